"""Write the DRAM traffic of the GEMM phases from an `ncu --set full` capture
into profiles/traffic.json (bench.py's `roofline.traffic`).

The three phases share one kernel instantiation, so the capture must list
them in a known order (e.g. `-k regex:pe_gemm --launch-skip S --launch-count 3`
over a middle iteration: Gram, Poly, Update).  Usage:
  ncu -i <rep> --page raw --csv > raw.csv
  python profiles/ncu_traffic.py raw.csv <workload> gram,poly,update [report-name]
Per launch: dram__bytes_read.sum + dram__bytes_write.sum (bytes); also records
the SM clock and tensor-pipe utilisation ncu saw for that launch."""
import csv
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def main(path, workload, labels, rep=None):
    rows = list(csv.reader(open(path)))
    h, units, data = rows[0], rows[1], rows[2:]
    ki = h.index("Kernel Name")
    data = [r for r in data if "pe_gemm" in r[ki]]
    labels = labels.split(",")
    assert len(data) >= len(labels), f"{len(data)} GEMM launches in {path}, {len(labels)} labels"

    def val(r, key):
        i = h.index(key)
        return float(r[i].replace(",", "")) * SCALE.get(units[i], 1.0)

    out_path = os.path.join(HERE, "traffic.json")
    tj = json.load(open(out_path)) if os.path.exists(out_path) else {}
    entry = {"_source": f"ncu --set full {rep or path}: dram__bytes_read.sum + dram__bytes_write.sum per launch "
                        f"({', '.join(labels)} in capture order), written by profiles/ncu_traffic.py"}
    for lab, r in zip(labels, data):
        entry[lab] = val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
        entry[f"{lab}_ncu"] = {
            "time_ms": val(r, "gpu__time_duration.sum") / 1e6 if units[h.index("gpu__time_duration.sum")] == "nsecond"
            else val(r, "gpu__time_duration.sum"),
            "sm_clock": r[h.index("sm__cycles_elapsed.avg.per_second")] + " " + units[h.index("sm__cycles_elapsed.avg.per_second")],
            "tensor_pipe_pct": r[h.index("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active")]
            if "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active" in h else None,
        }
    tj[workload] = entry
    json.dump(tj, open(out_path, "w"), indent=1)
    print(json.dumps(entry, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
