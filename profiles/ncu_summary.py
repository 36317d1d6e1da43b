"""Summarise an `ncu --set full` report (raw page CSV) into a markdown table of
the metrics the roofline discussion uses.  Usage:
  ncu -i <rep> --page raw --csv > raw.csv ; python profiles/ncu_summary.py raw.csv [title]"""
import csv
import sys

KEYS = [("gpu__time_duration.sum", "time"), ("sm__cycles_elapsed.avg.per_second", "SM clock"),
        ("dram__bytes_read.sum", "DRAM read"), ("dram__bytes_write.sum", "DRAM write"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
        ("lts__t_sector_hit_rate.pct", "L2 hit %"), ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %"),
        ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid"), ("launch__block_size", "block")]


def main(path, title=""):
    rows = list(csv.reader(open(path)))
    h, units, data = rows[0], rows[1], rows[2:]
    ki = h.index("Kernel Name")
    print(f"# ncu --set full summary {title}\n")
    print("| kernel | " + " | ".join(k[1] for k in KEYS) + " |")
    print("|---|" + "---|" * len(KEYS))
    for r in data:
        name = r[ki].split("(")[0].replace("void ", "")
        cells = []
        for k, _ in KEYS:
            i = h.index(k)
            cells.append(f"{r[i]} {units[i]}".strip())
        print(f"| `{name}` | " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main(sys.argv[1], " ".join(sys.argv[2:]))
