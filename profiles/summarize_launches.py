"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel launch count, total and mean device time, share of the total.
Usage: python profiles/summarize_launches.py <launches.csv> [title]"""
import collections
import csv
import sys

UNIT = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def main(path, title=""):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui, gi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("Grid Size")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi or not r[vi]:
            continue
        ours = "pe::pe_" in r[ki]
        name = r[ki].split("(")[0] if ours else r[ki][:48]
        us = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)
        a = agg.setdefault(name, [0, 0.0, set()])
        a[0] += 1
        a[1] += us
        a[2].add(r[gi])
    tot = sum(a[1] for a in agg.values())
    ours = sum(a[1] for k, a in agg.items() if "pe::pe_" in k)
    print(f"# Launch list {title}\n\nsource: `{path}` (ncu gpu__time_duration.sum, --clock-control none; "
          "cold-cache serialised launches: compare shares, not absolutes)\n")
    print("| kernel | launches | total us | mean us | share of all | share of pe:: | grids |")
    print("|---|---|---|---|---|---|---|")
    for k, (n, t, g) in sorted(agg.items(), key=lambda x: -x[1][1]):
        sh = f"{100 * t / ours:.1f}%" if "pe::pe_" in k else "-"
        print(f"| `{k}` | {n} | {t:.1f} | {t / n:.1f} | {100 * t / tot:.1f}% | {sh} | {' '.join(sorted(g))[:60]} |")


if __name__ == "__main__":
    main(sys.argv[1], " ".join(sys.argv[2:]))
