"""Per-kernel summary of an ncu launch list (--metrics gpu__time_duration.sum --csv):
launches, mean duration and share of the listed device time (developer tool).
usage: python scripts/launch_summary.py launches.csv [--only-mux]"""
import collections
import csv
import re
import sys


def main(path, only_mux):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            name = r[ki]
            if only_mux and "mux::" not in name:
                continue
            base = re.sub(r"[<(].*$", "", name.replace("void ", "").replace("(anonymous namespace)::", "").replace("<unnamed>::", ""))
            agg[base.split("::")[-1]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    print(f"| kernel | launches | mean us | share |\n|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"| {k} | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {100 * sum(v) / tot:.1f} % |")


if __name__ == "__main__":
    main(sys.argv[1], "--only-mux" in sys.argv)
