"""One CG iteration from an ncu launch list of a DFL_NO_GRAPH=1 solve
(tools/prof_kernels.py --solve): kernel names and durations between two
consecutive starts of the operator kernel."""
import csv
import re
import sys


def main(path, which=5):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h, d = rows[hi], rows[hi + 1:]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}
    seq = [(re.sub(r"\(.*", "", r[ki])[:70], float(r[vi].replace(",", "")) * scale[r[ui]]) for r in d if len(r) > vi]
    # iteration boundaries: the update kernel occurs once per CG iteration
    idx = [i for i, (n, _) in enumerate(seq) if "k_cg_update" in n]
    a, b = idx[which], idx[which + 1]
    tot = 0.0
    for n, v in seq[a - 2:b - 2]:
        print(f"{v:8.2f} {n}")
        tot += v
    print(f"iteration sum {tot:.1f} us ({len(idx)} iterations)")


if __name__ == "__main__":
    main(sys.argv[1])
