"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in data:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}.get(r[ui], 1.0)
        name = r[ki][:80]
        agg[name][0] += 1
        agg[name][1] += v
        tot += v
    print(f"{len(data)} launches, {tot / 1e3:.3f} ms total (serialised, cold-cache)")
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{t / tot * 100:6.2f}% {c:6d} x {t / c:9.2f} us  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
