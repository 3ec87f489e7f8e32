"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel count, total, share."""
import collections
import csv
import re
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        m = re.search(r"(\w+_kernel)(<[^(]*>)?", r[ki])
        name = (m.group(1) + (m.group(2) or "")) if m else r[ki][:40]
        v = float(r[vi].replace(",", ""))
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    print(f"{'kernel':44s} {'n':>6s} {'total_us':>10s} {'avg_us':>8s} {'share':>6s}")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{k:44s} {cnt[k]:6d} {v:10.1f} {v / cnt[k]:8.2f} {100 * v / T:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
