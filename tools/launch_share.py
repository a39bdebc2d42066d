"""Per-kernel share of an ncu launch list (--metrics gpu__time_duration.sum --csv)."""
import collections
import csv
import sys

SCALE = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}


def shares(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        tot[name] += float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
        cnt[name] += 1
    return tot, cnt


if __name__ == "__main__":
    tot, cnt = shares(sys.argv[1])
    s = sum(tot.values())
    print(f"{'kernel':60s} {'launches':>8s} {'ms':>10s} {'share':>6s}")
    for k in sorted(tot, key=tot.get, reverse=True)[:12]:
        print(f"{k[:60]:60s} {cnt[k]:8d} {tot[k]:10.3f} {100 * tot[k] / s:5.1f}%")
