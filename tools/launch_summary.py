"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel total device
time, share, launch count and mean duration (cold-cache, serialised: compare SHARES)."""
import collections
import csv
import sys


def summarise(path, top=20):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        v = float(r[vi].replace(",", "")) * {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0,
                                             "second": 1e3}.get(r[ui], 1e-6)
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    lines = [f"{'ms':>9} {'share':>6} {'launches':>8} {'mean_us':>9}  kernel"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:top]:
        lines.append(f"{v:9.2f} {100 * v / T:5.1f}% {cnt[k]:8d} {1e3 * v / cnt[k]:9.1f}  {k[:100]}")
    lines.append(f"total {T:.2f} ms over {sum(cnt.values())} launches")
    return "\n".join(lines)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(p)
        print(summarise(p))
