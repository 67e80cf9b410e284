"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) by kernel."""
import collections
import csv
import sys


def summarise(path, per=1):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[h + 1:]:
        name = r[ki].split("(")[0].replace("<unnamed>::", "")[:70]
        tot[name] += float(r[vi].replace(",", "")) / 1e6
        cnt[name] += 1
    s = sum(tot.values())
    out = []
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        out.append(f"{v / per:10.3f} ms {100 * v / s:5.1f}% {cnt[k] / per:7.1f}  {k}")
    out.append(f"total {s / per:.3f} ms per unit ({per} units), launches {sum(cnt.values())}")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 1))
