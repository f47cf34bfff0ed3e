"""Per-kernel totals of an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr, data = rows[hi], rows[hi + 1:]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in data:
    name = r[ki].split("(")[0]
    sc = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}.get(r[ui], 1e-9)
    v = float(r[vi].replace(",", "")) * sc
    tot[name] += v
    cnt[name] += 1
T = sum(tot.values())
for k in sorted(tot, key=lambda k: -tot[k])[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"{k[:64]:64s} n={cnt[k]:6d} total={tot[k] * 1e3:9.3f} ms avg={tot[k] / cnt[k] * 1e6:8.1f} us share={tot[k] / T * 100:5.1f}%")
