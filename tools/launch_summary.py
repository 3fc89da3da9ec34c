"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list per kernel name."""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[h]; ki = hdr.index('Kernel Name'); vi = hdr.index('Metric Value')
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
tot = defaultdict(float); cnt = defaultdict(int)
for r in rows[h + 1:]:
    try:
        v = float(r[vi].replace(',', ''))
    except (ValueError, IndexError):
        continue
    k = r[ki].split('(')[0].replace('void ', '').replace('<unnamed>::', '')
    tot[k] += v; cnt[k] += 1
T = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v / 1e6 / div:9.4f} ms/step {100 * v / T:5.1f}% launches={cnt[k] / div:7.1f} {k}")
print(f"total {T / 1e6 / div:.3f} ms/step")
