"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of
tools/ncu_target.py: per-kernel totals of the LAST build in the capture."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hi]
ik, iv, im = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
recs = [(r[ik], float(r[iv].replace(",", ""))) for r in rows[hi + 1:] if len(r) == len(h) and r[im] == "gpu__time_duration.sum"]
unit = next(r[h.index("Metric Unit")] for r in rows[hi + 1:] if len(r) == len(h))
# builds start with the first leaf kernel (small_elim) after a non-small kernel
starts = [i for i, (k, _) in enumerate(recs) if "small_elim" in k and (i == 0 or "small_elim" not in recs[i - 1][0])]
last = recs[starts[-1]:] if starts else recs
agg = defaultdict(lambda: [0, 0.0])
for k, t in last:
    name = k.split("(")[0].replace("void ", "").replace("dtnb::", "")
    name = name.split("<")[0]
    agg[name][0] += 1
    agg[name][1] += t
tot = sum(v[1] for v in agg.values())
print(f"| kernel | launches | sum of launch times ({unit}) | share |")
print("|---|---|---|---|")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"| {k} | {n} | {t:.1f} | {t / tot:.3f} |")
print(f"| total | {sum(v[0] for v in agg.values())} | {tot:.1f} | 1.000 |")
