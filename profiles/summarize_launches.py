import csv, sys
from collections import defaultdict
rows = list(csv.DictReader(l for l in open(sys.argv[1]) if not l.startswith('==')))
d = defaultdict(list)
for r in rows:
    d[(r['Kernel Name'][:40], r.get('Grid Size',''), r.get('Block Size',''))].append(float(r['Metric Value']))
tot = sum(sum(v)/len(v) for v in d.values())
for k, v in d.items():
    a = sum(v)/len(v)/1000
    print(f"{k[0]:42s} grid {k[1]:14s} n={len(v):3d} avg {a:7.2f} us  share {100*a*1000/tot:5.1f}%")
