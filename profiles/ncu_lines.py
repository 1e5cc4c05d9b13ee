"""Aggregate ncu warp-stall samples by CUDA source line (cuda,sass source view).

  ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > src.csv
  python profiles/ncu_lines.py src.csv [top]
"""
import collections
import csv
import sys


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cur = None
h = None
agg = collections.Counter()
src = {}
stall = collections.defaultdict(collections.Counter)
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if "Warp Stall Sampling (All Samples)" in r:
        h = r
        i_s = h.index("Warp Stall Sampling (All Samples)")
        sc = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
        continue
    if h is None or len(r) < len(h) or not r[0].isdigit():
        continue
    key = (cur, int(r[0]))
    if r[1].strip():
        src[key] = r[1].strip()
    agg[key] += num(r[i_s])
    for i in sc:
        stall[key][h[i][6:]] += num(r[i])
tot = sum(agg.values())
print("total samples", tot)
for key, v in agg.most_common(top):
    st = ", ".join(f"{n}={c:.0f}" for n, c in stall[key].most_common(2))
    print(f"{v:6.0f} {key[0]:18s}:{key[1]:4d} {src.get(key, '')[:72]:72s} {st}")
