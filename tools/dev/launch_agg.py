"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
frames = float(sys.argv[2]) if len(sys.argv) > 2 else 0
h, agg = None, collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if 'Kernel Name' in r:
        h = r
        continue
    if h and len(r) == len(h) and r[h.index('Metric Name')] == 'gpu__time_duration.sum':
        k = r[h.index('Kernel Name')].split('(')[0]
        agg[k][0] += 1
        agg[k][1] += float(r[h.index('Metric Value')].replace(',', ''))
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:12]:
    print(f"{k:40s} {v[0]:4d} {v[1] / 1e3:9.1f} us {100 * v[1] / tot:5.1f}%" + (f"  {v[1] / 1e3 / frames:.3f} us/frame" if frames else ""))
