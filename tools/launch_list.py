"""Per-kernel times of the last step from an ncu --metrics gpu__time_duration.sum csv."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[hi]; K = hdr.index('Kernel Name'); V = hdr.index('Metric Value')
names = [(r[K], float(r[V])) for r in rows[hi + 1:] if r[hdr.index('Metric Name')] == 'gpu__time_duration.sum']
proj = [i for i, (n, v) in enumerate(names) if 'k_project' in n]
step = names[proj[-1]:]
tot = sum(v for _, v in step)
print("kernels in last step:", len(step), "sum us %.1f" % (tot / 1e3))
agg = {}
for n, v in step:
    key = n.split('(')[0].replace('void ', '').replace('<unnamed>::', '')
    agg[key] = agg.get(key, 0) + v
for k, v in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"{v/1e3:9.1f} us {100*v/tot:5.1f}%  {k}")
