"""Print the kernels of the first target forward in an ncu launch-list CSV
(time, DRAM bytes, grid) and per-class sums."""
import csv, collections, sys
def load(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == 'ID')
    ix = {h: i for i, h in enumerate(rows[hi])}
    L = collections.OrderedDict()
    for r in rows[hi + 1:]:
        d = L.setdefault(r[ix['ID']], {'name': r[ix['Kernel Name']][:44], 'grid': r[ix['Grid Size']]})
        u = r[ix['Metric Unit']]; v = float(r[ix['Metric Value']].replace(',', ''))
        s = {'ns': 1e-3, 'nsecond': 1e-3, 'us': 1, 'usecond': 1, 'ms': 1e3, 'msecond': 1e3, 'byte': 1, 'Kbyte': 1e3,
             'Mbyte': 1e6, 'Gbyte': 1e9}.get(u, 1)
        d[r[ix['Metric Name']]] = v * s
    return list(L.values())
seq = load(sys.argv[1])
n = int(sys.argv[2]) if len(sys.argv) > 2 else 12
emb = [j for j, d in enumerate(seq) if 'embed' in d['name']]
for d in seq[emb[0]:emb[0] + n]:
    by = d.get('dram__bytes_read.sum', 0) + d.get('dram__bytes_write.sum', 0)
    t = d['gpu__time_duration.sum']
    print(f"  {d['name']:44s} {d['grid']:>14s} {t:8.1f}us {by / 1e6:8.1f}MB {by / t / 1e3:7.0f}GB/s")
