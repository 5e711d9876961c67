"""Summarise an ncu --csv launch list: per kernel (name+grid) count, time, DRAM bytes, GB/s."""
import csv, collections, sys
path = sys.argv[1]
first_embed_grid = sys.argv[2] if len(sys.argv) > 2 else None
rows = list(csv.reader(open(path)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == 'ID')
hdr = rows[hi]; ix = {h: i for i, h in enumerate(hdr)}
L = collections.OrderedDict()
for r in rows[hi + 1:]:
    d = L.setdefault(r[ix['ID']], {'name': r[ix['Kernel Name']], 'grid': r[ix['Grid Size']]})
    unit = r[ix['Metric Unit']]; v = float(r[ix['Metric Value']].replace(',', ''))
    scale = {'ns': 1e-3, 'nsecond': 1e-3, 'us': 1, 'usecond': 1, 'ms': 1e3, 'msecond': 1e3,
             'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}.get(unit, 1)
    d[r[ix['Metric Name']]] = v * scale
seq = list(L.values())
if first_embed_grid:
    emb = [j for j, d in enumerate(seq) if 'embed' in d['name'] and d['grid'] == first_embed_grid]
    start = emb[-1]
    nxt = [j for j, d in enumerate(seq) if 'embed' in d['name'] and j > start]
    seq = seq[start: nxt[0] if nxt else len(seq)]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for d in seq:
    key = d['name'].split('(')[0].replace('void ', '')[-42:] + ' ' + d['grid']
    a = agg[key]; a[0] += 1; a[1] += d.get('gpu__time_duration.sum', 0)
    a[2] += d.get('dram__bytes_read.sum', 0) + d.get('dram__bytes_write.sum', 0)
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':58s} {'n':>4s} {'total us':>10s} {'per us':>8s} {'%':>6s} {'GB/s':>8s} {'MB/launch':>9s}")
for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:58s} {n:4d} {t:10.1f} {t/n:8.2f} {100*t/tot:6.1f} {b/(t*1e-6)/1e9 if t else 0:8.0f} {b/n/1e6:9.2f}")
print(f"total {tot:.1f} us over {len(seq)} launches")
