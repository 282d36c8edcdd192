# Top stalled SASS instructions of an `ncu --page source --csv --print-source sass` export.
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; idx = hdr.index('Warp Stall Sampling (All Samples)'); ex = hdr.index('Instructions Executed')
cols = [c for c in hdr if c.startswith('stall_') and 'Not Issued' not in c]
ci = [hdr.index(c) for c in cols]
data = []
for k, r in enumerate(rows[2:]):
    try: v = float(r[idx])
    except: continue
    st = sorted(((float(r[i]), c[6:]) for i, c in zip(ci, cols)), reverse=True)[:2]
    data.append((v, k, r[1].strip()[:64], r[ex], st))
tot = sum(d[0] for d in data)
print('total samples', tot)
for v, k, src, e, st in sorted(data, reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{100*v/tot:5.1f}% #{k:5d} ex={e:>9} {src:64s} {st[0][1]}:{st[0][0]:.0f} {st[1][1]}:{st[1][0]:.0f}")
