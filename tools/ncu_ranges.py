"""Dev tool: stall reasons aggregated over source-line ranges (ncu source page CSV, cuda,sass)."""
import csv, sys
path = sys.argv[1]
ranges = {  # (file, lo, hi) -> name
    ('bm_hql.cuh', 183, 203): 'means', ('bm_hql.cuh', 205, 306): 'covariance', ('bm_hql.cuh', 307, 471): 'chol+nearest',
    ('bm_hql.cuh', 472, 546): 'quadforms', ('bm_hql.cuh', 547, 559): 'dmin', ('bm_hql.cuh', 560, 651): 'beta',
    ('bm_hql.cuh', 652, 680): 'staging', ('bm_hql.cuh', 681, 810): 'loo', ('bm_hql.cuh', 811, 870): 'alpha',
}
rows = list(csv.reader(open(path)))
hdr = next(r for r in rows if r and r[0] == 'Line No')
names = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
idx = {n: hdr.index(n) for n in names}
agg = {}
cur = None
for r in rows:
    if not r:
        continue
    if r[0] == 'File Path':
        cur = r[1].split('/')[-1]
        continue
    if r[0] and r[0].isdigit() and len(r) > 4:
        ln = int(r[0])
        key = 'other:' + (cur or '?')
        for (f, lo, hi), nm in ranges.items():
            if cur == f and lo <= ln <= hi:
                key = nm
        d = agg.setdefault(key, {n: 0.0 for n in names})
        for n in names:
            try:
                d[n] += float(r[idx[n]] or 0)
            except ValueError:
                pass
T = sum(sum(d.values()) for d in agg.values())
for k, d in sorted(agg.items(), key=lambda kv: -sum(kv[1].values())):
    s = sum(d.values())
    top = sorted(d.items(), key=lambda kv: -kv[1])[:5]
    print(f"{k:22s} {100 * s / T:5.1f}%  " + ", ".join(f"{n[6:]} {100 * v / s:.0f}%" for n, v in top))
