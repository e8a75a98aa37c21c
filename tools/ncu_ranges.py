"""Dev tool: stall reasons aggregated over source-line ranges (ncu source page CSV, cuda,sass)."""
import csv, sys
path = sys.argv[1]
ranges = {  # (file, lo, hi) -> name (line anchors of the round-1 final sources)
    ('bm_hql.cuh', 210, 246): 'hql:means', ('bm_hql.cuh', 247, 354): 'hql:covariance',
    ('bm_hql.cuh', 355, 526): 'hql:chol+nearest', ('bm_hql.cuh', 527, 599): 'hql:quadforms+dmin',
    ('bm_hql.cuh', 600, 704): 'hql:beta', ('bm_hql.cuh', 705, 739): 'hql:staging',
    ('bm_hql.cuh', 740, 866): 'hql:loo', ('bm_hql.cuh', 867, 925): 'hql:alpha',
    ('bm_conceal.cu', 294, 336): 'sched_pop', ('bm_conceal.cu', 337, 388): 'load_tile',
    ('bm_conceal.cu', 389, 471): 'gate:screen_chunk', ('bm_conceal.cu', 472, 629): 'gate:gather',
    ('bm_conceal.cu', 648, 822): 'estimate_patch', ('bm_conceal.cu', 823, 884): 'pick_and_extract',
    ('bm_conceal.cu', 885, 1035): 'k_conceal loop',
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
