"""Aggregate ncu source-page (cuda,sass) warp-stall samples per CUDA source line."""
import csv, sys
path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path)))
cur_file = None
tot = 0.0
lines = []
for r in rows:
    if not r:
        continue
    if r[0] == 'File Path':
        cur_file = r[1].split('/')[-1]
        continue
    if r[0] in ('Function Name', 'Line No'):
        continue
    if r[0] and r[0].isdigit() and len(r) > 4:
        try:
            v = float(r[4])
        except ValueError:
            continue
        tot += v
        lines.append((v, cur_file, int(r[0]), r[1].strip()[:100]))
lines.sort(reverse=True)
for v, f, l, s in lines[:top]:
    print(f"{100 * v / tot:5.1f}% {f}:{l}: {s}")


def reasons(path, top=25):
    """Per-line stall-reason breakdown (cuda,sass source page CSV)."""
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if r and r[0] == 'Line No')
    names = ['stall_barrier', 'stall_lg', 'stall_long_sb', 'stall_math', 'stall_mio', 'stall_short_sb', 'stall_wait',
             'stall_not_selected', 'stall_selected', 'stall_branch_resolving', 'stall_dispatch', 'stall_no_inst', 'stall_misc']
    idx = {n: hdr.index(n) for n in names}
    tot_cols = {n: 0.0 for n in names}
    cur = None
    lines = []
    for r in rows:
        if not r:
            continue
        if r[0] == 'File Path':
            cur = r[1].split('/')[-1]
            continue
        if r[0] and r[0].isdigit() and len(r) > 4:
            try:
                v = float(r[4])
            except ValueError:
                continue
            br = {n: float(r[idx[n]] or 0) for n in names}
            for n in names:
                tot_cols[n] += br[n]
            lines.append((v, cur, int(r[0]), br))
    lines.sort(key=lambda t: -t[0])
    T = sum(tot_cols.values())
    print('overall:', ', '.join(f"{n[6:]} {100 * v / T:.1f}%" for n, v in sorted(tot_cols.items(), key=lambda kv: -kv[1])[:8]))
    for v, f, l, br in lines[:top]:
        top3 = sorted(br.items(), key=lambda kv: -kv[1])[:3]
        print(f"{f}:{l} " + ", ".join(f"{n[6:]}={x:.0f}" for n, x in top3))


if __name__ == '__main__' and len(sys.argv) > 3:
    reasons(path, top)
