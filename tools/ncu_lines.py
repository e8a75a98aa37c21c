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
