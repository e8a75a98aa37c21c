"""Dev tool: FP64-pipe demand per CUDA source line from an ncu source page
(--page source --csv --print-source cuda,sass): DMMA counted as 8 DFMA-issue
equivalents (256 vs 32 FMAs), DFMA/DADD/DMUL/DSETP/DMNMX as 1."""
import csv, re, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
W = {"DMMA": 8, "DFMA": 1, "DADD": 1, "DMUL": 1, "DSETP": 1, "DMNMX": 1}
per = collections.Counter(); ops = collections.defaultdict(collections.Counter); src = {}
f = None; line = None; ie = None
for r in rows:
    if not r: continue
    if r[0] == "File Path": f = r[1].split("/")[-1]; continue
    if r[0] == "Line No": ie = r.index("Instructions Executed"); continue
    if r[0] == "Function Name": continue
    if r[0]:
        line = (f, int(r[0])); src[line] = r[1][:90]; continue
    if ie is None or len(r) <= ie or r[2] == "...": continue
    m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[3])
    if not m: continue
    op = m.group(2)
    if op in W:
        n = int(r[ie]); per[line] += W[op] * n; ops[line][op] += n
tot = sum(per.values())
print(f"FP64-pipe demand {tot:.3e} DFMA-issue equivalents")
for (fl, ln), v in per.most_common(top):
    print(f"{100*v/tot:5.1f}% {fl}:{ln} {dict(ops[(fl, ln)])}  | {src[(fl, ln)]}")
