"""Dev tool: the profiles/ summaries of one evidence run.

usage: ncu_summary.py <tag> <report.ncu-rep> <launches.csv> <commit>
writes profiles/ncu_<tag>_cfg5_k_conceal.txt (SOL, workload, scheduler, warp
state, launch, occupancy sections), profiles/ncu_<tag>_launches.txt (the
launch list with each kernel's share of the step) and
profiles/ncu_<tag>_cfg5_stalls_by_line.txt (warp-stall samples and shared-
memory bank-conflict excess per source line), and updates
profiles/ncu_traffic.json (dram bytes per k_conceal launch).
"""
import collections
import csv
import json
import os
import subprocess
import sys

tag, rep, launches, commit = sys.argv[1:5]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
prof = os.path.join(root, "profiles")


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


# sections
lines = ncu("--print-details", "all").split("\n")
keep = [("GPU Speed Of Light Throughput", 40), ("Compute Workload Analysis", 45), ("Memory Workload Analysis", 16),
        ("Scheduler Statistics", 34), ("Warp State Statistics", 34), ("Instruction Statistics", 20),
        ("Launch Statistics", 44), ("Occupancy", 40)]
out = lines[:3]
for name, cap in keep:
    for i, l in enumerate(lines):
        if l.strip() == f"Section: {name}":
            block = [l]
            j = i + 1
            while j < len(lines) and not lines[j].strip().startswith("Section:") and len(block) < cap:
                block.append(lines[j])
                j += 1
            out += block
            break
cmd = ("ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:_ZN2bm9k_conceal "
       "-s 3 -c 1 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e")
with open(os.path.join(prof, f"ncu_{tag}_cfg5_k_conceal.txt"), "w") as fh:
    fh.write(f"# {cmd}\n# commit {commit}; report {os.path.basename(rep)} (not committed)\n" + "\n".join(out) + "\n")

# launch list
rows = list(csv.reader(open(launches)))
i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[i]
ik, iv, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
agg = collections.defaultdict(list)
for r in rows[i + 1:]:
    if len(r) > iv and r[im] == "gpu__time_duration.sum":
        agg[r[ik]].append(float(r[iv].replace(",", "")))
tot = sum(sum(v) for v in agg.values())
lst = [f"# ncu launch list: python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e (cfg5, 256 x 1080p), commit {commit}",
       "# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised per launch)",
       "# launches        mean_ns   share  kernel"]
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    lst.append("%10d %14.0f %6.2f%%  %s" % (len(v), sum(v) / len(v), 100 * sum(v) / tot, k[:80]))
with open(os.path.join(prof, f"ncu_{tag}_launches.txt"), "w") as fh:
    fh.write("\n".join(lst) + "\n")

# stalls and bank conflicts per line
src = list(csv.reader(ncu("--page", "source", "--csv", "--print-source", "cuda,sass").splitlines()))
hdr = next(r for r in src if r and r[0] == "Line No")
iw = hdr.index("Warp Stall Sampling (All Samples)")
ix, iwf = hdr.index("L1 Wavefronts Shared Excessive"), hdr.index("L1 Wavefronts Shared")
names = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
idx = {n: hdr.index(n) for n in names}
cur, recs = None, []
for r in src:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0].isdigit() and len(r) > max(iw, ix):
        try:
            recs.append((float(r[iw] or 0), float(r[ix] or 0), float(r[iwf] or 0), cur, int(r[0]), r[1].strip()[:90],
                         {n: float(r[idx[n]] or 0) for n in names}))
        except ValueError:
            pass
ts = sum(x[0] for x in recs)
tx = sum(x[1] for x in recs)
tw = sum(x[2] for x in recs)
reason = collections.Counter()
for x in recs:
    reason.update(x[6])
rs = sum(reason.values())
txt = [f"# warp-stall samples per CUDA source line, bm::k_conceal, cfg5 (commit {commit}; tools/ncu_summary.py)",
       "overall: " + ", ".join(f"{n[6:]} {100 * v / rs:.1f}%" for n, v in reason.most_common(10))]
for x in sorted(recs, key=lambda x: -x[0])[:40]:
    top3 = sorted(x[6].items(), key=lambda kv: -kv[1])[:3]
    txt.append(f"{100 * x[0] / ts:5.1f}% {x[3]}:{x[4]}: {x[5]}   [" + ", ".join(f"{n[6:]} {int(v)}" for n, v in top3) + "]")
txt.append(f"\n# shared-memory wavefronts: {tw:.3g} total, {tx:.3g} ({100 * tx / max(tw, 1):.0f}%) excessive (bank conflicts); top lines by excess")
for x in sorted(recs, key=lambda x: -x[1])[:8]:
    txt.append(f"{100 * x[1] / max(tx, 1):5.1f}% of excess  {x[2]:.3g} wavefronts  {x[3]}:{x[4]} {x[5]}")
with open(os.path.join(prof, f"ncu_{tag}_cfg5_stalls_by_line.txt"), "w") as fh:
    fh.write("\n".join(txt) + "\n")

# traffic
raw = list(csv.reader(ncu("--page", "raw", "--csv").splitlines()))
h, u, v = raw[0], raw[1], raw[2]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
def get(name):
    k = h.index(name)
    return float(v[k].replace(",", "")) * scale[u[k]]
rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
tp = os.path.join(prof, "ncu_traffic.json")
d = json.load(open(tp)) if os.path.exists(tp) else {}
prev = d.get("cfg5", {})
d["cfg5"] = {"frames": 256, "kernel": "bm::k_conceal", "dram_bytes_per_launch": int(rd + wr), "dram_read": int(rd),
             "dram_write": int(wr), "source": f"{cmd} (profiles/ncu_{tag}_cfg5_k_conceal.txt, commit {commit})",
             "history": prev.get("history", []) + ([{"dram_bytes_per_launch": prev["dram_bytes_per_launch"],
                                                      "source": prev.get("source", "")}] if prev else [])}
json.dump(d, open(tp, "w"), indent=1)
print("ok", tag, int(rd + wr))
