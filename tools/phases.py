"""Dev tool: HQL phase cycle breakdown on a workload subset."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2205_11226_b200 as bm
from paper_2205_11226_b200 import _native
from paper_2205_11226_b200.profiles import conceal_batch
from paper_2205_11226_b200.synth import make_config
cfg = int(sys.argv[1]); nf = int(sys.argv[2]); prof = sys.argv[3]
kb = sys.argv[4] if len(sys.argv) > 4 else None
kb = None if kb is None else (int(kb) if kb.isdigit() else kb)
per_cta = 2 if kb == "cluster" else 1  # the cluster build's CTAs each count every phase
px, st = make_config(cfg, frames=nf)
p = bm.Profile.sentinel() if prof == 'sentinel' else bm.Profile.named(prof)
tp, ts = torch.from_numpy(px).cuda(), torch.from_numpy(st).cuda()
conceal_batch(tp, ts, p, kernel_build=kb)
_native.phase_cycles(reset=True)
r = conceal_batch(tp, ts, p, time_kernel=True, kernel_build=kb)
ph = {k: v // per_cta for k, v in _native.phase_cycles(reset=True).items()}
n_hql = r.summary['hql_patches']
tot = sum(v for k, v in ph.items() if not k.startswith('patch'))
print('kernel ms', _native.kernel_times_ms()[-1], 'hql patches', n_hql, r.summary['layer_counts'])
for k, v in ph.items():
    if k.startswith('patch'):
        print(f"{k:12s} total {v:.3e} cycles")
    else:
        print(f"{k:12s} {v / max(n_hql,1):10.0f} cycles/HQL patch  {100 * v / tot:5.1f}%")
kms = _native.kernel_times_ms()[-1]
busy = ph['patch_idl'] + ph['patch_hql']
grid = 2 * 148
print(f"IDL+HQL patch cycles {busy:.3e}; CTA capacity {grid * kms * 1e-3 * 1.965e9:.3e} -> utilisation {busy / (grid * kms * 1e-3 * 1.965e9):.2f}")
nidl = r.summary['layer_counts']['IDL']
for k in ('idl_pick', 'idl_gather', 'idl_estimate', 'idl_writeback'):
    print(f"{k:14s} {ph[k] / max(nidl, 1):9.0f} cycles/IDL patch")
cap = ph['cta_life']
print(f"CTA lifetime {cap:.3e} cycles over {ph['ctas']} CTAs (capacity {grid * kms * 1e-3 * 1.965e9:.3e})")
for k in ('patch_hql', 'patch_idl', 'patch_brl', 'dep_wait'):
    print(f"  {k:10s} {100 * ph[k] / cap:5.1f}% of CTA lifetime")
print(f"  other      {100 * (cap - ph['patch_hql'] - ph['patch_idl'] - ph['patch_brl'] - ph['dep_wait']) / cap:5.1f}%")
ns = max(ph['sidl_count'], 1)
print(f"small-m IDL patches (m < 64): {ph['sidl_count']}")
for k in ('sidl_setup', 'sidl_screen', 'sidl_ringsums', 'sidl_scan', 'sidl_dist_max', 'sidl_exp_sum', 'sidl_final'):
    print(f"  {k:14s} {ph[k] / ns:8.0f} cycles")
print(f"beta: loop(t0) {ph['beta_loop_t0'] / max(n_hql,1):.0f}  loop+reduce {ph['beta_loop_reduce'] / max(n_hql,1):.0f}  (phase total {ph['beta'] / max(n_hql,1):.0f})")
print(f"loo: loops(t0) {ph['loo_loops_t0'] / max(n_hql,1):.0f}  (phase total {ph['loo'] / max(n_hql,1):.0f})")
print("nearest (from HQL start): e2 %.0f sorted %.0f warp-merged %.0f all-merged %.0f final %.0f" % tuple(
    ph[k] / max(n_hql, 1) for k in ("e2_done", "nn_sorted", "nn_warp_merged", "nn_all_merged", "nearest")))
print(f"per-patch cycles: IDL {ph['patch_idl'] / max(nidl, 1):.0f}  HQL {ph['patch_hql'] / max(n_hql, 1):.0f}  BRL {ph['patch_brl'] / max(r.summary['layer_counts']['BRL'], 1):.0f}")
lt, nc, nb = ph.get('load_tile', 0), max(ph.get('load_tile_cells', 0), 1), ph.get('load_tile_nbufs', 0)
if ph.get('load_tile_cells', 0):
    byt = 2304 * 2 + 2048 * nb / nc  # u8 pixels + states of the 48x48 support, FP64 buffers of finished neighbours
    cyc = lt / nc
    print(f"staging (gather stage): {cyc:.0f} cycles/cell, {byt:.0f} B/cell ({nb / nc:.2f} neighbour buffers) "
          f"-> {byt / (cyc / 1.965e9) / 1e9:.1f} GB/s per CTA; {lt / ph['cta_life'] * 100:.1f}% of CTA time")
