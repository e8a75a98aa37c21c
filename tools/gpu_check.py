"""Quick GPU parity sweep over tests/golden (dev tool)."""
import glob, sys, time, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2205_11226_b200 as bm
from oracle import oracle
import parity

for f in sorted(glob.glob('tests/golden/*.npz')):
    z = np.load(f)
    t_phi, t_nu, forced = float(z['t_phi']), float(z['t_nu']), int(z['forced'])
    prof = bm.Profile('custom', t_phi, t_nu) if t_nu > 0 else None
    layer = None if forced < 0 else {0: 'BRL', 1: 'IDL', 2: 'HQL'}[forced]
    t0 = time.time()
    out, rep = bm.conceal_image(bm.ImageBuffer(z['pixels']), bm.LossMask(z['states']), prof, forced_layer=layer)
    dt = time.time() - t0
    from paper_2205_11226_b200.records import RECORD_DTYPE
    # rebuild record array from decisions for parity
    recs = np.zeros(len(rep.decisions), dtype=RECORD_DTYPE)
    for i, d in enumerate(rep.decisions):
        r = recs[i]
        r['row'], r['col'] = d.patch_origin
        r['layer'] = -1 if d.layer is None else {'BRL': 0, 'IDL': 1, 'HQL': 2}[d.layer.value]
        r['flags'] = (1 if d.fallback else 0) | (2 if d.deferred_fill else 0)
        r['rings_used'] = d.rings_used
        r['m_candidates'] = -1 if d.m_candidates is None else d.m_candidates
        r['n_y'] = d.n_y
        r['phi'] = np.nan if d.phi is None else d.phi
        r['nu'] = np.nan if d.nu is None else d.nu
        r['beta'] = np.nan if d.beta is None else d.beta
        r['alpha'] = np.nan if d.alpha is None else d.alpha
        r['beta_gap'] = np.nan if d.beta_gap is None else d.beta_gap
    g = z['records']
    res_g = parity.compare(z['out'], g, out.pixels, recs, z['states'], t_phi, t_nu)
    o_out, o_recs, _, _ = oracle.conceal(z['pixels'], z['states'], t_phi, t_nu, 10.0, forced)
    res_o = parity.compare(o_out, o_recs, out.pixels, recs, z['states'], t_phi, t_nu)
    print(f"{os.path.basename(f):42s} {dt*1e3:7.1f}ms vs-golden: {res_g.summary()}")
    print(f"{'':42s}           vs-oracle: {res_o.summary()}")
    for p in (res_g.problems[:3] + res_o.problems[:3]):
        print("     PROBLEM", p)
    for p in (res_g.allowed[:2] + res_o.allowed[:2]):
        print("     allowed", p)
