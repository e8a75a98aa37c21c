"""Dump GPU outputs/records for golden cases (dev tool)."""
import sys, os, glob
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2205_11226_b200 as bm
from paper_2205_11226_b200.profiles import conceal_batch
names = sys.argv[1:]
for nm in names:
    z = np.load(f'tests/golden/{nm}.npz')
    t_phi, t_nu, forced = float(z['t_phi']), float(z['t_nu']), int(z['forced'])
    layer = None if forced < 0 else {0: 'BRL', 1: 'IDL', 2: 'HQL'}[forced]
    px = torch.from_numpy(z['pixels'].copy()).cuda()
    st = torch.from_numpy(z['states'].copy()).cuda()
    r = conceal_batch(px, st, bm.Profile('custom', t_phi, t_nu), forced_layer=layer, want_f64=True, records=True)
    np.savez(f'gpurun_out/dump_{nm}.npz', out=r.recon_f64.cpu().numpy()[0], records=r.records)
    print(nm, r.summary)
