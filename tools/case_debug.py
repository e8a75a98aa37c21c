"""Dev tool: GPU vs golden record stream for one golden case, first mismatches in full."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, 'tests'))
import numpy as np, torch
import paper_2205_11226_b200 as bm
from paper_2205_11226_b200.profiles import conceal_batch
import parity
for nm in sys.argv[1:]:
    z = np.load(f'tests/golden/{nm}.npz')
    t_phi, t_nu, forced = float(z['t_phi']), float(z['t_nu']), int(z['forced'])
    layer = None if forced < 0 else ['BRL', 'IDL', 'HQL'][forced]
    r = conceal_batch(torch.from_numpy(z['pixels'].copy()).cuda(), torch.from_numpy(z['states'].copy()).cuda(),
                      bm.Profile('custom', t_phi, t_nu), forced_layer=layer, want_f64=True, records=True)
    g = r.records; ref = z['records']
    res = parity.compare(z['out'], ref, r.recon_f64.cpu().numpy()[0], g, z['states'], t_phi, t_nu)
    print(nm, res.summary())
    for p in res.problems[:4]: print('  P', p)
    for p in res.allowed[:4]: print('  A', p)
    np.savez(f'gpurun_out/dbg_{nm}.npz', out=r.recon_f64.cpu().numpy()[0], records=g)
