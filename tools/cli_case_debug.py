"""Dev tool: the CLI golden random run's frames (img_a, img_b, one batch as the
harness runs them) through conceal_batch per kernel build and forced layer,
against the oracle at the decision level (tests/parity.py)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np, torch
import parity
from oracle import oracle
from paper_2205_11226_b200 import Layer, Profile, conceal_batch, loss
from paper_2205_11226_b200.image import BlockGrid, ImageBuffer, apply_mask
from paper_2205_11226_b200.netpbm import read_pgm_bytes

G = os.path.join(ROOT, "tests", "golden", "aux", "cli")
px, st = [], []
for nm in ("img_a", "img_b"):
    img = read_pgm_bytes(open(os.path.join(G, nm + ".pgm"), "rb").read())
    H, W = img.shape
    m = loss.gen_random_mask(BlockGrid(W, H), 0.3, 5)
    px.append(apply_mask(ImageBuffer(img.astype(np.float64)), m).pixels.astype(np.float64))
    st.append(np.asarray(m.states))
codes = {None: -1, Layer.BRL: 0, Layer.IDL: 1, Layer.HQL: 2}
for fi in range(2):
  pxs, sts = np.ascontiguousarray(px[fi][None]), np.ascontiguousarray(st[fi][None])
  for forced in (Layer.HQL, None):
    prof = Profile.named("efficient")
    t_phi, t_nu = (prof.t_phi, prof.t_nu)
    o_out, o_rec, _, _ = oracle.conceal(pxs[0], sts[0], t_phi, t_nu, 10.0, codes[forced])
    for build in (None, 256, 512, "cluster"):
        res = conceal_batch(torch.from_numpy(pxs).cuda(), torch.from_numpy(sts).cuda(), prof, forced_layer=forced,
                            want_f64=True, records=True, kernel_build=build)
        pr = parity.compare(o_out, o_rec, res.recon_f64.cpu().numpy()[0], res.records, sts[0], t_phi, t_nu)
        print(fi, forced, build, res.summary.get("kernel_build"), pr.summary())
        for p in pr.problems[:4]: print("   problem", p)
        for p in pr.beta_ties[:4]: print("   tie", p)
