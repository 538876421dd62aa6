"""Small matvecs for compute-sanitizer: single plan (fused and split, leaf ops on/off,
symmetric near field on), a 3-rank loopback group, an adaptive sphere at p = 8.
    compute-sanitizer --tool memcheck python tools/sanitize_case.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1211_2517_b200 as K  # noqa: E402
import synth_inputs  # noqa: E402

dev = torch.device("cuda:0")
pts, q, cfg = synth_inputs.make("C1")
rng = np.random.default_rng(1)
g = rng.normal(size=(3000, 3))
sph = g / np.linalg.norm(g, axis=1, keepdims=True)
for P_, p, k, s in [(pts, 4, 24, 64), (sph, 8, 100, 16)]:
    Pt = torch.from_numpy(P_).to(dev)
    Q = torch.from_numpy(rng.uniform(-1, 1, P_.shape[0])).to(dev)
    for lo in (0, 1):
        for split in (False, True):
            pl = K.Plan(Pt, None, p=p, k=k, leaf_size=s, leaf_ops=lo, split_phases=split)
            out = pl.matvec(Q)
            torch.cuda.synchronize()
            pl.free()
    plans = [K.Plan(Pt, None, p=p, k=k, leaf_size=s, nranks=3, rank=r) for r in range(3)]
    K.fmm_matvec_group(plans, [Q] * 3, owned=False)
    torch.cuda.synchronize()
print("sanitize case done")
