"""One production-plan matvec of a config after warm-up (for ncu launch lists: the last
k_set_density launch starts the measured matvec).

    python tools/one_matvec.py C2 [--serial]   (--serial: a profiled plan, phases serialised)
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1211_2517_b200 as K  # noqa: E402
import synth_inputs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
pts, q, cfg = synth_inputs.make(name)
P, Q = torch.from_numpy(pts).cuda(), torch.from_numpy(q).cuda()
plan = K.Plan(P, Q, p=cfg["p"], k=cfg["k"], leaf_size=cfg["leaf"], profile="--serial" in sys.argv)
out = plan.matvec(Q)
for _ in range(3):
    plan.matvec(Q, out)
torch.cuda.synchronize()
