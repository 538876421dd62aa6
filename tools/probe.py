"""Run a few matvecs of one config (diagnostics target for ncu; not the bench).

    python tools/probe.py C2 [reps]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1211_2517_b200 as K  # noqa: E402
import synth_inputs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
pts, q, cfg = synth_inputs.make(name)
dev = torch.device("cuda:0")
P = torch.from_numpy(pts).to(dev)
Q = torch.from_numpy(q).to(dev)
plan = K.Plan(P, Q, p=cfg["p"], k=cfg["k"], leaf_size=cfg["leaf"])
out = torch.empty_like(Q)
for _ in range(reps):
    plan.matvec(Q, out)
torch.cuda.synchronize()
print("ok", name, float(out.abs().sum()))
