"""A few stage-2 matvecs (ncu target).  python tools/probe_stage2.py C2 1.0"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1211_2517_b200 as K  # noqa: E402
import synth_inputs  # noqa: E402

p, q, c = synth_inputs.make(sys.argv[1])
P, Q = torch.from_numpy(p).cuda(), torch.from_numpy(q).cuda()
pl = K.Plan(P, Q, p=c["p"], k=c["k"], leaf_size=c["leaf"], m2l_c2=float(sys.argv[2]))
for _ in range(2):
    pl.matvec(Q)
torch.cuda.synchronize()
print("ok")
