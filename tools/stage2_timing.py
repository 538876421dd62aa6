"""Matvec and M2L timing with the stage-2 low-rank cores (diagnostics).
    python tools/stage2_timing.py C2 [C2coef ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1211_2517_b200 as K  # noqa: E402
import synth_inputs  # noqa: E402

name = sys.argv[1]
coefs = [float(x) for x in sys.argv[2:]] or [0.0, 1.0, 10.0]
p, q, c = synth_inputs.make(name)
P = torch.from_numpy(p).cuda()
Q = torch.from_numpy(q).cuda()
for c2 in coefs:
    pl = K.Plan(P, Q, p=c["p"], k=c["k"], leaf_size=c["leaf"], m2l_c2=c2, profile=True)
    for _ in range(3):
        pl.matvec(Q)
    torch.cuda.synchronize()
    ts, m2l = [], []
    for _ in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pl.matvec(Q)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
        m2l.append(pl.get_info()["phase_ms"]["m2l"])
    inf = pl.get_info()
    ms, mm = sorted(ts)[3], sorted(m2l)[3]
    print(f"{name} C2={c2:g}: matvec {ms:.3f} ms, m2l {mm:.3f} ms, rank mean {inf['m2l_rank_mean']:.1f}, "
          f"M2L {inf['m2l_flops'] / mm / 1e9:.1f} TF/s algorithmic", flush=True)
    pl.free()
