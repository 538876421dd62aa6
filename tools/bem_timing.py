"""BEM collocation matvec on a refined-octahedron sphere mesh (diagnostics / profiles).
    python tools/bem_timing.py [levels=9] [leaf=128] [p=8] [k=100]"""
import json
import math
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1211_2517_b200 as K  # noqa: E402
import synth_inputs  # noqa: E402

lv = int(sys.argv[1]) if len(sys.argv) > 1 else 9
s = int(sys.argv[2]) if len(sys.argv) > 2 else 128
p = int(sys.argv[3]) if len(sys.argv) > 3 else 8
k = int(sys.argv[4]) if len(sys.argv) > 4 else 100
tri, cen, q = synth_inputs.sphere_bem(lv)
N = cen.shape[0]
d = 0.5 / math.sqrt(s)
dev = torch.device("cuda:0")
C, Tt, Q = (torch.from_numpy(x).to(dev) for x in (cen, tri, q))
t0 = time.perf_counter()
pl = K.Plan(C, None, p=p, k=k, leaf_size=s, d=d, triangles=Tt)  # production plan (near SpMV overlapped)
torch.cuda.synchronize()
setup = time.perf_counter() - t0
pp = K.Plan(C, None, p=p, k=k, leaf_size=s, d=d, triangles=Tt, profile=True)  # profiled twin: phases
for _ in range(3):
    pp.matvec(Q)
torch.cuda.synchronize()
inf = pp.get_info()
del pp
torch.cuda.empty_cache()
for _ in range(3):
    pl.matvec(Q)
torch.cuda.synchronize()
ts = []
for _ in range(7):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = pl.matvec(Q)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ones = pl.matvec(torch.ones(N, dtype=torch.float64, device=dev)).cpu().numpy()
ms = sorted(ts)[3]
print(json.dumps(dict(workload=f"BEM sphere octa-{lv}", N=N, leaf=s, p=p, k=inf["k"], d=d, setup_s=setup, ms=ms,
                      ms_note="production plan (near-field SpMV beside the far field); phase_ms from a profiled twin",
                      elements_per_s=N / (ms * 1e-3), phase_ms=inf["phase_ms"],
                      near_gb=inf["bem_near_bytes"] / 1e9, leafop_gb=inf["leaf_op_bytes"] / 1e9,
                      near_hbm_tbs=inf["bem_near_bytes"] / (inf["phase_ms"]["eval"] * 1e-3) / 1e12,
                      extrusion=inf["bem_extrusion"], unit_density_potential_maxdev=float(np.abs(ones - 1).max()))))

# GMRES (tolerance 1e-6 as P:539) on the Dirichlet problem with the structured data
# f = cos(3 theta) + N(0, 0.1) of the C3 recipe: the paper's T_it = solve time / iterations
f = Q.clone()
pl.gmres(f, restart=50, maxit=20, tol=1e-6)  # warm-up (workspace allocation)
torch.cuda.synchronize()
walls = []
for _ in range(3):  # host-driven solve: wall clock; the best of three (host jitter)
    t0 = time.perf_counter()
    x, gi = pl.gmres(f, restart=50, maxit=500, tol=1e-6)
    walls.append(time.perf_counter() - t0)
wall = min(walls)
r = f - pl.matvec(x)
print(json.dumps(dict(workload=f"BEM GMRES sphere octa-{lv}", N=N, p=p, k=inf["k"], tol=1e-6, restart=50,
                      iters=gi["iters"], relres=gi["relres"],
                      true_relres=float(torch.linalg.norm(r) / torch.linalg.norm(f)), solve_s=wall,
                      T_it_ms=wall / max(1, gi["iters"]) * 1e3, matvec_ms=gi["t_matvec_ms"],
                      solve_s_all=walls)))
