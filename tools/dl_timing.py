"""Single- vs double-layer matvec timing on a config (diagnostics): production plans
(default overlap), and the phases of a profiled twin.
    python tools/dl_timing.py C3"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1211_2517_b200 as K  # noqa: E402
import synth_inputs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
p, q, c = synth_inputs.make(name)
nrm = p / np.linalg.norm(p, axis=1, keepdims=True) if c["kind"] == "sphere_octa" else \
    np.random.default_rng(1).normal(size=p.shape)
nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
P, Q, Nt = (torch.from_numpy(x).cuda() for x in (p, q, nrm))
for layer, normals in (("single", None), ("double", Nt)):
    pl = K.Plan(P, Q, p=c["p"], k=c["k"], leaf_size=c["leaf"], normals=normals)
    for _ in range(3):
        pl.matvec(Q)
    torch.cuda.synchronize()
    ts = []
    for _ in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pl.matvec(Q)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    pl.free()
    pp = K.Plan(P, Q, p=c["p"], k=c["k"], leaf_size=c["leaf"], normals=normals, profile=True)
    for _ in range(3):
        pp.matvec(Q)
    torch.cuda.synchronize()
    ph = pp.get_info()["phase_ms"]
    pp.free()
    print(f"{name} {layer}: {sorted(ts)[3]:.3f} ms  ({c['N'] / sorted(ts)[3] / 1e-3:.3e} pts/s)  phases (serialised): "
          + " ".join(f"{k}={v:.3f}" for k, v in ph.items()), flush=True)
