"""Production-plan matvec time per config (no per-phase events, so the default overlap
of the near field with the far field is on).

    python tools/config_timing.py C3 C4 C5 [ovl=0 ovl=3 ovl=4]   (fmm_options.overlap; default -1)
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1211_2517_b200 as K  # noqa: E402
import synth_inputs  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("ovl=")]
ovl = [int(a[4:]) for a in sys.argv[1:] if a.startswith("ovl=")] or [-1]
for name, mode in [(n, m) for n in (args or ["C2"]) for m in ovl]:
    pts, q, cfg = synth_inputs.make(name)
    P, Q = torch.from_numpy(pts).cuda(), torch.from_numpy(q).cuda()
    plan = K.Plan(P, Q, p=cfg["p"], k=cfg["k"], leaf_size=cfg["leaf"], overlap=mode)
    out = plan.matvec(Q)
    for _ in range(2):
        plan.matvec(Q, out)
    torch.cuda.synchronize()
    ts = []
    for _ in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); plan.matvec(Q, out); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(json.dumps(dict(config=name, N=cfg["N"], ms_median=float(np.median(ts)), ms_min=float(np.min(ts)),
                          pts_per_s=cfg["N"] / (np.median(ts) * 1e-3), overlap=mode)))
    del plan, out
    torch.cuda.empty_cache()
