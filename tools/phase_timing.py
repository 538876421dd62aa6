"""Per-phase timing of one matvec config on the GPU (diagnostics, not the bench).

    python tools/phase_timing.py C2 [C4 ...] [reps] [ovl=4]  (profiled plans; near_ms = the k_near
    launches alone — in overlap mode 4 with the S2M / X streams they carry)
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1211_2517_b200 as K  # noqa: E402
import synth_inputs  # noqa: E402

ovl = int(([a[4:] for a in sys.argv[1:] if a.startswith("ovl=")] or [0])[0])
names = [a for a in sys.argv[1:] if not a.isdigit() and not a.startswith("ovl=")] or ["C2"]
reps = int(([a for a in sys.argv[1:] if a.isdigit()] or [5])[0])
for name in names:
    pts, q, cfg = synth_inputs.make(name)
    dev = torch.device("cuda:0")
    P = torch.from_numpy(pts).to(dev)
    Q = torch.from_numpy(q).to(dev)
    t0 = time.time()
    plan = K.Plan(P, Q, p=cfg["p"], k=cfg["k"], leaf_size=cfg["leaf"], profile=True, overlap=ovl)
    torch.cuda.synchronize()
    setup_s = time.time() - t0
    out = plan.matvec(Q)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts, phases, near = [], [], []
    for _ in range(reps):
        ev0.record()
        plan.matvec(Q, out)
        ev1.record()
        torch.cuda.synchronize()
        ts.append(ev0.elapsed_time(ev1))
        inf = plan.get_info()
        phases.append(inf["phase_ms"])
        near.append(inf["near_ms"])
    info = plan.get_info()
    ph = {k: float(np.median([p[k] for p in phases])) for k in phases[0]}
    print(json.dumps(dict(config=name, N=cfg["N"], setup_s=setup_s, ms=sorted(ts), phase_ms=ph,
                          near_ms=float(np.median(near)),
                          pts_per_s=cfg["N"] / (np.median(ts) * 1e-3),
                          info={k: info[k] for k in ("nboxes", "nleaves", "nlevels", "k", "kp", "nU", "nV", "nW", "nX",
                                                     "m2l_tiles", "precompute_ms", "tree_ms", "lists_ms", "schedule_ms")})))
    del plan, out
    torch.cuda.empty_cache()
