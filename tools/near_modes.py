"""Near-field mode comparison on the GPU (diagnostics): fmm_options.near_mode 0 (one-sided),
2 (warp-pair symmetric) and 1 (mutual leaf pairs, the default).

    python tools/near_modes.py C2 [reps]
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1211_2517_b200 as K  # noqa: E402
import synth_inputs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
modes = sys.argv[3].split(",") if len(sys.argv) > 3 else ["0", "2", "1"]
pts, q, cfg = synth_inputs.make(name)
dev = torch.device("cuda:0")
P = torch.from_numpy(pts).to(dev)
Q = torch.from_numpy(q).to(dev)
res, outs = {}, {}
for mode in modes:
    plan = K.Plan(P, Q, p=cfg["p"], k=cfg["k"], leaf_size=cfg["leaf"], profile=True, near_mode=int(mode))
    out = plan.matvec(Q)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts, ev = [], []
    for _ in range(reps):
        e0.record()
        plan.matvec(Q, out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
        ev.append(plan.get_info()["phase_ms"]["eval"])
    info = plan.get_info()
    outs[mode] = out.clone()
    res[mode] = dict(ms=float(np.median(ts)), eval_ms=float(np.median(ev)),
                     mutual_leaves=int(info["near_mutual_leaves"]), mutual_pairs=int(info["near_mutual_pairs"]),
                     sym_pairs=int(info["near_sym_pairs"]))
    del plan
    torch.cuda.empty_cache()
ref = outs[modes[0]]
for m in modes[1:]:
    res[m]["rel_diff_vs_" + modes[0]] = float((outs[m] - ref).norm() / ref.norm())
print(json.dumps(dict(config=name, N=cfg["N"], modes=res)))
