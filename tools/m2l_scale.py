"""M2L phase time vs the sibling / offset-major cost-model RED weight (diagnostics).

    KIFMM_M2L_RED_SCALE=0.5 python tools/m2l_scale.py C4
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1211_2517_b200 as K  # noqa: E402
import synth_inputs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
pts, q, cfg = synth_inputs.make(name)
P = torch.from_numpy(pts).cuda()
Q = torch.from_numpy(q).cuda()
plan = K.Plan(P, Q, p=cfg["p"], k=cfg["k"], leaf_size=cfg["leaf"], profile=True)
out = plan.matvec(Q)
ms, m2l = [], []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); plan.matvec(Q, out); e1.record(); torch.cuda.synchronize()
    ms.append(e0.elapsed_time(e1)); m2l.append(plan.get_info()["phase_ms"]["m2l"])
i = plan.get_info()
print(json.dumps(dict(config=name, scale=os.environ.get("KIFMM_M2L_RED_SCALE", "1"), ms=float(np.median(ms)),
                      m2l_ms=float(np.median(m2l)), fill=i["m2l_flops"] / i["m2l_exec_flops"],
                      tf_alg=i["m2l_flops"] / np.median(m2l) / 1e9)))
