"""M2L work fill per config (diagnostics): algorithmic flops (2 k^2 per V pair) against the
flops the sibling-class / offset-major kernels execute (absent sibling children included).

    python tools/m2l_fill.py C2 C3 C4
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1211_2517_b200 as K  # noqa: E402
import synth_inputs  # noqa: E402

for name in sys.argv[1:] or ["C2"]:
    pts, q, cfg = synth_inputs.make(name)
    plan = K.Plan(torch.from_numpy(pts).cuda(), p=cfg["p"], k=cfg["k"], leaf_size=cfg["leaf"])
    i = plan.get_info()
    print(json.dumps(dict(config=name, nV=i["nV"], m2l_flops=i["m2l_flops"], m2l_exec_flops=i["m2l_exec_flops"],
                          fill=i["m2l_flops"] / i["m2l_exec_flops"])))
    del plan
    torch.cuda.empty_cache()
