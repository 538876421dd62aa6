"""Setup-time breakdown (diagnostics): plan setup of a BASELINE config with
KIFMM_DEBUG_SETUP=1 (per-section host times of build_schedules on stderr).

    python tools/setup_timing.py C4
"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("KIFMM_DEBUG_SETUP", "1")
import paper_1211_2517_b200 as K  # noqa: E402
import synth_inputs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
pts, q, cfg = synth_inputs.make(name)
P = torch.from_numpy(pts).cuda()
for rep in range(2):
    torch.cuda.synchronize()
    t = time.perf_counter()
    pl = K.Plan(P, None, p=cfg["p"], k=cfg["k"], leaf_size=cfg["leaf"])
    torch.cuda.synchronize()
    i = pl.get_info()
    print(f"{name} setup {time.perf_counter() - t:.2f} s: precompute {i['precompute_ms']:.0f} ms, tree {i['tree_ms']:.0f}, "
          f"lists {i['lists_ms']:.0f}, schedule {i['schedule_ms']:.0f} ms", file=sys.stderr, flush=True)
    pl.free()
