"""Per-rank work of a Morton partition, measured on ONE GPU with a loopback group
(diagnostics; the ranks run one after another, so the per-rank phase events measure each
rank's own kernels).  Default: the weak-scaling workload of bench.py (R tiled unit cubes
of C2); with a config name, that one problem partitioned R ways (strong scaling).
    python tools/dist_balance.py R [C4] [leaf_ops=0|1|-1]
(compute-only strong-scaling efficiency = single_rank_ms / (R max_ms): the NCCL transfers
of a real multi-GPU run are not in it)"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1211_2517_b200 as K  # noqa: E402
import synth_inputs  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("leaf_ops=")]
lops = int(([a[9:] for a in sys.argv[1:] if a.startswith("leaf_ops=")] or ["-1"])[0])
R = int(args[0]) if args else 2
name = args[1] if len(args) > 1 else None
pts, q, cfg = synth_inputs.make(name, seed=0) if name else synth_inputs.make("C2", scale=R)
dev = torch.device("cuda:0")
P = torch.from_numpy(pts).to(dev)
plans = [K.Plan(P, None, p=cfg["p"], k=cfg["k"], leaf_size=cfg["leaf"], nranks=R, rank=r, profile=True,
                leaf_ops=lops) for r in range(R)]
perm = plans[0].export_tree()["perm"]
dens = []
for pl in plans:
    lo, hi = pl.owned_range
    dens.append(torch.from_numpy(q[perm[lo:hi]].copy()).to(dev))
for _ in range(3):
    K.fmm_matvec_group(plans, dens, owned=True)
torch.cuda.synchronize()
per_rank = []
for _ in range(5):
    K.fmm_matvec_group(plans, dens, owned=True)
    torch.cuda.synchronize()
    # only the phases recorded inside a rank's own stage calls (density and exchange span the
    # other ranks' work in a loopback group)
    per_rank.append([sum(v for k, v in pl.get_info()["phase_ms"].items() if k not in ("density", "exchange"))
                     for pl in plans])
ms = np.median(np.array(per_rank), axis=0)
infos = [pl.get_info() for pl in plans]
single = None
if name:  # the same problem on one rank (profiled plan), for the strong-scaling comparison
    del plans
    torch.cuda.empty_cache()
    one = K.Plan(P, None, p=cfg["p"], k=cfg["k"], leaf_size=cfg["leaf"], profile=True, leaf_ops=lops)
    Qd = torch.from_numpy(q).to(dev)
    for _ in range(3):
        one.matvec(Qd)
    torch.cuda.synchronize()
    single = float(sum(v for k, v in one.get_info()["phase_ms"].items() if k not in ("density", "exchange")))
print(json.dumps(dict(config=name or f"C2 x {R} tiles", leaf_ops=lops, single_rank_ms=single, ranks=R, N=cfg["N"], per_rank_compute_ms=[round(float(x), 3) for x in ms],
                      max_ms=float(ms.max()), mean_ms=float(ms.mean()), imbalance=float(ms.max() / ms.mean()),
                      owned=[i["own_hi"] - i["own_lo"] for i in infos],
                      ghost_q_rows=[i["ghost_q_recv"] for i in infos], ghost_dens=[i["ghost_d_recv"] for i in infos],
                      straddling_boxes=infos[0]["n_straddle"],
                      leaf_op_GB=[round(i["leaf_op_bytes"] / 1e9, 2) for i in infos],
                      ghost_MB_per_rank=[round((i["ghost_q_recv"] * i["kp"] + i["ghost_d_recv"]) * 8 / 1e6, 2)
                                         for i in infos])))
