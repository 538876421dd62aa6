"""One rank of a multi-process matvec over the NCCL shim (test helper for
tests/test_gpu_nccl_shim.py; run as a separate process per rank, all on cuda:0).

    python tests/shim_rank.py <workdir> <rank> <nranks> [overlap]

Reads workdir/case.npz (points, densities, operator tables, leaf size) and workdir/id.bin
(the shim's unique id), builds the rank's plan with the production NCCL transport
(KIFMM_NCCL_LIB points at the shim), and writes workdir/out_<rank>.npz: the REPLICATED
potential (caller order), the OWNED potentials of the rank's sorted range, and the range."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1211_2517_b200 as K  # noqa: E402

work, rank, nranks = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
overlap = int(sys.argv[4]) if len(sys.argv) > 4 else -1
d = np.load(os.path.join(work, "case.npz"))
uid = open(os.path.join(work, "id.bin"), "rb").read()
tb = {k[3:]: d[k] for k in d.files if k.startswith("tb_")}
for x in ("p", "n", "k"):
    tb[x] = int(tb[x])
tb["d"] = float(tb["d"])
dev = torch.device("cuda:0")
P = torch.from_numpy(d["pts"]).to(dev)
q = d["q"]
p, k, s = int(d["p"]), int(d["k"]), int(d["s"])
plan = K.Plan(P, None, p=p, k=k, leaf_size=s, tables=tb, nranks=nranks, rank=rank, nccl_id=uid, overlap=overlap)
assert plan.info["nranks"] == nranks
rep = plan.matvec(torch.from_numpy(q).to(dev)).cpu().numpy()   # REPLICATED: allgather inside
lo, hi = plan.owned_range
perm = plan.export_tree()["perm"]
own = plan.matvec_owned(torch.from_numpy(q[perm[lo:hi]].copy()).to(dev)).cpu().numpy()
# reuse, through the pipelined host-buffer batch (copy streams around the NCCL matvecs)
own2 = plan.matvec_owned_host_batch([q[perm[lo:hi]].copy()] * 2)[1]
np.savez(os.path.join(work, f"out_{rank}.npz"), rep=rep, own=own, own2=own2, lo=lo, hi=hi, perm=perm,
         overlap=plan.info["overlap"], ghost_q=plan.info["ghost_q_recv"], straddle=plan.info["n_straddle"])
plan.free()
