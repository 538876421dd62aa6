"""M2L algorithmic vs executed flops and rate per config (profiled plan; with
KIFMM_DEBUG_M2L=1 the column counts per class kind are printed at setup).

    python tools/m2l_info.py C2 C3 C4 C5
"""
import sys, torch, json
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1211_2517_b200 as K, synth_inputs
for name in sys.argv[1:]:
    pts, q, cfg = synth_inputs.make(name)
    P = torch.from_numpy(pts).cuda()
    pl = K.Plan(P, None, p=cfg["p"], k=cfg["k"], leaf_size=cfg["leaf"], profile=True)
    Q = torch.from_numpy(q).cuda()
    for _ in range(3): pl.matvec(Q)
    torch.cuda.synchronize()
    i = pl.get_info()
    print(name, json.dumps(dict(alg=i["m2l_flops"], exe=i["m2l_exec_flops"], ratio=i["m2l_exec_flops"]/i["m2l_flops"], m2l_ms=i["phase_ms"]["m2l"], alg_tf=i["m2l_flops"]/i["phase_ms"]["m2l"]/1e9, exe_tf=i["m2l_exec_flops"]/i["phase_ms"]["m2l"]/1e9)), flush=True)
    pl.free()
