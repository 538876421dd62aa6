import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1211_2517_b200 as K, synth_inputs
name = sys.argv[1] if len(sys.argv) > 1 else "C1"
pts, q, cfg = synth_inputs.make(name)
plan = K.Plan(torch.from_numpy(pts).cuda(), None, p=cfg["p"], k=cfg["k"], leaf_size=cfg["leaf"])
print(plan.get_info())
