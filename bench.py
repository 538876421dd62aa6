"""Benchmark: one FP64 KIFMM matvec per step (BASELINE.json metric: FMM matvec
points/sec (FP64) and the roofline fraction of the dominant kernel).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl ours|reference] [--weak]

Workload (default C4 = BASELINE.json configs[3], the config BASELINE runs at 1/2/4/8 GPUs):
N = 2^24 points on the torus R = 1, r = 0.3 (area-weighted, seed 0), densities U[-1,1],
p = 6 (n = 152), k = 60 (k_eff 61), leaf 128, adaptive octree.  C2 (configs[1]), C3 and
C5 (configs[4]: 2^26 points, the 8-GPU scale-out case, `--gpus 8 --config C5`) run with
--config.  A step is one whole fmm_matvec (permute, S2M, M2M, M2L, X, L2L, L2T, W, P2P,
unpermute) with the inputs resident in HBM; L2 is flushed (a 256 MiB write) between timed
steps, outside the timed events.  Multi-GPU (torchrun, N ranks): strong scaling, the SAME
problem partitioned over the ranks by Morton ranges (OWNED mode: each rank's owned
densities in, owned potentials out), ghost multipoles / densities exchanged over NCCL
inside every step; `value` = N / max-over-ranks step time.  `--weak` instead tiles N unit
cubes of the config (cube configs only).  `--impl reference` times the CPU oracle
(oracle/) on the host on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth_inputs  # noqa: E402


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C4")
    ap.add_argument("--weak", action="store_true", help="N > 1: tile N copies (cube configs) instead of strong scaling")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


METRIC = "FMM matvec points/sec (FP64)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 20 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)  # first sample lands before the timed loop starts
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is None:
            return
        time.sleep(0.05)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        self.rows = [[x.strip() for x in ln.split(",")] for ln in out.strip().splitlines() if ln.count(",") >= 5]

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 2 + i and r[2 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def oracle_sample(name: str, pts, q):
    """A bounded sample of the workload for the CPU oracle (the oracle runs at ~1e6
    points/s on a host, so the full C4 / C5 would take minutes per matvec): a contiguous
    piece of the same surface or volume with the workload's point density, so leaves,
    lists and the near/far work mix per point are those of the full problem.
      C1, C2, C3   the whole workload (seconds)
      C4           the torus sector 0 <= atan2(y, x) < 2 pi / 16 (1/16 of the points)
      C5           the points of the first of the 64 spheres (2^20 points)
    Returns (points, densities, description)."""
    if name == "C4":
        sel = np.arctan2(pts[:, 1], pts[:, 0])
        sel = (sel >= 0) & (sel < 2 * np.pi / 16)
        return np.ascontiguousarray(pts[sel]), np.ascontiguousarray(q[sel]), "torus sector 0 <= u < 2pi/16 of C4"
    if name == "C5":
        per = pts.shape[0] // 64
        return np.ascontiguousarray(pts[:per]), np.ascontiguousarray(q[:per]), "sphere 0 of C5's 64 spheres"
    return pts, q, f"the whole {name} workload"


def oracle_matvec_timer(pts, q, cfg, reps: int = 1):
    """Time the oracle (as it stands) on the host cores: one full matvec of (pts, q) per rep."""
    import oracle
    tb = oracle.precompute.build_tables(cfg["p"], cfg["k"])
    plan = oracle.Plan(pts, cfg["leaf"], tb["n"])
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        plan.matvec(tb, q)
        ts.append(time.perf_counter() - t0)
    return ts


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    pts, q, cfg = synth_inputs.make(args.config)
    sp, sq, what = oracle_sample(args.config, pts, q)
    ns = sp.shape[0]
    import oracle
    k_eff = int(oracle.precompute.build_tables(cfg["p"], cfg["k"])["k"])
    # warm-up and timed steps: each step one oracle matvec of the sample
    ts = oracle_matvec_timer(sp, sq, cfg, reps=args.warmup + args.steps)[args.warmup:]
    sec = float(np.mean(ts))
    value = ns / sec
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "strong" if not args.weak else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, cfg, 1, k_eff),
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": cpu_cores(), "kind": "oracle",
                         "sample": f"{what}: {ns} points, one oracle matvec per step (oracle/ C++ -O2 OpenMP)"},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(args, cfg, ws: int, k_eff: int) -> dict:
    """The workload a line measures (the same dict in both arms): no implementation details."""
    wl = args.config if ws == 1 or not args.weak else f"{args.config} x{ws} (weak: {ws} tiled copies)"
    return {"workload": wl, "N": cfg["N"], "N_per_gpu": cfg["N"] // ws, "p": cfg["p"], "k": cfg["k"], "k_eff": k_eff,
            "leaf_size": cfg["leaf"], "kind": cfg["kind"],
            "parallelism": "single" if ws == 1 else f"morton-partition{ws} (NCCL ghosts)"}


def ncu_evidence(config: str):
    """Per-config ncu numbers of the timed kernels (profiles/ncu_<config>.json: written from
    an `ncu --set full` capture of this config's bench command), or None."""
    f = os.path.join(ROOT, "profiles", f"ncu_{config}.json")
    return json.load(open(f)) if os.path.exists(f) else None


def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_1211_2517_b200 as K

    ws, rank, local = dist_env()
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # N = 1: the BASELINE workload itself.  N > 1: strong scaling, the same problem
    # partitioned over the ranks (every rank draws the same seeded cloud); --weak: N x the
    # points of the workload (tiled unit cubes for the cube configs)
    pts, q, cfg = synth_inputs.make(args.config, scale=ws if args.weak else 1)
    N = cfg["N"]
    stream = torch.cuda.current_stream()
    P = torch.from_numpy(pts).to(dev)
    Q = torch.from_numpy(q).to(dev)
    def new_nccl_id():  # one communicator per plan: rank 0's unique id, broadcast
        if ws == 1:
            return None
        box = [K.fmm_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        return box[0]

    nccl_id = new_nccl_id()
    t0 = time.perf_counter()
    # the production plan (timed steps, e2e): the mutual near field overlaps the far field
    # on a second stream, so per-phase events would not attribute time cleanly
    plan = K.Plan(P, Q, p=cfg["p"], k=cfg["k"], leaf_size=cfg["leaf"], nranks=ws, rank=rank, nccl_id=nccl_id)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    # a profiled twin of the same workload (phases serialised, per-phase CUDA events on the
    # launching stream): the per-phase breakdown and the M2L roofline
    pplan = K.Plan(P, Q, p=cfg["p"], k=cfg["k"], leaf_size=cfg["leaf"], profile=True, nranks=ws, rank=rank,
                   nccl_id=new_nccl_id())
    lo, hi = plan.owned_range
    if ws > 1:  # OWNED mode: densities / potentials of the owned points, sorted order
        perm = plan.export_tree()["perm"]
        Qin = torch.from_numpy(q[perm[lo:hi]].copy()).to(dev)
        out = torch.empty(hi - lo, dtype=torch.float64, device=dev)
        step = lambda: plan.matvec_owned(Qin, out)
        pstep = lambda: pplan.matvec_owned(Qin, out)
    else:
        Qin = Q
        out = torch.empty(N, dtype=torch.float64, device=dev)
        step = lambda: plan.matvec(Qin, out)
        pstep = lambda: pplan.matvec(Qin, out)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for _ in range(max(3, args.warmup)):
        step()
        pstep()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    phase_tot, launches = {}, 0
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(i & 0xFF)  # L2 flush outside the timed events
            evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
        torch.cuda.synchronize()
        launches = plan.get_info()["launches"] * args.steps
    if ws > 1:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    ms = float(np.sum(step_ms)) / args.steps
    if ws > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    # profiled pass: same steps, L2 flushed, phase events read per step
    for i in range(args.steps):
        flush.fill_(i & 0xFF)
        pstep()
        inf = pplan.get_info()  # waits for this step's phase events
        for kname, v in inf["phase_ms"].items():
            phase_tot[kname] = phase_tot.get(kname, 0.0) + v
    torch.cuda.synchronize()
    phase = {k: v / args.steps for k, v in phase_tot.items()}
    info = pplan.get_info()
    del pplan
    # ---- end to end through the C-ABI with host buffers (pinned), H2D + D2H inside the timing
    # (the batched call pipelines the steps: step i + 1's density is copied in and step
    # i - 1's potential copied out while step i computes; every step still copies its input
    # from and its result to pinned host memory inside the timed region)
    e2e_steps = max(5, args.steps // 2)
    if ws > 1:
        hq = torch.from_numpy(q[perm[lo:hi]].copy()).pin_memory()
        hp = [torch.empty(hi - lo, dtype=torch.float64).pin_memory() for _ in range(2)]
        e2e_call = lambda k: plan.matvec_owned_host_batch([hq.numpy()] * k, [hp[i & 1].numpy() for i in range(k)])
        e2e_bytes = 8 * (hi - lo)
        e2e_api = "fmm_matvec_owned_host_batch (pinned host buffers, owned points; copies overlapped with compute)"
    else:
        hq = torch.from_numpy(q).pin_memory()
        hp = [torch.empty(N, dtype=torch.float64).pin_memory() for _ in range(2)]
        e2e_call = lambda k: plan.matvec_host_batch([hq.numpy()] * k, [hp[i & 1].numpy() for i in range(k)])
        e2e_bytes = 8 * N
        e2e_api = "fmm_matvec_host_batch (pinned host buffers; copies overlapped with compute)"
    e2e_call(3)
    if ws > 1:
        dist.barrier()
    te = time.perf_counter()
    e2e_call(e2e_steps)
    e2e_s = (time.perf_counter() - te) / e2e_steps
    if ws > 1:
        t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
        tl = torch.tensor([launches], device=dev, dtype=torch.float64)
        dist.all_reduce(tl)
        launches = int(tl.item())
    if rank != 0:
        dist.destroy_process_group()
        return
    # ---- rooflines of the two candidate dominant kernels, from the profiled twin's live CUDA
    # events on the launching stream (phases serialised, L2 flushed, same steps)
    peaks = json.load(open(os.path.join(ROOT, "profiles", "fp64_peaks_r01.json")))
    ncu = ncu_evidence(args.config) if ws == 1 else None
    k = info["k"]
    m2l_flops = float(info["m2l_flops"])  # sum over this rank's V pairs of 2 k^2
    m2l_ms = phase["m2l"]
    m2l_peak = float(peaks["dmma_m8n8k4_tflops"])
    m2l_tf = m2l_flops / (m2l_ms * 1e-3) / 1e12
    m2l = {"bound": "tensor", "kernel": "M2L: k_m2l_sib16 (DMMA.8x8x4 FP64 via mma.sync m16n8k8)",
           "achieved": m2l_tf, "peak": m2l_peak, "unit": "TFLOP/s", "frac": m2l_tf / m2l_peak,
           "traffic": (ncu or {}).get("m2l", {}).get("dram_bytes_per_launch"),
           "tensor_pipe_active_pct_ncu": (ncu or {}).get("m2l", {}).get("tensor_pipe_active_pct"),
           "peak_source": "measured: tools/microbench/fp64_peaks.cu DMMA loop on this pool's B200 "
                          "(profiles/fp64_peaks_r01.json; MEASURED_PEAKS.json has no FP64 figure)",
           "per_unit": "2 k_eff^2 flops per V pair", "units_per_launch": info["nV_local"],
           "flops_per_launch": m2l_flops, "ms_per_launch": m2l_ms}
    # near field (P2P, FP64 ALU, issue-bound): the FP64 instructions of the minimal pair
    # formulation (13 per unordered mutual pair: 3 DADD, DMUL + 2 DFMA for r^2, 5 for the rsqrt
    # correction, 2 DFMA accumulations; 12 per one-sided pair) over the k_near launches alone
    # (fmm_info.near_ms), against the FP64 pipe's instruction rate (measured DFMA loop / 2)
    near = None
    if info["near_pairs"] > 0 and info["near_ms"] > 0:
        npair, pm = int(info["near_pairs"]), int(info["near_mutual_pairs"])
        instr = 13.0 * pm + 12.0 * (npair - 2 * pm)
        lane_peak = float(peaks["dfma_tflops"]) / 2  # T FP64 instruction-lanes / s (a DFMA = 2 flops)
        near_s = info["near_ms"] * 1e-3
        near = {"bound": "alu", "kernel": "k_near (P2P, mutual leaf pairs; every pass-shape launch of one matvec)",
                "achieved": instr / near_s / 1e12, "peak": lane_peak, "unit": "T FP64 instr-lanes/s",
                "frac": instr / near_s / 1e12 / lane_peak,
                "traffic": (ncu or {}).get("near", {}).get("dram_bytes_per_launch"),
                "fp64_pipe_active_pct_ncu": (ncu or {}).get("near", {}).get("fp64_pipe_active_pct"),
                "peak_source": "measured DFMA loop (profiles/fp64_peaks_r01.json) / 2 = 148 SMs x 64 FP64 lanes x clock",
                "per_unit": "13 FP64 instr per unordered mutual pair, 12 per one-sided pair",
                "directed_pairs": npair, "mutual_pairs": pm, "units_per_launch": npair,
                "pairs_per_s": npair / near_s, "ms_per_launch": info["near_ms"]}
    # the dominant kernel of this config is the one with the larger share of the step
    cand = [x for x in (m2l, near) if x is not None]
    roof = max(cand, key=lambda x: x["ms_per_launch"])
    roof = dict(roof, timed_in="profiled twin plan of the same workload: phases serialised on one stream, "
                                "CUDA events around the kernel's launches, L2 flushed, same step count",
                share_of_serial_step=roof["ms_per_launch"] / sum(phase.values()))
    if ncu:
        roof["ncu_source"] = ncu.get("source")
    # ---- cpu baseline: the oracle on the host cores, one full matvec (rank 0, N = 1 only)
    cpu = None
    if ws == 1 and not args.no_cpu_baseline:
        sp, sq, what = oracle_sample(args.config, pts, q)
        ts = oracle_matvec_timer(sp, sq, cfg, reps=1)
        cpu = {"value": sp.shape[0] / ts[0], "unit": "points/s", "cores": cpu_cores(), "kind": "oracle",
               "sample": f"{what}: one oracle matvec of {sp.shape[0]} points, oracle/ C++ -O2 OpenMP, {ts[0]:.2f} s"}
    value = N / (ms * 1e-3)
    config = workload_config(args, cfg, ws, k)
    ovl = int(plan.get_info()["overlap"])  # the production plan's mode (the profiled twin runs serialised)
    method = {"l2": "flushed (256 MiB write) between timed steps",
              "overlap": ovl,
              "near_field": ("mutual leaf pairs (k_near) on a second stream beside the far field (overlap mode 3)"
                             if ovl == 3 else
                             "mutual leaf pairs (k_near), serialised with the far field")}
    if ws > 1:
        method.update(mode="owned", ghost_q_rows_rank0=info["ghost_q_recv"], ghost_dens_rank0=info["ghost_d_recv"],
                      straddling_boxes=info["n_straddle"])
    line = {
        "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": ws, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak" if args.weak else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config, "method": method,
        "roofline": roof,
        "kernels": {"m2l": m2l, "p2p": near},
        "phase_ms": phase,
        "clocks": clk.summary(),
        "e2e": {"value": N / e2e_s, "unit": "points/s", "h2d_bytes_per_step": e2e_bytes,
                "d2h_bytes_per_step": e2e_bytes, "ms_per_step": e2e_s * 1e3, "api": e2e_api},
        "gpu_launches": launches,
        "setup_s": setup_s,
        "precompute_ms": info["precompute_ms"],
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
