"""Summarise an ncu report: key raw metrics + top source lines by stall samples.
    python tools/ncu_summary.py report.ncu-rep [--source]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2:]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "lts__t_bytes.sum", "l1tex__t_bytes.sum", "launch__grid_size", "launch__block_size"]
for v in vals:
    for h, u, x in zip(hdr, units, v):
        if h in want or (h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio")):
            try:
                if h.startswith("smsp__average") and float(x) < 0.05:
                    continue
            except ValueError:
                pass
            print(f"{h:90s} {x} {u}")
    print("-" * 40)
if "--source" in sys.argv:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(src)))
    r = [x for x in r if len(x) > 3]
    h = r[0]
    try:
        si = h.index("Warp Stall Sampling (All Samples)")
    except ValueError:
        si = None
    ii = h.index("Source") if "Source" in h else 1
    if si is not None:
        body = [x for x in r[1:] if len(x) > si and x[si].replace('.', '').isdigit()]
        body.sort(key=lambda x: -float(x[si]))
        tot = sum(float(x[si]) for x in body) or 1
        for x in body[:25]:
            print(f"{100*float(x[si])/tot:5.1f}%  {x[ii][:110]}")
