"""One line per kernel launch of an ncu report: time, pipe utilisations, SM balance, DRAM bytes.
    python tools/ncu_table.py report.ncu-rep"""
import csv, io, subprocess, sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, vals = rows[0], rows[2:]
col = {h: i for i, h in enumerate(hdr)}
def g(v, name):
    try:
        return float(v[col[name]].replace(",", ""))
    except (KeyError, ValueError):
        return float("nan")
print(f"{'kernel':34s} {'us':>8s} {'tensor%':>7s} {'fp64%':>6s} {'issue%':>6s} {'act/el':>6s} {'min/max':>7s} {'warps%':>6s} {'dramMB':>7s} {'regs':>4s} {'grid':>6s}")
for v in vals:
    name = v[col["Kernel Name"]].split("(")[0].replace("void ", "").replace("kifmm::", "")[:34]
    t = g(v, "gpu__time_duration.sum")
    unit = 1e-3 if "usecond" in rows[1][col["gpu__time_duration.sum"]] else 1.0
    print(f"{name:34s} {t * (1 if unit == 1e-3 else 1e3) if t == t else 0:8.1f} "
          f"{g(v, 'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active'):7.1f} "
          f"{g(v, 'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active'):6.1f} "
          f"{g(v, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):6.1f} "
          f"{g(v, 'sm__cycles_active.avg') / g(v, 'sm__cycles_elapsed.avg'):6.2f} "
          f"{g(v, 'sm__cycles_active.min') / g(v, 'sm__cycles_active.max'):7.2f} "
          f"{g(v, 'sm__warps_active.avg.pct_of_peak_sustained_active'):6.1f} "
          f"{(g(v, 'dram__bytes_read.sum') + g(v, 'dram__bytes_write.sum')) / (1 if 'Mbyte' in rows[1][col['dram__bytes_read.sum']] else 1e6):7.1f} "
          f"{g(v, 'launch__registers_per_thread'):4.0f} {g(v, 'launch__grid_size'):6.0f}")
