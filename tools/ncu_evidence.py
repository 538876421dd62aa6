"""Per-config ncu evidence for bench.py's roofline lines (profiles/ncu_<config>.json), from
the `ncu --set full` captures tools/gpu_profile.sh makes of one production matvec:
  near  every k_near launch of the matvec (one per pass shape): time-weighted FP64-pipe
        active %, DRAM bytes summed over the launches (one "launch" of the kernel family)
  m2l   the k_m2l_sib16 launch: tensor (DMMA) pipe active %, DRAM bytes
    python tools/ncu_evidence.py <knear.ncu-rep> <m2l.ncu-rep> <config> [tag]"""
import csv
import io
import json
import subprocess
import sys


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, r):
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                d[h] = v
                continue
            # times to ms, bytes to bytes (ncu picks the unit per value: a short kernel's
            # duration comes in us, a long one's in ms)
            scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "KB": 1e3, "MB": 1e6, "GB": 1e9,
                     "B": 1.0, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6,
                     "ns": 1e-6, "second": 1e3, "s": 1e3}.get(u, 1.0)
            d[h] = x * scale
        res.append(d)
    return res


def main():
    knear, m2l, cfg = sys.argv[1:4]
    tag = sys.argv[4] if len(sys.argv) > 4 else ""
    kn = [r for r in raw(knear) if "k_near" in r.get("Kernel Name", "")]
    t = sum(r["gpu__time_duration.sum"] for r in kn)
    near = {
        "kernel": f"k_near ({len(kn)} pass-shape launches of one matvec)",
        "fp64_pipe_active_pct": sum(r["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"] *
                                    r["gpu__time_duration.sum"] for r in kn) / t,
        "dram_bytes_per_launch": sum(r["dram__bytes_read.sum"] + r["dram__bytes_write.sum"] for r in kn),
        "ms_ncu": t,
        "shapes": {r["Kernel Name"].split("(")[0].split("::")[-1]: {
            "ms": round(r["gpu__time_duration.sum"], 4),
            "fp64_pipe_pct": round(r["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"], 2),
            "registers": r.get("launch__registers_per_thread"),
            "warps_active_pct": round(r["sm__warps_active.avg.pct_of_peak_sustained_active"], 2)} for r in kn},
    }
    mm = [r for r in raw(m2l) if "k_m2l" in r.get("Kernel Name", "")][0]
    m2 = {
        "kernel": mm["Kernel Name"].split("(")[0],
        "tensor_pipe_active_pct": mm["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"],
        "dram_bytes_per_launch": mm["dram__bytes_read.sum"] + mm["dram__bytes_write.sum"],
        "ms_ncu": mm["gpu__time_duration.sum"],
    }
    out = {"config": cfg, "near": near, "m2l": m2,
           "source": f"ncu --set full --clock-control none of tools/one_matvec.py {cfg} "
                     f"(tools/gpu_profile.sh {cfg} {tag}; cold-cache serialised launches)"}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
