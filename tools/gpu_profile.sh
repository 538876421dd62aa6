#!/bin/bash
# Measurement pass for one config on the GPU box (run under gpurun):
#   bench line, ncu launch list of one production matvec, ncu --set full of the two
#   candidate dominant kernels (k_near pass shapes, M2L), summarised on the box.
#   tools/gpu_profile.sh <config> <tag>
# The .ncu-rep files stay in /tmp on the box (they are tens of MB each; gpurun copies back at
# most 64 MB of gpurun_out); gpurun_out receives the bench line, the launch list and the
# per-config evidence JSON (tools/ncu_evidence.py).  No `timeout` around ncu: killing ncu in
# the middle of a replay can leave the GPU unusable — keep the profiled command small.
cfg=${1:-C4}; tag=${2:-r02}
o=gpurun_out
t=/tmp/kifmm_prof; mkdir -p $t
python bench.py --config $cfg --steps 10 --warmup 3 > $o/${tag}_bench_$cfg.log 2>&1 || { echo "bench failed"; tail -20 $o/${tag}_bench_$cfg.log; exit 1; }
tail -1 $o/${tag}_bench_$cfg.log
python tools/one_matvec.py $cfg > $t/plain_$cfg.log 2>&1 || { echo "one_matvec failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $t/launches_$cfg.csv \
    python tools/one_matvec.py $cfg > $t/ncu1_$cfg.log 2>&1 &&
python tools/launch_summary.py $t/launches_$cfg.csv $cfg > $o/${tag}_launches_$cfg.txt
# full sets: the k_near launches of the last matvec (skip the first three matvecs' launches)
nk=$(grep -c 'k_near' $t/launches_$cfg.csv)
per=$((nk / 4))
ncu --set full --clock-control none --import-source on -k regex:k_near -s $((3 * per)) -c $per \
    -o $t/knear_$cfg -f python tools/one_matvec.py $cfg > $t/ncu2_$cfg.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_m2l -s 3 -c 1 \
    -o $t/m2l_$cfg -f python tools/one_matvec.py $cfg > $t/ncu3_$cfg.log 2>&1
python tools/ncu_evidence.py $t/knear_$cfg.ncu-rep $t/m2l_$cfg.ncu-rep $cfg $tag > $o/ncu_${cfg}_${tag}.json
ls -la $o | grep $tag
