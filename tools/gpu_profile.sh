#!/bin/bash
# Measurement pass for one config on the GPU box (run under gpurun):
#   bench line, ncu launch list of one production matvec, ncu --set full of the two
#   candidate dominant kernels (k_near pass shapes, M2L).
#   tools/gpu_profile.sh <config> <tag>
cfg=${1:-C4}; tag=${2:-r02}
o=gpurun_out
python bench.py --config $cfg --steps 10 --warmup 3 > $o/${tag}_bench_$cfg.log 2>&1 || { echo "bench failed"; tail -20 $o/${tag}_bench_$cfg.log; exit 1; }
tail -1 $o/${tag}_bench_$cfg.log
python tools/one_matvec.py $cfg > $o/${tag}_plain_$cfg.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/${tag}_launches_$cfg.csv \
    python tools/one_matvec.py $cfg > $o/${tag}_ncu1_$cfg.log 2>&1 &&
python tools/launch_summary.py $o/${tag}_launches_$cfg.csv $cfg > $o/${tag}_launches_$cfg.txt
# full sets: the k_near launches of the last matvec (skip the first three matvecs' launches)
nk=$(grep -c 'k_near' $o/${tag}_launches_$cfg.csv)
per=$((nk / 4))
ncu --set full --clock-control none --import-source on -k regex:k_near -s $((3 * per)) -c $per \
    -o $o/${tag}_knear_$cfg -f python tools/one_matvec.py $cfg > $o/${tag}_ncu2_$cfg.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_m2l -s 3 -c 1 \
    -o $o/${tag}_m2l_$cfg -f python tools/one_matvec.py $cfg > $o/${tag}_ncu3_$cfg.log 2>&1
ls -la $o
