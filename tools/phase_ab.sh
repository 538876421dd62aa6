#!/bin/bash
# A/B of env-selected kernel variants on one config: tools/phase_ab.sh C2 "VAR=a" "VAR=b" ...
cfg=$1; shift
for v in "$@"; do echo "== $v"; env $v python tools/phase_timing.py $cfg 7 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('median ms %.4f'%sorted(d['ms'])[len(d['ms'])//2], {k:round(v,4) for k,v in d['phase_ms'].items()})"; done
