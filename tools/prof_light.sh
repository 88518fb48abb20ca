#!/bin/bash
# full ncu capture (source-level) of the light kernel at Scale (a relabelled level)
O=gpurun_out; T=${1:-plt}
mkdir -p $O
N="ncu --set full --clock-control none --import-source on"
B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-timing --config scale"
timeout 600 $N -k 'regex:light_kernel' -s 60 -c 1 -o $O/${T}_light -f $B > $O/${T}_l.log 2>&1
echo done > $O/${T}_done
