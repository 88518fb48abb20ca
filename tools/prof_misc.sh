#!/bin/bash
# source-level ncu captures of window_build and far_add at Scale
O=gpurun_out; T=${1:-pm}
mkdir -p $O
N="ncu --set full --clock-control none --import-source on"
B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-timing --config scale"
timeout 600 $N -k 'regex:window_build' -s 60 -c 1 -o $O/${T}_wb -f $B > $O/${T}_w.log 2>&1
timeout 600 $N -k 'regex:far_add' -s 20 -c 1 -o $O/${T}_far -f $B > $O/${T}_f.log 2>&1
timeout 600 $N -k 'regex:light_flush_perm' -s 1 -c 1 -o $O/${T}_lfp -f $B > $O/${T}_lfp.log 2>&1
echo done > $O/${T}_done
