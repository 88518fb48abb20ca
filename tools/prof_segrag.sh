#!/bin/bash
# source-level ncu capture of the segment kernel of the compacting chain at Text
O=gpurun_out; T=${1:-ps}
mkdir -p $O
N="ncu --set full --clock-control none --import-source on"
B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-timing --config text"
timeout 600 $N -k 'regex:segment_rag' -s 20 -c 1 -o $O/${T}_seg -f $B > $O/${T}_s.log 2>&1
echo done > $O/${T}_done
