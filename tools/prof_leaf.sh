#!/bin/bash
# full ncu capture (source-level) of the fused leaf kernel at Scale and Text
O=gpurun_out; T=${1:-pl}
mkdir -p $O
N="ncu --set full --clock-control none --import-source on"
for c in scale text; do
B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-timing --config $c"
timeout 600 $N -k 'regex:leaf_kernel' -s 300 -c 1 -o $O/${T}_leaf_$c -f $B > $O/${T}_l_$c.log 2>&1
done
echo done > $O/${T}_done
