#!/bin/bash
# full ncu captures (source-level) of the trie pass kernels at Scale
O=gpurun_out; T=${1:-pt}
mkdir -p $O
B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-timing"
N="ncu --set full --clock-control none --import-source on"
timeout 600 $N -k 'regex:tp_scatter' -s 400 -c 1 -o $O/${T}_tps -f $B > $O/${T}_t.log 2>&1
timeout 600 $N -k 'regex:tp_hist' -s 400 -c 1 -o $O/${T}_tph -f $B > $O/${T}_th.log 2>&1
echo done > $O/${T}_done
