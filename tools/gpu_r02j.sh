#!/bin/bash
# r02 pass j: ncu source-level captures: light (Scale level-5 batch), tp_scatter, segment_rag
O=gpurun_out; T=${1:-r02j}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${T}_build.log 2>&1
N="ncu --set full --clock-control none --import-source on"
B="python bench.py --config scale --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-timing"
timeout 900 $N -k 'regex:light_kernel' -s 100 -c 1 -o $O/${T}_light -f $B > $O/${T}_ncu_light.log 2>&1
timeout 900 $N -k 'regex:tp_scatter' -s 600 -c 1 -o $O/${T}_tps -f $B > $O/${T}_ncu_tps.log 2>&1
timeout 900 $N -k 'regex:segment_rag' -s 40 -c 1 -o $O/${T}_seg -f $B > $O/${T}_ncu_seg.log 2>&1
timeout 900 $N -k 'regex:epilogue_kernel' -s 0 -c 1 -o $O/${T}_epi -f $B > $O/${T}_ncu_epi.log 2>&1
echo done > $O/${T}_done
