#!/bin/bash
# profiles of the bench configuration (Scale): launch list of one step
# (gpu__time_duration, --clock-control none) and full captures of its top kernels
O=gpurun_out; T=${1:-r02z}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${T}_build.log 2>&1
B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-timing"
timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-e2e > $O/${T}_bench.json 2> $O/${T}_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${T}_launches.csv $B > $O/${T}_ncu_launch.log 2>&1
N="ncu --set full --clock-control none --import-source on"
timeout 600 $N -k 'regex:light_kernel' -s 30 -c 1 -o $O/${T}_light -f $B > $O/${T}_l.log 2>&1
timeout 600 $N -k 'regex:tp_scatter' -s 400 -c 1 -o $O/${T}_tps -f $B > $O/${T}_t.log 2>&1
timeout 600 $N -k 'regex:tp_hist' -s 400 -c 1 -o $O/${T}_tph -f $B > $O/${T}_th.log 2>&1
timeout 600 $N -k 'regex:leaf_kernel' -s 300 -c 1 -o $O/${T}_leaf -f $B > $O/${T}_s.log 2>&1
timeout 600 $N -k 'regex:far_add' -s 10 -c 1 -o $O/${T}_far -f $B > $O/${T}_f.log 2>&1
timeout 600 $N -k 'regex:epilogue_kernel' -s 0 -c 1 -o $O/${T}_epi -f $B > $O/${T}_e.log 2>&1
timeout 600 $N -k 'regex:window_build' -s 30 -c 1 -o $O/${T}_wb -f $B > $O/${T}_w.log 2>&1
echo done > $O/${T}_done
