#!/bin/bash
# r02 pass g: ncu full captures of the Scale light kernel (level-5 batch) and far_add
O=gpurun_out; T=${1:-r02g}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${T}_build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:light_kernel' -s 100 -c 1 \
  -o $O/${T}_light -f python bench.py --config scale --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-timing > $O/${T}_ncu_light.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:far_add' -s 0 -c 40 \
  -o $O/${T}_far -f python bench.py --config scale --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-timing > $O/${T}_ncu_far.log 2>&1
echo done > $O/${T}_done
