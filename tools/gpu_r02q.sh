#!/bin/bash
# r02 pass q: Scale tuning sweep (all exact; timing only)
O=gpurun_out; T=${1:-r02q}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${T}_build.log 2>&1
B="python bench.py --config scale --steps 5 --no-cpu-baseline --no-e2e --no-timing"
run() { n=$1; shift; timeout 600 $B "$@" > $O/${T}_$n.json 2> $O/${T}_$n.err; }
run base1
run wmin5 --window-min 5
run wmin12 --window-min 12
run near1k --far-near 1024
run bk32 --batch-keys 33554432
run bk128 --batch-keys 134217728
run flat4 --light-flat 4
run flat16 --light-flat 16
run ctas3 --light-ctas 3
run base2
echo done > $O/${T}_done
