#!/bin/bash
O=gpurun_out; T=${1:-r02w}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${T}_build.log 2>&1
B="python bench.py --steps 10 --no-cpu-baseline --no-e2e"
for r in 1 2 3; do timeout 600 $B --config scale > $O/${T}_scale_$r.json 2> $O/${T}_scale_$r.err; done
timeout 600 $B --config text > $O/${T}_text.json 2> $O/${T}_text.err
echo done > $O/${T}_done
