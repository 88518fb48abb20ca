#!/bin/bash
# r02 pass l: run-to-run variance of the pipelined step; pipeline off; light grid 3
O=gpurun_out; T=${1:-r02l}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${T}_build.log 2>&1
B="python bench.py --steps 10 --no-cpu-baseline --no-e2e --no-timing"
for r in 1 2; do
  timeout 600 $B --config scale > $O/${T}_scale_$r.json 2>&1
  timeout 600 $B --config scale --light-grid 3 > $O/${T}_scale_g3_$r.json 2>&1
  timeout 600 $B --config text > $O/${T}_text_$r.json 2>&1
  timeout 600 $B --config text --pipeline 0 > $O/${T}_text_p0_$r.json 2>&1
  timeout 600 $B --config protein > $O/${T}_protein_$r.json 2>&1
  timeout 600 $B --config protein --pipeline 0 > $O/${T}_protein_p0_$r.json 2>&1
done
timeout 600 $B --config scale --pipeline 0 > $O/${T}_scale_p0.json 2>&1
echo done > $O/${T}_done
