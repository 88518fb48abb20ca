#!/bin/bash
# validation after removing the steady-state cudaMemGetInfo / syncs from accumulate
O=gpurun_out; T=${1:-r02aa}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${T}_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${T}_pytest.log
GAKCO_HOST_TRACE=1 timeout 600 python tools/outlier.py scale 24 > $O/${T}_out.log 2> $O/${T}_out.err
B="python bench.py --steps 10 --no-cpu-baseline --no-e2e"
for r in 1 2 3; do timeout 600 $B --config scale > $O/${T}_scale_$r.json 2> $O/${T}_scale_$r.err; done
for c in text dna protein; do timeout 600 $B --config $c > $O/${T}_$c.json 2> $O/${T}_$c.err; done
echo done > $O/${T}_done
