#!/bin/bash
# r02 pass k: tests, bench lines (all configs), light-grid experiment, NEXT-3 sweeps w/ parity
O=gpurun_out; T=${1:-r02k}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${T}_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > $O/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${T}_pytest.log
B="python bench.py --steps 5 --no-cpu-baseline --no-e2e"
for c in scale text dna protein; do timeout 600 $B --config $c > $O/${T}_$c.json 2> $O/${T}_$c.err; done
timeout 600 $B --config scale --light-grid 2 > $O/${T}_scale_g2.json 2> $O/${T}_scale_g2.err
timeout 600 $B --config scale --light-grid 3 > $O/${T}_scale_g3.json 2> $O/${T}_scale_g3.err
timeout 1800 python tools/sweep.py --out $O/sweeps_r02.json > $O/${T}_sweep.log 2>&1; echo "sweep rc=$?" >> $O/${T}_sweep.log
echo done > $O/${T}_done
