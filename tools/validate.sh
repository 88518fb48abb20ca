#!/bin/bash
# validation pass: smoke, the Scale-path GPU tests, three Scale bench lines
#   gpurun --timeout 2400 -- "bash tools/validate.sh TAG"
O=gpurun_out; T=${1:-val}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${T}_smoke.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "window or relabel or far or full_config or paths or sharded or k_only" > $O/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${T}_pytest.log
B="python bench.py --steps 10 --no-cpu-baseline --no-e2e"
for r in 1 2 3; do timeout 600 $B --config scale > $O/${T}_scale_$r.json 2> $O/${T}_scale_$r.err; done
echo done > $O/${T}_done
