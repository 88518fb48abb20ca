#!/bin/bash
# iteration pass: GPU tests (all, or those matching $2), then bench lines of the
# configs in $3 (default "scale text")
O=gpurun_out; T=${1:-it}; K=${2:-}; C=${3:-scale text}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${T}_smoke.log
if [ -n "$K" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "$K" > $O/${T}_pytest.log 2>&1
else
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/${T}_pytest.log 2>&1
fi
echo "pytest rc=$?" >> $O/${T}_pytest.log
for c in $C; do timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-e2e --config $c > $O/${T}_$c.json 2> $O/${T}_$c.err; done
echo done > $O/${T}_done
