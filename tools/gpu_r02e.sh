#!/bin/bash
# r02 pass e: tests (PYTEST_K selects), bench lines Scale (far on / off) and Text
O=gpurun_out; T=${1:-r02e}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${T}_smoke.log
if [ -n "$PYTEST_K" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 -k "$PYTEST_K" > $O/${T}_pytest.log 2>&1
else
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > $O/${T}_pytest.log 2>&1
fi
echo "pytest rc=$?" >> $O/${T}_pytest.log
timeout 600 python bench.py --config scale --steps 5 --no-cpu-baseline --no-e2e > $O/${T}_bench_scale.json 2> $O/${T}_bench_scale.err
timeout 600 python bench.py --config scale --steps 5 --no-cpu-baseline --no-e2e --far-near 0 > $O/${T}_bench_scale_nofar.json 2> $O/${T}_bench_scale_nofar.err
timeout 600 python bench.py --config text --steps 5 --no-cpu-baseline --no-e2e > $O/${T}_bench_text.json 2> $O/${T}_bench_text.err
echo done > $O/${T}_done
