#!/bin/bash
# r02 pass d: tests, bench lines (far records gated, compaction), memcheck on the paths
O=gpurun_out; T=${1:-r02d}; KX=${2:-}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${T}_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 $KX > $O/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${T}_pytest.log
for c in scale text; do
  timeout 600 python bench.py --config $c --steps 5 --no-cpu-baseline --no-e2e > $O/${T}_bench_$c.json 2> $O/${T}_bench_$c.err
done
timeout 600 python bench.py --config scale --steps 5 --no-cpu-baseline --no-e2e --far-near 0 > $O/${T}_bench_scale_nofar.json 2> $O/${T}_bench_scale_nofar.err
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize.py > $O/${T}_memcheck.log 2>&1; echo "rc=$?" >> $O/${T}_memcheck.log
echo done > $O/${T}_done
