#!/bin/bash
# r02 pass i: full GPU tests (5-config digests), checked-library tests, bench lines
O=gpurun_out; T=${1:-r02i}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${T}_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > $O/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${T}_pytest.log
B="python bench.py --steps 5 --no-cpu-baseline --no-e2e"
timeout 600 $B --config scale > $O/${T}_scale.json 2> $O/${T}_scale.err
timeout 600 $B --config text > $O/${T}_text.json 2> $O/${T}_text.err
timeout 600 $B --config scale --far-near 0 > $O/${T}_scale_nofar.json 2> $O/${T}_scale_nofar.err
GAKCO_LIB=$PWD/paper_1704_07468_b200/libgakco_checked.so timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/${T}_pytest_checked.log 2>&1; echo "pytest rc=$?" >> $O/${T}_pytest_checked.log
echo done > $O/${T}_done
