#!/bin/bash
# r02 pass h: Scale light variants (far apply v3, register budgets), quick tests
O=gpurun_out; T=${1:-r02h}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${T}_smoke.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "far or relabel or window or sharded" > $O/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${T}_pytest.log
B="python bench.py --config scale --steps 5 --no-cpu-baseline --no-e2e"
timeout 600 $B > $O/${T}_scale.json 2> $O/${T}_scale.err
timeout 600 $B --far-near 0 > $O/${T}_scale_nofar.json 2> $O/${T}_scale_nofar.err
timeout 600 $B --light-ctas 4 > $O/${T}_scale_c4.json 2> $O/${T}_scale_c4.err
timeout 600 $B --light-ctas 6 > $O/${T}_scale_c6.json 2> $O/${T}_scale_c6.err
timeout 600 $B --light-ctas 4 --far-near 0 > $O/${T}_scale_c4_nofar.json 2> $O/${T}_scale_c4_nofar.err
timeout 600 $B --xl-compact 0 > $O/${T}_scale_nocompact.json 2> $O/${T}_scale_nocompact.err
echo done > $O/${T}_done
