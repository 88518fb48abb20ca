#!/bin/bash
O=gpurun_out; T=${1:-r02t}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${T}_smoke.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "window or relabel or far or full_config or paths or sharded" > $O/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${T}_pytest.log
B="python bench.py --config scale --steps 10 --no-cpu-baseline --no-e2e"
timeout 600 $B > $O/${T}_scale_1.json 2> $O/${T}_scale_1.err
timeout 600 $B --no-timing > $O/${T}_scale_2.json 2> $O/${T}_scale_2.err
timeout 600 $B > $O/${T}_scale_3.json 2> $O/${T}_scale_3.err
echo done > $O/${T}_done
