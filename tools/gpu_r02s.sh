#!/bin/bash
O=gpurun_out; T=${1:-r02s}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${T}_smoke.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "window or relabel or far or full_config or paths" > $O/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${T}_pytest.log
B="python bench.py --steps 5 --no-cpu-baseline --no-e2e"
timeout 600 $B --config scale > $O/${T}_scale_1.json 2> $O/${T}_scale_1.err
timeout 600 $B --config scale --no-timing > $O/${T}_scale_2.json 2> $O/${T}_scale_2.err
timeout 600 $B --config text > $O/${T}_text_1.json 2> $O/${T}_text_1.err
timeout 600 $B --config text --no-timing > $O/${T}_text_2.json 2> $O/${T}_text_2.err
echo done > $O/${T}_done
