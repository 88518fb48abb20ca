#!/bin/bash
# r02 pass f: sharded tests (p2p), Scale launch list + ncu full on light / far / trie / segment
O=gpurun_out; T=${1:-r02f}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${T}_smoke.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "sharded or far or relabel or window" > $O/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${T}_pytest.log
timeout 600 python bench.py --config scale --steps 5 --no-cpu-baseline --no-e2e > $O/${T}_bench_scale.json 2> $O/${T}_bench_scale.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${T}_launches_scale.csv \
  python bench.py --config scale --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-timing > $O/${T}_ncu_launch.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k 'regex:light_kernel|far_add|tp_scatter|tp_hist|segment_rag|window_build' -s 200 -c 16 \
  -o $O/${T}_scale_full -f python bench.py --config scale --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-timing > $O/${T}_ncu_full.log 2>&1
echo done > $O/${T}_done
