#!/bin/bash
# r02 pass c: tests (compaction), bench lines, ncu launch list of one Scale step, ncu full
# captures of the trie pass / light / far-record / segment kernels.
O=gpurun_out; T=${1:-r02c}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${T}_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=20 > $O/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${T}_pytest.log
for c in scale text; do
  timeout 600 python bench.py --config $c --steps 5 --no-cpu-baseline --no-e2e > $O/${T}_bench_$c.json 2> $O/${T}_bench_$c.err
  timeout 600 python bench.py --config $c --steps 5 --no-cpu-baseline --no-e2e --far-near 0 --xl-compact 0 > $O/${T}_bench_${c}_old.json 2> $O/${T}_bench_${c}_old.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${T}_launches_scale.csv \
  python bench.py --config scale --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-timing > $O/${T}_ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k 'regex:tp_scatter|tp_hist|light_kernel|far_|segment_rag' -s 30 -c 14 \
  -o $O/${T}_scale_full -f python bench.py --config scale --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-timing > $O/${T}_ncu_full.log 2>&1
echo done > $O/${T}_done
