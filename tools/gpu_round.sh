#!/bin/bash
# One GPU-box pass: build check, parity tests, bench lines, ncu launch list + full capture.
#   gpurun --timeout 2700 -- 'bash tools/gpu_round.sh TAG'
TAG=${1:-r01}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $O/${TAG}_smi.txt 2>&1
lscpu > $O/${TAG}_lscpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${TAG}_smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${TAG}_pytest.log
timeout 600 python bench.py > $O/${TAG}_bench_dna.json 2> $O/${TAG}_bench_dna.err
for c in protein text scale; do
  timeout 600 python bench.py --config $c --steps 3 --no-cpu-baseline > $O/${TAG}_bench_$c.json 2> $O/${TAG}_bench_$c.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/${TAG}_bench_ref.json 2> $O/${TAG}_bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file $O/${TAG}_launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $O/${TAG}_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k 'regex:gram4_kernel|gram2_kernel|light_kernel|radix_scatter2|radix_hist|segment_kernel|build_dense3|epilogue_kernel|trie_root' \
  -s ${SKIP:-40} -c 16 \
  -o $O/${TAG}_prof -f python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-timing > $O/${TAG}_ncu_full.log 2>&1
echo done > $O/${TAG}_done
