#!/bin/bash
# r02 first pass: tests, current bench lines on Scale / Text, peaks, Scale oracle digests.
O=gpurun_out; T=r02a
mkdir -p $O
lscpu > $O/${T}_lscpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${T}_smoke.log
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${T}_pytest.log
for c in scale text; do
  timeout 600 python bench.py --config $c --steps 5 --no-cpu-baseline > $O/${T}_bench_$c.json 2> $O/${T}_bench_$c.err
done
timeout 300 python tools/measure_peaks.py --out $O/${T}_peaks.json > $O/${T}_peaks.log 2>&1
timeout 2400 python -m oracle.make_digests scale --out $O/oracle_scale.json > $O/${T}_orc_scale.log 2>&1
echo done > $O/${T}_done
