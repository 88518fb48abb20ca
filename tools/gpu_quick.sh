#!/bin/bash
# Quick GPU pass: build, parity tests (optionally filtered), bench lines.
#   gpurun -- 'bash tools/gpu_quick.sh TAG "pytest -k expr" "configs"'
TAG=${1:-q}
KEXPR=${2:-}
CONFIGS=${3:-dna}
O=gpurun_out
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${TAG}_smoke.log
if [ -n "$KEXPR" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "$KEXPR" > $O/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${TAG}_pytest.log
else
  timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${TAG}_pytest.log
fi
for c in $CONFIGS; do
  timeout 600 python bench.py --config $c --steps 3 --no-cpu-baseline --no-e2e > $O/${TAG}_bench_$c.json 2> $O/${TAG}_bench_$c.err
  timeout 600 python bench.py --config $c --steps 3 --no-cpu-baseline --no-e2e --sort 0 > $O/${TAG}_bench_${c}_lsd.json 2> $O/${TAG}_bench_${c}_lsd.err
done
echo done > $O/${TAG}_done
