#!/bin/bash
# r02 pass b: new tests (sharded step, trie pass, far records, e2m1 sums, k-sweep, 5-config
# digests), bench lines on Scale / Text with the trie pass + far records and ablations.
O=gpurun_out; T=${1:-r02b}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${T}_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x --durations=15 > $O/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${T}_pytest.log
timeout 600 python bench.py --config scale --steps 5 --no-cpu-baseline > $O/${T}_bench_scale.json 2> $O/${T}_bench_scale.err
timeout 600 python bench.py --config scale --steps 5 --no-cpu-baseline --no-e2e --far-near 0 > $O/${T}_bench_scale_nofar.json 2> $O/${T}_bench_scale_nofar.err
timeout 600 python bench.py --config text --steps 5 --no-cpu-baseline --no-e2e > $O/${T}_bench_text.json 2> $O/${T}_bench_text.err
timeout 600 python bench.py --config text --steps 5 --no-cpu-baseline --no-e2e --trie-pass 0 > $O/${T}_bench_text_tp0.json 2> $O/${T}_bench_text_tp0.err
timeout 600 python bench.py --config dna --steps 20 --no-cpu-baseline --no-e2e > $O/${T}_bench_dna.json 2> $O/${T}_bench_dna.err
echo done > $O/${T}_done
