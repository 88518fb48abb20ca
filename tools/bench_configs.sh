#!/bin/bash
# bench lines of every config (Scale x3, Text, DNA, Protein, the default line)
O=gpurun_out; T=${1:-cfg}
mkdir -p $O
B="python bench.py --steps 10 --no-cpu-baseline --no-e2e"
for r in 1 2 3; do timeout 600 $B --config scale > $O/${T}_scale_$r.json 2> $O/${T}_scale_$r.err; done
for c in text dna protein; do timeout 600 $B --config $c > $O/${T}_$c.json 2> $O/${T}_$c.err; done
timeout 900 python bench.py > $O/${T}_default.json 2> $O/${T}_default.err
echo done > $O/${T}_done
