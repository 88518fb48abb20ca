#!/bin/bash
# round-end evidence pass: every config bench line, the Scale launch list + captures, the reference arm
bash tools/bench_configs.sh ${1:-r02f}
bash tools/prof_bench.sh ${1:-r02f}
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${1:-r02f}_reference.json 2> gpurun_out/${1:-r02f}_reference.err
