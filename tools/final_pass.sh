#!/bin/bash
# round-end evidence pass: every config bench line, the Scale launch list + captures, the reference arm
bash tools/bench_configs.sh r02z
bash tools/prof_bench.sh r02z
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02z_reference.json 2> gpurun_out/r02z_reference.err
