python bench.py --config dna --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/pg_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:bk_group -s 3 -c 1 -o gpurun_out/pg_group -f python bench.py --config dna --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-timing > gpurun_out/pg_ncu1.log 2>&1
