python bench.py --config dna --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/pbk_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:bk_group -s 20 -c 2 -o gpurun_out/pbk_group -f python bench.py --config dna --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-timing > gpurun_out/pbk_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:bk_pass -s 20 -c 4 -o gpurun_out/pbk_pass -f python bench.py --config dna --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-timing > gpurun_out/pbk_ncu2.log 2>&1
