python bench.py --config dna --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/pl_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:light_kernel -s 3 -c 1 -o gpurun_out/plight -f python bench.py --config dna --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-timing > gpurun_out/pl_ncu.log 2>&1
