python bench.py --config dna --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/pg2_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gram2 -s 4 -c 1 -o gpurun_out/pg2big -f python bench.py --config dna --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-timing > gpurun_out/pg2_ncu.log 2>&1
