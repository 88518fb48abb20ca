python bench.py --config dna --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/pgr_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gram_kernel -s 2 -c 2 -o gpurun_out/pgr_gram -f python bench.py --config dna --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-timing > gpurun_out/pgr_ncu.log 2>&1
