python bench.py --config dna --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/pg4_plain.log 2>&1 && \
bash tools/prof_list.sh lg4 --config dna && \
ncu --set full --clock-control none --import-source on -k regex:gram4 -s 4 -c 1 -o gpurun_out/pg4big -f python bench.py --config dna --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-timing > gpurun_out/pg4_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:build_dense -s 5 -c 1 -o gpurun_out/pbd -f python bench.py --config dna --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-timing > gpurun_out/pbd_ncu.log 2>&1
