python bench.py --config text --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ps_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:radix_scatter -s 30 -c 1 -o gpurun_out/psort -f python bench.py --config text --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-timing > gpurun_out/ps_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:segment_kernel -s 10 -c 1 -o gpurun_out/pseg -f python bench.py --config text --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-timing > gpurun_out/ps_ncu2.log 2>&1
