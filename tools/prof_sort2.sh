# ncu capture of the v2 LSD pass kernels on Text (one launch each, mid-step)
ARGS=${ARGS:---config text --sort 3}
ncu --set full --clock-control none --import-source on -k 'regex:radix_scatter2|radix_hist' -s 40 -c 2 \
  -o gpurun_out/psort2 -f python bench.py $ARGS --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-timing \
  > gpurun_out/psort2_ncu.log 2>&1
echo done > gpurun_out/psort2_done
