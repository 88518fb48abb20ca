# ncu capture of segment + encode_win on Text (one launch each, mid-step)
ARGS=${ARGS:---config text}
ncu --set full --clock-control none --import-source on -k regex:segment_kernel -s 20 -c 1 \
  -o gpurun_out/pseg2 -f python bench.py $ARGS --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-timing \
  > gpurun_out/pseg2_ncu.log 2>&1
echo done > gpurun_out/pseg2_done
