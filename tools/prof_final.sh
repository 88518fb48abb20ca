# Profile pass for profiles/: plain run, launch list, full capture of the main kernels of one DNA step.
TAG=${1:-r01c}
python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-timing > gpurun_out/${TAG}_ncu_list.log 2>&1
ncu --set full --clock-control none --import-source on \
  -k 'regex:gram4_kernel|light_kernel|radix_scatter|segment_kernel|encode_win|build_dense3|epilogue_kernel' \
  -s ${SKIP:-0} -c 16 -o gpurun_out/${TAG}_full -f \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-timing > gpurun_out/${TAG}_ncu_full.log 2>&1
ls -la gpurun_out/ > gpurun_out/${TAG}_ls.txt
echo done > gpurun_out/${TAG}_done
