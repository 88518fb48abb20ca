# Profile pass for profiles/: plain run, launch list, full capture of one DNA step.
TAG=${1:-r01c}
python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-timing > gpurun_out/${TAG}_ncu_list.log 2>&1
ncu --set full --clock-control none --import-source on -c 90 -o gpurun_out/${TAG}_full -f \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-timing > gpurun_out/${TAG}_ncu_full.log 2>&1
echo done > gpurun_out/${TAG}_done
