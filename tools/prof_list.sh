# launch list (per-kernel device time) of one bench step: prof_list.sh TAG "bench args"
TAG=$1; shift
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e "$@" > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-timing "$@" > gpurun_out/${TAG}_ncu.log 2>&1
