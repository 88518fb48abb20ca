# ncu capture of one late-level light launch (and the window build / Gram) on Scale
O=gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k 'regex:light_kernel|window_build|gram_kernel' -s 150 -c 3 \
  -o $O/plscale -f python bench.py --config scale --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-timing > $O/plscale.log 2>&1
echo done > $O/plscale_done
