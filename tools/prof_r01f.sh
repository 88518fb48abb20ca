# r01f evidence: DNA bench line (clocks), big-level ncu capture (DNA), trie-pass capture (Text)
O=gpurun_out
timeout 600 python bench.py > $O/r01g_bench_dna.json 2> $O/r01g_bench_dna.err
timeout 900 ncu --set full --clock-control none --import-source on \
  -k 'regex:gram4_kernel|light_kernel|radix_scatter2|radix_hist|segment_kernel|encode_win|build_dense3|epilogue_kernel' \
  -s 44 -c 18 -o $O/r01g_dna_big -f python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-timing > $O/r01g_ncu_dna.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k 'regex:radix_scatter2|radix_hist|hist_scan|segment_kernel|light_kernel' \
  -s 300 -c 8 -o $O/r01g_text -f python bench.py --config text --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-timing > $O/r01g_ncu_text.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
  --log-file $O/r01g_text_launches.csv python bench.py --config text --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-timing > $O/r01g_text_launch.log 2>&1
echo done > $O/r01g_done
