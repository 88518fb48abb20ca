bash tools/gpu_sweep.sh e1 "dna:;dna:--heavy-min 25;dna:--heavy-min 50;dna:--heavy-min 70;protein:;protein:--heavy-min 20;protein:--heavy-min 60" ""
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/e1_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/e1_pytest.log
