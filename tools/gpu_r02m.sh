#!/bin/bash
# r02 pass m: the driver's commands (bench default + reference arm), tests, D2H bandwidth
O=gpurun_out; T=${1:-r02m}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${T}_smoke.log
timeout 900 python bench.py > $O/${T}_bench_default.json 2> $O/${T}_bench_default.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/${T}_bench_ref.json 2> $O/${T}_bench_ref.err
python - > $O/${T}_d2h.log 2>&1 <<'PY'
import torch, time
d = torch.empty(200_000_000, dtype=torch.int64, device="cuda")
h = torch.empty(200_000_000, dtype=torch.int64).pin_memory()
for i in range(3):
    torch.cuda.synchronize(); t = time.perf_counter(); h.copy_(d, non_blocking=True); torch.cuda.synchronize()
    print("d2h GB/s", 1.6e9 / (time.perf_counter() - t))
    torch.cuda.synchronize(); t = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize()
    print("h2d GB/s", 1.6e9 / (time.perf_counter() - t))
PY
echo done > $O/${T}_done
