"""Measure the ceilings the roofline needs beyond MEASURED_PEAKS.json (B200 box).

  python tools/measure_peaks.py [--out profiles/peaks_r02.json]

* random u32 RED throughput (the light path's limiter) into an L2-resident
  (32 MB, DNA's accumulator) and a DRAM-resident (800 MB, Scale's triangle)
  array, fully random cells and 32-cell row segments (tools/micro.cu);
* int8 dense GEMM throughput through cuBLASLt (torch._int_mm, 8192^3), the
  library reference for the heavy Gram's kind::i8 peak;
* e2m1 (fp4) block-scaled GEMM through torch._scaled_mm where this torch build
  supports it (else recorded as unavailable).
Each number is the best of several CUDA-event-timed repetitions.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libmicro.so")


def build():
    src = os.path.join(HERE, "micro.cu")
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(src):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-O3", "-gencode",
                               "arch=compute_100a,code=sm_100a", "-Xcompiler", "-fPIC",
                               "-shared", "-o", LIB, src])
    return ctypes.CDLL(LIB)


def timed(fn, reps=10):
    best = float("inf")
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best / 1e3


def red(lib, mbytes, rowseg):
    cells = mbytes * (1 << 20) // 4
    acc = torch.zeros(cells, dtype=torch.int32, device="cuda")
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    blocks, threads, per = sms * 16, 256, 256
    s = torch.cuda.current_stream().cuda_stream
    lib.micro_red.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
                              ctypes.c_int, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p]
    seed = [1]

    def run():
        seed[0] += 1
        rc = lib.micro_red(acc.data_ptr(), cells, blocks, threads, per, seed[0], int(rowseg), s)
        assert rc == 0, rc
    run()
    t = timed(run)
    upd = blocks * threads * per
    return {"array_MB": mbytes, "pattern": "32-cell row segments" if rowseg else "random cells",
            "updates": upd, "seconds": t, "G_updates_per_s": upd / t / 1e9}


def int8_gemm(n=8192):
    a = torch.randint(-64, 64, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-64, 64, (n, n), dtype=torch.int8, device="cuda").t()
    t = timed(lambda: torch._int_mm(a, b))
    return {"shape": [n, n, n], "seconds": t, "TOPS": 2 * n ** 3 / t / 1e12,
            "how": "torch._int_mm (cuBLASLt int8 -> int32), best of 10"}


def fp4_gemm(n=8192):
    try:
        fp4 = torch.float4_e2m1fn_x2
        a = torch.randint(0, 256, (n, n // 2), dtype=torch.uint8, device="cuda").view(fp4)
        b = torch.randint(0, 256, (n, n // 2), dtype=torch.uint8, device="cuda").view(fp4)
        sa = torch.ones((n, n // 16), dtype=torch.float8_e4m3fn, device="cuda")
        sb = torch.ones((n, n // 16), dtype=torch.float8_e4m3fn, device="cuda")
        f = lambda: torch._scaled_mm(a, b.t(), sa, sb, out_dtype=torch.bfloat16)  # noqa: E731
        f()
        t = timed(f)
        return {"shape": [n, n, n], "seconds": t, "TFLOPS": 2 * n ** 3 / t / 1e12,
                "how": "torch._scaled_mm nvfp4 (e2m1, e4m3 block-16 scales), best of 10"}
    except Exception as e:  # noqa: BLE001
        return {"unavailable": f"{type(e).__name__}: {str(e)[:200]}"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "peaks_r02.json"))
    a = ap.parse_args()
    lib = build()
    out = {"gpu": torch.cuda.get_device_name(0),
           "red": [red(lib, mb, rs) for mb in (32, 800) for rs in (False, True)],
           "int8_gemm": int8_gemm(), "fp4_gemm": fp4_gemm()}
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    sys.exit(main())
