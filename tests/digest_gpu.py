"""The order-independent matrix digest of oracle/make_digests.py, evaluated with
torch on the device so that full-size GPU outputs (Scale: 45 GB) are compared
with the committed oracle digests without a host copy. Test infrastructure only;
pinned to the numpy restatement (tests/refs.digest_np) by
test_gpu_parity.py::test_digest_gpu_matches_numpy.

  H = sum over entries of mix(idx ^ mix(bits)) mod 2^64, idx = flat index,
  mix = the splitmix64 finaliser; evaluated in int64 (two's-complement wrap of
  the products and the sum gives the same bits as uint64; shifts are made logical
  by masking).
"""
from __future__ import annotations

import torch

_M1 = 0xbf58476d1ce4e5b9 - (1 << 64)
_M2 = 0x94d049bb133111eb - (1 << 64)


def _srl(z, s):
    return (z >> s) & ((1 << (64 - s)) - 1)


def _mix(z):
    z = (z ^ _srl(z, 30)) * _M1
    z = (z ^ _srl(z, 27)) * _M2
    return z ^ _srl(z, 31)


def digest_torch(t: torch.Tensor, chunk: int = 1 << 26) -> int:
    """Digest of a (device) int64 / float64 tensor's bits, flat row-major index."""
    flat = t.contiguous().view(torch.int64).reshape(-1)
    total = torch.zeros((), dtype=torch.int64, device=flat.device)
    for i0 in range(0, flat.numel(), chunk):
        blk = flat[i0:i0 + chunk]
        idx = torch.arange(i0, i0 + blk.numel(), dtype=torch.int64, device=flat.device)
        total += _mix(idx ^ _mix(blk)).sum()
    return int(total.item()) & ((1 << 64) - 1)
