"""Thin ctypes binding of libgakco.so (include/gakco.h): argument marshalling only.

Every step of the path runs in the CUDA library; this module only converts
pointers, sizes and status codes. There is no CPU fallback: if libgakco.so is
missing or CUDA is unavailable the calls raise.

Function names follow the C-ABI: gakco_create, gakco_set_shard, gakco_set_option,
gakco_accumulate, gakco_finalize, gakco_kernel, gakco_get_stats, gakco_num_masks,
gakco_last_error, gakco_destroy. `Plan` wraps a plan handle; `kernel_matrix` is
the one-call convenience used by the tests, smoke() and bench.py.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# (GAKCO_LIB selects another build of the same library, e.g. the bounds-checked one)
LIB_PATH = os.environ.get("GAKCO_LIB") or os.path.join(_PKG, "libgakco.so")

GAKCO_OK = 0
GAKCO_E_ARG = 1
GAKCO_E_SYMBOL = 2
GAKCO_E_RANGE = 3
GAKCO_E_NOMEM = 4
GAKCO_E_CUDA = 5
GAKCO_E_INTERNAL = 6

GAKCO_OPT_HEAVY_MIN_SEQS = 1
GAKCO_OPT_BATCH_KEYS = 2
GAKCO_OPT_TIMING = 3
GAKCO_OPT_SORT = 4
GAKCO_OPT_SORT_CTAS_PER_SM = 5
GAKCO_OPT_LIGHT_BINS = 6
GAKCO_OPT_GRAM_PAIR = 7
GAKCO_OPT_LIGHT_FLAT = 8
GAKCO_OPT_LIGHT_RELABEL = 9
GAKCO_OPT_GRAM_FP4 = 10
GAKCO_OPT_PIPELINE = 11
GAKCO_OPT_LEVEL_ORDER = 12
GAKCO_OPT_LIGHT_WINDOW = 13
GAKCO_OPT_WINDOW_MIN = 14
GAKCO_OPT_GRAM_EACH = 15
GAKCO_OPT_TRIE_PASS = 16
GAKCO_OPT_FAR_NEAR = 17
GAKCO_OPT_XL_COMPACT = 18
GAKCO_OPT_LIGHT_CTAS = 19
GAKCO_OPT_LIGHT_GRID = 20
GAKCO_OPT_FAR_BYTES = 21
GAKCO_OPT_RELABEL_HOST = 22
GAKCO_OPT_LEAF_FUSE = 23

EXPORTS = ("gakco_create", "gakco_set_shard", "gakco_set_option", "gakco_accumulate",
           "gakco_finalize", "gakco_kernel", "gakco_kernel_k", "gakco_kernel_rect",
           "gakco_get_stats", "gakco_stream_wait_level", "gakco_level_order", "gakco_pack_upper",
           "gakco_diag", "gakco_finalize_packed", "gakco_finalize_packed_sum", "gakco_ipc_alloc",
           "gakco_ipc_free", "gakco_ipc_handle", "gakco_ipc_open", "gakco_ipc_close",
           "gakco_pack_upper_peers", "gakco_stage_timeline", "gakco_zero_upper",
           "gakco_num_masks", "gakco_last_error", "gakco_status_string", "gakco_destroy")


class gakco_stats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in (
        "masks", "keys", "sort_passes", "triples", "groups_multi", "light_pairs",
        "heavy_groups", "heavy_macs", "launches")] + [(n, ctypes.c_double) for n in (
            "ms_encode", "ms_sort", "ms_segment", "ms_light", "ms_heavy", "ms_epilogue")] + [
        (n, ctypes.c_int64) for n in (
            "n_encode", "n_sort", "n_segment", "n_light", "n_heavy", "n_epilogue", "keys32",
            "sort_passes32", "grouping")] + [("ms_dense", ctypes.c_double)] + [
        (n, ctypes.c_int64) for n in ("n_dense", "n_pad", "gram_fp4", "heavy_macs_fp4",
                                        "win_groups", "win_macs", "far_records")] + [
        ("ms_far", ctypes.c_double), ("n_far", ctypes.c_int64), ("pass_keys", ctypes.c_int64),
        ("far_overflow", ctypes.c_int64), ("ms_host", ctypes.c_double)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


class GakcoError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"gakco status {status}: {msg}")
        self.status = status


_lib = None


def lib():
    """Load libgakco.so (raises if it was not built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run `python -m paper_1704_07468_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        P, i64, ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        L.gakco_create.argtypes = [ci, ci, ci, ci, ci, ctypes.POINTER(P)]
        L.gakco_set_shard.argtypes = [P, ci, ci]
        L.gakco_set_option.argtypes = [P, ci, i64]
        L.gakco_accumulate.argtypes = [P, P, P, i64, P, P]
        L.gakco_finalize.argtypes = [P, P, i64, P, P, P, P]
        L.gakco_kernel.argtypes = [P, P, P, i64, P, P, P, P, P]
        L.gakco_kernel_k.argtypes = [P, P, P, i64, P, P, P]
        L.gakco_kernel_rect.argtypes = [P, P, P, i64, i64, P, P, P, P, P, P]
        L.gakco_get_stats.argtypes = [P, ctypes.POINTER(gakco_stats)]
        L.gakco_stage_timeline.argtypes = [P, P, P, P, i64, ctypes.POINTER(i64)]
        L.gakco_zero_upper.argtypes = [P, P, i64, ci, P]
        L.gakco_stream_wait_level.argtypes = [P, ci, P]
        L.gakco_level_order.argtypes = [P, ctypes.POINTER(ci), ci]
        L.gakco_level_order.restype = ci
        L.gakco_pack_upper.argtypes = [P, P, i64, ci, i64, i64, P, ci, P]
        L.gakco_diag.argtypes = [P, P, i64, ci, P, P]
        L.gakco_finalize_packed.argtypes = [P, P, ci, i64, i64, i64, i64, P, P, P, P, P]
        L.gakco_finalize_packed_sum.argtypes = [P, P, ci, ci, i64, i64, i64, i64, P, P, P, P, P]
        L.gakco_ipc_alloc.argtypes = [ctypes.c_size_t, ci, ctypes.POINTER(P), P]
        L.gakco_ipc_free.argtypes = [P]
        L.gakco_ipc_handle.argtypes = [P, P]
        L.gakco_ipc_open.argtypes = [P, ci, ctypes.POINTER(P)]
        L.gakco_ipc_close.argtypes = [P]
        L.gakco_pack_upper_peers.argtypes = [P, P, i64, ci, ci, i64, ctypes.POINTER(P), ci, ci, ci, P]
        L.gakco_num_masks.argtypes = [P, ci]
        L.gakco_num_masks.restype = i64
        L.gakco_last_error.argtypes = [P]
        L.gakco_last_error.restype = ctypes.c_char_p
        L.gakco_status_string.argtypes = [ci]
        L.gakco_status_string.restype = ctypes.c_char_p
        L.gakco_destroy.argtypes = [P]
        L.gakco_destroy.restype = None
        for f in ("gakco_create", "gakco_set_shard", "gakco_set_option", "gakco_accumulate",
                  "gakco_finalize", "gakco_kernel", "gakco_kernel_k", "gakco_kernel_rect",
                  "gakco_get_stats", "gakco_stream_wait_level", "gakco_pack_upper",
                  "gakco_diag", "gakco_finalize_packed", "gakco_finalize_packed_sum",
                  "gakco_ipc_alloc", "gakco_ipc_free", "gakco_ipc_handle", "gakco_ipc_open",
                  "gakco_ipc_close", "gakco_pack_upper_peers", "gakco_stage_timeline",
                  "gakco_zero_upper"):
            getattr(L, f).restype = ci
        _lib = L
    return _lib


def _ptr(x):
    """Address of a torch tensor (host or device), numpy array, int or None."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    return x.data_ptr()  # torch.Tensor


def _stream(stream):
    if stream is None:
        return None
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream  # torch.cuda.Stream


def gakco_create(sigma, g, k, M, device=0):
    h = ctypes.c_void_p()
    st = lib().gakco_create(sigma, g, k, M, device, ctypes.byref(h))
    if st != GAKCO_OK:
        raise GakcoError(st, lib().gakco_status_string(st).decode())
    return h.value


def gakco_last_error(plan):
    return lib().gakco_last_error(plan).decode()


def _check(plan, st):
    if st != GAKCO_OK:
        raise GakcoError(st, gakco_last_error(plan))


def gakco_set_shard(plan, rank, world):
    _check(plan, lib().gakco_set_shard(plan, rank, world))


def gakco_set_option(plan, option, value):
    _check(plan, lib().gakco_set_option(plan, option, int(value)))


def gakco_accumulate(plan, codes, offsets, N, C, stream=None):
    _check(plan, lib().gakco_accumulate(plan, _ptr(codes), _ptr(offsets), N, _ptr(C),
                                        _stream(stream)))


def gakco_finalize(plan, C, N, Nm=None, K=None, Knorm=None, stream=None):
    _check(plan, lib().gakco_finalize(plan, _ptr(C), N, _ptr(Nm), _ptr(K), _ptr(Knorm),
                                      _stream(stream)))


def gakco_kernel(plan, codes, offsets, N, C=None, Nm=None, K=None, Knorm=None, stream=None):
    _check(plan, lib().gakco_kernel(plan, _ptr(codes), _ptr(offsets), N, _ptr(C), _ptr(Nm),
                                    _ptr(K), _ptr(Knorm), _stream(stream)))


def gakco_kernel_rect(plan, codes, offsets, N, NA, C=None, Nm=None, K=None, Knorm=None,
                      Kdiag=None, stream=None):
    _check(plan, lib().gakco_kernel_rect(plan, _ptr(codes), _ptr(offsets), N, NA, _ptr(C),
                                         _ptr(Nm), _ptr(K), _ptr(Knorm), _ptr(Kdiag),
                                         _stream(stream)))


def gakco_kernel_k(plan, codes, offsets, N, K=None, Knorm=None, stream=None):
    _check(plan, lib().gakco_kernel_k(plan, _ptr(codes), _ptr(offsets), N, _ptr(K), _ptr(Knorm),
                                      _stream(stream)))


def gakco_get_stats(plan):
    s = gakco_stats()
    _check(plan, lib().gakco_get_stats(plan, ctypes.byref(s)))
    return s.as_dict()


def gakco_stage_timeline(plan, cap=100000):
    """(stage, t0 ms, t1 ms) per stage event of the last call (GAKCO_OPT_TIMING)."""
    st = (ctypes.c_int32 * cap)()
    a = (ctypes.c_float * cap)()
    b = (ctypes.c_float * cap)()
    n = ctypes.c_int64(0)
    _check(plan, lib().gakco_stage_timeline(plan, st, a, b, cap, ctypes.byref(n)))
    return [(st[i], a[i], b[i]) for i in range(min(n.value, cap))]


def gakco_stream_wait_level(plan, m, stream=None):
    _check(plan, lib().gakco_stream_wait_level(plan, m, _stream(stream)))


def gakco_level_order(plan):
    buf = (ctypes.c_int * 64)()
    n = lib().gakco_level_order(plan, buf, 64)
    if n < 0:
        raise GakcoError(GAKCO_E_ARG, "null plan")
    return [buf[i] for i in range(min(n, 64))]


def gakco_pack_upper(plan, C, N, levels, begin, end, out, out_bytes, stream=None):
    _check(plan, lib().gakco_pack_upper(plan, _ptr(C), N, levels, begin, end, _ptr(out),
                                        out_bytes, _stream(stream)))


def gakco_diag(plan, C, N, levels, out, stream=None):
    _check(plan, lib().gakco_diag(plan, _ptr(C), N, levels, _ptr(out), _stream(stream)))


def gakco_finalize_packed(plan, Cp, in_bytes, ld, N, begin, end, Cdiag, Nm=None, K=None,
                          Knorm=None, stream=None):
    _check(plan, lib().gakco_finalize_packed(plan, _ptr(Cp), in_bytes, ld, N, begin, end,
                                             _ptr(Cdiag), _ptr(Nm), _ptr(K), _ptr(Knorm),
                                             _stream(stream)))


def gakco_finalize_packed_sum(plan, Cp, in_bytes, nsrc, ld, N, begin, end, Cdiag, Nm=None,
                              K=None, Knorm=None, stream=None):
    _check(plan, lib().gakco_finalize_packed_sum(plan, _ptr(Cp), in_bytes, nsrc, ld, N, begin, end,
                                                 _ptr(Cdiag), _ptr(Nm), _ptr(K), _ptr(Knorm),
                                                 _stream(stream)))


def gakco_pack_upper_peers(plan, Cm, N, level, levels, chunk, dst, P, rank, out_bytes, stream=None):
    arr = (ctypes.c_void_p * P)(*[int(d) for d in dst])
    _check(plan, lib().gakco_pack_upper_peers(plan, _ptr(Cm), N, level, levels, chunk, arr, P,
                                              rank, out_bytes, _stream(stream)))


def _ipc_check(st, what):
    if st != GAKCO_OK:
        raise GakcoError(st, what + ": " + lib().gakco_status_string(st).decode())


def gakco_ipc_alloc(nbytes, device=0):
    """(device pointer, 64-byte IPC handle) of a new cudaMalloc buffer."""
    ptr = ctypes.c_void_p()
    h = ctypes.create_string_buffer(64)
    _ipc_check(lib().gakco_ipc_alloc(nbytes, device, ctypes.byref(ptr), h), "ipc_alloc")
    return ptr.value, h.raw


def gakco_ipc_free(ptr):
    _ipc_check(lib().gakco_ipc_free(ptr), "ipc_free")


def gakco_ipc_open(handle, device=0):
    ptr = ctypes.c_void_p()
    _ipc_check(lib().gakco_ipc_open(ctypes.create_string_buffer(bytes(handle), 64), device,
                                    ctypes.byref(ptr)), "ipc_open")
    return ptr.value


def gakco_ipc_close(ptr):
    _ipc_check(lib().gakco_ipc_close(ptr), "ipc_close")


def gakco_num_masks(plan, shard_only=False):
    return int(lib().gakco_num_masks(plan, 1 if shard_only else 0))


def gakco_destroy(plan):
    lib().gakco_destroy(plan)


class Plan:
    """Owning wrapper of a gakco_plan."""

    def __init__(self, sigma, g, k, M=None, device=0):
        self.sigma, self.g, self.k = sigma, g, k
        self.M = g - k if M is None else M
        self.device = device
        self.h = gakco_create(sigma, g, k, self.M, device)

    def set_shard(self, rank, world):
        gakco_set_shard(self.h, rank, world)

    def set_option(self, option, value):
        gakco_set_option(self.h, option, value)

    def accumulate(self, codes, offsets, N, C, stream=None):
        gakco_accumulate(self.h, codes, offsets, N, C, stream)

    def finalize(self, C, N, Nm=None, K=None, Knorm=None, stream=None):
        gakco_finalize(self.h, C, N, Nm, K, Knorm, stream)

    def kernel(self, codes, offsets, N, C=None, Nm=None, K=None, Knorm=None, stream=None):
        gakco_kernel(self.h, codes, offsets, N, C, Nm, K, Knorm, stream)

    def kernel_k(self, codes, offsets, N, K=None, Knorm=None, stream=None):
        gakco_kernel_k(self.h, codes, offsets, N, K, Knorm, stream)

    def kernel_rect(self, codes, offsets, N, NA, C=None, Nm=None, K=None, Knorm=None,
                    Kdiag=None, stream=None):
        gakco_kernel_rect(self.h, codes, offsets, N, NA, C, Nm, K, Knorm, Kdiag, stream)

    def stats(self):
        return gakco_get_stats(self.h)

    def stage_timeline(self):
        return gakco_stage_timeline(self.h)

    def zero_upper(self, C, N, levels, stream=None):
        """Zero the upper triangles of `levels` N x N int64 matrices (device C)."""
        _check(self.h, lib().gakco_zero_upper(self.h, _ptr(C), N, levels, _stream(stream)))

    def stream_wait_level(self, m, stream=None):
        gakco_stream_wait_level(self.h, m, stream)

    def level_order(self):
        return gakco_level_order(self.h)

    def pack_upper(self, C, N, levels, begin, end, out, out_bytes, stream=None):
        gakco_pack_upper(self.h, C, N, levels, begin, end, out, out_bytes, stream)

    def diag(self, C, N, levels, out, stream=None):
        gakco_diag(self.h, C, N, levels, out, stream)

    def pack_upper_peers(self, Cm, N, level, levels, chunk, dst, P, rank, out_bytes, stream=None):
        gakco_pack_upper_peers(self.h, Cm, N, level, levels, chunk, dst, P, rank, out_bytes, stream)

    def finalize_packed_sum(self, Cp, in_bytes, nsrc, ld, N, begin, end, Cdiag, Nm=None, K=None,
                            Knorm=None, stream=None):
        gakco_finalize_packed_sum(self.h, Cp, in_bytes, nsrc, ld, N, begin, end, Cdiag, Nm, K,
                                  Knorm, stream)

    def finalize_packed(self, Cp, in_bytes, ld, N, begin, end, Cdiag, Nm=None, K=None, Knorm=None,
                        stream=None):
        gakco_finalize_packed(self.h, Cp, in_bytes, ld, N, begin, end, Cdiag, Nm, K, Knorm, stream)

    def num_masks(self, shard_only=False):
        return gakco_num_masks(self.h, shard_only)

    def close(self):
        if self.h:
            gakco_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def kernel_matrix(codes, offsets, sigma, g, k, M=None, device=0, plan=None, outputs=True,
                  stream=None):
    """All outputs on `device` as torch tensors: dict C, Nm, K, Knorm.

    `codes` / `offsets` may be numpy arrays (host) or torch tensors (host/device).
    """
    import torch
    M = g - k if M is None else M
    N = int(offsets.shape[0]) - 1
    dev = torch.device("cuda", device)
    own = plan is None
    plan = plan or Plan(sigma, g, k, M, device)
    try:
        C = torch.zeros((M + 1, N, N), dtype=torch.int64, device=dev)
        Nm = torch.empty((M + 1, N, N), dtype=torch.int64, device=dev) if outputs else None
        K = torch.empty((N, N), dtype=torch.int64, device=dev)
        Kn = torch.empty((N, N), dtype=torch.float64, device=dev) if outputs else None
        codes_c = np.ascontiguousarray(codes, dtype=np.uint8) if isinstance(codes, np.ndarray) else codes
        off_c = np.ascontiguousarray(offsets, dtype=np.int64) if isinstance(offsets, np.ndarray) else offsets
        if isinstance(codes_c, np.ndarray) and codes_c.size == 0:
            codes_c = np.zeros(1, dtype=np.uint8)
        with torch.cuda.device(dev):
            s = stream or torch.cuda.current_stream(dev)
            plan.kernel(codes_c, off_c, N, C, Nm, K, Kn, stream=s)
        return {"C": C, "Nm": Nm, "K": K, "Knorm": Kn}
    finally:
        if own:
            plan.close()


def kernel_matrix_rect(codes, offsets, NA, sigma, g, k, M=None, device=0, plan=None, stream=None):
    """Train x test block (NEXT-2): the corpus holds the NA training sequences, then
    the test sequences. Returns device tensors C, Nm (M+1, NA, NB), K, Knorm (NA, NB)
    and Kdiag (N,)."""
    import torch
    M = g - k if M is None else M
    N = int(offsets.shape[0]) - 1
    NB = N - NA
    dev = torch.device("cuda", device)
    own = plan is None
    plan = plan or Plan(sigma, g, k, M, device)
    try:
        C = torch.empty((M + 1, NA, NB), dtype=torch.int64, device=dev)
        Nm = torch.empty((M + 1, NA, NB), dtype=torch.int64, device=dev)
        K = torch.empty((NA, NB), dtype=torch.int64, device=dev)
        Kn = torch.empty((NA, NB), dtype=torch.float64, device=dev)
        Kd = torch.empty((N,), dtype=torch.int64, device=dev)
        codes_c = np.ascontiguousarray(codes, dtype=np.uint8) if isinstance(codes, np.ndarray) else codes
        off_c = np.ascontiguousarray(offsets, dtype=np.int64) if isinstance(offsets, np.ndarray) else offsets
        if isinstance(codes_c, np.ndarray) and codes_c.size == 0:
            codes_c = np.zeros(1, dtype=np.uint8)
        with torch.cuda.device(dev):
            s = stream or torch.cuda.current_stream(dev)
            plan.kernel_rect(codes_c, off_c, N, NA, C, Nm, K, Kn, Kd, stream=s)
        return {"C": C, "Nm": Nm, "K": K, "Knorm": Kn, "Kdiag": Kd}
    finally:
        if own:
            plan.close()
