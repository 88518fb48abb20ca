"""Mask-sharded multi-GPU orchestration (one process per GPU).

The C(g,m) masks are independent (Supp. §S:5.3) and C_m is an
integer sum over masks (Algorithm 1 line 17). Rank r of P processes
the masks whose global index (level by level m = 0..M, lexicographic within a
level) is congruent to r mod P — the rule gakco_set_shard implements in
libgakco.so — into its own zeroed C. Then (ShardedStep.step):

  * as each level's C_m becomes final on the device (gakco_stream_wait_level, no
    host sync), a comm stream packs its upper triangle (gakco_pack_upper: the only
    part gakco_accumulate writes, e(X,Y) = X N - X(X-1)/2 + (Y-X)) into 32-bit
    words when the summed value is bounded below 2^31, else int64, and reduce-
    scatters it over the process group (NCCL over NVLink on B200s): rank r receives
    the complete C_m of packed entries [r*chunk, (r+1)*chunk). The reduces of early
    levels overlap the accumulation of later ones;
  * the diagonals C_m(X,X) (gakco_diag, (M+1) x N int64) are all-reduced, since
    Knorm needs K(X,X) of every sequence;
  * every rank runs the epilogue (Eq. 9, Eq. 7, normalisation) on its own slice
    (gakco_finalize_packed): the outputs C, N_m, K, Knorm end sharded over the
    ranks as packed upper-triangle slices (symmetric matrices, reading A4).

Nothing here computes the method: every step runs in libgakco.so; this module
only moves buffers between the library and torch.distributed. With the gloo
backend (CPU tests) the collectives are staged through host memory.
"""
from __future__ import annotations

import contextlib
import os
import socket
import subprocess
import sys
from itertools import combinations
from math import comb


def masks(g: int, M: int):
    """Global mask order: (m, removed positions) for m = 0..M, lexicographic."""
    out = []
    for m in range(M + 1):
        out.extend((m, rem) for rem in combinations(range(g), m))
    return out


def shard_masks(g: int, M: int, rank: int, world: int):
    """Masks of rank `rank` of `world` (global index = rank mod world)."""
    return [mk for i, mk in enumerate(masks(g, M)) if i % world == rank]


def tri_size(N: int) -> int:
    """Entries of the packed upper triangle (diagonal included)."""
    return N * (N + 1) // 2


def tri_slice(N: int, rank: int, world: int):
    """(chunk, begin, end): rank's part of the packed triangle, chunk = ceil(T/world)."""
    T = tri_size(N)
    chunk = -(-T // world)
    b = min(T, rank * chunk)
    return chunk, b, min(T, b + chunk)


def word_bytes(g: int, M: int, nmax: int) -> int:
    """4 when every complete C_m(X,Y) <= C(g,m) n_max^2 stays below 2^31, else 8."""
    return 4 if all(comb(g, m) * nmax * nmax < 2 ** 31 for m in range(M + 1)) else 8


def tri_index(X, Y, N):
    """Packed index of (X, Y), X <= Y (numpy arrays or ints)."""
    return X * N - X * (X - 1) // 2 + (Y - X)


class ShardedStep:
    """One step of the mask-sharded path on this rank.

    plan: gakco.Plan (or a test double with the same methods) with set_shard(rank,
    world) applied. C: this rank's (M+1, N, N) int64 accumulator. After step()
    the rank's slice [begin, end) of the packed triangle is in Cp (complete C_m,
    word_bytes wide), Nm (M+1, chunk), K (chunk,), Knorm (chunk,).
    """

    def __init__(self, plan, N, g, k, M, nmax, device, group=None, backend=None,
                 outputs=True, exchange="auto"):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.plan, self.N, self.g, self.k, self.M = plan, N, g, k, M
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.backend = backend or (dist.get_backend(group) if dist.is_initialized() else "none")
        self.dev = torch.device(device)
        self.cuda = self.dev.type == "cuda"
        self.T = tri_size(N)
        self.chunk, self.begin, self.end = tri_slice(N, self.rank, self.world)
        self.wb = word_bytes(g, M, nmax)
        wdt = torch.int32 if self.wb == 4 else torch.int64
        L = M + 1
        # per-level packed buffers (zero pad past T), the reduced slice, diagonals
        self.pack = torch.zeros((L, self.chunk * self.world), dtype=wdt, device=self.dev)
        self.Cp = torch.zeros((L, self.chunk), dtype=wdt, device=self.dev)
        self.D = torch.zeros((L, N), dtype=torch.int64, device=self.dev)
        self.Nm = torch.empty((L, self.chunk), dtype=torch.int64, device=self.dev) if outputs else None
        self.K = torch.empty((self.chunk,), dtype=torch.int64, device=self.dev)
        self.Knorm = torch.empty((self.chunk,), dtype=torch.float64, device=self.dev) if outputs else None
        self.comm = torch.cuda.Stream(self.dev) if self.cuda else None
        # exchange: "p2p" = pack fused with the transfer over peer memory (CUDA IPC:
        # gakco_pack_upper_peers into the owners' receive buffers, the P contributions
        # summed inside gakco_finalize_packed_sum); "collective" = pack + reduce-scatter
        self.exchange = "collective"
        self._ipc_own, self._ipc_open = [], []
        if exchange in ("auto", "p2p") and self.cuda and self.world > 1 and \
                hasattr(plan, "pack_upper_peers"):
            try:
                self._setup_p2p()
                self.exchange = "p2p"
            except Exception:  # noqa: BLE001  (no IPC / peer access: the collective path)
                if exchange == "p2p":
                    raise
                self.close()
        self.parity = 0

    def _setup_p2p(self):
        from paper_1704_07468_b200 import gakco
        L, P = self.M + 1, self.world
        nbytes = P * L * self.chunk * self.wb
        dev = self.dev.index or 0
        mine = []
        for _ in range(2):  # two buffers: a step's packs never overwrite what a slower
            ptr, h = gakco.gakco_ipc_alloc(nbytes, dev)  # peer is still reading
            self._ipc_own.append(ptr)
            mine.append(h)
        allh = [None] * P
        self.dist.all_gather_object(allh, mine, group=self.group)
        self.dst = [[0] * P for _ in range(2)]
        for q in range(2):
            for d in range(P):
                if d == self.rank:
                    self.dst[q][d] = self._ipc_own[q]
                else:
                    ptr = gakco.gakco_ipc_open(allh[d][q], dev)
                    self._ipc_open.append(ptr)
                    self.dst[q][d] = ptr

    def close(self):
        """Release the peer mappings and receive buffers of the p2p exchange."""
        from paper_1704_07468_b200 import gakco
        for ptr in self._ipc_open:
            try:
                gakco.gakco_ipc_close(ptr)
            except Exception:  # noqa: BLE001
                pass
        for ptr in self._ipc_own:
            try:
                gakco.gakco_ipc_free(ptr)
            except Exception:  # noqa: BLE001
                pass
        self._ipc_open, self._ipc_own = [], []

    # -- collectives (NCCL on the device; gloo through host memory)
    def _reduce_scatter(self, out, inp):
        if self.world == 1:
            out.copy_(inp[: self.chunk])
        elif self.backend == "nccl":
            self.dist.reduce_scatter_tensor(out, inp, group=self.group)
        else:
            t = inp.cpu()
            self.dist.all_reduce(t, group=self.group)
            out.copy_(t[self.rank * self.chunk:(self.rank + 1) * self.chunk])

    def _all_reduce(self, t):
        if self.world == 1:
            return
        if self.backend == "nccl":
            self.dist.all_reduce(t, group=self.group)
        else:
            h = t.cpu()
            self.dist.all_reduce(h, group=self.group)
            t.copy_(h)

    def _nvtx(self, name):
        return self.torch.cuda.nvtx.range(name) if self.cuda else contextlib.nullcontext()

    def _on_comm(self):
        return self.torch.cuda.stream(self.comm) if self.cuda else contextlib.nullcontext()

    def step(self, codes, offsets, C, stream=None):
        """accumulate (this rank's masks) -> per-level pack + reduce-scatter (comm
        stream, overlapping later levels) -> diagonal all-reduce -> slice epilogue."""
        plan, N, L = self.plan, self.N, self.M + 1
        plan.zero_upper(C, N, L, stream)  # (accumulate adds into the upper triangles)
        plan.accumulate(codes, offsets, N, C, stream)
        cs = self.comm
        if self.exchange == "p2p":
            return self._step_p2p(C, stream)
        with self._on_comm(), self._nvtx("sharded exchange + slice epilogue"):
            for m in plan.level_order():
                plan.stream_wait_level(m, cs)
                plan.pack_upper(C[m], N, 1, 0, self.T, self.pack[m], self.wb, cs)
                self._reduce_scatter(self.Cp[m], self.pack[m])
            plan.diag(C, N, L, self.D, cs)
            self._all_reduce(self.D)
            plan.finalize_packed(self.Cp, self.wb, self.chunk, N, self.begin, self.end, self.D,
                                 self.Nm, self.K, self.Knorm, cs)
        if self.cuda:
            (stream or self.torch.cuda.current_stream(self.dev)).wait_stream(cs)
        return self.begin, self.end

    def _step_p2p(self, C, stream):
        plan, N, L, P, cs = self.plan, self.N, self.M + 1, self.world, self.comm
        q = self.parity
        with self._on_comm(), self._nvtx("p2p exchange + slice epilogue"):
            for m in plan.level_order():  # each level straight into its owners' buffers
                plan.stream_wait_level(m, cs)
                plan.pack_upper_peers(C[m], N, m, L, self.chunk, self.dst[q], P, self.rank,
                                      self.wb, cs)
            plan.diag(C, N, L, self.D, cs)
            self._all_reduce(self.D)
        cs.synchronize()      # this rank's writes into every owner are complete ...
        self.dist.barrier(group=self.group)  # ... and every other rank's into ours
        with self._on_comm():
            plan.finalize_packed_sum(self._ipc_own[q], self.wb, P, self.chunk, N, self.begin,
                                     self.end, self.D, self.Nm, self.K, self.Knorm, cs)
        (stream or self.torch.cuda.current_stream(self.dev)).wait_stream(cs)
        self.parity ^= 1
        return self.begin, self.end

    def complete_C(self):
        """This rank's slice of the complete C (M+1, end - begin) on the device (for the
        p2p exchange the sum of the receive buffer's contributions)."""
        cnt = self.end - self.begin
        if self.exchange != "p2p":
            return self.Cp[:, :cnt].long()
        from paper_1704_07468_b200 import gakco  # noqa: F401
        wdt = self.torch.int32 if self.wb == 4 else self.torch.int64
        q = self.parity ^ 1  # the buffer of the last step
        nel = self.world * (self.M + 1) * self.chunk
        buf = _tensor_from_ptr(self.torch, self._ipc_own[q], nel, wdt, self.dev)
        return buf.view(self.world, self.M + 1, self.chunk)[:, :, :cnt].long().sum(0)


def _tensor_from_ptr(torch, ptr, nel, dtype, dev):
    """A torch view of device memory owned by libgakco (test / inspection only)."""
    class _Arr:
        pass
    a = _Arr()
    a.__cuda_array_interface__ = {"shape": (nel,), "typestr": "<i4" if dtype == torch.int32 else "<i8",
                                  "data": (ptr, False), "version": 3}
    return torch.as_tensor(a, device=dev)


# ------------------------------------------------------------------ launcher
def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def launch(nprocs: int, script: str, args, env=None) -> int:
    """Run `script args` as nprocs ranks of one node under torch.distributed.run
    (rendezvous on 127.0.0.1); returns the exit code. bench.py re-launches itself
    through this when --gpus N > 1 is given without a torchrun environment."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nprocs}", "--master-addr=127.0.0.1",
           f"--master-port={free_port()}", script] + list(args)
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.call(cmd, env=e)
