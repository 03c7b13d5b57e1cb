"""Row-sharded LSAR sweep: one process per GPU.

Rows of the LSAR window (w = n - p_bar, lsar.cpp:63) are split into
contiguous blocks; rank g owns rows [row0_g, row0_g + w_g) and holds the
series slice y[row0_g .. row0_g + w_g + p_bar) (a p_bar-sample halo).  Per lag
p the only cross-rank traffic is

  * an allgather of each shard's (sum s_{p-1}, sum r_{p-1}^2)  ->  the global
    R_{p-1} = ||r_{p-1}||^2 (lsar.cpp:17-25), every shard's CDF mass and its
    offset (exclusive prefix in rank order);
  * for every CholeskyQR pass, an allreduce (sum) of the K x K Gram of the
    locally resolved sampled rows; every rank then factors the same matrix,
    so phi_p, the pass gates and the next preconditioner agree everywhere.

Sampling (sketch.cpp:20-59) stays the reference's: every rank evaluates the
same counter-RNG uniforms u_t and resolves only the draws whose global CDF
position u_t * S falls in its segment, keeping them in draw order.

The orchestration below is backend-agnostic: `GpuShard` drives the CUDA
kernels through the C ABI (tf_shard_*), and the CPU tests drive the same
loop with a numpy stand-in over gloo (tests/test_shard.py).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _abi
from .api import DataError, Engine, NumericalError, UsageError, derive_seed, _unpack, ptr


def shard_rows(w: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous balanced row blocks: (row0, rows) of `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise UsageError("invalid rank / world size")
    if w < world:
        raise DataError("fewer window rows than shards")
    base, extra = divmod(w, world)
    row0 = rank * base + min(rank, extra)
    return row0, base + (1 if rank < extra else 0)


class LocalComm:
    """world size 1 (no communication)."""
    rank, world = 0, 1

    def allgather(self, x: np.ndarray) -> np.ndarray:
        return np.asarray(x, dtype=np.float64)[None, :]

    def allreduce_sum(self, x: np.ndarray) -> np.ndarray:
        return np.asarray(x, dtype=np.float64)


class TorchComm:
    """torch.distributed collectives (gloo on CPU, nccl on GPU tensors)."""

    def __init__(self, group=None, device=None):
        import torch
        import torch.distributed as dist
        self._dist, self._torch, self._group = dist, torch, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        backend = dist.get_backend(group)
        self._dev = device or (torch.device("cuda", torch.cuda.current_device())
                               if backend == "nccl" else torch.device("cpu"))

    def allgather(self, x: np.ndarray) -> np.ndarray:
        t = self._torch.as_tensor(np.asarray(x, dtype=np.float64), device=self._dev)
        out = [self._torch.empty_like(t) for _ in range(self.world)]
        self._dist.all_gather(out, t, group=self._group)
        return np.stack([o.cpu().numpy() for o in out])

    def allreduce_sum(self, x: np.ndarray) -> np.ndarray:
        t = self._torch.as_tensor(np.asarray(x, dtype=np.float64), device=self._dev).clone()
        self._dist.all_reduce(t, op=self._dist.ReduceOp.SUM, group=self._group)
        return t.cpu().numpy()


class GpuShard:
    """Per-rank device state through tf_shard_* (csrc/engine.cu)."""

    def __init__(self, engine: Engine | None = None, device: int = 0):
        self.eng = engine or Engine(device)
        self._L = _abi.lib()

    def _ok(self, st):
        self.eng._check(st)

    def open(self, y_slice, p_bar: int, c: int, w_local: int):
        y = np.ascontiguousarray(y_slice, dtype=np.float64)
        self._ok(self._L.tf_upload_series(self.eng._ctx, ptr(y), y.size))
        self.eng._series_id = None
        self._ok(self._L.tf_shard_open(self.eng._ctx, int(p_bar), int(c), int(w_local)))

    def pass_(self, q: int, phi, r_prev: float):
        out = np.zeros(2)
        ph = None if q == 0 else np.ascontiguousarray(phi, dtype=np.float64)
        self._ok(self._L.tf_shard_pass(self.eng._ctx, int(q), ptr(ph) if ph is not None else None,
                                       float(r_prev), ptr(out)))
        return float(out[0]), float(out[1])

    def sample(self, seed_p: int, s_total: float, offset: float, r_glob: float, is_last: bool) -> int:
        k = C.c_int64(0)
        self._ok(self._L.tf_shard_sample(self.eng._ctx, C.c_uint64(seed_p), float(s_total), float(offset),
                                         float(r_glob), int(is_last), C.byref(k)))
        return int(k.value)

    def gram(self, p: int, pass_: int, r_prev: float) -> np.ndarray:
        g = np.zeros(int(self._L.tf_tpu_size(p + 1)))
        self._ok(self._L.tf_shard_gram(self.eng._ctx, int(p), int(pass_), float(r_prev), ptr(g)))
        return g

    def factor(self, p: int, pass_: int, G: np.ndarray, c_total: int):
        fl = np.zeros(3, np.int32)
        g = np.ascontiguousarray(G, dtype=np.float64)
        self._ok(self._L.tf_shard_factor(self.eng._ctx, int(p), int(pass_), ptr(g), int(c_total),
                                         ptr(fl, _abi._i32p)))
        return [int(v) for v in fl]

    def finish(self, p: int):
        phi = np.zeros(p)
        tau = np.zeros(1)
        self._ok(self._L.tf_shard_finish(self.eng._ctx, int(p), ptr(phi), ptr(tau)))
        return phi, float(tau[0])


@dataclass
class ShardFit:
    taus: np.ndarray
    coefs: list
    p_star: int
    local_draws: list  # per lag: number of draws this rank resolved
    row0: int
    rows: int


def lsar_fit_sharded(y, p_bar: int, c: int, seed: int, comm=None, backend=None) -> ShardFit:
    """lsar.cpp:100-124 over row-sharded shards (every rank passes the full
    series y -- or at least its slice -- and gets the same result)."""
    comm = comm or LocalComm()
    backend = backend or GpuShard()
    y = np.asarray(y, dtype=np.float64)
    n = y.size
    if p_bar < 1:
        raise UsageError("maximum lag must be at least 1")
    if n <= p_bar + 1:
        raise DataError(f"series too short for maximum lag {p_bar}")
    if c < p_bar:
        raise UsageError("sample count below maximum lag")
    w = n - p_bar
    row0, wl = shard_rows(w, comm.world, comm.rank)
    backend.open(y[row0:row0 + wl + p_bar], p_bar, c, wl)
    a, b = backend.pass_(0, None, 1.0)
    taus = np.zeros(p_bar)
    coefs = np.zeros(p_bar * (p_bar + 1) // 2)
    draws = []
    off_c = 0
    for p in range(1, p_bar + 1):
        ab = comm.allgather(np.array([a, b]))
        R = float(np.sum(ab[:, 1]))  # rank order: fixed
        if not R > 0.0:
            raise NumericalError("all-zero window; leverage undefined (lag 1)" if p == 1 else
                                 f"zero residual norm; sampling distribution undefined (lag {p})")
        mass = ab[:, 0] + ab[:, 1] / R
        S = float(np.sum(mass))
        offset = float(np.sum(mass[:comm.rank]))
        k = backend.sample(derive_seed(seed, p), S, offset, R, comm.rank == comm.world - 1)
        draws.append(k)
        G = comm.allreduce_sum(backend.gram(p, 0, R))
        fl = backend.factor(p, 0, G, c)
        if p >= 2 and fl[2]:
            G = comm.allreduce_sum(backend.gram(p, 1, R))
            backend.factor(p, 1, G, c)
        if p >= 2 and fl[0]:
            G = comm.allreduce_sum(backend.gram(p, 2, R))
            backend.factor(p, 2, G, c)
        phi, tau = backend.finish(p)
        taus[p - 1] = tau
        coefs[off_c:off_c + p] = phi
        off_c += p
        a, b = backend.pass_(p, phi, R)
    bound = 1.96 / np.sqrt(float(c))
    p_star = 0
    for h in range(p_bar, 0, -1):  # toeplitz.cpp:133-138
        if abs(taus[h - 1]) >= bound:
            p_star = h
            break
    return ShardFit(taus=taus, coefs=_unpack(coefs, p_bar), p_star=p_star, local_draws=draws,
                    row0=row0, rows=wl)
