"""Row-sharded LSAR sweep of one long series: one process per GPU.

Rows of the LSAR window (w = n - p_bar, lsar.cpp:63) are split into
contiguous balanced blocks; rank g owns rows [row0_g, row0_g + w_g) and holds
the series slice y[row0_g .. row0_g + w_g + p_bar) (a p_bar-sample halo).  Per
lag p the only cross-rank traffic is

  * an allgather of each shard's (sum s_{p-1}, sum r_{p-1}^2)  ->  the global
    R_{p-1} = ||r_{p-1}||^2 (lsar.cpp:17-25);
  * an allgather of each shard's local CDF total (built with the global R)
    -> the global total and this shard's segment [lo, hi) (prefix in rank
    order);
  * an allgather of the shards' double-double Gram partials of their sampled
    rows, summed in rank order, so every rank runs the same rank-revealing
    solve (toeplitz.cpp:57-85) and holds the same phi_p.

Sampling (sketch.cpp:20-59) stays the reference's: every rank evaluates the
same counter-RNG uniforms u_t and resolves only the draws with
lo <= u_t S < hi (compared against the prefix values themselves, so each draw
lands in exactly one shard), keeping them in draw order.

`NcclShard` is the product path: the lag loop runs inside libtoepfit_b200.so
(tf_lsar_sweep_sharded) with NCCL on the context stream; torch.distributed
only carries the NCCL unique id.  `lsar_fit_sharded` restates the same
protocol in Python over any `comm` (gloo on CPU in tests/test_shard.py, with
the numpy stand-in of tests/shard_numpy.py for the per-shard steps): it is
the executable specification the CUDA orchestration follows.
"""
from __future__ import annotations

import ctypes as C
import time
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


def global_R(ab: np.ndarray) -> float:
    """k_shard_R: the global ||r||^2 from the allgathered (sum s, sum r^2), rank order."""
    R = 0.0
    for r in range(ab.shape[0]):
        R += float(ab[r, 1])
    return R


def segment(s_loc: np.ndarray, rank: int) -> tuple[float, float, float]:
    """k_shard_seg: (S, lo, hi) from the allgathered local CDF totals, rank
    order: the global total and this shard's segment [lo, hi) (last: open)."""
    S = lo = hi = 0.0
    for r in range(s_loc.shape[0]):
        if r == rank:
            lo = S
        S += float(s_loc[r])
        if r == rank:
            hi = S
    if rank == s_loc.shape[0] - 1:
        hi = float("inf")
    return S, lo, hi


class LocalComm:
    """world size 1 (no communication)."""
    rank, world = 0, 1

    def allgather(self, x: np.ndarray) -> np.ndarray:
        return np.asarray(x, dtype=np.float64)[None, :]


class TorchComm:
    """torch.distributed collectives (gloo on CPU) for the protocol model."""

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


class NcclShard:
    """This rank's part of a row-sharded sweep on its GPU (product path)."""

    def __init__(self, engine: Engine, dist, world: int, rank: int, n: int, p_bar: int):
        import torch
        self.eng, self.world, self.rank, self.n, self.p_bar = engine, world, rank, int(n), int(p_bar)
        self.row0, self.w_local = shard_rows(self.n - self.p_bar, world, rank)
        L = _abi.lib()
        buf = C.create_string_buffer(128)
        if rank == 0:
            engine._check(L.tf_nccl_unique_id(buf, 128))
        t = torch.frombuffer(bytearray(buf.raw), dtype=torch.uint8).to(torch.device("cuda", torch.cuda.current_device()))
        dist.broadcast(t, 0)
        uid = bytes(t.cpu().numpy().tobytes())
        engine._check(L.tf_nccl_init(engine._ctx, uid, world, rank))

    def generate(self, roots, seed: int, innovations: str = "normal"):
        """The whole series generated on the device (identical on every rank), then cut to this slice."""
        self.eng.generate_series(roots, self.n, seed, innovations)
        self.eng._check(_abi.lib().tf_keep_slice(self.eng._ctx, self.row0, self.w_local + self.p_bar))
        self.eng._series_id = ("slice", self.row0)

    def upload_host(self, y):
        v = np.ascontiguousarray(np.asarray(y, dtype=np.float64)[self.row0:self.row0 + self.w_local + self.p_bar])
        self.eng._check(_abi.lib().tf_upload_series(self.eng._ctx, ptr(v), v.size))
        self.eng._series_id = None

    def lsar_sweep(self, c: int, seed: int, want_diag=False):
        return self.eng.lsar_sweep(self.p_bar, c, seed, want_diag=want_diag, n=self.w_local + self.p_bar,
                                   sharded=True)

    def e2e_step(self, c: int, seed: int) -> float:
        """Wall time of one end-to-end sharded fit: H2D of this rank's slice from
        pinned host memory, the sweep, D2H of the fit."""
        import torch
        m = self.w_local + self.p_bar
        pinned = torch.empty(m, dtype=torch.float64, pin_memory=True).numpy()
        self.eng.download_series_into(pinned)
        torch.cuda.synchronize()
        t0 = time.time()
        self.eng._check(_abi.lib().tf_upload_series(self.eng._ctx, ptr(pinned), m))
        self.lsar_sweep(c, seed)
        torch.cuda.synchronize()
        return time.time() - t0


@dataclass
class ShardFit:
    taus: np.ndarray
    coefs: list
    p_star: int
    local_draws: list  # per lag: number of draws this rank resolved
    row0: int
    rows: int


def lsar_fit_sharded(y, p_bar: int, c: int, seed: int, comm=None, backend=None) -> ShardFit:
    """The sharded protocol (lsar.cpp:100-124 over row blocks) in Python over
    `comm`, with `backend` doing the per-shard steps (tests: numpy stand-in).
    tf_lsar_sweep_sharded runs the same steps on the device."""
    comm = comm or LocalComm()
    if backend is None:
        raise UsageError("the protocol model needs a per-shard backend (the GPU path is NcclShard)")
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
        R = global_R(comm.allgather(np.array([a, b])))
        if not R > 0.0:
            raise NumericalError("all-zero window; leverage undefined (lag 1)" if p == 1 else
                                 f"zero residual norm; sampling distribution undefined (lag {p})")
        S, lo, hi = segment(comm.allgather(np.array([backend.local_total(R)]))[:, 0], comm.rank)
        k = backend.sample(derive_seed(seed, p), R, S, lo, hi)
        draws.append(k)
        parts = comm.allgather(backend.gram(p))  # this shard's Gram partial
        G = np.zeros_like(parts[0])
        for r in range(parts.shape[0]):  # rank order
            G = G + parts[r]
        phi = backend.solve(p, G)
        taus[p - 1] = phi[p - 1]
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
