"""Row-sharded LSAR sweep.  CPU: the protocol of
paper_2112_12994_b200/shard.py (the steps tf_lsar_sweep_sharded runs on the
device) at world size 2 over gloo with a numpy stand-in for the per-shard
steps must resolve exactly the single-shard draws and give the same fit, and
the CDF segments must partition the draws.  GPU: the in-library NCCL path
(tf_nccl_init + tf_lsar_sweep_sharded) at world size 1 reproduces
tf_lsar_sweep bit for bit (only one GPU is available to this build)."""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _series(n=3000, seed=3):
    from paper_2112_12994_b200 import gen
    return gen.simulate_roots(gen.ar_roots(5, 1.3, 3.0, seed), n, seed)


def _worker(rank, world, port, y, p_bar, c, seed, q):
    import torch.distributed as dist
    from paper_2112_12994_b200 import shard
    from shard_numpy import NumpyShard
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        fit = shard.lsar_fit_sharded(y, p_bar, c, seed, comm=shard.TorchComm(), backend=NumpyShard())
        q.put((rank, fit.taus, fit.p_star, fit.local_draws, fit.row0, fit.rows))
    finally:
        dist.destroy_process_group()


def test_shard_rows_partition():
    from paper_2112_12994_b200.shard import shard_rows
    for w, world in [(10, 3), (997, 8), (8, 8)]:
        blocks = [shard_rows(w, world, r) for r in range(world)]
        assert blocks[0][0] == 0 and sum(b for _, b in blocks) == w
        assert all(blocks[r][0] + blocks[r][1] == blocks[r + 1][0] for r in range(world - 1))
        assert max(b for _, b in blocks) - min(b for _, b in blocks) <= 1


def test_sharded_gloo_world2_matches_single():
    import multiprocessing as mp
    from paper_2112_12994_b200 import shard
    from shard_numpy import NumpyShard
    y, p_bar, c, seed = _series(), 6, 300, 17
    single = shard.lsar_fit_sharded(y, p_bar, c, seed, backend=NumpyShard())
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, y, p_bar, c, seed, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    (r0, t0, ps0, d0, row0a, rows0), (r1, t1, ps1, d1, row0b, rows1) = res
    assert row0a == 0 and row0b == rows0 and rows0 + rows1 == y.size - p_bar
    # every draw resolved by exactly one shard
    assert [a + b for a, b in zip(d0, d1)] == [c] * p_bar
    assert np.allclose(t0, t1, rtol=0, atol=0)  # identical on both ranks
    assert np.max(np.abs(t0 - single.taus) / np.maximum(np.abs(single.taus), 1e-3)) < 1e-9
    assert ps0 == ps1 == single.p_star


def test_sharded_numpy_matches_oracle_fixed_draws():
    # the numpy stand-in is faithful: same draws as the oracle's LSAR for one shard
    from oracle import oracle as orc
    from paper_2112_12994_b200 import shard
    from shard_numpy import NumpyShard
    y, p_bar, c, seed = _series(2500, 9), 5, 250, 4
    ref = orc.lsar_fit(y, p_bar, c, seed)
    fit = shard.lsar_fit_sharded(y, p_bar, c, seed, backend=NumpyShard())
    assert np.max(np.abs(fit.taus - ref.taus) / np.maximum(np.abs(ref.taus), 1e-3)) < 1e-8
    assert fit.p_star == ref.p_star


def test_segments_partition_the_draws():
    # k_shard_seg: each u S lands in exactly one shard's [lo, hi)
    from paper_2112_12994_b200.shard import segment
    rng = np.random.default_rng(5)
    for world in (2, 3, 8):
        s_loc = rng.exponential(size=world) * 10 ** rng.uniform(-3, 3, size=world)
        segs = [segment(s_loc, r) for r in range(world)]
        S = segs[0][0]
        assert all(sg[0] == S for sg in segs)
        u = np.concatenate([rng.random(20000), [0.0, 1.0 - 2 ** -53]])
        x = u * S
        owners = np.zeros(x.size, int)
        for _, lo, hi in segs:
            owners += (x >= lo) & (x < hi)
        assert (owners == 1).all()


def _nccl_world1():
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    return dist


@pytest.mark.gpu
def test_sharded_nccl_world1_matches_sweep_bitwise():
    import paper_2112_12994_b200 as tf
    from paper_2112_12994_b200 import shard
    y = _series(40000, 6)
    p_bar, c, seed = 24, 2000, 5
    ref = tf.lsar_fit(tf.TimeSeries(y), p_bar, c, seed, engine=tf.Engine(0), want_diag=True)
    dist = _nccl_world1()
    try:
        eng = tf.Engine(0)
        sh = shard.NcclShard(eng, dist, 1, 0, y.size, p_bar)
        sh.upload_host(y)
        taus, coefs, secs, pstar, d = sh.lsar_sweep(c, seed, want_diag="light")
        taus2, *_ = sh.lsar_sweep(c, seed)  # second call: the captured graph
    finally:
        dist.destroy_process_group()
    assert np.array_equal(taus, np.array(ref.pacf.taus)) and np.array_equal(taus2, taus)
    assert pstar == ref.p_star
    assert np.array_equal(d["method"], ref.diag["method"])


@pytest.mark.gpu
def test_sharded_nccl_world1_generated_slice():
    # the device generator + tf_keep_slice path (what bench.py --gpus N runs)
    import paper_2112_12994_b200 as tf
    from paper_2112_12994_b200 import gen, shard
    roots = gen.ar_roots(6, 1.2, 3.0, 77)
    n, p_bar, c, seed = 120000, 12, 3000, 9
    e1 = tf.Engine(0)
    e1.generate_series(roots, n, 77)
    taus_ref, _, _, ps_ref, _ = e1.lsar_sweep(p_bar, c, seed, n=n)
    dist = _nccl_world1()
    try:
        e2 = tf.Engine(0)
        sh = shard.NcclShard(e2, dist, 1, 0, n, p_bar)
        sh.generate(roots, 77)
        taus, _, _, ps, _ = sh.lsar_sweep(c, seed)
        t_e2e = sh.e2e_step(c, seed)
    finally:
        dist.destroy_process_group()
    assert np.array_equal(taus, taus_ref) and ps == ps_ref and t_e2e > 0


@pytest.mark.gpu
def test_sharded_nccl_world1_fft_pass_and_int8_gram(monkeypatch):
    """The row-sharded sweep on the long-lag kernels (TF_PASS=fft: the FFT pass
    with its double-double spectra from the shard's slice; TF_GRAM=i8: the INT8
    Gram with the shard's device-side draw count and the max|w| max|y|
    exponent bound) equals the single-GPU sweep bit for bit at world size 1."""
    import paper_2112_12994_b200 as tf
    from paper_2112_12994_b200 import shard
    monkeypatch.setenv("TF_PASS", "fft")
    monkeypatch.setenv("TF_GRAM", "i8")
    y = _series(50000, 8)
    p_bar, c, seed = 30, 2500, 13
    ref = tf.lsar_fit(tf.TimeSeries(y), p_bar, c, seed, engine=tf.Engine(0), want_diag=True)
    dist = _nccl_world1()
    try:
        eng = tf.Engine(0)
        sh = shard.NcclShard(eng, dist, 1, 0, y.size, p_bar)
        sh.upload_host(y)
        taus, coefs, secs, pstar, d = sh.lsar_sweep(c, seed, want_diag="light")
        taus2, *_ = sh.lsar_sweep(c, seed)
    finally:
        dist.destroy_process_group()
    assert np.array_equal(taus, np.array(ref.pacf.taus)) and np.array_equal(taus2, taus)
    assert pstar == ref.p_star
    assert np.array_equal(d["method"], ref.diag["method"])


@pytest.mark.gpu
def test_sharded_nccl_world1_long_shard_overlapped_fold(monkeypatch):
    """A shard of >= 2^24 rows takes the sharded loop's other branch: eager
    launches with each FFT lag's score update (k_fft_fold) on the side stream
    beside the replicated solve.  Same device code as the single-GPU sweep's
    split, so one rank through NCCL still equals it bit for bit (twice: the
    sharded loop must not depend on a graph it never captures)."""
    import paper_2112_12994_b200 as tf
    from paper_2112_12994_b200 import gen, shard
    monkeypatch.setenv("TF_PASS", "fft")
    roots = gen.ar_roots(6, 1.2, 3.0, 78)
    n, p_bar, c, seed = (1 << 24) + 5000, 10, 3000, 21
    e1 = tf.Engine(0)
    e1.generate_series(roots, n, 78)
    taus_ref, _, _, ps_ref, _ = e1.lsar_sweep(p_bar, c, seed, n=n)
    e1.close()
    dist = _nccl_world1()
    try:
        e2 = tf.Engine(0)
        sh = shard.NcclShard(e2, dist, 1, 0, n, p_bar)
        sh.generate(roots, 78)
        taus, _, _, ps, _ = sh.lsar_sweep(c, seed)
        taus2, _, _, ps2, _ = sh.lsar_sweep(c, seed)
    finally:
        dist.destroy_process_group()
    assert np.array_equal(taus, taus_ref) and ps == ps_ref
    assert np.array_equal(taus2, taus) and ps2 == ps
