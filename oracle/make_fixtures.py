"""Oracle fixtures at the BASELINE configurations (TEST INFRASTRUCTURE ONLY).

Runs the oracle restatement (oracle/toepfit_oracle.c, OpenMP-parallel; the
parallel loops are row / column independent, so results do not depend on the
thread count) on the BASELINE.json workloads once, on the CPU, and stores what
the GPU's deterministic-index tests (tests/test_gpu_fixtures.py) need:

  * per lag: phi (packed), tau, ||r_p||^2, sum s_p, the solve method (CPQR
    vs min-norm SVD, toeplitz.cpp:57-85) and rank, cond(A_S); and p*;
  * per lag a SHA-256 digest of the oracle's draws (index and weight bytes, in
    draw order) and the first 16 (index, weight) pairs.  The draws themselves
    (1e6-1e8 values) are not stored: the test re-derives them bit-exactly with
    orc_lsar_replay / orc_rh_replay (the oracle's own recursion fed with the
    stored coefficients / final approximation rows -- no solves, O(p_bar n)),
    checks the digests, and feeds them to the GPU sweep;
  * for RH: the halving level sizes and a digest of the concatenated levels
    (the GPU resolves them itself, bit-exactly), the upward-pass samples of
    every level (draw order), a strided subsample of the final scores.

Inputs are regenerated from the seeded generator (paper_2112_12994_b200/gen.py,
numpy + scipy.signal.lfilter: deterministic); the fixture records a SHA-256 of
the series so a test can tell a changed generator from a parity failure.

    OMP_NUM_THREADS=8 python oracle/make_fixtures.py [name ...]   (default: every case)
"""
from __future__ import annotations

import hashlib
import json
import lzma
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as orc  # noqa: E402
from paper_2112_12994_b200 import gen  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
SEED = 2112_12994   # series seed (gen.make_config_series default)
FIT_SEED = 20_211_229

# name: (generator config, n, p_bar, c, method, rh gaussian_rows or None, rh base or None)
CASES = {
    # C1 at full size (BASELINE configs[0])
    "c1_lsar": ("C1", 1_000_000, 100, 20_000, "lsar", None, None),
    # C2 (configs[1]): n = 1e7, p_bar = 200, s = 1e4, LSAR and RH with the defaults
    # (base 12060, g = ceil(8 ln 9,999,800) = 129, depth 10)
    "c2_lsar": ("C2", 10_000_000, 200, 10_000, "lsar", None, None),
    "c2_rh": ("C2", 10_000_000, 200, 10_000, "rh", None, None),
    # RH with explicit sketch widths and depth >= 2 on m ~ 2e5 (g = 129: the
    # C2 default width; g = 65: a one-column tail after a 64-column tile)
    "rh_g129": ("C2", 200_040, 40, 2_000, "rh", 129, 20_000),
    "rh_g65": ("C2", 200_040, 40, 2_000, "rh", 65, 20_000),
    # C4-shaped: AR(100), |root| in [1.05, 2] (configs[3]'s generator), p_bar =
    # 500 at reduced n and c (the full C4 draws, 1e8 indices, do not fit a
    # fixture); the sampled systems are numerically rank deficient from p ~ 30
    # on, so the reference's CPQR rank rule and min-norm SVD decide phi
    "c4s_lsar": ("C4", 1_000_000, 500, 20_000, "lsar", None, None),
}


def series_for(cfg: str, n: int) -> np.ndarray:
    y, _, _, _ = gen.make_config_series(cfg, seed=SEED, n=n)
    return np.ascontiguousarray(y)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def pack_i64(a: np.ndarray) -> np.ndarray:
    return np.frombuffer(lzma.compress(np.ascontiguousarray(a, np.int64).tobytes(), preset=9), np.uint8)


def unpack_i64(blob: np.ndarray, shape) -> np.ndarray:
    return np.frombuffer(lzma.decompress(blob.tobytes()), np.int64).reshape(shape).copy()


def draw_digests(idx: np.ndarray, w: np.ndarray) -> np.ndarray:
    """[lags][32] SHA-256 of each lag's (index bytes, weight bytes), draw order."""
    out = np.zeros((idx.shape[0], 32), np.uint8)
    for p in range(idx.shape[0]):
        h = hashlib.sha256(np.ascontiguousarray(idx[p], np.int64).tobytes())
        h.update(np.ascontiguousarray(w[p], np.float64).tobytes())
        out[p] = np.frombuffer(h.digest(), np.uint8)
    return out


def cond_of(a: np.ndarray) -> float:
    """cond_2 of a sampled system (c x p), via the R of a QR."""
    import scipy.linalg as sl
    p = a.shape[1]
    r = sl.qr(a, mode="r", check_finite=False)[0][:p, :p]
    sv = sl.svdvals(r, check_finite=False)
    return float(sv[0] / sv[-1]) if sv[-1] > 0 else float("inf")


def make(name: str) -> str:
    cfg, n, p_bar, c, method, g, base = CASES[name]
    y = series_for(cfg, n)
    t0 = time.time()
    out = {}
    meta = dict(name=name, config=cfg, n=n, p_bar=p_bar, c=c, method=method, series_seed=SEED,
                fit_seed=FIT_SEED, series_sha256=sha(y), generator="paper_2112_12994_b200/gen.py",
                oracle="oracle/toepfit_oracle.c")
    if method == "lsar":
        f = orc.lsar_fit(y, p_bar, c, FIT_SEED)
        out.update(rnorm2=f.rnorm2, ssum=f.ssum, method=f.method.astype(np.int32))
    else:
        rcfg = None
        if g is not None:
            rcfg = orc.RhCfg(base, c, g, orc.derive_seed(FIT_SEED, 0x5C07E5))
        f = orc.rh_fit(y, p_bar, c, FIT_SEED, cfg=rcfg, want_levels=True)
        lv = np.concatenate(f.levels) if f.levels else np.zeros(0, np.int64)
        m = n - p_bar
        step = max(1, m // 20000)
        out.update(level_sizes=f.level_sizes, levels_sha256=np.array(sha(lv)),
                   up_idx_lz=pack_i64(f.up_idx), up_w=f.up_w,
                   scores_sub=f.scores[::step].copy(), scores_step=np.array(step),
                   scores_sum=np.array(float(np.sum(f.scores))))
        meta.update(depth=int(f.depth), gaussian_rows=int(f.cfg.gaussian_rows),
                    base_threshold=int(f.cfg.base_threshold), cfg_seed=int(f.cfg.seed),
                    explicit_cfg=g is not None)
    t_fit = time.time() - t0
    idx, w = f.idx, f.w
    # cond(A_S) and the oracle's rank per lag (its own sampled system)
    conds = np.zeros(p_bar)
    ranks = np.zeros(p_bar, np.int32)
    meths = np.zeros(p_bar, np.int32)
    for p in range(1, p_bar + 1):
        if method == "lsar":
            a, b = orc.apply_sample(y, (n - p_bar) + p, p, idx[p - 1], w[p - 1])
        else:  # apply_sample(full, s, p), repeated_halving.cpp:221
            a, b = orc.apply_sample(y, n, p_bar, idx[p - 1], w[p - 1], width=p)
        conds[p - 1] = cond_of(a)
        _, meths[p - 1], ranks[p - 1] = orc.solve_exact(a, b)
    if method == "lsar":
        assert np.array_equal(meths, f.method), "oracle method mismatch on re-solve"
    else:
        out.update(method=meths)
    packed = np.concatenate([np.asarray(v) for v in f.coefs])
    out.update(digests=draw_digests(idx, w), wchk_idx=np.ascontiguousarray(idx[:, :16]),
               wchk_w=np.ascontiguousarray(w[:, :16]), taus=f.taus, coefs=packed, cond=conds, rank=ranks,
               p_star=np.array(f.p_star))
    meta.update(oracle_fit_seconds=round(t_fit, 1), omp_threads=os.environ.get("OMP_NUM_THREADS", "default"))
    out["meta"] = np.array(json.dumps(meta))
    os.makedirs(OUT, exist_ok=True)
    path = os.path.join(OUT, f"fix_{name}.npz")
    np.savez(path, **out)
    sz = os.path.getsize(path)
    print(f"{name}: oracle {t_fit:.1f}s, p*={f.p_star}, methods={np.bincount(out['method']).tolist()}, "
          f"cond max {np.max(conds):.2e}, {sz / 1e6:.2f} MB -> {path}", flush=True)
    return path


def load(name: str) -> dict:
    """Fixture -> dict of arrays, 'meta' (dict) and, for RH, 'up_idx' [depth][c]."""
    z = np.load(os.path.join(OUT, f"fix_{name}.npz"))
    d = {k: z[k] for k in z.files}
    d["meta"] = json.loads(str(d["meta"]))
    m = d["meta"]
    if m["method"] == "rh":
        d["up_idx"] = unpack_i64(d["up_idx_lz"], (m["depth"], m["c"]))
    return d


def unpack_coefs(packed: np.ndarray, p_bar: int) -> list:
    out, off = [], 0
    for p in range(1, p_bar + 1):
        out.append(packed[off:off + p])
        off += p
    return out


if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for nm in names:
        make(nm)

