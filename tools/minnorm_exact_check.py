"""Exact-arithmetic check of the rank-revealing solve (mpmath Gram, pivoted
Cholesky = CPQR, SVD min-norm) against the oracle on a C4-generator sampled
system: python tools/minnorm_exact_check.py p c.  Also dumps the cases that
tools/svd_debug.cu / tools/pchol_debug.cu replay on the GPU."""
import sys, numpy as np, mpmath as mp
sys.path.insert(0,'.')
from oracle import oracle as orc
from paper_2112_12994_b200 import gen
mp.mp.dps = 60
y, _, _, _ = gen.make_config_series("C4", n=300000)
p, c = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(p)
idx = rng.integers(0, y.size - p, size=c)
w = rng.uniform(0.5, 2.0, size=c)
a, b = orc.apply_sample(y, y.size, p, idx, w)
ref, m, rank = orc.solve_exact(a, b)
Af = np.column_stack([a[:, ::-1], b]); K = p + 1
# exact Gram via python ints: each double = mant * 2^e
from fractions import Fraction
M = [[mp.mpf(0)]*K for _ in range(K)]
cols = [[mp.mpf(float(v)) for v in Af[:, j]] for j in range(K)]
for i in range(K):
    for j in range(i, K):
        s = mp.fsum(cols[i][t] * cols[j][t] for t in range(c))
        M[i][j] = M[j][i] = s
perm = list(range(p)) + [p]
d = [M[j][j] for j in range(K)]
R = [[mp.mpf(0)]*K for _ in range(K)]
tol = max(c, p) * np.finfo(float).eps
rk = [mp.mpf(0)]*p; kend = p
for k in range(p):
    piv = max(range(k, p), key=lambda j: d[j])
    perm[k], perm[piv] = perm[piv], perm[k]; d[k], d[piv] = d[piv], d[k]
    if not d[k] > 0: kend = k; break
    rk[k] = mp.sqrt(d[k]); ck = perm[k]
    for j in range(k + 1, K):
        cj = perm[j]
        s = M[ck][cj] - mp.fsum(R[ck][i] * R[cj][i] for i in range(k))
        R[cj][k] = s / rk[k]
        if j < p: d[j] -= R[cj][k] ** 2
    R[ck][k] = rk[k]
mx = max(abs(v) for v in rk[:kend]); rank_e = sum(1 for v in rk[:kend] if abs(v) > tol * mx)
print("rank", rank_e, "oracle", rank, "rkk/max", [float(abs(v)/mx) for v in rk[:kend]][-10:])
Rp = np.zeros((p, p)); z = np.zeros(p)
for i in range(kend):
    for j in range(i, p): Rp[i, j] = float(R[perm[j]][i])
    z[i] = float(R[p][i])
U, S, Vt = np.linalg.svd(Rp)
keep = S >= tol * S[0]
x = Vt.T[:, keep] @ ((U[:, keep].T @ z) / S[keep])
phi = np.zeros(p)
for j in range(p): phi[p - 1 - perm[j]] = x[j]
print("phi err", np.max(np.abs(phi - ref)) / np.max(np.abs(ref)), "resid ratio", np.linalg.norm(a@phi-b)/np.linalg.norm(a@ref-b))
# --- emulate k_svd_minnorm on N = [R'^T; z^T]
m_ = p + 1
N = np.zeros((p, m_))  # N[c] = column c (length m)
for i in range(kend):
    for j in range(i, p): N[i, j] = float(R[perm[j]][i])
    N[i, p] = float(R[p][i])
nct = min(16, max(1, (p + 31) // 32)); nblk = 2 * nct; bw = max(1, (p + nblk - 1) // nblk)
def rr(n, r, t):
    a_ = n - 1 if t == 0 else (r + t) % (n - 1); b_ = (r - t + (n - 1)) % (n - 1); return a_, b_
eps = np.finfo(float).eps
for sweep in range(60):
    rot = 0
    for r in range(nblk - 1):
        for cta in range(nct):
            ba, bb = rr(nblk, r, cta); colof = [ba * bw, bb * bw]; nl = 2 * bw
            for sr in range(nl - 1):
                for t in range(bw):
                    u, v = rr(nl, sr, t)
                    gu = colof[u // bw] + u % bw; gv = colof[v // bw] + v % bw
                    if gu >= p or gv >= p: continue
                    xu, xv = N[gu], N[gv]
                    al = xu[:p] @ xu[:p]; be = xv[:p] @ xv[:p]; ga = xu[:p] @ xv[:p]
                    if ga == 0 or abs(ga) <= eps * np.sqrt(al * be): continue
                    rot = 1
                    zeta = (be - al) / (2 * ga); tt = (1.0 if zeta >= 0 else -1.0) / (abs(zeta) + np.sqrt(1 + zeta * zeta))
                    cs = 1 / np.sqrt(1 + tt * tt); sn = cs * tt
                    N[gu], N[gv] = cs * xu - sn * xv, sn * xu + cs * xv
    if not rot: break
print("sweeps", sweep + 1)
sig = np.sqrt((N[:, :p] ** 2).sum(1)); thr = max(sig.max() * tol, 2.2e-308)
x = sum(N[c, :p] * (N[c, p] / sig[c] ** 2) for c in range(p) if sig[c] >= thr)
phi2 = np.zeros(p)
for j in range(p): phi2[p - 1 - perm[j]] = x[j]
print("jacobi phi err", np.max(np.abs(phi2 - ref)) / np.max(np.abs(ref)), np.sum(sig >= thr))
# dump SVD input for the CUDA harness
N0 = np.zeros((p, m_))
for i in range(kend):
    for j in range(i, p): N0[i, j] = float(R[perm[j]][i])
    N0[i, p] = float(R[p][i])
with open('/root/repo/tools/svd_case.bin', 'wb') as f:
    np.array([p], np.int64).tofile(f); np.array([tol], np.float64).tofile(f)
    np.array(perm, np.int32).tofile(f); N0.tofile(f); phi2.tofile(f)
print("dumped")
Gh = np.array([[float(M[i][j]) for j in range(K)] for i in range(K)])
Gl = np.array([[float(M[i][j] - mp.mpf(Gh[i, j])) for j in range(K)] for i in range(K)])
with open('/root/repo/tools/pchol_case.bin', 'wb') as f:
    np.array([K, c], np.int64).tofile(f); Gh.tofile(f); Gl.tofile(f); phi2.tofile(f); np.array([rank_e], np.int64).tofile(f)
print("dumped pchol")
