"""Experiment: can the GPU's R factor reproduce the reference's CPQR rank rule
and min-norm answer on C4-shaped sampled systems?  Compares, per lag, the
oracle (Eigen-style CPQR on A, Jacobi-SVD min-norm) with the same rule applied
to the K x K R of [A | b] computed (H) by Householder QR, (C3) by shifted
CholeskyQR3 on A directly, (PC) by preconditioned CholeskyQR2 with the previous
lag's exact inverse factor, R = R_tot T^-1."""
import sys, numpy as np, scipy.linalg as sl
sys.path.insert(0, '/root/repo')
from oracle import oracle as orc
from oracle import make_fixtures as mf

fx = mf.load("c4s_lsar")
m = fx['meta']
y = mf.series_for(m['config'], m['n'])
n, pb, c = m['n'], m['p_bar'], m['c']
fx['idx'] = orc.lsar_replay(y, pb, c, m['fit_seed'], fx['coefs']).idx  # the oracle's draws
w = n - pb
eps = np.finfo(float).eps

def rule(R, p, tol):
    RX, z = R[:p, :p], R[:p, p]
    piv = sl.qr(RX, pivoting=True, mode='r')[0]
    d = np.abs(np.diag(piv))
    rank = int(np.sum(d > tol * d.max()))
    U, S, Vt = np.linalg.svd(RX)
    keep = S > tol * S[0]
    phi_svd = Vt.T[:, keep] @ ((U[:, keep].T @ z) / S[keep])
    phi_qr = sl.solve_triangular(RX, z) if rank == p else None
    return rank, (phi_qr if rank == p else phi_svd), d

def cqr3(Aug):
    K = Aug.shape[1]
    G = Aug.T @ Aug
    s = 11 * (Aug.shape[0] * K + K * (K + 1)) * eps * np.trace(G)
    R1 = np.linalg.cholesky(G + s * np.eye(K)).T
    Q1 = sl.solve_triangular(R1, Aug.T, trans='T').T
    R2 = np.linalg.cholesky(Q1.T @ Q1).T
    Q2 = sl.solve_triangular(R2, Q1.T, trans='T').T
    R3 = np.linalg.cholesky(Q2.T @ Q2).T
    return R3 @ R2 @ R1

prevR = None
for p in [int(a) for a in sys.argv[1:]] or [5, 12, 13, 20, 50, 100, 200, 300, 499, 500]:
    idx = fx['idx'][p - 1]
    wt = np.ones(c)
    A, b = orc.apply_sample(y, w + p, p, idx, wt)
    Aug = np.column_stack([A, b])
    tol = max(c, p) * eps
    phi_o, meth_o, rank_o = orc.solve_exact(A, b)
    R_H = sl.qr(Aug, mode='r')[0][:p + 1]
    rk_H, phi_H, d_H = rule(R_H, p, tol)
    try:
        R_C = cqr3(Aug)
        rk_C, phi_C, d_C = rule(R_C, p, tol)
    except np.linalg.LinAlgError:
        rk_C, phi_C = -1, np.full(p, np.nan)
    # preconditioned: exact inverse factor of the previous lag's columns (same rows)
    Rp = sl.qr(A if p > 1 else A, mode='r')[0][:p, :p]   # R of X (lag columns only)
    T = np.zeros((p + 1, p + 1)); T[:p, :p] = np.linalg.inv(Rp); T[p, p] = 1.0 / np.linalg.norm(b)
    Q1 = Aug @ T
    try:
        RA = np.linalg.cholesky(Q1.T @ Q1).T
        Q2 = sl.solve_triangular(RA, Q1.T, trans='T').T
        RB = np.linalg.cholesky(Q2.T @ Q2).T
        R_P = sl.solve(T.T, (RB @ RA).T).T   # R_tot T^-1
        rk_P, phi_P, _ = rule(R_P, p, tol)
    except np.linalg.LinAlgError:
        rk_P, phi_P = -1, np.full(p, np.nan)
    nrm = max(np.max(np.abs(phi_o)), 1e-300)
    bound = 1.96 / np.sqrt(c)
    print(f"p={p:3d} oracle rank {rank_o:3d} meth {meth_o} | H rank {rk_H:3d} dphi {np.max(np.abs(phi_H-phi_o))/nrm:.1e} dtau {abs(phi_H[-1]-phi_o[-1]):.1e}"
          f" | C3 rank {rk_C:3d} dphi {np.max(np.abs(phi_C-phi_o))/nrm:.1e} dtau {abs(phi_C[-1]-phi_o[-1]):.1e}"
          f" | PC rank {rk_P:3d} dphi {np.max(np.abs(phi_P-phi_o))/nrm:.1e} | tau {phi_o[-1]:+.4f} bound {bound:.4f}"
          f" | min|rkk|/max H {d_H.min()/d_H.max():.1e}", flush=True)
