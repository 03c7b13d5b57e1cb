"""CPU stand-in for the per-shard device steps (test infrastructure only):
the per-shard steps of the protocol (paper_2112_12994_b200/shard.py), in numpy,
so the sharded orchestration (collectives, offsets, draw ownership, pass
gating) is exercised over gloo without a GPU.  Plain normal-equation solve
of the sampled system; the counter RNG is the reference's (rng.hpp:23-35)."""
import numpy as np

GOLD = 0x9E3779B97F4A7C15
M64 = (1 << 64) - 1


def mix(z):
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def uniform(seed, t):
    return (mix((seed + (t + 1) * GOLD) & M64) >> 11) * 2.0 ** -53


class NumpyShard:
    def open(self, y_slice, p_bar, c, w_local):
        self.y = np.asarray(y_slice, dtype=np.float64)
        self.c, self.w = c, w_local
        self.s = np.zeros(w_local)
        self.r = np.zeros(w_local)

    def pass_(self, q, phi, r_prev):
        y, w = self.y, self.w
        rn = -y[q:q + w].copy()
        for j in range(q):
            rn += phi[j] * y[q - 1 - j:q - 1 - j + w]
        self.s = self.s + self.r ** 2 / r_prev if q > 0 else np.zeros(w)
        self.r = rn
        return float(self.s.sum()), float((rn ** 2).sum())

    def local_total(self, r_glob):
        return float(np.sum(self.s + self.r ** 2 / r_glob))

    def sample(self, seed_p, r_glob, s_total, lo, hi):
        mass = self.s + self.r ** 2 / r_glob
        cum = np.cumsum(mass)
        idx, wt = [], []
        for t in range(self.c):
            x = uniform(seed_p, t) * s_total
            if not (lo <= x < hi):
                continue
            v = x - lo
            i = min(int(np.searchsorted(cum, v, side="right")), self.w - 1)
            while mass[i] <= 0 and i > 0:
                i -= 1
            idx.append(i)
            wt.append(1.0 / np.sqrt(self.c * mass[i] / s_total))
        self.idx, self.wt = np.array(idx, np.int64), np.array(wt)
        return len(idx)

    def gram(self, p):
        K = p + 1
        if self.idx.size == 0:
            return np.zeros(K * K)
        A = self.wt[:, None] * np.stack([self.y[self.idx + a] for a in range(K)], 1)
        return (A.T @ A).ravel()

    def solve(self, p, G):
        K = p + 1
        G = np.asarray(G).reshape(K, K)
        phi_fwd = np.linalg.solve(G[:p, :p], G[:p, p])  # forward order, target last
        return phi_fwd[::-1].copy()
