"""Where does the FFT pass's rounding error come from?  (CPU experiment, numpy)

Overlap-save with N = 4096, D = 1024, two blocks per complex transform (the
k_fft.cuh scheme) on a C2 / C4-shaped series with the fixture's fitted phi at
the longest lag.  Variants round different stages from an extended-precision
(long double) evaluation, errors are max|r - r_exact| / max|r_exact| over the
rows; the direct fp64 FIR (the oracle's tap loop) is the yardstick.

    python tools/fft_precision.py C2 [nblocks]
"""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2112_12994_b200 import gen  # noqa: E402

N, D = 4096, 1024
L = N - D
LD = np.longdouble
CLD = np.clongdouble


def fft_ld(x, sign=-1):
    """iterative radix-2 DIT FFT in long double (x: complex long double, len 2^k)"""
    x = np.asarray(x, CLD).copy()
    n = x.size
    j = 0
    rev = np.zeros(n, np.int64)
    bits = n.bit_length() - 1
    for i in range(n):
        rev[i] = int(format(i, f"0{bits}b")[::-1], 2)
    x = x[rev]
    m = 2
    pi = LD("3.14159265358979323846264338327950288")
    while m <= n:
        k = np.arange(m // 2, dtype=LD)
        ang = sign * 2 * pi * k / LD(m)
        w = np.cos(ang) + 1j * np.sin(ang)
        w = w.astype(CLD)
        x = x.reshape(-1, m)
        a = x[:, : m // 2].copy()
        b = x[:, m // 2:] * w
        x[:, : m // 2] = a + b
        x[:, m // 2:] = a - b
        x = x.reshape(-1)
        m *= 2
    del j
    return x


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    nsb = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    fix = {"C2": "fix_c2_lsar", "C4": "fix_c4s_lsar"}[name]
    z = np.load(f"tests/golden/{fix}.npz")
    coefs = z["coefs"]
    pb = int(round((np.sqrt(8 * coefs.size + 1) - 1) / 2))
    q = pb
    phi = coefs[q * (q - 1) // 2:]
    y, _, _, _ = gen.make_config_series(name, n=200_000 + nsb * 2 * L + q + 64)
    i0 = 100_000
    rows = nsb * 2 * L
    seg = y[i0:i0 + rows + N]
    h = np.concatenate([[-1.0], phi])  # r(i) = sum_k h[k] y[q + i - k]
    # exact (long double) and direct fp64 residuals
    yl = seg.astype(LD)
    r_ex = np.zeros(rows, LD)
    r_d = np.zeros(rows)
    for k in range(q + 1):
        r_ex += LD(h[k]) * yl[q - k:q - k + rows]
    # direct fp64, the oracle's tap loop: acc = y[q+i]; acc -= phi_k y[q+i-k]
    acc = seg[q:q + rows].copy()
    for k in range(1, q + 1):
        acc = acc - phi[k - 1] * seg[q - k:q - k + rows]
    r_d = -acc
    scale = float(np.max(np.abs(r_ex)))
    print(f"{name}: q={q} max|phi|={np.max(np.abs(phi)):.3e} ||h||2={np.linalg.norm(h):.3e} "
          f"max|r|={scale:.3e} rms(y)={np.std(seg):.3e} sum|h||y|/|r| ~ "
          f"{np.sum(np.abs(h)) * np.std(seg) / np.std(r_ex.astype(float)):.2e}")
    print(f"  direct fp64 FIR (tap loop)          err {np.max(np.abs(r_d - r_ex.astype(float))) / scale:.3e}")

    # filter: f[D - q + k] = h[k]; output m = u + D is row (block base + u)
    f = np.zeros(N)
    f[D - q:D + 1] = h
    H64 = np.fft.fft(f) / N
    Hld = fft_ld(f.astype(CLD)) / LD(N)

    res = {k: np.zeros(rows) for k in ("all64", "Zex", "Hex", "ZHex", "ZHPex", "ld")}
    for sb in range(nsb):
        xa = seg[sb * 2 * L: sb * 2 * L + N]
        xb = seg[sb * 2 * L + L: sb * 2 * L + L + N]
        xc = xa + 1j * xb
        Z64 = np.fft.fft(xc)
        Zld = fft_ld(xa.astype(LD) + 1j * xb.astype(LD))
        Zr = Zld.astype(np.complex128)
        Hr = Hld.astype(np.complex128)
        outs = {
            "all64": np.fft.ifft(Z64 * H64) * N,
            "Zex": np.fft.ifft(Zr * H64) * N,
            "Hex": np.fft.ifft(Z64 * Hr) * N,
            "ZHex": np.fft.ifft(Zr * Hr) * N,
            "ZHPex": np.fft.ifft((Zld * Hld).astype(np.complex128)) * N,
            "ld": fft_ld(Zld * Hld, +1).astype(np.complex128),
        }
        for k, o in outs.items():
            res[k][sb * 2 * L: sb * 2 * L + L] = o.real[D:]
            res[k][sb * 2 * L + L: sb * 2 * L + 2 * L] = o.imag[D:]
    for k, v in res.items():
        print(f"  fft {k:6s}                         err {np.max(np.abs(v - r_ex.astype(float))) / scale:.3e}"
              f"   vs direct: {np.max(np.abs(v - r_d)) / scale:.3e}")
    # garbage outputs (wrap-around) magnitude
    o = np.fft.ifft(Z64 * H64) * N
    print(f"  |wrap outputs| max {np.max(np.abs(o.real[D - q:D])):.3e}, |valid| max {np.max(np.abs(o.real[D:])):.3e}")


if __name__ == "__main__":
    main()
