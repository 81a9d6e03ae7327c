#!/usr/bin/env python
"""Generate paper_1811_12498_b200/csrc/sph_basis.cuh: exact per-grade change of basis from
the far field's k3 <= 1 Taylor basis to scaled real solid harmonics.

The folded far-field weights W (moments.cu k_fold) multiply, at grade s, the 2s+1 Taylor
coefficients b^k of 1/r with k3 in {0, 1} (coulomb.hpp:37-48 restricted; harmonic fold).
Each b^k = N_k(x) / r^(2s+1) with N_k a harmonic homogeneous polynomial of degree s:

    N_0 = 1,  N_k = [(2s-1) sum_i x_i N_{k-e_i} - (s-1) r^2 sum_i N_{k-2e_i}] / s

(the reference recurrence with b^k = N_k / r^(2s+1) substituted).  The kernel evaluates
instead the real solid harmonics R_n^m (cos part C, sin part S) defined by

    C_m + i S_m = (x + i y)^m                               (n = m)
    R_{m+1}^m  = z R_m^m                                    (n = m + 1)
    R_n^m      = z R_{n-1}^m + beta_nm r^2 R_{n-2}^m,       beta_nm = -(n+m-1)(n-m-1)/((2n-1)(2n-3))

on the unit sphere (w_n^m = R_n^m(x/r)), so each value costs one DMUL + one DFMA, and
scales grade n by r^-(n+1) once per grade: R_n^m(x) / r^(2n+1) = w_n^m / r^(n+1).

Per grade, N_k = sum_m B[k][m] R_m exactly (both span the degree-s harmonic polynomials,
which are determined by their monomials with z-power <= 1).  B is solved here in exact
rational arithmetic, checked on every monomial, and written as doubles; the fold applies
W_hat[m] = sum_k B[k][m] W[k].  Grade ordering: Taylor index j <= s -> k = (s-j, j, 0),
j > s -> k = (s-1-b, b, 1) with b = j-s-1 (moments.cu k_fold); harmonic index 0 -> C_s^0,
2m-1 -> C_s^m, 2m -> S_s^m.
"""
import os
import sys
from fractions import Fraction

PMAX = 18  # kMaxOrder 16 + 2 (stresslet)


def padd(a, b, s=Fraction(1)):
    out = dict(a)
    for k, v in b.items():
        out[k] = out.get(k, 0) + s * v
        if out[k] == 0:
            del out[k]
    return out


def pscale(a, s):
    return {k: v * s for k, v in a.items()} if s != 0 else {}


def pmulx(a, i):
    out = {}
    for k, v in a.items():
        kk = list(k)
        kk[i] += 1
        out[tuple(kk)] = v
    return out


def pmulr2(a):
    out = {}
    for i in range(3):
        out = padd(out, pmulx(pmulx(a, i), i))
    return out


def laplacian(a):
    out = {}
    for k, v in a.items():
        for i in range(3):
            if k[i] >= 2:
                kk = list(k)
                kk[i] -= 2
                kk = tuple(kk)
                out[kk] = out.get(kk, 0) + v * k[i] * (k[i] - 1)
    return {k: v for k, v in out.items() if v != 0}


def taylor_index(s):
    ks = [(s - j, j, 0) for j in range(s + 1)]
    ks += [(s - 1 - b, b, 1) for b in range(s)]
    return ks


def taylor_polys(P):
    N = {(0, 0, 0): {(0, 0, 0): Fraction(1)}}
    for s in range(1, P + 1):
        for k in taylor_index(s):
            acc = {}
            for i in range(3):
                if k[i] >= 1:
                    km = list(k)
                    km[i] -= 1
                    acc = padd(acc, pmulx(N[tuple(km)], i), Fraction(2 * s - 1))
            acc2 = {}
            for i in range(3):
                if k[i] >= 2:
                    km = list(k)
                    km[i] -= 2
                    acc2 = padd(acc2, N[tuple(km)])
            acc = padd(acc, pmulr2(acc2), Fraction(-(s - 1)))
            N[k] = pscale(acc, Fraction(1, s))
    return N


def beta(n, m):
    return Fraction(-(n + m - 1) * (n - m - 1), (2 * n - 1) * (2 * n - 3))


def harmonic_polys(P):
    """R[(n, m, part)] with part 0 = cos, 1 = sin."""
    R = {(0, 0, 0): {(0, 0, 0): Fraction(1)}, (0, 0, 1): {}}
    for n in range(1, P + 1):
        # diagonal: (x + i y)^n
        c, s_ = R[(n - 1, n - 1, 0)], R[(n - 1, n - 1, 1)]
        R[(n, n, 0)] = padd(pmulx(c, 0), pmulx(s_, 1), Fraction(-1))
        R[(n, n, 1)] = padd(pmulx(s_, 0), pmulx(c, 1))
        for part in (0, 1):
            R[(n, n - 1, part)] = pmulx(R[(n - 1, n - 1, part)], 2)
        for m in range(0, n - 1):
            for part in (0, 1):
                R[(n, m, part)] = padd(pmulx(R[(n - 1, m, part)], 2), pmulr2(R[(n - 2, m, part)]), beta(n, m))
    return R


def harmonic_index(s):
    out = [(s, 0, 0)]
    for m in range(1, s + 1):
        out += [(s, m, 0), (s, m, 1)]
    return out


def solve_exact(A, Bm):
    """X with X A = Bm (A square, rows = basis), by Gauss-Jordan on A^T."""
    n = len(A)
    # solve A^T X^T = Bm^T
    M = [[A[c][r] for c in range(n)] + [Bm[k][r] for k in range(len(Bm))] for r in range(n)]
    W = len(M[0])
    for col in range(n):
        piv = next(r for r in range(col, n) if M[r][col] != 0)
        M[col], M[piv] = M[piv], M[col]
        inv = 1 / M[col][col]
        M[col] = [v * inv for v in M[col]]
        for r in range(n):
            if r != col and M[r][col] != 0:
                f = M[r][col]
                M[r] = [a - f * b for a, b in zip(M[r], M[col])]
    # X^T = M[:, n:]  -> X[k][m] = M[m][n + k]
    return [[M[m][n + k] for m in range(n)] for k in range(len(Bm))]


def main(out_path):
    N = taylor_polys(PMAX)
    R = harmonic_polys(PMAX)
    for key, poly in R.items():
        assert not laplacian(poly), f"R{key} not harmonic"
    mats = []
    for s in range(PMAX + 1):
        mons = taylor_index(s)
        hs = harmonic_index(s)
        Rm = [[R[h].get(mo, Fraction(0)) for mo in mons] for h in hs]
        Nm = [[N[k].get(mo, Fraction(0)) for mo in mons] for k in mons]
        X = solve_exact(Rm, Nm)  # N_k = sum_m X[k][m] R_m
        for ki, k in enumerate(mons):  # full check on every monomial
            acc = {}
            for mi, h in enumerate(hs):
                acc = padd(acc, R[h], X[ki][mi])
            assert padd(acc, N[k], Fraction(-1)) == {}, (s, k)
        mats.append(X)
    lines = [
        "// GENERATED by scripts/gen_sph_basis.py -- do not edit.",
        "// Per-grade change of basis B_s[j][m] (row = k3<=1 Taylor index j, column = solid",
        "// harmonic index m) for s = 0..%d, exact rationals rounded to double:" % PMAX,
        "// N_k = sum_m B_s[k][m] R_s^m; the fold applies W_hat[m] = sum_j B_s[j][m] W[j].",
        "#pragma once",
        "namespace st {",
        "constexpr int kSphPmax = %d;" % PMAX,
        "// offset of grade s: sum_{t<s} (2t+1)^2 = s(2s-1)(2s+1)/3",
        "__host__ __device__ constexpr int sph_off(int s) { return s * (2 * s - 1) * (2 * s + 1) / 3; }",
        "__device__ const double kSphB[] = {",
    ]
    for s, X in enumerate(mats):
        vals = [repr(float(v)) for row in X for v in row]
        lines.append("    // s = %d" % s)
        for i in range(0, len(vals), 6):
            lines.append("    " + ", ".join(vals[i:i + 6]) + ",")
    lines += ["};", "}  // namespace st", ""]
    with open(out_path, "w") as f:
        f.write("\n".join(lines))
    import numpy as np
    for s in (2, 6, 10, 14, 18):
        A = np.array([[float(v) for v in row] for row in mats[s]])
        print(f"grade {s:2d}: max|B| {np.abs(A).max():.3e}  cond {np.linalg.cond(A):.3e}")


if __name__ == "__main__":
    here = os.path.dirname(os.path.abspath(__file__))
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(here, "..", "paper_1811_12498_b200", "csrc",
                                                              "sph_basis.cuh")
    main(out)
