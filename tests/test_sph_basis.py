"""CPU: the far field's solid-harmonic change of basis (csrc/sph_basis.cuh).

1. the committed table is exactly what scripts/gen_sph_basis.py produces (the script
   solves it in rational arithmetic and checks it on every monomial);
2. in float64, sum_k W_k b^k(dx) over the k3 <= 1 Taylor coefficients of 1/r (the
   reference recurrence, coulomb.hpp:37-48) equals sum_m W_hat_m w_m(dx/r) / r^(n+1) with
   W_hat = B^T W and the kernel's two-op recurrence, to the rounding of the terms."""
import os
import re
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "paper_1811_12498_b200", "csrc", "sph_basis.cuh")
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import gen_sph_basis as G  # noqa: E402


def table():
    txt = open(HEADER).read().split("kSphB[] = {")[1].split("};")[0]
    txt = re.sub(r"//.*", "", txt)
    return np.array([float(x) for x in re.findall(r"[-+]?(?:\d+\.\d*|\.\d+|\d+)(?:e[-+]?\d+)?", txt)])


def off(s):
    return s * (2 * s - 1) * (2 * s + 1) // 3


def test_committed_table_is_generated(tmp_path):
    out = tmp_path / "sph.cuh"
    subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "gen_sph_basis.py"), str(out)], check=True,
                   capture_output=True)
    assert out.read_text() == open(HEADER).read()
    assert table().size == off(G.PMAX + 1)


def taylor_values(dx, P, dt):
    """b^k for k3 <= 1 per grade, by the reference recurrence restricted to that set."""
    dx = dx.astype(dt)
    rinv = 1 / np.sqrt((dx * dx).sum())
    ir2 = rinv * rinv
    b = {(0, 0, 0): rinv}
    out = [[rinv]]
    for s in range(1, P + 1):
        row = []
        for k in G.taylor_index(s):
            t1, t2 = dt(0), dt(0)
            for i in range(3):
                km = list(k)
                if k[i] >= 1:
                    km[i] -= 1
                    t1 += dx[i] * b[tuple(km)]
                    km[i] += 1
                if k[i] >= 2:
                    km[i] -= 2
                    t2 += b[tuple(km)]
            v = ((2 * s - 1) * t1 - (s - 1) * t2) * ir2 / s
            b[k] = v
            row.append(v)
        out.append(row)
    return out


def harmonic_values(dx, P):
    """The far kernel's arithmetic (far_eval.cuh): w on the unit sphere, scaled per grade."""
    rinv = 1 / np.sqrt((dx * dx).sum())
    xh, yh, zh = dx * rinv
    w = {(0, 0, 0): 1.0, (0, 0, 1): 0.0}
    out, pw = [[rinv]], rinv
    for n in range(1, P + 1):
        c, sn = w[(n - 1, n - 1, 0)], w[(n - 1, n - 1, 1)]
        w[(n, n, 0)], w[(n, n, 1)] = xh * c - yh * sn, xh * sn + yh * c
        for part in (0, 1):
            w[(n, n - 1, part)] = zh * w[(n - 1, n - 1, part)]
        for m in range(n - 1):
            for part in (0, 1):
                w[(n, m, part)] = zh * w[(n - 1, m, part)] + float(G.beta(n, m)) * w[(n - 2, m, part)]
        pw *= rinv
        out.append([w[h] * pw for h in G.harmonic_index(n)])
    return out


def test_change_of_basis_matches_taylor_form():
    B = table()
    rng = np.random.default_rng(7)
    for P in (1, 4, 8, 12, 18):
        worst = 0.0
        for _ in range(40):
            dx = rng.normal(size=3)
            dx *= rng.uniform(1.0, 3.0) / np.linalg.norm(dx)
            W = [rng.uniform(-1, 1, 2 * s + 1) * 0.5 ** s for s in range(P + 1)]
            tl = taylor_values(dx, P, np.longdouble)
            ref = sum(np.dot(np.array(W[s], dtype=np.longdouble), np.array(v)) for s, v in enumerate(tl))
            mag = float(sum(np.dot(np.abs(W[s]), np.abs(np.array(v, dtype=np.float64))) for s, v in enumerate(tl)))
            hv = harmonic_values(dx, P)
            new = sum(np.dot(B[off(s):off(s + 1)].reshape(2 * s + 1, 2 * s + 1).T @ W[s], hv[s])
                      for s in range(P + 1))
            worst = max(worst, abs(float(new - ref)) / mag)
        assert worst < 2e-15, (P, worst)
