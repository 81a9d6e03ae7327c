"""TEST INFRASTRUCTURE ONLY -- finite-difference checker for the Taylor coefficients.

Restates the reference's test support tests/support/finite_difference.hpp:1-112:
a^k = (1/k!) D_y^k K(x, y) by nested central first differences in 80-bit long double
(numpy.longdouble on x86-64), one Richardson step (4 L(h/2) - L(h)) / 3, and
h = 2e-3 * max(1, |x - y|).  Accurate to ~1e-6 relative for |k| <= 4."""
import numpy as np

ld = np.longdouble


def _nested(f, y, k, h):
    # finite_difference.hpp:30-45: difference along the first axis with k_a > 0, recurse
    for a in range(3):
        if k[a] > 0:
            km = list(k)
            km[a] -= 1
            yp, ym = y.copy(), y.copy()
            yp[a] += h
            ym[a] -= h
            return (_nested(f, yp, km, h) - _nested(f, ym, km, h)) / (ld(2) * h)
    return f(y)


def _derivative(f, y, k, h):
    # finite_difference.hpp:47-52
    coarse = _nested(f, y, k, h)
    fine = _nested(f, y, k, h * ld(0.5))
    return (ld(4) * fine - coarse) / ld(3)


def _factorial(k):
    r = ld(1)
    for a in range(3):
        for i in range(2, k[a] + 1):
            r *= i
    return r


def _step(x, y):
    d = np.asarray(x, ld) - np.asarray(y, ld)
    return ld(2e-3) * max(ld(1), np.sqrt(np.dot(d, d)))


def stokeslet_a_fd(x, y, k, i, j):
    """(1/k!) D_y^k S_ij(x, y), S_ij = delta_ij / r + d_i d_j / r^3 (finite_difference.hpp:77-98)."""
    xl = np.asarray(x, ld)

    def f(yy):
        d = xl - yy
        r2 = np.dot(d, d)
        r = np.sqrt(r2)
        return (ld(1) / r if i == j else ld(0)) + d[i] * d[j] / (r2 * r)

    return float(_derivative(f, np.asarray(y, ld), k, _step(x, y)) / _factorial(k))


def stresslet_a_fd(x, y, k, i, j, l):
    """(1/k!) D_y^k T_ijl(x, y), T_ijl = d_i d_j d_l / r^5 (finite_difference.hpp:85-89, 104-110)."""
    xl = np.asarray(x, ld)

    def f(yy):
        d = xl - yy
        r2 = np.dot(d, d)
        return d[i] * d[j] * d[l] / (r2 * r2 * np.sqrt(r2))

    return float(_derivative(f, np.asarray(y, ld), k, _step(x, y)) / _factorial(k))


def multi_indices(p):
    """Graded-lex multi-indices of grade <= p (multi_index.hpp:36-44)."""
    return [(k1, k2, s - k1 - k2) for s in range(p + 1) for k1 in range(s + 1) for k2 in range(s - k1 + 1)]
