"""ctypes front end to the CPU checkers -- TEST INFRASTRUCTURE ONLY.

Two checkers live under oracle/:

* ``liboracle.so`` -- oracle/stokes_oracle.c, a plain-C restatement of the
  reference path (every function cites /root/reference file:line);
* ``_ref/libstref.so`` -- the UNMODIFIED reference headers compiled in place by
  oracle/Makefile (ref_harness.cpp).  Present wherever ``make -C oracle`` ran
  with /root/reference mounted; it travels to the GPU box with gpurun.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline /
``--impl reference`` legs may import this module.  The product package
(paper_1811_12498_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OR_LIB = os.path.join(HERE, "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libstref.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_vp = C.c_void_p
_sz = C.c_size_t


class OracleError(RuntimeError):
    pass


class InvalidArgument(OracleError):
    pass


class DomainError(OracleError):
    pass


def _check(code: int, what: str):
    if code == 0:
        return
    if code == 1:
        raise InvalidArgument(what)
    if code == 2:
        raise DomainError(what)
    raise OracleError(f"{what}: status {code}")


def build(quiet: bool = True) -> None:
    """make -C oracle (liboracle.so always; _ref when /root/reference is mounted)."""
    out = subprocess.run(["make", "-C", HERE], capture_output=True, text=True)
    if out.returncode != 0:
        raise OracleError("oracle build failed:\n" + out.stdout + out.stderr)


def _opt(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64).ctypes.data_as(C.c_void_p)


_or = None
_ref = None


def _load_or():
    global _or
    if _or is None:
        if not os.path.exists(OR_LIB):
            build()
        L = C.CDLL(OR_LIB)
        L.or_tree_build.restype = _vp
        L.or_tree_build.argtypes = [_sz, _vp, _vp, _vp, _vp, C.c_int, C.c_int, C.POINTER(C.c_int)]
        L.or_tree_ncl.restype = _sz
        L.or_tree_ncl.argtypes = [_vp]
        L.or_tree_export.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp]
        L.or_tree_free.argtypes = [_vp]
        L.or_moments.argtypes = [_vp, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp, _vp]
        L.or_coulomb.argtypes = [_dp, C.c_int, _dp]
        L.or_taylor.argtypes = [_dp, _dp, C.c_int, C.c_int, _vp, _vp]
        L.or_farfield_pair.argtypes = [_dp, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp, _vp, _dp]
        L.or_treecode.argtypes = [_sz, _vp, _vp, _vp, _vp, _vp, _sz, C.c_int, C.c_double, C.c_int,
                                  C.c_int, C.c_int, C.c_int, C.c_int, _dp, _vp, _u64p]
        L.or_lists.argtypes = [_vp, C.c_double, _sz, _vp, _vp, _sz, _i32p, _i32p, _i64p, _i64p]
        L.or_direct_at.argtypes = [_sz, _vp, _vp, _vp, _vp, C.c_int, C.c_int, _i64p, _sz, C.c_int, _dp]
        L.or_direct_points.argtypes = [_sz, _vp, _vp, _vp, _vp, C.c_int, C.c_int, _dp, _sz, _dp]
        L.or_relative_error.argtypes = [_sz, _dp, _dp, C.POINTER(C.c_double)]
        L.or_mac.argtypes = [C.c_double, C.c_double, C.c_double]
        L.or_mac.restype = C.c_int
        L.or_generate.argtypes = [C.c_int, _sz, C.c_uint64, C.c_int, _vp, _vp, _vp, _vp]
        _or = L
    return _or


def have_ref() -> bool:
    return os.path.exists(REF_LIB)


def _load_ref():
    global _ref
    if _ref is None:
        if not have_ref():
            raise OracleError("oracle/_ref/libstref.so missing (run make -C oracle where /root/reference exists)")
        L = C.CDLL(REF_LIB)
        L.ref_parallel_velocity.argtypes = [_sz, _vp, _vp, _vp, _vp, C.c_int, C.c_double, C.c_int,
                                            C.c_int, C.c_int, C.c_int, C.c_int, _dp, _u64p, _dp]
        L.ref_ctx_new.restype = _vp
        L.ref_ctx_new.argtypes = [_sz, _vp, _vp, _vp, _vp, C.c_int, C.c_double, C.c_int, C.c_int,
                                  C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double),
                                  C.POINTER(C.c_double), C.POINTER(C.c_int)]
        L.ref_ctx_free.argtypes = [_vp]
        L.ref_ctx_ncl.restype = _sz
        L.ref_ctx_ncl.argtypes = [_vp]
        L.ref_ctx_export_tree.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp]
        L.ref_ctx_moments.argtypes = [_vp, _vp, _vp, _vp, _vp]
        L.ref_ctx_eval.argtypes = [_vp, _sz, _vp, _vp, C.c_int, _dp, _vp, _u64p]
        L.ref_direct_at.argtypes = [_sz, _vp, _vp, _vp, _vp, C.c_int, C.c_int, _i64p, _sz, C.c_int, _dp]
        L.ref_naive_direct.argtypes = [_sz, _vp, _vp, _vp, _vp, C.c_int, C.c_int, _dp]
        L.ref_coulomb.argtypes = [_dp, C.c_int, _dp]
        L.ref_taylor.argtypes = [_dp, C.c_int, C.c_int, _vp, _vp]
        L.ref_farfield_pair.argtypes = [_dp, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp, _vp, _dp]
        L.ref_relative_error.argtypes = [_sz, _dp, _dp, C.POINTER(C.c_double)]
        L.ref_sphere_particles.argtypes = [C.c_int, C.c_uint64, _dp, _dp, _dp, _dp]
        L.ref_cube_particles.argtypes = [_sz, C.c_double, C.c_uint64, _dp, _dp]
        L.ref_write_particles.argtypes = [C.c_char_p, _sz, _vp, _vp, _vp, _vp, C.c_int, C.c_int]
        L.ref_read_particles.argtypes = [C.c_char_p, _sz, C.POINTER(_sz), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                         _dp, _dp, _dp, _dp]
        _ref = L
    return _ref


def _arrs(ps):
    """ps: dict/obj with position, force_weight, dipole_weight, normal as (n,3) float64 or None."""
    get = (lambda k: ps.get(k)) if isinstance(ps, dict) else (lambda k: getattr(ps, k, None))
    keep = []
    ptrs = []
    for k in ("position", "force_weight", "dipole_weight", "normal"):
        a = get(k)
        if a is None or len(a) == 0:
            ptrs.append(None)
        else:
            a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1, 3)
            keep.append(a)
            ptrs.append(a.ctypes.data_as(C.c_void_p))
    n = len(get("position"))
    return n, ptrs, keep


def mi_count(p: int) -> int:
    return (p + 1) * (p + 2) * (p + 3) // 6


class Tree:
    """Exported cluster tree (same arrays from either checker)."""

    def __init__(self, ncl, be, geom, kids, meta, perm):
        self.ncl = ncl
        self.begin = be[:, 0]
        self.end = be[:, 1]
        self.center = geom[:, 0:3]
        self.radius = geom[:, 3]
        self.lo = geom[:, 4:7]
        self.hi = geom[:, 7:10]
        self.geom = geom
        self.children = kids
        self.n_children = meta[:, 0]
        self.is_leaf = meta[:, 1]
        self.to_original = perm

    @staticmethod
    def _export(fn, h, ncl, n):
        be = np.zeros((ncl, 2), np.int64)
        geom = np.zeros((ncl, 10), np.float64)
        kids = np.zeros((ncl, 8), np.int32)
        meta = np.zeros((ncl, 2), np.int32)
        perm = np.zeros(n, np.uint32)
        fn(h, be.ctypes.data, geom.ctypes.data, kids.ctypes.data, meta.ctypes.data, perm.ctypes.data)
        return Tree(ncl, be, geom, kids, meta, perm)


# ---------------------------------------------------------------- C restatement
def or_build_tree(ps, leaf_capacity: int, shrink: bool):
    L = _load_or()
    n, p, _keep = _arrs(ps)
    st = C.c_int(0)
    h = L.or_tree_build(n, p[0], p[1], p[2], p[3], leaf_capacity, int(shrink), C.byref(st))
    _check(st.value, "or_tree_build")
    try:
        return Tree._export(L.or_tree_export, h, L.or_tree_ncl(h), n)
    finally:
        L.or_tree_free(h)


def or_moments(ps, leaf_capacity, shrink, p, sto=True, stre=True):
    L = _load_or()
    n, ptr, _keep = _arrs(ps)
    st = C.c_int(0)
    h = L.or_tree_build(n, ptr[0], ptr[1], ptr[2], ptr[3], leaf_capacity, int(shrink), C.byref(st))
    _check(st.value, "or_tree_build")
    try:
        ncl = L.or_tree_ncl(h)
        E = mi_count(p)
        out = {k: np.zeros(ncl * m * E) for k, m in (("stok", 3), ("str", 9), ("trace", 1), ("sym", 6))}
        _check(L.or_moments(h, p, int(sto), int(stre), out["stok"].ctypes.data, out["str"].ctypes.data,
                            out["trace"].ctypes.data, out["sym"].ctypes.data), "or_moments")
        return {k: v.reshape(ncl, E, -1) for k, v in out.items()}
    finally:
        L.or_tree_free(h)


def or_coulomb(dx, pmax):
    b = np.zeros(mi_count(pmax) + 1)
    _check(_load_or().or_coulomb(np.ascontiguousarray(dx, np.float64), pmax, b), "or_coulomb")
    return b


def or_taylor(dx, order, pmax_b=None, sto=True, stre=True, b=None):
    """taylor_coeffs.hpp:13-46 for every multi-index of grade <= order:
    (a_sto[E,3,3] or None, a_str[E,3,3,3] or None); b defaults to or_coulomb(dx, pmax_b)."""
    pmax_b = order + (2 if stre else 1) if pmax_b is None else pmax_b
    b = or_coulomb(dx, pmax_b) if b is None else np.ascontiguousarray(b, np.float64)
    E = mi_count(order)
    a = np.zeros((E, 3, 3)) if sto else None
    t = np.zeros((E, 3, 3, 3)) if stre else None
    _check(_load_or().or_taylor(np.ascontiguousarray(dx, np.float64), b, pmax_b, order, _opt(a), _opt(t)),
           "or_taylor")
    return a, t


def or_farfield_pair(dx, p, stok=None, strm=None, trace=None, sym=None):
    u = np.zeros(3)
    _check(_load_or().or_farfield_pair(np.ascontiguousarray(dx, np.float64), p, int(stok is not None),
                                       int(strm is not None), _opt(stok), _opt(strm), _opt(trace),
                                       _opt(sym), u), "or_farfield_pair")
    return u


def or_treecode(ps, order, theta, leaf_capacity, shrink=True, sto=True, stre=True, targets=None,
                threads=None, per_target=False):
    """Returns (u[n_t,3] original order, stats dict, per-target counts[n_t,3] or None)."""
    L = _load_or()
    n, p, _keep = _arrs(ps)
    tg = None if targets is None else np.ascontiguousarray(targets, np.float64).reshape(-1, 3)
    nt = n if tg is None else len(tg)
    u = np.zeros((nt, 3))
    pt = np.zeros((nt, 3), np.uint64) if per_target else None
    s3 = np.zeros(3, np.uint64)
    threads = threads or os.cpu_count() or 1
    _check(L.or_treecode(n, p[0], p[1], p[2], p[3], None if tg is None else tg.ctypes.data, nt, order,
                         theta, leaf_capacity, int(shrink), int(sto), int(stre), threads, u.reshape(-1),
                         None if pt is None else pt.ctypes.data, s3), "or_treecode")
    stats = dict(farfield_evals=int(s3[0]), direct_pairs=int(s3[1]), clusters_visited=int(s3[2]))
    return u, stats, pt


def or_lists(ps, leaf_capacity, shrink, theta, tree_idx=None, xyz=None, cap=4096):
    """Per-target interaction lists (DFS order) for selected targets (tree indices or points)."""
    L = _load_or()
    n, p, _keep = _arrs(ps)
    st = C.c_int(0)
    h = L.or_tree_build(n, p[0], p[1], p[2], p[3], leaf_capacity, int(shrink), C.byref(st))
    _check(st.value, "or_tree_build")
    try:
        if xyz is not None:
            xyz = np.ascontiguousarray(xyz, np.float64).reshape(-1, 3)
            ns = len(xyz)
            ti = None
        else:
            ti = np.ascontiguousarray(tree_idx, np.uint32)
            ns = len(ti)
        far = np.full((ns, cap), -1, np.int32)
        near = np.full((ns, cap), -1, np.int32)
        nf = np.zeros(ns, np.int64)
        nn = np.zeros(ns, np.int64)
        _check(L.or_lists(h, theta, ns, None if ti is None else ti.ctypes.data,
                          None if xyz is None else xyz.ctypes.data, cap, far, near, nf, nn), "or_lists")
        return [far[i, :nf[i]].copy() for i in range(ns)], [near[i, :nn[i]].copy() for i in range(ns)]
    finally:
        L.or_tree_free(h)


def or_direct_at(ps, targets, sto=True, stre=True, threads=None):
    L = _load_or()
    n, p, _keep = _arrs(ps)
    tg = np.ascontiguousarray(targets, np.int64)
    u = np.zeros((len(tg), 3))
    _check(L.or_direct_at(n, p[0], p[1], p[2], p[3], int(sto), int(stre), tg, len(tg),
                          threads or os.cpu_count() or 1, u.reshape(-1)), "or_direct_at")
    return u


def or_direct_points(ps, xyz, sto=True, stre=True, threads=1):
    """Direct sum at disjoint points; `threads` host threads each take a contiguous block of
    points (ctypes releases the GIL during the C call)."""
    L = _load_or()
    n, p, _keep = _arrs(ps)
    xyz = np.ascontiguousarray(xyz, np.float64).reshape(-1, 3)
    u = np.zeros((len(xyz), 3))
    nt = len(xyz)
    threads = max(1, min(threads, nt))
    cuts = [nt * k // threads for k in range(threads + 1)]

    def part(k):
        a, b = cuts[k], cuts[k + 1]
        if b > a:
            _check(L.or_direct_points(n, p[0], p[1], p[2], p[3], int(sto), int(stre), xyz[a:b].reshape(-1), b - a,
                                      u[a:b].reshape(-1)), "or_direct_points")

    if threads == 1:
        part(0)
    else:
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(part, range(threads)))
    return u


def or_mac(radius, dist2, theta) -> bool:
    return bool(_load_or().or_mac(radius, dist2, theta))


def relative_error(u_ref, u_test) -> float:
    a = np.ascontiguousarray(u_ref, np.float64).reshape(-1)
    b = np.ascontiguousarray(u_test, np.float64).reshape(-1)
    if a.size != b.size:
        raise InvalidArgument("relative_error: field lengths differ")
    if a.size == 0:
        raise InvalidArgument("relative_error: empty fields")
    out = C.c_double(0)
    _check(_load_or().or_relative_error(a.size // 3, a, b, C.byref(out)), "relative_error")
    return out.value


# ---------------------------------------------------------------- reference in place
def ref_parallel_velocity(ps, order, theta, leaf_capacity, shrink=True, sto=True, stre=True, workers=1):
    L = _load_ref()
    n, p, _keep = _arrs(ps)
    u = np.zeros((n, 3))
    s3 = np.zeros(3, np.uint64)
    t4 = np.zeros(4)
    _check(L.ref_parallel_velocity(n, p[0], p[1], p[2], p[3], order, theta, leaf_capacity, int(shrink),
                                   int(sto), int(stre), workers, u.reshape(-1), s3, t4),
           "ref_parallel_velocity")
    stats = dict(farfield_evals=int(s3[0]), direct_pairs=int(s3[1]), clusters_visited=int(s3[2]))
    times = dict(build=t4[0], moments=t4[1], traverse=t4[2], total=t4[3])
    return u, stats, times


class RefContext:
    """Reference tree + moments built once; evaluate sampled or disjoint targets."""

    def __init__(self, ps, order, theta, leaf_capacity, shrink=True, sto=True, stre=True, workers=1):
        L = _load_ref()
        self.L = L
        n, p, self._keep = _arrs(ps)
        self.n = n
        self.order = order
        self.sto, self.stre = sto, stre
        tb, tm, st = C.c_double(0), C.c_double(0), C.c_int(0)
        self.h = L.ref_ctx_new(n, p[0], p[1], p[2], p[3], order, theta, leaf_capacity, int(shrink),
                               int(sto), int(stre), workers, C.byref(tb), C.byref(tm), C.byref(st))
        _check(st.value, "ref_ctx_new")
        self.t_build, self.t_moments = tb.value, tm.value

    def close(self):
        if self.h:
            self.L.ref_ctx_free(self.h)
            self.h = None

    __del__ = close

    def tree(self) -> Tree:
        return Tree._export(self.L.ref_ctx_export_tree, self.h, self.L.ref_ctx_ncl(self.h), self.n)

    def moments(self):
        ncl = self.L.ref_ctx_ncl(self.h)
        E = mi_count(self.order)
        out = {k: np.zeros(ncl * m * E) for k, m in (("stok", 3), ("str", 9), ("trace", 1), ("sym", 6))}
        self.L.ref_ctx_moments(self.h, out["stok"].ctypes.data, out["str"].ctypes.data,
                               out["trace"].ctypes.data, out["sym"].ctypes.data)
        return {k: v.reshape(ncl, E, -1) for k, v in out.items()}

    def eval(self, src_idx=None, xyz=None, threads=1):
        """Velocities (+ per-target visited/far/direct) at source indices or disjoint points."""
        if xyz is not None:
            xyz = np.ascontiguousarray(xyz, np.float64).reshape(-1, 3)
            nt = len(xyz)
            si = None
        else:
            si = np.ascontiguousarray(src_idx, np.int64)
            nt = len(si)
        u = np.zeros((nt, 3))
        pt = np.zeros((nt, 3), np.uint64)
        s3 = np.zeros(3, np.uint64)
        _check(self.L.ref_ctx_eval(self.h, nt, None if si is None else si.ctypes.data,
                                   None if xyz is None else xyz.ctypes.data, threads, u.reshape(-1),
                                   pt.ctypes.data, s3), "ref_ctx_eval")
        stats = dict(farfield_evals=int(s3[0]), direct_pairs=int(s3[1]), clusters_visited=int(s3[2]))
        return u, pt, stats


def ref_direct_at(ps, targets, sto=True, stre=True, threads=None):
    L = _load_ref()
    n, p, _keep = _arrs(ps)
    tg = np.ascontiguousarray(targets, np.int64)
    u = np.zeros((len(tg), 3))
    _check(L.ref_direct_at(n, p[0], p[1], p[2], p[3], int(sto), int(stre), tg, len(tg),
                           threads or os.cpu_count() or 1, u.reshape(-1)), "ref_direct_at")
    return u


def ref_naive_direct(ps, sto=True, stre=True):
    L = _load_ref()
    n, p, _keep = _arrs(ps)
    u = np.zeros((n, 3))
    _check(L.ref_naive_direct(n, p[0], p[1], p[2], p[3], int(sto), int(stre), u.reshape(-1)),
           "ref_naive_direct")
    return u


def ref_coulomb(dx, pmax):
    b = np.zeros(mi_count(pmax) + 1)
    _check(_load_ref().ref_coulomb(np.ascontiguousarray(dx, np.float64), pmax, b), "ref_coulomb")
    return b


def ref_taylor(dx, order, pmax_b=None, sto=True, stre=True):
    pmax_b = order + (2 if stre else 1) if pmax_b is None else pmax_b
    E = mi_count(order)
    a = np.zeros((E, 3, 3)) if sto else None
    t = np.zeros((E, 3, 3, 3)) if stre else None
    _check(_load_ref().ref_taylor(np.ascontiguousarray(dx, np.float64), pmax_b, order, _opt(a), _opt(t)),
           "ref_taylor")
    return a, t


def ref_farfield_pair(dx, p, stok=None, strm=None, trace=None, sym=None):
    u = np.zeros(3)
    _check(_load_ref().ref_farfield_pair(np.ascontiguousarray(dx, np.float64), p, int(stok is not None),
                                         int(strm is not None), _opt(stok), _opt(strm), _opt(trace),
                                         _opt(sym), u), "ref_farfield_pair")
    return u


def ref_sphere_particles(levels, seed):
    n = 20 * 4 ** levels
    a = [np.zeros((n, 3)) for _ in range(4)]
    _check(_load_ref().ref_sphere_particles(levels, seed, *[x.reshape(-1) for x in a]), "ref_sphere_particles")
    return dict(position=a[0], force_weight=a[1], dipole_weight=a[2], normal=a[3])


def ref_cube_particles(n, density, seed):
    a = [np.zeros((n, 3)) for _ in range(2)]
    _check(_load_ref().ref_cube_particles(n, density, seed, a[0].reshape(-1), a[1].reshape(-1)), "ref_cube_particles")
    return dict(position=a[0], force_weight=a[1])


def ref_write_particles(path, ps, sto=True, stre=True):
    n, p, _keep = _arrs(ps)
    _check(_load_ref().ref_write_particles(os.fsencode(str(path)), n, p[0], p[1], p[2], p[3], int(sto), int(stre)),
           "ref_write_particles")


def ref_read_particles(path, cap):
    a = [np.zeros((cap, 3)) for _ in range(4)]
    n, sto, stre = C.c_size_t(), C.c_int(), C.c_int()
    _check(_load_ref().ref_read_particles(os.fsencode(str(path)), cap, C.byref(n), C.byref(sto), C.byref(stre),
                                          *[x.reshape(-1) for x in a]), "ref_read_particles")
    k = n.value
    return dict(position=a[0][:k], force_weight=a[1][:k] if sto.value else None,
                dipole_weight=a[2][:k] if stre.value else None, normal=a[3][:k] if stre.value else None)


# ---------------------------------------------------------------- seeded inputs
GEN_KINDS = {"unit": 0, "cube": 1, "sphere": 2, "mixture": 3, "points": 4}


def generate(kind: str, n: int, seed: int, with_stresslets: bool = True) -> dict:
    """Seeded BASELINE inputs from the oracle's own C generator (or_generate; the recipes of
    DESIGN.md section 7).  The reference arm of bench.py builds its inputs with this, so it
    never loads the product library; tests/test_inputs_io.py pins the bytes to the
    product's st_generate by SHA-256."""
    L = _load_or()
    k = GEN_KINDS[kind]
    pos = np.empty((n, 3))
    f = None if k == 4 else np.empty((n, 3))
    h = np.empty((n, 3)) if (with_stresslets and k != 4) else None
    nu = np.empty((n, 3)) if (with_stresslets and k != 4) else None
    _check(L.or_generate(k, n, seed, 1 if with_stresslets else 0, _opt_out(pos), _opt_out(f), _opt_out(h),
                         _opt_out(nu)), "or_generate")
    if k == 4:
        return dict(position=pos)
    return dict(position=pos, force_weight=f, dipole_weight=h, normal=nu)


def _opt_out(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------- seeded inputs (pure Python)
_M64 = (1 << 64) - 1


class SplitMix64:
    """Restatement of rng.hpp:10-29 for small-n cross-checks of the product generator."""

    def __init__(self, seed: int):
        self.s = seed & _M64

    def next(self) -> int:
        self.s = (self.s + 0x9E3779B97F4A7C15) & _M64
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        return z ^ (z >> 31)

    def uniform01(self) -> float:
        return float(self.next() >> 11) * 2.0 ** -53

    def symmetric(self) -> float:
        return 2.0 * self.uniform01() - 1.0

    def unit(self):
        """testutil::random_unit (tests/support/test_helpers.hpp:22-28)."""
        while True:
            v = np.array([self.symmetric(), self.symmetric(), self.symmetric()])
            n2 = v[0] * v[0] + v[1] * v[1] + v[2] * v[2]
            if n2 > 1e-4 and n2 <= 1.0:
                return v * (1.0 / np.sqrt(n2))


def random_particles_py(n, seed, with_stresslets, lo=0.0, hi=1.0):
    """testutil::random_particles (tests/support/test_helpers.hpp:31-49), box [lo,hi)."""
    r = SplitMix64(seed)
    pos = np.zeros((n, 3)); f = np.zeros((n, 3))
    h = np.zeros((n, 3)) if with_stresslets else None
    nu = np.zeros((n, 3)) if with_stresslets else None
    for i in range(n):
        pos[i] = [lo + (hi - lo) * r.uniform01() for _ in range(3)]
        f[i] = [r.symmetric() for _ in range(3)]
        if with_stresslets:
            h[i] = [r.symmetric() for _ in range(3)]
            nu[i] = r.unit()
    return dict(position=pos, force_weight=f, dipole_weight=h, normal=nu)
