"""B200-native Stokeslet/stresslet treecode (arXiv 1811.12498 hot path).

Python mirror of the reference's public C++ API (namespace ``stokestree`` in
/root/reference/proj/include/stokestree/*.hpp) over the C ABI of
``libstokestree_b200.so`` (include/stokestree_c.h).  Names, argument meaning
and error behaviour follow the reference:

=========================================  ==========================================
reference (file:line)                      here
=========================================  ==========================================
KernelSelection (particles.hpp:13-25)       KernelSelection
ParticleSet / validate (particles.hpp:29-70) ParticleSet (arrays are (n, 3) float64)
TreecodeParams (engine.hpp:21-42)           TreecodeParams (+ ``devices``)
TraversalStats, VelocityResult (:44-64)     TraversalStats, VelocityResult
treecode_velocity (engine.hpp:185-189)      treecode_velocity
parallel_velocity (engine.hpp:194-196)      parallel_velocity
contracted_direct_velocity (kernels.hpp)    contracted_direct_velocity(_at)
naive_direct_velocity (kernels.hpp:89-118)  naive_direct_velocity
build_tree (cluster_tree.hpp:152-192)       build_tree -> ClusterTree
compute_moments (moments.hpp:140-175)       compute_moments -> ClusterMoments
coulomb_coeffs (coulomb.hpp:52-59)          coulomb_coeffs (batched)
stokeslet/stresslet_farfield (farfield.hpp) farfield_pairs (batched)
relative_error (error_metric.hpp:13-24)     relative_error
=========================================  ==========================================

std::invalid_argument -> :class:`InvalidArgument` (a ValueError),
std::domain_error -> :class:`DomainError` (an ArithmeticError), CUDA/runtime
failures -> :class:`StokesTreeError` (a RuntimeError).  There is no CPU
fallback: every compute call runs the sm_100a kernels and fails loudly without
a device or without the built library.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

__all__ = [
    "KernelSelection", "ParticleSet", "TreecodeParams", "TraversalStats", "VelocityResult",
    "ClusterTree", "ClusterMoments", "InvalidArgument", "DomainError", "StokesTreeError",
    "treecode_velocity", "parallel_velocity", "treecode_velocity_targets",
    "treecode_velocity_device", "treecode_velocity_sweep", "contracted_direct_velocity", "contracted_direct_velocity_at",
    "naive_direct_velocity", "build_tree", "compute_moments", "coulomb_coeffs",
    "farfield_pairs", "taylor_coeffs", "relative_error", "interaction_lists", "generate", "shard_cuts", "fp64_peak", "device_count",
    "mi_count", "lib_path", "load_library", "EXPORTED_SYMBOLS", "sphere_particles", "cube_particles",
    "write_particles", "read_particles", "treecode_velocity_sweep",
    "ipc_export", "ipc_open", "ipc_close", "release_workspace", "treecode_velocity_device_split",
    "ShardExchange",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
# ST_LIB_PATH: load another build of the library (A/B checks of kernel changes)
lib_path = os.environ.get("ST_LIB_PATH") or os.path.join(_HERE, "libstokestree_b200.so")

# every symbol declared in include/stokestree_c.h
EXPORTED_SYMBOLS = (
    "st_abi_version", "st_last_error", "st_device_count", "st_params_validate",
    "st_treecode_velocity", "st_treecode_velocity_ex", "st_treecode_velocity_device",
    "st_treecode_velocity_device_ev", "st_treecode_velocity_device_ev2",
    "st_direct_velocity", "st_direct_velocity_at", "st_naive_direct_velocity", "st_build_tree",
    "st_tree_num_clusters", "st_tree_num_particles", "st_tree_export", "st_tree_free",
    "st_compute_moments", "st_coulomb_coeffs", "st_farfield_pairs", "st_relative_error",
    "st_shard_cuts", "st_generate", "st_fp64_peak", "st_interaction_lists", "st_treecode_velocity_sweep",
    "st_sphere_count", "st_generate_sphere_icosa", "st_generate_cube_density", "st_write_particles",
    "st_read_particles", "st_loaded_copy", "st_loaded_free", "st_treecode_shard_device", "st_unbatch_device",
    "st_taylor_coeffs", "st_ipc_export", "st_ipc_open", "st_ipc_close", "st_release_workspace",
    "st_treecode_velocity_device_split", "st_nccl_unique_id", "st_nccl_comm_init", "st_nccl_comm_free",
    "st_treecode_velocity_nccl",
)

GEN_UNIT, GEN_CUBE, GEN_SPHERE, GEN_MIXTURE, GEN_POINTS = range(5)
_GEN = {"unit": GEN_UNIT, "cube": GEN_CUBE, "sphere": GEN_SPHERE, "mixture": GEN_MIXTURE,
        "points": GEN_POINTS}


class StokesTreeError(RuntimeError):
    """CUDA / NCCL / runtime failure (std::runtime_error in the reference)."""


class InvalidArgument(ValueError):
    """std::invalid_argument."""


class DomainError(ArithmeticError):
    """std::domain_error (coincident points, zero displacement, zero reference field)."""


# ------------------------------------------------------------------ C structs
class _Particles(C.Structure):
    _fields_ = [("n", C.c_size_t), ("position", C.c_void_p), ("force_weight", C.c_void_p),
                ("dipole_weight", C.c_void_p), ("normal", C.c_void_p)]


class _Params(C.Structure):
    _fields_ = [("order", C.c_int), ("theta", C.c_double), ("leaf_capacity", C.c_int),
                ("shrink", C.c_int), ("stokeslet", C.c_int), ("stresslet", C.c_int),
                ("workers", C.c_int), ("devices", C.c_int)]


class _Stats(C.Structure):
    _fields_ = [("farfield_evals", C.c_uint64), ("direct_pairs", C.c_uint64),
                ("clusters_visited", C.c_uint64), ("time_build_s", C.c_double),
                ("time_moments_s", C.c_double), ("time_traverse_s", C.c_double),
                ("time_total_s", C.c_double), ("time_far_s", C.c_double),
                ("time_near_s", C.c_double), ("time_h2d_s", C.c_double),
                ("time_d2h_s", C.c_double), ("gpu_launches", C.c_uint64)]


class ShardExchange(C.Structure):
    """st_shard_exchange (stokestree_c.h): the split moment pass's buffers on this rank."""
    _fields_ = [("shard", C.c_int), ("n_shards", C.c_int), ("w", C.c_void_p), ("w_row", C.c_size_t),
                ("ncl", C.c_size_t), ("w_cuts", C.POINTER(C.c_size_t)), ("m", C.c_void_p), ("m_row", C.c_size_t),
                ("n_units", C.c_size_t), ("m_cuts", C.POINTER(C.c_size_t)), ("stream", C.c_void_p)]

    def cuts(self, which):
        p = self.w_cuts if which == "w" else self.m_cuts
        return [int(p[i]) for i in range(self.n_shards + 1)]


EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(ShardExchange))

_lib = None


def load_library():
    """Load the in-tree CUDA library; raise loudly when it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(lib_path):
        raise StokesTreeError(
            f"CUDA library {lib_path} is missing: build it with `make -C paper_1811_12498_b200` "
            "(or __graft_entry__.build()); there is no CPU fallback")
    L = C.CDLL(lib_path)
    vp, sz, i, d = C.c_void_p, C.c_size_t, C.c_int, C.c_double
    P = C.POINTER
    L.st_abi_version.restype = i
    L.st_last_error.restype = C.c_char_p
    L.st_device_count.argtypes = [P(i)]
    L.st_params_validate.argtypes = [P(_Params)]
    L.st_treecode_velocity.argtypes = [P(_Particles), P(_Params), vp, P(_Stats)]
    L.st_treecode_velocity_ex.argtypes = [P(_Particles), vp, sz, P(_Params), vp, vp, P(_Stats)]
    L.st_treecode_velocity_device.argtypes = [P(_Particles), vp, sz, P(_Params), vp, i, i, vp, P(_Stats)]
    L.st_treecode_velocity_device_ev.argtypes = [P(_Particles), vp, sz, P(_Params), vp, i, i, vp, vp, P(_Stats)]
    L.st_treecode_velocity_device_ev2.argtypes = [P(_Particles), vp, sz, P(_Params), vp, i, i, vp, vp, vp,
                                                  P(_Stats)]
    L.st_direct_velocity.argtypes = [P(_Particles), i, i, sz, sz, vp]
    L.st_direct_velocity_at.argtypes = [P(_Particles), i, i, vp, sz, vp]
    L.st_naive_direct_velocity.argtypes = [P(_Particles), i, i, vp]
    L.st_build_tree.argtypes = [P(_Particles), i, i, P(vp)]
    L.st_tree_num_clusters.restype = sz
    L.st_tree_num_clusters.argtypes = [vp]
    L.st_tree_num_particles.restype = sz
    L.st_tree_num_particles.argtypes = [vp]
    L.st_tree_export.argtypes = [vp, vp, vp, vp, vp, vp]
    L.st_tree_free.argtypes = [vp]
    L.st_tree_free.restype = None
    L.st_compute_moments.argtypes = [vp, i, i, i, vp, vp, vp, vp]
    L.st_coulomb_coeffs.argtypes = [sz, vp, i, vp]
    L.st_taylor_coeffs.argtypes = [sz, vp, vp, i, i, vp, vp]
    L.st_farfield_pairs.argtypes = [sz, vp, i, i, i, vp, vp, vp, vp, vp]
    L.st_relative_error.argtypes = [sz, vp, vp, P(d)]
    L.st_shard_cuts.argtypes = [sz, vp, i, vp]
    L.st_generate.argtypes = [i, sz, C.c_uint64, i, vp, vp, vp, vp]
    L.st_fp64_peak.argtypes = [d, P(d)]
    L.st_treecode_velocity_sweep.argtypes = [P(_Particles), vp, sz, P(_Params), vp, i, vp, vp, P(_Stats)]
    L.st_interaction_lists.argtypes = [P(_Particles), P(_Params), vp, vp, sz, sz, vp, vp, vp, vp]
    L.st_treecode_shard_device.argtypes = [P(_Particles), vp, sz, P(_Params), i, i, vp, vp, P(sz), P(sz), vp,
                                           P(_Stats)]
    L.st_unbatch_device.argtypes = [sz, vp, vp, vp, vp]
    L.st_ipc_export.argtypes = [vp, C.c_char_p, C.POINTER(sz)]
    L.st_ipc_open.argtypes = [C.c_char_p, sz, C.POINTER(vp)]
    L.st_ipc_close.argtypes = [vp]
    L.st_nccl_unique_id.argtypes = [C.c_char_p]
    L.st_nccl_comm_init.argtypes = [C.c_char_p, i, i, P(vp)]
    L.st_nccl_comm_free.argtypes = [vp]
    L.st_nccl_comm_free.restype = None
    L.st_treecode_velocity_nccl.argtypes = [P(_Particles), vp, sz, P(_Params), vp, vp, vp, P(_Stats)]
    L.st_sphere_count.restype = sz
    L.st_sphere_count.argtypes = [i]
    L.st_generate_sphere_icosa.argtypes = [i, C.c_uint64, vp, vp, vp, vp]
    L.st_generate_cube_density.argtypes = [sz, d, C.c_uint64, vp, vp]
    L.st_write_particles.argtypes = [C.c_char_p, P(_Particles), i, i]
    L.st_read_particles.argtypes = [C.c_char_p, P(vp), P(sz), P(i), P(i)]
    L.st_loaded_copy.argtypes = [vp, vp, vp, vp, vp]
    L.st_loaded_free.argtypes = [vp]
    L.st_loaded_free.restype = None
    L.st_release_workspace.argtypes = []
    L.st_treecode_velocity_device_split.argtypes = [P(_Particles), vp, sz, P(_Params), vp, i, i, vp, EXCHANGE_FN,
                                                    vp, P(_Stats)]
    for name in EXPORTED_SYMBOLS:
        if name not in ("st_abi_version", "st_last_error", "st_tree_num_clusters",
                        "st_tree_num_particles", "st_tree_free", "st_sphere_count", "st_loaded_free"):
            getattr(L, name).restype = i
    _lib = L
    return L


def _check(code: int):
    if code == 0:
        return
    msg = load_library().st_last_error().decode()
    if code == 1:
        raise InvalidArgument(msg)
    if code == 2:
        raise DomainError(msg)
    raise StokesTreeError(msg)


def mi_count(p: int) -> int:
    """Entries with |k| <= p (multi_index.hpp:19-20)."""
    return (p + 1) * (p + 2) * (p + 3) // 6


# ------------------------------------------------------------------ data model
@dataclass(frozen=True)
class KernelSelection:
    stokeslet_enabled: bool = True
    stresslet_enabled: bool = True

    @staticmethod
    def stokeslet_only():
        return KernelSelection(True, False)

    @staticmethod
    def stresslet_only():
        return KernelSelection(False, True)

    @staticmethod
    def both():
        return KernelSelection(True, True)


def _as3(a):
    if a is None:
        return None
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.size == 0:
        return None
    return a.reshape(-1, 3)


@dataclass
class ParticleSet:
    """Structure of arrays, (n, 3) float64 each; h / nu may be None without stresslets."""
    position: np.ndarray
    force_weight: Optional[np.ndarray] = None
    dipole_weight: Optional[np.ndarray] = None
    normal: Optional[np.ndarray] = None

    def __post_init__(self):
        self.position = _as3(self.position)
        if self.position is None:
            self.position = np.zeros((0, 3))
        self.force_weight = _as3(self.force_weight)
        self.dipole_weight = _as3(self.dipole_weight)
        self.normal = _as3(self.normal)

    def size(self) -> int:
        return len(self.position)

    def _c(self, sel: Optional[KernelSelection] = None) -> _Particles:
        n = len(self.position)

        def ptr(a, needed=True):
            if a is None or not needed:
                return None
            if len(a) != n:  # mismatched length: hand the library a NULL array
                return None
            return a.ctypes.data

        sto = True if sel is None else sel.stokeslet_enabled
        stre = True if sel is None else sel.stresslet_enabled
        return _Particles(n, ptr(self.position), ptr(self.force_weight, sto),
                          ptr(self.dipole_weight, stre), ptr(self.normal, stre))


@dataclass
class TreecodeParams:
    kMaxOrder = 16
    order: int = 6
    theta: float = 0.5
    leaf_capacity: int = 2000
    shrink: bool = True
    kernels: KernelSelection = field(default_factory=KernelSelection)
    workers: int = 1
    devices: int = 1

    def _c(self) -> _Params:
        return _Params(int(self.order), float(self.theta), int(self.leaf_capacity), int(bool(self.shrink)),
                       int(self.kernels.stokeslet_enabled), int(self.kernels.stresslet_enabled),
                       int(self.workers), int(self.devices))

    def validate(self):
        """TreecodeParams::validate (engine.hpp:31-41)."""
        p = self._c()
        _check(load_library().st_params_validate(C.byref(p)))


@dataclass
class TraversalStats:
    farfield_evals: int = 0
    direct_pairs: int = 0
    clusters_visited: int = 0


@dataclass
class VelocityResult:
    velocity: np.ndarray
    stats: TraversalStats
    time_build_s: float = 0.0
    time_moments_s: float = 0.0
    time_traverse_s: float = 0.0
    time_total_s: float = 0.0
    time_far_s: float = 0.0
    time_near_s: float = 0.0
    time_h2d_s: float = 0.0
    time_d2h_s: float = 0.0
    gpu_launches: int = 0
    per_target: Optional[np.ndarray] = None


def _result(u, s: _Stats, per_target=None) -> VelocityResult:
    return VelocityResult(u, TraversalStats(int(s.farfield_evals), int(s.direct_pairs), int(s.clusters_visited)),
                          s.time_build_s, s.time_moments_s, s.time_traverse_s, s.time_total_s, s.time_far_s,
                          s.time_near_s, s.time_h2d_s, s.time_d2h_s, int(s.gpu_launches), per_target)


# ------------------------------------------------------------------ the treecode
def treecode_velocity_targets(ps: ParticleSet, targets, params: TreecodeParams,
                              per_target: bool = False) -> VelocityResult:
    """Treecode at explicit targets (None: the sources themselves, self excluded)."""
    L = load_library()
    cp = ps._c(params.kernels)
    prm = params._c()
    tg = _as3(targets) if targets is not None else None
    if targets is not None and tg is None:
        raise InvalidArgument("targets: empty target set")
    nt = ps.size() if tg is None else len(tg)
    u = np.zeros((nt, 3))
    pt = np.zeros((nt, 3), np.uint64) if per_target else None
    st = _Stats()
    _check(L.st_treecode_velocity_ex(C.byref(cp), None if tg is None else tg.ctypes.data,
                                     0 if tg is None else len(tg), C.byref(prm), u.ctypes.data,
                                     None if pt is None else pt.ctypes.data, C.byref(st)))
    return _result(u, st, pt)


def treecode_velocity(ps: ParticleSet, params: TreecodeParams, per_target: bool = False) -> VelocityResult:
    """Single-worker treecode (engine.hpp:185-189); velocities in original order."""
    return treecode_velocity_targets(ps, None, params, per_target)


def parallel_velocity(ps: ParticleSet, params: TreecodeParams, per_target: bool = False) -> VelocityResult:
    """Replicated-data driver (engine.hpp:194-196); bit-identical to treecode_velocity."""
    return treecode_velocity_targets(ps, None, params, per_target)


def treecode_velocity_sweep(ps: ParticleSet, params: TreecodeParams, orders, targets=None):
    """Velocities at several orders from one tree / moment pass / near-field pass.

    Returns (u[n_orders, n_t, 3], far_seconds[n_orders], VelocityResult with the shared
    counters and phase times)."""
    L = load_library()
    cp = ps._c(params.kernels)
    prm = params._c()
    od = np.ascontiguousarray(orders, dtype=np.int32)
    tg = _as3(targets) if targets is not None else None
    nt = ps.size() if tg is None else len(tg)
    u = np.zeros((len(od), nt, 3))
    fs = np.zeros(len(od))
    st = _Stats()
    _check(L.st_treecode_velocity_sweep(C.byref(cp), None if tg is None else tg.ctypes.data,
                                        0 if tg is None else len(tg), C.byref(prm), od.ctypes.data, len(od),
                                        u.ctypes.data, fs.ctypes.data, C.byref(st)))
    return u, fs, _result(None, st)


def treecode_shard_device(position_ptr, force_ptr, dipole_ptr, normal_ptr, n, params, u_batch_ptr,
                          batch_to_original_ptr=None, targets_ptr=None, n_targets=0, shard=0, n_shards=1,
                          stream=0):
    """Shard in batch order for all-gathers; returns (t0, t1, VelocityResult)."""
    L = load_library()
    cp = _Particles(n, position_ptr, force_ptr, dipole_ptr, normal_ptr)
    prm = params._c()
    st = _Stats()
    t0, t1 = C.c_size_t(), C.c_size_t()
    _check(L.st_treecode_shard_device(C.byref(cp), targets_ptr, n_targets, C.byref(prm), shard, n_shards,
                                      u_batch_ptr, batch_to_original_ptr, C.byref(t0), C.byref(t1), stream,
                                      C.byref(st)))
    return t0.value, t1.value, _result(None, st)


def unbatch_device(n, batch_to_original_ptr, u_batch_ptr, u_out_ptr, stream=0):
    _check(load_library().st_unbatch_device(n, batch_to_original_ptr, u_batch_ptr, u_out_ptr, stream))


def nccl_unique_id() -> bytes:
    """128-byte NCCL id (st_nccl_unique_id): rank 0 makes it, every rank passes it to NcclComm."""
    b = C.create_string_buffer(128)
    _check(load_library().st_nccl_unique_id(b))
    return b.raw


class NcclComm:
    """The library's own NCCL communicator (st_nccl_comm_init) on the current CUDA device."""

    def __init__(self, unique_id: bytes, n_ranks: int, rank: int):
        if len(unique_id) != 128:
            raise InvalidArgument("nccl: the unique id is 128 bytes")
        h = C.c_void_p()
        _check(load_library().st_nccl_comm_init(unique_id, int(n_ranks), int(rank), C.byref(h)))
        self.handle, self.n_ranks, self.rank = h.value, n_ranks, rank

    def close(self):
        if self.handle:
            load_library().st_nccl_comm_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def treecode_velocity_nccl(position_ptr: int, force_ptr: Optional[int], dipole_ptr: Optional[int],
                           normal_ptr: Optional[int], n: int, params: TreecodeParams, u_out_ptr: int,
                           comm: NcclComm, targets_ptr: Optional[int] = None, n_targets: int = 0,
                           stream: int = 0) -> VelocityResult:
    """One rank's call of the multi-GPU treecode with NCCL inside the library
    (st_treecode_velocity_nccl): every rank holds all inputs on its device; u_out receives
    every target's velocity (original order) on every rank; stats are the whole job's."""
    L = load_library()
    cp = _Particles(n, position_ptr, force_ptr, dipole_ptr, normal_ptr)
    prm = params._c()
    st = _Stats()
    _check(L.st_treecode_velocity_nccl(C.byref(cp), targets_ptr, n_targets, C.byref(prm), u_out_ptr, comm.handle,
                                       stream, C.byref(st)))
    return _result(None, st)


def ipc_export(device_ptr: int):
    """(64-byte CUDA IPC handle, offset) of the allocation holding ``device_ptr``; another
    process opens it with ipc_open and can pass the result as ``u_out_ptr`` of
    treecode_velocity_device(shard=rank, n_shards=world): its epilogue then stores the
    shard straight into this buffer (NVLink peer stores, no gather)."""
    h = C.create_string_buffer(64)
    off = C.c_size_t(0)
    _check(load_library().st_ipc_export(device_ptr, h, C.byref(off)))
    return h.raw, off.value


def ipc_open(handle: bytes, offset: int) -> int:
    if len(handle) != 64:
        raise InvalidArgument("ipc_open: a CUDA IPC handle is 64 bytes")
    p = C.c_void_p(0)
    _check(load_library().st_ipc_open(handle, offset, C.byref(p)))
    return p.value


def ipc_close(device_ptr: int) -> None:
    _check(load_library().st_ipc_close(device_ptr))


def treecode_velocity_device(position_ptr: int, force_ptr: Optional[int], dipole_ptr: Optional[int],
                             normal_ptr: Optional[int], n: int, params: TreecodeParams, u_out_ptr: int,
                             targets_ptr: Optional[int] = None, n_targets: int = 0, shard: int = 0,
                             n_shards: int = 1, stream: int = 0, weights_event: int = 0,
                             targets_event: int = 0) -> VelocityResult:
    """Device-resident call: raw device pointers (e.g. torch ``data_ptr()``) and a CUDA stream.
    weights_event (a cudaEvent_t handle, e.g. torch.cuda.Event.cuda_event): the weight
    arrays may still be in flight until it completes (st_treecode_velocity_device_ev);
    targets_event: likewise the disjoint targets, waited for before they are ordered
    (st_treecode_velocity_device_ev2)."""
    L = load_library()
    cp = _Particles(n, position_ptr, force_ptr, dipole_ptr, normal_ptr)
    prm = params._c()
    st = _Stats()
    _check(L.st_treecode_velocity_device_ev2(C.byref(cp), targets_ptr, n_targets, C.byref(prm), u_out_ptr,
                                             shard, n_shards, stream, targets_event or None, weights_event or None,
                                             C.byref(st)))
    return _result(None, st)


def treecode_velocity_device_split(position_ptr: int, force_ptr: Optional[int], dipole_ptr: Optional[int],
                                   normal_ptr: Optional[int], n: int, params: TreecodeParams, u_out_ptr: int,
                                   exchange, targets_ptr: Optional[int] = None, n_targets: int = 0, shard: int = 0,
                                   n_shards: int = 1, stream: int = 0) -> VelocityResult:
    """Device-resident shard call with the moment pass split over the ranks
    (st_treecode_velocity_device_split).  ``exchange(ex: ShardExchange) -> None`` is called
    once, on the call's stream, to move every rank's weight rows and unit moments into this
    rank's buffers (e.g. NCCL broadcasts); an exception in it fails the call."""
    L = load_library()
    cp = _Particles(n, position_ptr, force_ptr, dipole_ptr, normal_ptr)
    prm = params._c()
    st = _Stats()
    err = []

    def cb(_ctx, exp):
        try:
            exchange(exp.contents)
            return 0
        except BaseException as e:  # reported through the call's status
            err.append(e)
            return 1

    fn = EXCHANGE_FN(cb)
    code = L.st_treecode_velocity_device_split(C.byref(cp), targets_ptr, n_targets, C.byref(prm), u_out_ptr, shard,
                                               n_shards, stream, fn, None, C.byref(st))
    if err:
        raise err[0]
    _check(code)
    return _result(None, st)


def interaction_lists(ps: ParticleSet, params: TreecodeParams, target_index=None, points=None, cap: int = 4096):
    """Per-target far (accepted cluster) and near (leaf) lists in DFS order, pre-order ids."""
    L = load_library()
    cp = ps._c(params.kernels)
    prm = params._c()
    if points is not None:
        pts = _as3(points)
        n = len(pts)
        ti = None
    else:
        ti = np.ascontiguousarray(target_index, dtype=np.uint64)
        n = len(ti)
        pts = None
    far = np.full((n, cap), -1, np.int32)
    near = np.full((n, cap), -1, np.int32)
    nf = np.zeros(n, np.int64)
    nn = np.zeros(n, np.int64)
    _check(L.st_interaction_lists(C.byref(cp), C.byref(prm), None if ti is None else ti.ctypes.data,
                                  None if pts is None else pts.ctypes.data, n, cap, far.ctypes.data,
                                  near.ctypes.data, nf.ctypes.data, nn.ctypes.data))
    return [far[i, :min(nf[i], cap)].copy() for i in range(n)], [near[i, :min(nn[i], cap)].copy() for i in range(n)]


# ------------------------------------------------------------------ direct sums
def contracted_direct_velocity(ps: ParticleSet, sel: KernelSelection, first: int = 0,
                               last: Optional[int] = None) -> np.ndarray:
    """contracted_direct_velocity (kernels.hpp:123-136)."""
    L = load_library()
    last = ps.size() if last is None else last
    if first < 0 or last < 0:
        raise InvalidArgument("contracted_direct_velocity: bad target range")
    cp = ps._c(sel)
    u = np.zeros((max(last - first, 0), 3))
    _check(L.st_direct_velocity(C.byref(cp), int(sel.stokeslet_enabled), int(sel.stresslet_enabled), first,
                                last, u.ctypes.data))
    return u


def contracted_direct_velocity_at(ps: ParticleSet, sel: KernelSelection, targets) -> np.ndarray:
    """contracted_direct_velocity_at (kernels.hpp:139-150)."""
    L = load_library()
    tg = np.ascontiguousarray(targets, dtype=np.int64)
    if (tg < 0).any():
        raise InvalidArgument("contracted_direct_velocity_at: target out of range")
    tg = tg.astype(np.uint64)
    cp = ps._c(sel)
    u = np.zeros((len(tg), 3))
    _check(L.st_direct_velocity_at(C.byref(cp), int(sel.stokeslet_enabled), int(sel.stresslet_enabled),
                                   tg.ctypes.data, len(tg), u.ctypes.data))
    return u


def naive_direct_velocity(ps: ParticleSet, sel: KernelSelection) -> np.ndarray:
    """naive_direct_velocity (kernels.hpp:89-118): tensor-forming O(N^2) sum."""
    L = load_library()
    cp = ps._c(sel)
    u = np.zeros((ps.size(), 3))
    _check(L.st_naive_direct_velocity(C.byref(cp), int(sel.stokeslet_enabled), int(sel.stresslet_enabled),
                                      u.ctypes.data))
    return u


# ------------------------------------------------------------------ tree + moments
class ClusterTree:
    """build_tree output (cluster_tree.hpp:34-43), exported to host arrays, pre-order."""

    def __init__(self, handle, n, leaf_capacity, shrink, particles: ParticleSet):
        L = load_library()
        self._h = handle
        self.leaf_capacity = leaf_capacity
        self.shrink = shrink
        ncl = L.st_tree_num_clusters(handle)
        be = np.zeros((ncl, 2), np.int64)
        geom = np.zeros((ncl, 10))
        kids = np.zeros((ncl, 8), np.int32)
        meta = np.zeros((ncl, 2), np.int32)
        perm = np.zeros(n, np.uint32)
        _check(L.st_tree_export(handle, be.ctypes.data, geom.ctypes.data, kids.ctypes.data, meta.ctypes.data,
                                perm.ctypes.data))
        self.ncl = ncl
        self.begin, self.end = be[:, 0], be[:, 1]
        self.geom = geom
        self.center, self.radius = geom[:, 0:3], geom[:, 3]
        self.lo, self.hi = geom[:, 4:7], geom[:, 7:10]
        self.children, self.n_children, self.is_leaf = kids, meta[:, 0], meta[:, 1]
        self.to_original = perm
        self.to_tree = np.empty_like(perm)
        self.to_tree[perm] = np.arange(n, dtype=np.uint32)
        src = particles
        self.particles = ParticleSet(src.position[perm],
                                     None if src.force_weight is None else src.force_weight[perm],
                                     None if src.dipole_weight is None else src.dipole_weight[perm],
                                     None if src.normal is None else src.normal[perm])

    @property
    def clusters(self):
        return range(self.ncl)

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h and _lib is not None:
            _lib.st_tree_free(h)


def build_tree(ps: ParticleSet, leaf_capacity: int, shrink: bool) -> ClusterTree:
    """build_tree (cluster_tree.hpp:152-192), on the device."""
    L = load_library()
    cp = ps._c(None)
    h = C.c_void_p()
    _check(L.st_build_tree(C.byref(cp), int(leaf_capacity), int(bool(shrink)), C.byref(h)))
    return ClusterTree(h.value, ps.size(), leaf_capacity, shrink, ps)


@dataclass
class ClusterMoments:
    """ClusterMoments (moments.hpp:85-134): [ncl, E, {3, 9, 1, 6}] arrays."""
    order: int
    stok: Optional[np.ndarray]
    str: Optional[np.ndarray]
    trace: Optional[np.ndarray]
    sym: Optional[np.ndarray]

    def entry_count(self) -> int:
        return mi_count(self.order)


def compute_moments(tree: ClusterTree, p: int, sel: KernelSelection) -> ClusterMoments:
    """compute_moments (moments.hpp:140-175), on the device."""
    L = load_library()
    E = mi_count(max(p, 0))
    ncl = tree.ncl
    sto, stre = sel.stokeslet_enabled, sel.stresslet_enabled
    a = np.zeros((ncl, E, 3)) if sto else None
    b = np.zeros((ncl, E, 9)) if stre else None
    c = np.zeros((ncl, E, 1)) if stre else None
    d = np.zeros((ncl, E, 6)) if stre else None
    ptr = lambda x: None if x is None else x.ctypes.data
    _check(L.st_compute_moments(tree._h, int(p), int(sto), int(stre), ptr(a), ptr(b), ptr(c), ptr(d)))
    return ClusterMoments(p, a, b, c, d)


def coulomb_coeffs(dx, pmax: int) -> np.ndarray:
    """b^k for |k| <= pmax at each displacement (coulomb.hpp:28-59), graded-lex order."""
    L = load_library()
    d = np.ascontiguousarray(dx, np.float64).reshape(-1, 3)
    b = np.zeros((len(d), mi_count(max(pmax, 0))))
    _check(L.st_coulomb_coeffs(len(d), d.ctypes.data, int(pmax), b.ctypes.data))
    return b


def taylor_coeffs(dx, order: int, stokeslet: bool = True, stresslet: bool = True, b=None, pmax_b=None):
    """Explicit Taylor coefficients (taylor_coeffs.hpp:13-46) for every multi-index of grade
    <= order at each displacement: (a_sto [n, E, 3, 3] or None, a_str [n, E, 3, 3, 3] or None),
    a_sto[q, e, i, j] = a^k_ij and a_str[q, e, i, j, l] = a~^k_ijl.  ``b`` [n, E(pmax_b)] as
    coulomb_coeffs returns it; None = formed on the device at depth order+2 (order+1 if
    only the Stokeslet is asked for)."""
    L = load_library()
    d = np.ascontiguousarray(dx, np.float64).reshape(-1, 3)
    bb = None if b is None else np.ascontiguousarray(b, np.float64).reshape(len(d), -1)
    if pmax_b is None:
        pmax_b = _grade_of_count(bb.shape[1]) if bb is not None else order + (2 if stresslet else 1)
    E = mi_count(max(order, 0))
    a = np.zeros((len(d), E, 3, 3)) if stokeslet else None
    t = np.zeros((len(d), E, 3, 3, 3)) if stresslet else None
    ptr = lambda x: None if x is None else x.ctypes.data
    _check(L.st_taylor_coeffs(len(d), d.ctypes.data, ptr(bb), int(pmax_b), int(order), ptr(a), ptr(t)))
    return a, t


def _grade_of_count(n: int) -> int:
    p = 0
    while mi_count(p) < n:
        p += 1
    if mi_count(p) != n:
        raise InvalidArgument(f"taylor_coeffs: {n} coefficients is not E(p) for any p")
    return p


def farfield_pairs(dx, p: int, stok=None, strm=None, trace=None, sym=None) -> np.ndarray:
    """stokeslet_farfield + stresslet_farfield (farfield.hpp:30-96) for batches of pairs.

    ``stok`` [n, E, 3] and ``strm`` [n, E, 9] are per-pair moment blocks in the
    reference layout; pass None to disable a kernel."""
    L = load_library()
    d = np.ascontiguousarray(dx, np.float64).reshape(-1, 3)
    a = None if stok is None else np.ascontiguousarray(stok, np.float64)
    b = None if strm is None else np.ascontiguousarray(strm, np.float64)
    u = np.zeros((len(d), 3))
    ptr = lambda x: None if x is None else x.ctypes.data
    _check(L.st_farfield_pairs(len(d), d.ctypes.data, int(p), int(a is not None), int(b is not None), ptr(a),
                               ptr(b), None, None, u.ctypes.data))
    return u


def relative_error(u_ref, u_test) -> float:
    """E = sqrt(sum |u_ref - u|^2 / sum |u_ref|^2) (error_metric.hpp:13-24)."""
    a = np.ascontiguousarray(u_ref, np.float64).reshape(-1)
    b = np.ascontiguousarray(u_test, np.float64).reshape(-1)
    if a.size != b.size:
        raise InvalidArgument("relative_error: field lengths differ")
    out = C.c_double(0)
    _check(load_library().st_relative_error(a.size // 3, a.ctypes.data, b.ctypes.data, C.byref(out)))
    return out.value


# ------------------------------------------------------------------ inputs / planning
def generate(kind: str, n: int, seed: int, with_stresslets: bool = True) -> ParticleSet:
    """Seeded synthetic inputs: unit | cube | sphere | mixture | points."""
    L = load_library()
    k = _GEN[kind]
    pos = np.zeros((n, 3))
    if k == GEN_POINTS:
        _check(L.st_generate(k, n, seed, 0, pos.ctypes.data, None, None, None))
        return ParticleSet(pos)
    f = np.zeros((n, 3))
    h = np.zeros((n, 3)) if with_stresslets else None
    nu = np.zeros((n, 3)) if with_stresslets else None
    ptr = lambda x: None if x is None else x.ctypes.data
    _check(L.st_generate(k, n, seed, int(with_stresslets), pos.ctypes.data, f.ctypes.data, ptr(h), ptr(nu)))
    return ParticleSet(pos, f, h, nu)


def sphere_particles(levels: int, seed: int) -> ParticleSet:
    """The paper's icosahedral sphere geometry, N = 20 * 4^levels (testcases.hpp:66-106)."""
    L = load_library()
    if levels < 0:
        raise InvalidArgument("sphere_particles: levels must be >= 0")
    n = L.st_sphere_count(int(levels))
    pos, f, h, nu = (np.zeros((n, 3)) for _ in range(4))
    _check(L.st_generate_sphere_icosa(int(levels), seed, pos.ctypes.data, f.ctypes.data, h.ctypes.data,
                                      nu.ctypes.data))
    return ParticleSet(pos, f, h, nu)


def cube_particles(n: int, density: float = 2500.0, seed: int = 0) -> ParticleSet:
    """Stokeslets uniform in a cube of side (n/density)^(1/3) (testcases.hpp:108-124)."""
    L = load_library()
    if n < 1:
        raise InvalidArgument("cube_particles: n must be >= 1")
    if not density > 0:
        raise InvalidArgument("cube_particles: density must be > 0")
    pos, f = np.zeros((n, 3)), np.zeros((n, 3))
    _check(L.st_generate_cube_density(int(n), float(density), seed, pos.ctypes.data, f.ctypes.data))
    return ParticleSet(pos, f)


def write_particles(path, ps: ParticleSet, sel: KernelSelection) -> None:
    """write_particles (particle_io.hpp:34-58)."""
    cp = ps._c(sel)
    _check(load_library().st_write_particles(os.fsencode(str(path)), C.byref(cp), int(sel.stokeslet_enabled),
                                             int(sel.stresslet_enabled)))


def read_particles(path):
    """read_particles (particle_io.hpp:60-126) -> (ParticleSet, KernelSelection)."""
    L = load_library()
    h = C.c_void_p()
    n, sto, stre = C.c_size_t(), C.c_int(), C.c_int()
    _check(L.st_read_particles(os.fsencode(str(path)), C.byref(h), C.byref(n), C.byref(sto), C.byref(stre)))
    try:
        pos = np.zeros((n.value, 3))
        f = np.zeros((n.value, 3)) if sto.value else None
        hh = np.zeros((n.value, 3)) if stre.value else None
        nu = np.zeros((n.value, 3)) if stre.value else None
        ptr = lambda x: None if x is None else x.ctypes.data
        _check(L.st_loaded_copy(h.value, pos.ctypes.data, ptr(f), ptr(hh), ptr(nu)))
    finally:
        L.st_loaded_free(h.value)
    return ParticleSet(pos, f, hh, nu), KernelSelection(bool(sto.value), bool(stre.value))


def shard_cuts(weights, n_shards: int) -> np.ndarray:
    """Contiguous work-balanced shard boundaries over per-unit weights."""
    w = np.ascontiguousarray(weights, np.float64)
    cuts = np.zeros(n_shards + 1, np.uint64)
    _check(load_library().st_shard_cuts(len(w), w.ctypes.data if len(w) else None, int(n_shards),
                                        cuts.ctypes.data))
    return cuts.astype(np.int64)


def fp64_peak(seconds: float = 0.2) -> float:
    """Measured FP64 FMA throughput of the current device, TFLOP/s (FMA = 2 flop)."""
    out = C.c_double(0)
    _check(load_library().st_fp64_peak(float(seconds), C.byref(out)))
    return out.value


def release_workspace() -> None:
    """Return the library's cached device memory on the current device to the driver
    (st_release_workspace; synchronises the device)."""
    _check(load_library().st_release_workspace())


def device_count() -> int:
    out = C.c_int(0)
    load_library().st_device_count(C.byref(out))
    return out.value
