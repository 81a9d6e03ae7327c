// Drop-in C++ surface of the reference library (namespace stokestree,
// /root/reference/proj/include/stokestree/*.hpp) on top of the C ABI of
// libstokestree_b200.so (include/stokestree_c.h).  Every evaluation runs the
// sm_100a kernels; the small host pieces kept here are the value types, the
// index bookkeeping of MultiIndexTable, the per-pair tensor helpers and input
// validation, exactly as the reference exposes them.  Link with
// -lstokestree_b200.
#pragma once

#include <array>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <limits>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "stokestree_c.h"

namespace stokestree {

namespace abi {
[[noreturn]] inline void raise(st_status s) {
    const std::string m = st_last_error();
    if (s == ST_INVALID_ARGUMENT) throw std::invalid_argument(m);
    if (s == ST_DOMAIN_ERROR) throw std::domain_error(m);
    throw std::runtime_error(m);
}
inline void check(st_status s) {
    if (s != ST_OK) raise(s);
}
}  // namespace abi

// ------------------------------------------------------------------ vec3.hpp
struct Vec3 {
    double c[3]{0.0, 0.0, 0.0};
    constexpr Vec3() = default;
    constexpr Vec3(double x, double y, double z) : c{x, y, z} {}
    constexpr double& operator[](int i) { return c[i]; }
    constexpr const double& operator[](int i) const { return c[i]; }
    constexpr Vec3& operator+=(const Vec3& o) {
        for (int a = 0; a < 3; ++a) c[a] += o.c[a];
        return *this;
    }
    constexpr Vec3& operator-=(const Vec3& o) {
        for (int a = 0; a < 3; ++a) c[a] -= o.c[a];
        return *this;
    }
    constexpr Vec3& operator*=(double s) {
        for (double& v : c) v *= s;
        return *this;
    }
    friend constexpr Vec3 operator+(Vec3 a, const Vec3& b) { return a += b; }
    friend constexpr Vec3 operator-(Vec3 a, const Vec3& b) { return a -= b; }
    friend constexpr Vec3 operator*(Vec3 a, double s) { return a *= s; }
    friend constexpr Vec3 operator*(double s, Vec3 a) { return a *= s; }
    friend constexpr Vec3 operator/(Vec3 a, double s) { return a *= (1.0 / s); }
    friend constexpr Vec3 operator-(const Vec3& a) { return {-a.c[0], -a.c[1], -a.c[2]}; }
    friend constexpr bool operator==(const Vec3& a, const Vec3& b) {
        return a.c[0] == b.c[0] && a.c[1] == b.c[1] && a.c[2] == b.c[2];
    }
};
static_assert(sizeof(Vec3) == 3 * sizeof(double), "Vec3 arrays are handed to the C ABI as xyz doubles");

constexpr double dot(const Vec3& a, const Vec3& b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
constexpr double norm2(const Vec3& a) { return dot(a, a); }
inline double norm(const Vec3& a) { return std::sqrt(norm2(a)); }
inline Vec3 normalized(const Vec3& a) { return a / norm(a); }
inline bool all_finite(const Vec3& a) {
    return std::isfinite(a[0]) && std::isfinite(a[1]) && std::isfinite(a[2]);
}
using Mat3 = std::array<std::array<double, 3>, 3>;
using Ten3 = std::array<Mat3, 3>;

// ------------------------------------------------------------------ rng.hpp
class SplitMix64 {
public:
    explicit constexpr SplitMix64(uint64_t seed) : s_(seed) {}
    constexpr uint64_t next() {
        s_ += 0x9E3779B97F4A7C15ull;
        uint64_t z = s_;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    double uniform01() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
    double symmetric() { return 2.0 * uniform01() - 1.0; }

private:
    uint64_t s_;
};

// ------------------------------------------------------------------ particles.hpp
struct KernelSelection {
    bool stokeslet_enabled = true;
    bool stresslet_enabled = true;
    static constexpr KernelSelection stokeslet_only() { return {true, false}; }
    static constexpr KernelSelection stresslet_only() { return {false, true}; }
    static constexpr KernelSelection both() { return {true, true}; }
    friend constexpr bool operator==(KernelSelection a, KernelSelection b) = default;
};

struct ParticleSet {
    std::vector<Vec3> position, force_weight, dipole_weight, normal;
    std::size_t size() const { return position.size(); }
};

namespace detail {
inline const double* raw(const std::vector<Vec3>& v, std::size_t n) {
    return v.size() == n && n ? reinterpret_cast<const double*>(v.data()) : nullptr;
}
inline st_particles to_c(const ParticleSet& ps, KernelSelection sel) {
    const std::size_t n = ps.size();
    return st_particles{n, raw(ps.position, n), sel.stokeslet_enabled ? raw(ps.force_weight, n) : nullptr,
                        sel.stresslet_enabled ? raw(ps.dipole_weight, n) : nullptr,
                        sel.stresslet_enabled ? raw(ps.normal, n) : nullptr};
}
inline std::vector<Vec3> from_raw(const std::vector<double>& a) {
    std::vector<Vec3> v(a.size() / 3);
    for (std::size_t i = 0; i < v.size(); ++i) v[i] = Vec3{a[3 * i], a[3 * i + 1], a[3 * i + 2]};
    return v;
}
}  // namespace detail

// validate (particles.hpp:41-70): sizes, finiteness, unit normals (+-1e-12), host side.
inline void validate(const ParticleSet& ps, KernelSelection sel) {
    if (!sel.stokeslet_enabled && !sel.stresslet_enabled)
        throw std::invalid_argument("kernel selection: at least one kernel must be enabled");
    const std::size_t n = ps.size();
    if (n == 0) throw std::invalid_argument("particle set is empty");
    auto check = [n](const std::vector<Vec3>& a, const char* name) {
        if (a.size() != n)
            throw std::invalid_argument(std::string("particle array '") + name + "' has mismatched length");
        for (const Vec3& v : a)
            if (!all_finite(v))
                throw std::invalid_argument(std::string("particle array '") + name + "' contains a non-finite value");
    };
    check(ps.position, "position");
    if (sel.stokeslet_enabled) check(ps.force_weight, "force_weight");
    if (sel.stresslet_enabled) {
        check(ps.dipole_weight, "dipole_weight");
        check(ps.normal, "normal");
        for (std::size_t i = 0; i < n; ++i)
            if (std::abs(norm(ps.normal[i]) - 1.0) > 1e-12)
                throw std::invalid_argument("normal " + std::to_string(i) + " is not unit length");
    }
}

// ------------------------------------------------------------------ kernels.hpp
// Per-pair tensors (host helpers, as in the reference; not the evaluated path).
inline Mat3 stokeslet(const Vec3& x, const Vec3& y) {
    const Vec3 d = x - y;
    const double r2 = norm2(d);
    if (r2 == 0.0) throw std::domain_error("stokeslet: coincident points");
    const double ri = 1.0 / std::sqrt(r2), r3 = ri / r2;
    Mat3 s{};
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) s[i][j] = (i == j ? ri : 0.0) + d[i] * d[j] * r3;
    return s;
}
inline Ten3 stresslet(const Vec3& x, const Vec3& y) {
    const Vec3 d = x - y;
    const double r2 = norm2(d);
    if (r2 == 0.0) throw std::domain_error("stresslet: coincident points");
    const double r5 = 1.0 / (r2 * r2 * std::sqrt(r2));
    Ten3 t{};
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            for (int l = 0; l < 3; ++l) t[i][j][l] = d[i] * d[j] * d[l] * r5;
    return t;
}

inline std::vector<Vec3> naive_direct_velocity(const ParticleSet& ps, KernelSelection sel) {
    const st_particles c = detail::to_c(ps, sel);
    std::vector<Vec3> u(ps.size());
    abi::check(st_naive_direct_velocity(&c, sel.stokeslet_enabled, sel.stresslet_enabled,
                                        reinterpret_cast<double*>(u.data())));
    return u;
}
inline std::vector<Vec3> contracted_direct_velocity(const ParticleSet& ps, KernelSelection sel, std::size_t first,
                                                    std::size_t last) {
    const st_particles c = detail::to_c(ps, sel);
    std::vector<Vec3> u(last >= first ? last - first : 0);
    abi::check(st_direct_velocity(&c, sel.stokeslet_enabled, sel.stresslet_enabled, first, last,
                                  reinterpret_cast<double*>(u.data())));
    return u;
}
inline std::vector<Vec3> contracted_direct_velocity(const ParticleSet& ps, KernelSelection sel) {
    return contracted_direct_velocity(ps, sel, 0, ps.size());
}
inline std::vector<Vec3> contracted_direct_velocity_at(const ParticleSet& ps, KernelSelection sel,
                                                       const std::vector<std::size_t>& targets) {
    const st_particles c = detail::to_c(ps, sel);
    std::vector<Vec3> u(targets.size());
    abi::check(st_direct_velocity_at(&c, sel.stokeslet_enabled, sel.stresslet_enabled, targets.data(),
                                     targets.size(), reinterpret_cast<double*>(u.data())));
    return u;
}

// ------------------------------------------------------------------ multi_index.hpp
struct MultiIndex {
    int k[3]{0, 0, 0};
    constexpr int norm() const { return k[0] + k[1] + k[2]; }
    constexpr int operator[](int axis) const { return k[axis]; }
    friend constexpr bool operator==(const MultiIndex& a, const MultiIndex& b) {
        return a.k[0] == b.k[0] && a.k[1] == b.k[1] && a.k[2] == b.k[2];
    }
};

// Graded-lexicographic multi-index table (multi_index.hpp:26-180).  Positions are
// computed in closed form: entries before grade s are C(s+2,3); inside grade s,
// (k1,k2) sits at k1*(s+1) - k1*(k1-1)/2 + k2.  Out-of-table shifts map to the
// zero slot size() for the hot-path lookups and to kInvalid for shift().
class MultiIndexTable {
public:
    static constexpr int kInvalid = -1;
    explicit MultiIndexTable(int pmax) : pmax_(pmax) {
        if (pmax < 0) throw std::invalid_argument("MultiIndexTable: pmax must be >= 0");
        for (int s = 0; s <= pmax; ++s)
            for (int a = 0; a <= s; ++a)
                for (int b = 0; a + b <= s; ++b) entries_.push_back(MultiIndex{{a, b, s - a - b}});
    }
    static constexpr int count(int p) { return p < 0 ? 0 : (p + 1) * (p + 2) * (p + 3) / 6; }
    int pmax() const { return pmax_; }
    int size() const { return static_cast<int>(entries_.size()); }
    int zero_slot() const { return size(); }
    int size_at(int p) const {
        if (p < 0 || p > pmax_) throw std::invalid_argument("size_at: order out of range");
        return count(p);
    }
    int grade_begin(int s) const { return count(s - 1); }
    int grade_end(int s) const { return count(s); }
    const MultiIndex& operator[](int flat) const { return entries_[flat]; }
    int flat_index(int k1, int k2, int k3) const {
        if (k1 < 0 || k2 < 0 || k3 < 0) return kInvalid;
        const int s = k1 + k2 + k3;
        if (s > pmax_) return kInvalid;
        return count(s - 1) + k1 * (s + 1) - k1 * (k1 - 1) / 2 + k2;
    }
    int shift(int flat, int axis, int delta) const {
        if (axis < 0 || axis > 2) throw std::invalid_argument("shift: bad axis");
        if (delta != 1 && delta != -1 && delta != 2 && delta != -2)
            throw std::invalid_argument("shift: delta must be in {-2,-1,1,2}");
        MultiIndex m = entries_[flat];
        m.k[axis] += delta;
        return flat_index(m.k[0], m.k[1], m.k[2]);
    }
    int up(int flat, int axis) const { return at(flat, axis, 1); }
    int down(int flat, int axis) const { return at(flat, axis, -1); }
    int down2(int flat, int axis) const { return at(flat, axis, -2); }
    int up_down(int flat, int i, int j) const { return moved(flat, {i, j}, {1, -1}); }
    int up_up(int flat, int i, int j) const { return moved(flat, {i, j}, {1, 1}); }
    int up_up_down(int flat, int i, int j, int l) const { return moved3(flat, i, j, l); }
    int mono_axis(int flat) const {
        int a = 0;
        while (flat > 0 && entries_[flat].k[a] == 0) ++a;
        return flat > 0 ? a : 0;
    }
    int mono_parent(int flat) const { return flat > 0 ? down(flat, mono_axis(flat)) : 0; }
    static constexpr int sym_index(int i, int j) {
        const int lo = i < j ? i : j, hi = i < j ? j : i;
        return lo == 0 ? hi : lo == 1 ? 2 + hi : 5;
    }

private:
    int zero_or(int f) const { return f == kInvalid ? zero_slot() : f; }
    int at(int flat, int axis, int d) const {
        MultiIndex m = entries_[flat];
        m.k[axis] += d;
        return zero_or(flat_index(m.k[0], m.k[1], m.k[2]));
    }
    int moved(int flat, std::array<int, 2> ax, std::array<int, 2> d) const {
        MultiIndex m = entries_[flat];
        m.k[ax[0]] += d[0];
        m.k[ax[1]] += d[1];
        return zero_or(flat_index(m.k[0], m.k[1], m.k[2]));
    }
    int moved3(int flat, int i, int j, int l) const {
        MultiIndex m = entries_[flat];
        m.k[i] += 1;
        m.k[j] += 1;
        m.k[l] -= 1;
        return zero_or(flat_index(m.k[0], m.k[1], m.k[2]));
    }
    int pmax_;
    std::vector<MultiIndex> entries_;
};

// ------------------------------------------------------------------ coulomb.hpp
struct CoulombCoeffs {
    std::vector<double> b;
    Vec3 dx;
    double r2 = 0.0;
    int pmax = 0;
    double at(int flat) const { return flat == MultiIndexTable::kInvalid ? 0.0 : b[flat]; }
};

inline double coulomb_coeffs_into(const Vec3& dx, const MultiIndexTable& table, std::span<double> b) {
    if (b.size() != static_cast<std::size_t>(table.size()) + 1)
        throw std::invalid_argument("coulomb_coeffs_into: buffer size mismatch");
    abi::check(st_coulomb_coeffs(1, dx.c, table.pmax(), b.data()));
    b[table.zero_slot()] = 0.0;
    return norm2(dx);
}
inline CoulombCoeffs coulomb_coeffs(const Vec3& dx, const MultiIndexTable& table) {
    CoulombCoeffs c;
    c.b.resize(static_cast<std::size_t>(table.size()) + 1);
    c.dx = dx;
    c.pmax = table.pmax();
    c.r2 = coulomb_coeffs_into(dx, table, c.b);
    return c;
}

// ------------------------------------------------------------------ cluster_tree.hpp
struct Box {
    Vec3 lo, hi;
    Vec3 center() const { return (lo + hi) * 0.5; }
    bool contains(const Vec3& p) const {
        for (int a = 0; a < 3; ++a)
            if (!(p[a] >= lo[a] && p[a] <= hi[a])) return false;
        return true;
    }
};

struct Cluster {
    std::size_t begin = 0, end = 0;
    Vec3 center;
    double radius = 0.0;
    Box bbox;
    int32_t children[8];
    int n_children = 0;
    bool is_leaf = true;
    std::size_t count() const { return end - begin; }
};

struct ClusterTree {
    ParticleSet particles;
    std::vector<Cluster> clusters;
    std::vector<uint32_t> to_original;
    std::vector<uint32_t> to_tree;
    int leaf_capacity = 0;
    bool shrink = false;
    std::shared_ptr<st_tree> device;  // the device tree this host copy was exported from
    const Cluster& root() const { return clusters.front(); }
};

inline bool mac(double radius, double dist2, double theta) {
    return dist2 != 0.0 && radius * radius <= theta * theta * dist2;
}
inline bool mac(const Vec3& x, const Cluster& c, double theta) { return mac(c.radius, norm2(x - c.center), theta); }

inline ClusterTree build_tree(const ParticleSet& ps, int leaf_capacity, bool shrink) {
    const std::size_t n = ps.size();
    const st_particles c{n, detail::raw(ps.position, n), detail::raw(ps.force_weight, n),
                         detail::raw(ps.dipole_weight, n), detail::raw(ps.normal, n)};
    st_tree* h = nullptr;
    abi::check(st_build_tree(&c, leaf_capacity, shrink ? 1 : 0, &h));
    ClusterTree t;
    t.device.reset(h, st_tree_free);
    t.leaf_capacity = leaf_capacity;
    t.shrink = shrink;
    const std::size_t ncl = st_tree_num_clusters(h);
    std::vector<int64_t> be(2 * ncl);
    std::vector<double> geom(10 * ncl);
    std::vector<int32_t> kids(8 * ncl), meta(2 * ncl);
    t.to_original.resize(n);
    abi::check(st_tree_export(h, be.data(), geom.data(), kids.data(), meta.data(), t.to_original.data()));
    t.clusters.resize(ncl);
    for (std::size_t i = 0; i < ncl; ++i) {
        Cluster& cl = t.clusters[i];
        cl.begin = static_cast<std::size_t>(be[2 * i]);
        cl.end = static_cast<std::size_t>(be[2 * i + 1]);
        const double* g = &geom[10 * i];
        cl.center = Vec3{g[0], g[1], g[2]};
        cl.radius = g[3];
        cl.bbox = Box{Vec3{g[4], g[5], g[6]}, Vec3{g[7], g[8], g[9]}};
        for (int s = 0; s < 8; ++s) cl.children[s] = kids[8 * i + s];
        cl.n_children = meta[2 * i];
        cl.is_leaf = meta[2 * i + 1] != 0;
    }
    t.to_tree.resize(n);
    for (std::size_t k = 0; k < n; ++k) t.to_tree[t.to_original[k]] = static_cast<uint32_t>(k);
    auto gather = [&](const std::vector<Vec3>& src) {
        std::vector<Vec3> out;
        if (src.size() == n)
            for (std::size_t k = 0; k < n; ++k) out.push_back(src[t.to_original[k]]);
        return out;
    };
    t.particles = ParticleSet{gather(ps.position), gather(ps.force_weight), gather(ps.dipole_weight),
                              gather(ps.normal)};
    return t;
}

// ------------------------------------------------------------------ moments.hpp
struct StokesletMomentsView {
    std::span<const double> m;
};
struct StressletMomentsView {
    std::span<const double> mt, trace, sym;
};

class ClusterMoments {
public:
    ClusterMoments(int order, int count, std::size_t n_clusters, KernelSelection sel)
        : order_(order), count_(count), sel_(sel) {
        const std::size_t c = static_cast<std::size_t>(count) * n_clusters;
        if (sel.stokeslet_enabled) stok_.assign(3 * c, 0.0);
        if (sel.stresslet_enabled) {
            str_.assign(9 * c, 0.0);
            trace_.assign(c, 0.0);
            sym_.assign(6 * c, 0.0);
        }
    }
    int order() const { return order_; }
    int entry_count() const { return count_; }
    KernelSelection selection() const { return sel_; }
    StokesletMomentsView stokeslet_view(std::size_t cl) const { return {span_of(stok_, 3, cl)}; }
    StressletMomentsView stresslet_view(std::size_t cl) const {
        return {span_of(str_, 9, cl), span_of(trace_, 1, cl), span_of(sym_, 6, cl)};
    }
    std::span<double> stokeslet_slot(std::size_t cl) { return mut(stok_, 3, cl); }
    std::span<double> stresslet_slot(std::size_t cl) { return mut(str_, 9, cl); }
    std::span<double> trace_slot(std::size_t cl) { return mut(trace_, 1, cl); }
    std::span<double> sym_slot(std::size_t cl) { return mut(sym_, 6, cl); }
    double* raw_stok() { return stok_.data(); }
    double* raw_str() { return str_.data(); }
    double* raw_trace() { return trace_.data(); }
    double* raw_sym() { return sym_.data(); }

private:
    std::span<const double> span_of(const std::vector<double>& v, std::size_t w, std::size_t cl) const {
        const std::size_t c = static_cast<std::size_t>(count_);
        return std::span<const double>(v).subspan(w * c * cl, w * c);
    }
    std::span<double> mut(std::vector<double>& v, std::size_t w, std::size_t cl) {
        const std::size_t c = static_cast<std::size_t>(count_);
        return std::span<double>(v).subspan(w * c * cl, w * c);
    }
    int order_, count_;
    KernelSelection sel_;
    std::vector<double> stok_, str_, trace_, sym_;
};

// compute_moments (moments.hpp:140-175) on the device; `workers` is accepted and unused.
inline ClusterMoments compute_moments(const ClusterTree& tree, int p, KernelSelection sel,
                                      const MultiIndexTable& table, int workers = 1) {
    if (p < 0 || p > table.pmax()) throw std::invalid_argument("compute_moments: order outside table range");
    if (workers < 1) throw std::invalid_argument("compute_moments: workers must be >= 1");
    if (!tree.device) throw std::invalid_argument("compute_moments: tree was not produced by build_tree");
    ClusterMoments m(p, table.size_at(p), tree.clusters.size(), sel);
    abi::check(st_compute_moments(tree.device.get(), p, sel.stokeslet_enabled, sel.stresslet_enabled,
                                  m.raw_stok(), m.raw_str(), m.raw_trace(), m.raw_sym()));
    return m;
}

// ------------------------------------------------------------------ farfield.hpp
struct FarFieldWorkspace {
    std::vector<double> b;
    void resize_for(const MultiIndexTable& table) { b.resize(static_cast<std::size_t>(table.size()) + 1); }
};

// Eq. 25 / Eq. 30 (farfield.hpp:30-96), evaluated by the device far-field kernel
// from dx and the moments (ws.b is accepted for interface parity; the kernel
// forms its own coefficients by the same recurrence).
inline Vec3 stokeslet_farfield(const Vec3& dx, const StokesletMomentsView& m, int p, const MultiIndexTable& table,
                               const FarFieldWorkspace&) {
    if (table.pmax() < p + 1) throw std::invalid_argument("stokeslet_farfield: table too shallow for order");
    if (m.m.size() != static_cast<std::size_t>(3 * table.size_at(p)))
        throw std::invalid_argument("stokeslet_farfield: moment order mismatch");
    Vec3 u;
    abi::check(st_farfield_pairs(1, dx.c, p, 1, 0, m.m.data(), nullptr, nullptr, nullptr, u.c));
    return u;
}
// m.trace and m.sym must be the contractions of m.mt (as compute_moments produces them,
// moments.hpp:66-80): the device path recomputes them from m.mt (stokestree_c.h).
inline Vec3 stresslet_farfield(const Vec3& dx, const StressletMomentsView& m, int p, const MultiIndexTable& table,
                               const FarFieldWorkspace&) {
    if (table.pmax() < p + 2) throw std::invalid_argument("stresslet_farfield: table too shallow for order");
    if (m.trace.size() != static_cast<std::size_t>(table.size_at(p)))
        throw std::invalid_argument("stresslet_farfield: moment order mismatch");
    Vec3 u;
    abi::check(st_farfield_pairs(1, dx.c, p, 0, 1, nullptr, m.mt.data(), m.trace.data(), m.sym.data(), u.c));
    return u;
}

// ------------------------------------------------------------------ taylor_coeffs.hpp
// Explicit Taylor coefficients (taylor_coeffs.hpp:13-46), formed by the device kernel from
// the caller's coefficients (st_taylor_coeffs; a test/reference path, not the hot path).
inline double stokeslet_taylor_coeff(const MultiIndexTable& table, const CoulombCoeffs& coeffs, int flat_k, int i,
                                     int j) {
    if (flat_k < 0 || flat_k >= table.size())
        throw std::invalid_argument("stokeslet_taylor_coeff: multi-index out of table");
    const int s = table[flat_k].norm();
    if (s + 1 > coeffs.pmax) throw std::invalid_argument("stokeslet_taylor_coeff: coefficients not deep enough");
    std::vector<double> a(9 * static_cast<std::size_t>(MultiIndexTable::count(s)));
    abi::check(st_taylor_coeffs(1, coeffs.dx.c, coeffs.b.data(), coeffs.pmax, s, a.data(), nullptr));
    return a[9 * static_cast<std::size_t>(flat_k) + 3 * i + j];
}
inline double stresslet_taylor_coeff(const MultiIndexTable& table, const CoulombCoeffs& coeffs, int flat_k, int i,
                                     int j, int l) {
    if (flat_k < 0 || flat_k >= table.size())
        throw std::invalid_argument("stresslet_taylor_coeff: multi-index out of table");
    const int s = table[flat_k].norm();
    if (s + 2 > coeffs.pmax) throw std::invalid_argument("stresslet_taylor_coeff: coefficients not deep enough");
    std::vector<double> a(27 * static_cast<std::size_t>(MultiIndexTable::count(s)));
    abi::check(st_taylor_coeffs(1, coeffs.dx.c, coeffs.b.data(), coeffs.pmax, s, nullptr, a.data()));
    return a[27 * static_cast<std::size_t>(flat_k) + 9 * i + 3 * j + l];
}

// ------------------------------------------------------------------ engine.hpp
struct TreecodeParams {
    static constexpr int kMaxOrder = 16;
    int order = 6;
    double theta = 0.5;
    int leaf_capacity = 2000;
    bool shrink = true;
    KernelSelection kernels;
    int workers = 1;
    int devices = 1;  // new: GPUs used by parallel_velocity

    st_params to_c() const {
        return st_params{order, theta, leaf_capacity, shrink ? 1 : 0, kernels.stokeslet_enabled ? 1 : 0,
                         kernels.stresslet_enabled ? 1 : 0, workers, devices};
    }
    void validate() const {
        const st_params p = to_c();
        abi::check(st_params_validate(&p));
    }
};

struct TraversalStats {
    uint64_t farfield_evals = 0;
    uint64_t direct_pairs = 0;
    uint64_t clusters_visited = 0;
    TraversalStats& operator+=(const TraversalStats& o) {
        farfield_evals += o.farfield_evals;
        direct_pairs += o.direct_pairs;
        clusters_visited += o.clusters_visited;
        return *this;
    }
};

struct VelocityResult {
    std::vector<Vec3> velocity;  // original particle (or target) order
    TraversalStats stats;
    double time_build_s = 0.0;
    double time_moments_s = 0.0;
    double time_traverse_s = 0.0;
    double time_total_s = 0.0;
};

namespace detail {
inline VelocityResult run(const ParticleSet& ps, const std::vector<Vec3>* targets, const TreecodeParams& params) {
    params.validate();
    const st_particles c = to_c(ps, params.kernels);
    const st_params p = params.to_c();
    const std::size_t nt = targets ? targets->size() : ps.size();
    VelocityResult r;
    r.velocity.resize(nt);
    st_stats s{};
    abi::check(st_treecode_velocity_ex(&c, targets ? reinterpret_cast<const double*>(targets->data()) : nullptr,
                                       targets ? nt : 0, &p, reinterpret_cast<double*>(r.velocity.data()), nullptr,
                                       &s));
    r.stats = TraversalStats{s.farfield_evals, s.direct_pairs, s.clusters_visited};
    r.time_build_s = s.time_build_s;
    r.time_moments_s = s.time_moments_s;
    r.time_traverse_s = s.time_traverse_s;
    r.time_total_s = s.time_total_s;
    return r;
}
}  // namespace detail

// treecode_velocity (engine.hpp:185-189)
inline VelocityResult treecode_velocity(const ParticleSet& ps, const TreecodeParams& params) {
    TreecodeParams serial = params;
    serial.workers = 1;
    return detail::run(ps, nullptr, serial);
}
// parallel_velocity (engine.hpp:194-196): bit-identical to treecode_velocity.
inline VelocityResult parallel_velocity(const ParticleSet& ps, const TreecodeParams& params) {
    return detail::run(ps, nullptr, params);
}
// New: velocities at disjoint target points (nothing excluded).
inline VelocityResult treecode_velocity_at_points(const ParticleSet& ps, const std::vector<Vec3>& targets,
                                                  const TreecodeParams& params) {
    return detail::run(ps, &targets, params);
}
// New: give the device memory the library keeps between calls (its private pool, the near
// field's workspace) on the current device back to the driver (st_release_workspace).
inline void release_workspace() { abi::check(st_release_workspace()); }

// ------------------------------------------------------------------ error_metric.hpp
inline double relative_error(std::span<const Vec3> u_ref, std::span<const Vec3> u_test) {
    if (u_ref.size() != u_test.size()) throw std::invalid_argument("relative_error: field lengths differ");
    double out = 0.0;
    abi::check(st_relative_error(u_ref.size(), reinterpret_cast<const double*>(u_ref.data()),
                                 reinterpret_cast<const double*>(u_test.data()), &out));
    return out;
}

}  // namespace stokestree

// The reference umbrella also brings in the harness layer (bench, particle_io, testcases).
#include "stokestree/harness.hpp"
