// The reference's unit tests (proj/tests/test_*.cpp), restated case by case against the
// drop-in headers (include/stokestree/) -- the cases tests/cpp/dropin_test.cpp and the
// Python suites do not already carry.  Each function names the TEST_CASE it restates
// (file:line).  Catch2 is absent in this image, so CHECK is a local macro; the
// arithmetic, seeds and tolerances are the reference tests' own unless a comment says
// otherwise.  Modes: "host" (validation, index bookkeeping, host helpers, generators)
// or "all" (adds every case that runs the device path).  Exit code 0 = all passed.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "stokestree/cluster_tree.hpp"
#include "stokestree/coulomb.hpp"
#include "stokestree/engine.hpp"
#include "stokestree/error_metric.hpp"
#include "stokestree/farfield.hpp"
#include "stokestree/kernels.hpp"
#include "stokestree/moments.hpp"
#include "stokestree/multi_index.hpp"
#include "stokestree/taylor_coeffs.hpp"
#include "stokestree/testcases.hpp"

using namespace stokestree;

static int failures = 0;
static const char* current = "";
#define CHECK(cond)                                                                     \
    do {                                                                                \
        if (!(cond)) {                                                                  \
            std::printf("FAIL [%s] %s:%d: %s\n", current, __FILE__, __LINE__, #cond);   \
            ++failures;                                                                 \
        }                                                                               \
    } while (0)

template <class E, class F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

// ---- tests/support/test_helpers.hpp, restated
static double rel_diff(double a, double b) {
    const double s = std::max(std::abs(a), std::abs(b));
    return s == 0.0 ? 0.0 : std::abs(a - b) / s;
}
static double rel_diff(const Vec3& a, const Vec3& b) {
    const double s = std::max(norm(a), norm(b));
    return s == 0.0 ? 0.0 : norm(a - b) / s;
}
static Vec3 random_box_point(SplitMix64& r, double lo, double hi) {
    // braced initialisation evaluates left to right, as in the reference helper
    return Vec3{lo + (hi - lo) * r.uniform01(), lo + (hi - lo) * r.uniform01(), lo + (hi - lo) * r.uniform01()};
}
static Vec3 random_unit(SplitMix64& r) {
    for (;;) {
        const Vec3 v{r.symmetric(), r.symmetric(), r.symmetric()};
        const double n2 = norm2(v);
        if (n2 > 1e-4 && n2 <= 1.0) return v / std::sqrt(n2);
    }
}
static ParticleSet random_particles(std::size_t n, uint64_t seed, bool str) {
    SplitMix64 r(seed);
    ParticleSet ps;
    for (std::size_t i = 0; i < n; ++i) {
        ps.position.push_back(random_box_point(r, 0.0, 1.0));
        ps.force_weight.push_back({r.symmetric(), r.symmetric(), r.symmetric()});
        if (str) {
            ps.dipole_weight.push_back({r.symmetric(), r.symmetric(), r.symmetric()});
            ps.normal.push_back(random_unit(r));
        }
    }
    return ps;
}

// ---- tests/support/reference_farfield.hpp, restated
static Vec3 direct_at(const ParticleSet& ps, KernelSelection sel, const Vec3& x) {
    Vec3 u;
    for (std::size_t n = 0; n < ps.size(); ++n) {
        if (sel.stokeslet_enabled) {
            const Mat3 s = stokeslet(x, ps.position[n]);
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) u[i] += s[i][j] * ps.force_weight[n][j];
        }
        if (sel.stresslet_enabled) {
            const Ten3 t = stresslet(x, ps.position[n]);
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j)
                    for (int l = 0; l < 3; ++l) u[i] += t[i][j][l] * ps.dipole_weight[n][j] * ps.normal[n][l];
        }
    }
    return u;
}
struct SingleCluster {
    ClusterTree tree;
    Vec3 center;
    double radius = 0.0;
};
static SingleCluster make_cluster(const ParticleSet& ps) {
    SingleCluster sc{build_tree(ps, static_cast<int>(ps.size()) + 1, true), {}, 0.0};
    sc.center = sc.tree.root().center;
    sc.radius = sc.tree.root().radius;
    return sc;
}
static Vec3 stokeslet_uncontracted(const MultiIndexTable& t, const CoulombCoeffs& c, const StokesletMomentsView& m,
                                   int p) {
    Vec3 u;
    for (int e = 0; e < t.size_at(p); ++e)
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) u[i] += stokeslet_taylor_coeff(t, c, e, i, j) * m.m[3 * e + j];
    return u;
}
static Vec3 stresslet_uncontracted(const MultiIndexTable& t, const CoulombCoeffs& c, const StressletMomentsView& m,
                                   int p) {
    Vec3 u;
    for (int e = 0; e < t.size_at(p); ++e)
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j)
                for (int l = 0; l < 3; ++l) u[i] += stresslet_taylor_coeff(t, c, e, i, j, l) * m.mt[9 * e + 3 * j + l];
    return u;
}

// =============================================================== host cases
// test_multi_index.cpp:7-13
static void table_entry_counts() {
    CHECK(MultiIndexTable(0).size() == 1);
    CHECK(MultiIndexTable(2).size() == 10);
    CHECK(MultiIndexTable(10).size() == 286);
    CHECK(MultiIndexTable(0)[0] == (MultiIndex{{0, 0, 0}}));
}
// test_multi_index.cpp:15-29
static void graded_lexicographic_ordering() {
    const MultiIndexTable t(6);
    for (int e = 1; e < t.size(); ++e) {
        const MultiIndex &a = t[e - 1], &b = t[e];
        CHECK(a.norm() <= b.norm());
        if (a.norm() == b.norm())
            CHECK(a.k[0] < b.k[0] || (a.k[0] == b.k[0] && a.k[1] < b.k[1]) ||
                  (a.k[0] == b.k[0] && a.k[1] == b.k[1] && a.k[2] < b.k[2]));
    }
    for (int p = 0; p <= 6; ++p) CHECK(t.size_at(p) == (p + 1) * (p + 2) * (p + 3) / 6);
}
// test_multi_index.cpp:31-39, 41-54
static void flat_index_and_shifts() {
    const MultiIndexTable t(5);
    for (int e = 0; e < t.size(); ++e) CHECK(t.flat_index(t[e].k[0], t[e].k[1], t[e].k[2]) == e);
    CHECK(t.flat_index(-1, 0, 0) == MultiIndexTable::kInvalid);
    CHECK(t.flat_index(3, 2, 1) == MultiIndexTable::kInvalid);
    const MultiIndexTable t4(4);
    for (int e = 0; e < t4.size(); ++e)
        for (int axis = 0; axis < 3; ++axis)
            for (int delta : {-2, -1, 1, 2}) {
                int c[3] = {t4[e].k[0], t4[e].k[1], t4[e].k[2]};
                c[axis] += delta;
                CHECK(t4.shift(e, axis, delta) == t4.flat_index(c[0], c[1], c[2]));
            }
    CHECK(throws<std::invalid_argument>([&] { (void)t4.shift(0, 0, 3); }));
    CHECK(throws<std::invalid_argument>([&] { (void)t4.shift(0, 3, 1); }));
}
// test_multi_index.cpp:56-86
static void composite_lookups_zero_slot() {
    const MultiIndexTable t(3);
    const int zero = t.zero_slot();
    auto slot = [&](int a, int b, int c) {
        const int f = t.flat_index(a, b, c);
        return f == MultiIndexTable::kInvalid ? zero : f;
    };
    for (int e = 0; e < t.size(); ++e) {
        const MultiIndex& k = t[e];
        for (int i = 0; i < 3; ++i) {
            int c[3] = {k.k[0], k.k[1], k.k[2]};
            c[i] += 1;
            CHECK(t.up(e, i) == slot(c[0], c[1], c[2]));
            for (int j = 0; j < 3; ++j) {
                int d[3] = {k.k[0], k.k[1], k.k[2]};
                d[i] += 1;
                d[j] -= 1;
                CHECK(t.up_down(e, i, j) == slot(d[0], d[1], d[2]));
                for (int l = 0; l < 3; ++l) {
                    int g[3] = {k.k[0], k.k[1], k.k[2]};
                    g[i] += 1;
                    g[j] += 1;
                    g[l] -= 1;
                    CHECK(t.up_up_down(e, i, j, l) == slot(g[0], g[1], g[2]));
                }
            }
        }
    }
}
// test_multi_index.cpp:88-98
static void monomial_chain() {
    const MultiIndexTable t(5);
    for (int e = 1; e < t.size(); ++e) {
        const int parent = t.mono_parent(e);
        CHECK(parent < e);
        MultiIndex k = t[parent];
        k.k[t.mono_axis(e)] += 1;
        CHECK(k == t[e]);
    }
}
// test_kernels.cpp:38-68, 70-73
static void kernel_hand_values() {
    const Mat3 s = stokeslet({1, 0, 0}, {0, 0, 0});
    CHECK(std::abs(s[0][0] - 2.0) <= 1e-15 && std::abs(s[1][1] - 1.0) <= 1e-15 && std::abs(s[2][2] - 1.0) <= 1e-15);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            if (i != j) CHECK(s[i][j] == 0.0);
    CHECK(std::abs(stokeslet({2, 0, 0}, {0, 0, 0})[0][0] - 1.0) <= 1e-15);
    const Ten3 t = stresslet({1, 1, 1}, {0, 0, 0});
    const double expected = 1.0 / (9.0 * std::sqrt(3.0));
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            for (int l = 0; l < 3; ++l) CHECK(std::abs(t[i][j][l] - expected) <= 1e-14 * expected);
    const Ten3 ta = stresslet({1, 0, 0}, {0, 0, 0});
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            for (int l = 0; l < 3; ++l) CHECK(ta[i][j][l] == ((i | j | l) == 0 ? 1.0 : 0.0));
    CHECK(throws<std::domain_error>([] { (void)stokeslet({1, 2, 3}, {1, 2, 3}); }));
    CHECK(throws<std::domain_error>([] { (void)stresslet({1, 2, 3}, {1, 2, 3}); }));
}
// test_kernels.cpp:75-89 (independent unit-vector evaluation)
static void kernels_independent_evaluation() {
    SplitMix64 rng(11);
    for (int rep = 0; rep < 50; ++rep) {
        const Vec3 x = random_box_point(rng, -2.0, 2.0);
        Vec3 y = random_box_point(rng, -2.0, 2.0);
        if (norm2(x - y) < 1e-4) y[0] += 1.0;
        const Vec3 d = x - y;
        const double r = std::hypot(d[0], d[1], d[2]);
        const Vec3 e = d / r;
        const Mat3 s = stokeslet(x, y);
        const Ten3 t = stresslet(x, y);
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) {
                CHECK(rel_diff(s[i][j], ((i == j ? 1.0 : 0.0) + e[i] * e[j]) / r) < 1e-14);
                for (int l = 0; l < 3; ++l) CHECK(rel_diff(t[i][j][l], e[i] * e[j] * e[l] / (r * r)) < 1e-14);
            }
    }
}
// test_kernels.cpp:91-113.  The reference asks t[i][j][l] == t[l][j][i] == t[i][l][j]
// exactly; its own stresslet() forms (d_i d_j) d_l r^-5, so permuting l rounds
// differently and the reference fails 252 of those checks on these very points
// (measured: this case compiled against the reference headers).  Our stresslet() is the
// same expression, so those two are held to 2 ulp; every other identity stays exact.
static void kernel_symmetries() {
    SplitMix64 rng(17);
    for (int rep = 0; rep < 20; ++rep) {
        const Vec3 x = random_box_point(rng, -1.0, 1.0);
        Vec3 y = random_box_point(rng, -1.0, 1.0);
        if (norm2(x - y) < 1e-4) y[2] -= 1.0;
        const Mat3 s = stokeslet(x, y), sw = stokeslet(y, x);
        const Ten3 t = stresslet(x, y), tw = stresslet(y, x);
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) {
                CHECK(s[i][j] == s[j][i]);
                CHECK(s[i][j] == sw[i][j]);
                for (int l = 0; l < 3; ++l) {
                    CHECK(t[i][j][l] == t[j][i][l]);
                    CHECK(rel_diff(t[i][j][l], t[l][j][i]) <= 4.5e-16);
                    CHECK(rel_diff(t[i][j][l], t[i][l][j]) <= 4.5e-16);
                    CHECK(t[i][j][l] == -tw[i][j][l]);
                }
            }
    }
}
// test_kernels.cpp:115-128
static void kernel_scale_law() {
    SplitMix64 rng(23);
    const Vec3 x = random_box_point(rng, -1.0, 1.0);
    const Vec3 y = random_box_point(rng, 1.5, 3.0);
    const double c = 2.0;
    const Mat3 s1 = stokeslet(x, y), sc = stokeslet(x * c, y * c);
    const Ten3 t1 = stresslet(x, y), tc = stresslet(x * c, y * c);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            CHECK(rel_diff(sc[i][j], s1[i][j] / c) < 1e-14);
            for (int l = 0; l < 3; ++l) CHECK(rel_diff(tc[i][j][l], t1[i][j][l] / (c * c)) < 1e-14);
        }
}
// test_engine.cpp:139-161
static void parameter_validation() {
    TreecodeParams p;
    p.theta = 1.0;
    CHECK(throws<std::invalid_argument>([&] { p.validate(); }));
    p.theta = 0.0;
    CHECK(throws<std::invalid_argument>([&] { p.validate(); }));
    p.theta = 0.5;
    p.order = -1;
    CHECK(throws<std::invalid_argument>([&] { p.validate(); }));
    p.order = TreecodeParams::kMaxOrder + 1;
    CHECK(throws<std::invalid_argument>([&] { p.validate(); }));
    p.order = 6;
    p.leaf_capacity = 0;
    CHECK(throws<std::invalid_argument>([&] { p.validate(); }));
    p.leaf_capacity = 10;
    p.workers = 0;
    CHECK(throws<std::invalid_argument>([&] { p.validate(); }));
    p.workers = 1;
    p.kernels = {false, false};
    CHECK(throws<std::invalid_argument>([&] { p.validate(); }));
    p.kernels = KernelSelection::both();
    CHECK(!throws<std::exception>([&] { p.validate(); }));
}
// test_cluster_tree.cpp:220-226 and test_coulomb.cpp:27-30 (host-side checks)
static void input_validation() {
    ParticleSet empty;
    CHECK(throws<std::invalid_argument>([&] { (void)build_tree(empty, 10, false); }));
    ParticleSet one;
    one.position = {{0, 0, 0}};
    CHECK(throws<std::invalid_argument>([&] { (void)build_tree(one, 0, false); }));
    const MultiIndexTable t(2);
    CHECK(throws<std::domain_error>([&] { (void)coulomb_coeffs({0, 0, 0}, t); }));
}
// test_testcases.cpp (all six cases; the [slow] 81,920-particle one included)
static bool byte_identical(const ParticleSet& a, const ParticleSet& b) {
    auto eq = [](const std::vector<Vec3>& x, const std::vector<Vec3>& y) {
        return x.size() == y.size() && (x.empty() || std::memcmp(x.data(), y.data(), x.size() * sizeof(Vec3)) == 0);
    };
    return eq(a.position, b.position) && eq(a.force_weight, b.force_weight) && eq(a.dipole_weight, b.dipole_weight) &&
           eq(a.normal, b.normal);
}
static bool positions_distinct(const ParticleSet& ps) {
    std::vector<Vec3> s = ps.position;
    std::sort(s.begin(), s.end(), [](const Vec3& a, const Vec3& b) {
        if (a[0] != b[0]) return a[0] < b[0];
        if (a[1] != b[1]) return a[1] < b[1];
        return a[2] < b[2];
    });
    for (std::size_t i = 1; i < s.size(); ++i)
        if (s[i - 1] == s[i]) return false;
    return true;
}
static void testcases_generators() {
    for (int levels : {0, 1, 2, 3}) {
        const ParticleSet ps = sphere_particles({levels, 99});
        CHECK(ps.size() == (20u << (2 * levels)));
        for (const Vec3& p : ps.position) CHECK(std::abs(norm(p) - 1.0) <= 1e-14);
    }
    CHECK(sphere_particles({3, 0}).size() == 1280);
    const ParticleSet s2 = sphere_particles({2, 123});
    CHECK(s2.normal.size() == s2.size());
    for (std::size_t i = 0; i < s2.size(); ++i) {
        CHECK(s2.normal[i] == s2.position[i]);
        for (int c = 0; c < 3; ++c) CHECK(std::abs(s2.force_weight[i][c]) <= 1.0 && std::abs(s2.dipole_weight[i][c]) <= 1.0);
    }
    const ParticleSet big = sphere_particles({6, 2024});
    CHECK(big.size() == 81920);
    CHECK(positions_distinct(big));
    CHECK((CubeCaseConfig{2500, 2500.0, 0}.side() == 1.0));
    CHECK(std::abs(CubeCaseConfig{125000, 2500.0, 0}.side() - 3.6840314986) <= 1e-9 * 3.6840314986);
    const CubeCaseConfig cfg{10000, 2500.0, 77};
    const ParticleSet cube = cube_particles(cfg);
    const double L = cfg.side();
    CHECK(cube.size() == cfg.n);
    CHECK(cube.dipole_weight.empty() && cube.normal.empty());
    for (std::size_t i = 0; i < cube.size(); ++i)
        for (int c = 0; c < 3; ++c)
            CHECK(cube.position[i][c] >= 0.0 && cube.position[i][c] <= L && std::abs(cube.force_weight[i][c]) <= 1.0);
    CHECK(positions_distinct(cube));
    CHECK(byte_identical(sphere_particles({3, 42}), sphere_particles({3, 42})));
    CHECK(byte_identical(cube_particles({5000, 2500.0, 42}), cube_particles({5000, 2500.0, 42})));
    CHECK(!byte_identical(cube_particles({5000, 2500.0, 42}), cube_particles({5000, 2500.0, 43})));
}

// =============================================================== device cases
// test_coulomb.cpp:48-54
static void coulomb_zero_slot() {
    const MultiIndexTable t(5);
    const CoulombCoeffs c = coulomb_coeffs({0.3, -1.2, 0.4}, t);
    CHECK(c.b[t.zero_slot()] == 0.0);
    CHECK(c.b.size() == static_cast<std::size_t>(t.size()) + 1);
    CHECK(c.b[0] > 0.0);
}
// test_cluster_tree.cpp:52-61
static void single_particle_tree() {
    ParticleSet ps;
    ps.position = {{0.3, -0.2, 0.9}};
    ps.force_weight = {{1, 0, 0}};
    const ClusterTree tree = build_tree(ps, 2000, false);
    CHECK(tree.clusters.size() == 1);
    CHECK(tree.root().is_leaf);
    CHECK(tree.root().radius == 0.0);
    CHECK(tree.root().center == ps.position[0]);
}
static int tree_depth(const ClusterTree& tree, int id = 0) {
    const Cluster& c = tree.clusters[id];
    int d = 0;
    for (int s = 0; s < c.n_children; ++s) d = std::max(d, 1 + tree_depth(tree, c.children[s]));
    return d;
}
static void check_partition(const ClusterTree& tree) {
    const std::size_t n = tree.particles.size();
    std::vector<int> seen(n, 0);
    for (const Cluster& c : tree.clusters) {
        if (!c.is_leaf) {
            std::size_t cursor = c.begin;
            for (int s = 0; s < c.n_children; ++s) {
                const Cluster& ch = tree.clusters[c.children[s]];
                CHECK(ch.begin == cursor);
                cursor = ch.end;
            }
            CHECK(cursor == c.end);
            continue;
        }
        for (std::size_t t = c.begin; t < c.end; ++t) ++seen[t];
    }
    for (std::size_t t = 0; t < n; ++t) CHECK(seen[t] == 1);
    std::vector<uint32_t> perm(tree.to_original.begin(), tree.to_original.end());
    std::sort(perm.begin(), perm.end());
    for (std::size_t i = 0; i < n; ++i) CHECK(perm[i] == i);
}
// test_cluster_tree.cpp:85-101 ([slow] in the reference; 81,920 particles is quick here)
static void sphere_tree_structure() {
    const ParticleSet ps = sphere_particles({6, 42});
    CHECK(ps.size() == 81920);
    const ClusterTree tree = build_tree(ps, 2000, true);
    std::size_t leaf_total = 0;
    for (const Cluster& c : tree.clusters)
        if (c.is_leaf) {
            CHECK(c.count() <= 2000);
            leaf_total += c.count();
        }
    CHECK(leaf_total == ps.size());
    CHECK(tree_depth(tree) <= 20);
    check_partition(tree);
    for (const Vec3& p : tree.particles.position) CHECK(tree.root().bbox.contains(p));
}
// test_cluster_tree.cpp:116-125.  The reference's own trees break this claim: with shrink
// the centre moves to the tight box's midpoint and the radius about it can exceed the
// unshrunk one -- 429 clusters over the three seeds (measured: this case compiled against
// the reference headers).  Our trees are bit-exact with the reference's, so the case
// pins that count: same cluster count, and exactly the reference's 429 violations.
static void shrink_never_increases_radius() {
    int violations = 0;
    for (uint64_t seed : {1u, 2u, 3u}) {
        const ParticleSet ps = random_particles(4000, seed, false);
        const ClusterTree plain = build_tree(ps, 50, false), shrunk = build_tree(ps, 50, true);
        CHECK(plain.clusters.size() == shrunk.clusters.size());
        for (std::size_t i = 0; i < std::min(plain.clusters.size(), shrunk.clusters.size()); ++i)
            violations += !(shrunk.clusters[i].radius <= plain.clusters[i].radius);
    }
    CHECK(violations == 429);
}
// test_cluster_tree.cpp:165-179
static void single_particle_moments() {
    ParticleSet ps;
    ps.position = {{0.25, 0.5, -0.75}};
    ps.force_weight = {{1, 2, 3}};
    const ClusterTree tree = build_tree(ps, 10, true);
    const MultiIndexTable table(4);
    const ClusterMoments m = compute_moments(tree, 4, KernelSelection::stokeslet_only(), table);
    const auto sv = m.stokeslet_view(0);
    for (int e = 1; e < table.size_at(4); ++e)
        for (int j = 0; j < 3; ++j) CHECK(sv.m[3 * e + j] == 0.0);
    CHECK(sv.m[0] == 1.0 && sv.m[1] == 2.0 && sv.m[2] == 3.0);
}
// test_cluster_tree.cpp:181-218.  The reference's own stresslet moments differ from this
// pow() loop by up to 2.054e-13 (measured against the reference headers), above the
// case's 1e-14; the Stokeslet ones stay at 5e-16.  The device sums particles in a
// parallel order with FMA, so a cancelling entry can also leave 1e-14 here; the bound is
// 1e-12 (north_star's velocity bar) for every moment and contraction.
static void moments_definitional_loop() {
    const ParticleSet ps = random_particles(100, 77, true);
    const ClusterTree tree = build_tree(ps, 200, false);
    CHECK(tree.clusters.size() == 1);
    const int p = 3;
    const MultiIndexTable table(p);
    const ClusterMoments m = compute_moments(tree, p, KernelSelection::both(), table);
    const auto sv = m.stokeslet_view(0);
    const auto tv = m.stresslet_view(0);
    const Vec3 yc = tree.root().center;
    for (int e = 0; e < table.size_at(p); ++e) {
        const MultiIndex& k = table[e];
        double ms[3] = {0, 0, 0}, mt[3][3] = {};
        for (std::size_t n = 0; n < ps.size(); ++n) {
            const Vec3 d = tree.particles.position[n] - yc;
            const double mono = std::pow(d[0], k.k[0]) * std::pow(d[1], k.k[1]) * std::pow(d[2], k.k[2]);
            for (int j = 0; j < 3; ++j) {
                ms[j] += mono * tree.particles.force_weight[n][j];
                for (int l = 0; l < 3; ++l)
                    mt[j][l] += mono * tree.particles.dipole_weight[n][j] * tree.particles.normal[n][l];
            }
        }
        for (int j = 0; j < 3; ++j) {
            CHECK(rel_diff(sv.m[3 * e + j], ms[j]) < 1e-12);
            for (int l = 0; l < 3; ++l) CHECK(rel_diff(tv.mt[9 * e + 3 * j + l], mt[j][l]) < 1e-12);
        }
        CHECK(rel_diff(tv.trace[e], mt[0][0] + mt[1][1] + mt[2][2]) < 1e-12);
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j)
                CHECK(rel_diff(tv.sym[6 * e + MultiIndexTable::sym_index(i, j)], mt[i][j] + mt[j][i]) < 1e-12);
    }
}
// test_farfield.cpp:21-47
static void farfield_single_particle_cluster() {
    SplitMix64 rng(3);
    ParticleSet ps;
    ps.position = {random_box_point(rng, -0.5, 0.5)};
    ps.force_weight = {{0.3, -1.1, 0.7}};
    ps.dipole_weight = {{-0.2, 0.9, 0.4}};
    ps.normal = {random_unit(rng)};
    const SingleCluster sc = make_cluster(ps);
    CHECK(sc.radius == 0.0);
    CHECK(sc.center == ps.position[0]);
    const Vec3 x = ps.position[0] + Vec3{1.3, -0.4, 0.8};
    for (int p : {0, 3}) {
        const MultiIndexTable table(p + 2);
        const ClusterMoments m = compute_moments(sc.tree, p, KernelSelection::both(), table);
        FarFieldWorkspace ws;
        ws.resize_for(table);
        const Vec3 dx = x - sc.center;
        coulomb_coeffs_into(dx, table, ws.b);
        CHECK(rel_diff(stokeslet_farfield(dx, m.stokeslet_view(0), p, table, ws),
                       direct_at(ps, KernelSelection::stokeslet_only(), x)) < 1e-14);
        CHECK(rel_diff(stresslet_farfield(dx, m.stresslet_view(0), p, table, ws),
                       direct_at(ps, KernelSelection::stresslet_only(), x)) < 1e-14);
    }
}
// test_farfield.cpp:49-70
static void farfield_order_zero_monopole() {
    const ParticleSet ps = random_particles(40, 12, false);
    const SingleCluster sc = make_cluster(ps);
    const MultiIndexTable table(1);
    const ClusterMoments m = compute_moments(sc.tree, 0, KernelSelection::stokeslet_only(), table);
    FarFieldWorkspace ws;
    ws.resize_for(table);
    const Vec3 x = sc.center + Vec3{3.0, 1.0, -2.0};
    const Vec3 dx = x - sc.center;
    coulomb_coeffs_into(dx, table, ws.b);
    const Vec3 u = stokeslet_farfield(dx, m.stokeslet_view(0), 0, table, ws);
    Vec3 fsum;
    for (const Vec3& f : ps.force_weight) fsum += f;
    const Mat3 s = stokeslet(x, sc.center);
    Vec3 expected;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) expected[i] += s[i][j] * fsum[j];
    CHECK(rel_diff(u, expected) < 1e-13);
}
// test_farfield.cpp:72-100
static void farfield_contracted_equals_uncontracted() {
    SplitMix64 rng(2718);
    for (int pair = 0; pair < 12; ++pair) {
        const ParticleSet ps = random_particles(20 + pair * 5, 900 + pair, true);
        const SingleCluster sc = make_cluster(ps);
        const Vec3 dir = random_unit(rng);
        const double R = sc.radius * (1.5 + 2.5 * rng.uniform01());
        const Vec3 x = sc.center + dir * R;
        for (int p : {0, 2, 5}) {
            const MultiIndexTable table(p + 2);
            const ClusterMoments m = compute_moments(sc.tree, p, KernelSelection::both(), table);
            const Vec3 dx = x - sc.center;
            const CoulombCoeffs c = coulomb_coeffs(dx, table);
            FarFieldWorkspace ws;
            ws.b = c.b;
            CHECK(rel_diff(stokeslet_farfield(dx, m.stokeslet_view(0), p, table, ws),
                           stokeslet_uncontracted(table, c, m.stokeslet_view(0), p)) < 1e-12);
            CHECK(rel_diff(stresslet_farfield(dx, m.stresslet_view(0), p, table, ws),
                           stresslet_uncontracted(table, c, m.stresslet_view(0), p)) < 1e-12);
        }
    }
}
// test_farfield.cpp:123-139
static void farfield_zero_dipoles() {
    ParticleSet ps = random_particles(30, 217, true);
    for (Vec3& h : ps.dipole_weight) h = {0, 0, 0};
    const SingleCluster sc = make_cluster(ps);
    for (int p : {0, 4}) {
        const MultiIndexTable table(p + 2);
        const ClusterMoments m = compute_moments(sc.tree, p, KernelSelection::both(), table);
        FarFieldWorkspace ws;
        ws.resize_for(table);
        const Vec3 dx{2.0, -1.0, 1.5};
        coulomb_coeffs_into(dx, table, ws.b);
        CHECK(stresslet_farfield(dx, m.stresslet_view(0), p, table, ws) == (Vec3{0, 0, 0}));
    }
}
// test_farfield.cpp:141-168.  The reference's own errors (measured against its headers,
// below) halve at every step but one: the Stokeslet error goes 9.6008e-3 -> 5.2967e-3
// from p = 6 to 8 (ratio 1.81).  The case checks our errors equal the reference's to
// 1e-6 relative and keeps the >= 2 ratio everywhere the reference meets it.
static const double kRefDecaySto[6] = {3.772123425498e+00, 4.043395109165e-01, 1.053229570590e-01,
                                       9.600809639918e-03, 5.296708320533e-03, 8.729388631466e-04};
static const double kRefDecayStr[6] = {1.530152772136e+00, 5.688418188638e-01, 1.555222529598e-01,
                                       5.698450605266e-02, 1.559341833953e-02, 4.705758642547e-03};
static void farfield_geometric_decay() {
    const ParticleSet ps = random_particles(60, 555, true);
    const SingleCluster sc = make_cluster(ps);
    const Vec3 dir = normalized(Vec3{1.0, 0.7, -0.4});
    const Vec3 x = sc.center + dir * (sc.radius / 0.5);
    const Vec3 ex_sto = direct_at(ps, KernelSelection::stokeslet_only(), x);
    const Vec3 ex_str = direct_at(ps, KernelSelection::stresslet_only(), x);
    double es[6], et[6];
    for (int idx = 0; idx < 6; ++idx) {
        const int p = 2 * idx;
        const MultiIndexTable table(p + 2);
        const ClusterMoments m = compute_moments(sc.tree, p, KernelSelection::both(), table);
        FarFieldWorkspace ws;
        ws.resize_for(table);
        const Vec3 dx = x - sc.center;
        coulomb_coeffs_into(dx, table, ws.b);
        es[idx] = norm(stokeslet_farfield(dx, m.stokeslet_view(0), p, table, ws) - ex_sto);
        et[idx] = norm(stresslet_farfield(dx, m.stresslet_view(0), p, table, ws) - ex_str);
    }
    for (int idx = 0; idx < 6; ++idx) {
        CHECK(rel_diff(es[idx], kRefDecaySto[idx]) < 1e-6);
        CHECK(rel_diff(et[idx], kRefDecayStr[idx]) < 1e-6);
    }
    for (int idx = 0; idx + 1 < 6; ++idx) {
        if (idx != 3) CHECK(es[idx] / es[idx + 1] >= 2.0);
        CHECK(et[idx] / et[idx + 1] >= 2.0);
    }
}
// test_farfield.cpp:170-187
static void farfield_order_guards() {
    const ParticleSet ps = random_particles(10, 1, true);
    const SingleCluster sc = make_cluster(ps);
    const MultiIndexTable table(4);
    const ClusterMoments m = compute_moments(sc.tree, 2, KernelSelection::both(), table);
    FarFieldWorkspace ws;
    ws.resize_for(table);
    const Vec3 dx{3, 0, 0};
    coulomb_coeffs_into(dx, table, ws.b);
    CHECK(throws<std::invalid_argument>([&] { (void)stokeslet_farfield(dx, m.stokeslet_view(0), 3, table, ws); }));
    CHECK(throws<std::invalid_argument>([&] { (void)stresslet_farfield(dx, m.stresslet_view(0), 3, table, ws); }));
    const ClusterMoments m3 = compute_moments(sc.tree, 3, KernelSelection::both(), table);
    CHECK(throws<std::invalid_argument>([&] { (void)stresslet_farfield(dx, m3.stresslet_view(0), 3, table, ws); }));
}
// test_kernels.cpp:177-186
static void direct_target_ranges() {
    const ParticleSet ps = random_particles(40, 7, true);
    const auto full = contracted_direct_velocity(ps, KernelSelection::both());
    const auto mid = contracted_direct_velocity(ps, KernelSelection::both(), 10, 25);
    CHECK(mid.size() == 15);
    for (std::size_t i = 0; i < std::min<std::size_t>(mid.size(), 15); ++i) CHECK(mid[i] == full[i + 10]);
    CHECK(contracted_direct_velocity(ps, KernelSelection::both(), 5, 5).empty());
}
// test_engine.cpp:38-46
static void single_particle_zero_velocity() {
    ParticleSet ps;
    ps.position = {{1, 2, 3}};
    ps.force_weight = {{4, 5, 6}};
    TreecodeParams params;
    params.kernels = KernelSelection::stokeslet_only();
    CHECK(treecode_velocity(ps, params).velocity[0] == (Vec3{0, 0, 0}));
}
// test_engine.cpp:48-70
static void identical_across_runs_and_workers() {
    const ParticleSet ps = cube_particles({100000, 2500.0, 5});
    TreecodeParams params;
    params.order = 3;
    params.theta = 0.5;
    params.kernels = KernelSelection::stokeslet_only();
    params.shrink = false;
    params.workers = 1;
    const VelocityResult a = parallel_velocity(ps, params), a2 = parallel_velocity(ps, params);
    params.workers = 4;
    const VelocityResult b = parallel_velocity(ps, params);
    CHECK(a.velocity.size() == b.velocity.size());
    CHECK(std::memcmp(a.velocity.data(), a2.velocity.data(), a.velocity.size() * sizeof(Vec3)) == 0);
    CHECK(std::memcmp(a.velocity.data(), b.velocity.data(), a.velocity.size() * sizeof(Vec3)) == 0);
    CHECK(a.stats.farfield_evals == b.stats.farfield_evals);
    CHECK(a.stats.direct_pairs == b.stats.direct_pairs);
}
// test_engine.cpp:72-93 ([slow] in the reference).  The reference's own e6 is
// 5.253490138629e-4, just above the case's 5e-4 band (measured against its headers, with
// e0 = 8.303973923527e-2 and e10 = 3.224066145377e-5); north_star asks E equal to the
// reference's within 1%, so the band's upper edge becomes that.
static void sphere_accuracy_bands() {
    const ParticleSet ps = sphere_particles({5, 7});
    CHECK(ps.size() == 20480);
    const auto direct = contracted_direct_velocity(ps, KernelSelection::both());
    TreecodeParams params;
    params.theta = 0.5;
    params.kernels = KernelSelection::both();
    params.shrink = true;
    params.order = 6;
    const double e6 = relative_error(direct, treecode_velocity(ps, params).velocity);
    CHECK(e6 >= 5e-6);
    CHECK(std::abs(e6 - 5.253490138629e-4) <= 0.01 * 5.253490138629e-4);
    params.order = 0;
    const double e0 = relative_error(direct, treecode_velocity(ps, params).velocity);
    params.order = 10;
    const double e10 = relative_error(direct, treecode_velocity(ps, params).velocity);
    CHECK(e0 / e10 > 1e3);
    CHECK(std::abs(e0 - 8.303973923527e-2) <= 0.01 * 8.303973923527e-2);
    CHECK(std::abs(e10 - 3.224066145377e-5) <= 0.01 * 3.224066145377e-5);
}
// test_engine.cpp:95-105
static void high_order_small_theta() {
    const ParticleSet ps = sphere_particles({4, 11});
    const auto direct = contracted_direct_velocity(ps, KernelSelection::both());
    TreecodeParams params;
    params.order = 10;
    params.theta = 0.2;
    params.kernels = KernelSelection::both();
    params.shrink = true;
    CHECK(relative_error(direct, treecode_velocity(ps, params).velocity) < 1e-9);
}
// test_engine.cpp:107-123
static void smaller_theta_visits_more() {
    const ParticleSet ps = cube_particles({20000, 2500.0, 3});
    TreecodeParams params;
    params.order = 2;
    params.kernels = KernelSelection::stokeslet_only();
    params.shrink = false;
    params.leaf_capacity = 500;
    uint64_t visited[3];
    const double thetas[3] = {0.8, 0.5, 0.2};
    for (int i = 0; i < 3; ++i) {
        params.theta = thetas[i];
        visited[i] = treecode_velocity(ps, params).stats.clusters_visited;
    }
    CHECK(visited[0] <= visited[1]);
    CHECK(visited[1] <= visited[2]);
}
// test_engine.cpp:125-137
static void traversal_stats_consistent() {
    const ParticleSet ps = random_particles(5000, 62, false);
    TreecodeParams params;
    params.order = 4;
    params.theta = 0.6;
    params.leaf_capacity = 200;
    params.kernels = KernelSelection::stokeslet_only();
    const VelocityResult res = treecode_velocity(ps, params);
    CHECK(res.stats.farfield_evals > 0);
    CHECK(res.stats.direct_pairs > 0);
    CHECK(res.stats.clusters_visited >= ps.size());
    CHECK(res.time_total_s >= 0.0);
}

#define RUN(fn)          \
    do {                 \
        current = #fn;   \
        fn();            \
    } while (0)

int main(int argc, char** argv) {
    const std::string mode = argc > 1 ? argv[1] : "all";
    RUN(table_entry_counts);
    RUN(graded_lexicographic_ordering);
    RUN(flat_index_and_shifts);
    RUN(composite_lookups_zero_slot);
    RUN(monomial_chain);
    RUN(kernel_hand_values);
    RUN(kernels_independent_evaluation);
    RUN(kernel_symmetries);
    RUN(kernel_scale_law);
    RUN(parameter_validation);
    RUN(input_validation);
    RUN(testcases_generators);
    if (mode == "all") {
        RUN(coulomb_zero_slot);
        RUN(single_particle_tree);
        RUN(sphere_tree_structure);
        RUN(shrink_never_increases_radius);
        RUN(single_particle_moments);
        RUN(moments_definitional_loop);
        RUN(farfield_single_particle_cluster);
        RUN(farfield_order_zero_monopole);
        RUN(farfield_contracted_equals_uncontracted);
        RUN(farfield_zero_dipoles);
        RUN(farfield_geometric_decay);
        RUN(farfield_order_guards);
        RUN(direct_target_ranges);
        RUN(single_particle_zero_velocity);
        RUN(identical_across_runs_and_workers);
        RUN(sphere_accuracy_bands);
        RUN(high_order_small_theta);
        RUN(smaller_theta_visits_more);
        RUN(traversal_stats_consistent);
    }
    std::printf("%s: %d failure(s)\n", mode.c_str(), failures);
    return failures ? 1 : 0;
}
