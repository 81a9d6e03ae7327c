// Reference-style checks written against the drop-in headers (include/stokestree/),
// i.e. the way a user of the reference calls it.  Mirrors assertions of the
// reference's test_engine.cpp, test_kernels.cpp, test_cluster_tree.cpp,
// test_farfield.cpp and test_multi_index.cpp.  Exit code 0 = all passed.
// Modes: "host" (no GPU needed: validation and index bookkeeping) or "all".
#include <cstdio>
#include <cstring>
#include <string>

#include "stokestree/engine.hpp"
#include "stokestree/error_metric.hpp"
#include "stokestree/farfield.hpp"
#include "stokestree/kernels.hpp"
#include "stokestree/moments.hpp"
#include "stokestree/multi_index.hpp"
#include "stokestree/taylor_coeffs.hpp"

using namespace stokestree;

static int failures = 0;
#define CHECK(cond)                                                            \
    do {                                                                       \
        if (!(cond)) {                                                         \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);        \
            ++failures;                                                        \
        }                                                                      \
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
        ps.position.push_back({r.uniform01(), r.uniform01(), r.uniform01()});
        ps.force_weight.push_back({r.symmetric(), r.symmetric(), r.symmetric()});
        if (str) {
            ps.dipole_weight.push_back({r.symmetric(), r.symmetric(), r.symmetric()});
            ps.normal.push_back(random_unit(r));
        }
    }
    return ps;
}

static void host_checks() {
    TreecodeParams p;
    p.theta = 1.0;
    CHECK(throws<std::invalid_argument>([&] { p.validate(); }));
    p.theta = 0.5;
    p.order = TreecodeParams::kMaxOrder + 1;
    CHECK(throws<std::invalid_argument>([&] { p.validate(); }));
    p.order = 6;
    p.kernels = {false, false};
    CHECK(throws<std::invalid_argument>([&] { p.validate(); }));
    p.kernels = KernelSelection::both();
    p.validate();
    const MultiIndexTable t(6);
    CHECK(MultiIndexTable(10).size() == 286);
    for (int e = 0; e < t.size(); ++e) {
        const MultiIndex& k = t[e];
        CHECK(t.flat_index(k.k[0], k.k[1], k.k[2]) == e);
        for (int a = 0; a < 3; ++a)
            for (int d : {-2, -1, 1, 2}) {
                int c[3] = {k.k[0], k.k[1], k.k[2]};
                c[a] += d;
                CHECK(t.shift(e, a, d) == t.flat_index(c[0], c[1], c[2]));
            }
        if (e > 0) {
            MultiIndex q = t[t.mono_parent(e)];
            q.k[t.mono_axis(e)] += 1;
            CHECK(q == t[e]);
        }
    }
    CHECK(t.flat_index(3, 2, 2) == MultiIndexTable::kInvalid);
    const Mat3 s = stokeslet({1, 0, 0}, {0, 0, 0});
    CHECK(s[0][0] == 2.0 && s[1][1] == 1.0 && s[0][1] == 0.0);
    CHECK(throws<std::domain_error>([] { stokeslet({1, 2, 3}, {1, 2, 3}); }));
    ParticleSet bad = random_particles(10, 1, true);
    bad.normal[4] = bad.normal[4] * (1.0 + 1e-9);
    CHECK(throws<std::invalid_argument>([&] { validate(bad, KernelSelection::both()); }));
}

static void device_checks() {
    // vanishing theta degenerates to the direct sum (test_engine.cpp:12-24)
    {
        const ParticleSet ps = random_particles(3000, 9001, true);
        TreecodeParams p;
        p.order = 5;
        p.theta = 1e-9;
        p.leaf_capacity = 100;
        const VelocityResult r = treecode_velocity(ps, p);
        const auto d = contracted_direct_velocity(ps, KernelSelection::both());
        CHECK(r.stats.farfield_evals == 0);
        CHECK(relative_error(d, r.velocity) <= 1e-13);
    }
    // results identical across runs and worker counts (test_engine.cpp:48-70)
    {
        const ParticleSet ps = random_particles(20000, 5, false);
        TreecodeParams p;
        p.order = 3;
        p.kernels = KernelSelection::stokeslet_only();
        p.shrink = false;
        const VelocityResult a = parallel_velocity(ps, p);
        p.workers = 4;
        const VelocityResult b = parallel_velocity(ps, p);
        CHECK(std::memcmp(a.velocity.data(), b.velocity.data(), a.velocity.size() * sizeof(Vec3)) == 0);
        CHECK(a.stats.direct_pairs == b.stats.direct_pairs);
        // the library's cached device memory can be released between calls
        release_workspace();
        const VelocityResult c = parallel_velocity(ps, p);
        CHECK(std::memcmp(a.velocity.data(), c.velocity.data(), a.velocity.size() * sizeof(Vec3)) == 0);
    }
    // stored radius equals brute force recomputation (test_cluster_tree.cpp:103-114)
    {
        const ParticleSet ps = random_particles(3000, 5, false);
        for (bool shrink : {false, true}) {
            const ClusterTree tree = build_tree(ps, 100, shrink);
            for (const Cluster& c : tree.clusters) {
                double m = 0.0;
                for (std::size_t k = c.begin; k < c.end; ++k)
                    m = std::max(m, norm2(tree.particles.position[k] - c.center));
                CHECK(std::sqrt(m) == c.radius);
            }
        }
    }
    // zeroth moment is the weight sum (test_cluster_tree.cpp:141-163)
    {
        const ParticleSet ps = random_particles(500, 9, true);
        const ClusterTree tree = build_tree(ps, 64, true);
        const MultiIndexTable table(3);
        const ClusterMoments m = compute_moments(tree, 3, KernelSelection::both(), table);
        for (std::size_t c = 0; c < tree.clusters.size(); ++c) {
            Vec3 fs;
            for (std::size_t k = tree.clusters[c].begin; k < tree.clusters[c].end; ++k)
                fs += tree.particles.force_weight[k];
            for (int j = 0; j < 3; ++j)
                CHECK(std::abs(m.stokeslet_view(c).m[j] - fs[j]) <= 1e-13 * std::max(1.0, std::abs(fs[j])));
        }
    }
    // far field at p = 10, r/R = 0.2 within 1e-8 of the direct sum (test_farfield.cpp:102-121)
    {
        const ParticleSet ps = random_particles(50, 314, true);
        const ClusterTree tree = build_tree(ps, 51, true);
        const int p = 10;
        const MultiIndexTable table(p + 2);
        const ClusterMoments m = compute_moments(tree, p, KernelSelection::both(), table);
        FarFieldWorkspace ws;
        ws.resize_for(table);
        SplitMix64 rng(315);
        for (int rep = 0; rep < 5; ++rep) {
            const Vec3 x = tree.root().center + random_unit(rng) * (tree.root().radius / 0.2);
            const Vec3 dx = x - tree.root().center;
            coulomb_coeffs_into(dx, table, ws.b);
            const Vec3 u = stokeslet_farfield(dx, m.stokeslet_view(0), p, table, ws) +
                           stresslet_farfield(dx, m.stresslet_view(0), p, table, ws);
            Vec3 ex;
            for (std::size_t k = 0; k < ps.size(); ++k) {
                const Mat3 S = stokeslet(x, ps.position[k]);
                const Ten3 T = stresslet(x, ps.position[k]);
                for (int i = 0; i < 3; ++i)
                    for (int j = 0; j < 3; ++j) {
                        ex[i] += S[i][j] * ps.force_weight[k][j];
                        for (int l = 0; l < 3; ++l) ex[i] += T[i][j][l] * ps.dipole_weight[k][j] * ps.normal[k][l];
                    }
            }
            CHECK(norm(u - ex) / norm(ex) < 1e-8);
        }
    }
    // explicit Taylor coefficients (test_taylor_coeffs.cpp:33-66, 118-126)
    {
        const MultiIndexTable t2(2);
        CHECK(std::fabs(stokeslet_taylor_coeff(t2, coulomb_coeffs({1, 0, 0}, t2), 0, 0, 0) - 2.0) < 1e-14);
        CHECK(stokeslet_taylor_coeff(t2, coulomb_coeffs({0, 0, 1}, t2), 0, 0, 1) == 0.0);
        const double a = stresslet_taylor_coeff(t2, coulomb_coeffs({1, 1, 1}, t2), 0, 0, 0, 0);
        CHECK(std::fabs(a - 1.0 / (9.0 * std::sqrt(3.0))) < 1e-13 * a);
        const MultiIndexTable t3(3);
        const CoulombCoeffs c = coulomb_coeffs({1, 1, 0}, t3);
        bool threw = false;
        try { (void)stokeslet_taylor_coeff(t3, c, t3.size_at(3) - 1, 0, 0); } catch (const std::invalid_argument&) { threw = true; }
        CHECK(threw);
        threw = false;
        try { (void)stresslet_taylor_coeff(t3, c, t3.size_at(2) - 1, 0, 0, 0); } catch (const std::invalid_argument&) { threw = true; }
        CHECK(threw);
        // zeroth coefficient reproduces the tensors (test_taylor_coeffs.cpp:13-31)
        const Vec3 x{0.3, -0.7, 0.2}, y{-0.1, 0.4, 0.9};
        const CoulombCoeffs cx = coulomb_coeffs(x - y, t3);
        const Mat3 S = stokeslet(x, y);
        const Ten3 T = stresslet(x, y);
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) {
                CHECK(std::fabs(stokeslet_taylor_coeff(t3, cx, 0, i, j) - S[i][j]) <= 1e-12 * std::fabs(S[i][j]));
                for (int l = 0; l < 3; ++l)
                    CHECK(std::fabs(stresslet_taylor_coeff(t3, cx, 0, i, j, l) - T[i][j][l]) <=
                          1e-12 * std::fabs(T[i][j][l]));
            }
    }
    // coincident particles -> domain_error (test_kernels.cpp:188-196)
    {
        ParticleSet ps;
        ps.position = {{0, 0, 0}, {1, 1, 1}, {0, 0, 0}};
        ps.force_weight = {{1, 0, 0}, {1, 0, 0}, {1, 0, 0}};
        CHECK(throws<std::domain_error>([&] { contracted_direct_velocity(ps, KernelSelection::stokeslet_only()); }));
    }
}

int main(int argc, char** argv) {
    const std::string mode = argc > 1 ? argv[1] : "all";
    host_checks();
    if (mode == "all") device_checks();
    std::printf("%s: %d failure(s)\n", mode.c_str(), failures);
    return failures ? 1 : 0;
}
