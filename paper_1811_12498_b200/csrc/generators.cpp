// Seeded synthetic inputs for the BASELINE.json configurations (host side).
//
// These are input builders, not part of the evaluated path: the same bytes are
// handed to the CUDA path and to the CPU checkers.  The stream is SplitMix64
// exactly as rng.hpp:10-29 (uniform01 = (next()>>11)*2^-53, symmetric =
// 2u-1); the per-particle draw order follows testutil::random_particles
// (tests/support/test_helpers.hpp:31-49): position, f, then h and the
// rejection-sampled unit normal (random_unit, :22-28).  Recipes per config
// are documented in DESIGN.md ("Synthetic inputs").
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <vector>

#include "stokestree_c.h"

namespace {

struct SplitMix {
    uint64_t s;
    uint64_t next() {
        uint64_t z = (s += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    double u01() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
    double sym() { return 2.0 * u01() - 1.0; }
    // rejection-sampled unit vector; v * (1/sqrt(n2)) as Vec3::operator/ does (vec3.hpp:41)
    void unit(double* out) {
        for (;;) {
            const double a = sym(), b = sym(), c = sym();
            const double n2 = a * a + b * b + c * c;
            if (n2 > 1e-4 && n2 <= 1.0) {
                const double inv = 1.0 / std::sqrt(n2);
                out[0] = a * inv;
                out[1] = b * inv;
                out[2] = c * inv;
                return;
            }
        }
    }
};

}  // namespace

extern "C" st_status st_generate(int kind, size_t n, uint64_t seed, int with_stresslets,
                                 double* pos, double* f, double* h, double* nu) {
    if (!pos) return ST_INVALID_ARGUMENT;
    if (kind != ST_GEN_POINTS && !f) return ST_INVALID_ARGUMENT;
    if (with_stresslets && kind != ST_GEN_POINTS && (!h || !nu)) return ST_INVALID_ARGUMENT;
    SplitMix r{seed};
    double centre[16][3];
    if (kind == ST_GEN_MIXTURE)
        for (auto& c : centre)
            for (double& v : c) v = -0.5 + 1.0 * r.u01();
    constexpr double kTwoPi = 6.283185307179586;
    for (size_t i = 0; i < n; ++i) {
        double* p = pos + 3 * i;
        switch (kind) {
            case ST_GEN_UNIT:  // testutil::random_box_point(rng, 0, 1)
                for (int a = 0; a < 3; ++a) p[a] = 0.0 + 1.0 * r.u01();
                break;
            case ST_GEN_CUBE:
            case ST_GEN_POINTS:  // uniform in [-0.5, 0.5)^3
                for (int a = 0; a < 3; ++a) p[a] = -0.5 + 1.0 * r.u01();
                break;
            case ST_GEN_SPHERE:  // position = outward normal = rejection unit vector
                r.unit(p);
                break;
            case ST_GEN_MIXTURE: {  // 16 isotropic Gaussians, sigma 0.05 (Box-Muller)
                const double* c = centre[r.next() % 16];
                double z[4];
                for (int k = 0; k < 2; ++k) {
                    const double u1 = r.u01(), u2 = r.u01();
                    const double rad = std::sqrt(-2.0 * std::log(1.0 - u1));
                    z[2 * k] = rad * std::cos(kTwoPi * u2);
                    z[2 * k + 1] = rad * std::sin(kTwoPi * u2);
                }
                for (int a = 0; a < 3; ++a) p[a] = c[a] + 0.05 * z[a];
                break;
            }
            default:
                return ST_INVALID_ARGUMENT;
        }
        if (kind == ST_GEN_POINTS) continue;
        for (int a = 0; a < 3; ++a) f[3 * i + a] = r.sym();
        if (with_stresslets) {
            for (int a = 0; a < 3; ++a) h[3 * i + a] = r.sym();
            if (kind == ST_GEN_SPHERE) {
                for (int a = 0; a < 3; ++a) nu[3 * i + a] = p[a];
            } else {
                r.unit(nu + 3 * i);
            }
        } else if (nu && kind == ST_GEN_SPHERE) {
            for (int a = 0; a < 3; ++a) nu[3 * i + a] = p[a];
        }
    }
    return ST_OK;
}

// ------------------------------------------------------------------ the paper's geometries
// (testcases.hpp:40-124).  Same arithmetic order as the reference so the
// particle sets are bit-identical: Vec3 a / s is a * (1 / s) and normalized(v) = v / |v|.
namespace {

struct V3 {
    double x, y, z;
};
inline V3 add(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 mul(V3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
inline double n2(V3 a) { return a.x * a.x + a.y * a.y + a.z * a.z; }
inline V3 unit(V3 a) { return mul(a, 1.0 / std::sqrt(n2(a))); }
inline V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }

struct Tri {
    V3 a, b, c;
};

}  // namespace

extern "C" size_t st_sphere_count(int levels) {
    return levels < 0 || levels > 14 ? 0 : (size_t)20 << (2 * levels);
}

// Stokeslets + stresslets at the projected centroids of an icosahedron refined `levels`
// times (N = 20 * 4^levels); normals = positions; f then h drawn per particle.
extern "C" st_status st_generate_sphere_icosa(int levels, uint64_t seed, double* pos, double* f, double* h,
                                              double* nu) {
    if (levels < 0 || levels > 14 || !pos || !f || !h || !nu) return ST_INVALID_ARGUMENT;
    const double phi = (1.0 + std::sqrt(5.0)) / 2.0;
    V3 v[12];
    int nv = 0;
    for (double s1 : {-1.0, 1.0})
        for (double s2 : {-1.0, 1.0}) {
            v[nv++] = {0.0, s1, s2 * phi};
            v[nv++] = {s1, s2 * phi, 0.0};
            v[nv++] = {s2 * phi, 0.0, s1};
        }
    const double cut = 5.0;  // edge length^2 is 4; the next pair distance^2 is 4 phi^2
    std::vector<Tri> faces;
    for (int i = 0; i < 12; ++i)
        for (int j = i + 1; j < 12; ++j) {
            if (n2(sub(v[i], v[j])) > cut) continue;
            for (int k = j + 1; k < 12; ++k) {
                if (n2(sub(v[i], v[k])) > cut || n2(sub(v[j], v[k])) > cut) continue;
                faces.push_back({unit(v[i]), unit(v[j]), unit(v[k])});
            }
        }
    for (int l = 0; l < levels; ++l) {
        std::vector<Tri> next;
        next.reserve(faces.size() * 4);
        for (const Tri& t : faces) {
            const V3 ab = unit(mul(add(t.a, t.b), 0.5));
            const V3 bc = unit(mul(add(t.b, t.c), 0.5));
            const V3 ca = unit(mul(add(t.c, t.a), 0.5));
            next.push_back({t.a, ab, ca});
            next.push_back({ab, t.b, bc});
            next.push_back({ca, bc, t.c});
            next.push_back({ab, bc, ca});
        }
        faces.swap(next);
    }
    SplitMix r{seed};
    for (size_t i = 0; i < faces.size(); ++i) {
        const Tri& t = faces[i];
        const V3 c = unit(mul(add(add(t.a, t.b), t.c), 1.0 / 3.0));
        const double cc[3] = {c.x, c.y, c.z};
        for (int a = 0; a < 3; ++a) pos[3 * i + a] = nu[3 * i + a] = cc[a];
        for (int a = 0; a < 3; ++a) f[3 * i + a] = r.sym();
        for (int a = 0; a < 3; ++a) h[3 * i + a] = r.sym();
    }
    return ST_OK;
}

// Stokeslets uniform in [0, L)^3, L = (n / density)^(1/3); draw order x1 x2 x3 f1 f2 f3.
extern "C" st_status st_generate_cube_density(size_t n, double density, uint64_t seed, double* pos,
                                              double* f) {
    if (n < 1 || !(density > 0.0) || !pos || !f) return ST_INVALID_ARGUMENT;
    const double L = std::cbrt(static_cast<double>(n) / density);
    SplitMix r{seed};
    for (size_t i = 0; i < n; ++i) {
        for (int a = 0; a < 3; ++a) pos[3 * i + a] = L * r.u01();
        for (int a = 0; a < 3; ++a) f[3 * i + a] = r.sym();
    }
    return ST_OK;
}
