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
