// oracle/ref_harness.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Thin extern "C" shim that compiles the UNMODIFIED reference headers in place
// (-I/root/reference/proj/include; nothing is copied into this repo) into
// oracle/_ref/libstref.so, so tests and bench.py's reference arm can call the
// reference's own treecode through ctypes.  Built by oracle/Makefile with the
// reference's flags (g++ -std=c++20 -O2, no -march => no FMA).
//
// Exceptions map to status codes: 1 invalid_argument, 2 domain_error, 5 other.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <thread>
#include <vector>

#include "stokestree/cluster_tree.hpp"
#include "stokestree/coulomb.hpp"
#include "stokestree/engine.hpp"
#include "stokestree/error_metric.hpp"
#include "stokestree/farfield.hpp"
#include "stokestree/kernels.hpp"
#include "stokestree/moments.hpp"
#include "stokestree/multi_index.hpp"
#include "stokestree/particle_io.hpp"
#include "stokestree/taylor_coeffs.hpp"
#include "stokestree/testcases.hpp"

using namespace stokestree;

namespace {

int code_of(const std::exception_ptr& e) {
    try {
        std::rethrow_exception(e);
    } catch (const std::invalid_argument&) {
        return 1;
    } catch (const std::domain_error&) {
        return 2;
    } catch (...) {
        return 5;
    }
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

std::vector<Vec3> to_vec(const double* a, std::size_t n) {
    std::vector<Vec3> v;
    if (!a) return v;
    v.resize(n);
    for (std::size_t i = 0; i < n; ++i) v[i] = Vec3{a[3 * i], a[3 * i + 1], a[3 * i + 2]};
    return v;
}

ParticleSet make_ps(std::size_t n, const double* pos, const double* f, const double* h,
                    const double* nu) {
    ParticleSet ps;
    ps.position = to_vec(pos, n);
    ps.force_weight = to_vec(f, n);
    ps.dipole_weight = to_vec(h, n);
    ps.normal = to_vec(nu, n);
    return ps;
}

void put(double* out, std::size_t i, const Vec3& v) {
    out[3 * i] = v[0];
    out[3 * i + 1] = v[1];
    out[3 * i + 2] = v[2];
}

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

struct RefCtx {
    ClusterTree tree;
    MultiIndexTable table;
    ClusterMoments moments;
    TreecodeParams params;
    RefCtx(ClusterTree&& t, int pmax, ClusterMoments&& m, const TreecodeParams& p)
        : tree(std::move(t)), table(pmax), moments(std::move(m)), params(p) {}
};

}  // namespace

extern "C" {

// Full reference call: parallel_velocity (engine.hpp:194-196) with `workers` threads.
// u_out original order; stats3 = {farfield_evals, direct_pairs, clusters_visited};
// times4 = {build, moments, traverse, total} seconds.
int ref_parallel_velocity(std::size_t n, const double* pos, const double* f, const double* h,
                          const double* nu, int order, double theta, int n0, int shrink, int sto,
                          int str, int workers, double* u_out, uint64_t* stats3, double* times4) {
    return guarded([&] {
        const ParticleSet ps = make_ps(n, pos, f, h, nu);
        TreecodeParams p;
        p.order = order;
        p.theta = theta;
        p.leaf_capacity = n0;
        p.shrink = shrink != 0;
        p.kernels = KernelSelection{sto != 0, str != 0};
        p.workers = workers;
        const VelocityResult r = parallel_velocity(ps, p);
        for (std::size_t i = 0; i < r.velocity.size(); ++i) put(u_out, i, r.velocity[i]);
        if (stats3) {
            stats3[0] = r.stats.farfield_evals;
            stats3[1] = r.stats.direct_pairs;
            stats3[2] = r.stats.clusters_visited;
        }
        if (times4) {
            times4[0] = r.time_build_s;
            times4[1] = r.time_moments_s;
            times4[2] = r.time_traverse_s;
            times4[3] = r.time_total_s;
        }
    });
}

// Build tree + moments once (build_tree, compute_moments with `workers` threads).
void* ref_ctx_new(std::size_t n, const double* pos, const double* f, const double* h,
                  const double* nu, int order, double theta, int n0, int shrink, int sto, int str,
                  int workers, double* t_build, double* t_moments, int* status) {
    RefCtx* ctx = nullptr;
    *status = guarded([&] {
        const ParticleSet ps = make_ps(n, pos, f, h, nu);
        TreecodeParams p;
        p.order = order;
        p.theta = theta;
        p.leaf_capacity = n0;
        p.shrink = shrink != 0;
        p.kernels = KernelSelection{sto != 0, str != 0};
        p.workers = workers;
        p.validate();
        validate(ps, p.kernels);
        const double t0 = now_s();
        ClusterTree tree = build_tree(ps, n0, shrink != 0);
        const double t1 = now_s();
        const int pmax = order + (str ? 2 : 1);
        MultiIndexTable table(pmax);
        ClusterMoments m = compute_moments(tree, order, p.kernels, table, workers);
        const double t2 = now_s();
        ctx = new RefCtx(std::move(tree), pmax, std::move(m), p);
        if (t_build) *t_build = t1 - t0;
        if (t_moments) *t_moments = t2 - t1;
    });
    return ctx;
}

void ref_ctx_free(void* c) { delete static_cast<RefCtx*>(c); }

std::size_t ref_ctx_ncl(void* c) { return static_cast<RefCtx*>(c)->tree.clusters.size(); }

// Same layout as or_tree_export in stokes_oracle.c.
void ref_ctx_export_tree(void* c, int64_t* be, double* geom, int32_t* kids, int32_t* meta,
                         uint32_t* perm) {
    const ClusterTree& T = static_cast<RefCtx*>(c)->tree;
    for (std::size_t i = 0; i < T.clusters.size(); ++i) {
        const Cluster& cl = T.clusters[i];
        if (be) {
            be[2 * i] = static_cast<int64_t>(cl.begin);
            be[2 * i + 1] = static_cast<int64_t>(cl.end);
        }
        if (geom) {
            double* g = geom + 10 * i;
            for (int a = 0; a < 3; ++a) {
                g[a] = cl.center[a];
                g[4 + a] = cl.bbox.lo[a];
                g[7 + a] = cl.bbox.hi[a];
            }
            g[3] = cl.radius;
        }
        if (kids)
            for (int s = 0; s < 8; ++s) kids[8 * i + s] = s < cl.n_children ? cl.children[s] : -1;
        if (meta) {
            meta[2 * i] = cl.n_children;
            meta[2 * i + 1] = cl.is_leaf ? 1 : 0;
        }
    }
    if (perm) std::memcpy(perm, T.to_original.data(), sizeof(uint32_t) * T.to_original.size());
}

// Moments of every cluster (ClusterMoments layout, moments.hpp:85-134).
void ref_ctx_moments(void* c, double* stok, double* strm, double* trace, double* sym) {
    const RefCtx* ctx = static_cast<RefCtx*>(c);
    const std::size_t ncl = ctx->tree.clusters.size();
    const std::size_t E = static_cast<std::size_t>(ctx->moments.entry_count());
    for (std::size_t i = 0; i < ncl; ++i) {
        if (stok && ctx->params.kernels.stokeslet_enabled) {
            auto v = ctx->moments.stokeslet_view(i);
            std::memcpy(stok + 3 * E * i, v.m.data(), sizeof(double) * 3 * E);
        }
        if (strm && ctx->params.kernels.stresslet_enabled) {
            auto v = ctx->moments.stresslet_view(i);
            std::memcpy(strm + 9 * E * i, v.mt.data(), sizeof(double) * 9 * E);
            std::memcpy(trace + E * i, v.trace.data(), sizeof(double) * E);
            std::memcpy(sym + 6 * E * i, v.sym.data(), sizeof(double) * 6 * E);
        }
    }
}

// Traverse selected targets with detail::accumulate_velocity (engine.hpp:80-108), each
// with a fresh TraversalStats.  Targets: original source indices (self excluded by
// their tree index) when xyz == NULL, else disjoint points (skip = kNoSkip).  Threads
// split the list into contiguous segments.  per_target (3*nt: visited, far, direct).
int ref_ctx_eval(void* c, std::size_t nt, const int64_t* src_idx, const double* xyz,
                 int nthreads, double* u_out, uint64_t* per_target, uint64_t* stats3) {
    RefCtx* ctx = static_cast<RefCtx*>(c);
    const detail::TraversalContext tc{ctx->tree, ctx->moments, ctx->table, ctx->params.kernels,
                                      ctx->params.order, ctx->params.theta};
    if (nthreads < 1) nthreads = 1;
    if (static_cast<std::size_t>(nthreads) > nt) nthreads = nt ? static_cast<int>(nt) : 1;
    std::vector<std::exception_ptr> errs(nthreads);
    std::vector<TraversalStats> tot(nthreads);
    auto work = [&](int w) {
        try {
            FarFieldWorkspace ws;
            ws.resize_for(ctx->table);
            const std::size_t t0 = nt * w / nthreads, t1 = nt * (w + 1) / nthreads;
            for (std::size_t i = t0; i < t1; ++i) {
                TraversalStats s;
                Vec3 u;
                if (xyz) {
                    const Vec3 x{xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]};
                    detail::accumulate_velocity(tc, x, detail::kNoSkip, 0, u, ws, s);
                } else {
                    const std::size_t t = ctx->tree.to_tree[static_cast<std::size_t>(src_idx[i])];
                    detail::accumulate_velocity(tc, ctx->tree.particles.position[t], t, 0, u, ws, s);
                }
                put(u_out, i, u);
                if (per_target) {
                    per_target[3 * i] = s.clusters_visited;
                    per_target[3 * i + 1] = s.farfield_evals;
                    per_target[3 * i + 2] = s.direct_pairs;
                }
                tot[w] += s;
            }
        } catch (...) {
            errs[w] = std::current_exception();
        }
    };
    std::vector<std::thread> th;
    for (int w = 1; w < nthreads; ++w) th.emplace_back(work, w);
    work(0);
    for (auto& t : th) t.join();
    for (auto& e : errs)
        if (e) return code_of(e);
    TraversalStats all;
    for (auto& s : tot) all += s;
    if (stats3) {
        stats3[0] = all.farfield_evals;
        stats3[1] = all.direct_pairs;
        stats3[2] = all.clusters_visited;
    }
    return 0;
}

// contracted_direct_velocity_at (kernels.hpp:139-150), threaded over the target list.
int ref_direct_at(std::size_t n, const double* pos, const double* f, const double* h,
                  const double* nu, int sto, int str, const int64_t* targets, std::size_t nt,
                  int nthreads, double* u_out) {
    return guarded([&] {
        const ParticleSet ps = make_ps(n, pos, f, h, nu);
        const KernelSelection sel{sto != 0, str != 0};
        if (nthreads < 1) nthreads = 1;
        std::vector<std::exception_ptr> errs(nthreads);
        auto work = [&](int w) {
            try {
                const std::size_t t0 = nt * w / nthreads, t1 = nt * (w + 1) / nthreads;
                std::vector<std::size_t> sub;
                for (std::size_t i = t0; i < t1; ++i) sub.push_back(static_cast<std::size_t>(targets[i]));
                const auto u = contracted_direct_velocity_at(ps, sel, sub);
                for (std::size_t i = t0; i < t1; ++i) put(u_out, i, u[i - t0]);
            } catch (...) {
                errs[w] = std::current_exception();
            }
        };
        std::vector<std::thread> th;
        for (int w = 1; w < nthreads; ++w) th.emplace_back(work, w);
        work(0);
        for (auto& t : th) t.join();
        for (auto& e : errs)
            if (e) std::rethrow_exception(e);
    });
}

// naive_direct_velocity (kernels.hpp:89-118), tensor-forming oracle.
int ref_naive_direct(std::size_t n, const double* pos, const double* f, const double* h,
                     const double* nu, int sto, int str, double* u_out) {
    return guarded([&] {
        const auto u = naive_direct_velocity(make_ps(n, pos, f, h, nu), KernelSelection{sto != 0, str != 0});
        for (std::size_t i = 0; i < u.size(); ++i) put(u_out, i, u[i]);
    });
}

// coulomb_coeffs (coulomb.hpp:52-59): b_out sized E(pmax)+1.
int ref_coulomb(const double* dx, int pmax, double* b_out) {
    return guarded([&] {
        const MultiIndexTable t(pmax);
        const CoulombCoeffs c = coulomb_coeffs(Vec3{dx[0], dx[1], dx[2]}, t);
        std::memcpy(b_out, c.b.data(), sizeof(double) * c.b.size());
    });
}

// Explicit Taylor coefficients (taylor_coeffs.hpp:13-46) for every flat_k of grade <= order,
// from coulomb_coeffs at depth pmax_b; layouts as or_taylor.
int ref_taylor(const double* dx, int pmax_b, int order, double* a_sto, double* a_str) {
    return guarded([&] {
        const MultiIndexTable t(pmax_b);
        const CoulombCoeffs c = coulomb_coeffs(Vec3{dx[0], dx[1], dx[2]}, t);
        const int E = (order + 1) * (order + 2) * (order + 3) / 6;
        for (int e = 0; e < E; ++e)
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) {
                    if (a_sto) a_sto[e * 9 + 3 * i + j] = stokeslet_taylor_coeff(t, c, e, i, j);
                    if (a_str)
                        for (int l = 0; l < 3; ++l)
                            a_str[e * 27 + 9 * i + 3 * j + l] = stresslet_taylor_coeff(t, c, e, i, j, l);
                }
    });
}

// One far-field pair from explicit moments (farfield.hpp:30-96), Stokeslet + stresslet.
int ref_farfield_pair(const double* dx, int p, int sto, int str, const double* stok,
                      const double* strm, const double* trace, const double* sym, double* u) {
    return guarded([&] {
        const MultiIndexTable t(p + (str ? 2 : 1));
        const std::size_t E = static_cast<std::size_t>(t.size_at(p));
        FarFieldWorkspace ws;
        ws.resize_for(t);
        const Vec3 d{dx[0], dx[1], dx[2]};
        coulomb_coeffs_into(d, t, ws.b);
        Vec3 r;
        if (sto) r += stokeslet_farfield(d, StokesletMomentsView{std::span<const double>(stok, 3 * E)}, p, t, ws);
        if (str)
            r += stresslet_farfield(d,
                                    StressletMomentsView{std::span<const double>(strm, 9 * E),
                                                         std::span<const double>(trace, E),
                                                         std::span<const double>(sym, 6 * E)},
                                    p, t, ws);
        u[0] = r[0];
        u[1] = r[1];
        u[2] = r[2];
    });
}

// testcases.hpp:66-124 generators; arrays sized by the caller (sphere: 20*4^levels).
int ref_sphere_particles(int levels, uint64_t seed, double* pos, double* f, double* h, double* nu) {
    return guarded([&] {
        const ParticleSet ps = sphere_particles({levels, seed});
        for (std::size_t i = 0; i < ps.size(); ++i) {
            put(pos, i, ps.position[i]);
            put(f, i, ps.force_weight[i]);
            put(h, i, ps.dipole_weight[i]);
            put(nu, i, ps.normal[i]);
        }
    });
}

int ref_cube_particles(std::size_t n, double density, uint64_t seed, double* pos, double* f) {
    return guarded([&] {
        const ParticleSet ps = cube_particles({n, density, seed});
        for (std::size_t i = 0; i < ps.size(); ++i) {
            put(pos, i, ps.position[i]);
            put(f, i, ps.force_weight[i]);
        }
    });
}

// particle_io.hpp: write with the reference writer; read back into caller arrays (n known).
int ref_write_particles(const char* path, std::size_t n, const double* pos, const double* f, const double* h,
                        const double* nu, int sto, int str) {
    return guarded([&] { write_particles(path, make_ps(n, pos, f, h, nu), KernelSelection{sto != 0, str != 0}); });
}

int ref_read_particles(const char* path, std::size_t cap, std::size_t* n, int* sto, int* str, double* pos,
                       double* f, double* h, double* nu) {
    return guarded([&] {
        const LoadedParticles L = read_particles(path);
        *n = L.particles.size();
        *sto = L.selection.stokeslet_enabled;
        *str = L.selection.stresslet_enabled;
        for (std::size_t i = 0; i < L.particles.size() && i < cap; ++i) {
            put(pos, i, L.particles.position[i]);
            if (*sto) put(f, i, L.particles.force_weight[i]);
            if (*str) {
                put(h, i, L.particles.dipole_weight[i]);
                put(nu, i, L.particles.normal[i]);
            }
        }
    });
}

int ref_relative_error(std::size_t n, const double* ref, const double* test, double* out) {
    return guarded([&] {
        const auto a = to_vec(ref, n), b = to_vec(test, n);
        *out = relative_error(a, b);
    });
}

}  // extern "C"
