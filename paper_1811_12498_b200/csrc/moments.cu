// K2: moments of every cluster directly from its particles (moments.hpp:34-80,
// compute_moments :140-175), then the fold into far-field weights.
//
// Moments: one CTA per (cluster, chunk of <= kChunk particles).  Particles of a
// tile are staged in shared memory as powers d_a^0..d_a^p per axis plus their
// 12 weights (f, h (x) nu); thread e owns multi-indices e, e+256, ... and
// accumulates mono_k * w for every weight column.  Clusters spanning several
// chunks write per-chunk partials that a second kernel sums in chunk order, so
// the result is deterministic and identical on every GPU.
//
// Fold: the reference's contracted far fields (farfield.hpp
// Eq. 25 / Eq. 30) equal sum_k a^k_ij M_j^k + a~^k_ijl M~_jl^k with the exact
// Taylor coefficients a, a~ (taylor_coeffs.hpp:13-46).  Writing S and T with the
// free index carried by (x - y)_i gives u_i = Phi_i(dx) + dx_i Psi(dx) with four
// harmonic potentials, Phi_i = sum_q b_q alpha_i[q], Psi = sum_q b_q psi[q]:
//   Stokeslet, per k (|k| <= p):
//     alpha_i[k]          += (1 - k_i) M_i^k
//     alpha_i[k+e_j-e_i]  -= (k_j + 1) M_j^k            (j != i)
//     psi[k+e_j]          += (k_j + 1) M_j^k
//   stresslet:
//     psi[k+e_j+e_l]      += (k_j+1)(k_l+1+d_jl) M~_jl^k / 3
//     alpha_i[k-e_i+e_j+e_l] -= k_i (m!/k!) M~_jl^k / 3  (m = k-e_i+e_j+e_l)
//     alpha_i[k+e_i]      += (k_i + 1) tr(M~^k) / 3
// and, because 1/r is harmonic (sum_i (k_i+1)(k_i+2) b^{k+2e_i} = 0), every
// weight at k3 >= 2 is folded onto k3 - 2 until only k3 in {0,1} remain:
// (P+1)^2 coefficients instead of E(P).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "moments.cuh"
#include "sph_basis.cuh"
#include "tma.cuh"

namespace st {

namespace {

constexpr int kThreads = 256;
#ifndef ST_MOMENTS_TILE
#define ST_MOMENTS_TILE 32
#endif
constexpr int kTileP = ST_MOMENTS_TILE;  // particles per shared-memory tile
constexpr int kChunk = 8192;    // particles per work item
constexpr int kPmax = 16;
constexpr int kPow = kPmax + 1; // powers 0..p per axis
static_assert(kPmax + 2 <= kSphPmax, "solid-harmonic basis table too short");

__device__ __forceinline__ int find_item(const int32_t* __restrict__ off, int n, int item) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (off[mid] <= item) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// flat graded-lex index -> (k1,k2,k3) (multi_index.hpp:36-44)
__device__ __forceinline__ void mi_decode(int e, int& k1, int& k2, int& k3) {
    int s = 0;
    while (mi_count(s) <= e) ++s;
    int r = e - (s == 0 ? 0 : mi_count(s - 1));
    k1 = 0;
    while (r >= s - k1 + 1) {
        r -= s - k1 + 1;
        ++k1;
    }
    k2 = r;
    k3 = s - k1 - k2;
}

// Thread t owns multi-indices t, t+T, ..., t+(EPT-1)T (T = blockDim.x, sized to E), so a
// particle's 12 weights, read once as shared-memory broadcasts, feed 12*EPT FMAs.
template <int EPT, bool STO, bool STR>
__global__ void __launch_bounds__(kThreads)
    k_moments(int ncl_items, const int32_t* __restrict__ item_off, const int32_t* __restrict__ item_cl,
              int nmulti, const int4* __restrict__ info, const double4* __restrict__ geom,
              const double* __restrict__ src, int p, int E, const int32_t* __restrict__ part_slot,
              double* __restrict__ M, double* __restrict__ part) {
    constexpr int NC = (STO ? 3 : 0) + (STR ? 9 : 0);
    constexpr int NCP = (NC + 1) & ~1;  // padded to whole double2
    constexpr int C0 = STO ? 0 : 3;     // first combined column written
    __shared__ double s_pow[kTileP][3 * kPow + 1];
    __shared__ __align__(16) double s_w[kTileP][NCP];
    __shared__ int s_k[4 * kThreads][3];
    const int T = blockDim.x;

    const int item = blockIdx.x;
    const int ci = find_item(item_off, ncl_items, item);  // index into the cluster list
    const int v = item_cl[ci];
    const int chunk = item - item_off[ci];
    const int4 inf = info[v];
    const double4 g = geom[v];
    const int b = inf.x + chunk * kChunk;
    const int e_end = min(inf.y, b + kChunk);

    for (int t = threadIdx.x; t < EPT * T; t += T) {
        int k1 = 0, k2 = 0, k3 = 0;
        if (t < E) mi_decode(t, k1, k2, k3);
        s_k[t][0] = k1;
        s_k[t][1] = k2;
        s_k[t][2] = k3;
    }

    double acc[EPT][NCP];
#pragma unroll
    for (int j = 0; j < EPT; ++j)
#pragma unroll
        for (int c = 0; c < NCP; ++c) acc[j][c] = 0.0;

    // the tile's contiguous tree-ordered records arrive by TMA, one tile ahead of the
    // staging that reads them (no global-load latency between the tiles)
    __shared__ __align__(128) double s_raw[2][kTileP * 12];
    __shared__ __align__(8) uint64_t s_bar[2];
    if (threadIdx.x == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        mbar_fence_init();
        if (b < e_end) bulk_g2s(s_raw[0], src + 12 * (size_t)b, 96u * min(kTileP, e_end - b), &s_bar[0]);
    }
    int it = 0;
    for (int t0 = b; t0 < e_end; t0 += kTileP, ++it) {
        const int nt = min(kTileP, e_end - t0);
        const int cur = it & 1;
        __syncthreads();  // the previous tile's compute is done with s_pow / s_w
        if (threadIdx.x == 0 && t0 + kTileP < e_end)  // s_raw[cur ^ 1] was staged last iteration
            bulk_g2s(s_raw[cur ^ 1], src + 12 * (size_t)(t0 + kTileP), 96u * min(kTileP, e_end - t0 - kTileP),
                     &s_bar[cur ^ 1]);
        mbar_wait(&s_bar[cur], (it >> 1) & 1);
        // one thread per (particle, axis): the axis' power chain, f_a and the row h_a nu_l
        for (int x = threadIdx.x; x < 3 * nt; x += T) {
            const int q = x / 3, a = x - 3 * q;
            const double* r = s_raw[cur] + 12 * q;
            const double d = r[a] - (a == 0 ? g.x : a == 1 ? g.y : g.z);
            double pw = 1.0;
            s_pow[q][a * kPow] = 1.0;
            for (int k = 1; k <= p; ++k) {
                pw *= d;
                s_pow[q][a * kPow + k] = pw;
            }
            if (STO) s_w[q][a] = r[3 + a];
            if (STR)
                for (int l = 0; l < 3; ++l) s_w[q][(STO ? 3 : 0) + 3 * a + l] = r[6 + a] * r[9 + l];
            if (NCP > NC && a == 0) s_w[q][NCP - 1] = 0.0;
        }
        __syncthreads();
        int kk[EPT][3];
#pragma unroll
        for (int j = 0; j < EPT; ++j)
#pragma unroll
            for (int a = 0; a < 3; ++a) kk[j][a] = s_k[threadIdx.x + j * T][a];
        for (int q = 0; q < nt; ++q) {
            double w[NCP];
#pragma unroll
            for (int c = 0; c < NCP; c += 2) {
                const double2 x = *reinterpret_cast<const double2*>(&s_w[q][c]);
                w[c] = x.x;
                w[c + 1] = x.y;
            }
#pragma unroll
            for (int j = 0; j < EPT; ++j) {
                const double mono = s_pow[q][kk[j][0]] * s_pow[q][kPow + kk[j][1]] * s_pow[q][2 * kPow + kk[j][2]];
#pragma unroll
                for (int c = 0; c < NC; ++c) acc[j][c] = fma(mono, w[c], acc[j][c]);
            }
        }
    }
    const int slot = part_slot[ci];
    double* out = slot < 0 ? M + (size_t)v * E * 12 : part + ((size_t)slot + chunk) * E * 12;
#pragma unroll
    for (int j = 0; j < EPT; ++j) {
        const int e = threadIdx.x + j * T;
        if (e < E) {
#pragma unroll
            for (int c = 0; c < NC; ++c) out[(size_t)e * 12 + C0 + c] = acc[j][c];
        }
    }
}

// M2M (exact algebra): the moments of a cluster about its centre c_p from its children's
// moments about theirs, M_p[k] = sum_children sum_{j<=k} C(k,j) (c_c - c_p)^(k-j) M_c[j]
// (componentwise binomials).  The shift is separable, so it runs as three 1-D passes
// (z, then y, then x) through shared memory: every entry costs at most p+1 terms per pass
// instead of prod(k_a+1) (up to 80 at p = 10), which balanced the threads of a CTA.
// Children in slot order, fixed term order: deterministic.
template <int EPT, bool STO, bool STR>
__global__ void __launch_bounds__(kThreads)
    k_m2m(const int32_t* __restrict__ ids, const int32_t* __restrict__ children,
          const int32_t* __restrict__ nchild, const double4* __restrict__ geom, int p, int E,
          double* __restrict__ M) {
    constexpr int NC = (STO ? 3 : 0) + (STR ? 9 : 0);
    constexpr int C0 = STO ? 0 : 3;
    extern __shared__ __align__(16) double m2m_smem[];
    double* Ma = m2m_smem;                         // [E][12] child moments / y-pass output
    double* Mb = m2m_smem + (size_t)E * 12;        // [E][12] z-pass output
    double* A = m2m_smem + (size_t)E * 24;         // [3][p+1][p+1]: C(k,j) d^(k-j)
    const int T = blockDim.x;
    const int v = ids[blockIdx.x];
    const double4 gp = geom[v];
    int kk[EPT][3];
#pragma unroll
    for (int j = 0; j < EPT; ++j) {
        const int e = threadIdx.x + j * T;
        if (e < E) mi_decode(e, kk[j][0], kk[j][1], kk[j][2]);
        else kk[j][0] = kk[j][1] = kk[j][2] = 0;
    }
    double acc[EPT][NC];
#pragma unroll
    for (int j = 0; j < EPT; ++j)
#pragma unroll
        for (int c = 0; c < NC; ++c) acc[j][c] = 0.0;
    const int P1 = p + 1;
    // one 1-D pass along axis `ax`: out[k] = sum_{j_ax <= k_ax} A[ax][k_ax][j_ax] in[k with j_ax]
    auto pass = [&](int ax, const double* in, double* out, bool accumulate) {
#pragma unroll
        for (int jj = 0; jj < EPT; ++jj) {
            const int e = threadIdx.x + jj * T;
            if (e >= E) continue;
            int q[3] = {kk[jj][0], kk[jj][1], kk[jj][2]};
            const int ka = q[ax];
            double t[NC];
#pragma unroll
            for (int c = 0; c < NC; ++c) t[c] = 0.0;
            for (int j = 0; j <= ka; ++j) {
                q[ax] = j;
                const double cf = A[(ax * P1 + ka) * P1 + j];
                const double* mj = in + (size_t)mi_flat(q[0], q[1], q[2]) * 12 + C0;
#pragma unroll
                for (int c = 0; c < NC; ++c) t[c] = fma(cf, mj[c], t[c]);
            }
            if (accumulate) {
#pragma unroll
                for (int c = 0; c < NC; ++c) acc[jj][c] += t[c];
            } else {
#pragma unroll
                for (int c = 0; c < NC; ++c) out[(size_t)e * 12 + C0 + c] = t[c];
            }
        }
    };
    for (int ch = 0; ch < nchild[v]; ++ch) {
        const int u = children[8 * v + ch];
        const double4 gc = geom[u];
        __syncthreads();  // the previous child's passes are done with Ma, A
        for (int x = threadIdx.x; x < E * 12; x += T) Ma[x] = M[(size_t)u * E * 12 + x];
        for (int x = threadIdx.x; x < 3 * P1 * P1; x += T) {
            const int a = x / (P1 * P1), k = (x / P1) % P1, j = x % P1;
            const double d = a == 0 ? gc.x - gp.x : a == 1 ? gc.y - gp.y : gc.z - gp.z;
            double c = 0.0;
            if (j <= k) {
                c = 1.0;
                for (int t = 0; t < k - j; ++t) c *= d;
                // binomial C(k, j), exact in double for k <= 16
                double bn = 1.0;
                for (int t = 1; t <= j; ++t) bn = bn * (k - j + t) / t;
                c *= bn;
            }
            A[x] = c;
        }
        __syncthreads();
        pass(2, Ma, Mb, false);
        __syncthreads();
        pass(1, Mb, Ma, false);
        __syncthreads();
        pass(0, Ma, nullptr, true);
    }
#pragma unroll
    for (int jj = 0; jj < EPT; ++jj) {
        const int e = threadIdx.x + jj * T;
        if (e < E)
#pragma unroll
            for (int c = 0; c < NC; ++c) M[((size_t)v * E + e) * 12 + C0 + c] = acc[jj][c];
    }
}

// Sum the chunk partials of multi-chunk clusters in chunk order.
__global__ void k_reduce_parts(int ncl_items, const int32_t* __restrict__ item_off,
                               const int32_t* __restrict__ item_cl, const int32_t* __restrict__ part_slot,
                               int E, const double* __restrict__ part, double* __restrict__ M) {
    const int ci = blockIdx.y;
    const int slot = part_slot[ci];
    if (slot < 0) return;
    const int nch = item_off[ci + 1] - item_off[ci];
    const int v = item_cl[ci];
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < E * 12; x += gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int c = 0; c < nch; ++c) s += part[((size_t)slot + c) * E * 12 + x];
        M[(size_t)v * E * 12 + x] = s;
    }
}

__device__ __forceinline__ double fact_ratio(int q, int k) {  // q!/k! for |q-k| small
    double r = 1.0;
    for (int t = k + 1; t <= q; ++t) r *= t;
    for (int t = q + 1; t <= k; ++t) r /= t;
    return r;
}

// One CTA per moment block: gather the 4 weight columns for every |q| <= P, fold
// k3 >= 2 onto the harmonic basis, write W[blk][h][4].
template <bool STO, bool STR>
__global__ void __launch_bounds__(kThreads)
    k_fold(int p, int P, int Estride, const double* __restrict__ M, double* __restrict__ W,
           const int32_t* __restrict__ rows) {
    extern __shared__ double s_w[];  // [E(P)][4], then the cluster's moments [E(p)][12]
    const int EP = mi_count(P);
    const size_t blk = rows ? (size_t)rows[blockIdx.x] : (size_t)blockIdx.x;
    // moments of order p are the graded prefix of any higher-order block (multi_index.hpp:110-114);
    // staged once with coalesced loads: the fold reads each ~12 times at scattered indices
    double* sM = s_w + 4 * EP;
    {
        const double* g = M + blk * Estride * 12;
        const int cnt = mi_count(p) * 12;
        for (int i = threadIdx.x; i < cnt; i += blockDim.x) sM[i] = g[i];
        __syncthreads();
    }
    const double* Mb = sM;
    const double third = 1.0 / 3.0;

    for (int q = threadIdx.x; q < EP; q += blockDim.x) {
        int qk[3];
        mi_decode(q, qk[0], qk[1], qk[2]);
        const int nq = qk[0] + qk[1] + qk[2];
        double w4[4] = {0.0, 0.0, 0.0, 0.0};
        if (STO) {
            for (int i = 0; i < 3; ++i) {
                if (nq <= p) {
                    w4[i] += (1 - qk[i]) * Mb[(size_t)q * 12 + i];
                    for (int j = 0; j < 3; ++j) {
                        if (j == i || qk[j] < 1) continue;
                        int k[3] = {qk[0], qk[1], qk[2]};
                        k[j] -= 1;
                        k[i] += 1;
                        w4[i] -= qk[j] * Mb[(size_t)mi_flat(k[0], k[1], k[2]) * 12 + j];
                    }
                }
            }
            if (nq >= 1 && nq - 1 <= p)
                for (int j = 0; j < 3; ++j) {
                    if (qk[j] < 1) continue;
                    int k[3] = {qk[0], qk[1], qk[2]};
                    k[j] -= 1;
                    w4[3] += qk[j] * Mb[(size_t)mi_flat(k[0], k[1], k[2]) * 12 + j];
                }
        }
        if (STR) {
            for (int i = 0; i < 3; ++i) {
                if (nq >= 1 && nq - 1 <= p) {
                    for (int j = 0; j < 3; ++j)
                        for (int l = 0; l < 3; ++l) {
                            int k[3] = {qk[0], qk[1], qk[2]};
                            k[i] += 1;
                            k[j] -= 1;
                            k[l] -= 1;
                            if (k[0] < 0 || k[1] < 0 || k[2] < 0 || k[i] < 1) continue;
                            const double ratio = fact_ratio(qk[0], k[0]) * fact_ratio(qk[1], k[1]) *
                                                 fact_ratio(qk[2], k[2]);
                            w4[i] -= k[i] * ratio * third *
                                     Mb[(size_t)mi_flat(k[0], k[1], k[2]) * 12 + 3 + 3 * j + l];
                        }
                    if (qk[i] >= 1) {
                        int k[3] = {qk[0], qk[1], qk[2]};
                        k[i] -= 1;
                        const double* m = Mb + (size_t)mi_flat(k[0], k[1], k[2]) * 12 + 3;
                        w4[i] += qk[i] * third * ((m[0] + m[4]) + m[8]);
                    }
                }
            }
            if (nq >= 2 && nq - 2 <= p)
                for (int j = 0; j < 3; ++j)
                    for (int l = 0; l < 3; ++l) {
                        int k[3] = {qk[0], qk[1], qk[2]};
                        k[j] -= 1;
                        k[l] -= 1;
                        if (k[0] < 0 || k[1] < 0 || k[2] < 0) continue;
                        const double C = (double)(k[j] + 1) * (double)(k[l] + 1 + (j == l));
                        w4[3] += C * third * Mb[(size_t)mi_flat(k[0], k[1], k[2]) * 12 + 3 + 3 * j + l];
                    }
        }
        for (int c = 0; c < 4; ++c) s_w[4 * q + c] = w4[c];
    }
    // harmonic fold, highest k3 first: W[t] -= (t1-1)t1/((t3+2)(t3+1)) W[t-2e1+2e3]
    //                                        + (t2-1)t2/((t3+2)(t3+1)) W[t-2e2+2e3]
    for (int c3 = P; c3 >= 2; --c3) {
        __syncthreads();
        const int t3 = c3 - 2;
        const int rem = P - t3;  // t1 + t2 <= rem
        const int cnt = (rem + 1) * (rem + 2) / 2;
        for (int x = threadIdx.x; x < cnt; x += blockDim.x) {
            // enumerate (t1, t2) with t1 + t2 <= rem
            int t1 = 0, r = x;
            while (r >= rem - t1 + 1) {
                r -= rem - t1 + 1;
                ++t1;
            }
            const int t2 = r;
            const int tf = mi_flat(t1, t2, t3);
            const double den = (double)((t3 + 2) * (t3 + 1));
            double acc[4] = {s_w[4 * tf], s_w[4 * tf + 1], s_w[4 * tf + 2], s_w[4 * tf + 3]};
            if (t1 >= 2) {  // source q = t - 2e1 + 2e3, |q| = |t|
                const int qf = mi_flat(t1 - 2, t2, t3 + 2);
                const double cf = (double)((t1 - 1) * t1) / den;
                for (int c = 0; c < 4; ++c) acc[c] -= cf * s_w[4 * qf + c];
            }
            if (t2 >= 2) {  // source q = t - 2e2 + 2e3
                const int qf = mi_flat(t1, t2 - 2, t3 + 2);
                const double cf = (double)((t2 - 1) * t2) / den;
                for (int c = 0; c < 4; ++c) acc[c] -= cf * s_w[4 * qf + c];
            }
            for (int c = 0; c < 4; ++c) s_w[4 * tf + c] = acc[c];
        }
    }
    __syncthreads();
    // Change of basis per grade s, k3 <= 1 Taylor coefficients -> scaled real solid
    // harmonics (sph_basis.cuh, exact rationals from scripts/gen_sph_basis.py):
    // W_hat[m] = sum_j B_s[j][m] W[j], so far_eval sums W_hat against harmonics that cost
    // two DP ops each instead of the 4-5 of the Coulomb recurrence.
    const int H = harm_count(P);
    double* Wb = W + blk * H * 4;
    for (int h = threadIdx.x; h < H; h += blockDim.x) {
        int s = 0;
        while ((s + 1) * (s + 1) <= h) ++s;
        const int m = h - s * s, n = 2 * s + 1;
        const double* B = kSphB + sph_off(s);
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        for (int j = 0; j < n; ++j) {
            int k1, k2, k3;
            if (j <= s) { k1 = s - j; k2 = j; k3 = 0; }
            else { k2 = j - s - 1; k1 = s - 1 - k2; k3 = 1; }
            const int f = mi_flat(k1, k2, k3);
            const double b = B[j * n + m];
            for (int c = 0; c < 4; ++c) acc[c] = fma(b, s_w[4 * f + c], acc[c]);
        }
        for (int c = 0; c < 4; ++c) Wb[4 * h + c] = acc[c];
    }
}

__global__ void k_export(int nblk, int E, int sto, int str, const double* __restrict__ M,
                         double* __restrict__ stok, double* __restrict__ strm, double* __restrict__ trace,
                         double* __restrict__ sym) {
    const size_t x = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (x >= (size_t)nblk * E) return;
    const double* m = M + x * 12;
    if (sto)
        for (int j = 0; j < 3; ++j) stok[3 * x + j] = m[j];
    if (str) {
        const double* t = m + 3;
        for (int q = 0; q < 9; ++q) strm[9 * x + q] = t[q];
        trace[x] = t[0] + t[4] + t[8];
        double* s6 = sym + 6 * x;  // sym_index (multi_index.hpp:163-166)
        s6[0] = 2.0 * t[0];
        s6[3] = 2.0 * t[4];
        s6[5] = 2.0 * t[8];
        s6[1] = t[1] + t[3];
        s6[2] = t[2] + t[6];
        s6[4] = t[5] + t[7];
    }
}

__global__ void k_import(int nblk, int E, int sto, int str, const double* __restrict__ stok,
                         const double* __restrict__ strm, double* __restrict__ M) {
    const size_t x = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (x >= (size_t)nblk * E) return;
    double* m = M + x * 12;
    for (int j = 0; j < 3; ++j) m[j] = sto ? stok[3 * x + j] : 0.0;
    for (int q = 0; q < 9; ++q) m[3 + q] = str ? strm[9 * x + q] : 0.0;
}

template <int EPT>
void launch_moments_ept(bool sto, bool str, dim3 g, int threads, cudaStream_t s, int ncl_items, const int32_t* off,
                        const int32_t* cl, int nmulti, const int4* info, const double4* geom,
                        const double* src, int p, int E, const int32_t* slot, double* M, double* part) {
    if (sto && str)
        k_moments<EPT, true, true><<<g, threads, 0, s>>>(ncl_items, off, cl, nmulti, info, geom, src, p, E,
                                                          slot, M, part);
    else if (sto)
        k_moments<EPT, true, false><<<g, threads, 0, s>>>(ncl_items, off, cl, nmulti, info, geom, src, p, E,
                                                           slot, M, part);
    else
        k_moments<EPT, false, true><<<g, threads, 0, s>>>(ncl_items, off, cl, nmulti, info, geom, src, p, E,
                                                           slot, M, part);
    ST_LAUNCH("k_moments");
    count_launch();
}

}  // namespace

MomentsPlan plan_moments(const DevTree& tree, cudaStream_t s) {
    MomentsPlan pl;
    const int ncl = tree.ncl;
    // leaves: direct sums over their particles; internal clusters: M2M by level
    int4* hinfo = static_cast<int4*>(pinned_stage(sizeof(int4) * ncl));  // pinned: no staging stall
    int32_t* hlvl = static_cast<int32_t*>(pinned_stage(sizeof(int32_t) * ncl));
    ST_CUDA(cudaMemcpyAsync(hinfo, tree.info.get(), sizeof(int4) * ncl, cudaMemcpyDeviceToHost, s));
    ST_CUDA(cudaMemcpyAsync(hlvl, tree.bylevel.get(), sizeof(int32_t) * ncl, cudaMemcpyDeviceToHost, s));
    ST_CUDA(cudaStreamSynchronize(s));
    const std::vector<int4> info(hinfo, hinfo + ncl);
    const std::vector<int32_t> bylevel(hlvl, hlvl + ncl);
    pl.depth.assign(ncl, 0);
    for (size_t d = 0; d + 1 < tree.level_start.size(); ++d)
        for (int b = tree.level_start[d]; b < tree.level_start[d + 1]; ++b) pl.depth[bylevel[b]] = (int)d;
    for (int v = 0; v < ncl; ++v) {
        if (!info[v].w) continue;  // internal cluster
        const int cnt = info[v].y - info[v].x;
        const int nch = std::max(1, (cnt + kChunk - 1) / kChunk);
        pl.cl.push_back(v);
        pl.off.push_back(pl.items);
        pl.slot.push_back(nch > 1 ? pl.parts : -1);
        if (nch > 1) pl.parts += nch;
        pl.items += nch;
    }
    pl.off.push_back(pl.items);
    for (size_t d = 0; d + 1 < tree.level_start.size(); ++d) {
        std::vector<int32_t> ids;
        for (int b = tree.level_start[d]; b < tree.level_start[d + 1]; ++b)
            if (!info[bylevel[b]].w) ids.push_back(bylevel[b]);
        pl.lv.push_back(ids);
    }
    pl.info = std::move(info);
    return pl;
}

MomentsSplit split_moments(const MomentsPlan& full, int ncl, int nshards) {
    MomentsSplit sp;
    const std::vector<int4>& info = full.info;
    const int maxd = (int)full.lv.size();  // internal levels; leaves may sit one deeper
    int L = 0;
    for (;; ++L) {
        size_t units = 0;
        bool deeper = false;
        for (int v = 0; v < ncl; ++v) {
            const int d = full.depth[v];
            if (d == L || (d < L && info[v].w)) ++units;
            if (d > L) deeper = true;
        }
        if (units >= (size_t)4 * nshards || !deeper || L > maxd) break;
    }
    sp.depth = L;
    std::vector<double> wt;
    for (int v = 0; v < ncl; ++v) {
        const int d = full.depth[v];
        if (d == L || (d < L && info[v].w)) {
            sp.units.push_back(v);  // ascending v: pre-order
            wt.push_back((double)(info[v].y - info[v].x));
        }
    }
    sp.unit_cuts.assign(nshards + 1, 0);
    shard_cuts_host(sp.units.size(), wt.data(), nshards, sp.unit_cuts.data());
    sp.w_cuts.assign(nshards + 1, (size_t)ncl);
    sp.w_cuts[0] = 0;
    for (int r = 1; r < nshards; ++r)
        sp.w_cuts[r] = sp.unit_cuts[r] < sp.units.size() ? (size_t)sp.units[sp.unit_cuts[r]] : (size_t)ncl;
    for (int r = nshards - 1; r >= 1; --r) sp.w_cuts[r] = std::min(sp.w_cuts[r], sp.w_cuts[r + 1]);
    sp.top.assign(std::min<size_t>(L, full.lv.size()), {});
    for (size_t d = 0; d < sp.top.size(); ++d) {
        sp.top[d] = full.lv[d];  // internal clusters above L
        sp.top_ids.insert(sp.top_ids.end(), sp.top[d].begin(), sp.top[d].end());
    }
    return sp;
}

MomentsPlan shard_moments_plan(const MomentsPlan& full, const MomentsSplit& sp, int shard) {
    // clusters inside this rank's units: [units[u0], next(units[u1 - 1]))
    const size_t u0 = sp.unit_cuts[shard], u1 = sp.unit_cuts[shard + 1];
    MomentsPlan pl;
    pl.info = full.info;
    pl.depth = full.depth;
    pl.lv.assign(full.lv.size(), {});
    if (u0 >= u1) {
        pl.off.push_back(0);
        return pl;
    }
    const int lo = sp.units[u0], hi = full.info[sp.units[u1 - 1]].z;
    for (size_t i = 0; i < full.cl.size(); ++i) {
        const int v = full.cl[i];
        if (v < lo || v >= hi) continue;
        const int nch = full.off[i + 1] - full.off[i];
        pl.cl.push_back(v);
        pl.off.push_back(pl.items);
        pl.slot.push_back(nch > 1 ? pl.parts : -1);
        if (nch > 1) pl.parts += nch;
        pl.items += nch;
    }
    pl.off.push_back(pl.items);
    for (size_t d = sp.depth; d < full.lv.size(); ++d)
        for (int v : full.lv[d])
            if (v >= lo && v < hi) pl.lv[d].push_back(v);
    return pl;
}

MomentsPlan top_moments_plan(const MomentsSplit& sp) {
    MomentsPlan pl;
    pl.off.push_back(0);
    pl.lv = sp.top;
    return pl;
}

void compute_moments_device(const DevTree& tree, const double* src, int p, bool sto, bool str,
                            cudaStream_t s, DevArray<double>& M, const MomentsPlan* plan, bool keep) {
    static const bool dbg = getenv("ST_DEBUG_MOMENTS") != nullptr;
    auto stamp = [&](const char* what) {
        if (!dbg) return;
        ST_CUDA(cudaStreamSynchronize(s));
        static auto t0 = std::chrono::steady_clock::now();
        const auto t = std::chrono::steady_clock::now();
        fprintf(stderr, "[moments] %-12s %.3f ms\n", what, std::chrono::duration<double, std::milli>(t - t0).count());
        t0 = t;
    };
    stamp("enter");
    if (p < 0 || p > kPmax) fail(ST_INVALID_ARGUMENT, "compute_moments: order outside table range");
    const int E = mi_count(p);
    const int ncl = tree.ncl;
    MomentsPlan own;
    if (!plan) {
        own = plan_moments(tree, s);
        plan = &own;
    }
    const std::vector<int32_t>&off = plan->off, &cl = plan->cl, &slot = plan->slot;
    const int items = plan->items, parts = plan->parts;
    const std::vector<std::vector<int32_t>>& lv = plan->lv;
    const int nleaf = (int)cl.size();
    DevArray<int32_t> d_off(nleaf + 1, s), d_cl(nleaf, s), d_slot(nleaf, s), d_lvl(ncl, s);
    // pinned staging: a pageable upload would first wait for this stream to drain
    ST_CUDA(cudaMemcpyAsync(d_off.get(), pinned_copy(off.data(), nleaf + 1), sizeof(int32_t) * (nleaf + 1),
                            cudaMemcpyHostToDevice, s));
    ST_CUDA(cudaMemcpyAsync(d_cl.get(), pinned_copy(cl.data(), nleaf), sizeof(int32_t) * nleaf,
                            cudaMemcpyHostToDevice, s));
    ST_CUDA(cudaMemcpyAsync(d_slot.get(), pinned_copy(slot.data(), nleaf), sizeof(int32_t) * nleaf,
                            cudaMemcpyHostToDevice, s));
    {
        std::vector<int32_t> flat;
        for (const auto& ids : lv) flat.insert(flat.end(), ids.begin(), ids.end());
        if (!flat.empty())
            ST_CUDA(cudaMemcpyAsync(d_lvl.get(), pinned_copy(flat.data(), flat.size()), sizeof(int32_t) * flat.size(),
                                    cudaMemcpyHostToDevice, s));
    }
    stamp("host lists");
    if (!keep) {
        M.alloc((size_t)ncl * E * 12, s);
        M.zero();
    }
    DevArray<double> part((size_t)std::max(parts, 1) * E * 12, s);
    stamp("alloc");
    // entries per thread (block = E/EPT rounded up to a warp): 2 (106 registers) measured
    // fastest (4: 163 registers, 20% slower at cfg1); 4 once E/2 exceeds the 256-thread
    // launch bound (p >= 13).  ST_MOMENTS_EPT overrides (A/B checks).
    static const int ept_env = getenv("ST_MOMENTS_EPT") ? atoi(getenv("ST_MOMENTS_EPT")) : 0;
    int ept = ept_env == 1 || ept_env == 2 || ept_env == 4 ? ept_env : E >= 32 ? 2 : 1;
    while ((E + ept - 1) / ept > kThreads) ept *= 2;
    const int threads = std::max(32, ((E + ept - 1) / ept + 31) / 32 * 32);
    if (items) {
        dim3 g(items);
        switch (ept) {
            case 1: launch_moments_ept<1>(sto, str, g, threads, s, nleaf, d_off.get(), d_cl.get(), 0, tree.info.get(),
                                          tree.geom.get(), src, p, E, d_slot.get(), M.get(), part.get()); break;
            case 2: launch_moments_ept<2>(sto, str, g, threads, s, nleaf, d_off.get(), d_cl.get(), 0, tree.info.get(),
                                          tree.geom.get(), src, p, E, d_slot.get(), M.get(), part.get()); break;
            default: launch_moments_ept<4>(sto, str, g, threads, s, nleaf, d_off.get(), d_cl.get(), 0, tree.info.get(),
                                           tree.geom.get(), src, p, E, d_slot.get(), M.get(), part.get()); break;
        }
    }
    if (parts) {
        k_reduce_parts<<<dim3(std::max(1, (E * 12 + 255) / 256), nleaf), 256, 0, s>>>(
            nleaf, d_off.get(), d_cl.get(), d_slot.get(), E, part.get(), M.get());
        ST_LAUNCH("k_reduce_parts");
        count_launch();
    }
    stamp("leaves");
    // upward pass: deepest internal level first
    const size_t smem = sizeof(double) * ((size_t)E * 24 + 3 * (size_t)(p + 1) * (p + 1));
    size_t base = 0;
    std::vector<size_t> lvl_off;
    for (const auto& ids : lv) {
        lvl_off.push_back(base);
        base += ids.size();
    }
    for (int d = (int)lv.size() - 1; d >= 0; --d) {
        const int cnt = (int)lv[d].size();
        if (!cnt) continue;
        // one CTA per parent and few parents per level: as many threads as the launch
        // bound allows (the fewest entries per thread), unlike the leaf kernel
        const int mept = (E + kThreads - 1) / kThreads <= 1 ? 1 : (E + kThreads - 1) / kThreads <= 2 ? 2 : 4;
        const int mthreads = std::max(32, ((E + mept - 1) / mept + 31) / 32 * 32);
        auto go = [&](auto kern) {
            ST_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            kern<<<cnt, mthreads, smem, s>>>(d_lvl.get() + lvl_off[d], tree.children.get(), tree.nchild.get(),
                                             tree.geom.get(), p, E, M.get());
            ST_LAUNCH("k_m2m");
            count_launch();
        };
        auto pick = [&](auto ept_tag) {
            constexpr int EP = decltype(ept_tag)::value;
            if (sto && str) go(k_m2m<EP, true, true>);
            else if (sto) go(k_m2m<EP, true, false>);
            else go(k_m2m<EP, false, true>);
        };
        if (mept == 1) pick(std::integral_constant<int, 1>{});
        else if (mept == 2) pick(std::integral_constant<int, 2>{});
        else pick(std::integral_constant<int, 4>{});
    }
    stamp("m2m");
}

void fold_weights_device(const double* M, int nblk, int p, bool sto, bool str, cudaStream_t s,
                         DevArray<double>& W, int pstride) {
    const int P = p + (str ? 2 : 1);
    const size_t smem = sizeof(double) * (4 * mi_count(P) + 12 * mi_count(p));
    W.alloc((size_t)nblk * harm_count(P) * 4, s);
    if (nblk == 0) return;
    auto go = [&](auto kern) {
        ST_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern<<<nblk, kThreads, smem, s>>>(p, P, mi_count(pstride < 0 ? p : pstride), M, W.get(), nullptr);
        ST_LAUNCH("k_fold");
        count_launch();
    };
    if (sto && str) go(k_fold<true, true>);
    else if (sto) go(k_fold<true, false>);
    else go(k_fold<false, true>);
}

void fold_weights_rows_device(const double* M, const int32_t* rows, int n, int p, bool sto, bool str,
                              cudaStream_t s, double* W) {
    if (n <= 0) return;
    const int P = p + (str ? 2 : 1);
    const size_t smem = sizeof(double) * (4 * mi_count(P) + 12 * mi_count(p));
    auto go = [&](auto kern) {
        ST_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern<<<n, kThreads, smem, s>>>(p, P, mi_count(p), M, W, rows);
        ST_LAUNCH("k_fold");
        count_launch();
    };
    if (sto && str) go(k_fold<true, true>);
    else if (sto) go(k_fold<true, false>);
    else go(k_fold<false, true>);
}

__global__ void k_rows(const double* __restrict__ src, const int32_t* __restrict__ rows, int n, size_t len,
                       double* __restrict__ dst, int scatter) {
    const size_t i = blockIdx.y;
    for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < len; k += (size_t)gridDim.x * blockDim.x) {
        if (scatter) dst[(size_t)rows[i] * len + k] = src[i * len + k];
        else dst[i * len + k] = src[(size_t)rows[i] * len + k];
    }
}

void gather_rows_device(const double* src, const int32_t* rows, int n, size_t len, double* dst, bool scatter,
                        cudaStream_t s) {
    if (n <= 0 || !len) return;
    k_rows<<<dim3((unsigned)std::min<size_t>((len + 255) / 256, 64), (unsigned)n), 256, 0, s>>>(src, rows, n, len, dst,
                                                                                             scatter ? 1 : 0);
    ST_LAUNCH("k_rows");
    count_launch();
}

void export_moments_device(const double* M, int nblk, int p, bool sto, bool str, double* stok,
                           double* strm, double* trace, double* sym, cudaStream_t s) {
    const size_t n = (size_t)nblk * mi_count(p);
    if (!n) return;
    k_export<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(nblk, mi_count(p), sto, str, M, stok, strm, trace, sym);
    ST_LAUNCH("k_export");
    count_launch();
}

void import_moments_device(int nblk, int p, bool sto, bool str, const double* stok, const double* strm,
                           double* M, cudaStream_t s) {
    const size_t n = (size_t)nblk * mi_count(p);
    if (!n) return;
    k_import<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(nblk, mi_count(p), sto, str, stok, strm, M);
    ST_LAUNCH("k_import");
    count_launch();
}

}  // namespace st
