/*
 * oracle/stokes_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference treecode path (arXiv 1811.12498,
 * /root/reference/proj/include/stokestree/ headers) used as the CPU checker for
 * the CUDA product path.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  It is never linked into
 * or called by the product library.
 *
 * Every function cites the reference file:line it restates.  Compiled with
 * -ffp-contract=off so that no FMA contraction changes geometry bits (the
 * reference is built by GCC without -march, i.e. without FMA).
 *
 * Parity pin: this restatement is checked bit-for-bit (tree, permutation,
 * per-target interaction counts) and to <=1e-13 (velocities, moments) against
 * the reference headers compiled in place (oracle/_ref, see oracle/Makefile)
 * and against the reference's own hand values (tests/test_oracle.py).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_INVALID 1
#define OR_DOMAIN 2
#define OR_NOSKIP ((size_t)-1)

/* ------------------------------------------------------------------ */
/* vector helpers (vec3.hpp:48-52): norm2 = (a0*a0 + a1*a1) + a2*a2      */
/* ------------------------------------------------------------------ */
static double nrm2(const double a[3]) { return a[0] * a[0] + a[1] * a[1] + a[2] * a[2]; }

/* ------------------------------------------------------------------ */
/* multi-index table (multi_index.hpp:26-180)                          */
/* graded-lex: per grade s, k1 = 0..s, k2 = 0..s-k1, k3 = s-k1-k2 (:36-44) */
/* ------------------------------------------------------------------ */
typedef struct {
    int pmax;
    int n;          /* entries with |k| <= pmax */
    int (*k)[3];
    int *dense;     /* (pmax+1)^3 -> flat or -1 */
    int *goff;      /* grade offsets, pmax+2 */
} mi_table;

static int mi_count(int p) { return (p + 1) * (p + 2) * (p + 3) / 6; }

static int mi_flat(const mi_table *t, int a, int b, int c) {
    if (a < 0 || b < 0 || c < 0 || a + b + c > t->pmax) return -1;
    int side = t->pmax + 1;
    return t->dense[(a * side + b) * side + c];
}
/* out-of-table lookups map to the zero slot n (multi_index.hpp:47-52) */
static int mi_at(const mi_table *t, int a, int b, int c) {
    int f = mi_flat(t, a, b, c);
    return f < 0 ? t->n : f;
}

static void mi_init(mi_table *t, int pmax) {
    int side = pmax + 1;
    t->pmax = pmax;
    t->n = mi_count(pmax);
    t->k = malloc(sizeof(int[3]) * (size_t)t->n);
    t->dense = malloc(sizeof(int) * (size_t)side * side * side);
    t->goff = malloc(sizeof(int) * (size_t)(pmax + 2));
    for (int i = 0; i < side * side * side; ++i) t->dense[i] = -1;
    int e = 0;
    for (int s = 0; s <= pmax; ++s) {
        t->goff[s] = e;
        for (int k1 = 0; k1 <= s; ++k1)
            for (int k2 = 0; k2 + k1 <= s; ++k2) {
                int k3 = s - k1 - k2;
                t->k[e][0] = k1; t->k[e][1] = k2; t->k[e][2] = k3;
                t->dense[(k1 * side + k2) * side + k3] = e;
                ++e;
            }
    }
    t->goff[pmax + 1] = e;
}
static void mi_free(mi_table *t) { free(t->k); free(t->dense); free(t->goff); }

/* shifted lookup k + d (component deltas) with zero-slot mapping */
static int mi_shift(const mi_table *t, int e, int d0, int d1, int d2) {
    return mi_at(t, t->k[e][0] + d0, t->k[e][1] + d1, t->k[e][2] + d2);
}

/* ------------------------------------------------------------------ */
/* tree (cluster_tree.hpp:13-192)                                      */
/* ------------------------------------------------------------------ */
typedef struct {
    size_t begin, end;
    double center[3];
    double radius;
    double lo[3], hi[3];
    int32_t children[8];
    int n_children;
    int is_leaf;
} or_cluster;

typedef struct {
    size_t n;
    int n0, shrink;
    or_cluster *cl;
    size_t ncl, cap;
    uint32_t *to_original, *to_tree, *scratch;
    const double *pos_in;   /* original order, borrowed during build */
    double *pos, *f, *h, *nu; /* tree-ordered copies (NULL if absent) */
} or_tree;

/* tight_box (cluster_tree.hpp:58-69): std::min/max keep the first-seen value on ties */
static void tight_box(const double *pos, const uint32_t *idx, size_t b, size_t e, double lo[3],
                      double hi[3]) {
    for (int a = 0; a < 3; ++a) lo[a] = hi[a] = pos[3 * (size_t)idx[b] + a];
    for (size_t t = b + 1; t < e; ++t) {
        const double *p = pos + 3 * (size_t)idx[t];
        for (int a = 0; a < 3; ++a) {
            if (p[a] < lo[a]) lo[a] = p[a];
            if (hi[a] < p[a]) hi[a] = p[a];
        }
    }
}

static size_t push_cluster(or_tree *T) {
    if (T->ncl == T->cap) {
        T->cap = T->cap ? 2 * T->cap : 64;
        T->cl = realloc(T->cl, sizeof(or_cluster) * T->cap);
    }
    memset(&T->cl[T->ncl], 0, sizeof(or_cluster));
    T->cl[T->ncl].is_leaf = 1;
    return T->ncl++;
}

/* TreeBuilder::build (cluster_tree.hpp:81-143): pre-order ids, geometric bisection,
 * ties go up, stable counting-sort scatter, empty children pruned, depth cap 64. */
static int build_rec(or_tree *T, size_t b, size_t e, const double glo[3], const double ghi[3],
                     int depth) {
    const double *pos = T->pos_in;
    size_t id = push_cluster(T);
    {
        or_cluster *c = &T->cl[id];
        c->begin = b;
        c->end = e;
        if (T->shrink) {
            tight_box(pos, T->to_original, b, e, c->lo, c->hi);
        } else {
            for (int a = 0; a < 3; ++a) { c->lo[a] = glo[a]; c->hi[a] = ghi[a]; }
        }
        for (int a = 0; a < 3; ++a) c->center[a] = (c->lo[a] + c->hi[a]) * 0.5;
        double max2 = 0.0;
        for (size_t t = b; t < e; ++t) {
            const double *p = pos + 3 * (size_t)T->to_original[t];
            double d[3] = {p[0] - c->center[0], p[1] - c->center[1], p[2] - c->center[2]};
            double r2 = nrm2(d);
            if (max2 < r2) max2 = r2;
        }
        c->radius = sqrt(max2);
    }
    if (e - b <= (size_t)T->n0 || depth >= 64) return (int)id;

    double mid[3];
    for (int a = 0; a < 3; ++a) mid[a] = (glo[a] + ghi[a]) * 0.5;
    size_t counts[8] = {0}, offset[8], cursor[8];
    for (size_t t = b; t < e; ++t) {
        const double *p = pos + 3 * (size_t)T->to_original[t];
        int slot = (p[0] >= mid[0] ? 1 : 0) | (p[1] >= mid[1] ? 2 : 0) | (p[2] >= mid[2] ? 4 : 0);
        ++counts[slot];
    }
    size_t acc = b;
    for (int s = 0; s < 8; ++s) { offset[s] = acc; cursor[s] = acc; acc += counts[s]; }
    for (size_t t = b; t < e; ++t) {
        const double *p = pos + 3 * (size_t)T->to_original[t];
        int slot = (p[0] >= mid[0] ? 1 : 0) | (p[1] >= mid[1] ? 2 : 0) | (p[2] >= mid[2] ? 4 : 0);
        T->scratch[cursor[slot]++] = T->to_original[t];
    }
    memcpy(T->to_original + b, T->scratch + b, sizeof(uint32_t) * (e - b));

    int ids[8], nch = 0;
    for (int s = 0; s < 8; ++s) {
        if (!counts[s]) continue;
        double clo[3], chi[3];
        for (int a = 0; a < 3; ++a) {
            int up = (s >> a) & 1;
            clo[a] = up ? mid[a] : glo[a];
            chi[a] = up ? ghi[a] : mid[a];
        }
        ids[nch++] = build_rec(T, offset[s], offset[s] + counts[s], clo, chi, depth + 1);
    }
    or_cluster *c = &T->cl[id];
    c->is_leaf = 0;
    c->n_children = nch;
    for (int s = 0; s < nch; ++s) c->children[s] = ids[s];
    return (int)id;
}

static double *gather3(const double *src, const uint32_t *perm, size_t n) {
    if (!src) return NULL;
    double *out = malloc(sizeof(double) * 3 * n);
    for (size_t t = 0; t < n; ++t)
        for (int a = 0; a < 3; ++a) out[3 * t + a] = src[3 * (size_t)perm[t] + a];
    return out;
}

/* build_tree (cluster_tree.hpp:152-192): root cube = tight box centre +- side/2,
 * side = max extent * (1 + 1e-12). */
void *or_tree_build(size_t n, const double *pos, const double *f, const double *h,
                    const double *nu, int n0, int shrink, int *status) {
    if (n == 0 || n0 < 1) { *status = OR_INVALID; return NULL; }
    or_tree *T = calloc(1, sizeof(or_tree));
    T->n = n; T->n0 = n0; T->shrink = shrink; T->pos_in = pos;
    T->to_original = malloc(sizeof(uint32_t) * n);
    T->to_tree = malloc(sizeof(uint32_t) * n);
    T->scratch = malloc(sizeof(uint32_t) * n);
    for (size_t i = 0; i < n; ++i) T->to_original[i] = (uint32_t)i;
    double lo[3], hi[3];
    tight_box(pos, T->to_original, 0, n, lo, hi);
    double side = 0.0;
    for (int a = 0; a < 3; ++a) {
        double ext = hi[a] - lo[a];
        if (side < ext) side = ext;
    }
    side *= 1.0 + 1e-12;
    double rlo[3], rhi[3];
    for (int a = 0; a < 3; ++a) {
        double c = (lo[a] + hi[a]) * 0.5;
        double half = side * 0.5;
        rlo[a] = c - half;
        rhi[a] = c + half;
    }
    build_rec(T, 0, n, rlo, rhi, 0);
    for (size_t t = 0; t < n; ++t) T->to_tree[T->to_original[t]] = (uint32_t)t;
    T->pos = gather3(pos, T->to_original, n);
    T->f = gather3(f, T->to_original, n);
    T->h = gather3(h, T->to_original, n);
    T->nu = gather3(nu, T->to_original, n);
    T->pos_in = NULL;
    free(T->scratch); T->scratch = NULL;
    *status = OR_OK;
    return T;
}

size_t or_tree_ncl(const void *tp) { return ((const or_tree *)tp)->ncl; }

/* export: be[2*ncl] = begin,end; geom[10*ncl] = center3, radius, lo3, hi3;
 * kids[8*ncl]; meta[2*ncl] = n_children, is_leaf; perm[n] = to_original */
void or_tree_export(const void *tp, int64_t *be, double *geom, int32_t *kids, int32_t *meta,
                    uint32_t *perm) {
    const or_tree *T = tp;
    for (size_t i = 0; i < T->ncl; ++i) {
        const or_cluster *c = &T->cl[i];
        if (be) { be[2 * i] = (int64_t)c->begin; be[2 * i + 1] = (int64_t)c->end; }
        if (geom) {
            double *g = geom + 10 * i;
            for (int a = 0; a < 3; ++a) { g[a] = c->center[a]; g[4 + a] = c->lo[a]; g[7 + a] = c->hi[a]; }
            g[3] = c->radius;
        }
        if (kids) for (int s = 0; s < 8; ++s) kids[8 * i + s] = s < c->n_children ? c->children[s] : -1;
        if (meta) { meta[2 * i] = c->n_children; meta[2 * i + 1] = c->is_leaf; }
    }
    if (perm) memcpy(perm, T->to_original, sizeof(uint32_t) * T->n);
}

void or_tree_free(void *tp) {
    or_tree *T = tp;
    if (!T) return;
    free(T->cl); free(T->to_original); free(T->to_tree);
    free(T->pos); free(T->f); free(T->h); free(T->nu);
    free(T);
}

/* ------------------------------------------------------------------ */
/* moments (moments.hpp:34-80, 140-175)                                */
/* per cluster: stok[3E] (e*3+j), str[9E] (e*9+3j+l), trace[E], sym[6E] */
/* ------------------------------------------------------------------ */
static const int SYM[3][3] = {{0, 1, 2}, {1, 3, 4}, {2, 4, 5}};

static void cluster_moments(const or_tree *T, const or_cluster *c, const mi_table *t, int cnt,
                            int sto, int str, double *mono, double *stok, double *strm,
                            double *trace, double *sym) {
    /* monomial chain: entry e = entry parent(e) * d[axis(e)], axis = first nonzero (:97-102) */
    for (size_t n = c->begin; n < c->end; ++n) {
        const double *y = T->pos + 3 * n;
        double d[3] = {y[0] - c->center[0], y[1] - c->center[1], y[2] - c->center[2]};
        mono[0] = 1.0;
        for (int e = 1; e < cnt; ++e) {
            int ax = 0;
            while (t->k[e][ax] == 0) ++ax;
            int par = mi_shift(t, e, -(ax == 0), -(ax == 1), -(ax == 2));
            mono[e] = d[ax] * mono[par];
        }
        if (sto) {
            const double *f = T->f + 3 * n;
            for (int e = 0; e < cnt; ++e) {
                double s = mono[e];
                stok[3 * e + 0] += s * f[0];
                stok[3 * e + 1] += s * f[1];
                stok[3 * e + 2] += s * f[2];
            }
        }
        if (str) {
            const double *h = T->h + 3 * n, *nu = T->nu + 3 * n;
            double outer[9];
            for (int j = 0; j < 3; ++j)
                for (int l = 0; l < 3; ++l) outer[3 * j + l] = h[j] * nu[l];
            for (int e = 0; e < cnt; ++e) {
                double s = mono[e];
                for (int q = 0; q < 9; ++q) strm[9 * e + q] += s * outer[q];
            }
        }
    }
    if (str) { /* derive_stresslet_contractions (:67-80) */
        for (int e = 0; e < cnt; ++e) {
            const double *m = strm + 9 * e;
            trace[e] = m[0] + m[4] + m[8];
            double *s = sym + 6 * e;
            s[SYM[0][0]] = 2.0 * m[0];
            s[SYM[1][1]] = 2.0 * m[4];
            s[SYM[2][2]] = 2.0 * m[8];
            s[SYM[0][1]] = m[1] + m[3];
            s[SYM[0][2]] = m[2] + m[6];
            s[SYM[1][2]] = m[5] + m[7];
        }
    }
}

/* compute_moments for every cluster; buffers sized ncl * {3,9,1,6} * E(p), zero-filled here. */
int or_moments(const void *tp, int p, int sto, int str, double *stok, double *strm,
               double *trace, double *sym) {
    const or_tree *T = tp;
    if (p < 0) return OR_INVALID;
    mi_table t;
    mi_init(&t, p);
    int cnt = t.n;
    double *mono = malloc(sizeof(double) * (size_t)cnt);
    size_t E = (size_t)cnt;
    if (sto) memset(stok, 0, sizeof(double) * 3 * E * T->ncl);
    if (str) {
        memset(strm, 0, sizeof(double) * 9 * E * T->ncl);
        memset(trace, 0, sizeof(double) * E * T->ncl);
        memset(sym, 0, sizeof(double) * 6 * E * T->ncl);
    }
    for (size_t c = 0; c < T->ncl; ++c)
        cluster_moments(T, &T->cl[c], &t, cnt, sto, str, mono, sto ? stok + 3 * E * c : NULL,
                        str ? strm + 9 * E * c : NULL, str ? trace + E * c : NULL,
                        str ? sym + 6 * E * c : NULL);
    free(mono);
    mi_free(&t);
    return OR_OK;
}

/* ------------------------------------------------------------------ */
/* Coulomb coefficients (coulomb.hpp:28-50), b sized n+1, zero slot n  */
/* ------------------------------------------------------------------ */
static int coulomb(const double dx[3], const mi_table *t, double *b) {
    double r2 = nrm2(dx);
    if (!(r2 > 0.0)) return OR_DOMAIN;
    b[t->n] = 0.0;
    b[0] = 1.0 / sqrt(r2);
    for (int s = 1; s <= t->pmax; ++s) {
        double c1 = 2.0 * s - 1.0, c2 = s - 1.0, inv = 1.0 / (s * r2);
        for (int e = t->goff[s]; e < t->goff[s + 1]; ++e) {
            double acc = c1 * (dx[0] * b[mi_shift(t, e, -1, 0, 0)] + dx[1] * b[mi_shift(t, e, 0, -1, 0)] +
                               dx[2] * b[mi_shift(t, e, 0, 0, -1)]);
            if (s >= 2)
                acc -= c2 * (b[mi_shift(t, e, -2, 0, 0)] + b[mi_shift(t, e, 0, -2, 0)] +
                             b[mi_shift(t, e, 0, 0, -2)]);
            b[e] = acc * inv;
        }
    }
    return OR_OK;
}

int or_coulomb(const double dx[3], int pmax, double *b_out) {
    if (pmax < 0) return OR_INVALID;
    mi_table t;
    mi_init(&t, pmax);
    int st = coulomb(dx, &t, b_out);
    mi_free(&t);
    return st;
}

/* Explicit Taylor coefficients from b of depth pmax_b (taylor_coeffs.hpp:13-46), for every
   multi-index of grade <= order: a_sto[e*9 + 3i+j] (needs order+1 <= pmax_b),
   a_str[e*27 + 9i+3j+l] (needs order+2 <= pmax_b).  b is sized E(pmax_b)+1 (zero slot). */
int or_taylor(const double dx[3], const double *b, int pmax_b, int order, double *a_sto, double *a_str) {
    if (order < 0 || pmax_b < 0) return OR_INVALID;
    if ((a_sto && order + 1 > pmax_b) || (a_str && order + 2 > pmax_b)) return OR_INVALID;
    mi_table t;
    mi_init(&t, pmax_b);
    const int E = mi_count(order);
    for (int e = 0; e < E; ++e) {
        const int *k = t.k[e];
        for (int i = 0; i < 3; ++i) {
            int ui[3] = {0, 0, 0};
            ui[i] = 1;
            for (int j = 0; j < 3; ++j) {
                const double dij = i == j ? 1.0 : 0.0;
                if (a_sto) {
                    const double kip1 = k[i] + 1;
                    int ud[3] = {ui[0], ui[1], ui[2]};
                    ud[j] -= 1;
                    a_sto[e * 9 + 3 * i + j] = dij * b[e] + dx[j] * kip1 * b[mi_shift(&t, e, ui[0], ui[1], ui[2])] -
                                               (kip1 - dij) * b[mi_shift(&t, e, ud[0], ud[1], ud[2])];
                }
                if (!a_str) continue;
                for (int l = 0; l < 3; ++l) {
                    const double dil = i == l ? 1.0 : 0.0, djl = j == l ? 1.0 : 0.0;
                    int uu[3] = {ui[0], ui[1], ui[2]};
                    uu[j] += 1;
                    int uud[3] = {uu[0], uu[1], uu[2]};
                    uud[l] -= 1;
                    int ul[3] = {0, 0, 0};
                    ul[l] = 1;
                    const double t1 = dx[l] * (k[i] + 1) * (k[j] + 1 + dij) * b[mi_shift(&t, e, uu[0], uu[1], uu[2])];
                    const double t2 =
                        (k[i] + 1 - dil) * (k[j] + 1 + dij - djl) * b[mi_shift(&t, e, uud[0], uud[1], uud[2])];
                    const double t3 = dij * (k[l] + 1) * b[mi_shift(&t, e, ul[0], ul[1], ul[2])];
                    a_str[e * 27 + 9 * i + 3 * j + l] = (t1 - t2 + t3) / 3.0;
                }
            }
        }
    }
    mi_free(&t);
    return OR_OK;
}

/* stokeslet_farfield, Eq. 25 (farfield.hpp:30-53) */
static void sto_far(const double dx[3], const double *m3, int cnt, const mi_table *t,
                    const double *b, double u[3]) {
    double v[3] = {0, 0, 0};
    for (int e = 0; e < cnt; ++e) {
        const double *m = m3 + 3 * e;
        double be = b[e];
        double sigma = dx[0] * m[0] + dx[1] * m[1] + dx[2] * m[2];
        for (int i = 0; i < 3; ++i) {
            double kip1 = t->k[e][i] + 1;
            int up = mi_shift(t, e, i == 0, i == 1, i == 2);
            double s = b[up] * sigma;
            double sub = 0.0;
            for (int j = 0; j < 3; ++j) {
                int ud = mi_shift(t, e, (i == 0) - (j == 0), (i == 1) - (j == 1), (i == 2) - (j == 2));
                double term = b[ud] * m[j];
                sub = j == 0 ? term : sub + term;
            }
            s -= sub;
            v[i] += 2.0 * be * m[i] + kip1 * s;
        }
    }
    u[0] = v[0]; u[1] = v[1]; u[2] = v[2];
}

/* stresslet_farfield, Eq. 30 (farfield.hpp:61-96) */
static void str_far(const double dx[3], const double *mt9, const double *tr, const double *sy,
                    int cnt, const mi_table *t, const double *b, double u[3]) {
    double v[3] = {0, 0, 0};
    for (int e = 0; e < cnt; ++e) {
        const double *mt = mt9 + 9 * e;
        double mk = tr[e];
        const double *ms = sy + 6 * e;
        const int *k = t->k[e];
        double tau[3];
        for (int j = 0; j < 3; ++j)
            tau[j] = dx[0] * mt[3 * j + 0] + dx[1] * mt[3 * j + 1] + dx[2] * mt[3 * j + 2];
        for (int i = 0; i < 3; ++i) {
            double kip1 = k[i] + 1;
            double t1 = 0.0, t2 = 0.0;
            for (int j = 0; j < 3; ++j) {
                double cj = k[j] + 1 + (i == j ? 1 : 0);
                int uu = mi_shift(t, e, (i == 0) + (j == 0), (i == 1) + (j == 1), (i == 2) + (j == 2));
                t1 += cj * b[uu] * tau[j];
                double s3 = 0.0;
                for (int l = 0; l < 3; ++l) {
                    int uud = mi_shift(t, e, (i == 0) + (j == 0) - (l == 0), (i == 1) + (j == 1) - (l == 1),
                                       (i == 2) + (j == 2) - (l == 2));
                    double term = b[uud] * mt[3 * j + l];
                    s3 = l == 0 ? term : s3 + term;
                }
                t2 += cj * s3;
            }
            double t3 = b[mi_shift(t, e, i == 0, i == 1, i == 2)] * mk;
            double t4 = (k[0] + 1) * b[mi_shift(t, e, 1, 0, 0)] * ms[SYM[i][0]] +
                        (k[1] + 1) * b[mi_shift(t, e, 0, 1, 0)] * ms[SYM[i][1]] +
                        (k[2] + 1) * b[mi_shift(t, e, 0, 0, 1)] * ms[SYM[i][2]];
            v[i] += kip1 * (t1 - t2 + t3) + t4;
        }
    }
    double third = 1.0 / 3.0;
    u[0] = v[0] * third; u[1] = v[1] * third; u[2] = v[2] * third;
}

/* One particle-cluster far-field pair at order p (coulomb + Eq. 25 + Eq. 30). */
int or_farfield_pair(const double dx[3], int p, int sto, int str, const double *stok,
                     const double *strm, const double *trace, const double *sym, double u[3]) {
    if (p < 0) return OR_INVALID;
    mi_table t;
    mi_init(&t, p + (str ? 2 : 1));
    double *b = malloc(sizeof(double) * (size_t)(t.n + 1));
    int st = coulomb(dx, &t, b);
    u[0] = u[1] = u[2] = 0.0;
    if (st == OR_OK) {
        int cnt = mi_count(p);
        double w[3];
        if (sto) { sto_far(dx, stok, cnt, &t, b, w); for (int a = 0; a < 3; ++a) u[a] += w[a]; }
        if (str) { str_far(dx, strm, trace, sym, cnt, &t, b, w); for (int a = 0; a < 3; ++a) u[a] += w[a]; }
    }
    free(b);
    mi_free(&t);
    return st;
}


/* ------------------------------------------------------------------ */
/* contracted direct sum (kernels.hpp:45-83); ascending source order   */
/* ------------------------------------------------------------------ */
static int direct_add(const double *pos, const double *f, const double *h, const double *nu,
                      int sto, int str, const double x[3], size_t skip, size_t s0, size_t s1,
                      double u[3]) {
    for (size_t n = s0; n < s1; ++n) {
        if (n == skip) continue;
        const double *y = pos + 3 * n;
        double d[3] = {x[0] - y[0], x[1] - y[1], x[2] - y[2]};
        double r2 = nrm2(d);
        if (r2 == 0.0) return OR_DOMAIN;
        double rinv = 1.0 / sqrt(r2);
        double r3inv = rinv / r2;
        if (sto) {
            const double *fw = f + 3 * n;
            double s = (d[0] * fw[0] + d[1] * fw[1] + d[2] * fw[2]) * r3inv; /* s^mn */
            u[0] += fw[0] * rinv + d[0] * s;
            u[1] += fw[1] * rinv + d[1] * s;
            u[2] += fw[2] * rinv + d[2] * s;
        }
        if (str) {
            const double *hw = h + 3 * n, *nw = nu + 3 * n;
            double dh = d[0] * hw[0] + d[1] * hw[1] + d[2] * hw[2];
            double dn = d[0] * nw[0] + d[1] * nw[1] + d[2] * nw[2];
            double t = dh * dn * (r3inv / r2); /* t^mn */
            u[0] += d[0] * t;
            u[1] += d[1] * t;
            u[2] += d[2] * t;
        }
    }
    return OR_OK;
}

/* ------------------------------------------------------------------ */
/* traversal (engine.hpp:80-108) with per-target counters and optional */
/* interaction-list recording (far cluster ids / near leaf ids, DFS order) */
/* ------------------------------------------------------------------ */
typedef struct {
    const or_tree *T;
    const mi_table *tab;
    int p, cnt, sto, str;
    double theta;
    const double *stok, *strm, *trace, *sym; /* per-cluster moment blocks */
} trav_ctx;

typedef struct {
    uint64_t visited, far, direct;
    int32_t *far_list, *near_list; /* optional */
    size_t far_cap, near_cap, n_far, n_near;
    double *b;
    int err;
} trav_state;

static void accumulate(const trav_ctx *C, const double x[3], size_t skip, int cid, double u[3],
                       trav_state *S) {
    const or_cluster *c = &C->T->cl[cid];
    ++S->visited;
    double dx[3] = {x[0] - c->center[0], x[1] - c->center[1], x[2] - c->center[2]};
    double dist2 = nrm2(dx);
    /* mac (cluster_tree.hpp:47-50): equality accepted, dist2 == 0 never */
    int accept = dist2 != 0.0 && c->radius * c->radius <= C->theta * C->theta * dist2;
    if (accept) {
        if (coulomb(dx, C->tab, S->b) != OR_OK) { S->err = OR_DOMAIN; return; }
        size_t E = (size_t)C->cnt;
        double w[3];
        if (C->sto) {
            sto_far(dx, C->stok + 3 * E * cid, C->cnt, C->tab, S->b, w);
            u[0] += w[0]; u[1] += w[1]; u[2] += w[2];
        }
        if (C->str) {
            str_far(dx, C->strm + 9 * E * cid, C->trace + E * cid, C->sym + 6 * E * cid, C->cnt,
                    C->tab, S->b, w);
            u[0] += w[0]; u[1] += w[1]; u[2] += w[2];
        }
        ++S->far;
        if (S->far_list && S->n_far < S->far_cap) S->far_list[S->n_far] = cid;
        ++S->n_far;
        return;
    }
    if (c->is_leaf) {
        const or_tree *T = C->T;
        int st = direct_add(T->pos, T->f, T->h, T->nu, C->sto, C->str, x, skip, c->begin, c->end, u);
        if (st != OR_OK) { S->err = st; return; }
        int has_self = skip >= c->begin && skip < c->end;
        S->direct += (c->end - c->begin) - (has_self ? 1 : 0);
        if (S->near_list && S->n_near < S->near_cap) S->near_list[S->n_near] = cid;
        ++S->n_near;
        return;
    }
    for (int s = 0; s < c->n_children && !S->err; ++s) accumulate(C, x, skip, c->children[s], u, S);
}

typedef struct {
    const trav_ctx *C;
    const double *targets; /* NULL: sources (tree order), else original-order target positions */
    size_t t0, t1;
    double *u_out;         /* original order */
    uint64_t *per_target;  /* 3 per target (visited, far, direct), original order, or NULL */
    uint64_t tot[3];
    int err;
} seg_job;

static void *run_seg(void *arg) {
    seg_job *J = arg;
    const trav_ctx *C = J->C;
    trav_state S;
    memset(&S, 0, sizeof S);
    S.b = malloc(sizeof(double) * (size_t)(C->tab->n + 1));
    for (size_t t = J->t0; t < J->t1 && !J->err; ++t) {
        double u[3] = {0, 0, 0};
        uint64_t v0 = S.visited, f0 = S.far, d0 = S.direct;
        const double *x;
        size_t skip, out;
        if (J->targets) { x = J->targets + 3 * t; skip = OR_NOSKIP; out = t; }
        else { x = C->T->pos + 3 * t; skip = t; out = C->T->to_original[t]; }
        accumulate(C, x, skip, 0, u, &S);
        if (S.err) { J->err = S.err; break; }
        J->u_out[3 * out] = u[0]; J->u_out[3 * out + 1] = u[1]; J->u_out[3 * out + 2] = u[2];
        if (J->per_target) {
            J->per_target[3 * out] = S.visited - v0;
            J->per_target[3 * out + 1] = S.far - f0;
            J->per_target[3 * out + 2] = S.direct - d0;
        }
    }
    J->tot[0] = S.visited; J->tot[1] = S.far; J->tot[2] = S.direct;
    free(S.b);
    return NULL;
}

/* Full treecode (engine.hpp:133-196): tree, moments at p with table pmax = p+2 (stresslet)
 * or p+1, traversal of every target.  targets == NULL: targets are the sources (self
 * excluded by tree index); else nt disjoint targets (no exclusion).
 * stats3 = {farfield_evals, direct_pairs, clusters_visited}. */
int or_treecode(size_t n, const double *pos, const double *f, const double *h, const double *nu,
                const double *targets, size_t nt, int p, double theta, int n0, int shrink, int sto,
                int str, int nthreads, double *u_out, uint64_t *per_target, uint64_t *stats3) {
    if (p < 0 || p > 16 || !(theta > 0.0) || !(theta < 1.0) || n0 < 1 || (!sto && !str) || n == 0)
        return OR_INVALID;
    int st;
    or_tree *T = or_tree_build(n, pos, f, h, nu, n0, shrink, &st);
    if (st != OR_OK) return st;
    mi_table tab;
    mi_init(&tab, p + (str ? 2 : 1));
    size_t E = (size_t)mi_count(p);
    double *stok = sto ? malloc(sizeof(double) * 3 * E * T->ncl) : NULL;
    double *strm = str ? malloc(sizeof(double) * 9 * E * T->ncl) : NULL;
    double *trace = str ? malloc(sizeof(double) * E * T->ncl) : NULL;
    double *sym = str ? malloc(sizeof(double) * 6 * E * T->ncl) : NULL;
    or_moments(T, p, sto, str, stok, strm, trace, sym);
    trav_ctx C = {T, &tab, p, (int)E, sto, str, theta, stok, strm, trace, sym};
    size_t ntg = targets ? nt : n;
    if (nthreads < 1) nthreads = 1;
    if ((size_t)nthreads > ntg) nthreads = ntg ? (int)ntg : 1;
    seg_job *jobs = calloc((size_t)nthreads, sizeof(seg_job));
    pthread_t *th = calloc((size_t)nthreads, sizeof(pthread_t));
    for (int w = 0; w < nthreads; ++w) {
        jobs[w].C = &C; jobs[w].targets = targets;
        jobs[w].t0 = ntg * (size_t)w / (size_t)nthreads;
        jobs[w].t1 = ntg * (size_t)(w + 1) / (size_t)nthreads;
        jobs[w].u_out = u_out; jobs[w].per_target = per_target;
        pthread_create(&th[w], NULL, run_seg, &jobs[w]);
    }
    int err = OR_OK;
    uint64_t tot[3] = {0, 0, 0};
    for (int w = 0; w < nthreads; ++w) {
        pthread_join(th[w], NULL);
        if (jobs[w].err && !err) err = jobs[w].err;
        for (int a = 0; a < 3; ++a) tot[a] += jobs[w].tot[a];
    }
    if (stats3) { stats3[0] = tot[1]; stats3[1] = tot[2]; stats3[2] = tot[0]; }
    free(jobs); free(th);
    free(stok); free(strm); free(trace); free(sym);
    mi_free(&tab);
    or_tree_free(T);
    return err;
}

/* Per-target interaction lists (DFS order) for selected targets of a built tree:
 * far[i*cap ...] cluster ids accepted, near[i*cap ...] leaf ids summed directly.
 * Counts returned in nfar/nnear (may exceed cap: then lists are truncated).
 * targets_tree_idx: tree indices (self-excluding) or, if xyz != NULL, disjoint points. */
int or_lists(const void *tp, double theta, size_t nsel, const uint32_t *tree_idx,
             const double *xyz, size_t cap, int32_t *far, int32_t *near, int64_t *nfar,
             int64_t *nnear) {
    const or_tree *T = tp;
    mi_table tab;
    mi_init(&tab, 0);
    /* list recording only: run the traversal with zero moments of order 0 (values unused) */
    trav_ctx C = {T, &tab, 0, 1, 0, 0, theta, NULL, NULL, NULL, NULL};
    trav_state S;
    memset(&S, 0, sizeof S);
    S.b = malloc(sizeof(double) * 2);
    for (size_t i = 0; i < nsel; ++i) {
        S.far_list = far + i * cap; S.near_list = near + i * cap;
        S.far_cap = S.near_cap = cap; S.n_far = S.n_near = 0;
        double u[3] = {0, 0, 0};
        const double *x = xyz ? xyz + 3 * i : T->pos + 3 * (size_t)tree_idx[i];
        size_t skip = xyz ? OR_NOSKIP : tree_idx[i];
        /* no kernel enabled: the direct loop still checks coincidence but adds nothing */
        accumulate(&C, x, skip, 0, u, &S);
        nfar[i] = (int64_t)S.n_far; nnear[i] = (int64_t)S.n_near;
    }
    free(S.b);
    mi_free(&tab);
    return S.err;
}

/* contracted_direct_velocity_at (kernels.hpp:139-150) over original-order particles;
 * targets given as indices (skip = own index).  Multithreaded over targets. */
typedef struct {
    size_t n; const double *pos, *f, *h, *nu; int sto, str;
    const int64_t *tg; size_t t0, t1; double *u; int err;
} dir_job;

static void *run_dir(void *arg) {
    dir_job *J = arg;
    for (size_t i = J->t0; i < J->t1; ++i) {
        double u[3] = {0, 0, 0};
        size_t m = (size_t)J->tg[i];
        int st = direct_add(J->pos, J->f, J->h, J->nu, J->sto, J->str, J->pos + 3 * m, m, 0, J->n, u);
        if (st) { J->err = st; return NULL; }
        J->u[3 * i] = u[0]; J->u[3 * i + 1] = u[1]; J->u[3 * i + 2] = u[2];
    }
    return NULL;
}

int or_direct_at(size_t n, const double *pos, const double *f, const double *h, const double *nu,
                 int sto, int str, const int64_t *targets, size_t nt, int nthreads, double *u_out) {
    if (nthreads < 1) nthreads = 1;
    if ((size_t)nthreads > nt) nthreads = nt ? (int)nt : 1;
    dir_job *jobs = calloc((size_t)nthreads, sizeof(dir_job));
    pthread_t *th = calloc((size_t)nthreads, sizeof(pthread_t));
    for (int w = 0; w < nthreads; ++w) {
        dir_job J = {n, pos, f, h, nu, sto, str, targets, nt * (size_t)w / (size_t)nthreads,
                     nt * (size_t)(w + 1) / (size_t)nthreads, u_out, 0};
        jobs[w] = J;
        pthread_create(&th[w], NULL, run_dir, &jobs[w]);
    }
    int err = 0;
    for (int w = 0; w < nthreads; ++w) {
        pthread_join(th[w], NULL);
        if (jobs[w].err && !err) err = jobs[w].err;
    }
    free(jobs); free(th);
    return err;
}

/* direct velocity at arbitrary (disjoint) points, no exclusion (reftest::direct_at analogue
 * in contracted form; tests/support/reference_farfield.hpp:20-37). */
int or_direct_points(size_t n, const double *pos, const double *f, const double *h,
                     const double *nu, int sto, int str, const double *xyz, size_t nt,
                     double *u_out) {
    for (size_t i = 0; i < nt; ++i) {
        double u[3] = {0, 0, 0};
        int st = direct_add(pos, f, h, nu, sto, str, xyz + 3 * i, OR_NOSKIP, 0, n, u);
        if (st) return st;
        u_out[3 * i] = u[0]; u_out[3 * i + 1] = u[1]; u_out[3 * i + 2] = u[2];
    }
    return 0;
}

/* relative_error (error_metric.hpp:13-24) */
int or_relative_error(size_t n, const double *ref, const double *test, double *out) {
    if (n == 0) return OR_INVALID;
    double num = 0.0, den = 0.0;
    for (size_t i = 0; i < n; ++i) {
        double d[3] = {ref[3 * i] - test[3 * i], ref[3 * i + 1] - test[3 * i + 1], ref[3 * i + 2] - test[3 * i + 2]};
        num += nrm2(d);
        den += nrm2(ref + 3 * i);
    }
    if (den == 0.0) return OR_DOMAIN;
    *out = sqrt(num / den);
    return OR_OK;
}

/* mac (cluster_tree.hpp:47-50): accept iff dist2 != 0 and r*r <= theta*theta*dist2 */
int or_mac(double radius, double dist2, double theta) {
    if (dist2 == 0.0) return 0;
    return radius * radius <= theta * theta * dist2;
}

/* ------------------------------------------------------------------ */
/* Seeded BASELINE inputs, restated on the oracle side so that the      */
/* reference arm of bench.py never loads the product library.          */
/* Stream: SplitMix64 (rng.hpp:10-29): uniform01 = (next >> 11) 2^-53,  */
/* symmetric = 2u - 1.  Per-particle draw order of                      */
/* testutil::random_particles (tests/support/test_helpers.hpp:31-49):   */
/* position, f, then h and the rejection unit normal (random_unit,      */
/* :22-28; v * (1/sqrt(n2)) as vec3.hpp:41).  The BASELINE recipes      */
/* (cube, sphere surface, Gaussian mixture, target points) are those    */
/* of DESIGN.md section 7; tests/test_inputs_io.py pins the bytes to    */
/* the product's st_generate by SHA-256.                                */
/* kind: 0 unit box, 1 cube, 2 sphere surface, 3 mixture, 4 points.     */
/* ------------------------------------------------------------------ */
static uint64_t sm_next(uint64_t *s) {
    uint64_t z;
    *s += 0x9E3779B97F4A7C15ull;
    z = *s;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static double sm_u01(uint64_t *s) { return (double)(sm_next(s) >> 11) * (1.0 / 9007199254740992.0); }
static double sm_sym(uint64_t *s) { return 2.0 * sm_u01(s) - 1.0; }
static void sm_unit(uint64_t *s, double out[3]) {
    for (;;) {
        double v[3], n2, inv;
        v[0] = sm_sym(s);
        v[1] = sm_sym(s);
        v[2] = sm_sym(s);
        n2 = nrm2(v);
        if (n2 > 1e-4 && n2 <= 1.0) {
            inv = 1.0 / sqrt(n2);
            out[0] = v[0] * inv;
            out[1] = v[1] * inv;
            out[2] = v[2] * inv;
            return;
        }
    }
}

int or_generate(int kind, size_t n, uint64_t seed, int with_stresslets, double *pos, double *f,
                double *h, double *nu) {
    uint64_t s = seed;
    double centres[16][3];
    size_t i;
    int a, k;
    const double two_pi = 6.283185307179586;
    if (kind < 0 || kind > 4 || !pos) return OR_INVALID;
    if (kind != 4 && (!f || (with_stresslets && (!h || !nu)))) return OR_INVALID;
    if (kind == 3)
        for (k = 0; k < 16; ++k)
            for (a = 0; a < 3; ++a) centres[k][a] = -0.5 + 1.0 * sm_u01(&s);
    for (i = 0; i < n; ++i) {
        double *p = pos + 3 * i;
        if (kind == 0) {
            for (a = 0; a < 3; ++a) p[a] = 0.0 + 1.0 * sm_u01(&s);
        } else if (kind == 1 || kind == 4) {
            for (a = 0; a < 3; ++a) p[a] = -0.5 + 1.0 * sm_u01(&s);
        } else if (kind == 2) {
            sm_unit(&s, p);
        } else {
            const double *c = centres[sm_next(&s) % 16];
            double g[4];
            for (k = 0; k < 2; ++k) { /* Box-Muller, two normals per uniform pair */
                const double u1 = sm_u01(&s), u2 = sm_u01(&s);
                const double rad = sqrt(-2.0 * log(1.0 - u1));
                g[2 * k] = rad * cos(two_pi * u2);
                g[2 * k + 1] = rad * sin(two_pi * u2);
            }
            for (a = 0; a < 3; ++a) p[a] = c[a] + 0.05 * g[a];
        }
        if (kind == 4) continue;
        for (a = 0; a < 3; ++a) f[3 * i + a] = sm_sym(&s);
        if (!with_stresslets) {
            if (kind == 2 && nu)
                for (a = 0; a < 3; ++a) nu[3 * i + a] = p[a];
            continue;
        }
        for (a = 0; a < 3; ++a) h[3 * i + a] = sm_sym(&s);
        if (kind == 2) {
            for (a = 0; a < 3; ++a) nu[3 * i + a] = p[a];
        } else {
            sm_unit(&s, nu + 3 * i);
        }
    }
    return OR_OK;
}
