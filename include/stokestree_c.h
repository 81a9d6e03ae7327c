/*
 * stokestree_c.h -- C ABI of the B200-native treecode (libstokestree_b200.so).
 *
 * Drop-in boundary for the reference's public C++ entry points in
 * /root/reference/proj/include/stokestree/ (header-only C++20 library).  Every
 * entry point below names the reference interface it replaces (file:line).
 * The C++ shim (include/stokestree/ headers) re-exposes the reference's exact
 * names on top of this ABI; INTEGRATION.md shows the bindings.
 *
 * Conventions
 *  - Plain pointers and sizes only.  Vec3 arrays are interleaved x,y,z doubles
 *    (the reference's std::vector<Vec3> storage, vec3.hpp:9-46), n entries.
 *  - Host pointers unless the function name ends in _device.
 *  - Every call returns an st_status; on failure st_last_error() (thread-local)
 *    holds the message the reference would have thrown.
 *      ST_INVALID_ARGUMENT -> std::invalid_argument
 *      ST_DOMAIN_ERROR     -> std::domain_error
 *      ST_CUDA_ERROR / ST_NCCL_ERROR / ST_RUNTIME_ERROR -> std::runtime_error
 *  - All arithmetic is fp64 on the GPU.  There is no CPU fallback: without a
 *    usable sm_100 device every compute entry point fails with ST_CUDA_ERROR.
 */
#ifndef STOKESTREE_C_H
#define STOKESTREE_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ST_ABI_VERSION 1

typedef enum st_status {
    ST_OK = 0,
    ST_INVALID_ARGUMENT = 1,
    ST_DOMAIN_ERROR = 2,
    ST_CUDA_ERROR = 3,
    ST_NCCL_ERROR = 4,
    ST_RUNTIME_ERROR = 5
} st_status;

/* ParticleSet (particles.hpp:29-36).  dipole_weight/normal may be NULL when
 * stresslets are off; force_weight may be NULL when Stokeslets are off. */
typedef struct st_particles {
    size_t n;
    const double* position;
    const double* force_weight;
    const double* dipole_weight;
    const double* normal;
} st_particles;

/* TreecodeParams (engine.hpp:21-42) + KernelSelection (particles.hpp:13-25).
 * `workers` is validated (>= 1) and otherwise ignored: the GPU path is
 * bit-identical for every worker count, as the reference promises
 * (engine.hpp:163-169).  `devices` (new, trailing) is the GPU count (>= 1). */
typedef struct st_params {
    int order;          /* p in [0, 16]                      */
    double theta;       /* MAC parameter, strictly in (0, 1) */
    int leaf_capacity;  /* N0 >= 1                           */
    int shrink;         /* bool                              */
    int stokeslet;      /* bool                              */
    int stresslet;      /* bool                              */
    int workers;        /* >= 1, accepted and ignored        */
    int devices;        /* >= 1                              */
} st_params;

/* TraversalStats (engine.hpp:44-55) + VelocityResult timings (:57-64).
 * time_* are device (CUDA-event) seconds of the phases; time_far_s and
 * time_near_s are the far-field and near-field kernels alone. */
typedef struct st_stats {
    uint64_t farfield_evals;
    uint64_t direct_pairs;
    uint64_t clusters_visited;
    double time_build_s;
    double time_moments_s;
    double time_traverse_s;
    double time_total_s;
    double time_far_s;
    double time_near_s;
    double time_h2d_s;
    double time_d2h_s;
    uint64_t gpu_launches; /* kernels this call launched */
} st_stats;

typedef struct st_tree st_tree;

int st_abi_version(void);
const char* st_last_error(void);
/* Number of visible CUDA devices (0 when none / no driver). */
st_status st_device_count(int* out);

/* Device memory the library keeps between calls on the CURRENT device -- its private
 * stream-ordered pool (the process's default pool is never reconfigured) and the
 * near-field entry workspace -- goes back to the driver.  No reference counterpart (the
 * reference holds no device memory); call it when the host application needs the memory
 * back.  Synchronises the device. */
st_status st_release_workspace(void);

/* ---- validation (pure host, no GPU needed) ---- */
/* TreecodeParams::validate (engine.hpp:31-41). */
st_status st_params_validate(const st_params* params);

/* ---- the treecode path ---- */
/* treecode_velocity / parallel_velocity (engine.hpp:185-196, run_treecode :133-180):
 * validate (engine.hpp:31-41, particles.hpp:41-70), build the tree, compute the
 * moments, traverse every target; u_out[3n] in ORIGINAL particle order. */
st_status st_treecode_velocity(const st_particles* src, const st_params* params, double* u_out,
                               st_stats* stats);

/* Extended form.  targets == NULL: targets are the sources (self excluded by
 * tree index, engine.hpp:118-131).  Otherwise n_targets disjoint points
 * (xyz interleaved), nothing excluded (skip = kNoSkip, kernels.hpp:43) -- the
 * entry cfg4 needs, absent from the reference's public API.
 * per_target (optional, 3 * n_targets uint64, ORIGINAL target order):
 * {clusters_visited, farfield_evals, direct_pairs} of each target. */
st_status st_treecode_velocity_ex(const st_particles* src, const double* targets, size_t n_targets,
                                  const st_params* params, double* u_out, uint64_t* per_target,
                                  st_stats* stats);

/* Device-resident form: every pointer (src arrays, targets, u_out) is device
 * memory on the current device; work is issued on `stream` (cudaStream_t,
 * NULL = the legacy default stream).  shard / n_shards select a contiguous,
 * work-balanced range of the key-ordered target batches (n_shards = 1:
 * all); only that shard's entries of u_out are written.  This is the entry a
 * multi-process (one rank per GPU) driver uses; the tree and moments are
 * rebuilt redundantly and bit-identically on every rank. */
st_status st_treecode_velocity_device(const st_particles* src_device, const double* targets_device,
                                      size_t n_targets, const st_params* params,
                                      double* u_out_device, int shard, int n_shards,
                                      void* stream, st_stats* stats);
/* As st_treecode_velocity_device while the weight arrays (force_weight, dipole_weight,
 * normal) may still be in flight: the call waits for `weights_ready` (a cudaEvent_t, may
 * be NULL) after the tree build, which reads positions only -- so a caller uploading its
 * inputs copies positions (and targets) first and overlaps the rest with the build
 * (what st_treecode_velocity_ex does internally for host arrays). */
st_status st_treecode_velocity_device_ev(const st_particles* src_device, const double* targets_device,
                                         size_t n_targets, const st_params* params,
                                         double* u_out_device, int shard, int n_shards,
                                         void* stream, void* weights_ready, st_stats* stats);
/* As st_treecode_velocity_device_ev while the disjoint targets may also still be in flight:
 * the call waits for `targets_ready` (a cudaEvent_t, may be NULL) before it orders them --
 * beside the tree build, which then needs only the positions to have landed. */
st_status st_treecode_velocity_device_ev2(const st_particles* src_device, const double* targets_device,
                                          size_t n_targets, const st_params* params,
                                          double* u_out_device, int shard, int n_shards,
                                          void* stream, void* targets_ready, void* weights_ready,
                                          st_stats* stats);

/* Order sweep (new): velocities at every order in orders[n_orders] (params->order
 * ignored) from one tree, one moment pass at max(orders) -- order-p moments are the
 * graded prefix of higher-order ones (multi_index.hpp:110-114) -- and one near-field
 * pass (independent of p).  u_out[n_orders][3*n_t] in original order; each order's
 * field is bit-identical to st_treecode_velocity_ex at that order.  far_seconds
 * (optional, n_orders) receives each order's far-field kernel time.  stats are the
 * traversal counters (identical for every order). */
st_status st_treecode_velocity_sweep(const st_particles* src, const double* targets, size_t n_targets,
                                     const st_params* params, const int* orders, int n_orders,
                                     double* u_out, double* far_seconds, st_stats* stats);

/* Interaction lists (engine.hpp:80-108) of selected targets, for parity checks:
 * target_index[i] is a source index (targets = sources, self excluded) when
 * points == NULL, else points[3i..] is a disjoint target.  For each target, far[i*cap..]
 * receives the accepted clusters and near[i*cap..] the leaves summed directly, in the
 * reference's DFS order, as PRE-ORDER cluster ids (the reference's cluster ids);
 * n_far[i] / n_near[i] the full counts (lists truncated at cap). */
st_status st_interaction_lists(const st_particles* src, const st_params* params,
                               const size_t* target_index, const double* points, size_t n_sel,
                               size_t cap, int32_t* far, int32_t* near, int64_t* n_far,
                               int64_t* n_near);

/* ---- one process per GPU, moment pass split over the ranks ----
 * As st_treecode_velocity_device(shard, n_shards), but the moment pass is not replicated:
 * each rank computes the moments and far-field weights of its share of the tree (whole
 * subtrees, balanced by particle count), and the ranks exchange them through `exchange`,
 * which the library calls once per call (on every rank, also a rank with no targets),
 * after the rank's own rows are queued on `ex->stream` and before any far-field kernel.
 * The callback must make every rank's rows of ex->w and units of ex->m present in this
 * rank's buffers in stream order on ex->stream -- e.g. one NCCL broadcast per rank of
 * rows [w_cuts[r], w_cuts[r+1]) and units [m_cuts[r], m_cuts[r+1]) -- and return 0
 * (non-zero fails the call with ST_RUNTIME_ERROR).  The cut points are identical on every
 * rank.  The velocities are bit-identical to the replicated path's.  exchange == NULL or
 * n_shards == 1: the replicated path.  (DESIGN.md section 6.) */
typedef struct st_shard_exchange {
    int shard, n_shards;
    double* w;             /* device: folded far-field weights, ncl rows of w_row doubles   */
    size_t w_row, ncl;
    const size_t* w_cuts;  /* host, n_shards + 1: rank r produced rows [w_cuts[r], w_cuts[r+1]) */
    double* m;             /* device: moments of the n_units subtree roots, m_row doubles each */
    size_t m_row, n_units;
    const size_t* m_cuts;  /* host, n_shards + 1: rank r produced units [m_cuts[r], m_cuts[r+1]) */
    void* stream;          /* the call's stream (cudaStream_t): enqueue the exchange on it    */
} st_shard_exchange;
typedef int (*st_exchange_fn)(void* ctx, const st_shard_exchange* ex);
st_status st_treecode_velocity_device_split(const st_particles* src_device, const double* targets_device,
                                            size_t n_targets, const st_params* params, double* u_out_device,
                                            int shard, int n_shards, void* stream, st_exchange_fn exchange,
                                            void* ctx, st_stats* stats);

/* Shard evaluation for collective gathers (one rank per GPU): like
 * st_treecode_velocity_device but the shard's velocities are written in BATCH order
 * (octree-key order of 32-target batches) into u_batch[3*t0 .. 3*t1), so every rank owns a
 * contiguous slice [t0, t1) that an all-gather can move; batch_to_original (device,
 * n_targets uint32, optional) receives the permutation, identical on every rank. */
st_status st_treecode_shard_device(const st_particles* src_device, const double* targets_device,
                                   size_t n_targets, const st_params* params, int shard, int n_shards,
                                   double* u_batch_device, uint32_t* batch_to_original_device,
                                   size_t* t0, size_t* t1, void* stream, st_stats* stats);
/* u_out[3*batch_to_original[t] + a] = u_batch[3*t + a] for all t < n (device, stream). */
st_status st_unbatch_device(size_t n, const uint32_t* batch_to_original_device,
                            const double* u_batch_device, double* u_out_device, void* stream);

/* ---- one process per GPU: CUDA IPC of an output buffer (NVLink peer stores) ----
 * st_ipc_export: 64-byte handle of the allocation holding device pointer ptr, and ptr's
 * offset inside it.  st_ipc_open (in another process, on a GPU with peer access): the
 * same memory as a device pointer of this process; st_ipc_close releases it.  Passing
 * the opened pointer as u_out of st_treecode_velocity_device(shard = rank, n_shards =
 * world) makes every rank's epilogue kernel store its shard's velocities straight into
 * the owner's buffer in original order: the gather is fused into the kernel (replaces
 * the reference's per-worker writes into one shared output, engine.hpp:157-169). */
st_status st_ipc_export(const void* device_ptr, unsigned char handle[64], size_t* offset);
st_status st_ipc_open(const unsigned char handle[64], size_t offset, void** device_ptr);
st_status st_ipc_close(void* device_ptr);

/* ---- one process per GPU with NCCL inside the library (no torch.distributed needed) ----
 * Rank 0 calls st_nccl_unique_id and ships the 128-byte id to the other ranks by any means
 * (a file, a socket, MPI); every rank then calls st_nccl_comm_init(id, n_ranks, rank) with
 * its GPU current.  The library loads libnccl.so.2 at first use (the copy already in the
 * process when PyTorch is, else the system's); failures return ST_NCCL_ERROR. */
typedef struct st_comm st_comm;
st_status st_nccl_unique_id(unsigned char id[128]);
st_status st_nccl_comm_init(const unsigned char id[128], int n_ranks, int rank, st_comm** comm);
void st_nccl_comm_free(st_comm* comm);
/* The treecode on one rank of `comm` (replaces engine.hpp:157-169's worker threads over one
 * output with one rank per GPU): every rank holds all sources (and targets) on its device;
 * the moment pass is split over the ranks, its weight rows and subtree-root moments moved
 * by NCCL broadcasts on `stream`; the rank evaluates its work-balanced shard of the
 * key-ordered target batches; u_out (device, on every rank) receives every target's
 * velocity in original order and stats the whole job's counters (one NCCL sum: each
 * target has exactly one writer, so the values are one GPU's -- except that a component
 * exactly -0.0 comes back +0.0).  Every rank must make the call (collective). */
st_status st_treecode_velocity_nccl(const st_particles* src_device, const double* targets_device,
                                    size_t n_targets, const st_params* params, double* u_out_device,
                                    const st_comm* comm, void* stream, st_stats* stats);

/* ---- direct sums (O(N^2) oracle path) ---- */
/* contracted_direct_velocity(ps, sel, first, last) (kernels.hpp:123-136). */
st_status st_direct_velocity(const st_particles* src, int stokeslet, int stresslet, size_t first,
                             size_t last, double* u_out);
/* contracted_direct_velocity_at (kernels.hpp:139-150). */
st_status st_direct_velocity_at(const st_particles* src, int stokeslet, int stresslet,
                                const size_t* targets, size_t n_targets, double* u_out);
/* naive_direct_velocity (kernels.hpp:89-118): forms S_ij and T_ijl per pair. */
st_status st_naive_direct_velocity(const st_particles* src, int stokeslet, int stresslet,
                                   double* u_out);

/* ---- tree and moments ---- */
/* build_tree (cluster_tree.hpp:152-192).  Clusters in pre-order (id 0 = root). */
st_status st_build_tree(const st_particles* src, int leaf_capacity, int shrink, st_tree** out);
size_t st_tree_num_clusters(const st_tree* tree);
size_t st_tree_num_particles(const st_tree* tree);
/* Export (any pointer may be NULL):
 *   begin_end[2*ncl] (Cluster::begin/end), geom[10*ncl] = center xyz, radius,
 *   bbox lo xyz, bbox hi xyz; children[8*ncl] (-1 padded, slot order);
 *   meta[2*ncl] = n_children, is_leaf; to_original[n] (ClusterTree::to_original). */
st_status st_tree_export(const st_tree* tree, int64_t* begin_end, double* geom, int32_t* children,
                         int32_t* meta, uint32_t* to_original);
void st_tree_free(st_tree* tree);

/* compute_moments (moments.hpp:140-175) in the reference layout (:15-27):
 * stok[ncl*E*3], str[ncl*E*9], trace[ncl*E], sym[ncl*E*6], E = (p+1)(p+2)(p+3)/6.
 * Buffers of a disabled kernel may be NULL. */
st_status st_compute_moments(const st_tree* tree, int order, int stokeslet, int stresslet,
                             double* stok, double* str, double* trace, double* sym);

/* ---- per-pair far-field API, batched (coulomb.hpp:28-59, farfield.hpp:30-96) ---- */
/* b^k for every k with |k| <= pmax, graded-lex order (multi_index.hpp:36-44), at
 * n_pairs displacements dx[3*n_pairs]; b_out[n_pairs * E(pmax)]. */
st_status st_coulomb_coeffs(size_t n_pairs, const double* dx, int pmax, double* b_out);
/* Explicit Taylor coefficients (taylor_coeffs.hpp:13-46) for every multi-index e of grade
 * <= order: a_sto[(q*E(order) + e)*9 + 3i+j] = a^k_ij, a_str[(q*E(order) + e)*27 + 9i+3j+l]
 * = a~^k_ijl.  b is st_coulomb_coeffs' output at depth pmax_b (E(pmax_b) doubles per pair);
 * NULL = computed on the device from dx.  Either output may be NULL; a_sto needs
 * order+1 <= pmax_b and a_str order+2 <= pmax_b (else ST_INVALID_ARGUMENT, :18-19/:35-36). */
st_status st_taylor_coeffs(size_t n_pairs, const double* dx, const double* b, int pmax_b, int order,
                           double* a_sto, double* a_str);
/* stokeslet_farfield + stresslet_farfield for n_pairs (dx, moment block) pairs; moment
 * blocks in the reference layout, one block of E(p) entries per pair.  trace and sym
 * (StressletMomentsView, moments.hpp:103-134) are accepted for the signature but not
 * read: they are recomputed from str, which is how compute_moments defines them
 * (derive_stresslet_contractions, moments.hpp:66-80).  A caller whose trace/sym are not the contractions of its str
 * gets the far field of str. */
st_status st_farfield_pairs(size_t n_pairs, const double* dx, int order, int stokeslet,
                            int stresslet, const double* stok, const double* str,
                            const double* trace, const double* sym, double* u_out);

/* ---- metric (error_metric.hpp:13-24), host ---- */
st_status st_relative_error(size_t n, const double* u_ref, const double* u_test, double* out);

/* ---- multi-GPU planning (host, no GPU needed) ---- */
/* Contiguous work-balanced cut points: given per-unit weights w[n_units] (any
 * non-negative cost), write cuts[n_shards+1] with cuts[0] = 0, cuts[n_shards] =
 * n_units, such that shard s owns [cuts[s], cuts[s+1]) and the prefix-weight
 * boundaries are as close as possible to s/n_shards of the total. */
st_status st_shard_cuts(size_t n_units, const double* weights, int n_shards, size_t* cuts);

/* ---- seeded synthetic inputs (host) ---- */
enum {
    ST_GEN_UNIT = 0,    /* testutil::random_particles: positions in [0,1)^3       */
    ST_GEN_CUBE = 1,    /* BASELINE cfg0/1/3: positions in [-0.5,0.5)^3            */
    ST_GEN_SPHERE = 2,  /* cfg2: uniform on the unit sphere, nu = outward normal   */
    ST_GEN_MIXTURE = 3, /* cfg4 sources: 16 Gaussians, sigma 0.05                 */
    ST_GEN_POINTS = 4   /* cfg4 targets: positions only, [-0.5,0.5)^3              */
};
st_status st_generate(int kind, size_t n, uint64_t seed, int with_stresslets, double* pos,
                      double* f, double* h, double* nu);

/* The paper's own test geometries (testcases.hpp:40-124), bit-identical to the reference:
 * icosahedral sphere refined `levels` times (N = st_sphere_count(levels) = 20*4^levels;
 * normals = positions; f, h uniform in [-1,1]) and Stokeslets uniform in a cube of side
 * (n/density)^(1/3) (no stresslet arrays). */
size_t st_sphere_count(int levels);
st_status st_generate_sphere_icosa(int levels, uint64_t seed, double* pos, double* f, double* h,
                                   double* nu);
st_status st_generate_cube_density(size_t n, double density, uint64_t seed, double* pos, double* f);

/* ---- particle text format (particle_io.hpp:30-126), host ---- */
typedef struct st_loaded st_loaded;
/* write_particles: validates like validate(ps, sel), header "x [f] [h nu]", "%.17g" fields. */
st_status st_write_particles(const char* path, const st_particles* src, int stokeslet, int stresslet);
/* read_particles: returns a handle, the particle count and the selection the header declares
 * (errors: ST_RUNTIME_ERROR with the reference's message and line number). */
st_status st_read_particles(const char* path, st_loaded** out, size_t* n, int* stokeslet,
                            int* stresslet);
/* copy the loaded arrays (3n doubles each; absent blocks leave their buffer untouched) */
st_status st_loaded_copy(const st_loaded* loaded, double* pos, double* f, double* h, double* nu);
void st_loaded_free(st_loaded* loaded);

/* ---- measurement ---- */
/* FP64 FMA throughput probe (a DFMA-only kernel over every SM): TFLOP/s with
 * FMA = 2 flop, run for roughly `seconds`. */
st_status st_fp64_peak(double seconds, double* tflops);

#ifdef __cplusplus
}
#endif

#endif /* STOKESTREE_C_H */
