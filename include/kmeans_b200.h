/*
 * kmeans_b200.h — C ABI of the B200-native MTI-pruned Lloyd's k-means hot path.
 *
 * Method: Lloyd's k-means (§4.1) with Minimal Triangle
 * Inequality pruning (§3.3), merged MM step with per-thread
 * state and one reduction per iteration (§3.2) and the
 * distributed "merge global state" step (§7) realised as one
 * NCCL allreduce per iteration.  Readings of garbled/silent passages: DESIGN.md "Readings".
 *
 * One iteration t (kmeans_iterate) runs, on the context's CUDA stream:
 *   S1 geometry + drift  f(c) = ||C_t-1[c] - C_t-2[c]||, H = 1/2 ||C[c]-C[c']||,
 *                        s(c) = min_{c'!=c} H, neighbour lists sorted by H
 *   S2 MTI assignment    u += f(a); skip point iff u <= s(a); else tighten u = d(x, C[a]) and
 *                        skip candidate c' iff H[a][c'] >= u
 *   S3 reduction         per-cluster fp64 sums and counts, allreduced over ranks
 *   S4 update            C_t[c] = sum/count, or C_t-1[c] when the cluster is empty; stop iff changed <= tol
 * Iteration 1 has no bounds: every point evaluates all k centroids (S0).
 *
 * Precision ("exact mode"): fp32 points and fp32 screening distances with
 * rigorously rounded bounds derived from the fp64 master centroids; candidates whose fp32
 * error intervals overlap are re-evaluated in fp64, so assignments equal the fp64 argmin;
 * sums, counts and centroids are fp64.
 *
 * Conventions for every call:
 *   - returns km_status; KM_OK (0) on success.  On failure a thread-local message is
 *     available from kmeans_last_error() and the context is left unchanged unless stated.
 *   - a context is used by one host thread at a time; many contexts per process are allowed.
 *   - all work is enqueued on the context stream; calls that return host values synchronise it.
 */
#ifndef KMEANS_B200_H
#define KMEANS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t km_status;
enum {
    KM_OK = 0,
    KM_EARG = 1,        /* invalid argument (sizes, null or misaligned pointers, k > n_global, d > 64, k > 4096) */
    KM_ENONFINITE = 2,  /* NaN/Inf found in points or centroids (only when check_finite = 1) */
    KM_ECUDA = 3,       /* CUDA runtime error (message has cudaGetErrorString) */
    KM_ENCCL = 4,       /* NCCL error, or libnccl.so.2 could not be loaded for world > 1 */
    KM_ENOMEM = 5,      /* device allocation failed */
    KM_ESTATE = 6       /* call not valid in the current state (e.g. sse before any iteration) */
};

/* MTI: the paper's Minimal Triangle Inequality (knori, §3.3).  NONE: every distance
 * (knori-).  TI: Elkan's triangle inequality with an n x k lower-bound matrix, the baseline the
 * paper compares MTI with (§2, 876-885; claims 17-24); needs k * n_local * 4 bytes of
 * device memory for the bounds (KM_ENOMEM otherwise) and keeps the caller's row order. */
enum { KM_PRUNE_MTI = 0, KM_PRUNE_NONE = 1, KM_PRUNE_TI = 2 };

/* Row re-bucketing policy: the context keeps its own copy of
 * the points physically sorted by (assigned cluster, survivor-prefix class) so that warps
 * evaluate candidates with broadcast centroid reads.  AUTO re-sorts after iteration 1 and
 * whenever the points reassigned since the last sort exceed resort_fraction * n_local. */
enum { KM_RESORT_AUTO = 0, KM_RESORT_NEVER = 1, KM_RESORT_ALWAYS = 2 };

/* Candidate-evaluation engine of the MTI pass.  AUTO: TENSOR_CHUNKED when d pads
 * to 32 and k >= 512 (the dense-survivor regime, C5), else CUDA_CORE (measured on B200, DESIGN.md
 * "Engine choice").  CUDA_CORE: the CUDA-core
 * walk ("k_walk"; "k_walk_skip1" when the previous pass's clause-1 rate exceeds 15 %).  SCREEN:
 * the same walk split in two kernels ("k_screen": every row, minimum candidate value only, the
 * rows that provably stay are decided; "k_resolve": the queued rest, direct form + exact-mode
 * decision).  TENSOR: the tcgen05 TF32x3 kernel ("k_mti_tc"; d padded to 8, 16 or 32; measured
 * slower, opt-in).  TENSOR_SCREEN: the tcgen05 kernel screening (smallest column value only, rows
 * that provably stay decided; "k_mti_tc_screen") followed by k_resolve.  TENSOR_CHUNKED: the
 * tcgen05 screen over the whole neighbour list in 128-column chunks ("k_tcc", km_tcc.cu; no
 * column cap, for large k) followed by k_resolve.  All give the same (exact-mode) assignments.  Iteration 1 and KM_PRUNE_NONE
 * always use the CUDA-core dense kernel. */
enum { KM_ENGINE_AUTO = 0, KM_ENGINE_CUDA_CORE = 1, KM_ENGINE_TENSOR = 2, KM_ENGINE_SCREEN = 3,
       KM_ENGINE_TENSOR_SCREEN = 4, KM_ENGINE_TENSOR_CHUNKED = 5 };

typedef struct km_options {
    int32_t device;            /* CUDA device ordinal the context lives on */
    void *stream;              /* cudaStream_t, borrowed; NULL = the context creates its own */
    int32_t prune;             /* KM_PRUNE_MTI (knori), KM_PRUNE_NONE (knori-, all k distances) or
                                  KM_PRUNE_TI (Elkan baseline) */
    int32_t rank;              /* this process's rank, 0 <= rank < world */
    int32_t world;             /* number of ranks (GPUs); 1 = no collective */
    uint8_t nccl_unique_id[128]; /* ncclUniqueId from kmeans_nccl_unique_id() on rank 0 (world > 1) */
    int64_t n_global;          /* total rows over all ranks (used for k <= n_global); 0 = n_local * world */
    int32_t check_finite;      /* 1 = scan points and centroids for NaN/Inf at create (KM_ENONFINITE) */
    int32_t points_on_host;    /* 1 = points pointer is host memory (pinned preferred); copied at create */
    int32_t resort_policy;     /* KM_RESORT_* */
    float resort_fraction;     /* AUTO threshold; 0 = default (0.25 walk / tensor engines, 0.10 others) */
    int32_t engine;            /* KM_ENGINE_* (default AUTO) */
    int32_t spherical;         /* 1 = spherical k-means (§4.2 "sk-means", 1133-1140):
                                  the context's copy of every row is projected to the unit sphere once
                                  at create (x / ||x||, fp64, rounded to fp32), the initial centroids
                                  likewise (fp64), and every update re-normalises the mean (fp64);
                                  assignment = Euclidean argmin on the sphere = cosine argmax, so MTI
                                  applies unchanged.  A zero row or zero initial centroid is KM_EARG. */
    int32_t no_graph;          /* 1 = launch every kernel of an iteration eagerly; 0 (default) = from
                                  iteration 2 on, the iteration (S1-S4 + allreduce + counter read-back)
                                  is captured once per row buffer as a CUDA graph and replayed */
    int32_t force_comm;        /* 1 = create the NCCL communicator and run the allreduce even when
                                  world == 1 (a 1-rank communicator; needs nccl_unique_id): exercises
                                  the multi-GPU data path on one GPU */
    float resum_moves;         /* the walk, tensor-core and TI passes update the per-cluster sums by the
                                  rows that moved (reading B5); once the moves applied since
                                  the last full reduction exceed resum_moves * n_global, the sums are
                                  re-derived from every row (bounds fp64 drift).  0 = default 4;
                                  < 0 = never */
    int32_t reserved[3];
} km_options;

typedef struct km_iter_stats {
    int64_t changed;   /* points whose assignment changed (global, post-allreduce); iteration 1: n */
    int64_t dists;     /* point-centroid distances evaluated under the MTI semantics (global) */
    int64_t clause1;   /* points skipped by clause 1 (global) */
    int64_t refined;   /* points re-evaluated in fp64 by exact mode (global) */
    int64_t walk_steps; /* warp-steps of the MTI candidate walk (global); lane efficiency =
                           (dists - points tightened) / (32 * walk_steps) */
    int32_t empty;     /* clusters with no points after this iteration's assignment */
    int32_t resorted;  /* 1 if the rows were re-bucketed after this iteration's pass */
    float ms_iter;     /* device time of the whole iteration (CUDA events, this rank) */
    float ms_assign;   /* device time of the assignment(+reduction) kernel (this rank) */
    float ms_sort;     /* device time of re-bucketing (0 if none) */
    float ms_comm;     /* device time of the allreduce (0 if world == 1) */
    int64_t fallbacks; /* rows whose fp32 candidate intervals did not decide the winner and were
                          re-walked in the direct form (then refined in fp64 if still tied; global) */
} km_iter_stats;

typedef struct km_ctx km_ctx;

/* Fill *opt with defaults: device 0, NULL stream, MTI, rank 0, world 1, AUTO re-sort, AUTO engine. */
void kmeans_default_options(km_options *opt);

/* rank 0 only (world > 1): write a fresh ncclUniqueId (128 bytes) to out; the caller
 * broadcasts it to the other ranks and passes it in km_options.nccl_unique_id.  Loads
 * libnccl.so.2 dynamically (KM_ENCCL if unavailable). */
km_status kmeans_nccl_unique_id(uint8_t out[128]);

/*
 * Create a context for this rank's shard.
 *   n_local           rows held by this rank (>= 1); rank r of G conventionally holds rows
 *                     [floor(r n/G), floor((r+1) n/G)) of the global data
 *   d                 dimensions, 1 <= d <= 64
 *   k                 clusters, 1 <= k <= min(4096, n_global)
 *   points            n_local x d fp32, row-major, contiguous.  Device memory on opt->device
 *                     (borrowed: read during create only, never written) or host memory when
 *                     opt->points_on_host = 1.  Must be 4-byte aligned.
 *   init_centroids    k x d fp64 row-major host array (copied); identical on all ranks.
 *   opt               may be NULL (defaults).  Ownership of opt->stream stays with the caller.
 *   out               receives the context.
 * Collective over ranks when world > 1 (NCCL communicator creation).
 * Errors: KM_EARG, KM_ENONFINITE, KM_ECUDA, KM_ENCCL, KM_ENOMEM.
 */
km_status kmeans_create(int64_t n_local, int32_t d, int32_t k, const float *points,
                        const double *init_centroids, const km_options *opt, km_ctx **out);

/* One full iteration (S1-S4; S0 on the first call).  Collective when world > 1.
 * changed / dists (may be NULL) receive this iteration's global counts. */
km_status kmeans_iterate(km_ctx *ctx, int64_t *changed, int64_t *dists);

/* Iterate until changed <= tol (a count of points; BASELINE uses tol = 0) or max_iters
 * iterations have run in this call, then kmeans_finalize.  max_iters = 0 runs nothing
 * (iterations = 0, centroids unchanged).  iterations / dists_total (may be NULL) receive this
 * call's totals. */
km_status kmeans_run(km_ctx *ctx, int32_t max_iters, int64_t tol, int32_t *iterations,
                     int64_t *dists_total);

/* Re-derive C_T = per-cluster means of a_T from sums taken in one fixed order (DESIGN.md
 * reading B12; Lloyd's update): each rank sums its rows in its own row
 * order in blocks of 65536 rows (per block and cluster a sequential fp64 sum from 0, then the
 * block sums added from 0 in block order), then the ranks' sums are added.  The iterations keep
 * running sums updated by the moves of each pass (reading B5), whose fp64 rounding depends on
 * the order the moves are applied in; after finalize the centroids are bit-reproducible run to
 * run for the same assignments (world <= 2: independent of NCCL's reduction order).  The
 * centroids of the last pass are kept for the next drift, so iterating further stays sound.
 * Collective when world > 1.  No-op before iteration 1.  kmeans_run calls it. */
km_status kmeans_finalize(km_ctx *ctx);

/* n_local int32 assignments of the last assignment pass, in the caller's row order
 * (reading A9: not re-argmin against the final centroids).  out is host memory unless
 * out_is_device = 1 (device memory on the context device).  KM_ESTATE before iteration 1. */
km_status kmeans_get_assignments(km_ctx *ctx, int32_t *out, int32_t out_is_device);

/* Debug/verification: the n_local fp32 upper bounds u(x) kept by MTI after the last pass, in
 * the caller's row order.  After a pass that used centroids C_used, u(x_i) >= ||x_i - C_used[a_i]||
 * (exact real arithmetic on the fp64 C_used, bound loosened by drift and
 * tightened by U(u)).  out is host memory unless out_is_device = 1.  KM_ESTATE before iteration
 * 1 or with KM_PRUNE_NONE (no bounds are kept). */
km_status kmeans_get_bounds(km_ctx *ctx, float *out, int32_t out_is_device);

/* k x d fp64 current centroids C_T (host memory, caller-owned).  Identical on all ranks. */
km_status kmeans_get_centroids(km_ctx *ctx, double *out_host);

/* Replace the current centroids (k x d fp64 host).  The next iteration computes drift
 * against the centroids the last pass used, so the kept bounds stay sound (lockstep parity). */
km_status kmeans_set_centroids(km_ctx *ctx, const double *centroids_host);

/* Global SSE = sum_i ||x_i - C_T[a_T(i)]||^2 in fp64 (S5; Eq. 1 read as SSE).  Collective
 * when world > 1.  KM_ESTATE before iteration 1. */
km_status kmeans_sse(km_ctx *ctx, double *out);

/* Copy up to cap per-iteration records (oldest first); *count = records available. */
km_status kmeans_get_stats(km_ctx *ctx, km_iter_stats *out, int32_t cap, int32_t *count);

/* k-means++ D^2 seeding (§4.3, Eq. 2).
 * points: n x d fp32 row-major, device memory of `device` (borrowed) or host memory when
 * points_on_host = 1 (copied).  c_1 = row first_index; c_m (m = 2..k) = the row drawn with
 * probability D(x)^2 / sum D^2 using the caller's uniforms[m-2] in [0,1) (k-1 values, host).
 * The draw is exact and reproducible (reading B9): D^2 in fp64 summed in coordinate
 * order; the drawn row is the first row whose exact prefix sum of D^2 exceeds u times the exact
 * total (the sums are kept as 768-bit fixed-point integers, exact for any fp32 data).  Outputs (host, caller-owned): chosen[k] row indices, centroids k x d fp64 (the
 * chosen rows).  Errors: KM_EARG (sizes, NULLs, first_index out of range, uniforms outside
 * [0,1), fewer than k distinct rows), KM_ECUDA, KM_ENOMEM.  stream: cudaStream_t or NULL. */
km_status kmeans_seed_plusplus(int64_t n, int32_t d, int32_t k, const float *points, int32_t points_on_host,
                               int64_t first_index, const double *uniforms, int32_t device, void *stream,
                               int64_t *chosen, double *centroids);

/* Number of kernel launches this context has issued so far (for launch accounting). */
int64_t kmeans_launch_count(const km_ctx *ctx);

/* Bytes of device memory the context holds (points copy, per-row state, bounds, scratch). */
int64_t kmeans_device_bytes(const km_ctx *ctx);

/* Name of the kernel that runs the MTI assignment pass (S2+S3) of this context:
 * "k_walk" (CUDA-core walk engine), "k_mti_tc" (tcgen05 engine), "k_assign" (direct-form lane
 * walk, legacy), "k_assign_dense" (KM_PRUNE_NONE) or "k_ti" (KM_PRUNE_TI).  Static string; NULL ctx -> "". */
const char *kmeans_engine(const km_ctx *ctx);

/* Release all device memory, the internal stream (if created) and the NCCL communicator. */
void kmeans_destroy(km_ctx *ctx);

/* Thread-local message for the last failing call on this thread ("" if none). */
const char *kmeans_last_error(void);

/* Library version string. */
const char *kmeans_version(void);

#ifdef __cplusplus
}
#endif
#endif /* KMEANS_B200_H */
