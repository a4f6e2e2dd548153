// km_kernels.cuh — device-side building blocks and kernel launch interface for the
// MTI-pruned Lloyd's k-means hot path on sm_100a (B200).
//
// Layout in HBM (per rank):
//   X      n x DP fp32 row-major, DP = d padded to {4,8,16,32,64} with zeros, rows
//          physically bucketed by (assigned cluster, survivor-prefix class) after iteration 1
//   a, u   int32[n], fp32[n]   assignment and MTI upper bound, same row order as X
//   perm   int32[n]            caller row index of each stored row
//   Cneg   k x DP fp32         -fp32(C) (negated so x + (-c) is the IEEE x - c), zero padded
//   NL     k x ks uint64       per centroid c: (H[c][c'] as fp32 bits << 32 | c'), ascending,
//                               k-1 neighbours then sentinels (h = NaN, c = 0); ks = k rounded to even
//   f, s   fp32[k]             drift (rounded up) and 1/2 nearest-centroid distance (rounded down)
//   acc    k x (DP+1) fp64     per-cluster sums (DP slots, padded ones stay 0) and count
#pragma once
#ifndef KM_NB_MAX
#define KM_NB_MAX 32768   // re-bucketing: at most this many (cluster, prefix class) buckets (C5: Q = 32)
#endif
#include <cuda_runtime.h>
#include <stdint.h>

namespace km {

constexpr int kWarp = 32;
constexpr unsigned kFull = 0xffffffffu;
constexpr int kAssignThreads = 256;
constexpr int kChunkRows = 256;       // rows a warp claims per work-counter fetch

// assignment kernel modes
enum AssignMode : int {
    MODE_DENSE = 0,          // all k centroids, writes a/u, no reduction (iteration 1)
    MODE_DENSE_REDUCE = 1,   // all k centroids + fused reduction (knori-, t >= 2)
    MODE_MTI_REDUCE = 2,     // MTI clauses 1-3 + fused reduction (knori, t >= 2)
    MODE_REDUCE_ONLY = 3     // reduction of the current a (after the iteration-1 sort)
};

struct AssignParams {
    const float *X;        // n x DP
    int32_t *a;            // n
    float *u;              // n
    int64_t n;
    int32_t d, k;
    const float *Cneg;     // k x DP
    const double *C64;     // k x d master centroids of this pass
    const uint64_t *NL;    // k x ks (k-1 neighbours, then sentinels; + one spare row)
    int32_t ks;            // NL row stride: k rounded up to even
    const float *f;        // k
    const float *s;        // k
    const float *eps;      // device scalar: eps_C (rounded up)
    float g_up, g_dn;      // 1 + gamma (rounded up), 1 - gamma (rounded down)
    int32_t count_changed; // 1: count a_new != a_old
    double *acc;           // partial-sum slabs: nslab x k x (DP+1) (zeroed before launch)
    int32_t nslab;         // CTA b accumulates into slab b % nslab
    unsigned long long *counters;  // [0] changed [1] dists [2] clause1 [3] refined [4] walk warp-steps / TC columns [5] TC fallbacks [6] deferred rows
    int *work;             // dynamic chunk counter (zeroed before launch)
    // tensor-core MTI path (k_mti_tc, km_tc.cu)
    const float *Bop;      // k x nmax x KT: per-cluster B operand blocks (UMMA K-major layout)
    const float4 *Bmeta;   // k x nmax: {H, column centroid bits, |c'|^2 up, prefix max}
    int32_t nmax;          // columns per cluster block (multiple of 16, <= 256)
    int32_t tmem_cols;     // TMEM columns allocated per CTA (power of 2 >= 2 nmax)
    int32_t tile_chunk;    // 128-row tiles claimed per work-counter fetch
    unsigned long long *defer;   // n_alloc: (a << 32 | u_t bits) of rows whose distance count is deferred
    int *dcount;           // ntiles: deferred entries per 128-row tile
    int32_t nmeta;         // Bmeta entries per cluster (power of two >= nmax, NaN padded)
    // CUDA-core walk engine (k_walk, km_walk.cu)
    const float4 *Wblk;    // k x wpad/2 x DP/2: per-cluster candidate pairs, -2 c' interleaved by row
    const float *Wcc;      // k x wpad: |c'|^2 of the candidate rows
    const float2 *Wmeta;   // k x wpad: {prefix max of |c'|^2 (up), centroid bits}
    const float *WH;       // k x whs: H of the candidate rows (NaN past the list)
    int32_t whs;           // WH row stride (power of two >= wpad)
    int32_t wh_smem;       // 1: stage WH in shared memory
    int32_t wpad;          // candidate rows per cluster (>= k, even)
    int32_t wbits;         // key index bits (2^wbits >= wpad)
    // screen engines (k_screen, k_mti_tc<SCREEN>) -> k_resolve: per 32-row group g,
    // qrow[32 g .. 32 g + qcnt[g]) = the rows left undecided
    int *qrow;
    int *qcnt;
    const int16_t *rank;   // k x k: position of c' in c's neighbour list (tensor-screen epilogue)
    // column-chunked tensor-core screen (k_tcc, km_tcc.cu)
    const float *Bc;       // k x tcc_nch x (128 x (2 DP + 8)): B operand chunks (UMMA K-major)
    const float *Mh;       // k x hrow: H of the list, skewed (entry j at j + j / 32), NaN padded
    const float *Mx;       // k x nmeta: prefix max of |c'|^2 (up)
    int32_t tcc_nch;       // chunks per cluster list
};

struct PrepParams {
    const double *C;       // k x d (centroids of the coming pass)
    const double *Cprev;   // k x d (centroids of the previous pass)
    int32_t k, d, DP, sortN, ks;
    float *Cneg;           // k x DP
    float *f, *s;          // k
    uint64_t *NL;          // k x ks
    unsigned *eps_bits;    // fp32 bits of eps_C (atomicMax; zeroed before launch)
};

struct SortParams {
    const float *X; const int32_t *a; const float *u; const int32_t *perm;
    float *X2; int32_t *a2; float *u2; int32_t *perm2;
    uint32_t *keys;        // n bucket ids
    uint32_t *hist;        // NB x ntiles (counts, then exclusive offsets)
    uint32_t *totals;      // NB
    uint32_t *base;        // NB
    const uint64_t *NL; const float *s;
    uint32_t *lohist;      // k+1 counts of the prefix length p (quantile classes, k <= kQuantK)
    int32_t *qmap;         // k+1: p -> class (0 for p = 0, then Q-1 classes of equal population)
    int64_t n;
    int32_t ks;
    int32_t k, DP, Q, NB, ntiles, tile_rows;
};
constexpr int kQuantK = 8192;
constexpr int64_t kExactBlock = 65536;   // rows per block of the exact-order sums (reading B12)   // quantile prefix classes for k <= this (p packed in 13 bits)

// ---- launchers (km_kernels.cu) ----------------------------------------------------------
cudaError_t launch_prep(const PrepParams &p, cudaStream_t st);
cudaError_t launch_assign(int mode, int DP, bool csmem, const AssignParams &p, int grid,
                          cudaStream_t st);
int assign_grid(int mode, int DP, bool csmem, int k, int num_sms);
size_t assign_smem(int DP, bool csmem, int k);
cudaError_t launch_partials_reduce(const double *part, int parts, int64_t elems, double *acc,
                                  cudaStream_t st);
bool tc_supported(int DP);
int tc_kt_host(int DP);
size_t tc_plan(int DP, bool csmem, int k, int nmax, int num_sms, int *grid, int *tmem_cols);
cudaError_t launch_mti_tc(int DP, bool csmem, const AssignParams &p, int grid, bool screen, cudaStream_t st);
cudaError_t launch_prep_tc(const double *C, const uint64_t *NL, int k, int d, int DP, int ks, int nmax,
                           float *Bop, float4 *Bmeta, int16_t *rank, cudaStream_t st);
cudaError_t launch_resolve(int DP, bool csmem, const AssignParams &p, int g_resolve, cudaStream_t st);
cudaError_t launch_tcc(int DP, bool csmem, const AssignParams &p, int num_sms, const void *tmap, cudaStream_t st);
int tcc_make_tmap(void *out, const float *X, int64_t n_alloc, int DP);
cudaError_t launch_prep_tcc(const double *C, const uint64_t *NL, int k, int d, int DP, int ks, int nch, int nmeta,
                            float *Bc, float *Mh, float *Mx, int16_t *rank, cudaStream_t st);
int tcc_hrow_host(int k);
size_t tcc_smem(int DP, bool csmem, int k);
int tcc_nch_host(int k);
int tcc_ka_host(int DP);
int tcc_nmeta_host(int k);
int resolve_grid(int DP, bool csmem, int k, int num_sms);
cudaError_t launch_mti_count(const unsigned long long *defer, const int *dcount, int64_t ntiles,
                             unsigned long long *counters, const uint64_t *NL, int ks, int k, int num_sms,
                             cudaStream_t st);
int tc_nmeta_host(int nmax);
bool walk_supported(int DP);
cudaError_t launch_walk(int DP, bool csmem, const AssignParams &p, int grid, bool skip1, cudaStream_t st);
int walk_grid(int DP, bool csmem, int k, int kp, bool whs, int num_sms);
void screen_grids(int DP, bool csmem, int k, int whs, bool hs, int num_sms, int *g_screen, int *g_resolve);
cudaError_t launch_screen(int DP, bool csmem, const AssignParams &p, int g_screen, int g_resolve, bool skip1,
                          int *qrow, int *qcnt, int64_t n_alloc, cudaStream_t st);
cudaError_t launch_prep_walk(const double *C, const uint64_t *NL, int k, int d, int DP, int ks, int kp, int whs,
                             float4 *Wblk, float *Wcc, float2 *Wmeta, float *WH, cudaStream_t st);
int ti_grid(int DP, bool csmem, int k, int num_sms);
cudaError_t launch_ti(int DP, bool csmem, bool first, const AssignParams &p, float *L, const float *Hm, int grid,
                      cudaStream_t st);
cudaError_t launch_prep_ti(const uint64_t *NL, int k, int ks, float *Hm, cudaStream_t st);
cudaError_t launch_update(const double *acc, double *S, int delta, double *C, double *Cprev, int k, int d,
                          int DP, int *empty, int spherical, cudaStream_t st);
cudaError_t launch_sort(const SortParams &p, cudaStream_t st, int *launches);
cudaError_t launch_sse(const float *X, const int32_t *a, const double *C, int64_t n, int d,
                       int DP, double *out, cudaStream_t st);
int64_t exact_blocks(int64_t n);
cudaError_t launch_exact_sums(const float *X, const int32_t *a, const int32_t *perm, int64_t n, int DP, int k,
                              int32_t *inv, int32_t *ac, double *P, double *acc, bool identity, cudaStream_t st,
                              int *launches);
cudaError_t launch_unpermute(const int32_t *a, const int32_t *perm, int64_t n, int32_t *out,
                             cudaStream_t st);
cudaError_t launch_iota(int32_t *perm, int64_t n, cudaStream_t st);
cudaError_t launch_pad_rows(const float *X, float *Xp, int64_t n, int d, int DP, cudaStream_t st);
cudaError_t launch_check_finite(const float *X, int64_t count, int *flag, cudaStream_t st);
cudaError_t launch_normalize_rows(float *X, int64_t n, int d, int DP, int *flag, cudaStream_t st);
size_t seed_scratch_bytes(int64_t n);
cudaError_t seed_plusplus(const float *X, int64_t n, int d, int ldx, int k, int64_t first,
                          const double *u, double *D2, void *scratch, float *crow, int64_t *dsel,
                          int64_t *chosen, cudaStream_t st);

}  // namespace km
