// km_kernels.cu — sm_100a kernels for MTI-pruned Lloyd's k-means.
//
//   k_prep        S1: centroid geometry + drift from the fp64 master centroids
//                 (PAPER.md:990-991 drift f; PAPER.md:1036-1040 clause-1 radius; reading A1/A2)
//   k_assign      S0/S2(+S3): dense or MTI assignment with exact-mode fp64 refinement, fused
//                 with the per-cluster fp64 reduction
//   k_update      S4: centroid update, empty cluster keeps its centroid (reading A10)
//   k_sort_*      re-bucketing of rows by (cluster, survivor-prefix class): B200-specific
//                 layout step so warps walk one cluster's neighbour list with broadcast reads
//   k_sse         S5: SSE (Eq. 1 as SSE; reading A15)
#include "km_kernels.cuh"
#include "km_device.cuh"

#include <math.h>

#include <algorithm>

namespace km {

// ---------------------------------------------------------------------------------------
// k_assign: one lane = one row; a warp claims kChunkRows consecutive rows at a time.
template <int DP, int MODE, bool CSMEM>
__global__ void __launch_bounds__(kAssignThreads)
k_assign(AssignParams p)
{
    constexpr bool PRUNE = MODE == MODE_MTI_REDUCE;
    constexpr bool DENSE = MODE == MODE_DENSE || MODE == MODE_DENSE_REDUCE;
    constexpr bool ASSIGN = MODE != MODE_REDUCE_ONLY;
    constexpr bool REDUCE = MODE != MODE_DENSE;

    extern __shared__ __align__(16) float smem[];
    const int k = p.k;
    float *sC = smem;                               // k*DP (CSMEM)
    float *sF = smem + (CSMEM ? k * DP : 0);        // k
    float *sS = sF + k;                             // k
    if (ASSIGN) {
        if (CSMEM) {
            const float4 *src = reinterpret_cast<const float4 *>(p.Cneg);
            float4 *dst = reinterpret_cast<float4 *>(sC);
            for (int i = threadIdx.x; i < k * DP / 4; i += blockDim.x) dst[i] = src[i];
        }
        if (PRUNE)
            for (int i = threadIdx.x; i < k; i += blockDim.x) { sF[i] = p.f[i]; sS[i] = p.s[i]; }
    }
    __syncthreads();
    CRow<CSMEM> Cn;
    if constexpr (CSMEM) {
        uint32_t b = (uint32_t)__cvta_generic_to_shared(sC);
        asm volatile("mov.u32 %0, %0;" : "+r"(b));   // keep in a register (no re-materialisation)
        Cn.base = b;
    }
    else Cn.base = p.Cneg;
    // this CTA's private partial-sum slab: fp64 REDs from different CTAs never contend
    double *acc = p.acc + (int64_t)(blockIdx.x % p.nslab) * k * (DP + 1);
    const float eps = ASSIGN ? *p.eps : 0.f;
    const int lane = threadIdx.x & (kWarp - 1);
    const int64_t n = p.n;

    RunAcc<DP> ra;
    ra.clear();
    unsigned long long c_changed = 0, c_dists = 0, c_clause1 = 0, c_refined = 0;
    unsigned steps = 0;
    const int ks = p.ks;                        // NL row stride (even, >= k)

    // Row stream of this warp: chunks of kChunkRows rows claimed from a global counter (one
    // chunk ahead), batches of 32 rows (one per lane); the next batch's x, a, u are loaded
    // before the current batch is processed, so HBM latency overlaps the distance work.
    constexpr int kBatches = kChunkRows / kWarp;
    auto claim = [&]() -> int64_t {
        int c = 0;
        if (lane == 0) c = atomicAdd(p.work, 1);
        return (int64_t)__shfl_sync(kFull, c, 0) * kChunkRows;
    };
    int64_t chunk_row = claim(), ahead_row = claim();
    int b = 0;
    float nx[DP];
    int na = 0;
    float nu = 0.f;
    auto load = [&](int64_t row) {
        const bool v = row < n;
        const float4 *xr = reinterpret_cast<const float4 *>(p.X + (v ? row : 0) * DP);
#pragma unroll
        for (int j = 0; j < DP / 4; ++j) {
            float4 t = v ? __ldg(xr + j) : make_float4(0.f, 0.f, 0.f, 0.f);
            nx[4 * j] = t.x; nx[4 * j + 1] = t.y; nx[4 * j + 2] = t.z; nx[4 * j + 3] = t.w;
        }
        na = v ? __ldg(p.a + row) : 0;
        nu = (v && PRUNE) ? __ldg(p.u + row) : 0.f;
    };
    load(chunk_row + lane);

    while (chunk_row < n) {
        const int64_t row = chunk_row + b * kWarp + lane;
        const bool valid = row < n;
        float x[DP];
#pragma unroll
        for (int j = 0; j < DP; ++j) x[j] = nx[j];
        const int aold = na;
        const float uold = nu;
        // advance the stream and prefetch the next batch
        if (++b == kBatches || chunk_row + b * kWarp >= n) {
            b = 0;
            chunk_row = ahead_row;
            ahead_row = chunk_row < n ? claim() : ahead_row;
        }
        if (chunk_row < n) load(chunk_row + b * kWarp + lane);

        int anew = aold;
        if (ASSIGN) {
            float unew = 0.f;
            bool active = valid;
            if (PRUNE) {
                const float uu = valid ? __fadd_ru(uold, sF[aold]) : 0.f;  // u += f(a)
                const bool c1 = valid && uu <= sS[aold];                   // clause 1
                c_clause1 += c1;
                active = valid && !c1;
                unew = uu;
            }
            if (__any_sync(kFull, active)) {
                float bq = INFINITY, q2 = INFINITY, ut = 0.f;
                int bc = aold, ns = 0;
                if (DENSE) {
#pragma unroll 4
                    for (int c = 0; c < k; ++c) {
                        const float q = dist2<DP, CSMEM>(x, Cn, c);
                        q2 = fminf(q2, fmaxf(q, bq));
                        bc = q < bq ? c : bc;
                        bq = fminf(q, bq);
                    }
                    ns = k;
                } else {
                    // Every lane walks its own cluster's neighbour list (ascending H) in
                    // lockstep, two candidates per step; rows are bucketed by cluster, so
                    // lanes mostly share the list and centroid reads are broadcasts.  Steps =
                    // the longest walk in the warp, whatever the mix of clusters.
                    if (active) {                           // tighten: U(u) = d(x, C[a])
                        bq = dist2<DP, CSMEM>(x, Cn, aold);
                        bc = aold;
                        ut = upper_d(bq, p.g_up, eps);
                        ns = 1;
                    }
                    // NL rows (stride ks, even) end with sentinels (h = NaN, c = 0) and the
                    // array has a spare row, so pair loads never leave the allocation and
                    // every key's c is a valid centroid index, even past a lane's own walk.
                    const uint64_t *nl = p.NL + (int64_t)aold * ks;
                    bool walking = active;
                    ulonglong2 kp = __ldg(reinterpret_cast<const ulonglong2 *>(nl));
                    for (int j = 0;; j += 2) {
                        const bool w0 = walking && key_h(kp.x) < ut;   // clauses 2/3
                        const bool w1 = w0 && key_h(kp.y) < ut;
                        if (!__any_sync(kFull, w0)) break;
                        steps += 2;
                        const ulonglong2 np = __ldg(reinterpret_cast<const ulonglong2 *>(nl + j + 2));
                        const int c0 = key_c(kp.x), c1 = key_c(kp.y);
                        float q0 = dist2<DP, CSMEM>(x, Cn, c0);
                        float q1 = dist2<DP, CSMEM>(x, Cn, c1);
                        q0 = w0 ? q0 : INFINITY;
                        q1 = w1 ? q1 : INFINITY;
                        ns += (int)w0 + (int)w1;
                        // fp32 ties are resolved later: equal q makes q2 == bq -> refinement
                        q2 = fminf(q2, fmaxf(q0, bq));
                        bc = q0 < bq ? c0 : bc;
                        bq = fminf(q0, bq);
                        q2 = fminf(q2, fmaxf(q1, bq));
                        bc = q1 < bq ? c1 : bc;
                        bq = fminf(q1, bq);
                        walking = w1;
                        kp = np;
                    }
                }
                if (active) {
                    const float ub = upper_d(bq, p.g_up, eps);
                    const bool amb = q2 < INFINITY && lower_d(q2, p.g_dn, eps) <= ub;
                    if (amb) {
                        anew = refine64(p.X + row * DP, p.d, p.C64, k, aold,
                                        DENSE ? nullptr : p.NL + (int64_t)aold * ks, ut, &unew);
                        ++c_refined;
                    } else {
                        anew = bc;
                        unew = ub;
                    }
                    c_dists += (unsigned long long)ns;
                }
            }
            if (valid) {
                p.a[row] = anew;
                // knori- (no pruning after iteration 1) keeps no bound: a read + write only
                if (MODE != MODE_DENSE_REDUCE) p.u[row] = unew;
                if (p.count_changed) c_changed += (anew != aold);
            }
        }
        if (REDUCE) reduce_batch<DP>(ra, x, anew, valid, acc, p.d, lane);
    }
    if (REDUCE) ra.flush(acc, p.d, lane);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        c_changed += __shfl_xor_sync(kFull, c_changed, o);
        c_dists += __shfl_xor_sync(kFull, c_dists, o);
        c_clause1 += __shfl_xor_sync(kFull, c_clause1, o);
        c_refined += __shfl_xor_sync(kFull, c_refined, o);
    }
    if (lane == 0 && ASSIGN) {
        if (c_changed) atomicAdd(p.counters + 0, c_changed);
        if (c_dists) atomicAdd(p.counters + 1, c_dists);
        if (c_clause1) atomicAdd(p.counters + 2, c_clause1);
        if (c_refined) atomicAdd(p.counters + 3, c_refined);
        if (steps) atomicAdd(p.counters + 4, (unsigned long long)steps);   // warp-uniform count
    }
}

size_t assign_smem(int DP, bool csmem, int k)
{
    return (size_t)((csmem ? k * DP : 0) + 2 * k) * sizeof(float);
}

template <int DP, int MODE, bool CSMEM>
static cudaError_t launch_assign_t(const AssignParams &p, int grid, cudaStream_t st)
{
    const size_t sm = assign_smem(DP, CSMEM, p.k);
    if (sm > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k_assign<DP, MODE, CSMEM>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e != cudaSuccess) return e;
    }
    k_assign<DP, MODE, CSMEM><<<grid, kAssignThreads, sm, st>>>(p);
    return cudaGetLastError();
}

template <int DP, int MODE, bool CSMEM>
static int grid_t(int k, int num_sms)
{
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_assign<DP, MODE, CSMEM>, kAssignThreads,
                                                  assign_smem(DP, CSMEM, k));
    if (per_sm < 1) per_sm = 1;
    return per_sm * num_sms;
}

#define KM_DISPATCH_DP(DPV, FN, ...)                                   \
    switch (DPV) {                                                     \
    case 4: return FN<4, __VA_ARGS__>;                                 \
    case 8: return FN<8, __VA_ARGS__>;                                 \
    case 16: return FN<16, __VA_ARGS__>;                               \
    case 32: return FN<32, __VA_ARGS__>;                               \
    case 64: return FN<64, __VA_ARGS__>;                               \
    default: return nullptr;                                           \
    }

typedef cudaError_t (*assign_fn)(const AssignParams &, int, cudaStream_t);
typedef int (*grid_fn)(int, int);

template <int MODE, bool CSMEM>
static assign_fn pick_assign(int DP) { KM_DISPATCH_DP(DP, launch_assign_t, MODE, CSMEM) }
template <int MODE, bool CSMEM>
static grid_fn pick_grid(int DP) { KM_DISPATCH_DP(DP, grid_t, MODE, CSMEM) }

static assign_fn assign_table(int mode, int DP, bool cs)
{
    switch (mode * 2 + (cs ? 1 : 0)) {
    case 0: return pick_assign<MODE_DENSE, false>(DP);
    case 1: return pick_assign<MODE_DENSE, true>(DP);
    case 2: return pick_assign<MODE_DENSE_REDUCE, false>(DP);
    case 3: return pick_assign<MODE_DENSE_REDUCE, true>(DP);
    case 4: return pick_assign<MODE_MTI_REDUCE, false>(DP);
    case 5: return pick_assign<MODE_MTI_REDUCE, true>(DP);
    case 6: return pick_assign<MODE_REDUCE_ONLY, false>(DP);
    case 7: return pick_assign<MODE_REDUCE_ONLY, true>(DP);
    }
    return nullptr;
}

static grid_fn grid_table(int mode, int DP, bool cs)
{
    switch (mode * 2 + (cs ? 1 : 0)) {
    case 0: return pick_grid<MODE_DENSE, false>(DP);
    case 1: return pick_grid<MODE_DENSE, true>(DP);
    case 2: return pick_grid<MODE_DENSE_REDUCE, false>(DP);
    case 3: return pick_grid<MODE_DENSE_REDUCE, true>(DP);
    case 4: return pick_grid<MODE_MTI_REDUCE, false>(DP);
    case 5: return pick_grid<MODE_MTI_REDUCE, true>(DP);
    case 6: return pick_grid<MODE_REDUCE_ONLY, false>(DP);
    case 7: return pick_grid<MODE_REDUCE_ONLY, true>(DP);
    }
    return nullptr;
}

cudaError_t launch_assign(int mode, int DP, bool csmem, const AssignParams &p, int grid,
                          cudaStream_t st)
{
    assign_fn fn = assign_table(mode, DP, csmem);
    if (!fn) return cudaErrorInvalidValue;
    return fn(p, grid, st);
}

int assign_grid(int mode, int DP, bool csmem, int k, int num_sms)
{
    grid_fn fn = grid_table(mode, DP, csmem);
    return fn ? fn(k, num_sms) : num_sms;
}

// ---------------------------------------------------------------------------------------
// S1: per centroid c (one CTA): H[c][.] = 1/2 ||C[c] - C[.]|| rounded down to fp32, sorted
// ascending with ties by index -> NL[c]; s[c] = NL[c][0].h (k = 1: +inf); f[c] = drift
// rounded up; Cneg[c] = -fp32(C[c]); eps_C = max_c ||C[c] - fp32(C[c])|| rounded up.
// The fp64 values carry relative error <= (d+2) 2^-53 < 1e-14, absorbed by the 1 -/+ 1e-14
// factors before directed rounding to fp32.
__global__ void k_prep(PrepParams p)
{
    extern __shared__ uint64_t keys[];
    const int c = blockIdx.x, k = p.k, d = p.d, N = p.sortN;
    const double *Cc = p.C + (int64_t)c * d;
    for (int c2 = threadIdx.x; c2 < N; c2 += blockDim.x) {
        uint64_t key = ~0ull;
        if (c2 < k && c2 != c) {
            const double *C2 = p.C + (int64_t)c2 * d;
            double s = 0.0;
            for (int j = 0; j < d; ++j) {
                double t = Cc[j] - C2[j];
                s = fma(t, t, s);
            }
            float h = __double2float_rd(0.5 * sqrt(s) * (1.0 - 1e-14));
            key = ((uint64_t)__float_as_uint(h) << 32) | (uint32_t)c2;
        }
        keys[c2] = key;
    }
    for (int j = threadIdx.x; j < p.DP; j += blockDim.x)
        p.Cneg[(int64_t)c * p.DP + j] = j < d ? -(float)Cc[j] : 0.f;
    if (threadIdx.x == 0) {
        double se = 0.0, sf = 0.0;
        const double *Cp = p.Cprev + (int64_t)c * d;
        for (int j = 0; j < d; ++j) {
            double e = Cc[j] - (double)(float)Cc[j];
            se = fma(e, e, se);
            double t = Cc[j] - Cp[j];
            sf = fma(t, t, sf);
        }
        float eps = __double2float_ru(sqrt(se) * (1.0 + 1e-14));
        atomicMax(p.eps_bits, __float_as_uint(eps));
        p.f[c] = __double2float_ru(sqrt(sf) * (1.0 + 1e-14));
    }
    // bitonic sort (ascending) of N = 2^m keys
    for (int size = 2; size <= N; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            __syncthreads();
            for (int i = threadIdx.x; i < N / 2; i += blockDim.x) {
                int lo = (i / stride) * 2 * stride + (i % stride);
                int hi = lo + stride;
                bool asc = (lo & size) == 0;
                uint64_t A = keys[lo], B = keys[hi];
                if ((A > B) == asc) { keys[lo] = B; keys[hi] = A; }
            }
        }
    }
    __syncthreads();
    uint64_t *nl = p.NL + (int64_t)c * p.ks;     // k - 1 neighbours, then sentinels (h = NaN, c = 0)
    for (int j = threadIdx.x; j < p.ks; j += blockDim.x) nl[j] = j < k - 1 ? keys[j] : kSentinel;
    if (threadIdx.x == 0) p.s[c] = k > 1 ? __uint_as_float((uint32_t)(keys[0] >> 32)) : INFINITY;
}

cudaError_t launch_prep(const PrepParams &p, cudaStream_t st)
{
    size_t sm = (size_t)p.sortN * sizeof(uint64_t);
    k_prep<<<p.k, 256, sm, st>>>(p);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// S3 final step: acc[e] = sum over CTAs g (in order) of part[g][e]
__global__ void __launch_bounds__(1024) k_partials_reduce(const double *part, int parts, int64_t elems, double *acc)
{
    // block = 32 elements x 32 warps; warp w sums parts w, w+32, ... then a fixed-order tree
    __shared__ double red[32][33];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t e = (int64_t)blockIdx.x * 32 + lane;
    double s = 0.0;
    if (e < elems)
        for (int g = w; g < parts; g += 32) s += part[(int64_t)g * elems + e];
    red[w][lane] = s;
    __syncthreads();
    if (w == 0) {
        double t = 0.0;
        for (int i = 0; i < 32; ++i) t += red[i][lane];
        if (e < elems) acc[e] = t;
    }
}

cudaError_t launch_partials_reduce(const double *part, int parts, int64_t elems, double *acc,
                                   cudaStream_t st)
{
    k_partials_reduce<<<(unsigned)((elems + 31) / 32), 1024, 0, st>>>(part, parts, elems, acc);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// S4: C_new[c] = sums[c] / count[c] (IEEE fp64 division), or C_old[c] when empty (A10).
// S holds the running per-cluster sums | count: delta = 0 -> S = acc (full reduction of this
// pass), delta = 1 -> S += acc (acc holds only the moves of this pass),
// delta = 2 -> S = acc with C_prev kept (kmeans_finalize: C_T re-derived from exact-order sums of
// the same assignment; C_prev stays the centroids the last pass used, so the drift stays sound).
__global__ void k_update(const double *acc, double *S, int delta, double *C, double *Cprev, int k, int d,
                         int DP, int *empty, int spherical)
{
    const int c = blockIdx.x * blockDim.x + threadIdx.x;     // one thread per cluster
    if (c >= k) return;
    double *Sc = S + (int64_t)c * (DP + 1);
    const double *ac = acc + (int64_t)c * (DP + 1);
    const bool add = delta == 1, keep_prev = delta == 2;
    const double cnt = add ? Sc[DP] + ac[DP] : ac[DP];
    Sc[DP] = cnt;
    if (!(cnt > 0.5)) atomicAdd(empty, 1);
    for (int j = 0; j < d; ++j) {
        const double v = add ? Sc[j] + ac[j] : ac[j];
        Sc[j] = v;
        const int64_t ci = (int64_t)c * d + j;
        const double old = C[ci];
        if (!keep_prev) Cprev[ci] = old;
        C[ci] = cnt > 0.5 ? v / cnt : old;
    }
    if (spherical && cnt > 0.5) {
        // sk-means update: the mean re-normalised to unit length, in the oracle's
        // order (sequential fp64 sum of squares, correctly rounded sqrt and divisions); a zero mean
        // keeps the previous centroid
        double *Cc = C + (int64_t)c * d;
        double ss = 0.0;
        for (int j = 0; j < d; ++j) ss = __dadd_rn(ss, __dmul_rn(Cc[j], Cc[j]));
        if (ss > 0.0) {
            const double nrm = __dsqrt_rn(ss);
            for (int j = 0; j < d; ++j) Cc[j] = __ddiv_rn(Cc[j], nrm);
        } else {
            for (int j = 0; j < d; ++j) Cc[j] = Cprev[(int64_t)c * d + j];
        }
    }
}

cudaError_t launch_update(const double *acc, double *S, int delta, double *C, double *Cprev, int k, int d,
                          int DP, int *empty, int spherical, cudaStream_t st)
{
    k_update<<<(unsigned)((k + 127) / 128), 128, 0, st>>>(acc, S, delta, C, Cprev, k, d, DP, empty, spherical);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// Exact-order cluster sums (reading B12).  The rows are summed in the caller's row
// order, in blocks of kExactBlock rows: per block and cluster a sequential fp64 sum from 0 over
// the block's rows of that cluster in row order, then per cluster the block sums added from 0 in
// block order — one fixed order, independent of the physical (re-bucketed) row order, of the
// grid and of timing, so C_T is bit-reproducible run to run (and, being the order the oracle's
// reduction is defined with, bit-identical to the oracle's when the assignments agree).
__global__ void k_unpermute(const int32_t *a, const int32_t *perm, int64_t n, int32_t *out);
constexpr int kExactThreads = 128;     // clusters per CTA
constexpr int kExactTile = 4096;       // assignments staged in shared memory per step

__global__ void k_inv_perm(const int32_t *perm, int64_t n, int32_t *inv)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        inv[perm[i]] = (int32_t)i;
}

// CTA (block b, clusters [128 y, 128 y + 128)): every thread scans the block's caller-order
// assignments (broadcast from shared memory) and adds the rows of its own cluster in row order.
template <int DP>
__global__ void __launch_bounds__(kExactThreads) k_exact_block_sums(const float *X, const int32_t *inv,
                                                                   const int32_t *ac, int64_t n, int k,
                                                                   double *P)
{
    __shared__ __align__(16) int32_t sa[kExactTile];
    const int64_t r0 = (int64_t)blockIdx.x * kExactBlock;
    const int64_t r1 = r0 + kExactBlock < n ? r0 + kExactBlock : n;
    const int c = blockIdx.y * kExactThreads + threadIdx.x;
    double s[DP];
#pragma unroll
    for (int j = 0; j < DP; ++j) s[j] = 0.0;
    double cnt = 0.0;
    for (int64_t t0 = r0; t0 < r1; t0 += kExactTile) {
        const int m = (int)(r1 - t0 < kExactTile ? r1 - t0 : kExactTile);
        __syncthreads();
        for (int i = threadIdx.x; i < m; i += kExactThreads) sa[i] = ac[t0 + i];
        __syncthreads();
        for (int i = 0; i < m; ++i) {
            if (sa[i] != c) continue;
            const float4 *xr = reinterpret_cast<const float4 *>(X + (int64_t)inv[t0 + i] * DP);
#pragma unroll
            for (int j = 0; j < DP / 4; ++j) {
                const float4 v = __ldg(xr + j);
                s[4 * j] = __dadd_rn(s[4 * j], (double)v.x);
                s[4 * j + 1] = __dadd_rn(s[4 * j + 1], (double)v.y);
                s[4 * j + 2] = __dadd_rn(s[4 * j + 2], (double)v.z);
                s[4 * j + 3] = __dadd_rn(s[4 * j + 3], (double)v.w);
            }
            cnt += 1.0;
        }
    }
    if (c < k) {
        double *pb = P + ((int64_t)blockIdx.x * k + c) * (DP + 1);
#pragma unroll
        for (int j = 0; j < DP; ++j) pb[j] = s[j];
        pb[DP] = cnt;
    }
}

// The same sums as k_exact_block_sums, one CTA per 64 Ki-row block (k <= kExactListK), in four
// sub-blocks of 16 Ki rows taken in row order.  Per sub-block: a stable counting sort of its rows
// by cluster in shared memory (kExactSortWarps warps, each over a contiguous eighth: per-warp
// counts, an exclusive scan in (cluster, warp) order, then each warp places its rows in row
// order), so every cluster's rows form one list in row order; then one thread per (cluster,
// coordinate) continues its sequential fp64 sum (kept in P between sub-blocks) over its list.
// Bit-identical to k_exact_block_sums (the same additions in the same order), without every
// thread scanning all 65536 assignments of the block.  inv == nullptr: caller order = stored order.
constexpr int kExactListK = 1024;
constexpr int kExactSortWarps = 8;
constexpr int kExactListThreads = 512;
constexpr int kExactSub = 16384;

__host__ __device__ constexpr size_t exact_list_smem(int k)
{
    return (size_t)kExactSub * sizeof(uint16_t) + (size_t)(kExactSortWarps + 2) * k * sizeof(int) + 32 * sizeof(int);
}

template <int DP>
__global__ void __launch_bounds__(kExactListThreads) k_exact_list_sums(const float *X, const int32_t *inv,
                                                                      const int32_t *ac, int64_t n, int k,
                                                                      double *P)
{
    extern __shared__ __align__(16) uint8_t esm[];
    uint16_t *list = reinterpret_cast<uint16_t *>(esm);                       // kExactSub row offsets
    int *cnt = reinterpret_cast<int *>(esm + kExactSub * sizeof(uint16_t));    // [warp][cluster] -> offsets
    int *cbase = cnt + kExactSortWarps * k;                                     // cluster list start
    int *ctot = cbase + k;                                                      // cluster row count
    int *wsum = ctot + k;                                                       // scan scratch (32 ints)
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int nw = (int)(blockDim.x >> 5);
    constexpr int kSpan = kExactSub / kExactSortWarps;      // rows per sort warp
    constexpr int U = 8;                                    // assignment loads in flight per lane
    for (int sub = 0; sub < (int)(kExactBlock / kExactSub); ++sub) {
        const int64_t r0 = (int64_t)blockIdx.x * kExactBlock + (int64_t)sub * kExactSub;
        if (r0 >= n) break;
        const int m = (int)(n - r0 < kExactSub ? n - r0 : kExactSub);
        for (int i = tid; i < kExactSortWarps * k; i += blockDim.x) cnt[i] = 0;
        __syncthreads();
        const int w0 = w * kSpan, w1 = min(m, w0 + kSpan);
        if (w < kExactSortWarps) {                       // per-warp counts
            int *cw = cnt + w * k;
            for (int b = w0; b < w1; b += 32 * U) {
                int cv[U];
#pragma unroll
                for (int u = 0; u < U; ++u) { const int i = b + 32 * u + lane; cv[u] = i < w1 ? ac[r0 + i] : -1; }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const unsigned g = __match_any_sync(kFull, cv[u]);
                    if (cv[u] >= 0 && lane == __ffs(g) - 1) cw[cv[u]] += __popc(g);
                    __syncwarp();
                }
            }
        }
        __syncthreads();
        // cluster totals and their exclusive scan (cluster order), then per-warp offsets
        int run = 0;
        for (int c0 = 0; c0 < k; c0 += blockDim.x) {
            const int c = c0 + tid;
            int t = 0;
            if (c < k)
                for (int ww = 0; ww < kExactSortWarps; ++ww) t += cnt[ww * k + c];
            int incl = t;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(kFull, incl, o);
                if (lane >= o) incl += v;
            }
            if (lane == 31) wsum[w] = incl;
            __syncthreads();
            int wpre = 0, tot = 0;
            for (int ww = 0; ww < nw; ++ww) { wpre += ww < w ? wsum[ww] : 0; tot += wsum[ww]; }
            if (c < k) {
                const int base = run + wpre + incl - t;
                cbase[c] = base;
                ctot[c] = t;
                int o = base;
                for (int ww = 0; ww < kExactSortWarps; ++ww) {
                    const int v = cnt[ww * k + c];
                    cnt[ww * k + c] = o;
                    o += v;
                }
            }
            run += tot;
            __syncthreads();
        }
        if (w < kExactSortWarps) {                       // stable placement, row order per warp
            int *cw = cnt + w * k;
            for (int b = w0; b < w1; b += 32 * U) {
                int cv[U];
#pragma unroll
                for (int u = 0; u < U; ++u) { const int i = b + 32 * u + lane; cv[u] = i < w1 ? ac[r0 + i] : -1; }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int c = cv[u];
                    const unsigned g = __match_any_sync(kFull, c);
                    if (c >= 0) list[cw[c] + __popc(g & ((1u << lane) - 1u))] = (uint16_t)(b + 32 * u + lane);
                    __syncwarp();
                    if (c >= 0 && lane == __ffs(g) - 1) cw[c] += __popc(g);
                    __syncwarp();
                }
            }
        }
        __syncthreads();
        // sequential fp64 sums, one thread per (cluster, coordinate) (+ the count), continued
        // from the previous sub-block's value in P
        for (int item = tid; item < k * (DP + 1); item += blockDim.x) {
            const int c = item / (DP + 1), j = item % (DP + 1);
            double *pb = P + ((int64_t)blockIdx.x * k + c) * (DP + 1);
            const int t0 = cbase[c], t1 = t0 + ctot[c];
            if (j == DP) { pb[DP] = (sub ? pb[DP] : 0.0) + (double)(t1 - t0); continue; }
            double s = sub ? pb[j] : 0.0;
            int t = t0;
            for (; t + U <= t1; t += U) {                // U loads in flight, adds in row order
                float v[U];
#pragma unroll
                for (int q = 0; q < U; ++q) {
                    const int64_t row = r0 + list[t + q];
                    v[q] = __ldg(X + (int64_t)(inv ? inv[row] : row) * DP + j);
                }
#pragma unroll
                for (int q = 0; q < U; ++q) s = __dadd_rn(s, (double)v[q]);
            }
            for (; t < t1; ++t) {
                const int64_t row = r0 + list[t];
                s = __dadd_rn(s, (double)__ldg(X + (int64_t)(inv ? inv[row] : row) * DP + j));
            }
            pb[j] = s;
        }
        __syncthreads();
    }
}

// acc[c][j] = ((0 + P_0[c][j]) + P_1[c][j]) + ... in block order
__global__ void k_exact_merge(const double *P, int64_t nblk, int64_t elems, double *acc)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= elems) return;
    double s = 0.0;
    for (int64_t b = 0; b < nblk; ++b) s = __dadd_rn(s, P[b * elems + t]);
    acc[t] = s;
}

int64_t exact_blocks(int64_t n) { return (n + kExactBlock - 1) / kExactBlock; }

template <int DP>
static cudaError_t launch_exact_list(const float *X, const int32_t *inv, const int32_t *ac, int64_t n, int k,
                                     double *P, cudaStream_t st)
{
    const size_t sm = exact_list_smem(k);
    cudaError_t e = cudaFuncSetAttribute(k_exact_list_sums<DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    k_exact_list_sums<DP><<<(unsigned)exact_blocks(n), kExactListThreads, sm, st>>>(X, inv, ac, n, k, P);
    return cudaGetLastError();
}

// identity: the stored rows are in caller order (perm = iota, before the first re-bucketing), so
// the assignments and rows are read in place
cudaError_t launch_exact_sums(const float *X, const int32_t *a, const int32_t *perm, int64_t n, int DP, int k,
                              int32_t *inv, int32_t *ac, double *P, double *acc, bool identity, cudaStream_t st,
                              int *launches)
{
    const unsigned g = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16);
    if (k > kExactListK) identity = false;   // the scan kernel reads through inv
    if (identity) {
        inv = nullptr;
        ac = const_cast<int32_t *>(a);
    } else {
        k_inv_perm<<<g, 256, 0, st>>>(perm, n, inv);
        k_unpermute<<<g, 256, 0, st>>>(a, perm, n, ac);
        *launches += 2;
    }
    const int64_t nblk = exact_blocks(n);
    const int64_t elems = (int64_t)k * (DP + 1);
    if (k <= kExactListK) {
        cudaError_t e = cudaErrorInvalidValue;
        switch (DP) {
        case 4: e = launch_exact_list<4>(X, inv, ac, n, k, P, st); break;
        case 8: e = launch_exact_list<8>(X, inv, ac, n, k, P, st); break;
        case 16: e = launch_exact_list<16>(X, inv, ac, n, k, P, st); break;
        case 32: e = launch_exact_list<32>(X, inv, ac, n, k, P, st); break;
        case 64: e = launch_exact_list<64>(X, inv, ac, n, k, P, st); break;
        }
        if (e != cudaSuccess) return e;
        k_exact_merge<<<(unsigned)((elems + 255) / 256), 256, 0, st>>>(P, nblk, elems, acc);
        *launches += 2;
        return cudaGetLastError();
    }
    const dim3 grid((unsigned)nblk, (unsigned)((k + kExactThreads - 1) / kExactThreads));
    switch (DP) {
    case 4: k_exact_block_sums<4><<<grid, kExactThreads, 0, st>>>(X, inv, ac, n, k, P); break;
    case 8: k_exact_block_sums<8><<<grid, kExactThreads, 0, st>>>(X, inv, ac, n, k, P); break;
    case 16: k_exact_block_sums<16><<<grid, kExactThreads, 0, st>>>(X, inv, ac, n, k, P); break;
    case 32: k_exact_block_sums<32><<<grid, kExactThreads, 0, st>>>(X, inv, ac, n, k, P); break;
    case 64: k_exact_block_sums<64><<<grid, kExactThreads, 0, st>>>(X, inv, ac, n, k, P); break;
    default: return cudaErrorInvalidValue;
    }
    k_exact_merge<<<(unsigned)((elems + 255) / 256), 256, 0, st>>>(P, nblk, elems, acc);
    *launches += 2;
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// Re-bucketing (counting sort by bucket = a * Q + prefix class).  The prefix length
// p = #{c' : H[a][c'] < u} is the number of candidates the point would evaluate; rows of a
// bucket therefore have similar walk lengths, which keeps warp lanes busy.
__device__ __forceinline__ uint32_t bucket_class(int a, int lo, int k, int Q)
{
    int q = 0;
    if (lo > 0) {
        int64_t t = 1 + (int64_t)(lo - 1) * (Q - 1) / (k > 1 ? k - 1 : 1);
        q = (int)(t < Q - 1 ? t : Q - 1);
    }
    return (uint32_t)a * Q + q;
}

__device__ __forceinline__ uint32_t bucket_of(int a, float u, const uint64_t *NL, int k, int ks, int Q)
{
    if (Q == 1) return (uint32_t)a;
    const uint64_t *nl = NL + (int64_t)a * ks;
    int lo = 0, hi = k - 1;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (key_h(__ldg(nl + mid)) < u) lo = mid + 1; else hi = mid;
    }
    return bucket_class(a, lo, k, Q);
}

// Bucket keys + per-tile histograms.  For k <= kSortSmemK the H rows of all clusters are staged
// in shared memory, so the prefix search costs no dependent global loads.
constexpr int kSortSmemK = 128;

__global__ void k_sort_keys(SortParams p)
{
    extern __shared__ uint32_t sh[];
    const int k = p.k;
    const bool hs = p.Q > 1 && k <= kSortSmemK;
    float *sH = reinterpret_cast<float *>(sh + p.NB);   // k x k (row c: H[c][.] ascending, NaN pad)
    for (int b = threadIdx.x; b < p.NB; b += blockDim.x) sh[b] = 0;
    if (hs)
        for (int i = threadIdx.x; i < k * k; i += blockDim.x) {
            const int c = i / k, j = i % k;
            sH[i] = j < k - 1 ? key_h(p.NL[(int64_t)c * p.ks + j]) : __int_as_float(0x7fc00000);
        }
    __syncthreads();
    const int64_t r0 = (int64_t)blockIdx.x * p.tile_rows;
    int64_t r1 = r0 + p.tile_rows;
    if (r1 > p.n) r1 = p.n;
    for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
        const int a = p.a[r];
        const float u = p.u[r];
        uint32_t b;
        if (hs) {
            const float *h = sH + a * k;
            int lo = 0, hi = k - 1;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (h[mid] < u) lo = mid + 1; else hi = mid;
            }
            b = bucket_class(a, lo, k, p.Q);
        } else {
            b = bucket_of(a, u, p.NL, k, p.ks, p.Q);
        }
        p.keys[r] = b;
        atomicAdd(&sh[b], 1u);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < p.NB; b += blockDim.x)
        p.hist[(int64_t)b * p.ntiles + blockIdx.x] = sh[b];
}

// exclusive block scan helper (blockDim.x == 1024); returns exclusive prefix, *total = sum
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t *total)
{
    __shared__ uint32_t wsum[32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
        uint32_t s = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(kFull, s, o);
            if (lane >= o) s += y;
        }
        wsum[lane] = s;
    }
    __syncthreads();
    uint32_t incl = x + (w > 0 ? wsum[w - 1] : 0);
    *total = wsum[(blockDim.x >> 5) - 1];
    __syncthreads();
    return incl - v;
}

__global__ void k_scan_tiles(SortParams p)      // one CTA per bucket
{
    uint32_t *h = p.hist + (int64_t)blockIdx.x * p.ntiles;
    uint32_t carry = 0;
    for (int base = 0; base < p.ntiles; base += blockDim.x) {
        int i = base + threadIdx.x;
        uint32_t v = i < p.ntiles ? h[i] : 0, tot;
        uint32_t ex = block_excl_scan(v, &tot);
        if (i < p.ntiles) h[i] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) p.totals[blockIdx.x] = carry;
}

__global__ void k_scan_buckets(SortParams p)    // one CTA
{
    uint32_t carry = 0;
    for (int base = 0; base < p.NB; base += blockDim.x) {
        int i = base + threadIdx.x;
        uint32_t v = i < p.NB ? p.totals[i] : 0, tot;
        uint32_t ex = block_excl_scan(v, &tot);
        if (i < p.NB) p.base[i] = carry + ex;
        carry += tot;
    }
}

// Rows of a warp that go to the same bucket take consecutive slots (one smem atomic per bucket
// group, __match_any_sync), so a nearly sorted input is written back in coalesced runs.
// Rows of a warp that go to the same bucket take consecutive slots (one smem atomic per bucket
// group, __match_any_sync), so a nearly sorted input is written back in coalesced runs.  Each
// warp handles G groups of 32 rows per step with all loads issued first (memory parallelism).
// 32-byte global load / store (LDG/STG.E.ENL2.256): one transaction per 8-float row segment
__device__ __forceinline__ void ld256(const float4 *src, float4 &a, float4 &b)
{
    asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w) : "l"(src));
}
__device__ __forceinline__ void st256(float4 *dst, const float4 &a, const float4 &b)
{
    asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 :: "l"(dst), "f"(a.x), "f"(a.y), "f"(a.z), "f"(a.w), "f"(b.x), "f"(b.y), "f"(b.z), "f"(b.w)
                 : "memory");
}

template <int DP>
__global__ void __launch_bounds__(512) k_scatter(SortParams p)
{
    constexpr int G = DP <= 16 ? 4 : 2;
    extern __shared__ uint32_t cur[];
    for (int b = threadIdx.x; b < p.NB; b += blockDim.x)
        cur[b] = p.base[b] + p.hist[(int64_t)b * p.ntiles + blockIdx.x];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t r0 = (int64_t)blockIdx.x * p.tile_rows;
    int64_t r1 = r0 + p.tile_rows;
    if (r1 > p.n) r1 = p.n;
    for (int64_t rb = r0 + (threadIdx.x & ~31) * G; rb < r1; rb += (int64_t)blockDim.x * G) {
        uint32_t key[G];
        float4 xv[G][DP / 4];
        int32_t av[G], pv[G];
        float uv[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const int64_t r = rb + 32 * g + lane;
            const bool v = r < r1;
            key[g] = v ? __ldg(p.keys + r) : 0xffffffffu;
            const float4 *src = reinterpret_cast<const float4 *>(p.X + (v ? r : r0) * DP);
            if constexpr (DP >= 8) {
#pragma unroll
                for (int j = 0; j < DP / 4; j += 2) ld256(src + j, xv[g][j], xv[g][j + 1]);
            } else {
#pragma unroll
                for (int j = 0; j < DP / 4; ++j) xv[g][j] = __ldg(src + j);
            }
            av[g] = __ldg(p.a + (v ? r : r0));
            uv[g] = __ldg(p.u + (v ? r : r0));
            pv[g] = __ldg(p.perm + (v ? r : r0));
        }
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const bool v = key[g] != 0xffffffffu;
            const unsigned grp = __match_any_sync(kFull, key[g]);
            const int leader = __ffs(grp) - 1;
            uint32_t base = 0;
            if (v && lane == leader) base = atomicAdd(&cur[key[g]], (uint32_t)__popc(grp));
            base = __shfl_sync(kFull, base, leader);
            if (!v) continue;
            const int64_t dst = base + __popc(grp & ((1u << lane) - 1u));
            float4 *dx = reinterpret_cast<float4 *>(p.X2 + dst * DP);
            if constexpr (DP >= 8) {
#pragma unroll
                for (int j = 0; j < DP / 4; j += 2) st256(dx + j, xv[g][j], xv[g][j + 1]);
            } else {
#pragma unroll
                for (int j = 0; j < DP / 4; ++j) dx[j] = xv[g][j];
            }
            p.a2[dst] = av[g];
            p.u2[dst] = uv[g];
            p.perm2[dst] = pv[g];
        }
    }
}

cudaError_t launch_sort_tail(const SortParams &p, cudaStream_t st, int *launches);

template <int DP>
static cudaError_t launch_scatter(const SortParams &p, size_t sh, cudaStream_t st)
{
    if (sh > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k_scatter<DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh);
        if (e != cudaSuccess) return e;
    }
    k_scatter<DP><<<p.ntiles, 512, sh, st>>>(p);
    return cudaSuccess;
}

// Quantile prefix classes.  The walk's cost per warp is the largest prefix p in it, so rows are
// bucketed by p in classes of equal population (not equal width): pass 1 computes p per row and
// its histogram, one CTA turns the histogram into the class map, pass 2 forms the bucket keys.
__device__ __forceinline__ int prefix_len(const float *sH, bool hs, int a, float u, const uint64_t *NL, int k, int ks)
{
    int lo = 0, hi = k - 1;
    if (hs) {
        const float *h = sH + a * k;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (h[mid] < u) lo = mid + 1; else hi = mid;
        }
    } else {
        const uint64_t *nl = NL + (int64_t)a * ks;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (key_h(__ldg(nl + mid)) < u) lo = mid + 1; else hi = mid;
        }
    }
    return lo;
}

__global__ void k_sort_prefix(SortParams p)   // keys[r] = a << 13 | p, lohist[p] += 1
{
    extern __shared__ uint32_t shp[];
    const int k = p.k;
    const bool hs = k <= kSortSmemK;
    uint32_t *lh = shp;                                   // k+1
    float *sH = reinterpret_cast<float *>(shp + ((k + 4) & ~3));
    for (int i = threadIdx.x; i <= k; i += blockDim.x) lh[i] = 0;
    if (hs)
        for (int i = threadIdx.x; i < k * k; i += blockDim.x) {
            const int c = i / k, j = i % k;
            sH[i] = j < k - 1 ? key_h(p.NL[(int64_t)c * p.ks + j]) : __int_as_float(0x7fc00000);
        }
    __syncthreads();
    const int64_t r0 = (int64_t)blockIdx.x * p.tile_rows;
    int64_t r1 = r0 + p.tile_rows;
    if (r1 > p.n) r1 = p.n;
    for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
        const int a = p.a[r];
        const int lo = prefix_len(sH, hs, a, p.u[r], p.NL, k, p.ks);
        p.keys[r] = ((uint32_t)a << 13) | (uint32_t)lo;
        atomicAdd(&lh[lo], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i <= k; i += blockDim.x)
        if (lh[i]) atomicAdd(&p.lohist[i], lh[i]);
}

__global__ void k_sort_qmap(SortParams p)     // one CTA of 1024 threads
{
    const int k = p.k, Q = p.Q;
    __shared__ unsigned long long s_tot;
    uint32_t carry = 0, tot;
    // total rows with p >= 1
    unsigned long long part = 0;
    for (int i = 1 + threadIdx.x; i <= k; i += blockDim.x) part += p.lohist[i];
    if (threadIdx.x == 0) s_tot = 0;
    __syncthreads();
    atomicAdd(&s_tot, part);
    __syncthreads();
    const unsigned long long T1 = s_tot;
    for (int base = 1; base <= k; base += blockDim.x) {
        const int i = base + threadIdx.x;
        const uint32_t v = i <= k ? p.lohist[i] : 0;
        const uint32_t ex = block_excl_scan(v, &tot);
        if (i <= k) {
            const unsigned long long cum = (unsigned long long)carry + ex;   // rows with 1 <= p' < i
            int q = T1 ? (int)((unsigned long long)(Q - 1) * cum / T1) : 0;
            p.qmap[i] = 1 + min(q, Q - 2);
        }
        carry += tot;
    }
    if (threadIdx.x == 0) p.qmap[0] = 0;
}

__global__ void k_sort_keys_q(SortParams p)   // keys[r] = a * Q + qmap[p], per-tile histograms
{
    extern __shared__ uint32_t shq[];
    uint32_t *hst = shq;                                  // NB
    int *qm = reinterpret_cast<int *>(shq + p.NB);        // k+1
    for (int b = threadIdx.x; b < p.NB; b += blockDim.x) hst[b] = 0;
    for (int i = threadIdx.x; i <= p.k; i += blockDim.x) qm[i] = p.qmap[i];
    __syncthreads();
    const int64_t r0 = (int64_t)blockIdx.x * p.tile_rows;
    int64_t r1 = r0 + p.tile_rows;
    if (r1 > p.n) r1 = p.n;
    for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
        const uint32_t kv = p.keys[r];
        const uint32_t b = (kv >> 13) * (uint32_t)p.Q + (uint32_t)qm[kv & 8191u];
        p.keys[r] = b;
        atomicAdd(&hst[b], 1u);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < p.NB; b += blockDim.x)
        p.hist[(int64_t)b * p.ntiles + blockIdx.x] = hst[b];
}

cudaError_t launch_sort(const SortParams &p, cudaStream_t st, int *launches)
{
    if (p.Q > 1 && p.k <= kQuantK && p.lohist && p.qmap) {
        const size_t sp = (size_t)((p.k + 4) & ~3) * sizeof(uint32_t) +
                          (p.k <= kSortSmemK ? (size_t)p.k * p.k * sizeof(float) : 0);
        const size_t sq = (size_t)(p.NB + p.k + 1) * sizeof(uint32_t);
        if (sp > 48 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(k_sort_prefix, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sp);
            if (e != cudaSuccess) return e;
        }
        if (sq > 48 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(k_sort_keys_q, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sq);
            if (e != cudaSuccess) return e;
        }
        cudaError_t e = cudaMemsetAsync(p.lohist, 0, (size_t)(p.k + 1) * sizeof(uint32_t), st);
        if (e != cudaSuccess) return e;
        k_sort_prefix<<<p.ntiles, 512, sp, st>>>(p);
        k_sort_qmap<<<1, 1024, 0, st>>>(p);
        k_sort_keys_q<<<p.ntiles, 512, sq, st>>>(p);
        if (launches) *launches += 3;
        return launch_sort_tail(p, st, launches);
    }
    const size_t shk = (size_t)p.NB * sizeof(uint32_t) + (p.Q > 1 && p.k <= kSortSmemK ? (size_t)p.k * p.k * sizeof(float) : 0);
    if (shk > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k_sort_keys, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shk);
        if (e != cudaSuccess) return e;
    }
    k_sort_keys<<<p.ntiles, 512, shk, st>>>(p);
    if (launches) *launches += 1;
    return launch_sort_tail(p, st, launches);
}

cudaError_t launch_sort_tail(const SortParams &p, cudaStream_t st, int *launches)
{
    const size_t sh = (size_t)p.NB * sizeof(uint32_t);   // bucket cursors (NB <= KM_NB_MAX)
    k_scan_tiles<<<p.NB, 1024, 0, st>>>(p);
    k_scan_buckets<<<1, 1024, 0, st>>>(p);
    cudaError_t e = cudaSuccess;
    switch (p.DP) {
    case 4: e = launch_scatter<4>(p, sh, st); break;
    case 8: e = launch_scatter<8>(p, sh, st); break;
    case 16: e = launch_scatter<16>(p, sh, st); break;
    case 32: e = launch_scatter<32>(p, sh, st); break;
    case 64: e = launch_scatter<64>(p, sh, st); break;
    default: return cudaErrorInvalidValue;
    }
    if (e != cudaSuccess) return e;
    if (launches) *launches += 3;
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// S5: SSE in fp64 (x promoted, fp64 master centroids), block partials + one fp64 RED each.
__global__ void k_sse(const float *X, const int32_t *a, const double *C, int64_t n, int d, int DP,
                      double *out)
{
    __shared__ double red[32];
    double acc = 0.0;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x) {
        const float *x = X + r * DP;
        const double *c = C + (int64_t)a[r] * d;
        double s = 0.0;
        for (int j = 0; j < d; ++j) {
            double t = __dsub_rn((double)x[j], c[j]);
            s = __dadd_rn(s, __dmul_rn(t, t));
        }
        acc += s;
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
        if (threadIdx.x == 0) atomicAdd(out, v);
    }
}

cudaError_t launch_sse(const float *X, const int32_t *a, const double *C, int64_t n, int d,
                       int DP, double *out, cudaStream_t st)
{
    k_sse<<<148 * 8, 256, 0, st>>>(X, a, C, n, d, DP, out);
    return cudaGetLastError();
}

__global__ void k_unpermute(const int32_t *a, const int32_t *perm, int64_t n, int32_t *out)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[perm[i]] = a[i];
}

cudaError_t launch_unpermute(const int32_t *a, const int32_t *perm, int64_t n, int32_t *out,
                             cudaStream_t st)
{
    k_unpermute<<<148 * 8, 256, 0, st>>>(a, perm, n, out);
    return cudaGetLastError();
}

// X (n x d, contiguous) -> Xp (n x DP, zero padded)
__global__ void k_pad_rows(const float *X, float *Xp, int64_t n, int d, int DP)
{
    const int64_t tot = n * DP;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / DP;
        const int j = (int)(i - r * DP);
        Xp[i] = j < d ? X[r * d + j] : 0.f;
    }
}

cudaError_t launch_pad_rows(const float *X, float *Xp, int64_t n, int d, int DP, cudaStream_t st)
{
    k_pad_rows<<<148 * 8, 256, 0, st>>>(X, Xp, n, d, DP);
    return cudaGetLastError();
}

__global__ void k_iota(int32_t *perm, int64_t n)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        perm[i] = (int32_t)i;
}

cudaError_t launch_iota(int32_t *perm, int64_t n, cudaStream_t st)
{
    k_iota<<<148 * 8, 256, 0, st>>>(perm, n);
    return cudaGetLastError();
}

__global__ void k_check_finite(const float *X, int64_t count, int *flag)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x)
        if (!isfinite(X[i])) { *flag = 1; return; }
}

// sk-means: every row projected to the unit sphere once: x / ||x|| with the
// squared norm summed sequentially in fp64, a correctly rounded sqrt and division, rounded to
// fp32 — the oracle's normalize_rows step for step; *flag = 1 if a row has zero norm
__global__ void k_normalize_rows(float *X, int64_t n, int d, int DP, int *flag)
{
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        float *x = X + r * DP;
        double ss = 0.0;
        for (int j = 0; j < d; ++j) {
            const double v = (double)x[j];
            ss = __dadd_rn(ss, __dmul_rn(v, v));
        }
        if (!(ss > 0.0)) { *flag = 1; continue; }
        const double nrm = __dsqrt_rn(ss);
        for (int j = 0; j < d; ++j) x[j] = __double2float_rn(__ddiv_rn((double)x[j], nrm));
    }
}

cudaError_t launch_normalize_rows(float *X, int64_t n, int d, int DP, int *flag, cudaStream_t st)
{
    k_normalize_rows<<<148 * 8, 256, 0, st>>>(X, n, d, DP, flag);
    return cudaGetLastError();
}

cudaError_t launch_check_finite(const float *X, int64_t count, int *flag, cudaStream_t st)
{
    k_check_finite<<<148 * 8, 256, 0, st>>>(X, count, flag);
    return cudaGetLastError();
}

}  // namespace km
