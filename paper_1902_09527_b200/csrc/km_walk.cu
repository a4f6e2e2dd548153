// km_walk.cu — CUDA-core MTI assignment pass ("walk" engine) + fused fp64 reduction, sm_100a.
//
// Method: PAPER.md §3.3 (1026-1053): u += f(a) (drift, 1028-1030); clause 1 (u <= s(a): keep,
// no distance, 1036-1040); tighten U(u) = d(x, C[a]) (1033-1034); clauses 2/3: candidates c'
// with 1/2 d(a, c') < u (1042-1053, readings A1/A5/A6 of DESIGN.md); per-cluster sums fused
// into the same pass (§3.2, 1000-1011).  DESIGN.md "Walk engine".
//
// B200 realisation.  Rows are stored bucketed by cluster, so the 32 rows of a warp mostly share
// one cluster A (the cluster of lane 16).  Every lane walks A's neighbour list (ascending H)
// in lockstep, so each candidate row is ONE broadcast load for the warp:
//   * distances in the centred expansion form q_j = |x'|^2 + |c'_j|^2 - 2 x'.c'_j with
//     x' = x - C^[A], c'_j = C^[c_j] - C^[A] (k_prep_walk stores [-2 c'_j | |c'_j|^2, prefix
//     max, H, c_j] per candidate): DP/2 + 2 FMA-pipe instructions per candidate instead of the
//     2 DP of the direct form;
//   * lanes of A stop at their own prefix p = #{j : H[A][j] < u_t} (clauses 2/3); a lane of
//     another cluster a (a "misfit") takes the prefix H[A][j] < (u_t + d(x, A)) / 2: by the
//     triangle inequality no centroid outside it can beat a, and a itself is inside it;
//   * the warp evaluates up to its largest prefix; values past a lane's own prefix are true
//     distances of real centroids, so they never change the argmin (only the error bound,
//     which covers every evaluated column);
//   * best / second-best by packed keys (q bits, low bits = position) with integer min/max;
//   * exact mode: rigorous intervals decide the winner, otherwise the lane re-walks its own
//     list in the direct form with fp64 refinement (same decision procedure as k_assign).
// Distance counts (1 + #{c : H[a][c] < u_t}) of misfit lanes are deferred to k_mti_count.
//
// SKIP1 (for clause-1 points "no I/O
// requests are made" for their data): the a/u of a batch are staged one batch before its rows,
// the clause-1 test is taken on them, and only the rows that fail it are read from HBM.  The
// running sums are deltas of the moved rows (reading B5), so a clause-1 row's x is never needed.
// Chosen per pass by the host when the previous pass's clause-1 rate is high (C5, C2, C1).
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "km_device.cuh"
#include "km_kernels.cuh"

namespace km {

// One CTA per SM: the shared H rows and C are held once per SM rather than once per CTA, which
// leaves most of the 256 KB L1/shared array as L1 for the candidate tables (walk_threads below).
#ifndef KM_WALK_R32
#define KM_WALK_R32 2           // rows per lane at d = 32
#endif
#ifndef KM_WALK_HALVES
#define KM_WALK_HALVES 1        // d >= 32: consume each candidate pair block in two halves
#endif
#ifndef KM_WALK_CHUNK
#define KM_WALK_CHUNK 128       // measured: 64 1.73 ms, 128 1.67, 256 1.69, 512 1.73, 1024 1.80 (C3)
#endif
constexpr int kWalkChunk = KM_WALK_CHUNK;   // rows a warp claims per work-counter fetch
constexpr int kQueue = 64;             // mover-queue entries per warp (< 32 left + 32 new)

// floats of one warp's shared-memory region: staged rows x | a | u, mover queue (row, from, to)
// [, SKIP1: the second a | u slot]
__host__ __device__ constexpr int walk_warp_floats(int DP, int R, int skip1)
{
    return 32 * R * (DP + 2) + 3 * kQueue + (skip1 ? 64 * R : 0);
}

__host__ __device__ constexpr int walk_pair_f4(int DP) { return DP / 2; }   // float4 per candidate pair

// 32-byte read-only load (LDG.E.ENL2.256): two float4 in one instruction
__device__ __forceinline__ void ldg256(const float4 *src, float4 &a, float4 &b)
{
    asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
                 : "l"(src));
}

// FFMA2 with a scalar operand broadcast to both lanes: r = (a*b.x + c.x, a*b.y + c.y)
__device__ __forceinline__ float2 fma2s(float a, float2 b, float2 c)
{
    float2 r;
    asm("{\n\t.reg .b64 ra, rb, rc, rr;\n\t"
        "mov.b64 ra, {%2, %2};\n\tmov.b64 rb, {%3, %4};\n\tmov.b64 rc, {%5, %6};\n\t"
        "fma.rn.f32x2 rr, ra, rb, rc;\n\tmov.b64 {%0, %1}, rr;\n\t}"
        : "=f"(r.x), "=f"(r.y) : "f"(a), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return r;
}

// FADD2 with a scalar operand broadcast to both lanes: r = (a + b.x, a + b.y)
__device__ __forceinline__ float2 add2s(float a, float2 b)
{
    float2 r;
    asm("{\n\t.reg .b64 ra, rb, rr;\n\t"
        "mov.b64 ra, {%2, %2};\n\tmov.b64 rb, {%3, %4};\n\t"
        "add.rn.f32x2 rr, ra, rb;\n\tmov.b64 {%0, %1}, rr;\n\t}"
        : "=f"(r.x), "=f"(r.y) : "f"(a), "f"(b.x), "f"(b.y));
    return r;
}

// squared distances to the candidate pair (j, j+1) in the centred expansion form:
// (q_j, q_j+1) = (xx + cc_j, xx + cc_j+1) + sum_e x'_e (m_j[e], m_j+1[e]),  m = -2 c', cc = |c'|^2
// v: the pair's DP/2 float4 (coordinates interleaved by candidate); one FFMA2 (scalar x'_e
// broadcast) per coordinate
template <int DP>
__device__ __forceinline__ float2 q_pair(const float (&xc)[DP], float xx, float2 cc, const float4 (&v)[DP / 2])
{
    float2 s = add2s(xx, cc);
#pragma unroll
    for (int e = 0; e < DP / 2; ++e) {
        s = fma2s(xc[2 * e], make_float2(v[e].x, v[e].y), s);
        s = fma2s(xc[2 * e + 1], make_float2(v[e].z, v[e].w), s);
    }
    return s;
}

// #{j < NH : h[j] < T}, NH a power of two, h ascending with NaN padding: unrolled lower bound
template <int NH, typename P>
__device__ __forceinline__ int count_below_u(P h, float T)
{
    int base = 0;
#pragma unroll
    for (int half = NH >> 1; half >= 1; half >>= 1)
        base = h[base + half - 1] < T ? base + half : base;
    return base + (h[base] < T ? 1 : 0);
}

// shared-memory form: the running lower bound is kept as a byte address, so each step is one
// LDS with an immediate offset, one compare and one predicated add
template <int HALF>
__device__ __forceinline__ void cbs_step(uint32_t &a, float T)
{
    if constexpr (HALF >= 1) {
        float v;
        asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(v) : "r"(a), "n"((HALF - 1) * 4));
        if (v < T) a += HALF * 4;
        cbs_step<HALF / 2>(a, T);
    }
}
template <int NH>
__device__ __forceinline__ int count_below_s(const float *h, float T)
{
    const uint32_t a0 = (uint32_t)__cvta_generic_to_shared(h);
    uint32_t a = a0;
    cbs_step<NH / 2>(a, T);
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return (int)((a - a0) >> 2) + (v < T ? 1 : 0);
}

__device__ __forceinline__ void cp_async16(void *dst, const void *src)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src) : "memory");
}

// #{j < m : h[j] < T} for ascending h (NaN padding never compares below)
__device__ __forceinline__ int count_below_f(const float *__restrict__ h, int m, float T)
{
    int lo = 0, hi = m;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (h[mid] < T) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// One lane = R rows (rows r0 + lane + 32 i); the warp walks its cluster A's candidate rows once
// for all 32 R rows, so each broadcast load serves R rows per lane.
// Threads per CTA (one CTA per SM): as many warps as the register need of each row width
// allows — DP <= 8: 1024 (64 registers), 16: 512 (128), 32: 384 (168), 64: 256 (255); measured
// on B200 against 768 / 640 / 512 (DP 8) and 256 / 320 / 448 / 512 (DP 32), DESIGN.md §6.
#ifndef KM_WALK_T8
#define KM_WALK_T8 1024
#endif
#ifndef KM_WALK_T16
#define KM_WALK_T16 512
#endif
#ifndef KM_WALK_T32
#define KM_WALK_T32 384
#endif
__host__ __device__ constexpr int walk_threads_of(int DP)
{
    return DP <= 8 ? KM_WALK_T8 : (DP <= 16 ? KM_WALK_T16 : (DP <= 32 ? KM_WALK_T32 : 256));
}
template <int DP> constexpr int walk_threads() { return walk_threads_of(DP); }
static int walk_threads_rt(int DP) { return walk_threads_of(DP); }

// Staged row r, 16-byte part q (of DP/4) lives in float4 slot r (DP/4) + (q ^ g(r)): the lanes of
// a warp read part q of rows lane, lane + 32 with one LDS.128 each, and without the swizzle rows
// DP*4 bytes apart fall on the same banks (DP = 32: an 8-way conflict per quarter warp; ncu of
// C4: 474M shared bank conflicts, L1 throughput 88 %).  g spreads 8 consecutive rows over the 8
// 16-byte bank groups.
#ifndef KM_SWZ_MIN_DP
#define KM_SWZ_MIN_DP 8       // DP = 8: unswizzled 32-B rows read 2-way conflicted (ncu of C3: the
                              // staging writes and reads were 57 % of the shared wavefronts)
#endif
template <int DP>
__device__ __forceinline__ int stg_swz(int c)
{
    constexpr int P = DP / 4;                     // parts per row
    if constexpr (DP < KM_SWZ_MIN_DP) return c;
    const int r = c / P, q = c % P;
    const int g = P >= 8 ? (r & 7) : ((r * P) >> 3) & (P - 1);
    return r * P + (q ^ g);
}

#define KM_WALK_NAME k_walk
#define KM_SKIP1 0
#include "km_walk_body.cuh"
#undef KM_WALK_NAME
#undef KM_SKIP1
#define KM_WALK_NAME k_walk_skip1
#define KM_SKIP1 1
#include "km_walk_body.cuh"
#undef KM_WALK_NAME
#undef KM_SKIP1

// S1 (walk part): per cluster c (one CTA), the candidate rows of its neighbour list NL[c]:
//   Wblk[c][j] = -2 c'_j (DP floats), c'_j = fp32(C[c_j]) - fp32(C[c]) (RN);
//   Wcc[c][j] = |c'_j|^2 (RN, as used in q); Wmeta[c][j] = {prefix max of |c'|^2 rounded up, c_j};
//   WH[c][j] = H[c][c_j] (fp32, rounded down).  Rows j >= k-1 are dummies: q = xx + 1e30, H NaN.
__global__ void k_prep_walk(const double *C, const uint64_t *NL, int k, int d, int DP, int ks, int kp, int whs,
                            float4 *Wblk, float *Wcc, float2 *Wmeta, float *WH)
{
    const int c = blockIdx.x;
    const double *Cc = C + (int64_t)c * d;
    const uint64_t *nl = NL + (int64_t)c * ks;
    // pair P = rows (2P, 2P+1): float e of the pair block = coordinate e/2 of row 2P + (e & 1)
    float *blk = reinterpret_cast<float *>(Wblk + (int64_t)c * (kp / 2) * (DP / 2));
    extern __shared__ float scn[];
    for (int j = threadIdx.x; j < kp; j += blockDim.x) {
        const bool real = j < k - 1;
        const int cj = real ? key_c(nl[j]) : c;
        const double *Cj = C + (int64_t)cj * d;
        double cn2 = 0.0;
        float *pairp = blk + (int64_t)(j >> 1) * 2 * DP + (j & 1);
        for (int e = 0; e < DP; ++e) {
            const float v = (real && e < d) ? __fsub_rn((float)Cj[e], (float)Cc[e]) : 0.f;
            cn2 += (double)v * (double)v;
            pairp[2 * e] = -2.f * v;
        }
        Wcc[(int64_t)c * kp + j] = real ? (float)cn2 : 1e30f;
        scn[j] = real ? __double2float_ru(cn2 * (1.0 + 1e-12)) : 0.f;
        Wmeta[(int64_t)c * kp + j].y = __int_as_float(cj);
    }
    for (int j = threadIdx.x; j < whs; j += blockDim.x)
        WH[(int64_t)c * whs + j] = j < k - 1 ? key_h(nl[j]) : __int_as_float(0x7fc00000);
    __syncthreads();
    if (threadIdx.x == 0) {                      // prefix max of |c'|^2 (rounded up)
        float m = 0.f;
        for (int j = 0; j < kp; ++j) { m = fmaxf(m, scn[j]); Wmeta[(int64_t)c * kp + j].x = m; }
    }
}

cudaError_t launch_prep_walk(const double *C, const uint64_t *NL, int k, int d, int DP, int ks, int kp, int whs,
                             float4 *Wblk, float *Wcc, float2 *Wmeta, float *WH, cudaStream_t st)
{
    k_prep_walk<<<k, 128, (size_t)kp * sizeof(float), st>>>(C, NL, k, d, DP, ks, kp, whs, Wblk, Wcc, Wmeta, WH);
    return cudaGetLastError();
}

size_t walk_smem(int DP, bool csmem, int k, int whs, bool wh_smem, bool skip1)
{
    const int R = DP <= 16 ? 2 : (DP <= 32 ? KM_WALK_R32 : 1);
    const int k4 = (k + 3) & ~3;
    return (size_t)((csmem ? k * DP : 0) + 2 * k4 + (wh_smem ? k * whs : 0)) * sizeof(float) +
           (size_t)(walk_threads_rt(DP) / 32) * walk_warp_floats(DP, R, skip1 ? 1 : 0) * sizeof(float);
}

// rows per lane: 2 where the registers allow (the candidate loads are shared by both rows)
template <int DP> constexpr int walk_r() { return DP <= 16 ? 2 : (DP <= 32 ? KM_WALK_R32 : 1); }

typedef void (*walk_kernel_t)(AssignParams);

#define KM_WALK_PICK(K)                                                              \
    if (hs) {                                                                        \
        switch (whs) {                                                               \
        case 2: case 4: case 8: case 16: return K<DP, CSMEM, R, 16, true>;           \
        case 32: return K<DP, CSMEM, R, 32, true>;                                   \
        case 64: return K<DP, CSMEM, R, 64, true>;                                   \
        case 128: return K<DP, CSMEM, R, 128, true>;                                 \
        case 256: return K<DP, CSMEM, R, 256, true>;                                 \
        }                                                                            \
    } else {                                                                         \
        switch (whs) {                                                               \
        case 256: return K<DP, CSMEM, R, 256, false>;                                \
        case 512: return K<DP, CSMEM, R, 512, false>;                                \
        case 1024: return K<DP, CSMEM, R, 1024, false>;                              \
        case 2048: return K<DP, CSMEM, R, 2048, false>;                              \
        case 4096: return K<DP, CSMEM, R, 4096, false>;                              \
        }                                                                            \
    }                                                                                \
    return nullptr;

template <int DP, bool CSMEM, bool SK>
static walk_kernel_t walk_pick_s(int whs, bool hs)
{
    constexpr int R = walk_r<DP>();
    if constexpr (SK) {
        KM_WALK_PICK(k_walk_skip1)
    } else {
        KM_WALK_PICK(k_walk)
    }
}

template <int DP, bool CSMEM>
static walk_kernel_t walk_pick(int whs, bool hs, bool skip1)
{
    return skip1 ? walk_pick_s<DP, CSMEM, true>(whs, hs) : walk_pick_s<DP, CSMEM, false>(whs, hs);
}

static walk_kernel_t walk_kernel(int DP, bool csmem, int whs, bool hs, bool skip1)
{
    switch (DP * 2 + (csmem ? 1 : 0)) {
    case 8: return walk_pick<4, false>(whs, hs, skip1);
    case 9: return walk_pick<4, true>(whs, hs, skip1);
    case 16: return walk_pick<8, false>(whs, hs, skip1);
    case 17: return walk_pick<8, true>(whs, hs, skip1);
    case 32: return walk_pick<16, false>(whs, hs, skip1);
    case 33: return walk_pick<16, true>(whs, hs, skip1);
    case 64: return walk_pick<32, false>(whs, hs, skip1);
    case 65: return walk_pick<32, true>(whs, hs, skip1);
    case 128: return walk_pick<64, false>(whs, hs, skip1);
    case 129: return walk_pick<64, true>(whs, hs, skip1);
    }
    return nullptr;
}

bool walk_supported(int DP) { return DP == 4 || DP == 8 || DP == 16 || DP == 32 || DP == 64; }

cudaError_t launch_walk(int DP, bool csmem, const AssignParams &p, int grid, bool skip1, cudaStream_t st)
{
    walk_kernel_t kern = walk_kernel(DP, csmem, p.whs, p.wh_smem != 0, skip1);
    if (!kern) return cudaErrorInvalidValue;
    const size_t sm = walk_smem(DP, csmem, p.k, p.whs, p.wh_smem != 0, skip1);
    if (sm > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e != cudaSuccess) return e;
    }
    kern<<<grid, walk_threads_rt(DP), sm, st>>>(p);
    return cudaGetLastError();
}

int walk_grid(int DP, bool csmem, int k, int whs, bool hs, int num_sms)
{
    int best = 0;
    for (int sk = 0; sk < 2; ++sk) {     // both variants share one grid (one CTA per SM)
        walk_kernel_t kern = walk_kernel(DP, csmem, whs, hs, sk != 0);
        if (!kern) return num_sms;
        const size_t sm = walk_smem(DP, csmem, k, whs, hs, sk != 0);
        if (sm > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, walk_threads_rt(DP), sm);
        per_sm = per_sm < 1 ? 1 : per_sm;
        best = sk == 0 ? per_sm : std::min(best, per_sm);
    }
    return best * num_sms;
}

}  // namespace km
