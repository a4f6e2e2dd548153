// km_walk_common.cuh — helpers shared by the walk engine (km_walk.cu: k_walk, k_walk_skip1) and the
// screen/resolve engine (km_screen.cu): packed FFMA2/FADD2 with a broadcast scalar, 32-byte
// read-only loads, shared-memory H prefix search, cp.async staging, warp sizing, staging swizzle.
#pragma once
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
#ifndef KM_WALK_CHAINS2
#define KM_WALK_CHAINS2 0       // d >= 32 (halves): two FFMA2 accumulation chains per row
#endif
#ifndef KM_WALK_CHUNK
#define KM_WALK_CHUNK 128       // measured: 64 1.73 ms, 128 1.67, 256 1.69, 512 1.73, 1024 1.80 (C3)
#endif
struct km_true { static constexpr bool value = true; };
struct km_false { static constexpr bool value = false; };
constexpr int kWalkChunk = KM_WALK_CHUNK;   // rows a warp claims per work-counter fetch
constexpr int kQueue = 64;             // mover-queue entries per warp (< 32 left + 32 new)

// floats of one warp's shared-memory region: staged rows x | a | u, mover queue (row, from, to)
// [, SKIP1: the second a | u slot]
__host__ __device__ constexpr int walk_warp_floats(int DP, int R, int skip1)
{
    return 32 * R * (DP + 2) + 3 * kQueue + (skip1 ? 64 * R : 0);
}

__host__ __device__ constexpr int walk_pair_f4(int DP) { return DP / 2; }   // float4 per candidate pair

// Per-warp shared-memory copy of the head of the warp cluster's candidate table (KM_WALK_TAB 1):
// the first walk_tab_cap candidates of A's list (pair blocks + |c'|^2) are copied once per change
// of A with cp.async (a group of its own, committed before the next batch's rows) and then read
// with broadcast LDS instead of broadcast LDG: 5.0 against 8.2 SM cycles per 32-B block per warp
// (tools/probes/ldc_probe.cu), and no L1 miss on the walk's dependent path — at d = 32 the
// tables (k^2 x 132 B = 1.3 MB at k = 100) do not fit L1 and the walk runs 3 warps per
// sub-partition, so every miss showed as a long-scoreboard stall.  Measured: C4 6.28 -> 5.56 ms
// per pass; C3 (d = 8) 1.565 -> 1.559 ms, so only d = 32 takes it.  Only with the H rows in
// shared memory and without SKIP1.  Shared memory at d = 32: <= 186,240 B without the table for
// every k that keeps the H rows in shared memory (k <= 112), + 12 warps x 24 x 132 B = 224,256 B.
#ifndef KM_WALK_TAB
#define KM_WALK_TAB 1
#endif
#ifndef KM_WALK_TAB_CAP
#define KM_WALK_TAB_CAP 24      // even; 28 is the most that fits beside the H rows at k = 112
#endif
__host__ __device__ constexpr int walk_tab_cap(int DP, bool hs, int skip1)
{
    return (KM_WALK_TAB && hs && !skip1 && DP == 32) ? KM_WALK_TAB_CAP : 0;
}
__host__ __device__ constexpr int walk_tab_floats(int DP, bool hs, int skip1) { return walk_tab_cap(DP, hs, skip1) * (DP + 1); }

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

__device__ __forceinline__ void cp_async8(void *dst, const void *src)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src) : "memory");
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
// rows per lane: 2 where the registers allow (the candidate loads are shared by both rows)
#ifndef KM_WALK_R8
#define KM_WALK_R8 2            // rows per lane at d <= 8
#endif
template <int DP> constexpr int walk_r() { return DP <= 8 ? KM_WALK_R8 : (DP <= 16 ? 2 : (DP <= 32 ? KM_WALK_R32 : 1)); }
static inline int walk_r_rt(int DP) { return DP <= 8 ? KM_WALK_R8 : (DP <= 16 ? 2 : (DP <= 32 ? KM_WALK_R32 : 1)); }
// d = 32 with the H rows in global memory (large k, C5): three rows per lane at 256 threads per
// CTA — each candidate pair block a warp loads (256 B, delivered to all 32 lanes through the L1
// data pipe) then serves 96 rows; measured on C5: 28.0 -> 24.4 ms per pass; on C4 (H rows in
// shared memory) two rows at 384 threads stay faster (6.27 vs 7.60 ms)
#ifndef KM_WALK_R32G
#define KM_WALK_R32G 3
#endif
#ifndef KM_WALK_T32G
#define KM_WALK_T32G 256
#endif
__host__ __device__ constexpr int walk_threads_dr(int DP, int R)
{
    return (DP == 32 && R == KM_WALK_R32G && R != KM_WALK_R32) ? KM_WALK_T32G : walk_threads_of(DP);
}
static inline int walk_r_sel(int DP, bool hs) { return (DP == 32 && !hs) ? KM_WALK_R32G : walk_r_rt(DP); }
static inline int walk_threads_rt(int DP) { return walk_threads_of(DP); }

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

}  // namespace km
