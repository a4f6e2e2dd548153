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
// (q_j, q_j+1) = (xx + cc_j, xx + cc_j+1) + sum_e x'_e (m_j[e], m_j+1[e]),  m = -2 c'
// v: the pair's DP/2 float4 (coordinates interleaved by candidate); one FFMA2 per coordinate
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

template <int DP, bool CSMEM, int R, int NH, bool HSMEM>
__global__ void __launch_bounds__(walk_threads<DP>(), 1)
k_walk(AssignParams p)
{
    extern __shared__ __align__(16) float smem[];
    const int k = p.k;
    float *sC = smem;                               // k*DP (CSMEM)
    const int k4 = (k + 3) & ~3;                   // sections stay 16-B aligned
    float *sF = smem + (CSMEM ? k * DP : 0);        // k
    float *sS = sF + k4;                            // k
    float *sH = sS + k4;                            // k x NH H rows (HSMEM)
    // per-warp staging of the next batch (cp.async): x rows, then a, then u
    constexpr int kRowsB = 32 * R;
    float *stg = sH + (HSMEM ? k * NH : 0) + (threadIdx.x >> 5) * (kRowsB * (DP + 2) + 3 * kQueue);
    int *sQ = reinterpret_cast<int *>(stg + kRowsB * DP + 2 * kRowsB);   // mover queue: row, from, to
    if (CSMEM) {
        const float4 *src = reinterpret_cast<const float4 *>(p.Cneg);
        float4 *dst = reinterpret_cast<float4 *>(sC);
        for (int i = threadIdx.x; i < k * DP / 4; i += blockDim.x) dst[i] = src[i];
    }
    for (int i = threadIdx.x; i < k; i += blockDim.x) { sF[i] = p.f[i]; sS[i] = p.s[i]; }
    if (HSMEM)
        for (int i = threadIdx.x; i < k * NH; i += blockDim.x) sH[i] = p.WH[i];
    __syncthreads();
    CRow<CSMEM> Cn;
    if constexpr (CSMEM) {
        uint32_t b = (uint32_t)__cvta_generic_to_shared(sC);
        asm volatile("mov.u32 %0, %0;" : "+r"(b));
        Cn.base = b;
    } else {
        Cn.base = p.Cneg;
    }
    double *acc = p.acc + (int64_t)(blockIdx.x % p.nslab) * k * (DP + 1);
    const float eps = *p.eps;
    const int lane = threadIdx.x & 31;
    const int n = (int)p.n;                        // < 2^31 (kmeans_create enforces it)
    const int kp = p.wpad;                          // candidate rows per cluster block
    const int kcols = k - 1;
    const int ib = p.wbits;                         // key index bits
    const uint32_t kmask = ~((1u << ib) - 1u);
    const float qtrunc = 1.f + __uint_as_float((uint32_t)(127 - 23 + ib) << 23) * 1.0001f;   // 1 + 2^(ib-23)
    // expansion-form error: |q~ - |x'-c'|^2| <= kappa (xx + cmax)
    const float kappa = 2.f * (2.f * DP + 20.f) * 5.9604645e-8f;
    constexpr int kRows = 32 * R;                   // rows per warp batch

    // per-lane counters: 32 bits (a lane's rows and walk steps stay far below 2^32; registers
    // are what bounds the resident warps), widened for the warp reduction at the end
    unsigned long long c_dists = 0;
    unsigned c_changed32 = 0, c_clause132 = 0, c_refined32 = 0, c_fb32 = 0, steps32 = 0;

    constexpr int kBatches = kWalkChunk / kRows;
    auto claim = [&]() -> int {
        int c = 0;
        if (lane == 0) c = atomicAdd(p.work, 1);
        c = __shfl_sync(kFull, c, 0);
        return c < (n + kWalkChunk - 1) / kWalkChunk ? c * kWalkChunk : n;   // n: no more work
    };
    int chunk_row = claim(), ahead_row = claim();
    int bt = 0;
    // stage rows [r0, r0 + 32 R) of X, a, u into this warp's buffer (16-B cp.async per lane)
    auto stage = [&](int r0) {
        const float4 *xs = reinterpret_cast<const float4 *>(p.X + (size_t)r0 * DP);
        float4 *xd = reinterpret_cast<float4 *>(stg);
#pragma unroll
        for (int c = lane; c < kRowsB * DP / 4; c += 32) cp_async16(xd + c, xs + c);
        float *ad = stg + kRowsB * DP;
        if (lane < kRowsB / 4) cp_async16(ad + 4 * lane, p.a + r0 + 4 * lane);
        else if (lane < kRowsB / 2) cp_async16(ad + kRowsB + 4 * (lane - kRowsB / 4), p.u + r0 + 4 * (lane - kRowsB / 4));
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if (chunk_row < n) stage(chunk_row);
    // mover queue (shared memory, kQueue entries per warp; mq warp-uniform)
    int mq = 0;
    auto flush_moves = [&]() {
        __syncwarp();
        if (lane < min(mq, 32)) {
            const int mrow = sQ[lane], mfrom = sQ[kQueue + lane], mto = sQ[2 * kQueue + lane];
            float xr[DP];
            const float4 *src = reinterpret_cast<const float4 *>(p.X + (size_t)mrow * DP);
#pragma unroll
            for (int j = 0; j < DP / 4; ++j) {
                const float4 t = __ldg(src + j);
                xr[4 * j] = t.x; xr[4 * j + 1] = t.y; xr[4 * j + 2] = t.z; xr[4 * j + 3] = t.w;
            }
            move_delta<DP>(acc, p.d, mfrom, mto, xr);
        }
        __syncwarp();
        if (mq > 32) {   // keep the overflow (< 32 entries) at the front
            int e0 = 0, e1 = 0, e2 = 0;
            const bool mv = lane < mq - 32;
            if (mv) { e0 = sQ[32 + lane]; e1 = sQ[kQueue + 32 + lane]; e2 = sQ[2 * kQueue + 32 + lane]; }
            __syncwarp();
            if (mv) { sQ[lane] = e0; sQ[kQueue + lane] = e1; sQ[2 * kQueue + lane] = e2; }
            __syncwarp();
            mq -= 32;
        } else {
            mq = 0;
        }
    };

    while (chunk_row < n) {
        const int row0 = chunk_row + bt * kRows;
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncwarp();
        float x[R][DP];
        int aold[R];
        float uu[R];
        bool valid[R], active[R];
        unsigned amask = 0;
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const int r = 32 * i + lane;
#pragma unroll
            for (int j = 0; j < DP; j += 4) {
                const float4 t = *reinterpret_cast<const float4 *>(stg + r * DP + j);
                x[i][j] = t.x; x[i][j + 1] = t.y; x[i][j + 2] = t.z; x[i][j + 3] = t.w;
            }
            aold[i] = __float_as_int(stg[kRowsB * DP + r]);
            const float uold = stg[kRowsB * DP + kRowsB + r];
            const int row = row0 + r;
            valid[i] = row < n;
            if (!valid[i]) aold[i] = 0;
            uu[i] = valid[i] ? __fadd_ru(uold, sF[aold[i]]) : 0.f;          // u += f(a)
            const bool c1 = valid[i] && uu[i] <= sS[aold[i]];                  // clause 1
            active[i] = valid[i] && !c1;
            c_clause132 += c1;
            amask |= __ballot_sync(kFull, active[i]) ? (1u << i) : 0u;
        }
        __syncwarp();
        if (++bt == kBatches || chunk_row + bt * kRows >= n) {
            bt = 0;
            chunk_row = ahead_row;
            ahead_row = chunk_row < n ? claim() : ahead_row;
        }
        if (chunk_row < n) stage(chunk_row + bt * kRows);

        int anew[R];
        float unew[R], ut[R];
        bool defer[R];
#pragma unroll
        for (int i = 0; i < R; ++i) { anew[i] = aold[i]; unew[i] = uu[i]; ut[i] = 0.f; defer[i] = false; }
        if (amask) {
            // warp cluster A: the middle row's if active, else the first active row's
            const int mid = R == 1 ? 16 : 0;            // R = 2: lane 0 of the second half
            const unsigned m_mid = __ballot_sync(kFull, active[R - 1]);
            int A;
            if ((m_mid >> mid) & 1u) A = __shfl_sync(kFull, aold[R - 1], mid);
            else {
                const unsigned m0 = __ballot_sync(kFull, active[0]);
                A = m0 ? __shfl_sync(kFull, aold[0], __ffs(m0) - 1) : __shfl_sync(kFull, aold[R - 1], __ffs(m_mid) - 1);
            }
            float4 cA[DP / 4];
#pragma unroll
            for (int j = 0; j < DP / 4; ++j) cA[j] = Cn.ld(A, DP, 4 * j);
            float xc[R][DP], xx[R], lo[R], T[R];
            int pl[R];
            bool misfit[R];
            int pm = 0;
#pragma unroll
            for (int i = 0; i < R; ++i) {
                // x' = x - C^[A] (direct form's arithmetic), xx = |x'|^2
                float2 a0 = make_float2(0.f, 0.f), a1 = make_float2(0.f, 0.f);
#pragma unroll
                for (int j = 0; j < DP; j += 4) {
                    const float4 c = cA[j / 4];
                    const float2 t0 = add2(make_float2(x[i][j], x[i][j + 1]), make_float2(c.x, c.y));
                    const float2 t1 = add2(make_float2(x[i][j + 2], x[i][j + 3]), make_float2(c.z, c.w));
                    xc[i][j] = t0.x; xc[i][j + 1] = t0.y; xc[i][j + 2] = t1.x; xc[i][j + 3] = t1.y;
                    a0 = fma2(t0, t0, a0);
                    a1 = fma2(t1, t1, a1);
                }
                const float2 s2 = add2(a0, a1);
                xx[i] = s2.x + s2.y;
                misfit[i] = active[i] && aold[i] != A;
                lo[i] = 0.f; T[i] = 0.f; pl[i] = 0;
                if (active[i]) {
                    if (!misfit[i]) {
                        ut[i] = upper_d(xx[i], p.g_up, eps);
                        lo[i] = lower_d(xx[i], p.g_dn, eps);
                        T[i] = ut[i];
                    } else {
                        const float qo = dist2<DP, CSMEM>(x[i], Cn, aold[i]);
                        ut[i] = upper_d(qo, p.g_up, eps);
                        lo[i] = lower_d(qo, p.g_dn, eps);
                        T[i] = __fmul_ru(__fadd_ru(ut[i], upper_d(xx[i], p.g_up, eps)), 0.5f);
                    }
                    if constexpr (HSMEM) pl[i] = count_below_s<NH>(sH + A * NH, T[i]);
                    else pl[i] = count_below_u<NH>(p.WH + (int64_t)A * NH, T[i]);
                }
                pm = max(pm, pl[i]);
            }
            pm = __reduce_max_sync(kFull, pm);
            // the walk: candidates j < pm of A's list, two per step, keys (q & kmask) | j
            const float4 *blk = p.Wblk + (int64_t)A * (kp / 2) * walk_pair_f4(DP);
            const float2 *ccA = reinterpret_cast<const float2 *>(p.Wcc + (int64_t)A * kp);
            int m1[R], m2[R];
#pragma unroll
            for (int i = 0; i < R; ++i) { m1[i] = 0x7fffffff; m2[i] = 0x7fffffff; }
            for (int j = 0; j < pm; j += 2) {
                const float2 cc = __ldg(ccA + (j >> 1));
                float2 q[R];
                if constexpr (DP >= 32 && KM_WALK_HALVES && HSMEM) {   // (measured: +2 % on C4, -3.5 % on C5)
                    // wide rows: the pair block is consumed in two halves of DP/2 coordinates, so
                    // only DP/4 float4 of it are live at once (registers bound the resident warps)
#pragma unroll
                    for (int i = 0; i < R; ++i) q[i] = add2s(xx[i], cc);
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        float4 v[DP / 4];
#pragma unroll
                        for (int e = 0; e < DP / 4; e += 2)
                            ldg256(blk + (int64_t)(j >> 1) * walk_pair_f4(DP) + h * (DP / 4) + e, v[e], v[e + 1]);
#pragma unroll
                        for (int i = 0; i < R; ++i)
#pragma unroll
                            for (int e = 0; e < DP / 4; ++e) {
                                q[i] = fma2s(xc[i][h * (DP / 2) + 2 * e], make_float2(v[e].x, v[e].y), q[i]);
                                q[i] = fma2s(xc[i][h * (DP / 2) + 2 * e + 1], make_float2(v[e].z, v[e].w), q[i]);
                            }
                    }
                } else {
                    float4 v[DP / 2];
                    if constexpr (DP >= 32) {   // halves the load instructions where they dominate
#pragma unroll
                        for (int e = 0; e < DP / 2; e += 2)
                            ldg256(blk + (int64_t)(j >> 1) * walk_pair_f4(DP) + e, v[e], v[e + 1]);
                    } else {
#pragma unroll
                        for (int e = 0; e < DP / 2; ++e) v[e] = __ldg(blk + (int64_t)(j >> 1) * walk_pair_f4(DP) + e);
                    }
#pragma unroll
                    for (int i = 0; i < R; ++i) q[i] = q_pair<DP>(xc[i], xx[i], cc, v);
                }
#pragma unroll
                for (int i = 0; i < R; ++i) {
                    int k0, k1;
                    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(k0) : "r"(__float_as_uint(q[i].x)), "r"(kmask), "r"(j));
                    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(k1) : "r"(__float_as_uint(q[i].y)), "r"(kmask), "r"(j + 1));
                    const int lo2 = min(k0, k1), hi2 = max(k0, k1);
                    m2[i] = min(min(max(m1[i], lo2), m2[i]), hi2);
                    m1[i] = min(m1[i], lo2);
                }
            }
            steps32 += (unsigned)pm;
            // prefix max of |c'|^2 over the evaluated rows (bounds the error of every key)
            const float cmax = pm > 0 ? __ldg(p.Wmeta + (int64_t)A * kp + ((pm + 1) & ~1) - 1).x : 0.f;
            const float2 *mA = p.Wmeta + (int64_t)A * kp;
#pragma unroll
            for (int i = 0; i < R; ++i) {
                if (!active[i]) continue;
                // rigorous decision (same procedure as the tensor-core epilogue).  Fast paths in
                // the squared domain: a key value v with v > thr = (u_t + epsr)^2 + E has a lower
                // distance bound above u_t, the upper bound of the own cluster's distance.
                const float E = __fmul_ru(kappa, __fadd_ru(xx[i], cmax));
                const float epsr = __fadd_ru(eps, __fmul_ru(1.2e-7f, __fadd_ru(sqrt_up(xx[i]), sqrt_up(cmax))));
                const float ue = __fadd_ru(ut[i], epsr);
                const float thr = __fadd_ru(__fmul_ru(ue, ue), E);
                const float v1 = m1[i] == 0x7fffffff ? INFINITY : __int_as_float(m1[i] & kmask);
                const float v2 = m2[i] == 0x7fffffff ? INFINITY : __int_as_float(m2[i] & kmask);
                bool fallback = false, stay;
                if (!misfit[i]) {
                    stay = v1 > thr;
                } else {
                    // misfit: stays if A is farther than u_t and every candidate but the own
                    // cluster's column is: either all keys exceed thr, or only the best does not
                    // and the best is the own cluster (then any other key is >= m2 > thr)
                    const bool a_far = __fmul_rd(sqrt_dn(xx[i]), p.g_dn) > __fadd_ru(ut[i], eps);
                    stay = a_far && (v1 > thr ||
                                     (v2 > thr && __float_as_int(__ldg(&mA[m1[i] & ~kmask].y)) == aold[i]));
                }
                if (stay) {
                    unew[i] = ut[i];
                } else if (!misfit[i]) {
                    // moves to the best candidate if its interval is clear of the own cluster's
                    // and of every other candidate's (>= m2)
                    const float U1 = __fadd_ru(sqrt_up(__fadd_ru(__fmul_ru(fmaxf(v1, 0.f), qtrunc), E)), epsr);
                    const float L2 = v2 == INFINITY ? INFINITY
                                                    : fmaxf(0.f, __fsub_rd(sqrt_dn(fmaxf(__fsub_rd(v2, E), 0.f)), epsr));
                    if (U1 < fminf(lo[i], L2)) {
                        anew[i] = __float_as_int(__ldg(&mA[m1[i] & ~kmask].y));
                        unew[i] = U1;
                    } else {
                        fallback = true;
                    }
                } else {
                    auto U_of = [&](int key) {
                        const float v = fmaxf(__int_as_float(key & kmask), 0.f);
                        return __fadd_ru(sqrt_up(__fadd_ru(__fmul_ru(v, qtrunc), E)), epsr);
                    };
                    auto L_of = [&](int key) {
                        if (key == 0x7fffffff) return INFINITY;
                        const float v = __int_as_float(key & kmask);
                        return fmaxf(0.f, __fsub_rd(sqrt_dn(fmaxf(__fsub_rd(v, E), 0.f)), epsr));
                    };
                    const int cc1 = m1[i] != 0x7fffffff ? __float_as_int(__ldg(&mA[m1[i] & ~kmask].y)) : -1;
                    const int cc2 = m2[i] != 0x7fffffff ? __float_as_int(__ldg(&mA[m2[i] & ~kmask].y)) : -1;
                    float Uo = ut[i], Lo = lo[i], Ui = INFINITY, Li = INFINITY, Lother = INFINITY;
                    int ci = -1;
                    if (cc1 == aold[i]) {      // own cluster is the best candidate: merge
                        Uo = fminf(Uo, U_of(m1[i])); Lo = fmaxf(Lo, L_of(m1[i]));
                        ci = cc2;
                        if (ci >= 0) { Ui = U_of(m2[i]); Li = L_of(m2[i]); Lother = -1.f; }   // third unknown
                    } else {
                        ci = cc1;
                        if (ci >= 0) { Ui = U_of(m1[i]); Li = L_of(m1[i]); }
                        Lother = L_of(m2[i]);
                    }
                    const float UA = upper_d(xx[i], p.g_up, eps), LA = lower_d(xx[i], p.g_dn, eps);
                    if (Uo < fminf(Li, LA)) {
                        unew[i] = Uo;
                    } else if (UA < fminf(Lo, Li)) {
                        anew[i] = A; unew[i] = UA;
                    } else if (ci >= 0 && Ui < fminf(fminf(Lo, LA), Lother)) {
                        anew[i] = ci; unew[i] = Ui;
                    } else {
                        fallback = true;
                    }
                }
                if (fallback) {
                    ++c_fb32;
                    const uint64_t *nl = p.NL + (int64_t)aold[i] * p.ks;
                    float xr[DP];
                    {
                        const float4 *src = reinterpret_cast<const float4 *>(p.X + (size_t)(row0 + 32 * i + lane) * DP);
#pragma unroll
                        for (int j = 0; j < DP / 4; ++j) {
                            const float4 t = __ldg(src + j);
                            xr[4 * j] = t.x; xr[4 * j + 1] = t.y; xr[4 * j + 2] = t.z; xr[4 * j + 3] = t.w;
                        }
                    }
                    float bq = dist2<DP, CSMEM>(xr, Cn, aold[i]), q2 = INFINITY;
                    int bc = aold[i];
                    for (int j = 0; j < kcols; ++j) {
                        const uint64_t key = __ldg(nl + j);
                        if (!(key_h(key) < ut[i])) break;
                        const int c = key_c(key);
                        const float q = dist2<DP, CSMEM>(xr, Cn, c);
                        q2 = fminf(q2, fmaxf(q, bq));
                        bc = q < bq ? c : bc;
                        bq = fminf(q, bq);
                    }
                    const float ub = upper_d(bq, p.g_up, eps);
                    if (q2 < INFINITY && lower_d(q2, p.g_dn, eps) <= ub) {
                        anew[i] = refine64(p.X + (size_t)(row0 + 32 * i + lane) * DP, p.d, p.C64, k, aold[i], nl, ut[i], &unew[i]);
                        ++c_refined32;
                    } else {
                        anew[i] = bc;
                        unew[i] = ub;
                    }
                }
                // MTI distance count 1 + #{c : H[a][c] < u_t}; misfit rows: deferred
                if (!misfit[i]) {
                    c_dists += (unsigned long long)(1 + pl[i]);
                } else if constexpr (HSMEM) {      // own list's H row is in shared memory
                    c_dists += (unsigned long long)(1 + count_below_s<NH>(sH + aold[i] * NH, ut[i]));
                } else {
                    defer[i] = true;                 // counted by k_mti_count
                }
            }
        }
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const int rb = row0 + 32 * i;
            if constexpr (!HSMEM) {   // deferred counts: per 32-row group: defer[rb + i], dcount[rb / 32]
                const unsigned dm = __ballot_sync(kFull, defer[i]);
                if (defer[i])
                    p.defer[rb + __popc(dm & ((1u << lane) - 1u))] =
                        ((unsigned long long)(uint32_t)aold[i] << 32) | __float_as_uint(ut[i]);
                if (lane == 0 && rb < n) p.dcount[rb / 32] = __popc(dm);
            }
            if (valid[i]) {
                p.a[rb + lane] = anew[i];
                p.u[rb + lane] = unew[i];
            }
            // S3 as a delta (B5): movers are queued in shared memory and their fp64
            // deltas applied 32 at a time, so the REDs run with full warps
            {
                const bool mv = valid[i] && anew[i] != aold[i];
                const unsigned mm = __ballot_sync(kFull, mv);
                if (mm) {
                    c_changed32 += mv;
                    if (mv) {
                        const int slot = mq + __popc(mm & ((1u << lane) - 1u));
                        sQ[slot] = rb + lane; sQ[kQueue + slot] = aold[i]; sQ[2 * kQueue + slot] = anew[i];
                    }
                    mq += __popc(mm);
                    if (mq >= 32) flush_moves();
                }
            }
        }
    }
    flush_moves();
    unsigned long long c_changed = c_changed32, c_clause1 = c_clause132, c_refined = c_refined32,
                       c_fb = c_fb32, steps = steps32;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        c_changed += __shfl_xor_sync(kFull, c_changed, o);
        c_dists += __shfl_xor_sync(kFull, c_dists, o);
        c_clause1 += __shfl_xor_sync(kFull, c_clause1, o);
        c_refined += __shfl_xor_sync(kFull, c_refined, o);
        c_fb += __shfl_xor_sync(kFull, c_fb, o);
    }
    if (lane == 0) {
        if (c_changed) atomicAdd(p.counters + 0, c_changed);
        if (c_dists) atomicAdd(p.counters + 1, c_dists);
        if (c_clause1) atomicAdd(p.counters + 2, c_clause1);
        if (c_refined) atomicAdd(p.counters + 3, c_refined);
        if (steps) atomicAdd(p.counters + 4, steps);
        if (c_fb) atomicAdd(p.counters + 5, c_fb);
    }
}

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

size_t walk_smem(int DP, bool csmem, int k, int whs, bool wh_smem)
{
    const int R = DP <= 16 ? 2 : (DP <= 32 ? KM_WALK_R32 : 1);
    const int k4 = (k + 3) & ~3;
    return (size_t)((csmem ? k * DP : 0) + 2 * k4 + (wh_smem ? k * whs : 0)) * sizeof(float) +
           (size_t)(walk_threads_rt(DP) / 32) * (32 * R * (DP + 2) + 3 * kQueue) * sizeof(float);
}

// rows per lane: 2 where the registers allow (the candidate loads are shared by both rows)
template <int DP> constexpr int walk_r() { return DP <= 16 ? 2 : (DP <= 32 ? KM_WALK_R32 : 1); }

typedef void (*walk_kernel_t)(AssignParams);

template <int DP, bool CSMEM>
static walk_kernel_t walk_pick(int whs, bool hs)
{
    constexpr int R = walk_r<DP>();
    if (hs) {
        switch (whs) {
        case 2: case 4: case 8: case 16: return k_walk<DP, CSMEM, R, 16, true>;
        case 32: return k_walk<DP, CSMEM, R, 32, true>;
        case 64: return k_walk<DP, CSMEM, R, 64, true>;
        case 128: return k_walk<DP, CSMEM, R, 128, true>;
        case 256: return k_walk<DP, CSMEM, R, 256, true>;
        }
    } else {
        switch (whs) {
        case 256: return k_walk<DP, CSMEM, R, 256, false>;
        case 512: return k_walk<DP, CSMEM, R, 512, false>;
        case 1024: return k_walk<DP, CSMEM, R, 1024, false>;
        case 2048: return k_walk<DP, CSMEM, R, 2048, false>;
        case 4096: return k_walk<DP, CSMEM, R, 4096, false>;
        }
    }
    return nullptr;
}

static walk_kernel_t walk_kernel(int DP, bool csmem, int whs, bool hs)
{
    switch (DP * 2 + (csmem ? 1 : 0)) {
    case 8: return walk_pick<4, false>(whs, hs);
    case 9: return walk_pick<4, true>(whs, hs);
    case 16: return walk_pick<8, false>(whs, hs);
    case 17: return walk_pick<8, true>(whs, hs);
    case 32: return walk_pick<16, false>(whs, hs);
    case 33: return walk_pick<16, true>(whs, hs);
    case 64: return walk_pick<32, false>(whs, hs);
    case 65: return walk_pick<32, true>(whs, hs);
    case 128: return walk_pick<64, false>(whs, hs);
    case 129: return walk_pick<64, true>(whs, hs);
    }
    return nullptr;
}

bool walk_supported(int DP) { return DP == 4 || DP == 8 || DP == 16 || DP == 32 || DP == 64; }

cudaError_t launch_walk(int DP, bool csmem, const AssignParams &p, int grid, cudaStream_t st)
{
    walk_kernel_t kern = walk_kernel(DP, csmem, p.whs, p.wh_smem != 0);
    if (!kern) return cudaErrorInvalidValue;
    const size_t sm = walk_smem(DP, csmem, p.k, p.whs, p.wh_smem != 0);
    if (sm > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e != cudaSuccess) return e;
    }
    kern<<<grid, walk_threads_rt(DP), sm, st>>>(p);
    return cudaGetLastError();
}

int walk_grid(int DP, bool csmem, int k, int whs, bool hs, int num_sms)
{
    walk_kernel_t kern = walk_kernel(DP, csmem, whs, hs);
    if (!kern) return num_sms;
    const size_t sm = walk_smem(DP, csmem, k, whs, hs);
    if (sm > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, walk_threads_rt(DP), sm);
    return (per_sm < 1 ? 1 : per_sm) * num_sms;
}

}  // namespace km
