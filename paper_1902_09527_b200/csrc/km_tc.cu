// km_tc.cu — tensor-core (tcgen05, TF32 x3) MTI assignment + fused reduction for sm_100a.
//
// Same method and outputs as k_assign<MODE_MTI_REDUCE> (§3.3, 1026-1053: clause 1,
// tightening, clauses 2/3; §3.2, 1000-1011: fused per-cluster reduction); only the
// evaluation of the surviving candidates moves to the tensor cores.  DESIGN.md "Tensor-core
// MTI".  Per 128-row tile (rows bucketed by cluster, so a tile mostly shares its cluster A):
//
//   1. per row (CUDA cores): u += f(a); clause 1; tighten u = d(x, C[a]) in the direct fp32
//      form (rigorous gamma bound) -> ut; the row's x split into TF32 hi/lo written to smem.
//   2. candidates of the tile = prefix of A's neighbour list NL[A] with H < max ut (a prefix,
//      since NL[A] is sorted by H); their pre-split centroid rows [c_hi | c_hi | c_lo] are
//      staged in smem (cached across tiles of the same cluster).
//   3. one elected thread issues tcgen05.mma.kind::tf32 (M = 128, N = 16..256, K = 3 DP):
//      D[r][j] = x_hi.c_hi + x_lo.c_hi + x_hi.c_lo ~ x . c_j  (error <= (3DP+7) 2^-23 |x||c|)
//      accumulated in TMEM; completion is signalled through an mbarrier (tcgen05.commit).
//   4. epilogue: each thread reads its TMEM lane (tcgen05.ld 32x32b.x16), forms
//      q_j = |x|^2 + |c_j|^2 - 2 D and keeps the best / second best over its own survivors
//      (H[A][c_j] < ut, clauses 2/3).  All q carry one absolute error bound
//      E = (14 DP + 36) 2^-24 (|x|^2 + max |c|^2) (2x the derived bound); if the second
//      best's interval meets the best's, the row falls back to the CUDA-core direct walk,
//      whose own fp32 screen and fp64 refinement make the final decision (exact mode).
//   Rows whose cluster is not A ("misfits") also take the CUDA-core walk.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "km_device.cuh"
#include "km_kernels.cuh"

namespace km {
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ float tf32_rna(float x)
{
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

__device__ __forceinline__ void sts128(uint32_t addr, float a, float b, float c, float d)
{
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" :: "r"(addr), "f"(a), "f"(b), "f"(c), "f"(d));
}

// K-major, no-swizzle UMMA operand layout (core matrices of 8 rows x 16 B): element (r, e)
// of an R-row operand lives at K-block e/8 (R*32 B each), 8-row group r/8 (SBO = 256 B),
// 16-B chunk (e%8)/4 (LBO = 128 B), row r%8 (16 B), word e%4.
__device__ __forceinline__ uint32_t op_off(int r, int e, int R)
{
    return (uint32_t)((e >> 3) * (R * 32) + (r >> 3) * 256 + ((e & 7) >> 2) * 128 + (r & 7) * 16 + (e & 3) * 4);
}

__device__ __forceinline__ uint64_t sdesc(uint32_t addr)
{
    return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)(128 >> 4) << 16) |
           ((uint64_t)(256 >> 4) << 32) | (1ull << 46);   // version 1 (sm_100), no swizzle
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc)
{
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                 :: "r"(tmem_d), "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint32_t mbar)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(mbar));
}

__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t phase)
{
    asm volatile("{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
                 "@P1 bra DONE_%=;\n\tbra WAIT_%=;\n\tDONE_%=:\n\t}" :: "r"(mbar), "r"(phase));
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16])
{
    uint32_t r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

}  // namespace tc

constexpr int kTcRows = 128;

template <int DP, bool CSMEM>
__global__ void __launch_bounds__(kTcRows)
k_mti_tc(AssignParams p)
{
    constexpr int KT = 3 * DP;                  // [x_hi | x_lo | x_hi] . [c_hi | c_hi | c_lo]
    constexpr int G = 8;                        // tiles claimed per work-counter fetch
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) uint64_t s_mbar;
    __shared__ int s_firstA[2][4];
    __shared__ long long s_ahead[2];

    const int k = p.k, W = p.W, ks = p.ks;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    uint8_t *sA = smem;                                          // 128 x KT operand
    uint8_t *sB = sA + kTcRows * KT * 4;                         // W x KT operand
    float4 *sKey = reinterpret_cast<float4 *>(sB + W * KT * 4);  // W x {h, c bits, |c|^2, -}
    float *sC = reinterpret_cast<float *>(sKey + W);             // k x DP (CSMEM)
    float *sF = sC + (CSMEM ? k * DP : 0);
    float *sS = sF + k;
    const uint32_t aBase = tc::smem_u32(sA), bBase = tc::smem_u32(sB), mbar = tc::smem_u32(&s_mbar);

    if (CSMEM) {
        const float4 *src = reinterpret_cast<const float4 *>(p.Cneg);
        float4 *dst = reinterpret_cast<float4 *>(sC);
        for (int i = t; i < k * DP / 4; i += kTcRows) dst[i] = src[i];
    }
    for (int i = t; i < k; i += kTcRows) { sF[i] = p.f[i]; sS[i] = p.s[i]; }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     :: "r"(tc::smem_u32(&s_tmem)), "r"(p.tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(mbar), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;");
        s_ahead[0] = (long long)atomicAdd(p.work, 1) * G;
        s_ahead[1] = (long long)atomicAdd(p.work, 1) * G;
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = s_tmem;
    const uint32_t tlane = tmem + ((uint32_t)(warp * 32) << 16);

    CRow<CSMEM> Cn;
    if constexpr (CSMEM) {
        uint32_t b = tc::smem_u32(sC);
        asm volatile("mov.u32 %0, %0;" : "+r"(b));
        Cn.base = b;
    } else {
        Cn.base = p.Cneg;
    }
    double *acc = p.acc + (int64_t)(blockIdx.x % p.nslab) * k * (DP + 1);
    const float eps = *p.eps;
    const float kappa = (14.f * DP + 44.f) * 5.9604645e-8f;    // (14 DP + 44) 2^-24, DESIGN.md
    const int64_t n = p.n;
    const int64_t ntiles = (n + kTcRows - 1) / kTcRows;
    const bool partial_cols = W - 1 < k - 1;                    // columns do not cover all of NL[A]
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(W >> 3) << 17) |
                           ((uint32_t)(kTcRows >> 4) << 24);   // F32 += TF32 x TF32, K-major, 128 x W

    RunAcc<DP> ra;
    ra.clear();
    unsigned long long c_changed = 0, c_dists = 0, c_clause1 = 0, c_refined = 0;
    unsigned steps = 0;
    unsigned dbg_walk = 0, dbg_uncov = 0, dbg_mis = 0;   // diagnostics (counters 5..7)
    uint32_t phase = 0;
    int colA = -1;                        // cluster whose columns [A | NL[A][0..W-1)] are staged

    int64_t g_cur = s_ahead[0], g_next = s_ahead[1];
    __syncthreads();                      // everyone has read s_ahead before it is reused
    int64_t tile = g_cur;
    float nx[DP];
    int na = 0;
    float nu = 0.f;
    auto load = [&](int64_t tl) {
        const int64_t r = tl * kTcRows + t;
        const bool v = tl < ntiles && r < n;
        const float4 *xr = reinterpret_cast<const float4 *>(p.X + (v ? r : 0) * DP);
#pragma unroll
        for (int j = 0; j < DP / 4; ++j) {
            float4 q = v ? __ldg(xr + j) : make_float4(0.f, 0.f, 0.f, 0.f);
            nx[4 * j] = q.x; nx[4 * j + 1] = q.y; nx[4 * j + 2] = q.z; nx[4 * j + 3] = q.w;
        }
        na = v ? __ldg(p.a + r) : 0;
        nu = v ? __ldg(p.u + r) : 0.f;
    };
    if (tile < ntiles) load(tile);
    int it = 0;

    while (tile < ntiles) {
        const int par = it & 1;
        const int64_t row = tile * kTcRows + t;
        const bool valid = row < n;
        float x[DP];
#pragma unroll
        for (int j = 0; j < DP; ++j) x[j] = nx[j];
        const int aold = na;
        const bool switching = !(tile + 1 < min(g_cur + G, ntiles));
        if (switching && t == 0) s_ahead[par ^ 1] = (long long)atomicAdd(p.work, 1) * G;

        // ---- 1. per row: drift, clause 1, tighten (direct fp32 form), operand row -----------
        const float uu = valid ? __fadd_ru(nu, sF[aold]) : 0.f;         // u += f(a)
        const bool c1 = valid && uu <= sS[aold];                          // clause 1
        c_clause1 += c1;
        const bool active = valid && !c1;
        float q_own = INFINITY, ut = 0.f, xx = 0.f;
        if (active) {
            q_own = dist2<DP, CSMEM>(x, Cn, aold);                         // U(u) = d(x, C[a])
            ut = upper_d(q_own, p.g_up, eps);
        }
        {
            const unsigned am = __ballot_sync(kFull, active);
            const int fa = am ? __shfl_sync(kFull, aold, __ffs(am) - 1) : -1;
            if (lane == 0) s_firstA[par][warp] = fa;
        }
        __syncthreads();                                                   // (1)
        int64_t tile_next = tile + 1;
        if (switching) {
            g_cur = g_next;
            g_next = s_ahead[par ^ 1];
            tile_next = g_cur;
        }
        int A = -1;
#pragma unroll
        for (int w = 3; w >= 0; --w) A = s_firstA[par][w] >= 0 ? s_firstA[par][w] : A;

        float bq = q_own, q2 = INFINITY;
        int bc = aold, ns = active ? 1 : 0;
        bool walk = active;                      // rows not decided by the tensor cores
        bool prefetched = false;

        if (A >= 0) {
            const bool misfit = active && aold != A;
            // per-row column threshold: own rows take NL[A] candidates with H < ut (clauses 2/3);
            // misfit rows (cluster a != A) take the columns c with 2 H[A][c] - d(x,A) < d_best,
            // i.e. H[A][c] < (ut + d(x,A)) / 2 (triangle inequality around A), plus A itself
            float T = ut;
            if (misfit) {
                const float dA = upper_d(dist2<DP, CSMEM>(x, Cn, A), p.g_up, eps);
                T = __fmul_ru(__fadd_ru(ut, dA), 0.5f);
            }
            // ---- 2. operands, centred on C[A] (translation-invariant distances, small norms):
            //      row r: x' = x - C[A];  column j: c'_j = C[c_j] - C[A]  (fp32), split into TF32
            //      hi + lo, A' = [x'_hi | x'_lo | x'_hi], B' = [c'_hi | c'_hi | c'_lo]
            {
                float xc[DP];
#pragma unroll
                for (int j4 = 0; j4 < DP / 4; ++j4) {
                    const float4 ca = Cn.ld(A, DP, 4 * j4);        // -C[A]
                    xc[4 * j4] = x[4 * j4] + ca.x; xc[4 * j4 + 1] = x[4 * j4 + 1] + ca.y;
                    xc[4 * j4 + 2] = x[4 * j4 + 2] + ca.z; xc[4 * j4 + 3] = x[4 * j4 + 3] + ca.w;
                }
#pragma unroll
                for (int j = 0; j < DP; ++j) xx = fmaf(xc[j], xc[j], xx);
#pragma unroll
                for (int c = 0; c < DP / 4; ++c) {
                    float h[4], l[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        h[i] = tc::tf32_rna(xc[4 * c + i]);
                        l[i] = tc::tf32_rna(xc[4 * c + i] - h[i]);
                    }
                    tc::sts128(aBase + tc::op_off(t, 4 * c, kTcRows), h[0], h[1], h[2], h[3]);
                    tc::sts128(aBase + tc::op_off(t, DP + 4 * c, kTcRows), l[0], l[1], l[2], l[3]);
                    tc::sts128(aBase + tc::op_off(t, 2 * DP + 4 * c, kTcRows), h[0], h[1], h[2], h[3]);
                }
            }
            if (A != colA) {                      // columns [A | NL[A][0..W-1)], cached while A repeats
                for (int jj = t; jj < W; jj += kTcRows) {
                    uint64_t key;
                    if (jj == 0) key = ((uint64_t)__float_as_uint(-INFINITY) << 32) | (uint32_t)A;
                    else key = jj - 1 < ks ? __ldg(p.NL + (int64_t)A * ks + (jj - 1)) : kSentinel;
                    const int c = key_c(key);
                    float cs = 0.f;
#pragma unroll
                    for (int j4 = 0; j4 < DP / 4; ++j4) {
                        const float4 ca = Cn.ld(A, DP, 4 * j4), cj = Cn.ld(c, DP, 4 * j4);
                        const float v[4] = {ca.x - cj.x, ca.y - cj.y, ca.z - cj.z, ca.w - cj.w};  // c_j - c_A
                        float h[4], l[4];
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            cs = fmaf(v[i], v[i], cs);
                            h[i] = tc::tf32_rna(v[i]);
                            l[i] = tc::tf32_rna(v[i] - h[i]);
                        }
                        tc::sts128(bBase + tc::op_off(jj, 4 * j4, W), h[0], h[1], h[2], h[3]);
                        tc::sts128(bBase + tc::op_off(jj, DP + 4 * j4, W), h[0], h[1], h[2], h[3]);
                        tc::sts128(bBase + tc::op_off(jj, 2 * DP + 4 * j4, W), l[0], l[1], l[2], l[3]);
                    }
                    sKey[jj] = make_float4(key_h(key), __int_as_float(c), cs, 0.f);
                }
                colA = A;
            }
            tc::fence_async_smem();
            tc::fence_before();
            __syncthreads();                                               // (2)
            tc::fence_after();
            // ---- 3. MMA: D[128 x W] = A' . B'^T ----------------------------------------------
            if (t == 0) {
#pragma unroll
                for (int kb = 0; kb < KT / 8; ++kb)
                    tc::mma_tf32(tmem, tc::sdesc(aBase + kb * kTcRows * 32), tc::sdesc(bBase + kb * W * 32),
                                 idesc, kb > 0);
                tc::mma_commit(mbar);
            }
            load(tile_next);                      // overlap the next tile's loads with the MMA
            prefetched = true;
            tc::mbar_wait(mbar, phase);
            phase ^= 1;
            tc::fence_after();
            // ---- 4. epilogue: per-row best / second best over the taken columns (clauses 2/3 for
            //      own rows, the triangle bound around A for misfits; never the row's own
            //      cluster, which the direct tighten already evaluated)
            int j0 = 0;
            for (; j0 < W; j0 += 16) {
                if (!__any_sync(kFull, active && sKey[j0].x < T)) break;
                float v[16];
                tc::tmem_ld16(tlane + (uint32_t)j0, v);
                steps += 16;
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const float4 kk = sKey[j0 + i];
                    const int c = __float_as_int(kk.y);
                    const bool take = active && kk.x < T && c != aold;
                    float q = fmaf(-2.f, v[i], xx + kk.z);
                    q = take ? q : INFINITY;
                    ns += (take && !misfit);
                    q2 = fminf(q2, fmaxf(q, bq));
                    bc = q < bq ? c : bc;
                    bq = fminf(q, bq);
                }
            }
            tc::fence_before();
            if (active) {
                // the staged columns cover the row's candidates unless its prefix runs past them
                const bool covered = !partial_cols || !(sKey[W - 1].x < T);
                // every taken column has 2 H < 2 T, so |c'|^2 <= 4 T^2 (1 + 2^-20): one bound per row
                const float E = kappa * fmaf(4.000004f * T, T, xx);
                const float ub = __fadd_ru(__fsqrt_ru(__fadd_ru(bq, E)), eps);
                const float lb2 = q2 < INFINITY ? __fsub_rd(__fsqrt_rd(fmaxf(__fsub_rd(q2, E), 0.f)), eps) : INFINITY;
                walk = !covered || lb2 <= ub;            // TC-ambiguous or uncovered: direct walk
                dbg_walk += walk;
                dbg_uncov += !covered;
                dbg_mis += misfit;
                if (!walk && misfit) {
                    // MTI distance count of this row: 1 + #{c : H[a][c] < ut} (binary search)
                    const uint64_t *nl = p.NL + (int64_t)aold * ks;
                    int lo = 0, hi = k - 1;
                    while (lo < hi) {
                        const int mid = (lo + hi) >> 1;
                        if (key_h(__ldg(nl + mid)) < ut) lo = mid + 1; else hi = mid;
                    }
                    ns = 1 + lo;
                }
            }
        }
        if (!prefetched) load(tile_next);

        // ---- 5. rows left to the CUDA cores: direct-form walk + exact-mode decision ---------
        int anew = aold;
        float unew = uu;
        if (active) {
            if (walk) { bq = q_own; q2 = INFINITY; bc = aold; ns = 1; }
            const uint64_t *nl = p.NL + (int64_t)aold * ks;
            bool walking = walk;
            if (__any_sync(__activemask(), walking)) {
                ulonglong2 kp = walking ? __ldg(reinterpret_cast<const ulonglong2 *>(nl)) : make_ulonglong2(kSentinel, kSentinel);
                for (int j = 0;; j += 2) {
                    const bool w0 = walking && key_h(kp.x) < ut;
                    const bool w1 = w0 && key_h(kp.y) < ut;
                    if (!__any_sync(__activemask(), w0)) break;
                    steps += 2;
                    const ulonglong2 np = w1 ? __ldg(reinterpret_cast<const ulonglong2 *>(nl + j + 2)) : make_ulonglong2(kSentinel, kSentinel);
                    const int c0 = key_c(kp.x), c1 = key_c(kp.y);
                    float qa = dist2<DP, CSMEM>(x, Cn, c0);
                    float qb = dist2<DP, CSMEM>(x, Cn, c1);
                    qa = w0 ? qa : INFINITY;
                    qb = w1 ? qb : INFINITY;
                    ns += (int)w0 + (int)w1;
                    q2 = fminf(q2, fmaxf(qa, bq)); bc = qa < bq ? c0 : bc; bq = fminf(qa, bq);
                    q2 = fminf(q2, fmaxf(qb, bq)); bc = qb < bq ? c1 : bc; bq = fminf(qb, bq);
                    walking = w1;
                    kp = np;
                }
            }
            if (walk) {
                const float ub = upper_d(bq, p.g_up, eps);
                const bool amb = q2 < INFINITY && lower_d(q2, p.g_dn, eps) <= ub;
                if (amb) {
                    anew = refine64(p.X + row * DP, p.d, p.C64, k, aold, nl, ut, &unew);
                    ++c_refined;
                } else {
                    anew = bc;
                    unew = ub;
                }
            } else {
                anew = bc;
                // tight bound for the next pass: direct-form distance to the winner
                unew = bc == aold ? ut : upper_d(dist2<DP, CSMEM>(x, Cn, bc), p.g_up, eps);
            }
            c_dists += (unsigned long long)ns;
        }
        if (valid) {
            p.a[row] = anew;
            p.u[row] = unew;
            c_changed += (anew != aold);
        }
        reduce_batch<DP>(ra, x, anew, valid, acc, p.d, lane);
        tile = tile_next;
        ++it;
    }
    ra.flush(acc, p.d, lane);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        c_changed += __shfl_xor_sync(kFull, c_changed, o);
        c_dists += __shfl_xor_sync(kFull, c_dists, o);
        c_clause1 += __shfl_xor_sync(kFull, c_clause1, o);
        c_refined += __shfl_xor_sync(kFull, c_refined, o);
    }
    if (lane == 0) {
        if (c_changed) atomicAdd(p.counters + 0, c_changed);
        if (c_dists) atomicAdd(p.counters + 1, c_dists);
        if (c_clause1) atomicAdd(p.counters + 2, c_clause1);
        if (c_refined) atomicAdd(p.counters + 3, c_refined);
        if (steps) atomicAdd(p.counters + 4, (unsigned long long)steps);
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        dbg_walk += __shfl_xor_sync(kFull, dbg_walk, o);
        dbg_uncov += __shfl_xor_sync(kFull, dbg_uncov, o);
        dbg_mis += __shfl_xor_sync(kFull, dbg_mis, o);
    }
    if (lane == 0) {
        atomicAdd(p.counters + 5, (unsigned long long)dbg_walk);
        atomicAdd(p.counters + 6, (unsigned long long)dbg_uncov);
        atomicAdd(p.counters + 7, (unsigned long long)dbg_mis);
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(p.tmem_cols));
}

size_t tc_smem(int DP, bool csmem, int k, int W)
{
    const int KT = 3 * DP;
    return (size_t)kTcRows * KT * 4 + (size_t)W * KT * 4 + (size_t)W * 16 +
           (size_t)((csmem ? k * DP : 0) + 2 * k) * 4;
}

template <int DP, bool CSMEM>
static cudaError_t launch_tc_t(const AssignParams &p, int grid, cudaStream_t st)
{
    const size_t sm = tc_smem(DP, CSMEM, p.k, p.W);
    cudaError_t e = cudaFuncSetAttribute(k_mti_tc<DP, CSMEM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    k_mti_tc<DP, CSMEM><<<grid, kTcRows, sm, st>>>(p);
    return cudaGetLastError();
}

template <int DP, bool CSMEM>
static int tc_grid_t(int k, int W, int tmem_cols, int num_sms)
{
    const size_t sm = tc_smem(DP, CSMEM, k, W);
    cudaError_t e1 = cudaFuncSetAttribute(k_mti_tc<DP, CSMEM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int per_sm = 0;
    cudaError_t e2 = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mti_tc<DP, CSMEM>, kTcRows, sm);
    // The occupancy API reports 1 CTA/SM for kernels that allocate TMEM; compute the residency
    // from registers, shared memory and TMEM columns instead.
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k_mti_tc<DP, CSMEM>);
    int dev = 0, smem_sm = 0, regs_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
    const int regs_cta = ((fa.numRegs + 7) & ~7) * kTcRows;
    const int by_regs = regs_sm / std::max(1, regs_cta);
    const int by_smem = smem_sm / (int)(sm + fa.sharedSizeBytes + 1024);
    const int by_tmem = 512 / tmem_cols;
    const int calc = std::min(std::min(by_regs, by_smem), std::min(by_tmem, 16));
    if (getenv("KM_DEBUG"))
        fprintf(stderr, "[km] tc grid: DP=%d smem=%zu W=%d cols=%d occ_api=%d regs=%d by_regs=%d by_smem=%d by_tmem=%d -> %d (%s/%s)\n",
                DP, sm, W, tmem_cols, per_sm, fa.numRegs, by_regs, by_smem, by_tmem, calc,
                cudaGetErrorString(e1), cudaGetErrorString(e2));
    per_sm = calc;
    return std::max(1, per_sm) * num_sms;
}

bool tc_supported(int DP) { return DP == 8 || DP == 16 || DP == 32; }

cudaError_t launch_mti_tc(int DP, bool csmem, const AssignParams &p, int grid, cudaStream_t st)
{
    switch (DP * 2 + (csmem ? 1 : 0)) {
    case 16: return launch_tc_t<8, false>(p, grid, st);
    case 17: return launch_tc_t<8, true>(p, grid, st);
    case 32: return launch_tc_t<16, false>(p, grid, st);
    case 33: return launch_tc_t<16, true>(p, grid, st);
    case 64: return launch_tc_t<32, false>(p, grid, st);
    case 65: return launch_tc_t<32, true>(p, grid, st);
    }
    return cudaErrorInvalidValue;
}

int mti_tc_grid(int DP, bool csmem, int k, int W, int tmem_cols, int num_sms)
{
    switch (DP * 2 + (csmem ? 1 : 0)) {
    case 16: return tc_grid_t<8, false>(k, W, tmem_cols, num_sms);
    case 17: return tc_grid_t<8, true>(k, W, tmem_cols, num_sms);
    case 32: return tc_grid_t<16, false>(k, W, tmem_cols, num_sms);
    case 33: return tc_grid_t<16, true>(k, W, tmem_cols, num_sms);
    case 64: return tc_grid_t<32, false>(k, W, tmem_cols, num_sms);
    case 65: return tc_grid_t<32, true>(k, W, tmem_cols, num_sms);
    }
    return num_sms;
}

}  // namespace km
