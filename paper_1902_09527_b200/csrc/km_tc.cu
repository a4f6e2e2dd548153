// km_tc.cu — tensor-core (tcgen05, TF32 x3) MTI assignment + fused fp64 reduction for sm_100a.
//
// Same method and outputs as k_assign<MODE_MTI_REDUCE> (§3.3, 1026-1053: drift,
// clause 1, tightening U(u), clauses 2/3; §3.2, 1000-1011: fused per-cluster
// reduction); only the evaluation of the surviving candidates moves to the tensor cores.
// DESIGN.md "Tensor-core MTI".
//
// Rows are stored bucketed by cluster, so a 128-row tile mostly shares one cluster A (the
// cluster of its middle row).  Per tile, software-pipelined with the previous tile:
//
//   load     thread 0 streams tiles [x | a | u] into a STAGES-deep shared-memory ring with
//            cp.async.bulk (TMA bulk copies) + mbarrier complete_tx, tiles claimed in chunks
//            from a global counter (dynamic load balance, clusters stay contiguous per chunk)
//   prep(i)  per row (CUDA cores): u += f(a); clause 1 (u <= s(a) -> keep, 0 distances);
//            else centre x' = x - C^[A], tighten u_t = d(x, C^[a]) (direct fp32 form, rigorous
//            bound), column threshold T (= u_t for rows of A; (u_t + d(x,A))/2 for the other
//            rows: triangle inequality around A), p = #{j : H[A][j] < T} by binary search;
//            A operand row [x'hi | x'lo | x'hi | xx_hi | xx_lo | 1 | 1 | 0..] written to smem
//   mma(i)   one thread: D[128 x N] = A . B^T, tcgen05.mma.kind::tf32, K = KT, N = max p of
//            the tile rounded up to 16; B = k_prep's per-cluster block for A (columns = A's
//            neighbour list in ascending H, rows [-2c'hi | -2c'hi | -2c'lo | 1 | 1 | cc_hi |
//            cc_lo]) so D[r][j] ~ |x' - c'_j|^2 directly; committed to an mbarrier; TMEM is
//            double buffered so mma(i) overlaps epilogue(i-1)
//   epi(i-1) per row: tcgen05.ld 32x32b.x16 chunks while any lane of the warp has p > chunk;
//            packed keys (q bits & ~0xff | column) -> best / second best by integer min/max;
//            rigorous intervals decide the winner or send the row to the CUDA-core walk
//            (direct form + fp64 refinement: exact mode); a/u written; fp64 warp reduction
//
// Error model (measured on B200 by tools/probes/tc_acc_probe.cu:
// accumulation error <= (K/4 + 2) 2^-24 sum|a_k b_k|):  |D - |x' - c'|^2| <= E with
//   E = kappa (xx + cmax),  kappa = 2 (25 + DP/4 + KT/2) 2^-24  (2x the derived bound)
// where cmax bounds |c'_j|^2 over the columns the row's warp reads.  Centring roundings add
// <= 2^-24 (|x'| + |c'|) on the distance scale.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <initializer_list>

#include "km_device.cuh"
#include "km_kernels.cuh"
#include "km_tc_common.cuh"

namespace km {


constexpr int kTcRows = 128;
constexpr int kTcPrepWarps = 4;                  // warps 0-3: prep (one row per thread)
constexpr int kTcEpiWarp0 = 4;                   // warps 4-7: epilogue (TMEM lane quadrant = warp % 4)
constexpr int kTcProdWarp = 8;                   // warp 8: TMA producer
constexpr int kTcMmaWarp = 9;                    // warp 9: MMA issuer
constexpr int kTcThreads = 320;

__host__ __device__ constexpr int tc_kt(int DP) { return ((3 * DP + 4) + 7) & ~7; }

__host__ __device__ inline int tc_nmeta(int nmax) { int m = 16; while (m < nmax) m <<= 1; return m; }

// per-row state handed from the prep warps to the epilogue warps (one slot per TMEM buffer)
struct TcRow {
    int a;          // assignment before the pass
    int flags;      // bit0 valid, bit1 active (clause 1 failed), bit2 misfit (a != A), bit3 uncovered
    float uu;       // u + f(a) (clause-1 rows keep it)
    float ut;       // tightened upper bound of d(x, C[a]) (direct form)
    float lo;       // lower bound of d(x, C[a])
    float xx;       // |x - C^[A]|^2 (direct form)
    int p;          // columns below the row's threshold
    int pad;
};

struct TcInfo {      // per TMEM buffer: the tile in flight
    long long tile;  // -1 = end of stream
    int A;           // tile cluster
    int bslot;       // B operand slot
    int mslot;       // column-metadata slot
    int N;           // MMA columns (0: no MMA)
    int pw[4];       // per-warp columns the epilogue reads
};

struct TcCfg {       // pipeline depths and shared-memory layout (byte offsets, 1024-aligned base)
    int S, NA, NB;   // ring stages, A-operand buffers, B-operand buffers
    int stage_bytes, ring, aop, bop, bmeta, rstate, sc, sf, ss, total;
};

__host__ __device__ inline TcCfg tc_cfg(int DP, bool csmem, int k, int nmax, int S, int NA, int NB)
{
    TcCfg L;
    const int KT = tc_kt(DP);
    L.S = S; L.NA = NA; L.NB = NB;
    L.stage_bytes = kTcRows * DP * 4 + 2 * kTcRows * 4;
    L.ring = 0;
    L.aop = (L.ring + S * L.stage_bytes + 127) & ~127;
    L.bop = L.aop + NA * kTcRows * KT * 4;
    L.bmeta = L.bop + NB * nmax * KT * 4;
    L.rstate = L.bmeta + 2 * tc_nmeta(nmax) * 16;
    L.sc = L.rstate + 2 * kTcRows * (int)sizeof(TcRow);
    L.sf = L.sc + (csmem ? k * DP * 4 : 0);
    L.ss = L.sf + k * 4;
    L.total = L.ss + k * 4;
    return L;
}

// number of keys h[0..M) below T, M = power of two, keys ascending with NaN padding (NaN never
// compares below): branch-free lower bound in log2(M) fixed steps
template <int M>
__device__ __forceinline__ int count_below(const float4 *meta, float T)
{
    int base = 0;
#pragma unroll
    for (int half = M >> 1; half >= 1; half >>= 1)
        base = meta[base + half - 1].x < T ? base + half : base;
    return base + (meta[base].x < T ? 1 : 0);
}


__device__ __forceinline__ float tc_fmin3(float a, float b, float c)
{
    float r;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

// SCREEN (the "tensor-screen" engine): the epilogue keeps only the smallest column value of each
// row (the own column masked for rows of another cluster), decides the rows that provably stay
// and queues the rest (p.qrow / p.qcnt per 32-row group) for k_resolve (km_screen.cu), which
// takes the exact-mode decision and applies the moves.
template <int DP, bool CSMEM, int NMETA, bool SCREEN>
__global__ void __launch_bounds__(kTcThreads, 2)
k_mti_tc(AssignParams p, TcCfg L)
{
    constexpr int KT = tc_kt(DP);
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t s_full[8], s_sfree[8];
    __shared__ __align__(8) uint64_t s_aready[2], s_accfull[2], s_tfree[2];
    __shared__ __align__(8) uint64_t s_bbar[2];
    __shared__ long long s_meta[8];
    __shared__ TcInfo s_info[2];
    __shared__ uint32_t s_tmem;

    const int k = p.k, NMAX = p.nmax, S = L.S;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const uint32_t sbase = tc::smem_u32(smem);
    float *sC = reinterpret_cast<float *>(smem + L.sc);
    float *sF = reinterpret_cast<float *>(smem + L.sf);
    float *sS = reinterpret_cast<float *>(smem + L.ss);
    TcRow *rstate = reinterpret_cast<TcRow *>(smem + L.rstate);
    const float4 *meta0 = reinterpret_cast<const float4 *>(smem + L.bmeta);

    if (CSMEM) {
        const float4 *src = reinterpret_cast<const float4 *>(p.Cneg);
        float4 *dst = reinterpret_cast<float4 *>(sC);
        for (int i = t; i < k * DP / 4; i += kTcThreads) dst[i] = src[i];
    }
    for (int i = t; i < k; i += kTcThreads) { sF[i] = p.f[i]; sS[i] = p.s[i]; }
    {   // zero the A operand buffers once (rows of clause-1 threads are never written)
        float4 *za = reinterpret_cast<float4 *>(smem + L.aop);
        for (int i = t; i < L.NA * kTcRows * KT / 4; i += kTcThreads) za[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (warp == kTcMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     :: "r"(tc::smem_u32(&s_tmem)), "r"(p.tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) {
        for (int s = 0; s < S; ++s) {
            tc::mbar_init(tc::smem_u32(&s_full[s]), 1);
            tc::mbar_init(tc::smem_u32(&s_sfree[s]), 4);
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(tc::smem_u32(&s_aready[b]), kTcPrepWarps);
            tc::mbar_init(tc::smem_u32(&s_accfull[b]), 1);
            tc::mbar_init(tc::smem_u32(&s_tfree[b]), 4);
            tc::mbar_init(tc::smem_u32(&s_bbar[b]), 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const int64_t n = p.n;
    const int64_t ntiles = (n + kTcRows - 1) / kTcRows;

    if (warp == kTcProdWarp) {
        // ================= producer: tiles [x | a | u] -> ring stages (TMA bulk copies) ========
        if (lane == 0) {
            const int G = p.tile_chunk;
            int64_t q_next = 0, q_end = 0;
            for (int L_ = 0;; ++L_) {
                const int s = L_ % S;
                if (L_ >= S) tc::mbar_wait(tc::smem_u32(&s_sfree[s]), (uint32_t)(((L_ / S) - 1) & 1));
                if (q_next >= q_end) {
                    const int64_t c = atomicAdd(p.work, 1);
                    q_next = c * G;
                    q_end = q_next + G;
                }
                const int64_t tl = q_next < ntiles ? q_next : -1;
                ++q_next;
                s_meta[s] = tl;
                const uint32_t mb = tc::smem_u32(&s_full[s]);
                if (tl < 0) { tc::mbar_arrive(mb); break; }
                const uint32_t xb = kTcRows * DP * 4, ab = kTcRows * 4;
                tc::mbar_arrive_tx(mb, xb + 2 * ab);
                const uint32_t dst = sbase + L.ring + s * L.stage_bytes;
                tc::bulk_g2s(dst, p.X + tl * kTcRows * DP, xb, mb);
                tc::bulk_g2s(dst + xb, p.a + tl * kTcRows, ab, mb);
                tc::bulk_g2s(dst + xb + ab, p.u + tl * kTcRows, ab, mb);
            }
        }
    } else if (warp == kTcMmaWarp) {
        // ================= MMA issuer: D[b] = A[i % NA] . B[slot]^T ==========================
        if (lane == 0) {
            const uint32_t idesc_base = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kTcRows >> 4) << 24);
            for (int i = 0;; ++i) {
                const int b = i & 1;
                tc::mbar_wait(tc::smem_u32(&s_aready[b]), (uint32_t)((i >> 1) & 1));
                tc::fence_after();
                const TcInfo &inf = s_info[b];
                if (inf.tile < 0) { tc::mbar_arrive(tc::smem_u32(&s_accfull[b])); break; }
                const int N = inf.N;
                // TMEM buffer b was released by the epilogue of tile i - 2 (the prep warps waited
                // for that before handing over tile i)
                if (N > 0) {
                    const uint32_t idesc = idesc_base | ((uint32_t)(N >> 3) << 17);
                    const uint32_t ab = sbase + L.aop + (uint32_t)((i % L.NA) * kTcRows * KT * 4);
                    const uint32_t bb = sbase + L.bop + (uint32_t)(inf.bslot * NMAX * KT * 4);
#pragma unroll
                    for (int kb = 0; kb < KT / 8; ++kb)
                        tc::mma_tf32(s_tmem + (uint32_t)(b * NMAX), tc::sdesc(ab + kb * kTcRows * 32),
                                     tc::sdesc(bb + kb * NMAX * 32), idesc, kb > 0);
                    tc::mma_commit(tc::smem_u32(&s_accfull[b]));
                } else {
                    tc::mbar_arrive(tc::smem_u32(&s_accfull[b]));
                }
            }
        }
    } else if (warp < kTcPrepWarps) {
        // ================= prep: bounds, clause 1, tightening, A operand ====================
        const float eps = *p.eps;
        const int kcols = min(NMAX, k - 1);
        const bool full_list = kcols == k - 1;
        CRow<CSMEM> Cn;
        if constexpr (CSMEM) Cn.base = tc::smem_u32(sC); else Cn.base = p.Cneg;
        int slotA[2] = {-1, -1};                 // cluster whose B block / metadata sits in a slot
        long long slotLast[2] = {-1, -1};        // last tile that used the slot
        int bcur = 0;
        uint32_t bpar[2] = {0u, 0u};
        unsigned long long c_clause1 = 0;
        for (int i = 0;; ++i) {
            const int s = i % S, b = i & 1;
            tc::mbar_wait(tc::smem_u32(&s_full[s]), (uint32_t)((i / S) & 1));
            const int64_t tile = s_meta[s];
            // buffers of tile i - 2 (A operand when NA = 2, row state, TMEM) are free once its
            // epilogue finished
            if (i >= 2) tc::mbar_wait(tc::smem_u32(&s_tfree[b]), (uint32_t)(((i - 2) >> 1) & 1));
            if (L.NA == 1 && i >= 1)    // single A buffer: the previous MMA must have consumed it
                tc::mbar_wait(tc::smem_u32(&s_accfull[(i - 1) & 1]), (uint32_t)(((i - 1) >> 1) & 1));
            if (tile < 0) {
                if (t == 0) s_info[b].tile = -1;
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(tc::smem_u32(&s_aready[b]));
                break;
            }
            const uint8_t *stage = smem + L.ring + s * L.stage_bytes;
            const float *sx = reinterpret_cast<const float *>(stage);
            const int32_t *sa = reinterpret_cast<const int32_t *>(stage + kTcRows * DP * 4);
            const float *su = reinterpret_cast<const float *>(stage + kTcRows * DP * 4 + kTcRows * 4);
            const int vrows = (int)(n - tile * kTcRows < kTcRows ? n - tile * kTcRows : kTcRows);
            const int A = sa[vrows >> 1];                 // tile cluster: its middle row's
            // column block of A: reuse a slot, or load it into the other one
            int mslot;
            if (slotA[bcur] == A) {
                mslot = bcur;
            } else if (slotA[bcur ^ 1] == A && L.NB == 2) {
                mslot = bcur ^ 1;
            } else {
                mslot = bcur ^ 1;
                // the slot's previous user must be done: its epilogue (metadata) and MMA (B block)
                const long long last = slotLast[mslot];
                if (last >= 0 && last == i - 1)
                    tc::mbar_wait(tc::smem_u32(&s_tfree[last & 1]), (uint32_t)((last >> 1) & 1));
                if (L.NB == 1 && i >= 1)  // single B block: the previous MMA must be done
                    tc::mbar_wait(tc::smem_u32(&s_accfull[(i - 1) & 1]), (uint32_t)(((i - 1) >> 1) & 1));
                // all four prep warps are past their reads of the old slot (named barrier)
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (t == 0) {
                    const uint32_t bb = tc::smem_u32(&s_bbar[mslot]);
                    const int bsl = L.NB == 2 ? mslot : 0;
                    const uint32_t opb = (uint32_t)(NMAX * KT * 4), mtb = (uint32_t)(NMETA * 16);
                    tc::mbar_arrive_tx(bb, opb + mtb);
                    tc::bulk_g2s(sbase + L.bop + (uint32_t)(bsl * NMAX * KT * 4), p.Bop + (int64_t)A * NMAX * KT, opb, bb);
                    tc::bulk_g2s(sbase + L.bmeta + (uint32_t)(mslot * NMETA * 16), p.Bmeta + (int64_t)A * NMETA, mtb, bb);
                }
                tc::mbar_wait(tc::smem_u32(&s_bbar[mslot]), bpar[mslot]);
                bpar[mslot] ^= 1u;
                slotA[mslot] = A;
                bcur = mslot;
            }
            slotLast[mslot] = i;
            const float4 *meta = meta0 + mslot * NMETA;

            const int64_t row = tile * kTcRows + t;
            const bool valid = row < n;
            float x[DP];
#pragma unroll
            for (int j = 0; j < DP; j += 4) {
                const float4 v = *reinterpret_cast<const float4 *>(sx + t * DP + j);
                x[j] = v.x; x[j + 1] = v.y; x[j + 2] = v.z; x[j + 3] = v.w;
            }
            const int aold = valid ? sa[t] : 0;
            const float uu = valid ? __fadd_ru(su[t], sF[aold]) : 0.f;       // u += f(a)
            const bool c1 = valid && uu <= sS[aold];                           // clause 1
            const bool active = valid && !c1;
            const bool misfit = active && aold != A;
            c_clause1 += c1;
            TcRow st;
            st.a = aold; st.uu = uu; st.xx = 0.f; st.ut = 0.f; st.lo = 0.f; st.p = 0; st.pad = -1;
            if (SCREEN && misfit) st.pad = p.rank[(int64_t)A * k + aold];   // own column in A's list
            int flags = (valid ? 1 : 0) | (active ? 2 : 0) | (misfit ? 4 : 0);
            if (active) {
                // x' = x - C^[A] in the direct form's arithmetic (x + (-c)), xx = |x'|^2
                float xh[DP];
                float2 acc0 = make_float2(0.f, 0.f), acc1 = make_float2(0.f, 0.f);
#pragma unroll
                for (int j = 0; j < DP; j += 4) {
                    const float4 c = Cn.ld(A, DP, j);
                    const float2 t0 = add2(make_float2(x[j], x[j + 1]), make_float2(c.x, c.y));
                    const float2 t1 = add2(make_float2(x[j + 2], x[j + 3]), make_float2(c.z, c.w));
                    xh[j] = t0.x; xh[j + 1] = t0.y; xh[j + 2] = t1.x; xh[j + 3] = t1.y;
                    acc0 = fma2(t0, t0, acc0);
                    acc1 = fma2(t1, t1, acc1);
                }
                const float2 s2 = add2(acc0, acc1);
                const float xx = s2.x + s2.y;
                st.xx = xx;
                float T;
                if (!misfit) {
                    st.ut = upper_d(xx, p.g_up, eps);
                    st.lo = lower_d(xx, p.g_dn, eps);
                    T = st.ut;
                } else {
                    // misfit row: own distance in the direct form; columns by the triangle bound
                    // around A: any c with 2 H[A][c] - d(x,A) >= u_t cannot beat a (and the own
                    // cluster itself has H[A][a] <= (u_t + d(x,A)) / 2, so it is a column)
                    const float qo = dist2<DP, CSMEM>(x, Cn, aold);
                    st.ut = upper_d(qo, p.g_up, eps);
                    st.lo = lower_d(qo, p.g_dn, eps);
                    T = __fmul_ru(__fadd_ru(st.ut, upper_d(xx, p.g_up, eps)), 0.5f);
                }
                st.p = count_below<NMETA>(meta, T);
                if (!full_list && st.p >= kcols) flags |= 8;   // list continues past the staged columns
                // TF32 split by truncation (the tensor core truncates fp32 operands to TF32):
                // hi = x' with the low 13 bits cleared, lo = x' - hi (exact) passed as is
                const uint32_t ab = sbase + L.aop + (uint32_t)((i % L.NA) * kTcRows * KT * 4);
#pragma unroll
                for (int j = 0; j < DP; j += 4) {
                    float h[4], l[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        h[q] = __uint_as_float(__float_as_uint(xh[j + q]) & 0xFFFFE000u);
                        l[q] = xh[j + q] - h[q];
                    }
                    tc::sts128(ab + tc::op_off(t, j, kTcRows), h[0], h[1], h[2], h[3]);
                    tc::sts128(ab + tc::op_off(t, DP + j, kTcRows), l[0], l[1], l[2], l[3]);
                    tc::sts128(ab + tc::op_off(t, 2 * DP + j, kTcRows), h[0], h[1], h[2], h[3]);
                }
                const float xxh = __uint_as_float(__float_as_uint(xx) & 0xFFFFE000u);
                tc::sts128(ab + tc::op_off(t, 3 * DP, kTcRows), xxh, xx - xxh, 1.f, 1.f);
            }
            st.flags = flags;
            rstate[b * kTcRows + t] = st;
            const int pw = (__reduce_max_sync(kFull, active ? min(st.p, kcols) : 0) + 15) & ~15;
            if (lane == 0) s_info[b].pw[warp] = pw;
            tc::fence_async_smem();
            // the tile's MMA width: max over the four prep warps (named barrier among them)
            asm volatile("bar.sync 1, 128;" ::: "memory");
            if (t == 0) {
                TcInfo &inf = s_info[b];
                inf.tile = tile;
                inf.A = A;
                inf.bslot = L.NB == 2 ? mslot : 0;
                inf.mslot = mslot;
                inf.N = max(max(inf.pw[0], inf.pw[1]), max(inf.pw[2], inf.pw[3]));
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");
            tc::fence_before();
            if (lane == 0) tc::mbar_arrive(tc::smem_u32(&s_aready[b]));
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) c_clause1 += __shfl_xor_sync(kFull, c_clause1, o);
        if (lane == 0 && c_clause1) atomicAdd(p.counters + 2, c_clause1);
    } else {
        // ================= epilogue: best / second-best column, exact-mode decision ==========
        const int ew = warp - kTcEpiWarp0;            // TMEM lane quadrant
        const int r = ew * 32 + lane;                 // row within the tile
        const uint32_t tlane = s_tmem + ((uint32_t)(ew * 32) << 16);
        const float eps = *p.eps;
        const float kappa = 2.f * (58.f + DP / 4.f + KT / 2.f) * 5.9604645e-8f;
        CRow<CSMEM> Cn;
        if constexpr (CSMEM) Cn.base = tc::smem_u32(sC); else Cn.base = p.Cneg;
        double *acc = p.acc + (int64_t)(blockIdx.x % p.nslab) * k * (DP + 1);
        unsigned long long c_changed = 0, c_dists = 0, c_refined = 0, c_cols = 0, c_fb = 0;
        uint32_t qid[16];                             // column ids 0..15 kept in registers
#pragma unroll
        for (int q = 0; q < 16; ++q) { qid[q] = (uint32_t)q; asm volatile("" : "+r"(qid[q])); }
        for (int i = 0;; ++i) {
            const int s = i % S, b = i & 1;
            tc::mbar_wait(tc::smem_u32(&s_accfull[b]), (uint32_t)((i >> 1) & 1));
            tc::mbar_wait(tc::smem_u32(&s_aready[b]), (uint32_t)((i >> 1) & 1));   // acquire prep's writes
            tc::fence_after();
            const TcInfo inf = s_info[b];
            if (inf.tile < 0) break;
            const TcRow st = rstate[b * kTcRows + r];
            const int64_t tile = inf.tile;
            const int64_t row = tile * kTcRows + r;
            const bool valid = st.flags & 1, active = st.flags & 2, misfit = st.flags & 4;
            const bool uncovered = st.flags & 8;
            const float4 *meta = meta0 + inf.mslot * NMETA;
            if constexpr (SCREEN) {
                const int pw = inf.N > 0 ? inf.pw[ew] : 0;
                const int own = st.pad;
                float m = INFINITY;
                for (int c0 = 0; c0 < pw; c0 += 16) {
                    uint32_t rr[16];
                    tc::tmem_ld16(tlane + (uint32_t)(b * NMAX + c0), rr);
                    if (__any_sync(kFull, own >= c0 && own < c0 + 16)) {
#pragma unroll
                        for (int q = 0; q < 16; ++q)
                            if (c0 + q == own) rr[q] = 0x7f800000u;   // +inf: the own cluster is not a rival
                    }
#pragma unroll
                    for (int q = 0; q < 16; q += 2) m = tc_fmin3(m, __uint_as_float(rr[q]), __uint_as_float(rr[q + 1]));
                }
                if (lane == 0) c_cols += (unsigned long long)pw;
                const float cmax = pw > 0 ? meta[pw - 1].w : 0.f;
                tc::fence_before();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(tc::smem_u32(&s_tfree[b]));   // TMEM / A / row state / metadata free
                // stays iff every rival column's lower bound exceeds the own upper bound u_t
                // (squared domain: m > (u_t + epsr)^2 + E) and, for a row of another cluster, the
                // tile cluster A itself is farther than u_t
                bool decided = false;
                if (active && !uncovered) {
                    const float E = __fmul_ru(kappa, __fadd_ru(st.xx, cmax));
                    const float epsr = __fadd_ru(eps, __fmul_ru(1.2e-7f, __fadd_ru(sqrt_up(st.xx), sqrt_up(cmax))));
                    const float ue = __fadd_ru(st.ut, epsr);
                    const float thr = __fadd_ru(__fmul_ru(ue, ue), E);
                    decided = m > thr && (!misfit || lower_d(st.xx, p.g_dn, eps) > st.ut);
                    // MTI distance count 1 + #{c : H[a][c] < u_t}
                    if (decided)
                        c_dists += 1ull + (unsigned long long)(misfit ? count_below_nl(p.NL + (int64_t)st.a * p.ks, k - 1, st.ut)
                                                                      : st.p);
                }
                const bool qd = active && !decided;
                const unsigned qm = __ballot_sync(kFull, qd);
                const int64_t grp = tile * 4 + ew;
                if (tile * kTcRows + ew * 32 < n) {
                    if (qd) p.qrow[grp * 32 + __popc(qm & ((1u << lane) - 1u))] = (int)row;
                    if (lane == 0) p.qcnt[grp] = __popc(qm);
                }
                c_fb += qd;
                // clause-1 rows keep the loosened bound, decided rows the tightened one (queued
                // rows are rewritten by k_resolve)
                if (valid) p.u[row] = decided ? st.ut : st.uu;
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(tc::smem_u32(&s_sfree[s]));     // stage reusable
                continue;
            }
            const float *sx = reinterpret_cast<const float *>(smem + L.ring + s * L.stage_bytes);
            float x[DP];
#pragma unroll
            for (int j = 0; j < DP; j += 4) {
                const float4 v = *reinterpret_cast<const float4 *>(sx + r * DP + j);
                x[j] = v.x; x[j + 1] = v.y; x[j + 2] = v.z; x[j + 3] = v.w;
            }
            const int pw = inf.N > 0 ? inf.pw[ew] : 0;
            uint32_t m1 = 0x7fffffffu, m2 = 0x7fffffffu;   // packed keys: q bits, low byte = column
            for (int c0 = 0; c0 < pw; c0 += 16) {
                uint32_t rr[16];
                tc::tmem_ld16(tlane + (uint32_t)(b * NMAX + c0), rr);
                int kk[16];
#pragma unroll
                for (int q = 0; q < 16; ++q)      // key = q bits, low byte replaced by the column
                    asm("lop3.b32 %0, %1, 0xFFFFFF00, %2, 0xEA;" : "=r"(kk[q]) : "r"(rr[q]), "r"(qid[q]));
                int b1 = min(kk[0], min(kk[1], kk[2]));
#pragma unroll
                for (int q = 3; q < 16; q += 2) b1 = min(b1, min(kk[q], q + 1 < 16 ? kk[q + 1] : kk[q]));
                // second best = min over the other keys: (k - b1 - 1) as unsigned maps b1 to the
                // maximum and keeps the order of the rest (subtraction on the FMA pipe)
                const uint32_t moff = ~(uint32_t)b1;  // -(b1 + 1)
                uint32_t dd[16];
#pragma unroll
                for (int q = 0; q < 16; ++q) asm("mad.lo.u32 %0, %1, 1, %2;" : "=r"(dd[q]) : "r"(kk[q]), "r"(moff));
                uint32_t d2 = min(dd[0], min(dd[1], dd[2]));
#pragma unroll
                for (int q = 3; q < 16; q += 2) d2 = min(d2, min(dd[q], q + 1 < 16 ? dd[q + 1] : dd[q]));
                const uint32_t off = (uint32_t)b1 + 1u;
                const int g1 = b1 + c0, g2 = (int)(d2 + off) + c0;        // globalise the column
                const int n1 = min((int)m1, g1);
                m2 = (uint32_t)min(max((int)m1, g1), min((int)m2, g2));
                m1 = (uint32_t)n1;
            }
            if (lane == 0) c_cols += (unsigned long long)pw;
            // everything this tile needs from the metadata slot, before releasing the buffers
            const float cmax = pw > 0 ? meta[pw - 1].w : 0.f;
            const int cc1 = m1 != 0x7fffffffu ? __float_as_int(meta[m1 & 0xff].y) : -1;
            const int cc2 = m2 != 0x7fffffffu ? __float_as_int(meta[m2 & 0xff].y) : -1;
            tc::fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(tc::smem_u32(&s_tfree[b]));   // TMEM / A / row state / metadata free
            int anew = st.a;
            float unew = st.uu;
            if (active) {
                bool fallback = uncovered;
                const float E = __fmul_ru(kappa, __fadd_ru(st.xx, cmax));
                // eps_C + centring roundings 2^-24 (|x'| + |c'|) (+ slack for the roots)
                const float epsr = __fadd_ru(eps, __fmul_ru(1.2e-7f, __fadd_ru(sqrt_up(st.xx), sqrt_up(cmax))));
                const int k1 = (int)m1, k2 = (int)m2;
                // common case, in the squared domain: the best column's lower bound exceeds the own
                // upper bound, i.e. v1 - E > (ut + epsr)^2 (v1: truncated key value <= the TC value)
                const float ue = __fadd_ru(st.ut, epsr);
                const float thr = __fadd_ru(__fmul_ru(ue, ue), E);
                const bool stay_fast = !fallback && !misfit && (k1 == 0x7fffffff || __int_as_float(k1 & ~0xff) > thr);
                if (stay_fast) {
                    unew = st.ut;
                } else if (!fallback) {
                    // TC candidate intervals on the distance scale (key truncation: <= 2^-15 relative)
                    auto U_of = [&](int key) {
                        const float v = fmaxf(__int_as_float(key & ~0xff), 0.f);
                        return __fadd_ru(sqrt_up(__fadd_ru(__fmul_ru(v, 1.0000306f), E)), epsr);
                    };
                    auto L_of = [&](int key) {
                        if (key == 0x7fffffff) return INFINITY;
                        const float v = __int_as_float(key & ~0xff);
                        return fmaxf(0.f, __fsub_rd(sqrt_dn(fmaxf(__fsub_rd(v, E), 0.f)), epsr));
                    };
                    // own cluster: direct interval [lo, ut]; a misfit's own cluster is also a column
                    float Uo = st.ut, Lo = st.lo, Ui = INFINITY, Li = INFINITY, Lother = INFINITY;
                    int ci = -1;                               // best column other than the own cluster
                    if (cc1 == st.a) {                         // (misfit) own is the best column: merge
                        Uo = fminf(Uo, U_of(k1)); Lo = fmaxf(Lo, L_of(k1));
                        ci = cc2;
                        if (ci >= 0) { Ui = U_of(k2); Li = L_of(k2); Lother = -1.f; }   // third unknown
                    } else {
                        ci = cc1;
                        if (ci >= 0) { Ui = U_of(k1); Li = L_of(k1); }
                        Lother = L_of(k2);                     // (may be the own cluster's column)
                    }
                    // misfit rows also have the tile cluster A (distance sqrt(xx), direct form)
                    float UA = INFINITY, LA = INFINITY;
                    if (misfit) { UA = upper_d(st.xx, p.g_up, eps); LA = lower_d(st.xx, p.g_dn, eps); }
                    if (Uo < fminf(Li, LA)) {                                   // stays
                        unew = Uo;
                    } else if (misfit && UA < fminf(Lo, Li)) {                  // moves to A
                        anew = inf.A; unew = UA;
                    } else if (ci >= 0 && Ui < fminf(fminf(Lo, LA), Lother)) {  // moves to a column
                        anew = ci; unew = Ui;
                    } else {
                        fallback = true;
                    }
                }
                if (fallback) {
                    // CUDA-core MTI walk over NL[a] in the direct form + exact-mode refinement
                    ++c_fb;
                    const uint64_t *nl = p.NL + (int64_t)st.a * p.ks;
                    float bq = dist2<DP, CSMEM>(x, Cn, st.a), q2 = INFINITY;
                    int bc = st.a;
                    for (int j = 0; j < k - 1; ++j) {
                        const uint64_t key = __ldg(nl + j);
                        if (!(key_h(key) < st.ut)) break;
                        const int c = key_c(key);
                        const float q = dist2<DP, CSMEM>(x, Cn, c);
                        q2 = fminf(q2, fmaxf(q, bq));
                        bc = q < bq ? c : bc;
                        bq = fminf(q, bq);
                    }
                    const float ub = upper_d(bq, p.g_up, eps);
                    if (q2 < INFINITY && lower_d(q2, p.g_dn, eps) <= ub) {
                        anew = refine64(sx + r * DP, p.d, p.C64, k, st.a, nl, st.ut, &unew);
                        ++c_refined;
                    } else {
                        anew = bc;
                        unew = ub;
                    }
                }
                // MTI distance count 1 (tighten) + #{c : H[a][c] < u_t}: from the tile's columns
                // for rows of A; misfit / uncovered rows are counted by k_mti_count after the pass
                if (!misfit && !uncovered) c_dists += (unsigned long long)(1 + st.p);
            }
            {   // deferred counts: compacted per warp into defer[tile*128 + ew*32 + i], count dcount[tile*4 + ew]
                const bool defer = active && (misfit || uncovered);
                const unsigned dm = __ballot_sync(kFull, defer);
                if (defer)
                    p.defer[tile * kTcRows + ew * 32 + __popc(dm & ((1u << lane) - 1u))] =
                        ((unsigned long long)(uint32_t)st.a << 32) | __float_as_uint(st.ut);
                if (lane == 0) p.dcount[tile * 4 + ew] = __popc(dm);
            }
            if (valid) {
                p.a[row] = anew;
                p.u[row] = unew;
                c_changed += (anew != st.a);
            }
            if (valid && anew != st.a) move_delta<DP>(acc, p.d, st.a, anew, x);   // S3 as a delta (B5)
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(tc::smem_u32(&s_sfree[s]));     // stage reusable
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            c_changed += __shfl_xor_sync(kFull, c_changed, o);
            c_dists += __shfl_xor_sync(kFull, c_dists, o);
            c_refined += __shfl_xor_sync(kFull, c_refined, o);
            c_fb += __shfl_xor_sync(kFull, c_fb, o);
        }
        if (lane == 0) {
            if (c_changed) atomicAdd(p.counters + 0, c_changed);
            if (c_dists) atomicAdd(p.counters + 1, c_dists);
            if (c_refined) atomicAdd(p.counters + 3, c_refined);
            if (c_cols) atomicAdd(p.counters + 4, c_cols);
            if (c_fb) atomicAdd(p.counters + 5, c_fb);
        }
    }
    __syncwarp();
    tc::fence_before();
    __syncthreads();
    if (warp == kTcMmaWarp)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(s_tmem), "r"(p.tmem_cols));
}

// MTI distance counts of the rows the tensor-core pass deferred (misfit / uncovered rows):
// counters[1] += sum over entries (a, u_t) of 1 + #{c : H[a][c] < u_t}  (binary search in NL[a]);
// entries of (tile g, warp w) are defer[g*128 + w*32 .. + dcount[g*4 + w]).  One warp per pair.
__global__ void k_mti_count(const unsigned long long *defer, const int *dcount, int64_t ntiles,
                            unsigned long long *counters, const uint64_t *NL, int ks, int k)
{
    const int lane = threadIdx.x & 31;
    unsigned long long sum = 0;
    for (int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; g < ntiles * 4;
         g += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int cnt = dcount[g];
        if (lane < cnt) {
            const unsigned long long e = defer[g * 32 + lane];
            const int a = (int)(e >> 32);
            const float ut = __uint_as_float((uint32_t)e);
            sum += 1 + count_below_nl(NL + (int64_t)a * ks, k - 1, ut);
        }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) sum += __shfl_xor_sync(kFull, sum, o);
    if (lane == 0 && sum) atomicAdd(counters + 1, sum);
}

cudaError_t launch_mti_count(const unsigned long long *defer, const int *dcount, int64_t ntiles,
                             unsigned long long *counters, const uint64_t *NL, int ks, int k, int num_sms,
                             cudaStream_t st)
{
    k_mti_count<<<num_sms * 8, 256, 0, st>>>(defer, dcount, ntiles, counters, NL, ks, k);
    return cudaGetLastError();
}

// ---- host side: pipeline configuration, residency, launch ---------------------------------
// Deepest pipeline that fits: prefer 2 CTAs per SM, then ring depth, A/B double buffering.
static TcCfg pick_cfg(int DP, bool csmem, int k, int nmax, int optin, int smem_sm, int *ctas)
{
    const int static_bytes = 1024;
    for (int want = 2; want >= 1; --want) {
        const int budget = std::min(optin, smem_sm / want - 1024) - static_bytes;
        for (int S : {4, 3, 2})
            for (int NA : {2, 1})
                for (int NB : {2, 1}) {
                    TcCfg L = tc_cfg(DP, csmem, k, nmax, S, NA, NB);
                    if (L.total <= budget) { *ctas = want; return L; }
                }
    }
    *ctas = 0;
    return tc_cfg(DP, csmem, k, nmax, 2, 1, 1);
}

template <int DP, bool CSMEM, int NMETA>
static cudaError_t launch_tc_t(const AssignParams &p, const TcCfg &L, int grid, bool screen, cudaStream_t st)
{
    auto kern = screen ? k_mti_tc<DP, CSMEM, NMETA, true> : k_mti_tc<DP, CSMEM, NMETA, false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L.total);
    if (e != cudaSuccess) return e;
    kern<<<grid, kTcThreads, L.total, st>>>(p, L);
    return cudaGetLastError();
}

template <int DP, bool CSMEM>
static cudaError_t launch_tc_m(const AssignParams &p, const TcCfg &L, int grid, bool screen, cudaStream_t st)
{
    switch (p.nmeta) {
    case 16: return launch_tc_t<DP, CSMEM, 16>(p, L, grid, screen, st);
    case 32: return launch_tc_t<DP, CSMEM, 32>(p, L, grid, screen, st);
    case 64: return launch_tc_t<DP, CSMEM, 64>(p, L, grid, screen, st);
    case 128: return launch_tc_t<DP, CSMEM, 128>(p, L, grid, screen, st);
    case 256: return launch_tc_t<DP, CSMEM, 256>(p, L, grid, screen, st);
    }
    return cudaErrorInvalidValue;
}

bool tc_supported(int DP) { return DP == 8 || DP == 16 || DP == 32; }

int tc_kt_host(int DP) { return tc_kt(DP); }

int tc_nmeta_host(int nmax) { return tc_nmeta(nmax); }

// shared memory the tensor-core pass needs (0 if it does not fit one CTA) and its grid
size_t tc_plan(int DP, bool csmem, int k, int nmax, int num_sms, int *grid, int *tmem_cols)
{
    int dev = 0, optin = 0, smem_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    int ctas = 0;
    TcCfg L = pick_cfg(DP, csmem, k, nmax, optin, smem_sm, &ctas);
    int cols = 32;
    while (cols < 2 * nmax) cols <<= 1;
    ctas = std::min(ctas, 512 / cols);
    *tmem_cols = cols;
    *grid = std::max(1, ctas) * num_sms;
    return ctas > 0 ? (size_t)L.total : 0;
}

cudaError_t launch_mti_tc(int DP, bool csmem, const AssignParams &p, int grid, bool screen, cudaStream_t st)
{
    int dev = 0, optin = 0, smem_sm = 0, ctas = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    const TcCfg L = pick_cfg(DP, csmem, p.k, p.nmax, optin, smem_sm, &ctas);
    if (ctas == 0) return cudaErrorInvalidValue;
    switch (DP * 2 + (csmem ? 1 : 0)) {
    case 16: return launch_tc_m<8, false>(p, L, grid, screen, st);
    case 17: return launch_tc_m<8, true>(p, L, grid, screen, st);
    case 32: return launch_tc_m<16, false>(p, L, grid, screen, st);
    case 33: return launch_tc_m<16, true>(p, L, grid, screen, st);
    case 64: return launch_tc_m<32, false>(p, L, grid, screen, st);
    case 65: return launch_tc_m<32, true>(p, L, grid, screen, st);
    }
    return cudaErrorInvalidValue;
}

// ---------------------------------------------------------------------------------------
// S1 (tensor-core part): per cluster c, the B operand block and column metadata of its
// neighbour list (ascending H, as NL[c]); run after k_prep (which built NL).
//   B row j (column c_j = NL[c][j]): c' = fp32(C[c_j]) - fp32(C[c]) (RN), split TF32 hi/lo:
//     [-2 c'hi | -2 c'hi | -2 c'lo | 1 | 1 | cc_hi | cc_lo | 0 ..],  cc = |c'|^2
//   meta j: {H (fp32, rounded down), c_j bits, |c'|^2 rounded up, prefix max of that}
//   columns past the k-1 neighbours: q = xx + 1e30 (never a winner), meta {NaN, c, 0, prefix}
__global__ void k_prep_tc(const double *C, const uint64_t *NL, int k, int d, int DP, int ks, int nmax,
                          float *Bop, float4 *Bmeta, int16_t *rank)
{
    if (rank)   // rank[c][c'] = position of c' in c's neighbour list (the screen epilogue's own column)
        for (int j = threadIdx.x; j < k - 1; j += blockDim.x)
            rank[(int64_t)blockIdx.x * k + key_c(NL[(int64_t)blockIdx.x * ks + j])] = (int16_t)j;
    const int nmeta = tc_nmeta(nmax);
    extern __shared__ float4 smeta[];
    const int c = blockIdx.x, KT = tc_kt(DP);
    const double *Cc = C + (int64_t)c * d;
    const uint64_t *nl = NL + (int64_t)c * ks;
    float *B = Bop + (int64_t)c * nmax * KT;
    for (int j = threadIdx.x; j < nmax; j += blockDim.x) {
        const bool real = j < k - 1;
        const int cj = real ? key_c(nl[j]) : c;
        const double *Cj = C + (int64_t)cj * d;
        double cn2 = 0.0;
        for (int e = 0; e < DP; ++e) {
            const float v = e < d ? __fsub_rn((float)Cj[e], (float)Cc[e]) : 0.f;
            const float hi = tc::tf32_rna(v), lo = tc::tf32_rna(__fsub_rn(v, hi));
            cn2 += (double)v * (double)v;
            B[tc::op_off(j, e, nmax) / 4] = real ? -2.f * hi : 0.f;
            B[tc::op_off(j, DP + e, nmax) / 4] = real ? -2.f * hi : 0.f;
            B[tc::op_off(j, 2 * DP + e, nmax) / 4] = real ? -2.f * lo : 0.f;
        }
        const float ccf = real ? (float)cn2 : 1e30f;
        const float cch = tc::tf32_rna(ccf);
        const float ccl = real ? tc::tf32_rna((float)(cn2 - (double)cch)) : 0.f;
        B[tc::op_off(j, 3 * DP, nmax) / 4] = 1.f;
        B[tc::op_off(j, 3 * DP + 1, nmax) / 4] = 1.f;
        B[tc::op_off(j, 3 * DP + 2, nmax) / 4] = cch;
        B[tc::op_off(j, 3 * DP + 3, nmax) / 4] = ccl;
        for (int e = 3 * DP + 4; e < KT; ++e) B[tc::op_off(j, e, nmax) / 4] = 0.f;
        smeta[j] = make_float4(real ? key_h(nl[j]) : __int_as_float(0x7fc00000), __int_as_float(cj),
                               real ? __double2float_ru(cn2 * (1.0 + 1e-12)) : 0.f, 0.f);
    }
    __syncthreads();
    for (int j = nmax + threadIdx.x; j < nmeta; j += blockDim.x)
        smeta[j] = make_float4(__int_as_float(0x7fc00000), __int_as_float(c), 0.f, 0.f);
    __syncthreads();
    if (threadIdx.x == 0) {
        float m = 0.f;
        for (int j = 0; j < nmeta; ++j) { m = fmaxf(m, smeta[j].z); smeta[j].w = m; }
    }
    __syncthreads();
    for (int j = threadIdx.x; j < nmeta; j += blockDim.x) Bmeta[(int64_t)c * nmeta + j] = smeta[j];
}

cudaError_t launch_prep_tc(const double *C, const uint64_t *NL, int k, int d, int DP, int ks, int nmax,
                           float *Bop, float4 *Bmeta, int16_t *rank, cudaStream_t st)
{
    k_prep_tc<<<k, 128, (size_t)tc_nmeta(nmax) * sizeof(float4), st>>>(C, NL, k, d, DP, ks, nmax, Bop, Bmeta, rank);
    return cudaGetLastError();
}

}  // namespace km
