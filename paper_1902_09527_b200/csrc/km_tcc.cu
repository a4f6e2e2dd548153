// km_tcc.cu — column-chunked tensor-core MTI screen ("tensor-chunked" engine), sm_100a.
//
// Method: PAPER.md §3.3 (1026-1053): u += f(a), clause 1, tightening U(u), clauses 2/3 over the
// neighbour list of the row's cluster (readings A1/A5/A6); the rows that provably stay are decided
// here, the rest is queued for k_resolve (km_screen.cu), which takes the exact-mode decision and
// applies the moves (reading B5).  DESIGN.md §10.
//
// Why.  The CUDA-core walk delivers every candidate row to every lane through the L1 data pipe
// (256 B per candidate pair at d = 32), which bounds C5 — where a quarter of the active rows need
// nearly all 999 candidates — at ~0.5 wavefront per row-candidate.  Here the candidates of a
// 128-row tile (rows bucketed by cluster, the tile's cluster A = its middle row's) are evaluated
// by tcgen05.mma reading both operands from shared memory, 128 columns at a time:
//
//   producer warp   TMA bulk copies of the row tiles [x | a | u] into a 2-stage ring
//   4 prep warps    per row: u += f(a), clause 1, x' = x - C^[A], |x'|^2, the tightened bound
//                   u_t (rows of another cluster: direct distance to their own centroid, columns
//                   up to the triangle bound (u_t + d(x, A)) / 2), the prefix p = #{j : H[A][j] <
//                   T}; the A operand row [x'hi | x'lo | |x'|^2 hi, lo, 1, 1, 0..] (TF32 split by
//                   truncation, as the tensor core truncates)
//   MMA warp        per 128-column chunk of A's list: a TMA bulk copy of the chunk's B operand
//                   ([-2c'hi | -2c'lo | 1, 1, |c'|^2 hi, lo, 0..], c' = C^[c_j] - C^[A]) into a
//                   2-slot ring, then x'hi.c'hi + x'lo.c'hi + x'hi.c'lo + extras as four MMA groups
//                   sharing the operands (the TF32x3 products of k_mti_tc, K = 2 DP + 8 stored
//                   instead of 3 DP + 8) into a 2-buffer TMEM ring
//   4 epilogue warps per chunk: tcgen05.ld, the running minimum of each row's columns (the own
//                   column masked for rows of another cluster); per tile: the row stays iff the
//                   minimum exceeds (u_t + eps)^2 + E (the error model of k_mti_tc),
//                   else it is queued
//
// Exactness is k_mti_tc's (the same products, the same bound κ); every row it cannot decide goes
// to k_resolve.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include <cuda.h>

#include "km_device.cuh"
#include "km_kernels.cuh"
#include "km_tc_common.cuh"

namespace km {

constexpr int kCRows = 128;            // rows per tile (MMA M)
constexpr int kCNC = 128;              // columns per chunk (MMA N <= 128)
constexpr int kCThreads = 448;
constexpr int kCPrepW = 4;             // warps 0-3: prep group 0 (even tiles)
constexpr int kCPrepW1 = 10;           // warps 10-13: prep group 1 (odd tiles)
constexpr int kCEpiW0 = 4;             // warps 4-7: epilogue (TMEM lane quadrant = warp % 4)
constexpr int kCProdW = 8;             // warp 8: row-tile producer
constexpr int kCMmaW = 9;              // warp 9: B-chunk loads + MMA issue
constexpr int kCStages = 2;
// Slots.  A operand: 2 (released by the MMA commit of the tile's last chunk, not by the epilogue);
// row state / tile info: kRS (released by the epilogue); TMEM accumulators: kTB x 128 columns.
// Prep of tile i waits only for the MMAs of tile i - 2, so the epilogue of a tile overlaps the
// prep and MMAs of the next ones (with one slot ring for all three the period of two tiles was
// prep + MMA + epilogue: ~4000 cycles per tile on C5, the tensor pipe 23 % busy).
constexpr int kRS = 4;
constexpr int kTB = 4;

__host__ __device__ constexpr int tcc_ka(int DP) { return 2 * DP + 8; }

// per-row state handed from the prep warps to the epilogue warps, structure of arrays (one
// 4-byte word per lane: conflict-free), two tile slots
constexpr int kRowFields = 7;   // a, flags, uu, ut, xx, p, own
struct TccRow {
    int a;          // assignment before the pass
    int flags;      // bit0 valid, bit1 active (clause 1 failed), bit2 misfit (a != A)
    float uu;       // u + f(a)
    float ut;       // tightened upper bound of d(x, C[a])
    float xx;       // |x - C^[A]|^2
    int p;          // columns below the row's threshold
    int own;        // misfit: position of a in A's list, else -1
};
__device__ __forceinline__ void row_store(int *base, int b, int r, const TccRow &s)
{
    int *q = base + b * kRowFields * kCRows + r;
    q[0] = s.a; q[kCRows] = s.flags; q[2 * kCRows] = __float_as_int(s.uu); q[3 * kCRows] = __float_as_int(s.ut);
    q[4 * kCRows] = __float_as_int(s.xx); q[5 * kCRows] = s.p; q[6 * kCRows] = s.own;
}
__device__ __forceinline__ TccRow row_load(const int *base, int b, int r)
{
    const int *q = base + b * kRowFields * kCRows + r;
    TccRow s;
    s.a = q[0]; s.flags = q[kCRows]; s.uu = __int_as_float(q[2 * kCRows]); s.ut = __int_as_float(q[3 * kCRows]);
    s.xx = __int_as_float(q[4 * kCRows]); s.p = q[5 * kCRows]; s.own = q[6 * kCRows];
    return s;
}

struct TccInfo {
    long long tile;  // -1 = end of stream
    int A, N, nch;   // tile cluster, MMA columns (multiple of 16), chunks
    int pw[4];       // per-warp columns the epilogue reads
    float cm[4];     // per-warp prefix max of |c'|^2 over those columns
};

struct TccCfg {
    int stage_bytes, ring, aop, bop, meta, rstate, sc, sf, ss, total;
};

// The row tile [128 x DP] is loaded by a 2-D TMA tensor copy with the hardware swizzle whose span
// is the row (32 / 64 / 128 B for DP = 8 / 16 / 32): 16-byte piece q of row r lands at piece
// q ^ f(r), so the lanes of a warp (one row each) read their pieces without bank conflicts
// (unswizzled 128-byte rows put every lane's piece q in the same banks: 8-way conflicts,
// measured on C5).  Byte offset o of the dense tile is stored at o ^ (((o >> 7) & M) << 4).
__host__ __device__ constexpr int tcc_xs(int DP) { return DP * 4; }
__host__ __device__ constexpr int tcc_swz_mask(int DP) { return DP >= 32 ? 7 : (DP >= 16 ? 3 : 1); }
__device__ __forceinline__ uint32_t tcc_swz(uint32_t o, int M) { return o ^ (((o >> 7) & (uint32_t)M) << 4); }
// H of a cluster's list in shared memory, skewed (entry i at i + i / 32) so that the lanes'
// binary-search probes fall in distinct banks
__host__ __device__ constexpr int tcc_hs(int nmeta) { return nmeta + nmeta / 32 + 4; }

__host__ __device__ inline TccCfg tcc_cfg(int DP, bool csmem, int k, int nmeta)
{
    TccCfg L;
    const int KA = tcc_ka(DP);
    L.stage_bytes = (kCRows * tcc_xs(DP) + 2 * kCRows * 4 + 1023) & ~1023;   // swizzled tiles: 1 KB aligned
    L.ring = 0;
    L.aop = (L.ring + kCStages * L.stage_bytes + 127) & ~127;
    L.bop = L.aop + 2 * kCRows * KA * 4;
    L.meta = L.bop + 2 * kCNC * KA * 4;
    L.rstate = L.meta + ((2 * tcc_hs(nmeta) * 4 + 15) & ~15);
    L.sc = L.rstate + kRS * kCRows * kRowFields * 4;
    L.sf = L.sc + (csmem ? k * DP * 4 : 0);
    L.ss = L.sf + ((k + 3) & ~3) * 4;
    L.total = L.ss + ((k + 3) & ~3) * 4;
    return L;
}

// #{j < M : h[j] < T} over a skewed row (entry j at j + j / 32; ascending, NaN padded)
template <int M>
__device__ __forceinline__ int count_below_k(const float *h, float T)
{
    int base = 0;
#pragma unroll
    for (int half = M >> 1; half >= 1; half >>= 1) {
        const int j = base + half - 1;
        base = h[j + (j >> 5)] < T ? base + half : base;
    }
    return base + (h[base + (base >> 5)] < T ? 1 : 0);
}

__device__ __forceinline__ float tcc_fmin3(float a, float b, float c)
{
    float r;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

template <int DP, bool CSMEM, int NMETA>
__global__ void __launch_bounds__(kCThreads, 1)
k_tcc(AssignParams p, TccCfg L, const __grid_constant__ CUtensorMap tmap)
{
    constexpr int KA = tcc_ka(DP);
    constexpr uint32_t kBBytes = kCNC * KA * 4;
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t s_full[kCStages], s_sfree[kCStages];
    __shared__ __align__(8) uint64_t s_aready[kRS], s_efree[kRS], s_afree[2], s_bfull[2], s_bempty[2], s_tfull[kTB], s_tfree[kTB], s_mbar[2];
    __shared__ long long s_meta[kCStages];
    __shared__ TccInfo s_info[kRS];
    __shared__ uint32_t s_tmem;

    const int k = p.k;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const uint32_t sbase = tc::smem_u32(smem);
    float *sC = reinterpret_cast<float *>(smem + L.sc);
    float *sF = reinterpret_cast<float *>(smem + L.sf);
    float *sS = reinterpret_cast<float *>(smem + L.ss);
    int *rstate = reinterpret_cast<int *>(smem + L.rstate);
    const float *meta0 = reinterpret_cast<const float *>(smem + L.meta);
    constexpr int XS = tcc_xs(DP);
    constexpr int HS = tcc_hs(NMETA);

    if (CSMEM) {
        const float4 *src = reinterpret_cast<const float4 *>(p.Cneg);
        float4 *dst = reinterpret_cast<float4 *>(sC);
        for (int i = t; i < k * DP / 4; i += kCThreads) dst[i] = src[i];
    }
    for (int i = t; i < k; i += kCThreads) { sF[i] = p.f[i]; sS[i] = p.s[i]; }
    {   // zero the A operand buffers once (rows of clause-1 threads are never written)
        float4 *za = reinterpret_cast<float4 *>(smem + L.aop);
        for (int i = t; i < 2 * kCRows * KA / 4; i += kCThreads) za[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (warp == kCMmaW) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     :: "r"(tc::smem_u32(&s_tmem)), "r"(kTB * kCNC));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) {
        for (int s = 0; s < kCStages; ++s) {
            tc::mbar_init(tc::smem_u32(&s_full[s]), 1);
            tc::mbar_init(tc::smem_u32(&s_sfree[s]), kCPrepW);
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(tc::smem_u32(&s_afree[b]), 1);
            tc::mbar_init(tc::smem_u32(&s_bfull[b]), 1);
            tc::mbar_init(tc::smem_u32(&s_bempty[b]), 1);
            tc::mbar_init(tc::smem_u32(&s_mbar[b]), 1);
        }
        for (int b = 0; b < kRS; ++b) {
            tc::mbar_init(tc::smem_u32(&s_aready[b]), kCPrepW);
            tc::mbar_init(tc::smem_u32(&s_efree[b]), 4);
        }
        for (int b = 0; b < kTB; ++b) {
            tc::mbar_init(tc::smem_u32(&s_tfull[b]), 1);
            tc::mbar_init(tc::smem_u32(&s_tfree[b]), 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const int64_t n = p.n;
    const int64_t ntiles = (n + kCRows - 1) / kCRows;

    if (warp == kCProdW) {
        // ================= producer: row tiles [x (swizzled) | a | u] -> ring stages ========
        if (lane == 0) {
            const int G = p.tile_chunk;
            int64_t q_next = 0, q_end = 0;
            int nterm = 0;
            for (int L_ = 0;; ++L_) {
                const int s = L_ % kCStages;
                if (L_ >= kCStages) tc::mbar_wait(tc::smem_u32(&s_sfree[s]), (uint32_t)(((L_ / kCStages) - 1) & 1));
                if (q_next >= q_end && nterm == 0) {
                    const int64_t c = atomicAdd(p.work, 1);
                    q_next = c * G;
                    q_end = q_next + G;
                }
                const int64_t tl = q_next < ntiles && nterm == 0 ? q_next : -1;
                ++q_next;
                s_meta[s] = tl;
                const uint32_t mb = tc::smem_u32(&s_full[s]);
                if (tl < 0) {   // one end-of-stream tile per prep group (stage s is group s's)
                    tc::mbar_arrive(mb);
                    if (++nterm == kCStages) break;
                    continue;
                }
                const uint32_t xb = kCRows * DP * 4, ab = kCRows * 4;
                tc::mbar_arrive_tx(mb, xb + 2 * ab);
                const uint32_t dst = sbase + L.ring + s * L.stage_bytes;
                asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                             :: "r"(dst), "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(0), "r"((int)(tl * kCRows)), "r"(mb)
                             : "memory");
                tc::bulk_g2s(dst + xb, p.a + tl * kCRows, ab, mb);
                tc::bulk_g2s(dst + xb + ab, p.u + tl * kCRows, ab, mb);
            }
        }
    } else if (warp == kCMmaW) {
        // ================= B chunks + MMA: D[chunk] = A . B[chunk]^T ========================
        if (lane == 0) {
            const uint32_t idesc_base = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kCRows >> 4) << 24);
            const uint32_t bfull[2] = {tc::smem_u32(&s_bfull[0]), tc::smem_u32(&s_bfull[1])};
            const uint32_t bempty[2] = {tc::smem_u32(&s_bempty[0]), tc::smem_u32(&s_bempty[1])};
            uint32_t g = 0;                               // chunks issued so far
            // B slot j holds chunks with ch % 2 == j; a slot still holding the wanted chunk (same
            // cluster A, same chunk: consecutive tiles of a bucket) is not reloaded
            int nfill[2] = {0, 0}, tag[2] = {-1, -1};
            for (int i = 0;; ++i) {
                const int b = i & 1, rs = i % kRS;
                tc::mbar_wait(tc::smem_u32(&s_aready[rs]), (uint32_t)((i / kRS) & 1));
                tc::fence_after();
                const TccInfo &inf = s_info[rs];
                if (inf.tile < 0) break;
                const int A = inf.A, N = inf.N, nch = inf.nch;
                const uint32_t ab = sbase + L.aop + (uint32_t)(b * kCRows * KA * 4);
                const float *bsrc = p.Bc + (int64_t)A * p.tcc_nch * kCNC * KA;
                auto load_b = [&](int ch) {   // fill #nfill[j] of slot j = ch & 1 with chunk ch of A's list
                    const int j = ch & 1, want = (A << 8) | ch;
                    // the slot's previous use done (waited for every use, in order: a skipped wait
                    // would let the phase parity alias two uses later)
                    if (nfill[j] >= 1) tc::mbar_wait(bempty[j], (uint32_t)((nfill[j] - 1) & 1));
                    if (tag[j] == want) {
                        tc::mbar_arrive(bfull[j]);               // still there: an empty fill
                    } else {
                        tc::mbar_arrive_tx(bfull[j], kBBytes);
                        tc::bulk_g2s(sbase + L.bop + j * kBBytes, bsrc + (int64_t)ch * kCNC * KA, kBBytes, bfull[j]);
                        tag[j] = want;
                    }
                    ++nfill[j];
                };
                if (nch > 0) load_b(0);
                for (int ch = 0; ch < nch; ++ch, ++g) {
                    const int j = ch & 1, jt = g % kTB;
                    const int f = nfill[j] - 1;                  // this chunk's fill of slot j
                    if (ch + 1 < nch) load_b(ch + 1);            // next chunk's copy overlaps these MMAs
                    tc::mbar_wait(bfull[j], (uint32_t)(f & 1));
                    if (g >= kTB) tc::mbar_wait(tc::smem_u32(&s_tfree[jt]), ((g / kTB) - 1) & 1);
                    tc::fence_after();
                    const int w = min(kCNC, N - ch * kCNC);
                    const uint32_t idesc = idesc_base | ((uint32_t)(w >> 3) << 17);
                    const uint32_t bb = sbase + L.bop + j * kBBytes;
                    const uint32_t d = s_tmem + (uint32_t)(jt * kCNC);
#pragma unroll
                    for (int kb = 0; kb < DP / 8; ++kb)       // x'hi . c'hi
                        tc::mma_tf32(d, tc::sdesc(ab + kb * kCRows * 32), tc::sdesc(bb + kb * kCNC * 32), idesc, kb > 0);
#pragma unroll
                    for (int kb = 0; kb < DP / 8; ++kb)       // x'lo . c'hi
                        tc::mma_tf32(d, tc::sdesc(ab + (DP / 8 + kb) * kCRows * 32), tc::sdesc(bb + kb * kCNC * 32), idesc, 1);
#pragma unroll
                    for (int kb = 0; kb < DP / 8; ++kb)       // x'hi . c'lo
                        tc::mma_tf32(d, tc::sdesc(ab + kb * kCRows * 32), tc::sdesc(bb + (DP / 8 + kb) * kCNC * 32), idesc, 1);
                    tc::mma_tf32(d, tc::sdesc(ab + (DP / 4) * kCRows * 32), tc::sdesc(bb + (DP / 4) * kCNC * 32), idesc, 1);
                    tc::mma_commit(tc::smem_u32(&s_tfull[jt]));
                    tc::mma_commit(bempty[j]);
                }
                tc::mma_commit(tc::smem_u32(&s_afree[b]));   // A slot b free once these MMAs are done
            }
        }
    } else if (warp < kCPrepW || warp >= kCPrepW1) {
        // ================= prep: bounds, clause 1, tightening, prefix, A operand ============
        // two groups of 4 warps on alternate tiles (group pg: ring stage pg, A slot pg, H-row
        // slot pg), so one group's dependent loads overlap the other's
        const int pg = warp < kCPrepW ? 0 : 1;
        const int pt = t - (pg ? kCPrepW1 * 32 : 0);    // row in the tile
        const int pwarp = pt >> 5;
        const float eps = *p.eps;
        const int ncols = k - 1;
        CRow<CSMEM> Cn;
        if constexpr (CSMEM) Cn.base = tc::smem_u32(sC); else Cn.base = p.Cneg;
        int mA = -1;
        uint32_t mpar = 0u;
        unsigned long long c_clause1 = 0;
        for (int i = pg;; i += kCStages) {
            const int s = i % kCStages, b = i & 1, rs = i % kRS;
            tc::mbar_wait(tc::smem_u32(&s_full[s]), (uint32_t)((i / kCStages) & 1));
            const long long tile = s_meta[s];
            // A slot b is free once the MMAs of tile i - 2 are done; row state and info slot rs
            // once the epilogue of tile i - kRS is
            if (i >= 2) tc::mbar_wait(tc::smem_u32(&s_afree[b]), (uint32_t)(((i - 2) >> 1) & 1));
            if (i >= kRS) tc::mbar_wait(tc::smem_u32(&s_efree[rs]), (uint32_t)(((i / kRS) - 1) & 1));
            if (tile < 0) {
                if (pt == 0) s_info[rs].tile = -1;
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(tc::smem_u32(&s_aready[rs]));
                break;
            }
            const uint8_t *stage = smem + L.ring + s * L.stage_bytes;
            const uint32_t sxa = tc::smem_u32(stage);                                // swizzled row tile
            const int32_t *sa = reinterpret_cast<const int32_t *>(stage + kCRows * XS);
            const float *su = reinterpret_cast<const float *>(stage + kCRows * XS + kCRows * 4);
            const int vrows = (int)(n - tile * kCRows < kCRows ? n - tile * kCRows : kCRows);
            const int A = sa[vrows >> 1];
            const int ms = pg;
            if (mA != A) {   // every thread of the group finished the tile that read this slot
                if (pt == 0) {
                    const uint32_t mb = tc::smem_u32(&s_mbar[ms]);
                    const uint32_t hb = (uint32_t)(((HS * 4) + 15) & ~15);
                    tc::mbar_arrive_tx(mb, hb);
                    tc::bulk_g2s(sbase + L.meta + (uint32_t)(ms * hb), p.Mh + (int64_t)A * (hb / 4), hb, mb);
                }
                tc::mbar_wait(tc::smem_u32(&s_mbar[ms]), mpar);
                mpar ^= 1u;
                mA = A;
            }
            const float *meta = meta0 + ms * ((((HS * 4) + 15) & ~15) / 4);

            const int64_t row = tile * kCRows + pt;
            const bool valid = row < n;
            float x[DP];
#pragma unroll
            for (int j = 0; j < DP; j += 4) {
                const float4 v = lds128(sxa + tcc_swz((uint32_t)(pt * XS + j * 4), tcc_swz_mask(DP)));
                x[j] = v.x; x[j + 1] = v.y; x[j + 2] = v.z; x[j + 3] = v.w;
            }
            const int aold = valid ? sa[pt] : 0;
            const float uu = valid ? __fadd_ru(su[pt], sF[aold]) : 0.f;       // u += f(a)
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(tc::smem_u32(&s_sfree[s]));     // the stage is read
            const bool c1 = valid && uu <= sS[aold];                           // clause 1
            const bool active = valid && !c1;
            const bool misfit = active && aold != A;
            c_clause1 += c1;
            TccRow st;
            st.a = aold; st.uu = uu; st.xx = 0.f; st.ut = 0.f; st.p = 0;
            st.own = misfit ? p.rank[(int64_t)A * k + aold] : -1;
            st.flags = (valid ? 1 : 0) | (active ? 2 : 0) | (misfit ? 4 : 0);
            if (active) {
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
                    T = st.ut;
                } else {
                    // own distance in the direct form; columns by the triangle bound around A
                    const float qo = dist2<DP, CSMEM>(x, Cn, aold);
                    st.ut = upper_d(qo, p.g_up, eps);
                    T = __fmul_ru(__fadd_ru(st.ut, upper_d(xx, p.g_up, eps)), 0.5f);
                }
                st.p = min(count_below_k<NMETA>(meta, T), ncols);
                const uint32_t abuf = sbase + L.aop + (uint32_t)(b * kCRows * KA * 4);
#pragma unroll
                for (int j = 0; j < DP; j += 4) {
                    float h[4], l[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        h[q] = __uint_as_float(__float_as_uint(xh[j + q]) & 0xFFFFE000u);
                        l[q] = xh[j + q] - h[q];
                    }
                    tc::sts128(abuf + tc::op_off(pt, j, kCRows), h[0], h[1], h[2], h[3]);
                    tc::sts128(abuf + tc::op_off(pt, DP + j, kCRows), l[0], l[1], l[2], l[3]);
                }
                const float xxh = __uint_as_float(__float_as_uint(xx) & 0xFFFFE000u);
                tc::sts128(abuf + tc::op_off(pt, 2 * DP, kCRows), xxh, xx - xxh, 1.f, 1.f);
            }
            row_store(rstate, rs, pt, st);
            const int pw = (__reduce_max_sync(kFull, active ? st.p : 0) + 15) & ~15;
            if (lane == 0) {
                s_info[rs].pw[pwarp] = pw;
                s_info[rs].cm[pwarp] = pw > 0 ? __ldg(p.Mx + (int64_t)A * NMETA + pw - 1) : 0.f;
            }
            tc::fence_async_smem();
            asm volatile("bar.sync %0, 128;" :: "r"(1 + pg) : "memory");
            if (pt == 0) {
                TccInfo &inf = s_info[rs];
                inf.tile = tile;
                inf.A = A;
                inf.N = max(max(inf.pw[0], inf.pw[1]), max(inf.pw[2], inf.pw[3]));
                inf.nch = (inf.N + kCNC - 1) / kCNC;
            }
            asm volatile("bar.sync %0, 128;" :: "r"(1 + pg) : "memory");
            tc::fence_before();
            if (lane == 0) tc::mbar_arrive(tc::smem_u32(&s_aready[rs]));
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) c_clause1 += __shfl_xor_sync(kFull, c_clause1, o);
        if (lane == 0 && c_clause1) atomicAdd(p.counters + 2, c_clause1);
    } else if (warp < kCEpiW0 + 4) {
        // ================= epilogue: running minimum per chunk, decision, queue =============
        const int ew = warp - kCEpiW0;                 // TMEM lane quadrant
        const int r = ew * 32 + lane;
        const uint32_t tlane = s_tmem + ((uint32_t)(ew * 32) << 16);
        const float eps = *p.eps;
        constexpr int KT3 = ((3 * DP + 4) + 7) & ~7;       // the products of k_mti_tc's TF32x3 form
        const float kappa = 2.f * (58.f + DP / 4.f + KT3 / 2.f) * 5.9604645e-8f;   // k_mti_tc's κ
        unsigned long long c_dists = 0, c_cols = 0, c_queued = 0;
        uint32_t g = 0;
        for (int i = 0;; ++i) {
            const int rs = i % kRS;
            tc::mbar_wait(tc::smem_u32(&s_aready[rs]), (uint32_t)((i / kRS) & 1));
            tc::fence_after();
            const TccInfo inf = s_info[rs];
            if (inf.tile < 0) break;
            const TccRow st = row_load(rstate, rs, r);
            const bool valid = st.flags & 1, active = st.flags & 2, misfit = st.flags & 4;
            const int pw = inf.pw[ew];
            float m = INFINITY, m2 = INFINITY;
            for (int ch = 0; ch < inf.nch; ++ch, ++g) {
                const int j = g % kTB;
                tc::mbar_wait(tc::smem_u32(&s_tfull[j]), (g / kTB) & 1);
                tc::fence_after();
                const int c0 = ch * kCNC;
                const int cend = min(kCNC, pw - c0);
                for (int cc = 0; cc < cend; cc += 32) {    // cend: a multiple of 16
                    uint32_t rr[32];
                    if (cend - cc >= 32) tc::tmem_ld32(tlane + (uint32_t)(j * kCNC + cc), rr);
                    else {
                        uint32_t h16[16];
                        tc::tmem_ld16(tlane + (uint32_t)(j * kCNC + cc), h16);
#pragma unroll
                        for (int q = 0; q < 16; ++q) { rr[q] = h16[q]; rr[16 + q] = 0x7f800000u; }
                    }
                    const int base = c0 + cc;
                    if (__any_sync(kFull, st.own >= base && st.own < base + 32)) {
#pragma unroll
                        for (int q = 0; q < 32; ++q)
                            if (base + q == st.own) rr[q] = 0x7f800000u;   // the own cluster is no rival
                    }
#pragma unroll
                    for (int q = 0; q < 32; q += 4) {      // two independent min chains
                        m = tcc_fmin3(m, __uint_as_float(rr[q]), __uint_as_float(rr[q + 1]));
                        m2 = tcc_fmin3(m2, __uint_as_float(rr[q + 2]), __uint_as_float(rr[q + 3]));
                    }
                }
                tc::fence_before();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(tc::smem_u32(&s_tfree[j]));
            }
            m = fminf(m, m2);
            if (lane == 0) c_cols += (unsigned long long)pw;
            bool decided = false;
            if (active) {
                const float cmax = inf.cm[ew];
                const float E = __fmul_ru(kappa, __fadd_ru(st.xx, cmax));
                const float epsr = __fadd_ru(eps, __fmul_ru(1.2e-7f, __fadd_ru(sqrt_up(st.xx), sqrt_up(cmax))));
                const float ue = __fadd_ru(st.ut, epsr);
                const float thr = __fadd_ru(__fmul_ru(ue, ue), E);
                decided = m > thr && (!misfit || lower_d(st.xx, p.g_dn, eps) > st.ut);
                if (decided)
                    c_dists += 1ull + (unsigned long long)(misfit ? count_below_nl(p.NL + (int64_t)st.a * p.ks, k - 1, st.ut)
                                                                  : st.p);
            }
            const bool qd = active && !decided;
            const unsigned qm = __ballot_sync(kFull, qd);
            const int64_t tile = inf.tile;
            const int64_t grp = tile * 4 + ew;
            if (tile * kCRows + ew * 32 < n) {
                if (qd) p.qrow[grp * 32 + __popc(qm & ((1u << lane) - 1u))] = (int)(tile * kCRows + r);
                if (lane == 0) p.qcnt[grp] = __popc(qm);
            }
            c_queued += qd;
            if (valid) p.u[tile * kCRows + r] = decided ? st.ut : st.uu;
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(tc::smem_u32(&s_efree[rs]));
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            c_dists += __shfl_xor_sync(kFull, c_dists, o);
            c_queued += __shfl_xor_sync(kFull, c_queued, o);
        }
        if (lane == 0) {
            if (c_dists) atomicAdd(p.counters + 1, c_dists);
            if (c_cols) atomicAdd(p.counters + 4, c_cols);
            if (c_queued) atomicAdd(p.counters + 5, c_queued);
        }
    }
    __syncwarp();
    tc::fence_before();
    __syncthreads();
    if (warp == kCMmaW)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(s_tmem), "r"(kTB * kCNC));
}

// S1 (tensor-chunked part): per cluster c, the B operand chunks and column metadata of its
// neighbour list (ascending H, as NL[c]); run after k_prep.
//   column j (centroid c_j = NL[c][j]): c' = fp32(C[c_j]) - fp32(C[c]) (RN), split TF32 hi/lo (RN):
//     [-2 c'hi | -2 c'lo | 1, 1, cc_hi, cc_lo, 0, 0, 0, 0],  cc = |c'|^2;  chunk j / 128, row j % 128
//   meta j: {H (fp32, rounded down; NaN past the list), prefix max of |c'|^2 rounded up}
//   columns past the k-1 neighbours: q = xx + 1e30 (never a winner)
__global__ void k_prep_tcc(const double *C, const uint64_t *NL, int k, int d, int DP, int ks, int nch, int nmeta,
                           float *Bc, float *Mh, float *Mx, int16_t *rank)
{
    // rank[c][c'] = position of c' in c's neighbour list (the epilogue's own column)
    for (int j = threadIdx.x; j < k - 1; j += blockDim.x)
        rank[(int64_t)blockIdx.x * k + key_c(NL[(int64_t)blockIdx.x * ks + j])] = (int16_t)j;
    extern __shared__ float scc[];
    const int c = blockIdx.x, KA = tcc_ka(DP);
    const double *Cc = C + (int64_t)c * d;
    const uint64_t *nl = NL + (int64_t)c * ks;
    const int ncol = nch * kCNC;
    for (int j = threadIdx.x; j < ncol; j += blockDim.x) {
        const bool real = j < k - 1;
        const int cj = real ? key_c(nl[j]) : c;
        const double *Cj = C + (int64_t)cj * d;
        float *B = Bc + ((int64_t)c * nch + j / kCNC) * kCNC * KA;
        const int jr = j % kCNC;
        double cn2 = 0.0;
        for (int e = 0; e < DP; ++e) {
            const float v = (real && e < d) ? __fsub_rn((float)Cj[e], (float)Cc[e]) : 0.f;
            const float hi = tc::tf32_rna(v), lo = tc::tf32_rna(__fsub_rn(v, hi));
            cn2 += (double)v * (double)v;
            B[tc::op_off(jr, e, kCNC) / 4] = -2.f * hi;
            B[tc::op_off(jr, DP + e, kCNC) / 4] = -2.f * lo;
        }
        const float ccf = real ? (float)cn2 : 1e30f;
        const float cch = tc::tf32_rna(ccf);
        const float ccl = real ? tc::tf32_rna((float)(cn2 - (double)cch)) : 0.f;
        B[tc::op_off(jr, 2 * DP, kCNC) / 4] = 1.f;
        B[tc::op_off(jr, 2 * DP + 1, kCNC) / 4] = 1.f;
        B[tc::op_off(jr, 2 * DP + 2, kCNC) / 4] = cch;
        B[tc::op_off(jr, 2 * DP + 3, kCNC) / 4] = ccl;
        for (int e = 2 * DP + 4; e < KA; ++e) B[tc::op_off(jr, e, kCNC) / 4] = 0.f;
        if (j < nmeta) scc[j] = real ? __double2float_ru(cn2 * (1.0 + 1e-12)) : 0.f;
    }
    const int hrow = ((tcc_hs(nmeta) * 4 + 15) & ~15) / 4;   // skewed H row (padded to 16 B)
    for (int j = threadIdx.x; j < hrow; j += blockDim.x) Mh[(int64_t)c * hrow + j] = __int_as_float(0x7fc00000);
    __syncthreads();
    for (int j = threadIdx.x; j < nmeta; j += blockDim.x) {
        if (j >= ncol) scc[j] = 0.f;
        Mh[(int64_t)c * hrow + j + (j >> 5)] = j < k - 1 ? key_h(nl[j]) : __int_as_float(0x7fc00000);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float m = 0.f;
        for (int j = 0; j < nmeta; ++j) { m = fmaxf(m, scc[j]); Mx[(int64_t)c * nmeta + j] = m; }
    }
}

cudaError_t launch_prep_tcc(const double *C, const uint64_t *NL, int k, int d, int DP, int ks, int nch, int nmeta,
                            float *Bc, float *Mh, float *Mx, int16_t *rank, cudaStream_t st)
{
    k_prep_tcc<<<k, 128, (size_t)nmeta * sizeof(float), st>>>(C, NL, k, d, DP, ks, nch, nmeta, Bc, Mh, Mx, rank);
    return cudaGetLastError();
}

int tcc_nch_host(int k) { return std::max(1, (k - 1 + kCNC - 1) / kCNC); }
int tcc_ka_host(int DP) { return tcc_ka(DP); }
int tcc_nmeta_host(int k) { int m = 16; while (m < k) m <<= 1; return m; }
int tcc_hrow_host(int k) { return ((tcc_hs(tcc_nmeta_host(k)) * 4 + 15) & ~15) / 4; }

static int tcc_optin()
{
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return optin;
}

// shared memory the chunked tensor-core screen needs (0 if it does not fit one SM)
size_t tcc_smem(int DP, bool csmem, int k)
{
    const TccCfg L = tcc_cfg(DP, csmem, k, tcc_nmeta_host(k));
    return L.total + 2048 <= tcc_optin() ? (size_t)L.total : 0;
}

template <int DP, bool CSMEM, int NMETA>
static cudaError_t launch_tcc_t(const AssignParams &p, const TccCfg &L, int grid, const CUtensorMap &tm, cudaStream_t st)
{
    cudaError_t e = cudaFuncSetAttribute(k_tcc<DP, CSMEM, NMETA>, cudaFuncAttributeMaxDynamicSharedMemorySize, L.total);
    if (e != cudaSuccess) return e;
    k_tcc<DP, CSMEM, NMETA><<<grid, kCThreads, L.total, st>>>(p, L, tm);
    return cudaGetLastError();
}

template <int DP, bool CSMEM>
static cudaError_t launch_tcc_m(const AssignParams &p, const TccCfg &L, int nmeta, int grid, const CUtensorMap &tm,
                                cudaStream_t st)
{
    switch (nmeta) {
    case 16: return launch_tcc_t<DP, CSMEM, 16>(p, L, grid, tm, st);
    case 32: return launch_tcc_t<DP, CSMEM, 32>(p, L, grid, tm, st);
    case 64: return launch_tcc_t<DP, CSMEM, 64>(p, L, grid, tm, st);
    case 128: return launch_tcc_t<DP, CSMEM, 128>(p, L, grid, tm, st);
    case 256: return launch_tcc_t<DP, CSMEM, 256>(p, L, grid, tm, st);
    case 512: return launch_tcc_t<DP, CSMEM, 512>(p, L, grid, tm, st);
    case 1024: return launch_tcc_t<DP, CSMEM, 1024>(p, L, grid, tm, st);
    case 2048: return launch_tcc_t<DP, CSMEM, 2048>(p, L, grid, tm, st);
    }
    return cudaErrorInvalidValue;
}

// tmap: the CUtensorMap (128 bytes) of the row buffer p.X, from tcc_make_tmap
cudaError_t launch_tcc(int DP, bool csmem, const AssignParams &p, int num_sms, const void *tmap, cudaStream_t st)
{
    const int nmeta = tcc_nmeta_host(p.k);
    const TccCfg L = tcc_cfg(DP, csmem, p.k, nmeta);
    const CUtensorMap &tm = *reinterpret_cast<const CUtensorMap *>(tmap);
    switch (DP * 2 + (csmem ? 1 : 0)) {
    case 16: return launch_tcc_m<8, false>(p, L, nmeta, num_sms, tm, st);
    case 17: return launch_tcc_m<8, true>(p, L, nmeta, num_sms, tm, st);
    case 32: return launch_tcc_m<16, false>(p, L, nmeta, num_sms, tm, st);
    case 33: return launch_tcc_m<16, true>(p, L, nmeta, num_sms, tm, st);
    case 64: return launch_tcc_m<32, false>(p, L, nmeta, num_sms, tm, st);
    case 65: return launch_tcc_m<32, true>(p, L, nmeta, num_sms, tm, st);
    }
    return cudaErrorInvalidValue;
}

// 2-D tensor map of an n_alloc x DP fp32 row buffer: box 128 rows x DP, the row-span swizzle
// (tcc_swz); out: 128 bytes, 64-byte aligned.  Returns 0 on success.
int tcc_make_tmap(void *out, const float *X, int64_t n_alloc, int DP)
{
    typedef CUresult (*encode_t)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                 const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static encode_t fn = nullptr;
    if (!fn) {
        void *f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess || !f) return -1;
        fn = reinterpret_cast<encode_t>(f);
    }
    const cuuint64_t dims[2] = {(cuuint64_t)DP, (cuuint64_t)n_alloc};
    const cuuint64_t strides[1] = {(cuuint64_t)DP * 4};
    const cuuint32_t box[2] = {(cuuint32_t)DP, (cuuint32_t)kCRows};
    const cuuint32_t estr[2] = {1, 1};
    const CUtensorMapSwizzle sw = DP >= 32 ? CU_TENSOR_MAP_SWIZZLE_128B
                                           : (DP >= 16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
    const CUresult r = fn(reinterpret_cast<CUtensorMap *>(out), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(X),
                          dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : (int)r;
}

}  // namespace km
