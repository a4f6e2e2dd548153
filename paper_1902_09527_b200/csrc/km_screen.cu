// km_screen.cu — the MTI assignment pass as two kernels ("screen" engine), sm_100a.
//
// Method: PAPER.md §3.3 (1026-1053): u += f(a) (drift, 1028-1030); clause 1 (u <= s(a): keep, no
// distance, 1036-1040); tighten U(u) = d(x, C[a]) (1033-1034); clauses 2/3: candidates c' with
// 1/2 d(a, c') < u (1042-1053, readings A1/A5/A6 of DESIGN.md); per-cluster sums of the rows that
// moved (reading B5; §3.2, 1000-1011).  Same outputs as k_walk (km_walk.cu).
//
// Why two kernels.  On C3 the single-kernel walk spends ~9 of its ~23 warp-instructions per row in
// the candidate loop; the rest is per-row machinery that almost every row carries although few
// rows need it: the top-2 keys with candidate indices (7 ALU instructions per row and candidate
// pair), the move / misfit / fallback decision branches (a warp executes a branch when any of its
// 64 rows takes it), the mover queue.  But after the first iterations nearly every row stays
// where it is, and a row stays iff its best candidate's lower bound exceeds its own upper bound.
//
//   k_screen (phase 1, every row): the walk of k_walk restricted to the rows of the warp's
//     cluster A ("walk rows"), tracking only the minimum candidate value (one FMNMX3 per row and
//     candidate pair); a walk row whose minimum exceeds (u_t + eps)^2 + E stays (u = u_t, a
//     unchanged; squared domain, no root).  Every other active row — a row of another cluster
//     (a "misfit"), or a walk row that may move — is appended to a per-32-row-group queue.
//   k_resolve (phase 2, queued rows only): one lane per row, the row's own neighbour list NL[a]
//     in the direct form, best and second best, fp64 refinement when the fp32 intervals overlap
//     (the exact-mode decision of k_walk's fallback path); writes a, u, and the
//     fp64 deltas of the rows that moved (coordinate-parallel REDs into the per-SM slabs).
//
// Queue layout: for 32-row group g of the stored rows, qrow[32 g .. 32 g + qcnt[g]) holds the
// rows of the group that k_screen left undecided.  Every group is written by k_screen (no
// memset), so the queue needs no global atomics.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "km_device.cuh"
#include "km_kernels.cuh"
#include "km_walk_common.cuh"

namespace km {

constexpr int kResolveGroups = 32;       // 32-row groups per k_resolve task (1024 rows)
constexpr int kResolveThreads = 256;

// rows per lane and threads per CTA of k_screen: d <= 8 has registers to spare for more rows
// per lane (each candidate pair block a warp loads then serves 32 R rows: the broadcast loads'
// delivery to the registers, 32 lanes x 32 B per LDG.256, bounds the walk through the L1 data
// pipe), wider rows as k_walk
#ifndef KM_SCREEN_R8
#define KM_SCREEN_R8 2
#endif
#ifndef KM_SCREEN_T8
#define KM_SCREEN_T8 1024
#endif
template <int DP> constexpr int screen_r() { return DP <= 8 ? KM_SCREEN_R8 : walk_r<DP>(); }
__host__ __device__ constexpr int screen_threads_of(int DP) { return DP <= 8 ? KM_SCREEN_T8 : walk_threads_of(DP); }
static inline int screen_r_rt(int DP) { return DP <= 8 ? KM_SCREEN_R8 : walk_r_rt(DP); }

// floats of one warp's k_screen shared-memory region: staged rows x | a | u [, SKIP1: a | u of
// the following batch]
__host__ __device__ constexpr int screen_warp_floats(int DP, int R, int skip1)
{
    return 32 * R * (DP + 2) + (skip1 ? 64 * R : 0);
}

__device__ __forceinline__ float fmin3(float a, float b, float c)
{
    float r;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

template <int DP, int R, int NH, bool HSMEM, bool SKIP1>
__global__ void __launch_bounds__(screen_threads_of(DP), 1)
k_screen(AssignParams p, int *qrow, int *qcnt)
{
    extern __shared__ __align__(16) float smem[];
    const int k = p.k;
    const int k4 = (k + 3) & ~3;                   // sections stay 16-B aligned
    float *sF = smem;                               // k
    float *sS = sF + k4;                            // k
    float *sH = sS + k4;                            // k x NH H rows (HSMEM)
    constexpr int kRowsB = 32 * R;                  // rows per warp batch
    constexpr int kChunk = kWalkChunk > 2 * kRowsB ? kWalkChunk : 2 * kRowsB;   // rows per work claim
    float *stg = sH + (HSMEM ? k * NH : 0) + (threadIdx.x >> 5) * screen_warp_floats(DP, R, SKIP1);
    float *sAU2 = stg + kRowsB * (DP + 2);          // SKIP1: the second a | u slot
    for (int i = threadIdx.x; i < k; i += blockDim.x) { sF[i] = p.f[i]; sS[i] = p.s[i]; }
    if (HSMEM)
        for (int i = threadIdx.x; i < k * NH; i += blockDim.x) sH[i] = p.WH[i];
    __syncthreads();
    const float eps = *p.eps;
    const int lane = threadIdx.x & 31;
    const int n = (int)p.n;                        // < 2^31 (kmeans_create enforces it)
    const int kp = p.wpad;
    // expansion-form error: |q~ - |x'-c'|^2| <= kappa (xx + cmax)
    const float kappa = 2.f * (2.f * DP + 20.f) * 5.9604645e-8f;

    unsigned long long c_dists = 0;
    unsigned c_clause132 = 0, steps32 = 0, c_queued32 = 0;

    auto claim = [&]() -> int {
        int c = 0;
        if (lane == 0) c = atomicAdd(p.work, 1);
        c = __shfl_sync(kFull, c, 0);
        return c < (n + kChunk - 1) / kChunk ? c * kChunk : n;   // n: no more work
    };
    // stage rows [r0, r0 + 32 R) of X, a, u into this warp's buffer (16-B cp.async per lane)
    auto stage_au_to = [&](float *ad, int r0) {    // a then u of rows [r0, r0 + 32 R), 16 B per lane
#pragma unroll
        for (int c = lane; c < kRowsB / 2; c += 32) {
            if (c < kRowsB / 4) cp_async16(ad + 4 * c, p.a + r0 + 4 * c);
            else cp_async16(ad + kRowsB + 4 * (c - kRowsB / 4), p.u + r0 + 4 * (c - kRowsB / 4));
        }
    };
    auto stage = [&](int r0) {
        const float4 *xs = reinterpret_cast<const float4 *>(p.X + (size_t)r0 * DP);
        float4 *xd = reinterpret_cast<float4 *>(stg);
#pragma unroll
        for (int c = lane; c < kRowsB * DP / 4; c += 32) cp_async16(xd + stg_swz<DP>(c), xs + c);
        stage_au_to(stg + kRowsB * DP, r0);
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    // SKIP1: batch starts b0 (processed), b1 (rows staged), b2 (a/u staged)
    int sk_end = 0, sk_next = 0, b0 = n, b1 = n, b2 = n, slot = 0;
    auto next_batch = [&]() -> int {
        if (sk_next >= sk_end) {
            const int c = claim();
            if (c >= n) { sk_next = sk_end = n; return n; }
            sk_next = c;
            sk_end = min(c + kChunk, n);
        }
        const int b = sk_next;
        sk_next += kRowsB;
        return b;
    };
    auto au_slot = [&](int sl) -> float * { return sl ? sAU2 : stg + kRowsB * DP; };
    auto stage_au = [&](int r0, int sl) {          // a, u of rows [r0, r0 + 32 R) -> slot sl
        if (r0 < n) stage_au_to(au_slot(sl), r0);
    };
    // x of the rows of batch r0 that fail clause 1 (their a/u are in slot sl): clause-1 rows are
    // never read ("no I/O requests are made")
    auto stage_x_live = [&](int r0, int sl) {
        if (r0 >= n) return;
        const float *ad = au_slot(sl);
        unsigned live[R];
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const int r = 32 * i + lane;
            const int av = __float_as_int(ad[r]);
            const bool v = r0 + r < n;
            const bool l = v && !(__fadd_ru(ad[kRowsB + r], sF[v ? av : 0]) <= sS[v ? av : 0]);
            live[i] = __ballot_sync(kFull, l);
        }
        const float4 *xs = reinterpret_cast<const float4 *>(p.X + (size_t)r0 * DP);
        float4 *xd = reinterpret_cast<float4 *>(stg);
#pragma unroll
        for (int c = lane; c < kRowsB * DP / 4; c += 32) {
            const int r = c / (DP / 4);
            unsigned w = live[0];
#pragma unroll
            for (int i = 1; i < R; ++i) w = (r >> 5) == i ? live[i] : w;
            if ((w >> (r & 31)) & 1u) cp_async16(xd + stg_swz<DP>(c), xs + c);
        }
    };
    // without SKIP1 the work counter is fetched one chunk ahead by lane 0 and broadcast when that
    // chunk starts, so the atomic's round trip overlaps a whole chunk of work
    constexpr int kBatches = kChunk / kRowsB;
    const int nchunks = (n + kChunk - 1) / kChunk;
    int chunk_row = n, ahead_c = 0, bt = 0;
    if constexpr (SKIP1) {
        b0 = next_batch();
        b1 = b0 < n ? next_batch() : n;
        stage_au(b0, 0);
        asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncwarp();
        stage_x_live(b0, 0);
        stage_au(b1, 1);
        asm volatile("cp.async.commit_group;" ::: "memory");
        chunk_row = b0;
    } else {
        chunk_row = claim();
        if (lane == 0) ahead_c = atomicAdd(p.work, 1);
        if (chunk_row < n) stage(chunk_row);
    }

    while (chunk_row < n) {
        const int row0 = SKIP1 ? b0 : chunk_row + bt * kRowsB;
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
                const float4 t = reinterpret_cast<const float4 *>(stg)[stg_swz<DP>(r * (DP / 4) + j / 4)];
                x[i][j] = t.x; x[i][j + 1] = t.y; x[i][j + 2] = t.z; x[i][j + 3] = t.w;
            }
            const float *aus = SKIP1 ? au_slot(slot) : stg + kRowsB * DP;
            aold[i] = __float_as_int(aus[r]);
            const float uold = aus[kRowsB + r];
            valid[i] = row0 + r < n;
            if (!valid[i]) aold[i] = 0;
            uu[i] = valid[i] ? __fadd_ru(uold, sF[aold[i]]) : 0.f;          // u += f(a)
            const bool c1 = valid[i] && uu[i] <= sS[aold[i]];                  // clause 1
            active[i] = valid[i] && !c1;
            c_clause132 += c1;
            amask |= __ballot_sync(kFull, active[i]) ? (1u << i) : 0u;
        }
        __syncwarp();
        if constexpr (SKIP1) {
            // rows of b1 that fail clause 1 (their a/u are here), a/u of b2 into b0's slot
            b2 = b1 < n ? next_batch() : n;
            stage_x_live(b1, slot ^ 1);
            stage_au(b2, slot);
            asm volatile("cp.async.commit_group;" ::: "memory");
            b0 = b1;
            b1 = b2;
            slot ^= 1;
            chunk_row = b0;                         // loop condition
        } else {
            if (++bt == kBatches || chunk_row + bt * kRowsB >= n) {
                bt = 0;
                const int c = __shfl_sync(kFull, ahead_c, 0);
                chunk_row = c < nchunks ? c * kChunk : n;
                if (lane == 0 && chunk_row < n) ahead_c = atomicAdd(p.work, 1);
            }
            if (chunk_row < n) stage(chunk_row + bt * kRowsB);
        }

        bool stay[R];
        float ut[R];
#pragma unroll
        for (int i = 0; i < R; ++i) { stay[i] = false; ut[i] = 0.f; }
        if (amask) {
            // warp cluster A: the middle row's (row 32 R / 2) if active, else the first active row's
            constexpr int im = R / 2, mid = R == 1 ? 16 : 0;
            const unsigned m_mid = __ballot_sync(kFull, active[im]);
            int A;
            if ((m_mid >> mid) & 1u) A = __shfl_sync(kFull, aold[im], mid);
            else {
                int fi = -1, fl = 0;
#pragma unroll
                for (int i = R - 1; i >= 0; --i) {
                    const unsigned m = __ballot_sync(kFull, active[i]);
                    if (m) { fi = i; fl = __ffs(m) - 1; }
                }
                int av = aold[0];
#pragma unroll
                for (int i = 1; i < R; ++i) av = fi == i ? aold[i] : av;
                A = __shfl_sync(kFull, av, fl);
            }
            float4 cA[DP / 4];
#pragma unroll
            for (int j = 0; j < DP / 4; ++j) cA[j] = __ldg(reinterpret_cast<const float4 *>(p.Cneg + (int64_t)A * DP) + j);
            float xx[R];
            int pl[R];
            bool walk[R];
            int pm = 0;
#pragma unroll
            for (int i = 0; i < R; ++i) {
                // x' = x - C^[A] in place (the direct form's arithmetic), xx = |x'|^2
                float2 a0 = make_float2(0.f, 0.f), a1 = make_float2(0.f, 0.f);
#pragma unroll
                for (int j = 0; j < DP; j += 4) {
                    const float4 c = cA[j / 4];
                    const float2 t0 = add2(make_float2(x[i][j], x[i][j + 1]), make_float2(c.x, c.y));
                    const float2 t1 = add2(make_float2(x[i][j + 2], x[i][j + 3]), make_float2(c.z, c.w));
                    x[i][j] = t0.x; x[i][j + 1] = t0.y; x[i][j + 2] = t1.x; x[i][j + 3] = t1.y;
                    a0 = fma2(t0, t0, a0);
                    a1 = fma2(t1, t1, a1);
                }
                const float2 s2 = add2(a0, a1);
                xx[i] = s2.x + s2.y;
                walk[i] = active[i] && aold[i] == A;
                pl[i] = 0;
                if (walk[i]) {
                    ut[i] = upper_d(xx[i], p.g_up, eps);
                    if constexpr (HSMEM) pl[i] = count_below_s<NH>(sH + A * NH, ut[i]);
                    else pl[i] = count_below_u<NH>(p.WH + (int64_t)A * NH, ut[i]);
                }
                pm = max(pm, pl[i]);
            }
            pm = __reduce_max_sync(kFull, pm);
            // the walk: candidates j < pm of A's list, two per step; only the minimum is kept
            const float4 *blk = p.Wblk + (int64_t)A * (kp / 2) * walk_pair_f4(DP);
            const float2 *ccA = reinterpret_cast<const float2 *>(p.Wcc + (int64_t)A * kp);
            const float cmax = pm > 0 ? __ldg(p.Wmeta + (int64_t)A * kp + ((pm + 1) & ~1) - 1).x : 0.f;
            float m1[R];
#pragma unroll
            for (int i = 0; i < R; ++i) m1[i] = INFINITY;
            for (int j = 0; j < pm; j += 2) {
                const float2 cc = __ldg(ccA + (j >> 1));
                float2 q[R];
                if constexpr (DP >= 32 && KM_WALK_HALVES) {
                    // wide rows: the pair block is consumed in two halves of DP/2 coordinates
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
                                q[i] = fma2s(x[i][h * (DP / 2) + 2 * e], make_float2(v[e].x, v[e].y), q[i]);
                                q[i] = fma2s(x[i][h * (DP / 2) + 2 * e + 1], make_float2(v[e].z, v[e].w), q[i]);
                            }
                    }
                } else {
                    float4 v[DP / 2];
#pragma unroll
                    for (int e = 0; e < DP / 2; e += 2)      // 32-byte loads: half the L1 requests
                        ldg256(blk + (int64_t)(j >> 1) * walk_pair_f4(DP) + e, v[e], v[e + 1]);
#pragma unroll
                    for (int i = 0; i < R; ++i) q[i] = q_pair<DP>(x[i], xx[i], cc, v);
                }
#pragma unroll
                for (int i = 0; i < R; ++i) m1[i] = fmin3(m1[i], q[i].x, q[i].y);
            }
            steps32 += (unsigned)pm;
#pragma unroll
            for (int i = 0; i < R; ++i) {
                if (!walk[i]) continue;
                // stays iff the smallest candidate value's lower bound exceeds the own upper
                // bound u_t: v > thr = (u_t + epsr)^2 + E (squared domain).  Columns
                // past the row's own prefix are true distances of real centroids (or +1e30
                // dummies): they can only make the test fail, never pass wrongly.
                const float E = __fmul_ru(kappa, __fadd_ru(xx[i], cmax));
                const float epsr = __fadd_ru(eps, __fmul_ru(1.2e-7f, __fadd_ru(sqrt_up(xx[i]), sqrt_up(cmax))));
                const float ue = __fadd_ru(ut[i], epsr);
                const float thr = __fadd_ru(__fmul_ru(ue, ue), E);
                stay[i] = m1[i] > thr;
                // MTI distance count of a decided row: 1 (tightening) + #{c : H[a][c] < u_t}
                if (stay[i]) c_dists += (unsigned long long)(1 + pl[i]);
            }
        }
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const int rb = row0 + 32 * i;
            const bool qd = active[i] && !stay[i];
            const unsigned qm = __ballot_sync(kFull, qd);
            if (rb < n) {                               // warp-uniform
                if (qd) qrow[rb + __popc(qm & ((1u << lane) - 1u))] = rb + lane;
                if (lane == 0) qcnt[rb >> 5] = __popc(qm);
            }
            c_queued32 += qd;
            // clause-1 rows keep the loosened bound, decided rows the tightened one; queued rows
            // are rewritten by k_resolve (a full-warp store keeps the writes coalesced)
            if (valid[i]) p.u[rb + lane] = stay[i] ? ut[i] : uu[i];
        }
    }
    unsigned long long c_clause1 = c_clause132, steps = steps32, c_queued = c_queued32;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        c_dists += __shfl_xor_sync(kFull, c_dists, o);
        c_clause1 += __shfl_xor_sync(kFull, c_clause1, o);
        c_queued += __shfl_xor_sync(kFull, c_queued, o);
    }
    if (lane == 0) {
        if (c_dists) atomicAdd(p.counters + 1, c_dists);
        if (c_clause1) atomicAdd(p.counters + 2, c_clause1);
        if (steps) atomicAdd(p.counters + 4, steps);
        if (c_queued) atomicAdd(p.counters + 5, c_queued);
    }
}

// Phase 2: the queued rows.  A warp claims tasks of kResolveGroups 32-row groups from a work
// counter, then resolves the task's queued rows 32 at a time, one lane per row.
template <int DP, bool CSMEM>
__global__ void __launch_bounds__(kResolveThreads)
k_resolve(AssignParams p, const int *qrow, const int *qcnt, int ngroups, int *work)
{
    extern __shared__ __align__(16) float smem[];
    const int k = p.k, d = p.d;
    float *sC = smem;                                           // k x DP (CSMEM)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // per warp: movers' rows (32 x DP fp32) and (from, to)
    float *mx = smem + (CSMEM ? k * DP : 0) + warp * (32 * DP + 64);
    int *mft = reinterpret_cast<int *>(mx + 32 * DP);
    if (CSMEM) {
        const float4 *src = reinterpret_cast<const float4 *>(p.Cneg);
        float4 *dst = reinterpret_cast<float4 *>(sC);
        for (int i = threadIdx.x; i < k * DP / 4; i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();
    CRow<CSMEM> Cn;
    if constexpr (CSMEM) Cn.base = (uint32_t)__cvta_generic_to_shared(sC);
    else Cn.base = p.Cneg;
    const float eps = *p.eps;
    double *acc = p.acc + (int64_t)(blockIdx.x % p.nslab) * k * (DP + 1);
    const int ntasks = (ngroups + kResolveGroups - 1) / kResolveGroups;
    unsigned long long c_dists = 0;
    unsigned c_changed = 0, c_refined = 0;
    for (;;) {
        int t = 0;
        if (lane == 0) t = atomicAdd(work, 1);
        t = __shfl_sync(kFull, t, 0);
        if (t >= ntasks) break;
        const int g0 = t * kResolveGroups;
        const int cnt = lane < kResolveGroups && g0 + lane < ngroups ? qcnt[g0 + lane] : 0;
        int incl = cnt;                                         // inclusive scan over the groups
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += v;
        }
        const int total = __shfl_sync(kFull, incl, 31);
        for (int e0 = 0; e0 < total; e0 += 32) {
            const int e = e0 + lane;
            // group of entry e: the first g with incl[g] > e (branch-free search over the lanes)
            int g = 0;
#pragma unroll
            for (int h = kResolveGroups / 2; h >= 1; h >>= 1) {
                const int v = __shfl_sync(kFull, incl, g + h - 1);
                if (v <= e) g += h;
            }
            const int gex = __shfl_sync(kFull, incl - cnt, g);
            const bool has = e < total;
            int row = 0, aold = 0, anew = 0;
            float x[DP];
            if (has) {
                row = qrow[(int64_t)(g0 + g) * 32 + (e - gex)];
                aold = p.a[row];
                const float4 *src = reinterpret_cast<const float4 *>(p.X + (size_t)row * DP);
#pragma unroll
                for (int j = 0; j < DP / 4; ++j) {
                    const float4 v = __ldg(src + j);
                    x[4 * j] = v.x; x[4 * j + 1] = v.y; x[4 * j + 2] = v.z; x[4 * j + 3] = v.w;
                }
                // tighten (direct form, the same arithmetic as k_screen's |x - C^[A]|^2), then
                // clauses 2/3 over NL[a] in ascending H: best and second best (exact mode)
                const float qo = dist2<DP, CSMEM>(x, Cn, aold);
                const float ut = upper_d(qo, p.g_up, eps);
                const uint64_t *nl = p.NL + (int64_t)aold * p.ks;
                float bq = qo, q2 = INFINITY;
                int bc = aold, len = 0;
                for (int j = 0; j < k - 1; ++j) {
                    const uint64_t key = __ldg(nl + j);
                    if (!(key_h(key) < ut)) break;
                    const int c = key_c(key);
                    const float q = dist2<DP, CSMEM>(x, Cn, c);
                    q2 = fminf(q2, fmaxf(q, bq));
                    bc = q < bq ? c : bc;
                    bq = fminf(q, bq);
                    ++len;
                }
                float unew;
                const float ub = upper_d(bq, p.g_up, eps);
                if (q2 < INFINITY && lower_d(q2, p.g_dn, eps) <= ub) {
                    anew = refine64(p.X + (size_t)row * DP, d, p.C64, k, aold, nl, ut, &unew);
                    ++c_refined;
                } else {
                    anew = bc;
                    unew = ub;
                }
                c_dists += (unsigned long long)(1 + len);
                p.u[row] = unew;
                if (anew != aold) p.a[row] = anew;
            }
            // S3 as a delta (B5): the movers' rows staged in shared memory, then fp64 REDs with
            // lanes over (mover, coordinate), so each RED instruction writes whole row segments
            const bool mv = has && anew != aold;
            const unsigned mm = __ballot_sync(kFull, mv);
            if (mm) {
                c_changed += mv;
                if (mv) {
                    const int r = __popc(mm & ((1u << lane) - 1u));
#pragma unroll
                    for (int j = 0; j < DP; j += 4)
                        *reinterpret_cast<float4 *>(mx + r * DP + j) = make_float4(x[j], x[j + 1], x[j + 2], x[j + 3]);
                    mft[r] = aold;
                    mft[32 + r] = anew;
                }
                __syncwarp();
                constexpr int G = DP >= 32 ? 1 : 32 / DP;       // movers per step
                constexpr int CL = DP >= 32 ? 32 : DP;          // lanes per mover
                constexpr int NJ = DP >= 32 ? DP / 32 : 1;      // coordinates per lane per step
                const int nm = __popc(mm);
                const int sub = lane / CL, co = lane % CL;
                for (int m0 = 0; m0 < nm; m0 += G) {
                    const int m = m0 + sub;
                    if (m < nm) {
                        double *ra = acc + (int64_t)mft[m] * (DP + 1), *rb = acc + (int64_t)mft[32 + m] * (DP + 1);
#pragma unroll
                        for (int jj = 0; jj < NJ; ++jj) {
                            const int j = jj * CL + co;
                            if (j < d) {
                                const double v = (double)mx[m * DP + j];
                                atomicAdd(rb + j, v);
                                atomicAdd(ra + j, -v);
                            }
                        }
                        if (co == 0) {
                            atomicAdd(rb + DP, 1.0);
                            atomicAdd(ra + DP, -1.0);
                        }
                    }
                }
                __syncwarp();
            }
        }
    }
    unsigned long long ch = c_changed, rf = c_refined;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        ch += __shfl_xor_sync(kFull, ch, o);
        c_dists += __shfl_xor_sync(kFull, c_dists, o);
        rf += __shfl_xor_sync(kFull, rf, o);
    }
    if (lane == 0) {
        if (ch) atomicAdd(p.counters + 0, ch);
        if (c_dists) atomicAdd(p.counters + 1, c_dists);
        if (rf) atomicAdd(p.counters + 3, rf);
    }
}

// ---- host side ------------------------------------------------------------------------------
typedef void (*screen_kernel_t)(AssignParams, int *, int *);

#define KM_SCREEN_PICK(SK)                                                           \
    if (hs) {                                                                        \
        switch (whs) {                                                               \
        case 2: case 4: case 8: case 16: return k_screen<DP, R, 16, true, SK>;       \
        case 32: return k_screen<DP, R, 32, true, SK>;                               \
        case 64: return k_screen<DP, R, 64, true, SK>;                               \
        case 128: return k_screen<DP, R, 128, true, SK>;                             \
        case 256: return k_screen<DP, R, 256, true, SK>;                             \
        }                                                                            \
    } else {                                                                         \
        switch (whs) {                                                               \
        case 256: return k_screen<DP, R, 256, false, SK>;                            \
        case 512: return k_screen<DP, R, 512, false, SK>;                            \
        case 1024: return k_screen<DP, R, 1024, false, SK>;                          \
        case 2048: return k_screen<DP, R, 2048, false, SK>;                          \
        case 4096: return k_screen<DP, R, 4096, false, SK>;                          \
        }                                                                            \
    }                                                                                \
    return nullptr;

template <int DP>
static screen_kernel_t screen_pick(int whs, bool hs, bool skip1)
{
    constexpr int R = screen_r<DP>();
    if (skip1) {
        KM_SCREEN_PICK(true)
    } else {
        KM_SCREEN_PICK(false)
    }
}

static screen_kernel_t screen_kernel(int DP, int whs, bool hs, bool skip1)
{
    switch (DP) {
    case 4: return screen_pick<4>(whs, hs, skip1);
    case 8: return screen_pick<8>(whs, hs, skip1);
    case 16: return screen_pick<16>(whs, hs, skip1);
    case 32: return screen_pick<32>(whs, hs, skip1);
    case 64: return screen_pick<64>(whs, hs, skip1);
    }
    return nullptr;
}

static size_t screen_smem(int DP, int k, int whs, bool wh_smem, bool skip1)
{
    const int R = screen_r_rt(DP);
    const int k4 = (k + 3) & ~3;
    return (size_t)(2 * k4 + (wh_smem ? k * whs : 0)) * sizeof(float) +
           (size_t)(screen_threads_of(DP) / 32) * screen_warp_floats(DP, R, skip1 ? 1 : 0) * sizeof(float);
}

static size_t resolve_smem(int DP, bool csmem, int k)
{
    return (size_t)((csmem ? k * DP : 0) + (kResolveThreads / 32) * (32 * DP + 64)) * sizeof(float);
}

typedef void (*resolve_kernel_t)(AssignParams, const int *, const int *, int, int *);

static resolve_kernel_t resolve_kernel(int DP, bool csmem)
{
    switch (DP * 2 + (csmem ? 1 : 0)) {
    case 8: return k_resolve<4, false>;
    case 9: return k_resolve<4, true>;
    case 16: return k_resolve<8, false>;
    case 17: return k_resolve<8, true>;
    case 32: return k_resolve<16, false>;
    case 33: return k_resolve<16, true>;
    case 64: return k_resolve<32, false>;
    case 65: return k_resolve<32, true>;
    case 128: return k_resolve<64, false>;
    case 129: return k_resolve<64, true>;
    }
    return nullptr;
}

static cudaError_t set_smem(const void *kern, size_t sm)
{
    return sm > 48 * 1024 ? cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)
                          : cudaSuccess;
}

// grids (one screen CTA per SM; resolve: as many CTAs as fit), computed once per context
void screen_grids(int DP, bool csmem, int k, int whs, bool hs, int num_sms, int *g_screen, int *g_resolve)
{
    int best = 0;
    for (int sk = 0; sk < 2; ++sk) {
        screen_kernel_t kern = screen_kernel(DP, whs, hs, sk != 0);
        const size_t sm = screen_smem(DP, k, whs, hs, sk != 0);
        int per_sm = 1;
        if (kern && set_smem((const void *)kern, sm) == cudaSuccess)
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, screen_threads_of(DP), sm);
        per_sm = std::max(per_sm, 1);
        best = sk == 0 ? per_sm : std::min(best, per_sm);
    }
    *g_screen = best * num_sms;
    resolve_kernel_t rk = resolve_kernel(DP, csmem);
    const size_t rsm = resolve_smem(DP, csmem, k);
    int per_sm = 1;
    if (rk && set_smem((const void *)rk, rsm) == cudaSuccess)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rk, kResolveThreads, rsm);
    *g_resolve = std::max(per_sm, 1) * num_sms;
}

// p.work[0]: the screen's chunk counter, p.work[1]: the resolve task counter (both zeroed with
// the per-iteration scratch)
cudaError_t launch_screen(int DP, bool csmem, const AssignParams &p, int g_screen, int g_resolve, bool skip1,
                          int *qrow, int *qcnt, int64_t n_alloc, cudaStream_t st)
{
    screen_kernel_t sk = screen_kernel(DP, p.whs, p.wh_smem != 0, skip1);
    resolve_kernel_t rk = resolve_kernel(DP, csmem);
    if (!sk || !rk) return cudaErrorInvalidValue;
    const size_t sm = screen_smem(DP, p.k, p.whs, p.wh_smem != 0, skip1);
    cudaError_t e = set_smem((const void *)sk, sm);
    if (e != cudaSuccess) return e;
    sk<<<g_screen, screen_threads_of(DP), sm, st>>>(p, qrow, qcnt);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    (void)n_alloc;
    AssignParams q = p;
    q.qrow = qrow;
    q.qcnt = qcnt;
    return launch_resolve(DP, csmem, q, g_resolve, st);
}

// k_resolve over p.qrow / p.qcnt; its task counter is p.work[1]
cudaError_t launch_resolve(int DP, bool csmem, const AssignParams &p, int g_resolve, cudaStream_t st)
{
    resolve_kernel_t rk = resolve_kernel(DP, csmem);
    if (!rk) return cudaErrorInvalidValue;
    const size_t rsm = resolve_smem(DP, csmem, p.k);
    cudaError_t e = set_smem((const void *)rk, rsm);
    if (e != cudaSuccess) return e;
    const int ngroups = (int)((p.n + 31) / 32);
    rk<<<g_resolve, kResolveThreads, rsm, st>>>(p, p.qrow, p.qcnt, ngroups, p.work + 1);
    return cudaGetLastError();
}

int resolve_grid(int DP, bool csmem, int k, int num_sms)
{
    resolve_kernel_t rk = resolve_kernel(DP, csmem);
    const size_t rsm = resolve_smem(DP, csmem, k);
    int per_sm = 1;
    if (rk && set_smem((const void *)rk, rsm) == cudaSuccess)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rk, kResolveThreads, rsm);
    return std::max(per_sm, 1) * num_sms;
}

}  // namespace km
