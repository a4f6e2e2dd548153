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
#include "km_walk_common.cuh"

namespace km {


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
    const int R = walk_r_sel(DP, wh_smem);
    const int k4 = (k + 3) & ~3;
    return (size_t)((csmem ? k * DP : 0) + 2 * k4 + (wh_smem ? k * whs : 0)) * sizeof(float) +
           (size_t)(walk_threads_dr(DP, R) / 32) *
               (walk_warp_floats(DP, R, skip1 ? 1 : 0) + walk_tab_floats(DP, wh_smem, skip1 ? 1 : 0)) * sizeof(float);
}


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
        case 256: return K<DP, CSMEM, RG, 256, false>;                               \
        case 512: return K<DP, CSMEM, RG, 512, false>;                               \
        case 1024: return K<DP, CSMEM, RG, 1024, false>;                             \
        case 2048: return K<DP, CSMEM, RG, 2048, false>;                             \
        case 4096: return K<DP, CSMEM, RG, 4096, false>;                             \
        }                                                                            \
    }                                                                                \
    return nullptr;

template <int DP, bool CSMEM, bool SK>
static walk_kernel_t walk_pick_s(int whs, bool hs)
{
    constexpr int R = walk_r<DP>();
    constexpr int RG = DP == 32 ? KM_WALK_R32G : R;   // rows per lane when the H rows are global
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
#ifdef KM_WALK_FAST_BUILD      // A/B variant builds: only the row widths of C3 and C4 / C5
    case 17: return walk_pick<8, true>(whs, hs, skip1);
    case 64: return walk_pick<32, false>(whs, hs, skip1);
    case 65: return walk_pick<32, true>(whs, hs, skip1);
    default: return nullptr;
#else
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
#endif
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
    kern<<<grid, walk_threads_dr(DP, walk_r_sel(DP, p.wh_smem != 0)), sm, st>>>(p);
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
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, walk_threads_dr(DP, walk_r_sel(DP, hs)), sm);
        per_sm = per_sm < 1 ? 1 : per_sm;
        best = sk == 0 ? per_sm : std::min(best, per_sm);
    }
    return best * num_sms;
}

}  // namespace km
