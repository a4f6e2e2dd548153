// km_seed.cu — k-means++ D² seeding (§4.3 "k-means++", Eq. 2;
// SURVEY §8(f) NEXT-4), sm_100a.
//
// c_1 = X[first_index]; for m = 2..k: D(x) = min distance of x to the centres chosen so far,
// c_m = the row i drawn with probability D(x_i)² / Σ D² (Eq. 2).  The draw is made exact and
// reproducible (reading B9): the caller passes the k-1 uniforms u_m ∈ [0,1); every
// D² is summed in fp64 in coordinate order; Σ D² is taken hierarchically (rows of a kSeedBlock-row
// block in order, blocks of a kSeedGroup-block group in order, groups in order), and u_m · Σ D² is
// located top-down by the running sums of each level.  The oracle (`oracle/kmeanspp.py`)
// performs the same operations in the same order, so both pick the same rows.
#include <cuda_runtime.h>
#include <cstdint>

#include "km_device.cuh"
#include "km_kernels.cuh"

namespace km {

constexpr int64_t kSeedBlock = 1024;   // rows per block
constexpr int64_t kSeedGroup = 1024;   // blocks per group

// One warp per block of kSeedBlock rows: D2[i] = min(D2[i], Σ_j (x_ij - c_j)²) (fp64, coordinate
// order; first = 1: the distance itself), and the block's sum in row order — lane l holds row
// 32 t + l, lane 0 adds the 32 values in lane order (shuffles), so the sum is sequential.
__global__ void k_pp_update_sums(const float *X, int64_t n, int d, int ldx, const float *c, double *D2,
                                 int first, double *bsum, int64_t nb)
{
    const int lane = threadIdx.x & 31;
    const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (b >= nb) return;
    const int64_t r0 = b * kSeedBlock, r1 = r0 + kSeedBlock < n ? r0 + kSeedBlock : n;
    double s = 0.0;
    for (int64_t base = r0; base < r1; base += 32) {
        const int64_t i = base + lane;
        double v = 0.0;
        if (i < r1) {
            const float *x = X + i * ldx;
            double q = 0.0;
            for (int j = 0; j < d; ++j) {
                const double t = __dsub_rn((double)x[j], (double)c[j]);
                q = __dadd_rn(q, __dmul_rn(t, t));
            }
            v = first ? q : fmin(D2[i], q);
            D2[i] = v;
        }
        const int cnt = r1 - base < 32 ? (int)(r1 - base) : 32;
        for (int l = 0; l < cnt; ++l) s = __dadd_rn(s, __shfl_sync(0xffffffffu, v, l));
    }
    if (lane == 0) bsum[b] = s;
}

// one thread per group: the group's block sums in block order
__global__ void k_pp_group_sums(const double *bsum, int64_t nb, double *gsum, int64_t ng)
{
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= ng) return;
    const int64_t b0 = g * kSeedGroup, b1 = b0 + kSeedGroup < nb ? b0 + kSeedGroup : nb;
    double s = 0.0;
    for (int64_t b = b0; b < b1; ++b) s = __dadd_rn(s, bsum[b]);
    gsum[g] = s;
}

// first index in v[0..m) whose left-to-right running sum exceeds t (its start sum in *start),
// else -1
__device__ int64_t first_crossing(const double *v, int64_t m, double t, double *start)
{
    double run = 0.0;
    for (int64_t i = 0; i < m; ++i) {
        const double nxt = __dadd_rn(run, v[i]);
        if (nxt > t) { *start = run; return i; }
        run = nxt;
    }
    return -1;
}
__device__ int64_t last_positive(const double *v, int64_t m)
{
    for (int64_t i = m - 1; i >= 0; --i)
        if (v[i] > 0.0) return i;
    return -1;
}

// one warp (reading B9): u * total located top-down — group, block, row — by the running sums
// of each level in the oracle's order; where rounding leaves no crossing, the last positive
// entry.  *out = -1 if every D² is 0.
__global__ void k_pp_select(const double *D2, int64_t n, const double *bsum, int64_t nb, const double *gsum,
                            int64_t ng, double u, int64_t *out)
{
    const int lane = threadIdx.x & 31;
    int64_t b = -1;
    bool scan = true;
    double t2 = 0.0;
    if (lane == 0) {
        double total = 0.0;
        for (int64_t g = 0; g < ng; ++g) total = __dadd_rn(total, gsum[g]);
        const double target = __dmul_rn(u, total);
        double R = 0.0, P = 0.0;
        int64_t g = first_crossing(gsum, ng, target, &R);
        if (g < 0) { scan = false; g = last_positive(gsum, ng); }
        if (g >= 0) {
            const double *gb = bsum + g * kSeedGroup;
            const int64_t m = (g + 1) * kSeedGroup < nb ? kSeedGroup : nb - g * kSeedGroup;
            const double t1 = __dsub_rn(target, R);
            int64_t bi = -1;
            if (scan) { bi = first_crossing(gb, m, t1, &P); if (bi < 0) scan = false; }
            if (!scan) bi = last_positive(gb, m);
            b = g * kSeedGroup + bi;
            t2 = __dsub_rn(t1, P);
        }
    }
    b = __shfl_sync(0xffffffffu, b, 0);
    scan = __shfl_sync(0xffffffffu, scan, 0);
    if (b < 0) { if (lane == 0) *out = -1; return; }
    const int64_t r0 = b * kSeedBlock, r1 = r0 + kSeedBlock < n ? r0 + kSeedBlock : n;
    double part = 0.0;
    int64_t last = -1, found = -1;
    for (int64_t base = r0; base < r1 && found < 0; base += 32) {
        const int64_t i = base + lane;
        const double v = i < r1 ? D2[i] : 0.0;
        const int cnt = r1 - base < 32 ? (int)(r1 - base) : 32;
        for (int l = 0; l < cnt; ++l) {
            const double w = __shfl_sync(0xffffffffu, v, l);
            if (lane == 0 && found < 0) {
                part = __dadd_rn(part, w);
                if (w > 0.0) {
                    last = base + l;
                    if (scan && part > t2) found = base + l;
                }
            }
        }
        found = __shfl_sync(0xffffffffu, found, 0);
    }
    if (lane == 0) *out = found >= 0 ? found : last;
}

cudaError_t seed_plusplus(const float *X, int64_t n, int d, int ldx, int k, int64_t first,
                          const double *u, double *D2, double *bsum, float *crow, int64_t *dsel,
                          int64_t *chosen, cudaStream_t st)
{
    const int64_t nb = (n + kSeedBlock - 1) / kSeedBlock;
    const int64_t ng = (nb + kSeedGroup - 1) / kSeedGroup;
    double *gsum = bsum + nb;   // the caller allocates nb + ng doubles
    chosen[0] = first;
    for (int m = 1; m <= k; ++m) {
        const int64_t c = chosen[m - 1];
        cudaError_t e = cudaMemcpyAsync(crow, X + c * ldx, (size_t)d * sizeof(float), cudaMemcpyDeviceToDevice, st);
        if (e != cudaSuccess) return e;
        k_pp_update_sums<<<(unsigned)((nb * 32 + 127) / 128), 128, 0, st>>>(X, n, d, ldx, crow, D2, m == 1, bsum, nb);
        if (m == k) break;
        k_pp_group_sums<<<(unsigned)((ng + 127) / 128), 128, 0, st>>>(bsum, nb, gsum, ng);
        k_pp_select<<<1, 32, 0, st>>>(D2, n, bsum, nb, gsum, ng, u[m - 1], dsel);
        e = cudaMemcpyAsync(&chosen[m], dsel, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) return e;
        e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return e;
        if (chosen[m] < 0) return cudaErrorInvalidValue;   // fewer than k distinct rows
    }
    return cudaGetLastError();
}

}  // namespace km
