// km_seed.cu — k-means++ D² seeding (§4.3 "k-means++", Eq. 2;
// SURVEY §8(f) NEXT-4), sm_100a.
//
// c_1 = X[first_index]; for m = 2..k: D(x) = min distance of x to the centres chosen so far,
// c_m = the row i drawn with probability D(x_i)² / Σ D² (Eq. 2).  The draw is exact and
// reproducible (reading B9): the caller passes the k-1 uniforms u_m ∈ [0,1); every D²
// is the fp64 value Σ_j (x_j - c_j)² in coordinate order; the drawn row is the FIRST row whose
// exact prefix sum Σ_{j<=i} D_j² exceeds u · Σ_j D_j² (exact real arithmetic).
//
// Exactness on the GPU: every D² of fp32 data is a multiple of 2^-350 (differences of fp32
// values are multiples of 2^-149, squares and rounded sums of squares keep that) and below
// 2^300 for any n < 2^40, d <= 64, so D² · 2^384 is an integer below 2^688 and every sum of them
// is held exactly by a 768-bit fixed-point integer (12 x 64-bit limbs).  Per draw:
//   k_pp_update_sums  D² = min(D², |x - c|²) per row (fp64) and the exact sum of each 1024-row
//                     block (each lane sums its rows, then a shuffle tree — integer addition is
//                     associative, so the order does not matter);
//   k_pp_group_sums   exact sums of 1024-block groups;
//   k_pp_select       total T, target = floor(u · T) (u = mu / 2^s exactly), and the first row
//                     whose exact prefix exceeds the target: group, block, row, top-down.
// The blocking is only a search structure: the result is the flat definition's.
#include <cuda_runtime.h>
#include <cstdint>

#include "km_device.cuh"
#include "km_kernels.cuh"

namespace km {

constexpr int64_t kSeedBlock = 1024;   // rows per block
constexpr int64_t kSeedGroup = 1024;   // blocks per group
constexpr int kW = 12;                 // limbs of the fixed-point sums (768 bits)
constexpr int kLsbExp = -384;          // the fixed point's unit: 2^-384

struct Wide {
    uint64_t w[kW];
};

__device__ __forceinline__ void wzero(Wide &a)
{
#pragma unroll
    for (int i = 0; i < kW; ++i) a.w[i] = 0ull;
}

// a += b (carry chain)
__device__ __forceinline__ void wadd(Wide &a, const Wide &b)
{
    asm("add.cc.u64 %0, %0, %12;\n\t"
        "addc.cc.u64 %1, %1, %13;\n\t"
        "addc.cc.u64 %2, %2, %14;\n\t"
        "addc.cc.u64 %3, %3, %15;\n\t"
        "addc.cc.u64 %4, %4, %16;\n\t"
        "addc.cc.u64 %5, %5, %17;\n\t"
        "addc.cc.u64 %6, %6, %18;\n\t"
        "addc.cc.u64 %7, %7, %19;\n\t"
        "addc.cc.u64 %8, %8, %20;\n\t"
        "addc.cc.u64 %9, %9, %21;\n\t"
        "addc.cc.u64 %10, %10, %22;\n\t"
        "addc.u64 %11, %11, %23;"
        : "+l"(a.w[0]), "+l"(a.w[1]), "+l"(a.w[2]), "+l"(a.w[3]), "+l"(a.w[4]), "+l"(a.w[5]),
          "+l"(a.w[6]), "+l"(a.w[7]), "+l"(a.w[8]), "+l"(a.w[9]), "+l"(a.w[10]), "+l"(a.w[11])
        : "l"(b.w[0]), "l"(b.w[1]), "l"(b.w[2]), "l"(b.w[3]), "l"(b.w[4]), "l"(b.w[5]),
          "l"(b.w[6]), "l"(b.w[7]), "l"(b.w[8]), "l"(b.w[9]), "l"(b.w[10]), "l"(b.w[11]));
}

// v · 2^384 as a fixed-point integer (v >= 0); *bad = 1 if v is not a multiple of 2^-384
__device__ __forceinline__ Wide wfrom(double v, int *bad)
{
    Wide r;
    wzero(r);
    const uint64_t bits = (uint64_t)__double_as_longlong(v);
    int e = (int)((bits >> 52) & 0x7ff);
    uint64_t m = bits & 0xfffffffffffffull;
    if (m == 0 && e == 0) return r;
    if (e) m |= 1ull << 52; else e = 1;
    int sh = e - 1075 - kLsbExp;                 // v = m 2^(e - 1075) -> m 2^sh units
    if (sh < 0) {
        if (sh <= -53 || (m & ((1ull << -sh) - 1ull))) { *bad = 1; return r; }
        m >>= -sh;
        sh = 0;
    }
    const int li = sh >> 6, off = sh & 63;
    const uint64_t lo = m << off, hi = off ? (m >> (64 - off)) : 0ull;
#pragma unroll
    for (int i = 0; i < kW; ++i) r.w[i] = (i == li ? lo : 0ull) | (i == li + 1 ? hi : 0ull);
    return r;
}

// a > b
__device__ __forceinline__ bool wgt(const Wide &a, const Wide &b)
{
    for (int i = kW - 1; i >= 0; --i)
        if (a.w[i] != b.w[i]) return a.w[i] > b.w[i];
    return false;
}

__device__ __forceinline__ bool wzero_p(const Wide &a)
{
    uint64_t o = 0;
#pragma unroll
    for (int i = 0; i < kW; ++i) o |= a.w[i];
    return o == 0;
}

// floor(u · T) for u in [0, 1): u = mu 2^-s exactly (mu < 2^53, s >= 53); the 13-limb product
// mu · T shifted right by s bits
__device__ Wide wscale(const Wide &T, double u)
{
    Wide r;
    wzero(r);
    const uint64_t bits = (uint64_t)__double_as_longlong(u);
    int e = (int)((bits >> 52) & 0x7ff);
    uint64_t mu = bits & 0xfffffffffffffull;
    if (mu == 0 && e == 0) return r;
    if (e) mu |= 1ull << 52; else e = 1;
    const int s = 1075 - e;                      // u = mu 2^-s
    uint64_t p[kW + 1];
    uint64_t carry = 0;
    for (int i = 0; i < kW; ++i) {
        const uint64_t lo = T.w[i] * mu, hi = __umul64hi(T.w[i], mu);
        const uint64_t t = lo + carry;
        p[i] = t;
        carry = hi + (t < lo ? 1ull : 0ull);
    }
    p[kW] = carry;
    const int ls = s >> 6, bs = s & 63;
    for (int i = 0; i < kW; ++i) {
        const int j = i + ls;
        const uint64_t a = j <= kW ? p[j] : 0ull, b = j + 1 <= kW ? p[j + 1] : 0ull;
        r.w[i] = bs ? ((a >> bs) | (b << (64 - bs))) : a;
    }
    return r;
}

__device__ __forceinline__ Wide wshfl_down(const Wide &a, int off)
{
    Wide r;
#pragma unroll
    for (int i = 0; i < kW; ++i) r.w[i] = __shfl_down_sync(0xffffffffu, a.w[i], off);
    return r;
}

// One warp per block of kSeedBlock rows: D2[i] = min(D2[i], Σ_j (x_ij - c_j)²) (fp64, coordinate
// order; first = 1: the distance itself), and the block's exact sum.
__global__ void __launch_bounds__(128) k_pp_update_sums(const float *X, int64_t n, int d, int ldx, const float *c,
                                                        double *D2, int first, Wide *bsum, int64_t nb, int *bad)
{
    const int lane = threadIdx.x & 31;
    const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (b >= nb) return;
    const int64_t r0 = b * kSeedBlock, r1 = r0 + kSeedBlock < n ? r0 + kSeedBlock : n;
    Wide s;
    wzero(s);
    int badl = 0;
    for (int64_t i = r0 + lane; i < r1; i += 32) {
        const float *x = X + i * ldx;
        double q = 0.0;
        for (int j = 0; j < d; ++j) {
            const double t = __dsub_rn((double)x[j], (double)c[j]);
            q = __dadd_rn(q, __dmul_rn(t, t));
        }
        const double v = first ? q : fmin(D2[i], q);
        D2[i] = v;
        wadd(s, wfrom(v, &badl));
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        const Wide o = wshfl_down(s, off);
        wadd(s, o);
    }
    if (lane == 0) bsum[b] = s;
    if (__any_sync(0xffffffffu, badl) && lane == 0) *bad = 1;
}

// one thread per group: the exact sum of its blocks
__global__ void k_pp_group_sums(const Wide *bsum, int64_t nb, Wide *gsum, int64_t ng)
{
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= ng) return;
    const int64_t b0 = g * kSeedGroup, b1 = b0 + kSeedGroup < nb ? b0 + kSeedGroup : nb;
    Wide s;
    wzero(s);
    for (int64_t b = b0; b < b1; ++b) wadd(s, bsum[b]);
    gsum[g] = s;
}

// one thread: the first row whose exact prefix sum exceeds floor(u · T) — found group by group,
// then block by block, then row by row (every prefix exact).  *out = -1 if every D² is 0.
__global__ void k_pp_select(const double *D2, int64_t n, const Wide *bsum, int64_t nb, const Wide *gsum,
                            int64_t ng, double u, int64_t *out)
{
    Wide T;
    wzero(T);
    for (int64_t g = 0; g < ng; ++g) wadd(T, gsum[g]);
    if (wzero_p(T)) { *out = -1; return; }
    const Wide target = wscale(T, u);            // < T because u < 1
    Wide run;
    wzero(run);
    int64_t g = 0;
    for (; g < ng; ++g) {
        Wide nxt = run;
        wadd(nxt, gsum[g]);
        if (wgt(nxt, target)) break;
        run = nxt;
    }
    int64_t b = g * kSeedGroup;
    const int64_t b1 = b + kSeedGroup < nb ? b + kSeedGroup : nb;
    for (; b < b1; ++b) {
        Wide nxt = run;
        wadd(nxt, bsum[b]);
        if (wgt(nxt, target)) break;
        run = nxt;
    }
    const int64_t r0 = b * kSeedBlock, r1 = r0 + kSeedBlock < n ? r0 + kSeedBlock : n;
    int bad = 0;
    for (int64_t i = r0; i < r1; ++i) {
        wadd(run, wfrom(D2[i], &bad));
        if (wgt(run, target)) { *out = i; return; }
    }
    *out = -1;                                    // unreachable: the block's sum crosses
}

size_t seed_scratch_bytes(int64_t n)
{
    const int64_t nb = (n + kSeedBlock - 1) / kSeedBlock;
    const int64_t ng = (nb + kSeedGroup - 1) / kSeedGroup;
    return (size_t)(nb + ng) * sizeof(Wide) + 16;
}

cudaError_t seed_plusplus(const float *X, int64_t n, int d, int ldx, int k, int64_t first,
                          const double *u, double *D2, void *scratch, float *crow, int64_t *dsel,
                          int64_t *chosen, cudaStream_t st)
{
    const int64_t nb = (n + kSeedBlock - 1) / kSeedBlock;
    const int64_t ng = (nb + kSeedGroup - 1) / kSeedGroup;
    Wide *bsum = static_cast<Wide *>(scratch);
    Wide *gsum = bsum + nb;
    int *bad = reinterpret_cast<int *>(gsum + ng);
    cudaError_t e = cudaMemsetAsync(bad, 0, sizeof(int), st);
    if (e != cudaSuccess) return e;
    chosen[0] = first;
    for (int m = 1; m <= k; ++m) {
        const int64_t c = chosen[m - 1];
        e = cudaMemcpyAsync(crow, X + c * ldx, (size_t)d * sizeof(float), cudaMemcpyDeviceToDevice, st);
        if (e != cudaSuccess) return e;
        k_pp_update_sums<<<(unsigned)((nb * 32 + 127) / 128), 128, 0, st>>>(X, n, d, ldx, crow, D2, m == 1, bsum, nb, bad);
        if (m == k) break;
        k_pp_group_sums<<<(unsigned)((ng + 127) / 128), 128, 0, st>>>(bsum, nb, gsum, ng);
        k_pp_select<<<1, 1, 0, st>>>(D2, n, bsum, nb, gsum, ng, u[m - 1], dsel);
        e = cudaMemcpyAsync(&chosen[m], dsel, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) return e;
        e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return e;
        if (chosen[m] < 0) return cudaErrorInvalidValue;   // fewer than k distinct rows
    }
    int hbad = 0;
    e = cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return e;
    if (hbad) return cudaErrorNotSupported;          // a D² outside the fixed point (not fp32 data)
    return cudaGetLastError();
}

}  // namespace km
