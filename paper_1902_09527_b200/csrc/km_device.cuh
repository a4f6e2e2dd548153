// km_device.cuh — device helpers shared by the CUDA-core and tensor-core assignment kernels:
// packed fp32x2 distance, exact-mode interval bounds, fp64 refinement, warp reduction.
#pragma once
#include <math.h>
#include <stdint.h>

#include "km_kernels.cuh"

namespace km {

// ---------------------------------------------------------------------------------------
// packed fp32x2 arithmetic (sm_100a FADD2/FFMA2)
__device__ __forceinline__ float2 add2(float2 a, float2 b)
{
    float2 r;
    asm("{\n\t.reg .b64 ra, rb, rr;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "add.rn.f32x2 rr, ra, rb;\n\tmov.b64 {%0, %1}, rr;\n\t}"
        : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return r;
}

__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c)
{
    float2 r;
    asm("{\n\t.reg .b64 ra, rb, rc, rr;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
        "fma.rn.f32x2 rr, ra, rb, rc;\n\tmov.b64 {%0, %1}, rr;\n\t}"
        : "=f"(r.x), "=f"(r.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return r;
}

// Squared distance ||x - c||^2 in fp32, direct-difference form: t = x + (-c) (IEEE x - c),
// squares accumulated with fma in four interleaved partial sums.  Relative error of the
// result <= (DP/4 + 4) * 2^-24 (+O(2^-48)); DESIGN.md "Exact mode" bounds sqrt of it by gamma.
__device__ __forceinline__ float4 lds128(uint32_t addr)
{
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
}

// Centroid row source: shared memory (32-bit shared-window address) or global (__ldg).
template <bool SMEM> struct CRow;
template <> struct CRow<true> {
    uint32_t base;
    __device__ __forceinline__ float4 ld(int c, int DP, int j) const
    {
        return lds128(base + (uint32_t)((c * DP + j) * 4));
    }
};
template <> struct CRow<false> {
    const float *base;
    __device__ __forceinline__ float4 ld(int c, int DP, int j) const
    {
        return __ldg(reinterpret_cast<const float4 *>(base + (int64_t)c * DP + j));
    }
};

template <int DP, bool SMEM>
__device__ __forceinline__ float dist2(const float (&x)[DP], const CRow<SMEM> &cr, int cidx)
{
    float2 acc0 = make_float2(0.f, 0.f), acc1 = make_float2(0.f, 0.f);
#pragma unroll
    for (int j = 0; j < DP; j += 4) {
        float4 c = cr.ld(cidx, DP, j);
        float2 t0 = add2(make_float2(x[j], x[j + 1]), make_float2(c.x, c.y));
        float2 t1 = add2(make_float2(x[j + 2], x[j + 3]), make_float2(c.z, c.w));
        acc0 = fma2(t0, t0, acc0);
        acc1 = fma2(t1, t1, acc1);
    }
    float2 s = add2(acc0, acc1);
    return s.x + s.y;
}

// Directed square roots from the hardware approximation: sqrt.approx.ftz.f32 has max relative
// error 2^-23.25 over every normal input (exhaustive over [1, 4), tools/probes/sqrt_probe.cu
// on B200; the result scales exactly with the exponent), so a 2^-21 margin applied with a
// directed multiply bounds the true root from above / below.  FTZ: inputs below 2^-126 give 0
// (a valid lower bound); the upper bound is floored at sqrt(2^-126) < 1.1e-19.
__device__ __forceinline__ float sqrt_approx(float q)
{
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(q));
    return r;
}
__device__ __forceinline__ float sqrt_up(float q) { return fmaxf(__fmul_ru(sqrt_approx(q), 1.00000048f), 1.1e-19f); }
__device__ __forceinline__ float sqrt_dn(float q) { return __fmul_rd(sqrt_approx(q), 0.99999952f); }

// Rigorous distance interval of an fp32 squared distance q (exact mode):
// true d(x, C64[c]) in [lower, upper] (gamma folded into g_up/g_dn, eps = eps_C).
__device__ __forceinline__ float upper_d(float q, float g_up, float eps)
{
    return __fadd_ru(__fmul_ru(sqrt_up(q), g_up), eps);
}
__device__ __forceinline__ float lower_d(float q, float g_dn, float eps)
{
    return fmaxf(0.f, __fsub_rd(__fmul_rd(sqrt_dn(q), g_dn), eps));
}

constexpr uint64_t kSentinel = 0xffffffff00000000ull;   // h = NaN (never < u), c = 0
__device__ __forceinline__ float key_h(uint64_t key) { return __uint_as_float((uint32_t)(key >> 32)); }
__device__ __forceinline__ int key_c(uint64_t key) { return (int)(uint32_t)(key & 0xffffffffull); }

// fp64 re-evaluation (exact mode): argmin over {A} u {c' : H[A][c'] < ut} (MTI) or over
// all k (nl == nullptr), lowest index on ties; distances in the oracle's direct form.
static __device__ __noinline__ int refine64(const float *xrow, int d, const double *C64, int k, int A,
                                     const uint64_t *nl, float ut, float *unew)
{
    double best = INFINITY;
    int bc = 0x7fffffff;
    auto eval = [&](int c) {
        const double *cc = C64 + (int64_t)c * d;
        double s = 0.0;
        for (int j = 0; j < d; ++j) {
            double t = __dsub_rn((double)xrow[j], cc[j]);
            s = __dadd_rn(s, __dmul_rn(t, t));
        }
        if (s < best || (s == best && c < bc)) { best = s; bc = c; }
    };
    if (nl) {
        eval(A);
        for (int j = 0;; ++j) {          // row ends with a sentinel whose h is NaN
            uint64_t key = nl[j];
            if (!(key_h(key) < ut)) break;
            eval(key_c(key));
        }
    } else {
        for (int c = 0; c < k; ++c) eval(c);
    }
    *unew = __double2float_ru(sqrt(best) * (1.0 + 1e-12));
    return bc;
}

// ---------------------------------------------------------------------------------------
// warp transpose-reduction of DP fp64 values per lane: afterwards lane L holds, in v[0..W),
// the warp sums of components tr_base(L) + i.  Uses DP-1 (+log2(32/DP)) double shuffles.
template <int DP> struct Red {
    static constexpr int W = DP >= 32 ? DP / 32 : 1;
    static constexpr int LASTO = DP >= 32 ? 1 : 32 / DP;
};

template <int O, int Wc, int DP>
__device__ __forceinline__ void tr_step(double (&v)[DP], int lane)
{
    if constexpr (O >= 1) {
        if constexpr (Wc > 1) {
            const bool up = (lane & O) != 0;
#pragma unroll
            for (int i = 0; i < Wc / 2; ++i) {
                double send = up ? v[i] : v[i + Wc / 2];
                double keep = up ? v[i + Wc / 2] : v[i];
                v[i] = keep + __shfl_xor_sync(kFull, send, O);
            }
            tr_step<O / 2, Wc / 2, DP>(v, lane);
        } else {
            v[0] += __shfl_xor_sync(kFull, v[0], O);
            tr_step<O / 2, 1, DP>(v, lane);
        }
    }
}

template <int DP>
__device__ __forceinline__ int tr_base(int lane)
{
    int base = 0, w = DP;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        if (w > 1) {
            if (lane & o) base += w / 2;
            w >>= 1;
        }
    }
    return base;
}

// Per-warp run accumulator: the fp64 sums of the current run cluster R live in registers
// (lane-distributed components) and are flushed with fp64 RED to acc only when R changes.
template <int DP>
struct RunAcc {
    int R = -1;
    int cnt = 0;
    double v[Red<DP>::W];
    __device__ __forceinline__ void clear()
    {
#pragma unroll
        for (int i = 0; i < Red<DP>::W; ++i) v[i] = 0.0;
        cnt = 0;
    }
    __device__ __forceinline__ void flush(double *acc, int d, int lane)
    {
        if (R < 0) return;
        double *row = acc + (int64_t)R * (DP + 1);
        const bool writer = (lane & (Red<DP>::LASTO - 1)) == 0;
        const int base = tr_base<DP>(lane);
        if (writer) {
#pragma unroll
            for (int i = 0; i < Red<DP>::W; ++i)
                if (base + i < d && v[i] != 0.0) atomicAdd(row + base + i, v[i]);
        }
        if (lane == 0 && cnt) atomicAdd(row + DP, (double)cnt);
    }
};

template <int DP>
__device__ __forceinline__ void reduce_batch(RunAcc<DP> &ra, const float (&x)[DP], int anew,
                                             bool valid, double *acc, int d, int lane)
{
    unsigned mR = __ballot_sync(kFull, valid && anew == ra.R);
    if (mR == 0) {
        unsigned mv = __ballot_sync(kFull, valid);
        if (mv == 0) return;
        int M = __shfl_sync(kFull, anew, __ffs(mv) - 1);
        ra.flush(acc, d, lane);
        ra.clear();
        ra.R = M;
        mR = __ballot_sync(kFull, valid && anew == M);
    }
    const bool in = (mR >> lane) & 1u;
    // first transposition step (offset 16) on fp32 values, widened to fp64 when added
    constexpr int H = DP / 2;
    const bool up = (lane & 16) != 0;
    double v[H];
#pragma unroll
    for (int i = 0; i < H; ++i) {
        const float lo = in ? x[i] : 0.f, hi = in ? x[i + H] : 0.f;
        const float recv = __shfl_xor_sync(kFull, up ? lo : hi, 16);
        v[i] = (double)(up ? hi : lo) + (double)recv;
    }
    tr_step<8, H, H>(v, lane);
#pragma unroll
    for (int i = 0; i < Red<DP>::W; ++i) ra.v[i] += v[i];
    ra.cnt += __popc(mR);
    if (valid && !in) {      // lane leaves the warp's run cluster: direct fp64 RED
        double *row = acc + (int64_t)anew * (DP + 1);
#pragma unroll
        for (int j = 0; j < DP; ++j)          // compile-time indices keep x in registers
            if (j < d) atomicAdd(row + j, (double)x[j]);
        atomicAdd(row + DP, 1.0);
    }
}


// fp64 delta reduction of a row that moved from a to b: S[b] += x, S[a] -= x (counts +-1)
template <int DP>
__device__ __forceinline__ void move_delta(double *acc, int d, int a, int b, const float (&x)[DP])
{
    double *ra = acc + (int64_t)a * (DP + 1), *rb = acc + (int64_t)b * (DP + 1);
#pragma unroll
    for (int j = 0; j < DP; ++j)
        if (j < d) {
            const double v = (double)x[j];
            atomicAdd(rb + j, v);
            atomicAdd(ra + j, -v);
        }
    atomicAdd(rb + DP, 1.0);
    atomicAdd(ra + DP, -1.0);
}

}  // namespace km
