// km_ti.cu — Elkan's triangle-inequality (TI) pruning as the GPU baseline MTI is compared with
// (SURVEY §8(f) NEXT-3), sm_100a.
//
// Method: PAPER.md §2 (876-885): "triangle inequality (TI) with bounds" relying on "a sparse lower
// bound matrix of size O(kn)"; the paper's claims about it are PAPER.md:17-24 (MTI does at most
// 2x TI's distances, is >= 2x faster and uses up to 5x less memory).  Algorithm as the oracle's
// oracle_ti_pass (reading B10):
//   l[c] <- max(0, l[c] - f(c)) for every c;  u <- u + f(a0)
//   u <= s(a0): keep (clause 1, 0 distances)
//   else best = a0; for c = 0..k-1 (index order), c != best:
//     if u > l[c] and u > H[best][c]: tighten once (u = d(x, a0), l[a0] = u, 1 distance);
//       if still u > l[c] and u > H[best][c]: l[c] = d(x, c) (1 distance); c closer -> best = c, u = d
//
// B200 realisation.  One lane = one row, rows in the caller's order (TI keeps an n x k matrix
// per row, so the rows are never re-bucketed); the lower bounds are stored centroid-major within
// 32-row groups, so for every c the 32 lanes of a warp read and write one coalesced 128-B
// line — and the k lines of a 32-row group are contiguous (L[((i / 32) k + c) 32 + i % 32], so a warp
// streams one 128 k-byte block): the pass is bound by the 8 k bytes per row of lower-bound traffic (the O(nk)
// maintenance cost the paper attributes to TI).  Exact mode as in the MTI
// engines: bounds in fp32 with directed rounding (l rounded down, u up, H down), so every prune
// is sound; the winner among the evaluated candidates is certified by the top-2 intervals or
// re-evaluated in fp64 (refine64 over the MTI candidate set of a0, a superset of every
// candidate that can beat a0), so assignments equal the fp64 argmin.  S3: the rows that move
// add fp64 deltas (B5) to per-CTA slabs.  Iteration 1 (FIRST) evaluates every centroid and
// initialises l[c] = d(x, c).
#include "km_device.cuh"
#include "km_kernels.cuh"

namespace km {

constexpr int kTiThreads = 256;
constexpr int kTiBatch = 8;      // lower bounds loaded per batch (loads in flight per lane)

// resident CTAs per SM requested from ptxas (registers): 4 (64 registers) up to d = 16, 3 at 32
template <int DP> constexpr int ti_min_blocks() { return DP <= 16 ? 4 : (DP <= 32 ? 3 : 2); }

template <int DP, bool CSMEM, bool HSMEM, bool FIRST>
__global__ void __launch_bounds__(kTiThreads, ti_min_blocks<DP>())
k_ti(AssignParams p, float *__restrict__ L, const float *__restrict__ Hm)
{
    extern __shared__ __align__(16) float smem[];
    const int k = p.k;
    const int k4 = (k + 3) & ~3;
    float *sC = smem;                                  // k * DP (CSMEM)
    float *sF = smem + (CSMEM ? k * DP : 0);           // k
    float *sS = sF + k4;                               // k
    float *sH = sS + k4;                               // k * k (HSMEM)
    if (CSMEM) {
        const float4 *src = reinterpret_cast<const float4 *>(p.Cneg);
        float4 *dst = reinterpret_cast<float4 *>(sC);
        for (int i = threadIdx.x; i < k * DP / 4; i += blockDim.x) dst[i] = src[i];
    }
    for (int i = threadIdx.x; i < k; i += blockDim.x) { sF[i] = p.f[i]; sS[i] = p.s[i]; }
    if (HSMEM)
        for (int i = threadIdx.x; i < k * k; i += blockDim.x) sH[i] = Hm[i];
    __syncthreads();
    const float *H = HSMEM ? sH : Hm;
    CRow<CSMEM> Cn;
    if constexpr (CSMEM) Cn.base = (uint32_t)__cvta_generic_to_shared(sC);
    else Cn.base = p.Cneg;
    double *acc = p.acc + (int64_t)(blockIdx.x % p.nslab) * k * (DP + 1);
    const float eps = *p.eps;
    const int64_t n = p.n;
    const int lane = threadIdx.x & 31;
    unsigned long long c_changed = 0, c_dists = 0, c_clause1 = 0, c_refined = 0;

    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < n; base += stride) {
        const int64_t row = base + lane;
        const bool valid = row < n;
        float x[DP];
        {
            const float4 *xr = reinterpret_cast<const float4 *>(p.X + (valid ? row : 0) * DP);
#pragma unroll
            for (int j = 0; j < DP / 4; ++j) {
                const float4 t = valid ? __ldg(xr + j) : make_float4(0.f, 0.f, 0.f, 0.f);
                x[4 * j] = t.x; x[4 * j + 1] = t.y; x[4 * j + 2] = t.z; x[4 * j + 3] = t.w;
            }
        }
        float *Lr = L + (base >> 5) * (int64_t)k * 32 + lane;   // bound c of this row: Lr[32 c]
        int anew;
        float unew;
        if constexpr (FIRST) {
            // iteration 1: every centroid, l[c] = d(x, c) rounded down
            float bq = INFINITY, q2 = INFINITY;
            int bc = 0;
            for (int c = 0; c < k; ++c) {
                const float q = dist2<DP, CSMEM>(x, Cn, c);
                if (valid) Lr[32 * c] = lower_d(q, p.g_dn, eps);
                q2 = fminf(q2, fmaxf(q, bq));
                bc = q < bq ? c : bc;
                bq = fminf(q, bq);
            }
            const float ub = upper_d(bq, p.g_up, eps);
            anew = bc;
            unew = ub;
            if (valid && q2 < INFINITY && lower_d(q2, p.g_dn, eps) <= ub) {
                anew = refine64(p.X + row * DP, p.d, p.C64, k, 0, nullptr, 0.f, &unew);
                ++c_refined;
            }
        } else {
            const int a0 = valid ? __ldg(p.a + row) : 0;
            float ub = valid ? __fadd_ru(__ldg(p.u + row), sF[a0]) : 0.f;   // u += f(a0)
            const bool c1 = valid && ub <= sS[a0];                            // clause 1
            c_clause1 += c1;
            bool live = valid && !c1, tight = false;
            int best = a0;
            float bq = INFINITY, q2 = INFINITY, la = 0.f, ut = 0.f;
            unsigned nd = 0;
            // the lower bounds are streamed kTiBatch at a time (independent loads in flight:
            // the pass is bound by this O(nk) traffic)
            for (int c0 = 0; c0 < k; c0 += kTiBatch) {
                float lb[kTiBatch];
#pragma unroll
                for (int j = 0; j < kTiBatch; ++j)
                    lb[j] = (valid && c0 + j < k) ? __ldcs(Lr + 32 * (c0 + j)) : 0.f;
#pragma unroll
                for (int j = 0; j < kTiBatch; ++j) {
                    const int c = c0 + j;
                    if (c >= k) break;
                    float l = fmaxf(0.f, __fsub_rd(lb[j], sF[c]));
                    if (tight && c == a0) l = la;
                    if (live && c != best && ub > l && ub > H[best * k + c]) {
                        if (!tight) {                    // Elkan step 3a: u = d(x, C[a0]), once
                            bq = dist2<DP, CSMEM>(x, Cn, a0);
                            ub = upper_d(bq, p.g_up, eps);
                            ut = ub;
                            la = lower_d(bq, p.g_dn, eps);
                            tight = true;
                            ++nd;
                            if (a0 < c) Lr[32 * a0] = la;   // already written this pass
                        }
                        if (ub > l && ub > H[best * k + c]) {     // step 3b with the tightened u
                            const float q = dist2<DP, CSMEM>(x, Cn, c);
                            ++nd;
                            l = lower_d(q, p.g_dn, eps);
                            q2 = fminf(q2, fmaxf(q, bq));
                            if (q < bq) { bq = q; best = c; ub = upper_d(q, p.g_up, eps); }
                        }
                    }
                    if (valid) __stcs(Lr + 32 * c, l);
                }
            }
            anew = best;
            unew = ub;
            if (tight && q2 < INFINITY && lower_d(q2, p.g_dn, eps) <= upper_d(bq, p.g_up, eps)) {
                anew = refine64(p.X + row * DP, p.d, p.C64, k, a0, p.NL + (int64_t)a0 * p.ks, ut, &unew);
                ++c_refined;
            }
            c_dists += nd;
            if (valid && anew != a0) {
                ++c_changed;
                move_delta<DP>(acc, p.d, a0, anew, x);   // S3 as a delta (B5)
            }
        }
        if (valid) {
            p.a[row] = anew;
            p.u[row] = unew;
        }
    }
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
    }
}

// H in index order (k x k fp32, rounded down as k_prep's neighbour lists; H[c][c] = 0)
__global__ void k_prep_ti(const uint64_t *NL, int k, int ks, float *Hm)
{
    const int c = blockIdx.x;
    const uint64_t *nl = NL + (int64_t)c * ks;
    for (int j = threadIdx.x; j < k - 1; j += blockDim.x) {
        const uint64_t key = nl[j];
        Hm[(int64_t)c * k + key_c(key)] = key_h(key);
    }
    if (threadIdx.x == 0) Hm[(int64_t)c * k + c] = 0.f;
}

cudaError_t launch_prep_ti(const uint64_t *NL, int k, int ks, float *Hm, cudaStream_t st)
{
    k_prep_ti<<<k, 128, 0, st>>>(NL, k, ks, Hm);
    return cudaGetLastError();
}

static size_t ti_smem(int DP, bool csmem, bool hsmem, int k)
{
    const int k4 = (k + 3) & ~3;
    return (size_t)((csmem ? k * DP : 0) + 2 * k4 + (hsmem ? k * k : 0)) * sizeof(float);
}

bool ti_h_smem(int DP, bool csmem, int k) { return ti_smem(DP, csmem, true, k) <= 200 * 1024; }

typedef void (*ti_kernel_t)(AssignParams, float *, const float *);

template <int DP>
static ti_kernel_t ti_pick(bool cs, bool hs, bool first)
{
    switch ((cs ? 4 : 0) + (hs ? 2 : 0) + (first ? 1 : 0)) {
    case 0: return k_ti<DP, false, false, false>;
    case 1: return k_ti<DP, false, false, true>;
    case 2: return k_ti<DP, false, true, false>;
    case 3: return k_ti<DP, false, true, true>;
    case 4: return k_ti<DP, true, false, false>;
    case 5: return k_ti<DP, true, false, true>;
    case 6: return k_ti<DP, true, true, false>;
    case 7: return k_ti<DP, true, true, true>;
    }
    return nullptr;
}

static ti_kernel_t ti_kernel(int DP, bool cs, bool hs, bool first)
{
    switch (DP) {
    case 4: return ti_pick<4>(cs, hs, first);
    case 8: return ti_pick<8>(cs, hs, first);
    case 16: return ti_pick<16>(cs, hs, first);
    case 32: return ti_pick<32>(cs, hs, first);
    case 64: return ti_pick<64>(cs, hs, first);
    }
    return nullptr;
}

int ti_grid(int DP, bool csmem, int k, int num_sms)
{
    const bool hs = ti_h_smem(DP, csmem, k);
    int best = num_sms;
    for (int first = 0; first < 2; ++first) {
        ti_kernel_t kern = ti_kernel(DP, csmem, hs, first != 0);
        if (!kern) return num_sms;
        const size_t sm = ti_smem(DP, csmem, hs, k);
        if (sm > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kTiThreads, sm);
        best = (per_sm < 1 ? 1 : per_sm) * num_sms;
    }
    return best;
}

cudaError_t launch_ti(int DP, bool csmem, bool first, const AssignParams &p, float *L, const float *Hm, int grid,
                      cudaStream_t st)
{
    const bool hs = ti_h_smem(DP, csmem, p.k);
    ti_kernel_t kern = ti_kernel(DP, csmem, hs, first);
    if (!kern) return cudaErrorInvalidValue;
    const size_t sm = ti_smem(DP, csmem, hs, p.k);
    if (sm > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e != cudaSuccess) return e;
    }
    kern<<<grid, kTiThreads, sm, st>>>(p, L, Hm);
    return cudaGetLastError();
}

}  // namespace km
