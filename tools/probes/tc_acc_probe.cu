#include <cstdint>
#include <cstdio>
__device__ __forceinline__ uint32_t smem_u32(const void* p){ return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ float tf32_rna(float x){ uint32_t r; asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x)); return __uint_as_float(r); }
// D[128 x N] = A[128 x K] . B[N x K]^T, tf32, K-major, no swizzle
__global__ void k(const float* A, const float* B, float* D, int N, int K, int raw) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint32_t tmem_base_sh;
  __shared__ __align__(8) uint64_t mbar;
  const int t = threadIdx.x;
  uint8_t* sA = sm; uint8_t* sB = sm + 128 * K * 4;
  auto off = [](int r, int e, int R) { return (e / 8) * (R * 32) + (r / 8) * 256 + ((e % 8) / 4) * 128 + (r % 8) * 16 + (e % 4) * 4; };
  for (int e = 0; e < K; ++e) *(float*)(sA + off(t, e, 128)) = raw ? A[t * K + e] : tf32_rna(A[t * K + e]);
  for (int r = t; r < N; r += 128) for (int e = 0; e < K; ++e) *(float*)(sB + off(r, e, N)) = raw ? B[r * K + e] : tf32_rna(B[r * K + e]);
  if (t < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&tmem_base_sh)), "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(&mbar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base_sh;
  if (t == 0) {
    // instruction descriptor: c_format F32 (1<<4), a_format TF32 (2<<7), b_format TF32 (2<<10), K-major both, n_dim N>>3 at bit 17, m_dim 128>>4 at bit 24
    uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    for (int kb = 0; kb < K / 8; ++kb) {
      uint64_t da = 0, db = 0;
      uint32_t a0 = smem_u32(sA) + kb * 128 * 32, b0 = smem_u32(sB) + kb * N * 32;
      da = (uint64_t)((a0 >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
      db = (uint64_t)((b0 >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
      uint32_t acc = kb > 0;
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                   :: "r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&mbar)));
  }
  // wait phase 0
  asm volatile("{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\t"
               "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
               "@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}" :: "r"(smem_u32(&mbar)), "r"(0));
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int w = t / 32;
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t r[16];
    uint32_t taddr = tmem + ((uint32_t)(w * 32) << 16) + c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),"=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15]) : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 16; ++j) D[t * N + c0 + j] = __uint_as_float(r[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(128));
}

#include <random>
#include <cmath>
#include <cstring>
static float trunc19(float x){ uint32_t u; memcpy(&u,&x,4); u &= 0xFFFFE000u; float y; memcpy(&y,&u,4); return y; }
static float rna19(float x){ uint32_t u; memcpy(&u,&x,4); u += 0x1000u; u &= 0xFFFFE000u; float y; memcpy(&y,&u,4); return y; }
int main() {
  const int N = 112;
  float *A, *B, *D;
  cudaMallocManaged(&A, 128 * 128 * 4); cudaMallocManaged(&B, N * 128 * 4); cudaMallocManaged(&D, 128 * N * 4);
  std::mt19937_64 g(1);
  std::normal_distribution<double> nd(0, 1);
  std::uniform_int_distribution<int> ex(-6, 6);
  for (int K : {8, 32, 104}) for (int raw = 0; raw < 2; ++raw) {
    double worst = 0, worst_tr = 0, worst_rn = 0; double sumratio = 0; long cnt = 0;
    for (int trial = 0; trial < 6; ++trial) {
      for (int i = 0; i < 128 * K; ++i) A[i] = (float)(nd(g) * std::ldexp(1.0, ex(g)));
      for (int i = 0; i < N * K; ++i) B[i] = (float)(nd(g) * std::ldexp(1.0, ex(g)));
      if (trial >= 3) { // cancellation: B row n = -A row (n%128) partially
        for (int n = 0; n < N; ++n) for (int kk = 0; kk < K; ++kk) B[n*K+kk] = (kk % 2 ? -1.f : 1.f) * A[(n%128)*K + (kk ^ 1)];
      }
      int smem = (128 + N) * K * 4;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      k<<<1, 128, smem>>>(A, B, D, N, K, raw);
      cudaError_t e = cudaDeviceSynchronize();
      if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      for (int m = 0; m < 128; ++m) for (int n = 0; n < N; ++n) {
        double s = 0, sa = 0, st = 0, sr = 0;
        for (int kk = 0; kk < K; ++kk) {
          float a = A[m*K+kk], b = B[n*K+kk];
          double pa = raw ? (double)a : (double)rna19(a), pb = raw ? (double)b : (double)rna19(b);
          s += pa * pb; sa += fabs(pa * pb);
          st += (double)trunc19(a) * trunc19(b);
          sr += (double)rna19(a) * rna19(b);
        }
        double d = D[m*N+n];
        double r = fabs(d - (raw ? st : s)) / sa * 16777216.0;
        worst = fmax(worst, r); sumratio += r; ++cnt;
        worst_tr = fmax(worst_tr, fabs(d - st) / sa * 16777216.0);
        worst_rn = fmax(worst_rn, fabs(d - sr) / sa * 16777216.0);
      }
    }
    printf("K=%3d raw=%d  max|D-exact(tf32 inputs)|/sum|ab| = %.2f x 2^-24 (mean %.3f); vs trunc-inputs %.2f, vs rna-inputs %.2f\n",
           K, raw, worst, sumratio / cnt, worst_tr, worst_rn);
  }
  return 0;
}
