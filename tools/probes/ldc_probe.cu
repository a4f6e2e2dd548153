// Microbenchmark: how fast can a warp-uniform 32-byte candidate block reach the registers of all 32
// lanes?  LDG.256 broadcast (L1 data pipe), 2 x LDS.128 broadcast (shared memory, same pipe),
// vector LDC from the constant bank (indexed constant cache).  1024 threads per CTA, one CTA per
// SM; reports SM cycles per 32-B block per warp (all 32 warps of the SM loading concurrently).
#include <cstdio>
#include <cuda_runtime.h>

#define N_ITER 2048
__constant__ float4 Cc[4096];      // 64 KB

template <int OP>
__global__ void __launch_bounds__(1024, 1) k(const float4 *G, float *out, int base0, long long *cyc)
{
    __shared__ float4 S[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) S[i] = G[i];
    __syncthreads();
    // warp-uniform but opaque index
    int idx = __shfl_sync(0xffffffffu, base0 + (threadIdx.x >> 5) * 37, 0) & 1023;
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long t0 = clock64();
    for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int j = (idx + u * 2) & 2046;          // float4 index, even: 32-B aligned
            float4 a, b;
            if (OP == 0) {
                asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                             : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
                             : "l"(G + j));
            } else if (OP == 1) {
                a = S[j]; b = S[j + 1];
            } else {
                a = Cc[j]; b = Cc[j + 1];
            }
            acc[0] += a.x; acc[1] += a.y; acc[2] += a.z; acc[3] += a.w;
            acc[4] += b.x; acc[5] += b.y; acc[6] += b.z; acc[7] += b.w;
        }
        idx = (idx + 16 + (int)(acc[0] > 1e30f)) & 1023;   // dependence keeps the loop honest
    }
    long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 8; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main()
{
    float4 *G; float *out; long long *cyc;
    cudaMalloc(&G, 4096 * sizeof(float4)); cudaMemset(G, 0, 4096 * sizeof(float4));
    cudaMalloc(&out, 148 * 1024 * sizeof(float)); cudaMalloc(&cyc, 8);
    const char *names[3] = {"LDG.256 broadcast", "2 x LDS.128 broadcast", "LDC (constant bank, vector index)"};
    for (int op = 0; op < 3; ++op) {
        for (int rep = 0; rep < 2; ++rep) {
            if (op == 0) k<0><<<148, 1024>>>(G, out, 5, cyc);
            if (op == 1) k<1><<<148, 1024>>>(G, out, 5, cyc);
            if (op == 2) k<2><<<148, 1024>>>(G, out, 5, cyc);
            cudaDeviceSynchronize();
        }
        long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        printf("%-36s %8.2f SM cycles per 32-B block per warp (32 warps/SM)  err=%s\n", names[op],
               (double)c / (N_ITER * 8.0 * 32.0), cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
