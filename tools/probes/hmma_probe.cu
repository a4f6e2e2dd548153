// Throughput of legacy mma.sync m16n8k8 TF32 (HMMA) on B200: cycles per warp-MMA per SMSP.
#include <cstdio>
#include <cstdint>
__global__ void k(float *out, long long *cyc, int iters)
{
    uint32_t a[4], b[2];
    for (int i = 0; i < 4; ++i) a[i] = __float_as_uint(1.0f + threadIdx.x * 1e-3f + i);
    for (int i = 0; i < 2; ++i) b[i] = __float_as_uint(0.5f + i);
    float c[8][4];
    for (int m = 0; m < 8; ++m) for (int i = 0; i < 4; ++i) c[m][i] = 0.f;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int m = 0; m < 8; ++m)
            asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+f"(c[m][0]), "+f"(c[m][1]), "+f"(c[m][2]), "+f"(c[m][3])
                         : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
    long long t1 = clock64();
    float s = 0;
    for (int m = 0; m < 8; ++m) for (int i = 0; i < 4; ++i) s += c[m][i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main()
{
    float *out; long long *cyc;
    cudaMalloc(&out, 148 * 1024 * 4 * 4);
    cudaMallocManaged(&cyc, 8);
    for (int threads : {128, 256, 512, 1024}) {
        k<<<148, threads>>>(out, cyc, 2000);
        cudaDeviceSynchronize();
        const double wps = threads / 128.0;   // warps per SMSP
        printf("threads=%4d  cycles per warp-HMMA per SMSP = %.2f  (TF32 FMA/clk/SM = %.0f)\n", threads,
               (double)*cyc / (2000.0 * 8 * wps), 1024.0 * 4 / ((double)*cyc / (2000.0 * 8 * wps)));
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
