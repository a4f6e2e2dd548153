// Effective HBM bandwidth of gathering 32-B rows through a permutation (random vs sorted vs
// "mostly sorted": runs of 64 consecutive rows), B200.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <algorithm>
__global__ void gather(const float4 *X, const int *idx, float4 *out, int n)
{
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int r = idx[i];
        float4 a = X[2 * (size_t)r], b = X[2 * (size_t)r + 1];
        if (a.x == 1.2345f && b.y == 7.f) out[i] = a;   // keep the loads
    }
}
int main()
{
    const int n = 65608366;
    float4 *X; int *idx; float4 *out;
    cudaMalloc(&X, (size_t)n * 32); cudaMalloc(&idx, (size_t)n * 4); cudaMalloc(&out, 16 * 1024);
    cudaMemset(X, 0, (size_t)n * 32);
    std::vector<int> h(n);
    std::mt19937 g(1);
    for (int mode = 0; mode < 3; ++mode) {
        for (int i = 0; i < n; ++i) h[i] = i;
        if (mode == 1) std::shuffle(h.begin(), h.end(), g);
        if (mode == 2) {   // runs of 64 consecutive rows in random order (cluster-sorted, rows scattered)
            std::vector<int> blocks(n / 64);
            for (int b = 0; b < n / 64; ++b) blocks[b] = b;
            std::shuffle(blocks.begin(), blocks.end(), g);
            for (int b = 0; b < n / 64; ++b) for (int j = 0; j < 64; ++j) h[b * 64 + j] = blocks[b] * 64 + j;
        }
        cudaMemcpy(idx, h.data(), (size_t)n * 4, cudaMemcpyHostToDevice);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0);
            gather<<<148 * 8, 256>>>(X, idx, out, n);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (rep == 2) printf("mode %d (%s): %.3f ms, %.0f GB/s of rows (+idx)\n", mode,
                                 mode == 0 ? "sequential" : mode == 1 ? "random" : "runs of 64", ms,
                                 (double)n * 36 / ms / 1e6);
        }
    }
    return 0;
}
