// Max relative error of sqrt.approx.ftz.f32 and of sqrt.rn over [1, 4) (all fp32 values;
// sqrt(x * 4^e) = 2^e sqrt(x), so this range covers every normal input).
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cmath>
__global__ void k(unsigned long long *worst_bits, int mode)
{
    const uint32_t lo = 0x3f800000u, hi = 0x40800000u;   // [1, 4)
    double worst = 0;
    for (uint32_t b = lo + blockIdx.x * blockDim.x + threadIdx.x; b < hi; b += gridDim.x * blockDim.x) {
        const float x = __uint_as_float(b);
        float y;
        if (mode == 0) asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
        else { float r; asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); y = x * r; }
        const double e = fabs((double)y - sqrt((double)x)) / sqrt((double)x);
        worst = fmax(worst, e);
    }
    atomicMax(worst_bits, (unsigned long long)__double_as_longlong(worst));
}
int main()
{
    unsigned long long *w; cudaMallocManaged(&w, 8);
    for (int mode = 0; mode < 2; ++mode) {
        *w = 0; k<<<592, 256>>>(w, mode); cudaDeviceSynchronize();
        double v; memcpy(&v, w, 8);
        printf("%s max rel err = %.3e = 2^%.2f\n", mode ? "x*rsqrt.approx" : "sqrt.approx", v, log2(v));
    }
    return 0;
}
