// Microbenchmark: issue throughput of the instruction classes the MTI walk / epilogue uses,
// measured on B200 (cycles per warp-instruction per SM sub-partition).
#include <cstdio>
#include <cuda_runtime.h>

#define N_ITER 4096
template <int OP>
__global__ void k(float *out, float a0, float b0, int ia0, long long *cyc)
{
    float v[8];
    double dacc[4] = {0, 0, 0, 0};
    unsigned iv[8];
    for (int i = 0; i < 8; ++i) { v[i] = a0 + threadIdx.x * 1e-3f + i; iv[i] = ia0 + threadIdx.x + i * 7; }
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) {   // FFMA2 (3 reg)
                if (i < 4) asm volatile("{.reg .b64 ra, rb; mov.b64 ra, {%0,%1}; mov.b64 rb, {%2,%3}; fma.rn.f32x2 ra, ra, rb, ra; mov.b64 {%0,%1}, ra;}"
                             : "+f"(v[2*i]), "+f"(v[2*i+1]) : "f"(b0), "f"(a0));
            } else if (OP == 1) {   // FFMA 3-reg
                asm volatile("fma.rn.f32 %0, %0, %1, %0;" : "+f"(v[i]) : "f"(b0));
            } else if (OP == 2) {   // FADD2
                if (i < 4) asm volatile("{.reg .b64 ra, rb; mov.b64 ra, {%0,%1}; mov.b64 rb, {%2,%3}; add.rn.f32x2 ra, ra, rb; mov.b64 {%0,%1}, ra;}"
                             : "+f"(v[2*i]), "+f"(v[2*i+1]) : "f"(b0), "f"(a0));
            } else if (OP == 3) {   // FMNMX
                asm volatile("min.f32 %0, %0, %1;" : "+f"(v[i]) : "f"(v[(i + 3) & 7]));
            } else if (OP == 4) {   // FMNMX3
                asm volatile("min.f32 %0, %0, %1, %2;" : "+f"(v[i]) : "f"(v[(i + 3) & 7]), "f"(v[(i + 5) & 7]));
            } else if (OP == 5) {   // VIMNMX (u32)
                asm volatile("min.u32 %0, %0, %1;" : "+r"(iv[i]) : "r"(iv[(i + 3) & 7]));
            } else if (OP == 6) {   // LOP3
                asm volatile("lop3.b32 %0, %0, %1, %2, 0xE8;" : "+r"(iv[i]) : "r"(iv[(i + 3) & 7]), "r"(iv[(i + 5) & 7]));
            } else if (OP == 7) {   // FADD scalar
                asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(v[i]) : "f"(v[(i + 3) & 7]));
            } else if (OP == 8) {   // mixed: 1 FFMA2 + 1 FMNMX (dual issue across pipes?)
                if (i < 4) asm volatile("{.reg .b64 ra, rb; mov.b64 ra, {%0,%1}; mov.b64 rb, {%2,%3}; fma.rn.f32x2 ra, ra, rb, ra; mov.b64 {%0,%1}, ra;}"
                             : "+f"(v[2*i]), "+f"(v[2*i+1]) : "f"(b0), "f"(a0));
                asm volatile("min.u32 %0, %0, %1;" : "+r"(iv[i]) : "r"(iv[(i + 3) & 7]));
            } else if (OP == 10) {  // F2F.F64.F32 + DADD accumulate
                dacc[i & 3] += (double)v[i];
            } else if (OP == 11) {  // DADD only
                dacc[i & 3] += dacc[(i + 1) & 3];
            } else if (OP == 12) {  // SHFL
                v[i] = __shfl_xor_sync(0xffffffffu, v[i], 1 + (i & 3));
            } else if (OP == 13) {  // FSETP + SEL (predicated select)
                iv[i] = v[i] < v[(i + 3) & 7] ? iv[i] : iv[(i + 1) & 7];
            } else if (OP == 9) {   // FMUL imm / FFMA imm
                asm volatile("fma.rn.f32 %0, %0, 0f3F800001, 0f3F000000;" : "+f"(v[i]));
            }
        }
    }
    long long t1 = clock64();
    float s = 0; unsigned si = 0;
    for (int i = 0; i < 8; ++i) { s += v[i]; si ^= iv[i]; }
    s += (float)(dacc[0] + dacc[1] + dacc[2] + dacc[3]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s + si;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main()
{
    float *out; long long *cyc;
    cudaMalloc(&out, 148 * 1024 * 4 * 8);
    cudaMalloc(&cyc, 8);
    const char *names[] = {"FFMA2", "FFMA", "FADD2", "FMNMX", "FMNMX3", "IMNMX", "LOP3", "FADD", "FFMA2+IMNMX", "FFMA imm", "F2F+DADD", "DADD", "SHFL", "FSETP+SEL"};
    void (*ks[])(float *, float, float, int, long long *) = {k<0>, k<1>, k<2>, k<3>, k<4>, k<5>, k<6>, k<7>, k<8>, k<9>, k<10>, k<11>, k<12>, k<13>};
    for (int op = 0; op < 14; ++op) {
        for (int threads : {256, 1024}) {
            ks[op]<<<148, threads>>>(out, 1.0f, 0.999f, 3, cyc);
            cudaDeviceSynchronize();
            long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            // warps per SMSP = threads/32/4; instr per warp = N_ITER*8 (x2 for op 8)
            double wps = threads / 128.0;
            double instr = (double)N_ITER * ((op == 0 || op == 2) ? 4 : (op == 8 ? 12 : 8));
            printf("%-12s threads=%4d cycles/warp-instr/SMSP = %.3f\n", names[op], threads, c / (instr * wps));
        }
    }
    cudaError_t e = cudaGetLastError();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
