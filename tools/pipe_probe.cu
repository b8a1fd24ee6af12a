// Throughput probe: warp-instructions per SM-cycle for a few instruction
// kinds, 8 independent chains per thread, full occupancy.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pipe_probe tools/pipe_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096
template <int KIND>
__global__ void probe(float *out, float a0, float b0, int n) {
    float f[8];
    unsigned u[8];
    bool p[8];
#pragma unroll
    for (int k = 0; k < 8; k++) { f[k] = a0 + threadIdx.x + k; u[k] = threadIdx.x * 7 + k; p[k] = (threadIdx.x >> k) & 1; }
    for (int it = 0; it < n; it++) {
#pragma unroll
        for (int k = 0; k < 8; k++) {
            if (KIND == 0) {  // ISETP chain (predicate result fed back)
                asm volatile("{.reg .pred q; setp.le.u32 q, %1, %2; selp.u32 %0, %1, %2, q;}" : "=r"(u[k]) : "r"(u[k]), "r"(u[k ^ 1]));
            } else if (KIND == 1) {  // FSETP
                asm volatile("{.reg .pred q; setp.le.f32 q, %1, %2; selp.f32 %0, %1, %2, q;}" : "=f"(f[k]) : "f"(f[k]), "f"(f[k ^ 1]));
            } else if (KIND == 2) {  // FFMA
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f[k]) : "f"(b0), "f"(a0));
            } else if (KIND == 3) {  // IMAD
                asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(u[k]) : "r"((unsigned)n), "r"(u[k ^ 1]));
            } else if (KIND == 4) {  // LOP3
                asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(u[k]) : "r"(u[k ^ 1]), "r"(u[k ^ 2]));
            } else if (KIND == 5) {  // FMNMX
                asm volatile("min.f32 %0, %0, %1;" : "+f"(f[k]) : "f"(f[k ^ 1]));
            }
        }
    }
    float s = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) s += f[k] + u[k] + p[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int KIND>
float run(const char *name, float *out, int sms) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    int blocks = sms * 8, threads = 256;
    probe<KIND><<<blocks, threads>>>(out, 1.0f, 0.999f, 16);
    cudaEventRecord(e0);
    probe<KIND><<<blocks, threads>>>(out, 1.0f, 0.999f, ITERS);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double warp_insts = (double)blocks * threads / 32 * ITERS * 8;
    double cycles = ms * 1e-3 * clk * 1e3;
    printf("%-8s %8.3f ms  %.3f warp-inst/clk/SM (per the loop body's main op)\n", name, ms, warp_insts / cycles / sms);
    return ms;
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *out; cudaMalloc(&out, sms * 8 * 256 * sizeof(float));
    run<0>("ISETP", out, sms); run<1>("FSETP", out, sms); run<2>("FFMA", out, sms);
    run<3>("IMAD", out, sms); run<4>("LOP3", out, sms); run<5>("FMNMX", out, sms);
    return 0;
}
