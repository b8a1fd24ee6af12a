// l2_probe2.cu -- how the match-set scan's row layout and dependence shape
// L2 read bandwidth (round 2): random 128-byte lines read by 8-lane groups,
// (a) dense over a small buffer, (b) only the FIRST line of rows spaced
// `stride` lines apart (the scan's row-start lines: stride 12 = 1536-byte
// rows at 10K rules; 11 = odd), (c) dependent: each group's next line
// address depends on the line just read (the scan's step chain), K chains.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/l2_probe2 tools/l2_probe2.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int K, bool DEP>
__global__ void __launch_bounds__(256) rows_probe(const uint4 *__restrict__ p, uint32_t nrows, uint32_t stride,
                                                  int iters, uint32_t *out) {
    const int lane = threadIdx.x & 31, grp = lane / 8, gl = lane % 8;
    uint32_t x[K];
#pragma unroll
    for (int k = 0; k < K; k++) x[k] = 0x9E3779B9u * (blockIdx.x * 128u + (threadIdx.x >> 5) * 16u + grp * 4u + k + 1u);
    uint32_t acc = 0;
    for (int it = 0; it < iters; it++) {
        uint4 v[K];
#pragma unroll
        for (int k = 0; k < K; k++) {
            x[k] = x[k] * 1664525u + 1013904223u;
            const uint32_t row = (uint32_t)(((uint64_t)(x[k] >> 8) * nrows) >> 24);
            v[k] = __ldg(p + ((size_t)row * stride) * 8 + gl);
        }
#pragma unroll
        for (int k = 0; k < K; k++) {
            const uint32_t a = v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
            acc ^= a;
            if (DEP) x[k] ^= __shfl_sync(0xFFFFFFFFu, a, grp * 8) & 1u;  // next address waits for this line
        }
    }
    if (acc == 0x12345678u) *out = acc;
}

int main() {
    uint32_t *out;
    cudaMalloc(&out, 4);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const size_t bytes = (size_t)160 << 20;
    uint4 *p;
    cudaMalloc(&p, bytes);
    cudaMemset(p, 0, bytes);
    struct Cfg { const char *name; uint32_t nrows, stride; };
    const Cfg cfgs[] = {{"dense 10 MB", 80000, 1}, {"row starts, stride 12 (1536 B rows)", 80000, 12},
                        {"row starts, stride 11", 80000, 11}, {"dense 48 MB", 393216, 1}};
    for (const Cfg &c : cfgs) {
        for (int dep = 0; dep < 2; dep++) {
            for (int occ : {5, 8}) {
                const int iters = 2048;
                auto run = [&](int it) {
                    if (dep) rows_probe<4, true><<<sms * occ, 256>>>(p, c.nrows, c.stride, it, out);
                    else rows_probe<4, false><<<sms * occ, 256>>>(p, c.nrows, c.stride, it, out);
                };
                run(16);
                cudaEventRecord(a);
                run(iters);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                const double lines = (double)sms * occ * 256 / 8 * 4 * iters;
                printf("%-40s %s blocks/SM %d: %8.1f GB/s\n", c.name, dep ? "dependent " : "independent", occ,
                       lines * 128 / ms / 1e6);
            }
        }
    }
    return 0;
}
