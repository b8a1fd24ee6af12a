// l2_probe.cu -- L2 read bandwidth on this GPU: coalesced 16-byte loads over
// an L2-resident buffer (24-96 MB, replayed), and the same over a 2 GB
// buffer (HBM); 4 / 8 / 16 resident blocks per SM, best of 3.  The best
// L2-resident figure is the roofline peak of the match-set scan (bench.py).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/l2_probe tools/l2_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void rd16(const uint4 *__restrict__ p, size_t n16, int reps, uint32_t *out) {
    uint32_t acc = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int r = 0; r < reps; r++)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += stride) {
            const uint4 v = __ldg(p + i);
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
    if (acc == 0x12345678u) *out = acc;
}

// The match-set scan's access pattern: each group of 8 lanes reads one
// random 128-byte line (16 bytes per lane), K independent lines per lane in
// flight per iteration (the scan: 4, one per row), over an L2-resident buffer.
template <int K, int GL = 8>
__global__ void __launch_bounds__(256) rd_random_lines(const uint4 *__restrict__ p, uint32_t nlines, int iters,
                                                       uint32_t *out) {
    const int lane = threadIdx.x & 31, grp = lane / GL, gl = lane % GL;
    uint32_t x = 0x9E3779B9u * (blockIdx.x * 32u + (threadIdx.x >> 5) * 4u + grp + 1u);
    uint32_t acc = 0;
    for (int it = 0; it < iters; it++) {
        uint4 v[K];
#pragma unroll
        for (int k = 0; k < K; k++) {
            x = x * 1664525u + 1013904223u;           // per-group LCG (group-uniform)
            const uint32_t line = (uint32_t)(((uint64_t)(x >> 8) * nlines) >> 24);
            v[k] = __ldg(p + (size_t)line * GL + gl);
        }
#pragma unroll
        for (int k = 0; k < K; k++) acc ^= v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
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
    double best_l2 = 0, best_hbm = 0;
    for (size_t mb : {16, 32, 48, 64, 2048}) {
        const size_t bytes = mb << 20;
        uint4 *p;
        cudaMalloc(&p, bytes);
        cudaMemset(p, 1, bytes);
        const int reps = mb >= 1024 ? 3 : 60;
        for (int occ : {4, 8, 16}) {
            for (int t = 0; t < 3; t++) {
                rd16<<<sms * occ, 256>>>(p, bytes / 16, 1, out);
                cudaEventRecord(a);
                rd16<<<sms * occ, 256>>>(p, bytes / 16, reps, out);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                const double gbs = bytes * (double)reps / ms / 1e6;
                printf("rd16   %5zu MB x%2d  blocks/SM %2d: %8.1f GB/s\n", mb, reps, occ, gbs);
                if (mb >= 1024) best_hbm = gbs > best_hbm ? gbs : best_hbm;
                else best_l2 = gbs > best_l2 ? gbs : best_l2;
            }
        }
        cudaFree(p);
    }
    // random 128-byte lines, 8-lane groups, K lines in flight per lane
    double best_rl = 0;
    {
        const size_t bytes = (size_t)48 << 20;
        uint4 *p;
        cudaMalloc(&p, bytes);
        cudaMemset(p, 1, bytes);
        const uint32_t nlines = (uint32_t)(bytes / 128);
        for (int occ : {4, 5, 8}) {
            for (int K : {2, 4, 8}) {
                const int iters = 4096;
                auto run = [&](int it) {
                    if (K == 2) rd_random_lines<2><<<sms * occ, 256>>>(p, nlines, it, out);
                    else if (K == 4) rd_random_lines<4><<<sms * occ, 256>>>(p, nlines, it, out);
                    else rd_random_lines<8><<<sms * occ, 256>>>(p, nlines, it, out);
                };
                run(16);
                cudaEventRecord(a);
                run(iters);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                const double lines = (double)sms * occ * 256 / 8 * K * iters;
                const double gbs = lines * 128 / ms / 1e6;
                printf("random 128B lines  48 MB  blocks/SM %d  lines in flight/lane %d: %8.1f GB/s\n", occ, K, gbs);
                best_rl = gbs > best_rl ? gbs : best_rl;
            }
        }
        cudaFree(p);
    }
    // 64-byte random segments (4-lane groups): the 512-rule-step shape
    {
        const size_t bytes = (size_t)48 << 20;
        uint4 *p;
        cudaMalloc(&p, bytes);
        cudaMemset(p, 1, bytes);
        const uint32_t nseg = (uint32_t)(bytes / 64);
        for (int occ : {5, 8}) {
            const int iters = 4096;
            rd_random_lines<4, 4><<<sms * occ, 256>>>(p, nseg, 16, out);
            cudaEventRecord(a);
            rd_random_lines<4, 4><<<sms * occ, 256>>>(p, nseg, iters, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            const double segs = (double)sms * occ * 256 / 4 * 4 * iters;
            printf("random 64B segments 48 MB  blocks/SM %d  4 in flight/lane: %8.1f GB/s\n", occ, segs * 64 / ms / 1e6);
        }
        cudaFree(p);
    }
    printf("{\"l2_read_gbs\": %.1f, \"hbm_read_gbs\": %.1f, \"l2_random_line_read_gbs\": %.1f}\n", best_l2,
           best_hbm, best_rl);
    return 0;
}
