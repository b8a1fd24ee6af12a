// async_probe.cu -- can per-group asynchronous line fetches beat the
// lockstep walk?  Random 128-byte lines of an L2-resident buffer, 4 per step
// (the match-set scan's four rows), groups of 8 lanes, steps dependent (the
// next step's lines are chosen after the current ones are consumed):
//   lockstep: LDG.128 x 4 per lane, the warp waits for all 16 lines of its
//             4 groups every step (the shipped kernels' shape);
//   bulk:     one lane per group issues 4 cp.async.bulk copies (128 B each)
//             into the group's shared slot, completion on the group's
//             mbarrier; each step the warp polls (try_wait, non-blocking),
//             and only the groups whose lines landed consume and re-issue --
//             groups no longer wait for each other.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/async_probe tools/async_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t pick(uint32_t &x, uint32_t nlines) {
    x = x * 1664525u + 1013904223u;
    return (uint32_t)(((uint64_t)(x >> 8) * nlines) >> 24);
}

__global__ void __launch_bounds__(256) lockstep(const uint4 *__restrict__ p, uint32_t nlines, int steps,
                                                uint32_t *sink) {
    const int lane = threadIdx.x & 31, grp = lane / 8, gl = lane % 8;
    uint32_t x = 0x9E3779B9u * (blockIdx.x * 32u + (threadIdx.x >> 5) * 4u + (uint32_t)grp + 1u);
    uint32_t acc = 0;
    for (int s = 0; s < steps; s++) {
        uint4 v[4];
#pragma unroll
        for (int r = 0; r < 4; r++) v[r] = __ldg(p + (size_t)pick(x, nlines) * 8 + gl);
        const uint32_t a = (v[0].x & v[1].x & v[2].x & v[3].x) | (v[0].w & v[1].w & v[2].w & v[3].w);
        const unsigned b = __ballot_sync(0xFFFFFFFFu, a == 0x12345u);
        acc ^= a ^ b;
        x ^= (acc & 1u);  // the next step depends on this one
    }
    if (acc == 0x7654321u) *sink = acc;
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
                 "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t *bar, unsigned phase) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"((unsigned)__cvta_generic_to_shared(bar)), "r"(phase)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void bulk_g2s(void *sdst, const void *gsrc, unsigned bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (unsigned)__cvta_generic_to_shared(sdst)),
                 "l"(gsrc), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
                 : "memory");
}

template <int BUF>
__global__ void __launch_bounds__(256) bulk(const uint4 *__restrict__ p, uint32_t nlines, int steps,
                                            uint32_t *sink) {
    // per group: BUF slots of 4 lines (512 B each) in flight, one mbarrier per slot
    __shared__ __align__(128) uint4 s_line[8][4][BUF][4][8];
    __shared__ uint64_t s_bar[8][4][BUF];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, grp = lane / 8, gl = lane % 8;
    uint32_t x = 0x9E3779B9u * (blockIdx.x * 32u + (uint32_t)warp * 4u + (uint32_t)grp + 1u);
    if (gl == 0)
        for (int b = 0; b < BUF; b++) mbar_init(&s_bar[warp][grp][b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    auto issue = [&](int b) {
        if (gl == 0) {
            mbar_expect_tx(&s_bar[warp][grp][b], 512);
#pragma unroll
            for (int r = 0; r < 4; r++)
                bulk_g2s(&s_line[warp][grp][b][r][0], p + (size_t)pick(x, nlines) * 8, 128, &s_bar[warp][grp][b]);
        }
    };
    for (int b = 0; b < BUF; b++) issue(b);
    uint32_t phase = 0;  // bit b: parity of slot b
    int done = 0, slot = 0;
    uint32_t acc = 0;
    while (__any_sync(0xFFFFFFFFu, done < steps)) {
        const bool ready = done < steps && mbar_test(&s_bar[warp][grp][slot], (phase >> slot) & 1u);
        uint32_t a = 0;
        if (ready) {
            uint4 v[4];
#pragma unroll
            for (int r = 0; r < 4; r++) v[r] = s_line[warp][grp][slot][r][gl];
            a = (v[0].x & v[1].x & v[2].x & v[3].x) | (v[0].w & v[1].w & v[2].w & v[3].w);
        }
        const unsigned bb = __ballot_sync(0xFFFFFFFFu, ready && a == 0x12345u);
        if (ready) {
            acc ^= a ^ bb;
            x ^= (acc & 1u);
            __syncwarp(0xFFu << (grp * 8));  // the group's lanes have read the slot
            phase ^= 1u << slot;
            done++;
            if (done + BUF - 1 < steps) issue(slot);
            slot = slot + 1 == BUF ? 0 : slot + 1;
        }
    }
    if (acc == 0x7654321u) *sink = acc;
}

int main() {
    uint32_t *sink;
    cudaMalloc(&sink, 4);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t bytes = (size_t)48 << 20;
    uint4 *p;
    cudaMalloc(&p, bytes);
    cudaMemset(p, 0xFF, bytes);
    const uint32_t nlines = (uint32_t)(bytes / 128);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int steps = 2048;
    auto report = [&](const char *name, int occ, auto launch) {
        launch(64);
        cudaEventRecord(a);
        launch(steps);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const cudaError_t e = cudaGetLastError();
        const double lines = (double)sms * occ * 32 * 4 * steps;  // 32 groups per block, 4 lines per step
        printf("%-28s blocks/SM %d: %8.1f GB/s  (%.3f lines/SM-cycle @1.965 GHz) %s\n", name, occ,
               lines * 128 / ms / 1e6, lines / (ms * 1e-3) / sms / 1.965e9, e == cudaSuccess ? "" : cudaGetErrorString(e));
    };
    for (int occ : {4, 5, 6, 8}) {
        report("lockstep LDG x4", occ, [&](int s) { lockstep<<<sms * occ, 256>>>(p, nlines, s, sink); });
        report("bulk, 1 slot per group", occ, [&](int s) { bulk<1><<<sms * occ, 256>>>(p, nlines, s, sink); });
        report("bulk, 2 slots per group", occ, [&](int s) { bulk<2><<<sms * occ, 256>>>(p, nlines, s, sink); });
    }
    return 0;
}
