// Host-side copy probes for the e2e path (pageable input staging): memcpy
// bandwidth vs thread count, cudaHostRegister cost, and pageable H2D.
// nvcc -O2 -std=c++17 -o tools/host_probe tools/host_probe.cu -lpthread
#include <cuda_runtime.h>
#include "../paper_1312_4188_b200/csrc/hostpool.h"
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
int main() {
    const size_t n = 872u << 20;  // 64Mi packets x 13 B
    char *a = (char *)malloc(n), *b = (char *)malloc(n);
    memset(a, 1, n);
    memset(b, 2, n);
    char *pin;
    cudaHostAlloc(&pin, n, cudaHostAllocPortable);
    memset(pin, 3, n);
    for (int T : {1, 2, 4, 8, 12, 16}) {
        double best = 0;
        for (int rep = 0; rep < 3; rep++) {
            double t0 = now();
            std::vector<std::thread> th;
            for (int i = 0; i < T; i++) th.emplace_back([&, i] { size_t per = n / T; memcpy(pin + i * per, a + i * per, per); });
            for (auto &t : th) t.join();
            double gbs = n / (now() - t0) / 1e9;
            if (gbs > best) best = gbs;
        }
        printf("memcpy pageable->pinned T=%2d: %.1f GB/s\n", T, best);
    }
    for (int rep = 0; rep < 3; rep++) {
        double t0 = now();
        HostPool::get().copy(pin, a, n);
        double t1 = now();
        for (size_t off = 0; off < n; off += 32u << 20) HostPool::get().copy(pin + off, a + off, std::min<size_t>(32u << 20, n - off));
        double t2 = now();
        printf("HostPool (%d threads) one copy %.1f GB/s, 32 MB copies %.1f GB/s\n", HostPool::get().threads(),
               n / (t1 - t0) / 1e9, n / (t2 - t1) / 1e9);
    }
    void *d;
    cudaMalloc(&d, n);
    for (int rep = 0; rep < 3; rep++) {
        double t0 = now();
        cudaError_t e = cudaHostRegister(b, n, cudaHostRegisterDefault);
        double t1 = now();
        cudaMemcpy(d, b, n, cudaMemcpyHostToDevice);
        double t2 = now();
        cudaHostUnregister(b);
        double t3 = now();
        printf("cudaHostRegister %zu MB: %.1f ms (%s), H2D %.1f GB/s, unregister %.1f ms\n", n >> 20, (t1 - t0) * 1e3,
               cudaGetErrorString(e), n / (t2 - t1) / 1e9, (t3 - t2) * 1e3);
    }
    for (int rep = 0; rep < 2; rep++) {
        double t0 = now();
        cudaMemcpy(d, a, n, cudaMemcpyHostToDevice);
        double t1 = now();
        cudaMemcpy(d, pin, n, cudaMemcpyHostToDevice);
        double t2 = now();
        printf("H2D pageable %.1f GB/s, pinned %.1f GB/s\n", n / (t1 - t0) / 1e9, n / (t2 - t1) / 1e9);
    }
    return 0;
}
