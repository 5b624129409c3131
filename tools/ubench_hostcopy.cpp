// Host-side copy costs that bound the pageable drop-in path: memcpy bandwidth
// of 512 MiB with 1..16 threads (pageable -> pinned, pinned -> pageable), and
// the cost of cudaHostRegister / cudaHostUnregister of the same buffer.
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
#include <cuda_runtime.h>

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

static void pcopy(char* d, const char* s, size_t n, int t) {
    std::vector<std::thread> th;
    size_t part = (n + t - 1) / t;
    for (int i = 0; i < t; ++i) th.emplace_back([=] { size_t o = i * part; if (o < n) std::memcpy(d + o, s + o, std::min(part, n - o)); });
    for (auto& x : th) x.join();
}

int main() {
    const size_t n = size_t(512) << 20;
    std::vector<char> a(n, 1), b(n, 2);
    char* pin = nullptr;
    cudaHostAlloc(reinterpret_cast<void**>(&pin), n, cudaHostAllocDefault);
    std::memset(pin, 3, n);
    for (int t : {1, 2, 4, 8, 12, 16}) {
        pcopy(pin, a.data(), n, t);
        double t0 = now();
        for (int r = 0; r < 3; ++r) pcopy(pin, a.data(), n, t);
        double in = 3 * n / (now() - t0) / 1e9;
        t0 = now();
        for (int r = 0; r < 3; ++r) pcopy(b.data(), pin, n, t);
        double out = 3 * n / (now() - t0) / 1e9;
        std::printf("{\"threads\": %d, \"pageable_to_pinned_gbs\": %.1f, \"pinned_to_pageable_gbs\": %.1f}\n", t, in, out);
    }
    for (int r = 0; r < 3; ++r) {
        double t0 = now();
        cudaError_t e = cudaHostRegister(a.data(), n, cudaHostRegisterDefault);
        double t1 = now();
        cudaHostUnregister(a.data());
        double t2 = now();
        std::printf("{\"host_register_ms\": %.2f, \"unregister_ms\": %.2f, \"ok\": %d}\n", 1e3 * (t1 - t0), 1e3 * (t2 - t1), e == cudaSuccess);
    }
    return 0;
}
