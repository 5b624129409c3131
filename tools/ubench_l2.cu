// Microbenchmark: L2 read bandwidth of this B200 (the "builder-measured L2
// peak" SURVEY.md §8d asks the roofline to be reported against). Every SM
// streams 16-byte loads over a buffer that fits in L2 (32 MB of the 126 MB),
// repeatedly; one warm-up pass pulls it into L2. Also reports the HBM read
// bandwidth of a 4 GB buffer for comparison. Prints GB/s.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(1024) read_kernel(const float4* __restrict__ p, size_t n, int reps, float* out) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
             i += static_cast<size_t>(gridDim.x) * blockDim.x) {
            const float4 v = __ldcg(p + i);  // cache at L2 only (skip L1)
            acc.x += v.x;
            acc.y += v.y;
            acc.z += v.z;
            acc.w += v.w;
        }
    if (acc.x + acc.y + acc.z + acc.w == 1234.5f) out[threadIdx.x] = acc.x;
}

static double run(size_t bytes, int reps, int sms) {
    float4* p;
    float* out;
    cudaMalloc(&p, bytes);
    cudaMalloc(&out, 4096);
    cudaMemset(p, 0, bytes);
    const size_t n = bytes / sizeof(float4);
    read_kernel<<<sms * 2, 1024>>>(p, n, 1, out);  // warm (pulls an L2-sized buffer into L2)
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    read_kernel<<<sms * 2, 1024>>>(p, n, reps, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaFree(p);
    cudaFree(out);
    return static_cast<double>(bytes) * reps / (ms * 1e-3) / 1e9;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double best_l2 = 0, best_hbm = 0;
    for (int t = 0; t < 5; ++t) {
        const double l2 = run(size_t(32) << 20, 50, sms);
        const double hbm = run(size_t(4) << 30, 2, sms);
        best_l2 = l2 > best_l2 ? l2 : best_l2;
        best_hbm = hbm > best_hbm ? hbm : best_hbm;
    }
    printf("{\"l2_read_gbs\": %.1f, \"hbm_read_gbs\": %.1f, \"sms\": %d, \"how\": \"ld.global.cg float4 streams, 32 MB (L2-resident, 50 passes) and 4 GB (HBM) buffers, best of 5\"}\n",
           best_l2, best_hbm, sms);
    return 0;
}
