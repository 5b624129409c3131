// Microbenchmark: on-chip gather bandwidth per SM for the lmKAN access pattern
// (a warp-uniform, data-dependent node index; lanes read consecutive outputs).
//   mode 0: shared memory, LDS.128 (one 512-B row per warp per load)
//   mode 1: tensor memory, tcgen05.ld.32x32b.x2 (lane = output, column = node)
//   mode 2: both at once (do the two datapaths add?)
//   mode 3: FFMA-only control loop (issue ceiling)
// Prints bytes/clk/SM and the implied FMA/clk/SM for 4-byte coefficients.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t lcg(uint32_t& s) {
    s = s * 1664525u + 1013904223u;
    return s;
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) gather_bench(int iters, uint32_t seed, float* out, long long* cyc) {
    extern __shared__ float4 sh[];  // 256 rows x 32 float4 = 128 KB
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) sh[i] = make_float4(i, 1, 2, 3);
    if (MODE == 1 || MODE == 2) {
        if (warp == 0) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                static_cast<uint32_t>(__cvta_generic_to_shared(&tbase))));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
    }
    __syncthreads();
    if (MODE == 1 || MODE == 2) asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = (MODE == 1 || MODE == 2) ? tbase : 0;
    const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
    float acc = 0.f;
    uint32_t s = seed ^ (warp * 7919u);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0 || MODE == 2) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint32_t row = (lcg(s) >> 20) & 255;
                const float4 v = sh[row * 32 + lane];
                acc += v.x + v.y + v.z + v.w;
            }
        }
        if (MODE == 1 || MODE == 2) {
            uint32_t r[16];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint32_t col = (lcg(s) >> 20) & 255;
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];"
                             : "=r"(r[2 * k]), "=r"(r[2 * k + 1])
                             : "r"(base + lane_base + col));
            }
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int k = 0; k < 16; ++k) acc += __uint_as_float(r[k]);
        }
        if (MODE == 3) {
#pragma unroll
            for (int k = 0; k < 32; ++k) acc = fmaf(acc, 1.0001f, 0.5f);
        }
    }
    const long long t1 = clock64();
    if (lane == 0 && warp == 0) cyc[blockIdx.x] = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (MODE == 1 || MODE == 2) {
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
    }
}

template <int MODE>
void run(const char* name, int sms) {
    const int iters = 4096;
    float* out;
    long long* cyc;
    cudaMalloc(&out, sizeof(float) * sms * 512);
    cudaMalloc(&cyc, sizeof(long long) * sms);
    const int smem = 256 * 32 * 16;
    cudaFuncSetAttribute(gather_bench<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    gather_bench<MODE><<<sms, 512, smem>>>(16, 1, out, cyc);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    gather_bench<MODE><<<sms, 512, smem>>>(iters, 12345, out, cyc);
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    if (e != cudaSuccess) {
        printf("%s: error %s\n", name, cudaGetErrorString(e));
        return;
    }
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    long long c0;
    cudaMemcpy(&c0, cyc, sizeof(long long), cudaMemcpyDeviceToHost);
    double bytes_per_sm = 0;
    if (MODE == 0) bytes_per_sm = 16.0 * iters * 8 * 512;
    if (MODE == 1) bytes_per_sm = 16.0 * iters * 8 * 256;
    if (MODE == 2) bytes_per_sm = 16.0 * iters * 8 * (512 + 256);
    double fma_per_sm = MODE == 3 ? 16.0 * iters * 32 * 32 : bytes_per_sm / 4;
    printf("%-28s %8.3f ms  cycles=%lld  bytes/clk/SM=%7.1f  FMA-equiv/clk/SM=%7.1f  chip %.1f TB/s\n", name, ms,
           c0, bytes_per_sm / c0, fma_per_sm / c0, bytes_per_sm * sms / (ms * 1e-3) / 1e12);
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    printf("SMs=%d\n", sms);
    run<0>("smem LDS.128 row gather", sms);
    run<1>("tmem ld.32x32b.x2 gather", sms);
    run<2>("smem + tmem together", sms);
    run<3>("ffma issue control", sms);
    return 0;
}
