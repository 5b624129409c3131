// Microbenchmark for a TMEM-assisted gather: per "row", a warp loads two
// corners from shared memory (LDS.64, 2 outputs per lane, 256 B each) and two
// adjacent corners from tensor memory (tcgen05.ld.32x32b.x4, 4 columns per
// lane = 2 nodes x 2 outputs, 512 B), all at warp-uniform random node indices.
// Reports bytes/clk/SM for: SMEM-only (4 x LDS.64), TMEM-only (2 x .x4), and
// the mix. Also a pure .x4 / .x8 TMEM gather for the ceiling.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t lcg(uint32_t& s) {
    s = s * 1664525u + 1013904223u;
    return s;
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) mix_bench(int iters, uint32_t seed, float* out, long long* cyc) {
    extern __shared__ float2 sh[];  // 512 nodes x 32 lanes x float2 = 128 KB
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 512 * 32; i += blockDim.x) sh[i] = make_float2(i, 1);
    const bool tm = MODE != 0;
    if (tm) {
        if (warp == 0) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                static_cast<uint32_t>(__cvta_generic_to_shared(&tbase))));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
    }
    __syncthreads();
    if (tm) asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = tm ? tbase : 0;
    const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
    float acc = 0.f;
    uint32_t s = seed ^ (warp * 7919u);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        uint32_t r[32];
#pragma unroll
        for (int k = 0; k < 4; ++k) {  // 4 rows per iteration
            const uint32_t n1 = (lcg(s) >> 20) & 255, n2 = (lcg(s) >> 20) & 254;
            if (MODE == 0 || MODE == 2) {  // SMEM: corners (n1, n1+1) and, in mode 0, (n2, n2+1)
                const float2 a = sh[n1 * 32 + lane], b = sh[(n1 + 1) * 32 + lane];
                acc += a.x + a.y + b.x + b.y;
                if (MODE == 0) {
                    const float2 c = sh[n2 * 32 + lane], d = sh[(n2 + 1) * 32 + lane];
                    acc += c.x + c.y + d.x + d.y;
                }
            }
            if (MODE == 1 || MODE == 2) {  // TMEM: 4 columns = nodes (n2, n2+1) x 2 outputs
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(r[4 * k]), "=r"(r[4 * k + 1]), "=r"(r[4 * k + 2]), "=r"(r[4 * k + 3])
                             : "r"(base + lane_base + 2 * n2));
            }
            if (MODE == 1) {
                const uint32_t n3 = (lcg(s) >> 20) & 254;
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(r[16 + 4 * k]), "=r"(r[17 + 4 * k]), "=r"(r[18 + 4 * k]), "=r"(r[19 + 4 * k])
                             : "r"(base + lane_base + 2 * n3));
            }
        }
        if (tm) {
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int k = 0; k < 16; ++k) acc += __uint_as_float(r[k]);
            if (MODE == 1)
#pragma unroll
                for (int k = 16; k < 32; ++k) acc += __uint_as_float(r[k]);
        }
    }
    const long long t1 = clock64();
    if (lane == 0 && warp == 0) cyc[blockIdx.x] = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (tm) {
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
    }
}

template <int MODE>
void run(const char* name, int sms, double bytes_per_row) {
    const int iters = 4096;
    float* out;
    long long* cyc;
    cudaMalloc(&out, sizeof(float) * sms * 512);
    cudaMalloc(&cyc, sizeof(long long) * sms);
    const int smem = 512 * 32 * 8;
    cudaFuncSetAttribute(mix_bench<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    mix_bench<MODE><<<sms, 512, smem>>>(16, 1, out, cyc);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    mix_bench<MODE><<<sms, 512, smem>>>(iters, 12345, out, cyc);
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
    const double rows = 16.0 * iters * 4;  // per SM
    printf("%-34s %8.3f ms  cyc/row/SM=%6.2f  bytes/clk/SM=%7.1f  rows/clk/SM=%.3f\n", name, ms, c0 / rows,
           rows * bytes_per_row / c0, rows / c0);
    cudaFree(out);
    cudaFree(cyc);
}

int main(int argc, char** argv) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int mode = argc > 1 ? atoi(argv[1]) : -1;
    setvbuf(stdout, nullptr, _IONBF, 0);
    printf("SMs=%d (a 'row' = 4 corners x 64 outputs x 4 B = 1024 B)\n", sms);
    if (mode < 0 || mode == 0) run<0>("smem only: 4 x LDS.64", sms, 1024);
    if (mode < 0 || mode == 1) run<1>("tmem only: 2 x ld.32x32b.x4", sms, 1024);
    if (mode < 0 || mode == 2) run<2>("mix: 2 x LDS.64 + 1 x ld.x4", sms, 1024);
    return 0;
}
