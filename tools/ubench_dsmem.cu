// Microbenchmark: is a gather from a peer CTA's shared memory (DSMEM,
// ld.shared::cluster) served by the peer SM's port without costing the
// requester's? A 2-CTA cluster, every warp doing warp-uniform-row LDS.128
// gathers (512 B per instruction, as in the lmKAN gather kernel):
//   mode 0: all local;  mode 1: all remote (peer CTA's buffer);
//   mode 2: half local, half remote (alternating).
// If remote reads only load the peer's port, mode 2 moves ~2x the bytes of
// mode 0 per SM-clock (each SM's port serves its own local half plus the
// peer's remote half = the same wavefronts, while each SM receives both).
#include <cstdint>
#include <cstdio>
#include <cooperative_groups.h>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(512, 1)
    dsmem_bench(int iters, float* out, long long* cyc) {
    extern __shared__ float4 sh[];  // 256 rows x 32 float4 = 128 KB
    cg::cluster_group cluster = cg::this_cluster();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) sh[i] = make_float4(i, 1, 2, 3);
    cluster.sync();
    const unsigned peer = cluster.block_rank() ^ 1u;
    const float4* remote = cluster.map_shared_rank(sh, peer);
    uint32_t row = (warp * 37u + blockIdx.x * 11u) & 255u;
    float acc = 0.f;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            row = (row + 37u) & 255u;
            const bool rem = MODE == 1 || (MODE == 2 && (k & 1));
            const float4* b = rem ? remote : sh;
            const float4 v = b[row * 32 + lane];
            acc += v.x;
        }
    }
    const long long t1 = clock64();
    cluster.sync();  // the peer's buffer must outlive our reads
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int MODE>
void run(const char* name, int sms) {
    const int iters = 4096;
    float* out;
    long long* cyc;
    const int blocks = (sms / 2) * 2;
    cudaMalloc(&out, sizeof(float) * blocks * 512);
    cudaMalloc(&cyc, sizeof(long long) * blocks);
    const int smem = 256 * 32 * 16;
    cudaFuncSetAttribute(dsmem_bench<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    dsmem_bench<MODE><<<blocks, 512, smem>>>(16, out, cyc);
    dsmem_bench<MODE><<<blocks, 512, smem>>>(iters, out, cyc);
    const cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("%s: %s\n", name, cudaGetErrorString(e));
        return;
    }
    long long c0;
    cudaMemcpy(&c0, cyc, sizeof(long long), cudaMemcpyDeviceToHost);
    const double bytes = 16.0 * iters * 8 * 512;  // per CTA
    printf("%-34s cycles=%9lld  bytes/clk per SM (received)=%6.1f\n", name, c0, bytes / c0);
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<0>("local LDS.128 gathers", sms);
    run<1>("remote (DSMEM) gathers", sms);
    run<2>("half local / half remote", sms);
    return 0;
}
