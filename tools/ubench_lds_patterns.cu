// Microbenchmark: shared-memory wavefront cost of the LDS patterns the gather
// kernel's per-row loads can take (weights broadcast to a lane group, corner
// runs), and whether SHFL shares the shared-memory data path.
// Prints warp-instructions per clock per SM for each pattern; a pattern costing
// k wavefronts per instruction runs at ~1/k instr/clk.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t lcg(uint32_t& s) {
    s = s * 1664525u + 1013904223u;
    return s;
}

// P: 0 = 2 groups of 16 lanes (16 B each, contiguous), 1 = 4 groups of 8,
//    2 = 8 groups of 4, 3 = 32 distinct float4 (512 B), 4 = all lanes same,
//    5 = LDS.32 32 distinct (128 B), 6 = SHFL only, 7 = pattern 3 + 1 SHFL per LDS,
//    8 = LDS.64 16 groups of 2 (8 B), 9 = 4 groups of 8 but groups 128 B apart (bank conflict check)
template <int P>
__global__ void __launch_bounds__(512, 1) lds_bench(int iters, uint32_t seed, float* out, long long* cyc) {
    extern __shared__ float4 sh[];  // 1024 rows x 32 float4 = 512 KB? no: 256 rows x 32 float4 = 128 KB
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) sh[i] = make_float4(i, 1, 2, 3);
    __syncthreads();
    float acc = 0.f;
    uint32_t row = (seed + warp * 37u) & 255u;
    const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(sh));
    // lane byte offset inside the 512-B row for each pattern
    uint32_t loff = 0;
    if (P == 0) loff = (lane >> 4) * 16;
    if (P == 1) loff = (lane >> 3) * 16;
    if (P == 2) loff = (lane >> 2) * 16;
    if (P == 3 || P == 7) loff = lane * 16;
    if (P == 5) loff = lane * 4;
    if (P == 8) loff = (lane >> 1) * 8;
    if (P == 9) loff = (lane >> 3) * 128;
    if (P == 10 || P == 12) loff = (lane >> 4) * 8;
    if (P == 13) loff = (lane >> 4) * 4;
    const uint32_t lb = base + loff;
    uint32_t sv = lane, accu = 0;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        row = (row + 37u) & 127u;
        const uint32_t a = lb + (row << 9);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            uint32_t x = 0, y = 0, z = 0, w = 0;
            if (P <= 4 || P == 9) {
                asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "r"(a + k * 8192) : "memory");
            } else if (P == 5 || P == 13) {
                asm volatile("ld.shared.b32 %0, [%1];" : "=r"(x) : "r"(a + k * 8192) : "memory");
            } else if (P == 6) {
                asm volatile("shfl.sync.idx.b32 %0, %1, %2, 31, -1;" : "=r"(y) : "r"(sv), "r"((row + k) & 31));
            } else if (P == 7) {
                asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "r"(a + k * 8192) : "memory");
                asm volatile("shfl.sync.idx.b32 %0, %1, %2, 31, -1;" : "=r"(y) : "r"(sv), "r"((row + k) & 31));
            } else if (P == 8 || P == 10 || P == 11) {
                asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=r"(x), "=r"(y) : "r"(a + k * 8192) : "memory");
            }
            accu ^= x ^ y ^ z ^ w;
        }
    }
    acc = __uint_as_float(accu);
    const long long t1 = clock64();
    if (lane == 0 && warp == 0) cyc[blockIdx.x] = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int P>
void run(const char* name, int sms) {
    const int iters = 4096;
    float* out;
    long long* cyc;
    cudaMalloc(&out, sizeof(float) * sms * 512);
    cudaMalloc(&cyc, sizeof(long long) * sms);
    const int smem = 256 * 32 * 16;
    cudaFuncSetAttribute(lds_bench<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    lds_bench<P><<<sms, 512, smem>>>(16, 1, out, cyc);
    lds_bench<P><<<sms, 512, smem>>>(iters, 12345, out, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("%s: error %s\n", name, cudaGetErrorString(e));
        return;
    }
    long long c0;
    cudaMemcpy(&c0, cyc, sizeof(long long), cudaMemcpyDeviceToHost);
    const double instr = 16.0 * iters * 8;  // warp-instructions per SM (16 warps)
    printf("%-52s cycles=%9lld  warp-instr/clk/SM=%6.3f  clk/instr=%5.2f\n", name, c0, instr / c0, c0 / instr);
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    printf("SMs=%d (16 warps/SM, random 512-B row per instruction)\n", sms);
    run<0>("LDS.128 2 groups x16 lanes (32 B unique)", sms);
    run<1>("LDS.128 4 groups x8 lanes (64 B unique)", sms);
    run<2>("LDS.128 8 groups x4 lanes (128 B unique)", sms);
    run<3>("LDS.128 32 distinct (512 B)", sms);
    run<4>("LDS.128 all lanes same (16 B)", sms);
    run<5>("LDS.32 32 distinct (128 B)", sms);
    run<6>("SHFL.IDX only", sms);
    run<7>("LDS.128 32 distinct + 1 SHFL each", sms);
    run<8>("LDS.64 16 groups x2 lanes (128 B unique)", sms);
    run<9>("LDS.128 4 groups x8, groups 128 B apart", sms);
    run<10>("LDS.64 2 groups x16 lanes (16 B unique)", sms);
    run<11>("LDS.64 all lanes same (8 B)", sms);
    run<13>("LDS.32 2 groups x16 lanes (8 B unique)", sms);
    return 0;
}
