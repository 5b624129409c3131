// Which slot-release protocols of a bulk-copy ring does compute-sanitizer's
// racecheck accept? A 2-slot ring of 16 KB slots filled by cp.async.bulk
// (mbarrier complete_tx "full" barriers), 8 warps reading every slot, three
// release protocols for the refill (write-after-read) side:
//   0: atomic counter, the last warp out refills (the gather kernel's round-1 scheme)
//   1: per-warp arrivals on an "empty" mbarrier; a dedicated thread (warp 0,
//      lane 0) waits on it and refills (the textbook producer / consumer)
//   2: both: the atomic picks the refilling warp, which waits on the empty
//      mbarrier the warps arrived on before refilling
// nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo tools/ring_racecheck.cu -o tools/ring_racecheck
// compute-sanitizer --tool racecheck tools/ring_racecheck <variant>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "../paper_2509_07103_b200/csrc/device_common.cuh"

using namespace lmkan_b200;

__device__ __forceinline__ void mbar_arrive_release(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

template <int VARIANT>
__global__ void ring_kernel(const float* __restrict__ src, float* out, int units) {
    constexpr int kSlotFloats = 4096, kWarps = 8;
    __shared__ __align__(128) float ring[2][kSlotFloats];
    __shared__ uint64_t full[2], empty[2];
    __shared__ unsigned cnt[2];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < 2; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kWarps);
            cnt[s] = 0;
        }
        fence_barrier_init();
    }
    __syncthreads();
    auto issue = [&](int u) {
        const int s = u & 1;
        mbar_arrive_expect_tx(&full[s], kSlotFloats * 4);
        bulk_g2s(ring[s], src + static_cast<size_t>(u) * kSlotFloats, kSlotFloats * 4, &full[s], 0ull);
    };
    if (tid == 0) {
        issue(0);
        if (units > 1) issue(1);
    }
    float acc = 0.f;
    for (int u = 0; u < units; ++u) {
        const int s = u & 1;
        mbar_wait(&full[s], (u >> 1) & 1);
        for (int k = tid; k < kSlotFloats; k += kWarps * 32) acc += ring[s][k];
        __syncwarp();
        if (VARIANT == 0) {
            if (lane == 0 && atom_add_acq_rel_cta(&cnt[s], 1u) == kWarps - 1) {
                cnt[s] = 0;
                if (u + 2 < units) {
                    fence_proxy_async();
                    issue(u + 2);
                }
            }
        } else if (VARIANT == 1) {
            if (lane == 0) mbar_arrive_release(&empty[s]);
            if (tid == 0 && u + 2 < units) {
                mbar_wait(&empty[s], (u >> 1) & 1);
                fence_proxy_async();
                issue(u + 2);
            }
        } else {
            if (lane == 0) {
                mbar_arrive_release(&empty[s]);
                if (atomicAdd(&cnt[s], 1u) == kWarps - 1) {
                    cnt[s] = 0;
                    if (u + 2 < units) {
                        mbar_wait(&empty[s], (u >> 1) & 1);
                        fence_proxy_async();
                        issue(u + 2);
                    }
                }
            }
        }
    }
    out[blockIdx.x * blockDim.x + tid] = acc;
}

int main(int argc, char** argv) {
    const int variant = argc > 1 ? std::atoi(argv[1]) : 0;
    const int units = 8;
    float *src, *out;
    cudaMalloc(&src, sizeof(float) * 4096 * units);
    cudaMalloc(&out, sizeof(float) * 256 * 4);
    cudaMemset(src, 0, sizeof(float) * 4096 * units);
    if (variant == 0) ring_kernel<0><<<4, 256>>>(src, out, units);
    if (variant == 1) ring_kernel<1><<<4, 256>>>(src, out, units);
    if (variant == 2) ring_kernel<2><<<4, 256>>>(src, out, units);
    const cudaError_t e = cudaDeviceSynchronize();
    std::printf("variant %d: %s\n", variant, cudaGetErrorString(e));
    return e == cudaSuccess ? 0 : 1;
}
