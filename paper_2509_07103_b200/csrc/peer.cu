// Cross-GPU completion for the fused output all-gather (SURVEY.md §8e, config
// 5): every rank's gather kernel stores its output columns straight into the
// full-width Y of every peer (lmkan_b200_forward_f32_dests with peer pointers
// mapped over NVLink by lmkan_b200_ipc_open_handle). This barrier, enqueued on
// the same stream right after that kernel, makes the gathered Y usable: rank r
// publishes `epoch` into slot r of every rank's flag array (system-scope
// release after a system fence, so its Y stores are visible first) and waits
// until every slot of its own array holds `epoch` (acquire). A bounded spin
// turns a missing peer into an error instead of a hung GPU.
#include <cstdint>
#include <string>

#include "../../include/lmkan_b200.h"
#include "layer_impl.hpp"

using namespace lmkan_b200;

namespace {

__device__ __forceinline__ void st_release_sys(int* p, int v) {
    asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_sys(const int* p) {
    int v;
    asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

struct FlagPtrs {
    int* f[kMaxDest];
};

__global__ void peer_barrier_kernel(const FlagPtrs flags, int world, int rank, int epoch, long long timeout_cycles,
                                    int* status) {
    if (threadIdx.x != 0) return;
    __threadfence_system();  // this rank's earlier peer stores (Y) before the flags
#pragma unroll
    for (int q = 0; q < kMaxDest; ++q)
        if (q < world) st_release_sys(flags.f[q] + rank, epoch);
    const int* mine = flags.f[rank];
    const long long t0 = clock64();
    for (int q = 0; q < world; ++q) {
        while (ld_acquire_sys(mine + q) < epoch) {
            if (clock64() - t0 > timeout_cycles) {
                *status = 1 + q;  // peer q never arrived
                return;
            }
            __nanosleep(256);
        }
    }
}

}  // namespace

extern "C" {

int lmkan_b200_peer_barrier(int* const* flag_arrays, int world, int rank, int epoch, int timeout_ms, int* status_dev,
                            void* stream) {
    if (!flag_arrays || world < 1 || world > kMaxDest || rank < 0 || rank >= world || !status_dev || epoch <= 0)
        return api::set_error(LMKAN_B200_EINVAL, "peer_barrier: bad arguments");
    FlagPtrs fp{};
    for (int q = 0; q < world; ++q) {
        if (!flag_arrays[q]) return api::set_error(LMKAN_B200_EINVAL, "peer_barrier: null flag array");
        fp.f[q] = flag_arrays[q];
    }
    int dev = 0, khz = 1965000;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, dev);
    const long long cycles = static_cast<long long>(timeout_ms > 0 ? timeout_ms : 10000) * (khz > 0 ? khz : 1965000);
    peer_barrier_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(fp, world, rank, epoch, cycles, status_dev);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return api::cuda_error(e, "peer_barrier: launch");
    return LMKAN_B200_OK;
}

int lmkan_b200_device_pci_bus_id(int device, char* buf, int len) {
    if (!buf || len < 13) return api::set_error(LMKAN_B200_EINVAL, "device_pci_bus_id: buffer too small");
    const cudaError_t e = cudaDeviceGetPCIBusId(buf, len, device);
    if (e != cudaSuccess) return api::cuda_error(e, "device_pci_bus_id");
    return LMKAN_B200_OK;
}

int lmkan_b200_peer_access(int device, const char* peer_pci_bus_id) {
    if (!peer_pci_bus_id) return api::set_error(LMKAN_B200_EINVAL, "peer_access: null PCI bus id");
    int peer = -1;
    if (cudaDeviceGetByPCIBusId(&peer, peer_pci_bus_id) != cudaSuccess || peer < 0) {
        cudaGetLastError();
        return api::set_error(LMKAN_B200_EUNSUPPORTED, std::string("peer_access: GPU ") + peer_pci_bus_id +
                                                           " is not visible to this process (CUDA_VISIBLE_DEVICES)");
    }
    if (peer == device) return LMKAN_B200_OK;
    int can = 0;
    cudaError_t e = cudaDeviceCanAccessPeer(&can, device, peer);
    if (e != cudaSuccess) return api::cuda_error(e, "peer_access: cudaDeviceCanAccessPeer");
    if (!can)
        return api::set_error(LMKAN_B200_EUNSUPPORTED, "peer_access: GPU " + std::to_string(device) +
                                                           " cannot access GPU " + std::to_string(peer) +
                                                           " (no NVLink / PCIe peer path): the fused all-gather "
                                                           "needs peer access, use the NCCL gather instead");
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    e = cudaDeviceEnablePeerAccess(peer, 0);
    cudaSetDevice(prev);
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
        e = cudaSuccess;
    }
    if (e != cudaSuccess) return api::cuda_error(e, "peer_access: cudaDeviceEnablePeerAccess");
    return LMKAN_B200_OK;
}

}  // extern "C"
