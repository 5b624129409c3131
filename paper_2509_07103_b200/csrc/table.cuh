// Device table preparation: relayout from the reference layout, the counter-RNG
// fill and the export back to the reference layout.
#pragma once

#include "device_common.cuh"

namespace lmkan_b200 {

// ------------------------------------------------------- table preparation
// Reference layout src[node][pair][out_total] (layer.hpp:34-45) -> device layout
// dst[ot][pair][node][NS] for the output slice [out_begin, out_begin + n_out_local),
// zero padded to n_ot*OT; NS = OT, or 2 OT for a duplicated-node table (both
// copies of a node's OT outputs written). One thread per destination element
// (coalesced on both sides along the output index).
template <typename T>
__global__ void relayout_kernel(const T* __restrict__ src, float* __restrict__ dst, int pairs, int nodes,
                                int n_out_total, int out_begin, int n_out_local, int OT, int NS, int n_ot) {
    const size_t total = static_cast<size_t>(n_ot) * pairs * nodes * NS;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int qq = static_cast<int>(i % NS) % OT;  // both copies of a duplicated node
        size_t t = i / NS;
        const int node = static_cast<int>(t % nodes);
        t /= nodes;
        const int p = static_cast<int>(t % pairs);
        const int ot = static_cast<int>(t / pairs);
        const int ql = ot * OT + qq;
        float v = 0.f;
        if (ql < n_out_local)
            v = static_cast<float>(src[(static_cast<size_t>(node) * pairs + p) * n_out_total + out_begin + ql]);
        dst[i] = v;
    }
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

// Counter-based N(0,1) for flat reference index f (Box-Muller on one 64-bit hash).
__device__ __forceinline__ float hash_normal(uint64_t seed, uint64_t f) {
    const uint64_t h = splitmix64(seed ^ splitmix64(f));
    const float u1 = (static_cast<float>(h >> 40) + 0.5f) * (1.0f / 16777216.0f);  // (0,1)
    const float u2 = static_cast<float>((h >> 16) & 0xffffffu) * (1.0f / 16777216.0f);
    return sqrtf(-2.0f * logf(u1)) * cospif(2.0f * u2);
}

static __global__ void fill_random_kernel(float* __restrict__ dst, int pairs, int nodes, int n_out_total,
                                   int out_begin, int n_out_local, int OT, int NS, int n_ot, uint64_t seed,
                                   float scale) {
    const size_t total = static_cast<size_t>(n_ot) * pairs * nodes * NS;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int qq = static_cast<int>(i % NS) % OT;  // both copies of a duplicated node
        size_t t = i / NS;
        const int node = static_cast<int>(t % nodes);
        t /= nodes;
        const int p = static_cast<int>(t % pairs);
        const int ot = static_cast<int>(t / pairs);
        const int ql = ot * OT + qq;
        float v = 0.f;
        if (ql < n_out_local) {
            const uint64_t f = (static_cast<uint64_t>(node) * pairs + p) * n_out_total + out_begin + ql;
            v = scale * hash_normal(seed, f);
        }
        dst[i] = v;
    }
}

// Device table -> reference layout (doubles) for pairs [pb, pe), local outputs.
static __global__ void export_kernel(const float* __restrict__ table, double* __restrict__ dst, int pairs, int nodes,
                              int n_out_local, int OT, int NS, int pb, int pe) {
    const int np = pe - pb;
    const size_t total = static_cast<size_t>(nodes) * np * n_out_local;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int q = static_cast<int>(i % n_out_local);
        size_t t = i / n_out_local;
        const int pl = static_cast<int>(t % np);
        const int node = static_cast<int>(t / np);
        const int ot = q / OT, qq = q % OT;
        dst[i] = table[((static_cast<size_t>(ot) * pairs + pb + pl) * nodes + node) * NS + qq];
    }
}

// fp64 results that are exactly fp32 values (the gather accumulates in fp32)
// narrowed for a half-size D2H (host paths with fp64 Y; widened back on the host).
static __global__ void narrow_f64_kernel(const double* __restrict__ src, float* __restrict__ dst, size_t n) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        dst[i] = static_cast<float>(src[i]);
}

}  // namespace lmkan_b200
