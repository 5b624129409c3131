// Device-side types and PTX helpers shared by every lmKAN kernel (grid constants,
// input maps, output destinations, mbarrier / bulk-copy / shared-memory wrappers).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace lmkan_b200 {

constexpr int kMaxG = 255;     // largest grid (the packed node offset has 24 bits)
constexpr int kMaxThr = 256;   // threshold slots: L = the power of two >= G, at most 256
constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;

// Grid constants of a layer, resident in device memory (one allocation per
// layer); kernels copy them into shared memory at CTA start.
struct GridConst {
    const float* t32;   // [L] thresholds t_k, NaN-padded to L entries
    const double* t64;  // [L]
    const double* points;     // [G+1]
    const double* inv_h;      // [G] 1 / (points[i+1] - points[i]), the per-axis factors of inv_areas (grid.hpp:58-64)
    const double* inv_areas;  // [G*G]
    int G;
    int L;  // power of two >= G (search width)
};
__host__ __device__ constexpr int grid_L(int G) { return G <= 1 ? 1 : 2 * grid_L((G + 1) / 2); }

// Where the layer input x[r][col] lives: a dense row-major X (row stride n_in),
// or the implicit im2col view of an NHWC image batch that unfold_conv would
// materialize (conv.hpp:39-60): row r = (n, oy, ox) row-major over output
// positions, column col = (dy*k + dx)*C + ch -> img[n][oy*s + dy][ox*s + dx][ch].
// Both are "row base + column offset"; row_offset shifts r for row chunks.
struct InputMap {
    int conv;  // 0: dense X, 1: implicit im2col over an NHWC image batch
    int out_h, out_w, H, W, C, k, s;
    int64_t row_offset;
    int64_t npix;  // conv: pixels of the image batch, N*H*W (pixel-record stride, kModePixel)
};
__host__ __device__ inline int64_t in_rowbase(const InputMap& m, int64_t r, int n_in) {
    r += m.row_offset;
    if (!m.conv) return r * n_in;
    const int64_t per = static_cast<int64_t>(m.out_h) * m.out_w;
    const int64_t n = r / per;
    const int rem = static_cast<int>(r - n * per);
    const int oy = rem / m.out_w, ox = rem - oy * m.out_w;
    return ((n * m.H + static_cast<int64_t>(oy) * m.s) * m.W + static_cast<int64_t>(ox) * m.s) * m.C;
}
__host__ __device__ inline int in_coloff(const InputMap& m, int col) {
    if (!m.conv) return col;
    const int tap = col / m.C, ch = col - tap * m.C;
    const int dy = tap / m.k, dx = tap - dy * m.k;
    return (dy * m.W + dx) * m.C + ch;
}

// Where the layer output y[r][q] (local column q) goes: n row-major buffers
// base[d][r * ld + col0 + q]. The plain forward has one (Y, ld = n_out,
// col0 = 0); an output-sharded layer can write its columns straight into the
// full-width Y of every GPU (peer pointers mapped over NVLink), which fuses the
// all-gather of the shards into the gather kernel's epilogue.
constexpr int kMaxDest = 8;
template <typename XT>
struct OutDests {
    XT* base[kMaxDest];
    int64_t ld;
    int col0;
    int n;
};
template <typename XT>
__host__ __device__ inline OutDests<XT> single_dest(XT* Y, int n_out) {
    OutDests<XT> o{};
    o.base[0] = Y;
    o.ld = n_out;
    o.col0 = 0;
    o.n = 1;
    return o;
}
template <typename XT>
__host__ __device__ inline OutDests<XT> dests_at_row(OutDests<XT> o, int64_t r0) {
    for (int d = 0; d < o.n && d < kMaxDest; ++d) o.base[d] += r0 * o.ld;
    return o;
}

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
// 1-D bulk copy global -> shared, completion counted on `bar` (TMA engine; SASS UBLKCP).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// Predicated 128-bit shared-memory load: zeros (and no shared-memory traffic)
// when !pred. Keeps the slab-mode gather loop branch-free.
__device__ __forceinline__ float4 lds128_if(const void* p, bool pred) {
    float4 v;
    asm volatile(
        "{\n\t.reg .pred q;\n\t"
        "setp.ne.b32 q, %5, 0;\n\t"
        "mov.f32 %0, 0f00000000;\n\tmov.f32 %1, 0f00000000;\n\t"
        "mov.f32 %2, 0f00000000;\n\tmov.f32 %3, 0f00000000;\n\t"
        "@q ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n\t}"
        : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
        : "r"(smem_addr(p)), "r"(static_cast<int>(pred))
        : "memory");
    return v;
}
__device__ __forceinline__ float2 lds64_if(const void* p, bool pred) {
    float2 v;
    asm volatile(
        "{\n\t.reg .pred q;\n\t"
        "setp.ne.b32 q, %3, 0;\n\t"
        "mov.f32 %0, 0f00000000;\n\tmov.f32 %1, 0f00000000;\n\t"
        "@q ld.shared.v2.f32 {%0, %1}, [%2];\n\t}"
        : "=f"(v.x), "=f"(v.y)
        : "r"(smem_addr(p)), "r"(static_cast<int>(pred))
        : "memory");
    return v;
}
// 256-bit read-only global load (sm_100: LDG.E.ENL2.256); p 32-byte aligned.
__device__ __forceinline__ void ldg_v8(const float* p, float (&o)[8]) {
    asm volatile("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=f"(o[0]), "=f"(o[1]), "=f"(o[2]), "=f"(o[3]), "=f"(o[4]), "=f"(o[5]), "=f"(o[6]), "=f"(o[7])
                 : "l"(p));
}
__device__ __forceinline__ unsigned atom_add_acq_rel_cta(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(smem_addr(p)), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "LAB_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra LAB_WAIT_%=;\n\t}" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}

}  // namespace lmkan_b200
