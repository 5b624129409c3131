// K4 narrow_kernel: layers with n_out <= 4 (the methane head), whole table in
// shared memory.
#pragma once

#include "locate.cuh"

namespace lmkan_b200 {

// K4: narrow layers (n_out <= 4, e.g. the methane net's 128 -> 1 head). A
// padded 16-wide output tile would waste >= 3/4 of every gather, so instead the
// whole table, laid out [pair][node][NO] (NO = n_out rounded up to 1, 2 or 4),
// is made resident in shared memory once per CTA (bulk copy) and every lane
// owns one row: it walks the pairs in order (x loaded 4 pairs = one 32-byte
// sector at a time), locates and gathers its 4 corners per output. The
// per-(row, output) arithmetic is exactly the general kernel's (same FMA
// grouping, same pair order), so results are bitwise identical to it.
constexpr int kNarrowThreads = 1024;
__host__ __device__ inline uint32_t narrow_smem_bytes(int G, int pairs, int NO) {
    const uint32_t tab = static_cast<uint32_t>((G + 1) * (G + 1)) * pairs * NO * 4u;
    uint32_t o = (tab + 15u) & ~15u;
    o += static_cast<uint32_t>(grid_L(G)) * 8u + static_cast<uint32_t>(G + 1) * 8u + static_cast<uint32_t>(G) * 8u + 16u;
    return (o + 127u) & ~127u;
}

template <typename XT, int NO>
__global__ void __launch_bounds__(kNarrowThreads, 1)
    narrow_kernel(const XT* __restrict__ X, const OutDests<XT> out, int64_t rows, int n_in, int n_out,
                  const float* __restrict__ table, float gamma, const __grid_constant__ GridConst gc,
                  const InputMap im, int pair_block) {
    extern __shared__ __align__(1024) unsigned char smem[];
    const int G = gc.G, pairs = n_in / 2, nodes = (G + 1) * (G + 1);
    // bulk copies move multiples of 16 B: the copy includes the table
    // allocation's zeroed tail (alloc_layer rounds it up to 16 B)
    const uint32_t tab_bytes = (static_cast<uint32_t>(nodes) * pairs * NO * 4u + 15u) & ~15u;
    float* tab = reinterpret_cast<float*>(smem);
    uint32_t o = tab_bytes;
    XT* thr = reinterpret_cast<XT*>(smem + o);
    o += static_cast<uint32_t>(gc.L) * 8u;
    double* pts = reinterpret_cast<double*>(smem + o);
    o += static_cast<uint32_t>(G + 1) * 8u;
    double* inv = reinterpret_cast<double*>(smem + o);
    o += static_cast<uint32_t>(G) * 8u;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + ((o + 7u) & ~7u));
    const int tid = threadIdx.x;
    for (int k = tid; k < gc.L; k += kNarrowThreads) thr[k] = thr_of<XT>(gc)[k];
    for (int k = tid; k <= G; k += kNarrowThreads) pts[k] = gc.points[k];
    for (int k = tid; k < G; k += kNarrowThreads) inv[k] = gc.inv_h[k];
    if (tid == 0) {
        mbar_init(bar, 1);
        fence_barrier_init();
        mbar_arrive_expect_tx(bar, tab_bytes);
        const uint64_t pol = policy_evict_last();
        constexpr uint32_t kChunk = 32768;
        for (uint32_t c = 0; c < tab_bytes; c += kChunk)
            bulk_g2s(smem + c, reinterpret_cast<const char*>(table) + c, tab_bytes - c < kChunk ? tab_bytes - c : kChunk,
                     bar, pol);
    }
    __syncthreads();
    mbar_wait(bar, 0);
    const int rs1 = (G + 1) * NO;
    const bool vec4 = sizeof(XT) == 4 && !im.conv && (n_in & 7) == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0;
    // 256-bit loads (LDG.E.ENL2.256): a lane's 4 pairs in one instruction. The
    // lanes of a warp read 32 different rows, so every load instruction costs a
    // wavefront per row; one 32-B load instead of two 16-B ones halves them
    // (the kernel is L1-bound on these uncoalesced row reads).
    const bool vec8 = vec4 && (reinterpret_cast<uintptr_t>(X) & 31) == 0;
    for (int64_t r = static_cast<int64_t>(blockIdx.x) * kNarrowThreads + tid; r < rows;
         r += static_cast<int64_t>(gridDim.x) * kNarrowThreads) {
        float acc[NO], run[NO];  // run: pair-block running sum (fwd_fused_kernel's fold_main, in registers)
#pragma unroll
        for (int q = 0; q < NO; ++q) acc[q] = run[q] = 0.f;
        const XT* xr = X + in_rowbase(im, r, n_in);
        auto one_pair = [&](int p, XT x1, XT x2) {
            if (pair_block > 0 && p > 0 && p % pair_block == 0) {
#pragma unroll
                for (int q = 0; q < NO; ++q) {
                    run[q] = run[q] + acc[q];
                    acc[q] = 0.f;
                }
            }
            float2 ag;
            const int off = locate_ag<XT>(x1, x2, thr, pts, inv, G, gc.L, NO, G, ag);
            const float4 w = weights_ag(ag);
            const float* b = tab + static_cast<size_t>(p) * nodes * NO + off;
#pragma unroll
            for (int q = 0; q < NO; ++q)
                acc[q] += fmaf(w.w, b[rs1 + NO + q], fmaf(w.z, b[NO + q], fmaf(w.y, b[rs1 + q], w.x * b[q])));
        };
        int p = 0;
        if (vec8) {
            for (; p + 4 <= pairs; p += 4) {  // one 32-byte sector of the row = 4 pairs, one load
                float u[8];
                ldg_v8(reinterpret_cast<const float*>(xr) + 2 * p, u);
                one_pair(p, u[0], u[1]);
                one_pair(p + 1, u[2], u[3]);
                one_pair(p + 2, u[4], u[5]);
                one_pair(p + 3, u[6], u[7]);
            }
        } else if (vec4) {
            for (; p + 4 <= pairs; p += 4) {  // one 32-byte sector of the row = 4 pairs
                const float4 u = __ldg(reinterpret_cast<const float4*>(xr + 2 * p));
                const float4 v = __ldg(reinterpret_cast<const float4*>(xr + 2 * p + 4));
                one_pair(p, u.x, u.y);
                one_pair(p + 1, u.z, u.w);
                one_pair(p + 2, v.x, v.y);
                one_pair(p + 3, v.z, v.w);
            }
        }
        for (; p < pairs; ++p) one_pair(p, xr[in_coloff(im, 2 * p)], xr[in_coloff(im, 2 * p + 1)]);
        if (pair_block > 0 && pairs > pair_block) {
#pragma unroll
            for (int q = 0; q < NO; ++q) acc[q] = run[q] + acc[q];
        }
#pragma unroll
        for (int d = 0; d < kMaxDest; ++d) {
            if (d >= out.n) break;
            XT* yr = out.base[d] + out.col0 + r * out.ld;
#pragma unroll
            for (int q = 0; q < NO; ++q)
                if (q < n_out) yr[q] = static_cast<XT>(acc[q] * gamma);
        }
    }
}

}  // namespace lmkan_b200
