// Cell locate (stage 1: grid.hpp:14-101, layer.hpp:96-101): bit-exact cell
// indices from the threshold tables and the bilinear weights / records.
#pragma once

#include "device_common.cuh"

namespace lmkan_b200 {

// ------------------------------------------------------------- cell locate
// interval_index(x) == #{k : x >= t[k]} (thresholds derived from the reference
// function on the host, grid_host.hpp). Branchless binary search over the
// NaN-padded, power-of-two-long table: the predicate x >= t[k] is true on a
// prefix (t ascending) and false on the NaN padding, and false everywhere for
// x = NaN (-> cell 0, as the reference's clamp gives).
template <typename XT>
__device__ __forceinline__ int cell_index(XT x, const XT* thr, int L) {
    int i = 0;
    for (int step = L >> 1; step > 0; step >>= 1)
        if (x >= thr[i + step - 1]) i += step;
    return i;
}

// preamble (grid.hpp:87-101): gaps and weights in fp64 exactly as the
// reference orders them (a*c*inv == (a*c)*inv), then rounded to fp32.
// Returns node = i1*(G+1)+i2 and the weights {w00, w10, w01, w11}.
template <typename XT>
__device__ __forceinline__ void locate_pair(XT x1, XT x2, const XT* thr, const double* pts,
                                            const double* __restrict__ inv_areas, int G, int L,
                                            int& i1, int& i2, float4& w) {
    i1 = cell_index(x1, thr, L);
    i2 = cell_index(x2, thr, L);
    const double d1 = static_cast<double>(x1), d2 = static_cast<double>(x2);
    const double a = __dsub_rn(pts[i1 + 1], d1);
    const double b = __dsub_rn(d1, pts[i1]);
    const double c = __dsub_rn(pts[i2 + 1], d2);
    const double d = __dsub_rn(d2, pts[i2]);
    const double inv = __ldg(inv_areas + i1 * G + i2);
    w.x = __double2float_rn(__dmul_rn(__dmul_rn(a, c), inv));
    w.y = __double2float_rn(__dmul_rn(__dmul_rn(b, c), inv));
    w.z = __double2float_rn(__dmul_rn(__dmul_rn(a, d), inv));
    w.w = __double2float_rn(__dmul_rn(__dmul_rn(b, d), inv));
}

template <typename XT>
__device__ __forceinline__ const XT* thr_of(const GridConst& gc);
template <>
__device__ __forceinline__ const float* thr_of<float>(const GridConst& gc) { return gc.t32; }
template <>
__device__ __forceinline__ const double* thr_of<double>(const GridConst& gc) { return gc.t64; }

// K1: stage 1 alone, one thread per (row, pair), consecutive threads on
// consecutive pairs of a row (coalesced 8/16-byte x-pair loads).
template <typename XT>
__global__ void __launch_bounds__(256) locate_kernel(const XT* __restrict__ X, int64_t rows, int n_in,
                                                     const __grid_constant__ GridConst gc,
                                                     int32_t* __restrict__ o_i1, int32_t* __restrict__ o_i2,
                                                     float4* __restrict__ o_w) {
    __shared__ XT thr[kMaxThr];
    __shared__ double pts[kMaxThr + 1];
    for (int k = threadIdx.x; k < gc.L; k += blockDim.x) thr[k] = thr_of<XT>(gc)[k];
    for (int k = threadIdx.x; k <= gc.G; k += blockDim.x) pts[k] = gc.points[k];
    __syncthreads();
    const int pairs = n_in / 2;
    const int64_t total = rows * pairs;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = k / pairs;
        const int p = static_cast<int>(k - r * pairs);
        const XT* xr = X + r * n_in + 2 * p;
        int i1, i2;
        float4 w;
        locate_pair<XT>(xr[0], xr[1], thr, pts, gc.inv_areas, gc.G, gc.L, i1, i2, w);
        o_i1[k] = i1;
        o_i2[k] = i2;
        o_w[k] = w;
    }
}

// Fast cell index: an fp32 sigma estimate (MUFU exp) is VERIFIED against the
// two thresholds bracketing it (t_k = thr[k-1]; thr[G-1] is the NaN padding, so
// the top cell's upper test !(x >= NaN) always holds). Only if the verification
// fails (NaN input, or an estimate off by a cell: ~1e-6 of N(0,1) draws) does it
// fall back to the exact binary search. The result is therefore always
// #{k : x >= t_k}, i.e. the reference interval_index.
template <typename XT>
__device__ __forceinline__ int cell_index_fast(XT x, const XT* thr, int G, int L) {
    const float xf = static_cast<float>(x);
    // e = exp(-|x|) as one MUFU.EX2 (ftz: no range fix-up; the estimate is
    // verified against the exact thresholds below, so its accuracy only decides
    // how often the fallback search runs)
    float e;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(fabsf(xf) * -1.4426950408889634f));
    const float s = xf > 0.f ? 1.f - 0.5f * e : 0.5f * e;
    int i = static_cast<int>(s * static_cast<float>(G));
    i = i < 0 ? 0 : (i > G - 1 ? G - 1 : i);
    const XT lo = thr[i > 0 ? i - 1 : 0];
    const XT hi = thr[i];
    const bool ok = (i == 0 || x >= lo) && !(x >= hi) && x == x;
    return ok ? i : cell_index<XT>(x, thr, L);
}
// Slab split of a sheet along i1: slab s holds the node rows
// i1 in [s*H, min(G, s*H + H)], so every cell with i1 in [s*H, s*H + H) has all
// four corners inside slab s, and a slab is a contiguous byte range of the
// [node][OT] sheet. S = 1 (H = G) is the unsplit sheet. Large-G sheets are cut
// into slabs so that two of them fit in shared memory (double buffering).
__host__ __device__ inline int slab_node_rows(int G, int H, int s) {
    const int r = G + 1 - s * H;
    return r < H + 1 ? r : H + 1;
}

// Packed record offset: (slab << 24) | (node-within-slab * OT).
constexpr int kSlabShift = 24;
constexpr int kOffMask = (1 << kSlabShift) - 1;

// preamble (grid.hpp:87-101) in normalized cell coordinates, from grid
// constants held in shared memory: the cell index (bit-exact, thresholds) and
// ag = {alpha, gamma} = {a / h1, c / h2} (gaps and inverse widths in fp64,
// rounded to fp32). The reference weights are the bilinear products
// w00 = a c inv = alpha gamma, w10 = (1 - alpha) gamma, w01 = alpha (1 - gamma),
// w11 = (1 - alpha)(1 - gamma), since inv_areas = 1 / (h1 h2) (grid.hpp:58-64)
// and a + b = h1, c + d = h2 (weights_ag). Two floats per record instead of
// four: one 1-wavefront LDS.64 per row in the gather loop. Returns the packed
// slab / node offset.
//
// hsub >= 0 (bank-half-swapped plain OT = 16 sheets, see fwd_fused_kernel):
// the row is gathered by a lane group of parity hsub; node n's 64-B run sits on
// bank half n & 1 (sheet slots are 128-B aligned), so the packed offset names
// the member of {n, n+1} on the lane group's own half, n + sw, with
// sw = (n & 1) != hsub flagged in bit kSwapBit (unslabbed sheets only).
constexpr int kSwapBit = 30;
template <typename XT>
__device__ __forceinline__ int locate_ag(XT x1, XT x2, const XT* thr, const double* pts, const double* invh, int G,
                                         int L, int OT, int H, float2& ag, int hsub = -1) {
    const int i1 = cell_index_fast<XT>(x1, thr, G, L);
    const int i2 = cell_index_fast<XT>(x2, thr, G, L);
    ag.x = __double2float_rn(__dmul_rn(__dsub_rn(pts[i1 + 1], static_cast<double>(x1)), invh[i1]));
    ag.y = __double2float_rn(__dmul_rn(__dsub_rn(pts[i2 + 1], static_cast<double>(x2)), invh[i2]));
    if (hsub >= 0) {
        const int n = i1 * (G + 1) + i2, sw = (n & 1) != hsub;
        return (sw << kSwapBit) | ((n + sw) * OT);
    }
    if (H >= G) return (i1 * (G + 1) + i2) * OT;  // unslabbed sheet (the common case)
    const int s = (i1 >= H) + (i1 >= 2 * H) + (i1 >= 3 * H);  // slab (S <= 4), no integer division
    return (s << kSlabShift) | (((i1 - s * H) * (G + 1) + i2) * OT);
}

// The four bilinear weights {w00, w10, w01, w11} of a record (see locate_ag).
// For in-cell inputs they are the reference weights to ~1 fp32 ulp; on the
// unbounded edge cells (alpha or gamma outside [0, 1]) they extrapolate
// exactly like the reference's (grid.hpp:79-81) and still sum to 1.
__device__ __forceinline__ float4 weights_ag(float2 ag) {
    const float b = 1.f - ag.x, d = 1.f - ag.y;
    return make_float4(ag.x * ag.y, b * ag.y, ag.x * d, b * d);
}

// acc += ((w00 p00 + w10 p10) + w01 p01) + w11 p11 per output, fused
// multiply-adds in the reference's per-pair grouping (layer.hpp:129).
// PACKED: two outputs per instruction on the packed fp32x2 pipe (FMUL2 /
// FFMA2 / FADD2, sm_100). Every lane of a packed op is the same IEEE
// round-to-nearest operation, so the results are bit-identical to the scalar
// form at half the FP instruction count. It pays only where issue slots bind:
// the bank-half-swapped OT = 16 gather (config 5 shard 744 -> 698 ms); on the
// latency-bound gathers it measured slower (config 3 chain 5.86 -> 6.08 ms,
// config 2 +0.5%), so they keep the scalar form.
template <bool PACKED = false>
__device__ __forceinline__ float4 corner_term(const float4 w, const float4 p00, const float4 p10, const float4 p01,
                                              const float4 p11) {
#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 1000
    if constexpr (PACKED) {
        const float2 w0 = make_float2(w.x, w.x), w1 = make_float2(w.y, w.y), w2 = make_float2(w.z, w.z),
                     w3 = make_float2(w.w, w.w);
        const float2 lo = __ffma2_rn(w3, make_float2(p11.x, p11.y),
                                     __ffma2_rn(w2, make_float2(p01.x, p01.y),
                                                __ffma2_rn(w1, make_float2(p10.x, p10.y),
                                                           __fmul2_rn(w0, make_float2(p00.x, p00.y)))));
        const float2 hi = __ffma2_rn(w3, make_float2(p11.z, p11.w),
                                     __ffma2_rn(w2, make_float2(p01.z, p01.w),
                                                __ffma2_rn(w1, make_float2(p10.z, p10.w),
                                                           __fmul2_rn(w0, make_float2(p00.z, p00.w)))));
        return make_float4(lo.x, lo.y, hi.x, hi.y);
    }
#endif
    return make_float4(fmaf(w.w, p11.x, fmaf(w.z, p01.x, fmaf(w.y, p10.x, w.x * p00.x))),
                       fmaf(w.w, p11.y, fmaf(w.z, p01.y, fmaf(w.y, p10.y, w.x * p00.y))),
                       fmaf(w.w, p11.z, fmaf(w.z, p01.z, fmaf(w.y, p10.z, w.x * p00.z))),
                       fmaf(w.w, p11.w, fmaf(w.z, p01.w, fmaf(w.y, p10.w, w.x * p00.w))));
}
template <bool PACKED = false>
__device__ __forceinline__ void acc_add(float4& acc, const float4 t) {
#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 1000
    if constexpr (PACKED) {
        const float2 a = __fadd2_rn(make_float2(acc.x, acc.y), make_float2(t.x, t.y));
        const float2 b = __fadd2_rn(make_float2(acc.z, acc.w), make_float2(t.z, t.w));
        acc = make_float4(a.x, a.y, b.x, b.y);
        return;
    }
#endif
    acc.x += t.x;
    acc.y += t.y;
    acc.z += t.z;
    acc.w += t.w;
}
template <bool PACKED = false>
__device__ __forceinline__ void fma_corners(float4& acc, const float4 w, const float4 p00, const float4 p10,
                                            const float4 p01, const float4 p11) {
    acc_add<PACKED>(acc, corner_term<PACKED>(w, p00, p10, p01, p11));
}

}  // namespace lmkan_b200
