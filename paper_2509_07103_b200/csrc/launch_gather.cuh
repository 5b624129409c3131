// Gather-kernel launch templates (see layer_impl.hpp); included only by the
// gather_ot*.cu translation units, each instantiating one output-tile width.
#pragma once

#include <atomic>

#include "layer_impl.hpp"

namespace lmkan_b200 {

template <int OT, int RT, typename XT, int MODE, bool SLAB, int NW = kWarps, bool TAIL = false, bool DUP = false,
          bool GOFF = false>
cudaError_t launch_fused_t(const lmkan_b200_layer* L, const Plan& pl, const XT* X, const OutDests<XT>& Y, int64_t rows,
                           const float2* recW, const int* recO, const InputMap& im, const EmitRecords& emit,
                           const GridConst* gc_next, cudaStream_t st) {
    auto kern = fwd_fused_kernel<OT, RT, XT, MODE, SLAB, NW, TAIL, DUP, GOFF>;
    static std::atomic<bool> configured[64];  // per device: dynamic-smem opt-in done (idempotent)
    const int dev = L->device & 63;
    if (!configured[dev].load(std::memory_order_acquire)) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
        if (e != cudaSuccess) return e;
        configured[dev].store(true, std::memory_order_release);
    }
    dim3 grid(static_cast<unsigned>(pl.row_tiles), static_cast<unsigned>(L->n_ot));
    kern<<<grid, NW * 32, pl.smem, st>>>(X, Y, rows, L->n_in, L->n_out, L->table, L->pairs, pl.nbuf, pl.S,
                                           static_cast<float>(L->gamma), L->gc, recW, recO, pl.rows_pad, im, emit,
                                           emit.W ? *gc_next : L->gc, static_cast<int>(pl.row_tile),
                                           Y.n > 0 ? L->pair_block : 0, pl.cta_group);
    return cudaGetLastError();
}

template <int OT, typename XT, int MODE, bool SLAB, bool DUP = false>
cudaError_t launch_fused_rt(const lmkan_b200_layer* L, const Plan& pl, const XT* X, const OutDests<XT>& Y, int64_t rows,
                            const float2* recW, const int* recO, const InputMap& im, const EmitRecords& emit,
                           const GridConst* gc_next, cudaStream_t st) {
    // rows per thread: the planner's {16, 8, 4} float4 accumulators per thread / V
    constexpr int V = lane_vectors(OT, DUP ? 2 * OT : 0);
    constexpr int RT0 = 16 / V, RT1 = 8 / V, RT2 = 4 / V;
    if constexpr (MODE == kModeStaged && !SLAB && !DUP) {  // offsets from global: the tallest tile only (planner)
        if (pl.goff) {
            if (pl.row_tile < pl.sh.R)
                return launch_fused_t<OT, RT0, XT, MODE, false, kWarps, true, false, true>(L, pl, X, Y, rows, recW,
                                                                                           recO, im, emit, gc_next, st);
            return launch_fused_t<OT, RT0, XT, MODE, false, kWarps, false, false, true>(L, pl, X, Y, rows, recW, recO,
                                                                                        im, emit, gc_next, st);
        }
    }
    if constexpr (!SLAB) {  // small batches: fewer warps per CTA (RT2) so the grid still spans the GPU
        switch (pl.sh.NW) {
            case 8: return launch_fused_t<OT, RT2, XT, MODE, false, 8, false, DUP>(L, pl, X, Y, rows, recW, recO, im, emit, gc_next, st);
            case 4: return launch_fused_t<OT, RT2, XT, MODE, false, 4, false, DUP>(L, pl, X, Y, rows, recW, recO, im, emit, gc_next, st);
            case 2: return launch_fused_t<OT, RT2, XT, MODE, false, 2, false, DUP>(L, pl, X, Y, rows, recW, recO, im, emit, gc_next, st);
            case 1: return launch_fused_t<OT, RT2, XT, MODE, false, 1, false, DUP>(L, pl, X, Y, rows, recW, recO, im, emit, gc_next, st);
            default: break;
        }
    }
    if constexpr (!SLAB) {  // row tiles shortened to fill whole waves of SMs (planner: RT0 / RT1 only)
        if (pl.row_tile < pl.sh.R) {
            if (pl.RT == RT0)
                return launch_fused_t<OT, RT0, XT, MODE, false, kWarps, true, DUP>(L, pl, X, Y, rows, recW, recO, im, emit,
                                                                              gc_next, st);
            return launch_fused_t<OT, RT1, XT, MODE, false, kWarps, true, DUP>(L, pl, X, Y, rows, recW, recO, im, emit,
                                                                          gc_next, st);
        }
    }
    if (pl.RT == RT0) return launch_fused_t<OT, RT0, XT, MODE, SLAB, kWarps, false, DUP>(L, pl, X, Y, rows, recW, recO, im, emit, gc_next, st);
    if (pl.RT == RT1) return launch_fused_t<OT, RT1, XT, MODE, SLAB, kWarps, false, DUP>(L, pl, X, Y, rows, recW, recO, im, emit, gc_next, st);
    return launch_fused_t<OT, RT2, XT, MODE, SLAB, kWarps, false, DUP>(L, pl, X, Y, rows, recW, recO, im, emit, gc_next, st);
}

template <int OT, typename XT, bool DUP>
cudaError_t launch_gather(const lmkan_b200_layer* L, const Plan& pl, const XT* X, const OutDests<XT>& Y, int64_t rows,
                              const float2* recW, const int* recO, const InputMap& im, const EmitRecords& emit,
                           const GridConst* gc_next, cudaStream_t st) {
    if constexpr (DUP) {  // duplicated-node tables: unslabbed shared-memory sheets only (planner)
        if (pl.mode == kModeGlobal || pl.S > 1) return cudaErrorInvalidConfiguration;
        if (pl.mode == kModeFused && pl.pix)
            return launch_fused_rt<OT, XT, kModePixel, false, true>(L, pl, X, Y, rows, recW, recO, im, emit, gc_next, st);
        return pl.mode == kModeStaged
                   ? launch_fused_rt<OT, XT, kModeStaged, false, true>(L, pl, X, Y, rows, recW, recO, im, emit, gc_next, st)
                   : launch_fused_rt<OT, XT, kModeFused, false, true>(L, pl, X, Y, rows, recW, recO, im, emit, gc_next, st);
    } else {
        if (pl.mode == kModeFused && pl.pix && pl.S == 1)
            return launch_fused_rt<OT, XT, kModePixel, false>(L, pl, X, Y, rows, recW, recO, im, emit, gc_next, st);
        if (pl.mode == kModeGlobal)
            return launch_fused_t<OT, 4 / lane_vectors(OT), XT, kModeGlobal, false>(L, pl, X, Y, rows, recW, recO, im,
                                                                                   emit, gc_next, st);
        if (pl.mode == kModeStaged)
            return pl.S > 1 ? launch_fused_rt<OT, XT, kModeStaged, true>(L, pl, X, Y, rows, recW, recO, im, emit, gc_next, st)
                            : launch_fused_rt<OT, XT, kModeStaged, false>(L, pl, X, Y, rows, recW, recO, im, emit, gc_next, st);
        return pl.S > 1 ? launch_fused_rt<OT, XT, kModeFused, true>(L, pl, X, Y, rows, recW, recO, im, emit, gc_next, st)
                        : launch_fused_rt<OT, XT, kModeFused, false>(L, pl, X, Y, rows, recW, recO, im, emit, gc_next, st);
    }
}

}  // namespace lmkan_b200

#define LMKAN_B200_INSTANTIATE_GATHER(OT, DUP)                                                                   \
    template cudaError_t lmkan_b200::launch_gather<OT, float, DUP>(const lmkan_b200_layer*, const lmkan_b200::Plan&, \
                                                              const float*, const lmkan_b200::OutDests<float>&, \
                                                              int64_t, const float2*,                            \
                                                              const int*, const lmkan_b200::InputMap&,           \
                                                              const lmkan_b200::EmitRecords&,                    \
                                                              const lmkan_b200::GridConst*, cudaStream_t);       \
    template cudaError_t lmkan_b200::launch_gather<OT, double, DUP>(const lmkan_b200_layer*,                          \
                                                               const lmkan_b200::Plan&, const double*,           \
                                                               const lmkan_b200::OutDests<double>&,              \
                                                               int64_t, const float2*, const int*,               \
                                                               const lmkan_b200::InputMap&,                      \
                                                               const lmkan_b200::EmitRecords&,                   \
                                                               const lmkan_b200::GridConst*, cudaStream_t);
