// Internal host-side declarations shared by the C-ABI translation unit and the
// per-output-tile gather-launch translation units (compiled in parallel).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "kernels.cuh"

struct lmkan_b200_layer {
    int device = 0;
    int n_in = 0, n_out = 0, G = 0, pairs = 0, nodes = 0;
    int n_out_total = 0, out_begin = 0;
    double gamma = 0.0;
    int OT = 64, n_ot = 0;
    bool narrow = false;  // n_out <= 4: [pair][node][OT] table, K4 narrow kernel
    float* table = nullptr;
    size_t table_bytes = 0;
    double* d_inv = nullptr;
    lmkan_b200::GridConst gc{};
};

namespace lmkan_b200 {

struct Plan {
    int OT, RT, nbuf, mode, S;
    ShapeRT sh;
    uint32_t smem;
    int64_t row_tiles, rows_pad;
    int launches;
};

// Launch the gather kernel variant selected by `pl` for output tile OT
// (definitions in launch_gather.cuh, instantiated in gather_ot{16,32,64}.cu).
template <int OT, typename XT>
cudaError_t launch_gather(const lmkan_b200_layer* L, const Plan& pl, const XT* X, XT* Y, int64_t rows,
                          const float4* recW, const int* recO, const InputMap& im, cudaStream_t st);

}  // namespace lmkan_b200
