// Internal host-side declarations shared by the C-ABI translation unit and the
// per-output-tile gather-launch translation units (compiled in parallel).
#pragma once

#include <cstdint>
#include <string>
#include <cuda_runtime.h>

#include "kernels.cuh"

struct lmkan_b200_layer {
    int device = 0;
    int n_in = 0, n_out = 0, G = 0, pairs = 0, nodes = 0;
    int n_out_total = 0, out_begin = 0;
    double gamma = 0.0;
    int OT = 64, n_ot = 0;
    bool narrow = false;  // n_out <= 4: [pair][node][OT] table, K4 narrow kernel
    bool dup = false;     // OT = 16 duplicated-node table [ot][pair][node][2][OT] (conflict-free gathers)
    int ns = 64;          // node stride of the device table in floats (OT, or 2 OT when dup)
    int pair_block = 0;   // pair-block summation block (0: one running sum; see fwd_fused_kernel)
    int num_sms = 148;    // the device's SM count (queried at creation)
    // reference precision (lmkan_b200_layer_create_exact): fp64 table
    // [out_tile][pair][node][OT] (OT = 32 / 16 / 8 doubles) and the exact kernel
    // (csrc/exact.cu); no fp32 table
    bool exact = false;
    bool exact_gsheet = false;  // sheets read from L2 (too large for shared memory)
    double* table64 = nullptr;
    size_t table64_bytes = 0;
    float* table = nullptr;
    size_t table_bytes = 0;
    double* d_inv = nullptr;  // the grid constants block (GridConst's arrays), inv_areas first
    lmkan_b200::GridConst gc{};
    // bumped by every mutation after creation (set_gamma): captured CUDA graphs
    // of a model bake gamma into their kernel parameters and re-capture on change
    uint64_t version = 0;
};

namespace lmkan_b200 {

struct Plan {
    int OT, RT, nbuf, mode, S;
    ShapeRT sh;
    uint32_t smem;
    int64_t row_tiles, rows_pad;
    int launches;
    int64_t row_tile;  // rows per CTA tile, <= sh.R (smaller to balance the grid over the SMs)
    int goff = 0;      // staged: node offsets read from global into registers (fwd_fused_kernel)
    int pix = 0;       // fused conv: records per image pixel (kModePixel), recO = the pixel records
    int cta_group = 1; // output tiles per CTA-order group (cta_tile in gather.cuh; choose_cta_group)
};

// Launch the gather kernel variant selected by `pl` for output tile OT
// (definitions in launch_gather.cuh, instantiated in gather_ot{16,32,64}.cu and,
// for duplicated-node OT = 16 tables, gather_ot16d.cu).
template <int OT, typename XT, bool DUP = false>
cudaError_t launch_gather(const lmkan_b200_layer* L, const Plan& pl, const XT* X, const OutDests<XT>& Y, int64_t rows,
                          const float2* recW, const int* recO, const InputMap& im, const EmitRecords& emit,
                          const GridConst* gc_next, cudaStream_t st);

// Entry points shared with the other host translation units (model.cu):
// defined in lmkan_b200.cu next to the layer C-ABI.
namespace api {
int set_error(int code, const std::string& msg);  // thread-local lmkan_b200_last_error
int cuda_error(cudaError_t e, const char* what);  // maps a CUDA error to a status code
// Handle + grid constants + (uninitialised) device table for outputs
// [out_begin, out_begin + n_out_local) of an n_out_total-wide layer.
int alloc_layer(int n_in, int n_out_local, int n_out_total, int out_begin, int G, double gamma, int device,
                lmkan_b200_layer** out);
int forward_device(const lmkan_b200_layer* L, const float* X, float* Y, int64_t rows, cudaStream_t st);
// model_infer chain of full layers, fp32, activations through acts[2] except
// where a layer's epilogue emits the next layer's cell records (fused chain).
int forward_chain_f32(const lmkan_b200_layer* const* layers, int n, const float* X, float* Y, int64_t rows,
                      void* const* acts, cudaStream_t st);
int forward_device(const lmkan_b200_layer* L, const double* X, double* Y, int64_t rows, cudaStream_t st);
// reference-precision layers (csrc/exact.cu)
void exact_choose(int n_out, int G, int smem_cap, int& OT, bool& gsheet);
int exact_upload(lmkan_b200_layer* L, const double* P_host);
int exact_read_table(const lmkan_b200_layer* L, int pair_begin, int pair_end, double* dst_host);
int forward_exact(const lmkan_b200_layer* L, const float* X, float* Y, int64_t rows, cudaStream_t st);
int forward_exact(const lmkan_b200_layer* L, const double* X, double* Y, int64_t rows, cudaStream_t st);
}  // namespace api

}  // namespace lmkan_b200
