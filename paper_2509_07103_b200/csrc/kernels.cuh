// sm_100a device code for the lmKAN layer forward.
//
// Reference path (paths relative to /root/reference/proj/include/lmkan/):
//   stage 1  row_preambles -> preamble -> interval_index -> sigma
//            (layer.hpp:96-101, grid.hpp:87-101, grid.hpp:72-75, grid.hpp:14-17)
//   stage 2  y[q] += w00 p00[q] + w10 p10[q] + w01 p01[q] + w11 p11[q]; y *= gamma
//            (layer.hpp:116-133)
//
// Kernels:
//   locate_kernel     stage 1 alone -> (i1, i2, 4 fp32 weights) per (row, pair)
//                     (the parity/debug entry point lmkan_b200_locate_*)
//   records_kernel    K1: stage 1 for the staged path -> cell records laid out
//                     pair-major in exactly the order K2's warps consume them
//   fwd_fused_kernel  K2 (MODE staged): gather-accumulate; per pair the CTA's
//                     (G+1)^2 x OT coefficient sheet and its R cell records are
//                     streamed into shared memory by the bulk-copy engine
//                     (cp.async.bulk + mbarrier ring), warps gather float4 runs of
//                     the 4 corner nodes and accumulate R x OT in registers.
//                     K3 (MODE fused): same, cells located in-kernel per warp.
//                     MODE global: fallback reading sheets from L2 (huge G).
//   relayout / fill   one-time table preparation into [out_tile][pair][node][OT].
//
// Layout of the device code:
//   device_common.cuh  grid constants, input maps, output destinations, PTX helpers
//   locate.cuh         cell index / weights / records (stage 1)
//   gather.cuh         K1 records_kernel, K2/K3 fwd_fused_kernel (stage 2)
//   narrow.cuh         K4 narrow_kernel (n_out <= 4)
//   table.cuh          table relayout / random fill / export
#pragma once

#include "device_common.cuh"
#include "locate.cuh"
#include "gather.cuh"
#include "narrow.cuh"
#include "table.cuh"
