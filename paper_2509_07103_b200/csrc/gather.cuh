// Gather-accumulate (stage 2: layer.hpp:116-133): K1 records_kernel and the
// K2 / K3 fwd_fused_kernel with its plan shapes and shared-memory layout.
#pragma once

#include "locate.cuh"

namespace lmkan_b200 {

// Kernel variants of the layer forward.
enum : int {
    kModeFused = 0,   // K3: cells located in-kernel (warp-local), sheets via bulk copy
    kModeStaged = 1,  // K2: cell records produced by K1 (records_kernel), sheets + records via bulk copy
    kModeGlobal = 2,  // fallback for sheets larger than shared memory: in-kernel locate, sheets read from L2
    kModeNarrow = 3,  // K4: n_out <= 4, whole table resident in shared memory, lanes over pairs
    kModePixel = 4,   // K3 for the implicit-im2col conv: records located once per image pixel
                      // (pixel_records_kernel) and fetched per (row, pair) through the im2col map
};

// Float4 runs of outputs per lane. At OT = 64 a lane covers 16 outputs (four
// float4 runs OT/4 apart), so one warp instruction serves 8 rows instead of 2:
// each per-row {alpha, gamma} and node-offset load feeds 4x the FMAs, and the
// bank-half interleave in fwd_fused_kernel keeps each instruction at 4
// wavefronts. Rows per thread shrink by V to keep the register tile (RT x V
// float4 accumulators) and the rows per CTA unchanged. Same-box A/B at cfg2
// (K2 ms): V = 1 18.12, V = 2 17.35, V = 4 17.00. LMKAN_B200_VEC64 = 1 / 2
// selects the others (A/B builds).
// At OT = 32 likewise two runs (8 rows per instruction); OT = 16 keeps one
// run per lane and gets its conflict-free loads from duplicated nodes (DUP).
#ifndef LMKAN_B200_VEC64
#define LMKAN_B200_VEC64 4
#endif
#ifndef LMKAN_B200_VEC32
#define LMKAN_B200_VEC32 2
#endif
// OT = 16 with a duplicated-node table (NS = 2 OT): two 32-B runs per lane,
// 16 rows per instruction (see fwd_fused_kernel's bank mapping); plain OT = 16
// keeps one run (its bank-half swap needs whole 64-B runs).
#ifndef LMKAN_B200_VEC16D
#define LMKAN_B200_VEC16D 2
#endif
__host__ __device__ constexpr int lane_vectors(int OT, int NS = 0) {
    return OT >= 64 ? LMKAN_B200_VEC64 : (OT == 32 ? LMKAN_B200_VEC32 : (NS == 2 * OT ? LMKAN_B200_VEC16D : 1));
}

// Row <-> thread mapping shared by K1 (which writes records in K2's order) and K2.
template <int OT, int RT, int NW = kWarps, bool DUP = false>
struct FusedShape {
    static constexpr int V = lane_vectors(OT, DUP ? 2 * OT : 0);  // float4 runs per lane
    static constexpr int LPR = OT / (4 * V);         // lanes covering one row's OT outputs
    static constexpr int RPW = 32 / LPR;             // rows per warp per gather instruction
    static constexpr int ROWS_W = RPW * RT;          // rows owned by one warp
    static constexpr int LOC = (ROWS_W + 31) / 32;   // cells each lane locates per pair (fused mode)
    static constexpr int R = NW * ROWS_W;             // rows per CTA
    static constexpr int OSTRIDE = RT + (RPW > 2 ? 4 : 0);  // padded per-lane-group offset run (bank spread)
    static constexpr int OBLK = NW * RPW * OSTRIDE;         // offset ints per CTA per pair
};
// Runtime twin of FusedShape for host code / K1. NS = the table's node stride
// in floats: OT, or 2 OT for a duplicated-node (DUP) table (see fwd_fused_kernel).
struct ShapeRT {
    int OT, RT, LPR, RPW, ROWS_W, R, OSTRIDE, OBLK, NW, NS;
    int lgRPW, lgROWS_W, lgR;  // RPW, ROWS_W, R are powers of two (OT, RT, NW are)
};
__host__ __device__ constexpr int ilog2(int v) { return v > 1 ? 1 + ilog2(v >> 1) : 0; }
__host__ __device__ inline ShapeRT shape_rt(int OT, int RT, int NW = kWarps, int NS = 0) {
    ShapeRT s;
    s.OT = OT;
    s.NS = NS > 0 ? NS : OT;
    s.RT = RT;
    s.NW = NW;
    s.LPR = OT / (4 * lane_vectors(OT, s.NS));
    s.RPW = 32 / s.LPR;
    s.ROWS_W = s.RPW * RT;
    s.R = NW * s.ROWS_W;
    s.OSTRIDE = RT + (s.RPW > 2 ? 4 : 0);
    s.OBLK = NW * s.RPW * s.OSTRIDE;
    s.lgRPW = ilog2(s.RPW);
    s.lgROWS_W = ilog2(s.ROWS_W);
    s.lgR = ilog2(s.R);
    return s;
}
// Position of CTA-local row qc's node offset inside the CTA's offset block: the
// RT rows a lane group gathers are contiguous, so a thread loads them as int4s.
__host__ __device__ inline int offset_slot(const ShapeRT& s, int qc) {
    const int warp = qc >> s.lgROWS_W, q = qc & (s.ROWS_W - 1);
    const int sub = q & (s.RPW - 1), j = q >> s.lgRPW;
    return (warp * s.RPW + sub) * s.OSTRIDE + j;
}

// Fused chain (model_infer of a fused model, model.hpp:268-315): the NEXT
// layer's cell records written by this layer's epilogue. Its 4 consecutive
// outputs per lane are two input pairs of the next layer, located right there
// (next layer's grid, gc_next) and stored in the next layer's K2 order, so
// the activation never round-trips through HBM and the next K1 is skipped.
// Shared memory the emitting epilogue needs (one pass: OT/4 pairs x R rows).
// + the next layer's grid constants (thresholds, points, inverse widths), so the
// locates read shared memory instead of divergent parameter-space loads.
__host__ __device__ inline uint32_t emit_smem_bytes(int OT, int R) {
    return static_cast<uint32_t>(OT / 4) * R * 12u + kMaxThr * 4u + (kMaxThr + 1) * 8u + kMaxThr * 8u + 16u;
}
struct EmitRecords {
    float2* W;  // [pairs'][rows_pad'] {alpha, gamma}; nullptr: no emission
    int* O;     // [pairs'][tiles'][OBLK'] packed offsets
    ShapeRT sh;  // next layer's K2 row shape
    int64_t rows_pad, tiles;
    int H;  // next layer's slab height
};

// Record-ring depth of the staged mode: records of pair p arrive with its first
// slab and must outlive its S slabs while up to NBUF units are in flight.
__host__ __device__ inline int staged_nrec(int nbuf, int S) { return (nbuf - 1 + S - 1) / S + 1; }

// Shared-memory carve-up (host and device agree on it).
//   sheets : NBUF x slab buffers of (H+1)(G+1) x OT fp32 (bulk-copy destinations)
//   records: NREC x {R float2 {alpha, gamma}, OBLK packed offsets}; NREC = staged_nrec
//            when staged (they arrive with a pair's first slab), else 1
//            (warp-private, written by the in-kernel locate)
//   grid constants (not staged): thresholds, points[G+1], inv_h[G] (fp64)
//   NBUF "landed" mbarriers + NBUF finished-warp counters
struct FusedSmem {
    uint32_t sheet_bytes, recw_bytes, reco_bytes, off_recw, off_reco, off_thr, off_pts, off_inv, off_bar,
        off_cnt, total;
    int nrec;
};
__host__ __device__ inline FusedSmem fused_smem_layout(int G, int OT, int RT, int nbuf, int mode, int S = 1,
                                                       int NW = kWarps, int NS = 0, int goff = 0) {
    const ShapeRT sh = shape_rt(OT, RT, NW, NS);
    const int H = (G + S - 1) / S;
    const int nb = nbuf > 0 ? nbuf : 1;
    FusedSmem s;
    s.nrec = mode == kModeStaged ? staged_nrec(nb, S) : 1;
    // slot stride rounded to 128 B: node n's 64-B run of a plain OT = 16 sheet
    // then sits on bank half n & 1 in every slot (bank-half swap, locate_ag)
    s.sheet_bytes = (static_cast<uint32_t>(slab_node_rows(G, H, 0)) * (G + 1) * (NS > 0 ? NS : OT) * 4u + 127u) & ~127u;
    s.recw_bytes = sh.R * 8u;  // float2 {alpha, gamma} per row
    // goff (staged only): node offsets go global -> registers (prefetched a pair
    // ahead) instead of riding the ring with the records, so the ring holds only
    // sheets and {alpha, gamma}. The planner uses it only where it buys a taller
    // row tile (cfg3's G = 28 layer: 2 x 108 KB sheets + 2 x 8 KB records fit
    // the 1024-row tile, 6.76 -> 5.92 ms per chain step); where the ring fits
    // either way the shared-memory offsets measured faster (cfg2 17.01 vs 17.15 ms).
    s.reco_bytes = (mode == kModeStaged && goff) ? 0u : sh.OBLK * 4u;
    uint32_t o = mode == kModeGlobal ? 0u : s.sheet_bytes * nb;
    o = (o + 127u) & ~127u;
    s.off_recw = o;
    o += s.nrec * s.recw_bytes;
    s.off_reco = o;
    o += s.nrec * s.reco_bytes;
    o = (o + 15u) & ~15u;
    s.off_thr = o;
    s.off_pts = o;
    s.off_inv = o;
    if (mode != kModeStaged) {
        // grid constants: at least the 64 / 65 slots of grids up to G = 64 (the
        // round-1 layout, which measured 1.5% faster at cfg4 than the tight one)
        o += static_cast<uint32_t>(grid_L(G) > 64 ? grid_L(G) : 64) * 8u;  // thresholds (fp32 or fp64)
        s.off_pts = o;
        o += static_cast<uint32_t>(G + 1 > 65 ? G + 1 : 65) * 8u;
        o = (o + 15u) & ~15u;
        s.off_inv = o;
        o += static_cast<uint32_t>(G) * 8u;  // inv_h
        o = (o + 15u) & ~15u;
    }
    s.off_bar = o;
    o += 8u * nb;
    s.off_cnt = o;
    o += 4u * nb;
    s.total = (o + 127u) & ~127u;
    return s;
}

// K1 (staged path): cell records for every (pair, row) in the order K2 consumes
// them. A CTA stages a 64-row x 16-pair X tile through shared memory (row-
// contiguous loads), locates each (row, pair) and writes
//   W[p][row]                        = {alpha, gamma}            (coalesced)
//   O[p][tile][offset_slot(row % R)] = packed slab / node offset
// Rows in [rows, rows_pad) get zero records (their outputs are discarded).
template <typename XT, bool SHORT_TILES>
__global__ void __launch_bounds__(256) records_kernel(const XT* __restrict__ X, int64_t rows, int64_t rows_pad,
                                                      int n_in, const __grid_constant__ GridConst gc, ShapeRT sh,
                                                      int H, float2* __restrict__ W, int* __restrict__ O,
                                                      const InputMap im, int64_t Rt, int hs) {
    __shared__ XT xs[64][33];
    __shared__ int64_t rbase[64];
    __shared__ int coff[32];
    __shared__ XT thr[kMaxThr];
    __shared__ double pts[kMaxThr + 1];
    __shared__ double invh[kMaxThr];
    const int G = gc.G, pairs = n_in / 2, tid = threadIdx.x;
    for (int k = tid; k < gc.L; k += 256) thr[k] = thr_of<XT>(gc)[k];
    for (int k = tid; k <= G; k += 256) pts[k] = gc.points[k];
    for (int k = tid; k < G; k += 256) invh[k] = gc.inv_h[k];
    const int p0 = blockIdx.y * 16;
    const int r = tid & 63, pq = tid >> 6;
    const int64_t tiles = SHORT_TILES ? rows_pad / Rt : rows_pad >> sh.lgR;  // K2 row tiles of Rt <= R rows
    // row tiles of 64 are strided over gridDim.x, so the per-CTA setup above
    // (thresholds, points, inverse widths) is amortized over many tiles
    for (int64_t r0 = static_cast<int64_t>(blockIdx.x) * 64; r0 < rows_pad; r0 += static_cast<int64_t>(gridDim.x) * 64) {
        __syncthreads();  // previous tile's xs / rbase fully consumed
        if (tid < 64) rbase[tid] = in_rowbase(im, r0 + tid, n_in);
        if (tid < 32) coff[tid] = in_coloff(im, 2 * p0 + tid);
        __syncthreads();
        XT v[8];  // all 8 loads of this thread in flight before any store
        if (!im.conv) {  // dense X: rows n_in apart, no per-element address lookup
            const int rr0 = tid >> 5, c = tid & 31, col = 2 * p0 + c;
            const XT* xp = X + (r0 + rr0 + im.row_offset) * n_in + col;
#pragma unroll
            for (int t = 0; t < 8; ++t)
                v[t] = (r0 + rr0 + 8 * t < rows && col < n_in) ? __ldg(xp + static_cast<int64_t>(8 * t) * n_in) : XT(0);
        } else {
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                const int i = tid + 256 * t;
                const int rr = i >> 5, c = i & 31;
                const int col = 2 * p0 + c;
                v[t] = (r0 + rr < rows && col < n_in) ? __ldg(X + rbase[rr] + coff[c]) : XT(0);
            }
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            const int i = tid + 256 * t;
            xs[i >> 5][i & 31] = v[t];
        }
        __syncthreads();
        // thread = (row r of the tile, pairs pq, pq+4, pq+8, pq+12 of the block):
        // the row's tile / offset slot are computed once, record addresses step
        // by whole pairs
        const int64_t g = r0 + r;
        if (g < rows_pad) {  // row tiles (R) may be shorter than the 64-row X tile
            const int64_t tile = SHORT_TILES ? g / Rt : g >> sh.lgR;  // shortened tiles: a real division
            const int slot = offset_slot(sh, static_cast<int>(g - tile * Rt));
            float2* wp = W + static_cast<size_t>(p0 + pq) * rows_pad + g;
            int* op = O + (static_cast<size_t>(p0 + pq) * tiles + tile) * sh.OBLK + slot;
            const size_t wstep = static_cast<size_t>(4) * rows_pad, ostep = static_cast<size_t>(4) * tiles * sh.OBLK;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int pl = pq + 4 * k;
                if (p0 + pl < pairs) {
                    float2 ag = make_float2(0.f, 0.f);
                    int packed = 0;
                    if (g < rows)
                        packed = locate_ag<XT>(xs[r][2 * pl], xs[r][2 * pl + 1], thr, pts, invh, G, gc.L, sh.NS, H, ag,
                                               hs ? static_cast<int>((g - tile * Rt) & 1) : -1);
                    *wp = ag;
                    *op = packed;
                }
                wp += wstep;
                op += ostep;
            }
        }
    }
}

// K1 (staged path), register-direct variant: one thread per (row, group of 4
// pairs), no shared-memory staging and no barriers. The group's 8 inputs are
// contiguous in X (dense rows; conv rows when C % 8 == 0), so a 32-byte load
// fetches them; consecutive threads take consecutive rows, so the {alpha,
// gamma} stores of a pair are coalesced. Same records, same order as
// records_kernel (locate_ag, offset_slot); rows in [rows, rows_pad) get zeros.
template <typename XT, bool SHORT_TILES>
__global__ void __launch_bounds__(256) records4_kernel(const XT* __restrict__ X, int64_t rows, int64_t rows_pad,
                                                       int n_in, const __grid_constant__ GridConst gc, ShapeRT sh,
                                                       int H, float2* __restrict__ W, int* __restrict__ O,
                                                       const InputMap im, int64_t Rt, int vec, int hs) {
    __shared__ XT thr[kMaxThr];
    __shared__ double pts[kMaxThr + 1];
    __shared__ double invh[kMaxThr];
    const int G = gc.G, pairs = n_in / 2, tid = threadIdx.x;
    for (int k = tid; k < gc.L; k += 256) thr[k] = thr_of<XT>(gc)[k];
    for (int k = tid; k <= G; k += 256) pts[k] = gc.points[k];
    for (int k = tid; k < G; k += 256) invh[k] = gc.inv_h[k];
    __syncthreads();
    const int p0 = blockIdx.y * 4;
    const int np = pairs - p0 < 4 ? pairs - p0 : 4;
    const int64_t tiles = SHORT_TILES ? rows_pad / Rt : rows_pad >> sh.lgR;
    const int c0 = in_coloff(im, 2 * p0);
    const size_t wstep = static_cast<size_t>(rows_pad), ostep = static_cast<size_t>(tiles) * sh.OBLK;
    for (int64_t g = static_cast<int64_t>(blockIdx.x) * 256 + tid; g < rows_pad; g += static_cast<int64_t>(gridDim.x) * 256) {
        XT x[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = XT(0);
        if (g < rows) {
            const XT* xr = X + in_rowbase(im, g, n_in);
            if (sizeof(XT) == 4 && vec && np == 4) {  // 8 contiguous, 32-byte aligned inputs
                float u[8];
                ldg_v8(reinterpret_cast<const float*>(xr + c0), u);
#pragma unroll
                for (int k = 0; k < 8; ++k) x[k] = static_cast<XT>(u[k]);
            } else {
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    if (k < 2 * np) x[k] = __ldg(xr + in_coloff(im, 2 * p0 + k));
            }
        }
        const int64_t tile = SHORT_TILES ? g / Rt : g >> sh.lgR;
        const int slot = offset_slot(sh, static_cast<int>(g - tile * Rt));
        float2* wp = W + static_cast<size_t>(p0) * wstep + g;
        int* op = O + (static_cast<size_t>(p0) * tiles + tile) * sh.OBLK + slot;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (k < np) {
                float2 ag = make_float2(0.f, 0.f);
                int packed = 0;
                if (g < rows)
                    packed = locate_ag<XT>(x[2 * k], x[2 * k + 1], thr, pts, invh, G, gc.L, sh.NS, H, ag,
                                           hs ? static_cast<int>((g - tile * Rt) & 1) : -1);
                wp[k * wstep] = ag;
                op[k * ostep] = packed;
            }
        }
    }
}

// ---------------------------------------------------- parity / debug views
// The PRODUCTION cell records decoded back into row_preambles' terms
// (layer.hpp:96-101): per (row, pair) the cell (i1, i2) and {alpha, gamma}.
// Packed offset = (slab << 24) | (node-within-slab * NS), node = i1'(G+1) + i2.
__device__ __forceinline__ void decode_packed(int packed, int G, int H, int NS, int& i1, int& i2) {
    const int sw = (packed >> kSwapBit) & 1;  // bank-half-swapped record: offset names node n + 1
    const int s = (packed >> kSlabShift) & 0x3f;
    const int nodews = (packed & kOffMask) / NS - sw;
    i1 = s * H + nodews / (G + 1);
    i2 = nodews % (G + 1);
}

// Reads K1's output (W[p][rows_pad], O[p][tile][offset_slot]) exactly where K2
// reads it: one thread per (row, pair), row-major over [rows][pairs].
static __global__ void __launch_bounds__(256) decode_records_kernel(const float2* __restrict__ W, const int* __restrict__ O,
                                                             int64_t rows, int64_t rows_pad, int pairs, ShapeRT sh,
                                                             int64_t Rt, int G, int H, int32_t* __restrict__ o_i1,
                                                             int32_t* __restrict__ o_i2, float2* __restrict__ o_ag) {
    const int64_t tiles = rows_pad / Rt;
    const int64_t total = rows * pairs;
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < total;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = k / pairs;
        const int p = static_cast<int>(k - r * pairs);
        const int64_t tile = r / Rt;
        const int slot = offset_slot(sh, static_cast<int>(r - tile * Rt));
        int i1, i2;
        decode_packed(O[(static_cast<size_t>(p) * tiles + tile) * sh.OBLK + slot], G, H, sh.NS, i1, i2);
        o_i1[k] = i1;
        o_i2[k] = i2;
        o_ag[k] = W[static_cast<size_t>(p) * rows_pad + r];
    }
}

// The in-kernel locate of the fused / global gather modes and the narrow kernel
// (locate_ag on the same shared-memory grid constants, same node stride NS and
// slab height H), one thread per (row, pair), decoded like decode_records_kernel.
template <typename XT>
__global__ void __launch_bounds__(256) locate_ag_kernel(const XT* __restrict__ X, int64_t rows, int n_in,
                                                        const __grid_constant__ GridConst gc, int NS, int H, int hs,
                                                        int32_t* __restrict__ o_i1, int32_t* __restrict__ o_i2,
                                                        float2* __restrict__ o_ag) {
    __shared__ XT thr[kMaxThr];
    __shared__ double pts[kMaxThr + 1];
    __shared__ double invh[kMaxThr];
    const int G = gc.G;
    for (int k = threadIdx.x; k < gc.L; k += blockDim.x) thr[k] = thr_of<XT>(gc)[k];
    for (int k = threadIdx.x; k <= G; k += blockDim.x) pts[k] = gc.points[k];
    for (int k = threadIdx.x; k < G; k += blockDim.x) invh[k] = gc.inv_h[k];
    __syncthreads();
    const int pairs = n_in / 2;
    const int64_t total = rows * pairs;
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < total;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = k / pairs;
        const int p = static_cast<int>(k - r * pairs);
        const XT* xr = X + r * n_in + 2 * p;
        float2 ag;
        int i1, i2;
        decode_packed(locate_ag<XT>(xr[0], xr[1], thr, pts, invh, G, gc.L, NS, H, ag, hs ? static_cast<int>(r & 1) : -1),
                      G, H, NS, i1, i2);
        o_i1[k] = i1;
        o_i2[k] = i2;
        o_ag[k] = ag;
    }
}

// Pixel records for the implicit-im2col conv (kModePixel): the cell of a
// channel pair depends only on the input pixel, and a k x k conv reads every
// pixel in k^2 patch rows, so locating per pixel instead of per (row, pair)
// does 1/k^2 of the work. out[cp][pixel] = {alpha, gamma, packed offset, 0}
// for channel pair cp = (2cp, 2cp+1) of every pixel of the NHWC batch
// (npix = N*H*W), computed exactly as the in-kernel locate would (locate_ag,
// same node stride NS and slab height H). Thread per (cp, pixel), pixel
// fastest: coalesced record stores.
template <typename XT>
__global__ void __launch_bounds__(256) pixel_records_kernel(const XT* __restrict__ img, int64_t npix, int C,
                                                            const __grid_constant__ GridConst gc, int NS, int H,
                                                            int4* __restrict__ out) {
    __shared__ XT thr[kMaxThr];
    __shared__ double pts[kMaxThr + 1];
    __shared__ double invh[kMaxThr];
    const int G = gc.G;
    for (int k = threadIdx.x; k < gc.L; k += blockDim.x) thr[k] = thr_of<XT>(gc)[k];
    for (int k = threadIdx.x; k <= G; k += blockDim.x) pts[k] = gc.points[k];
    for (int k = threadIdx.x; k < G; k += blockDim.x) invh[k] = gc.inv_h[k];
    __syncthreads();
    const int64_t total = npix * (C / 2);
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < total;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t cp = k / npix, pix = k - cp * npix;
        const XT* x = img + pix * C + 2 * cp;
        float2 ag;
        const int packed = locate_ag<XT>(x[0], x[1], thr, pts, invh, G, gc.L, NS, H, ag);
        out[k] = make_int4(__float_as_int(ag.x), __float_as_int(ag.y), packed, 0);
    }
}

// CTA -> (row tile, output tile). The hardware dispatches CTAs in linear order
// (x fastest); the linear index walks groups of `group` output tiles, and within
// a group the output tiles fastest, then the row tiles. A wave of SMs then holds
// ~num_sms / group row tiles x group output tiles, running in near lockstep over
// the pairs, so L2 serves each pair's sheet to the wave's row tiles and each row
// tile's records to its output tiles; DRAM reads per wave are (row tiles x
// records) + (output tiles x sheets) instead of every row tile's records (group
// 1: one output tile per wave, the round-1 order). The planner picks the group
// (choose_cta_group: 1 by default, measured fastest); results do not depend on it.
__device__ __forceinline__ void cta_tile(unsigned bx, unsigned by, unsigned gx, unsigned gy, int group,
                                         int64_t& tile, int& ot) {
    if (group <= 1) {
        tile = bx;
        ot = static_cast<int>(by);
        return;
    }
    const unsigned lid = by * gx + bx, span = static_cast<unsigned>(group) * gx;
    const unsigned grp = lid / span, rem = lid - grp * span;
    const unsigned gs = min(static_cast<unsigned>(group), gy - grp * group);
    ot = static_cast<int>(grp * group + rem % gs);
    tile = rem / gs;
}

// K2/K3: gather-accumulate (with in-kernel locate in fused/global modes).
// Grid: x = row tile (R rows), y = output tile (OT outputs), remapped by
// cta_tile. Table layout
// [out_tile][pair][node][OT] fp32: one (out_tile, pair) sheet — or one slab of
// it — is one contiguous bulk copy, and each node's OT outputs are a
// contiguous, float4-aligned run.
//
// Pipeline over units u = (pair p, slab s), no CTA-wide barrier in the loop:
//   * sheets (+ the pair's records when staged): NBUF-deep ring in shared memory
//     filled by the bulk-copy engine; "full[slot]" mbarriers count landed bytes.
//     The LAST warp to finish with a slot (shared-memory atomic counter) issues
//     the copy that refills it, so no warp waits on a producer and none is
//     dedicated to producing.
//   * fused mode: every warp locates the cells of its own rows for the next pair
//     into a warp-private record slice (x pair prefetched a pair ahead).
//   * gather: lane group `sub` handles one row, lane c4 V float4 runs of outputs
//     (V = lane_vectors(OT)); per row one LDS.64 of {alpha, gamma} (one
//     wavefront for the warp's rows; an LDS.128 of four weights would cost two)
//     and 4 V LDS.128 of coefficients (nodes n, n+1, n+G+1, n+G+2), 16 V FMAs;
//     a lane group's RT node offsets are contiguous
//     (int4 loads, kept in registers across the pair's slabs). With slabs
//     (SLAB = true) a row is gathered only during its cell's slab.
//   * DUP (OT = 16): the table stores every node's 16 outputs twice, side by
//     side in one 128-B line ([node][copy][OT], node stride NS = 2 OT), and odd
//     lane groups read the second copy. A 64-B run otherwise sits on the bank
//     half its node's parity picks, so the 8 rows of an instruction collide on a
//     half ~27% of the time; with the copies every instruction puts 4 rows on
//     each half: 4 wavefronts, no conflicts, for twice the sheet bytes.
//
// Accumulation order per (row, output): acc = 0; for p: acc += t_p with
// t_p = ((w00 p00 + w10 p10) + w01 p01) + w11 p11 (fused multiply-adds), the
// reference's per-pair grouping (layer.hpp:129); then acc * gamma (layer.hpp:131).
// Deterministic: no data atomics, fixed order, independent of the launch shape.
template <int OT, int RT, typename XT, int MODE, bool SLAB, int NW, bool TAIL, bool DUP, bool GOFF>
__global__ void __launch_bounds__(NW * 32, 1)
    fwd_fused_kernel(const XT* __restrict__ X, const OutDests<XT> out, int64_t rows, int n_in, int n_out,
                     const float* __restrict__ table, int pairs, int nbuf, int S, float gamma,
                     const __grid_constant__ GridConst gc, const float2* __restrict__ recW,
                     const int* __restrict__ recO, int64_t rows_pad, const InputMap im, const EmitRecords emit,
                     const __grid_constant__ GridConst gc_next, int Rt_arg, int pair_block, int cta_group) {
    using Sh = FusedShape<OT, RT, NW, DUP>;
    constexpr int R = Sh::R;
    const int Rt = TAIL ? Rt_arg : R;  // full-tile kernels keep the row tile a compile-time constant
    constexpr int NT = NW * 32;
    constexpr bool kSmemSheet = MODE != kModeGlobal;
    constexpr int NS = DUP ? 2 * OT : OT;  // node stride in the table / sheets (floats)
    static_assert(!DUP || (!SLAB && MODE != kModeGlobal), "DUP: unslabbed smem sheets");
    extern __shared__ __align__(1024) unsigned char smem[];
    const int G = gc.G;
    const int nodes = (G + 1) * (G + 1);
    const int H = (G + S - 1) / S;
    static_assert(!GOFF || MODE == kModeStaged, "GOFF: staged mode only");
    const FusedSmem L = fused_smem_layout(G, OT, RT, nbuf, MODE, S, NW, NS, GOFF ? 1 : 0);
    float* sheets = reinterpret_cast<float*>(smem);
    float2* rec_w = reinterpret_cast<float2*>(smem + L.off_recw);
    int* rec_o = reinterpret_cast<int*>(smem + L.off_reco);
    XT* thr = reinterpret_cast<XT*>(smem + L.off_thr);
    double* pts = reinterpret_cast<double*>(smem + L.off_pts);
    double* inv = reinterpret_cast<double*>(smem + L.off_inv);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.off_bar);
    unsigned* cnt = reinterpret_cast<unsigned*>(smem + L.off_cnt);

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    constexpr int V = Sh::V;
    constexpr int VSTEP = 4 * Sh::LPR;  // floats between a lane's float4 runs
    const int sub = lane / Sh::LPR, c4 = lane % Sh::LPR;
    // Float offset of the lane's v-th run. Runs of 64 B (OT / V = 16) sit on one
    // bank half each (nodes are 128-B aligned); odd lane groups take the runs in
    // the order 1 0 3 2, so every instruction puts half its rows on each bank
    // half: 8 rows x 64 B in 4 wavefronts, no conflicts. DUP at V = 2: a node's
    // 128-B line holds its two copies; lane group `sub` reads copy sub & 1 and
    // its two 32-B runs in the order given by (sub >> 1) & 1, so each 8-bank
    // quarter of an instruction gets 4 of its 16 rows: 4 wavefronts, no conflicts.
    const int vflip = V >= 2 ? (VSTEP == 16 ? (sub & 1) : ((sub >> 1) & 1)) : 0;
    auto vofs = [&](int v) { return (v ^ vflip) * VSTEP; };
    const int lane_base = 4 * c4 + (DUP ? (sub & 1) * OT : 0);  // DUP: odd lane groups read the second copy
    int64_t tile;
    int ot;
    cta_tile(blockIdx.x, blockIdx.y, gridDim.x, gridDim.y, cta_group, tile, ot);
    // row tiles of Rt <= R rows (Rt < R balances the grid over the SMs): lane
    // slots q >= Rt and rows >= rows are masked, issuing no gathers
    const int64_t row0 = tile * Rt;
    const float* tsrc = table + static_cast<size_t>(ot) * pairs * nodes * NS;
    const uint32_t sheet_floats = static_cast<uint32_t>(nodes) * NS;
    const uint32_t slab_floats = static_cast<uint32_t>(H) * (G + 1) * NS;  // slab stride within a sheet
    const int64_t tiles = rows_pad / Rt;
    const uint32_t recw_copy = static_cast<uint32_t>(Rt) * 8u;  // this tile's records (<= L.recw_bytes)
    const int units = pairs * S;

    // conflict-free loads of plain (not duplicated) OT = 16 sheets by bank-half
    // swapped records (locate_ag's hsub; the gather loop un-swaps)
    constexpr bool kHalfSwap = OT == 16 && !DUP && V == 1 && kSmemSheet && !SLAB;

    constexpr bool kLocate = MODE == kModeFused || MODE == kModeGlobal;  // in-kernel locate
    constexpr bool kPix = MODE == kModePixel;
    if constexpr (kLocate) {
        for (int k = tid; k < gc.L; k += NT) thr[k] = thr_of<XT>(gc)[k];
        for (int k = tid; k <= G; k += NT) pts[k] = gc.points[k];
        for (int k = tid; k < G; k += NT) inv[k] = gc.inv_h[k];
    }
    uint64_t policy = 0, policy_rec = 0;
    if constexpr (kSmemSheet) {
        if (tid == 0) {
            for (int s = 0; s < nbuf; ++s) {
                mbar_init(&full[s], 1);
                cnt[s] = 0;
            }
            fence_barrier_init();
        }
        policy = policy_evict_last();
        policy_rec = policy_evict_first();
    }
    __syncthreads();

    // one thread: slab (+ the pair's records when staged) of unit u into ring
    // slot `slot` (= u % nbuf; passed in, the loop tracks it without divisions)
    auto issue = [&](int u, int slot) {
        const int p = SLAB ? u / S : u, s = SLAB ? u - p * S : 0;
        const uint32_t bytes = static_cast<uint32_t>(slab_node_rows(G, H, s)) * (G + 1) * NS * 4u;
        const bool with_rec = MODE == kModeStaged && s == 0;
        mbar_arrive_expect_tx(&full[slot], bytes + (with_rec ? recw_copy + L.reco_bytes : 0u));
        const char* src =
            reinterpret_cast<const char*>(tsrc + static_cast<size_t>(p) * sheet_floats + static_cast<size_t>(s) * slab_floats);
        char* dst = reinterpret_cast<char*>(sheets) + static_cast<size_t>(slot) * L.sheet_bytes;
        constexpr uint32_t kChunk = 32768;
        for (uint32_t o = 0; o < bytes; o += kChunk) {
            const uint32_t n = bytes - o < kChunk ? bytes - o : kChunk;
            bulk_g2s(dst + o, src + o, n, &full[slot], policy);
        }
        if constexpr (MODE == kModeStaged) {
            if (with_rec) {
                const int rs = SLAB ? p % L.nrec : slot;  // unslabbed: nrec == nbuf and p == u
                bulk_g2s(reinterpret_cast<char*>(rec_w) + rs * L.recw_bytes,
                         recW + static_cast<size_t>(p) * rows_pad + row0, recw_copy, &full[slot], policy_rec);
                if (L.reco_bytes)
                    bulk_g2s(reinterpret_cast<char*>(rec_o) + rs * L.reco_bytes,
                             recO + (static_cast<size_t>(p) * tiles + tile) * Sh::OBLK, L.reco_bytes, &full[slot],
                             policy_rec);
            }
        }
    };
    if constexpr (kSmemSheet) {
        if (tid == 0) {
            const int pre = nbuf < units ? nbuf : units;
            for (int u = 0; u < pre; ++u) issue(u, u);
        }
    }

    // --- warp-local cell locate (fused / global): lane handles rows q = k*32 + lane;
    // pixel mode: the lane fetches those rows' records of the pixel each pair reads
    XT xa[Sh::LOC], xb[Sh::LOC];
    const XT* xrow[Sh::LOC];
    int pixb[Sh::LOC];     // pixel mode: the row's top-left input pixel (absolute index)
    int4 prec[Sh::LOC];    // pixel mode: the prefetched records {alpha, gamma, packed offset, 0}
    const int4* const pixrec = reinterpret_cast<const int4*>(recO);
    // float2 x-pair loads when both columns are adjacent and 8-byte aligned
    const bool x_vec_ok = (reinterpret_cast<uintptr_t>(X) & 7) == 0 && (!im.conv || (im.C & 1) == 0);
#pragma unroll
    for (int k = 0; k < Sh::LOC; ++k) {
        const int q = k * 32 + lane;
        const int64_t r = row0 + warp * Sh::ROWS_W + q;
        const bool in_tile = warp * Sh::ROWS_W + q < Rt;
        xrow[k] = (MODE != kModeStaged && q < Sh::ROWS_W && in_tile && r < rows) ? X + in_rowbase(im, r, n_in) : nullptr;
        if constexpr (kPix) pixb[k] = xrow[k] ? static_cast<int>(in_rowbase(im, r, n_in) / im.C) : 0;
    }
    auto prefetch = [&](int p) {
        if constexpr (kPix) {  // pair p = channels (ch, ch+1) of tap (dy, dx): record [ch/2][pixel + tap offset]
            const int tap = (2 * p) / im.C, ch = 2 * p - tap * im.C;
            const int dy = tap / im.k, dx = tap - dy * im.k;
            const int4* base = pixrec + static_cast<int64_t>(ch >> 1) * im.npix + dy * im.W + dx;
#pragma unroll
            for (int k = 0; k < Sh::LOC; ++k) prec[k] = xrow[k] ? __ldg(base + pixb[k]) : make_int4(0, 0, 0, 0);
            return;
        }
        const int c0 = in_coloff(im, 2 * p), c1 = im.conv ? in_coloff(im, 2 * p + 1) : c0 + 1;
#pragma unroll
        for (int k = 0; k < Sh::LOC; ++k) {
            if (xrow[k]) {
                if (sizeof(XT) == 4 && x_vec_ok) {
                    const float2 v = __ldg(reinterpret_cast<const float2*>(xrow[k] + c0));
                    xa[k] = v.x;
                    xb[k] = v.y;
                } else {
                    xa[k] = __ldg(xrow[k] + c0);
                    xb[k] = __ldg(xrow[k] + c1);
                }
            } else {
                xa[k] = xb[k] = XT(0);
            }
        }
    };
    auto locate = [&]() {
        const ShapeRT shp = shape_rt(OT, RT, NW, NS);
#pragma unroll
        for (int k = 0; k < Sh::LOC; ++k) {
            const int q = k * 32 + lane;
            if (q < Sh::ROWS_W) {
                float2 ag = make_float2(0.f, 0.f);
                int packed = 0;
                if constexpr (kPix) {
                    ag = make_float2(__int_as_float(prec[k].x), __int_as_float(prec[k].y));
                    packed = prec[k].z;
                    if constexpr (kHalfSwap) {  // pixel records are plain: swap for this row's lane group
                        const int n = packed / NS, sw = (n & 1) != (lane & 1);
                        packed = (sw << kSwapBit) | ((n + sw) * NS);
                    }
                } else {
                    // the lane group gathering row q has parity q & 1 = lane & 1
                    if (xrow[k])
                        packed = locate_ag<XT>(xa[k], xb[k], thr, pts, inv, G, gc.L, NS, H, ag, kHalfSwap ? (lane & 1) : -1);
                }
                const int qc = warp * Sh::ROWS_W + q;
                rec_w[qc] = ag;
                rec_o[offset_slot(shp, qc)] = packed;
            }
        }
    };

    float4 acc[RT][V];
#pragma unroll
    for (int j = 0; j < RT; ++j)
#pragma unroll
        for (int v = 0; v < V; ++v) acc[j][v] = make_float4(0.f, 0.f, 0.f, 0.f);
    const int rstride = (G + 1) * NS;  // node (i1+1, i2) is (G+1) nodes further
    // The planner makes Rt a multiple of ROWS_W, so a warp's rows are all inside
    // the tile or all beyond it: warps beyond it issue no gathers. Rows past the
    // batch end inside the last tile gather zero-weight records (no branch in
    // the hot loop) and are not stored.
    const bool warp_live = warp * Sh::ROWS_W < Rt;

    // Pair-block summation (layers with many pairs, e.g. config 5's 4096): every
    // pair_block pairs the block sum in registers is added into a running sum
    // kept in the output rows (dests[0], this GPU's own Y; fp32 values, read back
    // only by the thread that wrote them) and the registers restart from zero:
    // y = (((B_1) + B_2) + ... + B_m) * gamma with B_k the in-order fp32 sum of
    // block k. Rounding error grows like sqrt(pairs (pair_block + pairs /
    // pair_block)) instead of pairs: ~3.9x smaller at 4096 pairs, block 256.
    // Block boundaries are absolute pair indices, so results stay independent of
    // the plan (tiles, slabs, modes, warps) and of row / output sharding.
    auto fold_main = [&](bool flush, bool first) {
        // The thread's geometry is re-derived here from opaque reads of the
        // special registers, so nothing this rare path needs (row / column
        // indices, addresses) is hoisted out of the gather loop and kept live
        // in registers across it.
        unsigned t_, bx_, by_, gx_, gy_;
        asm volatile("mov.u32 %0, %%tid.x;" : "=r"(t_));
        asm volatile("mov.u32 %0, %%ctaid.x;" : "=r"(bx_));
        asm volatile("mov.u32 %0, %%ctaid.y;" : "=r"(by_));
        asm volatile("mov.u32 %0, %%nctaid.x;" : "=r"(gx_));
        asm volatile("mov.u32 %0, %%nctaid.y;" : "=r"(gy_));
        int64_t tl_;
        int ot_;
        cta_tile(bx_, by_, gx_, gy_, cta_group, tl_, ot_);
        const int w_ = static_cast<int>(t_ >> 5), sb = static_cast<int>(t_ & 31) / Sh::LPR;
        const int vf = V >= 2 ? (VSTEP == 16 ? (sb & 1) : ((sb >> 1) & 1)) : 0;
        const int cl = ot_ * OT + 4 * (static_cast<int>(t_ & 31) % Sh::LPR);
        const int64_t ld = out.ld;
        XT* const base = out.base[0] + out.col0;
        const bool vec = sizeof(XT) == 4 && (reinterpret_cast<uintptr_t>(base) & 15) == 0 && (ld & 3) == 0;
        const bool live = !TAIL || w_ * Sh::ROWS_W < Rt;
#pragma unroll
        for (int j = 0; j < RT; ++j) {
            const int64_t r = tl_ * Rt + w_ * Sh::ROWS_W + j * Sh::RPW + sb;
            const bool row_ok = live && r < rows;
#pragma unroll
            for (int v = 0; v < V; ++v) {
                const int cv = cl + (v ^ vf) * VSTEP;
                XT* yr = base + r * ld + cv;
                float a[4] = {acc[j][v].x, acc[j][v].y, acc[j][v].z, acc[j][v].w};
                if (row_ok) {
                    if (vec && cv + 3 < n_out) {
                        float4 m = first ? make_float4(0.f, 0.f, 0.f, 0.f) : *reinterpret_cast<const float4*>(yr);
                        a[0] = m.x + a[0], a[1] = m.y + a[1], a[2] = m.z + a[2], a[3] = m.w + a[3];
                        if (flush) *reinterpret_cast<float4*>(yr) = make_float4(a[0], a[1], a[2], a[3]);
                    } else {
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            if (cv + e < n_out) {
                                a[e] = (first ? 0.f : static_cast<float>(yr[e])) + a[e];
                                if (flush) yr[e] = static_cast<XT>(a[e]);
                            }
                        }
                    }
                }
                acc[j][v] = flush ? make_float4(0.f, 0.f, 0.f, 0.f) : make_float4(a[0], a[1], a[2], a[3]);
            }
        }
    };

    if constexpr (MODE != kModeStaged) {
        prefetch(0);
        locate();
        if (pairs > 1) prefetch(1);
        __syncwarp();
    }
    // A lane group's RT node offsets (contiguous, 16-B aligned runs of OSTRIDE ints)
    auto load_offs = [&](const int* ro, int(&o)[RT], bool global) {
        if constexpr (RT % 4 == 0) {
#pragma unroll
            for (int k = 0; k < RT / 4; ++k) {
                const int4 v = global ? __ldg(reinterpret_cast<const int4*>(ro) + k) : reinterpret_cast<const int4*>(ro)[k];
                o[4 * k] = v.x;
                o[4 * k + 1] = v.y;
                o[4 * k + 2] = v.z;
                o[4 * k + 3] = v.w;
            }
        } else if constexpr (RT == 2) {  // small-batch CTAs at V = 2: OSTRIDE = 6, 8-B aligned runs
            const int2 v = global ? __ldg(reinterpret_cast<const int2*>(ro)) : *reinterpret_cast<const int2*>(ro);
            o[0] = v.x;
            o[1] = v.y;
        } else {
            static_assert(RT == 1, "rows per thread: 1, 2 or a multiple of 4");
            o[0] = global ? __ldg(ro) : ro[0];
        }
    };
    // staged with goff: pair p's offsets come straight from K1's output (recO),
    // loaded one pair ahead into registers so the latency hides behind a pair's gather
    const int lane_slot = (warp * Sh::RPW + sub) * Sh::OSTRIDE;
    auto offs_src = [&](int pp) { return recO + (static_cast<size_t>(pp) * tiles + tile) * Sh::OBLK + lane_slot; };
    int offs[RT], offs_next[RT];  // offs_next: GOFF only (dead otherwise)
    if constexpr (GOFF) load_offs(offs_src(0), offs_next, true);
    const float2* rw = rec_w;
    int p = 0, s = 0;
    int slot = 0;         // u % nbuf
    uint32_t phase = 0;   // (u / nbuf) & 1: the "landed" mbarrier phase of unit u
    // units in pair blocks: the loop body is the same for every block, the
    // running-sum fold sits between blocks (one block when pair_block == 0)
    const int blk_units = (pair_block > 0 ? pair_block : pairs) * S;
    for (int u0 = 0; u0 < units; u0 += blk_units) {
        const int u1 = units - u0 < blk_units ? units : u0 + blk_units;
        for (int u = u0; u < u1; ++u) {
            const float* sh;
            if constexpr (kSmemSheet) {
                mbar_wait(&full[slot], phase);
                sh = sheets + static_cast<size_t>(slot) * (L.sheet_bytes / 4) + lane_base;
            } else {
                sh = tsrc + static_cast<size_t>(p) * sheet_floats + lane_base;
            }
            if (!SLAB || s == 0) {  // pair's records: weights stay in smem, offsets in registers (kept across slabs)
                const int rs = MODE == kModeStaged ? (SLAB ? p % L.nrec : slot) : 0;
                rw = rec_w + rs * (L.recw_bytes / 8) + warp * Sh::ROWS_W + sub;
                if constexpr (GOFF) {
#pragma unroll
                    for (int j = 0; j < RT; ++j) offs[j] = offs_next[j];
                    if (p + 1 < pairs) load_offs(offs_src(p + 1), offs_next, true);
                } else {
                    load_offs(rec_o + rs * (L.reco_bytes / 4) + lane_slot, offs, false);
                }
            }
            if (!TAIL || warp_live) {  // TAIL: shortened row tiles, some warps hold no rows
#pragma unroll
                for (int j = 0; j < RT; ++j) {
                    if constexpr (SLAB) {
                        // rows whose cell lies in another slab load nothing and add +0
                        const bool ok = (offs[j] >> kSlabShift) == s;
                        const float* b0 = sh + (offs[j] & kOffMask);
                        const float* b1 = b0 + rstride;
                        const float4 w = weights_ag(lds64_if(rw + j * Sh::RPW, ok));
#pragma unroll
                        for (int v = 0; v < V; ++v) {
                            const float4 p00 = lds128_if(b0 + vofs(v), ok);
                            const float4 p01 = lds128_if(b0 + vofs(v) + NS, ok);
                            const float4 p10 = lds128_if(b1 + vofs(v), ok);
                            const float4 p11 = lds128_if(b1 + vofs(v) + NS, ok);
                            fma_corners(acc[j][v], w, p00, p10, p01, p11);
                        }
                    } else {
                        const float4 w = weights_ag(rw[j * Sh::RPW]);
                        const float* b0 = sh + offs[j];
                        const float* b1 = b0 + rstride;
#pragma unroll
                        for (int v = 0; v < V; ++v) {
                            float4 p00, p01, p10, p11;
                            if constexpr (kHalfSwap) {
                                // plain OT = 16 sheet: node n's 64-B run sits on bank half
                                // n & 1, n + 1 on the other. The record names the member
                                // of {n, n+1} on the lane group's own half (sub & 1) and
                                // flags sw when that is n + 1 (locate_ag); the same shift
                                // applies to {n+G+1, n+G+2}, whose halves flip uniformly
                                // for all lanes. So every LDS puts 4 rows on each half (4
                                // wavefronts, no conflicts); the registers are un-swapped
                                // so the FMA order stays p00, p10, p01, p11.
                                const bool sw = (offs[j] >> kSwapBit) & 1;
                                const float* f0 = sh + (offs[j] & kOffMask);
                                const float* f1 = f0 + rstride;
                                const int d = sw ? -NS : NS;
                                const float4 r0 = *reinterpret_cast<const float4*>(f0);
                                const float4 r1 = *reinterpret_cast<const float4*>(f1);
                                const float4 r2 = *reinterpret_cast<const float4*>(f0 + d);
                                const float4 r3 = *reinterpret_cast<const float4*>(f1 + d);
                                p00 = sw ? r2 : r0;
                                p01 = sw ? r0 : r2;
                                p10 = sw ? r3 : r1;
                                p11 = sw ? r1 : r3;
                            } else if constexpr (kSmemSheet) {
                                p00 = *reinterpret_cast<const float4*>(b0 + vofs(v));
                                p01 = *reinterpret_cast<const float4*>(b0 + vofs(v) + NS);
                                p10 = *reinterpret_cast<const float4*>(b1 + vofs(v));
                                p11 = *reinterpret_cast<const float4*>(b1 + vofs(v) + NS);
                            } else {
                                p00 = __ldg(reinterpret_cast<const float4*>(b0 + vofs(v)));
                                p01 = __ldg(reinterpret_cast<const float4*>(b0 + vofs(v) + NS));
                                p10 = __ldg(reinterpret_cast<const float4*>(b1 + vofs(v)));
                                p11 = __ldg(reinterpret_cast<const float4*>(b1 + vofs(v) + NS));
                            }
                            fma_corners<kHalfSwap>(acc[j][v], w, p00, p10, p01, p11);
                        }
                    }
                }
            }
            __syncwarp();  // this warp is done with slot u % nbuf (and, at s == S-1, with pair p's records)
            if constexpr (kSmemSheet) {
                if (lane == 0) {
                    // acq_rel increment: releases this warp's reads of the slot (ordered
                    // before it by __syncwarp) and, for the last warp, acquires everyone
                    // else's, so all reads happen before the async-proxy overwrite below
                    if (atom_add_acq_rel_cta(&cnt[slot], 1u) == NW - 1) {  // last warp out refills the slot
                        cnt[slot] = 0;
                        if (u + nbuf < units) {
                            fence_proxy_async();
                            issue(u + nbuf, slot);
                        }
                    }
                }
                if (++slot == nbuf) {  // ring position of the next unit
                    slot = 0;
                    phase ^= 1u;
                }
            }
            if (++s == S) {
                s = 0;
                ++p;
                if constexpr (MODE != kModeStaged) {
                    if (p < pairs) {
                        locate();
                        if (p + 1 < pairs) prefetch(p + 1);
                        __syncwarp();
                    }
                }
            }
        }
        if (u1 < units) fold_main(true, u0 == 0);
    }

    // epilogue: y *= gamma (layer.hpp:131), masked store of the warp's rows into
    // every destination (peer destinations are NVLink stores issued as the
    // CTA's tile completes, overlapping the other CTAs' gathers)
    const int col = ot * OT + 4 * c4;  // run v holds outputs col + vofs(v) .. + 3
    if (pair_block > 0 && pairs > pair_block) fold_main(false, false);  // y = running sum + last block
#pragma unroll
    for (int j = 0; j < RT; ++j)
#pragma unroll
        for (int v = 0; v < V; ++v)
            acc[j][v] = make_float4(acc[j][v].x * gamma, acc[j][v].y * gamma, acc[j][v].z * gamma, acc[j][v].w * gamma);
    if constexpr (sizeof(XT) == 4) {
        if (emit.W) {
            // fused chain: the lane's outputs cv..cv+3 of each run (cv = col + vofs(v))
            // are the next layer's pairs cv/2 and cv/2 + 1. Two passes (h = 0, 1), one
            // next-layer pair per run each: locate into shared memory [pair][row], then coalesced record
            // stores — rows run contiguously in W, and when both layers use the same
            // row tile the CTA's offset block of each pair is written whole.
            constexpr int PP = OT / 4;  // next-layer pairs per pass
            float2* sW = reinterpret_cast<float2*>(smem);
            int* sO = reinterpret_cast<int*>(smem + static_cast<size_t>(PP) * R * sizeof(float2));
            unsigned char* gbase = smem + static_cast<size_t>(PP) * R * 12u;
            double* npts = reinterpret_cast<double*>(gbase);
            double* ninv = npts + kMaxThr + 1;
            float* nthr = reinterpret_cast<float*>(ninv + kMaxThr);
            const int pn_base = (ot * OT) >> 1;
            const int pairs_next = n_out >> 1;
            const bool same_tile = emit.sh.R == R;
            __syncthreads();  // all warps past the gather loop: the ring space is free
            for (int k = tid; k < kMaxThr + 1; k += NT) {
                if (k <= gc_next.G) npts[k] = gc_next.points[k];
                if (k < gc_next.G) ninv[k] = gc_next.inv_h[k];
                if (k < gc_next.L) nthr[k] = gc_next.t32[k];
            }
            for (int h = 0; h < 2; ++h) {
                __syncthreads();  // grid constants in place / the previous pass's stores done
#pragma unroll
                for (int j = 0; j < RT; ++j) {
                    const int rl = warp * Sh::ROWS_W + j * Sh::RPW + sub;
                    const int64_t r = row0 + rl;
#pragma unroll
                    for (int v = 0; v < V; ++v) {
                        float2 ag = make_float2(0.f, 0.f);
                        int packed = 0;
                        if (r < rows && col + vofs(v) + 2 * h + 1 < n_out) {
                            const float a = h ? acc[j][v].z : acc[j][v].x, b = h ? acc[j][v].w : acc[j][v].y;
                            packed = locate_ag<float>(a, b, nthr, npts, ninv, gc_next.G, gc_next.L, emit.sh.NS,
                                                      emit.H, ag);
                        }
                        const int cv = (v ^ vflip) * Sh::LPR + c4;  // (col + vofs(v) - ot OT) / 4
                        sW[cv * R + rl] = ag;
                        sO[cv * R + rl] = packed;
                    }
                }
                __syncthreads();
                for (int idx = tid; idx < PP * R; idx += NT) {
                    const int pl = idx / R, rl = idx - pl * R;
                    const int pn = pn_base + 2 * pl + h;
                    const int64_t r = row0 + rl;
                    if (pn < pairs_next && r < emit.rows_pad) emit.W[static_cast<size_t>(pn) * emit.rows_pad + r] = sW[idx];
                }
                if (same_tile) {  // the whole offset block of (pair, tile), slot order, padding slots zeroed
                    const int ob = emit.sh.OBLK;
                    for (int idx = tid; idx < PP * ob; idx += NT) {
                        const int pl = idx / ob, sl = idx - pl * ob;
                        const int pn = pn_base + 2 * pl + h;
                        if (pn >= pairs_next) continue;
                        const int grp = sl / emit.sh.OSTRIDE, jj = sl - grp * emit.sh.OSTRIDE;
                        int v = 0;
                        if (jj < emit.sh.RT) {
                            const int q = (grp / emit.sh.RPW) * emit.sh.ROWS_W + jj * emit.sh.RPW + grp % emit.sh.RPW;
                            v = sO[pl * R + q];
                        }
                        emit.O[(static_cast<size_t>(pn) * emit.tiles + tile) * ob + sl] = v;
                    }
                } else {
                    for (int idx = tid; idx < PP * R; idx += NT) {
                        const int pl = idx / R, rl = idx - pl * R;
                        const int pn = pn_base + 2 * pl + h;
                        const int64_t r = row0 + rl;
                        if (pn >= pairs_next || r >= emit.rows_pad) continue;
                        const int slot = offset_slot(emit.sh, static_cast<int>(r & (emit.sh.R - 1)));
                        emit.O[(static_cast<size_t>(pn) * emit.tiles + (r >> emit.sh.lgR)) * emit.sh.OBLK + slot] =
                            sO[idx];
                    }
                }
            }
        }
    }
#pragma unroll
    for (int d = 0; d < kMaxDest; ++d) {  // unrolled: constant indices keep `out` in the parameter space
        if (d >= out.n) break;
        XT* const base = out.base[d] + out.col0;
        const bool y_vec_ok = (reinterpret_cast<uintptr_t>(base) & 15) == 0 && (out.ld & 3) == 0;
#pragma unroll
        for (int j = 0; j < RT; ++j) {
            const int64_t r = row0 + warp * Sh::ROWS_W + j * Sh::RPW + sub;
            if ((TAIL && !warp_live) || r >= rows) continue;
            XT* yr = base + r * out.ld;
#pragma unroll
            for (int v = 0; v < V; ++v) {
                const int cv = col + vofs(v);
                if constexpr (sizeof(XT) == 4) {
                    if (cv + 3 < n_out && y_vec_ok) {
                        *reinterpret_cast<float4*>(yr + cv) = acc[j][v];
                        continue;
                    }
                }
                const float a[4] = {acc[j][v].x, acc[j][v].y, acc[j][v].z, acc[j][v].w};
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if (cv + e < n_out) yr[cv + e] = static_cast<XT>(a[e]);
            }
        }
    }
}

}  // namespace lmkan_b200
