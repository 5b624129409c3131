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
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace lmkan_b200 {

constexpr int kMaxThr = 64;  // threshold slots (G <= 64)
constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;

struct GridConst {
    float t32[kMaxThr];   // thresholds, NaN-padded to L entries
    double t64[kMaxThr];
    double points[kMaxThr + 1];
    double inv_h[kMaxThr];  // 1 / (points[i+1] - points[i]), the per-axis factors of inv_areas (grid.hpp:58-64)
    const double* inv_areas;  // device [G*G]
    int G;
    int L;  // power of two >= G (search width)
};

// Where the layer input x[r][col] lives: a dense row-major X (row stride n_in),
// or the implicit im2col view of an NHWC image batch that unfold_conv would
// materialize (conv.hpp:39-60): row r = (n, oy, ox) row-major over output
// positions, column col = (dy*k + dx)*C + ch -> img[n][oy*s + dy][ox*s + dx][ch].
// Both are "row base + column offset"; row_offset shifts r for row chunks.
struct InputMap {
    int conv;  // 0: dense X, 1: implicit im2col over an NHWC image batch
    int out_h, out_w, H, W, C, k, s;
    int64_t row_offset;
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
    for (int k = threadIdx.x; k < kMaxThr; k += blockDim.x) thr[k] = thr_of<XT>(gc)[k];
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
    const float e = __expf(-fabsf(xf));
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
template <typename XT>
__device__ __forceinline__ int locate_ag(XT x1, XT x2, const XT* thr, const double* pts, const double* invh, int G,
                                         int L, int OT, int H, float2& ag) {
    const int i1 = cell_index_fast<XT>(x1, thr, G, L);
    const int i2 = cell_index_fast<XT>(x2, thr, G, L);
    ag.x = __double2float_rn(__dmul_rn(__dsub_rn(pts[i1 + 1], static_cast<double>(x1)), invh[i1]));
    ag.y = __double2float_rn(__dmul_rn(__dsub_rn(pts[i2 + 1], static_cast<double>(x2)), invh[i2]));
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

// Kernel variants of the layer forward.
enum : int {
    kModeFused = 0,   // K3: cells located in-kernel (warp-local), sheets via bulk copy
    kModeStaged = 1,  // K2: cell records produced by K1 (records_kernel), sheets + records via bulk copy
    kModeGlobal = 2,  // fallback for sheets larger than shared memory: in-kernel locate, sheets read from L2
    kModeNarrow = 3,  // K4: n_out <= 4, whole table resident in shared memory, lanes over pairs
};

// Row <-> thread mapping shared by K1 (which writes records in K2's order) and K2.
template <int OT, int RT, int NW = kWarps>
struct FusedShape {
    static constexpr int LPR = OT / 4;               // lanes covering one row's OT outputs (float4 each)
    static constexpr int RPW = 32 / LPR;             // rows per warp per gather instruction
    static constexpr int ROWS_W = RPW * RT;          // rows owned by one warp
    static constexpr int LOC = (ROWS_W + 31) / 32;   // cells each lane locates per pair (fused mode)
    static constexpr int R = NW * ROWS_W;             // rows per CTA
    static constexpr int OSTRIDE = RT + (RPW > 2 ? 4 : 0);  // padded per-lane-group offset run (bank spread)
    static constexpr int OBLK = NW * RPW * OSTRIDE;         // offset ints per CTA per pair
};
// Runtime twin of FusedShape for host code / K1.
struct ShapeRT {
    int OT, RT, LPR, RPW, ROWS_W, R, OSTRIDE, OBLK, NW;
    int lgRPW, lgROWS_W, lgR;  // RPW, ROWS_W, R are powers of two (OT, RT, NW are)
};
__host__ __device__ constexpr int ilog2(int v) { return v > 1 ? 1 + ilog2(v >> 1) : 0; }
__host__ __device__ inline ShapeRT shape_rt(int OT, int RT, int NW = kWarps) {
    ShapeRT s;
    s.OT = OT;
    s.RT = RT;
    s.NW = NW;
    s.LPR = OT / 4;
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
                                                       int NW = kWarps) {
    const ShapeRT sh = shape_rt(OT, RT, NW);
    const int H = (G + S - 1) / S;
    const int nb = nbuf > 0 ? nbuf : 1;
    FusedSmem s;
    s.nrec = mode == kModeStaged ? staged_nrec(nb, S) : 1;
    s.sheet_bytes = static_cast<uint32_t>(slab_node_rows(G, H, 0)) * (G + 1) * OT * 4u;
    s.recw_bytes = sh.R * 8u;  // float2 {alpha, gamma} per row
    s.reco_bytes = sh.OBLK * 4u;
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
        o += kMaxThr * 8u;
        s.off_pts = o;
        o += (kMaxThr + 1) * 8u;
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
template <typename XT>
__global__ void __launch_bounds__(256) records_kernel(const XT* __restrict__ X, int64_t rows, int64_t rows_pad,
                                                      int n_in, const __grid_constant__ GridConst gc, ShapeRT sh,
                                                      int H, float2* __restrict__ W, int* __restrict__ O,
                                                      const InputMap im) {
    __shared__ XT xs[64][33];
    __shared__ int64_t rbase[64];
    __shared__ int coff[32];
    __shared__ XT thr[kMaxThr];
    __shared__ double pts[kMaxThr + 1];
    __shared__ double invh[kMaxThr];
    const int G = gc.G, pairs = n_in / 2, tid = threadIdx.x;
    for (int k = tid; k < kMaxThr; k += 256) thr[k] = thr_of<XT>(gc)[k];
    for (int k = tid; k <= G; k += 256) pts[k] = gc.points[k];
    for (int k = tid; k < G; k += 256) invh[k] = gc.inv_h[k];
    const int p0 = blockIdx.y * 16;
    const int r = tid & 63, pq = tid >> 6;
    const int64_t tiles = rows_pad >> sh.lgR;
    // row tiles of 64 are strided over gridDim.x, so the per-CTA setup above
    // (thresholds, points, inverse widths) is amortized over many tiles
    for (int64_t r0 = static_cast<int64_t>(blockIdx.x) * 64; r0 < rows_pad; r0 += static_cast<int64_t>(gridDim.x) * 64) {
        __syncthreads();  // previous tile's xs / rbase fully consumed
        if (tid < 64) rbase[tid] = in_rowbase(im, r0 + tid, n_in);
        if (tid < 32) coff[tid] = in_coloff(im, 2 * p0 + tid);
        __syncthreads();
        XT v[8];  // all 8 loads of this thread in flight before any store
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            const int i = tid + 256 * t;
            const int rr = i >> 5, c = i & 31;
            const int col = 2 * p0 + c;
            v[t] = (r0 + rr < rows && col < n_in) ? __ldg(X + rbase[rr] + coff[c]) : XT(0);
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
            const int64_t tile = g >> sh.lgR;
            const int slot = offset_slot(sh, static_cast<int>(g & (sh.R - 1)));
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
                        packed = locate_ag<XT>(xs[r][2 * pl], xs[r][2 * pl + 1], thr, pts, invh, G, gc.L, sh.OT, H, ag);
                    *wp = ag;
                    *op = packed;
                }
                wp += wstep;
                op += ostep;
            }
        }
    }
}

// K2/K3: gather-accumulate (with in-kernel locate in fused/global modes).
// Grid: x = row tile (R rows), y = output tile (OT outputs). Table layout
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
//   * gather: lane group `sub` handles one row, lane c4 a float4 of outputs; per
//     row one LDS.64 of {alpha, gamma} (one wavefront for the warp's rows; an
//     LDS.128 of four weights would cost two) and 4 LDS.128 of coefficients
//     (nodes n, n+1, n+G+1, n+G+2), 16 FMAs; a lane group's RT node offsets are contiguous
//     (int4 loads, kept in registers across the pair's slabs). With slabs
//     (SLAB = true) a row is gathered only during its cell's slab.
//
// Accumulation order per (row, output): acc = 0; for p: acc += t_p with
// t_p = ((w00 p00 + w10 p10) + w01 p01) + w11 p11 (fused multiply-adds), the
// reference's per-pair grouping (layer.hpp:129); then acc * gamma (layer.hpp:131).
// Deterministic: no data atomics, fixed order, independent of the launch shape.
template <int OT, int RT, typename XT, int MODE, bool SLAB, int NW>
__global__ void __launch_bounds__(NW * 32, 1)
    fwd_fused_kernel(const XT* __restrict__ X, const OutDests<XT> out, int64_t rows, int n_in, int n_out,
                     const float* __restrict__ table, int pairs, int nbuf, int S, float gamma,
                     const __grid_constant__ GridConst gc, const float2* __restrict__ recW,
                     const int* __restrict__ recO, int64_t rows_pad, const InputMap im, const EmitRecords emit,
                     const __grid_constant__ GridConst gc_next) {
    using Sh = FusedShape<OT, RT, NW>;
    constexpr int R = Sh::R;
    constexpr int NT = NW * 32;
    constexpr bool kSmemSheet = MODE != kModeGlobal;
    extern __shared__ __align__(1024) unsigned char smem[];
    const int G = gc.G;
    const int nodes = (G + 1) * (G + 1);
    const int H = (G + S - 1) / S;
    const FusedSmem L = fused_smem_layout(G, OT, RT, nbuf, MODE, S, NW);
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
    const int sub = lane / Sh::LPR, c4 = lane % Sh::LPR;
    const int64_t tile = blockIdx.x;
    const int64_t row0 = tile * R;
    const int ot = blockIdx.y;
    const float* tsrc = table + static_cast<size_t>(ot) * pairs * nodes * OT;
    const uint32_t sheet_floats = static_cast<uint32_t>(nodes) * OT;
    const uint32_t slab_floats = static_cast<uint32_t>(H) * (G + 1) * OT;  // slab stride within a sheet
    const int64_t tiles = rows_pad / R;
    const int units = pairs * S;

    if constexpr (MODE != kModeStaged) {
        for (int k = tid; k < kMaxThr; k += NT) thr[k] = thr_of<XT>(gc)[k];
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

    auto issue = [&](int u) {  // one thread: slab (+ the pair's records when staged) of unit u
        const int p = u / S, s = u - p * S;
        const int slot = u % nbuf;
        const uint32_t bytes = static_cast<uint32_t>(slab_node_rows(G, H, s)) * (G + 1) * OT * 4u;
        const bool with_rec = MODE == kModeStaged && s == 0;
        mbar_arrive_expect_tx(&full[slot], bytes + (with_rec ? L.recw_bytes + L.reco_bytes : 0u));
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
                const int rs = p % L.nrec;
                bulk_g2s(reinterpret_cast<char*>(rec_w) + rs * L.recw_bytes,
                         recW + static_cast<size_t>(p) * rows_pad + row0, L.recw_bytes, &full[slot], policy_rec);
                bulk_g2s(reinterpret_cast<char*>(rec_o) + rs * L.reco_bytes,
                         recO + (static_cast<size_t>(p) * tiles + tile) * Sh::OBLK, L.reco_bytes, &full[slot],
                         policy_rec);
            }
        }
    };
    if constexpr (kSmemSheet) {
        if (tid == 0) {
            const int pre = nbuf < units ? nbuf : units;
            for (int u = 0; u < pre; ++u) issue(u);
        }
    }

    // --- warp-local cell locate (fused / global): lane handles rows q = k*32 + lane
    XT xa[Sh::LOC], xb[Sh::LOC];
    const XT* xrow[Sh::LOC];
    // float2 x-pair loads when both columns are adjacent and 8-byte aligned
    const bool x_vec_ok = (reinterpret_cast<uintptr_t>(X) & 7) == 0 && (!im.conv || (im.C & 1) == 0);
#pragma unroll
    for (int k = 0; k < Sh::LOC; ++k) {
        const int q = k * 32 + lane;
        const int64_t r = row0 + warp * Sh::ROWS_W + q;
        xrow[k] = (MODE != kModeStaged && q < Sh::ROWS_W && r < rows) ? X + in_rowbase(im, r, n_in) : nullptr;
    }
    auto prefetch = [&](int p) {
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
        const ShapeRT shp = shape_rt(OT, RT, NW);
#pragma unroll
        for (int k = 0; k < Sh::LOC; ++k) {
            const int q = k * 32 + lane;
            if (q < Sh::ROWS_W) {
                float2 ag = make_float2(0.f, 0.f);
                int packed = 0;
                if (xrow[k]) packed = locate_ag<XT>(xa[k], xb[k], thr, pts, inv, G, gc.L, OT, H, ag);
                const int qc = warp * Sh::ROWS_W + q;
                rec_w[qc] = ag;
                rec_o[offset_slot(shp, qc)] = packed;
            }
        }
    };

    float4 acc[RT];
#pragma unroll
    for (int j = 0; j < RT; ++j) acc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    const int rstride = (G + 1) * OT;  // node (i1+1, i2) is (G+1) nodes further

    if constexpr (MODE != kModeStaged) {
        prefetch(0);
        locate();
        if (pairs > 1) prefetch(1);
        __syncwarp();
    }
    int offs[RT];
    const float2* rw = rec_w;
    int p = 0, s = 0;
    for (int u = 0; u < units; ++u) {
        const float* sh;
        if constexpr (kSmemSheet) {
            const int slot = u % nbuf;
            mbar_wait(&full[slot], static_cast<uint32_t>((u / nbuf) & 1));
            sh = sheets + static_cast<size_t>(slot) * (L.sheet_bytes / 4) + 4 * c4;
        } else {
            sh = tsrc + static_cast<size_t>(p) * sheet_floats + 4 * c4;
        }
        if (!SLAB || s == 0) {  // pair's records: weights stay in smem, offsets to registers (kept across slabs)
            const int rs = MODE == kModeStaged ? p % L.nrec : 0;
            rw = rec_w + rs * (L.recw_bytes / 8) + warp * Sh::ROWS_W + sub;
            const int* ro = rec_o + rs * (L.reco_bytes / 4) + (warp * Sh::RPW + sub) * Sh::OSTRIDE;
#pragma unroll
            for (int k = 0; k < RT / 4; ++k) {
                const int4 v = reinterpret_cast<const int4*>(ro)[k];
                offs[4 * k] = v.x;
                offs[4 * k + 1] = v.y;
                offs[4 * k + 2] = v.z;
                offs[4 * k + 3] = v.w;
            }
        }
#pragma unroll
        for (int j = 0; j < RT; ++j) {
            float4 w, p00, p01, p10, p11;
            if constexpr (SLAB) {
                // rows whose cell lies in another slab load nothing and add +0
                const bool v = (offs[j] >> kSlabShift) == s;
                const float* b0 = sh + (offs[j] & kOffMask);
                const float* b1 = b0 + rstride;
                w = weights_ag(lds64_if(rw + j * Sh::RPW, v));
                p00 = lds128_if(b0, v);
                p01 = lds128_if(b0 + OT, v);
                p10 = lds128_if(b1, v);
                p11 = lds128_if(b1 + OT, v);
            } else {
                w = weights_ag(rw[j * Sh::RPW]);
                const float* b0 = sh + offs[j];
                const float* b1 = b0 + rstride;
                if constexpr (kSmemSheet) {
                    p00 = *reinterpret_cast<const float4*>(b0);
                    p01 = *reinterpret_cast<const float4*>(b0 + OT);
                    p10 = *reinterpret_cast<const float4*>(b1);
                    p11 = *reinterpret_cast<const float4*>(b1 + OT);
                } else {
                    p00 = __ldg(reinterpret_cast<const float4*>(b0));
                    p01 = __ldg(reinterpret_cast<const float4*>(b0 + OT));
                    p10 = __ldg(reinterpret_cast<const float4*>(b1));
                    p11 = __ldg(reinterpret_cast<const float4*>(b1 + OT));
                }
            }
            acc[j].x += fmaf(w.w, p11.x, fmaf(w.z, p01.x, fmaf(w.y, p10.x, w.x * p00.x)));
            acc[j].y += fmaf(w.w, p11.y, fmaf(w.z, p01.y, fmaf(w.y, p10.y, w.x * p00.y)));
            acc[j].z += fmaf(w.w, p11.z, fmaf(w.z, p01.z, fmaf(w.y, p10.z, w.x * p00.z)));
            acc[j].w += fmaf(w.w, p11.w, fmaf(w.z, p01.w, fmaf(w.y, p10.w, w.x * p00.w)));
        }
        __syncwarp();  // this warp is done with slot u % nbuf (and, at s == S-1, with pair p's records)
        if constexpr (kSmemSheet) {
            if (lane == 0) {
                const int slot = u % nbuf;
                // acq_rel increment: releases this warp's reads of the slot (ordered
                // before it by __syncwarp) and, for the last warp, acquires everyone
                // else's, so all reads happen before the async-proxy overwrite below
                if (atom_add_acq_rel_cta(&cnt[slot], 1u) == NW - 1) {  // last warp out refills the slot
                    cnt[slot] = 0;
                    if (u + nbuf < units) {
                        fence_proxy_async();
                        issue(u + nbuf);
                    }
                }
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

    // epilogue: y *= gamma (layer.hpp:131), masked store of the warp's rows into
    // every destination (peer destinations are NVLink stores issued as the
    // CTA's tile completes, overlapping the other CTAs' gathers)
    const int col = ot * OT + 4 * c4;
#pragma unroll
    for (int j = 0; j < RT; ++j) acc[j] = make_float4(acc[j].x * gamma, acc[j].y * gamma, acc[j].z * gamma,
                                                      acc[j].w * gamma);
    if constexpr (sizeof(XT) == 4) {
        if (emit.W) {
            // fused chain: this lane's outputs col..col+3 are the next layer's pairs
            // col/2 and col/2 + 1. Two passes (h = 0, 1), one next-layer pair per lane
            // each: locate into shared memory [pair][row], then coalesced record
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
                npts[k] = gc_next.points[k];
                if (k < kMaxThr) {
                    ninv[k] = gc_next.inv_h[k];
                    nthr[k] = gc_next.t32[k];
                }
            }
            for (int h = 0; h < 2; ++h) {
                __syncthreads();  // grid constants in place / the previous pass's stores done
#pragma unroll
                for (int j = 0; j < RT; ++j) {
                    const int rl = warp * Sh::ROWS_W + j * Sh::RPW + sub;
                    const int64_t r = row0 + rl;
                    float2 ag = make_float2(0.f, 0.f);
                    int packed = 0;
                    if (r < rows && col + 2 * h + 1 < n_out) {
                        const float a = h ? acc[j].z : acc[j].x, b = h ? acc[j].w : acc[j].y;
                        packed = locate_ag<float>(a, b, nthr, npts, ninv, gc_next.G, gc_next.L, emit.sh.OT, emit.H, ag);
                    }
                    sW[c4 * R + rl] = ag;
                    sO[c4 * R + rl] = packed;
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
            if (r >= rows) continue;
            XT* yr = base + r * out.ld;
            if constexpr (sizeof(XT) == 4) {
                if (col + 3 < n_out && y_vec_ok) {
                    *reinterpret_cast<float4*>(yr + col) = acc[j];
                    continue;
                }
            }
            const float v[4] = {acc[j].x, acc[j].y, acc[j].z, acc[j].w};
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (col + e < n_out) yr[col + e] = static_cast<XT>(v[e]);
        }
    }
}

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
    o += kMaxThr * 8u + (kMaxThr + 1) * 8u + static_cast<uint32_t>(G) * 8u + 16u;
    return (o + 127u) & ~127u;
}

template <typename XT, int NO>
__global__ void __launch_bounds__(kNarrowThreads, 1)
    narrow_kernel(const XT* __restrict__ X, const OutDests<XT> out, int64_t rows, int n_in, int n_out,
                  const float* __restrict__ table, float gamma, const __grid_constant__ GridConst gc,
                  const InputMap im) {
    extern __shared__ __align__(1024) unsigned char smem[];
    const int G = gc.G, pairs = n_in / 2, nodes = (G + 1) * (G + 1);
    const uint32_t tab_bytes = static_cast<uint32_t>(nodes) * pairs * NO * 4u;
    float* tab = reinterpret_cast<float*>(smem);
    uint32_t o = (tab_bytes + 15u) & ~15u;
    XT* thr = reinterpret_cast<XT*>(smem + o);
    o += kMaxThr * 8u;
    double* pts = reinterpret_cast<double*>(smem + o);
    o += (kMaxThr + 1) * 8u;
    double* inv = reinterpret_cast<double*>(smem + o);
    o += static_cast<uint32_t>(G) * 8u;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + ((o + 7u) & ~7u));
    const int tid = threadIdx.x;
    for (int k = tid; k < kMaxThr; k += kNarrowThreads) thr[k] = thr_of<XT>(gc)[k];
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
    for (int64_t r = static_cast<int64_t>(blockIdx.x) * kNarrowThreads + tid; r < rows;
         r += static_cast<int64_t>(gridDim.x) * kNarrowThreads) {
        float acc[NO];
#pragma unroll
        for (int q = 0; q < NO; ++q) acc[q] = 0.f;
        const XT* xr = X + in_rowbase(im, r, n_in);
        auto one_pair = [&](int p, XT x1, XT x2) {
            float2 ag;
            const int off = locate_ag<XT>(x1, x2, thr, pts, inv, G, gc.L, NO, G, ag);
            const float4 w = weights_ag(ag);
            const float* b = tab + static_cast<size_t>(p) * nodes * NO + off;
#pragma unroll
            for (int q = 0; q < NO; ++q)
                acc[q] += fmaf(w.w, b[rs1 + NO + q], fmaf(w.z, b[NO + q], fmaf(w.y, b[rs1 + q], w.x * b[q])));
        };
        int p = 0;
        if (vec4) {
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

// ------------------------------------------------------- table preparation
// Reference layout src[node][pair][out_total] (layer.hpp:34-45) -> device layout
// dst[ot][pair][node][OT] for the output slice [out_begin, out_begin + n_out_local),
// zero padded to n_ot*OT. One thread per destination element (coalesced on both
// sides along the output index).
template <typename T>
__global__ void relayout_kernel(const T* __restrict__ src, float* __restrict__ dst, int pairs, int nodes,
                                int n_out_total, int out_begin, int n_out_local, int OT, int n_ot) {
    const size_t total = static_cast<size_t>(n_ot) * pairs * nodes * OT;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int qq = static_cast<int>(i % OT);
        size_t t = i / OT;
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
                                   int out_begin, int n_out_local, int OT, int n_ot, uint64_t seed,
                                   float scale) {
    const size_t total = static_cast<size_t>(n_ot) * pairs * nodes * OT;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int qq = static_cast<int>(i % OT);
        size_t t = i / OT;
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
                              int n_out_local, int OT, int pb, int pe) {
    const int np = pe - pb;
    const size_t total = static_cast<size_t>(nodes) * np * n_out_local;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int q = static_cast<int>(i % n_out_local);
        size_t t = i / n_out_local;
        const int pl = static_cast<int>(t % np);
        const int node = static_cast<int>(t / np);
        const int ot = q / OT, qq = q % OT;
        dst[i] = table[((static_cast<size_t>(ot) * pairs + pb + pl) * nodes + node) * OT + qq];
    }
}

}  // namespace lmkan_b200
