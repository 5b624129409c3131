// sm_100a device code for the lmKAN layer forward.
//
// Reference path (paths relative to /root/reference/proj/include/lmkan/):
//   stage 1  row_preambles -> preamble -> interval_index -> sigma
//            (layer.hpp:96-101, grid.hpp:87-101, grid.hpp:72-75, grid.hpp:14-17)
//   stage 2  y[q] += w00 p00[q] + w10 p10[q] + w01 p01[q] + w11 p11[q]; y *= gamma
//            (layer.hpp:116-133)
//
// Kernels:
//   locate_kernel     K1: stage 1 alone -> (i1, i2, 4 fp32 weights) per (row, pair)
//   fwd_fused_kernel  K3: stage 1 + stage 2 in one kernel. A CTA owns a tile of R
//                     rows x OT outputs in registers and walks the pairs; per pair
//                     the (G+1)^2 x OT coefficient sheet is streamed into shared
//                     memory by the bulk-copy engine (cp.async.bulk + mbarrier,
//                     NBUF-deep ring) while the CTA locates the next pair's cells
//                     for its R rows into a shared-memory record ring. Warps then
//                     gather float4 runs of the 4 corner rows of each row's cell.
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
    const double* inv_areas;  // device [G*G]
    int G;
    int L;  // power of two >= G (search width)
};

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

// Shared-memory carve-up of the fused kernel (host and device agree on it).
struct FusedSmem {
    uint32_t sheet_bytes, off_recw, off_reco, off_thr, off_pts, off_bar, total;
};
__host__ __device__ inline FusedSmem fused_smem_layout(int nodes, int OT, int R, int nbuf) {
    FusedSmem s;
    s.sheet_bytes = static_cast<uint32_t>(nodes) * OT * 4u;
    uint32_t o = s.sheet_bytes * nbuf;
    s.off_recw = o;
    o += 2u * R * 16u;
    s.off_reco = o;
    o += 2u * R * 4u;
    o = (o + 15u) & ~15u;
    s.off_thr = o;
    o += kMaxThr * 8u;
    s.off_pts = o;
    o += (kMaxThr + 1) * 8u;
    o = (o + 15u) & ~15u;
    s.off_bar = o;
    o += 8u * nbuf;
    s.total = (o + 127u) & ~127u;
    return s;
}

template <int OT, int RT>
struct FusedShape {
    static constexpr int LPR = OT / 4;           // lanes covering one row's OT outputs (float4 each)
    static constexpr int RPW = 32 / LPR;         // rows per warp per instruction
    static constexpr int R = kWarps * RPW * RT;  // rows per CTA
};

// K3: fused locate + gather-accumulate. Grid: x = row tile (R rows), y = output
// tile (OT outputs). Table layout [out_tile][pair][node][OT] fp32, so the sheet of
// one (out_tile, pair) is one contiguous (G+1)^2*OT*4-byte bulk copy and each
// node's OT outputs are a contiguous, float4-aligned run.
//
// Accumulation order per (row, output): acc = 0; for p: acc += t_p with
// t_p = ((w00 p00 + w10 p10) + w01 p01) + w11 p11 (fused multiply-adds), the
// reference's per-pair grouping (layer.hpp:129); then acc * gamma (layer.hpp:131).
// Deterministic: no atomics, fixed order, independent of the launch shape.
template <int OT, int RT, typename XT>
__global__ void __launch_bounds__(kThreads, 1)
    fwd_fused_kernel(const XT* __restrict__ X, XT* __restrict__ Y, int64_t rows, int n_in, int n_out,
                     const float* __restrict__ table, int pairs, int nbuf, float gamma,
                     const __grid_constant__ GridConst gc) {
    using S = FusedShape<OT, RT>;
    constexpr int R = S::R;
    extern __shared__ __align__(1024) unsigned char smem[];
    const int G = gc.G;
    const int nodes = (G + 1) * (G + 1);
    const FusedSmem L = fused_smem_layout(nodes, OT, R, nbuf);
    float* sheets = reinterpret_cast<float*>(smem);
    float4* rec_w = reinterpret_cast<float4*>(smem + L.off_recw);
    int* rec_o = reinterpret_cast<int*>(smem + L.off_reco);
    XT* thr = reinterpret_cast<XT*>(smem + L.off_thr);
    double* pts = reinterpret_cast<double*>(smem + L.off_pts);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.off_bar);

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int sub = lane / S::LPR, c4 = lane % S::LPR;
    const int64_t row0 = static_cast<int64_t>(blockIdx.x) * R;
    const int ot = blockIdx.y;
    const float* tsrc = table + static_cast<size_t>(ot) * pairs * nodes * OT;
    const uint32_t sheet_floats = static_cast<uint32_t>(nodes) * OT;

    for (int k = tid; k < kMaxThr; k += kThreads) thr[k] = thr_of<XT>(gc)[k];
    for (int k = tid; k <= G; k += kThreads) pts[k] = gc.points[k];
    uint64_t policy = 0;
    if (tid == 0) {
        for (int s = 0; s < nbuf; ++s) mbar_init(&full[s], 1);
        fence_barrier_init();
        policy = policy_evict_last();
    }
    __syncthreads();

    auto issue_sheet = [&](int p) {  // tid 0 only
        const int s = p % nbuf;
        mbar_arrive_expect_tx(&full[s], L.sheet_bytes);
        const char* src = reinterpret_cast<const char*>(tsrc + static_cast<size_t>(p) * sheet_floats);
        char* dst = reinterpret_cast<char*>(sheets) + static_cast<size_t>(s) * L.sheet_bytes;
        constexpr uint32_t kChunk = 32768;
        for (uint32_t o = 0; o < L.sheet_bytes; o += kChunk) {
            const uint32_t n = L.sheet_bytes - o < kChunk ? L.sheet_bytes - o : kChunk;
            bulk_g2s(dst + o, src + o, n, &full[s], policy);
        }
    };
    if (tid == 0) {
        const int pre = nbuf < pairs ? nbuf : pairs;
        for (int p = 0; p < pre; ++p) issue_sheet(p);
    }

    auto locate = [&](int p, int buf) {
        for (int i = tid; i < R; i += kThreads) {
            const int64_t r = row0 + i;
            float4 w = make_float4(0.f, 0.f, 0.f, 0.f);
            int off = 0;
            if (r < rows) {
                const XT* xr = X + r * n_in + 2 * p;
                int i1, i2;
                locate_pair<XT>(xr[0], xr[1], thr, pts, gc.inv_areas, G, gc.L, i1, i2, w);
                off = (i1 * (G + 1) + i2) * OT;
            }
            rec_w[buf * R + i] = w;
            rec_o[buf * R + i] = off;
        }
    };

    float4 acc[RT];
#pragma unroll
    for (int j = 0; j < RT; ++j) acc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    const int rstride = (G + 1) * OT;  // node (i1+1, i2) is (G+1) nodes further

    locate(0, 0);
    __syncthreads();
    for (int p = 0; p < pairs; ++p) {
        if (p + 1 < pairs) locate(p + 1, (p + 1) & 1);
        const int s = p % nbuf;
        mbar_wait(&full[s], static_cast<uint32_t>((p / nbuf) & 1));
        const float* sh = sheets + static_cast<size_t>(s) * sheet_floats + 4 * c4;
        const float4* rw = rec_w + (p & 1) * R;
        const int* ro = rec_o + (p & 1) * R;
#pragma unroll
        for (int j = 0; j < RT; ++j) {
            const int rl = (j * kWarps + warp) * S::RPW + sub;
            const float4 w = rw[rl];
            const float* b0 = sh + ro[rl];
            const float* b1 = b0 + rstride;
            const float4 p00 = *reinterpret_cast<const float4*>(b0);
            const float4 p01 = *reinterpret_cast<const float4*>(b0 + OT);
            const float4 p10 = *reinterpret_cast<const float4*>(b1);
            const float4 p11 = *reinterpret_cast<const float4*>(b1 + OT);
            acc[j].x += fmaf(w.w, p11.x, fmaf(w.z, p01.x, fmaf(w.y, p10.x, w.x * p00.x)));
            acc[j].y += fmaf(w.w, p11.y, fmaf(w.z, p01.y, fmaf(w.y, p10.y, w.x * p00.y)));
            acc[j].z += fmaf(w.w, p11.z, fmaf(w.z, p01.z, fmaf(w.y, p10.z, w.x * p00.z)));
            acc[j].w += fmaf(w.w, p11.w, fmaf(w.z, p01.w, fmaf(w.y, p10.w, w.x * p00.w)));
        }
        __syncthreads();  // sheet slot s and record buffer (p&1) are free again
        if (tid == 0 && p + nbuf < pairs) {
            fence_proxy_async();
            issue_sheet(p + nbuf);
        }
    }

    // epilogue: y *= gamma (layer.hpp:131), masked store of the R x OT tile
    const int col = ot * OT + 4 * c4;
#pragma unroll
    for (int j = 0; j < RT; ++j) {
        const int64_t r = row0 + (j * kWarps + warp) * S::RPW + sub;
        if (r >= rows) continue;
        const float v[4] = {acc[j].x * gamma, acc[j].y * gamma, acc[j].z * gamma, acc[j].w * gamma};
        XT* yr = Y + r * n_out;
        if constexpr (sizeof(XT) == 4) {
            if (col + 3 < n_out && (n_out & 3) == 0) {
                *reinterpret_cast<float4*>(yr + col) = make_float4(v[0], v[1], v[2], v[3]);
                continue;
            }
        }
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if (col + e < n_out) yr[col + e] = static_cast<XT>(v[e]);
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

__global__ void fill_random_kernel(float* __restrict__ dst, int pairs, int nodes, int n_out_total,
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
__global__ void export_kernel(const float* __restrict__ table, double* __restrict__ dst, int pairs, int nodes,
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
