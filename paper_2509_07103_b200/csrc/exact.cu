// Reference-precision forward: lmkan_forward (layer.hpp:108-134) with the fp64
// table, fp64 weights and fp64 accumulation, every operation explicitly
// rounded in the reference's order (no FMA contraction), so Y is BIT-IDENTICAL
// to the reference's lmkan_forward:
//   weights  w00 = (a c) inv, w10 = (b c) inv, w01 = (a d) inv, w11 = (b d) inv
//            with a, b, c, d the cell gaps and inv = inv_areas[i1 G + i2]
//            (grid.hpp:94-100), cells from the fp64 thresholds (bit-exact);
//   per row  y = 0; for p in order: y += ((w00 p00 + w10 p10) + w01 p01) + w11 p11
//            (layer.hpp:121-129); y *= gamma (layer.hpp:131).
// Selected per layer (lmkan_b200_layer_create_exact, the C++ drop-in's
// LmKanLayer::precision = 64): the fast path stays the fp32 gather
// (north_star's 1e-5 contract); this one is for callers that need the
// reference's own numbers (its unit tests compare at 1e-12 .. 1e-14).
//
// Kernel: one CTA of 16 warps per (row tile, output tile). The table is laid
// out [out_tile][pair][node][OT] doubles (OT = 32, 16 or 8 outputs, the widest
// whose sheet double-buffers in shared memory); per pair the (G+1)^2 x OT
// sheet arrives by bulk copy (cp.async.bulk + mbarrier, two buffers, a CTA
// barrier per pair). A warp locates the cells of its rows into a warp-private
// record slice (fp64 weights) — or, with several output tiles, loads them from
// exact_records_kernel's staged records (launch_exact) — then every lane gathers one output of 32 / OT
// rows per instruction: LDS.64 of a 256-B (OT = 32) or 128-B (OT = 16) run is
// 2 wavefronts with no bank conflicts. Sheets too large for shared memory
// (G > ~40) are read from L2 directly.
#include <algorithm>
#include <cstdlib>
#include <string>

#include "../../include/lmkan_b200.h"
#include "layer_impl.hpp"

using namespace lmkan_b200;

namespace {

constexpr int kExactWarps = 16;

// Outputs per lane: NRUN runs of 2 doubles (one LDS.128 each), the runs OT/2
// apart: OT = 32 and 16 take 2 runs (8 / 4 lanes per row, 4 / 8 rows per
// instruction), OT = 8 one run (4 lanes, 8 rows). A row's record (four fp64
// weights + the node) is then shared by 4 lanes' worth of outputs, not 1:
// shared-load wavefronts per coefficient 13/8 -> ~37/32 at OT = 32.
constexpr int exact_nrun(int OT) { return OT >= 16 ? 2 : 1; }
constexpr int exact_lpr(int OT) { return OT / (2 * exact_nrun(OT)); }  // lanes per row
// rows per lane group: the register tile is RT rows x 2 NRUN doubles (32 doubles)
constexpr int exact_rt(int OT) { return 16 / exact_nrun(OT); }

struct ExactSmem {
    uint32_t sheet_bytes, off_recw, off_recn, off_thr, off_pts, off_bar, total;
};
__host__ __device__ inline ExactSmem exact_smem_layout(int G, int OT, bool gsheet) {
    const int rows_w = (32 / exact_lpr(OT)) * exact_rt(OT);
    ExactSmem s;
    s.sheet_bytes = (static_cast<uint32_t>((G + 1) * (G + 1)) * OT * 8u + 127u) & ~127u;
    uint32_t o = gsheet ? 0u : 2u * s.sheet_bytes;
    s.off_recw = o;
    o += kExactWarps * rows_w * 32u;  // double4 weights
    s.off_recn = o;
    o += kExactWarps * rows_w * 4u;  // node index
    o = (o + 15u) & ~15u;
    s.off_thr = o;
    o += static_cast<uint32_t>(grid_L(G)) * 8u;
    s.off_pts = o;
    o += static_cast<uint32_t>(G + 1) * 8u;
    o = (o + 15u) & ~15u;
    s.off_bar = o;
    o += 24u;  // two "landed" mbarriers + two finished-warp counters
    s.total = (o + 127u) & ~127u;
    return s;
}

// Cell records of the staged variant, [pair][rows]: the four fp64 weights and
// the node, computed exactly as the fused kernel's locate below (so Y is the
// same bits either way). One thread per (row, pair), rows fastest: a pair's
// stores are contiguous, and the x loads of consecutive pairs share sectors
// that L2 still holds.
template <typename XT>
__global__ void exact_records_kernel(const XT* __restrict__ X, int64_t rows, int n_in,
                                     const __grid_constant__ GridConst gc, double4* __restrict__ W,
                                     int* __restrict__ N) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int p = blockIdx.y;
    if (r >= rows) return;
    const int G = gc.G;
    const double x1 = static_cast<double>(__ldg(X + r * n_in + 2 * p));
    const double x2 = static_cast<double>(__ldg(X + r * n_in + 2 * p + 1));
    const int i1 = cell_index_fast<double>(x1, gc.t64, G, gc.L);
    const int i2 = cell_index_fast<double>(x2, gc.t64, G, gc.L);
    const double a = __dsub_rn(__ldg(gc.points + i1 + 1), x1), b = __dsub_rn(x1, __ldg(gc.points + i1));
    const double c = __dsub_rn(__ldg(gc.points + i2 + 1), x2), d = __dsub_rn(x2, __ldg(gc.points + i2));
    const double inv = __ldg(gc.inv_areas + i1 * G + i2);
    const size_t k = static_cast<size_t>(p) * rows + r;
    W[k] = make_double4(__dmul_rn(__dmul_rn(a, c), inv), __dmul_rn(__dmul_rn(b, c), inv),
                        __dmul_rn(__dmul_rn(a, d), inv), __dmul_rn(__dmul_rn(b, d), inv));
    N[k] = i1 * (G + 1) + i2;
}

template <int OT, typename XT, bool GSHEET, bool STAGED>
__global__ void __launch_bounds__(kExactWarps * 32, 1)
    exact_kernel(const XT* __restrict__ X, XT* __restrict__ Y, int64_t rows, int n_in, int n_out,
                 const double* __restrict__ table, int pairs, double gamma, const __grid_constant__ GridConst gc,
                 const double4* __restrict__ recW, const int* __restrict__ recN) {
    constexpr int RT = exact_rt(OT), NRUN = exact_nrun(OT), LPR = exact_lpr(OT), RPI = 32 / LPR;
    constexpr int ROWS_W = RPI * RT, LOC = (ROWS_W + 31) / 32;
    constexpr int R = kExactWarps * ROWS_W;
    extern __shared__ __align__(1024) unsigned char smem[];
    const int G = gc.G, nodes = (G + 1) * (G + 1);
    const ExactSmem Ls = exact_smem_layout(G, OT, GSHEET);
    double* sheets = reinterpret_cast<double*>(smem);
    double4* recw = reinterpret_cast<double4*>(smem + Ls.off_recw);
    int* recn = reinterpret_cast<int*>(smem + Ls.off_recn);
    double* thr = reinterpret_cast<double*>(smem + Ls.off_thr);
    double* pts = reinterpret_cast<double*>(smem + Ls.off_pts);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Ls.off_bar);
    unsigned* cnt = reinterpret_cast<unsigned*>(bar + 2);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int k = tid; k < gc.L; k += kExactWarps * 32) thr[k] = gc.t64[k];
    for (int k = tid; k <= G; k += kExactWarps * 32) pts[k] = gc.points[k];
    const int ot = blockIdx.y;
    const double* tsrc = table + static_cast<size_t>(ot) * pairs * nodes * OT;
    const uint32_t sheet_copy = static_cast<uint32_t>(nodes) * OT * 8u;
    uint64_t policy = 0;
    auto issue = [&](int p) {  // thread 0: sheet of pair p into buffer p & 1
        mbar_arrive_expect_tx(&bar[p & 1], sheet_copy);
        const char* src = reinterpret_cast<const char*>(tsrc + static_cast<size_t>(p) * nodes * OT);
        char* dst = reinterpret_cast<char*>(sheets) + (p & 1) * Ls.sheet_bytes;
        for (uint32_t o = 0; o < sheet_copy; o += 32768u)
            bulk_g2s(dst + o, src + o, sheet_copy - o < 32768u ? sheet_copy - o : 32768u, &bar[p & 1], policy);
    };
    if constexpr (!GSHEET) {
        if (tid == 0) {
            mbar_init(&bar[0], 1);
            mbar_init(&bar[1], 1);
            cnt[0] = cnt[1] = 0;
            fence_barrier_init();
            policy = policy_evict_last();
            issue(0);
            if (pairs > 1) issue(1);
        }
    }
    __syncthreads();

    const int64_t row0 = static_cast<int64_t>(blockIdx.x) * R + warp * ROWS_W;
    const int g = lane / LPR, c = lane % LPR;
    // run r of the lane: doubles 2c + (r ^ flip) OT/2 of a node's OT. At OT = 16 a
    // run is 64 B, on the bank half its index picks: odd lane groups take the runs
    // in the order 1 0, so every LDS.128 puts half its rows on each half.
    const int flip = (OT == 16 && NRUN == 2) ? (g & 1) : 0;
    auto run_ofs = [&](int r) { return 2 * c + (r ^ flip) * (OT / 2); };
    double4* wrec = recw + warp * ROWS_W;
    int* nrec = recn + warp * ROWS_W;
    double2 acc[RT][NRUN];
#pragma unroll
    for (int j = 0; j < RT; ++j)
#pragma unroll
        for (int r = 0; r < NRUN; ++r) acc[j][r] = make_double2(0.0, 0.0);

    // x pair (staged: the cell record) of the lane's rows, loaded one pair ahead
    // (the loads are in flight during the previous pair's gather)
    XT xa[LOC], xb[LOC];
    double4 pw[LOC];
    int pn[LOC];
    auto prefetch = [&](int p) {
#pragma unroll
        for (int k = 0; k < LOC; ++k) {
            const int64_t r = row0 + k * 32 + lane;
            const bool ok = k * 32 + lane < ROWS_W && r < rows;
            if constexpr (STAGED) {
                const size_t i = static_cast<size_t>(p) * rows + r;
                const double2* q = reinterpret_cast<const double2*>(recW + (ok ? i : 0));
                const double2 lo = ok ? __ldg(q) : make_double2(0.0, 0.0), hi = ok ? __ldg(q + 1) : make_double2(0.0, 0.0);
                pw[k] = make_double4(lo.x, lo.y, hi.x, hi.y);
                pn[k] = ok ? __ldg(recN + i) : 0;
            } else {
                xa[k] = ok ? __ldg(X + r * n_in + 2 * p) : XT(0);
                xb[k] = ok ? __ldg(X + r * n_in + 2 * p + 1) : XT(0);
            }
        }
    };
    prefetch(0);
    for (int p = 0; p < pairs; ++p) {
        // cells of the warp's rows for pair p (lane: rows q = k*32 + lane); the
        // warp-private records were last read by the previous pair's gather
        __syncwarp();
#pragma unroll
        for (int k = 0; k < LOC; ++k) {
            const int q = k * 32 + lane;
            if (q < ROWS_W) {
                const int64_t r = row0 + q;
                double4 w = make_double4(0.0, 0.0, 0.0, 0.0);
                int node = 0;
                if constexpr (STAGED) {
                    w = pw[k];
                    node = pn[k];
                } else if (r < rows) {
                    const double x1 = static_cast<double>(xa[k]);
                    const double x2 = static_cast<double>(xb[k]);
                    // the estimate-then-verify index (locate.cuh): the same cell as the
                    // exact search for every input, at one MUFU + two threshold loads
                    const int i1 = cell_index_fast<double>(x1, thr, G, gc.L);
                    const int i2 = cell_index_fast<double>(x2, thr, G, gc.L);
                    const double a = __dsub_rn(pts[i1 + 1], x1), b = __dsub_rn(x1, pts[i1]);
                    const double c = __dsub_rn(pts[i2 + 1], x2), d = __dsub_rn(x2, pts[i2]);
                    const double inv = __ldg(gc.inv_areas + i1 * G + i2);
                    w = make_double4(__dmul_rn(__dmul_rn(a, c), inv), __dmul_rn(__dmul_rn(b, c), inv),
                                     __dmul_rn(__dmul_rn(a, d), inv), __dmul_rn(__dmul_rn(b, d), inv));
                    node = i1 * (G + 1) + i2;
                }
                wrec[q] = w;
                nrec[q] = node;
            }
        }
        if (p + 1 < pairs) prefetch(p + 1);
        __syncwarp();
        const double* sh;
        if constexpr (GSHEET) {
            sh = tsrc + static_cast<size_t>(p) * nodes * OT;
        } else {
            mbar_wait(&bar[p & 1], static_cast<uint32_t>((p >> 1) & 1));
            sh = sheets + (p & 1) * (Ls.sheet_bytes / 8);
        }
#pragma unroll
        for (int j = 0; j < RT; ++j) {
            const int q = j * RPI + g;
            const double4 w = wrec[q];
            const double* b0 = sh + nrec[q] * OT;
            const double* b1 = b0 + (G + 1) * OT;
#pragma unroll
            for (int r = 0; r < NRUN; ++r) {
                const int o = run_ofs(r);
                double2 p00, p10, p01, p11;
                if constexpr (GSHEET) {
                    p00 = __ldg(reinterpret_cast<const double2*>(b0 + o));
                    p10 = __ldg(reinterpret_cast<const double2*>(b1 + o));
                    p01 = __ldg(reinterpret_cast<const double2*>(b0 + OT + o));
                    p11 = __ldg(reinterpret_cast<const double2*>(b1 + OT + o));
                } else {
                    p00 = *reinterpret_cast<const double2*>(b0 + o);
                    p10 = *reinterpret_cast<const double2*>(b1 + o);
                    p01 = *reinterpret_cast<const double2*>(b0 + OT + o);
                    p11 = *reinterpret_cast<const double2*>(b1 + OT + o);
                }
                // y += ((w00 p00 + w10 p10) + w01 p01) + w11 p11, every op rounded (layer.hpp:129)
                auto term = [&](double a, double b, double cc, double d) {
                    return __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(w.x, a), __dmul_rn(w.y, b)), __dmul_rn(w.z, cc)),
                                     __dmul_rn(w.w, d));
                };
                acc[j][r].x = __dadd_rn(acc[j][r].x, term(p00.x, p10.x, p01.x, p11.x));
                acc[j][r].y = __dadd_rn(acc[j][r].y, term(p00.y, p10.y, p01.y, p11.y));
            }
        }
        // slot release without a CTA barrier (as in fwd_fused_kernel): the last
        // warp to finish with buffer p & 1 refills it with pair p + 2 (acq_rel
        // counter: its own reads released, everyone else's acquired)
        if constexpr (!GSHEET) {
            __syncwarp();
            if (lane == 0 && atom_add_acq_rel_cta(&cnt[p & 1], 1u) == kExactWarps - 1) {
                cnt[p & 1] = 0;
                if (p + 2 < pairs) {
                    fence_proxy_async();
                    issue(p + 2);
                }
            }
        }
    }
#pragma unroll
    for (int j = 0; j < RT; ++j) {
        const int64_t row = row0 + j * RPI + g;
        if (row >= rows) continue;
#pragma unroll
        for (int r = 0; r < NRUN; ++r) {
            const int col = ot * OT + run_ofs(r);
            if (col < n_out) Y[row * n_out + col] = static_cast<XT>(__dmul_rn(acc[j][r].x, gamma));
            if (col + 1 < n_out) Y[row * n_out + col + 1] = static_cast<XT>(__dmul_rn(acc[j][r].y, gamma));
        }
    }
}

// Reference layout src[node][pair][n_out] (doubles) -> [ot][pair][node][OT].
__global__ void relayout64_kernel(const double* __restrict__ src, double* __restrict__ dst, int pairs, int nodes,
                                  int n_out, int OT, int n_ot) {
    const size_t total = static_cast<size_t>(n_ot) * pairs * nodes * OT;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int qq = static_cast<int>(i % OT);
        size_t t = i / OT;
        const int node = static_cast<int>(t % nodes);
        t /= nodes;
        const int p = static_cast<int>(t % pairs);
        const int q = static_cast<int>(t / pairs) * OT + qq;
        dst[i] = q < n_out ? src[(static_cast<size_t>(node) * pairs + p) * n_out + q] : 0.0;
    }
}

__global__ void export64_kernel(const double* __restrict__ table, double* __restrict__ dst, int pairs, int nodes,
                                int n_out, int OT, int pb, int pe) {
    const int np = pe - pb;
    const size_t total = static_cast<size_t>(nodes) * np * n_out;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int q = static_cast<int>(i % n_out);
        size_t t = i / n_out;
        const int pl = static_cast<int>(t % np);
        const int node = static_cast<int>(t / np);
        dst[i] = table[((static_cast<size_t>(q / OT) * pairs + pb + pl) * nodes + node) * OT + q % OT];
    }
}

unsigned blocks_for(size_t total) { return static_cast<unsigned>(std::min<size_t>((total + 255) / 256, 148 * 64)); }

template <int OT, typename XT, bool GS, bool STAGED>
cudaError_t launch_exact_t(const lmkan_b200_layer* L, const XT* X, XT* Y, int64_t rows, const double4* W,
                           const int* N, cudaStream_t st) {
    constexpr int R = kExactWarps * (32 / exact_lpr(OT)) * exact_rt(OT);
    auto kern = exact_kernel<OT, XT, GS, STAGED>;
    const uint32_t smem = exact_smem_layout(L->G, OT, GS).total;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    const int64_t tiles = (rows + R - 1) / R;
    dim3 grid(static_cast<unsigned>(tiles), static_cast<unsigned>(L->n_ot));
    kern<<<grid, kExactWarps * 32, smem, st>>>(X, Y, rows, L->n_in, L->n_out, L->table64, L->pairs, L->gamma, L->gc,
                                                W, N);
    return cudaGetLastError();
}

template <typename XT, bool STAGED>
cudaError_t launch_exact_k(const lmkan_b200_layer* L, const XT* X, XT* Y, int64_t rows, const double4* W,
                           const int* N, cudaStream_t st) {
    const bool gs = L->exact_gsheet;
    switch (L->OT) {
        case 32: return gs ? launch_exact_t<32, XT, true, STAGED>(L, X, Y, rows, W, N, st)
                           : launch_exact_t<32, XT, false, STAGED>(L, X, Y, rows, W, N, st);
        case 16: return gs ? launch_exact_t<16, XT, true, STAGED>(L, X, Y, rows, W, N, st)
                           : launch_exact_t<16, XT, false, STAGED>(L, X, Y, rows, W, N, st);
        default: return gs ? launch_exact_t<8, XT, true, STAGED>(L, X, Y, rows, W, N, st)
                           : launch_exact_t<8, XT, false, STAGED>(L, X, Y, rows, W, N, st);
    }
}

// Staged when several output tiles would otherwise each redo the fp64 locate
// of every (row, pair) (the locate is ~24% of the fused kernel's time at cfg2's
// 32 tiles: a timing-only build without it ran 38.9 vs 51.4 ms): K1 writes the
// records once (36 B per (row, pair), row chunks under the scratch cap), the
// gather kernel prefetches them a pair ahead. LMKAN_B200_EXACT_STAGED=0 keeps
// the fused kernel.
template <typename XT>
cudaError_t launch_exact(const lmkan_b200_layer* L, const XT* X, XT* Y, int64_t rows, cudaStream_t st) {
    const char* env = std::getenv("LMKAN_B200_EXACT_STAGED");
    if (L->n_ot < 2 || L->pairs > 65535 || (env && !std::atoi(env)))
        return launch_exact_k<XT, false>(L, X, Y, rows, nullptr, nullptr, st);
    const char* cap_env = std::getenv("LMKAN_B200_MAX_SCRATCH_MB");
    const size_t cap = static_cast<size_t>(cap_env ? std::atoi(cap_env) : 4096) << 20;
    const size_t per_row = static_cast<size_t>(L->pairs) * (sizeof(double4) + sizeof(int));
    const int64_t chunk = std::max<int64_t>(1024, static_cast<int64_t>(cap / per_row));
    for (int64_t r0 = 0; r0 < rows; r0 += chunk) {
        const int64_t n = std::min(chunk, rows - r0);
        double4* W = nullptr;
        int* N = nullptr;
        cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&W), static_cast<size_t>(n) * L->pairs * sizeof(double4), st);
        if (e != cudaSuccess) return e;
        e = cudaMallocAsync(reinterpret_cast<void**>(&N), static_cast<size_t>(n) * L->pairs * sizeof(int), st);
        if (e == cudaSuccess) {
            exact_records_kernel<XT><<<dim3(static_cast<unsigned>((n + 255) / 256), static_cast<unsigned>(L->pairs)),
                                       256, 0, st>>>(X + r0 * L->n_in, n, L->n_in, L->gc, W, N);
            e = cudaGetLastError();
        }
        if (e == cudaSuccess) e = launch_exact_k<XT, true>(L, X + r0 * L->n_in, Y + r0 * L->n_out, n, W, N, st);
        if (N) cudaFreeAsync(N, st);
        cudaFreeAsync(W, st);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace

namespace lmkan_b200::api {

// Output tile of a reference-precision layer: the widest of {32, 16, 8}
// doubles whose sheet double-buffers in shared memory next to the records;
// else 8 with sheets read from L2 (gsheet).
void exact_choose(int n_out, int G, int smem_cap, int& OT, bool& gsheet) {
    for (int ot : {32, 16, 8}) {
        if (ot > 8 && ot / 2 >= n_out) continue;  // do not pad a narrow layer by 2x
        if (static_cast<int>(exact_smem_layout(G, ot, false).total) <= smem_cap) {
            OT = ot;
            gsheet = false;
            return;
        }
    }
    OT = 8;
    gsheet = true;
}

int exact_upload(lmkan_b200_layer* L, const double* P_host) {
    const size_t count = static_cast<size_t>(L->nodes) * L->pairs * L->n_out;
    double* tmp = nullptr;
    cudaError_t e = cudaMalloc(&tmp, count * sizeof(double));
    if (e == cudaSuccess) e = cudaMemcpy(tmp, P_host, count * sizeof(double), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        const size_t total = L->table64_bytes / sizeof(double);
        relayout64_kernel<<<blocks_for(total), 256>>>(tmp, L->table64, L->pairs, L->nodes, L->n_out, L->OT, L->n_ot);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    cudaFree(tmp);
    return e == cudaSuccess ? LMKAN_B200_OK : cuda_error(e, "layer_create_exact: upload P");
}

int exact_read_table(const lmkan_b200_layer* L, int pb, int pe, double* dst_host) {
    const size_t count = static_cast<size_t>(L->nodes) * (pe - pb) * L->n_out;
    double* tmp = nullptr;
    cudaError_t e = cudaMalloc(&tmp, count * sizeof(double));
    if (e == cudaSuccess) {
        export64_kernel<<<blocks_for(count), 256>>>(L->table64, tmp, L->pairs, L->nodes, L->n_out, L->OT, pb, pe);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpy(dst_host, tmp, count * sizeof(double), cudaMemcpyDeviceToHost);
    cudaFree(tmp);
    return e == cudaSuccess ? LMKAN_B200_OK : cuda_error(e, "read_table");
}

int forward_exact(const lmkan_b200_layer* L, const float* X, float* Y, int64_t rows, cudaStream_t st) {
    const cudaError_t e = launch_exact<float>(L, X, Y, rows, st);
    return e == cudaSuccess ? LMKAN_B200_OK : cuda_error(e, "lmkan_forward: exact kernel launch");
}
int forward_exact(const lmkan_b200_layer* L, const double* X, double* Y, int64_t rows, cudaStream_t st) {
    const cudaError_t e = launch_exact<double>(L, X, Y, rows, st);
    return e == cudaSuccess ? LMKAN_B200_OK : cuda_error(e, "lmkan_forward: exact kernel launch");
}

}  // namespace lmkan_b200::api
