// C-ABI implementation of include/lmkan_b200.h (host side of the B200 path).
//
// Replaces, per DESIGN.md "Boundary":
//   lmkan::build_grid            grid.hpp:44-68     -> lmkan_b200_build_grid
//   lmkan::interval_index        grid.hpp:72-75     -> lmkan_b200_thresholds (+ device search)
//   lmkan::LmKanLayer + P        layer.hpp:24-61    -> lmkan_b200_layer (prepared device table)
//   lmkan::lmkan_forward         layer.hpp:108-134  -> lmkan_b200_forward_{f32,f64,host_f32,host_f64}
//   lmkan::detail::row_preambles layer.hpp:96-101   -> lmkan_b200_locate_{f32,f64}
// There is no CPU compute fallback: without an sm_100a device every compute
// entry point fails with LMKAN_B200_ENOSYS / ECUDA.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/lmkan_b200.h"
#include "grid_host.hpp"
#include "host_rng.hpp"
#include "kernels.cuh"
#include "layer_impl.hpp"
#include "host_pipeline.hpp"

using namespace lmkan_b200;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    if (e == cudaErrorMemoryAllocation)
        return fail(LMKAN_B200_ENOMEM, std::string(what) + ": " + cudaGetErrorString(e));
    if (e == cudaErrorNoKernelImageForDevice || e == cudaErrorInvalidDeviceFunction ||
        e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver)
        return fail(LMKAN_B200_ENOSYS, std::string(what) + ": " + cudaGetErrorString(e));
    return fail(LMKAN_B200_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CK(call)                                              \
    do {                                                      \
        cudaError_t _e = (call);                              \
        if (_e != cudaSuccess) return cuda_fail(_e, #call);   \
    } while (0)

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

int require_sm100(int device) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
        cudaGetLastError();
        return fail(LMKAN_B200_ENOSYS, "no CUDA device visible (the B200 path has no CPU fallback)");
    }
    if (device < 0 || device >= n) return fail(LMKAN_B200_EINVAL, "device ordinal out of range");
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device);
    if (major != 10 || minor != 0)
        return fail(LMKAN_B200_ENOSYS, "kernels are built for sm_100a (B200); device is sm_" +
                                           std::to_string(major) + std::to_string(minor));
    return LMKAN_B200_OK;
}

int max_smem_optin(int device) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    return v > 0 ? v : 232448;
}

// ---------------------------------------------------------------- planning
// float4 accumulators per thread (the register tile); rows per thread RT =
// choice / lane_vectors(OT), so the rows per CTA do not depend on V
constexpr int kRTChoices[] = {16, 8, 4};
constexpr int kMaxSlabs = 4;

int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}

// Output tile width for a layer: the widest of {64, 32, 16} (not padding a
// small layer by 2x or more) whose whole sheet can be double-buffered in shared
// memory; only if none can, the fewest i1-slabs (up to 3) that double-buffer,
// else the narrowest single-buffered. Unslabbed wins over wider: a slabbed
// sheet makes every row issue (predicated-off) loads in every slab (measured at
// G = 28: OT 32 unslabbed 7.0 ms, OT 16 8.6 ms, OT 32 two slabs 11.2 ms).
// Before that (G >= 12): the widest double-buffered unslabbed OT that still
// gives >= 3 output tiles, so the planner stages the cells (K1 locates each
// (row, pair) once for every output tile, K2 only gathers) instead of fusing
// the locate into one or two wide tiles. Measured (tools/ot_sweep.sh, same
// box), n_out = 64 as four OT = 16 tiles vs the wide tile: 576→64 G=16 262144
// rows 3.57 → 3.31 ms, 65536 rows 0.82 → 0.76, conv stage 3 0.307 → 0.283;
// 128→64 G=28 2^20 rows 3.40 (OT 32) → 3.06, 65536 rows 0.244 → 0.226; but
// 64→64 G=8 (81-node sheets, a cheap fused locate) 16384 rows 0.041 → 0.043
// and config 1's step +2.4%, hence G >= 12. n_out = 128 keeps OT = 32 (4.86 ms
// vs 5.67 at OT 16), n_out = 32 OT = 32 (fused; 0.27 vs 0.35 ms at OT 16).
bool out_tile_fits(int OT, int G, int want_buf, int S, int smem_cap) {
    for (int A : kRTChoices) {
        // (global offsets: the tallest tile, unslabbed, only; see make_plan)
        const FusedSmem s = fused_smem_layout(G, OT, A / lane_vectors(OT), want_buf, kModeStaged, S, kWarps, 0,
                                              A == kRTChoices[0] && S == 1 ? 1 : 0);
        if (static_cast<int>(s.total) <= smem_cap) return true;
    }
    return false;
}

int choose_out_tile(int n_out, int G, int smem_cap) {
    const int v = env_int("LMKAN_B200_OT", 0);
    if (v == 16 || v == 32 || v == 64) return v;
    if (G >= 12)
        for (int OT : {64, 32, 16})
            if ((n_out + OT - 1) / OT >= 3 && out_tile_fits(OT, G, 2, 1, smem_cap)) return OT;
    for (int want_buf : {2, 1}) {
        for (int S = 1; S <= (want_buf == 2 ? 3 : 1); ++S) {
            for (int OT : {64, 32, 16}) {
                if (OT > 16 && OT / 2 >= n_out) continue;
                if (out_tile_fits(OT, G, want_buf, S, smem_cap)) return OT;
            }
        }
    }
    return 16;
}

// Duplicated-node table for an OT = 16 layer (conflict-free 64-B gathers, see
// fwd_fused_kernel) when its doubled sheet still double-buffers unslabbed in
// both modes at the tallest row tile, so it never costs sheet reuse (cfg4's
// G = 16: 37 KB; not G = 28 / 32: 108 / 139 KB). LMKAN_B200_DUP16=0 disables.
bool choose_dup(int OT, int G, int smem_cap) {
    if (OT != 16 || !env_int("LMKAN_B200_DUP16", 1)) return false;
    const int RT = kRTChoices[0] / lane_vectors(OT, 2 * OT);
    return static_cast<int>(fused_smem_layout(G, OT, RT, 2, kModeFused, 1, kWarps, 2 * OT).total) <= smem_cap &&
           static_cast<int>(fused_smem_layout(G, OT, RT, 2, kModeStaged, 1, kWarps, 2 * OT).total) <= smem_cap;
}

// Pair-block summation (fwd_fused_kernel): layers with more than 1024 pairs sum
// blocks of b pairs (a power of two, b >= 4 sqrt(pairs)) and add the block sums
// in order. Rounding-error variance ~ pairs (b + pairs / b) instead of pairs^2:
// config 5 (4096 pairs, b = 256): 15x lower variance. Each fold is a
// read-modify-write of the CTA's output tile (L2), so b trades accuracy for
// traffic: config-5 shard step 810 ms unblocked, 819 ms at b = 256, 834 ms at
// b = 64 (same box). Depends only on the layer, never on the plan.
// LMKAN_B200_PAIR_BLOCK overrides (0 = off).
int choose_pair_block(int pairs) {
    if (const char* e = std::getenv("LMKAN_B200_PAIR_BLOCK")) return std::max(0, std::atoi(e));
    if (pairs <= 1024) return 0;
    int b = 1;
    while (static_cast<int64_t>(b) * b < 16LL * pairs) b <<= 1;
    return b;
}

// CTA order of the gather grid (cta_tile, gather.cuh): g output tiles per
// group; a wave of the SMs holds about num_sms / g row tiles x g output tiles.
// Measured (same box, tools/ab_ctagroup.sh): g > 1 cuts K2's DRAM reads —
// config 2 9.5 GB (g = 1) -> 6.4 (2) / 5.1 (4) / 6.1 (8), the config-5 shard
// 199 -> 165 GB (2), 530 (16), 650 (64) — but is never faster: config 2
// +0.06% at every g > 1, config 3 +0.6% at g = 4, config 5 +0.2% at g = 2 and
// +4% / +11% / +15% at g = 7 / 16 / 64. The kernels are bound by the shared-
// memory port with DRAM at 9-20% of its bandwidth, so the default stays the
// fastest order (g = 1, row tiles fastest). LMKAN_B200_CTA_GROUP overrides.
int choose_cta_group(const lmkan_b200_layer* L, const Plan&) {
    return std::max(1, std::min(env_int("LMKAN_B200_CTA_GROUP", 1), L->n_ot));
}

// Mode: staged (K1 + K2) when several output tiles re-read the same cells (the
// locate then runs once per (row, pair) instead of once per output tile and
// the gather kernel's shared-memory port serves only gathers); fused (K3)
// otherwise; global-sheet fallback when nothing fits shared memory.
// Within a mode: prefer double buffering with the fewest slabs, then the
// largest row tile that still fills the GPU with one wave of CTAs.
bool make_plan(const lmkan_b200_layer* L, int64_t rows, int smem_cap, Plan& out, int force_mode_arg = -1) {
    // ring depth: up to 8, as deep as shared memory allows (cfg4's 37 KB DUP
    // sheets: 5 slots, 0.2353 -> 0.2313 ms vs 4; cfg1/2/3/5 unchanged: their
    // sheets fit 2-4 slots); LMKAN_B200_MAX_NBUF overrides
    const int max_nbuf = std::max(2, std::min(16, env_int("LMKAN_B200_MAX_NBUF", 8)));
    const int force_rt = env_int("LMKAN_B200_RT", 0), force_nbuf = env_int("LMKAN_B200_NBUF", 0),
              force_s = env_int("LMKAN_B200_SLABS", 0);
    if (L->narrow) {
        const int64_t ctas = std::min<int64_t>(L->num_sms, (rows + kNarrowThreads - 1) / kNarrowThreads);
        out = Plan{L->OT, 1, 1, kModeNarrow, 1, shape_rt(16, 4), narrow_smem_bytes(L->G, L->pairs, L->OT), ctas,
                   rows, 1, 0};
        return static_cast<int>(out.smem) <= smem_cap;
    }
    int force_mode = force_mode_arg;
    if (const char* e = force_mode_arg >= 0 ? nullptr : std::getenv("LMKAN_B200_MODE")) {
        if (!std::strcmp(e, "fused")) force_mode = kModeFused;
        if (!std::strcmp(e, "staged")) force_mode = kModeStaged;
        if (!std::strcmp(e, "global")) force_mode = kModeGlobal;
    }
    // staged when >= 3 output tiles re-read the cells, or when the batch is too
    // small to give every SM a 16-warp CTA (the per-pair locate then sits on the
    // critical path of the few rows each CTA owns; measured 32 vs 47 us at cfg1)
    const int rt_small = kRTChoices[2] / lane_vectors(L->OT, L->ns);
    const int r_small = shape_rt(L->OT, rt_small, kWarps, L->ns).R;
    const bool small = ((rows + r_small - 1) / r_small) * L->n_ot < L->num_sms;
    const int NSt = L->ns;  // node stride of the table (2 OT for duplicated-node tables)
    const int pref = (L->n_ot >= 3 || small) ? kModeStaged : kModeFused;
    const int modes[3] = {pref, pref == kModeStaged ? kModeFused : kModeStaged, kModeGlobal};
    for (int mode : modes) {
        if (force_mode >= 0 && mode != force_mode) continue;
        const bool smem_sheet = mode != kModeGlobal;
        if (L->dup && !smem_sheet) continue;  // duplicated-node tables: shared-memory sheets only
        for (int min_buf : {2, 1}) {
            if (!smem_sheet && min_buf == 2) continue;
            for (int S = 1; S <= (smem_sheet ? kMaxSlabs : 1); ++S) {
                if (force_s && S != force_s) continue;
                if (S > 1 && (min_buf == 1 || L->dup)) continue;
                for (int A : kRTChoices) {
                    const int RT = A / lane_vectors(L->OT, L->ns);
                    if (force_rt && RT != force_rt) continue;
                    if (mode == kModeGlobal && A != kRTChoices[2]) continue;  // the global-sheet kernel is built for RT2 only
                    // warps per CTA: 16, or for batches too small to give half the
                    // SMs a 16-warp CTA at RT = 4, the largest of {8, 4, 2, 1} that
                    // does. (Not all SMs: conv stage 3's 16384 rows ran 0.307 ms as
                    // 128 CTAs of 16 warps and 0.423 ms as 256 of 8 — 1.7 waves of
                    // CTAs that each still stream every sheet.)
                    int NW = kWarps;
                    if (A == kRTChoices[2] && S == 1 && mode != kModeGlobal) {
                        const int force_nw = env_int("LMKAN_B200_NW", 0);
                        if (force_nw) {
                            NW = force_nw;
                        } else {
                            while (NW > 1 && ((rows + shape_rt(L->OT, RT, NW, NSt).R - 1) / shape_rt(L->OT, RT, NW, NSt).R) *
                                                     L->n_ot * 2 < L->num_sms)
                                NW >>= 1;
                        }
                    }
                    const ShapeRT sh = shape_rt(L->OT, RT, NW, NSt);
                    const int64_t tiles = (rows + sh.R - 1) / sh.R;
                    // a taller row tile reuses each sheet for more rows; take it while the
                    // grid still covers >= 3/4 of the SMs (cfg4: RT 16 with 128 CTAs 0.392 ms
                    // beat RT 8 with 256 CTAs = 1.7 waves, 0.404 ms)
                    if (!force_rt && A != kRTChoices[2] && tiles * L->n_ot * 4 < L->num_sms * 3) continue;
                    for (int nbuf = smem_sheet ? max_nbuf : 0; nbuf >= (smem_sheet ? min_buf : 0); --nbuf) {
                        if (force_nbuf && smem_sheet && nbuf != force_nbuf) continue;
                        const int units = L->pairs * S;
                        if (smem_sheet && nbuf > units && nbuf > 1) continue;
                        // staged: offsets through the ring, else (when only that fits) from global
                        int goff = 0;
                        FusedSmem s = fused_smem_layout(L->G, L->OT, RT, nbuf, mode, S, NW, NSt);
                        if (static_cast<int>(s.total) > smem_cap && mode == kModeStaged && A == kRTChoices[0] &&
                            S == 1 && NW == kWarps && !L->dup && env_int("LMKAN_B200_GOFF", 1)) {
                            goff = 1;
                            s = fused_smem_layout(L->G, L->OT, RT, nbuf, mode, S, NW, NSt, 1);
                        }
                        if (static_cast<int>(s.total) > smem_cap) continue;
                        // Balance: rows per tile Rt <= R so a grid of less than one wave
                        // fills the SMs: cfg4's 128 CTAs of 2048 rows become 147 of 1792
                        int64_t Rt = sh.R, nt = tiles;
                        if (env_int("LMKAN_B200_BALANCE", 1) && A >= 8 && NW == kWarps && S == 1 &&
                            mode != kModeGlobal) {
                            // only a grid of less than one wave: with more waves the tail is
                            // a small fraction and shortened tiles (less sheet reuse, idle
                            // warps) cost more than they save (cfg2's chunked host path:
                            // e2e 19.5 -> 21.0 ms when its 256-CTA chunks were balanced)
                            const int64_t ctas = tiles * L->n_ot;
                            const int64_t want = ctas < L->num_sms ? L->num_sms / L->n_ot : 0;
                            if (want > tiles) {
                                // whole warps only (a warp is all in or all out of the
                                // tile: no masked rows in the hot loop); also even
                                Rt = (rows + want - 1) / want;
                                Rt = std::min<int64_t>(sh.R, (Rt + sh.ROWS_W - 1) / sh.ROWS_W * sh.ROWS_W);
                                nt = (rows + Rt - 1) / Rt;
                            }
                        }
                        out = Plan{L->OT, RT, nbuf, mode, S, sh, s.total, nt, nt * Rt,
                                   mode == kModeStaged ? 2 : 1, Rt, goff};
                        out.cta_group = choose_cta_group(L, out);
                        return true;
                    }
                }
            }
        }
    }
    return false;
}

// Cap on the stream-ordered cell-record scratch of the staged mode; larger
// batches are processed in row chunks (LMKAN_B200_MAX_SCRATCH_MB overrides).
// implicit-im2col conv in the fused mode: records per image pixel (kModePixel)
bool pixel_eligible(const Plan& pl, const InputMap& im) {
    return pl.mode == kModeFused && pl.S == 1 && im.conv && im.C % 2 == 0 && im.npix > 0 &&
           im.npix < (int64_t(1) << 31) && env_int("LMKAN_B200_PIXREC", 1);
}

// Ring depth vs L1: the gather reads the pixel records through L1 (each is
// reused by up to k^2 patch rows), and L1 gets what the sheet ring leaves of
// the SM's 256 KB. When the CTA's records fit beside a shallower ring (>= 2
// slots), take the deepest ring that leaves them room — conv stage 2: 6 slots
// 0.276 ms at a 3.6% L1 hit rate, 2 slots 0.271 ms at 74% (ncu) — else keep
// the deepest (cfg4: 259 KB of records per CTA fit no L1; 5 slots beat 2 by 2.4%).
void pixel_ring_cap(const lmkan_b200_layer* L, const InputMap& im, Plan& plx) {
    if (env_int("LMKAN_B200_NBUF", 0) || !env_int("LMKAN_B200_PIX_L1", 1)) return;
    const double px_per_row = static_cast<double>(im.H) * im.W / (static_cast<double>(im.out_h) * im.out_w);
    const double foot = static_cast<double>(plx.row_tile) * px_per_row * (im.C / 2) * sizeof(int4);
    constexpr double kL1Smem = 256.0 * 1024;  // unified L1 / shared memory per SM
    for (int nb = plx.nbuf; nb >= 2; --nb) {
        const FusedSmem fs = fused_smem_layout(L->G, L->OT, plx.RT, nb, plx.mode, plx.S, plx.sh.NW, L->ns);
        if (foot <= kL1Smem - fs.total) {
            plx.nbuf = nb;
            plx.smem = fs.total;
            return;
        }
    }
}

size_t record_scratch_cap() { return static_cast<size_t>(env_int("LMKAN_B200_MAX_SCRATCH_MB", 4096)) << 20; }

// One launch group (K1 + K2 in staged mode, K3 otherwise) over `rows` rows.
template <typename XT, int NO>
cudaError_t launch_narrow(const lmkan_b200_layer* L, const Plan& pl, const XT* X, const OutDests<XT>& Y, int64_t rows,
                          const InputMap& im, cudaStream_t st) {
    static std::atomic<bool> configured[64];  // per device: dynamic-smem opt-in done (idempotent)
    if (!configured[L->device & 63].load(std::memory_order_acquire)) {
        cudaError_t e =
            cudaFuncSetAttribute(narrow_kernel<XT, NO>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
        if (e != cudaSuccess) return e;
        configured[L->device & 63].store(true, std::memory_order_release);
    }
    narrow_kernel<XT, NO><<<static_cast<unsigned>(pl.row_tiles), kNarrowThreads, pl.smem, st>>>(
        X, Y, rows, L->n_in, L->n_out, L->table, static_cast<float>(L->gamma), L->gc, im, L->pair_block);
    return cudaGetLastError();
}

// Records handed between the layers of a fused chain: `pre` (the records this
// layer would otherwise compute in K1) and `emit` (the next layer's records,
// written by this layer's epilogue).
struct ChainLink {
    const float2* preW = nullptr;
    const int* preO = nullptr;
    EmitRecords emit{};
    const GridConst* gc_next = nullptr;
};

// K1: the cell records of `rows` rows in K2's order (records4_kernel, or the
// shared-memory-tile records_kernel when reg4 is false).
// Records for the bank-half-swapped gather (plain OT = 16 sheets, unslabbed,
// shared-memory sheets: fwd_fused_kernel's kHalfSwap) carry the swap (locate_ag).
bool half_swap(const lmkan_b200_layer* L, const Plan& pl) {
    return L->OT == 16 && !L->dup && !L->narrow && pl.S == 1 && pl.mode != kModeGlobal;
}

template <typename XT>
void launch_records(const lmkan_b200_layer* L, const Plan& pl, const XT* X, int64_t rows, const InputMap& im,
                    float2* recW, int* recO, bool reg4, cudaStream_t st) {
    const int H = (L->G + pl.S - 1) / pl.S;
    const int hs = half_swap(L, pl) ? 1 : 0;
    if (reg4) {  // register-direct K1 (records4_kernel)
        const int64_t py = (L->pairs + 3) / 4;
        const int64_t gx = std::min<int64_t>((pl.rows_pad + 255) / 256,
                                             std::max<int64_t>(1, (L->num_sms * 8 + py - 1) / py));
        dim3 g1(static_cast<unsigned>(gx), static_cast<unsigned>(py));
        // 32-byte group loads: 8 contiguous inputs at 32-byte aligned offsets
        const bool vec = (reinterpret_cast<uintptr_t>(X) & 31) == 0 &&
                         (im.conv ? (im.C % 8 == 0) : (L->n_in % 8 == 0));
        if (pl.row_tile < pl.sh.R)
            records4_kernel<XT, true><<<g1, 256, 0, st>>>(X, rows, pl.rows_pad, L->n_in, L->gc, pl.sh, H, recW,
                                                          recO, im, pl.row_tile, vec ? 1 : 0, hs);
        else
            records4_kernel<XT, false><<<g1, 256, 0, st>>>(X, rows, pl.rows_pad, L->n_in, L->gc, pl.sh, H, recW,
                                                           recO, im, pl.row_tile, vec ? 1 : 0, hs);
    } else {
        const int64_t py = (L->pairs + 15) / 16;
        const int64_t gx = std::min<int64_t>((pl.rows_pad + 63) / 64, std::max<int64_t>(1, (L->num_sms * 32 + py - 1) / py));
        dim3 g1(static_cast<unsigned>(gx), static_cast<unsigned>(py));
        if (pl.row_tile < pl.sh.R)
            records_kernel<XT, true><<<g1, 256, 0, st>>>(X, rows, pl.rows_pad, L->n_in, L->gc, pl.sh, H, recW, recO,
                                                         im, pl.row_tile, hs);
        else
            records_kernel<XT, false><<<g1, 256, 0, st>>>(X, rows, pl.rows_pad, L->n_in, L->gc, pl.sh, H, recW, recO,
                                                          im, pl.row_tile, hs);
    }
}

template <typename XT>
int forward_rows(const lmkan_b200_layer* L, const Plan& pl, const XT* X, const OutDests<XT>& Y, int64_t rows,
                 const InputMap& im,
                 cudaStream_t st, cudaEvent_t ev_begin, cudaEvent_t ev_end, const ChainLink& link = ChainLink{}) {
    if (pl.mode == kModeNarrow) {
        if (ev_begin) cudaEventRecord(ev_begin, st);
        const cudaError_t e = L->OT == 1   ? launch_narrow<XT, 1>(L, pl, X, Y, rows, im, st)
                              : L->OT == 2 ? launch_narrow<XT, 2>(L, pl, X, Y, rows, im, st)
                                           : launch_narrow<XT, 4>(L, pl, X, Y, rows, im, st);
        if (ev_end) cudaEventRecord(ev_end, st);
        if (e != cudaSuccess) return cuda_fail(e, "lmkan_forward: narrow kernel launch");
        return LMKAN_B200_OK;
    }
    float2* recW = nullptr;
    int* recO = nullptr;
    if (pl.mode == kModeStaged && !link.preW) {
        // K1: cell records, stream-ordered scratch (pool memory is retained, see alloc_layer)
        const size_t wbytes = static_cast<size_t>(L->pairs) * pl.rows_pad * sizeof(float2);
        const size_t obytes = static_cast<size_t>(L->pairs) * pl.row_tiles * pl.sh.OBLK * sizeof(int);
        CK(cudaMallocAsync(reinterpret_cast<void**>(&recW), wbytes, st));
        cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&recO), obytes, st);
        if (e != cudaSuccess) {
            cudaFreeAsync(recW, st);
            return cuda_fail(e, "lmkan_forward: record scratch");
        }
        launch_records<XT>(L, pl, X, rows, im, recW, recO, env_int("LMKAN_B200_K1", 4) == 4, st);
        e = cudaGetLastError();
        if (e != cudaSuccess) {
            cudaFreeAsync(recW, st);
            cudaFreeAsync(recO, st);
            return cuda_fail(e, "lmkan_forward: records kernel launch");
        }
    }
    // implicit-im2col conv in the fused mode: locate once per image pixel
    // (pixel_records_kernel, 1/k^2 of the per-(row, pair) locates) and let the
    // gather fetch the records through the im2col map (kModePixel)
    Plan plx = pl;
    int4* pixrec = nullptr;
    if (pixel_eligible(pl, im) && !link.emit.W) {
        const int64_t nrec = im.npix * (im.C / 2);
        CK(cudaMallocAsync(reinterpret_cast<void**>(&pixrec), static_cast<size_t>(nrec) * sizeof(int4), st));
        // one wave of 8 blocks per SM, grid-stride: each block stages the grid
        // constants once (global -> shared) and amortises that over many records
        const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((nrec + 255) / 256, L->num_sms * 8));
        pixel_records_kernel<XT><<<blocks, 256, 0, st>>>(X, im.npix, im.C, L->gc, L->ns, L->G, pixrec);
        const cudaError_t e1 = cudaGetLastError();
        if (e1 != cudaSuccess) {
            cudaFreeAsync(pixrec, st);
            return cuda_fail(e1, "lmkan_forward: pixel records kernel launch");
        }
        plx.pix = 1;
        recO = reinterpret_cast<int*>(pixrec);
        pixel_ring_cap(L, im, plx);
    }
    cudaError_t e;
    if (ev_begin) cudaEventRecord(ev_begin, st);
    const float2* useW = link.preW ? link.preW : recW;
    const int* useO = link.preW ? link.preO : recO;
    switch (L->OT) {
        case 64: e = launch_gather<64, XT>(L, plx, X, Y, rows, useW, useO, im, link.emit, link.gc_next, st); break;
        case 32: e = launch_gather<32, XT>(L, plx, X, Y, rows, useW, useO, im, link.emit, link.gc_next, st); break;
        default:
            e = L->dup ? launch_gather<16, XT, true>(L, plx, X, Y, rows, useW, useO, im, link.emit, link.gc_next, st)
                       : launch_gather<16, XT>(L, plx, X, Y, rows, useW, useO, im, link.emit, link.gc_next, st);
            break;
    }
    if (ev_end) cudaEventRecord(ev_end, st);
    if (recW) cudaFreeAsync(recW, st);
    if (recO) cudaFreeAsync(recO, st);  // K1 records or the pixel records
    if (e != cudaSuccess) return cuda_fail(e, "lmkan_forward: gather kernel launch");
    return LMKAN_B200_OK;
}

template <typename XT>
int forward_device_dests(const lmkan_b200_layer* L, const XT* X, const OutDests<XT>& out, int64_t rows,
                         cudaStream_t st, cudaEvent_t ev_begin = nullptr, cudaEvent_t ev_end = nullptr,
                         InputMap im = InputMap{}) {
    if (!L) return fail(LMKAN_B200_EINVAL, "lmkan_forward: null layer");
    if (rows < 0) return fail(LMKAN_B200_EINVAL, "lmkan_forward: negative row count");
    if (rows == 0) return LMKAN_B200_OK;
    if (!X || out.n < 1 || out.n > kMaxDest) return fail(LMKAN_B200_EINVAL, "lmkan_forward: null X or Y");
    for (int d = 0; d < out.n; ++d)
        if (!out.base[d] || reinterpret_cast<uintptr_t>(out.base[d]) % sizeof(XT) != 0)
            return fail(LMKAN_B200_EINVAL, "lmkan_forward: X and Y must be aligned to their element size");
    if (reinterpret_cast<uintptr_t>(X) % sizeof(XT) != 0)
        return fail(LMKAN_B200_EINVAL, "lmkan_forward: X and Y must be aligned to their element size");
    if (out.col0 < 0 || out.ld < out.col0 + L->n_out)
        return fail(LMKAN_B200_EINVAL, "lmkan_forward: output row stride narrower than the layer's columns");
    DeviceGuard g(L->device);
    if (L->exact) {  // reference precision: plain [rows][n_out] output only
        if (out.n != 1 || out.col0 != 0 || out.ld != L->n_out || im.conv)
            return fail(LMKAN_B200_EINVAL, "lmkan_forward: reference-precision layers support the plain forward only");
        if (ev_begin) cudaEventRecord(ev_begin, st);
        const int rc = api::forward_exact(L, X, out.base[0], rows, st);
        if (ev_end) cudaEventRecord(ev_end, st);
        return rc;
    }
    const int cap = max_smem_optin(L->device);
    Plan pl;
    if (!make_plan(L, rows, cap, pl))
        return fail(LMKAN_B200_EINVAL, "lmkan_forward: no kernel variant fits shared memory (G too large)");
    int64_t chunk = rows;
    if (pl.mode == kModeStaged) {
        const size_t per_row = static_cast<size_t>(L->pairs) * (sizeof(float2) + sizeof(int) * 2);
        const int64_t max_rows = static_cast<int64_t>(record_scratch_cap() / per_row) / pl.sh.R * pl.sh.R;
        if (rows > max_rows) chunk = std::max<int64_t>(max_rows, pl.sh.R);
    }
    if ((chunk + pl.sh.R - 1) / pl.sh.R > 0x7fffffff)
        return fail(LMKAN_B200_EINVAL, "lmkan_forward: batch too large");
    for (int64_t r0 = 0; r0 < rows; r0 += chunk) {
        const int64_t n = std::min(chunk, rows - r0);
        Plan pc = pl;
        if (n != rows && !make_plan(L, n, cap, pc))
            return fail(LMKAN_B200_EINVAL, "lmkan_forward: no kernel variant fits shared memory");
        const bool first = r0 == 0, last = r0 + n >= rows;
        InputMap imc = im;
        imc.row_offset = r0;
        if (int rc = forward_rows<XT>(L, pc, X, dests_at_row(out, r0), n, imc, st, first ? ev_begin : nullptr,
                                      last ? ev_end : nullptr))
            return rc;
    }
    return LMKAN_B200_OK;
}

template <typename XT>
int forward_device(const lmkan_b200_layer* L, const XT* X, XT* Y, int64_t rows, cudaStream_t st,
                   cudaEvent_t ev_begin = nullptr, cudaEvent_t ev_end = nullptr, InputMap im = InputMap{}) {
    if (L && rows > 0 && !Y) return fail(LMKAN_B200_EINVAL, "lmkan_forward: null X or Y");
    return forward_device_dests<XT>(L, X, single_dest<XT>(Y, L ? L->n_out : 0), rows, st, ev_begin, ev_end, im);
}

template <typename XT>
int locate_device(const lmkan_b200_layer* L, const XT* X, int32_t* i1, int32_t* i2, float* w, int64_t rows,
                  cudaStream_t st) {
    if (!L) return fail(LMKAN_B200_EINVAL, "locate: null layer");
    if (rows <= 0) return rows == 0 ? LMKAN_B200_OK : fail(LMKAN_B200_EINVAL, "locate: negative rows");
    if (reinterpret_cast<uintptr_t>(w) % 16 != 0) return fail(LMKAN_B200_EINVAL, "locate: w must be 16-byte aligned");
    DeviceGuard g(L->device);
    const int64_t total = rows * L->pairs;
    const int64_t blocks = std::min<int64_t>((total + 255) / 256, L->num_sms * 16);
    locate_kernel<XT><<<static_cast<unsigned>(blocks), 256, 0, st>>>(X, rows, L->n_in, L->gc, i1, i2,
                                                                     reinterpret_cast<float4*>(w));
    CK(cudaGetLastError());
    return LMKAN_B200_OK;
}

// Production cell records decoded per (row, pair) (lmkan_b200_records_*):
// variant 0/1 = K1 (records4_kernel / records_kernel) of the layer's staged
// plan for `rows`, read back where K2 reads them; 2 = the in-kernel locate of
// the fused / global / narrow gather kernels.
template <typename XT>
int records_device(const lmkan_b200_layer* L, const XT* X, int32_t* i1, int32_t* i2, float* ag, int64_t rows,
                   int variant, cudaStream_t st) {
    if (!L) return fail(LMKAN_B200_EINVAL, "records: null layer");
    if (rows <= 0) return rows == 0 ? LMKAN_B200_OK : fail(LMKAN_B200_EINVAL, "records: negative rows");
    if (!X || !i1 || !i2 || !ag || reinterpret_cast<uintptr_t>(ag) % 8 != 0)
        return fail(LMKAN_B200_EINVAL, "records: null or misaligned output");
    if (variant < 0 || variant > 2) return fail(LMKAN_B200_EINVAL, "records: variant must be 0, 1 or 2");
    if (variant < 2 && L->narrow) return fail(LMKAN_B200_EINVAL, "records: narrow layers have no K1 records");
    if (L->exact) return fail(LMKAN_B200_EINVAL, "records: reference-precision layers keep fp64 records in-kernel");
    DeviceGuard g(L->device);
    const int cap = max_smem_optin(L->device);
    const int64_t total = rows * L->pairs;
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, L->num_sms * 16));
    float2* out_ag = reinterpret_cast<float2*>(ag);
    if (variant == 2) {
        int H = L->G, hs = 0;
        if (!L->narrow) {
            Plan pl;
            if (!make_plan(L, rows, cap, pl, kModeFused) && !make_plan(L, rows, cap, pl, kModeGlobal))
                return fail(LMKAN_B200_EINVAL, "records: no fused plan");
            H = (L->G + pl.S - 1) / pl.S;
            hs = half_swap(L, pl) ? 1 : 0;
        }
        locate_ag_kernel<XT><<<blocks, 256, 0, st>>>(X, rows, L->n_in, L->gc, L->ns, H, hs, i1, i2, out_ag);
        CK(cudaGetLastError());
        return LMKAN_B200_OK;
    }
    Plan pl;
    if (!make_plan(L, rows, cap, pl, kModeStaged)) return fail(LMKAN_B200_EINVAL, "records: no staged plan");
    float2* recW = nullptr;
    int* recO = nullptr;
    CK(cudaMallocAsync(reinterpret_cast<void**>(&recW), static_cast<size_t>(L->pairs) * pl.rows_pad * sizeof(float2), st));
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&recO),
                                    static_cast<size_t>(L->pairs) * pl.row_tiles * pl.sh.OBLK * sizeof(int), st);
    if (e == cudaSuccess) {
        launch_records<XT>(L, pl, X, rows, InputMap{}, recW, recO, variant == 0, st);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) {
        decode_records_kernel<<<blocks, 256, 0, st>>>(recW, recO, rows, pl.rows_pad, L->pairs, pl.sh, pl.row_tile, L->G,
                                                      (L->G + pl.S - 1) / pl.S, i1, i2, out_ag);
        e = cudaGetLastError();
    }
    cudaFreeAsync(recW, st);
    if (recO) cudaFreeAsync(recO, st);
    if (e != cudaSuccess) return cuda_fail(e, "records");
    return LMKAN_B200_OK;
}

int validate_shape(int n_in, int n_out, int G) {
    if (n_in <= 0 || n_in % 2 != 0)
        return fail(LMKAN_B200_EINVAL, "init_layer: n_in must be a positive even number");
    if (n_out <= 0) return fail(LMKAN_B200_EINVAL, "init_layer: n_out must be positive");
    if (G < 3) return fail(LMKAN_B200_EINVAL, "build_grid: G must be >= 3 (ghost rule needs two interior points)");
    if (G > kMaxG) return fail(LMKAN_B200_EINVAL, "build_grid: G > 255 is not supported by the B200 kernels");
    return LMKAN_B200_OK;
}

// Allocates the handle, grid constants and the (uninitialised) device table.
int alloc_layer(int n_in, int n_out_local, int n_out_total, int out_begin, int G, double gamma, int device,
                lmkan_b200_layer** out, bool exact = false) {
    if (!out) return fail(LMKAN_B200_EINVAL, "layer_create: null out pointer");
    *out = nullptr;
    if (int rc = validate_shape(n_in, n_out_total, G)) return rc;
    if (out_begin < 0 || n_out_local <= 0 || out_begin + n_out_local > n_out_total)
        return fail(LMKAN_B200_EINVAL, "layer_create: bad output slice");
    if (int rc = require_sm100(device)) return rc;
    DeviceGuard g(device);
    auto* L = new lmkan_b200_layer();
    L->device = device;
    L->n_in = n_in;
    L->n_out = n_out_local;
    L->n_out_total = n_out_total;
    L->out_begin = out_begin;
    L->G = G;
    L->pairs = n_in / 2;
    L->nodes = (G + 1) * (G + 1);
    L->gamma = gamma;
    {  // planning and grid sizing use the device's SM count (148 on B200)
        int sms = 0;
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) == cudaSuccess && sms > 0)
            L->num_sms = sms;
    }
    const int no = n_out_local <= 1 ? 1 : (n_out_local <= 2 ? 2 : 4);
    if (exact) {
        L->exact = true;
        api::exact_choose(n_out_local, G, max_smem_optin(device), L->OT, L->exact_gsheet);
    } else if (n_out_local <= 4 && env_int("LMKAN_B200_NARROW", 1) &&
        static_cast<int>(narrow_smem_bytes(G, n_in / 2, no)) <= max_smem_optin(device)) {
        L->narrow = true;
        L->OT = no;
    } else {
        L->OT = choose_out_tile(n_out_local, G, max_smem_optin(device));
        L->dup = choose_dup(L->OT, G, max_smem_optin(device));
    }
    L->ns = L->dup ? 2 * L->OT : L->OT;
    L->pair_block = choose_pair_block(L->pairs);
    L->n_ot = (n_out_local + L->OT - 1) / L->OT;
    std::vector<double> pts, inv, t64;
    std::vector<float> t32;
    host::build_grid(G, pts, inv);
    host::thresholds(G, t64, t32);
    GridConst& gc = L->gc;
    gc.G = G;
    gc.L = grid_L(G);
    // one device block holds the grid constants: inv_areas[G*G], t64[L],
    // points[G+1], inv_h[G] (doubles), then t32[L] (floats); thresholds are
    // NaN-padded to L entries (the search's upper padding)
    const size_t nd = static_cast<size_t>(G) * G + gc.L + (G + 1) + G;
    std::vector<double> blk(nd + (gc.L + 1) / 2, 0.0);
    double* hp = blk.data();
    std::copy(inv.begin(), inv.end(), hp);
    double* h64 = hp + static_cast<size_t>(G) * G;
    double* hpts = h64 + gc.L;
    double* hinvh = hpts + G + 1;
    float* h32 = reinterpret_cast<float*>(hinvh + G);
    for (int k = 0; k < gc.L; ++k) {
        h64[k] = k < G - 1 ? t64[k] : std::numeric_limits<double>::quiet_NaN();
        h32[k] = k < G - 1 ? t32[k] : std::numeric_limits<float>::quiet_NaN();
    }
    for (int k = 0; k <= G; ++k) hpts[k] = pts[k];
    for (int k = 0; k < G; ++k) hinvh[k] = 1.0 / (pts[k + 1] - pts[k]);
    L->table_bytes = exact ? 0 : static_cast<size_t>(L->n_ot) * L->pairs * L->nodes * L->ns * sizeof(float);
    L->table64_bytes = exact ? static_cast<size_t>(L->n_ot) * L->pairs * L->nodes * L->OT * sizeof(double) : 0;
    cudaError_t e = cudaMalloc(&L->d_inv, sizeof(double) * blk.size());
    if (e == cudaSuccess)
        e = cudaMemcpy(L->d_inv, blk.data(), sizeof(double) * blk.size(), cudaMemcpyHostToDevice);
    // the allocation is rounded up to 16 B and the tail zeroed: the narrow kernel
    // bulk-copies the whole table, and bulk copies move multiples of 16 B
    const size_t alloc_bytes = (L->table_bytes + 15) & ~static_cast<size_t>(15);
    if (e == cudaSuccess && exact) e = cudaMalloc(&L->table64, L->table64_bytes);
    if (e == cudaSuccess && !exact) e = cudaMalloc(&L->table, alloc_bytes);
    if (e == cudaSuccess && !exact && alloc_bytes > L->table_bytes)
        e = cudaMemset(reinterpret_cast<char*>(L->table) + L->table_bytes, 0, alloc_bytes - L->table_bytes);
    if (e != cudaSuccess) {
        cudaFree(L->d_inv);
        cudaFree(L->table64);
        cudaFree(L->table);
        delete L;
        return cuda_fail(e, "layer_create: device allocation");
    }
    gc.inv_areas = L->d_inv;
    gc.t64 = L->d_inv + static_cast<size_t>(G) * G;
    gc.points = gc.t64 + gc.L;
    gc.inv_h = gc.points + G + 1;
    gc.t32 = reinterpret_cast<const float*>(gc.inv_h + G);
    {  // keep stream-ordered scratch (cell records, host-path staging) in the pool between calls
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
            // no hidden cross-stream waits: with internal-dependency reuse an
            // allocation on one compute stream of the host pipeline may wait on a
            // free enqueued on the other, serialising the two streams
            // (LMKAN_B200_POOL_DEPS=1 restores the default for A/B runs)
            int deps = env_int("LMKAN_B200_POOL_DEPS", 0);
            cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowInternalDependencies, &deps);
        }
    }
    *out = L;
    return LMKAN_B200_OK;
}

// Blocks of 256 threads for the grid-stride preparation kernels (capped at 64
// per SM of a 148-SM B200; the loops cover any size).
unsigned fill_blocks(size_t total) {
    return static_cast<unsigned>(std::min<size_t>((total + 255) / 256, 148 * 64));
}

template <typename T>
int relayout_from_device(lmkan_b200_layer* L, const T* P_dev) {
    const size_t total = L->table_bytes / sizeof(float);
    relayout_kernel<T><<<fill_blocks(total), 256>>>(P_dev, L->table, L->pairs, L->nodes, L->n_out_total,
                                                    L->out_begin, L->n_out, L->OT, L->ns, L->n_ot);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    return LMKAN_B200_OK;
}

// Host-path pipeline state (streams, events, staging) per device, per host thread.
HostPipeline& host_pipeline(int device) {
    static thread_local HostPipeline hp[64];
    return hp[device & 63];
}

template <typename XT>
int forward_host(const lmkan_b200_layer* L, const XT* X, XT* Y, int64_t rows) {
    if (!L) return fail(LMKAN_B200_EINVAL, "lmkan_forward: null layer");
    if (rows < 0) return fail(LMKAN_B200_EINVAL, "lmkan_forward: negative row count");
    if (rows == 0) return LMKAN_B200_OK;
    if (!X || !Y) return fail(LMKAN_B200_EINVAL, "lmkan_forward: null X or Y");
    DeviceGuard g(L->device);
    HostPipeline& P = host_pipeline(L->device);
    CK(P.init(L->device));
    // Chunks flow H2D -> kernels -> D2H on three streams (host_pipeline.hpp).
    Plan pl;
    if (!make_plan(L, rows, max_smem_optin(L->device), pl))
        return fail(LMKAN_B200_EINVAL, "lmkan_forward: no kernel variant fits shared memory");
    // ~8 chunks of at least one wave of row tiles (cfg2: 8 measured best; fewer
    // expose more of the first H2D / last D2H, more shrink the grids below a
    // wave): LMKAN_B200_HOST_CHUNKS overrides
    const int64_t min_chunk = static_cast<int64_t>(pl.sh.R) * L->num_sms / std::max(1, L->n_ot);
    const int64_t nchunks = std::max(1, env_int("LMKAN_B200_HOST_CHUNKS", 8));
    int64_t chunk = std::max<int64_t>({(rows + nchunks - 1) / nchunks, min_chunk, 1});
    chunk = std::min(chunk, rows);
    // fp64 callers: Y crosses PCIe as fp32 (exact: every output is an fp32 sum
    // times an fp32 gamma) and is widened on the host; the slot's device Y holds
    // [fp32 Y | fp64 Y]
    const bool widen = sizeof(XT) == 8 && !L->exact && env_int("LMKAN_B200_HOST_F32_Y", 1) != 0;
    const size_t y32_bytes = (static_cast<size_t>(chunk) * L->n_out * sizeof(float) + 255) & ~static_cast<size_t>(255);
    CK(P.reserve(static_cast<size_t>(chunk) * L->n_in * sizeof(XT),
                 static_cast<size_t>(chunk) * L->n_out * sizeof(XT) + (widen ? y32_bytes : 0)));
    const ChunkSchedule cs(rows, chunk, env_int("LMKAN_B200_HOST_TAPER", 2));  // cfg2 e2e 3.51e6 -> 3.58e6 (2 levels vs none)
    return run_host_pipeline(
        P, cs.count(),
        [&](int64_t c, const void** h, size_t* b) {
            *h = X + cs.first(c) * L->n_in;
            *b = static_cast<size_t>(cs.size(c)) * L->n_in * sizeof(XT);
        },
        [&](int64_t c, void** h, size_t* b) {
            *h = Y + cs.first(c) * L->n_out;
            *b = static_cast<size_t>(cs.size(c)) * L->n_out * sizeof(XT);
        },
        [&](int64_t c, void* dX, void* dY, cudaStream_t st) {
            if (!widen)
                return forward_device<XT>(L, static_cast<const XT*>(dX), static_cast<XT*>(dY), cs.size(c), st);
            XT* y64 = reinterpret_cast<XT*>(static_cast<char*>(dY) + y32_bytes);
            if (int rc = forward_device<XT>(L, static_cast<const XT*>(dX), y64, cs.size(c), st)) return rc;
            const size_t n = static_cast<size_t>(cs.size(c)) * L->n_out;
            narrow_f64_kernel<<<fill_blocks(n), 256, 0, st>>>(reinterpret_cast<const double*>(y64),
                                                              static_cast<float*>(dY), n);
            const cudaError_t e = cudaGetLastError();
            return e == cudaSuccess ? LMKAN_B200_OK : cuda_fail(e, "lmkan_forward: narrow Y");
        },
        [](cudaError_t e, const char* what) { return cuda_fail(e, what); }, widen);
}

}  // namespace

namespace {
// Can layer A's gather epilogue produce layer B's cell records (fused chain)?
// Both full (unsliced) layers, A not narrow, B staged, and neither forward
// needs row chunking at this batch size.
bool chain_fusable(const lmkan_b200_layer* A, const Plan& pa, const lmkan_b200_layer* B, int64_t rows, int cap,
                   Plan& pb) {
    if (A->n_out != A->n_out_total || B->n_out != B->n_out_total || A->n_out != B->n_in) return false;
    if (pa.mode == kModeNarrow || A->device != B->device) return false;
    if (A->pair_block > 0) return false;  // the running sum lives in the (skipped) activation rows
    if (!make_plan(B, rows, cap, pb) || pb.mode != kModeStaged) return false;
    if (half_swap(B, pb)) return false;  // the emitter writes plain (unswapped) records
    if (pa.row_tile != pa.sh.R || pb.row_tile != pb.sh.R) return false;  // the emitter assumes full row tiles
    const lmkan_b200_layer* ls[2] = {A, B};
    const Plan* ps[2] = {&pa, &pb};
    for (int i = 0; i < 2; ++i) {
        if (ps[i]->mode != kModeStaged) continue;
        const size_t per_row = static_cast<size_t>(ls[i]->pairs) * (sizeof(float2) + sizeof(int) * 2);
        if (static_cast<size_t>(rows) * per_row > record_scratch_cap()) return false;
    }
    return true;
}
}  // namespace

namespace lmkan_b200::api {
// model_infer of a fused model (model.hpp:268-315) on one stream: layer b's
// gather epilogue writes layer b+1's cell records whenever chain_fusable, so
// that activation never goes to memory and layer b+1 skips its K1; otherwise
// the activation goes through acts[b & 1] as a plain forward.
int forward_chain_f32(const lmkan_b200_layer* const* layers, int n, const float* X, float* Y, int64_t rows,
                      void* const* acts, cudaStream_t st) {
    if (rows == 0) return LMKAN_B200_OK;
    const int cap = max_smem_optin(layers[0]->device);
    ChainLink pending;
    float2* pendW = nullptr;
    int* pendO = nullptr;
    const float* cur = X;
    int rc = LMKAN_B200_OK;
    for (int b = 0; b < n && rc == LMKAN_B200_OK; ++b) {
        const lmkan_b200_layer* L = layers[b];
        DeviceGuard g(L->device);
        Plan pl;
        if (!make_plan(L, rows, cap, pl))
            return fail(LMKAN_B200_EINVAL, "lmkan_forward: no kernel variant fits shared memory");
        const bool last = b + 1 == n;
        Plan pn;
        const bool fuse = !last && (!pending.preW || pl.mode == kModeStaged) &&
                          chain_fusable(L, pl, layers[b + 1], rows, cap, pn) &&
                          env_int("LMKAN_B200_CHAIN_FUSE", 0) != 0;  // opt-in: measured slower
        // a layer fed records by its predecessor must run its staged K2 on them
        if (pending.preW && pl.mode != kModeStaged)
            return fail(LMKAN_B200_EINVAL, "forward_chain: internal plan mismatch");
        float* dst = last ? Y : static_cast<float*>(acts[b & 1]);
        OutDests<float> out = single_dest<float>(dst, L->n_out);
        ChainLink link = pending;
        float2* emW = nullptr;
        int* emO = nullptr;
        if (fuse) {
            const lmkan_b200_layer* N = layers[b + 1];
            const size_t wbytes = static_cast<size_t>(N->pairs) * pn.rows_pad * sizeof(float2);
            const size_t obytes = static_cast<size_t>(N->pairs) * pn.row_tiles * pn.sh.OBLK * sizeof(int);
            cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&emW), wbytes, st);
            if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&emO), obytes, st);
            // rows in [rows, rows_pad) carry zero records (as K1 writes them); the last
            // row tile's offset block is zeroed whole, the epilogue fills its valid rows
            if (e == cudaSuccess && pn.rows_pad > rows)
                e = cudaMemset2DAsync(emW + rows, pn.rows_pad * sizeof(float2), 0,
                                      (pn.rows_pad - rows) * sizeof(float2), N->pairs, st);
            if (e == cudaSuccess)
                e = cudaMemset2DAsync(emO + (pn.row_tiles - 1) * pn.sh.OBLK, pn.row_tiles * pn.sh.OBLK * sizeof(int), 0,
                                      pn.sh.OBLK * sizeof(int), N->pairs, st);
            if (e != cudaSuccess) {
                rc = cuda_fail(e, "forward_chain: record buffers");
                break;
            }
            link.emit = EmitRecords{emW, emO, pn.sh, pn.rows_pad, pn.row_tiles, (N->G + pn.S - 1) / pn.S};
            pl.smem = std::max<uint32_t>(pl.smem, emit_smem_bytes(pl.OT, pl.sh.R));  // staging for the record stores
            link.gc_next = &N->gc;
            out.n = 0;  // the activation lives on only as the next layer's records
        }
        rc = forward_rows<float>(L, pl, cur, out, rows, InputMap{}, st, nullptr, nullptr, link);
        if (pendW) cudaFreeAsync(pendW, st);
        if (pendO) cudaFreeAsync(pendO, st);
        pendW = emW;
        pendO = emO;
        pending = ChainLink{};
        if (fuse) {
            pending.preW = emW;
            pending.preO = emO;
            cur = nullptr;  // a staged K2 reads only its records
        } else {
            cur = dst;
        }
    }
    if (pendW) cudaFreeAsync(pendW, st);
    if (pendO) cudaFreeAsync(pendO, st);
    return rc;
}

int set_error(int code, const std::string& msg) { return fail(code, msg); }
int cuda_error(cudaError_t e, const char* what) { return cuda_fail(e, what); }
int alloc_layer(int n_in, int n_out_local, int n_out_total, int out_begin, int G, double gamma, int device,
                lmkan_b200_layer** out) {
    return ::alloc_layer(n_in, n_out_local, n_out_total, out_begin, G, gamma, device, out);
}
int forward_device(const lmkan_b200_layer* L, const float* X, float* Y, int64_t rows, cudaStream_t st) {
    return ::forward_device<float>(L, X, Y, rows, st);
}
int forward_device(const lmkan_b200_layer* L, const double* X, double* Y, int64_t rows, cudaStream_t st) {
    return ::forward_device<double>(L, X, Y, rows, st);
}
}  // namespace lmkan_b200::api

// =================================================================== C-ABI
extern "C" {

const char* lmkan_b200_last_error(void) { return g_err.c_str(); }

const char* lmkan_b200_version(void) { return "lmkan_b200 0.1 (sm_100a, fused locate+gather, bulk-copy sheets)"; }

int lmkan_b200_build_grid(int G, double* points, double* inv_areas) {
    std::vector<double> p, inv;
    if (!host::build_grid(G, p, inv))
        return fail(LMKAN_B200_EINVAL, "build_grid: G must be >= 3 (ghost rule needs two interior points)");
    if (points) std::memcpy(points, p.data(), sizeof(double) * p.size());
    if (inv_areas) std::memcpy(inv_areas, inv.data(), sizeof(double) * inv.size());
    return LMKAN_B200_OK;
}

int lmkan_b200_thresholds(int G, double* t64, float* t32) {
    std::vector<double> a;
    std::vector<float> b;
    if (!host::thresholds(G, a, b))
        return fail(LMKAN_B200_EINVAL, "build_grid: G must be >= 3 (ghost rule needs two interior points)");
    if (t64) std::memcpy(t64, a.data(), sizeof(double) * a.size());
    if (t32) std::memcpy(t32, b.data(), sizeof(float) * b.size());
    return LMKAN_B200_OK;
}

int lmkan_b200_init_table(int n_in, int n_out, int G, uint64_t seed, double init_scale, double* P_out) {
    if (n_in <= 0 || n_in % 2 != 0)
        return fail(LMKAN_B200_EINVAL, "init_layer: n_in must be a positive even number");
    if (n_out <= 0) return fail(LMKAN_B200_EINVAL, "init_layer: n_out must be positive");
    if (G < 3) return fail(LMKAN_B200_EINVAL, "build_grid: G must be >= 3 (ghost rule needs two interior points)");
    if (!P_out) return fail(LMKAN_B200_EINVAL, "init_layer: null output");
    if (init_scale < 0.0) init_scale = 1.0 / std::sqrt(static_cast<double>(n_in / 2));
    const size_t count = static_cast<size_t>(G + 1) * (G + 1) * (n_in / 2) * n_out;
    host::NamedStream rs(seed, "lmkan.layer.init");
    for (size_t i = 0; i < count; ++i) P_out[i] = init_scale * rs.normal();
    return LMKAN_B200_OK;
}

int lmkan_b200_layer_create(int n_in, int n_out, int G, double gamma, const double* P_host, int device,
                            lmkan_b200_layer** out) {
    if (!P_host) return fail(LMKAN_B200_EINVAL, "layer_create: null P");
    if (int rc = alloc_layer(n_in, n_out, n_out, 0, G, gamma, device, out)) return rc;
    lmkan_b200_layer* L = *out;
    DeviceGuard g(device);
    const size_t count = static_cast<size_t>(L->nodes) * L->pairs * n_out;
    double* tmp = nullptr;
    cudaError_t e = cudaMalloc(&tmp, count * sizeof(double));
    if (e == cudaSuccess) e = cudaMemcpy(tmp, P_host, count * sizeof(double), cudaMemcpyHostToDevice);
    int rc = e == cudaSuccess ? relayout_from_device<double>(L, tmp) : cuda_fail(e, "layer_create: upload P");
    cudaFree(tmp);
    if (rc) {
        lmkan_b200_layer_destroy(L);
        *out = nullptr;
    }
    return rc;
}

int lmkan_b200_layer_create_exact(int n_in, int n_out, int G, double gamma, const double* P_host, int device,
                                  lmkan_b200_layer** out) {
    if (!P_host) return fail(LMKAN_B200_EINVAL, "layer_create: null P");
    if (int rc = alloc_layer(n_in, n_out, n_out, 0, G, gamma, device, out, true)) return rc;
    DeviceGuard g(device);
    const int rc = api::exact_upload(*out, P_host);
    if (rc) {
        lmkan_b200_layer_destroy(*out);
        *out = nullptr;
    }
    return rc;
}

int lmkan_b200_layer_create_device_f32_slice(int n_in, int n_out, int G, double gamma, const float* P_dev,
                                             int out_begin, int out_end, int device, lmkan_b200_layer** out) {
    if (!P_dev) return fail(LMKAN_B200_EINVAL, "layer_create: null P");
    if (int rc = alloc_layer(n_in, out_end - out_begin, n_out, out_begin, G, gamma, device, out)) return rc;
    DeviceGuard g(device);
    int rc = relayout_from_device<float>(*out, P_dev);
    if (rc) {
        lmkan_b200_layer_destroy(*out);
        *out = nullptr;
    }
    return rc;
}

int lmkan_b200_layer_create_device_f32(int n_in, int n_out, int G, double gamma, const float* P_dev, int device,
                                       lmkan_b200_layer** out) {
    return lmkan_b200_layer_create_device_f32_slice(n_in, n_out, G, gamma, P_dev, 0, n_out, device, out);
}

int lmkan_b200_layer_create_random(int n_in, int n_out, int G, double gamma, uint64_t seed, double scale,
                                   int out_begin, int out_end, int device, lmkan_b200_layer** out) {
    if (int rc = alloc_layer(n_in, out_end - out_begin, n_out, out_begin, G, gamma, device, out)) return rc;
    lmkan_b200_layer* L = *out;
    DeviceGuard g(device);
    const size_t total = L->table_bytes / sizeof(float);
    fill_random_kernel<<<fill_blocks(total), 256>>>(L->table, L->pairs, L->nodes, L->n_out_total, L->out_begin,
                                                    L->n_out, L->OT, L->ns, L->n_ot, seed, static_cast<float>(scale));
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        lmkan_b200_layer_destroy(L);
        *out = nullptr;
        return cuda_fail(e, "layer_create_random: fill");
    }
    return LMKAN_B200_OK;
}

int lmkan_b200_layer_read_table(const lmkan_b200_layer* L, int pair_begin, int pair_end, double* dst) {
    if (!L || !dst) return fail(LMKAN_B200_EINVAL, "read_table: null argument");
    if (pair_begin < 0 || pair_end > L->pairs || pair_begin >= pair_end)
        return fail(LMKAN_B200_EINVAL, "read_table: bad pair range");
    DeviceGuard g(L->device);
    if (L->exact) return api::exact_read_table(L, pair_begin, pair_end, dst);
    const size_t count = static_cast<size_t>(L->nodes) * (pair_end - pair_begin) * L->n_out;
    double* tmp = nullptr;
    CK(cudaMalloc(&tmp, count * sizeof(double)));
    export_kernel<<<fill_blocks(count), 256>>>(L->table, tmp, L->pairs, L->nodes, L->n_out, L->OT, L->ns, pair_begin,
                                               pair_end);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpy(dst, tmp, count * sizeof(double), cudaMemcpyDeviceToHost);
    cudaFree(tmp);
    if (e != cudaSuccess) return cuda_fail(e, "read_table");
    return LMKAN_B200_OK;
}

int lmkan_b200_layer_set_gamma(lmkan_b200_layer* L, double gamma) {
    if (!L) return fail(LMKAN_B200_EINVAL, "set_gamma: null layer");
    if (L->gamma != gamma) ++L->version;
    L->gamma = gamma;
    return LMKAN_B200_OK;
}

int lmkan_b200_layer_info(const lmkan_b200_layer* L, int* n_in, int* n_out, int* G, int* device,
                          size_t* table_bytes, int* out_tile) {
    if (!L) return fail(LMKAN_B200_EINVAL, "layer_info: null layer");
    if (n_in) *n_in = L->n_in;
    if (n_out) *n_out = L->n_out;
    if (G) *G = L->G;
    if (device) *device = L->device;
    if (table_bytes) *table_bytes = L->table_bytes;
    if (out_tile) *out_tile = L->OT;
    return LMKAN_B200_OK;
}

int lmkan_b200_layer_destroy(lmkan_b200_layer* L) {
    if (!L) return LMKAN_B200_OK;
    {
        DeviceGuard g(L->device);
        cudaFree(L->table);
        cudaFree(L->table64);
        cudaFree(L->d_inv);
    }
    delete L;
    return LMKAN_B200_OK;
}

int lmkan_b200_forward_f32(const lmkan_b200_layer* L, const float* X, float* Y, int64_t rows, void* stream) {
    return forward_device<float>(L, X, Y, rows, static_cast<cudaStream_t>(stream));
}
int lmkan_b200_forward_f32_timed(const lmkan_b200_layer* L, const float* X, float* Y, int64_t rows, void* stream,
                                 void* ev_begin, void* ev_end) {
    return forward_device<float>(L, X, Y, rows, static_cast<cudaStream_t>(stream), static_cast<cudaEvent_t>(ev_begin),
                                 static_cast<cudaEvent_t>(ev_end));
}
namespace {
// argument checks of unfold_conv (conv.hpp:40-45), then the layer width check
// (layer.hpp:110); fills the implicit-im2col input map.
int conv_map(const lmkan_b200_layer* L, int N, int H, int W, int C, int k, int s, InputMap& im) {
    if (!L) return fail(LMKAN_B200_EINVAL, "conv_forward: null layer");
    if (k < 1 || s < 1) return fail(LMKAN_B200_EINVAL, "unfold_conv: k and s must be positive");
    if (k > H || k > W) return fail(LMKAN_B200_EINVAL, "unfold_conv: kernel larger than image");
    if ((H - k) % s != 0 || (W - k) % s != 0)
        return fail(LMKAN_B200_EINVAL, "unfold_conv: (H-k) and (W-k) must be divisible by the stride");
    if (N < 0 || C < 1) return fail(LMKAN_B200_EINVAL, "conv_forward: bad image batch shape");
    if (static_cast<int64_t>(k) * k * C != L->n_in)
        return fail(LMKAN_B200_EINVAL, "lmkan_forward: expected width " + std::to_string(L->n_in) + ", got " +
                                           std::to_string(static_cast<int64_t>(k) * k * C));
    im = InputMap{};
    im.conv = 1;
    im.out_h = (H - k) / s + 1;
    im.out_w = (W - k) / s + 1;
    im.H = H;
    im.W = W;
    im.C = C;
    im.k = k;
    im.s = s;
    im.npix = static_cast<int64_t>(N) * H * W;
    return LMKAN_B200_OK;
}
}  // namespace

// Synchronous host conv: image chunks through the three-stream host pipeline
// (H2D, kernels and D2H of different chunks overlap; host_pipeline.hpp).
int lmkan_b200_conv_forward_host_f32(const lmkan_b200_layer* L, const float* img, int N, int H, int W, int C, int k,
                                     int s, float* Y, size_t /*workers*/) {
    InputMap im;
    if (int rc = conv_map(L, N, H, W, C, k, s, im)) return rc;
    if (N == 0) return LMKAN_B200_OK;
    if (!img || !Y) return fail(LMKAN_B200_EINVAL, "conv_forward: null image or output");
    DeviceGuard g(L->device);
    HostPipeline& P = host_pipeline(L->device);
    CK(P.init(L->device));
    const int64_t per_img = static_cast<int64_t>(im.out_h) * im.out_w;
    Plan pl;
    if (!make_plan(L, per_img * N, max_smem_optin(L->device), pl))
        return fail(LMKAN_B200_EINVAL, "lmkan_forward: no kernel variant fits shared memory");
    // chunks of at least one wave of 512-row tiles (a full-batch plan's taller
    // tile would otherwise make a single chunk), else ~8 chunks
    const int64_t wave_rows = static_cast<int64_t>(env_int("LMKAN_B200_CONV_CHUNK_ROWS", 512)) * L->num_sms /
                              std::max(1, L->n_ot);
    const int64_t min_imgs = (wave_rows + per_img - 1) / per_img;
    const int chunk = static_cast<int>(std::min<int64_t>(N, std::max<int64_t>({(N + 7) / 8, min_imgs, 1})));
    const size_t in_img = static_cast<size_t>(H) * W * C, out_img = static_cast<size_t>(per_img) * L->n_out;
    CK(P.reserve(sizeof(float) * in_img * chunk, sizeof(float) * out_img * chunk));
    const ChunkSchedule cs(N, chunk, env_int("LMKAN_B200_HOST_TAPER", 0));  // cfg4 e2e: tapering cost 15%
    return run_host_pipeline(
        P, cs.count(),
        [&](int64_t c, const void** h, size_t* b) {
            *h = img + cs.first(c) * in_img;
            *b = sizeof(float) * in_img * cs.size(c);
        },
        [&](int64_t c, void** h, size_t* b) {
            *h = Y + cs.first(c) * out_img;
            *b = sizeof(float) * out_img * cs.size(c);
        },
        [&](int64_t c, void* dI, void* dY, cudaStream_t st) {
            InputMap imc = im;
            imc.npix = static_cast<int64_t>(cs.size(c)) * H * W;  // the chunk's images only
            return forward_device<float>(L, static_cast<const float*>(dI), static_cast<float*>(dY),
                                         per_img * cs.size(c), st, nullptr, nullptr, imc);
        },
        [](cudaError_t e, const char* what) { return cuda_fail(e, what); });
}

int lmkan_b200_conv_plan(const lmkan_b200_layer* L, int N, int H, int W, int C, int k, int s, int* nbuf,
                         int* rows_per_cta, int* pixel_records) {
    InputMap im;
    if (int rc = conv_map(L, N, H, W, C, k, s, im)) return rc;
    Plan pl;
    const int64_t rows = static_cast<int64_t>(N) * im.out_h * im.out_w;
    if (!make_plan(L, std::max<int64_t>(rows, 1), max_smem_optin(L->device), pl))
        return fail(LMKAN_B200_EINVAL, "conv_plan: no kernel variant fits shared memory");
    const bool pix = pixel_eligible(pl, im);
    if (pix) pixel_ring_cap(L, im, pl);
    if (nbuf) *nbuf = pl.nbuf;
    if (rows_per_cta) *rows_per_cta = static_cast<int>(pl.row_tile > 0 ? pl.row_tile : pl.sh.R);
    if (pixel_records) *pixel_records = pix ? 1 : 0;
    return LMKAN_B200_OK;
}

int lmkan_b200_conv_forward_f32(const lmkan_b200_layer* L, const float* img, int N, int H, int W, int C, int k,
                                int s, float* Y, void* stream) {
    InputMap im;
    if (int rc = conv_map(L, N, H, W, C, k, s, im)) return rc;
    const int64_t rows = static_cast<int64_t>(N) * im.out_h * im.out_w;
    return forward_device<float>(L, img, Y, rows, static_cast<cudaStream_t>(stream), nullptr, nullptr, im);
}
int lmkan_b200_forward_f32_dests(const lmkan_b200_layer* L, const float* X, float* const* dests, int n_dest,
                                 int64_t ld, int col0, int64_t rows, void* stream) {
    if (!dests || n_dest < 1 || n_dest > kMaxDest)
        return fail(LMKAN_B200_EINVAL, "forward_dests: 1 to 8 destinations required");
    OutDests<float> out{};
    for (int d = 0; d < n_dest; ++d) out.base[d] = dests[d];
    out.n = n_dest;
    out.ld = ld;
    out.col0 = col0;
    return forward_device_dests<float>(L, X, out, rows, static_cast<cudaStream_t>(stream));
}
int lmkan_b200_ipc_get_handle(const void* dev_ptr, void* handle_out, uint64_t* offset_out) {
    if (!dev_ptr || !handle_out || !offset_out) return fail(LMKAN_B200_EINVAL, "ipc_get_handle: null argument");
    // the handle names the whole allocation (e.g. a caching-allocator segment):
    // report the pointer's offset inside it (cuMemGetAddressRange via the
    // runtime's driver entry point, no libcuda link)
    using AddrRange = int (*)(unsigned long long*, size_t*, unsigned long long);
    static AddrRange range = nullptr;
    if (!range) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
            return fail(LMKAN_B200_ECUDA, "ipc_get_handle: cuMemGetAddressRange unavailable");
        range = reinterpret_cast<AddrRange>(fn);
    }
    unsigned long long base = 0;
    size_t size = 0;
    if (range(&base, &size, reinterpret_cast<unsigned long long>(dev_ptr)) != 0)
        return fail(LMKAN_B200_ECUDA, "ipc_get_handle: pointer is not a device allocation");
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
    std::memcpy(handle_out, &h, sizeof(h));
    *offset_out = reinterpret_cast<unsigned long long>(dev_ptr) - base;
    return LMKAN_B200_OK;
}
namespace {
std::mutex g_ipc_mu;
std::vector<std::pair<void*, void*>> g_ipc_open;  // (returned pointer, mapped base)
}  // namespace
int lmkan_b200_ipc_open_handle(const void* handle, uint64_t offset, int device, void** dev_ptr) {
    if (!handle || !dev_ptr) return fail(LMKAN_B200_EINVAL, "ipc_open_handle: null argument");
    DeviceGuard g(device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    void* base = nullptr;
    CK(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    *dev_ptr = static_cast<char*>(base) + offset;
    std::lock_guard<std::mutex> lock(g_ipc_mu);
    g_ipc_open.emplace_back(*dev_ptr, base);
    return LMKAN_B200_OK;
}
int lmkan_b200_ipc_close(void* dev_ptr) {
    if (!dev_ptr) return LMKAN_B200_OK;
    void* base = nullptr;
    {
        std::lock_guard<std::mutex> lock(g_ipc_mu);
        for (auto it = g_ipc_open.begin(); it != g_ipc_open.end(); ++it)
            if (it->first == dev_ptr) {
                base = it->second;
                g_ipc_open.erase(it);
                break;
            }
    }
    if (!base) return fail(LMKAN_B200_EINVAL, "ipc_close: pointer was not opened by ipc_open_handle");
    CK(cudaIpcCloseMemHandle(base));
    return LMKAN_B200_OK;
}
int lmkan_b200_forward_f64(const lmkan_b200_layer* L, const double* X, double* Y, int64_t rows, void* stream) {
    return forward_device<double>(L, X, Y, rows, static_cast<cudaStream_t>(stream));
}
int lmkan_b200_forward_host_f64(const lmkan_b200_layer* L, const double* X, double* Y, int64_t rows,
                                size_t /*workers*/) {
    return forward_host<double>(L, X, Y, rows);
}
int lmkan_b200_forward_host_f32(const lmkan_b200_layer* L, const float* X, float* Y, int64_t rows,
                                size_t /*workers*/) {
    return forward_host<float>(L, X, Y, rows);
}
int lmkan_b200_locate_f32(const lmkan_b200_layer* L, const float* X, int32_t* i1, int32_t* i2, float* w,
                          int64_t rows, void* stream) {
    return locate_device<float>(L, X, i1, i2, w, rows, static_cast<cudaStream_t>(stream));
}
int lmkan_b200_locate_f64(const lmkan_b200_layer* L, const double* X, int32_t* i1, int32_t* i2, float* w,
                          int64_t rows, void* stream) {
    return locate_device<double>(L, X, i1, i2, w, rows, static_cast<cudaStream_t>(stream));
}

int lmkan_b200_records_f32(const lmkan_b200_layer* L, const float* X, int32_t* i1, int32_t* i2, float* ag,
                           int64_t rows, int variant, void* stream) {
    return records_device<float>(L, X, i1, i2, ag, rows, variant, static_cast<cudaStream_t>(stream));
}
int lmkan_b200_records_f64(const lmkan_b200_layer* L, const double* X, int32_t* i1, int32_t* i2, float* ag,
                           int64_t rows, int variant, void* stream) {
    return records_device<double>(L, X, i1, i2, ag, rows, variant, static_cast<cudaStream_t>(stream));
}

int lmkan_b200_lane_vectors(int out_tile) { return lane_vectors(out_tile); }
int lmkan_b200_layer_lane_vectors(const lmkan_b200_layer* L) {
    if (!L) return fail(LMKAN_B200_EINVAL, "lane_vectors: null layer"), 0;
    return L->narrow || L->exact ? 1 : lane_vectors(L->OT, L->ns);
}

int lmkan_b200_plan_cta_group(const lmkan_b200_layer* L, int64_t rows) {
    if (!L) return fail(LMKAN_B200_EINVAL, "plan_cta_group: null layer"), 0;
    if (L->exact || L->narrow) return 1;
    Plan pl;
    if (!make_plan(L, rows, max_smem_optin(L->device), pl)) return fail(LMKAN_B200_EINVAL, "plan: no variant fits"), 0;
    return pl.cta_group;
}

int lmkan_b200_plan(const lmkan_b200_layer* L, int64_t rows, int* out_tile, int* rows_per_thread, int* nbuf,
                    int* rows_per_cta_out, int* launches, int* mode, int* slabs, int* warps_per_cta) {
    if (!L) return fail(LMKAN_B200_EINVAL, "plan: null layer");
    if (L->exact) {  // mode 4: the reference-precision kernel (one launch, 16 warps per CTA)
        const int nrun = L->OT >= 16 ? 2 : 1, lpr = L->OT / (2 * nrun), rt = 16 / nrun;  // exact.cu's geometry
        if (out_tile) *out_tile = L->OT;
        if (rows_per_thread) *rows_per_thread = rt;
        if (nbuf) *nbuf = L->exact_gsheet ? 0 : 2;
        if (rows_per_cta_out) *rows_per_cta_out = 16 * (32 / lpr) * rt;
        if (launches) *launches = 1;
        if (mode) *mode = 4;
        if (slabs) *slabs = 1;
        if (warps_per_cta) *warps_per_cta = 16;
        return LMKAN_B200_OK;
    }
    Plan pl;
    if (!make_plan(L, rows, max_smem_optin(L->device), pl)) return fail(LMKAN_B200_EINVAL, "plan: no variant fits");
    if (out_tile) *out_tile = pl.OT;
    if (rows_per_thread) *rows_per_thread = pl.RT;
    if (nbuf) *nbuf = pl.nbuf;
    if (rows_per_cta_out) *rows_per_cta_out = static_cast<int>(pl.row_tile > 0 ? pl.row_tile : pl.sh.R);
    if (launches) *launches = pl.launches;
    if (mode) *mode = pl.mode;
    if (slabs) *slabs = pl.S;
    if (warps_per_cta) *warps_per_cta = pl.mode == kModeNarrow ? kNarrowThreads / 32 : pl.sh.NW;
    return LMKAN_B200_OK;
}

}  // extern "C"
