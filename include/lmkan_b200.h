/*
 * lmkan_b200.h — C-ABI of the B200-native (sm_100a) lmKAN layer forward.
 *
 * This is the drop-in boundary for the reference's layer-forward path. The
 * reference has no FFI: its interface is the inline C++ function
 *     void lmkan::lmkan_forward(const LmKanLayer&, const Matrix& X, Matrix& Y,
 *                               std::size_t workers = 0)          (layer.hpp:108-109)
 * over the types LmKanLayer (layer.hpp:24-61), SigmaGrid / build_grid
 * (grid.hpp:33-68) and Matrix (matrix.hpp:11-38). The C++ host API in
 * include/lmkan_b200/lmkan.hpp restates that interface on top of the entry
 * points below; a foreign-language binding (ctypes) binds
 * these symbols directly. Plain pointers and sizes only.
 *
 * Paths are relative to /root/reference/proj/include/lmkan/.
 *
 * Status codes: every entry point returns 0 on success, else one of
 * LMKAN_B200_E*; lmkan_b200_last_error() gives a thread-local message. The C++
 * wrapper maps EINVAL to std::invalid_argument with the reference message
 * format ("lmkan_forward: expected width N, got M", matrix.hpp:40-44) and the
 * rest to std::runtime_error.
 */
#ifndef LMKAN_B200_H
#define LMKAN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LMKAN_B200_OK 0
#define LMKAN_B200_EINVAL 1  /* maps to std::invalid_argument (matrix.hpp:40-44, layer.hpp:71-73, grid.hpp:45-46) */
#define LMKAN_B200_ECUDA 2   /* CUDA runtime / launch failure */
#define LMKAN_B200_ENOMEM 3  /* device or pinned-host allocation failed */
#define LMKAN_B200_ENOSYS 4  /* no sm_100a device / kernel image */
#define LMKAN_B200_EFORMAT 5 /* malformed / truncated LMK1 file: lmkan::FormatError (errors.hpp:23-26) */
#define LMKAN_B200_EUNSUPPORTED 6 /* valid LMK1 model with blocks outside the B200 path (mlp, bn, preconditioned) */

typedef struct lmkan_b200_layer lmkan_b200_layer; /* opaque prepared device layer */
typedef struct lmkan_b200_model lmkan_b200_model; /* opaque chain of device layers (a fused model) */

/* Thread-local message for the last failing call on this thread. */
const char* lmkan_b200_last_error(void);
/* Library build string (kernel arch, version). */
const char* lmkan_b200_version(void);

/* ---- grid (host-side, once per layer) ---- */

/* build_grid (grid.hpp:44-68): points[G+1] with ghost points, inv_areas[G*G].
 * EINVAL when G < 3. */
int lmkan_b200_build_grid(int G, double* points, double* inv_areas);

/* Cell-locate threshold tables derived from interval_index (grid.hpp:72-75):
 * t64[k-1] = min{double x : interval_index(x) >= k}, k = 1..G-1, and t32[k-1]
 * the smallest float >= t64[k-1]. Then interval_index(x) == #{k : x >= t[k]}
 * for every input, including +-0, +-inf and NaN (-> 0). Either pointer may be
 * NULL. */
int lmkan_b200_thresholds(int G, double* t64, float* t32);

/* init_layer's coefficient table (layer.hpp:69-86): P_out[i] = init_scale *
 * N(0,1) drawn in reference index order from RandomStream(seed,
 * "lmkan.layer.init") (rng.hpp:19-79: FNV-1a + splitmix64 keyed mt19937_64,
 * Box-Muller with one cached value). init_scale < 0 selects (n_in/2)^(-1/2)
 * (layer.hpp:63-65). Host-only; bit-identical to the reference on the same
 * libstdc++/glibc. P_out holds (G+1)^2 * (n_in/2) * n_out doubles. */
int lmkan_b200_init_table(int n_in, int n_out, int G, uint64_t seed, double init_scale, double* P_out);

/* ---- prepared layer handle ---- */

/* Replaces constructing/owning an LmKanLayer (layer.hpp:24-61) for the device:
 * P_host is the reference table, index order [i1][i2][pair][out] with out
 * fastest (layer.hpp:20-22, 34-45), (G+1)^2 * (n_in/2) * n_out doubles. It is
 * rounded to fp32 once and re-laid out on `device` as [out_tile][pair][node][OT]
 * (node = i1*(G+1)+i2). gamma is the lookup-branch weight (layer.hpp:29).
 * EINVAL if n_in is not a positive even number, n_out <= 0 or G < 3. */
int lmkan_b200_layer_create(int n_in, int n_out, int G, double gamma, const double* P_host,
                            int device, lmkan_b200_layer** out);
/* Reference-precision layer: the fp64 table, fp64 weights and fp64
 * accumulation in the reference's operation order with every operation
 * explicitly rounded (no FMA contraction), so lmkan_forward's Y is
 * BIT-IDENTICAL to the reference's (layer.hpp:108-134), for any G >= 3 that
 * the kernels take (<= 255). The forward entry points (device f32/f64,
 * host f32/f64) and lmkan_b200_layer_read_table accept it; the multi-dest,
 * conv and model-chain paths return EINVAL. About 2x the shared-memory
 * traffic of the fp32 gather per coefficient. */
int lmkan_b200_layer_create_exact(int n_in, int n_out, int G, double gamma, const double* P_host, int device,
                                  lmkan_b200_layer** out);
/* Same, from an fp32 table in reference layout already resident on `device`
 * (e.g. generated there); the relayout runs on the device. */
int lmkan_b200_layer_create_device_f32(int n_in, int n_out, int G, double gamma,
                                       const float* P_dev, int device, lmkan_b200_layer** out);
/* Output-sliced layer: keeps only outputs [out_begin, out_end) of the table
 * (exact, since y_q depends only on column q of P, layer.hpp:128-129). Used to
 * shard very wide layers over GPUs. P_dev is the FULL reference-layout table. */
int lmkan_b200_layer_create_device_f32_slice(int n_in, int n_out, int G, double gamma,
                                             const float* P_dev, int out_begin, int out_end,
                                             int device, lmkan_b200_layer** out);
/* Table generated on the device by a counter-based hash normal RNG:
 * P[i1][i2][pair][out] = scale * N(0,1)(seed, flat reference index), written
 * straight into the device layout (no host table, no 2x relayout memory). */
int lmkan_b200_layer_create_random(int n_in, int n_out, int G, double gamma, uint64_t seed,
                                   double scale, int out_begin, int out_end, int device,
                                   lmkan_b200_layer** out);
/* Copy the fp32 device table back in reference layout for pairs
 * [pair_begin, pair_end) and the layer's local outputs [0, n_out_local):
 * dst[node][pair - pair_begin][out] as doubles (for oracle checks). */
int lmkan_b200_layer_read_table(const lmkan_b200_layer* layer, int pair_begin, int pair_end,
                                double* dst);
int lmkan_b200_layer_set_gamma(lmkan_b200_layer* layer, double gamma);
/* Shape query: any pointer may be NULL. n_out is the layer's local width. */
int lmkan_b200_layer_info(const lmkan_b200_layer* layer, int* n_in, int* n_out, int* G,
                          int* device, size_t* table_bytes, int* out_tile);
int lmkan_b200_layer_destroy(lmkan_b200_layer* layer);

/* ---- forward ---- */

/* Device path (asynchronous on `stream`, a cudaStream_t or NULL for the
 * legacy default stream). X_dev: [rows][n_in] fp32 row-major, Y_dev:
 * [rows][n_out] fp32 row-major (layer-local n_out). Same semantics as
 * lmkan_forward (layer.hpp:108-134): y_q = gamma * sum_p f_qp(x_2p, x_2p+1),
 * cell indices bit-exact, fp32 accumulation in the reference pair order. */
int lmkan_b200_forward_f32(const lmkan_b200_layer* layer, const float* X_dev, float* Y_dev,
                           int64_t rows, void* stream);
/* Profiling variant of lmkan_b200_forward_f32: additionally records the
 * caller's CUDA events (cudaEvent_t, either may be NULL) on `stream` right
 * before and right after the gather kernel, so the dominant kernel can be
 * timed alone (bench.py's roofline). */
int lmkan_b200_forward_f32_timed(const lmkan_b200_layer* layer, const float* X_dev, float* Y_dev,
                                 int64_t rows, void* stream, void* ev_gather_begin,
                                 void* ev_gather_end);
/* Same, with fp64 inputs/outputs on the device (cells located in fp64 against
 * the fp64 thresholds, so indices stay bit-exact for any double X). */
int lmkan_b200_forward_f64(const lmkan_b200_layer* layer, const double* X_dev, double* Y_dev,
                           int64_t rows, void* stream);
/* Implicit-im2col convolution (the caller-side chain unfold_conv ->
 * lmkan_forward -> fold_output, conv.hpp:39-71 + layer.hpp:108-134, in one
 * device call): img_dev is an NHWC fp32 batch [N][H][W][C], taps k x k with
 * stride s, and the layer's n_in must equal k*k*C (columns ordered
 * (dy*k + dx)*C + ch as in unfold_conv). Patch rows are formed on the fly from
 * the image (no patch matrix); Y_dev is [N][out_h][out_w][n_out] NHWC, i.e.
 * fold_output's layout, out_h = (H-k)/s + 1. Same EINVAL conditions and
 * messages as unfold_conv. */
int lmkan_b200_conv_forward_f32(const lmkan_b200_layer* layer, const float* img_dev, int N, int H,
                                int W, int C, int k, int s, float* Y_dev, void* stream);
/* The same conv with host img / Y (synchronous): image chunks alternate over
 * two internal streams so the copies overlap the kernels. */
int lmkan_b200_conv_forward_host_f32(const lmkan_b200_layer* layer, const float* img, int N, int H, int W,
                                     int C, int k, int s, float* Y, size_t workers);
/* ---- output-sharded layers: the all-gather fused into the epilogue ----
 *
 * Forward writing the layer's (local) output columns into n_dest (1..8)
 * row-major fp32 buffers dests[d][r * ld + col0 + q]: on a GPU of an
 * output-sharded layer the destinations are the
 * full-width Y of every rank — its own and the peers', mapped over NVLink with
 * lmkan_b200_ipc_open_handle — so each CTA's tile reaches every GPU as NVLink
 * stores while the other CTAs are still gathering (no separate collective).
 * col0 = the shard's first column, ld = the full width. */
int lmkan_b200_forward_f32_dests(const lmkan_b200_layer* layer, const float* X_dev, float* const* dests,
                                 int n_dest, int64_t ld, int col0, int64_t rows, void* stream);
/* CUDA IPC plumbing for the peer destinations: the 64-byte handle
 * (cudaIpcMemHandle_t) of the allocation containing dev_ptr plus dev_ptr's
 * offset inside it (a caching allocator hands out pieces of larger segments);
 * opened in another process on `device` (peer access enabled lazily) as
 * base + offset; closed with the pointer open returned. */
int lmkan_b200_ipc_get_handle(const void* dev_ptr, void* handle_out, uint64_t* offset_out);
int lmkan_b200_ipc_open_handle(const void* handle, uint64_t offset, int device, void** dev_ptr);
int lmkan_b200_ipc_close(void* dev_ptr);
/* Device-side barrier on a stream: rank `rank` of `world` (<= 8) stores
 * `epoch` (> 0, increasing) into slot `rank` of every rank's int32[world] flag
 * array (flag_arrays[q], IPC-mapped; system-scope release after a system
 * fence) and spins until all slots of its own array reach `epoch` (acquire).
 * status (int32, device memory or pinned host memory) is set to 1 + q if peer
 * q did not arrive within timeout_ms (<= 0: 10 s), else left unchanged.
 * PeerGather (sharding.py) enqueues one before the fused forward (no rank
 * stores into a peer's Y before that peer's earlier stream work has consumed
 * it) and one after it (every rank's columns have landed). */
int lmkan_b200_peer_barrier(int* const* flag_arrays, int world, int rank, int epoch, int timeout_ms,
                            int* status_dev, void* stream);

/* Explicit peer access for the fused all-gather (instead of relying on the
 * lazy enable of cudaIpcOpenMemHandle): the PCI bus id of `device`
 * ("0000:1b:00.0", buf >= 13 bytes), and a check + enable of access from
 * `device` to the GPU with that bus id. EUNSUPPORTED with an explicit message
 * when the pair has no peer path (or the peer is not visible here). */
int lmkan_b200_device_pci_bus_id(int device, char* buf, int len);
int lmkan_b200_peer_access(int device, const char* peer_pci_bus_id);

/* Drop-in synchronous host paths: X/Y in host memory (pinned or pageable),
 * copies and kernels pipelined over row chunks on internal streams; returns
 * when Y is on the host. `workers` is accepted for signature parity with
 * lmkan_forward's workers argument (threading.hpp:24-28) and ignored. */
int lmkan_b200_forward_host_f64(const lmkan_b200_layer* layer, const double* X, double* Y,
                                int64_t rows, size_t workers);
int lmkan_b200_forward_host_f32(const lmkan_b200_layer* layer, const float* X, float* Y,
                                int64_t rows, size_t workers);

/* Debug / parity path: the cell-locate stage alone (row_preambles,
 * layer.hpp:96-101). i1, i2: [rows][pairs] int32; w: [rows][pairs][4] fp32 in
 * the order {w00, w10, w01, w11}, each the reference fp64 weight rounded to
 * fp32. All pointers are device pointers. */
int lmkan_b200_locate_f32(const lmkan_b200_layer* layer, const float* X_dev, int32_t* i1,
                          int32_t* i2, float* w, int64_t rows, void* stream);
int lmkan_b200_locate_f64(const lmkan_b200_layer* layer, const double* X_dev, int32_t* i1,
                          int32_t* i2, float* w, int64_t rows, void* stream);

/* Parity path for the PRODUCTION cell records (row_preambles, layer.hpp:96-101,
 * as the gather kernels consume them; the cell index is cell_index_fast's fp32
 * estimate verified against the thresholds). Per (row, pair), row-major
 * [rows][pairs]: i1, i2 int32 and ag float2 {alpha, gamma} = fp32 of
 * (points[i+1] - x) / (points[i+1] - points[i]) per axis (the gather forms the
 * reference weights w00 = alpha*gamma, w10 = (1-alpha)*gamma, w01 = alpha*(1-gamma),
 * w11 = (1-alpha)*(1-gamma) from them). variant 0: the output of K1
 * (records4_kernel) for the layer's staged plan at `rows`, decoded from where
 * K2 reads it (packed slab/node offsets + {alpha, gamma} rings); 1: the same
 * from the shared-memory-tile K1 (records_kernel); 2: the in-kernel locate of
 * the fused / global / narrow gather kernels (same shared-memory constants,
 * node stride and slab height). EINVAL for variants 0/1 on narrow (n_out <= 4)
 * layers. Device pointers; asynchronous on `stream`. */
int lmkan_b200_records_f32(const lmkan_b200_layer* layer, const float* X_dev, int32_t* i1, int32_t* i2,
                           float* ag, int64_t rows, int variant, void* stream);
int lmkan_b200_records_f64(const lmkan_b200_layer* layer, const double* X_dev, int32_t* i1, int32_t* i2,
                           float* ag, int64_t rows, int variant, void* stream);

/* Tuning / introspection: kernel variant chosen for `rows` (OT = output tile,
 * mode 4 = the reference-precision kernel of an exact layer,
 * RT = rows per thread, NBUF = sheet buffers, rows_per_cta = the row tile,
 * possibly shortened so the grid fills whole waves of SMs), the number of
 * kernel launches one forward issues, the mode (0 = fused locate+gather,
 * 1 = staged: cell-record kernel + gather kernel, 2 = global-sheet fallback)
 * the number of i1-slabs a sheet is streamed in and the warps per CTA (16,
 * fewer for batches too small to fill the GPU). Environment overrides for
 * experiments: LMKAN_B200_MODE=fused|staged|global, LMKAN_B200_RT,
 * LMKAN_B200_NBUF, LMKAN_B200_SLABS, LMKAN_B200_NW, LMKAN_B200_OT (at layer
 * creation). Any output pointer may be NULL. */
int lmkan_b200_plan(const lmkan_b200_layer* layer, int64_t rows, int* out_tile, int* rows_per_thread,
                    int* nbuf, int* rows_per_cta, int* launches, int* mode, int* slabs, int* warps_per_cta);
/* Float4 runs of outputs each gather lane covers at output tile `out_tile`
 * (4 at 64, 2 at 32, else 1): rows_per_thread x this = the per-thread register tile in
 * float4s, the quantity LMKAN_B200_RT / the small-batch path are sized by. */
int lmkan_b200_lane_vectors(int out_tile);
/* The same for a layer (duplicated-node OT = 16 tables use 2 runs of 32 B). */
int lmkan_b200_layer_lane_vectors(const lmkan_b200_layer* layer);
/* Output tiles per group of the gather grid's CTA order at `rows` rows (1: row
 * tiles fastest; DRAM-traffic knob only, results do not depend on it); 0 on error. */
int lmkan_b200_plan_cta_group(const lmkan_b200_layer* layer, int64_t rows);
/* Plan of an implicit-im2col conv call (lmkan_b200_conv_forward_*): the sheet
 * ring depth the gather kernel runs with (after the pixel-record L1 cap), its
 * rows per CTA, and whether cells are located once per image pixel. */
int lmkan_b200_conv_plan(const lmkan_b200_layer* layer, int N, int H, int W, int C, int k, int s, int* nbuf,
                         int* rows_per_cta, int* pixel_records);

/* ---- training path ----
 *
 * lmkan_backward (layer.hpp:141-202) in fp64: dP_dev (the fp64 table layout
 * [i1][i2][pair][out], (G+1)^2 * (n_in/2) * n_out doubles) is ADDED into, as
 * the reference does; dX_dev [rows][n_in] may be NULL. P_dev is the fp64
 * master table in reference layout (the layer handle supplies grid and gamma;
 * its fp32 table is forward-only). `workers` has the reference's meaning: rows
 * are split into that many contiguous chunks (threading.hpp:33-39), each
 * chunk's dP contributions summed in row order, chunk partials merged in
 * worker order, dX summed over outputs in order with the reference's
 * expression grouping — so dP and dX are BIT-IDENTICAL to the reference's
 * lmkan_backward with the same `workers`. workers = 0 picks a count that fills
 * the GPU (lmkan_b200_backward_workers). EINVAL for output-sliced layers. */
int lmkan_b200_backward_f64(const lmkan_b200_layer* layer, const double* P_dev, const double* X_dev,
                            const double* dY_dev, double* dP_dev, double* dX_dev, int64_t rows,
                            uint64_t workers, void* stream);
/* The worker count workers = 0 selects for `rows` rows. */
int64_t lmkan_b200_backward_workers(const lmkan_b200_layer* layer, int64_t rows);
/* Same with host arrays (synchronous). */
int lmkan_b200_backward_host_f64(const lmkan_b200_layer* layer, const double* P, const double* X,
                                 const double* dY, double* dP, double* dX, int64_t rows, size_t workers);

/* ---- models: the LMK1 container and the pure-lookup inference chain ----
 *
 * load_model (serialize.hpp:185-301) reads "LMK1" | u32 LE header length |
 * JSON header | raw LE tensors, P in [i1][i2][pair][out] order, f64 or f32.
 * model_infer (model.hpp:268-315) of a FUSED model (fuse_model,
 * fuse.hpp:105-140: every block a pure lookup layer — type "lmkan", mode
 * "none", no batch norm) is a chain of lmkan_forward calls; that chain is
 * what the B200 model object runs. */

/* load_model's validation without loading tensors (host only, no GPU): magic,
 * header JSON, format/version, dtype, block metadata, manifest order and byte
 * counts, truncated payload, trailing bytes — the same checks, in the same
 * order, with the same lmkan::FormatError messages (EFORMAT). pure_lookup = 1
 * when every block is a fused lookup block. Any output may be NULL. */
int lmkan_b200_lmk1_inspect(const char* path, int* n_blocks, int* dtype_bytes, int* pure_lookup);
/* Header metadata of one block: type 0 = lmkan, 1 = mlp, 2 = bn; mode 0 =
 * relu_first, 1 = relu_last, 2 = linear, 3 = none (model.hpp:27-43);
 * p_offset = byte offset of the block's P tensor in the file (lmkan blocks). */
int lmkan_b200_lmk1_block(const char* path, int block, int* type, int* n_in, int* n_out, int* G,
                          double* gamma, int* mode, int* has_bn, uint64_t* p_offset);
/* One lmkan block's table straight from the file to a device layer (outputs
 * [out_begin, out_end); out_end < 0 = all): streamed in 64 MB chunks through
 * pinned buffers, rounded to fp32 and re-laid out on the device. The sharded
 * loader for layers too wide for one GPU (config 5). */
int lmkan_b200_layer_load_lmk1(const char* path, int block, int out_begin, int out_end, int device,
                               lmkan_b200_layer** out);
/* load_model of a fused model onto `device`: EFORMAT as load_model throws
 * FormatError, EUNSUPPORTED if any block is not a pure lookup block. */
int lmkan_b200_model_load(const char* path, int device, lmkan_b200_model** out);
/* A chain over existing layers (borrowed: they must outlive the model). */
int lmkan_b200_model_create(lmkan_b200_layer* const* layers, int n_layers, lmkan_b200_model** out);
int lmkan_b200_model_info(const lmkan_b200_model* model, int* n_blocks, int* in_dim, int* out_dim,
                          int* device);
/* Borrowed pointer to block `block`'s layer (owned by the model). */
int lmkan_b200_model_layer(const lmkan_b200_model* model, int block, lmkan_b200_layer** layer);
/* model_infer on the device: X_dev [rows][in_dim] -> Y_dev [rows][out_dim],
 * intermediate activations kept in device buffers owned by the model. The
 * first call for a (rows, X, Y, stream) runs eagerly and captures a CUDA graph
 * of the chain that later calls replay (not on the legacy NULL stream;
 * LMKAN_B200_GRAPH=0 disables). Width mismatches between blocks fail with
 * precond_forward's message (model.hpp:59). Calls on one model serialize. */
int lmkan_b200_model_infer_f32(lmkan_b200_model* model, const float* X_dev, float* Y_dev, int64_t rows,
                               void* stream);
int lmkan_b200_model_infer_f64(lmkan_b200_model* model, const double* X_dev, double* Y_dev,
                               int64_t rows, void* stream);
/* Drop-in synchronous model_infer with host X/Y; `workers` ignored. */
int lmkan_b200_model_infer_host_f64(lmkan_b200_model* model, const double* X, double* Y, int64_t rows,
                                    size_t workers);
int lmkan_b200_model_infer_host_f32(lmkan_b200_model* model, const float* X, float* Y, int64_t rows,
                                    size_t workers);
int lmkan_b200_model_destroy(lmkan_b200_model* model);

#ifdef __cplusplus
}
#endif
#endif /* LMKAN_B200_H */
