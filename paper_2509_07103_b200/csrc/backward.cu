// Training path of the lmKAN layer on sm_100a: lmkan_backward
// (/root/reference/proj/include/lmkan/layer.hpp:141-202) in fp64.
//
// The reference accumulates, per (row, pair), gamma * w * dY into the four
// active nodes of dP and the analytic cell derivatives into dX; with one
// worker the dP sums run over rows in order (worker 0 adds straight into dP,
// layer.hpp:162-163) and each dX entry sums over outputs q in order
// (layer.hpp:182-191). Both kernels below keep exactly those orders and the
// reference's expression grouping with explicitly rounded fp64 operations
// (no FMA contraction), so dP and dX are bit-identical to the reference's
// lmkan_backward run with the same worker count, and deterministic:
//   dx kernel: one thread per (row, pair), the q loop in order;
//   dP kernel: one lane per (pair, output q, worker), the worker's contiguous
//              row chunk (threading.hpp:33-39) in order; worker 0 adds into dP,
//              the others into zeroed partial buffers merged in worker order
//              (layer.hpp:199-200). Each lane owns its dP column: no atomics.
//   With workers = 1 the dP sums are the plain row-ordered sums; workers = 0
//   picks enough row chunks to fill the GPU (lmkan_b200_backward_workers).
// The fp64 master table P is passed in reference layout (training keeps the
// fp64 P; the layer handle's fp32 device table serves the forward only).
#include <algorithm>
#include <string>

#include "../../include/lmkan_b200.h"
#include "layer_impl.hpp"

using namespace lmkan_b200;

namespace {

struct CellF64 {
    int i1, i2;
    double a, b, c, d;  // right/left gaps on both axes (grid.hpp:94-97)
};

// preamble (grid.hpp:87-101) in fp64, indices bit-exact (threshold count).
__device__ __forceinline__ CellF64 cell_f64(double x1, double x2, const double* thr, const double* pts, int G, int L) {
    CellF64 c;
    c.i1 = cell_index_fast<double>(x1, thr, G, L);
    c.i2 = cell_index_fast<double>(x2, thr, G, L);
    c.a = __dsub_rn(pts[c.i1 + 1], x1);
    c.b = __dsub_rn(x1, pts[c.i1]);
    c.c = __dsub_rn(pts[c.i2 + 1], x2);
    c.d = __dsub_rn(x2, pts[c.i2]);
    return c;
}

__global__ void __launch_bounds__(256) backward_dx_kernel(const double* __restrict__ P, const double* __restrict__ X,
                                                          const double* __restrict__ dY, double* __restrict__ dX,
                                                          int64_t rows, int n_in, int n_out, double gamma,
                                                          const __grid_constant__ GridConst gc) {
    __shared__ double thr[kMaxThr];
    __shared__ double pts[kMaxThr + 1];
    for (int k = threadIdx.x; k < gc.L; k += blockDim.x) thr[k] = gc.t64[k];
    for (int k = threadIdx.x; k <= gc.G; k += blockDim.x) pts[k] = gc.points[k];
    __syncthreads();
    const int pairs = n_in / 2, G = gc.G, G1 = G + 1;
    const size_t per_node = static_cast<size_t>(pairs) * n_out;
    const int64_t total = rows * pairs;
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < total;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = k / pairs;
        const int p = static_cast<int>(k - r * pairs);
        const double x1 = X[r * n_in + 2 * p], x2 = X[r * n_in + 2 * p + 1];
        const CellF64 c = cell_f64(x1, x2, thr, pts, G, gc.L);
        const size_t base = (static_cast<size_t>(c.i1) * G1 + c.i2) * per_node + static_cast<size_t>(p) * n_out;
        const double* p00 = P + base;
        const double* p10 = p00 + static_cast<size_t>(G1) * per_node;
        const double* p01 = p00 + per_node;
        const double* p11 = p10 + per_node;
        const double* g = dY + r * n_out;
        // layer.hpp:179-182: r2 = c, l2 = d, r1 = a, l1 = b
        double acc1 = 0.0, acc2 = 0.0;
        for (int q = 0; q < n_out; ++q) {
            const double gq = __dmul_rn(gamma, __ldg(g + q));
            const double v00 = __ldg(p00 + q), v10 = __ldg(p10 + q), v01 = __ldg(p01 + q), v11 = __ldg(p11 + q);
            const double t1 = __dadd_rn(__dmul_rn(__dsub_rn(v10, v00), c.c), __dmul_rn(__dsub_rn(v11, v01), c.d));
            const double t2 = __dadd_rn(__dmul_rn(__dsub_rn(v01, v00), c.a), __dmul_rn(__dsub_rn(v11, v10), c.b));
            acc1 = __dadd_rn(acc1, __dmul_rn(gq, t1));
            acc2 = __dadd_rn(acc2, __dmul_rn(gq, t2));
        }
        const double inv = __ldg(gc.inv_areas + c.i1 * G + c.i2);
        dX[r * n_in + 2 * p] = __dmul_rn(acc1, inv);
        dX[r * n_in + 2 * p + 1] = __dmul_rn(acc2, inv);
    }
}

// One lane per (pair, output, worker): lanes of a warp share the pair (and
// therefore the cell of every row) and cover 32 consecutive outputs; worker w
// owns rows [w * chunk, min(rows, (w + 1) * chunk)), threading.hpp:33-39, and
// accumulates them in order into dP (w == 0, layer.hpp:162) or into its zeroed
// partial buffer (w > 0, merged afterwards in worker order by merge_kernel).
__global__ void __launch_bounds__(128) backward_dp_kernel(const double* __restrict__ X, const double* __restrict__ dY,
                                                          double* __restrict__ dP, double* __restrict__ partials,
                                                          int64_t rows, int64_t chunk, int workers, int n_in,
                                                          int n_out, double gamma, const __grid_constant__ GridConst gc) {
    __shared__ double thr[kMaxThr];
    __shared__ double pts[kMaxThr + 1];
    for (int k = threadIdx.x; k < gc.L; k += blockDim.x) thr[k] = gc.t64[k];
    for (int k = threadIdx.x; k <= gc.G; k += blockDim.x) pts[k] = gc.points[k];
    __syncthreads();
    const int pairs = n_in / 2, G = gc.G, G1 = G + 1;
    const int chunks = (n_out + 31) / 32;
    const int64_t warp = blockIdx.x * static_cast<int64_t>(blockDim.x / 32) + threadIdx.x / 32;
    if (warp >= static_cast<int64_t>(pairs) * chunks * workers) return;
    const int w = static_cast<int>(warp % workers);
    const int64_t pc = warp / workers;
    const int p = static_cast<int>(pc / chunks);
    const int q = static_cast<int>(pc % chunks) * 32 + (threadIdx.x & 31);
    if (q >= n_out) return;
    const size_t per_node = static_cast<size_t>(pairs) * n_out;
    double* acc = w == 0 ? dP : partials + static_cast<size_t>(w - 1) * G1 * G1 * per_node;
    double* col = acc + static_cast<size_t>(p) * n_out + q;  // node 0 of this (pair, q) column
    const size_t s10 = static_cast<size_t>(G1) * per_node, s01 = per_node;
    const int64_t rb = min(rows, static_cast<int64_t>(w) * chunk), re = min(rows, rb + chunk);
    for (int64_t r = rb; r < re; ++r) {
        const double x1 = __ldg(X + r * n_in + 2 * p), x2 = __ldg(X + r * n_in + 2 * p + 1);
        const CellF64 c = cell_f64(x1, x2, thr, pts, G, gc.L);
        const double inv = __ldg(gc.inv_areas + c.i1 * G + c.i2);
        // preamble's weights (grid.hpp:98-101): (a * c) * inv etc.
        const double w00 = __dmul_rn(__dmul_rn(c.a, c.c), inv);
        const double w10 = __dmul_rn(__dmul_rn(c.b, c.c), inv);
        const double w01 = __dmul_rn(__dmul_rn(c.a, c.d), inv);
        const double w11 = __dmul_rn(__dmul_rn(c.b, c.d), inv);
        const double gq = __dmul_rn(gamma, __ldg(dY + r * n_out + q));
        double* d00 = col + (static_cast<size_t>(c.i1) * G1 + c.i2) * per_node;
        double* d10 = d00 + s10;
        double* d01 = d00 + s01;
        double* d11 = d10 + s01;
        *d00 = __dadd_rn(*d00, __dmul_rn(w00, gq));
        *d10 = __dadd_rn(*d10, __dmul_rn(w10, gq));
        *d01 = __dadd_rn(*d01, __dmul_rn(w01, gq));
        *d11 = __dadd_rn(*d11, __dmul_rn(w11, gq));
    }
}

// layer.hpp:199-200: dP[i] += buf[i] for every partial buffer, in worker order.
__global__ void merge_kernel(double* __restrict__ dP, const double* __restrict__ partials, size_t n, int parts) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        double v = dP[i];
        for (int k = 0; k < parts; ++k) v = __dadd_rn(v, partials[static_cast<size_t>(k) * n + i]);
        dP[i] = v;
    }
}

// Worker count for workers == 0: enough row chunks to fill the GPU (>= 256
// rows each, at most 256 chunks), capped so the partial buffers stay <= 1 GiB.
int64_t auto_workers(const lmkan_b200_layer* L, int64_t rows) {
    const size_t pbytes = static_cast<size_t>(L->nodes) * L->pairs * L->n_out * 8;
    int64_t w = std::min<int64_t>(256, std::max<int64_t>(1, rows / 256));
    const int64_t cap = static_cast<int64_t>((size_t(1) << 30) / std::max<size_t>(pbytes, 1)) + 1;
    return std::max<int64_t>(1, std::min(w, cap));
}

int backward_device(const lmkan_b200_layer* L, const double* P, const double* X, const double* dY, double* dP,
                    double* dX, int64_t rows, uint64_t workers_req, cudaStream_t st) {
    if (!L) return api::set_error(LMKAN_B200_EINVAL, "lmkan_backward: null layer");
    if (rows < 0) return api::set_error(LMKAN_B200_EINVAL, "lmkan_backward: negative row count");
    if (L->n_out != L->n_out_total)
        return api::set_error(LMKAN_B200_EINVAL, "lmkan_backward: output-sliced layers are forward-only");
    if (rows == 0) return LMKAN_B200_OK;
    if (!P || !X || !dY || !dP) return api::set_error(LMKAN_B200_EINVAL, "lmkan_backward: null argument");
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != L->device) cudaSetDevice(L->device);
    // layer.hpp:151-152: workers clamped to [1, rows]
    int64_t W = workers_req ? static_cast<int64_t>(std::min<uint64_t>(workers_req, 1u << 20)) : auto_workers(L, rows);
    W = std::max<int64_t>(1, std::min<int64_t>(W, rows));
    const int64_t chunk = (rows + W - 1) / W;  // threading.hpp:33
    const size_t n = static_cast<size_t>(L->nodes) * L->pairs * L->n_out;
    double* partials = nullptr;
    cudaError_t e = cudaSuccess;
    if (W > 1) {
        e = cudaMallocAsync(reinterpret_cast<void**>(&partials), n * 8 * (W - 1), st);
        if (e == cudaSuccess) e = cudaMemsetAsync(partials, 0, n * 8 * (W - 1), st);
    }
    const double gamma = L->gamma;
    const int pairs = L->pairs;
    if (e == cudaSuccess) {
        const int64_t warps = static_cast<int64_t>(pairs) * ((L->n_out + 31) / 32) * W;
        backward_dp_kernel<<<static_cast<unsigned>((warps + 3) / 4), 128, 0, st>>>(
            X, dY, dP, partials, rows, chunk, static_cast<int>(W), L->n_in, L->n_out, gamma, L->gc);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess && W > 1) {
        merge_kernel<<<static_cast<unsigned>(std::min<size_t>((n + 255) / 256, static_cast<size_t>(L->num_sms) * 16)), 256, 0, st>>>(
            dP, partials, n, static_cast<int>(W - 1));
        e = cudaGetLastError();
    }
    if (partials) cudaFreeAsync(partials, st);
    if (e == cudaSuccess && dX) {
        const int64_t total = rows * pairs;
        const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, L->num_sms * 32));
        backward_dx_kernel<<<blocks, 256, 0, st>>>(P, X, dY, dX, rows, L->n_in, L->n_out, gamma, L->gc);
        e = cudaGetLastError();
    }
    if (prev != L->device) cudaSetDevice(prev);
    if (e != cudaSuccess) return api::cuda_error(e, "lmkan_backward: launch");
    return LMKAN_B200_OK;
}

}  // namespace

extern "C" {

int lmkan_b200_backward_f64(const lmkan_b200_layer* layer, const double* P_dev, const double* X_dev,
                            const double* dY_dev, double* dP_dev, double* dX_dev, int64_t rows, uint64_t workers,
                            void* stream) {
    return backward_device(layer, P_dev, X_dev, dY_dev, dP_dev, dX_dev, rows, workers,
                           static_cast<cudaStream_t>(stream));
}

int64_t lmkan_b200_backward_workers(const lmkan_b200_layer* layer, int64_t rows) {
    if (!layer || rows <= 0) return 1;
    return std::max<int64_t>(1, std::min<int64_t>(auto_workers(layer, rows), rows));
}

int lmkan_b200_backward_host_f64(const lmkan_b200_layer* layer, const double* P, const double* X, const double* dY,
                                 double* dP, double* dX, int64_t rows, size_t workers) {
    if (!layer) return api::set_error(LMKAN_B200_EINVAL, "lmkan_backward: null layer");
    if (rows == 0) return LMKAN_B200_OK;
    if (!P || !X || !dY || !dP) return api::set_error(LMKAN_B200_EINVAL, "lmkan_backward: null argument");
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != layer->device) cudaSetDevice(layer->device);
    const size_t np = static_cast<size_t>(layer->nodes) * layer->pairs * layer->n_out;
    const size_t nx = static_cast<size_t>(rows) * layer->n_in, ny = static_cast<size_t>(rows) * layer->n_out;
    double *dPd = nullptr, *dXd = nullptr, *dYd = nullptr, *dPacc = nullptr, *dXo = nullptr;
    cudaStream_t st = nullptr;
    int rc = LMKAN_B200_OK;
    cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&dPd), np * 8, st);
    if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&dPacc), np * 8, st);
    if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&dXd), nx * 8, st);
    if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&dYd), ny * 8, st);
    if (e == cudaSuccess && dX) e = cudaMallocAsync(reinterpret_cast<void**>(&dXo), nx * 8, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dPd, P, np * 8, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dPacc, dP, np * 8, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dXd, X, nx * 8, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dYd, dY, ny * 8, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) rc = api::cuda_error(e, "lmkan_backward: host staging");
    if (rc == LMKAN_B200_OK) rc = backward_device(layer, dPd, dXd, dYd, dPacc, dXo, rows, workers, st);
    if (rc == LMKAN_B200_OK) {
        e = cudaMemcpyAsync(dP, dPacc, np * 8, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess && dX) e = cudaMemcpyAsync(dX, dXo, nx * 8, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) rc = api::cuda_error(e, "lmkan_backward: D2H");
    }
    for (double* ptr : {dPd, dPacc, dXd, dYd, dXo})
        if (ptr) cudaFreeAsync(ptr, st);
    if (st) {
        cudaStreamSynchronize(st);
        cudaStreamDestroy(st);
    }
    if (prev != layer->device) cudaSetDevice(prev);
    return rc;
}

}  // extern "C"
