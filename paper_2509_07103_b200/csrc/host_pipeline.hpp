// Host-memory entry points (the synchronous drop-in lmkan_forward, model_infer
// and conv on host buffers): rows are processed in chunks through a three-
// stream pipeline
//
//   copy-in stream     H2D of chunk c into slot c % kSlots
//   compute stream c%2 kernels of chunk c          (after its H2D and after the
//                                                   D2H that last used the slot's Y)
//   copy-out stream    D2H of chunk c               (after its kernels)
//
// so H2D of later chunks, kernels and D2H of earlier chunks all overlap, and the
// two copy directions run concurrently on their own copy engines. (Two streams
// each carrying H2D -> kernels -> D2H serialise a stream's next H2D behind its
// previous D2H: cfg4's host conv, where copies and kernels take about the same
// time, lost ~20% to that.) Two compute streams let the next chunk's CTAs fill
// the SMs left idle by the last partial wave of the current one (one compute
// stream cost cfg2's host path 19% of its e2e throughput).
#pragma once

#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

namespace lmkan_b200 {

// Chunk boundaries over `total` units (rows or images): chunks of `full` units,
// optionally tapered at both ends (full/4, full/2, full, ..., full, full/2,
// full/4) so the first H2D and the last kernels + D2H, which nothing overlaps,
// move less data. Tapering needs at least 2 full chunks' worth of units.
struct ChunkSchedule {
    std::vector<int64_t> start;  // start[c] .. start[c + 1]
    ChunkSchedule(int64_t total, int64_t full, bool taper) {
        full = full < 1 ? 1 : full;
        std::vector<int64_t> sizes;
        if (taper && full >= 4 && total >= 2 * full) {
            const int64_t edge[2] = {full / 4, full / 2};
            int64_t mid = total - 2 * (edge[0] + edge[1]);
            sizes = {edge[0], edge[1]};
            for (; mid > 0; mid -= full) sizes.push_back(mid < full ? mid : full);
            sizes.push_back(edge[1]);
            sizes.push_back(edge[0]);
        } else {
            for (int64_t r = total; r > 0; r -= full) sizes.push_back(r < full ? r : full);
        }
        start.assign(1, 0);
        for (int64_t z : sizes) start.push_back(start.back() + z);
    }
    int64_t count() const { return static_cast<int64_t>(start.size()) - 1; }
    int64_t first(int64_t c) const { return start[c]; }
    int64_t size(int64_t c) const { return start[c + 1] - start[c]; }
};

struct HostPipeline {
    static constexpr int kSlots = 3;
    int device = -1;
    cudaStream_t in = nullptr, out = nullptr, comp[2] = {nullptr, nullptr};
    cudaEvent_t h2d[kSlots] = {}, kdone[kSlots] = {}, d2h[kSlots] = {};
    void* dX[kSlots] = {};
    void* dY[kSlots] = {};
    size_t xcap = 0, ycap = 0;

    cudaError_t init(int dev) {
        if (in) return cudaSuccess;
        device = dev;
        cudaError_t e = cudaSuccess;
        for (cudaStream_t* s : {&in, &comp[0], &comp[1], &out})
            if (e == cudaSuccess) e = cudaStreamCreateWithFlags(s, cudaStreamNonBlocking);
        for (int i = 0; i < kSlots && e == cudaSuccess; ++i) {
            for (cudaEvent_t* ev : {&h2d[i], &kdone[i], &d2h[i]})
                if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
        }
        return e;
    }
    // Staging buffers of at least xb / yb bytes per slot (grown, never shrunk).
    cudaError_t reserve(size_t xb, size_t yb) {
        if (xb <= xcap && yb <= ycap) return cudaSuccess;
        cudaError_t e = cudaStreamSynchronize(comp[0]);
        if (e == cudaSuccess) e = cudaStreamSynchronize(comp[1]);
        if (e == cudaSuccess) e = cudaStreamSynchronize(in);
        if (e == cudaSuccess) e = cudaStreamSynchronize(out);
        if (e != cudaSuccess) return e;
        release();
        for (int i = 0; i < kSlots && e == cudaSuccess; ++i) {
            e = cudaMalloc(&dX[i], xb);
            if (e == cudaSuccess) e = cudaMalloc(&dY[i], yb);
        }
        if (e != cudaSuccess) {
            release();
            return e;
        }
        xcap = xb;
        ycap = yb;
        return cudaSuccess;
    }
    void release() {
        for (int i = 0; i < kSlots; ++i) {
            if (dX[i]) cudaFree(dX[i]);
            if (dY[i]) cudaFree(dY[i]);
            dX[i] = dY[i] = nullptr;
        }
        xcap = ycap = 0;
    }
    void destroy() {
        release();
        for (int i = 0; i < kSlots; ++i)
            for (cudaEvent_t* ev : {&h2d[i], &kdone[i], &d2h[i]}) {
                if (*ev) cudaEventDestroy(*ev);
                *ev = nullptr;
            }
        for (cudaStream_t s : {in, comp[0], comp[1], out})
            if (s) cudaStreamDestroy(s);
        in = out = comp[0] = comp[1] = nullptr;
    }
    // per-thread pipelines (host entry points) go away with their thread;
    // errors after the runtime has shut down (process exit) are ignored
    ~HostPipeline() { destroy(); }
};

// Runs `chunks` chunks through the pipeline. For chunk c:
//   src(c, &host_ptr, &bytes)  - host input to copy into the slot's dX
//   dst(c, &host_ptr, &bytes)  - host output to fill from the slot's dY
//   compute(c, dX, dY, stream) - enqueue the chunk's kernels; returns a status
// Blocks until every chunk's D2H has landed. Returns the first failing status
// (`cuda_fail(e, what)` maps CUDA errors).
template <class Src, class Dst, class Compute, class Fail>
int run_host_pipeline(HostPipeline& P, int64_t chunks, Src src, Dst dst, Compute compute, Fail cuda_fail) {
    constexpr int S = HostPipeline::kSlots;
    int rc = 0;
    if (chunks == 1) {  // nothing to overlap: one stream, no cross-stream events (small batches)
        const void* hs = nullptr;
        void* hd = nullptr;
        size_t xb = 0, yb = 0;
        src(0, &hs, &xb);
        dst(0, &hd, &yb);
        cudaStream_t st = P.comp[0];
        cudaError_t e = cudaMemcpyAsync(P.dX[0], hs, xb, cudaMemcpyHostToDevice, st);
        if (e != cudaSuccess) return cuda_fail(e, "host pipeline: H2D");
        if ((rc = compute(0, P.dX[0], P.dY[0], st)) != 0) {
            cudaStreamSynchronize(st);
            return rc;
        }
        e = cudaMemcpyAsync(hd, P.dY[0], yb, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        return e == cudaSuccess ? 0 : cuda_fail(e, "host pipeline: D2H");
    }
    for (int64_t c = 0; c < chunks && rc == 0; ++c) {
        const int b = static_cast<int>(c % S);
        const void* hs = nullptr;
        void* hd = nullptr;
        size_t xb = 0, yb = 0;
        src(c, &hs, &xb);
        dst(c, &hd, &yb);
        cudaError_t e = cudaSuccess;
        if (c >= S) e = cudaStreamWaitEvent(P.in, P.kdone[b], 0);  // chunk c - S has consumed dX[b]
        if (e == cudaSuccess) e = cudaMemcpyAsync(P.dX[b], hs, xb, cudaMemcpyHostToDevice, P.in);
        if (e == cudaSuccess) e = cudaEventRecord(P.h2d[b], P.in);
        cudaStream_t comp = P.comp[c & 1];
        if (e == cudaSuccess) e = cudaStreamWaitEvent(comp, P.h2d[b], 0);
        if (e == cudaSuccess && c >= S) e = cudaStreamWaitEvent(comp, P.d2h[b], 0);  // dY[b] drained
        if (e != cudaSuccess) {
            rc = cuda_fail(e, "host pipeline: H2D");
            break;
        }
        rc = compute(c, P.dX[b], P.dY[b], comp);
        if (rc) break;
        e = cudaEventRecord(P.kdone[b], comp);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(P.out, P.kdone[b], 0);
        if (e == cudaSuccess) e = cudaMemcpyAsync(hd, P.dY[b], yb, cudaMemcpyDeviceToHost, P.out);
        if (e == cudaSuccess) e = cudaEventRecord(P.d2h[b], P.out);
        if (e != cudaSuccess) rc = cuda_fail(e, "host pipeline: D2H");
    }
    for (cudaStream_t s : {P.in, P.comp[0], P.comp[1], P.out}) {
        const cudaError_t e = cudaStreamSynchronize(s);
        if (e != cudaSuccess && rc == 0) rc = cuda_fail(e, "host pipeline: stream sync");
    }
    return rc;
}

}  // namespace lmkan_b200
