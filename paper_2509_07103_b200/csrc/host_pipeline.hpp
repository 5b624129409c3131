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
//
// Pageable (ordinary malloc / std::vector) host buffers — the reference
// signature's Matrix — are staged through pinned slots: a pool of host threads
// copies chunk c+1's X into its pinned slot and chunk c-1's Y out of its slot
// while the GPU works on chunk c, so the copies still overlap (a
// cudaMemcpyAsync straight from pageable memory is synchronous, single-threaded
// and bounced through the driver's own small pinned buffer).
#pragma once

#include <algorithm>
#include <condition_variable>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>
#include <cuda_runtime.h>
#if defined(__SSE2__)
#include <emmintrin.h>
#endif

namespace lmkan_b200 {

// Chunk boundaries over `total` units (rows or images): chunks of `full` units,
// optionally tapered at both ends (levels = 2: full/4, full/2, full, ..., full,
// full/2, full/4) so the first H2D and the last kernels + D2H, which nothing
// overlaps, move less data. Tapering needs at least 2 full chunks' worth of units.
struct ChunkSchedule {
    std::vector<int64_t> start;  // start[c] .. start[c + 1]
    // levels: how many halvings taper each end (2: full/4, full/2, full, ...)
    ChunkSchedule(int64_t total, int64_t full, int levels) {
        full = full < 1 ? 1 : full;
        std::vector<int64_t> sizes;
        if (levels > 0 && full >= (int64_t(1) << levels) && total >= 2 * full) {
            std::vector<int64_t> edge;
            for (int l = levels; l >= 1; --l) edge.push_back(full >> l);
            int64_t mid = total;
            for (int64_t e : edge) mid -= 2 * e;
            sizes = edge;
            for (; mid > 0; mid -= full) sizes.push_back(mid < full ? mid : full);
            for (auto it = edge.rbegin(); it != edge.rend(); ++it) sizes.push_back(*it);
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

// Parallel host copies over a persistent pool of threads (the caller takes a
// share too). LMKAN_B200_COPY_THREADS overrides the pool size (default: the
// hardware threads, at most 32).
class CopyPool {
public:
    CopyPool() = default;
    CopyPool(const CopyPool&) = delete;
    CopyPool& operator=(const CopyPool&) = delete;
    ~CopyPool() { stop(); }

    // Both copies stream their stores past the caches (non-temporal), so the
    // destination is not read first: the pageable path is bound by host memory
    // bandwidth (tools/ubench_hostcopy.cpp), and every byte not moved counts.
    void copy(void* dst, const void* src, size_t bytes) {
        char* d = static_cast<char*>(dst);
        const char* s = static_cast<const char*>(src);
        parallel(bytes, 64, [=](size_t lo, size_t hi) { copy_nt(d + lo, s + lo, hi - lo); });
    }
    // dst[i] = double(src[i]): fp32 results widened into the caller's fp64 Y
    void widen(double* dst, const float* src, size_t count) {
        parallel(count, 16, [=](size_t lo, size_t hi) { widen_nt(dst + lo, src + lo, hi - lo); });
    }

    static void copy_nt(char* d, const char* s, size_t n) {
#if defined(__SSE2__)
        size_t i = 0;
        for (; i < n && (reinterpret_cast<uintptr_t>(d + i) & 15); ++i) d[i] = s[i];
        for (; i + 64 <= n; i += 64) {
            const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i));
            const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 16));
            const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 32));
            const __m128i e = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 48));
            _mm_stream_si128(reinterpret_cast<__m128i*>(d + i), a);
            _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 16), b);
            _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 32), c);
            _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 48), e);
        }
        _mm_sfence();
        if (i < n) std::memcpy(d + i, s + i, n - i);
#else
        std::memcpy(d, s, n);
#endif
    }
    static void widen_nt(double* d, const float* s, size_t n) {
        size_t i = 0;
#if defined(__SSE2__)
        for (; i < n && (reinterpret_cast<uintptr_t>(d + i) & 15); ++i) d[i] = static_cast<double>(s[i]);
        for (; i + 4 <= n; i += 4) {
            const __m128 v = _mm_loadu_ps(s + i);
            _mm_stream_pd(d + i, _mm_cvtps_pd(v));
            _mm_stream_pd(d + i + 2, _mm_cvtps_pd(_mm_movehl_ps(v, v)));
        }
        _mm_sfence();
#endif
        for (; i < n; ++i) d[i] = static_cast<double>(s[i]);
    }

private:
    template <class F>
    void parallel(size_t n, size_t align, F fn) {
        start();
        const size_t t = workers_.size() + 1;
        if (n < (size_t(1) << 18) || t == 1) {
            fn(0, n);
            return;
        }
        const size_t part = ((n + t - 1) / t + align - 1) / align * align;
        auto run_part = [=](size_t k) {
            const size_t lo = k * part;
            if (lo < n) fn(lo, std::min(n, lo + part));
        };
        {
            std::lock_guard<std::mutex> lk(mu_);
            job_fn_ = run_part;
            pending_ = workers_.size();
            ++job_;
        }
        cv_.notify_all();
        run_part(t - 1);  // the caller's share
        std::unique_lock<std::mutex> lk(mu_);
        done_.wait(lk, [&] { return pending_ == 0; });
    }
    void start() {
        if (started_) return;
        started_ = true;
        // all hardware threads (measured on a 16-core host: 4 / 8 / 16 threads
        // -> pageable cfg2 drop-in 47 / 34 / 28 ms per call)
        int n = static_cast<int>(std::thread::hardware_concurrency());
        if (const char* e = std::getenv("LMKAN_B200_COPY_THREADS")) n = std::atoi(e);
        n = std::max(1, std::min(n, 32));
        for (int i = 0; i + 1 < n; ++i) workers_.emplace_back([this, i] { run(static_cast<size_t>(i)); });
    }
    void stop() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            quit_ = true;
        }
        cv_.notify_all();
        for (auto& t : workers_) t.join();
        workers_.clear();
    }
    void run(size_t idx) {
        uint64_t seen = 0;
        for (;;) {
            std::unique_lock<std::mutex> lk(mu_);
            cv_.wait(lk, [&] { return quit_ || job_ != seen; });
            if (quit_) return;
            seen = job_;
            std::function<void(size_t)> fn = job_fn_;
            lk.unlock();
            fn(idx);
            lk.lock();
            if (--pending_ == 0) done_.notify_one();
        }
    }

    std::vector<std::thread> workers_;
    std::mutex mu_;
    std::condition_variable cv_, done_;
    bool started_ = false, quit_ = false;
    uint64_t job_ = 0;
    size_t pending_ = 0;
    std::function<void(size_t)> job_fn_;
};

// true when p is ordinary pageable host memory (not pinned / registered / managed)
inline bool is_pageable(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return a.type == cudaMemoryTypeUnregistered;
}

struct HostPipeline {
    static constexpr int kSlots = 3;
    int device = -1;
    cudaStream_t in = nullptr, out = nullptr, comp[2] = {nullptr, nullptr};
    cudaEvent_t h2d[kSlots] = {}, kdone[kSlots] = {}, d2h[kSlots] = {};
    void* dX[kSlots] = {};
    void* dY[kSlots] = {};
    size_t xcap = 0, ycap = 0;
    void* hX[kSlots] = {};  // pinned staging for pageable callers (allocated on first use)
    void* hY[kSlots] = {};
    size_t hxcap = 0, hycap = 0;
    CopyPool pool;

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
    // Pinned host staging slots of at least xb / yb bytes (pageable callers).
    cudaError_t reserve_pinned(size_t xb, size_t yb) {
        if (xb <= hxcap && yb <= hycap) return cudaSuccess;
        release_pinned();
        cudaError_t e = cudaSuccess;
        for (int i = 0; i < kSlots && e == cudaSuccess; ++i) {
            e = cudaHostAlloc(&hX[i], xb, cudaHostAllocDefault);
            if (e == cudaSuccess) e = cudaHostAlloc(&hY[i], yb, cudaHostAllocDefault);
        }
        if (e != cudaSuccess) {
            release_pinned();
            return e;
        }
        hxcap = xb;
        hycap = yb;
        return cudaSuccess;
    }
    void release_pinned() {
        for (int i = 0; i < kSlots; ++i) {
            if (hX[i]) cudaFreeHost(hX[i]);
            if (hY[i]) cudaFreeHost(hY[i]);
            hX[i] = hY[i] = nullptr;
        }
        hxcap = hycap = 0;
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
        release_pinned();
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
//
// widen_out: the device result is fp32 while the caller's Y is fp64 (dst gives
// the fp64 buffer and its byte count): the D2H moves the fp32 bytes (half) into
// a pinned slot and the host pool widens them into Y.
// LMKAN_B200_PIPE_TRACE=1: timing events around every chunk's H2D, kernels and
// D2H, printed to stderr (ms from the first H2D) after the call — the timeline
// a profiler would show, for tuning the chunking (not used otherwise).
struct PipeTrace {
    std::vector<cudaEvent_t> ev;  // per chunk: H2D begin / end, kernels begin / end, D2H begin / end
    explicit PipeTrace(int64_t chunks) {
        const char* e = std::getenv("LMKAN_B200_PIPE_TRACE");
        if (!e || !std::atoi(e)) return;
        ev.assign(static_cast<size_t>(chunks) * 6, nullptr);
        for (auto& x : ev) cudaEventCreate(&x);
    }
    void mark(int64_t c, int k, cudaStream_t st) {
        if (!ev.empty()) cudaEventRecord(ev[static_cast<size_t>(c) * 6 + k], st);
    }
    ~PipeTrace() {
        if (ev.empty()) return;
        const int64_t chunks = static_cast<int64_t>(ev.size()) / 6;
        for (int64_t c = 0; c < chunks; ++c) {
            float t[6] = {};
            for (int k = 0; k < 6; ++k) cudaEventElapsedTime(&t[k], ev[0], ev[static_cast<size_t>(c) * 6 + k]);
            std::fprintf(stderr, "pipe chunk %lld: h2d %.4f-%.4f  kern %.4f-%.4f  d2h %.4f-%.4f ms\n",
                         static_cast<long long>(c), t[0], t[1], t[2], t[3], t[4], t[5]);
        }
        for (auto x : ev) cudaEventDestroy(x);
    }
};

template <class Src, class Dst, class Compute, class Fail>
int run_host_pipeline(HostPipeline& P, int64_t chunks, Src src, Dst dst, Compute compute, Fail cuda_fail,
                      bool widen_out = false) {
    constexpr int S = HostPipeline::kSlots;
    int rc = 0;
    if (chunks == 1 && !widen_out) {  // nothing to overlap: one stream, no cross-stream events (small batches)
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
    // pageable caller buffers go through the pinned slots (see the header comment)
    const void* hs0 = nullptr;
    void* hd0 = nullptr;
    size_t xb0 = 0, yb0 = 0;
    src(0, &hs0, &xb0);
    dst(0, &hd0, &yb0);
    const bool stage_in = is_pageable(hs0), stage_out = widen_out || is_pageable(hd0);
    const size_t yscale = widen_out ? 2 : 1;  // host Y bytes per device Y byte
    if (stage_in || stage_out) {
        size_t xmax = 0, ymax = 0;
        for (int64_t c = 0; c < chunks; ++c) {
            const void* a = nullptr;
            void* d = nullptr;
            size_t xb = 0, yb = 0;
            src(c, &a, &xb);
            dst(c, &d, &yb);
            xmax = std::max(xmax, xb);
            ymax = std::max(ymax, yb);
        }
        const cudaError_t e = P.reserve_pinned(stage_in ? xmax : 0, stage_out ? ymax / yscale : 0);
        if (e != cudaSuccess) return cuda_fail(e, "host pipeline: pinned staging");
    }
    // copy chunk c's result out of its pinned slot into the caller's buffer
    auto drain = [&](int64_t c) -> int {
        if (!stage_out || c < 0) return 0;
        void* hd = nullptr;
        size_t yb = 0;
        dst(c, &hd, &yb);
        const cudaError_t e = cudaEventSynchronize(P.d2h[c % S]);
        if (e != cudaSuccess) return cuda_fail(e, "host pipeline: D2H");
        if (widen_out)
            P.pool.widen(static_cast<double*>(hd), static_cast<const float*>(P.hY[c % S]), yb / sizeof(double));
        else
            P.pool.copy(hd, P.hY[c % S], yb);
        return 0;
    };
    PipeTrace tr(chunks);
    for (int64_t c = 0; c < chunks && rc == 0; ++c) {
        const int b = static_cast<int>(c % S);
        const void* hs = nullptr;
        void* hd = nullptr;
        size_t xb = 0, yb = 0;
        src(c, &hs, &xb);
        dst(c, &hd, &yb);
        cudaError_t e = cudaSuccess;
        if (stage_in) {  // the slot's previous H2D (chunk c - S) has finished reading it
            if (c >= S) e = cudaEventSynchronize(P.h2d[b]);
            if (e != cudaSuccess) {
                rc = cuda_fail(e, "host pipeline: H2D");
                break;
            }
            P.pool.copy(P.hX[b], hs, xb);
            hs = P.hX[b];
        }
        if (stage_out) hd = P.hY[b];  // chunk c - S was drained from it at iteration c - 1
        if (c >= S) e = cudaStreamWaitEvent(P.in, P.kdone[b], 0);  // chunk c - S has consumed dX[b]
        tr.mark(c, 0, P.in);
        if (e == cudaSuccess) e = cudaMemcpyAsync(P.dX[b], hs, xb, cudaMemcpyHostToDevice, P.in);
        tr.mark(c, 1, P.in);
        if (e == cudaSuccess) e = cudaEventRecord(P.h2d[b], P.in);
        cudaStream_t comp = P.comp[c & 1];
        if (e == cudaSuccess) e = cudaStreamWaitEvent(comp, P.h2d[b], 0);
        if (e == cudaSuccess && c >= S) e = cudaStreamWaitEvent(comp, P.d2h[b], 0);  // dY[b] drained
        if (e != cudaSuccess) {
            rc = cuda_fail(e, "host pipeline: H2D");
            break;
        }
        tr.mark(c, 2, comp);
        rc = compute(c, P.dX[b], P.dY[b], comp);
        if (rc) break;
        tr.mark(c, 3, comp);
        e = cudaEventRecord(P.kdone[b], comp);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(P.out, P.kdone[b], 0);
        tr.mark(c, 4, P.out);
        if (e == cudaSuccess) e = cudaMemcpyAsync(hd, P.dY[b], yb / yscale, cudaMemcpyDeviceToHost, P.out);
        tr.mark(c, 5, P.out);
        if (e == cudaSuccess) e = cudaEventRecord(P.d2h[b], P.out);
        if (e != cudaSuccess) rc = cuda_fail(e, "host pipeline: D2H");
        // drain two chunks behind, so the GPU always has chunks c-1 and c queued
        // while the host copies (slot c % S's Y was drained at iteration c - 1)
        if (rc == 0) rc = drain(c - 2);
    }
    if (rc == 0) rc = drain(chunks - 2);
    if (rc == 0) rc = drain(chunks - 1);
    for (cudaStream_t s : {P.in, P.comp[0], P.comp[1], P.out}) {
        const cudaError_t e = cudaStreamSynchronize(s);
        if (e != cudaSuccess && rc == 0) rc = cuda_fail(e, "host pipeline: stream sync");
    }
    return rc;
}

}  // namespace lmkan_b200
