// Model-level host runtime of the B200 path: the LMK1 container loader and the
// pure-lookup inference chain.
//
// Reference (paths relative to /root/reference/proj/include/lmkan/):
//   load_model  serialize.hpp:185-301  LMK1 = "LMK1" | u32 LE header length |
//                                      JSON header | raw LE tensors (P in
//                                      [i1][i2][pair][out] order, f64 or f32)
//   model_infer model.hpp:268-315      blocks in sequence; for a fused model
//                                      (fuse_model, fuse.hpp:105-140) every
//                                      block is a pure lookup layer (mode none,
//                                      gamma folded, no batch norm), i.e. a
//                                      chain of lmkan_forward calls
//
// The loader validates a file exactly as load_model does (same checks, same
// FormatError messages) and then streams each lookup block's P from disk in
// fixed-size chunks through pinned host buffers to the device, where a kernel
// rounds it to fp32 and scatters it into the gather kernels' layout
// [out_tile][pair][node][OT]: no host copy of the whole table and no fp64
// device copy. The chain runs the layers back to back on one stream with
// device-resident intermediate activations, replayed from a CUDA graph once a
// (rows, X, Y, stream) shape has been seen.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <list>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/lmkan_b200.h"
#include "host_pipeline.hpp"
#include "json_mini.hpp"
#include "layer_impl.hpp"

using namespace lmkan_b200;

namespace {

// ------------------------------------------------------------ LMK1 header
enum BlockType { kLmkan = 0, kMlp = 1, kBn = 2 };
enum Mode { kReluFirst = 0, kReluLast = 1, kLinear = 2, kNone = 3 };

struct BnMeta {
    int dim = 0;
    bool affine = false;
};
struct BlockMeta {
    int type = kLmkan;
    int n_in = 0, n_out = 0, G = 0, mode = kNone;
    double gamma = 0.0;
    bool has_bn = false;
    BnMeta bn;
};
struct TensorMeta {
    std::string name;
    uint64_t count = 0;  // elements
    uint64_t offset = 0; // byte offset of the tensor in the file
};
struct Lmk1 {
    int elem = 8;  // 8 = f64, 4 = f32
    std::vector<BlockMeta> blocks;
    std::vector<TensorMeta> tensors;
    std::vector<int> p_tensor;  // per block: index of its ".P" tensor, -1 if none
};

struct FormatError {  // lmkan::FormatError (errors.hpp:23-26) -> EFORMAT
    std::string msg;
};
struct InvalidArgument {  // std::invalid_argument escaping load_model -> EINVAL
    std::string msg;
};

int mode_from_string(const std::string& s) {  // model.hpp:37-43
    if (s == "relu_first") return kReluFirst;
    if (s == "relu_last") return kReluLast;
    if (s == "linear") return kLinear;
    if (s == "none") return kNone;
    throw InvalidArgument{"unknown precond mode: " + s};
}
void activation_check(const std::string& s) {  // model.hpp:155-161
    if (s != "none" && s != "relu" && s != "tanh") throw InvalidArgument{"unknown activation: " + s};
}

BnMeta bn_from_meta(const json::Value& j) {  // serialize.hpp:102-107
    BnMeta bn;
    bn.dim = static_cast<int>(j.at("dim").as_int());
    bn.affine = j.at("affine").as_bool();
    (void)j.at("momentum").as_double();
    (void)j.at("epsilon").as_double();
    (void)j.at("batches_seen").as_int();
    return bn;
}

// Reads and validates an LMK1 file the way load_model does
// (serialize.hpp:185-270 and the payload-length checks of 272-299), without
// keeping tensor data. Throws FormatError with the reference messages.
Lmk1 read_lmk1(const std::string& path) {
    FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw FormatError{"load_model: cannot open " + path};
    std::unique_ptr<FILE, int (*)(FILE*)> guard(f, std::fclose);
    char magic[4] = {};
    if (std::fread(magic, 1, 4, f) != 4 || std::memcmp(magic, "LMK1", 4) != 0)
        throw FormatError{"load_model: bad magic, not an LMK1 model file"};
    unsigned char lenb[4];
    if (std::fread(lenb, 1, 4, f) != 4) throw FormatError{"load_model: truncated header length"};
    const uint32_t hlen = static_cast<uint32_t>(lenb[0]) | (static_cast<uint32_t>(lenb[1]) << 8) |
                          (static_cast<uint32_t>(lenb[2]) << 16) | (static_cast<uint32_t>(lenb[3]) << 24);
    std::string htext(hlen, '\0');
    if (hlen && std::fread(&htext[0], 1, hlen, f) != hlen) throw FormatError{"load_model: truncated header"};
    json::Value header;
    try {
        header = json::parse(htext);
    } catch (const std::exception& e) {
        throw FormatError{std::string("load_model: header is not valid JSON: ") + e.what()};
    }
    // header.value(key, default): the default applies when the key is absent
    // (a present key of the wrong type makes nlohmann throw; treat as mismatch)
    auto str_or = [&](const char* k, const char* d) -> std::string {
        const json::Value* v = header.find(k);
        if (!v) return d;
        if (v->type != json::Value::String) throw FormatError{"load_model: unsupported format/version"};
        return v->text;
    };
    if (header.type != json::Value::Object) throw FormatError{"load_model: unsupported format/version"};
    long long version = 0;
    if (const json::Value* v = header.find("version")) {
        try {
            version = v->as_int();
        } catch (const std::exception&) {
            version = -1;
        }
    }
    if (str_or("format", "") != "LMK1" || version != 1) throw FormatError{"load_model: unsupported format/version"};
    Lmk1 m;
    const std::string dtype = str_or("dtype", "f64");
    if (dtype != "f64" && dtype != "f32") throw FormatError{"load_model: unknown dtype " + dtype};
    m.elem = dtype == "f32" ? 4 : 8;

    try {  // block skeleton (serialize.hpp:222-264)
        const json::Value& blocks = header.at("blocks");
        if (blocks.type != json::Value::Array) throw std::runtime_error("blocks must be an array");
        for (const json::Value& jb : blocks.arr) {
            BlockMeta b;
            const std::string type = jb.at("type").as_string();
            if (type == "lmkan") {
                b.type = kLmkan;
                b.n_in = static_cast<int>(jb.at("n_in").as_int());
                b.n_out = static_cast<int>(jb.at("n_out").as_int());
                b.G = static_cast<int>(jb.at("G").as_int());
                if (b.G < 3)  // build_grid (grid.hpp:45-46), called from load_model
                    throw InvalidArgument{"build_grid: G must be >= 3 (ghost rule needs two interior points)"};
                b.gamma = jb.at("gamma").as_double();
                b.mode = mode_from_string(jb.at("mode").as_string());
            } else if (type == "mlp") {
                b.type = kMlp;
                b.n_in = static_cast<int>(jb.at("n_in").as_int());
                b.n_out = static_cast<int>(jb.at("n_out").as_int());
                activation_check(jb.at("act").as_string());
            } else if (type == "bn") {
                b.type = kBn;
                b.has_bn = true;
                b.bn = bn_from_meta(jb.at("bn"));
                m.blocks.push_back(b);
                continue;
            } else {
                throw FormatError{"load_model: unknown block type " + type};
            }
            if (b.n_in < 0 || b.n_out < 0) throw std::runtime_error("negative dimension");
            if (const json::Value* jbn = jb.find("bn")) {
                b.has_bn = true;
                b.bn = bn_from_meta(*jbn);
            }
            m.blocks.push_back(b);
        }
    } catch (const FormatError&) {
        throw;
    } catch (const std::exception& e) {
        throw FormatError{std::string("load_model: malformed block metadata: ") + e.what()};
    }

    // expected manifest, in for_each_tensor order (serialize.hpp:46-86)
    std::vector<std::pair<std::string, uint64_t>> expected;
    m.p_tensor.assign(m.blocks.size(), -1);
    auto bn_tensors = [&](const BnMeta& bn, const std::string& prefix) {
        expected.emplace_back(prefix + ".running_mean", bn.dim);
        expected.emplace_back(prefix + ".running_var", bn.dim);
        if (bn.affine) {
            expected.emplace_back(prefix + ".scale", bn.dim);
            expected.emplace_back(prefix + ".shift", bn.dim);
        }
    };
    for (size_t i = 0; i < m.blocks.size(); ++i) {
        const BlockMeta& b = m.blocks[i];
        const std::string prefix = "block" + std::to_string(i);
        if (b.type == kLmkan) {
            const uint64_t G1 = static_cast<uint64_t>(b.G) + 1;
            m.p_tensor[i] = static_cast<int>(expected.size());
            expected.emplace_back(prefix + ".P", G1 * G1 * static_cast<uint64_t>(b.n_in / 2) * b.n_out);
            if (b.mode != kNone) {
                expected.emplace_back(prefix + ".linW", static_cast<uint64_t>(b.n_out) * b.n_in);
                expected.emplace_back(prefix + ".linB", static_cast<uint64_t>(b.n_out));
            }
            if (b.has_bn) bn_tensors(b.bn, prefix + ".bn");
        } else if (b.type == kMlp) {
            expected.emplace_back(prefix + ".W", static_cast<uint64_t>(b.n_out) * b.n_in);
            expected.emplace_back(prefix + ".b", static_cast<uint64_t>(b.n_out));
            if (b.has_bn) bn_tensors(b.bn, prefix + ".bn");
        } else {
            bn_tensors(b.bn, prefix + ".bn");
        }
    }
    // manifest vs skeleton (serialize.hpp:275-284)
    const json::Value* manifest = header.find("tensors");
    try {
        if (!manifest) throw std::runtime_error("key 'tensors' not found");
        if (manifest->type != json::Value::Array) throw std::runtime_error("tensors must be an array");
    } catch (const std::exception& e) {
        throw FormatError{std::string("load_model: malformed block metadata: ") + e.what()};
    }
    if (manifest->arr.size() != expected.size())
        throw FormatError{"load_model: tensor manifest does not match block metadata"};
    uint64_t offset = 8ull + hlen;
    for (size_t i = 0; i < expected.size(); ++i) {
        const json::Value& entry = manifest->arr[i];
        std::string name;
        uint64_t bytes = 0;
        try {
            name = entry.at("name").as_string();
        } catch (const std::exception& e) {
            throw FormatError{std::string("load_model: malformed block metadata: ") + e.what()};
        }
        if (name != expected[i].first) throw FormatError{"load_model: manifest order mismatch at " + expected[i].first};
        try {
            bytes = entry.at("bytes").as_u64();
        } catch (const std::exception& e) {
            throw FormatError{std::string("load_model: malformed block metadata: ") + e.what()};
        }
        if (bytes != expected[i].second * m.elem)
            throw FormatError{"load_model: declared byte count mismatch at " + expected[i].first};
        m.tensors.push_back(TensorMeta{expected[i].first, expected[i].second, offset});
        offset += bytes;
    }
    // payload length: truncated tensors and trailing bytes (serialize.hpp:286-299)
    if (std::fseek(f, 0, SEEK_END) != 0) throw FormatError{"load_model: cannot open " + path};
    const uint64_t size = static_cast<uint64_t>(std::ftell(f));
    for (const TensorMeta& t : m.tensors)
        if (t.offset + t.count * m.elem > size) throw FormatError{"load_model: truncated payload at tensor " + t.name};
    if (size > offset) throw FormatError{"load_model: trailing bytes after declared payload"};
    return m;
}

bool pure_lookup(const BlockMeta& b) { return b.type == kLmkan && b.mode == kNone && !b.has_bn; }

int format_fail(const FormatError& e) { return api::set_error(LMKAN_B200_EFORMAT, e.msg); }
int format_fail(const InvalidArgument& e) { return api::set_error(LMKAN_B200_EINVAL, e.msg); }

// ------------------------------------------------------------ streaming load
// One chunk of the reference-layout table: flat reference indices
// [f0, f0 + n) of P[node][pair][out_total] -> device layout, outputs
// [out_begin, out_begin + n_out_local) only (output-sliced layers).
template <typename T>
__global__ void relayout_chunk_kernel(const T* __restrict__ src, uint64_t f0, uint64_t n, float* __restrict__ dst,
                                      int pairs, int nodes, int n_out_total, int out_begin, int n_out_local, int OT,
                                      int NS) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t f = f0 + i;
        const int q = static_cast<int>(f % n_out_total);
        const uint64_t t = f / n_out_total;
        const int p = static_cast<int>(t % pairs);
        const int node = static_cast<int>(t / pairs);
        const int ql = q - out_begin;
        if (ql < 0 || ql >= n_out_local) continue;
        const int ot = ql / OT, qq = ql - ot * OT;
        float* d = dst + ((static_cast<size_t>(ot) * pairs + p) * nodes + node) * NS + qq;
        const float v = static_cast<float>(src[i]);
        d[0] = v;
        if (NS > OT) d[OT] = v;  // duplicated-node table: both copies
    }
}

constexpr size_t kChunkBytes = 64u << 20;  // per pinned staging buffer

// Streams tensor `t` of the file into layer L's device table (outputs
// [L->out_begin, L->out_begin + L->n_out) of an L->n_out_total-wide table).
// Double-buffered: the host reads chunk c+1 while chunk c is copied and
// scattered on the device.
int stream_table(const std::string& path, const Lmk1& m, const TensorMeta& t, lmkan_b200_layer* L) {
    FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) return api::set_error(LMKAN_B200_EFORMAT, "load_model: cannot open " + path);
    std::unique_ptr<FILE, int (*)(FILE*)> guard(f, std::fclose);
    if (std::fseek(f, static_cast<long>(t.offset), SEEK_SET) != 0)
        return api::set_error(LMKAN_B200_EFORMAT, "load_model: truncated payload at tensor " + t.name);
    cudaStream_t st = nullptr;
    void* host[2] = {nullptr, nullptr};
    void* dev[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    int rc = LMKAN_B200_OK;
    auto cleanup = [&]() {
        if (st) cudaStreamSynchronize(st);
        for (int i = 0; i < 2; ++i) {
            if (host[i]) cudaFreeHost(host[i]);
            if (dev[i]) cudaFree(dev[i]);
            if (done[i]) cudaEventDestroy(done[i]);
        }
        if (st) cudaStreamDestroy(st);
    };
    cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
        e = cudaHostAlloc(&host[i], kChunkBytes, cudaHostAllocDefault);
        if (e == cudaSuccess) e = cudaMalloc(&dev[i], kChunkBytes);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming);
    }
    // zero padding of the last output tile
    if (e == cudaSuccess) e = cudaMemsetAsync(L->table, 0, L->table_bytes, st);
    if (e != cudaSuccess) {
        rc = api::cuda_error(e, "load_model: staging buffers");
        cleanup();
        return rc;
    }
    const uint64_t per_chunk = kChunkBytes / m.elem;
    uint64_t f0 = 0;
    for (int c = 0; f0 < t.count; ++c, f0 += per_chunk) {
        const int b = c & 1;
        const uint64_t n = std::min<uint64_t>(per_chunk, t.count - f0);
        if (c >= 2 && (e = cudaEventSynchronize(done[b])) != cudaSuccess) break;  // buffer b free again
        if (std::fread(host[b], m.elem, n, f) != n) {
            rc = api::set_error(LMKAN_B200_EFORMAT, "load_model: truncated payload at tensor " + t.name);
            break;
        }
        if ((e = cudaMemcpyAsync(dev[b], host[b], n * m.elem, cudaMemcpyHostToDevice, st)) != cudaSuccess) break;
        const unsigned blocks = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, static_cast<uint64_t>(L->num_sms) * 32));
        if (m.elem == 8)
            relayout_chunk_kernel<double><<<blocks, 256, 0, st>>>(static_cast<const double*>(dev[b]), f0, n, L->table,
                                                                   L->pairs, L->nodes, L->n_out_total, L->out_begin,
                                                                   L->n_out, L->OT, L->ns);
        else
            relayout_chunk_kernel<float><<<blocks, 256, 0, st>>>(static_cast<const float*>(dev[b]), f0, n, L->table,
                                                                  L->pairs, L->nodes, L->n_out_total, L->out_begin,
                                                                  L->n_out, L->OT, L->ns);
        if ((e = cudaGetLastError()) != cudaSuccess) break;
        if ((e = cudaEventRecord(done[b], st)) != cudaSuccess) break;
    }
    if (rc == LMKAN_B200_OK && e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (rc == LMKAN_B200_OK && e != cudaSuccess) rc = api::cuda_error(e, "load_model: table upload");
    cleanup();
    return rc;
}

int load_block(const std::string& path, const Lmk1& m, int block, int out_begin, int out_end, int device,
               lmkan_b200_layer** out) {
    const BlockMeta& b = m.blocks[block];
    if (b.type != kLmkan)
        return api::set_error(LMKAN_B200_EUNSUPPORTED,
                              "lmkan_b200: block " + std::to_string(block) + " is not an lmkan lookup block");
    if (out_end < 0) out_end = b.n_out;
    if (out_begin < 0 || out_end > b.n_out || out_begin >= out_end)
        return api::set_error(LMKAN_B200_EINVAL, "layer_load: bad output slice");
    if (int rc = api::alloc_layer(b.n_in, out_end - out_begin, b.n_out, out_begin, b.G, b.gamma, device, out))
        return rc;
    if (int rc = stream_table(path, m, m.tensors[m.p_tensor[block]], *out)) {
        lmkan_b200_layer_destroy(*out);
        *out = nullptr;
        return rc;
    }
    return LMKAN_B200_OK;
}

}  // namespace

// ------------------------------------------------------------ model object
struct lmkan_b200_model {
    std::vector<lmkan_b200_layer*> layers;
    bool owns = false;
    int device = 0;
    std::mutex mu;       // device-path state below
    std::mutex host_mu;  // host-path staging
    // Per-stream ping-pong buffers for the intermediate activations, so chains
    // in flight on different streams never share them.
    struct StreamActs {
        cudaStream_t st;
        void* acts[2];
        size_t bytes;
    };
    std::vector<StreamActs> acts;
    struct GraphEntry {
        int64_t rows;
        uint64_t versions;  // sum of the layers' mutation counters at capture
        int elem;  // sizeof(XT): f32 and f64 chains on the same buffers are different graphs
        const void* X;
        void* Y;
        cudaStream_t st;
        cudaGraphExec_t exec;
    };
    std::list<GraphEntry> graphs;  // most recent first, at most kMaxGraphs
    static constexpr size_t kMaxGraphs = 12;  // host pipeline: 3 slots x (full, tail) chunk + device calls
    // host path: H2D / chain / D2H pipeline (host_pipeline.hpp)
    HostPipeline hp;

    ~lmkan_b200_model() {
        for (auto& g : graphs) cudaGraphExecDestroy(g.exec);
        for (auto& a : acts)
            for (void* p : a.acts)
                if (p) cudaFree(p);
        hp.destroy();
        if (owns)
            for (auto* L : layers) lmkan_b200_layer_destroy(L);
    }
};

namespace {

int layer_width(const lmkan_b200_layer* L, int* n_in, int* n_out) {
    return lmkan_b200_layer_info(L, n_in, n_out, nullptr, nullptr, nullptr, nullptr);
}

// model.hpp:268-315 for a pure-lookup chain: widths are checked the way
// precond_forward does (model.hpp:59, require_width "precond_forward").
int check_chain(const lmkan_b200_model* M) {
    for (size_t b = 1; b < M->layers.size(); ++b) {
        int prev_out = 0, n_in = 0;
        layer_width(M->layers[b - 1], nullptr, &prev_out);
        layer_width(M->layers[b], &n_in, nullptr);
        if (prev_out != n_in)
            return api::set_error(LMKAN_B200_EINVAL, "precond_forward: expected width " + std::to_string(n_in) +
                                                         ", got " + std::to_string(prev_out));
    }
    return LMKAN_B200_OK;
}

// Ping-pong activation buffers of stream `st`, big enough for `rows` rows of
// every intermediate width. Growing them drops the graphs captured on `st`.
int ensure_acts(lmkan_b200_model* M, int64_t rows, size_t elem, cudaStream_t st, void** out) {
    size_t need = 0;
    for (size_t b = 0; b + 1 < M->layers.size(); ++b) {
        int n_out = 0;
        layer_width(M->layers[b], nullptr, &n_out);
        need = std::max(need, static_cast<size_t>(rows) * n_out * elem);
    }
    lmkan_b200_model::StreamActs* sa = nullptr;
    for (auto& a : M->acts)
        if (a.st == st) sa = &a;
    if (!sa) {
        M->acts.push_back({st, {nullptr, nullptr}, 0});
        sa = &M->acts.back();
    }
    if (sa->bytes < need) {
        if (sa->acts[0] || sa->acts[1]) {
            cudaStreamSynchronize(st);  // work (and graphs) using the old buffers must be done
            for (auto it = M->graphs.begin(); it != M->graphs.end();) {
                if (it->st == st) {
                    cudaGraphExecDestroy(it->exec);
                    it = M->graphs.erase(it);
                } else {
                    ++it;
                }
            }
            for (void*& p : sa->acts) {
                if (p) cudaFree(p);
                p = nullptr;
            }
            sa->bytes = 0;
        }
        for (void*& p : sa->acts) {
            cudaError_t e = cudaMalloc(&p, need);
            if (e != cudaSuccess) return api::cuda_error(e, "model_infer: activation buffers");
        }
        sa->bytes = need;
    }
    out[0] = sa->acts[0];
    out[1] = sa->acts[1];
    return LMKAN_B200_OK;
}

template <typename XT>
int run_chain(lmkan_b200_model* M, const XT* X, XT* Y, int64_t rows, cudaStream_t st, void* const* acts) {
    if constexpr (sizeof(XT) == 4)  // fp32: fused chain (next layer's records from the epilogue)
        return api::forward_chain_f32(M->layers.data(), static_cast<int>(M->layers.size()), X, Y, rows, acts, st);
    const XT* cur = X;
    const size_t n = M->layers.size();
    for (size_t b = 0; b < n; ++b) {
        XT* dst = b + 1 == n ? Y : static_cast<XT*>(acts[b & 1]);
        if (int rc = api::forward_device(M->layers[b], cur, dst, rows, st)) return rc;
        cur = dst;
    }
    return LMKAN_B200_OK;
}

bool graphs_enabled() {
    const char* e = std::getenv("LMKAN_B200_GRAPH");
    return !(e && e[0] == '0');
}

template <typename XT>
int infer_device(lmkan_b200_model* M, const XT* X, XT* Y, int64_t rows, cudaStream_t st) {
    if (!M) return api::set_error(LMKAN_B200_EINVAL, "model_infer: null model");
    if (rows < 0) return api::set_error(LMKAN_B200_EINVAL, "model_infer: negative row count");
    if (M->layers.empty()) return api::set_error(LMKAN_B200_EINVAL, "model_infer: empty model");
    if (rows == 0) return LMKAN_B200_OK;
    if (!X || !Y) return api::set_error(LMKAN_B200_EINVAL, "model_infer: null X or Y");
    std::lock_guard<std::mutex> lock(M->mu);
    if (int rc = check_chain(M)) return rc;
    int dev_prev = 0;
    cudaGetDevice(&dev_prev);
    if (dev_prev != M->device) cudaSetDevice(M->device);
    struct Restore {
        int d, cur;
        ~Restore() {
            if (d != cur) cudaSetDevice(d);
        }
    } restore{dev_prev, M->device};
    void* acts[2];
    if (int rc = ensure_acts(M, rows, sizeof(XT), st, acts)) return rc;
    // graph replay for a (rows, X, Y, stream) seen before (not on the legacy
    // stream, which cannot be captured, nor while the caller is capturing)
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    const bool graphable = graphs_enabled() && st != nullptr &&
                           cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusNone;
    uint64_t vsum = 0;
    for (const auto* L : M->layers) vsum += L->version;
    if (graphable) {
        for (auto it = M->graphs.begin(); it != M->graphs.end(); ++it) {
            if (it->rows == rows && it->versions == vsum && it->elem == static_cast<int>(sizeof(XT)) && it->X == X &&
                it->Y == Y && it->st == st) {
                M->graphs.splice(M->graphs.begin(), M->graphs, it);
                cudaError_t e = cudaGraphLaunch(M->graphs.front().exec, st);
                if (e != cudaSuccess) return api::cuda_error(e, "model_infer: graph launch");
                return LMKAN_B200_OK;
            }
        }
    }
    // first sight: run eagerly (validates every launch), then capture
    if (int rc = run_chain<XT>(M, X, Y, rows, st, acts)) return rc;
    if (!graphable) return LMKAN_B200_OK;
    cudaGraph_t g = nullptr;
    if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
        cudaGetLastError();
        return LMKAN_B200_OK;
    }
    const int rc = run_chain<XT>(M, X, Y, rows, st, acts);
    const cudaError_t e_end = cudaStreamEndCapture(st, &g);
    cudaGraphExec_t exec = nullptr;
    if (rc == LMKAN_B200_OK && e_end == cudaSuccess && g &&
        cudaGraphInstantiateWithFlags(&exec, g, cudaGraphInstantiateFlagAutoFreeOnLaunch) == cudaSuccess) {
        M->graphs.push_front({rows, vsum, static_cast<int>(sizeof(XT)), X, Y, st, exec});
        if (M->graphs.size() > lmkan_b200_model::kMaxGraphs) {
            cudaGraphExecDestroy(M->graphs.back().exec);
            M->graphs.pop_back();
        }
    }
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();  // a failed capture only costs the replay, not the result
    return LMKAN_B200_OK;
}

// Drop-in host path: row chunks through the model's three-stream host pipeline
// (H2D, chain and D2H of different chunks overlap, host_pipeline.hpp); each
// chunk shape replays its own captured graph of the chain.
template <typename XT>
int infer_host(lmkan_b200_model* M, const XT* X, XT* Y, int64_t rows) {
    if (!M || M->layers.empty()) return api::set_error(LMKAN_B200_EINVAL, "model_infer: null or empty model");
    if (rows < 0) return api::set_error(LMKAN_B200_EINVAL, "model_infer: negative row count");
    if (rows == 0) return LMKAN_B200_OK;
    if (!X || !Y) return api::set_error(LMKAN_B200_EINVAL, "model_infer: null X or Y");
    std::lock_guard<std::mutex> lock(M->host_mu);
    int n_in = 0, n_out = 0;
    layer_width(M->layers.front(), &n_in, nullptr);
    layer_width(M->layers.back(), nullptr, &n_out);
    int dev_prev = 0;
    cudaGetDevice(&dev_prev);
    if (dev_prev != M->device) cudaSetDevice(M->device);
    struct Restore {
        int d, cur;
        ~Restore() {
            if (d != cur) cudaSetDevice(d);
        }
    } restore{dev_prev, M->device};
    // ~4 chunks of at least 65536 rows (LMKAN_B200_MODEL_CHUNKS overrides the count)
    const char* ce = std::getenv("LMKAN_B200_MODEL_CHUNKS");
    const int64_t nch = std::max<int64_t>(1, ce ? std::atoi(ce) : 4);
    const int64_t chunk = std::min<int64_t>(rows, std::max<int64_t>((rows + nch - 1) / nch, 65536));
    HostPipeline& P = M->hp;
    cudaError_t e = P.init(M->device);
    if (e == cudaSuccess)
        e = P.reserve(sizeof(XT) * static_cast<size_t>(chunk) * n_in, sizeof(XT) * static_cast<size_t>(chunk) * n_out);
    if (e != cudaSuccess) return api::cuda_error(e, "model_infer: host staging");
    auto n_of = [&](int64_t c) { return std::min(chunk, rows - c * chunk); };
    return run_host_pipeline(
        P, (rows + chunk - 1) / chunk,
        [&](int64_t c, const void** h, size_t* b) {
            *h = X + c * chunk * n_in;
            *b = sizeof(XT) * static_cast<size_t>(n_of(c)) * n_in;
        },
        [&](int64_t c, void** h, size_t* b) {
            *h = Y + c * chunk * n_out;
            *b = sizeof(XT) * static_cast<size_t>(n_of(c)) * n_out;
        },
        [&](int64_t c, void* dX, void* dY, cudaStream_t st) {
            return infer_device<XT>(M, static_cast<const XT*>(dX), static_cast<XT*>(dY), n_of(c), st);
        },
        [](cudaError_t err, const char* what) { return api::cuda_error(err, what); });
}

}  // namespace

// =================================================================== C-ABI
extern "C" {

int lmkan_b200_lmk1_inspect(const char* path, int* n_blocks, int* dtype_bytes, int* pure_lookup_out) {
    if (!path) return api::set_error(LMKAN_B200_EINVAL, "lmk1_inspect: null path");
    try {
        const Lmk1 m = read_lmk1(path);
        if (n_blocks) *n_blocks = static_cast<int>(m.blocks.size());
        if (dtype_bytes) *dtype_bytes = m.elem;
        if (pure_lookup_out) {
            bool all = !m.blocks.empty();
            for (const auto& b : m.blocks) all = all && pure_lookup(b);
            *pure_lookup_out = all ? 1 : 0;
        }
    } catch (const FormatError& e) {
        return format_fail(e);
    } catch (const InvalidArgument& e) {
        return format_fail(e);
    }
    return LMKAN_B200_OK;
}

int lmkan_b200_lmk1_block(const char* path, int block, int* type, int* n_in, int* n_out, int* G, double* gamma,
                          int* mode, int* has_bn, uint64_t* p_offset) {
    if (!path) return api::set_error(LMKAN_B200_EINVAL, "lmk1_block: null path");
    try {
        const Lmk1 m = read_lmk1(path);
        if (block < 0 || block >= static_cast<int>(m.blocks.size()))
            return api::set_error(LMKAN_B200_EINVAL, "lmk1_block: block index out of range");
        const BlockMeta& b = m.blocks[block];
        if (type) *type = b.type;
        if (n_in) *n_in = b.n_in;
        if (n_out) *n_out = b.n_out;
        if (G) *G = b.G;
        if (gamma) *gamma = b.gamma;
        if (mode) *mode = b.mode;
        if (has_bn) *has_bn = b.has_bn ? 1 : 0;
        if (p_offset) *p_offset = m.p_tensor[block] >= 0 ? m.tensors[m.p_tensor[block]].offset : 0;
    } catch (const FormatError& e) {
        return format_fail(e);
    } catch (const InvalidArgument& e) {
        return format_fail(e);
    }
    return LMKAN_B200_OK;
}

int lmkan_b200_layer_load_lmk1(const char* path, int block, int out_begin, int out_end, int device,
                               lmkan_b200_layer** out) {
    if (!path || !out) return api::set_error(LMKAN_B200_EINVAL, "layer_load: null argument");
    *out = nullptr;
    try {
        const Lmk1 m = read_lmk1(path);
        if (block < 0 || block >= static_cast<int>(m.blocks.size()))
            return api::set_error(LMKAN_B200_EINVAL, "layer_load: block index out of range");
        return load_block(path, m, block, out_begin, out_end, device, out);
    } catch (const FormatError& e) {
        return format_fail(e);
    } catch (const InvalidArgument& e) {
        return format_fail(e);
    }
}

int lmkan_b200_model_load(const char* path, int device, lmkan_b200_model** out) {
    if (!path || !out) return api::set_error(LMKAN_B200_EINVAL, "model_load: null argument");
    *out = nullptr;
    Lmk1 m;
    try {
        m = read_lmk1(path);
    } catch (const FormatError& e) {
        return format_fail(e);
    } catch (const InvalidArgument& e) {
        return format_fail(e);
    }
    if (m.blocks.empty()) return api::set_error(LMKAN_B200_EUNSUPPORTED, "model_load: model has no blocks");
    for (size_t i = 0; i < m.blocks.size(); ++i) {
        const BlockMeta& b = m.blocks[i];
        if (!pure_lookup(b)) {
            static const char* kModeNames[] = {"relu_first", "relu_last", "linear", "none"};
            std::string what = b.type == kMlp ? "an mlp block" : b.type == kBn ? "a batch-norm block" : "an lmkan block";
            if (b.type == kLmkan && b.mode != kNone) what = std::string("a preconditioned lmkan block (mode ") +
                                                         kModeNames[b.mode] + ")";
            if (b.type != kBn && b.has_bn) what += " with a batch norm";
            return api::set_error(LMKAN_B200_EUNSUPPORTED,
                                  "model_load: block " + std::to_string(i) + " is " + what +
                                      "; the B200 path runs fused pure-lookup models (fuse_model, fuse.hpp:105-140)");
        }
    }
    auto M = std::make_unique<lmkan_b200_model>();
    M->owns = true;
    M->device = device;
    for (size_t i = 0; i < m.blocks.size(); ++i) {
        lmkan_b200_layer* L = nullptr;
        try {
            if (int rc = load_block(path, m, static_cast<int>(i), 0, -1, device, &L)) return rc;  // M frees earlier layers
        } catch (const FormatError& e) {
            return format_fail(e);
        }
        M->layers.push_back(L);
    }
    *out = M.release();
    return LMKAN_B200_OK;
}

int lmkan_b200_model_create(lmkan_b200_layer* const* layers, int n_layers, lmkan_b200_model** out) {
    if (!out || !layers || n_layers <= 0) return api::set_error(LMKAN_B200_EINVAL, "model_create: bad arguments");
    *out = nullptr;
    auto M = std::make_unique<lmkan_b200_model>();
    int dev0 = -1;
    for (int i = 0; i < n_layers; ++i) {
        if (!layers[i]) return api::set_error(LMKAN_B200_EINVAL, "model_create: null layer");
        if (layers[i]->exact)
            return api::set_error(LMKAN_B200_EINVAL, "model_create: reference-precision layers are not chained on the device");
        int d = 0;
        lmkan_b200_layer_info(layers[i], nullptr, nullptr, nullptr, &d, nullptr, nullptr);
        if (dev0 >= 0 && d != dev0) return api::set_error(LMKAN_B200_EINVAL, "model_create: layers on different devices");
        dev0 = d;
        M->layers.push_back(layers[i]);
    }
    M->device = dev0;
    M->owns = false;
    *out = M.release();
    return LMKAN_B200_OK;
}

int lmkan_b200_model_info(const lmkan_b200_model* M, int* n_blocks, int* in_dim, int* out_dim, int* device) {
    if (!M) return api::set_error(LMKAN_B200_EINVAL, "model_info: null model");
    if (n_blocks) *n_blocks = static_cast<int>(M->layers.size());
    if (in_dim) *in_dim = 0;
    if (out_dim) *out_dim = 0;
    if (!M->layers.empty()) {
        if (in_dim) layer_width(M->layers.front(), in_dim, nullptr);
        if (out_dim) layer_width(M->layers.back(), nullptr, out_dim);
    }
    if (device) *device = M->device;
    return LMKAN_B200_OK;
}

int lmkan_b200_model_layer(const lmkan_b200_model* M, int block, lmkan_b200_layer** layer) {
    if (!M || !layer) return api::set_error(LMKAN_B200_EINVAL, "model_layer: null argument");
    if (block < 0 || block >= static_cast<int>(M->layers.size()))
        return api::set_error(LMKAN_B200_EINVAL, "model_layer: block index out of range");
    *layer = M->layers[block];
    return LMKAN_B200_OK;
}

int lmkan_b200_model_infer_f32(lmkan_b200_model* M, const float* X, float* Y, int64_t rows, void* stream) {
    return infer_device<float>(M, X, Y, rows, static_cast<cudaStream_t>(stream));
}
int lmkan_b200_model_infer_f64(lmkan_b200_model* M, const double* X, double* Y, int64_t rows, void* stream) {
    return infer_device<double>(M, X, Y, rows, static_cast<cudaStream_t>(stream));
}
int lmkan_b200_model_infer_host_f64(lmkan_b200_model* M, const double* X, double* Y, int64_t rows,
                                    size_t /*workers*/) {
    return infer_host<double>(M, X, Y, rows);
}
int lmkan_b200_model_infer_host_f32(lmkan_b200_model* M, const float* X, float* Y, int64_t rows,
                                    size_t /*workers*/) {
    return infer_host<float>(M, X, Y, rows);
}

int lmkan_b200_model_destroy(lmkan_b200_model* M) {
    delete M;
    return LMKAN_B200_OK;
}

}  // extern "C"
