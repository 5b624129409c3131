// lmkan_b200/lmkan.hpp — C++ host API of the B200 lmKAN layer forward.
//
// Restates the reference's layer interface (paths relative to
// /root/reference/proj/include/lmkan/) on top of the C-ABI in lmkan_b200.h:
//   Matrix, require_width          matrix.hpp:11-44
//   SigmaGrid, build_grid           grid.hpp:33-68
//   sigma, interval_index, preamble grid.hpp:10-17, 72-101 (index: threshold form, bit-exact)
//   flops_main_term, param_count    costs.hpp:14-29
//   LmKanLayer                      layer.hpp:24-61 (same fields and P layout)
//   default_init_scale, init_layer  layer.hpp:63-86 (bit-identical table)
//   lmkan_forward                   layer.hpp:108-134 (same signature)
//   worker_count                    threading.hpp:11-19
//   lmkan_backward                  layer.hpp:141-202 (same signature; bit-
//                                   identical results for the same workers)
//   FormatError                     errors.hpp:23-26
//   load_model, model_infer         serialize.hpp:185-301, model.hpp:313-316,
//                                   for fused pure-lookup models (DeviceModel)
// Existing callers switch with `namespace lmkan = lmkan_b200;` (see
// INTEGRATION.md). Errors: std::invalid_argument where the reference throws it
// (same messages), std::runtime_error for CUDA failures. There is no CPU
// compute path: lmkan_forward runs on the layer's GPU (LmKanLayer::device).
//
// The layer keeps a prepared device table (fp32, [out_tile][pair][node][OT])
// next to the host P. It is rebuilt whenever P may have changed since the last
// forward (P is a ParamVector: non-const access bumps a generation counter, an
// O(1) check per call) or the shape / device changed.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <initializer_list>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <string_view>
#include <thread>
#include <vector>

#include "../lmkan_b200.h"

namespace lmkan_b200 {

// errors.hpp:23-26: malformed or truncated model file.
struct FormatError : std::runtime_error {
    explicit FormatError(const std::string& msg) : std::runtime_error(msg) {}
};

namespace detail {
inline void throw_status(int rc, const char* where) {
    if (rc == LMKAN_B200_OK) return;
    const std::string msg = lmkan_b200_last_error();
    if (rc == LMKAN_B200_EINVAL) throw std::invalid_argument(msg);
    if (rc == LMKAN_B200_EFORMAT) throw FormatError(msg);
    throw std::runtime_error(std::string(where) + ": " + msg);
}
}  // namespace detail

// Dense row-major matrix of doubles, rows = batch (matrix.hpp:11-38).
class Matrix {
public:
    Matrix() = default;
    Matrix(std::size_t rows, std::size_t cols, double fill = 0.0)
        : rows_(rows), cols_(cols), data_(rows * cols, fill) {}
    std::size_t rows() const { return rows_; }
    std::size_t cols() const { return cols_; }
    std::size_t size() const { return data_.size(); }
    double& operator()(std::size_t r, std::size_t c) { return data_[r * cols_ + c]; }
    double operator()(std::size_t r, std::size_t c) const { return data_[r * cols_ + c]; }
    double* row(std::size_t r) { return data_.data() + r * cols_; }
    const double* row(std::size_t r) const { return data_.data() + r * cols_; }
    double* data() { return data_.data(); }
    const double* data() const { return data_.data(); }
    void fill(double v) { std::fill(data_.begin(), data_.end(), v); }
    bool same_shape(const Matrix& o) const { return rows_ == o.rows_ && cols_ == o.cols_; }

private:
    std::size_t rows_ = 0, cols_ = 0;
    std::vector<double> data_;
};

// matrix.hpp:40-44 — same exception type and message.
inline void require_width(const Matrix& m, std::size_t cols, const char* what) {
    if (m.cols() != cols)
        throw std::invalid_argument(std::string(what) + ": expected width " + std::to_string(cols) + ", got " +
                                    std::to_string(m.cols()));
}

// grid.hpp:33-39
struct SigmaGrid {
    int G = 0;
    std::vector<double> points;     // G+1, ghost points at both ends
    std::vector<double> inv_areas;  // G*G, [i1*G + i2]
    std::vector<double> thresholds; // G-1 cell-locate thresholds (lmkan_b200_thresholds)
    double inv_area(int i1, int i2) const { return inv_areas[static_cast<std::size_t>(i1) * G + i2]; }
};

// grid.hpp:44-68 (throws std::invalid_argument for G < 3).
inline SigmaGrid build_grid(int G) {
    SigmaGrid g;
    g.G = G;
    g.points.assign(G >= 0 ? G + 1 : 0, 0.0);
    g.inv_areas.assign(G > 0 ? static_cast<std::size_t>(G) * G : 0, 0.0);
    detail::throw_status(lmkan_b200_build_grid(G, g.points.data(), g.inv_areas.data()), "build_grid");
    g.thresholds.assign(G - 1, 0.0);
    detail::throw_status(lmkan_b200_thresholds(G, g.thresholds.data(), nullptr), "build_grid");
    return g;
}

// grid.hpp:10-17: the percentile-grid generator (host, fp64; NaN propagates).
inline double sigma(double x) {
    const double t = std::exp(-std::fabs(x));
    return x > 0.0 ? 1.0 - 0.5 * t : 0.5 * t;
}

// grid.hpp:20-24: analytic inverse of sigma on (0, 1); std::domain_error outside.
inline double sigma_inv(double p) {
    if (!(p > 0.0 && p < 1.0)) throw std::domain_error("sigma_inv: p must lie in (0, 1)");
    if (p > 0.5) return -std::log(2.0 * (1.0 - p));
    return std::log(2.0 * p);
}

// grid.hpp:72-75, bit-exact: #{k : x >= t_k} (NaN -> 0).
inline int interval_index(const SigmaGrid& grid, double x) {
    int i = 0;
    for (double t : grid.thresholds) i += x >= t;
    return i;
}

// grid.hpp:77-101: cell indices and the four bilinear weights of one 2D
// argument pair (host, fp64, the reference's operation order).
struct Preamble {
    int i1 = 0, i2 = 0;
    double w00 = 0, w10 = 0, w01 = 0, w11 = 0;
};
inline Preamble preamble(const SigmaGrid& grid, double x1, double x2) {
    Preamble r;
    r.i1 = interval_index(grid, x1);
    r.i2 = interval_index(grid, x2);
    const double a = grid.points[r.i1 + 1] - x1;
    const double b = x1 - grid.points[r.i1];
    const double c = grid.points[r.i2 + 1] - x2;
    const double d = x2 - grid.points[r.i2];
    const double inv = grid.inv_area(r.i1, r.i2);
    r.w00 = a * c * inv;
    r.w10 = b * c * inv;
    r.w01 = a * d * inv;
    r.w11 = b * d * inv;
    return r;
}

// rng.hpp:19-79: the reference's named random stream, reproduced bit for bit
// (the same keying, engine and transforms) so data drawn by existing callers
// and tests is unchanged: key = splitmix64 finalizer of seed ^ (FNV-1a(name) +
// golden ratio), engine std::mt19937_64(key), uniforms from the top 53 bits,
// normals by Box-Muller returning the cosine half first and caching the sine.
class RandomStream {
public:
    RandomStream(std::uint64_t seed, std::string_view name) : key_(derive(seed, name)), eng_(key_) {}
    RandomStream split(std::string_view child) const { return RandomStream(key_, child); }
    std::uint64_t next_u64() { return eng_(); }
    double uniform() { return static_cast<double>(eng_() >> 11) * 0x1.0p-53; }
    double uniform_open() {
        double u = uniform();
        while (u == 0.0) u = uniform();
        return u;
    }
    double normal() {
        if (have_) {
            have_ = false;
            return spare_;
        }
        const double u1 = uniform_open(), u2 = uniform();
        const double rad = std::sqrt(-2.0 * std::log(u1)), ang = 2.0 * M_PI * u2;
        spare_ = rad * std::sin(ang);
        have_ = true;
        return rad * std::cos(ang);
    }

private:
    static std::uint64_t derive(std::uint64_t seed, std::string_view name) {
        std::uint64_t h = 0xcbf29ce484222325ull;
        for (unsigned char ch : name) h = (h ^ ch) * 0x100000001b3ull;
        std::uint64_t z = seed ^ (h + 0x9e3779b97f4a7c15ull);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    }
    std::uint64_t key_;
    std::mt19937_64 eng_;
    bool have_ = false;
    double spare_ = 0.0;
};

// func2d.hpp:14-24: one 2D function as its (G+1) x (G+1) node coefficients,
// row-major [i1 (G+1) + i2] (indices 0 and G sit on the ghost points).
struct Func2D {
    int G = 0;
    std::vector<double> coeffs;
    Func2D() = default;
    explicit Func2D(int G_, double fill = 0.0) : G(G_), coeffs(static_cast<std::size_t>(G_ + 1) * (G_ + 1), fill) {}
    double& at(int i1, int i2) { return coeffs[static_cast<std::size_t>(i1) * (G + 1) + i2]; }
    double at(int i1, int i2) const { return coeffs[static_cast<std::size_t>(i1) * (G + 1) + i2]; }
};

// func2d.hpp:26-48: the 1D hat basis function i in [0, G] at x, evaluated from
// the grid points alone (1 at points[i], 0 at its neighbours); the hats of the
// two unbounded edge intervals keep their slope out to +-infinity, as the
// ghost-point extrapolation of the lookup does.
inline double basis_weight_1d(const SigmaGrid& grid, int i, double x) {
    const int G = grid.G;
    if (i < 0 || i > G) throw std::out_of_range("basis_weight_1d: index outside [0, G]");
    const std::vector<double>& t = grid.points;
    const bool left_open = i == 1, right_open = i == G - 1;
    if (i == 0) return x < t[1] ? (t[1] - x) / (t[1] - t[0]) : 0.0;
    if (i == G) return x > t[G - 1] ? (x - t[G - 1]) / (t[G] - t[G - 1]) : 0.0;
    if (x < t[i]) return (left_open || x >= t[i - 1]) ? (x - t[i - 1]) / (t[i] - t[i - 1]) : 0.0;
    return (right_open || x <= t[i + 1]) ? (t[i + 1] - x) / (t[i + 1] - t[i]) : 0.0;
}

// func2d.hpp:50-57: the O(1) bilinear lookup of one 2D function.
inline double eval2d(const SigmaGrid& grid, const Func2D& f, double x1, double x2);

// func2d.hpp:62-73: the dense O(G^2) basis-product sum eval2d must equal.
inline double eval2d_dense_oracle(const SigmaGrid& grid, const Func2D& f, double x1, double x2) {
    double sum = 0.0;
    for (int i1 = 0; i1 <= grid.G; ++i1) {
        const double u = basis_weight_1d(grid, i1, x1);
        if (u == 0.0) continue;
        for (int i2 = 0; i2 <= grid.G; ++i2) sum += f.at(i1, i2) * u * basis_weight_1d(grid, i2, x2);
    }
    return sum;
}

// func2d.hpp:75-105: input derivatives of the bilinear cell form and the four
// coefficient weights of the active cell.
struct Grad2D {
    double df_dx1 = 0, df_dx2 = 0;
    int i1 = 0, i2 = 0;
    double w00 = 0, w10 = 0, w01 = 0, w11 = 0;
};
inline Grad2D grad2d(const SigmaGrid& grid, const Func2D& f, double x1, double x2);

// std::vector<double> with a mutation generation, the type of LmKanLayer::P.
// Every non-const access (element references, data(), iterators, assign /
// resize / clear / push_back, assignment, and the conversion to
// std::vector<double>& used by functions taking the reference's vector)
// bumps the generation; const access does not. lmkan_forward re-uploads the
// device table only when the generation moved since the last upload: O(1)
// per call instead of hashing P. Writes through a pointer or iterator taken
// BEFORE a forward and used after it are not seen; take it again (as the
// reference's own optimizer does every step, model.hpp:382-386) or call
// touch().
class ParamVector {
public:
    using vector_type = std::vector<double>;
    using value_type = double;
    using size_type = std::size_t;
    using iterator = vector_type::iterator;
    using const_iterator = vector_type::const_iterator;

    ParamVector() = default;
    explicit ParamVector(size_type n, double v = 0.0) : v_(n, v) {}
    ParamVector(std::initializer_list<double> l) : v_(l) {}
    ParamVector(const vector_type& v) : v_(v) {}
    ParamVector(vector_type&& v) : v_(std::move(v)) {}
    ParamVector(const ParamVector& o) : v_(o.v_) {}
    ParamVector(ParamVector&& o) noexcept : v_(std::move(o.v_)) { o.touch(); }
    ParamVector& operator=(const ParamVector& o) {
        v_ = o.v_;
        touch();
        return *this;
    }
    ParamVector& operator=(ParamVector&& o) noexcept {
        v_ = std::move(o.v_);
        touch();
        o.touch();
        return *this;
    }
    ParamVector& operator=(vector_type v) {
        v_ = std::move(v);
        touch();
        return *this;
    }

    // const access: no generation change
    size_type size() const { return v_.size(); }
    bool empty() const { return v_.empty(); }
    const double* data() const { return v_.data(); }
    const double& operator[](size_type i) const { return v_[i]; }
    const double& at(size_type i) const { return v_.at(i); }
    const double& front() const { return v_.front(); }
    const double& back() const { return v_.back(); }
    const_iterator begin() const { return v_.begin(); }
    const_iterator end() const { return v_.end(); }
    const_iterator cbegin() const { return v_.cbegin(); }
    const_iterator cend() const { return v_.cend(); }
    operator const vector_type&() const { return v_; }
    const vector_type& vec() const { return v_; }

    // mutable access: bumps the generation
    double* data() { return touch(), v_.data(); }
    double& operator[](size_type i) { return touch(), v_[i]; }
    double& at(size_type i) { return touch(), v_.at(i); }
    double& front() { return touch(), v_.front(); }
    double& back() { return touch(), v_.back(); }
    iterator begin() { return touch(), v_.begin(); }
    iterator end() { return touch(), v_.end(); }
    operator vector_type&() { return touch(), v_; }
    vector_type& vec() { return touch(), v_; }
    void assign(size_type n, double v) { touch(), v_.assign(n, v); }
    template <class It>
    void assign(It a, It b) { touch(), v_.assign(a, b); }
    void resize(size_type n, double v = 0.0) { touch(), v_.resize(n, v); }
    void clear() { touch(), v_.clear(); }
    void push_back(double v) { touch(), v_.push_back(v); }
    void swap(ParamVector& o) { touch(), o.touch(), v_.swap(o.v_); }
    void swap(vector_type& o) { touch(), v_.swap(o); }

    std::uint64_t generation() const { return gen_; }
    void touch() { ++gen_; }

    friend bool operator==(const ParamVector& a, const ParamVector& b) { return a.v_ == b.v_; }
    friend bool operator!=(const ParamVector& a, const ParamVector& b) { return a.v_ != b.v_; }
    friend bool operator==(const ParamVector& a, const vector_type& b) { return a.v_ == b; }
    friend bool operator!=(const ParamVector& a, const vector_type& b) { return a.v_ != b; }

private:
    vector_type v_;
    std::uint64_t gen_ = 0;
};

inline double eval2d(const SigmaGrid& grid, const Func2D& f, double x1, double x2) {
    const Preamble c = preamble(grid, x1, x2);
    const std::size_t row = static_cast<std::size_t>(grid.G) + 1, n = c.i1 * row + c.i2;
    const double* k = f.coeffs.data();
    return c.w00 * k[n] + c.w01 * k[n + 1] + c.w10 * k[n + row] + c.w11 * k[n + row + 1];
}

inline Grad2D grad2d(const SigmaGrid& grid, const Func2D& f, double x1, double x2) {
    const Preamble c = preamble(grid, x1, x2);
    Grad2D g;
    g.i1 = c.i1;
    g.i2 = c.i2;
    g.w00 = c.w00;
    g.w10 = c.w10;
    g.w01 = c.w01;
    g.w11 = c.w11;
    const double f00 = f.at(c.i1, c.i2), f10 = f.at(c.i1 + 1, c.i2);
    const double f01 = f.at(c.i1, c.i2 + 1), f11 = f.at(c.i1 + 1, c.i2 + 1);
    const double inv = grid.inv_area(c.i1, c.i2);
    const double lo1 = grid.points[c.i1], hi1 = grid.points[c.i1 + 1];
    const double lo2 = grid.points[c.i2], hi2 = grid.points[c.i2 + 1];
    g.df_dx1 = ((f10 - f00) * (hi2 - x2) + (f11 - f01) * (x2 - lo2)) * inv;
    g.df_dx2 = ((f01 - f00) * (hi1 - x1) + (f11 - f10) * (x1 - lo1)) * inv;
    return g;
}

namespace detail {
struct Prepared {
    lmkan_b200_layer* h = nullptr;
    int n_in = 0, n_out = 0, G = 0, device = 0;
    const double* data = nullptr;
    std::size_t size = 0;
    std::uint64_t generation = 0;
    int precision = 32;
    ~Prepared() {
        if (h) lmkan_b200_layer_destroy(h);
    }
};
}  // namespace detail

// Arithmetic of a layer's device forward: 32 = the fp32 gather (the product
// path, |y - y_ref| <= 1e-5 max(1, |y_ref|)); 64 = reference precision, Y
// bit-identical to the reference's lmkan_forward (lmkan_b200_layer_create_exact).
// New layers take LMKAN_B200_PRECISION (32 / 64 / fp32 / fp64), default 32.
inline int default_precision() {
    const char* e = std::getenv("LMKAN_B200_PRECISION");
    if (!e) return 32;
    const std::string v(e);
    return (v == "64" || v == "fp64" || v == "f64") ? 64 : 32;
}

// layer.hpp:24-61. Same public fields and the same P layout
// [i1][i2][pair][out] (out fastest); `device` selects the GPU.
struct LmKanLayer {
    int n_in = 0;
    int n_out = 0;
    SigmaGrid grid;
    ParamVector P;  // std::vector<double> semantics; tracks modifications (see ParamVector)
    double gamma = 0.0;
    int device = 0;
    int precision = default_precision();  // 32 or 64, see default_precision

    LmKanLayer() = default;
    // Copies share no device state: a copied layer (whose P the caller may then
    // edit) prepares its own table on first use.
    LmKanLayer(const LmKanLayer& o)
        : n_in(o.n_in), n_out(o.n_out), grid(o.grid), P(o.P), gamma(o.gamma), device(o.device),
          precision(o.precision) {}
    LmKanLayer& operator=(const LmKanLayer& o) {
        if (this != &o) {
            n_in = o.n_in; n_out = o.n_out; grid = o.grid; P = o.P; gamma = o.gamma; device = o.device;
            precision = o.precision;
            cache_.reset();
        }
        return *this;
    }
    LmKanLayer(LmKanLayer&&) = default;
    LmKanLayer& operator=(LmKanLayer&&) = default;

    int pairs() const { return n_in / 2; }
    std::size_t param_count() const { return P.size(); }
    std::size_t node_offset(int i1, int i2) const {
        const std::size_t per_node = static_cast<std::size_t>(pairs()) * n_out;
        return (static_cast<std::size_t>(i1) * (grid.G + 1) + i2) * per_node;
    }
    double* node_slice(int i1, int i2, int pair) {
        return P.data() + node_offset(i1, i2) + static_cast<std::size_t>(pair) * n_out;
    }
    const double* node_slice(int i1, int i2, int pair) const {
        return P.data() + node_offset(i1, i2) + static_cast<std::size_t>(pair) * n_out;
    }

    // layer.hpp:47-60: one function's (pair, out) coefficient sheet as a Func2D, and back.
    Func2D sheet(int pair, int out) const {
        Func2D f(grid.G);
        for (int i1 = 0; i1 <= grid.G; ++i1)
            for (int i2 = 0; i2 <= grid.G; ++i2) f.at(i1, i2) = node_slice(i1, i2, pair)[out];
        return f;
    }
    void set_sheet(int pair, int out, const Func2D& f) {
        double* base = P.data();  // one generation bump for the whole sheet
        for (int i1 = 0; i1 <= grid.G; ++i1)
            for (int i2 = 0; i2 <= grid.G; ++i2)
                base[node_offset(i1, i2) + static_cast<std::size_t>(pair) * n_out + out] = f.at(i1, i2);
    }

    // Drop the device table (e.g. to free GPU memory); rebuilt on next use.
    void release() const { cache_.reset(); }

    // The prepared device handle, (re)built when P was (possibly) modified
    // since the last call (ParamVector generation), or the shape / device changed.
    lmkan_b200_layer* prepared() const {
        if (!cache_ || cache_->generation != P.generation() || cache_->data != P.data() ||
            cache_->size != P.size() || cache_->n_in != n_in || cache_->n_out != n_out ||
            cache_->G != grid.G || cache_->device != device || cache_->precision != precision) {
            auto pr = std::make_shared<detail::Prepared>();
            if (precision == 64)
                detail::throw_status(
                    lmkan_b200_layer_create_exact(n_in, n_out, grid.G, gamma, P.data(), device, &pr->h), "lmkan_forward");
            else
                detail::throw_status(
                    lmkan_b200_layer_create(n_in, n_out, grid.G, gamma, P.data(), device, &pr->h), "lmkan_forward");
            pr->precision = precision;
            pr->n_in = n_in; pr->n_out = n_out; pr->G = grid.G; pr->device = device;
            pr->data = P.data();
            pr->size = P.size();
            pr->generation = P.generation();
            cache_ = std::move(pr);
        }
        detail::throw_status(lmkan_b200_layer_set_gamma(cache_->h, gamma), "lmkan_forward");
        return cache_->h;
    }

private:
    mutable std::shared_ptr<detail::Prepared> cache_;
};

// costs.hpp:14-29: main-term FMA count (k^d / d) * n_in * n_out and the
// 2D table size (G+1)^2 * (n_in/2) * n_out.
inline std::uint64_t flops_main_term(std::uint64_t n_in, std::uint64_t n_out, unsigned d = 2, unsigned k = 2) {
    if (d < 1) throw std::invalid_argument("flops_main_term: d must be >= 1");
    if (k < 2) throw std::invalid_argument("flops_main_term: spline order k must be >= 2");
    if (n_in % d != 0) throw std::invalid_argument("flops_main_term: d must divide n_in");
    std::uint64_t kd = 1;
    for (unsigned i = 0; i < d; ++i) kd *= k;
    return kd * (n_in / d) * n_out;
}

// layer.hpp:63-65
inline double default_init_scale(int n_in) { return 1.0 / std::sqrt(static_cast<double>(n_in / 2)); }

// costs.hpp:25-29
inline std::uint64_t param_count(const LmKanLayer& layer) {
    return static_cast<std::uint64_t>(layer.grid.G + 1) * (layer.grid.G + 1) * layer.pairs() * layer.n_out;
}

// layer.hpp:69-86: same validation, the same N(0, scale^2) table drawn from the
// same named stream (bit-identical), gamma = 0.
inline LmKanLayer init_layer(int n_in, int n_out, int G, std::uint64_t seed, double init_scale = -1.0) {
    if (n_in <= 0 || n_in % 2 != 0) throw std::invalid_argument("init_layer: n_in must be a positive even number");
    if (n_out <= 0) throw std::invalid_argument("init_layer: n_out must be positive");
    LmKanLayer layer;
    layer.n_in = n_in;
    layer.n_out = n_out;
    layer.grid = build_grid(G);
    layer.P.assign(static_cast<std::size_t>(G + 1) * (G + 1) * (n_in / 2) * n_out, 0.0);
    detail::throw_status(lmkan_b200_init_table(n_in, n_out, G, seed, init_scale, layer.P.data()), "init_layer");
    layer.gamma = 0.0;
    return layer;
}

// layer.hpp:108-134. Y is resized when its shape differs (layer.hpp:111-112).
// `workers` is accepted for signature compatibility and ignored (the GPU
// replaces the std::thread row split of threading.hpp:24-42). Blocks until Y
// holds the result.
inline void lmkan_forward(const LmKanLayer& layer, const Matrix& X, Matrix& Y, std::size_t workers = 0) {
    require_width(X, layer.n_in, "lmkan_forward");
    if (Y.rows() != X.rows() || Y.cols() != static_cast<std::size_t>(layer.n_out)) Y = Matrix(X.rows(), layer.n_out);
    if (X.rows() == 0) return;
    lmkan_b200_layer* h = layer.prepared();
    detail::throw_status(lmkan_b200_forward_host_f64(h, X.data(), Y.data(), static_cast<std::int64_t>(X.rows()),
                                                     workers),
                         "lmkan_forward");
}

// threading.hpp:11-19: LMKAN_THREADS if set, else hardware concurrency.
inline std::size_t worker_count() {
    if (const char* env = std::getenv("LMKAN_THREADS")) {
        const long n = std::strtol(env, nullptr, 10);
        if (n >= 1) return static_cast<std::size_t>(n);
    }
    const unsigned hc = std::thread::hardware_concurrency();
    return hc == 0 ? 1 : hc;
}

// layer.hpp:141-202. Same checks and messages; dP is added into; dX resized
// when its shape differs. `workers` keeps the reference's meaning (0 ->
// worker_count()): the rows are split into that many contiguous chunks and the
// per-chunk sums are merged in order, so the result is bit-identical to the
// reference's lmkan_backward with the same worker count. The device runs the
// fp64 master table P; a larger explicit `workers` spreads the dP sums over
// more of the GPU (still matching the reference run with that count).
inline void lmkan_backward(const LmKanLayer& layer, const Matrix& X, const Matrix& dY, std::vector<double>& dP,
                           Matrix* dX, std::size_t workers = 0) {
    require_width(X, layer.n_in, "lmkan_backward");
    require_width(dY, layer.n_out, "lmkan_backward");
    if (X.rows() != dY.rows()) throw std::invalid_argument("lmkan_backward: X and dY row counts differ");
    if (dP.size() != layer.P.size()) throw std::invalid_argument("lmkan_backward: dP size mismatch");
    if (dX && (dX->rows() != X.rows() || dX->cols() != X.cols())) *dX = Matrix(X.rows(), X.cols());
    if (workers == 0) workers = worker_count();
    if (X.rows() == 0) return;
    lmkan_b200_layer* h = layer.prepared();
    detail::throw_status(lmkan_b200_backward_host_f64(h, layer.P.data(), X.data(), dY.data(), dP.data(),
                                                      dX ? dX->data() : nullptr,
                                                      static_cast<std::int64_t>(X.rows()), workers),
                         "lmkan_backward");
}

// A fused pure-lookup model resident on one GPU: what load_model returns for a
// model that went through fuse_model (fuse.hpp:105-140), as a chain of device
// layers. Blocks of other kinds (mlp, batch norm, preconditioned lookup) are
// outside the B200 path: load_model throws std::runtime_error for them.
class DeviceModel {
public:
    DeviceModel() = default;
    explicit DeviceModel(lmkan_b200_model* h) : h_(h, &lmkan_b200_model_destroy) {
        detail::throw_status(lmkan_b200_model_info(h, &n_blocks_, &in_dim_, &out_dim_, &device_), "load_model");
    }
    int in_dim() const { return in_dim_; }
    int out_dim() const { return out_dim_; }
    int n_blocks() const { return n_blocks_; }
    int device() const { return device_; }
    lmkan_b200_model* handle() const { return h_.get(); }

private:
    std::shared_ptr<lmkan_b200_model> h_;
    int n_blocks_ = 0, in_dim_ = 0, out_dim_ = 0, device_ = 0;
};

// serialize.hpp:185-301: same validation and FormatError messages; the tables
// are streamed from the file straight into the device layout.
inline DeviceModel load_model(const std::string& path, int device = 0) {
    lmkan_b200_model* h = nullptr;
    detail::throw_status(lmkan_b200_model_load(path.c_str(), device, &h), "load_model");
    return DeviceModel(h);
}

// model.hpp:313-316 (inference forward). Width errors as precond_forward's
// require_width (model.hpp:59). `workers` is accepted and ignored.
inline Matrix model_infer(const DeviceModel& model, const Matrix& X, std::size_t workers = 0) {
    require_width(X, static_cast<std::size_t>(model.in_dim()), "precond_forward");
    Matrix Y(X.rows(), model.out_dim());
    if (X.rows() == 0) return Y;
    detail::throw_status(lmkan_b200_model_infer_host_f64(model.handle(), X.data(), Y.data(),
                                                         static_cast<std::int64_t>(X.rows()), workers),
                         "model_infer");
    return Y;
}

// Adapter for code that keeps the REFERENCE's own types (lmkan::LmKanLayer,
// lmkan::Matrix): duck-typed on their public members, prepares a device table
// per call (use LmKanLayer above to keep it resident).
template <class RefLayer, class RefMatrix>
void lmkan_forward_ref_types(const RefLayer& layer, const RefMatrix& X, RefMatrix& Y, int device = 0) {
    if (X.cols() != static_cast<std::size_t>(layer.n_in))
        throw std::invalid_argument("lmkan_forward: expected width " + std::to_string(layer.n_in) + ", got " +
                                    std::to_string(X.cols()));
    if (Y.rows() != X.rows() || Y.cols() != static_cast<std::size_t>(layer.n_out)) Y = RefMatrix(X.rows(), layer.n_out);
    if (X.rows() == 0) return;
    detail::Prepared pr;
    detail::throw_status(
        lmkan_b200_layer_create(layer.n_in, layer.n_out, layer.grid.G, layer.gamma, layer.P.data(), device, &pr.h),
        "lmkan_forward");
    detail::throw_status(lmkan_b200_forward_host_f64(pr.h, X.data(), Y.data(), static_cast<std::int64_t>(X.rows()), 0),
                         "lmkan_forward");
}

}  // namespace lmkan_b200
