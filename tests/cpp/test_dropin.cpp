// Drop-in test of the C++ host API (include/lmkan_b200/lmkan.hpp) on a GPU.
// Mirrors the forward cases of the reference's test_layer.cpp (cited per case)
// with the caller code unchanged apart from `namespace lmkan = lmkan_b200;`.
// The fp64 oracles used here (dense O(G^2) basis sum, linear sheets) are
// independent restatements in this file (func2d.hpp:32-73); tolerance is the
// fp32 contract |d| <= 1e-5 * max(1, |ref|) instead of the reference's fp64 1e-12.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <random>
#include <stdexcept>
#include <cstring>
#include <string>
#include <vector>

#include "lmkan_b200/lmkan.hpp"

namespace lmkan = lmkan_b200;
using namespace lmkan;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                           \
    do {                                                                   \
        ++g_checks;                                                        \
        if (!(c)) {                                                        \
            ++g_fail;                                                      \
            std::fprintf(stderr, "%s:%d CHECK failed: %s\n", __FILE__, __LINE__, #c); \
        }                                                                  \
    } while (0)
#define CHECK_THROWS_AS(expr, T)        \
    do {                                \
        bool ok = false;                \
        try {                           \
            expr;                       \
        } catch (const T&) {            \
            ok = true;                  \
        } catch (...) {                 \
        }                               \
        CHECK(ok);                      \
    } while (0)

static bool close_mixed(double y, double ref, double tol = 1e-5) {
    return std::abs(y - ref) <= tol * std::max(1.0, std::abs(ref));
}

static Matrix random_batch(std::size_t rows, std::size_t cols, std::mt19937_64& g, double scale = 1.0) {
    std::normal_distribution<double> n(0.0, 1.0);
    Matrix X(rows, cols);
    for (std::size_t i = 0; i < X.size(); ++i) X.data()[i] = scale * n(g);
    return X;
}

// func2d.hpp:32-48 restated: hat function i at x, edge segments unbounded.
static double basis_1d(const SigmaGrid& g, int i, double x) {
    const int G = g.G;
    const auto& p = g.points;
    if (i == 0) return x < p[1] ? (p[1] - x) / (p[1] - p[0]) : 0.0;
    if (i == G) return x > p[G - 1] ? (x - p[G - 1]) / (p[G] - p[G - 1]) : 0.0;
    if (x < p[i]) return (i == 1 || x >= p[i - 1]) ? (x - p[i - 1]) / (p[i] - p[i - 1]) : 0.0;
    return (i == G - 1 || x <= p[i + 1]) ? (p[i + 1] - x) / (p[i + 1] - p[i]) : 0.0;
}

// test_layer.cpp:20-32 restated: gamma * sum_p dense-oracle(sheet(p, q)).
static Matrix dense_reference(const LmKanLayer& L, const Matrix& X) {
    Matrix Y(X.rows(), L.n_out);
    const int G = L.grid.G;
    for (std::size_t r = 0; r < X.rows(); ++r)
        for (int q = 0; q < L.n_out; ++q) {
            double acc = 0.0;
            for (int p = 0; p < L.pairs(); ++p)
                for (int i1 = 0; i1 <= G; ++i1) {
                    const double b1 = basis_1d(L.grid, i1, X(r, 2 * p));
                    if (b1 == 0.0) continue;
                    for (int i2 = 0; i2 <= G; ++i2)
                        acc += L.node_slice(i1, i2, p)[q] * b1 * basis_1d(L.grid, i2, X(r, 2 * p + 1));
                }
            Y(r, q) = L.gamma * acc;
        }
    return Y;
}

static void test_init_layer() {  // test_layer.cpp:50-72
    const LmKanLayer layer = init_layer(4, 3, 4, 123);
    CHECK(layer.n_in == 4 && layer.n_out == 3);
    CHECK(layer.P.size() == 5u * 5u * 2u * 3u);
    CHECK(layer.gamma == 0.0);
    CHECK(layer.P == init_layer(4, 3, 4, 123).P);
    CHECK(layer.P != init_layer(4, 3, 4, 124).P);
    LmKanLayer zero = init_layer(4, 3, 4, 1, 0.0);
    zero.gamma = 1.0;
    std::mt19937_64 g(9);
    Matrix X = random_batch(16, 4, g), Y;
    lmkan_forward(zero, X, Y);
    for (std::size_t i = 0; i < Y.size(); ++i) CHECK(Y.data()[i] == 0.0);
    CHECK_THROWS_AS(init_layer(3, 2, 4, 0), std::invalid_argument);
    CHECK_THROWS_AS(init_layer(0, 2, 4, 0), std::invalid_argument);
    CHECK_THROWS_AS(build_grid(2), std::invalid_argument);
}

static void test_dense_oracle() {  // test_layer.cpp:74-99
    std::mt19937_64 g(11);
    for (int G : {3, 5, 12}) {
        LmKanLayer layer = init_layer(6, 5, G, 77 + G);
        layer.gamma = 0.8;
        const Matrix X = random_batch(64, 6, g, 1.5);
        Matrix Y;
        lmkan_forward(layer, X, Y);
        const Matrix R = dense_reference(layer, X);
        for (std::size_t i = 0; i < Y.size(); ++i) CHECK(close_mixed(Y.data()[i], R.data()[i]));
    }
}

static void test_width_mismatch() {  // test_layer.cpp:101-110
    LmKanLayer layer = init_layer(4, 2, 4, 5);
    Matrix X(3, 6), Y;
    CHECK_THROWS_AS(lmkan_forward(layer, X, Y), std::invalid_argument);
    try {
        lmkan_forward(layer, X, Y);
    } catch (const std::invalid_argument& e) {
        CHECK(std::string(e.what()) == "lmkan_forward: expected width 4, got 6");
    }
}

static void test_linear_sheets() {  // test_layer.cpp:112-145
    std::mt19937_64 g(12);
    std::normal_distribution<double> n(0.0, 1.0);
    LmKanLayer layer = init_layer(8, 3, 4, 99);
    layer.gamma = 0.6;
    double A[3][4], B[3][4], C[3][4];
    for (int q = 0; q < 3; ++q)
        for (int p = 0; p < 4; ++p) A[q][p] = n(g), B[q][p] = n(g), C[q][p] = n(g);
    for (int p = 0; p < 4; ++p)
        for (int q = 0; q < 3; ++q)
            for (int i = 0; i <= 4; ++i)
                for (int j = 0; j <= 4; ++j)
                    layer.node_slice(i, j, p)[q] =
                        A[q][p] * layer.grid.points[i] + B[q][p] * layer.grid.points[j] + C[q][p];
    const Matrix X = random_batch(32, 8, g, 2.0);
    Matrix Y;
    lmkan_forward(layer, X, Y);
    for (std::size_t r = 0; r < X.rows(); ++r)
        for (int q = 0; q < 3; ++q) {
            double want = 0.0;
            for (int p = 0; p < 4; ++p) want += A[q][p] * X(r, 2 * p) + B[q][p] * X(r, 2 * p + 1) + C[q][p];
            CHECK(close_mixed(Y(r, q), 0.6 * want));
        }
}

static void test_determinism_and_cache() {  // test_layer.cpp:228-239 + P edits
    LmKanLayer layer = init_layer(8, 6, 12, 2024);
    layer.gamma = 0.9;
    std::mt19937_64 g(15);
    const Matrix X = random_batch(33, 8, g);
    Matrix Y1, Y2;
    lmkan_forward(layer, X, Y1);
    lmkan_forward(layer, X, Y2);
    for (std::size_t i = 0; i < Y1.size(); ++i) CHECK(Y1.data()[i] == Y2.data()[i]);
    // finite-difference style edits on a copy (test_layer.cpp:198-205) see the edit
    LmKanLayer bumped = layer;
    for (double& v : bumped.P) v *= 2.0;
    Matrix Yb;
    lmkan_forward(bumped, X, Yb);
    for (std::size_t i = 0; i < Y1.size(); ++i) CHECK(close_mixed(Yb.data()[i], 2.0 * Y1.data()[i]));
    // in-place edit of the same layer
    for (double& v : layer.P) v = -v;
    lmkan_forward(layer, X, Y2);
    for (std::size_t i = 0; i < Y1.size(); ++i) CHECK(close_mixed(Y2.data()[i], -Y1.data()[i]));
    // gamma change only
    layer.gamma = 0.0;
    lmkan_forward(layer, X, Y2);
    for (std::size_t i = 0; i < Y2.size(); ++i) CHECK(Y2.data()[i] == 0.0);
    layer.gamma = 0.9;
    // every mutation route of P (a ParamVector) is seen by the next forward:
    // element reference, data() pointer (taken after the last forward, as the
    // reference's optimizer does, model.hpp:382-386), a std::vector<double>&
    // parameter, assign(), whole assignment; a const read is not a mutation
    auto scale_via = [&](int how, double f) {
        switch (how) {
            case 0: for (std::size_t i = 0; i < layer.P.size(); ++i) layer.P[i] *= f; break;
            case 1: { double* p = layer.P.data(); for (std::size_t i = 0; i < layer.P.size(); ++i) p[i] *= f; } break;
            case 2: { auto mul = [f](std::vector<double>& v) { for (double& x : v) x *= f; }; mul(layer.P); } break;
            case 3: { std::vector<double> v(layer.P.begin(), layer.P.end()); for (double& x : v) x *= f;
                      layer.P.assign(v.begin(), v.end()); } break;
            default: { std::vector<double> v = layer.P; for (double& x : v) x *= f; layer.P = v; } break;
        }
    };
    Matrix Yref;
    lmkan_forward(layer, X, Yref);
    for (int how = 0; how < 5; ++how) {
        const std::uint64_t g0 = layer.P.generation();
        const LmKanLayer& cl = layer;
        double sum = 0.0;
        for (std::size_t i = 0; i < cl.P.size(); ++i) sum += cl.P[i];  // const reads
        CHECK(layer.P.generation() == g0 && std::isfinite(sum));
        scale_via(how, -1.0);
        CHECK(layer.P.generation() != g0);
        Matrix Ys;
        lmkan_forward(layer, X, Ys);
        for (std::size_t i = 0; i < Ys.size(); ++i) CHECK(Ys.data()[i] == -Yref.data()[i]);
        scale_via(how, -1.0);
        lmkan_forward(layer, X, Ys);
        for (std::size_t i = 0; i < Ys.size(); ++i) CHECK(Ys.data()[i] == Yref.data()[i]);
    }
}

static void test_grid_helpers() {  // test_grid.cpp:34-48, 166-219 restated
    CHECK(sigma(0.0) == 0.5);
    CHECK(std::abs(sigma(-std::log(2.0)) - 0.25) < 1e-15);
    CHECK(std::abs(sigma(0.1) - 0.5475812909820202) < 1e-15);
    CHECK(std::isnan(sigma(std::nan(""))));
    const SigmaGrid g = build_grid(4);
    const Preamble at_node = preamble(g, g.points[1], g.points[2]);  // one-hot at a node
    CHECK(at_node.i1 == 1 && at_node.i2 == 2 && std::abs(at_node.w00 - 1.0) < 1e-12);
    const Preamble mid = preamble(g, 0.5 * (g.points[1] + g.points[2]), 0.5 * (g.points[2] + g.points[3]));
    CHECK(std::abs(mid.w00 - 0.25) < 1e-12 && std::abs(mid.w11 - 0.25) < 1e-12);
    std::mt19937_64 r(3);
    std::normal_distribution<double> n(0.0, 2.0);
    for (int t = 0; t < 100; ++t) {  // partition of unity
        const Preamble p = preamble(g, n(r), n(r));
        CHECK(std::abs(p.w00 + p.w10 + p.w01 + p.w11 - 1.0) <= 1e-12);
    }
    CHECK(flops_main_term(1024, 1024) == 2ull * 1024 * 1024);
    CHECK(param_count(init_layer(4, 3, 4, 1)) == 5ull * 5 * 2 * 3);
}

static void test_interval_index() {  // test_grid.cpp:108-114
    const SigmaGrid g4 = build_grid(4);
    CHECK(interval_index(g4, 0.1) == 2);
    CHECK(interval_index(g4, -100.0) == 0);
    CHECK(interval_index(g4, 100.0) == 3);
    CHECK(interval_index(g4, 1e308) == 3);
    CHECK(interval_index(g4, std::nan("")) == 0);
}

// test_layer.cpp:147-226 restated: zero upstream -> zero; compact support of
// one row; dP against central differences of the fp64 dense oracle (the map
// is linear in P); bitwise determinism for a fixed worker count.
static void test_backward() {
    LmKanLayer layer = init_layer(4, 3, 4, 321);
    layer.gamma = 0.5;
    std::mt19937_64 g(13);
    const Matrix X = random_batch(8, 4, g);
    std::vector<double> dP(layer.P.size(), 0.0);
    Matrix dX;
    lmkan_backward(layer, X, Matrix(8, 3, 0.0), dP, &dX);
    for (double v : dP) CHECK(v == 0.0);
    for (std::size_t i = 0; i < dX.size(); ++i) CHECK(dX.data()[i] == 0.0);
    CHECK(dX.rows() == 8 && dX.cols() == 4);

    LmKanLayer one = init_layer(2, 1, 4, 7);
    one.gamma = 1.0;
    Matrix X1(1, 2);
    X1(0, 0) = 0.2;
    X1(0, 1) = -0.4;
    std::vector<double> d1(one.P.size(), 0.0);
    lmkan_backward(one, X1, Matrix(1, 1, 1.0), d1, nullptr);
    int nonzero = 0;
    for (double v : d1) nonzero += v != 0.0;
    CHECK(nonzero == 4);

    for (int G : {3, 4}) {
        LmKanLayer L = init_layer(4, 3, G, 1000 + G);
        L.gamma = 0.7;
        const Matrix Xg = random_batch(8, 4, g);
        const Matrix dY = random_batch(8, 3, g);
        std::vector<double> dPg(L.P.size(), 0.0);
        lmkan_backward(L, Xg, dY, dPg, nullptr, 3);
        std::vector<double> again(L.P.size(), 0.0);
        lmkan_backward(L, Xg, dY, again, nullptr, 3);
        CHECK(again == dPg);
        auto loss = [&](const LmKanLayer& l) {
            const Matrix y = dense_reference(l, Xg);
            double acc = 0.0;
            for (std::size_t i = 0; i < y.size(); ++i) acc += y.data()[i] * dY.data()[i];
            return acc;
        };
        const double h = 1e-3;
        for (std::size_t i = 0; i < L.P.size(); i += 7) {
            LmKanLayer b = L;
            b.P[i] += h;
            const double hi = loss(b);
            b.P[i] -= 2 * h;
            const double lo = loss(b);
            const double fd = (hi - lo) / (2 * h);
            CHECK(std::abs(dPg[i] - fd) <= 1e-8 * std::max(1.0, std::abs(fd)));
        }
    }
    std::vector<double> bad(3, 0.0);
    CHECK_THROWS_AS(lmkan_backward(layer, X, Matrix(8, 3), bad, nullptr), std::invalid_argument);
    CHECK_THROWS_AS(lmkan_backward(layer, X, Matrix(7, 3), dP, nullptr), std::invalid_argument);
}

// serialize.hpp:185-301 + model.hpp:313-316 on a model the REFERENCE saved
// (tests/golden/lmk1/pure_f64.lmk1, fuse_model of a relu_first student):
// model_infer equals the chain of lmkan_forward calls over layers built from
// the file's own P tensors; corrupt files throw FormatError with load_model's
// message; unfused models are refused.
static void test_load_model(const std::string& gold) {
    const std::string path = gold + "/pure_f64.lmk1";
    const DeviceModel model = load_model(path);
    CHECK(model.n_blocks() == 3 && model.in_dim() == 6 && model.out_dim() == 3);
    std::ifstream in(path, std::ios::binary);
    std::vector<char> raw((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    std::vector<LmKanLayer> layers;
    for (int b = 0; b < 3; ++b) {
        int type, n_in, n_out, G, mode, has_bn;
        double gamma;
        std::uint64_t off;
        CHECK(lmkan_b200_lmk1_block(path.c_str(), b, &type, &n_in, &n_out, &G, &gamma, &mode, &has_bn, &off) == 0);
        LmKanLayer L;
        L.n_in = n_in;
        L.n_out = n_out;
        L.grid = build_grid(G);
        L.gamma = gamma;
        L.P.resize(static_cast<std::size_t>(G + 1) * (G + 1) * (n_in / 2) * n_out);
        std::memcpy(L.P.data(), raw.data() + off, L.P.size() * sizeof(double));
        layers.push_back(std::move(L));
    }
    std::mt19937_64 g(21);
    const Matrix X = random_batch(40, 6, g, 1.5);
    const Matrix Y = model_infer(model, X);
    Matrix cur = X;
    for (const LmKanLayer& L : layers) {
        Matrix nxt;
        lmkan_forward(L, cur, nxt);
        cur = nxt;
    }
    CHECK(Y.rows() == 40 && Y.cols() == 3);
    for (std::size_t i = 0; i < Y.size(); ++i) CHECK(close_mixed(Y.data()[i], cur.data()[i]));
    Matrix bad(2, 5);
    CHECK_THROWS_AS(model_infer(model, bad), std::invalid_argument);
    // corrupt file: bad magic
    const std::string tmp = "/tmp/lmkan_b200_bad_magic.lmk1";
    {
        std::ofstream o(tmp, std::ios::binary);
        o.write("LMK2", 4);
        o.write(raw.data() + 4, static_cast<std::streamsize>(raw.size() - 4));
    }
    try {
        load_model(tmp);
        CHECK(false);
    } catch (const FormatError& e) {
        CHECK(std::string(e.what()) == "load_model: bad magic, not an LMK1 model file");
    }
    CHECK_THROWS_AS(load_model(gold + "/student.lmk1"), std::runtime_error);
}

int main(int argc, char** argv) {
    test_init_layer();
    test_dense_oracle();
    test_width_mismatch();
    test_linear_sheets();
    test_determinism_and_cache();
    test_interval_index();
    test_grid_helpers();
    test_backward();
    if (argc > 1) test_load_model(argv[1]);
    std::printf("test_dropin: %d checks, %d failures\n", g_checks, g_fail);
    return g_fail == 0 ? 0 : 1;
}
