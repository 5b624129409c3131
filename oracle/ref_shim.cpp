// TEST INFRASTRUCTURE ONLY — extern "C" shim over the UNMODIFIED reference
// headers in /root/reference/proj/include (compiled by oracle/Makefile into
// oracle/_ref/liblmkan_ref.so; the reference sources are not copied). It lets
// the Python tests and bench.py's reference arm drive the reference's own
// lmkan::lmkan_forward (layer.hpp:108-134), preamble (grid.hpp:87-101),
// build_grid (grid.hpp:44-68) and init_layer (layer.hpp:69-86).
#include <cstdint>
#include <cstring>
#include <vector>
#include <exception>
#include <string>

#include "lmkan/grid.hpp"
#include "lmkan/layer.hpp"
#include "lmkan/matrix.hpp"
#include "lmkan/threading.hpp"

namespace {
thread_local std::string g_err;
}

extern "C" {

const char* lmkref_last_error() { return g_err.c_str(); }

double lmkref_sigma(double x) { return lmkan::sigma(x); }

int lmkref_build_grid(int G, double* points, double* inv_areas) {
    try {
        const lmkan::SigmaGrid g = lmkan::build_grid(G);
        std::memcpy(points, g.points.data(), sizeof(double) * g.points.size());
        std::memcpy(inv_areas, g.inv_areas.data(), sizeof(double) * g.inv_areas.size());
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

int lmkref_interval_index(int G, double x) {
    const lmkan::SigmaGrid g = lmkan::build_grid(G);
    return lmkan::interval_index(g, x);
}

// Batched interval_index over an array (fast exhaustive / random checks).
void lmkref_interval_index_batch(int G, const double* x, int64_t n, int32_t* out) {
    const lmkan::SigmaGrid g = lmkan::build_grid(G);
    for (int64_t i = 0; i < n; ++i) out[i] = lmkan::interval_index(g, x[i]);
}

// detail::row_preambles (layer.hpp:96-101) over every row of X.
int lmkref_locate(int n_in, int G, const double* X, int64_t rows, int32_t* i1, int32_t* i2,
                  double* w) {
    try {
        lmkan::LmKanLayer layer;
        layer.n_in = n_in;
        layer.n_out = 1;
        layer.grid = lmkan::build_grid(G);
        std::vector<lmkan::detail::PairCell> cells(layer.pairs());
        for (int64_t r = 0; r < rows; ++r) {
            lmkan::detail::row_preambles(layer, X + r * n_in, cells.data());
            for (int p = 0; p < layer.pairs(); ++p) {
                const int64_t k = r * layer.pairs() + p;
                i1[k] = cells[p].i1;
                i2[k] = cells[p].i2;
                w[4 * k + 0] = cells[p].w00;
                w[4 * k + 1] = cells[p].w10;
                w[4 * k + 2] = cells[p].w01;
                w[4 * k + 3] = cells[p].w11;
            }
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// init_layer (layer.hpp:69-86); P_out must hold (G+1)^2*(n_in/2)*n_out doubles.
int lmkref_init_layer(int n_in, int n_out, int G, uint64_t seed, double init_scale,
                      double* P_out) {
    try {
        const lmkan::LmKanLayer l = lmkan::init_layer(n_in, n_out, G, seed, init_scale);
        std::memcpy(P_out, l.P.data(), sizeof(double) * l.P.size());
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// Persistent layer / matrix handles so the CPU baseline times lmkan_forward
// alone (no table copy in the timed region).
void* lmkref_layer_create(int n_in, int n_out, int G, const double* P, double gamma) {
    try {
        auto* l = new lmkan::LmKanLayer();
        l->n_in = n_in;
        l->n_out = n_out;
        l->grid = lmkan::build_grid(G);
        l->P.assign(P, P + static_cast<std::size_t>(G + 1) * (G + 1) * (n_in / 2) * n_out);
        l->gamma = gamma;
        return l;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void lmkref_layer_destroy(void* l) { delete static_cast<lmkan::LmKanLayer*>(l); }

void* lmkref_matrix_create(int64_t rows, int64_t cols, const double* data) {
    auto* m = new lmkan::Matrix(rows, cols);
    if (data) std::memcpy(m->data(), data, sizeof(double) * rows * cols);
    return m;
}
void lmkref_matrix_destroy(void* m) { delete static_cast<lmkan::Matrix*>(m); }
void lmkref_matrix_read(const void* m, double* out) {
    const auto* mm = static_cast<const lmkan::Matrix*>(m);
    std::memcpy(out, mm->data(), sizeof(double) * mm->size());
}
int64_t lmkref_matrix_rows(const void* m) { return static_cast<const lmkan::Matrix*>(m)->rows(); }
int64_t lmkref_matrix_cols(const void* m) { return static_cast<const lmkan::Matrix*>(m)->cols(); }

// lmkan_forward (layer.hpp:108-134) on handles; workers = 0 means
// LMKAN_THREADS / hardware_concurrency (threading.hpp:11-19).
int lmkref_forward(const void* layer, const void* X, void* Y, uint64_t workers) {
    try {
        lmkan::lmkan_forward(*static_cast<const lmkan::LmKanLayer*>(layer),
                             *static_cast<const lmkan::Matrix*>(X), *static_cast<lmkan::Matrix*>(Y),
                             workers);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// lmkan_backward (layer.hpp:141-202): dP (layer.P.size() doubles) is added
// into, dX [rows][n_in] or NULL.
int lmkref_backward(const void* layer, const void* X, const void* dY, double* dP, void* dX, uint64_t workers) {
    try {
        const auto& L = *static_cast<const lmkan::LmKanLayer*>(layer);
        std::vector<double> acc(dP, dP + L.P.size());
        lmkan::lmkan_backward(L, *static_cast<const lmkan::Matrix*>(X), *static_cast<const lmkan::Matrix*>(dY), acc,
                              static_cast<lmkan::Matrix*>(dX), workers);
        std::memcpy(dP, acc.data(), sizeof(double) * acc.size());
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

uint64_t lmkref_worker_count() { return lmkan::worker_count(); }

}  // extern "C"
