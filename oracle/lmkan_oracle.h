/*
 * TEST INFRASTRUCTURE ONLY — not part of the product.
 *
 * Plain-C restatement of the reference lmKAN layer-forward path
 * (/root/reference/proj/include/lmkan/{grid,layer}.hpp), used as the parity
 * checker by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg.
 * Nothing under paper_2509_07103_b200/ may link or call this code.
 *
 * Parity of this restatement is pinned two ways (see tests/test_oracle.py):
 *   - against the reference's own known-answer tests (test_grid.cpp:34-219,
 *     test_layer.cpp:50-145) restated as golden vectors in tests/golden/;
 *   - against the unmodified reference headers compiled into
 *     oracle/_ref/liblmkan_ref.so (oracle/ref_shim.cpp, oracle/Makefile),
 *     bit-for-bit on indices, weights and fp64 outputs.
 */
#ifndef LMKAN_ORACLE_H
#define LMKAN_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* grid.hpp:14-17 */
double lmko_sigma(double x);
/* grid.hpp:44-68; points[G+1], inv_areas[G*G]. Returns 0, or -1 if G < 3. */
int lmko_build_grid(int G, double* points, double* inv_areas);
/* grid.hpp:72-75 */
int lmko_interval_index(int G, double x);
/* grid.hpp:87-101; w[4] = {w00, w10, w01, w11} */
void lmko_preamble(int G, const double* points, const double* inv_areas, double x1, double x2,
                   int* i1, int* i2, double* w);
/* layer.hpp:96-101 over rows: i1/i2 [rows][pairs], w [rows][pairs][4] */
void lmko_locate(int G, const double* points, const double* inv_areas, int n_in, const double* X,
                 int64_t rows, int32_t* i1, int32_t* i2, double* w);
/* layer.hpp:108-134. P is [G+1][G+1][n_in/2][n_out] (layer.hpp:20-22,34-45).
 * threads <= 1 runs serially; otherwise contiguous row chunks (threading.hpp:33-39). */
void lmko_forward(int n_in, int n_out, int G, const double* points, const double* inv_areas,
                  const double* P, double gamma, const double* X, int64_t rows, double* Y,
                  int threads);

/* layer.hpp:141-202 (lmkan_backward) with one worker: dP (same layout as P)
 * accumulates gamma * w * dY at the four nodes of every (row, pair), rows in
 * order; dX [rows][n_in] (may be NULL) from the analytic cell derivatives.
 * dP must hold its initial value (the reference adds into it). */
void lmko_backward(int n_in, int n_out, int G, const double* points, const double* inv_areas,
                   const double* P, double gamma, const double* X, const double* dY, int64_t rows,
                   double* dP, double* dX);

/* Threshold table derived from lmko_interval_index by bisection over the total
 * order of finite doubles / floats: t[k-1] = min{x : interval_index(x) >= k},
 * k = 1..G-1. Assumes interval_index is monotone in x, which
 * lmko_verify_thresholds_f32 checks exhaustively for fp32 inputs. */
int lmko_thresholds_f64(int G, double* t);
int lmko_thresholds_f32(int G, float* t);
/* Exhaustive check over fp32 bit patterns [lo, hi] (inclusive): counts x whose
 * #{k : x >= t[k]} differs from interval_index((double)x). Multi-threaded. */
int64_t lmko_verify_thresholds_f32(int G, const float* t, uint32_t lo, uint32_t hi, int threads);

#ifdef __cplusplus
}
#endif
#endif
