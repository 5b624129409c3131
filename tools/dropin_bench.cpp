// End-to-end timing of the reference-signature drop-in (bench.py's e2e leg):
//   lmkan_b200::lmkan_forward(const LmKanLayer&, const Matrix& X, Matrix& Y)
// i.e. the call an existing caller of lmkan::lmkan_forward (layer.hpp:108-134)
// makes after `namespace lmkan = lmkan_b200;`: fp64 X / Y in ordinary pageable
// host memory (std::vector inside Matrix), the table prepared from the host
// LmKanLayer::P on first use and reused while P is unmodified.
//   dropin_bench n_in n_out G rows steps warmup [device]
// Prints one JSON object: samples/s and ms per step (host wall clock over the
// timed calls; each call returns with Y on the host), plus a result checksum.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <random>

#include "lmkan_b200/lmkan.hpp"

int main(int argc, char** argv) {
    if (argc < 7) {
        std::fprintf(stderr, "usage: %s n_in n_out G rows steps warmup [device]\n", argv[0]);
        return 2;
    }
    const int n_in = std::atoi(argv[1]), n_out = std::atoi(argv[2]), G = std::atoi(argv[3]);
    const std::size_t rows = std::strtoull(argv[4], nullptr, 10);
    const int steps = std::atoi(argv[5]), warmup = std::atoi(argv[6]);
    const int device = argc > 7 ? std::atoi(argv[7]) : 0;
    try {
        lmkan_b200::LmKanLayer layer = lmkan_b200::init_layer(n_in, n_out, G, 1000);  // layer.hpp:69-86 table
        layer.gamma = 1.0;
        layer.device = device;
        lmkan_b200::Matrix X(rows, n_in), Y;
        std::mt19937_64 g(1234);
        std::normal_distribution<double> nd(0.0, 1.0);
        for (std::size_t i = 0; i < X.size(); ++i) X.data()[i] = nd(g);
        for (int i = 0; i < warmup; ++i) lmkan_b200::lmkan_forward(layer, X, Y);  // first call prepares the table
        const auto t0 = std::chrono::steady_clock::now();
        double check = 0.0;
        for (int i = 0; i < steps; ++i) {
            lmkan_b200::lmkan_forward(layer, X, Y);
            check += Y(0, 0);  // the step's result read on the host
        }
        const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        std::printf("{\"samples_per_s\": %.6g, \"ms_per_step\": %.6g, \"steps\": %d, \"warmup\": %d, \"rows\": %zu, "
                    "\"h2d_bytes_per_step\": %zu, \"d2h_bytes_per_step\": %zu, \"checksum\": %.17g}\n",
                    rows * steps / s, 1e3 * s / steps, steps, warmup, rows, rows * n_in * sizeof(double),
                    rows * n_out * sizeof(double), check);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "dropin_bench: %s\n", e.what());
        return 1;
    }
    return 0;
}
