/*
 * TEST INFRASTRUCTURE ONLY — exhaustive check that the threshold-count cell
 * index #{k : x >= t_k} equals the reference interval_index (grid.hpp:72-75)
 * for EVERY fp32 bit pattern (finite, +-inf, NaN). Usage:
 *   verify_thresholds G [threads]      -> prints "G=<G> mismatches=<n> thresholds=..."
 */
#include <stdio.h>
#include <stdlib.h>

#include "lmkan_oracle.h"

int main(int argc, char** argv) {
    if (argc < 2) {
        fprintf(stderr, "usage: %s G [threads]\n", argv[0]);
        return 2;
    }
    const int G = atoi(argv[1]);
    const int threads = argc > 2 ? atoi(argv[2]) : 8;
    float t[256];
    if (G < 3 || G > 257 || lmko_thresholds_f32(G, t) != 0) {
        fprintf(stderr, "bad G\n");
        return 2;
    }
    const long long bad = (long long)lmko_verify_thresholds_f32(G, t, 0u, 0xffffffffu, threads);
    printf("G=%d mismatches=%lld thresholds=", G, bad);
    for (int k = 0; k < G - 1; ++k) printf("%s%.9g", k ? "," : "", (double)t[k]);
    printf("\n");
    return bad == 0 ? 0 : 1;
}
