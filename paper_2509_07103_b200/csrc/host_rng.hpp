// Host-side restatement of the reference's named random stream (rng.hpp:19-79)
// so that lmkan_b200_init_table reproduces init_layer's table (layer.hpp:69-86)
// bit-for-bit: FNV-1a(name) mixed into the seed by a splitmix64 finalizer keys a
// std::mt19937_64; uniforms take the top 53 bits; normals are Box-Muller with
// one cached value (the sine half is returned on the next call).
#pragma once

#include <cmath>
#include <cstdint>
#include <random>
#include <string_view>

namespace lmkan_b200 {
namespace host {

class NamedStream {
public:
    NamedStream(std::uint64_t seed, std::string_view name) : eng_(key(seed, name)) {}

    double uniform() { return static_cast<double>(eng_() >> 11) * 0x1.0p-53; }
    double uniform_open() {
        for (;;) {
            const double u = uniform();
            if (u != 0.0) return u;
        }
    }
    double normal() {
        if (cached_valid_) {
            cached_valid_ = false;
            return cached_;
        }
        const double u1 = uniform_open();
        const double u2 = uniform();
        const double rad = std::sqrt(-2.0 * std::log(u1));
        const double ang = 2.0 * M_PI * u2;
        cached_ = rad * std::sin(ang);
        cached_valid_ = true;
        return rad * std::cos(ang);
    }

private:
    static std::uint64_t key(std::uint64_t seed, std::string_view name) {
        std::uint64_t h = 0xcbf29ce484222325ull;  // FNV-1a 64
        for (unsigned char ch : name) h = (h ^ ch) * 0x100000001b3ull;
        std::uint64_t z = seed ^ (h + 0x9e3779b97f4a7c15ull);  // splitmix64 finalizer
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    }
    std::mt19937_64 eng_;
    bool cached_valid_ = false;
    double cached_ = 0.0;
};

}  // namespace host
}  // namespace lmkan_b200
