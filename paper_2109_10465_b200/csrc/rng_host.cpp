// rng_host.cpp — see rng_host.h.
#include "rng_host.h"

#include <cstdint>
#include <random>

namespace moe {

uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

uint64_t derive_seed_tag(uint64_t seed, const char* tag) {
    uint64_t h = splitmix64(seed);
    for (const unsigned char* c = reinterpret_cast<const unsigned char*>(tag); *c; ++c)
        h = splitmix64(h ^ *c);
    return h;
}

uint64_t derive_seed_u64(uint64_t seed, uint64_t salt) { return splitmix64(splitmix64(seed) ^ salt); }

void permutation(uint64_t seed, int64_t n, uint32_t* out) {
    std::mt19937_64 eng(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = static_cast<uint32_t>(i);
    for (int64_t i = n; i > 1; --i) {
        const uint64_t range = static_cast<uint64_t>(i);
        const uint64_t limit = UINT64_MAX - UINT64_MAX % range;
        uint64_t x;
        do {
            x = eng();
        } while (x >= limit);
        const int64_t j = static_cast<int64_t>(x % range);
        const uint32_t t = out[i - 1];
        out[i - 1] = out[j];
        out[j] = t;
    }
}

}  // namespace moe
