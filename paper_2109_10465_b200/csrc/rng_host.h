// rng_host.h — the reference's seed derivation and mt19937_64 draws (host).
// rng.cpp:15-102 (relative to /root/reference/proj/core/src).  std::mt19937_64
// is fully specified by the C++ standard, so this is bit-exact with the
// reference's Rng.
#pragma once

#include <stdint.h>

#include <vector>

namespace moe {

uint64_t splitmix64(uint64_t x);                           // rng.cpp:15-20
uint64_t derive_seed_tag(uint64_t seed, const char* tag);  // rng.cpp:24-30
uint64_t derive_seed_u64(uint64_t seed, uint64_t salt);    // rng.cpp:32-34
// Rng(seed).permutation(n), rng.cpp:94-102 (Fisher-Yates, rejection uniform_int)
void permutation(uint64_t seed, int64_t n, uint32_t* out);

}  // namespace moe
