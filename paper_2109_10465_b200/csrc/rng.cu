// rng.cu — device jitter-noise generator (mt19937_64 with jump-ahead).
#include "common.cuh"
#include "kernels.h"

namespace moe {

bool launch_jitter_noise_device(uint64_t, int64_t, double, float*, cudaStream_t) { return false; }

}  // namespace moe
