// rts.cu — the Random Token Selection order on the device.
//
// assign_rts scans tokens in the order Rng(seed).permutation(T)
// (routing.cpp:180-187, rng.cpp:94-102): iota, then for i = T..2
// swap(p[i-1], p[uniform_int(i)]), uniform_int rejecting x >= UINT64_MAX -
// UINT64_MAX % i (rng.cpp:45-56).  The draws do not depend on the array, only
// on the mt19937_64 stream, so:
//
//   1. raw   the first T + kSpare outputs of mt19937_64(seed) (rng.cu jump-ahead
//            generator)
//   2. draw  step i uses raw output T - i: j_i = x % i, flagging any x >= limit
//            (probability < i / 2^64 per draw); a one-thread pass redoes the
//            draws sequentially with rejection only when a flag was raised
//   3. the shuffle itself is rebuilt in parallel.  Step i (processed from
//      i = T down to 2) fixes position i-1 forever, so
//          p[i-1] = value at j_i just before step i.
//      The value at position q just before step i is q itself unless an
//      earlier step s > i targeted q (j_s = q); the latest such step (the
//      smallest s > i) left there the value position s-1 held just before
//      step s — the same question one level up.  Each output position
//      follows that chain (expected O(log T) links) through per-position
//      step lists built with counting-sort atomics; the lists are used as
//      sets (min over members), so the result does not depend on the
//      atomics' order.
//
// Bit-exact with the reference's permutation for every seed and T.
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace moe {
namespace rts {

constexpr int kSpare = 64;          // raw outputs beyond T for rejected draws
constexpr int32_t kNone = 0x7fffffff;

__global__ void draw_kernel(const uint64_t* __restrict__ raw, int64_t n, int32_t* __restrict__ jv,
                            int32_t* __restrict__ cnt, uint32_t* __restrict__ flag) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x + 2;  // step i in [2, n]
    if (i > n) return;
    const uint64_t x = raw[n - i];
    const uint64_t range = static_cast<uint64_t>(i);
    const uint64_t limit = UINT64_MAX - UINT64_MAX % range;
    if (x >= limit) atomicOr(flag, 1u);
    const int32_t j = static_cast<int32_t>(x % range);
    jv[i] = j;
    atomicAdd(&cnt[j], 1);
}

// only when a draw was rejected: the draws again, sequentially, with rejection
__global__ void redraw_kernel(const uint64_t* __restrict__ raw, int64_t n, int32_t* __restrict__ jv,
                              int32_t* __restrict__ cnt, uint32_t* __restrict__ flag,
                              uint32_t* __restrict__ layer_flags) {
    if (!(*flag & 1u) || threadIdx.x != 0) return;
    for (int64_t q = 0; q < n; ++q) cnt[q] = 0;
    int64_t k = 0;
    for (int64_t i = n; i > 1; --i) {
        const uint64_t range = static_cast<uint64_t>(i);
        const uint64_t limit = UINT64_MAX - UINT64_MAX % range;
        uint64_t x;
        do {
            if (k >= n + kSpare) {  // more rejections than spare outputs (never expected)
                if (layer_flags) atomicOr(layer_flags, MOE_FLAG_RTS_OVERFLOW_DEV);
                return;
            }
            x = raw[k++];
        } while (x >= limit);
        jv[i] = static_cast<int32_t>(x % range);
        ++cnt[jv[i]];
    }
}

// exclusive scan of cnt[0..n) into off / cursor (one CTA, chunked)
__global__ void scan_kernel(const int32_t* __restrict__ cnt, int64_t n, int32_t* __restrict__ off,
                            int32_t* __restrict__ cursor) {
    __shared__ int32_t part[1024];
    const int64_t per = (n + blockDim.x - 1) / blockDim.x;
    const int64_t b = threadIdx.x * per, e = min(n, b + per);
    int32_t s = 0;
    for (int64_t q = b; q < e; ++q) s += cnt[q];
    part[threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        int32_t acc = 0;
        for (unsigned w = 0; w < blockDim.x; ++w) {
            const int32_t v = part[w];
            part[w] = acc;
            acc += v;
        }
    }
    __syncthreads();
    int32_t acc = part[threadIdx.x];
    for (int64_t q = b; q < e; ++q) {
        off[q] = acc;
        cursor[q] = acc;
        acc += cnt[q];
    }
}

__global__ void place_kernel(const int32_t* __restrict__ jv, int64_t n, int32_t* __restrict__ cursor,
                             int32_t* __restrict__ list) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x + 2;
    if (i > n) return;
    list[atomicAdd(&cursor[jv[i]], 1)] = static_cast<int32_t>(i);
}

// nxt[i] = min{s > i : j_s = j_i} (i = 1 stands for position 0 with j_1 = 0);
// first2[q] = min{s > q + 1 : j_s = q}
__global__ void link_kernel(const int32_t* __restrict__ jv, int64_t n, const int32_t* __restrict__ off,
                            const int32_t* __restrict__ cnt, const int32_t* __restrict__ list,
                            int32_t* __restrict__ nxt, int32_t* __restrict__ first2) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x + 1;  // 1..n
    if (i > n) return;
    {
        const int32_t j = i == 1 ? 0 : jv[i];
        int32_t best = kNone;
        for (int32_t u = off[j], ue = off[j] + cnt[j]; u < ue; ++u) {
            const int32_t s = list[u];
            if (s > i && s < best) best = s;
        }
        nxt[i] = best;
    }
    {
        const int64_t q = i - 1;  // positions 0..n-1
        int32_t best = kNone;
        for (int32_t u = off[q], ue = off[q] + cnt[q]; u < ue; ++u) {
            const int32_t s = list[u];
            if (s > q + 1 && s < best) best = s;
        }
        first2[q] = best;
    }
}

__global__ void walk_kernel(const int32_t* __restrict__ jv, int64_t n, const int32_t* __restrict__ nxt,
                            const int32_t* __restrict__ first2, uint32_t* __restrict__ perm) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x + 1;  // fixes position i-1
    if (i > n) return;
    int32_t s = nxt[i];
    int32_t v = i == 1 ? 0 : jv[i];
    while (s != kNone) {
        v = s - 1;
        s = first2[s - 1];
    }
    perm[i - 1] = static_cast<uint32_t>(v);
}

}  // namespace rts

size_t rts_scratch_bytes(int64_t n) {
    // raw [n + spare] u64 + jv, cnt, off, cursor, list, nxt, first2 [n + 2] i32 + flag
    return sizeof(uint64_t) * static_cast<size_t>(n + rts::kSpare) + 7 * sizeof(int32_t) * static_cast<size_t>(n + 2) + 64;
}

void launch_rts_order(uint64_t seed, int64_t n, void* scratch, uint32_t* perm, uint32_t* layer_flags,
                      cudaStream_t st) {
    using namespace rts;
    if (n <= 0) return;
    uint64_t* raw = static_cast<uint64_t*>(scratch);
    int32_t* jv = reinterpret_cast<int32_t*>(raw + n + kSpare);
    int32_t* cnt = jv + (n + 2);
    int32_t* off = cnt + (n + 2);
    int32_t* cursor = off + (n + 2);
    int32_t* list = cursor + (n + 2);
    int32_t* nxt = list + (n + 2);
    int32_t* first2 = nxt + (n + 2);
    uint32_t* flag = reinterpret_cast<uint32_t*>(first2 + (n + 2));
    MOE_CUDA_CHECK(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (n + 2), st));
    MOE_CUDA_CHECK(cudaMemsetAsync(flag, 0, sizeof(uint32_t), st));
    launch_mt64_raw_device(seed, n + kSpare, raw, st);
    const unsigned g = static_cast<unsigned>(ceil_div(n + 1, static_cast<int64_t>(256)));
    if (n >= 2) {
        draw_kernel<<<g, 256, 0, st>>>(raw, n, jv, cnt, flag);
        MOE_LAUNCH_CHECK();
        redraw_kernel<<<1, 32, 0, st>>>(raw, n, jv, cnt, flag, layer_flags);
        MOE_LAUNCH_CHECK();
    }
    scan_kernel<<<1, 1024, 0, st>>>(cnt, n, off, cursor);
    MOE_LAUNCH_CHECK();
    if (n >= 2) {
        place_kernel<<<g, 256, 0, st>>>(jv, n, cursor, list);
        MOE_LAUNCH_CHECK();
    }
    link_kernel<<<g, 256, 0, st>>>(jv, n, off, cnt, list, nxt, first2);
    MOE_LAUNCH_CHECK();
    walk_kernel<<<g, 256, 0, st>>>(jv, n, nxt, first2, perm);
    MOE_LAUNCH_CHECK();
}

}  // namespace moe
