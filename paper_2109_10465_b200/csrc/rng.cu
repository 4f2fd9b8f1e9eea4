// rng.cu — the reference's jitter-noise stream generated on the device.
//
// gate_forward draws T*d values Rng(jitter_seed).uniform(1-eps, 1+eps) in
// row-major order (routing.cpp:62-70; rng.cpp:36-43): one mt19937_64 stream,
// strictly sequential.  To generate it on 148 SMs we jump ahead:
//
//  * mt19937_64 is GF(2)-linear.  Its raw word sequence x[k] (k >= 1) obeys
//    the recurrence whose characteristic polynomial phi(t) (degree 19937) we
//    recover once with Berlekamp-Massey; then x[k + e] = XOR_i g_i x[k + i]
//    with g = t^e mod phi.
//  * Chunk c of the stream starts at raw word o_c = 312 + c*J.  Its 312-word
//    window is XOR_{i: g_c,i = 1} base[j + i] with g_c = t^(o_c - 1) mod phi
//    and base = x[1 .. BASE] generated once per call from the seed.
//  * From its window each CTA regenerates its J outputs with the ordinary
//    block twist (shift-invariant) and tempering, producing the reference's
//    noise bit-for-bit (noise = lo + (hi - lo) * ((out >> 11) * 2^-53), the
//    f64 expression of rng.cpp:41-42, rounded to fp32 for the gate GEMM).
//
// The jump polynomials depend only on (J, P) — not on the seed — and are
// computed on the host once per geometry and cached.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace moe {

namespace mt {

constexpr int N = 312, M = 156, DEG = 19937;
constexpr uint64_t A = 0xB5026F5AA96619E9ULL, UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
constexpr int W = (DEG + 63) / 64 + 1;  // words of a polynomial of degree < DEG (+1 spare)
constexpr int kJumpR = 10;              // window words per lane in the jump

__host__ __device__ __forceinline__ uint64_t temper(uint64_t z) {
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    z ^= z >> 43;
    return z;
}
__host__ __device__ __forceinline__ uint64_t twist(uint64_t lo_word, uint64_t hi_word, uint64_t mid) {
    const uint64_t y = (lo_word & UM) | (hi_word & LM);
    return mid ^ (y >> 1) ^ ((y & 1ULL) ? A : 0ULL);
}

// ---------------------------------------------------------------- host: GF(2)
using Poly = std::vector<uint64_t>;

static inline int getbit(const Poly& p, long i) { return (p[i >> 6] >> (i & 63)) & 1; }
static inline void flipbit(Poly& p, long i) { p[i >> 6] ^= 1ULL << (i & 63); }

// dst ^= src << sh (bit shift), over dst's length
static void xor_shifted(Poly& dst, const Poly& src, long sh) {
    const long ws = sh >> 6;
    const int bs = static_cast<int>(sh & 63);
    const long n = static_cast<long>(dst.size());
    for (long i = static_cast<long>(src.size()) - 1; i >= 0; --i) {
        const uint64_t v = src[i];
        if (!v) continue;
        const long d0 = i + ws;
        if (d0 < n) dst[d0] ^= v << bs;
        if (bs && d0 + 1 < n) dst[d0 + 1] ^= v >> (64 - bs);
    }
}

// Characteristic polynomial of the raw word sequence (bit 0 of x[k], k >= 1),
// via Berlekamp-Massey over 2*DEG+64 terms.  Returns P(t) with P[DEG] = 1.
static Poly charpoly() {
    const long n2 = 2L * DEG + 64;
    // raw words x[1..n2] of mt19937_64 seeded with a generic seed
    std::vector<uint64_t> x(static_cast<size_t>(n2 + N + 1));
    x[0] = 5489ULL;
    for (int i = 1; i < N; ++i) x[i] = 6364136223846793005ULL * (x[i - 1] ^ (x[i - 1] >> 62)) + i;
    for (long k = N; k < static_cast<long>(x.size()); ++k) x[k] = twist(x[k - N], x[k - N + 1], x[k - N + M]);
    // sequence s_n = bit0(x[n+1]); stored reversed for windowed parities
    const long words = (n2 + 63) / 64 + 2;
    Poly R(static_cast<size_t>(words), 0);  // R bit (n2-1-n) = s_n
    for (long n = 0; n < n2; ++n)
        if (x[n + 1] & 1ULL) flipbit(R, n2 - 1 - n);
    const long pw = (DEG + 64) / 64 + 2;
    Poly Cp(static_cast<size_t>(pw), 0), Bp(static_cast<size_t>(pw), 0), Tp;
    Cp[0] = 1;
    Bp[0] = 1;
    long L = 0, m = 1;
    for (long n = 0; n < n2; ++n) {
        // d = sum_{i=0..L} c_i s_{n-i} = parity(C & (R >> (n2-1-n)) over L+1 bits)
        const long off = n2 - 1 - n;
        int par = 0;
        uint64_t acc = 0;
        // C has no bits above L, so no masking is needed
        const long lw = L / 64 + 1;
        const long w0 = off >> 6;
        const int b0 = static_cast<int>(off & 63);
        for (long i = 0; i < lw && w0 + i < words; ++i) {
            uint64_t r = R[w0 + i] >> b0;
            if (b0 && w0 + i + 1 < words) r |= R[w0 + i + 1] << (64 - b0);
            acc ^= Cp[i] & r;
        }
        par = __builtin_popcountll(acc) & 1;
        if (!par) {
            ++m;
        } else if (2 * L <= n) {
            Tp = Cp;
            xor_shifted(Cp, Bp, m);
            L = n + 1 - L;
            Bp = Tp;
            m = 1;
        } else {
            xor_shifted(Cp, Bp, m);
            ++m;
        }
    }
    if (L != DEG) throw Status(6, "mt19937_64 characteristic polynomial: unexpected degree");
    // P(t) = t^L C(1/t): P_k = c_{L-k}
    Poly P(static_cast<size_t>(W), 0);
    for (long k = 0; k <= L; ++k)
        if (getbit(Cp, L - k)) flipbit(P, k);
    return P;
}

struct Field {
    Poly P;
    Field() : P(charpoly()) {}
    // r (degree < 2*DEG) reduced mod P in place; result degree < DEG
    void reduce(Poly& r) const {
        for (long i = static_cast<long>(r.size()) * 64 - 1; i >= DEG; --i)
            if (getbit(r, i)) xor_shifted(r, P, i - DEG);
        r.resize(W);
    }
    Poly mul(const Poly& a, const Poly& b) const {
        Poly r(2 * W, 0);
        for (long i = 0; i < DEG; ++i)
            if (getbit(a, i)) xor_shifted(r, b, i);
        reduce(r);
        return r;
    }
    Poly sqr(const Poly& a) const {
        Poly r(2 * W, 0);
        for (long i = 0; i < DEG; ++i)
            if (getbit(a, i)) flipbit(r, 2 * i);
        reduce(r);
        return r;
    }
    Poly pow_t(uint64_t e) const {  // t^e mod P
        Poly r(W, 0);
        r[0] = 1;
        for (int b = 63; b >= 0; --b) {
            r = sqr(r);
            if ((e >> b) & 1) {  // r *= t
                Poly s(2 * W, 0);
                for (size_t i = 0; i < r.size(); ++i) s[i] = r[i];
                Poly t(2 * W, 0);
                xor_shifted(t, s, 1);
                reduce(t);
                r = t;
            }
        }
        return r;
    }
};

static const Field& field() {
    static std::unique_ptr<Field> f;
    static std::once_flag once;
    std::call_once(once, [] { f.reset(new Field()); });
    return *f;
}

// ---------------------------------------------------------------- device
// One CTA per chunk, 768 threads (24 warps), three overlapped phases:
//   1. base: x[1 .. BASE] regenerated from the seed in shared memory (every
//      CTA redundantly).  The host computes the 312 init words (a serial
//      nonlinear recurrence) and passes them as a kernel parameter; warp 0
//      twists blocks b = 1 .. kBaseBlocks in registers and publishes each
//      one on its own mbarrier.
//   2. jump (warps 1..23): the chunk's 312-word window =
//      XOR_{i : g_c,i} x[1 + j + i].  The bit range is cut into runs of
//      kRun 10-bit groups dealt round-robin to the jump warps, so all of them
//      advance through the base together right behind warp 0 and the base
//      costs only its first few blocks of latency.
//   3. generation: warp 0 runs the block recurrence (the serial critical
//      path) in registers and publishes each 312-word block into a
//      shared-memory ring (a full mbarrier per slot; one empty mbarrier per
//      half ring, waited once per 18 blocks); 18 emitter warps (those not on
//      warp 0's SM sub-partition) temper, convert and store whole blocks,
//      round-robin.
constexpr int kJumpWarps = 23;                        // warps 1..23 run the jump
constexpr int kChunkThreads = 32 * (kJumpWarps + 1);  // + warp 0: base producer, then twister
constexpr int kRun = 11;                              // 10-bit groups per run
constexpr int kRunsPerWarp = 8;
constexpr int kGroups = kJumpWarps * kRunsPerWarp * kRun;  // bits >= DEG of g are zero
static_assert(kGroups * kJumpR >= DEG, "jump groups cover the polynomial");
// the last lane's register window reads up to x[(kGroups + 32) * R]
constexpr int BASE = (kGroups + 33) * kJumpR;
constexpr int kBaseBlocks = BASE / N;                 // block b holds x[312b .. 312b + 311]
constexpr int kBaseAlloc = (kBaseBlocks + 2) * N;     // sb words (block stores never need a bound)
constexpr int kEmitters = kJumpWarps - kJumpWarps / 4;  // warps w in 1..23 with w % 4 != 0
constexpr int kRing = 2 * kEmitters;                  // ring slots: two halves of kEmitters
constexpr int kSlot = 320;                            // words per slot: A half [0,160), B half [160,320)
static_assert(kRing * kSlot <= BASE, "ring reuses the base region after the jump");

struct InitWords {  // x[0 .. 311] of init_genrand64(seed), host-computed
    uint64_t x[N];
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ uint32_t shfl_idx0(uint32_t v) {
    uint32_t r;
    asm volatile("shfl.sync.idx.b32 %0, %1, 0, 0x1f, 0xffffffff;" : "=r"(r) : "r"(v));
    return r;
}
__device__ __forceinline__ uint32_t shfl_down1(uint32_t v) {
    uint32_t r;
    asm volatile("shfl.sync.down.b32 %0, %1, 1, 0x1f, 0xffffffff;" : "=r"(r) : "r"(v));
    return r;
}
__device__ __forceinline__ uint64_t join(uint32_t lo, uint32_t hi) {
    return (static_cast<uint64_t>(hi) << 32) | lo;
}

// twist(lo, hi, mid) = mid ^ mix(lo, hi)
__device__ __forceinline__ uint64_t mix(uint64_t lo_word, uint64_t hi_word) {
    const uint64_t y = (lo_word & UM) | (hi_word & LM);
    return (y >> 1) ^ ((y & 1ULL) ? A : 0ULL);
}
// twist3(lo, hi, mid) = mix(lo, hi) ^ mid on 32-bit halves: y's high half is
// lo's, the low half merges lo's top bit with hi's low 31; one funnel shift,
// and the conditional A is a 32-bit sign-spread mask shared by both halves
// (9 ALU operations instead of the 64-bit form's ~12).
__device__ __forceinline__ uint64_t twist3(uint64_t lo_word, uint64_t hi_word, uint64_t mid) {
    const uint32_t lo_l = static_cast<uint32_t>(lo_word), lo_h = static_cast<uint32_t>(lo_word >> 32);
    const uint32_t hi_l = static_cast<uint32_t>(hi_word);
    const uint32_t y_l = (lo_l & 0x80000000u) | (hi_l & 0x7fffffffu);
    const uint32_t r_l = __funnelshift_r(y_l, lo_h, 1);
    const uint32_t r_h = lo_h >> 1;
    const uint32_t m = static_cast<uint32_t>(static_cast<int32_t>(hi_l << 31) >> 31);
    const uint32_t o_l = (r_l ^ static_cast<uint32_t>(mid)) ^ (static_cast<uint32_t>(A) & m);
    const uint32_t o_h = (r_h ^ static_cast<uint32_t>(mid >> 32)) ^ (static_cast<uint32_t>(A >> 32) & m);
    return (static_cast<uint64_t>(o_h) << 32) | o_l;
}

// One warp advances the 312-word state by one block, in registers.  Lane l
// holds the word pairs j = 5l + r and j + 156 (r < 5): A[r] = o[j],
// B[r] = o[j + 156] (lane 31's r >= 1, j >= 156, are padding).  Both halves
// of the block twist are then lane-local:
//   new[j]       = mix(o[j], o[j+1])         ^ o[j+156]   = mix(A[r], A[r+1]) ^ B[r]
//   new[j + 156] = mix(o[j+156], o[j+157])   ^ new[j]     = mix(B[r], B[r+1]) ^ newA[r]
// with the r+1 = 5 neighbours from lane l+1, and lane 31 (j = 155, 311 only)
// taking o[156] and new[0] from lane 0 (lane 31 rebuilds new[0] =
// mix(o[0], o[1]) ^ o[156] itself).  All cross-lane inputs are words r <= 1
// of the OLD block, so they are shuffled as soon as those are computed, one
// block ahead: the shuffle latency hides under the rest of the twist instead
// of heading the serial chain.  mix(lo, hi) reads lo's top 33 bits and hi's
// low 31, so the hi operands (a_next, b_next, o1) move only their low halves.
struct WarpTwister {
    uint64_t A[5], B[5];
    uint64_t a_next, b_next, o156, o0, o1;  // cross-lane inputs of the next twist

    __device__ __forceinline__ void fetch() {
        a_next = shfl_down1(static_cast<uint32_t>(A[0]));
        b_next = shfl_down1(static_cast<uint32_t>(B[0]));
        o156 = join(shfl_idx0(static_cast<uint32_t>(B[0])), shfl_idx0(static_cast<uint32_t>(B[0] >> 32)));
        o0 = join(shfl_idx0(static_cast<uint32_t>(A[0])), shfl_idx0(static_cast<uint32_t>(A[0] >> 32)));
        o1 = shfl_idx0(static_cast<uint32_t>(A[1]));
    }
    __device__ __forceinline__ void twist(int lane) {
        uint64_t nA[5];
        nA[0] = twist3(A[0], lane == 31 ? o156 : A[1], B[0]);  // j = 155 on lane 31
        nA[1] = twist3(A[1], A[2], B[1]);
        const uint64_t new0 = twist3(o0, o1, o156);
        const uint64_t nB0 = twist3(B[0], lane == 31 ? new0 : B[1], nA[0]);  // j = 311 on lane 31
        const uint64_t an = shfl_down1(static_cast<uint32_t>(nA[0]));
        const uint64_t bn = shfl_down1(static_cast<uint32_t>(nB0));
        const uint64_t p156 = join(shfl_idx0(static_cast<uint32_t>(nB0)), shfl_idx0(static_cast<uint32_t>(nB0 >> 32)));
        const uint64_t p0 = join(shfl_idx0(static_cast<uint32_t>(nA[0])), shfl_idx0(static_cast<uint32_t>(nA[0] >> 32)));
        const uint64_t p1 = shfl_idx0(static_cast<uint32_t>(nA[1]));
#pragma unroll
        for (int r = 2; r < 5; ++r) nA[r] = twist3(A[r], r < 4 ? A[r + 1] : a_next, B[r]);
#pragma unroll
        for (int r = 1; r < 5; ++r) B[r] = twist3(B[r], r < 4 ? B[r + 1] : b_next, nA[r]);
        B[0] = nB0;
#pragma unroll
        for (int r = 0; r < 5; ++r) A[r] = nA[r];
        a_next = an;
        b_next = bn;
        o156 = p156;
        o0 = p0;
        o1 = p1;
    }
};

__global__ void __launch_bounds__(kChunkThreads, 1)
chunk_kernel(const __grid_constant__ InitWords init, const uint16_t* __restrict__ masks, int64_t J,
             int64_t count, double lo, double span, float* __restrict__ noise,
             uint64_t* __restrict__ raw_out, unsigned long long* __restrict__ tdbg) {
    extern __shared__ uint64_t sm[];
    uint64_t* sb = sm;                                   // x[k] at sb[k-1]; later the ring [kRing][kSlot]
    uint64_t* win = sb + kBaseAlloc;                     // jump result [N]
    uint64_t* pad = win + N;                             // sink for lane 31's padding words [16]
    uint64_t* bb = pad + 16;                             // base block mbarriers [kBaseBlocks + 1]
    uint64_t* full = bb + kBaseBlocks + 1;               // ring mbarriers [kRing]
    uint64_t* empty = full + kRing;                      // half-ring mbarriers [2]
    uint16_t* sg = reinterpret_cast<uint16_t*>(empty + 2);  // g_c masks [kGroups]
    uint64_t* ring = sb;
    const int c = blockIdx.x;
    const int64_t q0 = static_cast<int64_t>(c) * J;
    if (q0 >= count) return;
    const int t = threadIdx.x;
    const int warp = t >> 5, lane = t & 31;
    auto stamp = [&](int k) {  // debug phase timeline (MOE_B200_RNG_TIMING)
        if (tdbg) {
            unsigned long long ns;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
            tdbg[c * 8 + k] = ns;
        }
    };
    if (t == 0) stamp(0);
    for (int i = t; i < kGroups; i += kChunkThreads) sg[i] = masks[static_cast<int64_t>(c) * kGroups + i];
    for (int i = t; i < N; i += kChunkThreads) win[i] = 0;
    if (t == 0) {
        for (int i = 1; i <= kBaseBlocks; ++i) mbar_init(&bb[i], 32);
        for (int i = 0; i < kRing; ++i) mbar_init(&full[i], 32);  // all twister lanes arrive
        mbar_init(&empty[0], 32 * kEmitters);                     // every emitter lane, once per lap
        mbar_init(&empty[1], 32 * kEmitters);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    pdl_wait();  // the noise buffer may still be read by the previous kernels
    pdl_trigger();
    __syncthreads();
    constexpr int R = kJumpR;
    if (warp == 0) {
        // ---- 1. base: blocks b = 1 .. kBaseBlocks of x, each published on bb[b]
        WarpTwister tw;
#pragma unroll
        for (int r = 0; r < 5; ++r) {
            const int j = min(lane * 5 + r, M - 1);
            tw.A[r] = init.x[j];
            tw.B[r] = init.x[j + M];
            if (j == lane * 5 + r) {  // block 0: x[1 .. 311] (published with block 1)
                if (j >= 1) sb[j - 1] = tw.A[r];
                sb[j + M - 1] = tw.B[r];
            }
        }
        tw.fetch();
        for (int b = 1; b <= kBaseBlocks; ++b) {
            tw.twist(lane);
            uint64_t* dst = sb + b * N - 1 + lane * 5;  // x[312b + j] at sb[312b + j - 1]
#pragma unroll
            for (int r = 0; r < 5; ++r) *((lane == 31 && r > 0) ? pad + r : dst + r) = tw.A[r];
#pragma unroll
            for (int r = 0; r < 5; ++r) *((lane == 31 && r > 0) ? pad + 8 + r : dst + r + M) = tw.B[r];
            mbar_arrive(&bb[b]);
        }
        if (lane == 0) stamp(1);
    } else {
        // ---- 2. jump.  Lane l owns R consecutive window words j = l*R + r
        // in registers and slides a register window over the base, so each
        // bit costs one shared load plus (if set) R XORs; bits are taken in
        // pairs so two set bits cost one 3-input XOR pass (acc ^ a ^ b).
        // Masks are warp-uniform (no divergence).  Partial windows meet in
        // `win` via shared atomic XOR.
        const int jw = warp - 1;
        const int j0 = lane * R;
        uint64_t acc[R], wr[R];
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = 0;
        for (int run = 0; run < kRunsPerWarp; ++run) {
            const int g0 = (run * kJumpWarps + jw) * kRun;
            // last word this run reads: x[(g0 + kRun + 32) * R]
            const int blk = (g0 + kRun + 32) * R / N;
            mbar_wait(&bb[blk], 0);
#pragma unroll
            for (int r = 0; r < R; ++r) wr[r] = sb[g0 * R + j0 + r];
            for (int g = 0; g < kRun; ++g) {
                const int i = (g0 + g) * R;
                const uint32_t m = sg[g0 + g];
                uint64_t nx[R];
#pragma unroll
                for (int q = 0; q < R; ++q) nx[q] = sb[i + j0 + R + q];
#pragma unroll
                for (int s2 = 0; s2 < R; s2 += 2) {
                    const uint32_t pr = (m >> s2) & 3u;
                    // bit s2 reads wr[(s2+r)%R]; bit s2+1 reads wr[(s2+1+r)%R],
                    // except r = R-1: the slot s2 refill (nx[s2])
                    if (pr == 3u) {
#pragma unroll
                        for (int r = 0; r < R; ++r)
                            acc[r] ^= wr[(s2 + r) % R] ^ (r == R - 1 ? nx[s2] : wr[(s2 + 1 + r) % R]);
                    } else if (pr == 1u) {
#pragma unroll
                        for (int r = 0; r < R; ++r) acc[r] ^= wr[(s2 + r) % R];
                    } else if (pr == 2u) {
#pragma unroll
                        for (int r = 0; r < R; ++r) acc[r] ^= (r == R - 1 ? nx[s2] : wr[(s2 + 1 + r) % R]);
                    }
                    wr[s2] = nx[s2];
                    wr[s2 + 1] = nx[s2 + 1];
                }
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r)
            if (j0 + r < N) atomicXor(reinterpret_cast<unsigned long long*>(&win[j0 + r]), acc[r]);
    }
    __syncthreads();  // base no longer read: its space becomes the ring
    if (t == 0) stamp(2);
    // ---- 3. generation.  Block b -> ring slot b % kRing, emitter b % kEmitters.
    const int64_t n = min(J, count - q0);
    const int nblk = static_cast<int>((n + N - 1) / N);
    if (warp == 0) {
        WarpTwister tw;
#pragma unroll
        for (int r = 0; r < 5; ++r) {
            const int j = min(lane * 5 + r, M - 1);
            tw.A[r] = win[j];
            tw.B[r] = win[j + M];
        }
        tw.fetch();
        int slot = 0;
        uint32_t lap = 0;
        const long long cyc0 = clock64();
        long long wait_cyc = 0;
        for (int b = 0; b < nblk; ++b) {
            if (b > 0) tw.twist(lane);
            // slots of half h are rewritten once all emitters released them
            if (lap > 0 && (slot == 0 || slot == kEmitters)) {
                const long long w0 = clock64();
                mbar_wait(&empty[slot != 0], (lap - 1) & 1);
                wait_cyc += clock64() - w0;
            }
            uint64_t* dst = ring + slot * kSlot + lane * 5;  // lane 31's r > 0 hit the pads
#pragma unroll
            for (int r = 0; r < 5; ++r) {
                dst[r] = tw.A[r];
                dst[r + kSlot / 2] = tw.B[r];
            }
            mbar_arrive(&full[slot]);
            if (++slot == kRing) {
                slot = 0;
                ++lap;
            }
        }
        if (lane == 0) {
            stamp(3);
            if (tdbg) tdbg[c * 8 + 6] = static_cast<unsigned long long>(clock64() - cyc0);
            if (tdbg) tdbg[c * 8 + 7] = static_cast<unsigned long long>(wait_cyc);
        }
    } else if (warp & 3) {  // not on warp 0's SM sub-partition (warp w runs on SMSP w % 4)
        const int k = (warp >> 2) * 3 + (warp & 3) - 1;  // 0 .. kEmitters-1
        for (int b = k; b < nblk; b += kEmitters) {
            const int slot = b % kRing;
            mbar_wait(&full[slot], (b / kRing) & 1);
            const uint64_t* src = ring + slot * kSlot;
            const int64_t qb = static_cast<int64_t>(b) * N;
#pragma unroll
            for (int it = 0; it < kSlot / 32; ++it) {
                const int p = lane + 32 * it;  // slot position; 156..159 and 316..319 are pads
                const int i = p < kSlot / 2 ? p : p - (kSlot / 2 - M);
                const int64_t q = qb + i;
                if ((p < M || p >= kSlot / 2) && p < kSlot / 2 + M && q < n) {
                    const uint64_t out = temper(src[p]);
                    if (raw_out) raw_out[q0 + q] = out;
                    if (noise) {
                        // lo + (hi - lo) * u53 * 2^-53 in f64 without
                        // contraction, exactly as the reference (rng.cpp:36-43)
                        const double uu = static_cast<double>(out >> 11) * 0x1.0p-53;
                        noise[q0 + q] = static_cast<float>(__dadd_rn(lo, __dmul_rn(span, uu)));
                    }
                }
            }
            mbar_arrive(&empty[slot >= kEmitters]);
        }
        if (lane == 0 && warp == 1) stamp(4);
    }
}

// Jump masks for chunk length J and P chunks: g_c = t^(311 + c*J) mod phi,
// repacked as kJumpR-bit groups (one uint16 per group) for the device loop.
struct Table {
    int64_t J = 0;
    int P = 0;
    uint16_t* dev = nullptr;  // [P][kGroups]
};

static std::mutex g_mu;
static std::map<std::pair<int64_t, int>, Table> g_tables;

static const Table& table_for(int64_t J, int P) {
    std::lock_guard<std::mutex> lk(g_mu);
    auto key = std::make_pair(J, P);
    auto it = g_tables.find(key);
    if (it != g_tables.end()) return it->second;
    const Field& F = field();
    std::vector<uint16_t> host(static_cast<size_t>(P) * kGroups, 0);
    Poly g = F.pow_t(311);
    const Poly step = F.pow_t(static_cast<uint64_t>(J));
    for (int c = 0; c < P; ++c) {
        uint16_t* dst = host.data() + static_cast<size_t>(c) * kGroups;
        for (long i = 0; i < DEG; ++i)
            if (getbit(g, i)) dst[i / kJumpR] |= static_cast<uint16_t>(1u << (i % kJumpR));
        if (c + 1 < P) g = F.mul(g, step);
    }
    Table t;
    t.J = J;
    t.P = P;
    MOE_CUDA_CHECK(cudaMalloc(&t.dev, sizeof(uint16_t) * host.size()));
    MOE_CUDA_CHECK(cudaMemcpy(t.dev, host.data(), sizeof(uint16_t) * host.size(), cudaMemcpyHostToDevice));
    return g_tables.emplace(key, t).first->second;
}

void generate(uint64_t seed, int64_t count, double lo, double hi, float* noise, uint64_t* raw,
              cudaStream_t st, int max_ctas = kNumSMs) {
    if (count <= 0) return;
    const int P = static_cast<int>(std::min<int64_t>(std::max(1, max_ctas), ceil_div(count, 4096)));
    const int64_t J = ceil_div(count, P);
    const Table& tab = table_for(J, P);
    const size_t smem = sizeof(uint64_t) * (kBaseAlloc + N + 16 + kBaseBlocks + 1 + kRing + 2) +
                        sizeof(uint16_t) * kGroups;
    InitWords init;  // init_genrand64 (rng.cpp: std::mt19937_64 seeding)
    init.x[0] = seed;
    for (int i = 1; i < N; ++i)
        init.x[i] = 6364136223846793005ULL * (init.x[i - 1] ^ (init.x[i - 1] >> 62)) + static_cast<uint64_t>(i);
    static bool attr = false;
    if (!attr) {
        MOE_CUDA_CHECK(cudaFuncSetAttribute(chunk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(smem)));
        attr = true;
    }
    static unsigned long long* tdbg = nullptr;
    static const bool timing = std::getenv("MOE_B200_RNG_TIMING") != nullptr;
    if (timing && !tdbg) MOE_CUDA_CHECK(cudaMalloc(&tdbg, sizeof(unsigned long long) * 8 * kNumSMs));
    // debug (timing runs only): =1 drops the stores, timing the recurrence alone
    static const bool null_out = timing && std::getenv("MOE_B200_RNG_NULL_OUT") != nullptr;
    if (null_out) noise = nullptr, raw = nullptr;
    static const bool pair_tpc = [] {
        const char* e = std::getenv("MOE_B200_PF_TPC");
        return !(e && e[0] == '0');
    }();
    if (pair_tpc && P < kNumSMs && P % 2 == 0) {
        // a generator sharing the GPU with persistent GEMMs: CTAs in clusters of
        // two, so they hold whole TPCs and leave the other TPCs' SM pairs to the
        // cta_group::2 GEMM kernels
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[1].val.programmaticStreamSerializationAllowed = pdl_on() ? 1 : 0;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(P);
        cfg.blockDim = dim3(kChunkThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cfg.attrs = at;
        cfg.numAttrs = 2;
        MOE_CUDA_CHECK(cudaLaunchKernelEx(&cfg, chunk_kernel, init, static_cast<const uint16_t*>(tab.dev), J, count, lo,
                                          hi - lo, noise, raw, timing ? tdbg : nullptr));
        count_launch();
    } else {
        launch_pdl(chunk_kernel, dim3(P), dim3(kChunkThreads), smem, st, init, tab.dev, J, count, lo, hi - lo,
                   noise, raw, timing ? tdbg : nullptr);
    }
    if (timing) {  // debug: per-phase times averaged over CTAs (synchronises)
        std::vector<unsigned long long> h(8 * static_cast<size_t>(P));
        MOE_CUDA_CHECK(cudaStreamSynchronize(st));
        MOE_CUDA_CHECK(cudaMemcpy(h.data(), tdbg, sizeof(unsigned long long) * h.size(),
                                  cudaMemcpyDeviceToHost));
        double ph[4] = {0, 0, 0, 0};
        for (int c = 0; c < P; ++c)
            for (int k = 0; k < 4; ++k) ph[k] += double(static_cast<long long>(h[c * 8 + k + 1] - h[c * 8 + k])) / P;
        double cyc = 0;
        double wcyc = 0;
        for (int c = 0; c < P; ++c) cyc += double(h[c * 8 + 6]) / P, wcyc += double(h[c * 8 + 7]) / P;
        std::fprintf(stderr, "[rng] twister empty-wait %.0f cycles/block\n", wcyc / double(ceil_div(J, (int64_t)N)));
        std::fprintf(stderr, "[rng] P=%d J=%lld base %.1f us, jump %.1f us, twister %.1f us (%.0f cycles/block), emit tail %.1f us\n",
                     P, static_cast<long long>(J), ph[0] / 1e3, ph[1] / 1e3, ph[2] / 1e3,
                     cyc / double(ceil_div(J, (int64_t)N)), ph[3] / 1e3);
    }
}

}  // namespace mt


bool launch_jitter_noise_device(uint64_t seed, int64_t count, double eps, float* noise,
                                cudaStream_t st, int max_ctas) {
    mt::generate(seed, count, 1.0 - eps, 1.0 + eps, noise, nullptr, st, max_ctas);
    return true;
}

void launch_mt64_raw_device(uint64_t seed, int64_t count, uint64_t* out, cudaStream_t st) {
    mt::generate(seed, count, 0.0, 1.0, nullptr, out, st);
}

// host-only check of the jump machinery (no GPU): raw outputs [c*J, c*J + n)
// of chunk c computed from the jump polynomial, for CPU tests.
void host_mt64_chunk(uint64_t seed, int64_t J, int P, int c, int64_t n, uint64_t* out) {
    using namespace mt;
    const Field& F = field();
    const Poly g = F.pow_t(311 + static_cast<uint64_t>(c) * J);
    (void)P;
    std::vector<uint64_t> x(static_cast<size_t>(BASE + N + 1));
    x[0] = seed;
    for (int i = 1; i < N; ++i) x[i] = 6364136223846793005ULL * (x[i - 1] ^ (x[i - 1] >> 62)) + i;
    for (size_t k = N; k < x.size(); ++k) x[k] = twist(x[k - N], x[k - N + 1], x[k - N + M]);
    uint64_t s[N];
    for (int j = 0; j < N; ++j) {
        uint64_t acc = 0;
        for (long i = 0; i < DEG; ++i)
            if (getbit(g, i)) acc ^= x[1 + j + i];
        s[j] = acc;
    }
    for (int64_t q = 0; q < n; ++q) {
        if (q > 0 && q % N == 0) {
            uint64_t t[N];
            for (int i = 0; i < N; ++i) t[i] = s[i];
            for (int i = 0; i < N - M; ++i) t[i] = twist(s[i], s[i + 1], s[i + M]);
            for (int i = N - M; i < N - 1; ++i) t[i] = twist(s[i], s[i + 1], t[i + M - N]);
            t[N - 1] = twist(s[N - 1], t[0], t[M - 1]);
            for (int i = 0; i < N; ++i) s[i] = t[i];
        }
        out[q] = temper(s[q % N]);
    }
}

}  // namespace moe
