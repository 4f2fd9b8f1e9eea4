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
//    and base = x[1 .. 20249) generated once per call from the seed.
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
// One CTA per chunk, 768 threads, three phases:
//   1. base: x[1 .. BASE] regenerated from the seed in shared memory (every
//      CTA redundantly) by the warp twister below;
//   2. jump: the chunk's 312-word window = XOR_{i : g_c,i} x[1 + j + i], all
//      32 warps;
//   3. generation: warp 0 runs the block recurrence (the serial critical
//      path) entirely in registers and publishes each 312-word block into a
//      shared-memory ring (mbarrier full/empty per slot); 18 emitter warps
//      (those not on warp 0's SM sub-partition) temper, convert and store
//      whole blocks, round-robin.
constexpr int kChunkThreads = 768;
constexpr int kJumpWarps = kChunkThreads / 32;
// bits per warp in the jump, a multiple of kJumpR so each warp's range is
// whole R-bit mask groups; bits >= DEG of g are zero.
constexpr int kGroupsPerWarp = (DEG + kJumpWarps * kJumpR - 1) / (kJumpWarps * kJumpR);
constexpr int kGroups = kJumpWarps * kGroupsPerWarp;
// the last lane's register window reads up to kGroups*R + 32*R + R words
constexpr int BASE = kGroups * kJumpR + 32 * kJumpR + kJumpR;
constexpr int kBaseBlocks = (BASE + N) / N;  // x[312*b ..] blocks b = 1..kBaseBlocks
constexpr int kEmitters = kJumpWarps / 4 * 3;  // warps w with w % 4 != 0
constexpr int kRing = 2 * kEmitters;         // ring slots (a multiple of kEmitters)
static_assert(kRing * N <= BASE, "ring reuses the base region after the jump");

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
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

// twist(lo, hi, mid) = mid ^ mix(lo, hi)
__device__ __forceinline__ uint64_t mix(uint64_t lo_word, uint64_t hi_word) {
    const uint64_t y = (lo_word & UM) | (hi_word & LM);
    return (y >> 1) ^ ((y & 1ULL) ? A : 0ULL);
}

// One warp advances the 312-word state by one block, in registers.  Lane l
// holds the word pairs j = 5l + r and j + 156 (r < 5, j < 156): A[r] = o[j],
// B[r] = o[j + 156].  Then both halves of the block twist are lane-local:
//   new[j]       = mix(o[j], o[j+1])         ^ o[j+156]   = mix(A[r], A[r+1]) ^ B[r]
//   new[j + 156] = mix(o[j+156], o[j+157])   ^ new[j]     = mix(B[r], B[r+1]) ^ newA[r]
// with the r+1 = 5 neighbours from lane l+1, and lane 31 (j = 155, 311 only)
// taking o[156] and new[0] from lane 0.
__device__ __forceinline__ void warp_twist(uint64_t (&Aw)[5], uint64_t (&Bw)[5], int lane) {
    // all cross-lane inputs are fetched up front (one batch of shuffles):
    // lane 31 also rebuilds new[0] = mix(o[0], o[1]) ^ o[156] from lane 0's
    // old words instead of waiting for lane 0's result
    const uint64_t a_next = __shfl_down_sync(0xffffffffu, Aw[0], 1);
    const uint64_t b_next = __shfl_down_sync(0xffffffffu, Bw[0], 1);
    const uint64_t o156 = __shfl_sync(0xffffffffu, Bw[0], 0);
    const uint64_t o0 = __shfl_sync(0xffffffffu, Aw[0], 0);
    const uint64_t o1 = __shfl_sync(0xffffffffu, Aw[1], 0);
    uint64_t nA[5];
#pragma unroll
    for (int r = 0; r < 5; ++r) {
        uint64_t hi = r < 4 ? Aw[r + 1] : a_next;
        if (r == 0 && lane == 31) hi = o156;  // j = 155
        nA[r] = mix(Aw[r], hi) ^ Bw[r];
    }
    const uint64_t new0 = mix(o0, o1) ^ o156;
#pragma unroll
    for (int r = 0; r < 5; ++r) {
        uint64_t hi = r < 4 ? Bw[r + 1] : b_next;
        if (r == 0 && lane == 31) hi = new0;  // j = 311
        Bw[r] = mix(Bw[r], hi) ^ nA[r];
        Aw[r] = nA[r];
    }
}

__global__ void __launch_bounds__(kChunkThreads, 1)
chunk_kernel(uint64_t seed, const uint16_t* __restrict__ masks, int64_t J, int64_t count,
             double lo, double span, float* __restrict__ noise, uint64_t* __restrict__ raw_out,
             unsigned long long* __restrict__ tdbg) {
    extern __shared__ uint64_t sm[];
    uint64_t* sb = sm;                                   // x[1 .. BASE]; later the ring [kRing][N]
    uint64_t* win = sb + BASE;                           // jump result [N]
    uint64_t* full = win + N;                            // mbarriers [kRing]
    uint64_t* empty = full + kRing;                      // mbarriers [kRing]
    uint16_t* sg = reinterpret_cast<uint16_t*>(empty + kRing);  // g_c masks [kGroups]
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
        for (int i = 0; i < kRing; ++i) {
            mbar_init(&full[i], 32);   // all twister lanes arrive
            mbar_init(&empty[i], 32);  // all lanes of the slot's emitter arrive
        }
    }
    // ---- 1. base sequence: init_genrand64 (thread 0), then warp 0 twists
    // blocks b = 1.. in registers and writes x[312b + j] to sb[312b + j - 1].
    if (warp == 0) {
        if (lane == 0) {
            uint64_t v = seed;
            win[0] = v;  // x[0] (scratch; win is cleared again below)
            for (int i = 1; i < N; ++i) {
                v = 6364136223846793005ULL * (v ^ (v >> 62)) + static_cast<uint64_t>(i);
                sb[i - 1] = v;
            }
        }
        __syncwarp();
        uint64_t Aw[5], Bw[5];
#pragma unroll
        for (int r = 0; r < 5; ++r) {
            const int j = lane * 5 + r;
            Aw[r] = j == 0 ? win[0] : (j < M ? sb[j - 1] : 0);
            Bw[r] = j < M ? sb[j + M - 1] : 0;
        }
        __syncwarp();
        if (lane == 0) win[0] = 0;
        for (int b = 1; b <= kBaseBlocks; ++b) {
            warp_twist(Aw, Bw, lane);
#pragma unroll
            for (int r = 0; r < 5; ++r) {
                const int j = lane * 5 + r;
                const int k = b * N + j;
                if (j < M) {
                    if (k <= BASE) sb[k - 1] = Aw[r];
                    if (k + M <= BASE) sb[k + M - 1] = Bw[r];
                }
            }
        }
    }
    __syncthreads();
    if (t == 0) stamp(1);
    // ---- 2. jump.  Warp w takes mask groups [w*G, (w+1)*G); lane l owns
    // R consecutive window words j = l*R + r in registers and slides a
    // register window over the base, so each bit costs one shared load plus
    // (if set) R XORs; the mask is warp-uniform (no divergence).  Partial
    // windows meet in `win` via shared atomic XOR.
    {
        constexpr int R = kJumpR;
        const int i0 = warp * kGroupsPerWarp * R;
        const int j0 = lane * R;
        uint64_t acc[R], wr[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            acc[r] = 0;
            wr[r] = sb[i0 + j0 + r];
        }
        const uint16_t* gm = sg + warp * kGroupsPerWarp;
        for (int g = 0; g < kGroupsPerWarp; ++g) {
            const int i = i0 + g * R;
            const uint32_t m = gm[g];
#pragma unroll
            for (int s = 0; s < R; ++s) {
                if (m & (1u << s)) {
#pragma unroll
                    for (int r = 0; r < R; ++r) acc[r] ^= wr[(s + r) % R];
                }
                wr[s] = sb[i + j0 + R + s];
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
        uint64_t Aw[5], Bw[5];
#pragma unroll
        for (int r = 0; r < 5; ++r) {
            const int j = lane * 5 + r;
            Aw[r] = j < M ? win[j] : 0;
            Bw[r] = j < M ? win[j + M] : 0;
        }
        // Every lane arrives on full[] (count 32), one block late, so the
        // release never waits on stores still in flight; the empty[] check
        // for the next slot is issued before the twist so its latency hides.
        int slot = 0, prev = -1;
        uint32_t lap = 0;
        for (int b = 0; b < nblk; ++b) {
            const bool ready = b < kRing || mbar_test(&empty[slot], lap ^ 1u);
            if (b > 0) warp_twist(Aw, Bw, lane);
            if (prev >= 0) mbar_arrive(&full[prev]);
            if (!ready) mbar_wait(&empty[slot], lap ^ 1u);
            uint64_t* dst = ring + slot * N + lane * 5;
#pragma unroll
            for (int r = 0; r < 5; ++r) {
                if (lane * 5 + r < M) {
                    dst[r] = Aw[r];
                    dst[r + M] = Bw[r];
                }
            }
            prev = slot;
            if (++slot == kRing) {
                slot = 0;
                lap ^= 1u;
            }
        }
        if (prev >= 0) mbar_arrive(&full[prev]);
        if (lane == 0) stamp(3);
    } else if (warp & 3) {
        const int k = (warp >> 2) * 3 + (warp & 3) - 1;  // 0 .. kEmitters-1
        for (int b = k; b < nblk; b += kEmitters) {
            const int slot = b % kRing;
            mbar_wait(&full[slot], (b / kRing) & 1);
            const uint64_t* src = ring + slot * N;
            const int64_t qb = static_cast<int64_t>(b) * N;
#pragma unroll
            for (int it = 0; it < (N + 31) / 32; ++it) {
                const int i = lane + 32 * it;
                const int64_t q = qb + i;
                if (i < N && q < n) {
                    const uint64_t out = temper(src[i]);
                    if (raw_out) raw_out[q0 + q] = out;
                    if (noise) {
                        // lo + (hi - lo) * u53 * 2^-53 in f64 without
                        // contraction, exactly as the reference (rng.cpp:36-43)
                        const double uu = static_cast<double>(out >> 11) * 0x1.0p-53;
                        noise[q0 + q] = static_cast<float>(__dadd_rn(lo, __dmul_rn(span, uu)));
                    }
                }
            }
            mbar_arrive(&empty[slot]);
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
              cudaStream_t st) {
    if (count <= 0) return;
    const int P = static_cast<int>(std::min<int64_t>(kNumSMs, ceil_div(count, 4096)));
    const int64_t J = ceil_div(count, P);
    const Table& tab = table_for(J, P);
    const size_t smem = sizeof(uint64_t) * (BASE + N + 2 * kRing) + sizeof(uint16_t) * kGroups;
    static bool attr = false;
    if (!attr) {
        MOE_CUDA_CHECK(cudaFuncSetAttribute(chunk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(smem)));
        attr = true;
    }
    static unsigned long long* tdbg = nullptr;
    static const bool timing = std::getenv("MOE_B200_RNG_TIMING") != nullptr;
    if (timing && !tdbg) MOE_CUDA_CHECK(cudaMalloc(&tdbg, sizeof(unsigned long long) * 8 * kNumSMs));
    chunk_kernel<<<P, kChunkThreads, smem, st>>>(seed, tab.dev, J, count, lo, hi - lo, noise, raw,
                                                 timing ? tdbg : nullptr);
    MOE_LAUNCH_CHECK();
    if (timing) {  // debug: per-phase times averaged over CTAs (synchronises)
        std::vector<unsigned long long> h(8 * static_cast<size_t>(P));
        MOE_CUDA_CHECK(cudaStreamSynchronize(st));
        MOE_CUDA_CHECK(cudaMemcpy(h.data(), tdbg, sizeof(unsigned long long) * h.size(),
                                  cudaMemcpyDeviceToHost));
        double ph[4] = {0, 0, 0, 0};
        for (int c = 0; c < P; ++c)
            for (int k = 0; k < 4; ++k) ph[k] += double(static_cast<long long>(h[c * 8 + k + 1] - h[c * 8 + k])) / P;
        std::fprintf(stderr, "[rng] P=%d J=%lld base %.1f us, jump %.1f us, twister %.1f us, emit tail %.1f us\n",
                     P, static_cast<long long>(J), ph[0] / 1e3, ph[1] / 1e3, ph[2] / 1e3, ph[3] / 1e3);
    }
}

}  // namespace mt


bool launch_jitter_noise_device(uint64_t seed, int64_t count, double eps, float* noise,
                                cudaStream_t st) {
    mt::generate(seed, count, 1.0 - eps, 1.0 + eps, noise, nullptr, st);
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
