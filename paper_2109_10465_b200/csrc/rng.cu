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
// base words x[1 .. BASE]: DEG + N are needed by the jump; the sliding
// window of the last lane reads up to 32*kJumpR + 2*kJumpR words past DEG.
constexpr int BASE = DEG + 32 * kJumpR + 2 * kJumpR + 8;
constexpr int kThreads = 320;

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

// Jump table for chunk length J and P chunks: g_c = t^(311 + c*J) mod phi.
struct Table {
    int64_t J = 0;
    int P = 0;
    uint64_t* dev = nullptr;  // [P][W]
};

static std::mutex g_mu;
static std::map<std::pair<int64_t, int>, Table> g_tables;

static const Table& table_for(int64_t J, int P) {
    std::lock_guard<std::mutex> lk(g_mu);
    auto key = std::make_pair(J, P);
    auto it = g_tables.find(key);
    if (it != g_tables.end()) return it->second;
    const Field& F = field();
    std::vector<uint64_t> host(static_cast<size_t>(P) * W);
    Poly g = F.pow_t(311);
    const Poly step = F.pow_t(static_cast<uint64_t>(J));
    for (int c = 0; c < P; ++c) {
        std::memcpy(host.data() + static_cast<size_t>(c) * W, g.data(), sizeof(uint64_t) * W);
        if (c + 1 < P) g = F.mul(g, step);
    }
    Table t;
    t.J = J;
    t.P = P;
    MOE_CUDA_CHECK(cudaMalloc(&t.dev, sizeof(uint64_t) * host.size()));
    MOE_CUDA_CHECK(cudaMemcpy(t.dev, host.data(), sizeof(uint64_t) * host.size(), cudaMemcpyHostToDevice));
    return g_tables.emplace(key, t).first->second;
}

// ---------------------------------------------------------------- device
// Base sequence x[1 .. BASE] from the seed (single CTA).
__global__ void __launch_bounds__(kThreads) base_kernel(uint64_t seed, uint64_t* __restrict__ base) {
    __shared__ uint64_t s[N];
    if (threadIdx.x == 0) {
        uint64_t v = seed;
        s[0] = v;
        for (int i = 1; i < N; ++i) {
            v = 6364136223846793005ULL * (v ^ (v >> 62)) + static_cast<uint64_t>(i);
            s[i] = v;
        }
    }
    __syncthreads();
    // x[1..311]
    for (int i = threadIdx.x + 1; i < N; i += blockDim.x) base[i - 1] = s[i];
    // twist blocks: x[312*b .. 312*b + 311]
    const int nblk = (BASE + 1 + N - 1) / N;  // enough blocks to cover x[BASE]
    for (int b = 1; b <= nblk; ++b) {
        const int i = threadIdx.x;
        uint64_t v0 = 0;
        if (i < N - M) v0 = twist(s[i], s[i + 1], s[i + M]);
        __syncthreads();
        if (i < N - M) s[i] = v0;
        __syncthreads();
        uint64_t v1 = 0;
        if (i >= N - M && i < N - 1) v1 = twist(s[i], s[i + 1], s[i + M - N]);
        __syncthreads();
        if (i >= N - M && i < N - 1) s[i] = v1;
        __syncthreads();
        if (i == N - 1) s[N - 1] = twist(s[N - 1], s[0], s[M - 1]);
        __syncthreads();
        for (int q = threadIdx.x; q < N; q += blockDim.x) {
            const long k = static_cast<long>(b) * N + q;  // raw index
            if (k - 1 < BASE) base[k - 1] = s[q];
        }
        __syncthreads();
    }
}

// New word i of the next 312-block computed from the OLD block only (the
// reference twist updates in place; words >= 156 read already-updated words
// 0..155, which we recompute locally), so a block needs one barrier.
__device__ __forceinline__ uint64_t next_word(const uint64_t* __restrict__ o, int i) {
    if (i < N - M) return twist(o[i], o[i + 1], o[i + M]);
    if (i < N - 1) return twist(o[i], o[i + 1], twist(o[i - (N - M)], o[i - (N - M) + 1], o[i]));
    // i == N-1: needs new[0] and new[M-1]
    const uint64_t n0 = twist(o[0], o[1], o[M]);
    const uint64_t nm = twist(o[M - 1], o[M], o[N - 1]);
    return twist(o[N - 1], n0, nm);
}

constexpr int kChunkThreads = 2 * N + 16;  // 640 = 20 warps
constexpr int kRing = 4;                    // generation ring depth (312-word blocks)
constexpr int kBarFull = 1, kBarEmpty = kBarFull + kRing, kBarTw = kBarEmpty + kRing;

__device__ __forceinline__ void bar_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int count) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// One CTA per chunk: jump to the chunk's window, then generate J outputs.
__global__ void __launch_bounds__(kChunkThreads, 1)
chunk_kernel(const uint64_t* __restrict__ base, const uint64_t* __restrict__ jump, int64_t J,
             int64_t count, double lo, double span, float* __restrict__ noise,
             uint64_t* __restrict__ raw_out) {
    extern __shared__ uint64_t sm[];
    uint64_t* sb = sm;              // base [BASE]
    uint64_t* sg = sm + BASE;       // g_c  [W]
    uint64_t* s0 = sg + W;          // ping [N]
    const int c = blockIdx.x;
    const int64_t q0 = static_cast<int64_t>(c) * J;
    if (q0 >= count) return;
    for (int i = threadIdx.x; i < BASE; i += blockDim.x) sb[i] = base[i];
    for (int i = threadIdx.x; i < W; i += blockDim.x) sg[i] = jump[static_cast<int64_t>(c) * W + i];
    __syncthreads();
    // window word j = XOR_{i : g_i} base[j + i].  Warp w takes bit range
    // [w*L, (w+1)*L) of g; lane l owns R consecutive words j = l*R + r in
    // registers and slides a register window over base, so each bit costs one
    // shared load plus R predicated XORs (g's bit is warp-uniform: no
    // divergence).  Partial windows meet in shared memory via atomic XOR.
    const int t = threadIdx.x;
    const int warp = t >> 5, lane = t & 31;
    for (int i = t; i < N; i += blockDim.x) s0[i] = 0;
    __syncthreads();
    {
        constexpr int R = kJumpR;
        const int nwarps = blockDim.x >> 5;
        const int L = (DEG + nwarps - 1) / nwarps;
        const int i0 = warp * L, i1 = min(DEG, i0 + L);
        const int j0 = lane * R;
        uint64_t acc[R], win[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            acc[r] = 0;
            win[r] = sb[i0 + j0 + r];
        }
        for (int i = i0; i < i1; i += R) {
#pragma unroll
            for (int s = 0; s < R; ++s) {
                const int ii = i + s;
                if (ii < i1 && ((sg[ii >> 6] >> (ii & 63)) & 1ULL)) {
#pragma unroll
                    for (int r = 0; r < R; ++r) acc[r] ^= win[(s + r) % R];
                }
                win[s] = sb[i + j0 + R + s];
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r)
            if (j0 + r < N) atomicXor(reinterpret_cast<unsigned long long*>(&s0[j0 + r]), acc[r]);
    }
    __syncthreads();
    // Generation, warp-specialised.  Warps 0-9 ("twisters") run only the block
    // recurrence — the serial critical path — into a kRing-deep ring of
    // 312-word blocks; warps 10-19 ("emitters") temper, convert and store each
    // completed block.  Named barriers: FULL[slot] (twisters arrive, emitters
    // wait), EMPTY[slot] (emitters arrive, twisters wait), TW (twisters only).
    // Block 0 (the jump window) is already in ring slot 0.
    const int64_t n = min(J, count - q0);
    const int64_t nblk = (n + N - 1) / N;
    uint64_t* ring = s0;  // [kRing][N] (s0 and the following smem)
    constexpr int kTw = 10 * 32;
    const bool twister = t < kTw;
    if (twister) {
        bar_arrive(kBarFull + 0, kChunkThreads);
        for (int64_t b = 1; b < nblk; ++b) {
            const int slot = static_cast<int>(b % kRing);
            if (b >= kRing) bar_sync(kBarEmpty + slot, kChunkThreads);  // slot's old block consumed
            const uint64_t* prev = ring + static_cast<int>((b - 1) % kRing) * N;
            uint64_t v = 0;
            if (t < N) v = next_word(prev, t);
            if (t < N) ring[slot * N + t] = v;
            bar_sync(kBarTw, kTw);  // whole block written before it is the next input
            bar_arrive(kBarFull + slot, kChunkThreads);
        }
    } else {
        const int u = t - kTw;
        for (int64_t b = 0; b < nblk; ++b) {
            const int slot = static_cast<int>(b % kRing);
            bar_sync(kBarFull + slot, kChunkThreads);
            const int64_t q = b * N + u;
            if (u < N && q < n) {
                const uint64_t out = temper(ring[slot * N + u]);
                if (raw_out) raw_out[q0 + q] = out;
                if (noise) {
                    const double uu = static_cast<double>(out >> 11) * 0x1.0p-53;
                    noise[q0 + q] = static_cast<float>(lo + span * uu);
                }
            }
            if (b + kRing < nblk) bar_arrive(kBarEmpty + slot, kChunkThreads);
        }
    }
}

struct Scratch {
    uint64_t* base = nullptr;
    Scratch() { MOE_CUDA_CHECK(cudaMalloc(&base, sizeof(uint64_t) * BASE)); }
};
static Scratch& scratch() {
    static Scratch* s = new Scratch();
    return *s;
}

void generate(uint64_t seed, int64_t count, double lo, double hi, float* noise, uint64_t* raw,
              cudaStream_t st) {
    if (count <= 0) return;
    const int P = static_cast<int>(std::min<int64_t>(kNumSMs, ceil_div(count, 4096)));
    const int64_t J = ceil_div(count, P);
    const Table& tab = table_for(J, P);
    Scratch& sc = scratch();
    base_kernel<<<1, kThreads, 0, st>>>(seed, sc.base);
    MOE_LAUNCH_CHECK();
    const size_t smem = sizeof(uint64_t) * (BASE + W + kRing * N);
    static bool attr = false;
    if (!attr) {
        MOE_CUDA_CHECK(cudaFuncSetAttribute(chunk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(smem)));
        attr = true;
    }
    chunk_kernel<<<P, kChunkThreads, smem, st>>>(sc.base, tab.dev, J, count, lo, hi - lo, noise, raw);
    MOE_LAUNCH_CHECK();
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
