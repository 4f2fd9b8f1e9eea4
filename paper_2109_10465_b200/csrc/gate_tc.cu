// gate_tc.cu — the three gate GEMMs on 5th-gen tensor cores (kind::tf32).
//
// The router's dense gate (routing.cpp:62-71 forward; ops.cpp:137-138 and
// 223-228 backward) is T x d x E with E small (64 in BASELINE C3): three
// HBM-streaming GEMMs whose FLOPs fit the tensor cores many times over.  On
// the bf16 path they run here instead of on the FMA pipes:
//
//   logits  L[t][e]   = sum_j (x[t][j] noise[t][j]) WgT[e][j]       (3xTF32)
//   dWg     dW[j][e]  = sum_t (x[t][j] noise[t][j]) dL[t][e]        (TF32, split-K)
//   dx      dx[t][j]  = noise[t][j] sum_e dL[t][e] Wg[j][e]          (TF32)
//                       + sum_k dX[row_k(t)][j] + (dy[t][j] if no route kept)
//
// One CTA per output tile (two per SM), 128 threads.  All four warps stage
// the next K step from global memory into registers while the tensor core
// works on the current one, transform it (x * noise, tf32 rounding, the
// hi/lo split of 3xTF32) and store it in the 128B-swizzled layout the MMA
// reads; thread 0 issues tcgen05.mma into a TMEM accumulator and commits to a
// per-buffer mbarrier, so a buffer is rewritten only after its MMAs retire.
// The epilogue reads TMEM with tcgen05.ld (thread = accumulator row).
//
// Precision: the logits decide routing, so they use the 3xTF32 split
// (a = a_hi + a_lo, products hi*hi + hi*lo + lo*hi: ~2^-21 relative per term,
// the accuracy of the fp32 FMA path).  dWg and dx feed bf16 tensors and fp32
// weight gradients and use single TF32 (2^-11 per operand).
#include "common.cuh"
#include "kernels.h"
#include "tc_ptx.cuh"

namespace moe {
namespace gtc {

using namespace tc;

constexpr int NT = 128;   // logits, dx: 4 warps (epilogue rows = TMEM lanes)
constexpr int NTS = 512;  // dWg: 16 warps stage and transform each K step
constexpr int BM = 128;  // accumulator rows (TMEM lanes)
constexpr int BK = 32;   // fp32 K elements per step = one 128 B swizzle row

__device__ __forceinline__ float tf32_rna(float v) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
    return __uint_as_float(r);
}
__device__ __forceinline__ void split_tf32(float v, float& hi, float& lo) {
    hi = tf32_rna(v);
    lo = tf32_rna(v - hi);
}
// byte offset of 16-byte chunk `c` (0..7) of row `r` in a 128B-swizzled tile
__device__ __forceinline__ uint32_t swz(int r, int c) { return r * 128 + ((c ^ (r & 7)) << 4); }

__device__ __forceinline__ void st4(uint8_t* base, uint32_t off, float a, float b, float c, float d) {
    *reinterpret_cast<float4*>(base + off) = make_float4(a, b, c, d);
}

template <class T>
__device__ __forceinline__ void ld4(const T* p, float (&v)[4]) {
    if constexpr (sizeof(T) == 2) {
        const uint2 u = __ldg(reinterpret_cast<const uint2*>(p));
        const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(&u.x);
        const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&u.y);
        v[0] = __low2float(a); v[1] = __high2float(a); v[2] = __low2float(b); v[3] = __high2float(b);
    } else {
        const float4 u = __ldg(reinterpret_cast<const float4*>(p));
        v[0] = u.x; v[1] = u.y; v[2] = u.z; v[3] = u.w;
    }
}

// Raw 4-element loads kept unconverted in registers until the data is used,
// so a prefetch does not stall on the conversion (bf16: 8 B, fp32: 16 B).
template <class T> struct Raw4;
template <> struct Raw4<__nv_bfloat16> {
    uint2 u;
    __device__ __forceinline__ void load(const __nv_bfloat16* p) { u = __ldg(reinterpret_cast<const uint2*>(p)); }
    __device__ __forceinline__ void zero() { u = make_uint2(0u, 0u); }
    __device__ __forceinline__ void get(float (&v)[4]) const {
        v[0] = __uint_as_float(u.x << 16); v[1] = __uint_as_float(u.x & 0xffff0000u);
        v[2] = __uint_as_float(u.y << 16); v[3] = __uint_as_float(u.y & 0xffff0000u);
    }
};
template <> struct Raw4<float> {
    float4 u;
    __device__ __forceinline__ void load(const float* p) { u = __ldg(reinterpret_cast<const float4*>(p)); }
    __device__ __forceinline__ void zero() { u = make_float4(0.f, 0.f, 0.f, 0.f); }
    __device__ __forceinline__ void get(float (&v)[4]) const { v[0] = u.x; v[1] = u.y; v[2] = u.z; v[3] = u.w; }
};

// Shared setup: barriers + TMEM allocation (warp 0), returns the TMEM base.
__device__ __forceinline__ uint32_t setup(uint64_t* bars, int nbars, uint32_t* tslot, uint32_t cols) {
    if (threadIdx.x == 0) {
        for (int i = 0; i < nbars; ++i) mbar_init(&bars[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tslot)),
                     "r"(cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    return *tslot;
}
__device__ __forceinline__ void teardown(uint32_t tmem, uint32_t cols) {
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(cols));
    }
}
// all producers' smem writes -> visible to the tensor core; thread 0 then
// issues the step's MMAs through `issue` and commits them to `bar`.
template <class F>
__device__ __forceinline__ void publish_and_issue(uint64_t* bar, F issue) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        tc_fence_after();
        issue();
        tc_commit(bar);
    }
}

// ---- cp.async staging: each K step's raw operand bytes are copied global ->
// shared by all threads with 16-byte cp.async (no registers held), kRaw
// steps ahead of the transform, so ~3 steps of loads are in flight per CTA.
constexpr int kRaw = 4;
__device__ __forceinline__ void cp16(void* dst, const void* src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
                 "r"(valid ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// ============================================================== logits
// CTA = 128 tokens x E experts, K range = one split of d.  A = x*noise
// (K-major, hi/lo), B = WgT = Wg^T [E][d] (K-major, hi/lo).  (kind::tf32
// operands must be K-major: an MN-major tf32 descriptor reads as zeros.)
// The tensor core's fp32 accumulation loses ~2^-24 of the running sum per
// MMA; spreading the K steps over kNAcc accumulators (summed in the
// epilogue) keeps the 3xTF32 logits at fp32-FMA-path accuracy for d = 2048.
constexpr int kNAcc = 4;
template <int E>
struct LogitsSmem {
    static constexpr uint32_t A = BM * 128;      // 16 KB per hi / lo
    static constexpr uint32_t B = E * 128;       // E rows x 128 B
    static constexpr uint32_t buf = 2 * A + 2 * B;
    static constexpr uint32_t bytes = 1024 + 2 * buf + 256;
};

constexpr int NTL = 256;  // logits: 8 warps stage / transform, 2 CTAs per SM
template <class TX, int E>
__global__ void __launch_bounds__(NTL, 2)
logits_kernel(const TX* __restrict__ x, const float* __restrict__ noise, const float* __restrict__ wgt,
              float* __restrict__ out, int64_t T, int d, int k_per_split) {
    using S = LogitsSmem<E>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in the shared window
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + 2 * S::buf);  // [2] per-buffer MMA done, [2] final
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 4);
    const int tid = threadIdx.x;
    const int64_t t0 = (int64_t)blockIdx.x * BM;
    const int kb = blockIdx.y * k_per_split;
    const int nsteps = k_per_split / BK;
    out += (int64_t)blockIdx.y * T * E;
    const uint32_t tmem = setup(bars, 3, tslot, kNAcc * E);
    pdl_wait();  // barriers and TMEM are set up; now the predecessor's data
    pdl_trigger();

    // producer mapping: A: chunk c = tid % 8 (4 k), rows tid/8 + 32 i (i < 4)
    //                   B: chunk c = tid % 8, rows e = tid/8 + 32 i (i < E/32)
    // The raw loads run two K steps ahead in two register slots, so ~2 steps
    // of x / noise are in flight per CTA while the tensor core works.
    const int ac = tid & 7, ar = tid >> 3;
    constexpr int NA = BM / 32, NB = E / 32;
    Raw4<TX> xa0[NA], xa1[NA];
    Raw4<float> na0[NA], na1[NA], wb0[NB], wb1[NB];
    auto load = [&](int step, Raw4<TX> (&xa)[NA], Raw4<float> (&na)[NA], Raw4<float> (&wb)[NB]) {
        if (step >= nsteps) return;
        const int k0 = kb + step * BK;
#pragma unroll
        for (int i = 0; i < NA; ++i) {
            const int64_t t = t0 + ar + 32 * i;
            if (t < T) {
                xa[i].load(x + t * d + k0 + 4 * ac);
                if (noise) na[i].load(noise + t * d + k0 + 4 * ac);
            } else {
                xa[i].zero();
            }
        }
#pragma unroll
        for (int i = 0; i < NB; ++i) wb[i].load(wgt + (int64_t)(ar + 32 * i) * d + k0 + 4 * ac);
    };
    auto store = [&](uint8_t* buf, const Raw4<TX> (&xa)[NA], const Raw4<float> (&na)[NA],
                     const Raw4<float> (&wb)[NB]) {
        uint8_t* ahi = buf;
        uint8_t* alo = buf + S::A;
        uint8_t* bhi = buf + 2 * S::A;
        uint8_t* blo = bhi + S::B;
#pragma unroll
        for (int i = 0; i < NA; ++i) {
            float xv[4], nv[4] = {1.f, 1.f, 1.f, 1.f}, h[4], l[4];
            xa[i].get(xv);
            if (noise) na[i].get(nv);
#pragma unroll
            for (int q = 0; q < 4; ++q) split_tf32(noise ? xv[q] * nv[q] : xv[q], h[q], l[q]);
            const uint32_t off = swz(ar + 32 * i, ac);
            st4(ahi, off, h[0], h[1], h[2], h[3]);
            st4(alo, off, l[0], l[1], l[2], l[3]);
        }
#pragma unroll
        for (int i = 0; i < NB; ++i) {
            float wv[4], h[4], l[4];
            wb[i].get(wv);
#pragma unroll
            for (int j = 0; j < 4; ++j) split_tf32(wv[j], h[j], l[j]);
            const uint32_t off = swz(ar + 32 * i, ac);
            st4(bhi, off, h[0], h[1], h[2], h[3]);
            st4(blo, off, l[0], l[1], l[2], l[3]);
        }
    };
    constexpr uint32_t idesc = make_idesc_tf32(BM, E, 0, 0);
    auto step = [&](int s, Raw4<TX> (&xa)[NA], Raw4<float> (&na)[NA], Raw4<float> (&wb)[NB]) {
        const int b = s & 1;
        uint8_t* buf = sm + b * S::buf;
        if (s >= 2) mbar_wait(&bars[b], ((s - 2) >> 1) & 1);
        store(buf, xa, na, wb);
        load(s + 2, xa, na, wb);  // two steps ahead, in flight during the MMAs
        publish_and_issue(&bars[b], [&] {
            const uint32_t a = smem_u32(buf), bb = a + 2 * S::A;
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk) {
                const uint64_t ah = sdesc(a + kk * 32, 16, 1024);
                const uint64_t al = sdesc(a + S::A + kk * 32, 16, 1024);
                const uint64_t bh = sdesc(bb + kk * 32, 16, 1024);
                const uint64_t bl = sdesc(bb + S::B + kk * 32, 16, 1024);
                const uint32_t acc = tmem + kk * E;  // accumulator kk of kNAcc
                tc_mma_tf32(acc, ah, bh, idesc, s ? 1u : 0u);
                tc_mma_tf32(acc, ah, bl, idesc, 1u);
                tc_mma_tf32(acc, al, bh, idesc, 1u);
            }
        });
    };
    load(0, xa0, na0, wb0);
    load(1, xa1, na1, wb1);
    for (int s = 0; s < nsteps; s += 2) {
        step(s, xa0, na0, wb0);
        if (s + 1 < nsteps) step(s + 1, xa1, na1, wb1);
    }
    if (tid == 0) tc_commit(&bars[2]);
    mbar_wait(&bars[2], 0);
    tc_fence_after();
    // epilogue: warp w reads TMEM lanes 32 (w % 4) .. +31, columns half w / 4
    const int warp = tid >> 5, lane = tid & 31;
    const int64_t t = t0 + (warp & 3) * 32 + lane;
    const int c = (warp >> 2) * 32;
    static_assert(E == 64, "logits epilogue: two 32-column halves");
    float sum[32];
#pragma unroll
    for (int q = 0; q < kNAcc; ++q) {  // the accumulators, summed in fixed order
        uint32_t v[32];
        tmem_ld32(tmem + ((uint32_t)((warp & 3) * 32) << 16) + q * E + c, v);
#pragma unroll
        for (int j = 0; j < 32; ++j) sum[j] = q ? sum[j] + __uint_as_float(v[j]) : __uint_as_float(v[j]);
    }
    if (t < T) {
        float* o = out + t * E + c;
#pragma unroll
        for (int j = 0; j < 32; j += 4)
            *reinterpret_cast<float4*>(o + j) = make_float4(sum[j], sum[j + 1], sum[j + 2], sum[j + 3]);
    }
    teardown(tmem, kNAcc * E);
}

// ============================================================== dWg
// CTA = 128 j x E, K = the split's tokens.  A(j, t) = x[t][j] noise[t][j],
// B(e, t) = dL[t][e], both K-major (t contiguous): each step's raw tiles are
// copied row-major (coalesced along j / e) and read transposed by the
// transform into the swizzled operand layout.
template <int E>
struct DwSmem {
    static constexpr uint32_t RX = BK * BM * 2;   // raw x  [32 t][128 j] bf16  8 KB
    static constexpr uint32_t RN = BK * BM * 4;   // raw n  [32][128] fp32     16 KB
    static constexpr uint32_t RL = BK * E * 4;    // raw dL [32][E]  fp32       8 KB
    static constexpr uint32_t raw = RX + RN + RL;
    static constexpr uint32_t A = BM * 128;       // 128 rows x 128 B
    static constexpr uint32_t B = E * 128;
    static constexpr uint32_t buf = A + B;
    static constexpr uint32_t bytes = 1024 + 2 * buf + kRaw * raw + 256;
};

template <class TX, int E>
__global__ void __launch_bounds__(NTS, 1)
dw_kernel(const TX* __restrict__ x, const float* __restrict__ noise, const float* __restrict__ dL,
          float* __restrict__ part, int64_t T, int d, int64_t t_per_split) {
    static_assert(sizeof(TX) == 2, "gate_tc dw: bf16 activations");
    using S = DwSmem<E>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in the shared window
    uint8_t* raw = sm + 2 * S::buf;
    uint64_t* bars = reinterpret_cast<uint64_t*>(raw + kRaw * S::raw);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 4);
    const int tid = threadIdx.x;
    const int j0 = blockIdx.x * BM;
    const int64_t tb = (int64_t)blockIdx.y * t_per_split;
    const int64_t te = min(T, tb + t_per_split);
    const int nsteps = te > tb ? (int)((te - tb + BK - 1) / BK) : 0;
    part += (int64_t)blockIdx.y * d * E;
    const uint32_t tmem = setup(bars, 3, tslot, E < 32 ? 32 : E);
    pdl_wait();  // barriers and TMEM are set up; now the predecessor's data
    pdl_trigger();

    auto issue = [&](int step) {
        if (step < nsteps) {
            uint8_t* r = raw + (step % kRaw) * S::raw;
            const int64_t k0 = tb + (int64_t)step * BK;
#pragma unroll
            for (int i = 0; i < BK * 16 / NTS; ++i) {  // x: 32 rows x 16 chunks (8 bf16)
                const int q = tid + NTS * i, row = q >> 4, c = q & 15;
                const int64_t t = k0 + row;
                cp16(r + row * 256 + c * 16, x + (t < te ? t : 0) * d + j0 + 8 * c, t < te);
            }
            if (noise) {
#pragma unroll
                for (int i = 0; i < BK * 32 / NTS; ++i) {  // noise: 32 rows x 32 chunks
                    const int q = tid + NTS * i, row = q >> 5, c = q & 31;
                    const int64_t t = k0 + row;
                    cp16(r + S::RX + row * 512 + c * 16, noise + (t < te ? t : 0) * d + j0 + 4 * c, t < te);
                }
            }
#pragma unroll
            for (int i = 0; i < E * 8 / NTS; ++i) {  // dL: 32 rows x E/4 chunks
                const int q = tid + NTS * i, row = q / (E / 4), c = q % (E / 4);
                const int64_t t = k0 + row;
                cp16(r + S::RX + S::RN + row * (E * 4) + c * 16, dL + (t < te ? t : 0) * E + 4 * c, t < te);
            }
        }
        cp_commit();
    };
    auto store = [&](const uint8_t* r, uint8_t* buf) {  // raw (row-major) -> transposed, swizzled, tf32
        const __nv_bfloat16* rx = reinterpret_cast<const __nv_bfloat16*>(r);
        const float* rn = reinterpret_cast<const float*>(r + S::RX);
        const float* rl = reinterpret_cast<const float*>(r + S::RX + S::RN);
        const int j = tid % BM;  // A row; this thread's chunks c = tid/BM + (NTS/BM) i
#pragma unroll
        for (int c = tid / BM; c < 8; c += NTS / BM) {
            float v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int tt = 4 * c + u;
                const float xv = __bfloat162float(rx[tt * BM + j]);
                v[u] = tf32_rna(noise ? xv * rn[tt * BM + j] : xv);
            }
            st4(buf, swz(j, c), v[0], v[1], v[2], v[3]);
        }
        constexpr int RPT = E * 8 / NTS;  // B chunks per thread
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            const int q = tid + NTS * i;
            const int e = q % E, c = q / E;
            st4(buf + S::A, swz(e, c), tf32_rna(rl[(4 * c) * E + e]), tf32_rna(rl[(4 * c + 1) * E + e]),
                tf32_rna(rl[(4 * c + 2) * E + e]), tf32_rna(rl[(4 * c + 3) * E + e]));
        }
    };
    constexpr uint32_t idesc = make_idesc_tf32(BM, E, 0, 0);
#pragma unroll
    for (int s = 0; s < kRaw - 1; ++s) issue(s);
    for (int s = 0; s < nsteps; ++s) {
        const int b = s & 1;
        uint8_t* buf = sm + b * S::buf;
        issue(s + kRaw - 1);
        cp_wait<kRaw - 1>();
        __syncthreads();
        if (s >= 2) mbar_wait(&bars[b], ((s - 2) >> 1) & 1);
        store(raw + (s % kRaw) * S::raw, buf);
        publish_and_issue(&bars[b], [&] {
            const uint32_t a = smem_u32(buf), bb = a + S::A;
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk)
                tc_mma_tf32(tmem, sdesc(a + kk * 32, 16, 1024), sdesc(bb + kk * 32, 16, 1024), idesc,
                            (s | kk) ? 1u : 0u);
        });
    }
    cp_wait<0>();
    if (tid == 0) tc_commit(&bars[2]);
    mbar_wait(&bars[2], 0);
    tc_fence_after();
    const int warp = tid >> 5, lane = tid & 31;
    const int quarter = warp & 3;
    const int j = j0 + quarter * 32 + lane;
    for (int c = 32 * (warp >> 2); c < E; c += 32 * (NTS / 128)) {
        uint32_t v[32];
        tmem_ld32(tmem + ((uint32_t)(quarter * 32) << 16) + c, v);
        float* o = part + (int64_t)j * E + c;
#pragma unroll
        for (int q = 0; q < 32; q += 4) {
            const float4 w = nsteps > 0 ? make_float4(__uint_as_float(v[q]), __uint_as_float(v[q + 1]),
                                                      __uint_as_float(v[q + 2]), __uint_as_float(v[q + 3]))
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
            *reinterpret_cast<float4*>(o + q) = w;
        }
    }
    teardown(tmem, E < 32 ? 32 : E);
}

// ============================================================== dx
// CTA = 128 tokens x 256 columns of d, K = E (all steps resident).
// A(t, e) = dL[t][e] (K-major), B(j, e) = Wg[j][e] (K-major).  The epilogue
// assembles dx = acc * noise + gathered dX rows (+ dy / dres), ops.cpp:137-138.
constexpr int XN = 256;
template <int E>
struct DxSmem {
    static constexpr int steps = E / BK;
    static constexpr uint32_t A = BM * 128;
    static constexpr uint32_t B = XN * 128;
    static constexpr uint32_t bytes = 1024 + steps * (A + B) + 256;
};

template <class TIO, int E>
__global__ void __launch_bounds__(NT, 2)
dx_kernel(int64_t T, int d, int K, int cap_pad, const float* __restrict__ dL, const float* __restrict__ wg,
          const float* __restrict__ noise, const TIO* __restrict__ dX, const int32_t* __restrict__ choice,
          const int32_t* __restrict__ pos, const TIO* __restrict__ dy, bool residual_is_x,
          TIO* __restrict__ dx, TIO* __restrict__ dres) {
    static_assert(sizeof(TIO) == 2, "gate_tc dx: bf16 tensors");
    using S = DxSmem<E>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in the shared window
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + S::steps * (S::A + S::B));
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2);
    const int tid = threadIdx.x;
    const int64_t t0 = (int64_t)blockIdx.x * BM;
    const int j0 = blockIdx.y * XN;
    const uint32_t tmem = setup(bars, 1, tslot, XN);
    pdl_wait();  // barriers and TMEM are set up; now the predecessor's data
    pdl_trigger();
    // stage all K steps: A 8 chunks / thread / step, B 16 chunks / thread / step
#pragma unroll
    for (int s = 0; s < S::steps; ++s) {
        uint8_t* a = sm + s * (S::A + S::B);
        uint8_t* b = a + S::A;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int q = tid + NT * i;
            const int r = q >> 3, c = q & 7;
            const int64_t t = t0 + r;
            float v[4] = {0.f, 0.f, 0.f, 0.f};
            if (t < T) ld4<float>(dL + t * E + s * BK + 4 * c, v);
            st4(a, swz(r, c), tf32_rna(v[0]), tf32_rna(v[1]), tf32_rna(v[2]), tf32_rna(v[3]));
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int q = tid + NT * i;
            const int r = q >> 3, c = q & 7;
            float v[4];
            ld4<float>(wg + (int64_t)(j0 + r) * E + s * BK + 4 * c, v);
            st4(b, swz(r, c), tf32_rna(v[0]), tf32_rna(v[1]), tf32_rna(v[2]), tf32_rna(v[3]));
        }
    }
    // this thread's output row and its dispatch rows (tokens t0 + tid)
    const int warp = tid >> 5, lane = tid & 31;
    const int64_t t = t0 + warp * 32 + lane;
    int64_t rows[2] = {-1, -1};
    bool any = false;
    if (t < T) {
        #pragma unroll
        for (int k = 0; k < 2; ++k) {  // K <= 2
            if (k >= K) break;
            const int32_t p = pos[t * K + k];
            if (p >= 0) {
                rows[k] = (int64_t)choice[t * K + k] * cap_pad + p;
                any = true;
            }
        }
    }
    constexpr uint32_t idesc = make_idesc_tf32(BM, XN, 0, 0);
    publish_and_issue(&bars[0], [&] {
#pragma unroll
        for (int s = 0; s < S::steps; ++s) {
            const uint32_t a = smem_u32(sm + s * (S::A + S::B)), b = a + S::A;
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk)
                tc_mma_tf32(tmem, sdesc(a + kk * 32, 16, 1024), sdesc(b + kk * 32, 16, 1024), idesc,
                            (s | kk) ? 1u : 0u);
        }
    });
    mbar_wait(&bars[0], 0);
    tc_fence_after();
    // Epilogue.  tcgen05.ld hands thread i accumulator row i; the global
    // traffic (noise, gathered dX rows, dy, dx) is row-major.  Each warp owns
    // its 32 rows and runs its own pipeline over the 32-column chunks: the
    // chunk's row segments are copied global -> shared with cp.async (16 B,
    // 8 adjacent lanes per 128 B row segment, zero-filled for dropped routes)
    // two chunks ahead, the accumulator chunk is bounced through shared
    // memory, and the combine walks 4 rows x 8 column groups per instruction.
    // The operand tiles are free now and hold the stages.
    constexpr int kWS = 8192;  // bytes per warp-stage: noise [32][32] f32, g0/g1 [32][32] bf16
    static_assert(2 * 4 * kWS + 4 * 32 * 33 * 4 + 128 * 2 * 4 <= S::steps * (S::A + S::B), "epilogue fits the operand tiles");
    float* stile = reinterpret_cast<float*>(sm + 2 * 4 * kWS) + warp * (32 * 33);  // [32 rows][33]
    int32_t* srows = reinterpret_cast<int32_t*>(sm + 2 * 4 * kWS + 4 * 32 * 33 * 4);  // [128][2]
    srows[tid * 2 + 0] = t < T ? (int32_t)rows[0] : -1;
    srows[tid * 2 + 1] = t >= T ? -1 : (any ? (int32_t)rows[1] : -2);  // -2: no route kept (residual)
    __syncwarp();
    const int32_t* wrows = srows + warp * 64;
    const int64_t tw = t0 + warp * 32;  // this warp's first token
    auto issue = [&](int c, int stage) {
        uint8_t* base = sm + (stage * 4 + warp) * kWS;
        const int64_t jc = j0 + c;
#pragma unroll
        for (int i = 0; i < 8; ++i) {  // noise: 32 rows x 8 x 16 B
            const int q = lane + 32 * i, r = q >> 3, c16 = q & 7;
            const bool ok = noise != nullptr && tw + r < T;
            cp16(base + r * 128 + c16 * 16, ok ? noise + (tw + r) * d + jc + 4 * c16 : noise, ok);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {  // dX rows of routes 0 / 1 (or dy): 32 rows x 4 x 16 B each
            const int q = lane + 32 * i, r = q >> 2, c16 = q & 3;
            const int32_t r0 = wrows[r * 2 + 0], r1 = wrows[r * 2 + 1];
            cp16(base + 4096 + r * 64 + c16 * 16, r0 >= 0 ? dX + (int64_t)r0 * d + jc + 8 * c16 : dX, r0 >= 0);
            const TIO* s1 = r1 >= 0 ? dX + (int64_t)r1 * d + jc + 8 * c16
                                    : (r1 == -2 ? dy + (tw + r) * d + jc + 8 * c16 : dX);
            cp16(base + 6144 + r * 64 + c16 * 16, s1, r1 != -1);
        }
        cp_commit();
    };
    const int sub = lane >> 3, cg = lane & 7;  // row within a group of 4, 4-column group
    constexpr int NCH = XN / 32;
    issue(0, 0);
    issue(32, 1);
#pragma unroll 1
    for (int ci = 0; ci < NCH; ++ci) {
        const int c = ci * 32, stage = ci & 1;
        uint32_t u[32];
        tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + c, u);
#pragma unroll
        for (int q = 0; q < 32; ++q) stile[lane * 33 + q] = __uint_as_float(u[q]);
        cp_wait<1>();  // this lane's copies of chunk ci have landed
        __syncwarp();  // ... and everyone's; stile visible too
        const uint8_t* base = sm + (stage * 4 + warp) * kWS;
        const int64_t j = j0 + c + 4 * cg;
#pragma unroll
        for (int it = 0; it < 8; ++it) {
            const int rl = it * 4 + sub;
            const int64_t tt = tw + rl;
            if (tt >= T) continue;
            const int32_t r1 = wrows[rl * 2 + 1];
            const float4 n4 = noise ? *reinterpret_cast<const float4*>(base + rl * 128 + cg * 16)
                                    : make_float4(1.f, 1.f, 1.f, 1.f);
            const uint2 g0 = *reinterpret_cast<const uint2*>(base + 4096 + rl * 64 + cg * 8);
            const uint2 g1 = *reinterpret_cast<const uint2*>(base + 6144 + rl * 64 + cg * 8);
            float v[4];
#pragma unroll
            for (int w = 0; w < 4; ++w) v[w] = stile[rl * 33 + 4 * cg + w];
            v[0] *= n4.x; v[1] *= n4.y; v[2] *= n4.z; v[3] *= n4.w;
            auto add4 = [&](const uint2& g) {
                v[0] += __uint_as_float(g.x << 16); v[1] += __uint_as_float(g.x & 0xffff0000u);
                v[2] += __uint_as_float(g.y << 16); v[3] += __uint_as_float(g.y & 0xffff0000u);
            };
            add4(g0);  // zero unless route 0 kept
            if (r1 == -2) {  // no route kept: the residual carries dy (in g1)
                if (residual_is_x) add4(g1);
                else if (dres) *reinterpret_cast<uint2*>(dres + tt * d + j) = g1;
            } else {
                add4(g1);  // zero unless route 1 kept
                if (!residual_is_x && dres) *reinterpret_cast<uint2*>(dres + tt * d + j) = make_uint2(0u, 0u);
            }
            const __nv_bfloat162 lo2 = __floats2bfloat162_rn(v[0], v[1]);
            const __nv_bfloat162 hi2 = __floats2bfloat162_rn(v[2], v[3]);
            *reinterpret_cast<uint2*>(dx + tt * d + j) =
                make_uint2(*reinterpret_cast<const uint32_t*>(&lo2), *reinterpret_cast<const uint32_t*>(&hi2));
        }
        __syncwarp();  // stage and stile consumed
        if (ci + 2 < NCH) issue(c + 64, stage);
        else cp_commit();  // keep one group per chunk so wait_group<1> stays exact
    }
    teardown(tmem, XN);
}

template <class K>
void set_smem(K kernel, uint32_t bytes) {
    MOE_CUDA_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(bytes)));
}

}  // namespace gtc

bool gate_tc_ok(int d, int E) { return E == 64 && d % gtc::XN == 0 && d >= gtc::XN; }

int gate_tc_logit_splits(int64_t T, int d) {
    // two CTAs per SM resident: aim for ~2 x 148 CTAs, K per split a multiple of 32
    const int64_t tiles = ceil_div(T, (int64_t)gtc::BM);
    int s = 1;
    while (s < kMaxGateSplits && tiles * (2 * s) <= 2 * kNumSMs && (d / (2 * s)) % gtc::BK == 0) s *= 2;
    return s;
}

template <class TX>
void launch_gate_tc_logits(const TX* x, const float* noise, const float* wgt, float* logits, int64_t T,
                           int d, int E, int splits, cudaStream_t st) {
    constexpr int kE = 64;
    if (E != kE) throw Status(6, "gate_tc: E must be 64");
    auto k = gtc::logits_kernel<TX, kE>;
    static bool attr = false;
    if (!attr) { gtc::set_smem(k, gtc::LogitsSmem<kE>::bytes); attr = true; }
    dim3 grid((unsigned)ceil_div(T, (int64_t)gtc::BM), (unsigned)splits);
    launch_pdl(k, dim3(grid), dim3(gtc::NTL), gtc::LogitsSmem<kE>::bytes, st, x, noise, wgt, logits, T, d, d / splits);
}

template <class TX>
void launch_gate_tc_dw(const TX* x, const float* noise, const float* dL, float* part, int64_t T, int d,
                       int E, int splits, cudaStream_t st) {
    constexpr int kE = 64;
    if (E != kE) throw Status(6, "gate_tc: E must be 64");
    auto k = gtc::dw_kernel<TX, kE>;
    static bool attr = false;
    if (!attr) { gtc::set_smem(k, gtc::DwSmem<kE>::bytes); attr = true; }
    const int64_t tps = round_up(ceil_div(T, (int64_t)splits), (int64_t)gtc::BK);
    dim3 grid((unsigned)(d / gtc::BM), (unsigned)splits);
    launch_pdl(k, dim3(grid), dim3(gtc::NTS), gtc::DwSmem<kE>::bytes, st, x, noise, dL, part, T, d, tps);
}

template <class TIO>
void launch_gate_tc_dx(int64_t T, int d, int E, int K, int cap_pad, const float* dL, const float* wg,
                       const float* noise, const TIO* dX, const int32_t* choice, const int32_t* pos,
                       const TIO* dy, bool residual_is_x, TIO* dx, TIO* dres, cudaStream_t st) {
    constexpr int kE = 64;
    if (E != kE) throw Status(6, "gate_tc: E must be 64");
    auto k = gtc::dx_kernel<TIO, kE>;
    static bool attr = false;
    if (!attr) { gtc::set_smem(k, gtc::DxSmem<kE>::bytes); attr = true; }
    dim3 grid((unsigned)ceil_div(T, (int64_t)gtc::BM), (unsigned)(d / gtc::XN));
    launch_pdl(k, dim3(grid), dim3(gtc::NT), gtc::DxSmem<kE>::bytes, st, T, d, K, cap_pad, dL, wg, noise, dX, choice, pos, dy,
                                                     residual_is_x, dx, dres);
}

#define INST(T)                                                                                         \
    template void launch_gate_tc_logits<T>(const T*, const float*, const float*, float*, int64_t, int, \
                                           int, int, cudaStream_t);                                    \
    template void launch_gate_tc_dw<T>(const T*, const float*, const float*, float*, int64_t, int, int, \
                                       int, cudaStream_t);                                             \
    template void launch_gate_tc_dx<T>(int64_t, int, int, int, int, const float*, const float*,        \
                                       const float*, const T*, const int32_t*, const int32_t*, const T*, \
                                       bool, T*, T*, cudaStream_t);
INST(__nv_bfloat16)
#undef INST

}  // namespace moe
