// gate_bwd.cu — the gate weight gradient of the bf16 path as a TMA-fed,
// warp-specialised tcgen05 kernel (ops.cpp:223-228 jitter-mul backward and
// the gate GEMM's weight closure, ops.cpp:135-144 matmul_at_acc):
//
//   dWg[j][e] = sum_t g[t][j] dL[t][e],   g = x[t][j] * noise[t][j]  (fp32)
//
// The reduction runs over tokens, which are the ROWS of every operand in HBM,
// so the operands are MN-major.  tcgen05 reads MN-major operands only for
// 16-bit (and 8-bit) types — an MN-major tf32 descriptor reads zeros
// (scripts/micro/tf32_mma.cu) — so the products use the 3xBF16 split:
// g = g_hi + g_lo and dL = l_hi + l_lo (bf16 each, exact residuals), summed
// as hi*hi + hi*lo + lo*hi by kind::f16 MMAs with fp32 accumulation.  That is
// ~2^-16 relative per product, finer than the TF32 operands (2^-11) of the
// transposing kernel it replaces (gate_tc.cu dw_kernel), and needs no
// transpose: every tile is read and written along its rows.
//
//   warp 0      TMA producer: per 32-token step x [32 x 128] bf16, noise
//               [32 x 128] fp32 and dL [32 x 64] fp32 of this CTA's column
//               block (128-byte rows, 128B swizzle) into a kStages-deep ring
//   warps 2..5  split, in place: the hi / lo bf16 tiles of g overwrite the
//               noise tile, those of dL the dL tile (each thread loads its
//               inputs, the four warps sync on a named barrier, then store);
//               after the last step they drain the accumulator from TMEM
//   warp 1      MMA: M = 128 columns of d, N = 64 experts, K = 16 tokens,
//               3 products per K step, one fp32 accumulator in TMEM
//
// A CTA owns 128 columns of d and a token split (a multiple of 32 tokens, so
// splits never overlap); its [128 x 64] partial goes to part[split] and the
// splits are summed in fixed order by launch_splitk_reduce.  The kernel
// streams x, noise and dL once (T·d·(2+4) + T·E·4 bytes).
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "gemm_tc.h"
#include "kernels.h"
#include "tc_ptx.cuh"

namespace moe {
namespace gbw {

using namespace tc;

constexpr int E = 64;
constexpr int BJ = 128;      // columns of d per CTA (MMA M)
constexpr int BT = 32;       // tokens per step
constexpr int kStages = 6;
constexpr int kTw = 8;        // split warps (two per SM sub-partition)
constexpr int kThreads = 64 + 32 * kTw;
constexpr uint32_t kBox = BT * 128;               // one [32 rows x 128 B] box
constexpr uint32_t kN = 4 * kBox;                 // noise / g: 4 boxes of 32 columns
constexpr uint32_t kX = 2 * kBox;                 // x: 2 boxes of 64 bf16 columns
constexpr uint32_t kL = 2 * kBox;                 // dL: 2 boxes of 32 experts
constexpr uint32_t kStage = kN + kX + kL;         // 32 KB
constexpr uint32_t kSmem = 1024 + kStages * kStage + 256;

struct __align__(64) Params {
    CUtensorMap tmX, tmN, tmL;
    float* part;
    int64_t T;
    int64_t tps;  // tokens per split (multiple of BT)
    int d;
    int has_noise;
};

__device__ __forceinline__ float4 lds128f(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t swz(int r, int c) { return r * 128 + ((c ^ (r & 7)) << 4); }

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
#ifdef MOE_GBW_INT_PACK
    // round-to-nearest-even on the integer pipes (finite values and infinities)
    uint32_t ua = __float_as_uint(a), ub = __float_as_uint(b);
    ua += 0x7FFFu + ((ua >> 16) & 1u);
    ub += 0x7FFFu + ((ub >> 16) & 1u);
    return __byte_perm(ua, ub, 0x7632);
#else
    const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
#endif
}
// hi / lo bf16 split of 8 fp32 values: hi = bf16(v), lo = bf16(v - hi)
__device__ __forceinline__ void split8(const float (&v)[8], uint4& hi, uint4& lo) {
    uint32_t h[4], l[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        h[i] = pack_bf16(v[2 * i], v[2 * i + 1]);
        const float h0 = __uint_as_float(h[i] << 16), h1 = __uint_as_float(h[i] & 0xffff0000u);
        l[i] = pack_bf16(v[2 * i] - h0, v[2 * i + 1] - h1);
    }
    hi = make_uint4(h[0], h[1], h[2], h[3]);
    lo = make_uint4(l[0], l[1], l[2], l[3]);
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts128u(uint32_t a, const uint4& v) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ void named_sync_split() { asm volatile("bar.sync 1, %0;" ::"n"(32 * kTw) : "memory"); }

// kind::f16 instruction descriptor: bf16 A / B (both MN-major), fp32 D
__host__ __device__ constexpr uint32_t idesc_bf16_mn(int M, int N) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) | (static_cast<uint32_t>(N >> 3) << 17) |
           (static_cast<uint32_t>(M >> 4) << 24);
}

__global__ void __launch_bounds__(kThreads, 1) dw_kernel(const __grid_constant__ Params p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + kStages * kStage);
    uint64_t* ready = full + kStages;
    uint64_t* empty = ready + kStages;
    uint64_t* done = empty + kStages;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int j0 = blockIdx.x * BJ;
    const int64_t tb = static_cast<int64_t>(blockIdx.y) * p.tps;
    const int64_t te = min(p.T, tb + p.tps);
    const int nsteps = te > tb ? static_cast<int>((te - tb + BT - 1) / BT) : 0;

    if (threadIdx.x == 0) {
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&ready[i], 32 * kTw);
            mbar_init(&empty[i], 1);
        }
        mbar_init(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        prefetch_tmap(&p.tmX);
        prefetch_tmap(&p.tmN);
        prefetch_tmap(&p.tmL);
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                     "r"(E));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    pdl_wait();  // dL and the activations of the predecessors
    pdl_trigger();

    if (warp == 0) {
        if (lane == 0) {
            const uint32_t bytes = p.has_noise ? kStage : kStage - kN;
            for (int s = 0; s < nsteps; ++s) {
                const int st = s % kStages;
                if (s >= kStages) mbar_wait(&empty[st], ((s / kStages) - 1) & 1);
                uint8_t* base = sm + st * kStage;
                const int32_t row = static_cast<int32_t>(tb + static_cast<int64_t>(s) * BT);
                mbar_expect_tx(&full[st], bytes);
                if (p.has_noise) {
#pragma unroll
                    for (int b = 0; b < 4; ++b) tma_load_2d(&p.tmN, &full[st], base + b * kBox, j0 + 32 * b, row);
                }
#pragma unroll
                for (int b = 0; b < 2; ++b) tma_load_2d(&p.tmX, &full[st], base + kN + b * kBox, j0 + 64 * b, row);
#pragma unroll
                for (int b = 0; b < 2; ++b) tma_load_2d(&p.tmL, &full[st], base + kN + kX + b * kBox, 32 * b, row);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_bf16_mn(BJ, E);
            for (int s = 0; s < nsteps; ++s) {
                const int st = s % kStages;
                mbar_wait(&ready[st], (s / kStages) & 1);
                tc_fence_after();
                const uint32_t gh = smem_u32(sm + st * kStage), gl = gh + 2 * kBox;   // [32 t][128 j] bf16 each
                const uint32_t lh = gh + kN + kX, ll = lh + kBox;                      // [32 t][64 e] bf16 each
#pragma unroll
                for (int k = 0; k < BT / 16; ++k) {
                    const uint32_t o = k * 2048;  // 16 token rows
                    tc_mma(tmem, sdesc(gh + o, kBox, 1024), sdesc(lh + o, kBox, 1024), idesc, (s | k) ? 1u : 0u);
                    tc_mma(tmem, sdesc(gh + o, kBox, 1024), sdesc(ll + o, kBox, 1024), idesc, 1u);
                    tc_mma(tmem, sdesc(gl + o, kBox, 1024), sdesc(lh + o, kBox, 1024), idesc, 1u);
                }
                tc_commit(&empty[st]);
            }
            tc_commit(done);  // fires after every MMA above (also when nsteps == 0)
        }
    } else {
        // ---- split (32 * kTw threads), then the epilogue
        constexpr int NTT = 32 * kTw;
        constexpr int GU = 512 / NTT, LU = 256 / NTT;  // (row, chunk) pairs per thread
        const int tt = threadIdx.x - 64;
        for (int s = 0; s < nsteps; ++s) {
            const int st = s % kStages;
            mbar_wait(&full[st], (s / kStages) & 1);
            const uint32_t base = smem_u32(sm + st * kStage);
            // g: 32 rows x 16 chunks of 8 columns; thread -> (row, chunk) pairs
            uint4 ghi[GU], glo[GU];
            uint32_t gofs[GU];
#pragma unroll
            for (int u = 0; u < GU; ++u) {
                const int q = tt + NTT * u;
                const int r = q >> 4, c8 = q & 15;          // row, 8-column chunk (columns 8*c8 ..)
                const int xb = c8 >> 3, xc = c8 & 7;        // x box (64 columns) and its 16-byte chunk
                const uint4 xr = lds128(base + kN + xb * kBox + swz(r, xc));
                float v[8];
                v[0] = __uint_as_float(xr.x << 16); v[1] = __uint_as_float(xr.x & 0xffff0000u);
                v[2] = __uint_as_float(xr.y << 16); v[3] = __uint_as_float(xr.y & 0xffff0000u);
                v[4] = __uint_as_float(xr.z << 16); v[5] = __uint_as_float(xr.z & 0xffff0000u);
                v[6] = __uint_as_float(xr.w << 16); v[7] = __uint_as_float(xr.w & 0xffff0000u);
                if (p.has_noise) {
                    const int nb = c8 >> 2, nc = (c8 & 3) * 2;  // noise box (32 columns), first 16-byte chunk
                    const float4 n0 = lds128f(base + nb * kBox + swz(r, nc));
                    const float4 n1 = lds128f(base + nb * kBox + swz(r, nc + 1));
                    v[0] *= n0.x; v[1] *= n0.y; v[2] *= n0.z; v[3] *= n0.w;
                    v[4] *= n1.x; v[5] *= n1.y; v[6] *= n1.z; v[7] *= n1.w;
                }
                split8(v, ghi[u], glo[u]);
                gofs[u] = xb * kBox + swz(r, xc);  // same place in the [32 x 128] bf16 hi / lo tiles
            }
            // dL: 32 rows x 8 chunks of 8 experts
            uint4 lhi[LU], llo[LU];
            uint32_t lofs[LU];
#pragma unroll
            for (int u = 0; u < LU; ++u) {
                const int q = tt + NTT * u;
                const int r = q >> 3, c8 = q & 7;
                const int lb = c8 >> 2, lc = (c8 & 3) * 2;
                const float4 a = lds128f(base + kN + kX + lb * kBox + swz(r, lc));
                const float4 b = lds128f(base + kN + kX + lb * kBox + swz(r, lc + 1));
                const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
                split8(v, lhi[u], llo[u]);
                lofs[u] = swz(r, c8);
            }
            named_sync_split();  // every input of this step is in registers: overwrite in place
#pragma unroll
            for (int u = 0; u < GU; ++u) {
                sts128u(base + gofs[u], ghi[u]);
                sts128u(base + 2 * kBox + gofs[u], glo[u]);
            }
#pragma unroll
            for (int u = 0; u < LU; ++u) {
                sts128u(base + kN + kX + lofs[u], lhi[u]);
                sts128u(base + kN + kX + kBox + lofs[u], llo[u]);
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor core
            mbar_arrive(&ready[st]);
        }
        mbar_wait(done, 0);
        tc_fence_after();
        const int quarter = warp & 3;  // TMEM lanes this warp may read
        const int j = j0 + quarter * 32 + lane;
        float* o = p.part + (static_cast<int64_t>(blockIdx.y) * p.d + j) * E;
        constexpr int CW = E * 4 / kTw;  // accumulator columns per warp (kTw / 4 warps per quarter)
        const int cb = ((warp - 2) >> 2) * CW;
#pragma unroll
        for (int c = cb; c < cb + CW; c += 32) {
            uint32_t v[32];
            tmem_ld32(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + c, v);
#pragma unroll
            for (int q = 0; q < 32; q += 4) {
                const float4 w = nsteps > 0 ? make_float4(__uint_as_float(v[q]), __uint_as_float(v[q + 1]),
                                                          __uint_as_float(v[q + 2]), __uint_as_float(v[q + 3]))
                                            : make_float4(0.f, 0.f, 0.f, 0.f);
                *reinterpret_cast<float4*>(o + c + q) = w;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(E));
    }
}

}  // namespace gbw

// ============================================================== dx
// dx[t][j] = noise[t][j] * sum_e dLr[t][e] WgR[j][e]          (ops.cpp:137-138, 223-228)
//          + sum_{k kept} dX[row_k(t)][j]                      (routing.cpp:245-253)
//          + dy[t][j] if no route was kept and the residual is x (routing.cpp:337-342)
// dres[t] = dy[t] or 0 when the residual was passed explicitly.
//
// Persistent, warp-specialised.  Tile = 128 tokens x 64 columns of d.  dLr
// and WgR are the tf32-rounded (rna) copies written by the router backward
// and launch_gate_round_wg, so the MMA operands come straight from TMA; the
// noise tile rides in the same stage for the epilogue.
//   warp 0       TMA: A = dLr [128 t x 64 e], B = WgR [64 j x 64 e] (K-major,
//                128B swizzle), N = noise [128 t x 64 j] fp32
//   warp 1       MMA: kind::tf32, M = 128, N = 64, K = 64 into one of two
//                TMEM accumulators
//   warps 2..9   epilogue: warp w owns TMEM lane quarter w % 4 and column
//                half (w - 2) / 4 (32 columns): accumulator * noise (from
//                the stage, row per thread) + the dispatch-backward rows and
//                dy (row per thread, 64-byte vectors), bf16, staged per warp
//                [32 x 32] (64B swizzle) and written with TMA tensor stores.
namespace gdx {
using namespace tc;
using gbw::lds128f;
using gbw::pack_bf16;
using gbw::sts128u;
using gbw::swz;
constexpr int BMT = 128, BN = 64;
constexpr int kStages = 3;
constexpr int kEpiWarps = 8;
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr uint32_t kA = BMT * 256;           // [128 t][64 e] fp32 = 2 atoms of [128][32]; per token tile
constexpr uint32_t kB = BN * 256;            // [64 j][64 e] fp32
constexpr uint32_t kNt = BMT * BN * 4;       // [128 t][64 j] fp32 = 2 boxes of [128][32]
constexpr uint32_t kStage = kB + kNt;        // 48 KB
constexpr uint32_t kOut = 32 * 64;           // [32 rows][32 bf16] = 2 KB per warp
constexpr uint32_t kSmem = 1024 + kStages * kStage + 2 * kA + kEpiWarps * kOut + 256;

struct __align__(64) Params {
    CUtensorMap tmA, tmB, tmN, tmO;
    const __nv_bfloat16* dX;
    const int32_t* choice;
    const int32_t* pos;
    const __nv_bfloat16* dy;
    __nv_bfloat16* dres;
    int64_t T;
    int d, K, cap_pad, residual_is_x, has_noise;
};

__device__ __forceinline__ void add8(float (&v)[8], const uint4& u) {
    v[0] += __uint_as_float(u.x << 16); v[1] += __uint_as_float(u.x & 0xffff0000u);
    v[2] += __uint_as_float(u.y << 16); v[3] += __uint_as_float(u.y & 0xffff0000u);
    v[4] += __uint_as_float(u.z << 16); v[5] += __uint_as_float(u.z & 0xffff0000u);
    v[6] += __uint_as_float(u.w << 16); v[7] += __uint_as_float(u.w & 0xffff0000u);
}

__global__ void __launch_bounds__(kThreads, 1) dx_kernel(const __grid_constant__ Params p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* abuf = sm + kStages * kStage;   // [2][kA]: dLr of the current / next token tile
    uint8_t* obuf = abuf + 2 * kA;
    uint64_t* full = reinterpret_cast<uint64_t*>(obuf + kEpiWarps * kOut);
    uint64_t* empty = full + kStages;
    uint64_t* tfull = empty + kStages;
    uint64_t* tempty = tfull + 2;
    uint64_t* afull = tempty + 2;
    uint64_t* aempty = afull + 2;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(aempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int NJ = p.d / BN;
    const int ntiles = static_cast<int>((p.T + BMT - 1) / BMT) * NJ;
    // a contiguous run of tiles per CTA (token tile major, column block fastest),
    // so the dLr tile changes once per NJ tiles
    const int t_begin = static_cast<int>(static_cast<int64_t>(ntiles) * blockIdx.x / gridDim.x);
    const int t_end = static_cast<int>(static_cast<int64_t>(ntiles) * (blockIdx.x + 1) / gridDim.x);

    if (threadIdx.x == 0) {
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1 + kEpiWarps);  // MMA commit + every epilogue warp done with the noise
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], kEpiWarps);
            mbar_init(&afull[i], 1);
            mbar_init(&aempty[i], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        prefetch_tmap(&p.tmA);
        prefetch_tmap(&p.tmB);
        prefetch_tmap(&p.tmN);
        prefetch_tmap(&p.tmO);
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                     "r"(2 * BN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    pdl_wait();
    pdl_trigger();

    if (warp == 0) {
        if (lane == 0) {
            int i = 0, na = 0, prev = -1;
            for (int tile = t_begin; tile < t_end; ++tile, ++i) {
                const int tt = tile / NJ;
                const int32_t t0 = tt * BMT, j0 = (tile % NJ) * BN;
                if (tt != prev) {  // next token tile: its dLr into the other A buffer
                    const int ab = na & 1;
                    if (na >= 2) mbar_wait(&aempty[ab], ((na >> 1) - 1) & 1);
                    mbar_expect_tx(&afull[ab], kA);
#pragma unroll
                    for (int b = 0; b < 2; ++b) tma_load_2d(&p.tmA, &afull[ab], abuf + ab * kA + b * (kA / 2), 32 * b, t0);
                    ++na;
                    prev = tt;
                }
                const int st = i % kStages;
                if (i >= kStages) mbar_wait(&empty[st], ((i / kStages) - 1) & 1);
                uint8_t* base = sm + st * kStage;
                mbar_expect_tx(&full[st], p.has_noise ? kStage : kB);
#pragma unroll
                for (int b = 0; b < 2; ++b) tma_load_2d(&p.tmB, &full[st], base + b * (kB / 2), 32 * b, j0);
                if (p.has_noise) {
#pragma unroll
                    for (int b = 0; b < 2; ++b)
                        tma_load_2d(&p.tmN, &full[st], base + kB + b * (kNt / 2), j0 + 32 * b, t0);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = make_idesc_tf32(BMT, BN, 0, 0);
            int i = 0, na = 0, prev = -1;
            uint32_t a = 0;
            for (int tile = t_begin; tile < t_end; ++tile, ++i) {
                const int st = i % kStages, acc = i & 1;
                const int tt = tile / NJ;
                if (tt != prev) {
                    const int ab = na & 1;
                    mbar_wait(&afull[ab], (na >> 1) & 1);
                    a = smem_u32(abuf + ab * kA);
                    ++na;
                    prev = tt;
                }
                mbar_wait(&full[st], (i / kStages) & 1);
                if (i >= 2) mbar_wait(&tempty[acc], ((i >> 1) - 1) & 1);
                tc_fence_after();
                const uint32_t b = smem_u32(sm + st * kStage);
#pragma unroll
                for (int k = 0; k < 8; ++k) {  // K = 64 experts, 8 per MMA
                    const uint32_t o = (k & 3) * 32;  // K = 8 tf32 = 32 B inside a 128 B atom
                    tc_mma_tf32(tmem + acc * BN, sdesc(a + (k >> 2) * (kA / 2) + o, 16, 1024),
                                sdesc(b + (k >> 2) * (kB / 2) + o, 16, 1024), idesc, k ? 1u : 0u);
                }
                tc_commit(&empty[st]);
                tc_commit(&tfull[acc]);
                if (tile + 1 == t_end || (tile + 1) / NJ != tt) tc_commit(&aempty[(na - 1) & 1]);  // last use of this dLr
            }
        }
    } else {
        const int ew = warp - 2;
        const int quarter = warp & 3, half = ew >> 2;
        const int rl = quarter * 32 + lane;  // tile row = TMEM lane
        uint8_t* ob = obuf + ew * kOut;
        // Software pipeline over this CTA's tiles: the routing entries of tile
        // i+2 and the dispatch-backward rows of tile i+1 are in flight while
        // tile i is combined, so no tile waits a full memory latency for them.
        struct Route {
            int32_t pos[2], ch[2];
        };
        auto fetch_route = [&](int tile, Route& rt) {  // raw loads; decoded one iteration later
            rt.pos[0] = rt.pos[1] = -1;
            rt.ch[0] = rt.ch[1] = 0;
            if (tile >= t_end) return;
            const int64_t t = static_cast<int64_t>(tile / NJ) * BMT + rl;
            if (t >= p.T) return;
            rt.pos[0] = p.pos[t * p.K];
            rt.ch[0] = p.choice[t * p.K];
            if (p.K > 1) {
                rt.pos[1] = p.pos[t * p.K + 1];
                rt.ch[1] = p.choice[t * p.K + 1];
            }
        };
        struct Rows {
            int64_t r0, r1;
            bool none;
        };
        auto decode = [&](int tile, const Route& rt) {
            Rows r{-1, -1, false};
            if (tile >= t_end) return r;
            const int64_t t = static_cast<int64_t>(tile / NJ) * BMT + rl;
            if (t >= p.T) return r;
            if (rt.pos[0] >= 0) r.r0 = static_cast<int64_t>(rt.ch[0]) * p.cap_pad + rt.pos[0];
            if (rt.pos[1] >= 0) r.r1 = static_cast<int64_t>(rt.ch[1]) * p.cap_pad + rt.pos[1];
            r.none = rt.pos[0] < 0 && rt.pos[1] < 0;
            return r;
        };
        auto fetch_rows = [&](int tile, const Rows& r, uint4 (&g)[2][4]) {
            const int64_t t = static_cast<int64_t>(tile / NJ) * BMT + rl;
            const int jb = (tile % NJ) * BN + 32 * half;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                g[0][c] = r.r0 >= 0 ? __ldg(reinterpret_cast<const uint4*>(p.dX + r.r0 * p.d + jb) + c)
                                    : make_uint4(0, 0, 0, 0);
                const __nv_bfloat16* s1 = r.r1 >= 0 ? p.dX + r.r1 * p.d + jb : (r.none ? p.dy + t * p.d + jb : nullptr);
                g[1][c] = s1 ? __ldg(reinterpret_cast<const uint4*>(s1) + c) : make_uint4(0, 0, 0, 0);
            }
        };
        const int g0 = t_begin, gs = 1;
        Route rt_a, rt_b;
        fetch_route(g0, rt_a);
        Rows rows = decode(g0, rt_a);
        uint4 gA[2][4], gB[2][4];  // ping-pong: the current tile's rows / the next tile's (in flight)
        if (g0 < t_end) fetch_rows(g0, rows, gA);
        fetch_route(g0 + gs, rt_b);  // tile i+1's routing entries
        auto body = [&](const int tile, const int i, uint4 (&g)[2][4], uint4 (&gn)[2][4]) {
            const int st = i % kStages, acc = i & 1;
            const int64_t t = static_cast<int64_t>(tile / NJ) * BMT + rl;
            const int j0 = (tile % NJ) * BN + 32 * half;
            const int64_t r1 = rows.r1;
            const bool none = rows.none;
            // tile i+1: decode its routes, start its row loads; tile i+2: its routes
            const Rows rows_next = decode(tile + gs, rt_b);
            fetch_route(tile + 2 * gs, rt_b);  // before the row loads (keeps their scoreboards apart)
            if (tile + gs < t_end) fetch_rows(tile + gs, rows_next, gn);
            mbar_wait(&full[st], (i / kStages) & 1);
            mbar_wait(&tfull[acc], (i >> 1) & 1);
            tc_fence_after();
            uint32_t u[32];
            tmem_ld32(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + acc * BN + 32 * half, u);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
            float v[32];
            const uint32_t nb = smem_u32(sm + st * kStage + kB + half * (kNt / 2));
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                float4 n = make_float4(1.f, 1.f, 1.f, 1.f);
                if (p.has_noise) n = lds128f(nb + swz(rl, c));
                v[4 * c] = __uint_as_float(u[4 * c]) * n.x;
                v[4 * c + 1] = __uint_as_float(u[4 * c + 1]) * n.y;
                v[4 * c + 2] = __uint_as_float(u[4 * c + 2]) * n.z;
                v[4 * c + 3] = __uint_as_float(u[4 * c + 3]) * n.w;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);  // this warp is done with the stage's noise
            const bool add1 = r1 >= 0 || (none && p.residual_is_x);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                float w8[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) w8[q] = v[8 * c + q];
                add8(w8, g[0][c]);
                if (add1) add8(w8, g[1][c]);
#pragma unroll
                for (int q = 0; q < 8; ++q) v[8 * c + q] = w8[q];
            }
            if (!p.residual_is_x && p.dres && t < p.T) {  // explicit residual: dres = dy (no route kept) or 0
                uint4* dr = reinterpret_cast<uint4*>(p.dres + t * p.d + j0);
#pragma unroll
                for (int c = 0; c < 4; ++c) dr[c] = none ? g[1][c] : make_uint4(0, 0, 0, 0);
            }
            // stage [32 rows][32 bf16] (64B rows, 64B swizzle) and store with TMA
            uint8_t* sb = ob;
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            __syncwarp();
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                uint4 o;
                o.x = pack_bf16(v[8 * c], v[8 * c + 1]);
                o.y = pack_bf16(v[8 * c + 2], v[8 * c + 3]);
                o.z = pack_bf16(v[8 * c + 4], v[8 * c + 5]);
                o.w = pack_bf16(v[8 * c + 6], v[8 * c + 7]);
                sts128u(smem_u32(sb) + lane * 64 + ((c ^ ((lane >> 1) & 3)) << 4), o);
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
                asm volatile(
                    "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                        reinterpret_cast<uint64_t>(&p.tmO)),
                    "r"(smem_u32(sb)), "r"(j0), "r"(static_cast<int32_t>(t - lane))
                    : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            rows = rows_next;
        };
        for (int tile = g0, i = 0; tile < t_end; tile += 2, i += 2) {
            body(tile, i, gA, gB);
            if (tile + 1 < t_end) body(tile + 1, i + 1, gB, gA);
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        __syncwarp();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * BN));
    }
}

__global__ void round_wg_kernel(const float* __restrict__ wg, float* __restrict__ out, int64_t n) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) out[i] = tf32_rna_dev(wg[i]);
}
}  // namespace gdx


bool gate_dw_tma_ok(int d, int E) { return E == gbw::E && d % gbw::BJ == 0; }

// splits: token splits (grid = d/128 x splits); part [splits][d][E]
void launch_gate_dw_tma(const __nv_bfloat16* x, const float* noise, const float* dL, float* part, int64_t T, int d,
                        int splits, cudaStream_t st) {
    using namespace gbw;
    static bool attr = false;
    if (!attr) {
        MOE_CUDA_CHECK(cudaFuncSetAttribute(dw_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(kSmem)));
        attr = true;
    }
    Params p{};
    p.tmX = tc::make_map_2d(x, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, T, d, 64, BT, true);
    p.tmN = tc::make_map_2d(noise ? static_cast<const void*>(noise) : static_cast<const void*>(x),
                            CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, noise ? T : 1, noise ? d : 32, 32, noise ? BT : 1,
                            true);
    p.tmL = tc::make_map_2d(dL, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, T, E, 32, BT, true);
    p.part = part;
    p.T = T;
    p.tps = round_up(ceil_div(T, static_cast<int64_t>(splits)), static_cast<int64_t>(BT));
    p.d = d;
    p.has_noise = noise != nullptr;
    launch_pdl(dw_kernel, dim3(static_cast<unsigned>(d / BJ), static_cast<unsigned>(splits)), dim3(kThreads), kSmem,
               st, p);
}

}  // namespace moe

namespace moe {
bool gate_dx_tma_ok(int d, int E, int K) { return E == gdx::BN && d % gdx::BN == 0 && K <= 2; }

void launch_gate_round_wg(const float* wg, float* wgr, int d, int E, cudaStream_t st) {
    const int64_t n = static_cast<int64_t>(d) * E;
    launch_pdl(gdx::round_wg_kernel, dim3(static_cast<unsigned>(ceil_div(n, static_cast<int64_t>(256)))), dim3(256), 0,
               st, wg, wgr, n);
}

void launch_gate_dx_tma(int64_t T, int d, int K, int cap_pad, const float* dLr, const float* wgr, const float* noise,
                        const __nv_bfloat16* dX, const int32_t* choice, const int32_t* pos, const __nv_bfloat16* dy,
                        bool residual_is_x, __nv_bfloat16* dx, __nv_bfloat16* dres, cudaStream_t st) {
    using namespace gdx;
    static bool attr = false;
    if (!attr) {
        MOE_CUDA_CHECK(cudaFuncSetAttribute(dx_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(kSmem)));
        attr = true;
    }
    Params p{};
    p.tmA = tc::make_map_2d(dLr, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, T, BN, 32, BMT, true);
    p.tmB = tc::make_map_2d(wgr, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, d, BN, 32, BN, true);
    p.tmN = tc::make_map_2d(noise ? noise : wgr, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, noise ? T : d, noise ? d : BN, 32,
                            noise ? BMT : BN, true);
    p.tmO = tc::make_map_2d_swz(dx, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, T, d, 32, 32, 64);
    p.dX = dX;
    p.choice = choice;
    p.pos = pos;
    p.dy = dy;
    p.dres = dres;
    p.T = T;
    p.d = d;
    p.K = K;
    p.cap_pad = cap_pad;
    p.residual_is_x = residual_is_x ? 1 : 0;
    p.has_noise = noise != nullptr;
    const int64_t tiles = ceil_div(T, static_cast<int64_t>(BMT)) * (d / BN);
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(tiles, kNumSMs));
    launch_pdl(dx_kernel, dim3(grid), dim3(kThreads), kSmem, st, p);
}
}  // namespace moe
