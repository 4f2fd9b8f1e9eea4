// gemm_tc.cu — grouped expert GEMMs on 5th-gen tensor cores (sm_100a).
//
// The expert FFN of the reference (routing.cpp:397-406; kernels::matmul_acc /
// matmul_bt_acc / matmul_at_acc, ops.cpp:16-60) is >98% of the layer's work.
// Here it is a persistent, warp-specialised tcgen05 kernel:
//
//   warp 0      TMA producer: cp.async.bulk.tensor 128B-swizzled A/B tiles
//               into a kStages-deep shared-memory ring (mbarrier full/empty)
//   warp 1      MMA issuer: one thread issues tcgen05.mma.cta_group::1.kind::f16
//               (bf16 x bf16 -> fp32, M=128 N=256 K=16) into a TMEM accumulator;
//               tcgen05.commit releases smem stages and publishes finished tiles
//   warps 2..5  epilogue: tcgen05.ld 32x32b.x32 TMEM -> registers, fused
//               bias / ReLU / ReLU-mask, bf16 pack, 16-byte stores
//   TMEM        2 x 256 fp32 columns: the epilogue of tile i overlaps the MMAs
//               of tile i+1
//
// Two problem kinds share the machinery:
//   ROW    C[row, n] = epi(sum_k A[row,k] W_g(k,n))  — fwd1/fwd2 (W N-major)
//          and dgrad1/dgrad2 (W K-major); rows are the occupied rows of each
//          (origin rank, local expert) segment, tiles are compacted on device
//          from the per-segment counts, so no host sync and no empty tiles.
//   WGRAD  C_g[m, n] = sum_{rows of group g} A[row,m] B[row,n] — dW1/dW2
//          (both operands MN-major; the K loop walks the group's segments).
#include <cuda.h>

#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "gemm_tc.h"
#include "tc_ptx.cuh"

namespace moe {

namespace tc {

constexpr int BM = 128, BN = 256, BK = 64;
constexpr int kThreads = 192;  // 6 warps
constexpr uint32_t kTileABytes = BM * BK * 2;  // 16 KB
constexpr uint32_t kTileBBytes = BN * BK * 2;  // 32 KB
constexpr uint32_t kStageBytes = kTileABytes + kTileBBytes;
// epilogue staging: per epilogue warp, 1-2 buffers of 32 rows x 64 bf16 (128 B
// rows, 128B-swizzled) drained by TMA bulk tensor stores
constexpr uint32_t kStageCBytes = 32 * 64 * 2;  // 4 KB
constexpr int kMaxSegs = 1024;
constexpr int kMaxGroups = 256;

enum Kind { ROW = 0, WGRAD = 1 };


// Pipeline shape per kind.  ROW (fwd/dgrad, K = d or f) is MMA/HBM-streaming:
// 4 x 48 KB stages keep ~3 stages in flight, enough to cover TMA latency at
// the MMA's ~94 B/clk consumption (3 stages starved the MMA).  WGRAD (K = the
// expert's rows, ~128 on one GPU) is bound by its dW stores: 3 stages and a
// double-buffered epilogue.
#ifndef MOE_WG_STAGES
#define MOE_WG_STAGES 3
#endif
#ifndef MOE_WG_EPIBUFS
#define MOE_WG_EPIBUFS 2
#endif
#ifndef MOE_WG_EPIWARPS
#define MOE_WG_EPIWARPS 4
#endif
template <int KIND> struct KCfg {
    static constexpr int stages = KIND == ROW ? 4 : MOE_WG_STAGES;
    static constexpr int epi_bufs = KIND == ROW ? 1 : MOE_WG_EPIBUFS;
    static constexpr int epi_warps = KIND == ROW ? 4 : MOE_WG_EPIWARPS;  // 4 or 8 (two per TMEM lane quarter)
    static constexpr int threads = 64 + 32 * epi_warps;
    static constexpr uint32_t epi_bytes = epi_warps * epi_bufs * kStageCBytes;
    static constexpr size_t smem = 1024 /*align slack*/ + stages * kStageBytes + epi_bytes +
                                   1024 /*barriers*/ + 4 * (kMaxSegs + 3 * kMaxGroups + 8);
};

struct __align__(64) Params {
    CUtensorMap tmA;
    CUtensorMap tmB;
    CUtensorMap tmC;  // output, box {64 cols, 32 rows}, 128B swizzle
    void* C;
    const float* bias;
    const __nv_bfloat16* mask;
    const int32_t* counts;
    int64_t N;       // output columns
    int64_t K;       // ROW: reduction length
    int64_t M;       // WGRAD: output rows per group
    int ep, El, cap_pad;
    int epi;
    int b_mn;        // ROW: 1 if W is N-major
    float* colsum;   // ROW: optional per-32-row-block column sums of C
    int c_peer;      // ROW: store origin rank r's rows through tmC_peer[r]
    int c_mode;      // WGRAD: bit 0 accumulate into C, bit 1 C is fp32 (direct stores, no TMA)
    int tmem_x64;    // epilogue TMEM loads: 1 = one x64 load per chunk, 0 = two x32 loads
    uint64_t* relu_bits;  // ROW: ReLU mask bits [rows][N/64] (written by EPI_BIAS_RELU, read by EPI_RELU_MASK)
    CUtensorMap tmC_peer[8];  // [El*cap_pad, N] slices in the origin ranks' buffers
};

// Instruction descriptor, kind::f16: bf16 A/B, fp32 D, M=128, N=256.
__host__ __device__ constexpr uint32_t make_idesc(uint32_t a_mn, uint32_t b_mn) {
    return (1u << 4)            // D format f32
           | (1u << 7)          // A format bf16
           | (1u << 10)         // B format bf16
           | (a_mn << 15)       // A major (0 = K, 1 = MN)
           | (b_mn << 16)       // B major
           | ((BN >> 3) << 17)  // N
           | ((BM >> 4) << 24); // M
}

// ------------------------------------------------------------ tile scheduler
struct Sched {
    int32_t* seg_cnt;   // [nseg] counts
    int32_t* grp_mt;    // [El] m-tiles of the group
    int32_t* grp_base;  // [El+1] first tile of the group
    int total;
};

// ROW: tiles ordered (group, n-tile, m-tile) so the CTAs running at the same
// time share the group's weight tile through L2.
__device__ __forceinline__ void row_tile(const Params& p, const Sched& s, int NT, int t, int& seg,
                                         int& mt, int& nt) {
    int le = 0;
    while (le + 1 < p.El && s.grp_base[le + 1] <= t) ++le;
    const int local = t - s.grp_base[le];
    const int gm = s.grp_mt[le];
    nt = local / gm;
    int mi = local % gm;
    for (int r = 0; r < p.ep; ++r) {
        const int sg = r * p.El + le;
        const int c = (s.seg_cnt[sg] + BM - 1) / BM;
        if (mi < c) {
            seg = sg;
            mt = mi;
            return;
        }
        mi -= c;
    }
    seg = le;
    mt = 0;
}

template <int KIND>
__global__ void __launch_bounds__(KCfg<KIND>::threads, 1) grouped_gemm_kernel(const __grid_constant__ Params p) {
    constexpr int kStages = KCfg<KIND>::stages;
    constexpr int kEpiW = KCfg<KIND>::epi_warps;
    constexpr int kEpiBufs = KCfg<KIND>::epi_bufs;
    constexpr uint32_t kEpiBytes = KCfg<KIND>::epi_bytes;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in the shared window
    uint8_t* tiles = smem;
    uint8_t* cstage = smem + kStages * kStageBytes;  // [4 warps][2][4 KB]
    uint8_t* misc = cstage + kEpiBytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(misc);
    uint64_t* empty = full + kStages;
    uint64_t* tfull = empty + kStages;   // [2]
    uint64_t* tempty = tfull + 2;        // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    int32_t* seg_cnt = reinterpret_cast<int32_t*>(misc + 1024);
    int32_t* grp_mt = seg_cnt + kMaxSegs;
    int32_t* grp_base = grp_mt + kMaxGroups;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nseg = p.ep * p.El;

    // ---- setup: barriers, TMEM, schedule
    if (warp == 0 && lane == 0) {
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 32 * kEpiW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        prefetch_tmap(&p.tmA);
        prefetch_tmap(&p.tmB);
        prefetch_tmap(&p.tmC);
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    pdl_wait();  // barriers, TMEM and tensor maps are set up; now the predecessor's data
    pdl_trigger();
    for (int i = threadIdx.x; i < nseg; i += blockDim.x) seg_cnt[i] = p.counts[i];
    __syncthreads();
    Sched s{seg_cnt, grp_mt, grp_base, 0};
    int NT, MT;
    if (KIND == ROW) {
        NT = static_cast<int>(p.N / BN);
        for (int g = threadIdx.x; g < p.El; g += blockDim.x) {
            int m = 0;
            for (int r = 0; r < p.ep; ++r) m += (seg_cnt[r * p.El + g] + BM - 1) / BM;
            grp_mt[g] = m;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int acc = 0;
            for (int g = 0; g < p.El; ++g) {
                grp_base[g] = acc;
                acc += grp_mt[g] * NT;
            }
            grp_base[p.El] = acc;
        }
        __syncthreads();
        s.total = grp_base[p.El];
        MT = 0;
    } else {
        NT = static_cast<int>(p.N / BN);
        MT = static_cast<int>(p.M / BM);
        s.total = p.El * MT * NT;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ================= TMA producer =================
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int t = blockIdx.x; t < s.total; t += gridDim.x) {
                if (KIND == ROW) {
                    int seg, mt, nt;
                    row_tile(p, s, NT, t, seg, mt, nt);
                    const int le = seg % p.El;
                    const int32_t arow = seg * p.cap_pad + mt * BM;
                    const int nkb = static_cast<int>((p.K + BK - 1) / BK);
                    for (int kb = 0; kb < nkb; ++kb) {
                        mbar_wait(&empty[stage], phase ^ 1);
                        uint8_t* sa = tiles + stage * kStageBytes;
                        uint8_t* sb = sa + kTileABytes;
                        mbar_expect_tx(&full[stage], kStageBytes);
                        tma_load_2d(&p.tmA, &full[stage], sa, kb * BK, arow);
                        if (p.b_mn) {  // W [El*K, N]: 4 boxes {64 n, 64 k}
#pragma unroll
                            for (int j = 0; j < BN / 64; ++j)
                                tma_load_2d(&p.tmB, &full[stage], sb + j * (64 * BK * 2),
                                            nt * BN + j * 64, static_cast<int32_t>(le * p.K) + kb * BK);
                        } else {       // W [El*N, K]: one box {64 k, 256 n}
                            tma_load_2d(&p.tmB, &full[stage], sb, kb * BK,
                                        static_cast<int32_t>(le * p.N) + nt * BN);
                        }
                        if (++stage == kStages) { stage = 0; phase ^= 1; }
                    }
                } else {
                    const int g = t / (MT * NT);
                    const int rem = t % (MT * NT);
                    const int mt = rem / NT, nt = rem % NT;
                    for (int r = 0; r < p.ep; ++r) {
                        const int seg = r * p.El + g;
                        const int nkb = (seg_cnt[seg] + BK - 1) / BK;
                        for (int kb = 0; kb < nkb; ++kb) {
                            mbar_wait(&empty[stage], phase ^ 1);
                            uint8_t* sa = tiles + stage * kStageBytes;
                            uint8_t* sb = sa + kTileABytes;
                            const int32_t row = seg * p.cap_pad + kb * BK;
                            mbar_expect_tx(&full[stage], kStageBytes);
#pragma unroll
                            for (int j = 0; j < BM / 64; ++j)
                                tma_load_2d(&p.tmA, &full[stage], sa + j * (64 * BK * 2), mt * BM + j * 64, row);
#pragma unroll
                            for (int j = 0; j < BN / 64; ++j)
                                tma_load_2d(&p.tmB, &full[stage], sb + j * (64 * BK * 2), nt * BN + j * 64, row);
                            if (++stage == kStages) { stage = 0; phase ^= 1; }
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ================= MMA issuer =================
        if (lane == 0) {
            const uint32_t a_mn = KIND == WGRAD ? 1u : 0u;
            const uint32_t b_mn = KIND == WGRAD ? 1u : static_cast<uint32_t>(p.b_mn);
            const uint32_t idesc = make_idesc(a_mn, b_mn);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int t = blockIdx.x; t < s.total; t += gridDim.x) {
                int nkb;
                if (KIND == ROW) {
                    nkb = static_cast<int>((p.K + BK - 1) / BK);
                } else {
                    const int g = t / (MT * NT);
                    nkb = 0;
                    for (int r = 0; r < p.ep; ++r) nkb += (seg_cnt[r * p.El + g] + BK - 1) / BK;
                }
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t tmem_d = tmem_base + acc * BN;
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(tiles + stage * kStageBytes);
                    const uint32_t sb = sa + kTileABytes;
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) {
                        uint64_t ad, bd;
                        if (a_mn) ad = sdesc(sa + k * 2048, 64 * BK * 2, 1024);
                        else      ad = sdesc(sa + k * 32, 16, 1024);
                        if (b_mn) bd = sdesc(sb + k * 2048, 64 * BK * 2, 1024);
                        else      bd = sdesc(sb + k * 32, 16, 1024);
                        tc_mma(tmem_d, ad, bd, idesc, (kb | k) ? 1u : 0u);
                    }
                    tc_commit(&empty[stage]);  // smem stage free once these MMAs retire
                    if (++stage == kStages) { stage = 0; phase ^= 1; }
                }
                tc_commit(&tfull[acc]);  // accumulator ready (also fires if nkb == 0)
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
            }
        }
    } else {
        // ================= epilogue (warps 2..) =================
        const int quarter = warp & 3;  // TMEM lane quarter this warp may access
        const int ew = warp - 2;
        // with 8 epilogue warps, two per lane quarter split the tile's columns
        const int c_begin = kEpiW == 8 ? (ew >> 2) * (BN / 2) : 0;
        const int c_end = kEpiW == 8 ? c_begin + BN / 2 : BN;
        const int row_in_tile = quarter * 32 + lane;
        int acc = 0;
        uint32_t acc_phase = 0;
        uint32_t cbuf = 0;
        for (int t = blockIdx.x; t < s.total; t += gridDim.x) {
            int64_t crow;
            int64_t ncol0;
            bool valid;
            bool have_acc = true;
            int le = 0;
            if (KIND == ROW) {
                int seg, mt, nt;
                row_tile(p, s, NT, t, seg, mt, nt);
                le = seg % p.El;
                const int m = mt * BM + row_in_tile;
                valid = m < seg_cnt[seg];
                crow = static_cast<int64_t>(seg) * p.cap_pad + m;
                ncol0 = static_cast<int64_t>(nt) * BN;
            } else {
                const int g = t / (MT * NT);
                const int rem = t % (MT * NT);
                const int mt = rem / NT, nt = rem % NT;
                int nrows = 0;
                for (int r = 0; r < p.ep; ++r) nrows += seg_cnt[r * p.El + g];
                have_acc = nrows > 0;
                valid = true;
                crow = static_cast<int64_t>(g) * p.M + mt * BM + row_in_tile;
                ncol0 = static_cast<int64_t>(nt) * BN;
            }
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const uint32_t tbase = tmem_base + acc * BN + (static_cast<uint32_t>(quarter * 32) << 16);
            const int32_t box_row = static_cast<int32_t>(crow - lane);  // this warp's 32 rows
            // expert parallelism: origin rank r's rows go straight to its buffer
            const int32_t slice_rows = p.El * p.cap_pad;
            const int peer_r = (KIND == ROW && p.c_peer) ? box_row / slice_rows : -1;
            const CUtensorMap* out_map = peer_r >= 0 ? &p.tmC_peer[peer_r] : &p.tmC;
            const int32_t out_row = peer_r >= 0 ? box_row - peer_r * slice_rows : box_row;
#pragma unroll 1
            for (int c = c_begin; c < c_end; c += 64) {
                float f[64];
                if (p.tmem_x64) {  // one 32x32b.x64 TMEM load (one wait) per 64-column chunk
                    uint32_t v[64];
                    tmem_ld64(tbase + c, v);
#pragma unroll
                    for (int j = 0; j < 64; ++j) f[j] = __uint_as_float(v[j]);
                } else {
                    uint32_t v[32];
                    tmem_ld32(tbase + c, v);
#pragma unroll
                    for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[j]);
                    tmem_ld32(tbase + c + 32, v);
#pragma unroll
                    for (int j = 0; j < 32; ++j) f[32 + j] = __uint_as_float(v[j]);
                }
                if (c + 64 == c_end) {  // accumulator fully read: MMA may reuse it
                    tc_fence_before();
                    mbar_arrive(&tempty[acc]);
                }
                if (!have_acc || !valid) {
#pragma unroll
                    for (int j = 0; j < 64; ++j) f[j] = 0.f;
                } else if (KIND == ROW) {
                    if (p.epi == EPI_BIAS || p.epi == EPI_BIAS_RELU) {
                        const float* b = p.bias + static_cast<int64_t>(le) * p.N + ncol0 + c;
#pragma unroll
                        for (int j = 0; j < 64; j += 4) {
                            const float4 bb = __ldg(reinterpret_cast<const float4*>(b + j));
                            f[j] += bb.x; f[j + 1] += bb.y; f[j + 2] += bb.z; f[j + 3] += bb.w;
                        }
                        if (p.epi == EPI_BIAS_RELU) {
#pragma unroll
                            for (int j = 0; j < 64; ++j) f[j] = f[j] > 0.f ? f[j] : 0.f;
                        }
                    } else if (p.epi == EPI_RELU_MASK) {
                        if (p.relu_bits) {  // 64 mask bits of this row and chunk
                            const uint64_t mb = __ldg(reinterpret_cast<const unsigned long long*>(
                                p.relu_bits + crow * (p.N / 64) + (ncol0 + c) / 64));
#pragma unroll
                            for (int j = 0; j < 64; ++j)
                                if (!((mb >> j) & 1ull)) f[j] = 0.f;
                        } else {
                            const uint4* mp = reinterpret_cast<const uint4*>(p.mask + crow * p.N + ncol0 + c);
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                uint4 u = __ldg(mp + q);
                                const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
                                for (int j = 0; j < 8; ++j)
                                    if (!(__bfloat162float(h[j]) > 0.f)) f[q * 8 + j] = 0.f;
                            }
                        }
                    }
                }
                if (KIND == ROW && p.colsum)
                    epi_colsum64(f, lane, p.colsum + static_cast<int64_t>(box_row / 32) * p.N + ncol0 + c);
                if (KIND == WGRAD && p.c_mode) {
                    // fp32 and / or accumulating dW: this thread's row of 64
                    // columns straight to global (read-modify-write when accumulating)
                    const int64_t o = crow * p.N + ncol0 + c;
                    if (p.c_mode & 2) {
                        float4* dst = reinterpret_cast<float4*>(static_cast<float*>(p.C) + o);
#pragma unroll
                        for (int q = 0; q < 16; ++q) {
                            float4 v = make_float4(f[4 * q], f[4 * q + 1], f[4 * q + 2], f[4 * q + 3]);
                            if (p.c_mode & 1) {
                                const float4 old = dst[q];
                                v.x += old.x; v.y += old.y; v.z += old.z; v.w += old.w;
                            }
                            dst[q] = v;
                        }
                    } else {
                        uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.C) + o);
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            const uint4 old = dst[q];
                            const __nv_bfloat162* ob = reinterpret_cast<const __nv_bfloat162*>(&old);
                            uint4 u;
                            __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
                            for (int j = 0; j < 4; ++j)
                                h2[j] = __floats2bfloat162_rn(f[q * 8 + 2 * j] + __low2float(ob[j]),
                                                              f[q * 8 + 2 * j + 1] + __high2float(ob[j]));
                            dst[q] = u;
                        }
                    }
                    continue;
                }
                // stage the warp's 32 x 64 bf16 block (128B-swizzled rows) and
                // hand it to the TMA engine; two buffers alternate per warp
                uint8_t* sbuf = cstage + ((ew * kEpiBufs + (cbuf % kEpiBufs)) * kStageCBytes);
                if (lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kEpiBufs - 1) : "memory");
                __syncwarp();
                bool staged = false;
                if constexpr (KIND == ROW) {
                    if (p.relu_bits && p.epi == EPI_BIAS_RELU) {  // the ReLU mask as bits for dgrad2
                        uint64_t mb = 0;
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            uint4 u;
                            __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
                            for (int j = 0; j < 4; ++j)
                                h2[j] = __floats2bfloat162_rn(f[q * 8 + 2 * j], f[q * 8 + 2 * j + 1]);
                            const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
                            for (int j = 0; j < 4; ++j) {  // stored value > 0 (ReLU output: sign bit clear)
                                mb |= static_cast<uint64_t>((w4[j] & 0xffffu) != 0u) << (q * 8 + 2 * j);
                                mb |= static_cast<uint64_t>((w4[j] >> 16) != 0u) << (q * 8 + 2 * j + 1);
                            }
                            sts128(smem_u32(sbuf) + lane * 128 + ((q ^ (lane & 7)) << 4), u);
                        }
                        p.relu_bits[crow * (p.N / 64) + (ncol0 + c) / 64] = mb;
                        staged = true;
                    }
                }
                if (!staged) {
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        uint4 u;
                        __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
                        for (int j = 0; j < 4; ++j) h2[j] = __floats2bfloat162_rn(f[q * 8 + 2 * j], f[q * 8 + 2 * j + 1]);
                        sts128(smem_u32(sbuf) + lane * 128 + ((q ^ (lane & 7)) << 4), u);
                    }
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) {
                    asm volatile(
                        "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                            reinterpret_cast<uint64_t>(out_map)),
                        "r"(smem_u32(sbuf)), "r"(static_cast<int32_t>(ncol0 + c)), "r"(out_row)
                        : "memory");
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
                ++cbuf;
            }
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        __syncwarp();
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
    }
}

// ===================================================================== 2-CTA
// cta_group::2 variant for the compute-bound regime (experts with >= 2 row
// tiles, i.e. expert parallelism or large T).  A CTA pair (cluster of 2) owns a
// 256 x 256 output tile: each CTA stages its own 128 rows of A and HALF of B
// (128 of the 256 columns), so a stage is 32 KB per CTA and 6 stages fit; the
// leader issues tcgen05.mma.cta_group::2 (M=256, N=256) reading both CTAs'
// shared memory and writing each CTA's TMEM half.  Both CTAs' TMA loads
// complete on the leader's full barrier; MMA completion is multicast to both
// CTAs' empty / tmem-full barriers; both epilogues arrive on the leader's
// tmem-empty barrier.
namespace pair {

constexpr int kStages = 6;
constexpr uint32_t kHalfB = 128 * BK * 2;             // 16 KB
constexpr uint32_t kStage = kTileABytes + kHalfB;     // 32 KB
constexpr uint32_t kEpi = 4 * kStageCBytes;           // one staging buffer per epilogue warp
constexpr size_t kSmem = 1024 + kStages * kStage + kEpi + 1024 + 4 * (kMaxSegs + 3 * kMaxGroups + 8);

__device__ __forceinline__ uint32_t cta_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.aligned;\nbarrier.cluster.wait.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t leader_addr(const void* p) {  // same offset in CTA 0
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(0));
    return r;
}
__device__ __forceinline__ void tma_load_2d_pair(const CUtensorMap* map, uint32_t leader_bar,
                                                 void* dst, int32_t c0, int32_t c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void mma2(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                     uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void commit2(uint64_t* bar) {  // arrive on bar in both CTAs
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;" ::"r"(smem_u32(bar)),
        "h"(static_cast<uint16_t>(3))
        : "memory");
}
__device__ __forceinline__ void arrive_remote(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

__host__ __device__ constexpr uint32_t idesc2(uint32_t a_mn, uint32_t b_mn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (a_mn << 15) | (b_mn << 16) | ((BN >> 3) << 17) |
           ((256 >> 4) << 24);
}

// ROW: pair-tile t -> (group, n-tile, m-pair); this CTA takes m-tile 2*mp+rank
// of the group's m-tile list (segment-major).  valid = that m-tile exists.
__device__ __forceinline__ void row_pair_tile(const Params& p, const Sched& s, int NT, int t,
                                              uint32_t rank, int& seg, int& mt, int& nt,
                                              bool& valid) {
    int le = 0;
    while (le + 1 < p.El && s.grp_base[le + 1] <= t) ++le;
    const int local = t - s.grp_base[le];
    const int gmp = (s.grp_mt[le] + 1) / 2;
    nt = local / gmp;
    const int mp = local % gmp;
    int want = 2 * mp + static_cast<int>(rank);
    valid = want < s.grp_mt[le];
    if (!valid) want = 2 * mp;  // stage the partner's rows; results are masked
    for (int r = 0; r < p.ep; ++r) {
        const int sg = r * p.El + le;
        const int c = (s.seg_cnt[sg] + BM - 1) / BM;
        if (want < c) {
            seg = sg;
            mt = want;
            return;
        }
        want -= c;
    }
    seg = le;
    mt = 0;
    valid = false;
}

template <int KIND>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
gemm2_kernel(const __grid_constant__ Params p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in the shared window
    uint8_t* tiles = smem;
    uint8_t* cstage = smem + kStages * kStage;
    uint8_t* misc = cstage + kEpi;
    uint64_t* full = reinterpret_cast<uint64_t*>(misc);
    uint64_t* empty = full + kStages;
    uint64_t* tfull = empty + kStages;   // [2]
    uint64_t* tempty = tfull + 2;        // [2] (leader's are used)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    int32_t* seg_cnt = reinterpret_cast<int32_t*>(misc + 1024);
    int32_t* grp_mt = seg_cnt + kMaxSegs;
    int32_t* grp_base = grp_mt + kMaxGroups;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cta_rank();
    const bool leader = rank == 0;
    const int pair_id = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const int nseg = p.ep * p.El;

    if (warp == 0 && lane == 0) {
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 256);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        prefetch_tmap(&p.tmA);
        prefetch_tmap(&p.tmB);
        prefetch_tmap(&p.tmC);
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    pdl_wait();  // barriers, TMEM and tensor maps are set up; now the predecessor's data
    pdl_trigger();
    for (int i = threadIdx.x; i < nseg; i += blockDim.x) seg_cnt[i] = p.counts[i];
    __syncthreads();
    Sched s{seg_cnt, grp_mt, grp_base, 0};
    const int NT = static_cast<int>(p.N / BN);
    int MTP = 0;
    if (KIND == ROW) {
        for (int g = threadIdx.x; g < p.El; g += blockDim.x) {
            int m = 0;
            for (int r = 0; r < p.ep; ++r) m += (seg_cnt[r * p.El + g] + BM - 1) / BM;
            grp_mt[g] = m;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int acc = 0;
            for (int g = 0; g < p.El; ++g) {
                grp_base[g] = acc;
                acc += ((grp_mt[g] + 1) / 2) * NT;
            }
            grp_base[p.El] = acc;
        }
        __syncthreads();
        s.total = grp_base[p.El];
    } else {
        MTP = static_cast<int>(p.M / (2 * BM));
        s.total = p.El * MTP * NT;
    }
    tc_fence_before();
    cluster_sync();  // barriers of both CTAs initialised before any remote arrive
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ================= TMA producer (both CTAs) =================
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int t = pair_id; t < s.total; t += npairs) {
                int nkb_total = 0;
                int seg = 0, mt = 0, nt = 0, g = 0;
                bool valid = true;
                if (KIND == ROW) {
                    row_pair_tile(p, s, NT, t, rank, seg, mt, nt, valid);
                    nkb_total = static_cast<int>((p.K + BK - 1) / BK);
                } else {
                    g = t / (MTP * NT);
                    const int rem = t % (MTP * NT);
                    mt = 2 * (rem / NT) + static_cast<int>(rank);
                    nt = rem % NT;
                }
                const int le = seg % p.El;
                auto load_stage = [&](int32_t a_c0, int32_t a_c1, int32_t kcoord, int32_t rowk) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* sa = tiles + stage * kStage;
                    uint8_t* sb = sa + kTileABytes;
                    const uint32_t lbar = leader_addr(&full[stage]);
                    if (leader) mbar_expect_tx(&full[stage], 2 * kStage);
                    if (KIND == ROW) {
                        tma_load_2d_pair(&p.tmA, lbar, sa, a_c0, a_c1);
                        const int n_half = nt * BN + static_cast<int>(rank) * 128;
                        if (p.b_mn) {
#pragma unroll
                            for (int j = 0; j < 2; ++j)
                                tma_load_2d_pair(&p.tmB, lbar, sb + j * (64 * BK * 2), n_half + j * 64, kcoord);
                        } else {
                            tma_load_2d_pair(&p.tmB, lbar, sb, rowk, static_cast<int32_t>(le * p.N) + n_half);
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < BM / 64; ++j)
                            tma_load_2d_pair(&p.tmA, lbar, sa + j * (64 * BK * 2), mt * BM + j * 64, a_c1);
                        const int n_half = nt * BN + static_cast<int>(rank) * 128;
#pragma unroll
                        for (int j = 0; j < 2; ++j)
                            tma_load_2d_pair(&p.tmB, lbar, sb + j * (64 * BK * 2), n_half + j * 64, a_c1);
                    }
                    if (++stage == kStages) { stage = 0; phase ^= 1; }
                };
                if (KIND == ROW) {
                    const int32_t arow = seg * p.cap_pad + mt * BM;
                    for (int kb = 0; kb < nkb_total; ++kb)
                        load_stage(kb * BK, arow, static_cast<int32_t>(le * p.K) + kb * BK, kb * BK);
                } else {
                    for (int r = 0; r < p.ep; ++r) {
                        const int sg = r * p.El + g;
                        const int nkb = (seg_cnt[sg] + BK - 1) / BK;
                        for (int kb = 0; kb < nkb; ++kb) load_stage(0, sg * p.cap_pad + kb * BK, 0, 0);
                    }
                }
                (void)valid;
            }
        }
    } else if (warp == 1) {
        // ================= MMA issuer (leader only) =================
        if (leader && lane == 0) {
            const uint32_t a_mn = KIND == WGRAD ? 1u : 0u;
            const uint32_t b_mn = KIND == WGRAD ? 1u : static_cast<uint32_t>(p.b_mn);
            const uint32_t idesc = idesc2(a_mn, b_mn);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int t = pair_id; t < s.total; t += npairs) {
                int nkb;
                if (KIND == ROW) {
                    nkb = static_cast<int>((p.K + BK - 1) / BK);
                } else {
                    const int g = t / (MTP * NT);
                    nkb = 0;
                    for (int r = 0; r < p.ep; ++r) nkb += (seg_cnt[r * p.El + g] + BK - 1) / BK;
                }
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t tmem_d = tmem_base + acc * BN;
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(tiles + stage * kStage);
                    const uint32_t sb = sa + kTileABytes;
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) {
                        uint64_t ad, bd;
                        if (a_mn) ad = sdesc(sa + k * 2048, 64 * BK * 2, 1024);
                        else      ad = sdesc(sa + k * 32, 16, 1024);
                        if (b_mn) bd = sdesc(sb + k * 2048, 64 * BK * 2, 1024);
                        else      bd = sdesc(sb + k * 32, 16, 1024);
                        mma2(tmem_d, ad, bd, idesc, (kb | k) ? 1u : 0u);
                    }
                    commit2(&empty[stage]);
                    if (++stage == kStages) { stage = 0; phase ^= 1; }
                }
                commit2(&tfull[acc]);
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
            }
        }
    } else {
        // ================= epilogue (warps 2..5, both CTAs) =================
        const int quarter = warp & 3;
        const int row_in_tile = quarter * 32 + lane;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = pair_id; t < s.total; t += npairs) {
            int64_t crow, ncol0;
            bool valid;
            bool have_acc = true;
            int le = 0;
            if (KIND == ROW) {
                int seg, mt, nt;
                bool tvalid;
                row_pair_tile(p, s, NT, t, rank, seg, mt, nt, tvalid);
                le = seg % p.El;
                const int m = mt * BM + row_in_tile;
                valid = tvalid && m < seg_cnt[seg];
                crow = static_cast<int64_t>(seg) * p.cap_pad + m;
                ncol0 = static_cast<int64_t>(nt) * BN;
                if (!tvalid) crow = -1;  // nothing of this CTA's half is stored
            } else {
                const int g = t / (MTP * NT);
                const int rem = t % (MTP * NT);
                const int mt = 2 * (rem / NT) + static_cast<int>(rank), nt = rem % NT;
                int nrows = 0;
                for (int r = 0; r < p.ep; ++r) nrows += seg_cnt[r * p.El + g];
                have_acc = nrows > 0;
                valid = true;
                crow = static_cast<int64_t>(g) * p.M + mt * BM + row_in_tile;
                ncol0 = static_cast<int64_t>(nt) * BN;
            }
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const uint32_t tbase = tmem_base + acc * BN + (static_cast<uint32_t>(quarter * 32) << 16);
            const bool store = crow >= 0;
            const int32_t box_row = static_cast<int32_t>(crow - lane);
            const int32_t slice_rows = p.El * p.cap_pad;
            const int peer_r = (KIND == ROW && p.c_peer) ? box_row / slice_rows : -1;
            const CUtensorMap* out_map = peer_r >= 0 ? &p.tmC_peer[peer_r] : &p.tmC;
            const int32_t out_row = peer_r >= 0 ? box_row - peer_r * slice_rows : box_row;
#pragma unroll 1
            for (int c = 0; c < BN; c += 64) {
                float f[64];
                if (p.tmem_x64) {  // one 32x32b.x64 TMEM load (one wait) per 64-column chunk
                    uint32_t v[64];
                    tmem_ld64(tbase + c, v);
#pragma unroll
                    for (int j = 0; j < 64; ++j) f[j] = __uint_as_float(v[j]);
                } else {
                    uint32_t v[32];
                    tmem_ld32(tbase + c, v);
#pragma unroll
                    for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[j]);
                    tmem_ld32(tbase + c + 32, v);
#pragma unroll
                    for (int j = 0; j < 32; ++j) f[32 + j] = __uint_as_float(v[j]);
                }
                if (c + 64 == BN) {  // both CTAs arrive on the leader's tmem-empty barrier
                    tc_fence_before();
                    arrive_remote(leader_addr(&tempty[acc]));
                }
                if (!store) continue;
                if (!have_acc || !valid) {
#pragma unroll
                    for (int j = 0; j < 64; ++j) f[j] = 0.f;
                } else if (KIND == ROW) {
                    if (p.epi == EPI_BIAS || p.epi == EPI_BIAS_RELU) {
                        const float* b = p.bias + static_cast<int64_t>(le) * p.N + ncol0 + c;
#pragma unroll
                        for (int j = 0; j < 64; j += 4) {
                            const float4 bb = __ldg(reinterpret_cast<const float4*>(b + j));
                            f[j] += bb.x; f[j + 1] += bb.y; f[j + 2] += bb.z; f[j + 3] += bb.w;
                        }
                        if (p.epi == EPI_BIAS_RELU) {
#pragma unroll
                            for (int j = 0; j < 64; ++j) f[j] = f[j] > 0.f ? f[j] : 0.f;
                        }
                    } else if (p.epi == EPI_RELU_MASK) {
                        if (p.relu_bits) {  // 64 mask bits of this row and chunk
                            const uint64_t mb = __ldg(reinterpret_cast<const unsigned long long*>(
                                p.relu_bits + crow * (p.N / 64) + (ncol0 + c) / 64));
#pragma unroll
                            for (int j = 0; j < 64; ++j)
                                if (!((mb >> j) & 1ull)) f[j] = 0.f;
                        } else {
                            const uint4* mp = reinterpret_cast<const uint4*>(p.mask + crow * p.N + ncol0 + c);
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                uint4 u = __ldg(mp + q);
                                const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
                                for (int j = 0; j < 8; ++j)
                                    if (!(__bfloat162float(h[j]) > 0.f)) f[q * 8 + j] = 0.f;
                            }
                        }
                    }
                }
                if (KIND == ROW && p.colsum)
                    epi_colsum64(f, lane, p.colsum + static_cast<int64_t>(box_row / 32) * p.N + ncol0 + c);
                uint8_t* sbuf = cstage + quarter * kStageCBytes;
                if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                __syncwarp();
                bool staged = false;
                if constexpr (KIND == ROW) {
                    if (p.relu_bits && p.epi == EPI_BIAS_RELU) {  // the ReLU mask as bits for dgrad2
                        uint64_t mb = 0;
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            uint4 u;
                            __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
                            for (int j = 0; j < 4; ++j)
                                h2[j] = __floats2bfloat162_rn(f[q * 8 + 2 * j], f[q * 8 + 2 * j + 1]);
                            const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
                            for (int j = 0; j < 4; ++j) {  // stored value > 0 (ReLU output: sign bit clear)
                                mb |= static_cast<uint64_t>((w4[j] & 0xffffu) != 0u) << (q * 8 + 2 * j);
                                mb |= static_cast<uint64_t>((w4[j] >> 16) != 0u) << (q * 8 + 2 * j + 1);
                            }
                            sts128(smem_u32(sbuf) + lane * 128 + ((q ^ (lane & 7)) << 4), u);
                        }
                        p.relu_bits[crow * (p.N / 64) + (ncol0 + c) / 64] = mb;
                        staged = true;
                    }
                }
                if (!staged) {
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        uint4 u;
                        __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
                        for (int j = 0; j < 4; ++j) h2[j] = __floats2bfloat162_rn(f[q * 8 + 2 * j], f[q * 8 + 2 * j + 1]);
                        sts128(smem_u32(sbuf) + lane * 128 + ((q ^ (lane & 7)) << 4), u);
                    }
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) {
                    asm volatile(
                        "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                            reinterpret_cast<uint64_t>(out_map)),
                        "r"(smem_u32(sbuf)), "r"(static_cast<int32_t>(ncol0 + c)), "r"(out_row)
                        : "memory");
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
            }
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        __syncwarp();
    }
    __syncthreads();
    cluster_sync();  // the partner's MMAs may still read this CTA's smem / TMEM
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
    }
}

}  // namespace pair

// ------------------------------------------------------------ host side
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn get_encode() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    });
    if (!fn) throw Status(6, "cuTensorMapEncodeTiled unavailable");
    return fn;
}

// 2D bf16 tensor [rows, cols] row-major, box {box_cols (inner), box_rows}, 128B swizzle
CUtensorMap make_map(const void* base, int64_t rows, int64_t cols, int box_cols, int box_rows) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols * 2)};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                              strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Status(6, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return m;
}

// general 2D map: [rows, cols] row-major of `esz`-byte elements, box {box_cols, box_rows}
CUtensorMap make_map_2d(const void* base, CUtensorMapDataType dt, int esz, int64_t rows, int64_t cols,
                        int box_cols, int box_rows, bool swizzle128) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols * esz)};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = get_encode()(&m, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE,
                              swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Status(6, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return m;
}

// the same with an explicit swizzle span (0, 32, 64 or 128 bytes)
CUtensorMap make_map_2d_swz(const void* base, CUtensorMapDataType dt, int esz, int64_t rows, int64_t cols,
                            int box_cols, int box_rows, int swizzle_bytes) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols * esz)};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
    const cuuint32_t estr[2] = {1, 1};
    const CUtensorMapSwizzle sw = swizzle_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                  : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                  : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                        : CU_TENSOR_MAP_SWIZZLE_NONE;
    CUresult r = get_encode()(&m, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Status(6, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return m;
}

int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = kNumSMs;
    }
    return n;
}
// SMs for a persistent grid that leaves `reserve` SMs to a co-running kernel
int grid_sms(int reserve) { return std::max(2, num_sms() - std::max(0, reserve)); }

template <int KIND>
void launch(const Params& p, int64_t max_tiles, cudaStream_t st, int reserve) {
    static bool attr = false;
    if (!attr) {
        MOE_CUDA_CHECK(cudaFuncSetAttribute(grouped_gemm_kernel<KIND>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(KCfg<KIND>::smem)));
        attr = true;
    }
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(grid_sms(reserve), max_tiles)));
    launch_pdl(grouped_gemm_kernel<KIND>, dim3(grid), dim3(KCfg<KIND>::threads), KCfg<KIND>::smem, st, p);
}


template <int KIND>
void launch_pair(const Params& p, int64_t max_pair_tiles, cudaStream_t st, int reserve) {
    static bool attr = false;
    if (!attr) {
        MOE_CUDA_CHECK(cudaFuncSetAttribute(pair::gemm2_kernel<KIND>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(pair::kSmem)));
        attr = true;
    }
    const int npairs = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(grid_sms(reserve) / 2, max_pair_tiles)));
    launch_pdl(pair::gemm2_kernel<KIND>, dim3(2 * npairs), dim3(kThreads), pair::kSmem, st, p);
}

// 2-CTA pairs pay off when the MMA is the bottleneck: every expert has >= 2
// row tiles (ROW) / K spans >= 256 rows (WGRAD).  MOE_B200_PAIR=0/1 forces.
static int tmem_x64() {  // MOE_B200_TMEM_X64=0: two x32 TMEM loads per epilogue chunk
    static int v = [] {
        const char* e = std::getenv("MOE_B200_TMEM_X64");
        return e ? std::atoi(e) : 1;
    }();
    return v;
}
static int pair_override() {
    static int v = [] {
        const char* e = std::getenv("MOE_B200_PAIR");
        return e ? std::atoi(e) : -1;
    }();
    return v;
}
static int wg_pair_override() {  // MOE_B200_WG_PAIR=0/1: weight-gradient GEMMs only
    static int v = [] {
        const char* e = std::getenv("MOE_B200_WG_PAIR");
        return e ? std::atoi(e) : pair_override();
    }();
    return v;
}

}  // namespace tc

static bool g_tc_enabled = true;
void tc_set_enabled(bool on) { g_tc_enabled = on; }
bool tc_enabled() { return g_tc_enabled; }

bool tc_row_gemm_supported(const RowGemmArgs& a) {
    return g_tc_enabled && a.N % tc::BN == 0 && a.K % tc::BK == 0 && a.cap_pad % tc::BM == 0 &&
           a.ep * a.El <= tc::kMaxSegs && a.El <= tc::kMaxGroups;
}

bool tc_wgrad_gemm_supported(const WgradGemmArgs& a) {
    return g_tc_enabled && a.N % tc::BN == 0 && a.M % tc::BM == 0 && a.cap_pad % tc::BK == 0 &&
           a.ep * a.El <= tc::kMaxSegs && a.El <= tc::kMaxGroups;
}

void launch_row_gemm_tc(const RowGemmArgs& a, cudaStream_t st) {
    tc::Params p{};
    const int64_t rows = static_cast<int64_t>(a.ep) * a.El * a.cap_pad;
    p.tmA = tc::make_map(a.A, rows, a.K, tc::BK, tc::BM);
    if (a.w_nmajor)
        p.tmB = tc::make_map(a.W, static_cast<int64_t>(a.El) * a.K, a.N, 64, tc::BK);
    else
        p.tmB = tc::make_map(a.W, static_cast<int64_t>(a.El) * a.N, a.K, tc::BK, tc::BN);
    p.tmC = tc::make_map(a.C, rows, a.N, 64, 32);
    p.C = a.C;
    p.bias = a.bias;
    p.mask = static_cast<const __nv_bfloat16*>(a.mask);
    p.counts = a.counts;
    p.N = a.N;
    p.K = a.K;
    p.M = 0;
    p.ep = a.ep;
    p.El = a.El;
    p.cap_pad = a.cap_pad;
    p.epi = a.epi;
    p.b_mn = a.w_nmajor ? 1 : 0;
    p.colsum = a.epi == EPI_RELU_MASK ? a.colsum : nullptr;
    p.relu_bits = (a.epi == EPI_RELU_MASK || a.epi == EPI_BIAS_RELU) ? a.relu_bits : nullptr;
    p.c_peer = 0;
    if (a.c_peer) {
        if (a.ep > 8) throw Status(8, "row gemm: peer stores support at most 8 ranks");
        for (int r = 0; r < a.ep; ++r)
            p.tmC_peer[r] = tc::make_map(a.c_peer[r], static_cast<int64_t>(a.El) * a.cap_pad, a.N, 64, 32);
        p.c_peer = 1;
    }
    p.tmem_x64 = tc::tmem_x64();
    const int64_t max_tiles = rows / tc::BM * (a.N / tc::BN);
    const int ov = tc::pair_override();
    const bool use_pair = ov >= 0 ? ov == 1 : static_cast<int64_t>(a.ep) * a.cap_pad >= 2 * tc::BM;
    if (use_pair) {
        if (!a.w_nmajor)  // each CTA stages 128 of the 256 weight rows
            p.tmB = tc::make_map(a.W, static_cast<int64_t>(a.El) * a.N, a.K, tc::BK, 128);
        tc::launch_pair<tc::ROW>(p, (max_tiles + 1) / 2, st, a.sm_reserve);
    } else {
        tc::launch<tc::ROW>(p, max_tiles, st, a.sm_reserve);
    }
}

void launch_wgrad_gemm_tc(const WgradGemmArgs& a, cudaStream_t st) {
    tc::Params p{};
    const int64_t rows = static_cast<int64_t>(a.ep) * a.El * a.cap_pad;
    p.tmA = tc::make_map(a.A, rows, a.M, 64, tc::BK);
    p.tmB = tc::make_map(a.B, rows, a.N, 64, tc::BK);
    p.tmC = tc::make_map(a.C, static_cast<int64_t>(a.El) * a.M, a.N, 64, 32);
    p.C = a.C;
    p.counts = a.counts;
    p.N = a.N;
    p.M = a.M;
    p.K = 0;
    p.ep = a.ep;
    p.El = a.El;
    p.cap_pad = a.cap_pad;
    p.epi = EPI_NONE;
    p.b_mn = 1;
    p.c_mode = a.c_mode;
    p.tmem_x64 = tc::tmem_x64();
    const int64_t max_tiles = static_cast<int64_t>(a.El) * (a.M / tc::BM) * (a.N / tc::BN);
    const int ov = tc::wg_pair_override();
    const bool use_pair = a.c_mode == 0 && (a.M / tc::BM) % 2 == 0 &&
                          (ov >= 0 ? ov == 1 : static_cast<int64_t>(a.ep) * a.cap_pad >= 4 * tc::BK);
    if (use_pair)
        tc::launch_pair<tc::WGRAD>(p, max_tiles / 2, st, a.sm_reserve);
    else
        tc::launch<tc::WGRAD>(p, max_tiles, st, a.sm_reserve);
}

}  // namespace moe
