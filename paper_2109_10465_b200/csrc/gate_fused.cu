// gate_fused.cu — the fused gate of the bf16 path: logits, softmax, top-1 /
// top-2, balance-loss partials and the balance-loss finalize in ONE kernel
// (routing.cpp:51-101 gate_forward + routing.cpp:348-374 balance_loss).
//
// A cluster of two CTAs owns 128 tokens; CTA r reduces half of d:
//
//   warp 0      TMA producer: raw x (bf16) and jitter (fp32) tiles [128 x 64]
//               (128 B row segments, 128B-swizzled) into a 2-deep ring, and
//               the pre-split tf32 hi / lo halves of
//               Wg^T [64 x 32] (128B-swizzled, read by the MMA in place) into
//               a 3-deep ring
//   warps 2..5  transform: g = x * noise, 3xTF32 split g = hi + lo, written
//               into the 128B-swizzled K-major A operand (2-deep ring)
//   warp 1      MMA: tcgen05.mma kind::tf32, M=128 N=64 K=8, hi*hi + hi*lo +
//               lo*hi into four TMEM accumulators (one per K=8 sub-step,
//               summed in fixed order: fp32-FMA accuracy at d = 2048)
//   epilogue    the two CTAs swap their partial logits for each other's 64
//               rows through distributed shared memory (st.shared::cluster),
//               then each thread owns one token row: softmax (ops.cpp:77-90),
//               top-1 / top-2 with the reference's tie rules (routing.cpp:
//               77-92), probabilities / choices / gate_prob stores, and the
//               per-64-row column sums and first-choice counts of the balance
//               loss (reduced in fixed order by balance_finalize_kernel on the
//               side stream, off the routing's critical path).
//
// No logits or split-K partials go to HBM: the kernel reads x (and the
// jitter) once and writes P, the decision and the small balance partials.
#include <cuda.h>

#include <cstdlib>

#include "common.cuh"
#include "gemm_tc.h"
#include "kernels.h"
#include "tc_ptx.cuh"

namespace moe {
unsigned long long* g_gate_stamps = nullptr;  // probe 8 (debug)
namespace gf {

using namespace tc;

// Experts: the kernel is instantiated for EP = 16, 32, 64 TMEM columns per
// accumulator (the MMA's N); E = 8 runs on the EP = 16 instance with the B
// operand's rows 8..15 zero and those columns masked out of the routing.
#ifndef MOE_GATE_TS
#define MOE_GATE_TS 1
#endif
#ifndef MOE_GATE_BBYTES
#define MOE_GATE_BBYTES 65536
#endif
#ifndef MOE_GATE_RAW
#define MOE_GATE_RAW (MOE_GATE_TS ? 3 : 2)
#endif
constexpr int BM = 128;            // tokens per cluster
constexpr int BK = 32;             // fp32 K elements per MMA step (one 128 B swizzle row)
constexpr int BKR = 64;            // K elements per raw stage (x rows of 128 B: full DRAM bursts)
constexpr int kRaw = MOE_GATE_RAW; // raw x / noise ring depth (the A ring's smem goes here under TS)
constexpr int kOp = MOE_GATE_TS ? 4 : 2;  // A-operand ring depth (MMA steps)
#ifndef MOE_GATE_N2
#define MOE_GATE_N2 MOE_GATE_TS
#endif
// TMEM accumulators.  N2 (TS only): B hi and lo sit back to back in the B stage,
// so hi.hi and hi.lo are ONE MMA with N = 2E into an accumulator of 2E columns
// ([hh + lh | hl], summed in the epilogue) and lo.hi a second one with N = E:
// two MMA instructions per K step of 8 instead of three.
constexpr int kNAcc = MOE_GATE_N2 ? 2 : 4;
constexpr int kAccW = MOE_GATE_N2 ? 2 : 1;  // accumulator width in units of E
constexpr int kTw = 8;             // transform warps (two per SM sub-partition)
constexpr int kThreads = 32 * (2 + kTw);
constexpr uint32_t kRawX = BM * BKR * 2;       // 16 KB bf16 x   [128 rows x 128 B], 128B swizzle
constexpr uint32_t kRawN = BM * BKR * 4;       // 32 KB fp32 noise: two [128 x 128 B] halves, swizzled
constexpr uint32_t kRawStage = kRawX + kRawN;                // 48 KB
// without jitter (eval) a raw stage is the 16 KB x tile, so the same bytes
// hold 3x the stages: more loads in flight for the same shared memory
constexpr int kRawMax = 3 * kRaw;
constexpr uint32_t kOpStage = 2 * BM * 128;                  // 32 KB (A hi, A lo)
constexpr uint32_t kOpSmem = MOE_GATE_TS ? 0 : kOp * kOpStage; // A lives in TMEM under TS
// SM2: the eval-only (no jitter) instance for EP = 16 sized for TWO CTAs per SM
// (smem ~103 KB, 256 TMEM columns, <= 102 registers): without jitter the main
// loop is a latency chain (TMA -> transform -> MMA), and a second resident
// CTA runs a second chain on the same SM.
template <int EP, bool SM2 = false> struct GCfg {
    static constexpr uint32_t kRawB = EP * 128;              // per hi / lo: 8 KB at EP = 64
    static constexpr uint32_t kBStage = 2 * kRawB;
    // B (Wg^T hi / lo) ring depth in MMA steps: 64 KB of B in flight under TS
    // (L2 latency ~1 us against ~0.5 us per step), 3 steps without
    static constexpr int kB = SM2 ? 8 : MOE_GATE_TS ? (MOE_GATE_BBYTES / kBStage < 16 ? static_cast<int>(MOE_GATE_BBYTES / kBStage) : 16) : 3;
    static constexpr int kRawT = SM2 ? 1 : kRaw;             // raw stages with jitter (SM2: unused)
    static constexpr int kRawE = SM2 ? 4 : kRawMax;          // raw stages without jitter (16 KB each)
    static constexpr int kRawM = kRawT > kRawE ? kRawT : kRawE;
    static constexpr uint32_t kRawBytes = SM2 ? kRawE * kRawX : kRaw * kRawStage;
    static constexpr int kOpD = SM2 ? 2 : kOp;               // A ring depth (MMA steps)
    static constexpr uint32_t kRecv = 64 * EP * 4;           // peer's partials for my rows
    static constexpr uint32_t kSmem = 1024 + kRawBytes + kB * kBStage + kOpSmem + kRecv + 512;
    static constexpr int kMinBlocks = SM2 ? 2 : 1;
    static_assert((2 * kRawM + 2 * kB + 2 * kOpD + 1) * 8 + 4 <= 512, "barrier area");
    static_assert(!SM2 || (MOE_GATE_TS && kSmem + 1024 <= 232448 / 2), "SM2 shared memory");
};

struct __align__(64) Params {
    CUtensorMap tmX, tmN, tmBh, tmBl;
    float* probs;
    int32_t* choice;
    float* gate_prob;
    float* colsum_part;   // [parts][E], part = 64 tokens
    int32_t* count_part;  // [parts][E]
    uint32_t* flags;
    int64_t T;
    int d, K, nparts, has_noise;
    int ne;     // experts (<= the instance's EP; probs / partials rows are ne wide)
    int csize;  // CTAs per 128-token tile: 2 (a cluster, each CTA half of d) or 1 (one CTA, all of d)
    int probe;  // timing probes (MOE_B200_GATE_PROBE): 1 no split math, 2 no MMA, 8 phase timestamps
    unsigned long long* stamps;  // probe 8: [CTA][8] %globaltimer at phase boundaries
};

// Round to tf32, nearest with ties away from zero, on the integer pipes:
// adding half an ulp of bit 13 to the sign-magnitude bits and clearing the 13
// low bits is exactly cvt.rna.tf32.f32 (carries into the exponent round up to
// the next binade or to infinity; infinities and NaNs keep their class), but
// two ALU operations instead of a conversion on the XU pipe, which the
// transform's two roundings per element otherwise saturate.
__device__ __forceinline__ float tf32_rna(float v) {
#ifdef MOE_GATE_CVT_RNA
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
    return __uint_as_float(r);
#else
    return __uint_as_float((__float_as_uint(v) + 0x1000u) & 0xFFFFE000u);
#endif
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t map_peer(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_cluster_v4(uint32_t addr, float a, float b, float c, float d) {
    asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a), "f"(b), "f"(c),
                 "f"(d)
                 : "memory");
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t swz(int r, int c) { return r * 128 + ((c ^ (r & 7)) << 4); }
// probe 16 (debug): per-stage timeline of CTAs 0..7, [cta][64] ns:
// [r] producer issued raw stage r, [16+r] transform saw it land, [32+r]
// transform done with it, [48+r] MMA issued its second step
// (scripts/micro/gate_timeline.py)
// (compiled in only with -DMOE_GATE_TIMELINE, so the hot loop carries no probe branch)
__device__ __forceinline__ void tl(const Params& p, int slot) {
#ifdef MOE_GATE_TIMELINE
    if (!(p.probe & 16) || blockIdx.x >= 8 || slot >= 64) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.stamps[blockIdx.x * 64 + slot] = t;
#else
    (void)p;
    (void)slot;
#endif
}
__device__ __forceinline__ void stamp(const Params& p, int i) {
    if (!(p.probe & 8)) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.stamps[blockIdx.x * 8 + i] = t;
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// A operand in TMEM (tcgen05.mma ... [a_tmem], b_desc): the 3xTF32 products
// re-read A three times, and with A in shared memory those reads (with the
// transform's stores) saturate its bandwidth.  The transform then
// writes hi / lo with tcgen05.st: 32 lanes = 32 token rows of the warp's lane
// quarter, 16 K columns per warp (two warps per quarter).
__device__ __forceinline__ void tc_mma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}

template <int E, bool SM2>
__global__ void __launch_bounds__(kThreads, GCfg<E, SM2>::kMinBlocks) gate_kernel(const __grid_constant__ Params p) {
    using C = GCfg<E, SM2>;
    constexpr int kOp = C::kOpD;
    constexpr int kRaw = C::kRawT;
    constexpr int kRawMax = C::kRawE;  // the no-jitter ring depth (the ring's max)
    // TMEM: kNAcc accumulators of E columns, then (TS) kOp stages of A hi / lo [128 x 32] each
    constexpr uint32_t kTmemA = kNAcc * kAccW * E;
    constexpr uint32_t kTmemCols = MOE_GATE_TS ? (kTmemA + kOp * 64 <= 256 ? 256 : 512) : kTmemA;
    constexpr uint32_t kRawB = C::kRawB;
    constexpr uint32_t kBStage = C::kBStage;
    constexpr uint32_t kRecv = C::kRecv;
    constexpr int kB = C::kB;
    static_assert(C::kRawM == (kRaw > kRawMax ? kRaw : kRawMax), "ring");
    const int ne = p.ne;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* raw = sm;
    uint8_t* bst = raw + C::kRawBytes;
    uint8_t* op = bst + kB * kBStage;
    float* recv = reinterpret_cast<float*>(op + kOpSmem);
    uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(recv) + kRecv);
    uint64_t* raw_full = bars;
    uint64_t* raw_empty = raw_full + C::kRawM;
    uint64_t* b_full = raw_empty + C::kRawM;
    uint64_t* b_empty = b_full + kB;
    uint64_t* op_full = b_empty + kB;
    uint64_t* op_empty = op_full + kOp;
    uint64_t* acc_full = op_empty + kOp;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(acc_full + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const int cs = p.csize;
    const int64_t t0 = static_cast<int64_t>(blockIdx.x / cs) * BM;
    const int kspan = p.d / cs;
    const int kbase = static_cast<int>(rank) * kspan;
    const int nsteps = kspan / BK;   // MMA steps
    const int nraw = kspan / BKR;    // raw stages (two MMA steps each)
    // every cluster walks its K range from a different starting stage, so the
    // 128 CTAs do not all read the same Wg^T tile from L2 at the same time
    const int nr = p.has_noise ? kRaw : kRawMax;  // raw ring depth and stage stride
    const uint32_t rstride = p.has_noise ? kRawStage : kRawX;
    const int kskew = static_cast<int>((blockIdx.x / cs) % nraw);

    if (threadIdx.x == 0) stamp(p, 0);
    if (threadIdx.x == 0) {
        for (int i = 0; i < C::kRawM; ++i) {
            mbar_init(&raw_full[i], 1);
            mbar_init(&raw_empty[i], kTw);  // the transform warps have read x / noise
        }
        for (int i = 0; i < kB; ++i) {
            mbar_init(&b_full[i], 1);
            mbar_init(&b_empty[i], 1);    // the MMAs of the step have read B
        }
        for (int i = 0; i < kOp; ++i) {
            mbar_init(&op_full[i], kTw);
            mbar_init(&op_empty[i], 1);
        }
        mbar_init(acc_full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        prefetch_tmap(&p.tmX);
        prefetch_tmap(&p.tmN);
        prefetch_tmap(&p.tmBh);
        prefetch_tmap(&p.tmBl);
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    pdl_wait();  // x, the jitter stream and the split gate weights come from predecessors
    pdl_trigger();
    if (threadIdx.x == 0) stamp(p, 1);

    if (warp == 0) {
        // ---------------- TMA producer
        if (lane == 0) {
            const uint32_t bytes = kRawX + (p.has_noise ? kRawN : 0);
            for (int r = 0; r < nraw; ++r) {
                const int rs = r % nr;
                const int k0 = kbase + ((r + kskew) % nraw) * BKR;
                if (r >= nr) mbar_wait(&raw_empty[rs], ((r / nr) - 1) & 1);
                uint8_t* st = raw + rs * rstride;
                if (r < 16) tl(p, r);
                mbar_expect_tx(&raw_full[rs], bytes);
                tma_load_2d(&p.tmX, &raw_full[rs], st, k0, static_cast<int32_t>(t0));
                if (p.has_noise) {
                    tma_load_2d(&p.tmN, &raw_full[rs], st + kRawX, k0, static_cast<int32_t>(t0));
                    tma_load_2d(&p.tmN, &raw_full[rs], st + kRawX + kRawN / 2, k0 + BK, static_cast<int32_t>(t0));
                }
            }
        } else if (lane == 1) {
            // B runs on its own lane, so a B stage held by the MMAs never
            // delays the next x / noise issue
            for (int s = 0; s < nsteps; ++s) {
                const int bs = s % kB;
                const int k0 = kbase + (((s >> 1) + kskew) % nraw) * BKR + (s & 1) * BK;
                if (s >= kB) mbar_wait(&b_empty[bs], ((s / kB) - 1) & 1);
#ifdef MOE_GATE_BSTALE  // timing probe only: B loaded once, then reused (wrong logits)
                if (s >= kB) { mbar_arrive(&b_full[bs]); continue; }
#endif
                uint8_t* bt = bst + bs * kBStage;
                mbar_expect_tx(&b_full[bs], kBStage);
                tma_load_2d(&p.tmBh, &b_full[bs], bt, k0, 0);
                tma_load_2d(&p.tmBl, &b_full[bs], bt + kRawB, k0, 0);
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer
        if (lane == 0) {
            constexpr uint32_t idesc = make_idesc_tf32(BM, E, 0, 0);
            for (int s = 0; s < nsteps; ++s) {
                const int bs = s % kB, os = s % kOp;
                mbar_wait(&b_full[bs], (s / kB) & 1);
#ifndef MOE_GATE_NOOPWAIT  // timing probe only: MMAs do not wait for the transform
                mbar_wait(&op_full[os], (s / kOp) & 1);
#endif
                if ((s & 1) && (s >> 1) < 16) tl(p, 48 + (s >> 1));
                tc_fence_after();
                const uint32_t b = smem_u32(bst + bs * kBStage);
#if MOE_GATE_TS
                const uint32_t ta = tmem + kTmemA + os * 64;  // hi at +0, lo at +32 columns
#pragma unroll
                for (int kk = 0; kk < BK / 8; ++kk) {
                    if (p.probe & 2) break;
                    const uint64_t bh = sdesc(b + kk * 32, 16, 1024);
#if MOE_GATE_N2
                    constexpr uint32_t idesc2 = make_idesc_tf32(BM, 2 * E, 0, 0);
                    const uint32_t acc = tmem + (kk % kNAcc) * 2 * E;
                    tc_mma_tf32_ts(acc, ta + kk * 8, bh, idesc2, (s || kk >= kNAcc) ? 1u : 0u);  // [hh | hl]
                    tc_mma_tf32_ts(acc, ta + 32 + kk * 8, bh, idesc, 1u);                      // += lh
#else
                    const uint64_t bl = sdesc(b + kRawB + kk * 32, 16, 1024);
                    const uint32_t acc = tmem + kk * E;
                    tc_mma_tf32_ts(acc, ta + kk * 8, bh, idesc, s ? 1u : 0u);
                    tc_mma_tf32_ts(acc, ta + kk * 8, bl, idesc, 1u);
                    tc_mma_tf32_ts(acc, ta + 32 + kk * 8, bh, idesc, 1u);
#endif
                }
#else
                const uint32_t a = smem_u32(op + os * kOpStage);
#pragma unroll
                for (int kk = 0; kk < BK / 8; ++kk) {
                    if (p.probe & 2) break;
                    const uint64_t ah = sdesc(a + kk * 32, 16, 1024);
                    const uint64_t al = sdesc(a + BM * 128 + kk * 32, 16, 1024);
                    const uint64_t bh = sdesc(b + kk * 32, 16, 1024);
                    const uint64_t bl = sdesc(b + kRawB + kk * 32, 16, 1024);
                    const uint32_t acc = tmem + kk * E;
                    tc_mma_tf32(acc, ah, bh, idesc, s ? 1u : 0u);
                    tc_mma_tf32(acc, ah, bl, idesc, 1u);
                    tc_mma_tf32(acc, al, bh, idesc, 1u);
                }
#endif
                tc_commit(&op_empty[os]);  // A operand stage free
                tc_commit(&b_empty[bs]);   // B stage free
            }
            tc_commit(acc_full);
        }
    } else {
#if MOE_GATE_TS
        // ---------------- transform: g = x * noise -> tf32 hi / lo into TMEM.
        // Warp w owns TMEM lane quarter w % 4 (token rows 32q + lane) and one
        // half of each op stage's 32 K columns; each thread reads its own row.
        const int tw = warp - 2;
        const int q4 = warp & 3, hf = tw >> 2;
        const int row = q4 * 32 + lane;
        for (int r = 0; r < nraw; ++r) {
            const int rs = r % nr;
            mbar_wait(&raw_full[rs], (r / nr) & 1);
            if (tw == 0 && lane == 0 && r < 16) tl(p, 16 + r);
            const uint8_t* st = raw + rs * rstride;
            for (int h = 0; h < 2; ++h) {
                const int s = 2 * r + h, os = s % kOp;
                // x: 16 bf16 = two 16 B chunks (columns 32h + 16hf ..) of the row
                const int kx = 4 * h + 2 * hf;
                const uint4 x0 = *reinterpret_cast<const uint4*>(st + row * 128 + ((kx ^ (row & 7)) << 4));
                const uint4 x1 = *reinterpret_cast<const uint4*>(st + row * 128 + (((kx + 1) ^ (row & 7)) << 4));
                float g[16];
                {
                    const uint32_t xw[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        g[2 * i] = __uint_as_float(xw[i] << 16);
                        g[2 * i + 1] = __uint_as_float(xw[i] & 0xffff0000u);
                    }
                }
                if (p.has_noise) {  // noise half h: [128 rows][32 fp32], chunks 4hf .. 4hf+3
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const float4 nv = *reinterpret_cast<const float4*>(st + kRawX + h * (kRawN / 2) + swz(row, 4 * hf + i));
                        g[4 * i] *= nv.x; g[4 * i + 1] *= nv.y; g[4 * i + 2] *= nv.z; g[4 * i + 3] *= nv.w;
                    }
                }
                uint32_t hi[16], lo[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const float hv = (p.probe & 1) ? g[i] : tf32_rna(g[i]);
                    hi[i] = __float_as_uint(hv);
                    lo[i] = __float_as_uint((p.probe & 1) ? g[i] : tf32_rna(g[i] - hv));
                }
                if (s >= kOp) mbar_wait(&op_empty[os], ((s / kOp) - 1) & 1);
                tc_fence_after();
                const uint32_t ta = tmem + (static_cast<uint32_t>(q4 * 32) << 16) + kTmemA + os * 64 + 16 * hf;
                tmem_st16(ta, hi);
                tmem_st16(ta + 32, lo);
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&op_full[os]);
            }
            if (lane == 0) mbar_arrive(&raw_empty[rs]);
            if (tw == 0 && lane == 0 && r < 16) tl(p, 32 + r);
        }
    }
#else

        const int tw = warp - 2;  // rows [16 tw, 16 tw + 16)
        const int c = lane & 7;   // 4-element K chunk of the 32-element MMA step
        for (int r = 0; r < nraw; ++r) {
            const int rs = r % nr;
            mbar_wait(&raw_full[rs], (r / nr) & 1);
            if (tw == 0 && lane == 0 && r < 16) tl(p, 16 + r);
            const uint8_t* st = raw + rs * rstride;
            for (int h = 0; h < 2; ++h) {
                const int s = 2 * r + h, os = s % kOp;
                if (s >= kOp) mbar_wait(&op_empty[os], ((s / kOp) - 1) & 1);
                const uint32_t ahi = smem_u32(op + os * kOpStage);
                const uint32_t alo = ahi + BM * 128;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int row = tw * 16 + (lane >> 3) + 4 * j;
                    // x: 128 B rows, 16 B chunk (4h + c/2) swizzled with row % 8
                    const uint2 xv = *reinterpret_cast<const uint2*>(
                        st + row * 128 + ((((h << 2) + (c >> 1)) ^ (row & 7)) << 4) + ((c & 1) << 3));
                    float g[4] = {__uint_as_float(xv.x << 16), __uint_as_float(xv.x & 0xffff0000u),
                                  __uint_as_float(xv.y << 16), __uint_as_float(xv.y & 0xffff0000u)};
                    if (p.has_noise) {
                        const float4 nv = *reinterpret_cast<const float4*>(st + kRawX + h * (kRawN / 2) + swz(row, c));
                        g[0] *= nv.x; g[1] *= nv.y; g[2] *= nv.z; g[3] *= nv.w;
                    }
                    float hi[4], lo[4];
                    if (p.probe & 1) {
#pragma unroll
                        for (int q = 0; q < 4; ++q) hi[q] = lo[q] = g[q];
                    } else {
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            hi[q] = tf32_rna(g[q]);
                            lo[q] = tf32_rna(g[q] - hi[q]);
                        }
                    }
                    const uint32_t off = swz(row, c);
                    sts128(ahi + off, make_uint4(__float_as_uint(hi[0]), __float_as_uint(hi[1]),
                                                 __float_as_uint(hi[2]), __float_as_uint(hi[3])));
                    sts128(alo + off, make_uint4(__float_as_uint(lo[0]), __float_as_uint(lo[1]),
                                                 __float_as_uint(lo[2]), __float_as_uint(lo[3])));
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(&op_full[os]);
            }
            if (lane == 0) mbar_arrive(&raw_empty[rs]);
            if (tw == 0 && lane == 0 && r < 16) tl(p, 32 + r);
        }
    }
#endif

    // ---------------- epilogue
    float L[E];
    const bool epi = warp >= 2 && warp < 6;  // one epilogue warp per TMEM lane quarter
    const int q = warp & 3;                 // TMEM lane quarter of this warp
    const int row = q * 32 + lane;          // token row inside the cluster tile
    const bool mine = cs == 1 || (row >> 6) == static_cast<int>(rank);
    if (epi) {
        mbar_wait(acc_full, 0);
        tc_fence_after();
        if (warp == 2 && lane == 0) stamp(p, 2);
#pragma unroll
        for (int a = 0; a < kNAcc * kAccW; ++a) {
            if constexpr (E == 16) {
                uint32_t v[16];
                tmem_ld16(tmem + (static_cast<uint32_t>(q * 32) << 16) + a * E, v);
#pragma unroll
                for (int j = 0; j < 16; ++j) L[j] = a ? L[j] + __uint_as_float(v[j]) : __uint_as_float(v[j]);
            } else {
#pragma unroll
                for (int h = 0; h < E / 32; ++h) {
                    uint32_t v[32];
                    tmem_ld32(tmem + (static_cast<uint32_t>(q * 32) << 16) + a * E + h * 32, v);
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        L[h * 32 + j] = a ? L[h * 32 + j] + __uint_as_float(v[j]) : __uint_as_float(v[j]);
                }
            }
        }
        if (!mine) {  // the peer CTA owns this row: ship my half-d partial logits there
            const uint32_t dst = map_peer(smem_u32(recv + (row & 63) * E), rank ^ 1u);
#pragma unroll
            for (int j = 0; j < E; j += 4) st_cluster_v4(dst + 4 * j, L[j], L[j + 1], L[j + 2], L[j + 3]);
        }
    }
    __syncwarp();    // producer / MMA lanes rejoin their warps before the aligned cluster barrier
    if (warp == 2 && lane == 0) stamp(p, 3);
    cluster_sync();  // every partial has landed; both CTAs stay resident until here
    if (warp == 2 && lane == 0) stamp(p, 4);
    // owner warps: logits = own half + peer half, then the row's routing
    float* sP = reinterpret_cast<float*>(raw);               // [64 or 128][E + 1]: the raw ring is idle after the loop
    int32_t* sC = reinterpret_cast<int32_t*>(sP + 128 * (E + 1));
    const int64_t t = t0 + row;
    uint32_t flag = 0;
    if (epi && mine) {
        if (cs == 2) {
            const float* pr = recv + (row & 63) * E;
#pragma unroll
            for (int j = 0; j < E; ++j) L[j] += pr[j];
        }
        const int lr = cs == 1 ? row : (row & 63);
        if (t < p.T) {
#pragma unroll
            for (int j = 0; j < E; ++j)
                if (j >= ne) L[j] = -INFINITY;  // padded experts (E = 8 on the 16-column instance)
            float mx = L[0];
#pragma unroll
            for (int j = 1; j < E; ++j) mx = fmaxf(mx, L[j]);
            float s = 0.f;
#pragma unroll
            for (int j = 0; j < E; ++j) {
                L[j] = __expf(L[j] - mx);  // L now holds exp (ex2.approx: ~2 ulp)
                s += L[j];
            }
            const float sinv = 1.0f / s;
            float psum = 0.f;
            int c0 = 0;
            float b0 = 0.f;  // running best, in registers (no dynamic indexing of L)
#pragma unroll
            for (int j = 0; j < E; ++j) {
                const float pj = L[j] * sinv;
                if (!finite_f(pj)) flag |= MOE_FLAG_NONFINITE_DEV;
                L[j] = pj;
                psum += pj;
                if (j == 0 || pj > b0) {  // strict >, lowest index wins
                    b0 = pj;
                    c0 = j;
                }
            }
            if (fabsf(psum - 1.0f) > kProbRowTol) flag |= MOE_FLAG_PROB_ROWS_DEV;
            float4* po = reinterpret_cast<float4*>(p.probs + t * ne);
#pragma unroll
            for (int j = 0; j < E; j += 4)
                if (j < ne) po[j / 4] = make_float4(L[j], L[j + 1], L[j + 2], L[j + 3]);
            p.choice[t * p.K] = c0;
            p.gate_prob[t * p.K] = b0;
            if (p.K == 2) {  // second choice: initial candidate c0 == 0 ? 1 : 0 (routing.cpp:84-91)
                int c1 = c0 == 0 ? 1 : 0;
                float b1 = c0 == 0 ? L[1] : L[0];
#pragma unroll
                for (int j = 0; j < E; ++j)
                    if (j != c0 && L[j] > b1) {
                        b1 = L[j];
                        c1 = j;
                    }
                p.choice[t * p.K + 1] = c1;
                p.gate_prob[t * p.K + 1] = b1;
            }
#pragma unroll
            for (int j = 0; j < E; ++j) sP[lr * (E + 1) + j] = L[j];
            sC[lr] = c0;
        } else {
#pragma unroll
            for (int j = 0; j < E; ++j) sP[lr * (E + 1) + j] = 0.f;
            sC[lr] = -1;
        }
    }
    // the two owner warps of this CTA: column sums / first-choice counts of their 64 rows
    // (one CTA per tile: both pairs of epilogue warps, each over its 64 rows)
    const bool owner_warp = epi && (cs == 1 || (q >> 1) == static_cast<int>(rank));
    if (owner_warp) {
        const int half = cs == 1 ? (q >> 1) : 0;
        if (half == 0) asm volatile("bar.sync 1, 64;" ::: "memory");
        else asm volatile("bar.sync 2, 64;" ::: "memory");
        const int j = row & 63;  // expert
        const int rb = 64 * half;
        float cs4[4] = {0.f, 0.f, 0.f, 0.f};  // four interleaved partial sums, fixed order
        int cnt = 0;
        if (j < ne) {
#pragma unroll 4
            for (int r = 0; r < 64; ++r) {
                cs4[r & 3] += sP[(rb + r) * (E + 1) + j];
                cnt += sC[rb + r] == j;
            }
        }
        const float csum = (cs4[0] + cs4[1]) + (cs4[2] + cs4[3]);
        const int part = static_cast<int>((t0 >> 6) + (cs == 1 ? half : static_cast<int>(rank)));
        if (part < p.nparts && j < ne) {
            p.colsum_part[static_cast<int64_t>(part) * ne + j] = csum;
            p.count_part[static_cast<int64_t>(part) * ne + j] = cnt;
        }
        flag = __reduce_or_sync(0xffffffffu, flag);
        if (lane == 0 && flag) atomicOr(p.flags, flag);
        if (lane == 0) stamp(p, 5);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
    }
}

// Wg [d][ne] -> Wg^T split into tf32 hi / lo halves [EP][d] (the B operand),
// rows ne..EP-1 zero
__global__ void split_kernel(const float* __restrict__ wg, float* __restrict__ hi, float* __restrict__ lo, int d,
                             int ne, int EP) {
    pdl_wait();
    pdl_trigger();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= d * EP) return;
    const int j = i / EP, e = i % EP;
    const float v = e < ne ? wg[static_cast<int64_t>(j) * ne + e] : 0.f;
    const float h = tf32_rna(v);
    hi[static_cast<int64_t>(e) * d + j] = h;
    lo[static_cast<int64_t>(e) * d + j] = tf32_rna(v - h);
}

// the kernel instance (TMEM columns per accumulator) for ne experts
inline int padded_experts(int ne) { return ne <= 16 ? 16 : ne; }

}  // namespace gf

bool gate_fused_ok(int d, int E) {
    return (E == 8 || E == 16 || E == 32 || E == 64) && d % (2 * gf::BKR) == 0 && d >= 2 * gf::BKR;
}

size_t gate_split_floats(int d, int E) { return 2 * static_cast<size_t>(d) * gf::padded_experts(E); }

void launch_gate_split(const float* wg, float* wsplit, int d, int E, cudaStream_t st) {
    const int EP = gf::padded_experts(E);
    launch_pdl(gf::split_kernel, dim3(static_cast<unsigned>(ceil_div(static_cast<int64_t>(d) * EP, 256))), dim3(256),
               0, st, wg, wsplit, wsplit + static_cast<int64_t>(d) * EP, d, E, EP);
}

namespace {
bool gate_sm2_on() {  // MOE_B200_GATE_SM2=0: the eval E <= 16 gate on the one-CTA-per-SM instance
    static const bool on = [] {
        const char* e = std::getenv("MOE_B200_GATE_SM2");
        return !(e && e[0] == '0');
    }();
    return on;
}
}  // namespace

int gate_fused_parts(int64_t T) { return static_cast<int>(ceil_div(T, static_cast<int64_t>(64))); }

namespace {
template <int EP, bool SM2>
void launch_gate_fused_ep(const __nv_bfloat16* x, const float* noise, const float* wsplit, int64_t T, int d, int K,
                          int E, float* probs, int32_t* choice, float* gate_prob, float* colsum_part,
                          int32_t* count_part, uint32_t* flags, cudaStream_t st) {
    using namespace gf;
    constexpr uint32_t kSmem = GCfg<EP, SM2>::kSmem;
    static bool attr = false;
    if (!attr) {
        MOE_CUDA_CHECK(cudaFuncSetAttribute(gate_kernel<EP, SM2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(kSmem)));
        attr = true;
    }
    Params p{};
    p.tmX = tc::make_map_2d(x, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, T, d, BKR, BM, true);
    p.tmN = tc::make_map_2d(noise ? noise : wsplit, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, noise ? T : EP, d, BK,
                            noise ? BM : EP, true);
    p.tmBh = tc::make_map_2d(wsplit, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, EP, d, BK, EP, true);
    p.tmBl = tc::make_map_2d(wsplit + static_cast<int64_t>(d) * EP, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, EP, d, BK,
                             EP, true);
    p.probs = probs;
    p.choice = choice;
    p.gate_prob = gate_prob;
    p.colsum_part = colsum_part;
    p.count_part = count_part;
    p.flags = flags;
    p.T = T;
    p.d = d;
    p.K = K;
    p.ne = E;
    const unsigned tiles = static_cast<unsigned>(ceil_div(T, static_cast<int64_t>(BM)));
    // more tiles than one wave of CTA pairs: one CTA per tile takes all of d,
    // halving the per-CTA setup / pipeline fill / epilogue per byte
    // (SM2: two resident CTAs per SM, so pairs pay up to one tile per SM)
    p.csize = tiles > static_cast<unsigned>(SM2 ? kNumSMs : kNumSMs / 2) && d % BKR == 0 ? 1 : 2;
    p.nparts = gate_fused_parts(T);
    p.has_noise = noise != nullptr;
    static const int probe = [] {
        const char* e = std::getenv("MOE_B200_GATE_PROBE");
        return e ? std::atoi(e) : 0;
    }();
    p.probe = probe;
    static unsigned long long* stamps = nullptr;
    if ((probe & 24) && !stamps) MOE_CUDA_CHECK(cudaMalloc(&stamps, 8 * 8 * 4096));
    p.stamps = stamps;
    if (probe & 24) g_gate_stamps = stamps;
    cudaLaunchAttribute attrs[2];
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = static_cast<unsigned>(p.csize);
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[1].val.programmaticStreamSerializationAllowed = pdl_on() ? 1 : 0;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(p.csize) * tiles);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kSmem;
    cfg.stream = st;
    cfg.attrs = attrs;
    cfg.numAttrs = 2;
    MOE_CUDA_CHECK(cudaLaunchKernelEx(&cfg, gate_kernel<EP, SM2>, p));
    count_launch();
}
}  // namespace

void launch_gate_fused(const __nv_bfloat16* x, const float* noise, const float* wsplit, int64_t T, int d, int K,
                       int E, float* probs, int32_t* choice, float* gate_prob, float* colsum_part,
                       int32_t* count_part, uint32_t* flags, cudaStream_t st) {
    switch (gf::padded_experts(E)) {
        case 16:
            if (!noise && gate_sm2_on())
                launch_gate_fused_ep<16, true>(x, noise, wsplit, T, d, K, E, probs, choice, gate_prob, colsum_part,
                                               count_part, flags, st);
            else
                launch_gate_fused_ep<16, false>(x, noise, wsplit, T, d, K, E, probs, choice, gate_prob, colsum_part,
                                                count_part, flags, st);
            break;
        case 32: launch_gate_fused_ep<32, false>(x, noise, wsplit, T, d, K, E, probs, choice, gate_prob, colsum_part,
                                          count_part, flags, st); break;
        case 64: launch_gate_fused_ep<64, false>(x, noise, wsplit, T, d, K, E, probs, choice, gate_prob, colsum_part,
                                          count_part, flags, st); break;
        default: throw Status(6, "gate_fused: experts must be 8, 16, 32 or 64");
    }
}

// debug: copy the probe-8 phase timestamps of the last launch (ncta x 8 u64)
int gate_fused_stamps(unsigned long long* host, int ncta) {
    if (!g_gate_stamps) return 0;
    cudaDeviceSynchronize();
    cudaMemcpy(host, g_gate_stamps, sizeof(unsigned long long) * 8 * ncta, cudaMemcpyDeviceToHost);
    return ncta;
}

}  // namespace moe
