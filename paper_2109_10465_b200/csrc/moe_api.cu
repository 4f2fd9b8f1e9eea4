// moe_api.cu — host orchestration of the B200 MoE layer behind the C ABI in
// include/moe_b200.h.  Implements moe_layer_forward (routing.cpp:376-424),
// the explicit backward of the tape it builds, the per-stage operators
// (routing.hpp:60-118) and real expert parallelism over NCCL
// (simulate_expert_parallel_step, parallel.cpp:231-366, made physical).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <map>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/moe_b200.h"
#include "common.cuh"
#include "gemm_tc.h"
#include "kernels.h"
#include "rng_host.h"

using namespace moe;

namespace {

#define NCCL_CHECK(expr)                                                                   \
    do {                                                                                   \
        ncclResult_t _r = (expr);                                                          \
        if (_r != ncclSuccess)                                                             \
            throw Status(MOE_NCCL, std::string(#expr) + ": " + ncclGetErrorString(_r));    \
    } while (0)

// bytes allocated through DevMem by the handle being created / bound (for
// moe_workspace_bytes); handles are created one at a time per thread
thread_local size_t* g_ws_counter = nullptr;
struct DevMem {
    void* p = nullptr;
    size_t bytes = 0;
    void alloc(size_t b) {
        if (b == 0) b = 16;
        MOE_CUDA_CHECK(cudaMalloc(&p, b));
        bytes = b;
        if (g_ws_counter) *g_ws_counter += b;
    }
    ~DevMem() {
        if (p) cudaFree(p);
    }
    template <class T> T* as() const { return static_cast<T*>(p); }
};

int validate_cfg(const moe_router_cfg* c, std::string& why) {
    // routing.cpp:13-23
    if (c->num_experts < 1) { why = "router: num_experts must be >= 1"; return MOE_CONFIG; }
    if (c->capacity_factor_train <= 0.0 || c->capacity_factor_eval <= 0.0) {
        why = "router: capacity factors must be positive"; return MOE_CONFIG;
    }
    if (c->balance_coeff < 0.0) { why = "router: balance_coeff must be >= 0"; return MOE_CONFIG; }
    if (c->jitter_eps < 0.0) { why = "router: jitter_eps must be >= 0"; return MOE_CONFIG; }
    if (c->group_count < 1) { why = "router: group_count must be >= 1"; return MOE_CONFIG; }
    if (c->top_k != 1 && c->top_k != 2) { why = "router: top_k must be 1 or 2"; return MOE_CONFIG; }
    if (c->top_k > c->num_experts) { why = "router: top_k exceeds num_experts"; return MOE_CONFIG; }
    if (c->assignment_mode < 0 || c->assignment_mode > 2) { why = "make_assignment: unknown mode"; return MOE_CONFIG; }
    return MOE_OK;
}

int capacity_of(int64_t tokens, const moe_router_cfg* c, int phase) {
    // routing.cpp:43-49 — computed in double, independent of top_k
    const double cf = phase == MOE_TRAIN ? c->capacity_factor_train : c->capacity_factor_eval;
    const double v = cf * static_cast<double>(tokens) / static_cast<double>(c->num_experts);
    return std::max<int>(1, static_cast<int>(std::ceil(v)));
}

}  // namespace

namespace moe {
static std::atomic<uint64_t> g_launches{0};
uint64_t count_launch() { return g_launches.fetch_add(1, std::memory_order_relaxed) + 1; }
bool pdl_on() {
    static const bool on = [] {
        const char* e = std::getenv("MOE_B200_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}
}  // namespace moe

namespace {
// Per-stage CUDA-event timeline (SURVEY §5 "per-call stats": stage times).
struct Prof {
    bool on = false;
    std::vector<std::pair<const char*, cudaEvent_t>> marks;
    std::vector<cudaEvent_t> pool;
    std::map<std::string, std::pair<double, int64_t>> acc;
    std::vector<std::string> order;
    cudaEvent_t get() {
        if (!pool.empty()) {
            cudaEvent_t e = pool.back();
            pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        MOE_CUDA_CHECK(cudaEventCreate(&e));
        return e;
    }
    void mark(const char* name, cudaStream_t st) {
        if (!on) return;
        cudaEvent_t e = get();
        MOE_CUDA_CHECK(cudaEventRecord(e, st));
        marks.emplace_back(name, e);
    }
    void drain() {  // fold recorded marks into the accumulators
        if (marks.empty()) return;
        MOE_CUDA_CHECK(cudaEventSynchronize(marks.back().second));
        for (size_t i = 1; i < marks.size(); ++i) {
            const char* nm = marks[i].first;
            if (std::strcmp(nm, "begin") == 0) continue;
            float ms = 0.f;
            MOE_CUDA_CHECK(cudaEventElapsedTime(&ms, marks[i - 1].second, marks[i].second));
            auto it = acc.find(nm);
            if (it == acc.end()) {
                order.emplace_back(nm);
                acc[nm] = {ms, 1};
            } else {
                it->second.first += ms;
                it->second.second += 1;
            }
        }
        for (auto& m : marks) pool.push_back(m.second);
        marks.clear();
    }
    ~Prof() {
        for (auto& m : marks) cudaEventDestroy(m.second);
        for (auto e : pool) cudaEventDestroy(e);
    }
};
}  // namespace

struct moe_handle {
    Prof prof;
    void mark(const char* n) { prof.mark(n, stream); }
    moe_router_cfg cfg{};
    moe_layer_dims dims{};
    cudaStream_t stream = nullptr;
    std::string err;
    int E = 0, K = 0, El = 0, ep = 1, rank = 0;
    int64_t Tmax = 0, d = 0, f = 0;
    int cap_pad_max = 0;
    size_t esz = 4;  // activation element size
    ncclComm_t comm = nullptr;
    // side stream for backward work independent of the expert GEMMs, and a
    // comm stream for the dX all-to-all (owned by the handle)
    cudaStream_t side = nullptr, comm_stream = nullptr;
    cudaEvent_t ev_a = nullptr, ev_b = nullptr, ev_c = nullptr, ev_side = nullptr, ev_comm = nullptr;
    // NVLink peer map (CUDA IPC) of the receive buffers: [buffer][rank]
    enum { P_X = 0, P_O, P_DO, P_DX, P_CNT, P_FLAG, P_DWG, P_NBUF };
    bool ipc = false;
    void* peer[P_NBUF][8] = {};
    DevMem bar;       // 1-int NCCL all-reduce (barrier fallback, MOE_B200_EP_BARRIER=nccl)
    DevMem flags_ipc; // [8] u64 barrier flags, written by the peers over NVLink
    bool no_peer_epi = std::getenv("MOE_B200_PEER_EPI") && std::getenv("MOE_B200_PEER_EPI")[0] == '0';
    DevMem shape_all; // [ep + 1] i64: all-gathered per-rank token counts (NCCL transport)
    DevMem dwg_x;     // [d*E] fp32 staging of this rank's dWg for the fixed-order sum over ranks
    unsigned long long epoch = 0;
    bool nccl_barrier = false;
    bool defer_balance = false;
    bool gemm_tc = false;        // bf16 expert GEMMs on tcgen05 (decided at create)
    bool gate_fused = false;     // bf16 gate in one cluster kernel (gate_fused.cu)
    bool rcb_fused = true;       // single rank: combine backward folded into router_bwd
    bool rcb_ep = true;
    bool peer_dispatch = true;   // EP (IPC): the dispatch gather stores rows into the owners' buffers (MOE_B200_PEER_DISPATCH=0: copy pass)          // ... also under EP (MOE_B200_RCB_EP=0: two kernels, dO exchange next to router_bwd)
    // EP: gate dW + its all-reduce before the expert backward (MOE_B200_DW_EARLY=1).
    // Off by default: the all-reduce's barrier after the weight gradients is
    // the exchange point that orders this step's last read of Xr (dW1) before
    // the peers' dispatch stores of the next step; with it moved, the next
    // dispatch exchange first runs an extra barrier.
    bool dw_early = false;
    bool gate_dw_tma = false;    // dWg by the TMA-fed MN-major kernel (gate_bwd.cu)
    bool gate_dx_tma = false;    // dx by the persistent TMA-fed kernel (gate_bwd.cu)
    bool relu_bits_on = true;    // dgrad2 reads the ReLU mask as bits (MOE_B200_RELU_BITS=0: reads H)
    DevMem wsplit;               // [2][E][d] tf32 hi / lo halves of Wg^T
    size_t ws_bytes = 0;         // device bytes allocated by this handle  // forward under EP: the balance loss runs next to the dispatch exchange
    ~moe_handle() {
        for (int b = 0; b < P_NBUF; ++b)
            for (int r = 0; r < 8; ++r)
                if (ipc && r != rank && peer[b][r]) cudaIpcCloseMemHandle(peer[b][r]);
        for (cudaEvent_t e : {ev_a, ev_b, ev_c, ev_side, ev_comm, ev_pf, ev_rts, ev_bal})
            if (e) cudaEventDestroy(e);
        if (side) cudaStreamDestroy(side);
        if (comm_stream) cudaStreamDestroy(comm_stream);
        if (pf_stream) cudaStreamDestroy(pf_stream);
    }

    // workspace
    DevMem logits, probs, choice, gate_prob, wts, slot, pos, row_src, kept, counts_r;
    DevMem colsum_part, count_part, fcoef, fcount, aux_scratch, noise, ord, flags;
    DevMem hist, base, gkept;
    DevMem Xloc, Xr, H, Or, Oloc, dOloc, dOr, dH, dXr, dXloc;
    DevMem dL, dLr, dxg, dwg_part, wgt;
    DevMem hbits;                // ReLU mask of H as bits [R][f/64] (fwd1 epilogue -> dgrad2 epilogue)
    DevMem bal_term, bal_done;  // balance_finalize per-expert terms + CTA counter
    // jitter stream double buffer: `noise` is the current forward's stream;
    // `noise_pf` receives a stream generated ahead of use (moe_prefetch_jitter)
    DevMem noise_pf;
    bool pf_req = false, pf_valid = false;
    uint64_t pf_req_seed = 0, pf_seed = 0;
    int64_t pf_req_count = 0, pf_count = 0;
    cudaEvent_t ev_pf = nullptr, ev_rts = nullptr, ev_bal = nullptr;
    bool bal_pending = false;  // balance finalize on the side stream not yet joined
    cudaStream_t pf_stream = nullptr;  // the next forward's jitter generator (prefetch)
    int pf_sms = 0;                    // SMs it runs on (MOE_B200_PF_SMS; 0: 10 on one GPU, 18 under EP)
    bool pf_hold = false;              // keep them reserved through the dW2 GEMM
    int pf_reserve = 0;                // SMs the expert GEMMs leave to it right now
    int wmode = 0;                     // weight-gradient output mode of this backward (WgradGemmArgs::c_mode)
    // moe_backward_ex(MOE_GRAD_ACCUMULATE): the non-weight grads land here first
    DevMem acc_dx, acc_dres, acc_dgw, acc_db1, acc_db2;
    DevMem rts_scratch;         // rts.cu working set
    bool rts_host = false;      // MOE_B200_RTS_HOST=1: RTS order from the host
    DevMem db1_part;            // [rows/32][f] column sums from the dgrad2 epilogue
    // float64 path (dtype MOE_F64): logits, probabilities, gate_prob, weights,
    // noise, dL, dw [T*K], f_e [E]
    DevMem f_logits, f_probs, f_gp, f_w, f_noise, f_dL, f_dw, f_fval;
    AssignScratch as{};
    std::vector<uint32_t> host_ord;

    // forward context
    bool fwd_valid = false;
    int64_t T = 0;
    int cap = 0, dec_cap = 0, cap_pad = 0, phase = 0, mode = 0;
    bool jitter_on = false, has_residual = false;
    const void* x = nullptr;
    const float* gate_w = nullptr;
    const void* w1 = nullptr;
    const void* w2 = nullptr;
    double last_logical_traffic = 0.0, last_actual_sent = 0.0;

    void* loc(DevMem& a, DevMem& b) { return ep == 1 ? a.p : b.p; }
};

namespace {

template <class F>
moe_status guarded(moe_handle* h, F&& fn) {
    try {
        fn();
        if (h) h->err.clear();
        return MOE_OK;
    } catch (const Status& s) {
        if (h) h->err = s.what();
        return static_cast<moe_status>(s.code);
    } catch (const std::exception& e) {
        if (h) h->err = e.what();
        return MOE_CUDA;
    }
}

void require(bool ok, int code, const char* msg) {
    if (!ok) throw Status(code, msg);
}

ncclDataType_t nccl_type(size_t esz) { return esz == 2 ? ncclBfloat16 : ncclFloat32; }

// All-to-all of equal chunks: rank r sends chunk s of `send` to rank s and
// receives rank s's chunk r into chunk s of `recv` (parallel.cpp:294-307,
// fixed (sender, expert) order).
void all_to_all(moe_handle* h, const void* send, void* recv, size_t chunk_elems,
                ncclDataType_t ty, size_t esz) {
    // own chunk: device-local copy; peers: one NCCL group of send/recv pairs
    MOE_CUDA_CHECK(cudaMemcpyAsync(static_cast<char*>(recv) + h->rank * chunk_elems * esz,
                                   static_cast<const char*>(send) + h->rank * chunk_elems * esz,
                                   chunk_elems * esz, cudaMemcpyDeviceToDevice, h->stream));
    NCCL_CHECK(ncclGroupStart());
    for (int s = 0; s < h->ep; ++s) {
        if (s == h->rank) continue;
        NCCL_CHECK(ncclSend(static_cast<const char*>(send) + s * chunk_elems * esz, chunk_elems, ty,
                            s, h->comm, h->stream));
        NCCL_CHECK(ncclRecv(static_cast<char*>(recv) + s * chunk_elems * esz, chunk_elems, ty, s,
                            h->comm, h->stream));
    }
    NCCL_CHECK(ncclGroupEnd());
}

// Expert-parallel exchange over NVLink: this rank stores chunk s of `send`
// straight into chunk `rank` of peer s's receive buffer `buf` (IPC-mapped),
// then one 4-byte NCCL all-reduce acts as the barrier that makes every
// peer's stores visible before the receiver reads (stream order on each rank
// puts the stores before its all-reduce).  Write-after-read safety comes from
// the exchange points already between a buffer's last read and its next write
// (see DESIGN.md §7).  Falls back to NCCL send/recv when IPC is unavailable.
struct XSpec {
    const void* send;
    void* recv;
    int buf;
    size_t chunk_elems;
    ncclDataType_t ty;
    size_t esz;
};

void peer_barrier(moe_handle* h, const ShapeCheck* sc = nullptr);
// sc: also verify that every rank passed the same token count (the dispatch
// exchange; parallel.cpp:245-253), see ShapeCheck in kernels.h.
void exchange(moe_handle* h, std::initializer_list<XSpec> specs, bool local_only = false,
              const ShapeCheck* sc = nullptr) {
    if (!h->ipc) {
        NCCL_CHECK(ncclGroupStart());
        for (const XSpec& x : specs) all_to_all(h, x.send, x.recv, x.chunk_elems, x.ty, x.esz);
        NCCL_CHECK(ncclGroupEnd());
        if (sc) {
            long long* all = h->shape_all.as<long long>();
            launch_fill_i64(all + h->ep, sc->tokens, h->stream);
            NCCL_CHECK(ncclAllGather(all + h->ep, all, 1, ncclInt64, h->comm, h->stream));
            launch_ep_shape_check(all, h->ep, *sc, h->stream);
        }
        return;
    }
    PeerCopyJobs jobs{};
    jobs.n = 0;
    require(specs.size() * static_cast<size_t>(local_only ? 1 : h->ep) <= static_cast<size_t>(kMaxCopies),
            MOE_UNSUPPORTED, "exchange: too many peer copies for one launch");
    for (const XSpec& x : specs) {
        const size_t bytes = x.chunk_elems * x.esz;
        if (local_only) {  // publish this rank's buffer in its own exported slot, then barrier
            jobs.src[jobs.n] = x.send;
            jobs.dst[jobs.n] = x.recv;
            jobs.bytes[jobs.n] = static_cast<int64_t>(bytes);
            ++jobs.n;
            continue;
        }
        for (int s = 0; s < h->ep; ++s) {
            jobs.src[jobs.n] = static_cast<const char*>(x.send) + s * bytes;
            char* dst = s == h->rank ? static_cast<char*>(x.recv) : static_cast<char*>(h->peer[x.buf][s]);
            jobs.dst[jobs.n] = dst + h->rank * bytes;
            jobs.bytes[jobs.n] = static_cast<int64_t>(bytes);
            ++jobs.n;
        }
    }
    launch_peer_copy(jobs, h->stream);
    if (std::getenv("MOE_B200_PROFILE_BARRIER")) h->mark("xchg_copy");
    peer_barrier(h, sc);
}

// All ranks' stores into each other's receive buffers (peer copies or GEMM
// epilogues storing over NVLink) complete before any rank reads its own.
void peer_barrier(moe_handle* h, const ShapeCheck* sc) {
    if (h->nccl_barrier) {
        NCCL_CHECK(ncclAllReduce(h->bar.p, h->bar.p, 1, ncclInt32, ncclSum, h->comm, h->stream));
        if (sc) {
            long long* all = h->shape_all.as<long long>();
            launch_fill_i64(all + h->ep, sc->tokens, h->stream);
            NCCL_CHECK(ncclAllGather(all + h->ep, all, 1, ncclInt64, h->comm, h->stream));
            launch_ep_shape_check(all, h->ep, *sc, h->stream);
        }
    } else {
        PeerFlags pf{};
        for (int r = 0; r < h->ep; ++r) pf.f[r] = static_cast<unsigned long long*>(h->peer[moe_handle::P_FLAG][r]);
        launch_ipc_barrier(pf, h->flags_ipc.as<unsigned long long>(), h->rank, h->ep, ++h->epoch, h->stream, sc);
    }
}

// Bootstrap blob of one rank for the NVLink peer map: its dims (checked for
// agreement) and the CUDA-IPC handles of its receive buffers.
struct EpBlob {
    int64_t max_tokens, d, f;
    int32_t E, K, dtype, ep, rank, pad;
    cudaIpcMemHandle_t mem[moe_handle::P_NBUF];
};

// Export: allocate the flag / dWg staging buffers, zero the flags (before any
// peer can see them) and describe this rank's receive buffers.
void ipc_export(moe_handle* h, EpBlob* out) {
    if (!h->flags_ipc.p) {
        h->flags_ipc.alloc(8 * 16);
        h->dwg_x.alloc(4 * static_cast<size_t>(h->d) * h->E);
    }
    MOE_CUDA_CHECK(cudaMemset(h->flags_ipc.p, 0, 8 * 16));
    h->epoch = 0;
    void* bufs[moe_handle::P_NBUF] = {h->Xr.p,          h->Oloc.p,      h->dOr.p,    h->dXloc.p,
                                      h->counts_r.p,    h->flags_ipc.p, h->dwg_x.p};
    std::memset(out, 0, sizeof(EpBlob));
    out->max_tokens = h->Tmax;
    out->d = h->d;
    out->f = h->f;
    out->E = h->E;
    out->K = h->K;
    out->dtype = h->esz == 2 ? MOE_BF16 : MOE_F32;
    out->ep = h->ep;
    out->rank = h->rank;
    for (int b = 0; b < moe_handle::P_NBUF; ++b) MOE_CUDA_CHECK(cudaIpcGetMemHandle(&out->mem[b], bufs[b]));
    MOE_CUDA_CHECK(cudaDeviceSynchronize());
}

// Import: check that every rank built the same layer, then open the peers'
// receive buffers (rank order).  Ranks may share a device.
void ipc_import(moe_handle* h, const EpBlob* all) {
    for (int r = 0; r < h->ep; ++r) {
        const EpBlob& b = all[r];
        require(b.ep == h->ep && b.rank == r, MOE_CONFIG, "moe_ep_import: blobs must be all ranks in rank order");
        require(b.E == h->E && b.K == h->K && b.d == h->d && b.f == h->f && b.dtype == all[h->rank].dtype,
                MOE_CONFIG, "moe_ep_import: ranks built different layers");
        // parallel.cpp:245-253: the fixed-shape exchange needs the same token geometry everywhere
        require(b.max_tokens == h->Tmax, MOE_UNIFORM_SHAPE,
                "simulate: per-rank token counts must be identical (All-to-All requires the same "
                "tensor shape on every rank)");
    }
    void* bufs[moe_handle::P_NBUF] = {h->Xr.p,          h->Oloc.p,      h->dOr.p,    h->dXloc.p,
                                      h->counts_r.p,    h->flags_ipc.p, h->dwg_x.p};
    for (int r = 0; r < h->ep; ++r)
        for (int b = 0; b < moe_handle::P_NBUF; ++b) {
            if (r == h->rank) {
                h->peer[b][r] = bufs[b];
                continue;
            }
            MOE_CUDA_CHECK(cudaIpcOpenMemHandle(&h->peer[b][r], all[r].mem[b],
                                                cudaIpcMemLazyEnablePeerAccess));
        }
    h->ipc = true;
}

void ipc_setup(moe_handle* h) {
    // export the receive buffers, all-gather the blobs over NCCL, open peers'
    std::vector<EpBlob> all(static_cast<size_t>(h->ep));
    EpBlob mine;
    ipc_export(h, &mine);
    DevMem dev;
    dev.alloc(sizeof(EpBlob) * h->ep);
    char* base = static_cast<char*>(dev.p);
    MOE_CUDA_CHECK(cudaMemcpy(base + h->rank * sizeof(EpBlob), &mine, sizeof(EpBlob), cudaMemcpyHostToDevice));
    NCCL_CHECK(ncclAllGather(base + h->rank * sizeof(EpBlob), base, sizeof(EpBlob), ncclUint8, h->comm,
                             h->stream));
    MOE_CUDA_CHECK(cudaStreamSynchronize(h->stream));
    MOE_CUDA_CHECK(cudaMemcpy(all.data(), base, sizeof(EpBlob) * h->ep, cudaMemcpyDeviceToHost));
    ipc_import(h, all.data());
    const char* bt = std::getenv("MOE_B200_EP_BARRIER");
    h->nccl_barrier = bt && std::string(bt) == "nccl";
    MOE_CUDA_CHECK(cudaDeviceSynchronize());  // flags zeroed everywhere before first use
    NCCL_CHECK(ncclAllReduce(h->bar.p, h->bar.p, 1, ncclInt32, ncclSum, h->comm, h->stream));
    MOE_CUDA_CHECK(cudaStreamSynchronize(h->stream));
}

// Returns true iff the GEMM also produced the per-block column sums `colsum`.
template <class TIO>
bool row_gemm(moe_handle* h, const TIO* A, const TIO* W, TIO* C, const float* bias,
              const TIO* mask, const int32_t* counts, int64_t N, int64_t K, bool w_nmajor,
              int epi, int nseg_ep, float* colsum = nullptr, void* const* c_peer = nullptr,
              bool* peered = nullptr, uint64_t* relu_bits = nullptr) {
    RowGemmArgs a;
    a.A = A;
    a.W = W;
    a.C = C;
    a.bias = bias;
    a.mask = mask;
    a.counts = counts;
    a.N = N;
    a.K = K;
    a.ep = nseg_ep;
    a.El = h->El;
    a.cap_pad = h->cap_pad;
    a.w_nmajor = w_nmajor;
    a.epi = epi;
    a.colsum = colsum;
    a.sm_reserve = h->pf_reserve;
    a.relu_bits = relu_bits;
    if constexpr (std::is_same<TIO, __nv_bfloat16>::value) {
        if (tc_row_gemm_supported(a)) {
            a.c_peer = c_peer;
            if (peered) *peered = c_peer != nullptr;
            launch_row_gemm_tc(a, h->stream);
            return colsum != nullptr;
        }
    }
    launch_row_gemm_simt<TIO>(a, h->stream);
    return false;
}

template <class TIO>
void wgrad_gemm(moe_handle* h, const TIO* A, const TIO* B, void* C, int64_t M, int64_t N,
                const int32_t* counts, int nseg_ep) {
    WgradGemmArgs a;
    a.A = A;
    a.B = B;
    a.C = C;
    a.counts = counts;
    a.M = M;
    a.N = N;
    a.ep = nseg_ep;
    a.El = h->El;
    a.cap_pad = h->cap_pad;
    a.sm_reserve = h->pf_reserve;
    a.c_mode = h->wmode;
    if constexpr (std::is_same<TIO, __nv_bfloat16>::value) {
        if (tc_wgrad_gemm_supported(a)) {
            launch_wgrad_gemm_tc(a, h->stream);
            return;
        }
    }
    launch_wgrad_gemm_simt<TIO>(a, h->stream);
}

// Tensor-core gate GEMMs (gate_tc.cu) serve the bf16 path when the shape fits.
template <class TIO>
bool use_gate_tc(const moe_handle* h) {
    return std::is_same<TIO, __nv_bfloat16>::value && tc_enabled() &&
           gate_tc_ok(static_cast<int>(h->d), h->E);
}

// ---------------------------------------------------------------------------
// router: gate -> softmax/top-k -> balance loss -> assignment
// ---------------------------------------------------------------------------
void balance_finalize(moe_handle* h, int64_t T, float* aux);
template <class TIO>
void route(moe_handle* h, int64_t T, const TIO* x, const float* gate_w, int phase, uint64_t seed,
           float* aux) {
    const int E = h->E, K = h->K;
    cudaStream_t st = h->stream;
    const bool jitter = phase == MOE_TRAIN && h->cfg.jitter_eps > 0.0;
    const bool gtc = use_gate_tc<TIO>(h);
    // fused gate (gate_fused.cu): one cluster kernel for logits, softmax,
    // top-k and the balance loss; MOE_B200_GATE_FUSED=0 keeps the split kernels
    const bool fused = std::is_same<TIO, __nv_bfloat16>::value && h->gate_fused;
    if (fused) {
        // tf32 hi / lo halves of Wg^T for the fused gate's B operand: a 4 us kernel
        // on the main stream (PDL hands over to the gate; a side-stream launch
        // cost more in cross-stream wait than it overlapped)
        launch_gate_split(gate_w, h->wsplit.as<float>(), static_cast<int>(h->d), E, st);
    } else if (gtc) {  // Wg^T for the logits' B operand, on the side stream next to the jitter generator
        MOE_CUDA_CHECK(cudaEventRecord(h->ev_a, st));
        MOE_CUDA_CHECK(cudaStreamWaitEvent(h->side, h->ev_a, 0));
        launch_gate2_transpose(gate_w, h->wgt.as<float>(), static_cast<int>(h->d), E, h->side);
        MOE_CUDA_CHECK(cudaEventRecord(h->ev_b, h->side));
    }
    if (jitter) {
        // routing.cpp:62-70: noise stream Rng(derive_seed(seed, "jitter")), row-major
        // generated on the device by jump-ahead (rng.cu)
        const uint64_t js = derive_seed_tag(seed, "jitter");
        if (h->pf_valid && h->pf_seed == js && h->pf_count == T * h->d) {
            // generated ahead of use during the previous backward: swap it in
            MOE_CUDA_CHECK(cudaStreamWaitEvent(st, h->ev_pf, 0));
            std::swap(h->noise.p, h->noise_pf.p);
        } else {
            launch_jitter_noise_device(js, T * h->d, h->cfg.jitter_eps, h->noise.as<float>(), st);
        }
        h->pf_valid = false;
        h->mark("jitter_noise");
    }
    if (fused) {
        if constexpr (std::is_same<TIO, __nv_bfloat16>::value) {
            launch_gate_fused(x, jitter ? h->noise.as<float>() : nullptr, h->wsplit.as<float>(), T,
                              static_cast<int>(h->d), K, E, h->probs.as<float>(), h->choice.as<int32_t>(),
                              h->gate_prob.as<float>(), h->colsum_part.as<float>(), h->count_part.as<int32_t>(),
                              h->flags.as<uint32_t>(), st);
        }
        h->mark("gate_fused");
        // aux and f_e / T from the per-64-token partials, on the side stream (the
        // assignment and the expert GEMMs do not need them); forward_impl joins it
        MOE_CUDA_CHECK(cudaEventRecord(h->ev_a, st));
        MOE_CUDA_CHECK(cudaStreamWaitEvent(h->side, h->ev_a, 0));
        launch_balance_finalize(h->colsum_part.as<float>(), h->count_part.as<int32_t>(), gate_fused_parts(T), T, E,
                                h->cfg.balance_coeff, aux ? aux : h->aux_scratch.as<float>(), h->fcoef.as<float>(),
                                h->fcount.as<int32_t>(), h->bal_term.as<double>(), h->bal_done.as<unsigned>(),
                                h->side);
        MOE_CUDA_CHECK(cudaEventRecord(h->ev_bal, h->side));
        h->bal_pending = true;
        h->jitter_on = jitter;
        return;
    }
    // logits = (x * noise) @ gate_w  (routing.cpp:71)
    int nsplit = 1;
    if (gtc) {
        if constexpr (std::is_same<TIO, __nv_bfloat16>::value) {
            nsplit = gate_tc_logit_splits(T, static_cast<int>(h->d));
            MOE_CUDA_CHECK(cudaStreamWaitEvent(st, h->ev_b, 0));
            launch_gate_tc_logits<TIO>(x, jitter ? h->noise.as<float>() : nullptr, h->wgt.as<float>(),
                                       h->logits.as<float>(), T, static_cast<int>(h->d), E, nsplit, st);
        }
    } else if (gate2_ok(static_cast<int>(h->d), E)) {
        nsplit = gate2_logit_splits(T, static_cast<int>(h->d), E);
        launch_gate2_logits<TIO>(x, jitter ? h->noise.as<float>() : nullptr, gate_w,
                                 h->logits.as<float>(), T, static_cast<int>(h->d), E, nsplit, st);
    } else if (gate_fast_ok(static_cast<int>(h->d), E)) {
        nsplit = gate_logit_splits(T, static_cast<int>(h->d), E);
        launch_gate_logits<TIO>(x, jitter ? h->noise.as<float>() : nullptr, gate_w,
                                h->logits.as<float>(), T, static_cast<int>(h->d), E, nsplit, st);
    } else {
        launch_gemm_dense<TIO>(x, h->d, 1, jitter ? h->noise.as<float>() : nullptr, gate_w, E, 1,
                               h->logits.as<float>(), T, E, h->d, 1, st);
    }
    h->mark("gate_logits");
    launch_softmax_topk(h->logits.as<float>(), nsplit, T, E, K, h->probs.as<float>(),
                        h->choice.as<int32_t>(), h->gate_prob.as<float>(),
                        h->colsum_part.as<float>(), h->count_part.as<int32_t>(),
                        h->flags.as<uint32_t>(), st);
    h->mark("softmax_topk");
    if (!h->defer_balance) balance_finalize(h, T, aux);
    h->jitter_on = jitter;
}

// aux loss and the per-expert gradient coefficients (routing.cpp:348-374)
void balance_finalize(moe_handle* h, int64_t T, float* aux) {
    launch_balance_finalize(h->colsum_part.as<float>(), h->count_part.as<int32_t>(),
                            softmax_parts(T), T, h->E, h->cfg.balance_coeff,
                            aux ? aux : h->aux_scratch.as<float>(), h->fcoef.as<float>(),
                            h->fcount.as<int32_t>(), h->bal_term.as<double>(),
                            h->bal_done.as<unsigned>(), h->stream);
    h->mark("balance_loss");
}

// routing.cpp:180-187: the RTS priority order Rng(seed).permutation(T), built on
// the device (rts.cu) on stream `st`; MOE_B200_RTS_HOST=1 computes it on the host
void rts_order(moe_handle* h, int64_t T, uint64_t aseed, cudaStream_t st) {
    if (h->rts_host) {
        h->host_ord.resize(static_cast<size_t>(T));
        permutation(aseed, T, h->host_ord.data());
        MOE_CUDA_CHECK(cudaMemcpyAsync(h->ord.p, h->host_ord.data(), sizeof(uint32_t) * T,
                                       cudaMemcpyHostToDevice, st));
    } else {
        launch_rts_order(aseed, T, h->rts_scratch.p, h->ord.as<uint32_t>(), h->flags.as<uint32_t>(), st);
    }
}

void assign(moe_handle* h, int64_t T, const int32_t* choice, int cap, int mode, uint64_t aseed,
            int32_t* slot_out, bool ord_ready = false) {
    const uint32_t* ord = nullptr;
    if (mode == MOE_RTS) {
        if (!ord_ready) rts_order(h, T, aseed, h->stream);
        ord = h->ord.as<uint32_t>();
    }
    if (mode == MOE_GROUPED && T % h->cfg.group_count != 0)
        throw Status(MOE_CONFIG, "assign_grouped: group_count must divide the token count");
    launch_assign(T, h->E, h->K, cap, mode, h->cfg.group_count, choice, ord, h->cap_pad, h->as,
                  slot_out, h->pos.as<int32_t>(), h->row_src.as<int32_t>(),
                  h->kept.as<int32_t>(), h->flags.as<uint32_t>(), h->stream);
}

void set_geometry(moe_handle* h, int64_t T, int phase, int& mode) {
    h->cap = capacity_of(T, &h->cfg, phase);
    mode = phase == MOE_EVAL ? MOE_PLAIN : h->cfg.assignment_mode;  // routing.cpp:194-196
    const int G = h->cfg.group_count;
    h->dec_cap = mode == MOE_GROUPED ? G * ((h->cap + G - 1) / G) : h->cap;
    h->cap_pad = static_cast<int>(round_up(h->dec_cap, kRowAlign));
    if (h->cap_pad > h->cap_pad_max) throw Status(MOE_SHAPE, "capacity exceeds workspace");
}

// SMs of the jitter prefetch: 10 next to one GPU's HBM-bound expert GEMMs;
// 18 under EP, where the generator must finish inside a shorter window
// (forward + dgrad of a ~1.9 ms step; N=2 sweep: 12-14 SMs overrun it in some
// runs, 16-20 give 8.76-8.82M tokens/s vs 8.23M without prefetch, 24 costs
// the GEMMs more).  Its CTAs hold whole TPCs (rng.cu), so the cta_group::2
// GEMMs lose SM pairs, not single SMs.
int pf_sms_of(const moe_handle* h) { return h->pf_sms > 0 ? h->pf_sms : (h->ep > 1 ? 18 : 10); }

template <class TIO>
void forward_impl(moe_handle* h, int64_t T, const TIO* x, const float* gate_w, const TIO* w1,
                  const float* b1, const TIO* w2, const float* b2, int phase, uint64_t seed,
                  const TIO* residual, TIO* y, float* aux, int32_t* expert_id, int32_t* slot,
                  float* gate_prob) {
    require(T >= 1 && T <= h->Tmax, MOE_SHAPE, "moe_forward: token count outside [1, max_tokens]");
    require(x && gate_w && w1 && b1 && w2 && b2 && y, MOE_SHAPE, "moe_forward: null tensor");
    require(phase == MOE_TRAIN || phase == MOE_EVAL, MOE_CONFIG, "moe_forward: bad phase");
    cudaStream_t st = h->stream;
    const int E = h->E, K = h->K, El = h->El, ep = h->ep;
    int mode;
    set_geometry(h, T, phase, mode);
    h->fwd_valid = false;
    h->mark("begin");
    h->defer_balance = ep > 1;
    route<TIO>(h, T, x, gate_w, phase, seed, aux);
    h->defer_balance = false;
    if (mode == MOE_RTS) {  // the priority order on the side stream, next to the gate kernels
        MOE_CUDA_CHECK(cudaEventRecord(h->ev_a, st));
        MOE_CUDA_CHECK(cudaStreamWaitEvent(h->side, h->ev_a, 0));
        rts_order(h, T, derive_seed_tag(seed, "assign"), h->side);
        MOE_CUDA_CHECK(cudaEventRecord(h->ev_rts, h->side));
        MOE_CUDA_CHECK(cudaStreamWaitEvent(st, h->ev_rts, 0));
    }
    assign(h, T, h->choice.as<int32_t>(), h->cap, mode, derive_seed_tag(seed, "assign"),
           h->slot.as<int32_t>(), true);
    // Jitter stream of the NEXT forward (moe_prefetch_jitter): generated on its
    // own stream by pf_sms CTAs (one chunk of the stream per SM) while this
    // call's expert GEMMs (forward and dgrad) run on the other SMs, instead of
    // heading the next forward on all of them.  This forward's gate has
    // already consumed its own stream.
    h->pf_reserve = 0;
    if (h->pf_req) {
        MOE_CUDA_CHECK(cudaEventRecord(h->ev_a, st));
        MOE_CUDA_CHECK(cudaStreamWaitEvent(h->pf_stream, h->ev_a, 0));
        launch_jitter_noise_device(h->pf_req_seed, h->pf_req_count, h->cfg.jitter_eps, h->noise_pf.as<float>(),
                                   h->pf_stream, pf_sms_of(h));
        MOE_CUDA_CHECK(cudaEventRecord(h->ev_pf, h->pf_stream));
        h->pf_valid = true;
        h->pf_seed = h->pf_req_seed;
        h->pf_count = h->pf_req_count;
        h->pf_req = false;
        h->pf_reserve = pf_sms_of(h);
    }
    h->mark("assign");
    if (ep == 1) launch_combine_weights(T, E, K, h->gate_prob.as<float>(), h->wts.as<float>(), st);
    // dispatch (routing.cpp:396): un-jittered x into [E, cap_pad, d]
    TIO* Xloc = static_cast<TIO*>(h->loc(h->Xr, h->Xloc));
    // under EP with NVLink-mapped buffers the gather stores each row straight
    // into its expert owner's receive buffer (no local copy, no copy pass)
    // (not with MOE_B200_DW_EARLY=1: there the barrier that orders the previous
    // step's dW1 read of Xr before these stores comes only with the exchange)
    const bool peer_dispatch = ep > 1 && h->ipc && !h->no_peer_epi && h->peer_dispatch && !h->dw_early && ep <= 8;
    RowDst rd{};
    if (peer_dispatch) {
        rd.El = El;
        rd.ep = ep;
        const size_t slot = static_cast<size_t>(h->rank) * El * h->cap_pad * h->d * h->esz;
        for (int r = 0; r < ep; ++r)
            rd.p[r] = (r == h->rank ? static_cast<char*>(h->Xr.p) : static_cast<char*>(h->peer[moe_handle::P_X][r])) + slot;
    }
    launch_dispatch_gather<TIO>(x, h->d, E, K, h->cap_pad, h->row_src.as<int32_t>(),
                                h->kept.as<int32_t>(), Xloc, h->flags.as<uint32_t>(), st,
                                peer_dispatch ? &rd : nullptr);
    h->mark("dispatch");
    const int32_t* counts = h->kept.as<int32_t>();
    if (ep > 1) {
        // forward all-to-all: counts then rows (fixed-shape [E_local, cap_pad, d] slices), on
        // the comm stream while the balance loss and the combine weights compute
        MOE_CUDA_CHECK(cudaEventRecord(h->ev_c, st));
        MOE_CUDA_CHECK(cudaStreamWaitEvent(h->comm_stream, h->ev_c, 0));
        cudaStream_t saved = h->stream;
        h->stream = h->comm_stream;
        // the exchange also checks that every rank passed the same T (else
        // MOE_FLAG_UNIFORM_SHAPE and zero received counts)
        const ShapeCheck sc{static_cast<long long>(T), h->flags.as<uint32_t>(), h->counts_r.as<int32_t>(), E};
        // (dW1 of the previous step reads Xr after the last barrier when the
        // gate's all-reduce ran early: order it before the peers' stores)
        if (h->dw_early && h->ipc) peer_barrier(h);
        if (peer_dispatch)  // rows already stored: counts + the barrier (with the shape check)
            exchange(h, {{h->kept.p, h->counts_r.p, moe_handle::P_CNT, static_cast<size_t>(El), ncclInt32, 4}},
                     false, &sc);
        else
            exchange(h, {{h->kept.p, h->counts_r.p, moe_handle::P_CNT, static_cast<size_t>(El), ncclInt32, 4},
                         {Xloc, h->Xr.p, moe_handle::P_X, static_cast<size_t>(El) * h->cap_pad * h->d,
                          nccl_type(h->esz), h->esz}}, false, &sc);
        h->stream = saved;
        MOE_CUDA_CHECK(cudaEventRecord(h->ev_comm, h->comm_stream));
        if (!h->bal_pending) balance_finalize(h, T, aux);  // (the fused gate's runs on the side stream)
        launch_combine_weights(T, E, K, h->gate_prob.as<float>(), h->wts.as<float>(), st);
        MOE_CUDA_CHECK(cudaStreamWaitEvent(st, h->ev_comm, 0));
        counts = h->counts_r.as<int32_t>();
        const double slice = static_cast<double>(El) * h->cap * h->d;
        h->last_logical_traffic = 2.0 * slice * 8.0 * (ep - 1);
        h->last_actual_sent = 2.0 * static_cast<double>(El) * h->cap_pad * h->d * h->esz * (ep - 1);
        h->mark("a2a_dispatch");
    }
    // expert FFN on occupied rows only (routing.cpp:399-405)
    // (the ReLU mask also goes out as bits, which dgrad2 reads instead of H)
    row_gemm<TIO>(h, h->Xr.as<TIO>(), w1, h->H.as<TIO>(), b1, nullptr, counts, h->f, h->d, true,
                  EPI_BIAS_RELU, ep, nullptr, nullptr, nullptr, h->relu_bits_on ? h->hbits.as<uint64_t>() : nullptr);
    h->mark("ffn1_fwd");
    // under EP with NVLink-mapped buffers the fwd2 epilogue stores each origin
    // rank's rows straight into that rank's O receive buffer (no copy pass)
    void* opeer[8] = {};
    const bool want_peer = ep > 1 && h->ipc && !h->no_peer_epi;
    if (want_peer)
        for (int r = 0; r < ep; ++r)
            opeer[r] = static_cast<char*>(h->peer[moe_handle::P_O][r]) +
                       static_cast<size_t>(h->rank) * El * h->cap_pad * h->d * h->esz;
    bool peered = false;
    row_gemm<TIO>(h, h->H.as<TIO>(), w2, h->Or.as<TIO>(), b2, nullptr, counts, h->d, h->f, true,
                  EPI_BIAS, ep, nullptr, want_peer ? opeer : nullptr, &peered);
    h->mark("ffn2_fwd");
    TIO* Oloc = h->Or.as<TIO>();
    if (peered) {
        peer_barrier(h);
        Oloc = h->Oloc.as<TIO>();
        h->mark("a2a_combine");
    } else if (ep > 1) {
        exchange(h, {{h->Or.p, h->Oloc.p, moe_handle::P_O, static_cast<size_t>(El) * h->cap_pad * h->d,
                      nccl_type(h->esz), h->esz}});
        Oloc = h->Oloc.as<TIO>();
        h->mark("a2a_combine");
    }
    // combine (routing.cpp:421, 258-298)
    launch_combine<TIO>(Oloc, T, h->d, E, K, h->cap_pad, h->choice.as<int32_t>(),
                        h->pos.as<int32_t>(), h->wts.as<float>(), residual ? residual : x, y,
                        h->flags.as<uint32_t>(), st);
    h->mark("combine");
    if (h->bal_pending) {  // the balance loss (side stream) is part of this call's outputs
        MOE_CUDA_CHECK(cudaStreamWaitEvent(st, h->ev_bal, 0));
        h->bal_pending = false;
    }
    const size_t nk = static_cast<size_t>(T * K);
    if (expert_id)
        MOE_CUDA_CHECK(cudaMemcpyAsync(expert_id, h->choice.p, 4 * nk, cudaMemcpyDeviceToDevice, st));
    if (slot) MOE_CUDA_CHECK(cudaMemcpyAsync(slot, h->slot.p, 4 * nk, cudaMemcpyDeviceToDevice, st));
    if (gate_prob)
        MOE_CUDA_CHECK(cudaMemcpyAsync(gate_prob, h->gate_prob.p, 4 * nk, cudaMemcpyDeviceToDevice, st));
    h->T = T;
    h->phase = phase;
    h->mode = mode;
    h->has_residual = residual != nullptr;
    h->x = x;
    h->gate_w = gate_w;
    h->w1 = w1;
    h->w2 = w2;
    h->fwd_valid = true;
}

template <class TIO>
void backward_impl(moe_handle* h, const TIO* dy, float daux, TIO* dx, float* dgate_w, void* dw1,
                   float* db1, void* dw2, float* db2, TIO* dres) {
    require(h->fwd_valid, MOE_SHAPE, "moe_backward: no forward context on this handle");
    require(dy && dx && dgate_w && dw1 && db1 && dw2 && db2, MOE_SHAPE, "moe_backward: null tensor");
    require(!h->has_residual || dres, MOE_SHAPE, "moe_backward: dresidual required");
    cudaStream_t st = h->stream;
    const int64_t T = h->T, d = h->d, f = h->f;
    const int E = h->E, K = h->K, El = h->El, ep = h->ep;
    const TIO* x = static_cast<const TIO*>(h->x);
    const TIO* w1 = static_cast<const TIO*>(h->w1);
    const TIO* w2 = static_cast<const TIO*>(h->w2);
    const TIO* Oloc = ep > 1 ? h->Oloc.as<TIO>() : h->Or.as<TIO>();
    h->mark("begin");
    // combine backward: dO rows = w * dy[t]
    TIO* dOloc = static_cast<TIO*>(h->loc(h->dOr, h->dOloc));
    const bool rcb = (ep == 1 || h->rcb_ep) && h->rcb_fused && E <= 64;
    // the persistent dx kernel reads tf32-rounded dL (written next to dL by the router backward)
    const bool dx_tma = std::is_same<TIO, __nv_bfloat16>::value && use_gate_tc<TIO>(h) && h->gate_dx_tma;
    float* dLr = dx_tma ? h->dLr.as<float>() : nullptr;
    // under EP with NVLink-mapped buffers the fused kernel stores the dO rows
    // straight into the expert owners' dO buffers (the exchange is a barrier)
    const bool peer_do = rcb && ep > 1 && h->ipc && !h->no_peer_epi && h->peer_dispatch && ep <= 8;
    RowDst rdo{};
    if (peer_do) {
        rdo.El = El;
        rdo.ep = ep;
        const size_t slot = static_cast<size_t>(h->rank) * El * h->cap_pad * d * h->esz;
        for (int r = 0; r < ep; ++r)
            rdo.p[r] = (r == h->rank ? static_cast<char*>(h->dOr.p) : static_cast<char*>(h->peer[moe_handle::P_DO][r])) + slot;
    }
    if (rcb) {  // one pass over dy: dO rows and the routing / softmax backward -> dL
        launch_router_combine_bwd<TIO>(T, static_cast<int>(d), E, K, dy, Oloc, h->cap_pad,
                                       h->choice.as<int32_t>(), h->pos.as<int32_t>(),
                                       h->gate_prob.as<float>(), h->probs.as<float>(),
                                       h->fcoef.as<float>(), daux, h->wts.as<float>(),
                                       h->kept.as<int32_t>(), dOloc, h->dL.as<float>(), st, dLr,
                                       peer_do ? &rdo : nullptr);
        h->mark("combine_router_bwd");
    } else {
        launch_combine_bwd_gather<TIO>(dy, d, E, K, h->cap_pad, h->row_src.as<int32_t>(),
                                       h->kept.as<int32_t>(), h->wts.as<float>(), dOloc, st);
        h->mark("combine_bwd");
    }
    const int32_t* counts = h->kept.as<int32_t>();
    if (ep > 1) {  // dO to the expert owners on the comm stream, next to the router backward
        MOE_CUDA_CHECK(cudaEventRecord(h->ev_c, st));
        MOE_CUDA_CHECK(cudaStreamWaitEvent(h->comm_stream, h->ev_c, 0));
        cudaStream_t saved = h->stream;
        h->stream = h->comm_stream;
        if (peer_do)
            peer_barrier(h);  // every rank's dO rows have landed
        else
            exchange(h, {{dOloc, h->dOr.p, moe_handle::P_DO, static_cast<size_t>(El) * h->cap_pad * d,
                          nccl_type(h->esz), h->esz}});
        h->stream = saved;
        MOE_CUDA_CHECK(cudaEventRecord(h->ev_comm, h->comm_stream));
        counts = h->counts_r.as<int32_t>();
    }
    // routing weights / balance loss / softmax backward -> dL
    if (!rcb) {
        launch_router_bwd<TIO>(T, static_cast<int>(d), E, K, dy, Oloc, h->cap_pad,
                               h->choice.as<int32_t>(), h->pos.as<int32_t>(),
                               h->gate_prob.as<float>(), h->probs.as<float>(), h->fcoef.as<float>(),
                               daux, h->dL.as<float>(), st, dLr);
        h->mark("router_bwd");
    }
    if (ep > 1) {
        MOE_CUDA_CHECK(cudaStreamWaitEvent(st, h->ev_comm, 0));
        h->mark("a2a_dO");
    }
    const float* noise = h->jitter_on ? h->noise.as<float>() : nullptr;
    const bool fast = gate_fast_ok(static_cast<int>(d), E);
    const bool g2 = gate2_ok(static_cast<int>(d), E);
    cudaStream_t side = h->side;
    // gate dW (tensor cores: split-K + fixed-order reduce) and, under EP, its
    // sum over ranks on the comm stream (the gate is replicated)
    const bool gtc = use_gate_tc<TIO>(h);
    // one CTA per SM: (d/128 column tiles) x splits <= 148
    // (leaving the jitter prefetch's SMs alone while it may still run)
    const int tc_dw_splits = static_cast<int>(std::max<int64_t>(
        1, std::min<int64_t>({16, (kNumSMs - h->pf_reserve) / std::max<int64_t>(1, d / 128), (T + 31) / 32})));
    auto gate_dw = [&] {
        if constexpr (std::is_same<TIO, __nv_bfloat16>::value) {
            if (h->gate_dw_tma)
                launch_gate_dw_tma(x, noise, h->dL.as<float>(), h->dwg_part.as<float>(), T, static_cast<int>(d),
                                   tc_dw_splits, st);
            else
                launch_gate_tc_dw<TIO>(x, noise, h->dL.as<float>(), h->dwg_part.as<float>(), T,
                                       static_cast<int>(d), E, tc_dw_splits, st);
        }
        launch_splitk_reduce(h->dwg_part.as<float>(), tc_dw_splits, d * E, dgate_w, st);
        h->mark("gate_dw");
    };
    auto dwg_allreduce = [&] {
        MOE_CUDA_CHECK(cudaEventRecord(h->ev_c, st));
        MOE_CUDA_CHECK(cudaStreamWaitEvent(h->comm_stream, h->ev_c, 0));
        if (h->ipc) {  // stage, barrier, every rank sums all ranks' copies in rank order (deterministic)
            cudaStream_t saved = h->stream;
            h->stream = h->comm_stream;
            exchange(h, {{dgate_w, h->dwg_x.p, moe_handle::P_DWG, static_cast<size_t>(d * E), ncclFloat32, 4}},
                     /*local_only=*/true);
            h->stream = saved;
            const float* srcs[8] = {};
            for (int r = 0; r < ep; ++r) srcs[r] = static_cast<const float*>(h->peer[moe_handle::P_DWG][r]);
            launch_sum_ranks(srcs, ep, d * E, dgate_w, h->comm_stream);
        } else {
            NCCL_CHECK(ncclAllReduce(dgate_w, dgate_w, static_cast<size_t>(d * E), ncclFloat32, ncclSum,
                                     h->comm, h->comm_stream));
        }
        MOE_CUDA_CHECK(cudaEventRecord(h->ev_comm, h->comm_stream));
    };
    // EP: dW of the gate first, so its all-reduce overlaps the expert backward
    // instead of trailing the gate dx kernel (one GPU keeps it after the weight
    // gradients, where the jitter prefetch no longer holds SMs)
    const bool dw_early = gtc && ep > 1 && h->dw_early;
    if (dw_early) {
        gate_dw();
        dwg_allreduce();
    }
    // expert backward: dH = (dO W2^T) * [H > 0]; dX = dH W1^T; dW2 = H^T dO; dW1 = X^T dH
    // db1 = colsum(dH) comes out of the dgrad2 epilogue on the tensor-core path
    const bool db1_fused = row_gemm<TIO>(h, h->dOr.as<TIO>(), w2, h->dH.as<TIO>(), nullptr,
                                         h->H.as<TIO>(), counts, f, d, false, EPI_RELU_MASK, ep,
                                         h->db1_part.as<float>(), nullptr, nullptr,
                                         h->relu_bits_on ? h->hbits.as<uint64_t>() : nullptr);
    h->mark("ffn2_dgrad");
    if (db1_fused) launch_colsum_parts(h->db1_part.as<float>(), f, ep, El, h->cap_pad, counts, db1, st);
    // under EP with NVLink-mapped buffers the dgrad1 epilogue returns dX rows
    // straight into the origin ranks' dX buffers (no copy pass)
    void* xpeer[8] = {};
    const bool want_peer = ep > 1 && h->ipc && !h->no_peer_epi;
    if (want_peer)
        for (int r = 0; r < ep; ++r)
            xpeer[r] = static_cast<char*>(h->peer[moe_handle::P_DX][r]) +
                       static_cast<size_t>(h->rank) * El * h->cap_pad * d * h->esz;
    bool dx_peered = false;
    row_gemm<TIO>(h, h->dH.as<TIO>(), w1, h->dXr.as<TIO>(), nullptr, nullptr, counts, d, f, false,
                  EPI_NONE, ep, nullptr, want_peer ? xpeer : nullptr, &dx_peered);
    h->mark("ffn1_dgrad");
    TIO* dXloc = h->dXr.as<TIO>();
    if (ep > 1) {  // return dX to its origin ranks while the weight gradients compute
        MOE_CUDA_CHECK(cudaEventRecord(h->ev_c, st));
        MOE_CUDA_CHECK(cudaStreamWaitEvent(h->comm_stream, h->ev_c, 0));
        cudaStream_t saved = h->stream;
        h->stream = h->comm_stream;
        if (dx_peered)
            peer_barrier(h);
        else
            exchange(h, {{h->dXr.p, h->dXloc.p, moe_handle::P_DX, static_cast<size_t>(El) * h->cap_pad * d,
                          nccl_type(h->esz), h->esz}});
        h->stream = saved;
        MOE_CUDA_CHECK(cudaEventRecord(h->ev_comm, h->comm_stream));
        dXloc = h->dXloc.as<TIO>();
    }
    // Side stream, next to the weight-gradient GEMMs (persistent kernels that
    // leave ~40 KB of shared memory, most registers and the FMA pipes free;
    // the dgrad GEMMs before them fill shared memory, so nothing co-runs there):
    //   db2 = colsum(dO), db1 = colsum(dH) when not fused into the dgrad2
    //   epilogue, and on the FMA path dWg = (x*noise)^T dL and
    //   dxg = (dL Wg^T) * noise.  On the tensor-core path the gate GEMMs run on
    //   the main stream after the weight gradients (gate_tc.cu).
    MOE_CUDA_CHECK(cudaEventRecord(h->ev_a, st));
    MOE_CUDA_CHECK(cudaStreamWaitEvent(side, h->ev_a, 0));
    const int dw_splits = static_cast<int>(std::min<int64_t>(16, std::max<int64_t>(1, T / 512)));
    if (!gtc) {
        if (fast) {
            launch_gate_dw<TIO>(x, noise, h->dL.as<float>(), h->dwg_part.as<float>(), T,
                                static_cast<int>(d), E, dw_splits, side);
        } else {
            launch_gemm_dense<TIO>(x, 1, d, noise, h->dL.as<float>(), E, 1, h->dwg_part.as<float>(),
                                   d, E, T, dw_splits, side);
        }
        launch_splitk_reduce(h->dwg_part.as<float>(), dw_splits, d * E, dgate_w, side);
        if (g2) {
            launch_gate2_transpose(h->gate_w, h->wgt.as<float>(), static_cast<int>(d), E, side);
            launch_gate2_dxg(T, static_cast<int>(d), E, h->dL.as<float>(), h->wgt.as<float>(), noise,
                             h->dxg.as<float>(), side);
        }
    }
    if (dx_tma) launch_gate_round_wg(h->gate_w, h->wgt.as<float>(), static_cast<int>(d), E, side);
    launch_colsum_groups<TIO>(h->dOr.as<TIO>(), d, ep, El, h->cap_pad, counts, db2, side);
    if (!db1_fused) launch_colsum_groups<TIO>(h->dH.as<TIO>(), f, ep, El, h->cap_pad, counts, db1, side);
    MOE_CUDA_CHECK(cudaEventRecord(h->ev_side, side));
    // the prefetched jitter stream is done by now (measured), so the weight
    // gradients take every SM (MOE_B200_PF_HOLD=1 keeps the reserve for dW2 too)
    if (!h->pf_hold) h->pf_reserve = 0;
    wgrad_gemm<TIO>(h, h->H.as<TIO>(), h->dOr.as<TIO>(), dw2, f, d, counts, ep);
    h->mark("ffn2_wgrad");
    h->pf_reserve = 0;
    wgrad_gemm<TIO>(h, h->Xr.as<TIO>(), h->dH.as<TIO>(), dw1, d, f, counts, ep);
    h->mark("ffn1_wgrad");
    if (gtc && !dw_early) gate_dw();
    MOE_CUDA_CHECK(cudaStreamWaitEvent(st, h->ev_side, 0));
    if (ep > 1) MOE_CUDA_CHECK(cudaStreamWaitEvent(st, h->ev_comm, 0));
    h->mark("bwd_join");
    if (ep > 1 && !dw_early) dwg_allreduce();
    if (gtc) {  // dx = (dL Wg^T) * noise + dispatch bwd + residual, one tensor-core kernel
        if constexpr (std::is_same<TIO, __nv_bfloat16>::value) {
            if (dx_tma)
                launch_gate_dx_tma(T, static_cast<int>(d), K, h->cap_pad, dLr, h->wgt.as<float>(), noise, dXloc,
                                   h->choice.as<int32_t>(), h->pos.as<int32_t>(), dy, !h->has_residual, dx, dres, st);
            else
                launch_gate_tc_dx<TIO>(T, static_cast<int>(d), E, K, h->cap_pad, h->dL.as<float>(),
                                       h->gate_w, noise, dXloc, h->choice.as<int32_t>(),
                                       h->pos.as<int32_t>(), dy, !h->has_residual, dx, dres, st);
        }
    } else if (g2) {  // dx = dxg (side stream, noise applied) + dispatch bwd + residual
        launch_dx_assemble<TIO>(T, d, E, K, h->cap_pad, h->dxg.as<float>(), nullptr, dXloc,
                                h->choice.as<int32_t>(), h->pos.as<int32_t>(), dy,
                                !h->has_residual, dx, dres, st);
    } else if (fast) {  // same, 64x64 tiles
        launch_gate_dx<TIO>(T, static_cast<int>(d), E, K, h->cap_pad, h->dL.as<float>(), h->gate_w,
                            noise, dXloc, h->choice.as<int32_t>(), h->pos.as<int32_t>(), dy,
                            !h->has_residual, dx, dres, st);
    } else {
        launch_gemm_dense<float>(h->dL.as<float>(), E, 1, nullptr, h->gate_w, 1, E,
                                 h->dxg.as<float>(), T, d, E, 1, st);
        launch_dx_assemble<TIO>(T, d, E, K, h->cap_pad, h->dxg.as<float>(), noise, dXloc,
                                h->choice.as<int32_t>(), h->pos.as<int32_t>(), dy,
                                !h->has_residual, dx, dres, st);
    }
    h->mark("gate_dx");
    if (ep > 1) {
        MOE_CUDA_CHECK(cudaStreamWaitEvent(st, h->ev_comm, 0));
        h->mark("allreduce_dgate_w");
    }
}

// ---------------------------------------------------------------------------
// float64 path (f64_layer.cu): moe_layer_forward and its tape backward at the
// reference's precision, for f64 callers (the tape adapter)
// ---------------------------------------------------------------------------
void forward_f64(moe_handle* h, int64_t T, const double* x, const double* gate_w, const double* w1,
                 const double* b1, const double* w2, const double* b2, int phase, uint64_t seed,
                 const double* residual, double* y, double* aux, int32_t* expert_id, int32_t* slot,
                 double* gate_prob) {
    require(T >= 1 && T <= h->Tmax, MOE_SHAPE, "moe_forward: token count outside [1, max_tokens]");
    require(x && gate_w && w1 && b1 && w2 && b2 && y && aux, MOE_SHAPE, "moe_forward: null tensor");
    require(phase == MOE_TRAIN || phase == MOE_EVAL, MOE_CONFIG, "moe_forward: bad phase");
    cudaStream_t st = h->stream;
    const int E = h->E, K = h->K;
    const int d = static_cast<int>(h->d);
    int mode;
    set_geometry(h, T, phase, mode);
    h->fwd_valid = false;
    const bool jitter = phase == MOE_TRAIN && h->cfg.jitter_eps > 0.0;
    double* noise = jitter ? h->f_noise.as<double>() : nullptr;
    if (jitter) {  // routing.cpp:62-70: Rng(derive_seed(seed, "jitter")), row-major
        launch_mt64_raw_device(derive_seed_tag(seed, "jitter"), T * h->d, h->f_noise.as<uint64_t>(), st);
        launch_f64_noise(h->f_noise.as<uint64_t>(), T * h->d, 1.0 - h->cfg.jitter_eps, 1.0 + h->cfg.jitter_eps, st);
    }
    int32_t* choice = h->choice.as<int32_t>();
    launch_f64_gate(x, noise, gate_w, h->f_logits.as<double>(), h->f_probs.as<double>(), T, d, E, K, choice,
                    h->f_gp.as<double>(), h->flags.as<uint32_t>(), st);
    launch_f64_balance(h->f_probs.as<double>(), choice, T, E, K, h->cfg.balance_coeff, aux,
                       h->f_fval.as<double>(), st);
    assign(h, T, choice, h->cap, mode, derive_seed_tag(seed, "assign"), h->slot.as<int32_t>());
    launch_f64_weights(h->f_gp.as<double>(), T, E, K, h->f_w.as<double>(), st);
    launch_f64_dispatch(x, h->d, E, K, h->cap_pad, h->row_src.as<int32_t>(), h->kept.as<int32_t>(),
                        h->Xr.as<double>(), st);
    const int32_t* kept = h->kept.as<int32_t>();
    launch_f64_seg_gemm(h->Xr.as<double>(), w1, h->H.as<double>(), b1, nullptr, kept, E, h->cap_pad, h->d, h->f,
                        true, 2, st);
    launch_f64_seg_gemm(h->H.as<double>(), w2, h->Or.as<double>(), b2, nullptr, kept, E, h->cap_pad, h->f, h->d,
                        true, 1, st);
    launch_f64_combine(h->Or.as<double>(), residual ? residual : x, T, h->d, K, h->cap_pad, choice,
                       h->pos.as<int32_t>(), h->f_w.as<double>(), y, h->flags.as<uint32_t>(), st);
    const size_t nk = static_cast<size_t>(T * K);
    if (expert_id) MOE_CUDA_CHECK(cudaMemcpyAsync(expert_id, choice, 4 * nk, cudaMemcpyDeviceToDevice, st));
    if (slot) MOE_CUDA_CHECK(cudaMemcpyAsync(slot, h->slot.p, 4 * nk, cudaMemcpyDeviceToDevice, st));
    if (gate_prob) MOE_CUDA_CHECK(cudaMemcpyAsync(gate_prob, h->f_gp.p, 8 * nk, cudaMemcpyDeviceToDevice, st));
    h->T = T;
    h->phase = phase;
    h->mode = mode;
    h->has_residual = residual != nullptr;
    h->jitter_on = jitter;
    h->x = x;
    h->gate_w = reinterpret_cast<const float*>(gate_w);
    h->w1 = w1;
    h->w2 = w2;
    h->fwd_valid = true;
}

void backward_f64(moe_handle* h, const double* dy, double daux, double* dx, double* dgate_w, double* dw1,
                  double* db1, double* dw2, double* db2, double* dres, bool acc) {
    require(h->fwd_valid, MOE_SHAPE, "moe_backward: no forward context on this handle");
    require(dy && dx && dgate_w && dw1 && db1 && dw2 && db2, MOE_SHAPE, "moe_backward: null tensor");
    require(!h->has_residual || dres, MOE_SHAPE, "moe_backward: dresidual required");
    cudaStream_t st = h->stream;
    const int64_t T = h->T;
    const int E = h->E, K = h->K, d = static_cast<int>(h->d);
    const int64_t f = h->f;
    const double* x = static_cast<const double*>(h->x);
    const double* gw = reinterpret_cast<const double*>(h->gate_w);
    const double* w1 = static_cast<const double*>(h->w1);
    const double* w2 = static_cast<const double*>(h->w2);
    const double* noise = h->jitter_on ? h->f_noise.as<double>() : nullptr;
    const int32_t* choice = h->choice.as<int32_t>();
    const int32_t* pos = h->pos.as<int32_t>();
    const int32_t* kept = h->kept.as<int32_t>();
    const int cp = h->cap_pad;
    launch_f64_combine_bwd(dy, h->Or.as<double>(), T, d, K, cp, choice, pos, h->f_w.as<double>(),
                           h->dOr.as<double>(), h->f_dw.as<double>(), st);
    launch_f64_router_bwd(h->f_probs.as<double>(), h->f_gp.as<double>(), h->f_dw.as<double>(), choice,
                          h->f_fval.as<double>(), daux, T, E, K, h->f_dL.as<double>(), st);
    launch_f64_seg_gemm(h->dOr.as<double>(), w2, h->dH.as<double>(), nullptr, h->H.as<double>(), kept, E, cp, d,
                        f, false, 3, st);
    launch_f64_seg_gemm(h->dH.as<double>(), w1, h->dXr.as<double>(), nullptr, nullptr, kept, E, cp, f, d, false,
                        0, st);
    launch_f64_seg_wgrad(h->H.as<double>(), h->dOr.as<double>(), dw2, kept, E, cp, f, d, acc, st);
    launch_f64_seg_wgrad(h->Xr.as<double>(), h->dH.as<double>(), dw1, kept, E, cp, d, f, acc, st);
    launch_f64_seg_wgrad(nullptr, h->dOr.as<double>(), db2, kept, E, cp, 1, d, acc, st);
    launch_f64_seg_wgrad(nullptr, h->dH.as<double>(), db1, kept, E, cp, 1, f, acc, st);
    launch_f64_gate_dw(x, noise, h->f_dL.as<double>(), dgate_w, T, d, E, acc, st);
    launch_f64_dx(h->f_dL.as<double>(), gw, noise, h->dXr.as<double>(), dy, T, d, E, K, cp, choice, pos,
                  !h->has_residual, dx, dres, acc, st);
}

void alloc_workspace(moe_handle* h) {
    const int E = h->E, K = h->K;
    const int64_t T = h->Tmax, d = h->d, f = h->f;
    // largest capacity over both phases, grouped rounding included
    moe_router_cfg c = h->cfg;
    int capmax = std::max(capacity_of(T, &c, MOE_TRAIN), capacity_of(T, &c, MOE_EVAL));
    const int G = c.group_count;
    capmax = std::max(capmax, G * ((capmax + G - 1) / G));
    h->cap_pad_max = static_cast<int>(round_up(capmax, kRowAlign));
    const int64_t R = static_cast<int64_t>(E) * h->cap_pad_max;
    const size_t es = h->esz;
    h->logits.alloc(4 * T * E * kMaxGateSplits);  // split-K partials
    h->probs.alloc(4 * T * E);
    h->choice.alloc(4 * T * K);
    h->gate_prob.alloc(4 * T * K);
    h->wts.alloc(4 * T * K);
    h->slot.alloc(4 * T * K);
    h->pos.alloc(4 * T * K);
    h->row_src.alloc(4 * R);
    h->kept.alloc(4 * E);
    h->counts_r.alloc(4 * E);
    const int nparts = softmax_parts(T);
    h->colsum_part.alloc(4 * static_cast<size_t>(nparts) * E);
    h->count_part.alloc(4 * static_cast<size_t>(nparts) * E);
    h->fcoef.alloc(4 * E);
    h->fcount.alloc(4 * E);
    h->bal_term.alloc(8 * E);
    h->bal_done.alloc(16);
    MOE_CUDA_CHECK(cudaMemset(h->bal_done.p, 0, 16));
    h->aux_scratch.alloc(16);
    h->noise.alloc(4 * T * d);
    h->noise_pf.alloc(4 * T * d);
    h->ord.alloc(4 * T);
    h->rts_scratch.alloc(rts_scratch_bytes(T));
    {
        const char* r = std::getenv("MOE_B200_RTS_HOST");
        h->rts_host = r && r[0] == '1';
    }
    h->flags.alloc(16);
    MOE_CUDA_CHECK(cudaMemset(h->flags.p, 0, 16));
    const size_t sints = assign_scratch_ints(T, E, K, G);
    h->hist.alloc(4 * sints);
    h->base.alloc(4 * sints);
    h->gkept.alloc(4 * (2 * static_cast<size_t>(G) * E + 64));
    h->as.hist = h->hist.as<int32_t>();
    h->as.base = h->base.as<int32_t>();
    h->as.gkept = h->gkept.as<int32_t>();
    h->as.max_chunks = static_cast<int>(sints / (2 * static_cast<size_t>(K) * E));
    h->as.max_groups = G;
    h->Xr.alloc(es * R * d);
    h->H.alloc(es * R * f);
    h->hbits.alloc(static_cast<size_t>(R) * (f / 64 + 1) * 8);
    h->Or.alloc(es * R * d);
    h->dOr.alloc(es * R * d);
    h->dH.alloc(es * R * f);
    h->dXr.alloc(es * R * d);
    if (es == 2) h->db1_part.alloc(4 * static_cast<size_t>(R / 32 + 1) * f);
    if (h->ep > 1) {
        h->bar.alloc(16);
        MOE_CUDA_CHECK(cudaMemset(h->bar.p, 0, 16));
        h->shape_all.alloc(8 * (static_cast<size_t>(h->ep) + 1));
        h->Xloc.alloc(es * R * d);
        h->Oloc.alloc(es * R * d);
        h->dOloc.alloc(es * R * d);
        h->dXloc.alloc(es * R * d);
    }
    // buffers start finite (zero) so padded tensor-core tiles never see NaN garbage
    for (DevMem* m : {&h->Xr, &h->H, &h->Or, &h->dOr, &h->dH, &h->dXr})
        MOE_CUDA_CHECK(cudaMemset(m->p, 0, m->bytes));
    if (es == 8) {
        h->f_logits.alloc(8 * T * E);
        h->f_probs.alloc(8 * T * E);
        h->f_gp.alloc(8 * T * K);
        h->f_w.alloc(8 * T * K);
        h->f_noise.alloc(8 * T * d);
        h->f_dL.alloc(8 * T * E);
        h->f_dw.alloc(8 * T * K);
        h->f_fval.alloc(8 * E);
    }
    h->dL.alloc(4 * T * E);
    h->dLr.alloc(4 * T * E);
    h->dxg.alloc(4 * T * d);
    h->dwg_part.alloc(4 * 16 * d * E);
    h->wgt.alloc(4 * d * E);
    h->wsplit.alloc(4 * (gate_fused_ok(static_cast<int>(d), E) ? gate_split_floats(static_cast<int>(d), E) : 2 * d * E));
    {
        const char* g = std::getenv("MOE_B200_GATE_FUSED");
        h->gate_fused = es == 2 && gate_fused_ok(static_cast<int>(d), E) && !(g && g[0] == '0');
        const char* r = std::getenv("MOE_B200_RCB_FUSED");
        h->rcb_fused = !(r && r[0] == '0');
        const char* pdp = std::getenv("MOE_B200_PEER_DISPATCH");
        h->peer_dispatch = !(pdp && pdp[0] == '0');
        const char* re = std::getenv("MOE_B200_RCB_EP");
        h->rcb_ep = !(re && re[0] == '0');
        const char* de = std::getenv("MOE_B200_DW_EARLY");
        h->dw_early = de && de[0] == '1';
        const char* gd = std::getenv("MOE_B200_GATE_DW_TMA");
        h->gate_dw_tma = gate_dw_tma_ok(static_cast<int>(d), E) && !(gd && gd[0] == '0');
        const char* rb = std::getenv("MOE_B200_RELU_BITS");
        h->relu_bits_on = !(rb && rb[0] == '0');
        const char* gx = std::getenv("MOE_B200_GATE_DX_TMA");
        h->gate_dx_tma = gate_dx_tma_ok(static_cast<int>(d), E, K) && !(gx && gx[0] == '0');
    }
    MOE_CUDA_CHECK(cudaDeviceSynchronize());
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

int moe_abi_version(void) { return MOE_B200_ABI_VERSION; }

void moe_debug_set_tensor_cores(int enabled) { tc_set_enabled(enabled != 0); }

void moe_router_cfg_default(moe_router_cfg* c) {
    c->num_experts = 8;
    c->capacity_factor_train = 1.0;
    c->capacity_factor_eval = 2.0;
    c->jitter_eps = 0.01;
    c->balance_coeff = 0.01;
    c->assignment_mode = MOE_PLAIN;
    c->group_count = 1;
    c->top_k = 1;
    c->rng_seed = 0;
}

moe_status moe_router_cfg_validate(const moe_router_cfg* cfg) {
    std::string why;
    return static_cast<moe_status>(validate_cfg(cfg, why));
}

moe_status moe_capacity(int64_t tokens, const moe_router_cfg* cfg, int phase, int* cap_out) {
    if (tokens < 1) return MOE_CONFIG;  // routing.cpp:44
    std::string why;
    const int st = validate_cfg(cfg, why);
    if (st) return static_cast<moe_status>(st);
    *cap_out = capacity_of(tokens, cfg, phase);
    return MOE_OK;
}

uint64_t moe_derive_seed_tag(uint64_t seed, const char* tag) { return derive_seed_tag(seed, tag); }
uint64_t moe_derive_seed_u64(uint64_t seed, uint64_t salt) { return derive_seed_u64(seed, salt); }
moe_status moe_rng_permutation(uint64_t seed, int64_t n, uint32_t* out_host) {
    return guarded(nullptr, [&] {
        require(n >= 0 && (n == 0 || out_host), MOE_SHAPE, "permutation: output required");
        moe::permutation(seed, n, out_host);
    });
}
moe_status moe_convert_f64(const double* src, int64_t n, int dtype, void* dst, void* stream) {
    return guarded(nullptr, [&] {
        require(src && dst && n >= 0, MOE_SHAPE, "convert_f64: src and dst required");
        require(dtype == MOE_F32 || dtype == MOE_BF16, MOE_CONFIG, "convert_f64: dtype");
        launch_convert_f64(src, n, dtype == MOE_BF16, dst, static_cast<cudaStream_t>(stream));
    });
}

moe_status moe_create(const moe_router_cfg* cfg, const moe_layer_dims* dims, moe_handle** out) {
    if (!cfg || !dims || !out) return MOE_SHAPE;
    *out = nullptr;
    std::unique_ptr<moe_handle> h(new moe_handle());
    moe_status s = guarded(h.get(), [&] {
        std::string why;
        const int st = validate_cfg(cfg, why);
        if (st) throw Status(st, why);
        require(dims->max_tokens >= 1 && dims->d_model >= 1 && dims->d_ff >= 1, MOE_SHAPE,
                "moe_create: dims must be positive");
        require(dims->dtype == MOE_F32 || dims->dtype == MOE_BF16 || dims->dtype == MOE_F64, MOE_CONFIG,
                "moe_create: dtype");
        require(dims->dtype != MOE_F64 || std::max(1, dims->ep_size) == 1, MOE_UNSUPPORTED,
                "moe_create: the float64 path is single-rank");
        const int ep = std::max(1, dims->ep_size);
        require(cfg->num_experts % ep == 0, MOE_CONFIG,
                "simulate: expert_parallel must divide num_experts");
        require(ep == 1 || cfg->top_k == 1, MOE_CONFIG, "simulate: only top-1 routing is simulated");
        require(dims->ep_rank >= 0 && dims->ep_rank < ep, MOE_CONFIG, "moe_create: ep_rank");
        h->cfg = *cfg;
        h->dims = *dims;
        h->E = cfg->num_experts;
        h->K = cfg->top_k;
        h->ep = ep;
        h->rank = dims->ep_rank;
        h->El = h->E / ep;
        h->Tmax = dims->max_tokens;
        h->d = dims->d_model;
        h->f = dims->d_ff;
        h->esz = dims->dtype == MOE_BF16 ? 2 : dims->dtype == MOE_F64 ? 8 : 4;
        {
            struct Count {  // RAII: never leave the counter pointing at a failed handle
                explicit Count(size_t* c) { g_ws_counter = c; }
                ~Count() { g_ws_counter = nullptr; }
            } count(&h->ws_bytes);
            alloc_workspace(h.get());
        }
        if (h->esz == 2) {
            // The bf16 path's expert GEMMs run on tcgen05 when the shape tiles
            // (d, f multiples of 256); otherwise they run on the fp32-accumulating
            // SIMT kernels, ~20x slower.  That choice is explicit: logged once
            // here, reported by moe_gemm_path, and an error under MOE_B200_REQUIRE_TC=1.
            RowGemmArgs ra{};
            ra.N = h->f;
            ra.K = h->d;
            ra.ep = h->ep;
            ra.El = h->El;
            ra.cap_pad = kRowAlign;
            RowGemmArgs rb = ra;
            rb.N = h->d;
            rb.K = h->f;
            WgradGemmArgs wa{};
            wa.M = h->f;
            wa.N = h->d;
            wa.ep = h->ep;
            wa.El = h->El;
            wa.cap_pad = kRowAlign;
            WgradGemmArgs wb = wa;
            wb.M = h->d;
            wb.N = h->f;
            h->gemm_tc = tc_row_gemm_supported(ra) && tc_row_gemm_supported(rb) &&
                         tc_wgrad_gemm_supported(wa) && tc_wgrad_gemm_supported(wb);
            if (!h->gemm_tc) {
                const char* req = std::getenv("MOE_B200_REQUIRE_TC");
                if (req && req[0] == '1')
                    throw Status(MOE_UNSUPPORTED,
                                 "moe_create: bf16 expert GEMMs need d_model and d_ff multiples of 256 "
                                 "for tcgen05 (MOE_B200_REQUIRE_TC=1)");
                const char* q = std::getenv("MOE_B200_QUIET");
                if (!(q && q[0] == '1'))
                    std::fprintf(stderr,
                                 "[moe_b200] bf16 layer d_model=%lld d_ff=%lld: expert GEMMs use the SIMT "
                                 "kernels (tcgen05 tiles need multiples of 256)\n",
                                 static_cast<long long>(h->d), static_cast<long long>(h->f));
            }
        }
        MOE_CUDA_CHECK(cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking));
        MOE_CUDA_CHECK(cudaStreamCreateWithFlags(&h->comm_stream, cudaStreamNonBlocking));
        MOE_CUDA_CHECK(cudaStreamCreateWithFlags(&h->pf_stream, cudaStreamNonBlocking));
        if (const char* v = std::getenv("MOE_B200_PF_SMS")) h->pf_sms = std::max(1, std::min(64, std::atoi(v)));
        if (const char* v = std::getenv("MOE_B200_PF_HOLD")) h->pf_hold = v[0] == '1';
        for (cudaEvent_t* e : {&h->ev_a, &h->ev_b, &h->ev_c, &h->ev_side, &h->ev_comm, &h->ev_pf, &h->ev_rts,
                                &h->ev_bal})
            MOE_CUDA_CHECK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    });
    if (s == MOE_OK) *out = h.release();
    return s;
}

moe_status moe_destroy(moe_handle* h) {
    if (!h) return MOE_OK;
    if (h->comm) ncclCommDestroy(h->comm);
    delete h;
    return MOE_OK;
}

const char* moe_last_error(const moe_handle* h) { return h ? h->err.c_str() : ""; }

moe_status moe_set_stream(moe_handle* h, void* s) {
    if (!h) return MOE_SHAPE;
    h->stream = static_cast<cudaStream_t>(s);
    return MOE_OK;
}

moe_status moe_profile_enable(moe_handle* h, int on) {
    if (!h) return MOE_SHAPE;
    return guarded(h, [&] {
        h->prof.drain();
        h->prof.acc.clear();
        h->prof.order.clear();
        h->prof.on = on != 0;
    });
}

moe_status moe_profile_read(moe_handle* h, int max_stages, char* names, double* ms_total,
                            int64_t* calls, int* n_out) {
    if (!h) return MOE_SHAPE;
    return guarded(h, [&] {
        h->prof.drain();
        int n = 0;
        for (const std::string& nm : h->prof.order) {
            if (n >= max_stages) break;
            const auto& a = h->prof.acc[nm];
            std::strncpy(names + 32 * n, nm.c_str(), 31);
            names[32 * n + 31] = 0;
            ms_total[n] = a.first;
            calls[n] = a.second;
            ++n;
        }
        *n_out = n;
    });
}

uint64_t moe_kernel_launch_count(void) { return g_launches.load(); }

moe_status moe_check(moe_handle* h, uint32_t* flags_out) {
    if (!h) return MOE_SHAPE;
    uint32_t fl = 0;
    moe_status s = guarded(h, [&] {
        MOE_CUDA_CHECK(cudaStreamSynchronize(h->stream));
        MOE_CUDA_CHECK(cudaMemcpy(&fl, h->flags.p, 4, cudaMemcpyDeviceToHost));
        MOE_CUDA_CHECK(cudaMemset(h->flags.p, 0, 4));
        if (h->comm) {  // expert-parallel communicator: surface asynchronous NCCL failures
            ncclResult_t async = ncclSuccess;
            NCCL_CHECK(ncclCommGetAsyncError(h->comm, &async));
            if (async != ncclSuccess)
                throw Status(MOE_NCCL, std::string("NCCL asynchronous error: ") + ncclGetErrorString(async));
        }
    });
    if (flags_out) *flags_out = fl;
    if (s) return s;
    if (fl & MOE_FLAG_NONFINITE) {
        h->err = "non-finite value produced by the MoE layer";
        return MOE_NONFINITE;
    }
    if (fl & MOE_FLAG_CHOICE_RANGE) {
        h->err = "assignment: choice out of expert range";
        return MOE_CONFIG;
    }
    if (fl & MOE_FLAG_UNIFORM_SHAPE) {  // parallel.cpp:245-253
        h->err = "simulate: per-rank token counts must be identical (All-to-All requires the same "
                 "tensor shape on every rank)";
        return MOE_UNIFORM_SHAPE;
    }
    if (fl & MOE_FLAG_RTS_OVERFLOW_DEV) {
        h->err = "assign_rts: more rejected uniform_int draws than spare generator outputs";
        return MOE_CUDA;
    }
    if (fl & MOE_FLAG_PROB_ROWS) {
        h->err = "balance_loss: probs rows must sum to 1";
        return MOE_INVALID_ARG;
    }
    return MOE_OK;
}

moe_status moe_forward(moe_handle* h, int64_t T, const void* x, const float* gate_w,
                       const void* w1, const float* b1, const void* w2, const float* b2,
                       int phase, uint64_t seed, const void* residual, void* y, float* aux,
                       int32_t* expert_id, int32_t* slot, float* gate_prob) {
    if (!h) return MOE_SHAPE;
    return guarded(h, [&] {
        require(h->esz != 8, MOE_CONFIG, "moe_forward: float64 handle, use moe_forward_f64");
        if (h->esz == 2) {
            using B = __nv_bfloat16;
            forward_impl<B>(h, T, static_cast<const B*>(x), gate_w, static_cast<const B*>(w1), b1,
                            static_cast<const B*>(w2), b2, phase, seed,
                            static_cast<const B*>(residual), static_cast<B*>(y), aux, expert_id,
                            slot, gate_prob);
        } else {
            forward_impl<float>(h, T, static_cast<const float*>(x), gate_w,
                                static_cast<const float*>(w1), b1, static_cast<const float*>(w2),
                                b2, phase, seed, static_cast<const float*>(residual),
                                static_cast<float*>(y), aux, expert_id, slot, gate_prob);
        }
    });
}

moe_status moe_backward(moe_handle* h, const void* dy, float daux, void* dx, float* dgate_w,
                        void* dw1, float* db1, void* dw2, float* db2, void* dresidual) {
    return moe_backward_ex(h, dy, daux, dx, dgate_w, dw1, db1, dw2, db2, dresidual, 0u);
}

moe_status moe_backward_ex(moe_handle* h, const void* dy, float daux, void* dx, float* dgate_w, void* dw1,
                           float* db1, void* dw2, float* db2, void* dresidual, unsigned flags) {
    if (!h) return MOE_SHAPE;
    return guarded(h, [&] {
        require(h->esz != 8, MOE_CONFIG, "moe_backward: float64 handle, use moe_backward_f64");
        require((flags & ~(MOE_GRAD_ACCUMULATE | MOE_GRAD_WEIGHTS_F32)) == 0u, MOE_CONFIG,
                "moe_backward_ex: unknown flag");
        const bool acc = flags & MOE_GRAD_ACCUMULATE;
        // dW1 / dW2: written or accumulated by the weight-gradient GEMM epilogue itself,
        // in the activation dtype or (MOE_GRAD_WEIGHTS_F32) in fp32
        h->wmode = (acc ? 1 : 0) | ((flags & MOE_GRAD_WEIGHTS_F32) && h->esz == 2 ? 2 : 0);
        struct Reset {
            moe_handle* h;
            ~Reset() { h->wmode = 0; }
        } reset{h};
        void* udx = dx;
        void* ures = dresidual;
        float *udgw = dgate_w, *udb1 = db1, *udb2 = db2;
        const int64_t T = h->T, d = h->d, f = h->f, E = h->E, El = h->El;
        if (acc) {  // the other grads go to scratch, then dst += scratch (tensor.cpp:31-36 semantics)
            require(h->fwd_valid && dx && dgate_w && db1 && db2, MOE_SHAPE, "moe_backward: null tensor");
            auto need = [](DevMem& m, size_t b) {
                if (m.bytes < b) {
                    if (m.p) MOE_CUDA_CHECK(cudaFree(m.p));
                    m.p = nullptr;
                    m.alloc(b);
                }
            };
            need(h->acc_dx, h->esz * h->Tmax * d);
            need(h->acc_dgw, 4 * d * E);
            need(h->acc_db1, 4 * El * f);
            need(h->acc_db2, 4 * El * d);
            dx = h->acc_dx.p;
            dgate_w = h->acc_dgw.as<float>();
            db1 = h->acc_db1.as<float>();
            db2 = h->acc_db2.as<float>();
            if (dresidual) {
                need(h->acc_dres, h->esz * h->Tmax * d);
                dresidual = h->acc_dres.p;
            }
        }
        if (h->esz == 2) {
            using B = __nv_bfloat16;
            backward_impl<B>(h, static_cast<const B*>(dy), daux, static_cast<B*>(dx), dgate_w, dw1, db1, dw2, db2,
                             static_cast<B*>(dresidual));
        } else {
            backward_impl<float>(h, static_cast<const float*>(dy), daux, static_cast<float*>(dx), dgate_w, dw1,
                                 db1, dw2, db2, static_cast<float*>(dresidual));
        }
        if (acc) {
            const bool bf = h->esz == 2;
            launch_add_into(udx, dx, T * d, bf, h->stream);
            if (ures) launch_add_into(ures, dresidual, T * d, bf, h->stream);
            launch_add_into(udgw, dgate_w, d * E, false, h->stream);
            launch_add_into(udb1, db1, El * f, false, h->stream);
            launch_add_into(udb2, db2, El * d, false, h->stream);
        }
    });
}

moe_status moe_forward_f64(moe_handle* h, int64_t T, const double* x, const double* gate_w, const double* w1,
                           const double* b1, const double* w2, const double* b2, int phase, uint64_t seed,
                           const double* residual, double* y, double* aux, int32_t* expert_id, int32_t* slot,
                           double* gate_prob) {
    if (!h) return MOE_SHAPE;
    return guarded(h, [&] {
        require(h->esz == 8, MOE_CONFIG, "moe_forward_f64: handle was not created with MOE_F64");
        forward_f64(h, T, x, gate_w, w1, b1, w2, b2, phase, seed, residual, y, aux, expert_id, slot, gate_prob);
    });
}

moe_status moe_backward_f64(moe_handle* h, const double* dy, double daux, double* dx, double* dgate_w,
                            double* dw1, double* db1, double* dw2, double* db2, double* dresidual,
                            int accumulate) {
    if (!h) return MOE_SHAPE;
    return guarded(h, [&] {
        require(h->esz == 8, MOE_CONFIG, "moe_backward_f64: handle was not created with MOE_F64");
        backward_f64(h, dy, daux, dx, dgate_w, dw1, db1, dw2, db2, dresidual, accumulate != 0);
    });
}

moe_status moe_last_decision_stats(moe_handle* h, int* capacity, int64_t* drop_count,
                                   int64_t* kept_per_expert) {
    if (!h) return MOE_SHAPE;
    return guarded(h, [&] {
        require(h->fwd_valid, MOE_SHAPE, "no forward on this handle");
        std::vector<int32_t> kept(static_cast<size_t>(h->E));
        MOE_CUDA_CHECK(cudaStreamSynchronize(h->stream));
        MOE_CUDA_CHECK(cudaMemcpy(kept.data(), h->kept.p, 4 * h->E, cudaMemcpyDeviceToHost));
        int64_t total = 0;
        for (int e = 0; e < h->E; ++e) {
            total += kept[e];
            if (kept_per_expert) kept_per_expert[e] = kept[e];
        }
        if (capacity) *capacity = h->dec_cap;
        if (drop_count) *drop_count = h->T * h->K - total;
    });
}

moe_status moe_grad_sqnorm(const void* grad, int64_t n, int grad_dtype, double* acc_dev, void* stream) {
    return guarded(nullptr, [&] {
        require(grad && acc_dev && n >= 0, MOE_SHAPE, "grad_sqnorm: grad and acc required");
        require(grad_dtype == MOE_F32 || grad_dtype == MOE_BF16, MOE_CONFIG, "grad_sqnorm: dtype");
        launch_grad_sqnorm(grad, n, grad_dtype == MOE_BF16, acc_dev, static_cast<cudaStream_t>(stream));
    });
}
moe_status moe_clip_scale(const double* sq_dev, double clip_norm, double* scale_dev, void* stream) {
    return guarded(nullptr, [&] {
        require(sq_dev && scale_dev, MOE_SHAPE, "clip_scale: sq and scale required");
        launch_clip_scale(sq_dev, clip_norm, scale_dev, static_cast<cudaStream_t>(stream));
    });
}
moe_status moe_adam_update(float* theta, float* m, float* v, const void* grad, int64_t n,
                           int grad_dtype, void* theta_bf16, const double* scale_dev, double lr,
                           double beta1, double beta2, double eps, int64_t step, void* stream) {
    return guarded(nullptr, [&] {
        // optim.cpp:22-24
        require(lr > 0.0, MOE_CONFIG, "adam: learning rate must be positive");
        require(theta && m && v && grad && n >= 0 && step >= 1, MOE_SHAPE, "adam: bad arguments");
        require(grad_dtype == MOE_F32 || grad_dtype == MOE_BF16, MOE_CONFIG, "adam: grad dtype");
        launch_adam(theta, m, v, grad, n, grad_dtype == MOE_BF16, static_cast<__nv_bfloat16*>(theta_bf16),
                    scale_dev, lr, beta1, beta2, eps, step, static_cast<cudaStream_t>(stream));
    });
}

moe_status moe_prefetch_jitter(moe_handle* h, uint64_t seed, int64_t tokens) {
    if (!h) return MOE_SHAPE;
    return guarded(h, [&] {
        require(tokens >= 1 && tokens <= h->Tmax, MOE_SHAPE, "prefetch_jitter: tokens outside [1, max_tokens]");
        if (h->cfg.jitter_eps <= 0.0) return;  // no jitter stream in this configuration
        h->pf_req = true;
        h->pf_req_seed = derive_seed_tag(seed, "jitter");  // routing.cpp:386
        h->pf_req_count = tokens * h->d;
    });
}

moe_status moe_accumulate_decision_stats(moe_handle* h, int64_t* util_dev, int64_t* hist_dev) {
    if (!h) return MOE_SHAPE;
    return guarded(h, [&] {
        require(h->fwd_valid, MOE_SHAPE, "no forward on this handle");
        require(util_dev && hist_dev, MOE_SHAPE, "decision stats: util[E] and hist[10] required");
        launch_decision_stats(h->T, h->E, h->K, h->choice.as<int32_t>(), h->pos.as<int32_t>(), util_dev,
                              hist_dev, h->stream);
    });
}

moe_status moe_gate(moe_handle* h, int64_t T, const void* x, const float* gate_w, int phase,
                    uint64_t jitter_seed, float* probs, int32_t* choice, float* gate_prob) {
    if (!h) return MOE_SHAPE;
    return guarded(h, [&] {
        require(T >= 1 && T <= h->Tmax, MOE_SHAPE, "gate_forward: x [T,d] and gate_w [d,E] required");
        h->fwd_valid = false;  // the per-stage gate reuses the forward's noise / logits scratch
        cudaStream_t st = h->stream;
        const int E = h->E, K = h->K;
        const bool jitter = phase == MOE_TRAIN && h->cfg.jitter_eps > 0.0;
        if (jitter)
            launch_jitter_noise_device(jitter_seed, T * h->d, h->cfg.jitter_eps,
                                       h->noise.as<float>(), st);
        const float* nz = jitter ? h->noise.as<float>() : nullptr;
        if (h->esz == 2)
            launch_gemm_dense<__nv_bfloat16>(static_cast<const __nv_bfloat16*>(x), h->d, 1, nz,
                                             gate_w, E, 1, h->logits.as<float>(), T, E, h->d, 1, st);
        else
            launch_gemm_dense<float>(static_cast<const float*>(x), h->d, 1, nz, gate_w, E, 1,
                                     h->logits.as<float>(), T, E, h->d, 1, st);
        launch_softmax_topk(h->logits.as<float>(), 1, T, E, K, probs, choice, gate_prob,
                            h->colsum_part.as<float>(), h->count_part.as<int32_t>(),
                            h->flags.as<uint32_t>(), st);
    });
}

moe_status moe_assign_mode(moe_handle* h, int64_t T, const int32_t* choice, int cap, int mode,
                           int group_count, uint64_t rts_seed, int32_t* slot, int* capacity_host) {
    if (!h) return MOE_SHAPE;
    moe_status s = guarded(h, [&] {
        require(T >= 1 && T <= h->Tmax, MOE_SHAPE, "assign: token count");
        require(mode >= 0 && mode <= 2, MOE_CONFIG, "make_assignment: unknown mode");
        require(cap >= 1, MOE_CONFIG, "assign: capacity must be >= 1");
        if (mode == MOE_GROUPED)
            require(group_count >= 1 && T % group_count == 0, MOE_CONFIG,
                    "assign_grouped: group_count must divide the token count");
        const int G = mode == MOE_GROUPED ? group_count : 1;
        require(G <= h->as.max_groups || G == 1, MOE_CONFIG, "assign: group_count exceeds handle");
        const int dec_cap = mode == MOE_GROUPED ? G * ((cap + G - 1) / G) : cap;
        require(round_up(dec_cap, kRowAlign) <= h->cap_pad_max, MOE_SHAPE, "assign: capacity exceeds workspace");
        h->cap_pad = static_cast<int>(round_up(dec_cap, kRowAlign));
        moe_router_cfg saved = h->cfg;
        h->cfg.group_count = G;
        MOE_CUDA_CHECK(cudaMemsetAsync(slot, 0xff, 4 * static_cast<size_t>(T * h->K), h->stream));
        assign(h, T, choice, cap, mode, rts_seed, slot);
        h->cfg = saved;
        h->fwd_valid = false;
        if (capacity_host) *capacity_host = dec_cap;
    });
    if (s) return s;
    return moe_check(h, nullptr);
}

moe_status moe_assign(moe_handle* h, int64_t T, const int32_t* choice, int phase,
                      uint64_t assign_seed, int32_t* slot, int* capacity_host) {
    if (!h) return MOE_SHAPE;
    const int cap = capacity_of(T, &h->cfg, phase);
    const int mode = phase == MOE_EVAL ? MOE_PLAIN : h->cfg.assignment_mode;
    return moe_assign_mode(h, T, choice, cap, mode, h->cfg.group_count, assign_seed, slot,
                           capacity_host);
}

moe_status moe_dispatch(moe_handle* h, int64_t T, const void* x, const int32_t* expert_id,
                        const int32_t* slot, int capacity, void* buf, uint8_t* occupancy) {
    if (!h) return MOE_SHAPE;
    return guarded(h, [&] {
        if (h->esz == 2)
            launch_dispatch_ref<__nv_bfloat16>(static_cast<const __nv_bfloat16*>(x), T, h->d, h->E,
                                               h->K, capacity, expert_id, slot,
                                               static_cast<__nv_bfloat16*>(buf), occupancy, h->stream);
        else
            launch_dispatch_ref<float>(static_cast<const float*>(x), T, h->d, h->E, h->K, capacity,
                                       expert_id, slot, static_cast<float*>(buf), occupancy,
                                       h->stream);
    });
}

moe_status moe_combine(moe_handle* h, int64_t T, const void* expert_out, const int32_t* expert_id,
                       const int32_t* slot, int capacity, const void* residual,
                       const float* weights, void* y) {
    if (!h) return MOE_SHAPE;
    return guarded(h, [&] {
        if (h->esz == 2)
            launch_combine_ref<__nv_bfloat16>(static_cast<const __nv_bfloat16*>(expert_out), T, h->d,
                                              h->E, h->K, capacity, expert_id, slot, weights,
                                              static_cast<const __nv_bfloat16*>(residual),
                                              static_cast<__nv_bfloat16*>(y), h->stream);
        else
            launch_combine_ref<float>(static_cast<const float*>(expert_out), T, h->d, h->E, h->K,
                                      capacity, expert_id, slot, weights,
                                      static_cast<const float*>(residual), static_cast<float*>(y),
                                      h->stream);
    });
}

moe_status moe_balance_loss(moe_handle* h, int64_t T, const float* probs,
                            const int32_t* expert_id, double alpha, float* loss) {
    if (!h) return MOE_SHAPE;
    moe_status s = guarded(h, [&] {
        require(T >= 1 && T <= h->Tmax, MOE_SHAPE, "balance_loss: probs must be [T, E]");
        // reuse the softmax kernel's reductions: logits = log(probs) is not
        // needed; compute partials directly from probs via a dedicated pass
        launch_balance_from_probs(probs, T, h->E, h->K, expert_id, alpha, loss,
                                  h->colsum_part.as<float>(), h->count_part.as<int32_t>(),
                                  h->flags.as<uint32_t>(), h->bal_term.as<double>(),
                                  h->bal_done.as<unsigned>(), h->stream);
    });
    if (s) return s;
    return moe_check(h, nullptr);
}

size_t moe_ep_unique_id_size(void) { return sizeof(ncclUniqueId); }

moe_status moe_ep_get_unique_id(void* id_out) {
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return MOE_NCCL;
    std::memcpy(id_out, &id, sizeof(id));
    return MOE_OK;
}

moe_status moe_ep_init(moe_handle* h, const void* unique_id) {
    if (!h) return MOE_SHAPE;
    return guarded(h, [&] {
        require(h->ep > 1, MOE_CONFIG, "moe_ep_init: ep_size must be > 1");
        ncclUniqueId id;
        std::memcpy(&id, unique_id, sizeof(id));
        NCCL_CHECK(ncclCommInitRank(&h->comm, h->ep, id, h->rank));
        // NVLink peer map for the exchanges (single node, <= 8 ranks, 16-byte
        // aligned count chunks); MOE_B200_EP_TRANSPORT=nccl keeps NCCL send/recv.
        const char* tr = std::getenv("MOE_B200_EP_TRANSPORT");
        const bool want_ipc = !(tr && std::string(tr) == "nccl");
        if (want_ipc && h->ep <= 8 && (h->El * 4) % 16 == 0) ipc_setup(h);
    });
}

moe_status moe_workspace_bytes(const moe_handle* h, size_t* bytes_out) {
    if (!h || !bytes_out) return MOE_SHAPE;
    *bytes_out = h->ws_bytes;
    return MOE_OK;
}

moe_status moe_gemm_path(const moe_handle* h, int* path_out) {
    if (!h || !path_out) return MOE_SHAPE;
    *path_out = h->esz == 2 && h->gemm_tc && tc_enabled() ? MOE_GEMM_TCGEN05 : MOE_GEMM_SIMT;
    return MOE_OK;
}

size_t moe_ep_blob_size(void) { return sizeof(EpBlob); }

moe_status moe_ep_export(moe_handle* h, void* blob_out) {
    if (!h) return MOE_SHAPE;
    return guarded(h, [&] {
        require(h->ep > 1, MOE_CONFIG, "moe_ep_export: ep_size must be > 1");
        require(blob_out, MOE_SHAPE, "moe_ep_export: blob required");
        require(h->ep <= 8 && (h->El * 4) % 16 == 0, MOE_UNSUPPORTED,
                "moe_ep_export: the NVLink peer map needs ep <= 8 and experts per rank % 4 == 0");
        require(!h->ipc && !h->comm, MOE_CONFIG, "moe_ep_export: handle already bound");
        ipc_export(h, static_cast<EpBlob*>(blob_out));
    });
}

moe_status moe_ep_import(moe_handle* h, const void* all_blobs) {
    if (!h) return MOE_SHAPE;
    return guarded(h, [&] {
        require(h->flags_ipc.p && !h->ipc, MOE_CONFIG, "moe_ep_import: call moe_ep_export first");
        require(all_blobs, MOE_SHAPE, "moe_ep_import: blobs required");
        ipc_import(h, static_cast<const EpBlob*>(all_blobs));
    });
}

moe_status moe_ep_traffic(moe_handle* h, double* logical_bytes_host, double* actual_bytes_sent) {
    if (!h) return MOE_SHAPE;
    return guarded(h, [&] {
        // A2ATrafficLog (parallel.hpp:83-91): fixed-shape f64 bytes per
        // direction pair = forward slice + reverse slice of [E/ep, cap, d].
        if (logical_bytes_host) {
            const double pair = 2.0 * h->El * static_cast<double>(h->cap) * h->d * 8.0;
            for (int i = 0; i < h->ep; ++i)
                for (int j = 0; j < h->ep; ++j) logical_bytes_host[i * h->ep + j] = i == j ? 0.0 : pair;
        }
        if (actual_bytes_sent) *actual_bytes_sent = h->last_actual_sent;
    });
}

}  // extern "C"

// ---- debug entry points for the device mt19937_64 generator (tests) ------
namespace moe {
void host_mt64_chunk(uint64_t seed, int64_t J, int P, int c, int64_t n, uint64_t* out);
void launch_mt64_raw_device(uint64_t seed, int64_t count, uint64_t* out, cudaStream_t st);
}  // namespace moe

extern "C" {
moe_status moe_debug_mt64_chunk_host(uint64_t seed, int64_t J, int c, int64_t n, uint64_t* out) {
    return guarded(nullptr, [&] { moe::host_mt64_chunk(seed, J, 1, c, n, out); });
}
moe_status moe_debug_mt64_device(uint64_t seed, int64_t count, uint64_t* out_dev) {
    return guarded(nullptr, [&] {
        moe::launch_mt64_raw_device(seed, count, out_dev, nullptr);
        MOE_CUDA_CHECK(cudaDeviceSynchronize());
    });
}
moe_status moe_debug_gate_tc_logits(const void* x, const float* noise, const float* gate_w,
                                    float* logits_part, int64_t T, int d, int E, int splits) {
    return guarded(nullptr, [&] {
        require(moe::gate_tc_ok(d, E), MOE_SHAPE, "gate_tc: unsupported shape");
        float* wgt = nullptr;
        MOE_CUDA_CHECK(cudaMalloc(&wgt, sizeof(float) * static_cast<size_t>(d) * E));
        moe::launch_gate2_transpose(gate_w, wgt, d, E, nullptr);
        moe::launch_gate_tc_logits<__nv_bfloat16>(static_cast<const __nv_bfloat16*>(x), noise, wgt,
                                                  logits_part, T, d, E, splits, nullptr);
        MOE_CUDA_CHECK(cudaDeviceSynchronize());
        MOE_CUDA_CHECK(cudaFree(wgt));
        MOE_CUDA_CHECK(cudaDeviceSynchronize());
    });
}
moe_status moe_debug_gate_tc_dw(const void* x, const float* noise, const float* dL, float* dw_part,
                                int64_t T, int d, int E, int splits) {
    return guarded(nullptr, [&] {
        require(moe::gate_tc_ok(d, E), MOE_SHAPE, "gate_tc: unsupported shape");
        moe::launch_gate_tc_dw<__nv_bfloat16>(static_cast<const __nv_bfloat16*>(x), noise, dL, dw_part, T,
                                              d, E, splits, nullptr);
        MOE_CUDA_CHECK(cudaDeviceSynchronize());
    });
}
moe_status moe_debug_gate_tc_dx(int64_t T, int d, int E, int K, int cap_pad, const float* dL,
                                const float* gate_w, const float* noise, const void* dX,
                                const int32_t* choice, const int32_t* pos, const void* dy,
                                int residual_is_x, void* dx, void* dres) {
    using B = __nv_bfloat16;
    return guarded(nullptr, [&] {
        require(moe::gate_tc_ok(d, E), MOE_SHAPE, "gate_tc: unsupported shape");
        moe::launch_gate_tc_dx<B>(T, d, E, K, cap_pad, dL, gate_w, noise, static_cast<const B*>(dX), choice,
                                  pos, static_cast<const B*>(dy), residual_is_x != 0, static_cast<B*>(dx),
                                  static_cast<B*>(dres), nullptr);
        MOE_CUDA_CHECK(cudaDeviceSynchronize());
    });
}
moe_status moe_debug_gate_stamps(uint64_t* host, int ncta, int* n_out) {
    *n_out = moe::gate_fused_stamps(reinterpret_cast<unsigned long long*>(host), ncta);
    return MOE_OK;
}
moe_status moe_debug_rts_order(uint64_t seed, int64_t n, uint32_t* perm_dev) {
    return guarded(nullptr, [&] {
        void* scratch = nullptr;
        MOE_CUDA_CHECK(cudaMalloc(&scratch, moe::rts_scratch_bytes(n)));
        moe::launch_rts_order(seed, n, scratch, perm_dev, nullptr, nullptr);
        MOE_CUDA_CHECK(cudaDeviceSynchronize());
        MOE_CUDA_CHECK(cudaFree(scratch));
    });
}
moe_status moe_debug_jitter_device(uint64_t seed, int64_t count, double eps, float* out_dev) {
    return guarded(nullptr, [&] {
        moe::launch_jitter_noise_device(seed, count, eps, out_dev, nullptr);
        MOE_CUDA_CHECK(cudaDeviceSynchronize());
    });
}
}
