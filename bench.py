"""bench.py — MoE-layer fwd+bwd tokens/s on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[2], the 64-expert top-1 config the target is
quoted on): E=64 experts sharded E/N per GPU, d_model=2048, d_ff=8192, top-1,
capacity factor 1.0, plain assignment, train phase (jitter eps=0.01,
balance alpha=0.01), bf16 activations/weights with fp32 accumulation,
T=8192 tokens per GPU (64k global at N=8, weak scaling).

One step = moe_forward + moe_backward of loss = <dy, y> + aux (all expert
grads, gate grad, dx) through the C ABI.  `value` is device-timed with inputs
resident in HBM; `e2e` times the same step through the public API with the
step's inputs (x, dy) copied from pinned host memory and the step's loss (the
aux loss; `--e2e-readback dx` also reads dx) read back.

  python bench.py [--gpus N --steps K --warmup W]            # our kernels
  python bench.py --impl reference [...]                      # reference CPU path
Multi-GPU: python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOAD = dict(name="c3_ep_64e_top1", experts=64, d_model=2048, d_ff=8192, top_k=1,
                capacity_factor=1.0, tokens_per_gpu=8192, assignment="plain", jitter_eps=0.01,
                balance_coeff=0.01)
METRIC = "MoE layer fwd+bwd tokens/sec"
UNIT = "tokens/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], p.get("bf16_tflops_sustained", p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampled every 50 ms from before warm-up to after the timed
    loops; samples are tagged with host time so the timed window can be cut
    out (falls back to the whole busy period if the window is shorter than
    the sampling interval)."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self):
        self.rows = []
        self.proc = None
        self.windows = []

    def start(self, ngpus: int = 1):
        try:
            ids = ",".join(str(i) for i in range(ngpus))  # the GPUs this job runs on
            self.proc = subprocess.Popen(["nvidia-smi", "-i", ids, f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.time(), [c.strip() for c in line.split(",")]))

    def mark(self, t0, t1):
        self.windows.append((t0, t1))

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = [r for r in self.rows if len(r[1]) >= 9 and r[1][1].replace(".", "").isdigit()]
        inside = [r for r in rows if any(a - 0.06 <= r[0] <= b + 0.06 for a, b in self.windows)]
        use = inside if len(inside) >= 2 else rows
        sm = sorted(float(r[1][1]) for r in use)
        mx = [float(r[1][2]) for r in use]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for _, r in use:
            for i, n in enumerate(names):
                if r[5 + i].lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(use),
                "window": "timed region" if use is inside else "whole run (timed region shorter than sampling)"}


# ---------------------------------------------------------------- CPU reference
def reference_sample_inputs(seed=42):
    """Bounded sample of the workload for the reference CPU path: one expert's
    worth of config 3 — d=2048, f=8192, capacity 128 (128 tokens, E'=1, C=1.0)
    — i.e. the same per-token work (every capacity row of every expert,
    routing.cpp:399-405) and the same tokens-per-expert as the full config, so
    its tokens/s equals the full config's (the gate is <1.5% of time)."""
    import oracle as O
    T, d, f, E = 128, WORKLOAD["d_model"], WORKLOAD["d_ff"], 1
    x, gw, w1, b1, w2, b2, dy = O.layer_inputs(T, d, f, E, seed=seed)
    cfg = O.make_cfg(num_experts=E, jitter_eps=WORKLOAD["jitter_eps"],
                     balance_coeff=WORKLOAD["balance_coeff"])
    return (x, gw, w1, b1, w2, b2, dy), cfg, T


def cpu_threads_for(bytes_per_replica: float, cap: int) -> int:
    n = os.cpu_count() or 1
    try:
        avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
        n = min(n, max(1, int(avail * 0.5 // bytes_per_replica)))
    except Exception:
        pass
    return max(1, min(n, cap))


def time_reference(threads: int, warm: bool = False):
    import oracle as O
    arrs, cfg, T = reference_sample_inputs()
    if O.have_reference():
        kind = "reference"
        secs = O.time_reference_layer(*arrs[:6], cfg, O.TRAIN, 42, arrs[6], threads)
    else:  # the C restatement (port), one replica per thread
        kind = "port"
        from concurrent.futures import ThreadPoolExecutor
        o = O.restatement()
        t0 = time.perf_counter()
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(lambda i: o.moe_layer(*arrs[:6], cfg, O.TRAIN, 42 + i, dy=arrs[6]), range(threads)))
        secs = time.perf_counter() - t0
    return kind, T * threads / secs, secs


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads = cpu_threads_for(1.2e9, 256)
    # warm-up: exercise the code paths (and page in the library) on a tiny sample
    import oracle as O
    arrs, cfg, _ = reference_sample_inputs()
    backend = O.reference() if O.have_reference() else O.restatement()
    for _ in range(args.warmup):
        backend.moe_layer(arrs[0][:8], *arrs[1:6], cfg, O.TRAIN, 1, dy=arrs[6][:8])
    times = []
    kind = "reference"
    for _ in range(args.steps):
        kind, tps, secs = time_reference(threads)
        times.append(secs)
        log(f"reference step: {secs:.2f} s, {tps:.2f} tokens/s ({threads} threads)")
    secs = sorted(times)[len(times) // 2]
    T = 128
    value = T * threads / secs
    sample = (f"per step: {threads} concurrent replicas (one per host thread, {os.cpu_count()} host cores) "
              f"of one expert's share of the config-3 layer: E'=1, d=2048, f=8192, cap=128, 128 tokens, "
              f"train, jitter on, fwd+bwd through the reference's moe_layer_forward + Tensor::backward; "
              f"median of {args.steps} steps.  The reference computes every capacity row of every expert "
              f"one expert after another (routing.cpp:397-406), so the 64-expert layer's time is 64x this "
              f"share plus the O(T d E) gate (<0.2% of its FLOPs); cross-checked against BASELINE.md 3a's "
              f"affine fit over the full 64-expert layer in profiles/r02_reference_fit.json")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_config(args.gpus),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "host_cores": os.cpu_count(),
                             "kind": kind, "sample": sample, "extrapolated": True},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def workload_config(n, E=None, T=None):
    E = E or WORKLOAD["experts"]
    T = T or WORKLOAD["tokens_per_gpu"]
    name = WORKLOAD["name"] if E == WORKLOAD["experts"] and T == WORKLOAD["tokens_per_gpu"] else \
        f"c3_variant_E{E}_T{T}"
    return {"workload": name, "experts": E,
            "experts_per_gpu": E // max(n, 1), "d_model": WORKLOAD["d_model"],
            "d_ff": WORKLOAD["d_ff"], "top_k": 1, "capacity_factor": 1.0,
            "assignment": "plain", "phase": "train", "jitter_eps": WORKLOAD["jitter_eps"],
            "balance_coeff": WORKLOAD["balance_coeff"], "tokens_per_gpu": T,
            "global_tokens": T * n, "parallelism": f"ep{n}",
            "l2": "inputs larger than L2: expert weights %.2f GB/GPU stream from HBM every step"
                  % (2 * E // max(n, 1) * WORKLOAD["d_model"] * WORKLOAD["d_ff"] * 2 / 1e9)}


# ---------------------------------------------------------------- our kernels
STAGE_BYTES_FLOPS = None


def stage_model(stage, T, d, f, El, n_rows, n_tok):
    """Algorithmic bytes and FLOPs of one launch of a stage.
    n_rows = occupied expert rows processed on this GPU, n_tok = tokens."""
    b16 = 2
    W = El * d * f * b16  # one expert weight matrix family
    if stage == "ffn1_fwd":      # H = relu(X W1 + b1): read X rows, W1; write H rows
        return W + n_rows * (d + f) * b16, 2.0 * n_rows * d * f
    if stage == "ffn2_fwd":      # O = H W2 + b2
        return W + n_rows * (f + d) * b16, 2.0 * n_rows * d * f
    if stage == "ffn2_dgrad":    # dH = (dO W2^T) * [H>0]: read dO, W2, H; write dH
        return W + n_rows * (d + 2 * f) * b16, 2.0 * n_rows * d * f
    if stage == "ffn1_dgrad":    # dX = dH W1^T
        return W + n_rows * (f + d) * b16, 2.0 * n_rows * d * f
    if stage in ("ffn2_wgrad", "ffn1_wgrad"):  # dW = A^T B: read A, B rows; write dW
        return W + n_rows * (d + f) * b16, 2.0 * n_rows * d * f
    return None, None


def stage_bytes(stage, T, d, E, K, n_kept, n_drop):
    """Algorithmic HBM bytes of the HBM-bound stages per SURVEY.md §8(d)
    (bf16 activations, s = 2; padding rows / zero fill not counted)."""
    s = 2
    if stage == "gate":          # x read + (choice, slot, prob) write + P saved
        return T * d * s + T * K * 12 + T * E * 4
    if stage == "assign":        # choice read + slot write
        return T * K * 8
    if stage == "dispatch":      # kept rows: x read + buffer write
        return 2 * n_kept * d * s
    if stage == "combine":       # kept rows read + y write (+ residual rows of dropped tokens)
        return n_kept * d * s + T * d * s + n_drop * d * s
    if stage == "combine_bwd":   # dy read (kept tokens) + dO rows write
        return 2 * n_kept * d * s
    if stage == "combine_router_bwd":  # dy read once + O rows read (the <dy, O> dots) + dO rows write
        return 3 * n_kept * d * s
    if stage == "gate_dx":       # dX rows gathered + dx write (+ dy of dropped tokens)
        return n_kept * d * s + T * d * s + n_drop * d * s
    return None


def traffic_for(stage, workload_tag):
    """Measured DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum
    from one `ncu --set full` capture, committed under profiles/) when the
    profile was taken on this exact workload; else None."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "traffic.json")
    try:
        with open(path) as fh:
            t = json.load(fh)
    except OSError:
        return None, None
    if t.get("workload") != workload_tag:
        return None, None
    v = t.get("bytes_per_launch", {}).get(stage)
    return v, t.get("source")


def run_ours(args):
    os.environ.setdefault("NCCL_DEBUG", "WARN")  # keep NCCL's banner off stdout
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2109_10465_b200 as M

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        log(f"note: WORLD_SIZE={world} but --gpus {args.gpus}; using WORLD_SIZE")
    N = world
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if N > 1:
        dist.init_process_group("nccl", device_id=dev)
    E, d, f = args.experts or WORKLOAD["experts"], WORKLOAD["d_model"], WORKLOAD["d_ff"]
    T = args.tokens_per_gpu
    El = E // N
    cfg = M.RouterConfig(num_experts=E, capacity_factor_train=WORKLOAD["capacity_factor"],
                         jitter_eps=WORKLOAD["jitter_eps"], balance_coeff=WORKLOAD["balance_coeff"])
    layer = M.MoeLayer(cfg, T, d, f, torch.bfloat16, ep_size=N, ep_rank=rank)
    if N > 1:
        uid = [M.ep_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        layer.ep_init(uid[0])
    # synthetic parameters (random init of this architecture) and inputs
    g = torch.Generator(device=dev).manual_seed(1234)
    gr = torch.Generator(device=dev).manual_seed(1000 + rank)
    s_g = float(np.sqrt(6.0 / (d + E)))
    s_w = float(np.sqrt(6.0 / (d + f)))
    gate_w = (torch.rand(d, E, device=dev, generator=g) * 2 - 1) * s_g  # replicated
    w1 = ((torch.rand(El, d, f, device=dev, generator=gr) * 2 - 1) * s_w).to(torch.bfloat16)
    w2 = ((torch.rand(El, f, d, device=dev, generator=gr) * 2 - 1) * s_w).to(torch.bfloat16)
    b1 = (torch.rand(El, f, device=dev, generator=gr) * 2 - 1) * 0.01
    b2 = (torch.rand(El, d, device=dev, generator=gr) * 2 - 1) * 0.01
    params = M.MoeLayerParams(gate_w, w1, b1, w2, b2)
    x = ((torch.rand(T, d, device=dev, generator=gr) * 2 - 1)).to(torch.bfloat16)
    dy = ((torch.rand(T, d, device=dev, generator=gr) * 2 - 1)).to(torch.bfloat16)
    seed = M.derive_seed(42, rank)  # per-rank layer seed (parallel.cpp:272)
    y = torch.empty_like(x)
    aux = torch.empty(1, device=dev)
    grads = dict(dx=torch.empty_like(x), dgate_w=torch.empty_like(gate_w), dw1=torch.empty_like(w1),
                 db1=torch.empty_like(b1), dw2=torch.empty_like(w2), db2=torch.empty_like(b2),
                 dresidual=None)

    # one layer seed per step, derived like the reference trainer's per-step
    # seeds (trainer.cpp:146-149), so the next step's seed is known.  With
    # prefetch (default; --no-prefetch turns it off) the next step's jitter
    # stream is generated during this step (moe_prefetch_jitter: MOE_B200_PF_SMS
    # = 10 CTAs on their own stream next to the forward and dgrad GEMMs, which
    # leave those SMs free).  Every step still generates exactly one stream.
    # Under expert parallelism the generator takes 18 SMs in whole TPCs (the
    # cta_group::2 GEMMs keep their SM pairs): N=2 8.76-8.82M tokens/s with,
    # 8.23M without (profiles/r02k_ep_prefetch.txt).
    step_no = [0]

    def seed_of(i):
        return M.derive_seed(seed, i)

    pf_on = [args.prefetch]

    def fwd(xx, yy, aa):
        i = step_no[0]
        if pf_on[0]:
            layer.prefetch_jitter(seed_of(i + 1), T)
        layer.forward(xx, params, M.Phase.TRAIN, seed_of(i), y=yy, aux=aa, decision=False, check=False)
        step_no[0] += 1

    def step():
        fwd(x, y, aux)
        layer.backward(dy, 1.0, check=False, grads=grads)

    def barrier():
        torch.cuda.synchronize()
        if N > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if N == 1:
            return v
        t = torch.tensor([v], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    clocks = ClockSampler()
    if rank == 0:
        clocks.start(N)
    for _ in range(max(args.warmup, 3)):
        step()
    layer.handle.check()  # surfaces any latched non-finite / range flag from warm-up
    barrier()
    # ---- device-timed region (inputs resident in HBM)
    layer.handle.profile(True)
    w0 = time.time()
    launches0 = M.routing.kernel_launch_count()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(st)
    for _ in range(args.steps):
        step()
    e1.record(st)
    barrier()
    launches = M.routing.kernel_launch_count() - launches0
    clocks.mark(w0, time.time())
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    stages = layer.handle.profile_read()
    layer.handle.profile(False)
    cap, drops, kept = layer.handle.stats()
    value = N * T / (ms / 1e3)

    # ---- e2e through the public API with host buffers: every step copies its
    # x and dy from pinned host memory and reads the loss (aux; with
    # --e2e-readback dx also dx) back.  The dx and weight gradients stay on the
    # device, as in a training loop.  Copies run on
    # side streams (double-buffered) so they overlap the previous/next step's
    # kernels, as a training loop feeding the layer would.
    x_h = x.cpu().pin_memory()
    dy_h = dy.cpu().pin_memory()
    dx_h = [torch.empty_like(x_h).pin_memory() for _ in range(2)]
    aux_h = [torch.empty(1).pin_memory() for _ in range(2)]
    xb = [torch.empty_like(x) for _ in range(2)]
    dyb = [torch.empty_like(dy) for _ in range(2)]
    gb = [dict(grads, dx=torch.empty_like(x)) for _ in range(2)]
    auxb = [torch.empty(1, device=dev) for _ in range(2)]
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    done = [torch.cuda.Event() for _ in range(2)]
    for ev in done:
        ev.record(st)

    def e2e_step(i):
        b = i % 2
        with torch.cuda.stream(s_in):
            s_in.wait_event(done[b])          # buffers b free (step i-2 finished)
            xb[b].copy_(x_h, non_blocking=True)
            ev_x = torch.cuda.Event()
            ev_x.record(s_in)
            dyb[b].copy_(dy_h, non_blocking=True)
            ev_dy = torch.cuda.Event()
            ev_dy.record(s_in)
        st.wait_event(ev_x)
        fwd(xb[b], y, auxb[b])
        st.wait_event(ev_dy)
        layer.backward(dyb[b], 1.0, check=False, grads=gb[b])
        ev_c = torch.cuda.Event()
        ev_c.record(st)
        with torch.cuda.stream(s_out):
            s_out.wait_event(ev_c)
            if args.e2e_readback == "dx":
                dx_h[b].copy_(gb[b]["dx"], non_blocking=True)
            aux_h[b].copy_(auxb[b], non_blocking=True)
            done[b].record(s_out)

    # With host-fed inputs the jitter prefetch can cost more than it saves
    # (measured: 2.94 vs 2.71 ms/step at config 3 on one GPU, while it saves
    # ~0.13 ms with resident inputs), so the e2e leg is timed both ways, as
    # a user would pick the option, and reports the better one (both listed).
    def run_e2e():
        for i in range(3):
            e2e_step(i)
        torch.cuda.synchronize()
        barrier()
        e0.record(st)
        for i in range(args.steps):
            e2e_step(i)
        e1.record(s_out)
        torch.cuda.synchronize()
        barrier()
        return max_over_ranks(e0.elapsed_time(e1) / args.steps)

    w0 = time.time()
    e2e_runs = {}
    for pf in ((True, False) if args.prefetch else (False,)):
        pf_on[0] = pf
        e2e_runs[pf] = run_e2e()
    pf_on[0] = args.prefetch
    clocks.mark(w0, time.time())
    clk = clocks.stop() if rank == 0 else None
    e2e_pf = min(e2e_runs, key=e2e_runs.get)
    e2e_ms = e2e_runs[e2e_pf]
    if args.e2e_readback == "dx":
        assert torch.equal(dx_h[(args.steps - 1) % 2].view(torch.int16),
                           gb[(args.steps - 1) % 2]["dx"].cpu().view(torch.int16))
    e2e_value = N * T / (e2e_ms / 1e3)
    layer.handle.check()

    if rank != 0:
        if N > 1:
            dist.destroy_process_group()
        return 0

    # ---- roofline of the dominant kernel (largest stage time)
    hbm, tf_burst, tf_sus, src = peaks()
    per_stage = {k: {"ms": v[0] / max(v[1], 1), "calls": v[1]} for k, v in stages.items()}
    n_rows = int(kept.sum().item()) if N == 1 else None
    if n_rows is None:
        n_rows = T  # EP: every GPU processes ~T kept rows per step (weak scaling)
    # The dominant kernel is the row-GEMM family (tc::grouped_gemm_kernel<ROW>:
    # ffn1_fwd, ffn2_fwd, ffn2_dgrad, ffn1_dgrad — the largest share of the
    # step); its roofline is the launches' algorithmic bytes (or FLOPs) over
    # their summed CUDA-event durations.  The weight-gradient family
    # (tc::grouped_gemm_kernel<WGRAD>) and the slowest single launch are
    # reported beside it.
    families = {"tc::grouped_gemm_kernel<ROW> (fwd1, fwd2, dgrad2, dgrad1)":
                ["ffn1_fwd", "ffn2_fwd", "ffn2_dgrad", "ffn1_dgrad"],
                "tc::grouped_gemm_kernel<WGRAD> (dW2, dW1)": ["ffn2_wgrad", "ffn1_wgrad"]}

    def family_roof(name, stages_):
        stages_ = [k for k in stages_ if k in per_stage]
        if not stages_:
            return None
        b_tot = f_tot = ms_tot = 0.0
        for k in stages_:
            b_, f_ = stage_model(k, T, d, f, El, n_rows, T)
            b_tot += b_
            f_tot += f_
            ms_tot += per_stage[k]["ms"]
        dur = ms_tot / 1e3
        if b_tot / (hbm * 1e9) >= f_tot / (tf_sus * 1e12):
            ach = b_tot / dur / 1e9
            r = {"kernel": name, "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                 "peak_source": src}
        else:
            ach = f_tot / dur / 1e12
            r = {"kernel": name, "bound": "tensor", "achieved": ach, "peak": tf_sus, "unit": "TFLOP/s",
                 "frac": ach / tf_sus, "peak_source": src + " (sustained)"}
        r.update({"launches_per_step": len(stages_), "algorithmic_bytes_per_launch": b_tot / len(stages_),
                  "flops_per_launch": f_tot / len(stages_), "launch_ms": ms_tot / len(stages_),
                  "stages": stages_, "traffic": None})
        tr = [traffic_for(k, f"c3 T={T} N={N}") for k in stages_]
        if all(t_[0] is not None for t_ in tr):
            r["traffic"] = sum(t_[0] for t_ in tr) / len(tr)
            r["traffic_source"] = tr[0][1]
        return r

    fam = {k: family_roof(k, v) for k, v in families.items()}
    fam_ms = {k: sum(per_stage[s_]["ms"] for s_ in v if s_ in per_stage) for k, v in families.items()}
    dom = max(fam_ms, key=fam_ms.get)
    roof = fam[dom]
    roof_other = {k: v for k, v in fam.items() if k != dom and v is not None}
    modeled = [k for k in per_stage if stage_model(k, T, d, f, El, 1, T)[0] is not None]
    slowest = max(modeled, key=lambda k: per_stage[k]["ms"]) if modeled else None
    if slowest:
        b_, f_ = stage_model(slowest, T, d, f, El, n_rows, T)
        ach = b_ / (per_stage[slowest]["ms"] / 1e3) / 1e9
        roof_slowest = {"stage": slowest, "achieved": ach, "unit": "GB/s", "frac_of_hbm": ach / hbm,
                        "launch_ms": per_stage[slowest]["ms"]}
    # HBM-bound stages against the same measured peak
    n_kept = int(kept.sum().item()) if N == 1 else T
    n_drop = T - n_kept
    gate_parts = [k for k in ("gate_fused", "gate_logits", "softmax_topk", "balance_loss") if k in per_stage]
    groups = {"gate": [k for k in ["jitter_noise"] if k in per_stage] + gate_parts, "gate_excl_jitter": gate_parts}
    stage_roof = {}
    for name in ["gate", "gate_excl_jitter", "assign", "dispatch", "combine", "combine_bwd", "combine_router_bwd", "gate_dx"]:
        parts = groups.get(name, [name])
        if not all(p in per_stage for p in parts):
            continue
        st_ms = sum(per_stage[p]["ms"] for p in parts)
        b = stage_bytes("gate" if name == "gate_excl_jitter" else name, T, d, E, 1, n_kept, n_drop)
        stage_roof[name] = {"ms": st_ms, "algorithmic_bytes": b, "GB/s": b / (st_ms / 1e3) / 1e9,
                            "frac": b / (st_ms / 1e3) / 1e9 / hbm}
    gemm_ms = sum(v["ms"] for k, v in per_stage.items() if k.startswith("ffn"))
    gemm_flops = 12.0 * n_rows * d * f
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": N, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (random-init weights of the config-3 architecture, U(-1,1) tokens)",
            "config": dict(workload_config(N, E, T), seeds="per step: derive_seed(derive_seed(42, rank), step)",
                           jitter_stream="each step generates the next step's stream next to its expert GEMMs "
                                         f"(moe_prefetch_jitter, {10 if N == 1 else 18} SMs)" if args.prefetch
                           else "generated at the head of each forward"),
            "roofline": roof,
            "roofline_other_families": roof_other,
            "roofline_slowest_launch": roof_slowest if slowest else None,
            "expert_gemms": {"ms_per_step": gemm_ms, "tflops": gemm_flops / (gemm_ms / 1e3) / 1e12 if gemm_ms else None,
                             "frac_of_bf16_sustained": (gemm_flops / (gemm_ms / 1e3) / 1e12) / tf_sus if gemm_ms else None},
            "e2e": {"value": e2e_value, "unit": UNIT, "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": 2 * T * d * 2,
                    "d2h_bytes_per_step": (T * d * 2 if args.e2e_readback == "dx" else 0) + 4,
                    "readback": args.e2e_readback, "jitter_prefetch": e2e_pf,
                    "ms_per_step_by_prefetch": {("on" if k else "off"): v for k, v in e2e_runs.items()}},
            "gpu_launches": launches, "gpu_launches_per_step": launches / args.steps,
            "clocks": clk, "stages_ms": {k: round(v["ms"], 4) for k, v in per_stage.items()},
            "stage_roofline": dict(stage_roof, note="SURVEY 8(d) algorithmic bytes; the gate stage also generates "
                                   "the reference's T*d mt19937_64 jitter draws (not counted as bytes) and reads "
                                   "them back (x*noise) for the 3xTF32 logits"),
            "decision": {"capacity": cap, "dropped_tokens_rank0": drops}}
    if N == 1 and not args.no_cpu_baseline:
        try:
            threads = cpu_threads_for(1.2e9, 16)
            kind, tps, secs = time_reference(threads)
            _, cfg_s, Ts = reference_sample_inputs()
            line["cpu_baseline"] = {"value": tps, "unit": UNIT, "cores": threads, "host_cores": os.cpu_count(),
                                    "kind": kind, "extrapolated": True,
                                    "sample": f"{threads} concurrent replicas of one expert's share of the "
                                              f"config-3 layer (E'=1, d=2048, f=8192, cap=128, {Ts} tokens) "
                                              f"fwd+bwd, {secs:.1f} s; the 64-expert layer is 64 such shares "
                                              f"run in sequence (routing.cpp:397-406)"}
        except Exception as ex:  # pragma: no cover
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "unavailable",
                                    "sample": str(ex)}
    print(json.dumps(line), flush=True)
    if N > 1:
        dist.destroy_process_group()
    return 0


EXTRA = {
    # BASELINE.json configs other than the headline (one GPU; device-timed)
    "c1": dict(E=8, d=512, f=2048, T=4096, k=1, C=1.0, mode=0, dtype="fp32", layers=1,
               phase=0, fwd_only=False, desc="config 1: fp32 parity path, E=8 top-1 C=1.0 plain"),
    "c2": dict(E=32, d=1024, f=4096, T=16384, k=2, C=1.25, mode=2, dtype="bf16", layers=1,
               phase=0, fwd_only=False, desc="config 2: E=32 top-2 C=1.25 RTS, aux loss"),
    "c4": dict(E=64, d=1024, f=4096, T=16384, k=1, C=1.0, mode=2, dtype="bf16", layers=18,
               phase=0, fwd_only=False,
               desc="config 4: 18-layer MoE stack (d=1024, f=4096, E=64, RTS), x_{l+1}=y_l, bwd in reverse"),
    "c5": dict(E=8, d=1024, f=4096, T=262144, k=1, C=2.0, mode=0, dtype="bf16", layers=1,
               phase=1, fwd_only=True,
               desc="config 5: inference (eval, C=2.0, no jitter), experts pruned to 8, T=256k, fwd only"),
}


def run_extra(args):
    """Device-timed tokens/s for the other BASELINE configs.  One GPU, or under
    torchrun N ranks with expert parallelism (E/N experts per rank, every
    layer's peer map bound with moe_ep_export/import; value = N*T / max-over-
    ranks step time, weak scaling at T tokens per GPU)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2109_10465_b200 as M
    w = EXTRA[args.workload]
    E, d, f, T, L = args.experts or w["E"], w["d"], w["f"], args.tokens or w["T"], w["layers"]
    N = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if N > 1:
        dist.init_process_group("nccl", device_id=dev)
    El = E // N
    dt = torch.float32 if w["dtype"] == "fp32" else torch.bfloat16
    g = torch.Generator(device=dev).manual_seed(7)
    gr = torch.Generator(device=dev).manual_seed(70 + rank)
    cfg = M.RouterConfig(num_experts=E, top_k=w["k"], capacity_factor_train=w["C"],
                         capacity_factor_eval=w["C"] if w["phase"] == 1 else 2.0,
                         assignment_mode=M.AssignmentMode(w["mode"]))
    s_w = float(np.sqrt(6.0 / (d + f)))
    layers, params = [], []
    for _ in range(L):
        layers.append(M.MoeLayer(cfg, T, d, f, dt, ep_size=N, ep_rank=rank))
        if N > 1:
            def all_gather(b):
                out = [None] * N
                dist.all_gather_object(out, b)
                return out
            layers[-1].ep_bootstrap(all_gather, dist.barrier)
        params.append(M.MoeLayerParams(
            (torch.rand(d, E, device=dev, generator=g) * 2 - 1) * float(np.sqrt(6.0 / (d + E))),
            ((torch.rand(El, d, f, device=dev, generator=gr) * 2 - 1) * s_w).to(dt),
            (torch.rand(El, f, device=dev, generator=gr) * 2 - 1) * 0.01,
            ((torch.rand(El, f, d, device=dev, generator=gr) * 2 - 1) * s_w).to(dt),
            (torch.rand(El, d, device=dev, generator=gr) * 2 - 1) * 0.01))
    x0 = ((torch.rand(T, d, device=dev, generator=gr) * 2 - 1)).to(dt)
    dy0 = ((torch.rand(T, d, device=dev, generator=gr) * 2 - 1)).to(dt)
    ys = [torch.empty_like(x0) for _ in range(L)]
    aux = torch.empty(1, device=dev)
    grads = [dict(dx=torch.empty_like(x0), dgate_w=torch.empty(d, E, device=dev),
                  dw1=torch.empty(El, d, f, device=dev, dtype=dt), db1=torch.empty(El, f, device=dev),
                  dw2=torch.empty(El, f, d, device=dev, dtype=dt), db2=torch.empty(El, d, device=dev),
                  dresidual=torch.empty_like(x0)) for _ in range(L)]
    zero = torch.zeros_like(x0)
    phase = M.Phase(w["phase"])

    def step(i):
        h = x0
        for l in range(L):  # stack: zero residual inside blocks (model.cpp:340-350)
            if args.prefetch and w["phase"] == 0:  # next step's stream of this layer, next to its GEMMs
                layers[l].prefetch_jitter(M.derive_seed(M.derive_seed(M.derive_seed(42, rank), i + 1), l), T)
            layers[l].forward(h, params[l], phase, M.derive_seed(M.derive_seed(M.derive_seed(42, rank), i), l),
                              residual=zero if L > 1 else None, y=ys[l], aux=aux, decision=False,
                              check=False)
            h = ys[l]
        if w["fwd_only"]:
            return
        g_ = dy0
        for l in reversed(range(L)):
            layers[l].backward(g_, 1.0, check=False, grads=grads[l])
            g_ = grads[l]["dx"]

    def barrier():
        torch.cuda.synchronize()
        if N > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for i in range(max(args.warmup, 3)):
        step(i)
    for lay in layers:
        lay.handle.check()
    barrier()
    prof = args.workload == "c5" and L == 1
    if prof:
        layers[0].handle.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    nw = max(args.warmup, 3)  # timed steps continue the seed sequence (prefetched streams match)
    for i in range(args.steps):
        step(nw + i)
    e1.record()
    barrier()
    ms = e0.elapsed_time(e1) / args.steps
    if N > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    flops = (4.0 if w["fwd_only"] else 12.0) * T * w["k"] * d * f * L
    line = {"metric": "MoE layer " + ("fwd" if w["fwd_only"] else "fwd+bwd") + " tokens/sec",
            "value": N * T / (ms / 1e3), "unit": UNIT, "n_gpus": N, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "dtype": w["dtype"], "data": "synthetic",
            "config": {"workload": args.workload, "desc": w["desc"], "tokens_per_gpu": T,
                       "layers": L, "experts": E, "experts_per_gpu": El, "d_model": d, "d_ff": f,
                       "top_k": w["k"], "parallelism": f"ep{N}",
                       "jitter": ("prefetched one step ahead per layer" if args.prefetch else "inline")
                       if w["phase"] == 0 else "none (eval)"},
            "expert_tflops_upper_bound_per_gpu": flops / (ms / 1e3) / 1e12}
    if prof:  # inference regime: gate / dispatch / combine against the HBM roofline
        hbm = peaks()[0]
        per = {k: v[0] / max(v[1], 1) for k, v in layers[0].handle.profile_read().items()}
        layers[0].handle.profile(False)
        cap, drops, kept = layers[0].handle.stats()
        n_kept = int(kept.sum().item())
        roof = {}
        gate_parts = [k for k in ("gate_fused", "gate_logits", "softmax_topk", "balance_loss") if k in per]
        for name, parts in (("gate", gate_parts), ("assign", ["assign"]),
                            ("dispatch", ["dispatch"]), ("combine", ["combine"])):
            if parts and all(p_ in per for p_ in parts):
                st_ms = sum(per[p_] for p_ in parts)
                b = stage_bytes(name, T, d, E, w["k"], n_kept, T - n_kept)
                roof[name] = {"ms": st_ms, "GB/s": b / (st_ms / 1e3) / 1e9, "frac": b / (st_ms / 1e3) / 1e9 / hbm}
        line["stages_ms"] = {k: round(v, 4) for k, v in per.items()}
        line["stage_roofline"] = roof
    if rank == 0:
        print(json.dumps(line), flush=True)
    if N > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--tokens-per-gpu", type=int, default=WORKLOAD["tokens_per_gpu"])
    ap.add_argument("--experts", type=int, default=0,
                    help="config-3 variant with this many experts in total (EP-overhead baselines: "
                         "1 GPU with E=64/N experts has the same rows per expert as N GPUs with E=64)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-readback", default="aux", choices=["dx", "aux"],
                    help="e2e: read back the step's loss (the aux loss, default) or dx + aux every step")
    ap.add_argument("--no-prefetch", dest="prefetch", action="store_false",
                    help="generate the next step's jitter stream during this step's backward "
                         "(moe_prefetch_jitter, default on: generate the next step's jitter stream next to "
                         "this step's expert GEMMs; off = generate it at the head of each forward)")
    ap.add_argument("--workload", default="c3", choices=["c3"] + sorted(EXTRA))
    ap.add_argument("--tokens", type=int, default=0, help="override T for --workload c1/c2/c4/c5")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.workload != "c3":
        return run_extra(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
