"""CPU, world_size 2 (gloo): the expert-parallel exchange protocol of the CUDA
path (moe_api.cu forward_impl / backward_impl), executed with the oracle as the
per-rank compute, must reproduce the reference's expert-parallel step.

Protocol (parallel.cpp:260-338, made physical):
  * rank r gates its own T tokens with seed derive_seed(seed, r) and builds
    the dispatch buffer [E, cap, d] (expert-major, fixed shape);
  * all_to_all: chunk s = experts [s*E/ep, (s+1)*E/ep) goes to rank s; rank s
    receives [ep(origin), E_local, cap, d] plus the per-(origin, expert) kept
    counts;
  * rank s runs its E_local experts on every origin's slice;
  * reverse all_to_all returns [E_local, cap, d] slices to their origins;
  * each rank combines locally with weight E * gate_prob.
"""
import os

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from tests.golden import load as G


def _ffn(x, w1, b1, w2, b2):
    h = np.maximum(x @ w1 + b1, 0.0)
    return h @ w2 + b2


def _worker(rank, world, port, name, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg, phase, seed, inp, z = G.load_ep(name)
        o = O.restatement()
        ep, T, d = inp["xs"].shape
        E = cfg.num_experts
        El = E // ep
        x = inp["xs"][rank]
        rs = o.derive_seed(seed, rank)
        _, choice, gp, _ = o.gate_forward(x, inp["gate_w"], cfg, phase, o.derive_seed(rs, "jitter"))
        slot, cap = o.assign(choice, E, o.capacity(T, cfg, phase),
                             mode=O.PLAIN if phase == O.EVAL else cfg.assignment_mode,
                             rts_seed=o.derive_seed(rs, "assign"))
        buf, occ = o.dispatch(x, choice, slot, 1, E, cap)
        kept = np.bincount(choice[slot >= 0], minlength=E).astype(np.int32)
        # forward all-to-all of counts and fixed-shape slices
        send = torch.from_numpy(buf.reshape(ep, El * cap * d).copy())
        recv = torch.empty_like(send)
        dist.all_to_all_single(recv, send)
        cnt_recv = torch.empty(ep * El, dtype=torch.int32)
        dist.all_to_all_single(cnt_recv, torch.from_numpy(kept))
        recv = recv.numpy().reshape(ep, El, cap, d)
        cnt_recv = cnt_recv.numpy().reshape(ep, El)
        # owner computes its experts on occupied rows of every origin's slice
        out = np.zeros_like(recv)
        for r in range(ep):
            for le in range(El):
                e = rank * El + le
                n = int(cnt_recv[r, le])
                out[r, le, :n] = _ffn(recv[r, le, :n], inp["w1"][e], inp["b1"][e], inp["w2"][e],
                                      inp["b2"][e])
        back = torch.empty(ep * El * cap * d, dtype=torch.float64)
        dist.all_to_all_single(back, torch.from_numpy(out.reshape(-1).copy()))
        O_loc = back.numpy().reshape(E * cap, d)
        y = o.combine(O_loc, choice, slot, 1, E, cap, x, gp * E)
        ok = (np.array_equal(choice, z["expert_id"][rank]) and np.array_equal(slot, z["slot"][rank])
              and float(np.max(np.abs(y - z["ys"][rank]))) < 1e-12)
        q.put((rank, ok, float(np.max(np.abs(y - z["ys"][rank])))))
    finally:
        dist.destroy_process_group()


def test_ep_exchange_protocol_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29800 + os.getpid() % 100
    procs = [ctx.Process(target=_worker, args=(r, 2, port, "ep2_e4_rts", q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
