"""CPU tests: pin the oracle (C restatement) against the reference's own
known-answer tests and against golden vectors produced by the reference itself.

Ports of /root/reference/proj/tests/test_routing.cpp and test_parallel.cpp
cases are named after the reference TEST_CASE/SUBCASE they follow.
"""
import numpy as np
import pytest

import oracle as O
from tests.golden import load as G

BACKENDS = ["restatement"] + (["reference"] if O.have_reference() else [])


@pytest.fixture(params=BACKENDS)
def be(request):
    return O.restatement() if request.param == "restatement" else O.reference()


# --- rng.cpp / survey KATs ------------------------------------
def test_mt19937_64_conformance(be):
    # C++ standard [rand.predef]: 10000th output of default-seeded mt19937_64
    assert int(be.mt64(5489, 1, skip=9999)[0]) == 9981545732273789042


def test_derive_seed_kats(be):
    assert be.derive_seed(42, "jitter") == 4217090220841641567
    assert be.derive_seed(42, "assign") == 11878108427965954893


def test_permutation_kat(be):
    assert be.permutation(be.derive_seed(42, "assign"), 8).tolist() == [0, 4, 1, 2, 7, 5, 3, 6]


def test_restatement_stream_matches_reference():
    if not O.have_reference():
        pytest.skip("oracle/_ref not built")
    o, r = O.restatement(), O.reference()
    for seed in (0, 1, 42, 2**63 + 5):
        assert np.array_equal(o.mt64(seed, 2000, skip=313), r.mt64(seed, 2000, skip=313))
        assert np.array_equal(o.permutation(seed, 1000), r.permutation(seed, 1000))
        assert o.derive_seed(seed, 7) == r.derive_seed(seed, 7)


# --- test_routing.cpp:43-50 capacity formula ----------------------------------
def test_capacity_formula(be):
    cfg = O.make_cfg(num_experts=8)
    assert be.capacity(64, cfg, O.TRAIN) == 8
    assert be.capacity(64, cfg, O.EVAL) == 16
    assert be.capacity(1, cfg, O.TRAIN) == 1
    cfg.capacity_factor_train = 1.3
    assert be.capacity(10, cfg, O.TRAIN) == 2


def test_capacity_ignores_top_k(be):
    # routing.cpp:43-49: capacity does not scale with top_k
    assert be.capacity(16384, O.make_cfg(num_experts=32, top_k=2, capacity_factor_train=1.25),
                       O.TRAIN) == 640


def test_config_validation(be):
    with pytest.raises(O.OracleError) as e:
        be.capacity(10, O.make_cfg(num_experts=2, top_k=3), O.TRAIN)
    assert e.value.status == 2
    with pytest.raises(O.OracleError):
        be.capacity(0, O.make_cfg(), O.TRAIN)


# --- test_routing.cpp:52-103 gate_forward -------------------------------------
def test_gate_tie_goes_to_expert0():
    o = O.restatement()
    P, ch, gp, _ = o.gate_forward(np.array([[0.3, -0.4]]), np.zeros((2, 2)),
                                  O.make_cfg(num_experts=2), O.EVAL, 0)
    assert P[0, 0] == pytest.approx(0.5, rel=1e-15) and ch[0] == 0


def test_gate_eps0_train_equals_eval():
    o = O.restatement()
    x = O.uniform(11, 30, -1, 1).reshape(6, 5)
    w = O.uniform(12, 20, -1, 1).reshape(5, 4)
    cfg = O.make_cfg(num_experts=4, jitter_eps=0.0)
    a = o.gate_forward(x, w, cfg, O.TRAIN, 123)
    b = o.gate_forward(x, w, cfg, O.EVAL, 456)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_gate_parity_routing_histogram():
    o = O.restatement()
    x = np.array([[-1.0 if t % 2 == 0 else 1.0] for t in range(9)])
    _, ch, _, _ = o.gate_forward(x, np.array([[1.0, -1.0]]), O.make_cfg(num_experts=2), O.EVAL, 0)
    assert ch.tolist() == [1 if t % 2 == 0 else 0 for t in range(9)]
    assert np.bincount(ch).tolist() == [4, 5]


def test_jitter_bounded_and_deterministic():
    o = O.restatement()
    x = O.uniform(3, 30, -1, 1).reshape(6, 5)
    w = O.uniform(4, 20, -1, 1).reshape(5, 4)
    cfg = O.make_cfg(num_experts=4)
    a = o.gate_forward(x, w, cfg, O.TRAIN, 77)
    b = o.gate_forward(x, w, cfg, O.TRAIN, 77)
    assert np.array_equal(a[0], b[0])
    assert a[3].min() >= 0.99 and a[3].max() < 1.01


# --- test_routing.cpp:117-246 assignment --------------------------------------
def test_assign_plain_suffix_drops(be):
    assert be.assign([0, 0, 0, 0], 1, 2)[0].tolist() == [0, 1, -1, -1]


def test_assign_plain_hand_simulated(be):
    s, _ = be.assign([1, 1, 1, 0, 0, 0], 2, 2)
    assert (s >= 0).tolist() == [True, True, False, True, True, False]


def test_assign_plain_top2_k_major_kat(be):
    # t2's first choice dropped, its second choice kept.
    s, cap = be.assign([0, 1, 0, 1, 0, 2], 3, 2, top_k=2)
    assert s.tolist() == [0, 0, 1, 1, -1, 0] and cap == 2


def test_assign_grouped_kats(be):
    s, cap = be.assign([0] * 6, 1, 3, mode=O.GROUPED, group_count=2)
    assert s.tolist() == [0, 1, -1, 2, 3, -1] and cap == 4
    s, _ = be.assign([0, 0, 0, 0], 1, 2, mode=O.GROUPED, group_count=2)
    assert (s >= 0).tolist() == [True, False, True, False]
    s, _ = be.assign([0, 1, 1, 0], 2, 2, mode=O.GROUPED, group_count=2)
    assert (s >= 0).all()
    with pytest.raises(O.OracleError):
        be.assign([0, 0, 0], 1, 2, mode=O.GROUPED, group_count=2)


def test_assign_grouped_g1_equals_plain(be):
    ch = (O.restatement().mt64(41, 48) % np.uint64(4)).astype(np.int32)
    a = be.assign(ch, 4, 5)
    b = be.assign(ch, 4, 5, mode=O.GROUPED, group_count=1)
    assert a[1] == b[1] and np.array_equal(a[0], b[0])


def test_rts_no_drops_when_capacity_suffices(be):
    for seed in range(32):
        assert (be.assign([0, 1, 0, 1, 2, 2], 3, 2, mode=O.RTS, rts_seed=seed)[0] >= 0).all()


def test_rts_keep_frequency():
    # test_routing.cpp:208-224 — 4 tokens on one expert with cap 2 -> 1/2
    o = O.restatement()
    kept = np.zeros(4)
    for s in range(10000):
        kept += o.assign([0, 0, 0, 0], 1, 2, mode=O.RTS, rts_seed=s)[0] >= 0
    assert np.allclose(kept / 10000, 0.5, atol=0.03)


def test_capacity_never_exceeded_fuzz(be):
    rng = np.random.default_rng(51)
    for _ in range(50):
        E = int(rng.integers(1, 7))
        T = 6 + int(rng.integers(0, 60)) // E * E
        cap = int(rng.integers(1, 6))
        K = 1 if E == 1 else int(rng.integers(1, 3))
        ch = rng.integers(0, E, size=T * K).astype(np.int32)
        if K == 2:  # distinct experts per token, as the gate produces
            ch[1::2] = np.where(ch[1::2] == ch[0::2], (ch[0::2] + 1) % E, ch[1::2])
        G = int(rng.integers(1, 5))
        while T % G:
            G -= 1
        for mode in (O.PLAIN, O.GROUPED, O.RTS):
            s, c = be.assign(ch, E, cap, top_k=K, mode=mode, group_count=G, rts_seed=int(rng.integers(1 << 62)))
            kept = s >= 0
            assert (s[kept] < c).all()
            pairs = set(zip(ch[kept].tolist(), s[kept].tolist()))
            assert len(pairs) == int(kept.sum())


# --- test_routing.cpp:286-364 dispatch / combine -------------------------------
def test_dispatch_combine_roundtrip_bit_exact():
    o = O.restatement()
    rng = np.random.default_rng(61)
    for _ in range(100):
        E, T, cap, d = (int(rng.integers(1, 6)), int(rng.integers(1, 25)), int(rng.integers(1, 5)),
                        int(rng.integers(1, 9)))
        x = rng.uniform(-1, 1, (T, d))
        ch = rng.integers(0, E, T).astype(np.int32)
        s, c = o.assign(ch, E, cap, mode=O.RTS, rts_seed=int(rng.integers(1 << 62)))
        buf, occ = o.dispatch(x, ch, s, 1, E, c)
        y = o.combine(buf, ch, s, 1, E, c, x, np.ones(T))
        assert np.array_equal(y, x)
        assert (buf[occ == 0] == 0).all()


def test_combine_hand_built():
    o = O.restatement()
    x = np.array([[1.0, 2.0], [-1.0, 0.5], [3.0, 3.0]])
    ch = np.array([0, 1, 0], np.int32)
    s, c = o.assign(ch, 2, 1)
    y = o.combine(np.array([[2.0, 4.0], [1.0, -0.5]]), ch, s, 1, 2, c, x, np.array([0.5, 0.25, 0.9]))
    assert y.ravel().tolist() == [1.0, 2.0, 0.25, -0.125, 3.0, 3.0]


# --- test_routing.cpp:367-435 balance loss -------------------------------------
def test_balance_loss_closed_forms():
    o = O.restatement()
    assert o.balance_loss(np.full((8, 4), 0.25), np.arange(8) % 4, 1, 0.01) == pytest.approx(0.01, rel=1e-12)
    P = np.zeros((6, 4))
    P[:, 0] = 1
    assert o.balance_loss(P, np.zeros(6), 1, 0.01) == pytest.approx(0.04, rel=1e-12)
    with pytest.raises(O.OracleError) as e:
        o.balance_loss(np.full((2, 2), 0.4), np.zeros(2), 1, 0.01)
    assert e.value.status == 5


# --- golden vectors from the reference itself ----------------------------------
def _close(a, b, tol=1e-10):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.abs(b)))) <= tol


@pytest.mark.parametrize("name", G.layer_names())
def test_restatement_vs_reference_golden(name):
    cfg, phase, seed, daux, inp, z = G.load_layer(name)
    out = O.restatement().moe_layer(inp["x"], inp["gate_w"], inp["w1"], inp["b1"], inp["w2"],
                                    inp["b2"], cfg, phase, seed, residual=inp["residual"],
                                    dy=inp["dy"], daux=daux)
    assert np.array_equal(out.expert_id, z["expert_id"])
    assert np.array_equal(out.slot, z["slot"])
    assert out.capacity == int(z["capacity"])
    assert _close(out.y, z["y"]) and _close(out.aux, z["aux"]) and _close(out.gate_prob, z["gate_prob"])
    for k in ("dx", "dgate_w", "db1", "db2", "dw1", "dw2", "dresidual"):
        if k in z:
            assert _close(getattr(out, k), z[k]), k
    if "dw1_rowsum" in z:
        assert _close(out.dw1.sum(2), z["dw1_rowsum"]) and _close(out.dw2.sum(1), z["dw2_colsum"])


@pytest.mark.parametrize("name", G.ep_names())
def test_restatement_ep_vs_reference_golden(name):
    cfg, phase, seed, inp, z = G.load_ep(name)
    ys, eid, slot, gp, cap, traffic = O.restatement().ep_forward(
        inp["xs"], inp["gate_w"], inp["w1"], inp["b1"], inp["w2"], inp["b2"], cfg, phase, seed)
    assert np.array_equal(eid, z["expert_id"]) and np.array_equal(slot, z["slot"])
    assert cap == int(z["capacity"])
    assert np.array_equal(ys, z["ys"])
    assert np.array_equal(traffic, z["traffic"])


def test_ep_equals_per_rank_single_rank():
    # test_parallel.cpp:209-225 contract: each rank's output equals
    # moe_layer_forward on its own tokens with seed derive_seed(seed, r).
    cfg, phase, seed, inp, z = G.load_ep("ep2_e4_rts")
    o = O.restatement()
    for r in range(inp["xs"].shape[0]):
        out = o.moe_layer(inp["xs"][r], inp["gate_w"], inp["w1"], inp["b1"], inp["w2"], inp["b2"],
                          cfg, phase, o.derive_seed(seed, r))
        assert np.array_equal(out.y, z["ys"][r])


def test_ep_traffic_closed_form():
    # test_parallel.cpp:268-293: symmetric; 2 * E_local * cap * d * 8 bytes per pair
    cfg, phase, seed, inp, z = G.load_ep("ep4_e8_plain_eval")
    ep, T, d = inp["xs"].shape
    cap = int(z["capacity"])
    tr = z["traffic"]
    assert np.array_equal(tr, tr.T) and np.all(np.diag(tr) == 0)
    El = cfg.num_experts // ep
    assert tr[0, 1] == 2 * El * cap * d * 8


def test_c1_golden_decisions_restatement():
    """Full-size config 1 decisions from the reference (fixture) reproduced by the
    restatement's gate + assignment (forward decisions only; seconds)."""
    z = G.load_c1()
    T, d, f, E = (int(v) for v in z["spec"][:4])
    x, gw, *_ = O.layer_inputs(T, d, f, E, seed=int(z["spec"][8]))
    from oracle.margin import margin_guard
    cfg = O.make_cfg(num_experts=E)
    x = margin_guard(x, gw, cfg, O.TRAIN, 42)
    assert _close(x.sum(1), z["x_rowsum"], 0)
    o = O.restatement()
    _, ch, gp, _ = o.gate_forward(x, gw, cfg, O.TRAIN, o.derive_seed(42, "jitter"))
    s, cap = o.assign(ch, E, o.capacity(T, cfg, O.TRAIN))
    assert np.array_equal(ch, z["expert_id"]) and np.array_equal(s, z["slot"])
    assert _close(gp, z["gate_prob"], 1e-14)
