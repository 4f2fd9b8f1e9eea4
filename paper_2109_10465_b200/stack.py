"""The reference's MoE caller restated over the B200 layer (SURVEY.md §8(f)
rows 1 and 3).

* ``MoeStack`` — the ``run_moe`` lambda of ``forward`` (model.cpp:340-350)
  applied layer after layer on a residual stream: every MoE layer gets a
  ZERO residual (so dropped tokens contribute 0, model.cpp:342), the seed
  ``derive_seed(step_seed, moe_ordinal)`` (model.cpp:345-346), its aux loss
  is added to the running ``aux_loss`` (model.cpp:347) and its decision is
  appended to ``decisions`` (model.cpp:348); the caller adds the layer's
  output to the stream (``enc_x = add(enc_x, ffn_out)``, model.cpp:366).
  Attention, layer norms and embeddings between the MoE layers are outside
  this path (SURVEY §2 marks the transformer OUT); ``between`` lets a
  caller insert them.  ``backward`` runs the layers' explicit backward in
  reverse order through the same stream (the tape order of tensor.cpp:156-187).
* ``DropHistogram`` / ``UtilizationCounts`` — trainer.cpp:15-29 and
  surgery.cpp:100-122, accumulated on the device from each layer's decision
  by ``moe_accumulate_decision_stats`` (integer adds: exact).

The multitask trainer's optimizer step (trainer.cpp:181-183, optim.cpp:21-57)
is ``paper_2109_10465_b200.optim.Adam``.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import torch

from . import _lib as L
from .routing import MoeLayer, MoeLayerParams, Phase, RouterConfig, _check, _p, derive_seed


class DropHistogram:
    """trainer.hpp:31-42: dropped routes by token-position octile."""

    def __init__(self, device="cuda"):
        self.dev = torch.zeros(10, dtype=torch.int64, device=device)  # [8 buckets, dropped, routed]

    def accumulate(self, layer: MoeLayer):
        """DropHistogram::accumulate(decision) for the layer's last forward."""
        _check(L.load().moe_accumulate_decision_stats(layer.handle.h, _p(_scratch_util(layer)),
                                                      _p(self.dev)), layer.handle.h)

    @property
    def buckets(self):
        return [int(v) for v in self.dev[:8].tolist()]

    @property
    def total_dropped(self) -> int:
        return int(self.dev[8].item())

    @property
    def total_routed(self) -> int:
        return int(self.dev[9].item())

    def dropped_fraction(self) -> float:
        r = self.total_routed
        return 0.0 if r == 0 else self.total_dropped / r


def _scratch_util(layer: MoeLayer) -> torch.Tensor:
    u = getattr(layer, "_util_scratch", None)
    if u is None:
        u = layer._util_scratch = torch.zeros(layer.cfg.num_experts, dtype=torch.int64, device="cuda")
    return u


@dataclass
class UtilizationCounts:
    """surgery.hpp UtilizationCounts: first-choice counts per (layer, expert)."""
    per_layer: list = field(default_factory=list)  # device int64 [E] per layer
    total_tokens: int = 0

    def accumulate(self, layer_index: int, layer: MoeLayer, hist: torch.Tensor | None = None):
        while len(self.per_layer) <= layer_index:
            self.per_layer.append(torch.zeros(layer.cfg.num_experts, dtype=torch.int64, device="cuda"))
        h = hist if hist is not None else torch.zeros(10, dtype=torch.int64, device="cuda")
        _check(L.load().moe_accumulate_decision_stats(layer.handle.h, _p(self.per_layer[layer_index]),
                                                      _p(h)), layer.handle.h)

    def as_lists(self):
        return [[int(v) for v in u.tolist()] for u in self.per_layer]


class MoeStack:
    """A stack of MoE layers called the way model.cpp:323-392 calls them."""

    def __init__(self, cfg: RouterConfig, n_layers: int, max_tokens: int, d_model: int, d_ff: int,
                 dtype: torch.dtype = torch.bfloat16, ep_size: int = 1, ep_rank: int = 0):
        self.cfg = cfg
        self.layers = [MoeLayer(cfg, max_tokens, d_model, d_ff, dtype, ep_size, ep_rank)
                       for _ in range(n_layers)]
        self.dtype = dtype
        self.drops = DropHistogram()
        self.util = UtilizationCounts()

    def ep_init(self, unique_ids):
        for layer, uid in zip(self.layers, unique_ids):
            layer.ep_init(uid)

    def forward(self, x: torch.Tensor, params: list, phase: Phase, seed: int, between=None,
                stats: bool = True, next_seed: int | None = None):
        """Returns (stream_out, aux_loss [1] fp32, decisions).  ``between(l, h)``
        (optional) maps the stream before MoE layer l (e.g. a layer norm).
        ``next_seed`` (training): the next step's seed; each layer then
        generates its next jitter stream during this call, next to its expert
        GEMMs (moe_prefetch_jitter), instead of at the head of its next forward."""
        h = x
        aux_sum = torch.zeros(1, device=x.device, dtype=torch.float32)
        decisions = []
        self._zero = torch.zeros_like(x)
        self._inputs = []
        for ordinal, (layer, p) in enumerate(zip(self.layers, params)):
            inp = between(ordinal, h) if between is not None else h
            if next_seed is not None and phase == Phase.TRAIN:
                layer.prefetch_jitter(derive_seed(next_seed, ordinal), inp.shape[0])
            y, aux, dec = layer.forward(inp, p, phase, derive_seed(seed, ordinal), residual=self._zero,
                                        check=False)
            aux_sum += aux
            decisions.append(dec)
            if stats:  # one device pass feeds both statistics
                self.util.accumulate(ordinal, layer, hist=self.drops.dev)
            h = h + y  # enc_x = add(enc_x, ffn_out)
            self._inputs.append(inp)
        for layer in self.layers:
            layer.handle.check()
        self.util.total_tokens += x.shape[0]
        return h, aux_sum, decisions

    def backward(self, dy: torch.Tensor, daux: float = 1.0):
        """Gradient of <dy, stream_out> + daux * aux_loss.  Returns (dx, per-layer
        parameter grads).  Valid when ``between`` was None (identity)."""
        g = dy
        grads = [None] * len(self.layers)
        for ordinal in range(len(self.layers) - 1, -1, -1):
            layer = self.layers[ordinal]
            gl = layer.backward(g.contiguous(), daux, check=False,
                                grads=None)
            grads[ordinal] = gl
            g = g + gl["dx"]  # stream: d(h + y(h))/dh
        for layer in self.layers:
            layer.handle.check()
        return g, grads
