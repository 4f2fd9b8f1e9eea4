"""Expert optimizer step on the device.

``Adam`` mirrors AdamOptimizer (optim.hpp:19-42, optim.cpp:10-57): one
shared step counter, one (m, v) pair per registered parameter, optional
global-norm clipping over ALL registered gradients, bias-corrected update.
Parameters are fp32 master tensors on the device; for bf16 layers an
optional bf16 shadow (the tensor the forward reads) is rewritten in the same
pass.  Every kernel is ``libmoe_b200.so`` (optim.cu); this class only sequences
them on the current stream.  Under expert parallelism call ``step`` with
``allreduce=fn`` to sum the squared norm over ranks before clipping.
"""
from __future__ import annotations

import torch

from . import _lib as L
from .routing import ConfigError, _check, _p

_DT = {torch.float32: 0, torch.bfloat16: 1}


class Adam:
    def __init__(self, params, beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8,
                 shadows=None):
        self.params = list(params)
        for p in self.params:
            if p.dtype != torch.float32 or not p.is_cuda or not p.is_contiguous():
                raise ConfigError("adam: parameters must be contiguous fp32 CUDA tensors (masters)")
        self.shadows = list(shadows) if shadows is not None else [None] * len(self.params)
        self.m = [torch.zeros_like(p) for p in self.params]
        self.v = [torch.zeros_like(p) for p in self.params]
        self.beta1, self.beta2, self.eps = beta1, beta2, eps
        self.step_count = 0
        dev = self.params[0].device if self.params else "cuda"
        self._sq = torch.zeros(1, dtype=torch.float64, device=dev)
        self._scale = torch.ones(1, dtype=torch.float64, device=dev)

    def step(self, grads, lr: float, clip_norm: float = 0.0, allreduce=None):
        """AdamOptimizer::step(lr, clip_norm) with ``grads[i]`` the gradient of
        params[i] (fp32 or bf16; None = zero gradient, optim.cpp:44)."""
        if lr <= 0.0:
            raise ConfigError("adam: learning rate must be positive")  # optim.cpp:22-24
        lib = L.load()
        stream = C_stream()
        scale = None
        if clip_norm > 0.0:
            self._sq.zero_()
            for g in grads:
                if g is None:
                    continue
                _check(lib.moe_grad_sqnorm(_p(g), g.numel(), _DT[g.dtype], _p(self._sq), stream))
            if allreduce is not None:
                allreduce(self._sq)
            _check(lib.moe_clip_scale(_p(self._sq), float(clip_norm), _p(self._scale), stream))
            scale = self._scale
        self.step_count += 1
        for p, m, v, g, sh in zip(self.params, self.m, self.v, grads, self.shadows):
            if g is None:
                g = torch.zeros_like(p)
            if g.numel() != p.numel():
                raise ConfigError("adam: gradient does not match its parameter")
            _check(lib.moe_adam_update(_p(p), _p(m), _p(v), _p(g.contiguous()), p.numel(), _DT[g.dtype],
                                       _p(sh), _p(scale), float(lr), self.beta1, self.beta2, self.eps,
                                       self.step_count, stream))


def C_stream():
    import ctypes
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
