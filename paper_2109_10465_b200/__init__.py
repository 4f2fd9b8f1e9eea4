"""paper_2109_10465_b200 — B200-native MoE layer (arXiv 2109.10465 hot path).

The product is libmoe_b200.so (hand-written sm_100a kernels behind the C ABI
in include/moe_b200.h).  This package is its Python host side: a mirror of
the reference's operator API (routing.hpp) over ctypes.
"""
from . import _lib
from .routing import (KDROPPED, AssignmentMode, ConfigError, DispatchBuffer, ExpertFfn,
                      GateResult, InvalidArgument, MoeError, MoeHandle, MoeLayer,
                      MoeLayerParams, MoeLayerResult, NonFiniteError, Phase, RouterConfig,
                      RoutingDecision, ShapeError, UniformShapeError, assign_grouped,
                      assign_plain, assign_rts, balance_loss, capacity, combine, derive_seed,
                      dispatch, ep_unique_id, gate_forward, make_assignment, moe_layer_forward)
from .stack import DropHistogram, MoeStack, UtilizationCounts
from . import checkpoint, optim  # noqa: F401  (checkpoint -> device layout; Adam step)

__all__ = [n for n in dir() if not n.startswith("_")]
