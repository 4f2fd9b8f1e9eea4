"""Checkpoint -> device weight layout.

Reads the reference's on-disk checkpoint (checkpoint.cpp: ``manifest.json``
+ ``tensors.bin``, f64 records with CRC32, version ``moe-forge-ckpt/1``),
prunes experts exactly as ``prune_experts`` (surgery.cpp:135-212), and packs
each MoE layer's per-expert records (``<layer>.moe.expert<e>.{w1,b1,w2,b2}``,
gate ``<layer>.moe.gate``, model.cpp:85-100) into the device layout the
B200 layer reads: w1 [E, d, f], w2 [E, f, d] in the layer dtype, b1/b2/gate
fp32.  The f64 -> bf16/fp32 conversion runs on the device
(``moe_convert_f64``); the host only reads bytes and checks them.
"""
from __future__ import annotations

import json
import os
import re
import zlib
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from .routing import MoeError, MoeLayerParams, _check, _p

VERSION = "moe-forge-ckpt/1"  # checkpoint.hpp:12


class CheckpointError(MoeError):
    """moeforge::CheckpointError (checkpoint.hpp)."""


@dataclass
class TensorRecord:
    name: str
    role: str            # "non_expert" | "expert" | "gate"
    shape: list
    data: np.ndarray     # f64, flat
    layer: int = -1
    expert: int = -1


@dataclass
class Checkpoint:
    arch: dict
    tensors: list = field(default_factory=list)

    def at(self, name: str) -> TensorRecord:
        for r in self.tensors:
            if r.name == name:
                return r
        raise CheckpointError("checkpoint: no tensor named " + name)

    def num_moe_layers(self) -> int:  # model.hpp:32-34
        a = self.arch
        return a["enc_layers"] // a["moe_every"] + a["dec_layers"] // a["moe_every"]


def load_checkpoint(path) -> Checkpoint:
    """load_checkpoint (checkpoint.cpp:253-287) with read_manifest's checks."""
    path = str(path)
    try:
        with open(os.path.join(path, "manifest.json")) as fh:
            j = json.load(fh)
    except OSError:
        raise CheckpointError("cannot open manifest in " + path) from None
    if j.get("version") != VERSION:
        raise CheckpointError("checkpoint version mismatch: found " + str(j.get("version")))
    blob_path = os.path.join(path, "tensors.bin")
    try:
        size = os.path.getsize(blob_path)
    except OSError:
        raise CheckpointError("cannot open blob in " + path) from None
    if size != j["blob_size"]:
        raise CheckpointError(f"blob truncated or oversized: expected {j['blob_size']} bytes, found {size}")
    ck = Checkpoint(arch=j["arch"])
    with open(blob_path, "rb") as fh:
        for rec in j["tensors"]:
            if rec.get("dtype") != "f64":
                raise CheckpointError("manifest: unsupported dtype " + str(rec.get("dtype")))
            count = rec["length"] // 8
            if rec["length"] % 8 or count != int(np.prod(rec["shape"], dtype=np.int64)):
                raise CheckpointError("record " + rec["name"] + " length does not match shape")
            fh.seek(rec["offset"])
            raw = fh.read(rec["length"])
            if len(raw) != rec["length"]:
                raise CheckpointError("blob truncated while reading " + rec["name"])
            if zlib.crc32(raw) != rec["crc32"]:
                raise CheckpointError("checksum failure on tensor " + rec["name"])
            ck.tensors.append(TensorRecord(rec["name"], rec["role"], list(rec["shape"]),
                                           np.frombuffer(raw, dtype="<f8").copy(),
                                           rec.get("layer", -1), rec.get("expert", -1)))
    return ck


_EXPERT = re.compile(r"^(.*\.moe)\.expert(\d+)(\..*)$")


def prune_experts(ck: Checkpoint, k: int, strategy: str = "top_utilization", counts=None,
                  seed: int = 0) -> Checkpoint:
    """surgery.cpp:135-212.  strategy 'top_utilization' keeps, per MoE layer,
    the k most-used experts (stable sort by count, descending; then
    ascending index order); 'random' keeps the first k of Rng(seed).permutation(E),
    sorted, for every layer.  Gate columns follow the kept experts."""
    E = ck.arch["num_experts"]
    if k < 1 or k > E:
        raise ValueError("prune_experts: k must be in [1, num_experts]")
    nl = ck.num_moe_layers()
    if strategy == "top_utilization":
        if counts is None or len(counts) != nl:
            raise ValueError("prune_experts: utilization counts missing or mismatched")
        kept = []
        for layer in range(nl):
            c = [int(v) for v in counts[layer]]
            if len(c) != E:
                raise ValueError("prune_experts: counts do not cover all experts")
            order = sorted(range(E), key=lambda e: -c[e])  # Python's sort is stable
            kept.append(sorted(order[:k]))
    else:
        perm = (L.load() and _permutation(seed, E))
        kept = [sorted(perm[:k])] * nl
    out = Checkpoint(arch=dict(ck.arch, num_experts=k))
    for r in ck.tensors:
        if r.role == "non_expert":
            out.tensors.append(r)
        elif r.role == "gate":
            keep = kept[r.layer]
            d = r.shape[0]
            g = r.data.reshape(d, E)[:, keep]
            out.tensors.append(TensorRecord(r.name, r.role, [d, k], np.ascontiguousarray(g).ravel(), r.layer))
        else:
            m = _EXPERT.match(r.name)
            keep = kept[r.layer]
            if r.expert in keep:
                j = keep.index(r.expert)
                out.tensors.append(TensorRecord(f"{m.group(1)}.expert{j}{m.group(3)}", r.role, r.shape,
                                                r.data, r.layer, j))
    # the reference enumerates specs of the pruned arch: gate, then experts 0..k-1
    # per layer in spec order; records above keep that relative order
    return out


def _permutation(seed: int, n: int):
    out = np.empty(n, dtype=np.uint32)
    _check(L.load().moe_rng_permutation(seed, n, out.ctypes.data))
    return [int(v) for v in out]


def moe_layer_prefixes(ck: Checkpoint) -> list:
    """Gate record names in MoE-ordinal order -> layer prefixes."""
    gates = sorted((r for r in ck.tensors if r.role == "gate"), key=lambda r: r.layer)
    return [r.name[: -len(".moe.gate")] for r in gates]


def _to_device(data: np.ndarray, shape, dtype: torch.dtype, device) -> torch.Tensor:
    src = torch.from_numpy(np.ascontiguousarray(data, dtype=np.float64)).to(device)
    dst = torch.empty(*shape, dtype=dtype, device=device)
    code = {torch.float32: 0, torch.bfloat16: 1}[dtype]
    stream = torch.cuda.current_stream(device).cuda_stream
    import ctypes
    _check(L.load().moe_convert_f64(_p(src), src.numel(), code, _p(dst), ctypes.c_void_p(stream)))
    return dst


def moe_layer_params(ck: Checkpoint, moe_ordinal: int, dtype: torch.dtype = torch.bfloat16,
                     device="cuda", experts=None) -> MoeLayerParams:
    """Pack MoE layer `moe_ordinal` into the device layout.  `experts` (a
    range) selects the local shard under expert parallelism
    (parallel.cpp:260-265)."""
    prefix = moe_layer_prefixes(ck)[moe_ordinal]
    E = ck.arch["num_experts"]
    d, f = ck.arch["d_model"], ck.arch["ffn_dim"]
    ex = list(experts) if experts is not None else list(range(E))
    gate = ck.at(prefix + ".moe.gate")
    if gate.shape != [d, E]:
        raise CheckpointError("checkpoint: gate " + gate.name + " does not match the architecture")

    def stack(suffix, shape):
        parts = []
        for e in ex:
            r = ck.at(f"{prefix}.moe.expert{e}.{suffix}")
            if r.shape != list(shape):
                raise CheckpointError("checkpoint: record " + r.name + " does not match architecture layout")
            parts.append(r.data)
        return np.concatenate(parts)

    El = len(ex)
    return MoeLayerParams(
        _to_device(gate.data, (d, E), torch.float32, device),
        _to_device(stack("w1", (d, f)), (El, d, f), dtype, device),
        _to_device(stack("b1", (f,)), (El, f), torch.float32, device),
        _to_device(stack("w2", (f, d)), (El, f, d), dtype, device),
        _to_device(stack("b2", (d,)), (El, d), torch.float32, device))
