"""Seeded synthetic inputs and workload shapes shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no RoPE, no softmax, no schedule):
only the five BASELINE.json workload shapes and a counter-keyed Gaussian
generator.  Both sides (``oracle/`` and ``paper_2605_01858_b200``) consume the
exact same rounded tensors produced here; neither side imports the other.

Input recipe: every tensor is i.i.d. N(0, 1) times
``scale`` (1.0 for c1, 0.5 for c2..c5, BASELINE.json configs), drawn in fp64 by
numpy's PCG64 keyed by (base seed, config id, stream, layer, kind, index), then
rounded to the config dtype (round-to-nearest-even).  The shapes follow the
paper's LLaVA-OV-7B streaming workload: 196 tokens per frame,
1 FPS, 28 query / 4 KV heads of dim 128, sink + past + instant budgets
(PAPER.md:295).  These synthetic streams stand in for StreamingBench /
OVO-Bench videos, which are not available and are not reproduced here.
"""
from __future__ import annotations

import dataclasses
from typing import Dict

import numpy as np
import torch

# kinds of tensors drawn per (stream, layer, index)
SINK_K, SINK_V = 0, 1          # the A sink tokens (first append)            [A][Hkv][d]
FRM_K, FRM_V = 2, 3            # raw K/V of frame f                           [tpf][Hkv][d]
INST_Q = 4                     # instant-build queries at step t              [C_t][Hq][d]
QRY_Q, QRY_K, QRY_V = 5, 6, 7  # query chunk at step t (K/V transient)        [q][Hq|Hkv][d]
UPD_Q = 8                      # queries of the frame leaving the buffer at t [tpf][Hq][d]
BST_K, BST_V = 9, 10           # re-encoded (boosted) newest frame at step t  [n_boost][Hkv][d]
IK_K, IK_V = 11, 12            # real-model mode: the step's instant K/V (Eq. 7 output) [C_t][Hkv][d]
PST_K, PST_V = 13, 14          # real-model mode: frame f's Eq. 5 K/V (stored in U)    [tpf][Hkv][d]

KIND_NAMES = {SINK_K: "SINK_K", SINK_V: "SINK_V", FRM_K: "FRM_K", FRM_V: "FRM_V",
              INST_Q: "INST_Q", QRY_Q: "QRY_Q", QRY_K: "QRY_K", QRY_V: "QRY_V", UPD_Q: "UPD_Q",
              BST_K: "BST_K", BST_V: "BST_V", IK_K: "IK_K", IK_V: "IK_V", PST_K: "PST_K", PST_V: "PST_V"}


@dataclasses.dataclass(frozen=True)
class StreamConfig:
    """One BASELINE.json workload.  Budgets in frames as in the paper."""
    name: str
    cfg_id: int
    num_streams: int        # S
    num_layers: int         # N
    num_q_heads: int        # Hq
    num_kv_heads: int       # Hkv
    head_dim: int           # d
    rope_theta: float
    tokens_per_frame: int   # tpf
    sink_tokens: int        # A   (l_A)
    past_frames: int        # l_U (W = l_U * tpf tokens)
    instant_frames: int     # l_I (C = l_I * tpf tokens)
    query_tokens: int       # q
    num_frames: int         # stream length
    dtype: str              # "bf16" | "fp32"
    scale: float            # input std
    seed: int = 0
    max_position: int = 32768

    @property
    def W(self) -> int:
        return self.past_frames * self.tokens_per_frame

    @property
    def C(self) -> int:
        return self.instant_frames * self.tokens_per_frame

    @property
    def torch_dtype(self):
        return torch.bfloat16 if self.dtype == "bf16" else torch.float32

    def replace(self, **kw) -> "StreamConfig":
        return dataclasses.replace(self, **kw)


# BASELINE.json "configs", in order.
CONFIGS: Dict[str, StreamConfig] = {
    "c1": StreamConfig("c1", 1, 1, 1, 2, 1, 64, 1e4, 16, 4, 4, 1, 8, 20, "fp32", 1.0),
    "c2": StreamConfig("c2", 2, 1, 1, 28, 4, 128, 1e6, 196, 4, 32, 4, 64, 64, "bf16", 0.5),
    "c3": StreamConfig("c3", 3, 1, 28, 28, 4, 128, 1e6, 196, 4, 64, 8, 64, 256, "bf16", 0.5),
    "c4": StreamConfig("c4", 4, 1, 1, 28, 4, 128, 1e6, 196, 4, 128, 8, 64, 4096, "bf16", 0.5),
    "c5": StreamConfig("c5", 5, 64, 4, 28, 4, 128, 1e6, 196, 4, 32, 4, 32, 128, "bf16", 0.5),
}


def _rng(cfg: StreamConfig, stream: int, layer: int, kind: int, index: int) -> np.random.Generator:
    ss = np.random.SeedSequence([cfg.seed, cfg.cfg_id, stream, layer, kind, index])
    return np.random.Generator(np.random.PCG64(ss))


def draw(cfg: StreamConfig, stream: int, layer: int, kind: int, index: int, shape) -> torch.Tensor:
    """N(0,1)*scale drawn in fp64, rounded (RNE) to the config dtype.  CPU tensor."""
    x = _rng(cfg, stream, layer, kind, index).standard_normal(size=tuple(shape)) * cfg.scale
    return torch.from_numpy(x).to(cfg.torch_dtype)


def sink_kv(cfg: StreamConfig, stream: int, layer: int):
    shp = (cfg.sink_tokens, cfg.num_kv_heads, cfg.head_dim)
    return draw(cfg, stream, layer, SINK_K, 0, shp), draw(cfg, stream, layer, SINK_V, 0, shp)


def frame_kv(cfg: StreamConfig, stream: int, layer: int, frame: int):
    shp = (cfg.tokens_per_frame, cfg.num_kv_heads, cfg.head_dim)
    return draw(cfg, stream, layer, FRM_K, frame, shp), draw(cfg, stream, layer, FRM_V, frame, shp)


def instant_q(cfg: StreamConfig, stream: int, layer: int, step: int, n_inst: int):
    return draw(cfg, stream, layer, INST_Q, step, (n_inst, cfg.num_q_heads, cfg.head_dim))


def update_q(cfg: StreamConfig, stream: int, layer: int, step: int):
    return draw(cfg, stream, layer, UPD_Q, step, (cfg.tokens_per_frame, cfg.num_q_heads, cfg.head_dim))


def boost_kv(cfg: StreamConfig, stream: int, layer: int, step: int, n_boost: int):
    """Raw K/V of the newest frame re-encoded at a higher resolution (n_boost tokens)."""
    shp = (n_boost, cfg.num_kv_heads, cfg.head_dim)
    return draw(cfg, stream, layer, BST_K, step, shp), draw(cfg, stream, layer, BST_V, step, shp)


def instant_kv(cfg: StreamConfig, stream: int, layer: int, step: int, n_inst: int):
    """Real-model mode: the K/V the caller's Eq. 7 build produced for the step's C_t instant
    tokens (fresh every step: the instant cache is rebuilt per step)."""
    shp = (n_inst, cfg.num_kv_heads, cfg.head_dim)
    return draw(cfg, stream, layer, IK_K, step, shp), draw(cfg, stream, layer, IK_V, step, shp)


def past_kv(cfg: StreamConfig, stream: int, layer: int, frame: int):
    """Real-model mode: frame f's K/V from its Eq. 5 update (stored in U when it leaves the
    buffer); distinct from any instant K/V of the same frame."""
    shp = (cfg.tokens_per_frame, cfg.num_kv_heads, cfg.head_dim)
    return draw(cfg, stream, layer, PST_K, frame, shp), draw(cfg, stream, layer, PST_V, frame, shp)


def batch_boost_kv(cfg: StreamConfig, step: int, n_boost: int, streams=None, layers=None):
    """[S][N][n_boost][Hkv][d] stacked boosted K and V."""
    streams = range(cfg.num_streams) if streams is None else streams
    layers = range(cfg.num_layers) if layers is None else layers
    ks, vs = [], []
    for s in streams:
        kl, vl = [], []
        for l in layers:
            k, v = boost_kv(cfg, s, l, step, n_boost)
            kl.append(k); vl.append(v)
        ks.append(torch.stack(kl)); vs.append(torch.stack(vl))
    return torch.stack(ks), torch.stack(vs)


def query_qkv(cfg: StreamConfig, stream: int, layer: int, step: int, n_q: int | None = None):
    n_q = cfg.query_tokens if n_q is None else n_q
    q = draw(cfg, stream, layer, QRY_Q, step, (n_q, cfg.num_q_heads, cfg.head_dim))
    k = draw(cfg, stream, layer, QRY_K, step, (n_q, cfg.num_kv_heads, cfg.head_dim))
    v = draw(cfg, stream, layer, QRY_V, step, (n_q, cfg.num_kv_heads, cfg.head_dim))
    return q, k, v


def batch_frame_kv(cfg: StreamConfig, frame: int, streams=None, layers=None):
    """[S][N][tpf][Hkv][d] stacked K and V for one frame over streams x layers."""
    streams = range(cfg.num_streams) if streams is None else streams
    layers = range(cfg.num_layers) if layers is None else layers
    ks, vs = [], []
    for s in streams:
        kl, vl = [], []
        for l in layers:
            k, v = frame_kv(cfg, s, l, frame)
            kl.append(k); vl.append(v)
        ks.append(torch.stack(kl)); vs.append(torch.stack(vl))
    return torch.stack(ks), torch.stack(vs)


def batch_sink_kv(cfg: StreamConfig, streams=None, layers=None):
    streams = range(cfg.num_streams) if streams is None else streams
    layers = range(cfg.num_layers) if layers is None else layers
    ks, vs = [], []
    for s in streams:
        kl, vl = [], []
        for l in layers:
            k, v = sink_kv(cfg, s, l)
            kl.append(k); vl.append(v)
        ks.append(torch.stack(kl)); vs.append(torch.stack(vl))
    return torch.stack(ks), torch.stack(vs)


def batch_instant_q(cfg: StreamConfig, step: int, n: int, streams=None, layers=None):
    """[S][N][n][Hq][d]; n = number of instant tokens (the caller's schedule decides it)."""
    streams = range(cfg.num_streams) if streams is None else streams
    layers = range(cfg.num_layers) if layers is None else layers
    return torch.stack([torch.stack([instant_q(cfg, s, l, step, n) for l in layers]) for s in streams])


def batch_query_qkv(cfg: StreamConfig, step: int, streams=None, layers=None, n_q=None):
    streams = range(cfg.num_streams) if streams is None else streams
    layers = range(cfg.num_layers) if layers is None else layers
    qs, ks, vs = [], [], []
    for s in streams:
        ql, kl, vl = [], [], []
        for l in layers:
            q, k, v = query_qkv(cfg, s, l, step, n_q)
            ql.append(q); kl.append(k); vl.append(v)
        qs.append(torch.stack(ql)); ks.append(torch.stack(kl)); vs.append(torch.stack(vl))
    return torch.stack(qs), torch.stack(ks), torch.stack(vs)
