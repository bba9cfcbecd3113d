"""Flat little-endian snapshot of a DSCache handle's streaming state (checkpoint / resume).

SURVEY.md §5 "Checkpoint / resume"; SPEC.md:341 ("a flat binary layout ... little-endian
... bit-exact round trip").  The state later steps read is the sink A, the ring U (raw
un-rotated K/V: position ids are assigned at load, so a slab restored
anywhere is valid) and each layer's frame counter; everything else (C_t, P_t, slots, ids,
the last evicted frame) is the library's closed form of that counter (dscache_get_state).

Layout (all little-endian):
  b"DSCK"  u32 version (1)
  i32 x 17 config fields (dscache_config minus `device`, which may differ on resume), f64 rope_theta
  i32 R (ring slots), i32 element bytes
  per layer:  i64 frames_seen, i32 sink_filled, i32 0
  per (stream, layer), stream-major:  sink K, sink V  [Hkv][A][d];  ring K, ring V  [Hkv][R][d]
              (bf16 as its raw 16-bit pattern, fp32 as IEEE single)
  u32 crc32 of everything before it

Host logic only: no arithmetic of the method lives here (only byte moves).
"""
from __future__ import annotations

import struct
import zlib

import numpy as np
import torch

MAGIC = b"DSCK"
VERSION = 1
_INT_FIELDS = ("num_streams", "num_layers", "num_q_heads", "num_kv_heads", "head_dim", "kv_head_offset",
               "tokens_per_frame", "sink_tokens", "past_frames", "instant_frames", "max_query_tokens",
               "max_position", "rope_style", "dtype", "attn_impl", "instant_source")


def _cfg_words(cfg) -> list:
    return [int(getattr(cfg, f)) for f in _INT_FIELDS]


def _header(cfg, R: int, elem: int) -> bytes:
    ints = _cfg_words(cfg)
    return (MAGIC + struct.pack("<I", VERSION) + struct.pack("<%di" % len(ints), *ints)
            + struct.pack("<d", float(cfg.rope_theta)) + struct.pack("<ii", R, elem))


def _elem(cfg) -> int:
    return 2 if int(cfg.dtype) == 0 else 4


def _to_bytes(t: torch.Tensor) -> bytes:
    t = t.contiguous().cpu()
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().astype("<i2", copy=False).tobytes()
    return t.numpy().astype("<f4", copy=False).tobytes()


def _from_bytes(buf: bytes, shape, elem: int) -> torch.Tensor:
    if elem == 2:
        a = np.frombuffer(buf, dtype="<i2").astype(np.int16).reshape(shape)
        return torch.from_numpy(a.copy()).view(torch.bfloat16)
    a = np.frombuffer(buf, dtype="<f4").astype(np.float32).reshape(shape)
    return torch.from_numpy(a.copy())


def pack(cfg, R: int, counters, slabs) -> bytes:
    """counters: [(frames_seen, sink_filled)] per layer; slabs: {(s, l): (sink_k, sink_v, ring_k, ring_v)}."""
    S, N = int(cfg.num_streams), int(cfg.num_layers)
    if len(counters) != N:
        raise ValueError("one (frames_seen, sink_filled) pair per layer")
    parts = [_header(cfg, R, _elem(cfg))]
    for f, sf in counters:
        parts.append(struct.pack("<qii", int(f), int(sf), 0))
    shapes = [(cfg.num_kv_heads, cfg.sink_tokens, cfg.head_dim)] * 2 + [(cfg.num_kv_heads, R, cfg.head_dim)] * 2
    for s in range(S):
        for l in range(N):
            for t, shp in zip(slabs[(s, l)], shapes):
                if tuple(t.shape) != tuple(shp):
                    raise ValueError(f"slab of (stream {s}, layer {l}) has shape {tuple(t.shape)}, expected {shp}")
                parts.append(_to_bytes(t))
    body = b"".join(parts)
    return body + struct.pack("<I", zlib.crc32(body) & 0xFFFFFFFF)


def unpack(blob: bytes, cfg, R: int):
    """Inverse of pack for a handle of config `cfg` (ValueError on any mismatch or corruption)."""
    if len(blob) < 8 or blob[:4] != MAGIC:
        raise ValueError("not a DSCache snapshot")
    body, (crc,) = blob[:-4], struct.unpack("<I", blob[-4:])
    if zlib.crc32(body) & 0xFFFFFFFF != crc:
        raise ValueError("snapshot checksum mismatch")
    elem = _elem(cfg)
    head = _header(cfg, R, elem)
    (version,) = struct.unpack_from("<I", body, 4)
    if version != VERSION:
        raise ValueError(f"snapshot version {version}, expected {VERSION}")
    if body[:len(head)] != head:
        raise ValueError("snapshot was taken with a different configuration")
    off = len(head)
    S, N = int(cfg.num_streams), int(cfg.num_layers)
    counters = []
    for _ in range(N):
        f, sf, _z = struct.unpack_from("<qii", body, off)
        counters.append((f, sf))
        off += 16
    Hkv, A, d = int(cfg.num_kv_heads), int(cfg.sink_tokens), int(cfg.head_dim)
    shapes = [(Hkv, A, d)] * 2 + [(Hkv, R, d)] * 2
    slabs = {}
    for s in range(S):
        for l in range(N):
            ts = []
            for shp in shapes:
                nb = shp[0] * shp[1] * shp[2] * elem
                if off + nb > len(body):
                    raise ValueError("snapshot truncated")
                ts.append(_from_bytes(body[off:off + nb], shp, elem))
                off += nb
            slabs[(s, l)] = tuple(ts)
    if off != len(body):
        raise ValueError("snapshot has trailing bytes")
    return counters, slabs
