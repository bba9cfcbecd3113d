"""Host logic of the checkpoint format (paper_2605_01858_b200/checkpoint.py): flat
little-endian layout and bit-exact round trip, corruption and config checks."""
import struct
import zlib

import pytest
import torch

import dscache_synth as synth
from paper_2605_01858_b200 import checkpoint as CK
from paper_2605_01858_b200.dscache import Config


def _cfg(c, dtype=None):
    return Config(c.num_streams, c.num_layers, c.num_q_heads, c.num_kv_heads, c.head_dim, 0, c.tokens_per_frame,
                  c.sink_tokens, c.past_frames, c.instant_frames, c.query_tokens, c.max_position, c.rope_theta, 0,
                  (0 if c.dtype == "bf16" else 1) if dtype is None else dtype, 0, 0, 0)


def _state(cfg, R, seed=0):
    g = torch.Generator().manual_seed(seed)
    dt = torch.bfloat16 if cfg.dtype == 0 else torch.float32
    Hkv, A, d = cfg.num_kv_heads, cfg.sink_tokens, cfg.head_dim
    slabs = {}
    for s in range(cfg.num_streams):
        for l in range(cfg.num_layers):
            slabs[(s, l)] = tuple(torch.randn(shp, generator=g).to(dt) for shp in
                                  [(Hkv, A, d)] * 2 + [(Hkv, R, d)] * 2)
    counters = [(1000 + 3 * l, 1) for l in range(cfg.num_layers)]
    return counters, slabs


def _bits(t):
    return t.view(torch.int16) if t.dtype == torch.bfloat16 else t.view(torch.int32)


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_round_trip_is_bit_exact(name):
    c = synth.CONFIGS[name].replace(num_streams=2, num_layers=3, past_frames=2, instant_frames=1)
    cfg = _cfg(c)
    R = (c.past_frames + c.instant_frames + 1) * c.tokens_per_frame
    counters, slabs = _state(cfg, R)
    slabs[(0, 0)][2].view(-1)[0] = float("nan")          # any bit pattern survives
    blob = CK.pack(cfg, R, counters, slabs)
    c2, s2 = CK.unpack(blob, cfg, R)
    assert c2 == counters
    for key, ts in slabs.items():
        for x, y in zip(ts, s2[key]):
            assert torch.equal(_bits(x), _bits(y))
    assert CK.pack(cfg, R, c2, s2) == blob


def test_layout_is_flat_little_endian():
    c = synth.CONFIGS["c1"].replace(num_streams=1, num_layers=1)
    cfg = _cfg(c)
    R = 8
    Hkv, A, d = cfg.num_kv_heads, cfg.sink_tokens, cfg.head_dim
    counters = [(5, 1)]
    vals = [torch.arange(n, dtype=torch.float32).reshape(shp) + 0.5 * i
            for i, (n, shp) in enumerate([(Hkv * A * d, (Hkv, A, d))] * 2 + [(Hkv * R * d, (Hkv, R, d))] * 2)]
    blob = CK.pack(cfg, R, counters, {(0, 0): tuple(vals)})
    assert blob[:4] == b"DSCK" and struct.unpack_from("<I", blob, 4) == (1,)
    off = 8 + 4 * 16
    assert struct.unpack_from("<d", blob, off) == (c.rope_theta,)
    assert struct.unpack_from("<ii", blob, off + 8) == (R, 4)
    assert struct.unpack_from("<qii", blob, off + 16) == (5, 1, 0)
    p = off + 32
    assert struct.unpack_from("<3f", blob, p) == (0.0, 1.0, 2.0)               # sink K row 0, fp32 LE
    assert struct.unpack_from("<f", blob, p + Hkv * A * d * 4) == (0.5,)        # sink V starts after sink K
    assert len(blob) == p + 4 * (2 * Hkv * A * d + 2 * Hkv * R * d) + 4
    assert struct.unpack("<I", blob[-4:]) == (zlib.crc32(blob[:-4]) & 0xFFFFFFFF,)


def test_corruption_and_mismatch_are_rejected():
    c = synth.CONFIGS["c2"].replace(num_streams=1, num_layers=2, past_frames=1, instant_frames=1)
    cfg = _cfg(c)
    R = 3 * c.tokens_per_frame
    counters, slabs = _state(cfg, R)
    blob = CK.pack(cfg, R, counters, slabs)
    bad = bytearray(blob)
    bad[100] ^= 1
    with pytest.raises(ValueError, match="checksum"):
        CK.unpack(bytes(bad), cfg, R)
    with pytest.raises(ValueError, match="configuration"):
        CK.unpack(blob, _cfg(c.replace(past_frames=2)), R)
    with pytest.raises(ValueError, match="configuration"):
        CK.unpack(blob, _cfg(c, dtype=1), R)
    with pytest.raises(ValueError):
        CK.unpack(blob[:-10] + struct.pack("<I", zlib.crc32(blob[:-10]) & 0xFFFFFFFF)[:0], cfg, R)
    with pytest.raises(ValueError, match="not a DSCache"):
        CK.unpack(b"XXXX" + blob[4:], cfg, R)
    other = dict(slabs)
    other[(0, 1)] = slabs[(0, 1)][:2] + (slabs[(0, 1)][2][:, :-1], slabs[(0, 1)][3])
    with pytest.raises(ValueError, match="shape"):
        CK.pack(cfg, R, counters, other)
