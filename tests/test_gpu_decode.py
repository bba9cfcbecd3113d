"""Decode through the memory-bound decode kernel (decode.cu) and
the sampled-past variant (zeta_decode, reading Q24) vs the fp64 oracle;
position ids bit-exact through the debug export."""
import numpy as np
import pytest
import torch

import dscache_synth as synth
from oracle import dscache_oracle as O
from oracle.workload import StreamInputs, step_schedule
from tests.gpu_harness import _batch, assert_close
from paper_2605_01858_b200 import dscache as D

pytestmark = pytest.mark.gpu


def _stream_to(cfg, dsc, t, exact, gen, dev):
    A, tpf, Hkv, d = cfg.sink_tokens, cfg.tokens_per_frame, cfg.num_kv_heads, cfg.head_dim
    if A > 0:
        skv = {sl: synth.sink_kv(cfg, *sl) for sl in exact}
        dsc.append_frame(_batch(cfg, (A, Hkv, d), exact, lambda s, l: skv[(s, l)][0], dev, gen),
                         _batch(cfg, (A, Hkv, d), exact, lambda s, l: skv[(s, l)][1], dev, gen))
    for f in range(t + 1):
        kv = {sl: synth.frame_kv(cfg, *sl, f) for sl in exact}
        dsc.append_frame(_batch(cfg, (tpf, Hkv, d), exact, lambda s, l: kv[(s, l)][0], dev, gen),
                         _batch(cfg, (tpf, Hkv, d), exact, lambda s, l: kv[(s, l)][1], dev, gen))


def _self_and_q(cfg, s, l, n_self, n_q):
    g = torch.Generator().manual_seed(1000 * s + 10 * l + n_self)
    ks = (torch.randn(n_self, cfg.num_kv_heads, cfg.head_dim, generator=g) * cfg.scale).to(cfg.torch_dtype)
    vs = (torch.randn(n_self, cfg.num_kv_heads, cfg.head_dim, generator=g) * cfg.scale).to(cfg.torch_dtype)
    q = (torch.randn(n_q, cfg.num_q_heads, cfg.head_dim, generator=g) * cfg.scale).to(cfg.torch_dtype)
    return q, ks, vs


def check_decode(cfg, t, exact, n_self, n_q, stride, debug=False):
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev)
    gen.manual_seed(55 + cfg.cfg_id)
    dsc = D.DSCache.from_config(cfg.replace(query_tokens=max(cfg.query_tokens, n_self)))
    if debug:
        dbg = torch.full((cfg.num_streams, cfg.num_layers, dsc.debug_len()), -1, dtype=torch.int32, device=dev)
        dsc.set_debug(None, dbg, False)
    _stream_to(cfg, dsc, t, exact, gen, dev)
    sq = {sl: _self_and_q(cfg, *sl, n_self, n_q) for sl in exact}
    q = _batch(cfg, (n_q, cfg.num_q_heads, cfg.head_dim), exact, lambda s, l: sq[(s, l)][0], dev, gen)
    ks = _batch(cfg, (n_self, cfg.num_kv_heads, cfg.head_dim), exact, lambda s, l: sq[(s, l)][1], dev, gen)
    vs = _batch(cfg, (n_self, cfg.num_kv_heads, cfg.head_dim), exact, lambda s, l: sq[(s, l)][2], dev, gen)
    o = dsc.decode(q, ks, vs, past_stride=stride)
    torch.cuda.synchronize()
    sch = step_schedule(cfg, t)
    for (s, l) in exact:
        inp = StreamInputs(cfg, s, l)
        qq, kk, vv = (x.double().numpy() for x in sq[(s, l)])
        ref = O.decode_output_sampled(sch, inp.sink(), inp.frame_kv, qq, kk, vv, stride, cfg.rope_theta)
        assert_close(o[s, l].float().cpu(), ref, cfg.dtype, f"{cfg.name} decode t={t} s={s} l={l} n_self={n_self} "
                                                            f"n_q={n_q} stride={stride}")
    ids = dbg.cpu().numpy() if debug else None
    R = dsc.R
    dsc.close()
    return ids, R


@pytest.mark.parametrize("t", [0, 2, 3, 4, 10, 35, 36, 50])
@pytest.mark.parametrize("stride", [1, 2, 3])
def test_decode_kernel_c2_steps_and_strides(lib, t, stride):
    cfg = synth.CONFIGS["c2"]
    check_decode(cfg, t, [(0, 0)], 64 + 16, 1, stride)


@pytest.mark.parametrize("n_self,n_q", [(1, 1), (65, 2), (64 + 40, 2), (300, 1)])
def test_decode_kernel_c2_lengths(lib, n_self, n_q):
    cfg = synth.CONFIGS["c2"]
    check_decode(cfg, 40, [(0, 0)], n_self, n_q, 1)
    check_decode(cfg, 40, [(0, 0)], n_self, n_q, 2)


@pytest.mark.parametrize("stride", [1, 2])
def test_decode_kernel_c5_multistream(lib, stride):
    cfg = synth.CONFIGS["c5"]
    check_decode(cfg, 40, [(0, 0), (7, 3), (63, 1)], 48, 1, stride)


def test_decode_kernel_no_sink_and_l_i_zero(lib):
    cfg = synth.CONFIGS["c2"].replace(sink_tokens=0)
    check_decode(cfg, 37, [(0, 0)], 20, 1, 2)
    cfg = synth.CONFIGS["c2"].replace(instant_frames=0, past_frames=6, num_frames=20)
    check_decode(cfg, 15, [(0, 0)], 20, 2, 2)


@pytest.mark.parametrize("stride", [1, 2])
def test_decode_kernel_ids_bit_exact(lib, stride):
    """Every id the decode kernel applied (kv head 0): sink j -> j, kept past + instant ring
    slots -> consecutive ids from A (frames not kept stay untouched), self j -> the ids after
    them, queries the last n_q ids."""
    cfg = synth.CONFIGS["c2"]
    t, n_self, n_q = 44, 70, 2
    ids, R = check_decode(cfg, t, [(0, 0)], n_self, n_q, stride, debug=True)
    blk = ids[0, 0]
    A, tpf = cfg.sink_tokens, cfg.tokens_per_frame
    M = max(cfg.C, max(cfg.query_tokens, n_self))
    sch = step_schedule(cfg, t)
    kept = list(sch.past_frames)[::-1][::stride][::-1]
    assert np.array_equal(blk[:A], np.arange(A))
    frames = kept + list(sch.instant_frames)
    slots = np.concatenate([O.ring_slots(f, tpf, cfg.instant_frames, cfg.past_frames) for f in frames])
    assert np.array_equal(blk[A + slots], A + np.arange(len(slots)))
    touched = np.zeros(R, bool); touched[slots] = True
    assert np.all(blk[A:A + R][~touched] == -1)
    L = A + len(slots)
    assert np.array_equal(blk[A + R:A + R + n_self], L + np.arange(n_self))
    assert np.array_equal(blk[A + R + M:A + R + M + n_q], L + n_self - n_q + np.arange(n_q))


@pytest.mark.parametrize("stride", [2, 3])
def test_decode_sampled_off_the_decode_kernel(lib, stride):
    """The sampled past through the SIMT kernel: fp32 (c1) and bf16 with more than 16 query
    rows per kv head (c2, n_q = 3 -> 21 rows)."""
    check_decode(synth.CONFIGS["c1"].replace(num_frames=40), 19, [(0, 0)], 12, 2, stride)
    check_decode(synth.CONFIGS["c2"], 40, [(0, 0)], 70, 3, stride)


def test_decode_stride_errors(lib):
    cfg = synth.CONFIGS["c1"]
    dsc = D.DSCache.from_config(cfg)
    dev = torch.device("cuda", 0)
    z = torch.zeros(1, 1, cfg.sink_tokens, cfg.num_kv_heads, cfg.head_dim, device=dev)
    f = torch.zeros(1, 1, cfg.tokens_per_frame, cfg.num_kv_heads, cfg.head_dim, device=dev)
    dsc.append_frame(z, z)
    dsc.append_frame(f, f)
    q = torch.zeros(1, 1, 1, cfg.num_q_heads, cfg.head_dim, device=dev)
    kv = torch.zeros(1, 1, 2, cfg.num_kv_heads, cfg.head_dim, device=dev)
    dsc.decode(q, kv, kv)
    with pytest.raises(D.DSCacheError) as e:
        dsc.decode(q, kv, kv, past_stride=0)
    assert e.value.status == D.E_ARG
    dsc.close()
