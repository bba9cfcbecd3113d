"""Checkpoint / resume on the GPU ("bit-exact round trip").

A handle snapshotted after T1 steps and restored into a fresh handle of the same config
must (1) report the same counters (dscache_get_state), (2) hold the same ring and sink
bytes, slot for slot, and (3) produce bit-identical outputs to the uninterrupted handle
for the following steps (same kernels, same inputs).  The uninterrupted handle is itself
oracle-parity-tested (test_gpu_parity.py); the restore is checked across the ring wrap
(eviction active) and from before the first frame.
"""
import pytest
import torch

import dscache_synth as synth
from paper_2605_01858_b200 import dscache as D

pytestmark = pytest.mark.gpu


def _inputs(cfg, t, gen, dev, dt):
    S, N, tpf, Hq, Hkv, d = (cfg.num_streams, cfg.num_layers, cfg.tokens_per_frame, cfg.num_q_heads,
                             cfg.num_kv_heads, cfg.head_dim)
    C_t = min(t + 1, cfg.instant_frames) * tpf
    n_q = cfg.query_tokens

    def r(*shape):
        return (torch.randn(shape, generator=gen, device=dev, dtype=torch.float32) * cfg.scale).to(dt)
    return (r(S, N, tpf, Hkv, d), r(S, N, tpf, Hkv, d), r(S, N, C_t, Hq, d),
            r(S, N, n_q, Hq, d), r(S, N, n_q, Hkv, d), r(S, N, n_q, Hkv, d))


def _run(handles, cfg, t0, t1, gen, dev, fused):
    outs = []
    for t in range(t0, t1):
        k, v, qi, q, ks, vs = _inputs(cfg, t, gen, dev, handles[0].torch_dtype)
        step = []
        for h in handles:
            if fused:
                oi, o = h.step(k, v, qi, q, ks, vs)
            else:
                h.append_frame(k, v)
                oi = h.build_instant(qi)
                o = h.attend(q, ks, vs)
            step.append((oi.clone(), o.clone()))
        outs.append(step)
    torch.cuda.synchronize()
    return outs


def _sink(cfg, h, gen, dev):
    if cfg.sink_tokens == 0:
        return
    shape = (cfg.num_streams, cfg.num_layers, cfg.sink_tokens, cfg.num_kv_heads, cfg.head_dim)
    sk = (torch.randn(shape, generator=gen, device=dev) * cfg.scale).to(h.torch_dtype)
    sv = (torch.randn(shape, generator=gen, device=dev) * cfg.scale).to(h.torch_dtype)
    h.append_frame(sk, sv)


CASES = {
    "c1": synth.CONFIGS["c1"],
    "c2": synth.CONFIGS["c2"],
    "c2_multi": synth.CONFIGS["c2"].replace(name="c2_multi", num_streams=3, num_layers=2, past_frames=6,
                                            instant_frames=2, query_tokens=16),
}


@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("name,t_snap", [("c1", 7), ("c1", 0), ("c2", 40), ("c2_multi", 11), ("c2_multi", 0)])
def test_snapshot_restore_resumes_bit_exact(lib, name, t_snap, fused):
    cfg = CASES[name]
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev)
    gen.manual_seed(77 + t_snap)
    a = D.DSCache.from_config(cfg)
    _sink(cfg, a, gen, dev)
    _run([a], cfg, 0, t_snap, gen, dev, fused)
    blob = a.snapshot()
    b = D.DSCache.from_config(cfg)
    b.restore(blob)
    for l in range(cfg.num_layers):
        assert b.state(l) == a.state(l), f"layer {l}"
    for s in range(cfg.num_streams):
        for l in range(cfg.num_layers):
            for x, y in zip(a.copy_ring(s, l) + a.copy_sink(s, l), b.copy_ring(s, l) + b.copy_sink(s, l)):
                assert torch.equal(x.view(torch.int16) if x.dtype == torch.bfloat16 else x.view(torch.int32),
                                   y.view(torch.int16) if y.dtype == torch.bfloat16 else y.view(torch.int32))
    assert b.snapshot() == blob
    n_more = cfg.past_frames + cfg.instant_frames + 2          # past the next wrap of the ring
    outs = _run([a, b], cfg, t_snap, t_snap + n_more, gen, dev, fused)
    for t, ((oa_i, oa), (ob_i, ob)) in enumerate(outs):
        assert torch.equal(oa_i, ob_i), f"O_inst differs {t_snap + t} steps in"
        assert torch.equal(oa, ob), f"O differs {t_snap + t} steps in"
    for l in range(cfg.num_layers):
        assert b.state(l) == a.state(l)
    # decode (NEXT-2) over the resumed cache, dense and with the 0.5 FPS past stride
    S, N, Hq, Hkv, d = cfg.num_streams, cfg.num_layers, cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim
    n_self = cfg.query_tokens + 5
    dt = a.torch_dtype
    ks = torch.randn((S, N, n_self, Hkv, d), generator=gen, device=dev).to(dt)
    vs = torch.randn((S, N, n_self, Hkv, d), generator=gen, device=dev).to(dt)
    q = torch.randn((S, N, 1, Hq, d), generator=gen, device=dev).to(dt)
    for stride in (1, 2):
        assert torch.equal(a.decode(q, ks, vs, past_stride=stride), b.decode(q, ks, vs, past_stride=stride))


def test_restore_rejects_other_config(lib):
    cfg = CASES["c2_multi"]
    a = D.DSCache.from_config(cfg)
    blob = a.snapshot()
    b = D.DSCache.from_config(cfg.replace(past_frames=7))
    with pytest.raises(ValueError):
        b.restore(blob)


def test_set_state_validation(lib):
    cfg = CASES["c2_multi"]
    h = D.DSCache.from_config(cfg)
    with pytest.raises(D.DSCacheError) as e:
        h.set_state(0, 3, 0)                      # frames without a sink
    assert e.value.status == D.E_STATE
    with pytest.raises(D.DSCacheError) as e:
        h.set_state(cfg.num_layers, 0, 0)
    assert e.value.status == D.E_ARG
    with pytest.raises(D.DSCacheError) as e:
        h.set_state(0, -1, 1)
    assert e.value.status == D.E_ARG
    h.set_state(0, 9, 1)                           # closed form of the counters (Eq. 3/6)
    st = h.state(0)
    lI, lU, tpf = cfg.instant_frames, cfg.past_frames, cfg.tokens_per_frame
    assert st["frames_seen"] == 9 and st["last_evicted_frame"] == 9 - 1 - lI - lU
    assert st["instant_tokens"] == lI * tpf and st["past_tokens"] == lU * tpf


@pytest.mark.parametrize("t_snap", [2, 9])
def test_snapshot_restore_external_instant_mode(lib, t_snap):
    """Real-model mode (NEXT-1): U holds the caller's Eq. 5 K/V (append_past); a restored
    handle resumes update_attend / build_instant_ext / attend_ext bit-identically."""
    cfg = CASES["c2_multi"]
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev)
    gen.manual_seed(991 + t_snap)
    S, N, tpf, Hq, Hkv, d, lI, nq = (cfg.num_streams, cfg.num_layers, cfg.tokens_per_frame, cfg.num_q_heads,
                                     cfg.num_kv_heads, cfg.head_dim, cfg.instant_frames, cfg.query_tokens)
    dt = torch.bfloat16

    def r(*shape):
        return (torch.randn(shape, generator=gen, device=dev) * cfg.scale).to(dt)

    def advance(hs, t):
        e = t - lI
        if e >= 0:
            kp, vp = r(S, N, tpf, Hkv, d), r(S, N, tpf, Hkv, d)
            for h in hs:
                h.append_past(kp, vp)
        else:
            for h in hs:
                h.append_past(None, None)
        C_t = min(t + 1, lI) * tpf
        qi, ki, vi = r(S, N, C_t, Hq, d), r(S, N, C_t, Hkv, d), r(S, N, C_t, Hkv, d)
        q, ks, vs = r(S, N, nq, Hq, d), r(S, N, nq, Hkv, d), r(S, N, nq, Hkv, d)
        qu = r(S, N, tpf, Hq, d) if e >= 0 else None
        res = []
        for h in hs:
            out = [h.build_instant_ext(qi, ki, vi).clone(), h.attend_ext(q, ks, vs, ki, vi).clone()]
            if qu is not None:
                out.append(h.update_attend(qu, active_frames=cfg.past_frames).clone())
            res.append(out)
        return res

    a = D.DSCache.from_config(cfg, instant_source=D.INSTANT_EXTERNAL)
    _sink(cfg, a, gen, dev)
    for t in range(t_snap):
        advance([a], t)
    torch.cuda.synchronize()
    b = D.DSCache.from_config(cfg, instant_source=D.INSTANT_EXTERNAL)
    b.restore(a.snapshot())
    for t in range(t_snap, t_snap + cfg.past_frames + lI + 2):
        ra, rb = advance([a, b], t)
        torch.cuda.synchronize()
        for x, y in zip(ra, rb):
            assert torch.equal(x, y), f"step {t}"
