"""Real-model mode (instant_source = DSCACHE_INSTANT_EXTERNAL) through the
C ABI vs the fp64 oracle: U holds each frame's Eq. 5 K/V (dscache_append_past),
the Eq. 5 attention runs over [sink | zeta(U_{t-1}) | own K/V] (dscache_update_attend),
Eq. 7 and Eq. 8 read the caller's instant K/V (dscache_build_instant_ext / _attend_ext,
PAPER.md:224, 230).  Exact (stream, layer) slots get the seeded synth inputs; every other
slot gets device-side random data through the same launches (isolation check)."""
import numpy as np
import pytest
import torch

import dscache_synth as synth
from oracle import dscache_oracle as O
from oracle.workload import StreamInputs, step_schedule
from tests.gpu_harness import _batch, assert_close
from paper_2605_01858_b200 import dscache as D

pytestmark = pytest.mark.gpu


def _np(x):
    return x.double().numpy()


def run_ext(cfg, capture, exact, l_L=None, impl=D.IMPL_AUTO):
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev)
    gen.manual_seed(4321 + cfg.cfg_id)
    dsc = D.DSCache.from_config(cfg, attn_impl=impl, instant_source=D.INSTANT_EXTERNAL)
    A, tpf, Hkv, Hq, d, lI = (cfg.sink_tokens, cfg.tokens_per_frame, cfg.num_kv_heads, cfg.num_q_heads,
                              cfg.head_dim, cfg.instant_frames)
    if A > 0:
        skv = {sl: synth.sink_kv(cfg, *sl) for sl in exact}
        sk = _batch(cfg, (A, Hkv, d), exact, lambda s, l: skv[(s, l)][0], dev, gen)
        sv = _batch(cfg, (A, Hkv, d), exact, lambda s, l: skv[(s, l)][1], dev, gen)
        dsc.append_frame(sk, sv)
    out = {}
    for t in range(max(capture) + 1):
        e = t - lI
        if e >= 0:
            pk = {sl: synth.past_kv(cfg, *sl, e) for sl in exact}
            kp = _batch(cfg, (tpf, Hkv, d), exact, lambda s, l: pk[(s, l)][0], dev, gen)
            vp = _batch(cfg, (tpf, Hkv, d), exact, lambda s, l: pk[(s, l)][1], dev, gen)
            dsc.append_past(kp, vp)
        else:
            dsc.append_past(None, None)
        st = dsc.state(0)
        C_t = min(t + 1, lI) * tpf
        assert st["instant_tokens"] == C_t and st["frames_seen"] == t + 1
        if t not in capture:
            continue
        rec = {}
        if e >= 0 and l_L is not None:
            qu = _batch(cfg, (tpf, Hq, d), exact, lambda s, l: synth.update_q(cfg, s, l, t), dev, gen)
            rec["upd"] = dsc.update_attend(qu, active_frames=l_L)
        ikv = {sl: synth.instant_kv(cfg, *sl, t, C_t) for sl in exact}
        ki = _batch(cfg, (C_t, Hkv, d), exact, lambda s, l: ikv[(s, l)][0], dev, gen)
        vi = _batch(cfg, (C_t, Hkv, d), exact, lambda s, l: ikv[(s, l)][1], dev, gen)
        if C_t > 0:
            qi = _batch(cfg, (C_t, Hq, d), exact, lambda s, l: synth.instant_q(cfg, s, l, t, C_t), dev, gen)
            rec["inst"] = dsc.build_instant_ext(qi, ki, vi)
        qkv = {sl: synth.query_qkv(cfg, *sl, t, cfg.query_tokens) for sl in exact}
        q = _batch(cfg, (cfg.query_tokens, Hq, d), exact, lambda s, l: qkv[(s, l)][0], dev, gen)
        ks = _batch(cfg, (cfg.query_tokens, Hkv, d), exact, lambda s, l: qkv[(s, l)][1], dev, gen)
        vs = _batch(cfg, (cfg.query_tokens, Hkv, d), exact, lambda s, l: qkv[(s, l)][2], dev, gen)
        rec["o"] = dsc.attend_ext(q, ks, vs, ki, vi)
        torch.cuda.synchronize()
        out[t] = {k: {sl: v[sl].float().cpu() for sl in exact} for k, v in rec.items()}
    impl_used = dsc.attn_impl()
    dsc.close()
    return out, impl_used


def check_ext(cfg, capture, exact, l_L=None, impl=D.IMPL_AUTO):
    res, _ = run_ext(cfg, capture, exact, l_L, impl)
    for t in capture:
        sch = step_schedule(cfg, t)
        for (s, l) in exact:
            inp = StreamInputs(cfg, s, l)
            pkv = lambda f, s=s, l=l: tuple(_np(x) for x in synth.past_kv(cfg, s, l, f))   # noqa: E731
            ki, vi = (_np(x) for x in synth.instant_kv(cfg, s, l, t, sch.C_t))
            if "upd" in res[t]:
                qu = _np(synth.update_q(cfg, s, l, t))
                ref = O.cumulative_update_output(t, cfg.instant_frames, cfg.past_frames, l_L, inp.sink(), pkv,
                                                 qu, cfg.rope_theta, cfg.tokens_per_frame)
                assert_close(res[t]["upd"][(s, l)], ref, cfg.dtype, f"{cfg.name} ext upd t={t} s={s} l={l}")
            if "inst" in res[t]:
                qi = inp.instant_q(t, sch.C_t)
                ref = O.instant_cache_output_ext(sch, inp.sink(), ki, vi, qi, cfg.rope_theta)
                assert_close(res[t]["inst"][(s, l)], ref, cfg.dtype, f"{cfg.name} ext O_inst t={t} s={s} l={l}")
            q, ks, vs = inp.query(t)
            ref = O.attend_output_ext(sch, inp.sink(), pkv, ki, vi, q, ks, vs, cfg.rope_theta)
            assert_close(res[t]["o"][(s, l)], ref, cfg.dtype, f"{cfg.name} ext O t={t} s={s} l={l}")
    return res


def test_ext_c1_fp32_all_steps(lib):
    cfg = synth.CONFIGS["c1"]
    check_ext(cfg, list(range(cfg.num_frames)), [(0, 0)], l_L=cfg.past_frames)


def test_ext_c2_bf16(lib):
    cfg = synth.CONFIGS["c2"]
    check_ext(cfg, [0, 3, 4, 5, 20, 36, 37, 63], [(0, 0)], l_L=cfg.past_frames)


def test_ext_c5_multistream(lib):
    cfg = synth.CONFIGS["c5"]
    check_ext(cfg, [2, 36, 127], [(0, 0), (7, 3), (63, 1)], l_L=8)


@pytest.mark.parametrize("name,t", [("c1", 9), ("c2", 3), ("c2", 40), ("c5", 36)])
def test_ext_decode_parity(lib, name, t):
    """dscache_decode_ext: the last n_q of n_self self tokens over [sink | U (Eq. 5 K/V) |
    the step's instant K/V | self] vs the oracle."""
    cfg = synth.CONFIGS[name]
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev)
    gen.manual_seed(99)
    exact = [(0, 0)] if cfg.num_streams == 1 else [(0, 0), (63, 3)]
    n_self, n_q = cfg.query_tokens + 5, 2
    dsc = D.DSCache.from_config(cfg.replace(query_tokens=n_self), instant_source=D.INSTANT_EXTERNAL)
    A, tpf, Hkv, Hq, d, lI = (cfg.sink_tokens, cfg.tokens_per_frame, cfg.num_kv_heads, cfg.num_q_heads,
                              cfg.head_dim, cfg.instant_frames)
    skv = {sl: synth.sink_kv(cfg, *sl) for sl in exact}
    dsc.append_frame(_batch(cfg, (A, Hkv, d), exact, lambda s, l: skv[(s, l)][0], dev, gen),
                     _batch(cfg, (A, Hkv, d), exact, lambda s, l: skv[(s, l)][1], dev, gen))
    for step in range(t + 1):
        e = step - lI
        if e >= 0:
            pk = {sl: synth.past_kv(cfg, *sl, e) for sl in exact}
            dsc.append_past(_batch(cfg, (tpf, Hkv, d), exact, lambda s, l: pk[(s, l)][0], dev, gen),
                            _batch(cfg, (tpf, Hkv, d), exact, lambda s, l: pk[(s, l)][1], dev, gen))
        else:
            dsc.append_past(None, None)
    C_t = dsc.state(0)["instant_tokens"]
    ikv = {sl: synth.instant_kv(cfg, *sl, t, C_t) for sl in exact}
    ki = _batch(cfg, (C_t, Hkv, d), exact, lambda s, l: ikv[(s, l)][0], dev, gen)
    vi = _batch(cfg, (C_t, Hkv, d), exact, lambda s, l: ikv[(s, l)][1], dev, gen)
    g = torch.Generator().manual_seed(5)
    selfkv = {sl: ((torch.randn(n_self, Hkv, d, generator=g) * cfg.scale).to(cfg.torch_dtype),
                   (torch.randn(n_self, Hkv, d, generator=g) * cfg.scale).to(cfg.torch_dtype),
                   (torch.randn(n_q, Hq, d, generator=g) * cfg.scale).to(cfg.torch_dtype)) for sl in exact}
    ks = _batch(cfg, (n_self, Hkv, d), exact, lambda s, l: selfkv[(s, l)][0], dev, gen)
    vs = _batch(cfg, (n_self, Hkv, d), exact, lambda s, l: selfkv[(s, l)][1], dev, gen)
    q = _batch(cfg, (n_q, Hq, d), exact, lambda s, l: selfkv[(s, l)][2], dev, gen)
    o = dsc.decode_ext(q, ks, vs, ki, vi)
    torch.cuda.synchronize()
    sch = step_schedule(cfg, t)
    for (s, l) in exact:
        inp = StreamInputs(cfg, s, l)
        pkv = lambda f, s=s, l=l: tuple(_np(x) for x in synth.past_kv(cfg, s, l, f))   # noqa: E731
        kk_, vv_ = (_np(x) for x in ikv[(s, l)])
        ref = O.attend_output_ext(sch, inp.sink(), pkv, kk_, vv_, _np(selfkv[(s, l)][2]), _np(selfkv[(s, l)][0]),
                                  _np(selfkv[(s, l)][1]), cfg.rope_theta)
        assert_close(o[s, l].float().cpu(), ref, cfg.dtype, f"{name} decode_ext t={t} s={s} l={l}")
    dsc.close()


def test_ext_differs_from_ring_mode(lib):
    """Negative control: the same ring content read through the default mode (ring K/V
    for the buffer frames) gives a different Eq. 8 answer than the caller's instant K/V."""
    cfg = synth.CONFIGS["c2"]
    t = 20
    res, _ = run_ext(cfg, [t], [(0, 0)])
    inp = StreamInputs(cfg, 0, 0)
    sch = step_schedule(cfg, t)
    pkv = lambda f: tuple(_np(x) for x in synth.past_kv(cfg, 0, 0, f))   # noqa: E731
    q, ks, vs = inp.query(t)
    ki, vi = (_np(x) for x in synth.instant_kv(cfg, 0, 0, t, sch.C_t))
    right = O.attend_output_ext(sch, inp.sink(), pkv, ki, vi, q, ks, vs, cfg.rope_theta)
    wrong = O.attend_output(sch, inp.sink(), pkv, q, ks, vs, cfg.rope_theta)
    g = res[t]["o"][(0, 0)].double().numpy()
    assert np.linalg.norm(g - wrong) > 5 * np.linalg.norm(g - right)


def test_ext_mode_errors(lib):
    cfg = synth.CONFIGS["c2"]
    h = D.DSCache.from_config(cfg, instant_source=D.INSTANT_EXTERNAL)
    x = torch.zeros(1, 1, cfg.tokens_per_frame, cfg.num_kv_heads, cfg.head_dim, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(D.DSCacheError) as e:
        h.append_past(None, None)                    # sink first
    assert e.value.status == D.E_STATE
    s = torch.zeros(1, 1, cfg.sink_tokens, cfg.num_kv_heads, cfg.head_dim, dtype=torch.bfloat16, device="cuda")
    h.append_frame(s, s)
    with pytest.raises(D.DSCacheError) as e:
        h.append_frame(x, x)                         # frames enter via append_past in this mode
    assert e.value.status == D.E_CONFIG
    with pytest.raises(D.DSCacheError) as e:
        h.append_past(x, x)                          # nothing leaves the buffer at step 0
    assert e.value.status == D.E_ARG
    h.append_past(None, None)
    q = torch.zeros(1, 1, 4, cfg.num_q_heads, cfg.head_dim, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(D.DSCacheError) as e:
        kv = q[:, :, :, :cfg.num_kv_heads].contiguous()
        h.attend(q, kv, kv)
    assert e.value.status == D.E_CONFIG
    h.close()
    r = D.DSCache.from_config(cfg)
    r.append_frame(s, s)
    with pytest.raises(D.DSCacheError) as e:
        r.append_past(None, None)
    assert e.value.status == D.E_CONFIG
    r.close()
