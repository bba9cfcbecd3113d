"""GPU parity of the CUDA path (through the C ABI) against the fp64 oracle.

Bar (BASELINE.json north_star): ring slots, eviction order and position ids
bit-exact; fp32 configs max abs <= 1e-4; bf16 configs max abs <= 2e-2 AND
relative L2 <= 5e-3 (the binding check, SURVEY §8(c) "Tolerances"), per
(step, stream, layer, output kind).
"""
import numpy as np
import pytest
import torch

import dscache_synth as synth
from oracle import dscache_oracle as O
from oracle.workload import StreamInputs, expected_ring, oracle_step, step_schedule
from tests.gpu_harness import assert_close, errors, run_stream
from paper_2605_01858_b200 import dscache as D

pytestmark = pytest.mark.gpu

REPORT = []


def _check_steps(cfg, res, steps, exact, style=O.SPLIT_HALF, tag=""):
    for t in steps:
        for (s, l) in exact:
            sch, o_inst, o = oracle_step(cfg, s, l, t, style=style)
            g_inst, g_o = res[t][(s, l)]
            if sch.C_t > 0:
                ma, rl = assert_close(g_inst, o_inst, cfg.dtype, f"{tag} O_inst t={t} s={s} l={l}")
                REPORT.append((cfg.name + tag, "O_inst", t, s, l, ma, rl))
            ma, rl = assert_close(g_o, o, cfg.dtype, f"{tag} O t={t} s={s} l={l}")
            REPORT.append((cfg.name + tag, "O", t, s, l, ma, rl))


def test_c1_fp32_all_steps(lib):
    cfg = synth.CONFIGS["c1"]
    steps = list(range(cfg.num_frames))
    res = run_stream(cfg, steps, [(0, 0)])
    assert res["impl"] == {"build_instant": "simt", "attend": "simt"}
    _check_steps(cfg, res, steps, [(0, 0)])


def test_c1_adjacent_rope_style(lib):
    cfg = synth.CONFIGS["c1"]
    steps = [0, 5, 19]
    dev_cfg = cfg
    res = run_stream_style(dev_cfg, steps, D.ROPE_ADJACENT)
    _check_steps(cfg, res, steps, [(0, 0)], style=O.ADJACENT, tag="-adj")


def run_stream_style(cfg, steps, style):
    # same as run_stream, through a handle created with the adjacent-pair RoPE flag
    orig = D.DSCache.from_config

    def patched(c, device=0, **kw):
        kw["rope_style"] = style
        return orig(c, device, **kw)
    D.DSCache.from_config = patched
    try:
        return run_stream(cfg, steps, [(0, 0)])
    finally:
        D.DSCache.from_config = orig


def test_c2_bf16_tcgen05(lib):
    cfg = synth.CONFIGS["c2"]
    steps = [0, 1, 3, 4, 35, 36, 37, 63]
    res = run_stream(cfg, steps, [(0, 0)])
    assert res["impl"] == {"build_instant": "tcgen05", "attend": "tcgen05"}
    _check_steps(cfg, res, steps, [(0, 0)])


def test_c2_bf16_simt_crosscheck(lib):
    cfg = synth.CONFIGS["c2"]
    steps = [3, 40]
    res = run_stream(cfg, steps, [(0, 0)], impl=D.IMPL_SIMT)
    assert res["impl"] == {"build_instant": "simt", "attend": "simt"}
    _check_steps(cfg, res, steps, [(0, 0)], tag="-simt")


def test_zero_output_negative_control(lib):
    # an all-zero output must FAIL the bf16 bar (rel L2 = 1): the tolerance is not vacuous
    cfg = synth.CONFIGS["c2"]
    sch, o_inst, o = oracle_step(cfg, 0, 0, 40)
    with pytest.raises(AssertionError):
        assert_close(torch.zeros(o.shape), o, "bf16", "zero control")
    # and off-by-one positions / a dropped sink in the reference must be detected too
    res = run_stream(cfg, [40], [(0, 0)])
    g_inst, g_o = res[40][(0, 0)]
    inp = StreamInputs(cfg, 0, 0)
    q, ks, vs = inp.query(40)
    sink = inp.sink()
    shifted = O.attend_output(sch, sink, inp.frame_kv, q, ks, vs, cfg.rope_theta)   # correct
    assert errors(g_o, shifted)[1] < 5e-3
    # reference with every id + 1 for the keys only (relative distances broken by one)
    frames = sch.past_frames + sch.instant_frames
    kk = np.concatenate([sink[0]] + [inp.frame_kv(f)[0] for f in frames] + [ks])
    vv = np.concatenate([sink[1]] + [inp.frame_kv(f)[1] for f in frames] + [vs])
    pk = np.arange(len(kk))
    bad = O.gqa_attention(q, pk[-len(q):], kk, vv, pk + 1, cfg.rope_theta)
    assert errors(g_o, bad)[1] > 5e-3
    nosink = O.gqa_attention(q, pk[-len(q):] - cfg.sink_tokens, kk[cfg.sink_tokens:], vv[cfg.sink_tokens:],
                             pk[cfg.sink_tokens:] - cfg.sink_tokens, cfg.rope_theta)
    assert errors(g_o, nosink)[1] > 5e-3


def test_ring_slots_sink_and_eviction_bit_exact(lib):
    for name, steps in (("c1", [0, 4, 5, 13, 19]), ("c2", [0, 36, 37, 50])):
        cfg = synth.CONFIGS[name]
        res = run_stream(cfg, steps, [(0, 0)], ring_capture=[(0, 0)])
        inp = StreamInputs(cfg, 0, 0)
        for t in steps:
            k, v = res["ring"][(t, 0, 0)]
            sch = step_schedule(cfg, t)
            exp = expected_ring(cfg, sch, inp)
            st = res["state"][t]
            assert st["past_tokens"] == sch.P_t and st["instant_tokens"] == sch.C_t
            assert st["last_evicted_frame"] == (sch.evicted[0] if sch.evicted else -1)
            for slot, (ek, ev) in exp.items():
                assert torch.equal(k[:, slot].double(), torch.from_numpy(ek)), (name, t, slot)
                assert torch.equal(v[:, slot].double(), torch.from_numpy(ev)), (name, t, slot)
        sk, sv = res["sink"][(0, 0)]
        ek, ev = inp.sink()
        assert torch.equal(sk.double(), torch.from_numpy(ek).permute(1, 0, 2))
        assert torch.equal(sv.double(), torch.from_numpy(ev).permute(1, 0, 2))


def test_poison_evicted_slots_and_outputs_unchanged(lib):
    cfg = synth.CONFIGS["c2"]
    steps = [40, 41]
    clean = run_stream(cfg, steps, [(0, 0)])
    pois = run_stream(cfg, steps, [(0, 0)], poison=True, ring_capture=[(0, 0)])
    for t in steps:
        assert torch.equal(clean[t][(0, 0)][1], pois[t][(0, 0)][1])
        assert torch.equal(clean[t][(0, 0)][0], pois[t][(0, 0)][0])
        sch = step_schedule(cfg, t)
        ev = sch.evicted[0]
        slots = O.ring_slots(ev, cfg.tokens_per_frame, cfg.instant_frames, cfg.past_frames)
        k, _ = pois["ring"][(t, 0, 0)]
        assert torch.all(k[:, slots].float() > 1e29)


def _check_ids(cfg, dbg_b, dbg_a, t, what=""):
    """Bit-exact position ids one (stream, layer) applied at step t (its debug block)."""
    R = (cfg.past_frames + cfg.instant_frames + 1) * cfg.tokens_per_frame
    A = cfg.sink_tokens
    M = max(cfg.C, cfg.query_tokens)
    sch = step_schedule(cfg, t)
    bk, bq, ak, aq = O.position_ids(sch, cfg.query_tokens)
    # attend: sink ids, ring slot -> id, self ids, query ids
    assert np.array_equal(dbg_a[:A], ak[:A]), what
    frames = sch.past_frames + sch.instant_frames
    slots = np.concatenate([O.ring_slots(f, cfg.tokens_per_frame, cfg.instant_frames, cfg.past_frames)
                            for f in frames])
    assert np.array_equal(dbg_a[A + slots], ak[A:A + len(slots)]), what
    in_window = np.zeros(R, bool); in_window[slots] = True
    assert np.all(dbg_a[A:A + R][~in_window] == -1), what
    nq = cfg.query_tokens
    assert np.array_equal(dbg_a[A + R:A + R + nq], ak[A + len(slots):]), what
    assert np.array_equal(dbg_a[A + R + M:A + R + M + nq], aq), what
    # build: sink ids, instant slots -> A + i, query ids A + i
    islots = np.concatenate([O.ring_slots(f, cfg.tokens_per_frame, cfg.instant_frames, cfg.past_frames)
                             for f in sch.instant_frames])
    assert np.array_equal(dbg_b[:A], bk[:A]), what
    assert np.array_equal(dbg_b[A + islots], bk[A:]), what
    assert np.array_equal(dbg_b[A + R + M:A + R + M + sch.C_t], bq), what


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_debug_position_ids_bit_exact(lib, name):
    cfg = synth.CONFIGS[name]
    steps = [0, 3, 37] if name == "c2" else [0, 3, 7, 19]
    res = run_stream(cfg, steps, [(0, 0)], debug=True)
    for t in steps:
        dbg_b, dbg_a = (x[0, 0] for x in res["dbg"][t])
        _check_ids(cfg, dbg_b, dbg_a, t, f"{name} t={t}")


@pytest.mark.parametrize("name,steps,exact", [
    # the bench's own path: dscache_step (one fused launch, staged pre-rotated build window)
    ("c5", [0, 35, 36, 127], [(0, 0), (0, 3), (7, 0), (7, 3), (63, 0), (63, 3)]),
    ("c3", [0, 71, 72, 255], [(0, 0), (0, 13), (0, 27)]),
])
def test_fused_step_ring_eviction_ids_bit_exact(lib, name, steps, exact):
    """Ring slot contents, eviction bookkeeping and every applied position id, bit-exact,
    through dscache_step on the configurations the bench times (c5: 64 streams x 4 layers;
    c3: 28 layers), plus value parity of the same fused steps."""
    cfg = synth.CONFIGS[name]
    res = run_stream(cfg, steps, exact, fused=True, debug=True, ring_capture=exact)
    _check_steps(cfg, res, steps, exact, tag="-fused-exact")
    for t in steps:
        sch = step_schedule(cfg, t)
        st = res["state"][t]
        assert st["past_tokens"] == sch.P_t and st["instant_tokens"] == sch.C_t
        assert st["last_evicted_frame"] == (sch.evicted[0] if sch.evicted else -1)
        dbg_b, dbg_a = res["dbg"][t]
        for (s, l) in exact:
            _check_ids(cfg, dbg_b[s, l], dbg_a[s, l], t, f"{name} t={t} s={s} l={l}")
            exp = expected_ring(cfg, sch, StreamInputs(cfg, s, l))
            slots = np.array(sorted(exp))
            ek = np.stack([exp[int(x)][0] for x in slots], axis=1)   # [Hkv, n, d]
            ev = np.stack([exp[int(x)][1] for x in slots], axis=1)
            k, v = res["ring"][(t, s, l)]
            assert np.array_equal(k[:, slots].double().numpy(), ek), (name, t, s, l)
            assert np.array_equal(v[:, slots].double().numpy(), ev), (name, t, s, l)
        # every other (stream, layer) applied the same ids (kv head 0 of each block)
        ref_b, ref_a = dbg_b[exact[0]], dbg_a[exact[0]]
        assert np.array_equal(dbg_a.reshape(-1, dbg_a.shape[-1]), np.broadcast_to(ref_a, (dbg_a.shape[0] * dbg_a.shape[1], ref_a.shape[0])))
        assert np.array_equal(dbg_b.reshape(-1, dbg_b.shape[-1]), np.broadcast_to(ref_b, (dbg_b.shape[0] * dbg_b.shape[1], ref_b.shape[0])))


def test_decoupling_instant_independent_of_past(lib):
    # Eq. 7: O_inst bitwise unchanged when every past frame holds other data
    cfg = synth.CONFIGS["c2"]
    t = 45
    sch = step_schedule(cfg, t)
    gen = torch.Generator().manual_seed(7)

    def override(s, l, f):
        if f in sch.instant_frames:
            return None
        shp = (cfg.tokens_per_frame, cfg.num_kv_heads, cfg.head_dim)
        return ((torch.randn(shp, generator=gen) * 3).to(torch.bfloat16),
                (torch.randn(shp, generator=gen) * 3).to(torch.bfloat16))
    a = run_stream(cfg, [t], [(0, 0)])
    b = run_stream(cfg, [t], [(0, 0)], past_override=override)
    assert torch.equal(a[t][(0, 0)][0], b[t][(0, 0)][0])
    assert not torch.equal(a[t][(0, 0)][1], b[t][(0, 0)][1])


@pytest.mark.parametrize("variant", ["no_sink", "lI0_uniform", "lU0_window", "layerwise"])
def test_edge_configs_tcgen05(lib, variant):
    base = synth.CONFIGS["c2"].replace(tokens_per_frame=128, past_frames=6, instant_frames=3, num_frames=16,
                                       query_tokens=37, num_layers=2)
    if variant == "no_sink":
        cfg = base.replace(sink_tokens=0)
    elif variant == "lI0_uniform":
        cfg = base.replace(instant_frames=0)
    elif variant == "lU0_window":
        cfg = base.replace(past_frames=0)
    else:
        cfg = base
    steps = [0, 2, 9, 10, 15]
    res = run_stream(cfg, steps, [(0, 0), (0, 1)], layer_by_layer=(variant == "layerwise"))
    assert res["impl"]["attend"] == "tcgen05"
    _check_steps(cfg, res, steps, [(0, 0), (0, 1)], tag="-" + variant)


@pytest.mark.parametrize("variant", ["odd_tpf_wrap", "big_sink_multi_extra", "tiny_frames"])
def test_logical_tiles_mirror_and_narrow_widths(lib, variant):
    """64-key logical window tiles read through the ring's mirror rows (windows that wrap
    around slot R-1), tile widths that are not multiples of 64 (narrow QK^T N / PV K),
    several sink+self tiles, and the tcgen05 path for tpf < 64 (any tpf is eligible)."""
    base = synth.CONFIGS["c2"].replace(num_frames=17, num_layers=1)
    if variant == "odd_tpf_wrap":        # R = 8 * 40 = 320 slots: the window wraps every few steps
        cfg = base.replace(tokens_per_frame=40, sink_tokens=3, past_frames=5, instant_frames=2, query_tokens=21)
    elif variant == "big_sink_multi_extra":   # A + q = 134 > 2 tiles of sink/self keys
        cfg = base.replace(tokens_per_frame=100, sink_tokens=70, past_frames=3, instant_frames=2, query_tokens=64)
    else:                                 # 24-token frames: every tile narrow or partial
        cfg = base.replace(tokens_per_frame=24, sink_tokens=5, past_frames=4, instant_frames=3, query_tokens=9)
    steps = list(range(0, cfg.num_frames, 2)) + [cfg.num_frames - 1]
    res = run_stream(cfg, steps, [(0, 0)])
    assert res["impl"] == {"build_instant": "tcgen05", "attend": "tcgen05"}
    _check_steps(cfg, res, steps, [(0, 0)], tag="-" + variant)


def test_c3_28_layers_sampled(lib):
    cfg = synth.CONFIGS["c3"]
    steps = [0, 7, 8, 71, 72, 100, 255]
    exact = [(0, 0), (0, 13), (0, 27)]
    res = run_stream(cfg, steps, exact)
    _check_steps(cfg, res, steps, exact)


def test_c4_long_stream_sampled(lib):
    cfg = synth.CONFIGS["c4"]
    steps = [0, 8, 136, 272, 1000, 2047, 4095]
    res = run_stream(cfg, steps, [(0, 0)], debug=True)
    _check_steps(cfg, res, steps, [(0, 0)])
    dbg_b, dbg_a = res["dbg"][4095]
    assert dbg_a[0, 0].max() == 26723 and dbg_a.max() < cfg.max_position


def test_c5_multistream_sampled(lib):
    cfg = synth.CONFIGS["c5"]
    steps = [0, 35, 36, 127]
    exact = [(0, 0), (7, 3), (63, 0), (63, 3)]
    res = run_stream(cfg, steps, exact)
    _check_steps(cfg, res, steps, exact)


@pytest.mark.parametrize("name,steps,exact", [
    ("c2", [0, 3, 4, 36, 37, 63], [(0, 0)]),
    ("c5", [0, 36, 127], [(0, 0), (63, 3)]),
    # c3 / c4: the fused launch runs on list-scheduled per-CTA work lists
    ("c3", [0, 9, 75], [(0, 0), (0, 27)]),
    ("c4", [0, 140], [(0, 0)]),
])
def test_fused_step_parity_and_bitwise_equal_to_three_calls(lib, name, steps, exact):
    # dscache_step = append + build_instant + attend in one persistent tcgen05 launch:
    # within the bar against the oracle AND bitwise equal to the three separate calls
    cfg = synth.CONFIGS[name]
    fused = run_stream(cfg, steps, exact, fused=True)
    _check_steps(cfg, fused, steps, exact, tag="-fused")
    sep = run_stream(cfg, steps, exact)
    for t in steps:
        for sl in exact:
            a, b = fused[t][sl], sep[t][sl]
            assert torch.equal(a[1], b[1]), (t, sl)
            assert (a[0] is None) == (b[0] is None) and (a[0] is None or torch.equal(a[0], b[0])), (t, sl)


@pytest.mark.parametrize("variant", ["no_sink", "lI0_uniform", "lU0_window", "small_multi"])
def test_fused_step_edge_configs(lib, variant):
    base = synth.CONFIGS["c2"].replace(tokens_per_frame=128, past_frames=6, instant_frames=3, num_frames=16,
                                       query_tokens=37, num_layers=2)
    cfg = {"no_sink": base.replace(sink_tokens=0), "lI0_uniform": base.replace(instant_frames=0),
           "lU0_window": base.replace(past_frames=0),
           "small_multi": base.replace(num_streams=3, query_tokens=1)}[variant]
    exact = [(0, 0), (cfg.num_streams - 1, 1)]
    steps = [0, 2, 9, 10, 15]
    res = run_stream(cfg, steps, exact, fused=True)
    _check_steps(cfg, res, steps, exact, tag="-fused-" + variant)


def test_errors_through_the_abi(lib):
    cfg = synth.CONFIGS["c2"]
    with pytest.raises(D.DSCacheError) as e:
        D.DSCache.from_config(cfg, max_position=7000)
    assert e.value.status == D.E_POS_OVERFLOW
    h = D.DSCache.from_config(cfg)
    q = torch.zeros(1, 1, 64, 28, 128, dtype=torch.bfloat16, device="cuda")
    kv = torch.zeros(1, 1, 64, 4, 128, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(D.DSCacheError) as e:
        h.attend(q, kv, kv)
    assert e.value.status == D.E_STATE
    bad = torch.zeros(1, 1, 5, 4, 128, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(D.DSCacheError) as e:
        h.append_frame(bad, bad)
    assert e.value.status == D.E_ARG
    h.close()




@pytest.mark.parametrize("name,l_L,steps", [("c2", 32, [4, 5, 20, 36, 37, 50]), ("c2", 8, [4, 12, 40]),
                                           ("c5", 32, [4, 35, 36, 127])])
def test_update_attend_eq5_parity(lib, name, l_L, steps):
    # NEXT-1: attention inside phi(X_{t-l_I}, [C_a, zeta(U_{t-1})]) (Eq. 5), through the ABI
    cfg = synth.CONFIGS[name]
    exact = [(0, 0)] if name == "c2" else [(0, 0), (63, 3)]
    res = run_stream(cfg, steps, exact, update_lL=l_L)
    for t in steps:
        for (s, l) in exact:
            inp = StreamInputs(cfg, s, l)
            qu = synth.update_q(cfg, s, l, t).double().numpy()
            ref = O.cumulative_update_output(t, cfg.instant_frames, cfg.past_frames, l_L, inp.sink(), inp.frame_kv,
                                             qu, cfg.rope_theta, cfg.tokens_per_frame)
            ma, rl = assert_close(res["upd"][t][(s, l)], ref, cfg.dtype, f"upd t={t} s={s} l={l} lL={l_L}")
            REPORT.append((cfg.name + "-upd", "O_upd", t, s, l, ma, rl))


def test_update_attend_simt_paths(lib):
    # fp32 config (SIMT kernel) and l_I = 0 (window may fill the ring: SIMT kernel)
    for cfg, l_L in ((synth.CONFIGS["c1"], 3), (synth.CONFIGS["c2"].replace(instant_frames=0, tokens_per_frame=128,
                                                                              past_frames=6, num_frames=12), 6)):
        steps = [2, 7, 11]
        res = run_stream(cfg, steps, [(0, 0)], update_lL=l_L)
        for t in steps:
            inp = StreamInputs(cfg, 0, 0)
            qu = synth.update_q(cfg, 0, 0, t).double().numpy()
            ref = O.cumulative_update_output(t, cfg.instant_frames, cfg.past_frames, l_L, inp.sink(), inp.frame_kv,
                                             qu, cfg.rope_theta, cfg.tokens_per_frame)
            ma, rl = assert_close(res["upd"][t][(0, 0)], ref, cfg.dtype, f"upd {cfg.name} t={t}")
            REPORT.append((cfg.name + "-upd", "O_upd", t, 0, 0, ma, rl))




@pytest.mark.parametrize("n_self,n_q", [(64 + 1, 1), (64 + 40, 1), (300, 5), (64, 64)])
def test_decode_parity(lib, n_self, n_q):
    # NEXT-2: the last n_q tokens of [query chunk | generated] over [sink|past|instant|self]
    import torch as _t
    cfg = synth.CONFIGS["c2"].replace(num_frames=40)
    t = 39
    dev = _t.device("cuda", 0)
    h = D.DSCache.from_config(cfg)
    sk, sv = synth.sink_kv(cfg, 0, 0)
    h.append_frame(sk[None, None].to(dev), sv[None, None].to(dev))
    for f in range(t + 1):
        k, v = synth.frame_kv(cfg, 0, 0, f)
        h.append_frame(k[None, None].to(dev), v[None, None].to(dev))
    g = _t.Generator().manual_seed(n_self)
    ks = (_t.randn(n_self, 4, 128, generator=g) * 0.5).to(_t.bfloat16)
    vs = (_t.randn(n_self, 4, 128, generator=g) * 0.5).to(_t.bfloat16)
    q = (_t.randn(n_q, 28, 128, generator=g) * 0.5).to(_t.bfloat16)
    o = h.decode(q[None, None].to(dev), ks[None, None].to(dev), vs[None, None].to(dev))
    _t.cuda.synchronize()
    inp = StreamInputs(cfg, 0, 0)
    ref = O.decode_output(step_schedule(cfg, t), inp.sink(), inp.frame_kv, q.double().numpy(), ks.double().numpy(),
                          vs.double().numpy(), cfg.rope_theta)
    ma, rl = assert_close(o[0, 0].float().cpu(), ref, "bf16", f"decode n_self={n_self} n_q={n_q}")
    REPORT.append(("c2-decode", "O_dec", t, n_self, n_q, ma, rl))
    h.close()




@pytest.mark.parametrize("n_parts", [2, 3, 8])
def test_context_parallel_partials_combine(lib, n_parts):
    """NEXT-4 building blocks: the attend split into n_parts key ranges (dscache_attend_partial),
    merged by dscache_combine_partials == the oracle attend; also == dscache_attend up to
    rounding.  8 parts = the 8-GPU context split of one stream (P3)."""
    import torch as _t
    cfg = synth.CONFIGS["c5"].replace(num_streams=2, num_layers=2, num_frames=40)
    t = 39
    dev = _t.device("cuda", 0)
    h = D.DSCache.from_config(cfg)
    S, N = cfg.num_streams, cfg.num_layers
    sink = [[synth.sink_kv(cfg, s, l) for l in range(N)] for s in range(S)]
    h.append_frame(_t.stack([_t.stack([sink[s][l][0] for l in range(N)]) for s in range(S)]).to(dev),
                   _t.stack([_t.stack([sink[s][l][1] for l in range(N)]) for s in range(S)]).to(dev))
    for f in range(t + 1):
        kv = [[synth.frame_kv(cfg, s, l, f) for l in range(N)] for s in range(S)]
        h.append_frame(_t.stack([_t.stack([kv[s][l][0] for l in range(N)]) for s in range(S)]).to(dev),
                       _t.stack([_t.stack([kv[s][l][1] for l in range(N)]) for s in range(S)]).to(dev))
    qkv = [[synth.query_qkv(cfg, s, l, t) for l in range(N)] for s in range(S)]
    q, ks, vs = (_t.stack([_t.stack([qkv[s][l][i] for l in range(N)]) for s in range(S)]).to(dev) for i in range(3))
    parts = [h.attend_partial(q, ks, vs, r, n_parts) for r in range(n_parts)]
    o = h.combine_partials(_t.stack([p[0] for p in parts]), _t.stack([p[1] for p in parts]))
    o_full = h.attend(q, ks, vs)
    _t.cuda.synchronize()
    for s in range(S):
        for l in range(N):
            _, _, ref = oracle_step(cfg, s, l, t)
            ma, rl = assert_close(o[s, l].float().cpu(), ref, "bf16", f"context-parallel {n_parts} parts s={s} l={l}")
            REPORT.append((f"c5-cp{n_parts}", "O", t, s, l, ma, rl))
    diff = (o.float() - o_full.float()).norm() / o_full.float().norm()
    assert diff.item() < 5e-3, diff.item()
    with pytest.raises(D.DSCacheError):
        h.attend_partial(q, ks, vs, 0, 10_000)          # parts without keys are refused
    h.close()


@pytest.mark.parametrize("name", ["c1", "c2", "c5"])
def test_build_instant_newest_parity(lib, name):
    # NEXT-3: the incremental instant rows == the last tpf rows of the exact Eq. 7 build
    import torch as _t
    cfg = synth.CONFIGS[name]
    steps = [0, 2, 3, 10, cfg.num_frames - 1]
    dev = _t.device("cuda", 0)
    exact = [(0, 0)] if cfg.num_streams == 1 else [(0, 0), (63, 3)]
    h = D.DSCache.from_config(cfg)
    S, N, tpf = cfg.num_streams, cfg.num_layers, cfg.tokens_per_frame
    def batch(fn, shape):
        t_ = (_t.randn((S, N) + shape, device=dev) * cfg.scale).to(cfg.torch_dtype)
        for (s_, l_) in exact:
            t_[s_, l_] = fn(s_, l_).to(dev)
        return t_
    shp = (cfg.sink_tokens, cfg.num_kv_heads, cfg.head_dim)
    h.append_frame(batch(lambda s_, l_: synth.sink_kv(cfg, s_, l_)[0], shp),
                   batch(lambda s_, l_: synth.sink_kv(cfg, s_, l_)[1], shp))
    for t in range(max(steps) + 1):
        fshp = (tpf, cfg.num_kv_heads, cfg.head_dim)
        kv = {sl: synth.frame_kv(cfg, sl[0], sl[1], t) for sl in exact}
        h.append_frame(batch(lambda s_, l_: kv[(s_, l_)][0], fshp), batch(lambda s_, l_: kv[(s_, l_)][1], fshp))
        if t not in steps:
            continue
        C_t = h.state(0)["instant_tokens"]
        qn = batch(lambda s_, l_: synth.instant_q(cfg, s_, l_, t, C_t)[C_t - tpf:], (tpf, cfg.num_q_heads, cfg.head_dim))
        o = h.build_instant_newest(qn)
        _t.cuda.synchronize()
        for (s_, l_) in exact:
            sch, o_inst, _ = oracle_step(cfg, s_, l_, t)
            ma, rl = assert_close(o[s_, l_].float().cpu(), o_inst[sch.C_t - tpf:], cfg.dtype, f"newest t={t}")
            REPORT.append((name + "-newest", "O_new", t, s_, l_, ma, rl))
    h.close()


@pytest.mark.parametrize("name,boost", [("c1", 1.0), ("c1", 2.25), ("c2", 1.0), ("c2", 2.25), ("c2", 4.0),
                                        ("c5", 4.0)])
def test_boosted_newest_frame_parity(lib, name, boost):
    """NEXT-4 resolution boost: build_instant_boost / attend_boost vs the fp64 oracle, with
    n_boost = boost * tpf re-encoded tokens (x1.5 / x2 spatial -> 2.25x / 4x tokens); t = 0
    has no older instant frame (window of the build empty), and boost = 1 with the ring's own
    frame must reproduce the plain build / attend."""
    import torch as _t
    cfg = synth.CONFIGS[name]
    steps = [0, 2, 3, 10, cfg.num_frames - 1]
    dev = _t.device("cuda", 0)
    exact = [(0, 0)] if cfg.num_streams == 1 else [(0, 0), (37, 2)]
    h = D.DSCache.from_config(cfg)
    S, N, tpf = cfg.num_streams, cfg.num_layers, cfg.tokens_per_frame
    nb = int(round(boost * tpf))
    def batch(fn, shape):
        t_ = (_t.randn((S, N) + shape, device=dev) * cfg.scale).to(cfg.torch_dtype)
        for (s_, l_) in exact:
            t_[s_, l_] = fn(s_, l_).to(dev)
        return t_
    shp = (cfg.sink_tokens, cfg.num_kv_heads, cfg.head_dim)
    h.append_frame(batch(lambda s_, l_: synth.sink_kv(cfg, s_, l_)[0], shp),
                   batch(lambda s_, l_: synth.sink_kv(cfg, s_, l_)[1], shp))
    bshp = (nb, cfg.num_kv_heads, cfg.head_dim)
    for t in range(max(steps) + 1):
        fshp = (tpf, cfg.num_kv_heads, cfg.head_dim)
        kv = {sl: synth.frame_kv(cfg, sl[0], sl[1], t) for sl in exact}
        k_f = batch(lambda s_, l_: kv[(s_, l_)][0], fshp)
        v_f = batch(lambda s_, l_: kv[(s_, l_)][1], fshp)
        h.append_frame(k_f, v_f)
        if t not in steps:
            continue
        C_t = h.state(0)["instant_tokens"]
        n_inst = C_t - tpf + nb
        if boost == 1.0:      # the newest frame "re-encoded" as itself
            bkv = {sl: kv[sl] for sl in exact}
            kb, vb = k_f.clone(), v_f.clone()
        else:
            bkv = {sl: synth.boost_kv(cfg, sl[0], sl[1], t, nb) for sl in exact}
            kb = batch(lambda s_, l_: bkv[(s_, l_)][0], bshp)
            vb = batch(lambda s_, l_: bkv[(s_, l_)][1], bshp)
        qi = batch(lambda s_, l_: synth.instant_q(cfg, s_, l_, t, n_inst), (n_inst, cfg.num_q_heads, cfg.head_dim))
        qkv = {sl: synth.query_qkv(cfg, sl[0], sl[1], t) for sl in exact}
        qshp = (cfg.query_tokens, cfg.num_q_heads, cfg.head_dim)
        kshp = (cfg.query_tokens, cfg.num_kv_heads, cfg.head_dim)
        q = batch(lambda s_, l_: qkv[(s_, l_)][0], qshp)
        kq = batch(lambda s_, l_: qkv[(s_, l_)][1], kshp)
        vq = batch(lambda s_, l_: qkv[(s_, l_)][2], kshp)
        oi = h.build_instant_boost(qi, kb, vb)
        o = h.attend_boost(q, kq, vq, kb, vb)
        if boost == 1.0:
            oi_plain = h.build_instant(qi)
            o_plain = h.attend(q, kq, vq)
        _t.cuda.synchronize()
        for (s_, l_) in exact:
            inp = StreamInputs(cfg, s_, l_)
            sch = step_schedule(cfg, t)
            f64 = lambda x: x.double().numpy()
            kb64, vb64 = f64(bkv[(s_, l_)][0]), f64(bkv[(s_, l_)][1])
            ref_i = O.instant_cache_output_boosted(sch, inp.sink(), inp.frame_kv, f64(synth.instant_q(cfg, s_, l_, t, n_inst)),
                                                   kb64, vb64, cfg.rope_theta)
            qq, kk, vv = (f64(x) for x in qkv[(s_, l_)])
            ref = O.attend_output_boosted(sch, inp.sink(), inp.frame_kv, qq, kk, vv, kb64, vb64, cfg.rope_theta)
            ma, rl = assert_close(oi[s_, l_].float().cpu(), ref_i, cfg.dtype, f"boost build t={t}")
            REPORT.append((f"{name}-boost{boost}", "O_inst", t, s_, l_, ma, rl))
            ma, rl = assert_close(o[s_, l_].float().cpu(), ref, cfg.dtype, f"boost attend t={t}")
            REPORT.append((f"{name}-boost{boost}", "O", t, s_, l_, ma, rl))
        if boost == 1.0:     # same keys, same ids: the plain calls agree to rounding
            assert (oi.float() - oi_plain.float()).abs().max().item() <= (1e-5 if cfg.dtype == "fp32" else 2e-2)
            assert (o.float() - o_plain.float()).abs().max().item() <= (1e-5 if cfg.dtype == "fp32" else 2e-2)
    h.close()


def test_boost_abi_errors(lib):
    import ctypes
    cfg = synth.CONFIGS["c2"]
    dev = torch.device("cuda", 0)
    h = D.DSCache.from_config(cfg)
    buf = torch.zeros(1 << 22, dtype=cfg.torch_dtype, device=dev)
    p = ctypes.c_void_p(buf.data_ptr())
    L = D._lib
    assert L.dscache_build_instant_boost(h._h, 0, 1, p, p, p, 5, p, None) == D.E_STATE   # no frame yet
    A = cfg.sink_tokens
    sk = torch.zeros((1, 1, A, cfg.num_kv_heads, cfg.head_dim), dtype=cfg.torch_dtype, device=dev)
    fk = torch.zeros((1, 1, cfg.tokens_per_frame, cfg.num_kv_heads, cfg.head_dim), dtype=cfg.torch_dtype, device=dev)
    h.append_frame(sk, sk)
    h.append_frame(fk, fk)
    assert L.dscache_build_instant_boost(h._h, 0, 1, p, p, p, 0, p, None) == D.E_ARG      # n_boost < 1
    assert L.dscache_build_instant_boost(h._h, 0, 1, None, p, p, 5, p, None) == D.E_ARG   # null q
    assert L.dscache_attend_boost(h._h, 0, 1, p, p, p, 0, p, p, 5, p, None) == D.E_ARG    # n_q < 1
    assert L.dscache_attend_boost(h._h, 0, 1, p, p, p, 4, p, p, 0, p, None) == D.E_ARG    # n_boost < 1
    big = cfg.max_position
    assert L.dscache_build_instant_boost(h._h, 0, 1, p, p, p, big, p, None) == D.E_POS_OVERFLOW
    torch.cuda.synchronize()
    h.close()


@pytest.mark.parametrize("name", ["c2", "c5"])
def test_host_pipeline_equals_device_step(lib, name):
    """pipeline.HostStepPipeline (pinned host inputs, 3 streams, 2 slots) gives the same bits
    as DSCache.step on device-resident inputs, step after step (warm-up with C_t < C included)."""
    from paper_2605_01858_b200.pipeline import HostStepPipeline
    cfg = synth.CONFIGS[name]
    dev = torch.device("cuda", 0)
    S, N, tpf, Hkv, Hq, d, A = (cfg.num_streams, cfg.num_layers, cfg.tokens_per_frame, cfg.num_kv_heads,
                                cfg.num_q_heads, cfg.head_dim, cfg.sink_tokens)
    C, q = cfg.C, cfg.query_tokens
    g = torch.Generator().manual_seed(5)
    r = lambda *sh: (torch.randn(sh, generator=g) * cfg.scale).to(cfg.torch_dtype).pin_memory()   # noqa: E731
    a, b = D.DSCache.from_config(cfg), D.DSCache.from_config(cfg)
    sk, sv = r(S, N, A, Hkv, d), r(S, N, A, Hkv, d)
    for h in (a, b):
        h.append_frame(sk.to(dev), sv.to(dev))
    pipe = HostStepPipeline(b, q)
    outs = []
    for t in range(cfg.instant_frames + 3):
        C_t = min(t + 1, cfg.instant_frames) * tpf
        hk, hv, hqi = r(S, N, tpf, Hkv, d), r(S, N, tpf, Hkv, d), r(S, N, C_t, Hq, d)
        hq, hks, hvs = r(S, N, q, Hq, d), r(S, N, q, Hkv, d), r(S, N, q, Hkv, d)
        oi_ref, o_ref = a.step(hk.to(dev), hv.to(dev), hqi.to(dev), hq.to(dev), hks.to(dev), hvs.to(dev))
        ho = torch.empty(S, N, q, Hq, d, dtype=cfg.torch_dtype).pin_memory()
        hoi = torch.empty(S, N, C_t, Hq, d, dtype=cfg.torch_dtype).pin_memory()
        pipe.submit(hk, hv, hqi, hq, hks, hvs, ho, o_inst_host=hoi)
        outs.append((o_ref, ho, oi_ref, hoi))
    pipe.synchronize()
    torch.cuda.synchronize()
    for o_ref, ho, oi_ref, hoi in outs:
        assert torch.equal(o_ref.cpu(), ho)
        assert torch.equal(oi_ref.cpu(), hoi)   # O_inst of warm-up steps (C_t < C) included
    a.close(); b.close()


def test_zz_print_report(lib):
    for r in REPORT:
        print("PARITY %-16s %-6s t=%-5d s=%-3d l=%-3d max_abs=%.3e rel_l2=%.3e" % r)
