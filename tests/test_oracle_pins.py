"""Pins of the fp64 oracle against things other than itself (all CPU, -m "not gpu").

Each test names what fixes the expected value: a closed form, a textbook special
case, a library routine, a hand-derived golden value (tests/golden/), brute
force, or an invariant the paper states.  A plausible mistake anywhere in the
oracle (dropped term, wrong sign or index, transposed operand, wrong pairing,
off-by-one position, wrong GQA map, missing sink, wrong eviction) fails at
least one of them.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

import dscache_synth as synth
from oracle import dscache_oracle as O
from oracle.workload import StreamInputs, oracle_step, step_schedule

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "schedule_spot_values.json")
RNG = np.random.default_rng(12345)


# --------------------------------------------------------------------------- RoPE
def test_rope_position_zero_is_identity_bitwise():
    # SPEC.md:113 "any x at position 0 -> x unchanged"; cos 0 = 1, sin 0 = 0 exactly.
    x = RNG.standard_normal((7, 3, 128))
    for style in (O.SPLIT_HALF, O.ADJACENT):
        assert np.array_equal(O.rope(x, np.zeros(7), 1e6, style), x)


def test_rope_d2_is_textbook_rotation():
    # d = 2 has one pair with theta_0 = base^0 = 1: (1, 0) at position p -> (cos p, sin p).
    for p in [0, 1, 2, 5, 17, 1000]:
        y = O.rope(np.array([[1.0, 0.0]]), np.array([p]), 1e4)
        assert np.allclose(y[0], [math.cos(p), math.sin(p)], atol=1e-15, rtol=0)
        y = O.rope(np.array([[0.0, 1.0]]), np.array([p]), 1e4)
        assert np.allclose(y[0], [-math.sin(p), math.cos(p)], atol=1e-15, rtol=0)


def test_rope_split_half_pairing():
    # e_i (i < d/2) only mixes with e_{i+d/2}: a mistaken adjacent pairing fails here.
    d, p, base = 128, 9, 1e6
    for i in [0, 1, 37, 63]:
        e = np.zeros((1, d)); e[0, i] = 1.0
        y = O.rope(e, np.array([p]), base)[0]
        nz = set(np.nonzero(np.abs(y) > 1e-300)[0].tolist())
        assert nz <= {i, i + d // 2}
        assert abs(y[i] ** 2 + y[i + d // 2] ** 2 - 1.0) < 1e-14


def test_rope_matches_qwen2_library_rotary():
    # Library routine: transformers' Qwen2 rotary embedding (the LLaVA-OV-7B LM) computes
    # inv_freq = 1 / base^(arange(0, d, 2)/d) and rotate_half pairing; its cos/sin are fp32.
    from transformers import Qwen2Config
    from transformers.models.qwen2 import modeling_qwen2 as m
    hcfg = Qwen2Config(hidden_size=28 * 128, num_attention_heads=28, num_key_value_heads=4, rope_theta=1e6)
    rot = m.Qwen2RotaryEmbedding(hcfg)
    n = 40
    pos = torch.arange(n)[None]
    cos, sin = rot(torch.zeros(1, 1, n, 128, dtype=torch.float64), pos)
    q = torch.randn(1, 28, n, 128, dtype=torch.float64)
    k = torch.randn(1, 4, n, 128, dtype=torch.float64)
    qe, ke = m.apply_rotary_pos_emb(q, k, cos.double(), sin.double())
    ours_q = O.rope(q[0].permute(1, 0, 2).numpy(), np.arange(n), 1e6)
    ours_k = O.rope(k[0].permute(1, 0, 2).numpy(), np.arange(n), 1e6)
    assert np.abs(ours_q - qe[0].permute(1, 0, 2).numpy()).max() < 2e-5   # fp32 angle error at p < 40
    assert np.abs(ours_k - ke[0].permute(1, 0, 2).numpy()).max() < 2e-5


def test_rope_adjacent_spec_worked_example():
    # SPEC.md:116 worked example (tests/golden/rope_adjacent_d4.json): head_dim 4, x = [1, 0, 1, 0]
    # at position 1, base 1e4 -> pair (0, 1) rotated by 1 rad, pair (2, 3) by 1e4^(-1/2) = 0.01 rad.
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "rope_adjacent_d4.json")))
    y = O.rope(np.array([g["x"]]), np.array([g["position"]]), g["base"], O.ADJACENT)[0]
    expect = [math.cos(1.0), math.sin(1.0), math.cos(0.01), math.sin(0.01)]
    assert np.abs(y - np.array(expect)).max() < 1e-15


def test_rope_adjacent_pairing_and_frequencies_by_unit_vectors():
    # Rotating a unit vector e_{2i} (resp. e_{2i+1}) by the pair rotation of angle p*theta_i gives
    # cos/sin in coordinates 2i, 2i+1 only (a split-half or shifted pairing fails), with
    # theta_i = base^(-2i/d) (a wrong frequency index fails).
    d, base = 16, 1e4
    for p in [1, 3, 250]:
        for i in range(d // 2):
            ang = p * base ** (-2.0 * i / d)
            e = np.zeros((1, d)); e[0, 2 * i] = 1.0
            y = O.rope(e, np.array([p]), base, O.ADJACENT)[0]
            ref = np.zeros(d); ref[2 * i] = math.cos(ang); ref[2 * i + 1] = math.sin(ang)
            assert np.abs(y - ref).max() < 1e-14
            e = np.zeros((1, d)); e[0, 2 * i + 1] = 1.0
            y = O.rope(e, np.array([p]), base, O.ADJACENT)[0]
            ref = np.zeros(d); ref[2 * i] = -math.sin(ang); ref[2 * i + 1] = math.cos(ang)
            assert np.abs(y - ref).max() < 1e-14


def test_rope_adjacent_is_split_half_under_interleave_permutation():
    # The two pairings are the same rotation in different coordinate orders: with P the
    # permutation taking interleaved (a0 b0 a1 b1 ..) to halves (a0 a1 .. b0 b1 ..),
    # adjacent(x) = P^-1 split_half(P x).  Split-half is pinned to transformers' Qwen2
    # rotary above, so this pins the adjacent branch to the same library routine.
    d = 64
    perm = np.concatenate([np.arange(0, d, 2), np.arange(1, d, 2)])   # P x = x[perm]
    inv = np.argsort(perm)
    x = RNG.standard_normal((50, 3, d))
    pos = RNG.integers(0, 30000, 50)
    a = O.rope(x, pos, 1e6, O.ADJACENT)
    b = O.rope(x[..., perm], pos, 1e6, O.SPLIT_HALF)[..., inv]
    assert np.abs(a - b).max() < 1e-12


def test_rope_isometry():
    x = RNG.standard_normal((500, 128))
    p = RNG.integers(0, 30000, 500)
    y = O.rope(x, p, 1e6)
    assert np.allclose(np.linalg.norm(y, axis=1), np.linalg.norm(x, axis=1), rtol=1e-13, atol=0)


def test_rope_group_property():
    # R(p2) R(p1) = R(p1 + p2): rotations compose additively.
    x = RNG.standard_normal((300, 64))
    p1 = RNG.integers(0, 20000, 300); p2 = RNG.integers(0, 20000, 300)
    for style in (O.SPLIT_HALF, O.ADJACENT):
        a = O.rope(O.rope(x, p1, 1e4, style), p2, 1e4, style)
        b = O.rope(x, p1 + p2, 1e4, style)
        assert np.abs(a - b).max() < 1e-9


def test_rope_shift_invariance_1e5_trials():
    # PAPER.md:662-664 <f(q,i), f(k,j)> = g(q, k, i-j); SPEC.md:137 bound 1e-10 (we hold 1e-10).
    n = 100_000
    q = RNG.standard_normal((n, 64)); k = RNG.standard_normal((n, 64))
    j = RNG.integers(0, 4000, n); i = j + RNG.integers(0, 4000, n); s = RNG.integers(-j, 4000)
    a = np.sum(O.rope(q, i, 1e4) * O.rope(k, j, 1e4), axis=1)
    b = np.sum(O.rope(q, i + s, 1e4) * O.rope(k, j + s, 1e4), axis=1)
    assert np.abs(a - b).max() <= 1e-10
    # and i == j gives <q, k> (both rotations cancel)
    c = np.sum(O.rope(q, j, 1e4) * O.rope(k, j, 1e4), axis=1)
    assert np.abs(c - np.sum(q * k, axis=1)).max() <= 1e-10


# --------------------------------------------------------------------------- schedule (Eq. 3/5/6)
def closed_form(cfg, t):
    """Independent derivation of the FIFO state (SURVEY §8(a)2 closed form)."""
    lI, lU, tpf = cfg.instant_frames, cfg.past_frames, cfg.tokens_per_frame
    inst = list(range(max(0, t - lI + 1), t + 1))
    past = list(range(max(0, t - lI - lU + 1), t - lI + 1))
    ev = [t - lI - lU] if t - lI - lU >= 0 else []
    return inst, past, ev


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c5"])
def test_fifo_matches_closed_form_every_step(name):
    cfg = synth.CONFIGS[name]
    for t in range(cfg.num_frames):
        sch = step_schedule(cfg, t)
        inst, past, ev = closed_form(cfg, t)
        assert sch.instant_frames == inst and sch.past_frames == past and sch.evicted == ev, t


def test_fifo_matches_closed_form_c4_sampled():
    cfg = synth.CONFIGS["c4"]
    for t in [0, 7, 8, 135, 136, 137, 272, 1000, 2047, 4095]:
        sch = step_schedule(cfg, t)
        inst, past, ev = closed_form(cfg, t)
        assert sch.instant_frames == inst and sch.past_frames == past and sch.evicted == ev, t


def test_schedule_golden_spot_values():
    g = json.load(open(GOLDEN))
    for name in ("c1", "c2"):
        cfg = synth.CONFIGS[name]
        for t, v in g[name]["P_t"].items():
            assert step_schedule(cfg, int(t)).P_t == v
        for t, v in g[name]["C_t"].items():
            assert step_schedule(cfg, int(t)).C_t == v
        fe = g[name]["first_eviction"]
        assert step_schedule(cfg, fe["step"]).evicted == [fe["frame"]]
        assert step_schedule(cfg, fe["step"] - 1).evicted == []
    for name in ("c1", "c2", "c4"):
        cfg = synth.CONFIGS[name]
        t = cfg.num_frames - 1
        sch = step_schedule(cfg, t)
        bk, bq, ak, aq = O.position_ids(sch, cfg.query_tokens)
        ctx_max = int(ak[-1 - cfg.query_tokens])
        assert ctx_max == g[name]["max_context_key_id"]
        assert int(aq.max()) == g[name]["max_query_id"]
        assert int(aq.max()) < cfg.max_position
    c4 = synth.CONFIGS["c4"]
    assert c4.sink_tokens + c4.num_frames * c4.tokens_per_frame == g["c4"]["total_tokens"]


def test_ring_slack_frame_is_next_frames_slots():
    # R = (l_U + l_I + 1) tpf: the frame evicted at t occupies exactly the slots frame t+1 will
    # take (the slack frame), and the window frames never collide.
    for name in ("c1", "c2", "c5"):
        cfg = synth.CONFIGS[name]
        for t in range(cfg.num_frames - 1):
            sch = step_schedule(cfg, t)
            used = np.concatenate([O.ring_slots(f, cfg.tokens_per_frame, cfg.instant_frames, cfg.past_frames)
                                   for f in sch.past_frames + sch.instant_frames])
            assert len(set(used.tolist())) == len(used)
            for e in sch.evicted:
                assert np.array_equal(
                    O.ring_slots(e, cfg.tokens_per_frame, cfg.instant_frames, cfg.past_frames),
                    O.ring_slots(t + 1, cfg.tokens_per_frame, cfg.instant_frames, cfg.past_frames))


def test_position_ids_bounded_for_every_config():
    # PAPER.md:236 "positional indices remain bounded"; north_star: below W+C+sink for keys.
    for cfg in synth.CONFIGS.values():
        for t in (0, cfg.num_frames - 1):
            sch = step_schedule(cfg, t)
            bk, bq, ak, aq = O.position_ids(sch, cfg.query_tokens)
            assert ak[: len(ak) - cfg.query_tokens].max() < cfg.sink_tokens + cfg.W + cfg.C
            assert aq.max() < cfg.sink_tokens + cfg.W + cfg.C + cfg.query_tokens <= cfg.max_position


# --------------------------------------------------------------------------- attention core
def test_softmax_attention_matches_torch_sdpa_fp64():
    # Library routine: torch scaled_dot_product_attention with a boolean mask (fp64, CPU).
    nq, nk, d = 37, 91, 64
    q = RNG.standard_normal((nq, d)); k = RNG.standard_normal((nk, d)); v = RNG.standard_normal((nk, 48))
    vis = RNG.random((nq, nk)) < 0.6
    vis[:, 0] = True
    ours = O.softmax_attention(q, k, v, vis)
    ref = torch.nn.functional.scaled_dot_product_attention(
        torch.from_numpy(q)[None], torch.from_numpy(k)[None], torch.from_numpy(v)[None],
        attn_mask=torch.from_numpy(vis)[None])[0].numpy()
    assert np.abs(ours - ref).max() < 1e-13


def test_gqa_head_map_matches_repeat_kv_sdpa():
    # HF repeat_kv convention (reading Q10): query head h uses kv head h // (Hq/Hkv).
    nq, hq, hkv, d = 5, 28, 4, 32
    q = RNG.standard_normal((nq, hq, d)); k = RNG.standard_normal((11, hkv, d)); v = RNG.standard_normal((11, hkv, d))
    pos_k = np.arange(11); pos_q = 6 + np.arange(5)
    ours = O.gqa_attention(q, pos_q, k, v, pos_k, 1e4)
    qr = torch.from_numpy(O.rope(q, pos_q, 1e4)).permute(1, 0, 2)
    kr = torch.from_numpy(O.rope(k, pos_k, 1e4)).permute(1, 0, 2).repeat_interleave(hq // hkv, 0)
    vv = torch.from_numpy(v).permute(1, 0, 2).repeat_interleave(hq // hkv, 0)
    mask = torch.from_numpy(pos_k[None, :] <= pos_q[:, None])
    ref = torch.nn.functional.scaled_dot_product_attention(qr, kr, vv, attn_mask=mask).permute(1, 0, 2).numpy()
    assert np.abs(ours - ref).max() < 1e-13


# --------------------------------------------------------------------------- closed forms on the step
def _zero_q_inputs(cfg, id_in_v):
    """Inputs with Q = 0 (uniform softmax) and V[.][0] = position id if id_in_v."""
    inp = StreamInputs(cfg, 0, 0)

    class Z(StreamInputs):
        pass
    z = Z(cfg, 0, 0)
    z.instant_q = lambda t, n: np.zeros((n, cfg.num_q_heads, cfg.head_dim))
    base_query = inp.query
    z.query = lambda t, n_q=None: (np.zeros_like(base_query(t, n_q)[0]),) + base_query(t, n_q)[1:]
    return z


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_zero_query_gives_mean_of_visible_values(name):
    # Q = 0 -> every score 0 -> O = mean of the visible V.  Build row i sees A + i + 1 keys,
    # attend row i sees A + P_t + C_t + i + 1 keys (sink, past, instant, self[0..i]).
    cfg = synth.CONFIGS[name].replace(num_frames=12)
    z = _zero_q_inputs(cfg, False)
    for t in (0, 1, 4, 11):
        sch, o_inst, o = oracle_step(cfg, 0, 0, t, inputs=z)
        sk, sv = z.sink()
        vals = [sv] + [z.frame_kv(f)[1] for f in sch.past_frames + sch.instant_frames]
        ctx = np.concatenate(vals)
        _, _, vself = z.query(t)
        grp = cfg.num_q_heads // cfg.num_kv_heads
        for h in (0, cfg.num_q_heads - 1):
            g = h // grp
            allv = np.concatenate([ctx[:, g], vself[:, g]])
            L = len(ctx)
            for i in (0, cfg.query_tokens - 1):
                assert np.abs(o[i, h] - allv[: L + i + 1].mean(0)).max() < 1e-12
            inst_v = np.concatenate([sv] + [z.frame_kv(f)[1] for f in sch.instant_frames])[:, g]
            for i in (0, sch.C_t - 1):
                assert np.abs(o_inst[i, h] - inst_v[: cfg.sink_tokens + i + 1].mean(0)).max() < 1e-12


def test_zero_query_position_id_encoding():
    # V[j][0] = id(j), Q = 0  ->  O[i][0] = mean(0..lim_i) = lim_i / 2 exactly; pins the visible
    # *set* and the ids (an off-by-one position or a dropped sink shifts the mean).
    cfg = synth.CONFIGS["c1"]
    A, tpf = cfg.sink_tokens, cfg.tokens_per_frame
    for t in (0, 3, 7, 19):
        sch = step_schedule(cfg, t)
        d, hkv = cfg.head_dim, cfg.num_kv_heads
        def fr(f):
            k = np.zeros((tpf, hkv, d)); v = np.zeros((tpf, hkv, d))
            return k, v
        # value column 0 carries the id the *context* assigns: fill after concatenation
        frames = sch.past_frames + sch.instant_frames
        id_of = {}
        for n, f in enumerate(frames):
            id_of[f] = A + n * tpf + np.arange(tpf)
        def frv(f):
            k, v = fr(f)
            v[:, :, 0] = id_of[f][:, None]
            return k, v
        sink = (np.zeros((A, hkv, d)), np.zeros((A, hkv, d)))
        sink[1][:, :, 0] = np.arange(A)[:, None]
        nq = cfg.query_tokens
        L = A + sch.P_t + sch.C_t
        vself = np.zeros((nq, hkv, d)); vself[:, :, 0] = (L + np.arange(nq))[:, None]
        o = O.attend_output(sch, sink, frv, np.zeros((nq, cfg.num_q_heads, d)), np.zeros((nq, hkv, d)),
                            vself, cfg.rope_theta)
        assert np.abs(o[:, :, 0] - ((L + np.arange(nq)) / 2.0)[:, None]).max() < 1e-12
        # instant build: ids A + i inside [sink | instant] only
        id_of = {f: A + n * tpf + np.arange(tpf) for n, f in enumerate(sch.instant_frames)}
        oi = O.instant_cache_output(sch, sink, frv, np.zeros((sch.C_t, cfg.num_q_heads, d)), cfg.rope_theta)
        assert np.abs(oi[:, :, 0] - ((A + np.arange(sch.C_t)) / 2.0)[:, None]).max() < 1e-12


def test_single_visible_key_returns_its_value():
    # A = 0: instant row 0 sees only instant key 0 -> O_inst[0] = v_0 for every head.
    cfg = synth.CONFIGS["c1"].replace(sink_tokens=0)
    inp = StreamInputs(cfg, 0, 0)
    for t in (0, 6):
        sch, o_inst, _ = oracle_step(cfg, 0, 0, t, inputs=inp)
        v0 = inp.frame_kv(sch.instant_frames[0])[1][0]
        for h in range(cfg.num_q_heads):
            assert np.abs(o_inst[0, h] - v0[h // (cfg.num_q_heads // cfg.num_kv_heads)]).max() < 1e-15


# --------------------------------------------------------------------------- brute force
def _brute_rope(vec, p, base):
    d = len(vec); h = d // 2
    out = list(vec)
    for i in range(h):
        th = base ** (-2.0 * i / d)
        c, s = math.cos(p * th), math.sin(p * th)
        a, b = vec[i], vec[i + h]
        out[i] = a * c - b * s
        out[i + h] = a * s + b * c
    return out


def _brute_attend(qv, qpos, keys, base):
    """keys: list of (pos, k, v); pure-Python softmax over keys with pos <= qpos."""
    qr = _brute_rope(qv, qpos, base)
    sc = []
    for (p, k, v) in keys:
        if p <= qpos:
            kr = _brute_rope(k, p, base)
            sc.append((sum(a * b for a, b in zip(qr, kr)) / math.sqrt(len(qv)), v))
    m = max(s for s, _ in sc)
    w = [math.exp(s - m) for s, _ in sc]
    den = sum(w)
    return [sum(wi * v[c] for wi, (_, v) in zip(w, sc)) / den for c in range(len(sc[0][1]))]


def test_brute_force_full_history_tiny_stream():
    """Keep EVERY token ever appended (full history); slice the window from the end of the
    history as PAPER.md:113-114 / Eq. 6 describe (the last l_W = (l_U + l_I) frames behind
    the sink), and recompute both attentions with pure-Python loops."""
    cfg = synth.StreamConfig("tiny", 99, 1, 1, 4, 2, 8, 1e4, 3, 2, 2, 2, 3, 9, "fp32", 1.0)
    inp = StreamInputs(cfg, 0, 0)
    sk, sv = inp.sink()
    A, tpf, lI, lU = cfg.sink_tokens, cfg.tokens_per_frame, cfg.instant_frames, cfg.past_frames
    grp = cfg.num_q_heads // cfg.num_kv_heads
    history = []   # (frame, k [Hkv,d], v)
    for t in range(cfg.num_frames):
        fk, fv = inp.frame_kv(t)
        history += [(t, fk[j], fv[j]) for j in range(tpf)]
        sch, o_inst, o = oracle_step(cfg, 0, 0, t, inputs=inp)
        window = history[-(lU + lI) * tpf:]                 # P_{l_P - l_W : l_P}
        inst = history[-lI * tpf:]                          # the buffer B_t
        q, ks, vs = inp.query(t)
        nq = q.shape[0]
        for h in range(cfg.num_q_heads):
            g = h // grp
            keys = [(j, list(sk[j, g]), list(sv[j, g])) for j in range(A)]
            keys += [(A + n, list(k[g]), list(v[g])) for n, (_, k, v) in enumerate(window)]
            L = len(keys)
            keys += [(L + i, list(ks[i, g]), list(vs[i, g])) for i in range(nq)]
            for i in range(nq):
                ref = _brute_attend(list(q[i, h]), L + i, keys, cfg.rope_theta)
                assert np.abs(np.array(ref) - o[i, h]).max() < 1e-12
            ikeys = [(j, list(sk[j, g]), list(sv[j, g])) for j in range(A)]
            ikeys += [(A + n, list(k[g]), list(v[g])) for n, (_, k, v) in enumerate(inst)]
            qi = inp.instant_q(t, sch.C_t)
            for i in range(sch.C_t):
                ref = _brute_attend(list(qi[i, h]), A + i, ikeys, cfg.rope_theta)
                assert np.abs(np.array(ref) - o_inst[i, h]).max() < 1e-12


# --------------------------------------------------------------------------- paper invariants
def _abs_attend(cfg, sch, inp, t, pos_mode):
    """Attend computed with *absolute* ids (standard cache, Eq. 1 / App. B): stream token
    a has id a (A = 0), the query chunk follows the newest frame."""
    tpf = cfg.tokens_per_frame
    frames = sch.past_frames + sch.instant_frames
    ks = np.concatenate([inp.frame_kv(f)[0] for f in frames])
    vs = np.concatenate([inp.frame_kv(f)[1] for f in frames])
    pk = np.concatenate([f * tpf + np.arange(tpf) for f in frames])
    q, kq, vq = inp.query(t)
    nq = q.shape[0]
    pq = (t + 1) * tpf + np.arange(nq)
    if pos_mode == "shuffled":
        pk = RNG.permutation(pk)
    kk = np.concatenate([ks, kq]); vv = np.concatenate([vs, vq]); pp = np.concatenate([pk, pq])
    return O.gqa_attention(q, pq, kk, vv, pp, cfg.rope_theta)


def test_proposition_rebased_equals_absolute_ids_with_eviction():
    # Proposition 3.2 (proof "Case eviction" PAPER.md:647-684): with no sink
    # (A = 0) the contiguous re-basing is a distance-preserving shift of the absolute ids,
    # so outputs are identical; a shuffled-position negative control must differ.
    cfg = synth.CONFIGS["c1"].replace(sink_tokens=0, num_frames=12)
    inp = StreamInputs(cfg, 0, 0)
    for t in (2, 5, 6, 11):               # before and after the first eviction (t = 5)
        sch, _, o = oracle_step(cfg, 0, 0, t, inputs=inp)
        assert np.abs(o - _abs_attend(cfg, sch, inp, t, "abs")).max() < 1e-12
    sch, _, o = oracle_step(cfg, 0, 0, 11, inputs=inp)
    assert np.abs(o - _abs_attend(cfg, sch, inp, 11, "shuffled")).max() > 1e-3


def test_proposition_with_sink_before_first_eviction():
    # Before any eviction the contiguous ids ARE the absolute ids (sink 0..A-1, then the stream).
    cfg = synth.CONFIGS["c1"]
    inp = StreamInputs(cfg, 0, 0)
    A, tpf = cfg.sink_tokens, cfg.tokens_per_frame
    for t in (0, 2, 4):
        sch, _, o = oracle_step(cfg, 0, 0, t, inputs=inp)
        assert not sch.evicted and sch.past_frames[:1] in ([], [0])
        sk, sv = inp.sink()
        frames = sch.past_frames + sch.instant_frames
        q, kq, vq = inp.query(t)
        kk = np.concatenate([sk] + [inp.frame_kv(f)[0] for f in frames] + [kq])
        vv = np.concatenate([sv] + [inp.frame_kv(f)[1] for f in frames] + [vq])
        pk = np.concatenate([np.arange(A)] + [A + f * tpf + np.arange(tpf) for f in frames]
                            + [A + (t + 1) * tpf + np.arange(len(q))])
        ref = O.gqa_attention(q, pk[-len(q):], kk, vv, pk, cfg.rope_theta)
        assert np.abs(o - ref).max() < 1e-12


def test_rerotation_invariant():
    # north_star: raw (position-agnostic) keys rotated at the reassigned ids == keys stored
    # rotated at absolute ids (Eq. 1) and explicitly re-rotated by (new - abs).
    cfg = synth.CONFIGS["c2"].replace(num_frames=40)
    inp = StreamInputs(cfg, 0, 0)
    t = 39
    sch = step_schedule(cfg, t)
    A, tpf = cfg.sink_tokens, cfg.tokens_per_frame
    frames = sch.past_frames + sch.instant_frames
    k_raw = np.concatenate([inp.frame_kv(f)[0] for f in frames])
    abs_id = np.concatenate([A + f * tpf + np.arange(tpf) for f in frames])
    new_id = A + np.arange(len(abs_id))
    k_abs = O.rope(k_raw, abs_id, cfg.rope_theta)                     # standard cache
    k_re = O.rope(k_abs, new_id - abs_id, cfg.rope_theta)             # re-rotated
    assert np.abs(k_re - O.rope(k_raw, new_id, cfg.rope_theta)).max() < 1e-9


def _uniform_window_attend(cfg, t, inp, n_tokens):
    """Reference for the reductions: the sink + the last n_tokens stream tokens (a plain
    sliding window), then the query chunk."""
    tpf, A = cfg.tokens_per_frame, cfg.sink_tokens
    toks_k = np.concatenate([inp.frame_kv(f)[0] for f in range(t + 1)])
    toks_v = np.concatenate([inp.frame_kv(f)[1] for f in range(t + 1)])
    wk, wv = toks_k[len(toks_k) - min(n_tokens, len(toks_k)):], toks_v[len(toks_v) - min(n_tokens, len(toks_v)):]
    sk, sv = inp.sink()
    q, kq, vq = inp.query(t)
    kk = np.concatenate([sk, wk, kq]); vv = np.concatenate([sv, wv, vq])
    pk = np.arange(len(kk))
    return O.gqa_attention(q, pk[-len(q):], kk, vv, pk, cfg.rope_theta)


def test_reduction_lI0_is_uniform_cache():
    # PAPER.md:295 / 488: DSCache with l_I = 0 is the uniform streaming cache (window l_U).
    cfg = synth.CONFIGS["c1"].replace(instant_frames=0, past_frames=5)
    inp = StreamInputs(cfg, 0, 0)
    for t in (0, 3, 9, 19):
        sch, o_inst, o = oracle_step(cfg, 0, 0, t, inputs=inp)
        assert sch.C_t == 0 and o_inst.shape[0] == 0
        assert np.abs(o - _uniform_window_attend(cfg, t, inp, cfg.W)).max() < 1e-12


def test_reduction_lU0_is_sliding_window():
    # l_U = 0 degenerates to a sliding-window model over the buffer.
    cfg = synth.CONFIGS["c1"].replace(instant_frames=3, past_frames=0)
    inp = StreamInputs(cfg, 0, 0)
    for t in (0, 2, 8, 19):
        sch, _, o = oracle_step(cfg, 0, 0, t, inputs=inp)
        assert sch.P_t == 0
        assert np.abs(o - _uniform_window_attend(cfg, t, inp, cfg.C)).max() < 1e-12


def test_instant_cache_decoupled_from_past():
    # Eq. 7 / PAPER.md:221,226: I is built from the buffer and sink alone -> bitwise unchanged
    # when every past frame's K/V is replaced by garbage; the final attend does change.
    cfg = synth.CONFIGS["c1"]
    inp = StreamInputs(cfg, 0, 0)
    t = 15
    sch, o_inst, o = oracle_step(cfg, 0, 0, t, inputs=inp)

    class Garbage(StreamInputs):
        def _frame_kv(self, f):
            k, v = StreamInputs._frame_kv(self, f)
            if f in sch.past_frames:
                return 1e3 * RNG.standard_normal(k.shape), 1e3 * RNG.standard_normal(v.shape)
            return k, v
    g = Garbage(cfg, 0, 0)
    sch2, o_inst2, o2 = oracle_step(cfg, 0, 0, t, inputs=g)
    assert np.array_equal(o_inst, o_inst2)
    assert np.abs(o - o2).max() > 1e-3


# --------------------------------------------------------------------------- Eq. 5 update attention (NEXT-1)
def _upd_cfg():
    return synth.StreamConfig("upd", 98, 1, 1, 4, 2, 8, 1e4, 3, 2, 4, 2, 3, 12, "fp32", 1.0)


@pytest.mark.parametrize("l_L", [0, 2, 4, 9])
def test_update_attention_brute_force_full_history(l_L):
    """Eq. 5: phi(X_{t-l_I}, [C_a, zeta(U_{t-1})]); zeta = the newest l_L frames of U_{t-1}
    (PAPER.md:202).  Reference from the full history: U_{t-1} holds the last min(e, l_U)
    frames before e = t - l_I, so zeta = frames [e - min(l_L, l_U, e), e); pure-Python loops."""
    cfg = _upd_cfg()
    inp = StreamInputs(cfg, 0, 0)
    sk, sv = inp.sink()
    A, tpf, lI, lU = cfg.sink_tokens, cfg.tokens_per_frame, cfg.instant_frames, cfg.past_frames
    grp = cfg.num_q_heads // cfg.num_kv_heads
    for t in range(lI, cfg.num_frames):
        e = t - lI
        nz = min(l_L, lU, e)
        frames = list(range(e - nz, e + 1))
        qu = f64_of(synth.update_q(cfg, 0, 0, t))
        o = O.cumulative_update_output(t, lI, lU, l_L, (sk, sv), inp.frame_kv, qu, cfg.rope_theta, tpf)
        for h in range(cfg.num_q_heads):
            g = h // grp
            keys = [(j, list(sk[j, g]), list(sv[j, g])) for j in range(A)]
            n = A
            for f in frames:
                fk, fv = inp.frame_kv(f)
                for j in range(tpf):
                    keys.append((n, list(fk[j, g]), list(fv[j, g])))
                    n += 1
            for i in range(tpf):
                ref = _brute_attend(list(qu[i, h]), A + nz * tpf + i, keys, cfg.rope_theta)
                assert np.abs(np.array(ref) - o[i, h]).max() < 1e-12


def test_update_attention_zero_query_mean():
    # Q = 0: token i of the leaving frame sees A + |zeta| + i + 1 keys -> O = their mean V
    cfg = synth.CONFIGS["c1"]
    inp = StreamInputs(cfg, 0, 0)
    sk, sv = inp.sink()
    tpf, lI, lU = cfg.tokens_per_frame, cfg.instant_frames, cfg.past_frames
    for t, l_L in ((1, 4), (7, 2), (19, 4), (19, 0)):
        e = t - lI
        nz = min(l_L, lU, e)
        vals = np.concatenate([sv] + [inp.frame_kv(f)[1] for f in range(e - nz, e + 1)])
        o = O.cumulative_update_output(t, lI, lU, l_L, (sk, sv), inp.frame_kv,
                                       np.zeros((tpf, cfg.num_q_heads, cfg.head_dim)), cfg.rope_theta, tpf)
        L0 = cfg.sink_tokens + nz * tpf
        for i in (0, tpf - 1):
            assert np.abs(o[i, 0] - vals[: L0 + i + 1, 0].mean(0)).max() < 1e-12
    with pytest.raises(ValueError):
        O.cumulative_update_output(0, 1, lU, 4, (sk, sv), inp.frame_kv,
                                   np.zeros((tpf, cfg.num_q_heads, cfg.head_dim)), cfg.rope_theta, tpf)


def f64_of(x):
    return x.double().numpy()


# --------------------------------------------------------------------------- decode (NEXT-2)
def test_decode_equals_attend_when_self_is_the_query_chunk():
    # n_q = n_self: decode_output is the Eq. 8 attend itself
    cfg = synth.CONFIGS["c1"]
    inp = StreamInputs(cfg, 0, 0)
    sch = step_schedule(cfg, 9)
    q, ks, vs = inp.query(9)
    a = O.attend_output(sch, inp.sink(), inp.frame_kv, q, ks, vs, cfg.rope_theta)
    b = O.decode_output(sch, inp.sink(), inp.frame_kv, q, ks, vs, cfg.rope_theta)
    assert np.array_equal(a, b)


def test_decode_token_by_token_matches_brute_force():
    """A decode step (n_q = 1) after g generated tokens == pure-Python attention of that
    token over sink + window + query chunk + generated tokens, ids consecutive."""
    cfg = _upd_cfg()
    inp = StreamInputs(cfg, 0, 0)
    t = 10
    sch = step_schedule(cfg, t)
    sk, sv = inp.sink()
    q, kq, vq = inp.query(t)
    gen = np.random.default_rng(3)
    kg = gen.standard_normal((4, cfg.num_kv_heads, cfg.head_dim))
    vg = gen.standard_normal((4, cfg.num_kv_heads, cfg.head_dim))
    qg = gen.standard_normal((4, cfg.num_q_heads, cfg.head_dim))
    grp = cfg.num_q_heads // cfg.num_kv_heads
    frames = sch.past_frames + sch.instant_frames
    for g in range(4):
        k_self = np.concatenate([kq, kg[: g + 1]]); v_self = np.concatenate([vq, vg[: g + 1]])
        o = O.decode_output(sch, (sk, sv), inp.frame_kv, qg[g:g + 1], k_self, v_self, cfg.rope_theta)
        for h in range(cfg.num_q_heads):
            gh = h // grp
            keys = [(j, list(sk[j, gh]), list(sv[j, gh])) for j in range(cfg.sink_tokens)]
            n = cfg.sink_tokens
            for f in frames:
                fk, fv = inp.frame_kv(f)
                for j in range(cfg.tokens_per_frame):
                    keys.append((n, list(fk[j, gh]), list(fv[j, gh]))); n += 1
            for j in range(len(k_self)):
                keys.append((n, list(k_self[j, gh]), list(v_self[j, gh]))); n += 1
            ref = _brute_attend(list(qg[g, h]), n - 1, keys, cfg.rope_theta)
            assert np.abs(np.array(ref) - o[0, h]).max() < 1e-12


# --------------------------------------------------------------------------- boosted newest frame (NEXT-4)
def test_boost_with_the_buffer_frame_reduces_to_eq7_and_eq8():
    """Re-encoding the newest frame as itself (n_boost = tpf, the ring's own K/V) must give
    the plain instant cache (Eq. 7) and the plain final attention (Eq. 8)."""
    cfg = synth.CONFIGS["c1"]
    inp = StreamInputs(cfg, 0, 0)
    for t in (0, 2, 9):
        sch = step_schedule(cfg, t)
        k, v = inp.frame_kv(sch.instant_frames[-1])
        qi = inp.instant_q(t, sch.C_t)
        a = O.instant_cache_output(sch, inp.sink(), inp.frame_kv, qi, cfg.rope_theta)
        b = O.instant_cache_output_boosted(sch, inp.sink(), inp.frame_kv, qi, k, v, cfg.rope_theta)
        assert np.array_equal(a, b)
        q, ks, vs = inp.query(t)
        a = O.attend_output(sch, inp.sink(), inp.frame_kv, q, ks, vs, cfg.rope_theta)
        b = O.attend_output_boosted(sch, inp.sink(), inp.frame_kv, q, ks, vs, k, v, cfg.rope_theta)
        assert np.array_equal(a, b)


@pytest.mark.parametrize("n_boost", [1, 7])
def test_boost_brute_force_full_history(n_boost):
    """Pure-Python loops over the full token history: the buffer B_t is the last l_I frames
    of the history; its newest frame is swapped for n_boost re-encoded tokens
    in both the instant build and the final cache; ids consecutive from 0."""
    cfg = _upd_cfg()
    inp = StreamInputs(cfg, 0, 0)
    sk, sv = inp.sink()
    A, tpf, lI, lU = cfg.sink_tokens, cfg.tokens_per_frame, cfg.instant_frames, cfg.past_frames
    grp = cfg.num_q_heads // cfg.num_kv_heads
    gen = np.random.default_rng(11)
    history = []
    for t in range(7):
        fk, fv = inp.frame_kv(t)
        history += [(k, v) for k, v in zip(fk, fv)]
        sch = step_schedule(cfg, t)
        kb = gen.standard_normal((n_boost, cfg.num_kv_heads, cfg.head_dim))
        vb = gen.standard_normal((n_boost, cfg.num_kv_heads, cfg.head_dim))
        inst = history[-min(t + 1, lI) * tpf:][:-tpf]           # buffer minus its newest frame
        window = history[-min(t + 1, lI + lU) * tpf:][:-tpf]    # past + older instant frames
        qi = gen.standard_normal((len(inst) + n_boost, cfg.num_q_heads, cfg.head_dim))
        q, kq, vq = inp.query(t)
        oi = O.instant_cache_output_boosted(sch, (sk, sv), inp.frame_kv, qi, kb, vb, cfg.rope_theta)
        o = O.attend_output_boosted(sch, (sk, sv), inp.frame_kv, q, kq, vq, kb, vb, cfg.rope_theta)
        for h in range(cfg.num_q_heads):
            g = h // grp
            base = [(j, list(sk[j, g]), list(sv[j, g])) for j in range(A)]
            keys = base + [(A + n, list(k[g]), list(v[g])) for n, (k, v) in enumerate(inst)]
            keys += [(A + len(inst) + j, list(kb[j, g]), list(vb[j, g])) for j in range(n_boost)]
            for i in range(qi.shape[0]):
                ref = _brute_attend(list(qi[i, h]), A + i, keys, cfg.rope_theta)
                assert np.abs(np.array(ref) - oi[i, h]).max() < 1e-12
            keys = base + [(A + n, list(k[g]), list(v[g])) for n, (k, v) in enumerate(window)]
            keys += [(A + len(window) + j, list(kb[j, g]), list(vb[j, g])) for j in range(n_boost)]
            L = len(keys)
            keys += [(L + i, list(kq[i, g]), list(vq[i, g])) for i in range(q.shape[0])]
            for i in range(q.shape[0]):
                ref = _brute_attend(list(q[i, h]), L + i, keys, cfg.rope_theta)
                assert np.abs(np.array(ref) - o[i, h]).max() < 1e-12


def test_boost_leaves_older_instant_rows_and_ignores_the_past():
    """Causality: instant tokens before the newest frame never see it, so their rows equal
    the plain Eq. 7 rows; and the boosted build is independent of U."""
    cfg = synth.CONFIGS["c1"]
    inp = StreamInputs(cfg, 0, 0)
    t = 9
    sch = step_schedule(cfg, t)
    qi = inp.instant_q(t, sch.C_t)
    kb, vb = (x.double().numpy() for x in synth.boost_kv(cfg, 0, 0, t, 3 * cfg.tokens_per_frame))
    older = sch.C_t - cfg.tokens_per_frame
    q_b = np.concatenate([qi[:older], np.random.default_rng(5).standard_normal((kb.shape[0],) + qi.shape[1:])])
    plain = O.instant_cache_output(sch, inp.sink(), inp.frame_kv, qi, cfg.rope_theta)
    boosted = O.instant_cache_output_boosted(sch, inp.sink(), inp.frame_kv, q_b, kb, vb, cfg.rope_theta)
    assert np.allclose(plain[:older], boosted[:older], rtol=0, atol=1e-13)
    # poison every past frame: the build must not change
    sch2 = O.StepSchedule(sch.t, sch.instant_frames, [], [], sch.tokens_per_frame, sch.sink_tokens)
    again = O.instant_cache_output_boosted(sch2, inp.sink(), inp.frame_kv, q_b, kb, vb, cfg.rope_theta)
    assert np.array_equal(boosted, again)


# --------------------------------------------------------------------------- real-model mode (NEXT-1)
def test_ext_with_the_buffer_kv_reduces_to_eq7_and_eq8():
    """Supplying the buffer frames' own K/V as the instant K/V and the frame K/V as the
    Eq. 5 K/V must give the ring-mode Eq. 7 / Eq. 8 results exactly (same keys, same order)."""
    cfg = synth.CONFIGS["c1"]
    inp = StreamInputs(cfg, 0, 0)
    for t in (0, 2, 9):
        sch = step_schedule(cfg, t)
        ki = np.concatenate([inp.frame_kv(f)[0] for f in sch.instant_frames])
        vi = np.concatenate([inp.frame_kv(f)[1] for f in sch.instant_frames])
        qi = inp.instant_q(t, sch.C_t)
        a = O.instant_cache_output(sch, inp.sink(), inp.frame_kv, qi, cfg.rope_theta)
        b = O.instant_cache_output_ext(sch, inp.sink(), ki, vi, qi, cfg.rope_theta)
        assert np.array_equal(a, b)
        q, ks, vs = inp.query(t)
        a = O.attend_output(sch, inp.sink(), inp.frame_kv, q, ks, vs, cfg.rope_theta)
        b = O.attend_output_ext(sch, inp.sink(), inp.frame_kv, ki, vi, q, ks, vs, cfg.rope_theta)
        assert np.array_equal(a, b)


def _np(x):
    return x.double().numpy()


def test_ext_brute_force_full_history():
    """Pure-Python loops over the full token history in the real-model mode: U holds, for
    each frame that left the buffer, the K/V of its Eq. 5 update, the newest
    l_U of them (Eq. 6); I_t is the step's own instant K/V (Eq. 7), distinct
    from anything in U; [C_a, U_t, I_t] (Eq. 8) plus the query chunk, ids 0..."""
    cfg = _upd_cfg()
    inp = StreamInputs(cfg, 0, 0)
    sk, sv = inp.sink()
    A, tpf, lI, lU = cfg.sink_tokens, cfg.tokens_per_frame, cfg.instant_frames, cfg.past_frames
    grp = cfg.num_q_heads // cfg.num_kv_heads
    pkv = lambda f: tuple(_np(x) for x in synth.past_kv(cfg, 0, 0, f))   # noqa: E731
    left = []   # frames that left the buffer, oldest first: (k, v) per token of past_kv
    for t in range(cfg.num_frames):
        if t - lI >= 0:
            pk, pv = pkv(t - lI)
            left += list(zip(pk, pv))
        sch = step_schedule(cfg, t)
        C_t = min(t + 1, lI) * tpf
        ki, vi = (_np(x) for x in synth.instant_kv(cfg, 0, 0, t, C_t))
        qi = inp.instant_q(t, C_t)
        q, kq, vq = inp.query(t)
        oi = O.instant_cache_output_ext(sch, (sk, sv), ki, vi, qi, cfg.rope_theta)
        o = O.attend_output_ext(sch, (sk, sv), pkv, ki, vi, q, kq, vq, cfg.rope_theta)
        past = left[-lU * tpf:] if lU > 0 else []
        for h in range(cfg.num_q_heads):
            g = h // grp
            base = [(j, list(sk[j, g]), list(sv[j, g])) for j in range(A)]
            keys = base + [(A + n, list(ki[n, g]), list(vi[n, g])) for n in range(C_t)]
            for i in range(C_t):
                ref = _brute_attend(list(qi[i, h]), A + i, keys, cfg.rope_theta)
                assert np.abs(np.array(ref) - oi[i, h]).max() < 1e-12
            keys = base + [(A + n, list(k[g]), list(v[g])) for n, (k, v) in enumerate(past)]
            keys += [(A + len(past) + n, list(ki[n, g]), list(vi[n, g])) for n in range(C_t)]
            L = len(keys)
            keys += [(L + i, list(kq[i, g]), list(vq[i, g])) for i in range(q.shape[0])]
            for i in range(q.shape[0]):
                ref = _brute_attend(list(q[i, h]), L + i, keys, cfg.rope_theta)
                assert np.abs(np.array(ref) - o[i, h]).max() < 1e-12


def test_ext_reads_the_instant_kv_not_u_for_buffer_frames():
    """Negative control + causality: poisoning the Eq. 5 K/V of frames still in the buffer
    changes nothing (I_t, not U, holds them: PAPER.md:226, 230), while swapping the instant
    K/V for the frames' Eq. 5 K/V does change the answer."""
    cfg = _upd_cfg()
    inp = StreamInputs(cfg, 0, 0)
    t = 9
    sch = step_schedule(cfg, t)
    C_t = sch.C_t
    ki, vi = (_np(x) for x in synth.instant_kv(cfg, 0, 0, t, C_t))
    q, kq, vq = inp.query(t)
    pkv = lambda f: tuple(_np(x) for x in synth.past_kv(cfg, 0, 0, f))   # noqa: E731
    inst = set(sch.instant_frames)
    poisoned = lambda f: tuple(np.full_like(x, 1e3) for x in pkv(f)) if f in inst else pkv(f)   # noqa: E731
    a = O.attend_output_ext(sch, inp.sink(), pkv, ki, vi, q, kq, vq, cfg.rope_theta)
    b = O.attend_output_ext(sch, inp.sink(), poisoned, ki, vi, q, kq, vq, cfg.rope_theta)
    assert np.array_equal(a, b)
    k2 = np.concatenate([pkv(f)[0] for f in sch.instant_frames])
    v2 = np.concatenate([pkv(f)[1] for f in sch.instant_frames])
    c = O.attend_output_ext(sch, inp.sink(), pkv, k2, v2, q, kq, vq, cfg.rope_theta)
    assert np.abs(a - c).max() > 1e-3


# --------------------------------------------------------------------------- approximate instant cache (NEXT-3)
def _approx(cfg, inp, t, period, capture=()):
    return O.instant_cache_output_approx(t, period, cfg.instant_frames, cfg.past_frames, cfg.tokens_per_frame,
                                         inp.sink(), inp.frame_kv, inp.instant_q, cfg.rope_theta,
                                         capture=capture)


def test_approx_period_one_and_refresh_steps_are_exact_eq7():
    """period = 1 rebuilds every step (the exact Eq. 7 cache); with any period, a refresh step
    (t mod period == 0) equals the exact build of that step ("periodically refreshed")."""
    cfg = synth.CONFIGS["c1"].replace(instant_frames=4)
    inp = StreamInputs(cfg, 0, 0)
    steps = list(range(12))
    for period, check in ((1, steps), (4, [0, 4, 8]), (3, [0, 3, 6, 9])):
        got = _approx(cfg, inp, max(steps), period, capture=steps)
        for t in check:
            sch = step_schedule(cfg, t)
            ref = O.instant_cache_output(sch, inp.sink(), inp.frame_kv, inp.instant_q(t, sch.C_t), cfg.rope_theta)
            assert np.allclose(got[t], ref, rtol=0, atol=1e-13), (period, t)


def test_approx_incremental_rows_are_the_last_rows_of_eq7():
    """Between refreshes the newest frame's rows are the last tpf rows of the exact Eq. 7
    build of that step (causality: they do not see the other instant queries)."""
    cfg = synth.CONFIGS["c1"].replace(instant_frames=4)
    inp = StreamInputs(cfg, 0, 0)
    tpf = cfg.tokens_per_frame
    got = _approx(cfg, inp, 11, 5, capture=range(12))
    for t in (1, 2, 7, 11):
        sch = step_schedule(cfg, t)
        ref = O.instant_cache_output(sch, inp.sink(), inp.frame_kv, inp.instant_q(t, sch.C_t), cfg.rope_theta)
        assert np.allclose(got[t][-tpf:], ref[-tpf:], rtol=0, atol=1e-13)


@pytest.mark.parametrize("period", [2, 3, 100])
def test_approx_brute_force_closed_form(period):
    """Pure-Python loops: frame f's rows at step t were built at s_f = max(f, P*floor(t/P))
    with the queries of step s_f, over [sink | frames max(0, s_f - l_I + 1) .. f] at ids 0..
    (PAPER.md:236); a frame is never rebuilt between refreshes ("reuse of
    buffer-frame caches").  period 100 > t: purely incremental rows (s_f = f for f > 0)."""
    cfg = synth.StreamConfig("apx", 97, 1, 1, 4, 2, 8, 1e4, 3, 2, 0, 3, 1, 10, "fp32", 1.0)
    inp = StreamInputs(cfg, 0, 0)
    sk, sv = inp.sink()
    A, tpf, lI = cfg.sink_tokens, cfg.tokens_per_frame, cfg.instant_frames
    grp = cfg.num_q_heads // cfg.num_kv_heads
    steps = list(range(cfg.num_frames))
    got = _approx(cfg, inp, max(steps), period, capture=steps)
    for t in steps:
        r = period * (t // period)
        buf = list(range(max(0, t - lI + 1), t + 1))
        assert got[t].shape[0] == len(buf) * tpf
        for n, f in enumerate(buf):
            s_f = max(f, r)
            b = max(0, s_f - lI + 1)
            ctx = list(range(b, f + 1))
            qs = inp.instant_q(s_f, (min(s_f + 1, lI)) * tpf)
            for h in range(cfg.num_q_heads):
                g = h // grp
                keys = [(j, list(sk[j, g]), list(sv[j, g])) for j in range(A)]
                for m, fr in enumerate(ctx):
                    fk, fv = inp.frame_kv(fr)
                    keys += [(A + m * tpf + j, list(fk[j, g]), list(fv[j, g])) for j in range(tpf)]
                for j in range(tpf):
                    row = (f - b) * tpf + j
                    ref = _brute_attend(list(qs[row, h]), A + row, keys, cfg.rope_theta)
                    assert np.abs(np.array(ref) - got[t][n * tpf + j, h]).max() < 1e-12, (t, f, j, h)


def test_approx_differs_from_exact_between_refreshes():
    """Negative control: between refreshes, once a frame has left the buffer since the older
    rows were built, the reused rows differ from the exact Eq. 7 rows (the "residual
    accumulation" of PAPER.md:779); the newest frame's rows never do."""
    cfg = synth.CONFIGS["c1"].replace(instant_frames=4)
    inp = StreamInputs(cfg, 0, 0)
    tpf = cfg.tokens_per_frame
    t = 10                                  # period 8: refresh at 8, l_I = 4
    got = _approx(cfg, inp, t, 8)[t]
    sch = step_schedule(cfg, t)
    ref = O.instant_cache_output(sch, inp.sink(), inp.frame_kv, inp.instant_q(t, sch.C_t), cfg.rope_theta)
    assert np.abs(got[:-tpf] - ref[:-tpf]).max() > 1e-3
    assert np.allclose(got[-tpf:], ref[-tpf:], rtol=0, atol=1e-13)


# --------------------------------------------------------------------------- sampled decode (zeta_decode)
def test_decode_sampled_stride_one_is_decode():
    cfg = synth.CONFIGS["c1"]
    inp = StreamInputs(cfg, 0, 0)
    sch = step_schedule(cfg, 12)
    q, ks, vs = inp.query(12)
    a = O.decode_output(sch, inp.sink(), inp.frame_kv, q[-1:], ks, vs, cfg.rope_theta)
    b = O.decode_output_sampled(sch, inp.sink(), inp.frame_kv, q[-1:], ks, vs, 1, cfg.rope_theta)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("stride", [2, 3, 50])
def test_decode_sampled_brute_force(stride):
    """PAPER.md:695 ("sample the cumulative KV cache at 0.5 FPS during decoding", stride 2 at
    1 FPS): pure-Python attention of one decode token over [sink | past frames f with
    (newest past frame - f) % stride == 0 | instant | self], ids consecutive from 0.  A
    stride beyond l_U keeps the newest past frame alone."""
    cfg = synth.StreamConfig("dec", 96, 1, 1, 4, 2, 8, 1e4, 2, 2, 6, 2, 3, 14, "fp32", 1.0)
    inp = StreamInputs(cfg, 0, 0)
    t = 12
    sch = step_schedule(cfg, t)
    sk, sv = inp.sink()
    q, kq, vq = inp.query(t)
    grp = cfg.num_q_heads // cfg.num_kv_heads
    newest = t - cfg.instant_frames                      # newest frame of U_t (Eq. 3 / 5)
    oldest = newest - cfg.past_frames + 1
    kept = [f for f in range(oldest, newest + 1) if (newest - f) % stride == 0]
    o = O.decode_output_sampled(sch, (sk, sv), inp.frame_kv, q[-1:], kq, vq, stride, cfg.rope_theta)
    if stride > cfg.past_frames:
        assert kept == [newest]
    for h in range(cfg.num_q_heads):
        gh = h // grp
        keys = [(j, list(sk[j, gh]), list(sv[j, gh])) for j in range(cfg.sink_tokens)]
        n = cfg.sink_tokens
        for f in kept + list(range(t - cfg.instant_frames + 1, t + 1)):
            fk, fv = inp.frame_kv(f)
            for j in range(cfg.tokens_per_frame):
                keys.append((n, list(fk[j, gh]), list(fv[j, gh]))); n += 1
        for j in range(len(kq)):
            keys.append((n, list(kq[j, gh]), list(vq[j, gh]))); n += 1
        ref = _brute_attend(list(q[-1, h]), n - 1, keys, cfg.rope_theta)
        assert np.abs(np.array(ref) - o[0, h]).max() < 1e-12


def test_ext_decode_reduces_to_decode():
    """Real-model decoding (the last n_q of n_self self tokens over [C_a, U, I, self]) with the
    buffer's own K/V as the instant K/V and the frame K/V as U equals decode_output."""
    cfg = synth.CONFIGS["c1"]
    inp = StreamInputs(cfg, 0, 0)
    t = 11
    sch = step_schedule(cfg, t)
    ki = np.concatenate([inp.frame_kv(f)[0] for f in sch.instant_frames])
    vi = np.concatenate([inp.frame_kv(f)[1] for f in sch.instant_frames])
    q, ks, vs = inp.query(t)
    gen = np.random.default_rng(21)
    kg = np.concatenate([ks, gen.standard_normal((3,) + ks.shape[1:])])
    vg = np.concatenate([vs, gen.standard_normal((3,) + vs.shape[1:])])
    qg = gen.standard_normal((2,) + q.shape[1:])
    a = O.decode_output(sch, inp.sink(), inp.frame_kv, qg, kg, vg, cfg.rope_theta)
    b = O.attend_output_ext(sch, inp.sink(), inp.frame_kv, ki, vi, qg, kg, vg, cfg.rope_theta)
    assert np.array_equal(a, b)
