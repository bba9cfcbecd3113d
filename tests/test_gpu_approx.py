"""Approximate instant cache (reading Q23) through
the C ABI vs the fp64 oracle's step-by-step replay (instant_cache_output_approx): full Eq. 7
rebuilds every `period` steps, the newest frame's rows alone in between, the rows of every
buffer frame kept in the caller's row ring (frame f at rows (f mod l_I) * tpf)."""
import numpy as np
import pytest
import torch

import dscache_synth as synth
from oracle import dscache_oracle as O
from oracle.workload import StreamInputs
from tests.gpu_harness import _batch, assert_close
from paper_2605_01858_b200 import dscache as D

pytestmark = pytest.mark.gpu


def ring_rows(o_ring, cfg, t):
    """The row ring reordered to B_t oldest first: [C_t][Hq][d]."""
    tpf, lI = cfg.tokens_per_frame, cfg.instant_frames
    frames = range(max(0, t - lI + 1), t + 1)
    return torch.cat([o_ring[(f % lI) * tpf:(f % lI + 1) * tpf] for f in frames])


def run_approx(cfg, period, capture, exact, skip=()):
    """Returns ({t: {(s,l): rows}}, {t: n_rows}); steps in `skip` make no approximate build."""
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev)
    gen.manual_seed(777 + cfg.cfg_id)
    dsc = D.DSCache.from_config(cfg)
    A, tpf, Hkv, Hq, d = cfg.sink_tokens, cfg.tokens_per_frame, cfg.num_kv_heads, cfg.num_q_heads, cfg.head_dim
    if A > 0:
        skv = {sl: synth.sink_kv(cfg, *sl) for sl in exact}
        dsc.append_frame(_batch(cfg, (A, Hkv, d), exact, lambda s, l: skv[(s, l)][0], dev, gen),
                         _batch(cfg, (A, Hkv, d), exact, lambda s, l: skv[(s, l)][1], dev, gen))
    ring = dsc.approx_ring()
    out, nrows = {}, {}
    for t in range(max(capture) + 1):
        kv = {sl: synth.frame_kv(cfg, *sl, t) for sl in exact}
        dsc.append_frame(_batch(cfg, (tpf, Hkv, d), exact, lambda s, l: kv[(s, l)][0], dev, gen),
                         _batch(cfg, (tpf, Hkv, d), exact, lambda s, l: kv[(s, l)][1], dev, gen))
        if t in skip:
            continue
        C_t = dsc.state(0)["instant_tokens"]
        n = dsc.approx_rows(ring, period)
        nrows[t] = n
        qi = _batch(cfg, (n, Hq, d), exact, lambda s, l: synth.instant_q(cfg, s, l, t, C_t)[C_t - n:], dev, gen)
        dsc.build_instant_approx(qi, ring, period)
        if t in capture:
            torch.cuda.synchronize()
            out[t] = {(s, l): ring_rows(ring[s, l], cfg, t).float().cpu() for (s, l) in exact}
    dsc.close()
    return out, nrows


def check_approx(cfg, period, capture, exact):
    res, nrows = run_approx(cfg, period, capture, exact)
    tpf = cfg.tokens_per_frame
    for t, n in nrows.items():
        C_t = min(t + 1, cfg.instant_frames) * tpf
        assert n == (C_t if t % period == 0 else tpf), (t, n)
    for (s, l) in exact:
        inp = StreamInputs(cfg, s, l)
        ref = O.instant_cache_output_approx(max(capture), period, cfg.instant_frames, cfg.past_frames, tpf,
                                            inp.sink(), inp.frame_kv, inp.instant_q, cfg.rope_theta,
                                            capture=capture)
        for t in capture:
            assert_close(res[t][(s, l)], ref[t], cfg.dtype, f"{cfg.name} approx P={period} t={t} s={s} l={l}")


@pytest.mark.parametrize("period", [1, 3, 8])
def test_approx_c1_fp32_simt(lib, period):
    cfg = synth.CONFIGS["c1"].replace(instant_frames=4)
    check_approx(cfg, period, list(range(cfg.num_frames)), [(0, 0)])


@pytest.mark.parametrize("period", [4, 3])
def test_approx_c2_bf16_tcgen05(lib, period):
    cfg = synth.CONFIGS["c2"]
    check_approx(cfg, period, [0, 1, 3, 4, 5, 6, 7, 9, 13, 14], [(0, 0)])


def test_approx_c5_multistream_staged_refresh(lib):
    cfg = synth.CONFIGS["c5"]
    check_approx(cfg, 4, [2, 4, 5, 7, 9], [(0, 0), (7, 3), (63, 1)])


def test_approx_state_machine_forces_refresh(lib):
    """A skipped step, another period or another row ring invalidates the reused rows: the
    next build is a refresh (C_t query rows) and then equals the exact Eq. 7 build."""
    cfg = synth.CONFIGS["c2"]
    res, nrows = run_approx(cfg, 4, [6, 9], [(0, 0)], skip=(5,))
    C = cfg.instant_frames * cfg.tokens_per_frame
    assert nrows[6] == C and nrows[7] == cfg.tokens_per_frame and nrows[8] == C
    inp = StreamInputs(cfg, 0, 0)
    from oracle.workload import step_schedule
    sch = step_schedule(cfg, 6)
    ref = O.instant_cache_output(sch, inp.sink(), inp.frame_kv, inp.instant_q(6, sch.C_t), cfg.rope_theta)
    assert_close(res[6][(0, 0)], ref, cfg.dtype, "refresh after a skipped step")
    dsc = D.DSCache.from_config(cfg)
    z = torch.zeros(1, 1, cfg.sink_tokens, cfg.num_kv_heads, cfg.head_dim, dtype=torch.bfloat16, device="cuda")
    dsc.append_frame(z, z)
    f = torch.zeros(1, 1, cfg.tokens_per_frame, cfg.num_kv_heads, cfg.head_dim, dtype=torch.bfloat16, device="cuda")
    ring, ring2 = dsc.approx_ring(), dsc.approx_ring()
    for t in range(3):
        dsc.append_frame(f, f)
        n = dsc.approx_rows(ring, 4)
        q = torch.zeros(1, 1, n, cfg.num_q_heads, cfg.head_dim, dtype=torch.bfloat16, device="cuda")
        dsc.build_instant_approx(q, ring, 4)
    dsc.append_frame(f, f)
    assert dsc.approx_rows(ring, 4) == cfg.tokens_per_frame
    assert dsc.approx_rows(ring2, 4) == 4 * cfg.tokens_per_frame       # another ring
    assert dsc.approx_rows(ring, 5) == 4 * cfg.tokens_per_frame        # another period
    q = torch.zeros(1, 1, 4 * cfg.tokens_per_frame, cfg.num_q_heads, cfg.head_dim, dtype=torch.bfloat16,
                    device="cuda")
    with pytest.raises(D.DSCacheError) as e:
        dsc.build_instant_approx(q, ring, 4)                           # tpf rows expected
    assert e.value.status == D.E_ARG
    with pytest.raises(D.DSCacheError) as e:
        dsc.approx_rows(ring, 0)
    assert e.value.status == D.E_ARG
    dsc.close()
