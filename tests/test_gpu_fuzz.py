"""Randomised shapes through the C ABI vs the fp64 oracle: a fixed-seed sample of small
configurations spanning the parameter space the header allows -- head_dim 64 / 128, bf16 /
fp32, split-half / adjacent RoPE, GQA group 1..7, tokens per frame 1..130, sink 0..130,
l_I 0..4, l_U 0..5, query chunks 1..64, several streams and layers -- each streamed through
warm-up and steady-state steps with the split calls and with the fused dscache_step
(ring-slot layout, eviction and ids are exercised by every step; values compared with the
oracle at the north_star bars).  The tcgen05 kernel serves the bf16 / d128 / split-half
cases, the SIMT kernel the rest."""
import numpy as np
import pytest

import dscache_synth as synth
from oracle import dscache_oracle as O
from tests.gpu_harness import run_stream
from tests.test_gpu_parity import _check_steps, run_stream_style
from paper_2605_01858_b200 import dscache as D

pytestmark = pytest.mark.gpu


def _configs(n=32, seed=2024):
    rng = np.random.default_rng(seed)
    out = []
    for k in range(n):
        d = int(rng.choice([64, 128], p=[0.3, 0.7]))
        dtype = str(rng.choice(["bf16", "fp32"], p=[0.75, 0.25]))
        hkv = int(rng.choice([1, 2, 4]))
        grp = int(rng.choice([1, 2, 4, 7]))
        tpf = int(rng.choice([1, 3, 16, 50, 130]))
        A = int(rng.choice([0, 1, 5, 130]))
        lI = int(rng.integers(0, 5))
        lU = int(rng.integers(0 if lI > 0 else 1, 6))
        q = int(rng.choice([1, 7, 64]))
        S, N = int(rng.integers(1, 4)), int(rng.integers(1, 3))
        frames = lI + lU + 3
        style = int(rng.choice([O.SPLIT_HALF, O.ADJACENT], p=[0.8, 0.2]))
        cfg = synth.StreamConfig(f"fz{k}", 200 + k, S, N, hkv * grp, hkv, d, float(rng.choice([1e4, 1e6])), tpf, A,
                                 lU, lI, q, frames, dtype, 0.5 if dtype == "bf16" else 1.0)
        out.append((cfg, style))
    return out


CASES = _configs()


@pytest.mark.parametrize("idx", range(len(CASES)))
def test_fuzz_split_calls(lib, idx):
    cfg, style = CASES[idx]
    steps = sorted({0, max(0, cfg.instant_frames - 1), cfg.instant_frames + cfg.past_frames, cfg.num_frames - 1})
    exact = sorted({(0, 0), (cfg.num_streams - 1, cfg.num_layers - 1)})
    if style == O.ADJACENT:
        res = run_stream_style(cfg, steps, D.ROPE_ADJACENT)
        exact = [(0, 0)]
    else:
        res = run_stream(cfg, steps, exact)
    _check_steps(cfg, res, steps, exact, style=style, tag=f"-fuzz{idx}")


@pytest.mark.parametrize("idx", [i for i, (c, st) in enumerate(CASES) if st == O.SPLIT_HALF])
def test_fuzz_fused_step(lib, idx):
    cfg, style = CASES[idx]
    steps = sorted({0, cfg.instant_frames + cfg.past_frames, cfg.num_frames - 1})
    exact = sorted({(0, 0), (cfg.num_streams - 1, cfg.num_layers - 1)})
    res = run_stream(cfg, steps, exact, fused=True)
    _check_steps(cfg, res, steps, exact, style=style, tag=f"-fuzzstep{idx}")


@pytest.mark.parametrize("idx", [i for i, (c, st) in enumerate(CASES) if st == O.SPLIT_HALF])
def test_fuzz_decode(lib, idx):
    """Decode (and the sampled past) on the same shapes: the decode kernel where it applies
    (bf16, d 128, <= 16 query rows per kv head), else the attention or SIMT kernel."""
    from tests.test_gpu_decode import check_decode
    cfg, _ = CASES[idx]
    n_q = 1 + idx % 2
    stride = 1 + (idx // 2) % 3
    exact = sorted({(0, 0), (cfg.num_streams - 1, cfg.num_layers - 1)})
    check_decode(cfg, cfg.num_frames - 1, exact, cfg.query_tokens + 3, n_q, stride)


@pytest.mark.parametrize("idx", [i for i, (c, st) in enumerate(CASES) if st == O.SPLIT_HALF and c.instant_frames > 0])
def test_fuzz_approx(lib, idx):
    """The approximate instant cache (refresh state machine) on the same shapes, every step."""
    from tests.test_gpu_approx import check_approx
    cfg, _ = CASES[idx]
    period = 1 + idx % 4
    check_approx(cfg, period, list(range(cfg.num_frames)), sorted({(0, 0), (cfg.num_streams - 1, cfg.num_layers - 1)}))


@pytest.mark.parametrize("idx", [i for i, (c, st) in enumerate(CASES) if st == O.SPLIT_HALF])
def test_fuzz_ext(lib, idx):
    """The real-model mode (caller instant K/V, Eq. 5 K/V in U, Eq. 5 attention) on the same shapes."""
    from tests.test_gpu_ext import check_ext
    cfg, _ = CASES[idx]
    steps = sorted({0, cfg.instant_frames + cfg.past_frames, cfg.num_frames - 1})
    check_ext(cfg, steps, sorted({(0, 0), (cfg.num_streams - 1, cfg.num_layers - 1)}),
              l_L=max(1, cfg.past_frames) if cfg.past_frames > 0 else None)
