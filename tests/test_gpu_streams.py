"""Concurrent use of the library from several CUDA streams (per-call split-KV
workspace, per-handle schedule cache).  include/dscache.h: every call is stream-ordered on
the stream passed in; layers may be advanced separately.  Results computed concurrently
on two streams must be bit-identical to the same calls issued one after another."""
import pytest
import torch

import dscache_synth as synth
from paper_2605_01858_b200 import dscache as D

pytestmark = pytest.mark.gpu


def _r(gen, dev, dt, scale, *shape):
    return (torch.randn(shape, generator=gen, device=dev) * scale).to(dt)


def _frames(cfg, n, seed, dt, dev):
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    S, N, tpf, Hq, Hkv, d, q = (cfg.num_streams, cfg.num_layers, cfg.tokens_per_frame, cfg.num_q_heads,
                                cfg.num_kv_heads, cfg.head_dim, cfg.query_tokens)
    sink = (_r(gen, dev, dt, cfg.scale, S, N, cfg.sink_tokens, Hkv, d), _r(gen, dev, dt, cfg.scale, S, N, cfg.sink_tokens, Hkv, d))
    steps = []
    for t in range(n):
        C_t = min(t + 1, cfg.instant_frames) * tpf
        steps.append(dict(k=_r(gen, dev, dt, cfg.scale, S, N, tpf, Hkv, d), v=_r(gen, dev, dt, cfg.scale, S, N, tpf, Hkv, d),
                          qi=_r(gen, dev, dt, cfg.scale, S, N, C_t, Hq, d), q=_r(gen, dev, dt, cfg.scale, S, N, q, Hq, d),
                          ks=_r(gen, dev, dt, cfg.scale, S, N, q, Hkv, d), vs=_r(gen, dev, dt, cfg.scale, S, N, q, Hkv, d)))
    return sink, steps


def _layer_calls(h, st, l, stream):
    sl = slice(l, l + 1)
    oi = torch.empty_like(st["qi"][:, sl])
    o = torch.empty_like(st["q"][:, sl])
    args = dict(layer_begin=l, layer_count=1, stream=stream)
    h.build_instant(st["qi"][:, sl].contiguous(), o_inst=oi, **args)
    h.attend(st["q"][:, sl].contiguous(), st["ks"][:, sl].contiguous(), st["vs"][:, sl].contiguous(), o=o, **args)
    return oi, o


def test_layers_on_two_streams_match_serial(lib):
    # one stream, two layers: few work items, so the attend takes the split-KV path (workspace)
    cfg = synth.CONFIGS["c2"].replace(name="c2_2l", num_layers=2, past_frames=8)
    dev = torch.device("cuda", 0)
    dt = torch.bfloat16
    sink, steps = _frames(cfg, 14, 5, dt, dev)
    outs = {}
    for mode in ("serial", "concurrent"):
        h = D.DSCache.from_config(cfg)
        h.append_frame(*sink)
        s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        res = []
        for st in steps:
            h.append_frame(st["k"], st["v"])
            with torch.no_grad():
                if mode == "serial":
                    r = [_layer_calls(h, st, l, torch.cuda.current_stream()) for l in range(2)]
                else:
                    # inputs are made contiguous on the current stream; the side streams wait for it
                    cur = torch.cuda.current_stream()
                    s1.wait_stream(cur); s2.wait_stream(cur)
                    with torch.cuda.stream(s1):
                        r0 = _layer_calls(h, st, 0, s1)
                    with torch.cuda.stream(s2):
                        r1 = _layer_calls(h, st, 1, s2)
                    cur.wait_stream(s1); cur.wait_stream(s2)
                    for t in r0 + r1:
                        t.record_stream(cur)
                    r = [r0, r1]
            res.append([(a.clone(), b.clone()) for a, b in r])
        torch.cuda.synchronize()
        outs[mode] = res
        h.close()
    for t, (ra, rb) in enumerate(zip(outs["serial"], outs["concurrent"])):
        for l in range(2):
            assert torch.equal(ra[l][0], rb[l][0]), f"O_inst step {t} layer {l}"
            assert torch.equal(ra[l][1], rb[l][1]), f"O step {t} layer {l}"


def test_two_handles_two_shapes_interleaved(lib):
    # two handles whose launch shapes differ every warm-up step, driven from two streams with
    # no host synchronisation in between (schedule tables must not be rewritten under a reader)
    cfgs = [synth.CONFIGS["c2"].replace(name="x", past_frames=5, instant_frames=3),
            synth.CONFIGS["c2"].replace(name="y", num_streams=3, past_frames=3, instant_frames=2, query_tokens=16)]
    dev = torch.device("cuda", 0)
    data = [_frames(c, 12, 11 + i, torch.bfloat16, dev) for i, c in enumerate(cfgs)]
    outs = {}
    for mode in ("serial", "concurrent"):
        hs = [D.DSCache.from_config(c) for c in cfgs]
        streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
        cur = torch.cuda.current_stream()
        for h, (sink, _) in zip(hs, data):
            h.append_frame(*sink)
        for s in streams:
            s.wait_stream(cur)
        res = [[], []]
        for t in range(12):
            for i, (h, (_, steps)) in enumerate(zip(hs, data)):
                st = steps[t]
                s = streams[i] if mode == "concurrent" else cur
                oi = torch.empty_like(st["qi"]); o = torch.empty_like(st["q"])
                with torch.cuda.stream(s):
                    h.step(st["k"], st["v"], st["qi"], st["q"], st["ks"], st["vs"], o_inst=oi, o=o, stream=s)
                res[i].append((oi, o))
        for s in streams:
            cur.wait_stream(s)
        torch.cuda.synchronize()
        outs[mode] = res
        for h in hs:
            h.close()
    for i in range(2):
        for t in range(12):
            assert torch.equal(outs["serial"][i][t][0], outs["concurrent"][i][t][0]), f"handle {i} O_inst step {t}"
            assert torch.equal(outs["serial"][i][t][1], outs["concurrent"][i][t][1]), f"handle {i} O step {t}"
