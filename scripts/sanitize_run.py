"""Small workload that drives every kernel of the library once or twice, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool memcheck python scripts/sanitize_run.py

c1 (fp32: SIMT attention), a shrunk c2 (bf16, tcgen05 kernel: fused step with staged
build, split-KV attend + combine, update attention, boost), the decode kernel (plain,
sampled past, split-KV last-CTA merge), the approximate instant cache and the external
instant (real-model) mode.  Prints one line per phase; exit code 0 when every call
returned without an error."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import dscache_synth as synth  # noqa: E402
from paper_2605_01858_b200 import dscache as D  # noqa: E402


def rnd(*shape, dt=torch.bfloat16):
    return (torch.randn(shape, device="cuda") * 0.5).to(dt)


def stream(cfg, steps, **kw):
    dt = cfg.torch_dtype
    S, N, Hq, Hkv, d, tpf = cfg.num_streams, cfg.num_layers, cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim, cfg.tokens_per_frame
    h = D.DSCache.from_config(cfg, **kw)
    if cfg.sink_tokens:
        h.append_frame(rnd(S, N, cfg.sink_tokens, Hkv, d, dt=dt), rnd(S, N, cfg.sink_tokens, Hkv, d, dt=dt))
    for t in range(steps):
        k, v = rnd(S, N, tpf, Hkv, d, dt=dt), rnd(S, N, tpf, Hkv, d, dt=dt)
        n_inst = min(t + 1, cfg.instant_frames) * tpf
        qi = rnd(S, N, n_inst, Hq, d, dt=dt)
        q, ks, vs = rnd(S, N, cfg.query_tokens, Hq, d, dt=dt), rnd(S, N, cfg.query_tokens, Hkv, d, dt=dt), \
            rnd(S, N, cfg.query_tokens, Hkv, d, dt=dt)
        h.step(k, v, qi, q, ks, vs)
    torch.cuda.synchronize()
    return h


def main():
    torch.manual_seed(0)
    c1 = synth.CONFIGS["c1"]
    h = stream(c1, 8)
    h.close()
    print("c1 fp32 SIMT steps ok", flush=True)

    c2 = synth.CONFIGS["c2"].replace(past_frames=6, num_frames=16, query_tokens=32)
    h = stream(c2, 12)
    S, N, Hq, Hkv, d, tpf = 1, 1, c2.num_q_heads, c2.num_kv_heads, 128, c2.tokens_per_frame
    q, ks, vs = rnd(S, N, 32, Hq, d), rnd(S, N, 32, Hkv, d), rnd(S, N, 32, Hkv, d)
    h.attend(q, ks, vs)                                   # split-KV attend + combine
    h.update_attend(rnd(S, N, tpf, Hq, d), active_frames=4)
    n_boost = 2 * tpf
    C = c2.instant_frames * tpf
    h.build_instant_boost(rnd(S, N, C - tpf + n_boost, Hq, d), rnd(S, N, n_boost, Hkv, d), rnd(S, N, n_boost, Hkv, d))
    h.attend_boost(q, ks, vs, rnd(S, N, n_boost, Hkv, d), rnd(S, N, n_boost, Hkv, d))
    torch.cuda.synchronize()
    print("c2 tcgen05 fused steps / split attend / update / boost ok", flush=True)
    for stride in (1, 2):
        for n_q in (1, 2):
            h.decode(rnd(S, N, n_q, Hq, d), rnd(S, N, 40, Hkv, d), rnd(S, N, 40, Hkv, d), past_stride=stride)
    torch.cuda.synchronize()
    print("decode kernel (strides 1/2, n_q 1/2, split-KV merge) ok", flush=True)
    ring = h.approx_ring()
    for t in range(5):
        h.append_frame(rnd(S, N, tpf, Hkv, d), rnd(S, N, tpf, Hkv, d))
        n = h.approx_rows(ring, 3)
        h.build_instant_approx(rnd(S, N, n, Hq, d), ring, 3)
    torch.cuda.synchronize()
    h.close()
    print("approximate instant cache ok", flush=True)

    e = D.DSCache.from_config(c2, instant_source=D.INSTANT_EXTERNAL)
    e.append_frame(rnd(S, N, c2.sink_tokens, Hkv, d), rnd(S, N, c2.sink_tokens, Hkv, d))
    for t in range(7):
        leave = t - c2.instant_frames
        if leave >= 0:
            e.append_past(rnd(S, N, tpf, Hkv, d), rnd(S, N, tpf, Hkv, d))
            e.update_attend(rnd(S, N, tpf, Hq, d))
        else:
            e.append_past(None, None)
        C_t = e.state(0)["instant_tokens"]
        ki, vi = rnd(S, N, C_t, Hkv, d), rnd(S, N, C_t, Hkv, d)
        e.build_instant_ext(rnd(S, N, C_t, Hq, d), ki, vi)
        e.attend_ext(q, ks, vs, ki, vi)
    torch.cuda.synchronize()
    e.close()
    print("external-instant mode ok", flush=True)


if __name__ == "__main__":
    main()
