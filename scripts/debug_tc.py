"""TC vs SIMT on the GPU for a small stream: per-row error pattern of build_instant / attend."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dscache_synth as synth  # noqa: E402
from paper_2605_01858_b200 import dscache as D  # noqa: E402

cfg = synth.CONFIGS["c2"].replace(tokens_per_frame=int(sys.argv[1]) if len(sys.argv) > 1 else 128, past_frames=2,
                                  instant_frames=1, num_frames=8, query_tokens=40)
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(0)
A, tpf, Hkv, Hq, d = cfg.sink_tokens, cfg.tokens_per_frame, cfg.num_kv_heads, cfg.num_q_heads, 128


def r(*s):
    return (torch.randn(s, device=dev, generator=g) * 0.5).to(torch.bfloat16)


hs = {impl: D.DSCache.from_config(cfg, attn_impl=impl) for impl in (D.IMPL_TC, D.IMPL_SIMT)}
sk, sv = r(1, 1, A, Hkv, d), r(1, 1, A, Hkv, d)
frames = [(r(1, 1, tpf, Hkv, d), r(1, 1, tpf, Hkv, d)) for _ in range(cfg.num_frames)]
for h in hs.values():
    h.append_frame(sk, sv)
for t in range(cfg.num_frames):
    for h in hs.values():
        h.append_frame(*frames[t])
    C = hs[D.IMPL_TC].state(0)["instant_tokens"]
    qi = r(1, 1, C, Hq, d)
    q, ks, vs = r(1, 1, 40, Hq, d), r(1, 1, 40, Hkv, d), r(1, 1, 40, Hkv, d)
    out = {}
    for impl, h in hs.items():
        out[impl] = (h.build_instant(qi).float(), h.attend(q, ks, vs).float())
    torch.cuda.synchronize()
    for k, name in ((0, "build"), (1, "attend")):
        a, b = out[D.IMPL_TC][k][0, 0], out[D.IMPL_SIMT][k][0, 0]   # [rows][Hq][d]
        err = (a - b).norm(dim=-1) / b.norm(dim=-1).clamp_min(1e-9)   # [rows][Hq]
        bad = (err > 2e-2).nonzero()
        print(f"t={t} {name}: rel {((a - b).norm() / b.norm()).item():.3e}  bad rows {bad.shape[0]}/{err.numel()}",
              "first bad (i,h):", bad[:6].tolist(), "max err", err.max().item())
