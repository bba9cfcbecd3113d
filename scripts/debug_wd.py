"""Run one config's fused step with DSC_WATCHDOG=1 and print the kernel's watchdog records
(which warp waited on which barrier when the pipeline stalled).

    DSC_WATCHDOG=1 python scripts/debug_wd.py [--config c2] [--streams S]
"""
import argparse
import os
import sys

os.environ.setdefault("DSC_WATCHDOG", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import dscache_synth as synth  # noqa: E402
from paper_2605_01858_b200 import dscache as D  # noqa: E402

NAMES = ["QR0", "QR1", "QR2", "QF0", "QF1", "QF2", "KR0", "KR1", "KF0", "KF1", "KE0", "KE1", "VR0", "VR1", "VE0",
         "VE1", "S0", "S1", "P0", "P1", "O0", "O1", "OF0", "OF1"]
ROLE = {**{w: f"softmax{w // 4}" for w in range(8)}, **{w: "rotation" for w in range(8, 12)}, 12: "copyK", 13: "copyV",
        14: "mma", 15: "idle"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--streams", type=int, default=0)
    ap.add_argument("--steps", type=int, default=0)
    ap.add_argument("--api", default="fused")
    args = ap.parse_args()
    cfg = synth.CONFIGS[args.config]
    if args.streams:
        cfg = cfg.replace(num_streams=args.streams)
    dev = torch.device("cuda", 0)
    h = D.DSCache.from_config(cfg)
    S, N, A, tpf, Hkv, Hq, d = (cfg.num_streams, cfg.num_layers, cfg.sink_tokens, cfg.tokens_per_frame,
                                cfg.num_kv_heads, cfg.num_q_heads, cfg.head_dim)

    def r(*s):
        return (torch.randn(s, device=dev) * cfg.scale).to(torch.bfloat16)
    try:
        h.append_frame(r(S, N, A, Hkv, d), r(S, N, A, Hkv, d))
        steps = args.steps or (cfg.instant_frames + cfg.past_frames + 2)
        for t in range(steps):
            C_t = min(t + 1, cfg.instant_frames) * tpf
            q = cfg.query_tokens
            if args.api == "fused":
                h.step(r(S, N, tpf, Hkv, d), r(S, N, tpf, Hkv, d), r(S, N, C_t, Hq, d), r(S, N, q, Hq, d),
                       r(S, N, q, Hkv, d), r(S, N, q, Hkv, d))
            else:
                h.append_frame(r(S, N, tpf, Hkv, d), r(S, N, tpf, Hkv, d))
                h.build_instant(r(S, N, C_t, Hq, d))
                h.attend(r(S, N, q, Hq, d), r(S, N, q, Hkv, d), r(S, N, q, Hkv, d))
            torch.cuda.synchronize()
            print(f"step {t} ok", flush=True)
    except Exception as e:  # noqa: BLE001
        print("FAILED:", str(e).splitlines()[0])
    recs = D.watchdog_records()
    print(f"{len(recs or [])} watchdog records")
    for cta, warp, b, par, clk in sorted(recs or [], key=lambda x: x[4]):
        print(f"  cta {cta:3d} warp {warp:2d} ({ROLE.get(warp, '?'):9s}) waits {NAMES[b] if b < len(NAMES) else b} parity {par}  clk {clk}")


if __name__ == "__main__":
    main()
