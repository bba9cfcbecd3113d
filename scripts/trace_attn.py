"""Per-CTA event timeline of the tcgen05 attention kernel (build_instant and attend)
on a steady-state c5-shaped workload.  Prints, per tile, the cycle at which each
pipeline event happened relative to the CTA start.

    python scripts/trace_attn.py [--streams 8] [--ctas 2]
"""
import argparse
import os
import sys

import torch

# the event timeline is compiled only into the DSC_TRACE=1 variant of the library
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_01858_b200 import _build as _B  # noqa: E402
from paper_2605_01858_b200 import dscache as _D  # noqa: E402
if "DSCACHE_LIB" not in os.environ:
    _defs = [d for d in os.environ.get("DSC_TRACE_DEFS", "").split() if d]
    _D.load_library(_B.build_variant("trace" + "_".join(d.replace("=", "") for d in _defs), ["DSC_TRACE=1"] + _defs))

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dscache_synth as synth  # noqa: E402
from paper_2605_01858_b200 import dscache as D  # noqa: E402

EV = ["K_issue", "V_issue", "KR", "KF(mma)", "S0", "S1", "P0", "P1", "PV0", "PV1", "Q", "start", "end", "VF(mma)"] + [f"Pw{i}" for i in range(8)] + ["max_h0", "max_h1", "exp_h0", "exp_h1", "packed", "resc", "Kdone", "Qdone", "Qloaded", "Qstart", "QKiss", "PV0iss", "PV1iss", "epi0", "epi1"]
NE = 40


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--streams", type=int, default=8)
    ap.add_argument("--ctas", type=int, default=2)
    ap.add_argument("--config", default="c5")
    args = ap.parse_args()
    cfg = synth.CONFIGS[args.config].replace(num_streams=args.streams)
    dev = torch.device("cuda", 0)
    h = D.DSCache.from_config(cfg)
    S, N, A, tpf, Hkv, Hq, d = cfg.num_streams, cfg.num_layers, cfg.sink_tokens, cfg.tokens_per_frame, \
        cfg.num_kv_heads, cfg.num_q_heads, cfg.head_dim

    def r(*s):
        return (torch.randn(s, device=dev) * cfg.scale).to(torch.bfloat16)
    h.append_frame(r(S, N, A, Hkv, d), r(S, N, A, Hkv, d))
    for t in range(cfg.instant_frames + cfg.past_frames):
        h.append_frame(r(S, N, tpf, Hkv, d), r(S, N, tpf, Hkv, d))
    C, q = cfg.C, cfg.query_tokens
    qi, qq, kk, vv = r(S, N, C, Hq, d), r(S, N, q, Hq, d), r(S, N, q, Hkv, d), r(S, N, q, Hkv, d)
    h.build_instant(qi); h.attend(qq, kk, vv)      # warm
    torch.cuda.synchronize()
    for name in ("build_instant", "attend"):
        buf = torch.zeros(args.ctas * NE * 64, dtype=torch.int64, device=dev)
        h.set_trace(buf, args.ctas)
        if name == "build_instant":
            h.build_instant(qi)
        else:
            h.attend(qq, kk, vv)
        torch.cuda.synchronize()
        h.set_trace(None)
        tr = buf.view(args.ctas, NE, 64).cpu()
        for c in range(args.ctas):
            t0 = int(tr[c, 11, 0])
            end = int(tr[c, 12, 0]) - t0
            ntiles = int((tr[c, 8] != 0).sum())
            print(f"== {name} CTA {c}: tiles {ntiles}, total {end} cycles, Q ready at {int(tr[c, 10, 0]) - t0}")
            pro = [int(tr[c, 11, j]) - t0 if int(tr[c, 11, j]) else -1 for j in (1, 2, 3)]
            print(f"   prologue: CTA sync {pro[0]}, copy-WG setmaxnreg {pro[1]}, first item decoded {pro[2]}")
            cols = [0, 1, 2, 28, 3, 32, 13, 4, 6, 8, 33, 5, 7, 9, 34] + [22, 26]
            print("tile " + " ".join(f"{EV[e]:>8}" for e in cols))
            # steady-state summary over tiles 2..ntiles-2 (cycles): tile period at the S0 wait,
            # softmax time per Q tile (S ready -> P arrived), P -> next S latency (PV + QK MMAs)
            def ev(e, j):
                return int(tr[c, e, j]) - t0 if int(tr[c, e, j]) else None
            per, sm0, sm1, lat0, rot, klat, vlat = [], [], [], [], [], [], []
            for j in range(2, min(ntiles, 64) - 1):
                a, b = ev(4, j), ev(4, j + 1)
                if a is not None and b is not None and b > a:
                    per.append(b - a)
                if ev(4, j) is not None and ev(6, j) is not None:
                    sm0.append(ev(6, j) - ev(4, j))
                if ev(5, j) is not None and ev(7, j) is not None:
                    sm1.append(ev(7, j) - ev(5, j))
                if ev(6, j) is not None and ev(4, j + 1) is not None:
                    lat0.append(ev(4, j + 1) - ev(6, j))
                if ev(2, j) is not None and ev(28, j) is not None:
                    rot.append(ev(28, j) - ev(2, j))
                if ev(0, j) is not None and ev(2, j) is not None:
                    klat.append(ev(2, j) - ev(0, j))
                if ev(1, j) is not None and ev(13, j) is not None:
                    vlat.append(ev(13, j) - ev(1, j))
            med = lambda v: sorted(v)[len(v) // 2] if v else -1
            print(f"   summary: median tile period {med(per)}, softmax0 {med(sm0)}, softmax1 {med(sm1)}, "
                  f"P0->S0next {med(lat0)}, K rotate {med(rot)}, K issue->landed {med(klat)}, "
                  f"V issue->MMA {med(vlat)}")
            # item switches of softmax WG0 (indexed by the next item's first tile)
            sw = []
            for j in range(1, 64):
                qs, ql, qd, e0, e1 = (ev(31, j), ev(30, j), ev(29, j), ev(35, j), ev(36, j))
                if qs is not None and e1 is not None:
                    sw.append((j, qs, ql - qs if ql else -1, qd - ql if (qd and ql) else -1, e0 - qd if (e0 and qd) else -1,
                               e1 - e0 if (e1 and e0) else -1))
            # per-warp P arrival spread (the P barrier completes at the LAST warp) vs the MMA's
            # PV issue: tiles 2..ntiles-2
            spread, last_to_pv = [], []
            for j in range(2, min(ntiles, 64) - 1):
                pw = [ev(14 + w_, j) for w_ in range(4)]
                if all(x is not None for x in pw) and ev(8, j) is not None:
                    spread.append(max(pw) - min(pw))
                    last_to_pv.append(ev(8, j) - max(pw))
            print(f"   P0 warp spread (median) {med(spread)}, last P0 warp -> PV0 issue (median) {med(last_to_pv)}")
            lag = [[] for _ in range(8)]
            for j in range(2, min(ntiles, 64) - 1):
                pw = [ev(14 + w_, j) for w_ in range(8)]
                for h0 in (0, 4):
                    grp_ = pw[h0:h0 + 4]
                    if all(x is not None for x in grp_):
                        for w_ in range(4):
                            lag[h0 + w_].append(grp_[w_] - min(grp_))
            print("   P lag behind the WG's first warp, median per softmax warp 0..7: " + " ".join(str(med(l)) for l in lag))
            kw = [ev(3, j) - ev(27, j) for j in range(4, min(ntiles, 64) - 1) if ev(3, j) is not None and ev(27, j) is not None]
            print(f"   MMA K(g+2) wait (median / max) {med(kw)} / {max(kw) if kw else -1}")
            for t in sw[:6]:
                print(f"   switch @tile {t[0]}: start {t[1]}, Q cp.async issue {t[2]}, Q wait+rotate {t[3]}, "
                      f"wait last PV {t[4]}, O read+store {t[5]}")
            for j in range(min(ntiles, 64)):
                row = [int(tr[c, e, j]) - t0 if int(tr[c, e, j]) else -1 for e in cols]
                print(f"{j:4d} " + " ".join(f"{x:8d}" for x in row))
    h.close()


if __name__ == "__main__":
    main()
