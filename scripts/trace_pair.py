"""Event timeline of the v8 pair kernel (attn_fa.cu namespace pr, PR_TRACE=1 variant) on one
steady-state fused step (dscache_step) of a BASELINE config.

    python scripts/trace_pair.py [--config c5] [--lib PATH] [--items 8] [--first-item 0]

Leader CTA (0): per tile the MMA warp's issue times of S(g) and PV(g), when its waits were
satisfied (K ready, V ready, P ready), and the leader's own softmax S -> P span; per item the
Q-ready / O-free waits and the rotation warpgroup's Q prep and epilogue spans.  clock64 is
per SM, so only events of one CTA are compared.
"""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_01858_b200 import _build as _B  # noqa: E402
from paper_2605_01858_b200 import dscache as _D  # noqa: E402

NE, NI = 32, 1024
EV = dict(S_ISS=0, PV_ISS=1, KF_OK=2, VR_OK=3, P_OK=4, SM_S=5, SM_P=6, CPK=7, CPV=8, FWV=9, ROT=10,
          ITEM=12, Q_START=13, Q_FREE=14, Q_END=15, EPI_O=16, EPI_END=17, QR_OK=18, OF_OK=19, END=20, KR_FW=21,
          S_MMA=22, PV_MMA=23, S_FENCE=24, ROT_PRE=25, ROT_KR=26, ROT_RR=27, ROT9=28, ROT10=29, ROT11=30)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--lib", default=None)
    ap.add_argument("--items", type=int, default=8)
    ap.add_argument("--first-item", type=int, default=0)
    ap.add_argument("--tiles", type=int, default=6)
    args = ap.parse_args()
    lib = args.lib or _B.build_variant("ptrace", ["PR_TRACE=1"])
    _D.load_library(lib)
    import dscache_synth as synth
    from paper_2605_01858_b200 import dscache as D
    cfg = synth.CONFIGS[args.config]
    dev = torch.device("cuda", 0)
    h = D.DSCache.from_config(cfg)
    S, N, A, tpf, Hkv, Hq, d = (cfg.num_streams, cfg.num_layers, cfg.sink_tokens, cfg.tokens_per_frame,
                                cfg.num_kv_heads, cfg.num_q_heads, cfg.head_dim)
    g = torch.Generator(device=dev).manual_seed(0)

    def r(*s):
        return (torch.randn(s, device=dev, generator=g) * cfg.scale).to(torch.bfloat16)
    h.append_frame(r(S, N, A, Hkv, d), r(S, N, A, Hkv, d))
    for _ in range(cfg.instant_frames + cfg.past_frames - 1):
        h.append_frame(r(S, N, tpf, Hkv, d), r(S, N, tpf, Hkv, d))
    C, q = cfg.C, cfg.query_tokens
    k, v = r(S, N, tpf, Hkv, d), r(S, N, tpf, Hkv, d)
    qi, qq, kk, vv = r(S, N, C, Hq, d), r(S, N, q, Hq, d), r(S, N, q, Hkv, d), r(S, N, q, Hkv, d)
    for _ in range(3):
        h.step(k, v, qi, qq, kk, vv)
    torch.cuda.synchronize()
    nct = 2
    buf = torch.zeros(nct * NE * NI, dtype=torch.int64, device=dev)
    h.set_trace(buf, nct)
    h.step(k, v, qi, qq, kk, vv)
    torch.cuda.synchronize()
    h.set_trace(None)
    tr = buf.view(nct, NE, NI).cpu()
    t = tr[0]
    t0 = int(t[EV["ITEM"], 0])

    def ev(e, i, tt=t, base=t0):
        x = int(tt[EV[e], i])
        return x - base if x else None
    n_items = int((t[EV["ITEM"]] > 0).sum())
    n_tiles = int((t[EV["PV_ISS"]] > 0).sum())
    end = ev("END", 0)
    print(f"=== leader CTA 0: {n_items} items, {n_tiles} tiles, end {end} clk, {end / max(n_tiles, 1):.0f} clk per tile")
    # item boundaries in global tiles (S issue order: an item's first S follows PV of the previous)
    item_start_clk = [ev("ITEM", i) for i in range(n_items)]
    s_iss = [ev("S_ISS", gg) for gg in range(n_tiles)]
    bounds = []
    gi = 0
    for i in range(n_items):
        while gi < n_tiles and (s_iss[gi] is None or s_iss[gi] < item_start_clk[i]):
            gi += 1
        bounds.append(gi)
    bounds.append(n_tiles)
    for i in range(args.first_item, min(n_items, args.first_item + args.items)):
        g0, g1 = bounds[i], bounds[i + 1]
        span = (ev("ITEM", i + 1) if i + 1 < n_items else end) - ev("ITEM", i)
        print(f"item {i}: tiles {g0}..{g1 - 1} ({g1 - g0}), span {span} clk ({span / max(g1 - g0, 1):.0f}/tile)  "
              f"QR_ok {ev('QR_OK', i)} OF_ok {ev('OF_OK', i)} | Qprep [{ev('Q_START', i)}, free {ev('Q_FREE', i)}, "
              f"end {ev('Q_END', i)}] epi [O {ev('EPI_O', i)}, end {ev('EPI_END', i)}]")
        for gg in range(g0, min(g1, g0 + args.tiles)):
            f = {e: ev(e, gg) for e in ("S_ISS", "PV_ISS", "KF_OK", "VR_OK", "P_OK", "SM_S", "SM_P", "CPK", "CPV", "FWV", "ROT", "KR_FW")}
            print("   g%-4d " % gg + " ".join(f"{k}={v}" for k, v in f.items()))
    # steady-state period statistics over all tiles
    import statistics as st

    def dif(a, b):
        out = []
        for gg in range(n_tiles):
            x, y = ev(a, gg), ev(b, gg)
            if x is not None and y is not None:
                out.append(x - y)
        return out
    for name, a, b in [("S issue -> softmax sees S", "SM_S", "S_ISS"), ("softmax S -> P", "SM_P", "SM_S"),
                       ("softmax P -> MMA P ok", "P_OK", "SM_P"), ("P ok -> PV issued", "PV_ISS", "P_OK"),
                       ("V TMA -> fwd", "FWV", "CPV"), ("K TMA -> fwd", "KR_FW", "CPK"),
                       ("MMA: KF ok -> fence done", "S_FENCE", "KF_OK"), ("MMA: 8 QK MMAs", "S_MMA", "S_FENCE"),
                       ("MMA: S commits", "S_ISS", "S_MMA"), ("MMA: P ok -> PV MMAs done", "PV_MMA", "P_OK"),
                       ("MMA: PV commits", "PV_ISS", "PV_MMA"), ("rot: pre -> KR ok", "ROT_KR", "ROT_PRE"),
                       ("rot: KR ok -> rotated", "ROT_RR", "ROT_KR"), ("rot: rotated -> arrived", "ROT", "ROT_RR"),
                       ("MMA: PV(g) -> S(g+3) start", None, None)]:
        d_ = dif(a, b) if a else [ev("KF_OK", gg + 3) - ev("PV_ISS", gg) for gg in range(n_tiles - 3)
                                   if ev("KF_OK", gg + 3) is not None and ev("PV_ISS", gg) is not None]
        if d_:
            print(f"{name:28s}: median {st.median(d_):7.0f}  p90 {sorted(d_)[int(0.9 * len(d_))]:7.0f}  n {len(d_)}")
    per = [s_iss[gg + 1] - s_iss[gg] for gg in range(n_tiles - 1) if s_iss[gg] is not None and s_iss[gg + 1] is not None]
    if per:
        print(f"S issue period: median {st.median(per):.0f}")
    # the peer (CTA 1): its own clock; intervals only
    tp = tr[1]

    def evp(e, i):
        x = int(tp[EV[e], i])
        return x if x else None
    print("=== peer CTA 1 (own clock)")
    for name, a, b in [("softmax S -> P", "SM_P", "SM_S"), ("V TMA -> fwd", "FWV", "CPV"),
                       ("softmax P(g) -> S(g+1) seen", None, None)]:
        d_ = []
        for gg in range(n_tiles - 1):
            if a is None:
                x, y = evp("SM_S", gg + 1), evp("SM_P", gg)
            else:
                x, y = evp(a, gg), evp(b, gg)
            if x is not None and y is not None:
                d_.append(x - y)
        if d_:
            print(f"{name:28s}: median {st.median(d_):7.0f}  p90 {sorted(d_)[int(0.9 * len(d_))]:7.0f}  n {len(d_)}")
    d_ = [ev("ROT_PRE", gg + 1) - ev("ROT", gg) for gg in range(n_tiles - 1)
          if ev("ROT_PRE", gg + 1) is not None and ev("ROT", gg) is not None]
    if d_:
        print(f"rot: arrived(g) -> pre(g+1) : median {st.median(d_):7.0f}")
    for name, e in [("peer S seen period", "SM_S"), ("peer V fwd period", "FWV"), ("peer V TMA period", "CPV")]:
        xs = [evp(e, gg) for gg in range(n_tiles)]
        pp = [xs[i + 1] - xs[i] for i in range(len(xs) - 1) if xs[i] is not None and xs[i + 1] is not None]
        if pp:
            print(f"{name:28s}: median {st.median(pp):7.0f}")
    d_ = []
    for gg in range(n_tiles - 1):
        x, y = ev("SM_S", gg + 1), ev("SM_P", gg)
        if x is not None and y is not None:
            d_.append(x - y)
    if d_:
        print(f"leader softmax P(g) -> S(g+1) seen: median {st.median(d_):7.0f}")
    print("   g: PV(g-3)end S_start S_end | ROT8..11 lead | ROT8..11 peer | P_lead")
    for gg in range(200, 212):
        def q(e, tt):
            x = int(tt[EV[e], gg])
            return x - int(t[EV["SM_S"], 200]) if x else None
        pv3 = ev("PV_ISS", gg - 3) - ev("SM_S", 200) if ev("PV_ISS", gg - 3) is not None else None
        print(f"   {gg}: {pv3} {q('KF_OK', t)} {q('S_ISS', t)} | {q('ROT', t)} {q('ROT9', t)} {q('ROT10', t)} {q('ROT11', t)} | "
              f"{q('ROT', tp)} {q('ROT9', tp)} {q('ROT10', tp)} {q('ROT11', tp)} | {q('SM_P', t)}")
    print("   g   : S_ISS  PV_ISS | P_lead  ROT_l  ROT_p  FWV_l  FWV_p | S gate: PV(g-3) / KF")
    for gg in range(200, 216):
        def q(e, tt):
            x = int(tt[EV[e], gg]) if gg < NI else 0
            return x - int(t[EV["SM_S"], 200]) if x else None
        pv3 = ev("PV_ISS", gg - 3) - ev("SM_S", 200) if ev("PV_ISS", gg - 3) is not None else None
        print(f"   {gg}: {q('S_ISS', t)} {q('PV_ISS', t)} | {q('SM_P', t)} {q('ROT', t)} {q('ROT', tp)} {q('FWV', t)} {q('FWV', tp)} | {pv3}")
    for gg in range(200, 204):
        print("   peer g%-4d " % gg + " ".join(f"{k}={(evp(k, gg) or 0) - (evp('SM_S', 200) or 0)}" for k in ("SM_S", "SM_P", "CPK", "CPV", "FWV", "ROT")))
        print("   lead g%-4d " % gg + " ".join(f"{k}={(ev(k, gg) or 0) - (ev('SM_S', 200) or 0)}" for k in ("SM_S", "SM_P", "CPK", "CPV", "FWV", "ROT", "VR_OK", "P_OK", "PV_ISS", "S_ISS")))


if __name__ == "__main__":
    main()
