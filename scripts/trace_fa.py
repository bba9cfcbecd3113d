"""Event timeline of the v7 tcgen05 kernel (attn_fa.cu, FA_TRACE=1 variant) on one
steady-state fused step (dscache_step) of a BASELINE config.

    python scripts/trace_fa.py [--config c5] [--ctas 2] [--lib PATH]

Per traced CTA: item list with start / end cycles, the MMA warp's per-tile waits (P0, P1,
K, V), the softmax latency S -> P per Q tile, and a split of the CTA's time into tile
periods and item switches.
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
EV = {"MMA_P0": 0, "MMA_P1": 1, "MMA_K": 2, "MMA_V": 3, "SM0_S": 4, "SM0_P": 5, "SM1_S": 6, "SM1_P": 7,
      "ROT_KR": 8, "ROT_KF": 9, "CPK": 10, "CPV": 11, "MMA_ITEM": 12, "MMA_Q0": 13, "MMA_Q1": 14, "EPI0_O": 15,
      "EPI0_END": 16, "QE_START": 17, "QE_END": 18, "QO_START": 19, "QO_FREE": 20, "QO_END": 21, "MMA_OF": 22,
      "EPI1_O": 23, "EPI1_END": 24, "END": 25, "SMX_LD0": 26, "SMX_EX0": 27, "SMX_LD1": 28, "SMX_EX1": 29, "MMA_PV0I": 30, "MMA_S0I": 31}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--ctas", type=int, default=2)
    ap.add_argument("--lib", default=None)
    ap.add_argument("--items", type=int, default=12, help="items printed per CTA")
    ap.add_argument("--tiles", type=int, default=4, help="tiles printed per item")
    ap.add_argument("--first-item", type=int, default=0, help="first item printed per CTA")
    args = ap.parse_args()
    lib = args.lib or _B.build_variant("trace", ["FA_TRACE=1"])
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
    buf = torch.zeros(args.ctas * NE * NI, dtype=torch.int64, device=dev)
    h.set_trace(buf, args.ctas)
    h.step(k, v, qi, qq, kk, vv)
    torch.cuda.synchronize()
    h.set_trace(None)
    tr = buf.view(args.ctas, NE, NI).cpu()
    for c in range(args.ctas):
        t = tr[c]
        t0 = int(t[EV["MMA_ITEM"], 0])
        rel = lambda e, i: int(t[EV[e], i]) - t0 if int(t[EV[e], i]) else None  # noqa: E731
        n_items = int((t[EV["MMA_ITEM"]] > 0).sum())
        end = rel("END", 0)
        print(f"=== CTA {c}: {n_items} items, MMA warp end at {end} clk")
        starts = [rel("MMA_ITEM", i) for i in range(n_items)]
        # tiles per item from the per-tile MMA_P0 events between item starts
        p0 = [rel("MMA_P0", g_) for g_ in range(NI)]
        ntile = sum(1 for x in p0 if x is not None)
        gi = 0
        rows = []
        for i in range(n_items):
            nxt = starts[i + 1] if i + 1 < n_items else end
            tiles = []
            while gi < ntile and p0[gi] is not None and (nxt is None or p0[gi] < nxt):
                tiles.append(gi)
                gi += 1
            rows.append((i, starts[i], nxt, tiles))
        sm_lat = []
        for i, st, nx, tiles in rows[args.first_item:args.first_item + args.items]:
            q0, q1, of = rel("MMA_Q0", i), rel("MMA_Q1", i), rel("MMA_OF", i)
            print(f" item {i:3d}: start {st:8d}  Q0 +{(q0 or st) - st:5d} Q1 +{(q1 or st) - st:5d} OF +{(of or st) - st:5d}"
                  f"  tiles {len(tiles):3d}  dur {((nx or st) - st):7d}  per tile {((nx or st) - st) / max(len(tiles), 1):7.0f}")
            print(f"    epi0 of prev: O-ready {rel('EPI0_O', i - 1) if i else None} end {rel('EPI0_END', i - 1) if i else None}"
                  f"  epi1: O-ready {rel('EPI1_O', i - 1) if i else None} end {rel('EPI1_END', i - 1) if i else None}"
                  f"  Q0 prep {rel('QE_START', i)}..{rel('QE_END', i)}  Q1 prep {rel('QO_START', i)} free {rel('QO_FREE', i)} end {rel('QO_END', i)}")
            for g_ in tiles[:args.tiles]:
                s0, p0_, s1, p1 = rel("SM0_S", g_), rel("SM0_P", g_), rel("SM1_S", g_), rel("SM1_P", g_)
                print(f"    g {g_:4d}: S0 {s0} P0 {p0_} (sm {p0_ - s0 if s0 and p0_ else '-'})  S1 {s1} P1 {p1} "
                      f"(sm {p1 - s1 if s1 and p1 else '-'})  mmaP0 {rel('MMA_P0', g_)} mmaP1 {rel('MMA_P1', g_)} "
                      f"K {rel('MMA_K', g_)} V {rel('MMA_V', g_)} | cpK {rel('CPK', g_)} cpV {rel('CPV', g_)} "
                      f"rotKR {rel('ROT_KR', g_)} rotKF {rel('ROT_KF', g_)}")
        for g_ in range(ntile):
            s0, p0_ = rel("SM0_S", g_), rel("SM0_P", g_)
            if s0 is not None and p0_ is not None:
                sm_lat.append(p0_ - s0)
        parts = {"S->ld0": [], "ld0->ex0": [], "ex0->ld1": [], "ld1->ex1": [], "ex1->P": []}
        for g_ in range(ntile):
            ev = [rel(e, g_) for e in ("SM0_S", "SMX_LD0", "SMX_EX0", "SMX_LD1", "SMX_EX1", "SM0_P")]
            if all(x is not None for x in ev):
                for (k_, a_, b_) in zip(parts, ev, ev[1:]):
                    parts[k_].append(b_ - a_)
        mparts = {"P0->PV0issued": [], "PV0issued->Kready": [], "Kready->S0issued": [], "S0issued->S0done": []}
        for g_ in range(ntile - 1):
            ev = [rel("MMA_P0", g_), rel("MMA_PV0I", g_), rel("MMA_K", g_ + 1), rel("MMA_S0I", g_ + 1), rel("SM0_S", g_ + 1)]
            if all(x is not None for x in ev):
                for (k_, a_, b_) in zip(mparts, ev, ev[1:]):
                    mparts[k_].append(b_ - a_)
        if mparts["P0->PV0issued"]:
            print(" MMA warp steps (median clk): " + ", ".join(f"{k_} {sorted(v)[len(v) // 2]}" for k_, v in mparts.items()))
        if parts["S->ld0"]:
            print(" softmax0 warp0 steps (median clk): " + ", ".join(
                f"{k_} {sorted(v)[len(v) // 2]}" for k_, v in parts.items()))
        if sm_lat:
            sm_lat.sort()
            print(f" softmax0 S->P latency: median {sm_lat[len(sm_lat) // 2]} p10 {sm_lat[len(sm_lat) // 10]} "
                  f"p90 {sm_lat[9 * len(sm_lat) // 10]} over {len(sm_lat)} tiles")
        # MMA-side gaps: P0(g) -> P0(g+1) within an item
        per = []
        for i, st, nx, tiles in rows:
            for a, b in zip(tiles, tiles[1:]):
                per.append(p0[b] - p0[a])
        if per:
            per.sort()
            print(f" tile period (MMA P0->P0 inside items): median {per[len(per) // 2]} p10 {per[len(per) // 10]} "
                  f"p90 {per[9 * len(per) // 10]} over {len(per)}")
        sw = []
        for (i, st, nx, tiles), (i2, st2, nx2, tiles2) in zip(rows, rows[1:]):
            if tiles and tiles2:
                sw.append(p0[tiles2[0]] - p0[tiles[-1]])
        if sw:
            sw.sort()
            print(f" item switch (last P0 -> next item's first P0): median {sw[len(sw) // 2]} p90 {sw[9 * len(sw) // 10]}"
                  f" total {sum(sw)} of {end}")
        qo = [(rel("QO_START", i), rel("QO_FREE", i), rel("QO_END", i)) for i in range(n_items)]
        qo = [(a, b, c_) for a, b, c_ in qo if a is not None and c_ is not None]
        if qo:
            print(" Q1 prep (start, free-wait, load+rotate): median wait "
                  f"{sorted(b - a for a, b, c_ in qo)[len(qo) // 2]} median load+rot {sorted(c_ - b for a, b, c_ in qo)[len(qo) // 2]}")
    h.close()


if __name__ == "__main__":
    main()
