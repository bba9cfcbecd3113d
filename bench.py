#!/usr/bin/env python3
"""DSCache streaming hot-path benchmark (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl ours|reference]

A *step* is one pass of the whole hot path for every (stream, layer) a rank
holds: append the new frame's raw K/V (ring append + FIFO eviction), build the
instant cache (Eq. 7), and attend the query chunk over [sink|past|instant|self]
(Eq. 8), all through the C ABI on one CUDA stream.  Default workload is c5
(BASELINE.json configs[4]: 64 independent streams x 4 layers of the 7B
attention shape), the configuration the metric is quoted on "at 1/2/4/8 GPUs";
for N > 1 its 64 streams are partitioned across ranks (rank r holds streams
[r*64/N, (r+1)*64/N)), with no collective on the data path.  Timed steps are
steady state (the window is full: l_I + l_U frames appended before timing).

value = frames processed by all ranks / max-over-ranks device time (frames/s,
one frame per stream per step).  The ring (3.8 GB for c5) is far larger than
L2, so no L2 flush is needed; for configs whose working set fits in L2 the
bench flushes L2 between steps and times each step separately.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import dscache_synth as synth  # noqa: E402

METRIC = "frames/s per stream and attention TFLOP/s (% B200 bf16 peak) at 1/2/4/8 GPUs"
L2_BYTES = 126 * 1024 * 1024


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"bf16_tflops": d["bf16_tflops"], "bf16_tflops_sustained": d.get("bf16_tflops_sustained"),
                "hbm_gbs": d["hbm_gbs"], "source": "measured (MEASURED_PEAKS.json)"}
    return {"bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "hbm_gbs": 6650.0,
            "source": "fallback (B200_PROFILING.md)"}


# ----------------------------------------------------------------------------- workload arithmetic
# the attention kernel the library runs (attn_fa.cu): v8 = the CTA-pair kernel (default), v7 with DSC_FA=7
FA_VER = "7" if os.environ.get("DSC_FA", "")[:1] == "7" else "8"
FA_KERNEL = {"8": "attn_pair_kernel (v8: tcgen05.mma.cta_group::2 CTA-pair rotate-on-load GQA flash attention)",
             "7": "attn_fa_kernel (v7 tcgen05 rotate-on-load GQA flash attention)"}[FA_VER]


def traffic_key(args, world: int) -> str:
    key = f"{args.config}|{args.mode}|{args.api}|boost{args.boost:g}|world{world}|layerseq{int(args.layer_seq)}"
    if FA_VER == "8" and args.mode != "decode":   # v8 captures are keyed apart from the v7 ones
        key = "v8|" + key
    if getattr(args, "approx", 0):
        key += f"|approx{args.approx}"
    if getattr(args, "instant_frames", None):
        key += f"|lI{args.instant_frames}"
    if args.mode == "decode":
        key += f"|nq{args.decode_nq}|gen{args.decode_gen}|stride{args.decode_stride}"
    return key


def config_dict(cfg, args, world: int, S_local=None):
    """The `config` object of the JSON line, shared by both arms (same workload description)."""
    A, P, C, q = steady_counts(cfg)
    par = "single GPU"
    if world > 1:
        par = {"kvsplit": f"KV-head split x{world} (NCCL all-gather of O)",
               "context": f"context split x{world} (NCCL all-gather of partials + merge)"}.get(
                   args.mode, f"stream partition x{world}")
    return {"workload": f"{cfg.name}: {cfg.num_streams} streams x {cfg.num_layers} layers, Hq={cfg.num_q_heads} "
                        f"Hkv={cfg.num_kv_heads} d={cfg.head_dim}, tpf={cfg.tokens_per_frame}, A={A}, "
                        f"W={cfg.past_frames}f, C={cfg.instant_frames}f, q={q}",
            "config_id": cfg.name, "streams": cfg.num_streams, "layers": cfg.num_layers, "query_tokens": q,
            "parallelism": par, "mode": args.mode, "api": args.api, "layer_sequential": bool(args.layer_seq),
            "n_boost": int(round(args.boost * cfg.tokens_per_frame)) if args.boost > 0 else 0,
            "approx_period": getattr(args, "approx", 0) or None,
            "steady_state": True}


def steady_counts(cfg, n_q=None):
    """Steady-state token counts per (stream, layer): A, P = W, C, q."""
    n_q = cfg.query_tokens if n_q is None else n_q
    return cfg.sink_tokens, cfg.W, cfg.C, n_q


def flops_per_unit(cfg, n_boost=0, newest_only=False):
    """Algorithmic FLOPs of one (stream, layer) step: 4 * d * Hq * visible (query, key) pairs.
    build: instant token i sees A + i + 1 keys; attend: query i sees A + P + C + i + 1 keys.
    With a boosted newest frame (n_boost tokens) the instant segment holds C - tpf + n_boost.
    newest_only (approximate instant cache between refreshes): only the last tpf instant rows."""
    A, P, C, q = steady_counts(cfg)
    if n_boost:
        C = C - cfg.tokens_per_frame + n_boost
    k = 4 * cfg.head_dim * cfg.num_q_heads
    build = k * (C * A + C * (C + 1) // 2)
    if newest_only:
        first = C - cfg.tokens_per_frame          # rows C - tpf .. C - 1
        build = k * (cfg.tokens_per_frame * A + (C * (C + 1) - first * (first + 1)) // 2)
    attend = k * (q * (A + P + C) + q * (q + 1) // 2)
    return build, attend


def bytes_per_unit(cfg):
    """Algorithmic HBM bytes of one (stream, layer) step (each context K/V row read once,
    Q read, O written, append read + written; eviction moves nothing)."""
    A, P, C, q = steady_counts(cfg)
    e = 2 if cfg.dtype == "bf16" else 4
    row_kv = cfg.num_kv_heads * cfg.head_dim * e
    row_q = cfg.num_q_heads * cfg.head_dim * e
    build = (A + C) * 2 * row_kv + 2 * C * row_q
    attend = (A + P + C) * 2 * row_kv + 2 * q * row_kv + 2 * q * row_q
    append = 2 * 2 * cfg.tokens_per_frame * row_kv
    return build, attend, append


class L2Flush:
    """Evicts the working set from L2 between timed steps by READING a buffer twice the L2
    size: the lines it leaves behind are clean, so the next step pays no write-back of the
    flush itself (a write-based flush leaves ~126 MB of dirty lines that the timed kernel
    would have to write back)."""

    def __init__(self, dev):
        self.buf = torch.ones(2 * L2_BYTES // 4, dtype=torch.float32, device=dev)
        self.out = torch.empty((), dtype=torch.float32, device=dev)

    def __call__(self):
        torch.amax(self.buf, dim=0, out=self.out)


# ----------------------------------------------------------------------------- clocks
def clock_snapshot(device_index: int):
    """One nvidia-smi reading (sm MHz, max MHz, active reasons), or None."""
    q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    try:
        out = subprocess.run(["nvidia-smi", "-i", str(device_index), f"--query-gpu={q}", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True, timeout=10).stdout.strip().split(",")
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        return {"sm_mhz": float(out[0]), "sm_max_mhz": float(out[1]),
                "reasons": [n for n, v in zip(names, out[2:6]) if v.strip().lower().startswith("active")]}
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi sampling every 50 ms while the GPU runs the step loop.  The sampled window
    covers the timed steps and, when they take less than HOLD_S, untimed repetitions of the
    same step right after them (so short timed regions still get clock samples)."""
    HOLD_S = 0.3

    def __init__(self, device_index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(device_index), f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = []
        for line in open(self.f.name):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        loaded = [x for x in sm if x > 500] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ----------------------------------------------------------------------------- distributed
def dist_setup(n_gpus: int):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def stream_range(S: int, world: int, rank: int):
    from paper_2605_01858_b200.dist import stream_partition
    return stream_partition(S, world, rank)


# ----------------------------------------------------------------------------- our arm
def run_ours(args, cfg, world, rank, local):
    from paper_2605_01858_b200 import dscache as D
    dev = torch.device("cuda", local)
    kvsplit = args.mode == "kvsplit"
    context = args.mode == "context"
    if context:
        # P3: one stream, every rank holds its whole cache and attends over 1/G of its keys;
        # the (O_r, lse_r) partials are all-gathered (NCCL) and merged by the combine kernel
        cfg = cfg.replace(num_streams=1)
        lcfg = cfg
        S = 1
        dsc = D.DSCache.from_config(lcfg, device=local)
    elif kvsplit:
        # P2: one stream, rank r holds KV heads [r*Hkv/G, (r+1)*Hkv/G) and their q heads
        from paper_2605_01858_b200.dist import kv_head_partition
        kv_lo, kv_n, q_lo, q_n = kv_head_partition(cfg.num_q_heads, cfg.num_kv_heads, world, rank)
        cfg = cfg.replace(num_streams=1)
        lcfg = cfg.replace(num_q_heads=q_n, num_kv_heads=kv_n)
        S = 1
        dsc = D.DSCache.from_config(lcfg, device=local, kv_head_offset=kv_lo)
    else:
        lo, hi = stream_range(cfg.num_streams, world, rank)
        S = hi - lo
        lcfg = cfg.replace(num_streams=S)
        dsc = D.DSCache.from_config(lcfg, device=local)
    A, P, C, q = steady_counts(cfg)
    N, Hq, Hkv, d, tpf = cfg.num_layers, lcfg.num_q_heads, lcfg.num_kv_heads, cfg.head_dim, cfg.tokens_per_frame
    dt = cfg.torch_dtype
    g = torch.Generator(device=dev)
    g.manual_seed(1000 + rank)

    def rnd(*shape):
        return (torch.randn(shape, device=dev, generator=g) * cfg.scale).to(dt)

    # device-resident synthetic input pool (values cycle; positions / slots never repeat)
    POOL = 4
    frames = [(rnd(S, N, tpf, Hkv, d), rnd(S, N, tpf, Hkv, d)) for _ in range(POOL)]
    if args.layer_seq and S != 1:
        raise SystemExit("--layer-seq times one stream's layers in order (c3); use a single-stream config")
    n_boost = int(round(args.boost * tpf)) if args.boost > 0 else 0
    Cq = C - tpf + n_boost if n_boost else C          # instant rows built per step
    q_inst = [rnd(S, N, Cq, Hq, d) for _ in range(2)]
    boost_kv = [(rnd(S, N, n_boost, Hkv, d), rnd(S, N, n_boost, Hkv, d)) for _ in range(2)] if n_boost else None
    qry = [(rnd(S, N, q, Hq, d), rnd(S, N, q, Hkv, d), rnd(S, N, q, Hkv, d)) for _ in range(2)]
    o_inst = torch.empty(S, N, Cq, Hq, d, dtype=dt, device=dev)
    o = torch.empty(S, N, q, Hq, d, dtype=dt, device=dev)
    stream = torch.cuda.current_stream(dev)
    if A > 0:
        dsc.append_frame(rnd(S, N, A, Hkv, d), rnd(S, N, A, Hkv, d))
    fill = cfg.instant_frames + cfg.past_frames - 1
    for t in range(fill):
        dsc.append_frame(*frames[t % POOL])
    tcount = [fill]

    gathered = [None]
    hgather = None
    if kvsplit and world > 1:
        from paper_2605_01858_b200.dist import AsyncHeadGather
        hgather = AsyncHeadGather((S, N, q, Hq, d), dt, dev, nbuf=2)

    fused = args.api == "fused"
    approx = getattr(args, "approx", 0)
    if approx:
        if args.layer_seq or n_boost or context or kvsplit:
            raise SystemExit("--approx runs the stream-partition mode with split calls")
        ring = dsc.approx_ring()
        q_new = [rnd(S, N, tpf, Hq, d) for _ in range(2)]
    fb_full, fa_ = flops_per_unit(lcfg, n_boost)
    fb_new, _ = flops_per_unit(lcfg, n_boost, newest_only=True)
    build_flops = [0]          # per (stream, layer), summed over the counted steps

    def step(i):
        t = tcount[0]
        qq = qry[i & 1]
        o_ = hgather.slot(stream) if hgather is not None else o   # P2: rotating O slots (side-stream gather)
        if context:     # P3 (NEXT-4): key-range split of one stream's attend, partials merged
            from paper_2605_01858_b200.dist import context_parallel_attend
            dsc.append_frame(*frames[t % POOL])
            dsc.build_instant(q_inst[i & 1], o_inst)
            if world > 1:
                gathered[0] = context_parallel_attend(dsc, qq[0], qq[1], qq[2])
            else:
                dsc.attend(qq[0], qq[1], qq[2], o)
        elif args.layer_seq:   # layer r+1 consumes layer r: one fused step per layer, in order
            fk, fv = frames[t % POOL]
            for l in range(N):
                dsc.step(fk[:, l:l + 1], fv[:, l:l + 1], q_inst[i & 1][:, l:l + 1], qq[0][:, l:l + 1],
                         qq[1][:, l:l + 1], qq[2][:, l:l + 1], o_inst=o_inst[:, l:l + 1], o=o[:, l:l + 1],
                         layer_begin=l, layer_count=1)
        elif n_boost:     # NEXT-4 resolution boost: the newest frame re-encoded (n_boost tokens)
            dsc.append_frame(*frames[t % POOL])
            dsc.build_instant_boost(q_inst[i & 1], *boost_kv[i & 1], o_inst=o_inst)
            dsc.attend_boost(qq[0], qq[1], qq[2], *boost_kv[i & 1], o=o)
        elif approx:    # NEXT-3: refresh every `approx` steps, otherwise the newest frame's rows only
            dsc.append_frame(*frames[t % POOL])
            n = dsc.approx_rows(ring, approx)
            dsc.build_instant_approx(q_inst[i & 1] if n != tpf or C == tpf else q_new[i & 1], ring, approx)
            build_flops[0] += fb_full if n != tpf or C == tpf else fb_new
            dsc.attend(qq[0], qq[1], qq[2], o)
        elif fused:     # dscache_step: append + build_instant + attend, one attention launch
            dsc.step(*frames[t % POOL], q_inst[i & 1], qq[0], qq[1], qq[2], o_inst=o_inst, o=o_)
        else:
            dsc.append_frame(*frames[t % POOL])
            dsc.build_instant(q_inst[i & 1], o_inst)
            dsc.attend(qq[0], qq[1], qq[2], o_)
        if kvsplit and world > 1:           # the only exchange of P2: head-major all-gather of O,
            gathered[0] = hgather.launch(stream)   # on a side stream, overlapped with the next step
        tcount[0] += 1

    ring_bytes = 2 * S * N * Hkv * dsc.R * d * (2 if cfg.dtype == "bf16" else 4)
    flush = ring_bytes < 2 * L2_BYTES
    scratch = L2Flush(dev) if flush else None
    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    assert dsc.state(0)["past_tokens"] == P and dsc.state(0)["instant_tokens"] == C

    dsc.profile(True)
    dsc.profile_read(reset=True)
    build_flops[0] = 0
    barrier(world)
    torch.cuda.synchronize()
    snap_before = clock_snapshot(local) if rank == 0 else None
    clocks = ClockSampler(local) if rank == 0 else None
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if flush:
        total_ms = 0.0
        for i in range(args.steps):
            scratch()
            ev[i][0].record(stream)
            step(i)
            if hgather is not None:
                hgather.wait(stream)
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        total_ms = sum(a.elapsed_time(b) for a, b in ev)
    else:
        ev[0][0].record(stream)
        for i in range(args.steps):
            step(i)
        if hgather is not None:
            hgather.wait(stream)            # the last step's gather is part of the timed work
        ev[0][1].record(stream)
        torch.cuda.synchronize()
        total_ms = ev[0][0].elapsed_time(ev[0][1])
    timed_build_flops = build_flops[0]
    # the attention launches of exactly the timed steps (the clock hold loop below is not profiled)
    prof = dsc.profile_read(reset=True)
    dsc.profile(False)
    if clocks:
        # short timed regions: keep the same step loop running (untimed) so the sampler sees
        # the clocks of this workload for at least HOLD_S
        t_hold = time.perf_counter()
        i = args.steps
        while time.perf_counter() - t_hold < clocks.HOLD_S - total_ms / 1e3:
            for _ in range(4):
                step(i)
                i += 1
            torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    clk = clocks.stop() if clocks else None
    if clk is not None:
        clk["window"] = "timed steps + untimed repetitions of the same step up to %.1f s" % ClockSampler.HOLD_S
        clk["snapshot_before"], clk["snapshot_after"] = snap_before, clock_snapshot(local)
    t_max = max_over_ranks(total_ms, world)

    # e2e: the same step through the public API with pinned host buffers, H2D of every
    # input of the step and D2H of the query answer O inside the timed region
    graph = None
    if getattr(args, "graph", False) and world == 1 and not (context or kvsplit or args.layer_seq or n_boost or approx):
        graph = time_graph(args, dsc, step, scratch, dev)
    e2e = (run_e2e(args, cfg, lcfg, dsc, S, dev, stream, world, kvsplit) if not (n_boost or approx) else
           {"skipped": ("boost" if n_boost else "approx") + " mode times the device-resident path only"})
    impl = dsc.attn_impl()
    dsc.close()

    fb, fa = flops_per_unit(lcfg, n_boost)
    if approx:
        fb = timed_build_flops / args.steps     # refresh / newest-only mix of the timed steps
    units = S * N
    frames_total = cfg.num_streams * args.steps
    value = frames_total / (t_max / 1e3)
    attn_flops_step_local = units * (fb + fa)
    attn_ms = prof["ms_build"] + prof["ms_attend"]
    n_launch = prof["n_build"] + prof["n_attend"]
    pk = peaks()
    achieved = (attn_flops_step_local * args.steps) / (attn_ms / 1e3) / 1e12 if attn_ms > 0 else None
    step_tflops = attn_flops_step_local * args.steps / (total_ms / 1e3) / 1e12
    # DRAM bytes per attention launch from an ncu --set full capture of exactly this launch
    # shape (profiles/ncu_traffic.json, written by scripts/summarize_profile.py); null if
    # this (config, mode, api, boost, world, layers-seq) combination was never captured
    traffic, traffic_tag = None, None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            rec = json.load(open(tp)).get(traffic_key(args, world), {})
            traffic, traffic_tag = rec.get("dram_bytes_per_launch"), rec.get("tag")
        except Exception:
            traffic = None
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "frames/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(t_max / args.steps, 4), "higher_is_better": True,
        "scaling": "strong",   # the config's total work (all its streams) is fixed as N grows
        "vs_baseline": None, "dtype": "bf16" if cfg.dtype == "bf16" else "f32", "data": "synthetic",
        "config": dict(config_dict(cfg, args, world),
                       l2=("flushed between steps (read-only flush of 2x L2)" if flush else "inputs larger than L2 (ring %.2f GB)" % (ring_bytes / 1e9)),
                       input_pool=f"{POOL} distinct frames cycled (positions never repeat)"),
        "value_is": "aggregate frames/s over all streams and GPUs (one frame per stream per step); "
                    "frames_per_s_per_stream = value / streams",
        "frames_per_s_per_stream": round(value / cfg.num_streams, 3),
        "attention_tflops_per_gpu_step": round(step_tflops, 2),
        "attention_pct_peak_step": round(100 * step_tflops / pk["bf16_tflops"], 2),
        "roofline": {"bound": "tensor", "kernel": FA_KERNEL,
                     "achieved": round(achieved, 2) if achieved else None, "peak": pk["bf16_tflops"],
                     "peak_source": pk["source"] + " bf16 burst", "unit": "TFLOP/s",
                     "frac": round(achieved / pk["bf16_tflops"], 4) if achieved else None,
                     # context: the step loop runs ~0.1-0.3 s at 1.9-1.97 GHz (the clocks line), i.e. the
                     # burst conditions; the cuBLAS sustained figure was taken power-capped at ~1.3 GHz
                     "peak_sustained": pk.get("bf16_tflops_sustained"),
                     "frac_vs_sustained": (round(achieved / pk["bf16_tflops_sustained"], 4)
                                           if achieved and pk.get("bf16_tflops_sustained") else None),
                     "traffic": traffic, "traffic_source": (f"ncu --set full, profiles/{traffic_tag}_ncu_full.md"
                                                            if traffic else "not captured for this launch shape"),
                     "launches": n_launch,
                     "algorithmic_flops_per_launch": (attn_flops_step_local * args.steps) / max(n_launch, 1)},
        "gpu_launches": prof["kernel_launches"],
        "attn_impl": impl,
        "clocks": clk,
        "e2e": e2e,
    }
    if graph is not None:
        graph["value"] = round(cfg.num_streams / (graph["ms_per_step"] / 1e3), 2)
        line["graph"] = graph
    if getattr(args, "whole_stream", False) and world == 1 and not (context or kvsplit or args.layer_seq or n_boost
                                                                     or approx):
        line["whole_stream"] = time_whole_stream(cfg, dev)
    return line


def time_graph(args, dsc, step, flush, dev):
    """The same steady-state step sequence replayed from one CUDA graph (SURVEY §8(d) graph
    vs eager): K steps are captured once (the library's host bookkeeping runs at capture;
    the launches' ring offsets and ids are baked in, so a replay re-executes those K steps'
    work -- a timing device, not a stream continuation).  With an L2 flush between steps the
    flushes are captured too and a flush-only graph's time is subtracted."""
    K = args.steps
    s = torch.cuda.Stream(dev)
    s.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(s):
        for i in range(2):                  # warm on the capture stream (launch shapes cached)
            step(i)
    torch.cuda.synchronize()

    def capture(body):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s, capture_error_mode="relaxed"):
            for i in range(K):
                body(i)
        return g

    def timed(g):
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            a.record(s)
            g.replay()
            b.record(s)
        torch.cuda.synchronize()
        return a.elapsed_time(b)

    def body(i):
        if flush is not None:
            flush()
        step(i)
    try:
        ms = timed(capture(body))
        ms_flush = timed(capture(lambda i: flush())) if flush is not None else 0.0
    except Exception as e:          # capture not possible for this mode: say why, keep the line
        return {"skipped": f"graph capture failed: {type(e).__name__}: {str(e)[:120]}"}
    return {"ms_per_step": round((ms - ms_flush) / K, 4), "steps_captured": K,
            "flush_ms_subtracted_per_step": round(ms_flush / K, 4),
            "note": "the timed steps replayed from one CUDA graph (no host launch overhead); eager = ms_per_step"}


def time_whole_stream(cfg, dev):
    """Whole-stream average next to the steady state: a fresh handle fed every
    frame of the config's stream from frame 0 (warm-up steps with a partial window included),
    one fused step per frame, timed end to end on the device."""
    from paper_2605_01858_b200 import dscache as D
    S, N, A, tpf, Hkv, Hq, d = (cfg.num_streams, cfg.num_layers, cfg.sink_tokens, cfg.tokens_per_frame,
                                cfg.num_kv_heads, cfg.num_q_heads, cfg.head_dim)
    g = torch.Generator(device=dev)
    g.manual_seed(77)

    def rnd(*shape):
        return (torch.randn(shape, device=dev, generator=g) * cfg.scale).to(cfg.torch_dtype)
    h = D.DSCache.from_config(cfg, device=dev.index or 0)
    fk, fv = rnd(S, N, tpf, Hkv, d), rnd(S, N, tpf, Hkv, d)
    qi_full = rnd(S * N * cfg.C * Hq * d)
    q, ks, vs = rnd(S, N, cfg.query_tokens, Hq, d), rnd(S, N, cfg.query_tokens, Hkv, d), rnd(S, N, cfg.query_tokens, Hkv, d)
    o = torch.empty(S, N, cfg.query_tokens, Hq, d, dtype=cfg.torch_dtype, device=dev)
    oi_full = torch.empty(S * N * cfg.C * Hq * d, dtype=cfg.torch_dtype, device=dev)
    if A > 0:
        h.append_frame(rnd(S, N, A, Hkv, d), rnd(S, N, A, Hkv, d))
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for t in range(cfg.num_frames):
        n_inst = h.state(0)["next_instant_tokens"]
        qi = qi_full[:S * N * n_inst * Hq * d].view(S, N, n_inst, Hq, d)
        oi = oi_full[:S * N * n_inst * Hq * d].view(S, N, n_inst, Hq, d)
        h.step(fk, fv, qi, q, ks, vs, o_inst=oi, o=o)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    h.close()
    return {"frames": cfg.num_frames, "ms_total": round(ms, 3), "ms_per_step": round(ms / cfg.num_frames, 4),
            "value": round(S * cfg.num_frames / (ms / 1e3), 2), "unit": "frames/s",
            "note": "fresh handle, every frame of the stream from frame 0 (partial windows included), device time"}


def decode_bytes_per_unit(cfg, n_self, n_q, past_tokens=None):
    """Algorithmic HBM bytes of one (stream, layer) decode launch: every key of [sink | past |
    instant | self] read once per KV head (K and V), the n_q query rows read, O written."""
    A, P, C, _ = steady_counts(cfg)
    P = P if past_tokens is None else past_tokens
    e = 2 if cfg.dtype == "bf16" else 4
    keys = A + P + C + n_self
    return keys * 2 * cfg.num_kv_heads * cfg.head_dim * e + 2 * n_q * cfg.num_q_heads * cfg.head_dim * e


def run_decode(args, cfg, world, rank, local):
    """--mode decode: one autoregressive token per stream per
    step over C_{t+1} = [sink | past | instant] plus the transient self segment (the query
    chunk and the tokens generated so far, n_self = q + G), for every layer; memory-bound."""
    from paper_2605_01858_b200 import dscache as D
    dev = torch.device("cuda", local)
    lo, hi = stream_range(cfg.num_streams, world, rank)
    S = hi - lo
    lcfg = cfg.replace(num_streams=S)
    n_q = args.decode_nq
    n_self = cfg.query_tokens + args.decode_gen
    lcfg = lcfg.replace(query_tokens=max(cfg.query_tokens, n_self))
    dsc = D.DSCache.from_config(lcfg, device=local)
    A, P, C, _ = steady_counts(cfg)
    N, Hq, Hkv, d, tpf = cfg.num_layers, cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim, cfg.tokens_per_frame
    dt = cfg.torch_dtype
    g = torch.Generator(device=dev)
    g.manual_seed(2000 + rank)

    def rnd(*shape):
        return (torch.randn(shape, device=dev, generator=g) * cfg.scale).to(dt)
    if A > 0:
        dsc.append_frame(rnd(S, N, A, Hkv, d), rnd(S, N, A, Hkv, d))
    fk, fv = rnd(S, N, tpf, Hkv, d), rnd(S, N, tpf, Hkv, d)
    for _ in range(cfg.instant_frames + cfg.past_frames):
        dsc.append_frame(fk, fv)
    assert dsc.state(0)["past_tokens"] == P and dsc.state(0)["instant_tokens"] == C
    qs = [rnd(S, N, n_q, Hq, d) for _ in range(2)]
    ks, vs = rnd(S, N, n_self, Hkv, d), rnd(S, N, n_self, Hkv, d)
    o = torch.empty(S, N, n_q, Hq, d, dtype=dt, device=dev)
    stream = torch.cuda.current_stream(dev)
    stride = args.decode_stride

    def step(i):
        if stride > 1:
            dsc.decode(qs[i & 1], ks, vs, o=o, past_stride=stride)
        else:
            dsc.decode(qs[i & 1], ks, vs, o=o)

    ring_bytes = 2 * S * N * Hkv * dsc.R * d * (2 if cfg.dtype == "bf16" else 4)
    flush = ring_bytes < 2 * L2_BYTES
    scratch = L2Flush(dev) if flush else None
    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    dsc.profile(True)
    dsc.profile_read(reset=True)
    barrier(world)
    torch.cuda.synchronize()
    clocks = ClockSampler(local) if rank == 0 else None
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if flush:
        for i in range(args.steps):
            scratch()
            ev[i][0].record(stream)
            step(i)
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        total_ms = sum(a.elapsed_time(b) for a, b in ev)
    else:
        ev[0][0].record(stream)
        for i in range(args.steps):
            step(i)
        ev[0][1].record(stream)
        torch.cuda.synchronize()
        total_ms = ev[0][0].elapsed_time(ev[0][1])
    prof = dsc.profile_read(reset=True)
    dsc.profile(False)
    if clocks:
        t_hold = time.perf_counter()
        i = args.steps
        while time.perf_counter() - t_hold < clocks.HOLD_S - total_ms / 1e3:
            for _ in range(16):
                step(i)
                i += 1
            torch.cuda.synchronize()
    barrier(world)
    clk = clocks.stop() if clocks else None
    impl = dsc.attn_impl()
    kept_past = P if stride <= 1 else ((cfg.past_frames + stride - 1) // stride) * tpf
    dsc.close()
    t_max = max_over_ranks(total_ms, world)
    units = S * N
    bytes_step = units * decode_bytes_per_unit(cfg, n_self, n_q, kept_past)
    traffic, traffic_tag = None, None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            rec = json.load(open(tp)).get(traffic_key(args, world), {})
            traffic, traffic_tag = rec.get("dram_bytes_per_launch"), rec.get("tag")
        except Exception:
            traffic = None
    attn_ms = prof["ms_attend"] + prof["ms_build"]
    pk = peaks()
    achieved = bytes_step * args.steps / (attn_ms / 1e3) / 1e9 if attn_ms > 0 else None
    value = cfg.num_streams * args.steps / (t_max / 1e3)
    return {
        "metric": "decode tokens/s (one token per stream per step, all layers) and HBM GB/s", "value": round(value, 2),
        "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(t_max / args.steps, 4), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16" if cfg.dtype == "bf16" else "f32", "data": "synthetic",
        "config": dict(config_dict(cfg, args, world), decode_n_q=n_q, decode_n_self=n_self, past_stride=stride,
                       kept_past_tokens=kept_past,
                       l2=("flushed between steps (read-only flush of 2x L2)" if flush else "inputs larger than L2 (ring %.2f GB)" % (ring_bytes / 1e9))),
        "value_is": "aggregate decode tokens/s over all streams (each token passes every layer of the handle)",
        "roofline": {"bound": "hbm", "kernel": ("decode_kernel (mma.sync m16n8k16, GQA rows packed per kv head, TMA ring tiles)"
                                                if cfg.dtype == "bf16" and cfg.head_dim == 128 and n_q * (Hq // Hkv) <= 16
                                                else "attention kernel (n_q * Hq/Hkv > 16 or not bf16/d128)"),
                     "achieved": round(achieved, 1) if achieved else None, "peak": pk["hbm_gbs"],
                     "peak_source": pk["source"] + " HBM copy", "unit": "GB/s",
                     "frac": round(achieved / pk["hbm_gbs"], 4) if achieved else None, "traffic": traffic,
                     "traffic_source": (f"ncu --set full, profiles/{traffic_tag}_ncu_full.md" if traffic
                                        else "not captured for this launch shape"),
                     "algorithmic_bytes_per_step": bytes_step, "launches": prof["n_build"] + prof["n_attend"]},
        "gpu_launches": prof["kernel_launches"], "attn_impl": impl, "clocks": clk,
        "e2e": {"skipped": "decode mode times the device-resident path only"},
    }


def run_e2e(args, cfg, lcfg, dsc, S, dev, stream, world, kvsplit):
    N, Hq, Hkv, d, tpf = cfg.num_layers, lcfg.num_q_heads, lcfg.num_kv_heads, cfg.head_dim, cfg.tokens_per_frame
    A, P, C, q = steady_counts(cfg)
    dt = cfg.torch_dtype
    steps = max(3, min(args.steps, 10))

    def host(*shape):
        return (torch.randn(shape) * cfg.scale).to(dt).pin_memory()
    hk, hv = host(S, N, tpf, Hkv, d), host(S, N, tpf, Hkv, d)
    hqi = host(S, N, C, Hq, d)
    hq, hks, hvs = host(S, N, q, Hq, d), host(S, N, q, Hkv, d), host(S, N, q, Hkv, d)
    ho = torch.empty(S, N, q, Hq * (world if kvsplit else 1), d, dtype=dt).pin_memory()
    h2d = sum(t.numel() * t.element_size() for t in (hk, hv, hqi, hq, hks, hvs))
    d2h = ho.numel() * ho.element_size()
    fused = args.api == "fused"

    def one():
        k = hk.to(dev, non_blocking=True); v = hv.to(dev, non_blocking=True)
        qi = hqi.to(dev, non_blocking=True)
        qq, ks, vs = (hq.to(dev, non_blocking=True), hks.to(dev, non_blocking=True),
                      hvs.to(dev, non_blocking=True))
        if fused:
            oi, o = dsc.step(k, v, qi, qq, ks, vs)
        else:
            dsc.append_frame(k, v)
            oi = dsc.build_instant(qi)
            o = dsc.attend(qq, ks, vs)
        if kvsplit and world > 1:
            from paper_2605_01858_b200.dist import gather_heads
            o = gather_heads(o)
        ho.copy_(o, non_blocking=True)
        del oi
    pipelined = fused and not (kvsplit and world > 1)
    if pipelined:
        # the public host-fed path: step i+1's H2D overlaps step i's kernels and step i-1's D2H
        from paper_2605_01858_b200.pipeline import HostStepPipeline
        pipe = HostStepPipeline(dsc, q)

        def one():
            pipe.submit(hk, hv, hqi, hq, hks, hvs, ho)
    one()
    torch.cuda.synchronize()
    barrier(world)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if pipelined:
        pipe.synchronize()
        a.record(pipe.h2d)          # before the first H2D of the timed steps
        for _ in range(steps):
            one()
        pipe.d2h.wait_stream(pipe.compute)
        b.record(pipe.d2h)          # after the last D2H
    else:
        a.record(stream)
        for _ in range(steps):
            one()
        b.record(stream)
    torch.cuda.synchronize()
    ms = max_over_ranks(a.elapsed_time(b), world)
    return {"value": round(cfg.num_streams * steps / (ms / 1e3), 2), "unit": "frames/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": steps,
            "note": "pinned host inputs (frame K/V, Q_inst, Q, K_self, V_self) copied H2D and the query "
                    "answer O copied D2H every step" + (
                        ", through pipeline.HostStepPipeline (DSCache.step on a compute stream; the next step's "
                        "H2D and the previous step's D2H overlap it, 2 buffer slots)" if pipelined else
                        ", through DSCache.step (or append_frame/build_instant/attend with --api split), one stream")}


# ----------------------------------------------------------------------------- oracle (cpu baseline / reference arm)
def oracle_sample(cfg, budget_s: float):
    """Time the fp64 oracle on (stream, layer) units of the steady-state workload."""
    from oracle.workload import StreamInputs, oracle_step
    try:
        from threadpoolctl import threadpool_info
        threads = max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        threads = os.cpu_count()
    t_steady = cfg.instant_frames + cfg.past_frames
    units, t0 = 0, time.perf_counter()
    times = []
    while True:
        s, l = units % cfg.num_streams, (units // cfg.num_streams) % cfg.num_layers
        inp = StreamInputs(cfg, s, l)
        a = time.perf_counter()
        oracle_step(cfg, s, l, t_steady + units % 4, inputs=inp)
        times.append(time.perf_counter() - a)
        units += 1
        if time.perf_counter() - t0 > budget_s or units >= 64:
            break
    per_unit = float(np.mean(times))
    step_s = per_unit * cfg.num_streams * cfg.num_layers
    return {"value": round(cfg.num_streams / step_s, 6), "unit": "frames/s", "cores": threads,
            "kind": "oracle", "units": units,
            "sample": f"{units} steady-state (stream, layer) units of {cfg.name} (build_instant + attend, fp64 "
                      f"numpy), {per_unit:.3f} s/unit, extrapolated to {cfg.num_streams * cfg.num_layers} "
                      f"units per step",
            "cpu": _cpu_model()}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def run_reference(args, cfg):
    per_step = []
    cb = None
    for i in range(args.warmup + args.steps):
        r = oracle_sample(cfg, budget_s=max(2.0, 60.0 / (args.warmup + args.steps)))
        if i >= args.warmup:
            per_step.append(r)
        cb = r
    value = float(np.mean([r["value"] for r in per_step]))
    fb, fa = flops_per_unit(cfg)
    return {"metric": METRIC, "value": round(value, 6), "unit": "frames/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(1e3 * cfg.num_streams / value, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": config_dict(cfg, args, 1),
            "reference_note": "fp64 CPU oracle (oracle/), the tier's reference arm: each timed step runs a "
                              "bounded sample of (stream, layer) units and is extrapolated to the full step",
            "extrapolated": True, "units_run": [r["units"] for r in per_step],
            "cpu_baseline": {"value": round(value, 6), "unit": "frames/s", "cores": cb["cores"], "kind": "oracle",
                             "sample": cb["sample"], "cpu": cb["cpu"]},
            "e2e": {"value": round(value, 6), "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def _free_port() -> int:
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    return port


def dry_run(args, cfg):
    """Every rank computes what it would hold (P1 streams / P2 KV heads / P3 key split) and
    rank 0 prints the gathered plan: the N-rank launch path without GPU work."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    from paper_2605_01858_b200.dist import kv_head_partition, stream_partition
    if args.mode in ("kvsplit", "context"):
        cfg = cfg.replace(num_streams=1)   # the single-stream modes (as run_ours)
    if args.mode == "kvsplit":
        part = dict(zip(("kv_lo", "kv_count", "q_lo", "q_count"),
                        kv_head_partition(cfg.num_q_heads, cfg.num_kv_heads, world, rank)))
    elif args.mode == "context":
        part = {"key_part": rank, "key_parts": world}
    else:
        lo, hi = stream_partition(cfg.num_streams, world, rank)
        part = {"streams": [lo, hi]}
    part["rank"] = rank
    plan = [part]
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        plan = [None] * world
        dist.all_gather_object(plan, part)
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "mode": args.mode, "config": config_dict(cfg, args, world),
                          "partition": plan}), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c5")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="streams", choices=["streams", "kvsplit", "context", "decode"],
                    help="streams: P1 stream partition (default); kvsplit: P2 KV-head split of one stream; "
                         "context: P3 key-range split of one stream's attend (NEXT-4)")
    ap.add_argument("--layer-seq", action="store_true",
                    help="one fused step per layer, layers in order (a real model's dependency; c3)")
    ap.add_argument("--dry-run", action="store_true",
                    help="launch the N ranks and print each rank's partition, no GPU work (gloo without CUDA)")
    ap.add_argument("--api", default="fused", choices=["fused", "split"],
                    help="fused: DSCache.step (one attention launch per step); split: three calls")
    ap.add_argument("--boost", type=float, default=0.0,
                    help="> 0: resolution-boosted newest frame with boost*tpf tokens (SURVEY NEXT-4), split calls")
    ap.add_argument("--approx", type=int, default=0,
                    help="> 0: approximate instant cache refreshed every APPROX steps (SURVEY NEXT-3), split calls")
    ap.add_argument("--instant-frames", type=int, default=None, help="override l_I of the config (frames)")
    ap.add_argument("--decode-gen", type=int, default=16, help="decode mode: tokens generated so far (self = q + G)")
    ap.add_argument("--decode-nq", type=int, default=1, help="decode mode: query rows per launch")
    ap.add_argument("--decode-stride", type=int, default=1,
                    help="decode mode: keep every STRIDE-th past frame (zeta_decode, PAPER.md:695)")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the graph-replay and whole-stream timings added to the line at N = 1")
    ap.add_argument("--graph", action="store_true", help="(default at N = 1) time the timed steps replayed from one CUDA graph")
    ap.add_argument("--whole-stream", action="store_true",
                    help="(default at N = 1) time a fresh handle over every frame of the config's stream")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if not args.no_extras and int(os.environ.get("WORLD_SIZE", "1")) == 1 and args.gpus == 1:
        args.graph = args.whole_stream = True
    cfg = synth.CONFIGS[args.config]
    if args.instant_frames is not None:
        cfg = cfg.replace(instant_frames=args.instant_frames)
    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # not launched by torchrun: launch N ranks of this same command (one process per GPU)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)
    if world_env != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world_env}: launch N ranks with torchrun "
                                   f"or omit WORLD_SIZE"}), flush=True)
        return 2
    if args.dry_run:
        return dry_run(args, cfg)
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        if rank != 0:
            return 0
        print(json.dumps(run_reference(args, cfg)), flush=True)
        return 0
    world, rank, local = dist_setup(args.gpus)
    line = run_decode(args, cfg, world, rank, local) if args.mode == "decode" else run_ours(args, cfg, world, rank, local)
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline and args.mode != "decode":
            line["cpu_baseline"] = oracle_sample(cfg, args.cpu_budget)
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
