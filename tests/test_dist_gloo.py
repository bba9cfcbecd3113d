"""Multi-process (world_size 2, gloo on CPU) checks of the multi-GPU host logic.

The GPU box has one GPU, so the N>1 paths are covered here: each rank stands in
for one GPU and computes its shard with the fp64 oracle (the CUDA backend's
stand-in on CPU); the tests check the partitions (P1 streams, P2 KV-head groups,
P3 context split), the head-major all-gather and the partial gather + merge of
paper_2605_01858_b200.dist against the unsharded oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import dscache_synth as synth
from paper_2605_01858_b200.dist import (gather_heads, gather_partials, kv_head_partition, merge_partials,
                                        stream_partition)


def test_stream_partition_covers_every_stream_once():
    for S in (1, 5, 8, 64):
        for world in (1, 2, 3, 4, 8):
            got = []
            for r in range(world):
                lo, hi = stream_partition(S, world, r)
                assert 0 <= lo <= hi <= S
                got += list(range(lo, hi))
            assert got == list(range(S))
            sizes = [stream_partition(S, world, r)[1] - stream_partition(S, world, r)[0] for r in range(world)]
            assert max(sizes) - min(sizes) <= 1


def test_kv_head_partition_keeps_gqa_groups_together():
    for world in (1, 2, 4):
        qs, ks = [], []
        for r in range(world):
            kv_lo, kv_n, q_lo, q_n = kv_head_partition(28, 4, world, r)
            ks += list(range(kv_lo, kv_lo + kv_n))
            qs += list(range(q_lo, q_lo + q_n))
            for h in range(q_lo, q_lo + q_n):          # every local q head reads a local kv head
                assert kv_lo <= h // 7 < kv_lo + kv_n
        assert ks == list(range(4)) and qs == list(range(28))
    with pytest.raises(ValueError):
        kv_head_partition(28, 4, 8, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_attend(cfg, s, t, heads=None):
    """Oracle O [q, Hq(_local), d] of stream s at step t, optionally on a KV-head shard."""
    from oracle.workload import StreamInputs, step_schedule
    from oracle import dscache_oracle as O
    inp = StreamInputs(cfg, s, 0)
    sch = step_schedule(cfg, t)
    sk, sv = inp.sink()
    q, ks, vs = inp.query(t)
    frame = inp.frame_kv
    if heads is not None:
        kv_lo, kv_n, q_lo, q_n = heads
        sk, sv = sk[:, kv_lo:kv_lo + kv_n], sv[:, kv_lo:kv_lo + kv_n]
        q = q[:, q_lo:q_lo + q_n]
        ks, vs = ks[:, kv_lo:kv_lo + kv_n], vs[:, kv_lo:kv_lo + kv_n]
        frame = lambda f: tuple(x[:, kv_lo:kv_lo + kv_n] for x in inp.frame_kv(f))   # noqa: E731
    return O.attend_output(sch, (sk, sv), frame, q, ks, vs, cfg.rope_theta)


def _small_cfg():
    # c2's head layout (28 q / 4 kv heads, GQA 7) on a short, small-frame stream
    return synth.CONFIGS["c2"].replace(num_streams=4, tokens_per_frame=8, past_frames=3, instant_frames=2,
                                       query_tokens=5, num_frames=8, head_dim=32)


def _worker_kv_split(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = _small_cfg()
    heads = kv_head_partition(cfg.num_q_heads, cfg.num_kv_heads, world, rank)
    t = 6
    local = torch.from_numpy(_oracle_attend(cfg, 0, t, heads))       # [q, Hq/G, d]
    full = gather_heads(local[None, None])                          # [1, 1, q, Hq, d]
    if rank == 0:
        out_q.put(full[0, 0].numpy())
    dist.barrier()
    dist.destroy_process_group()


def _worker_async_gather(rank, world, port, out_q):
    """AsyncHeadGather over 3 steps with 2 rotating slots: each step's gathered output is the
    unsharded oracle of that step (the slot reuse never leaks the previous step's heads)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_01858_b200.dist import AsyncHeadGather
    cfg = _small_cfg()
    heads = kv_head_partition(cfg.num_q_heads, cfg.num_kv_heads, world, rank)
    g = AsyncHeadGather((1, 1, cfg.query_tokens, heads[3], cfg.head_dim), torch.float64, "cpu", nbuf=2)
    outs = []
    for t in (5, 6, 7):
        g.slot().copy_(torch.from_numpy(_oracle_attend(cfg, 0, t, heads))[None, None])
        outs.append(g.launch())
    g.wait()
    if rank == 0:
        out_q.put([o[0, 0].numpy() for o in outs])
    dist.barrier()
    dist.destroy_process_group()


def _worker_streams(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = _small_cfg()
    lo, hi = stream_partition(cfg.num_streams, world, rank)
    t = 7
    digests = torch.zeros(cfg.num_streams, dtype=torch.float64)
    for s in range(lo, hi):                      # this rank's streams only; no data-path collective
        digests[s] = float(np.abs(_oracle_attend(cfg, s, t)).sum())
    dist.all_reduce(digests)                     # end-of-run digest gather (not on the hot path)
    if rank == 0:
        out_q.put(digests.numpy())
    dist.barrier()
    dist.destroy_process_group()


def _run(worker, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


def test_kv_head_split_allgather_matches_unsharded_oracle():
    full = _run(_worker_kv_split)
    ref = _oracle_attend(_small_cfg(), 0, 6)
    assert full.shape == ref.shape
    assert np.abs(full - ref).max() < 1e-12


def test_async_head_gather_rotating_slots():
    outs = _run(_worker_async_gather)
    for t, full in zip((5, 6, 7), outs):
        ref = _oracle_attend(_small_cfg(), 0, t)
        assert np.abs(full - ref).max() < 1e-12


def test_stream_partition_two_ranks_matches_single_process():
    digests = _run(_worker_streams)
    cfg = _small_cfg()
    ref = np.array([np.abs(_oracle_attend(cfg, s, 7)).sum() for s in range(cfg.num_streams)])
    assert np.allclose(digests, ref, rtol=0, atol=1e-12)


def _partial_attend(cfg, s, t, part, n_parts):
    """fp64 partial of the attend over the n_parts-way contiguous split of its context
    keys (plain softmax over the subset, built from the oracle's key assembly and RoPE):
    (O_part [q, Hq, d], lse_part [q, Hq] in log2 units)."""
    from oracle.workload import StreamInputs, step_schedule
    from oracle import dscache_oracle as O
    inp = StreamInputs(cfg, s, 0)
    sch = step_schedule(cfg, t)
    sk, sv = inp.sink()
    q, ks, vs = inp.query(t)
    frames = list(sch.past_frames) + list(sch.instant_frames)
    hkv, d = sk.shape[1], sk.shape[2]
    K = O._cat([sk] + [inp.frame_kv(f)[0] for f in frames] + [ks], hkv, d)
    V = O._cat([sv] + [inp.frame_kv(f)[1] for f in frames] + [vs], hkv, d)
    nk, nq = K.shape[0], q.shape[0]
    pos_k = np.arange(nk)
    pos_q = (nk - nq) + np.arange(nq)
    qr = O.rope(np.asarray(q, np.float64), pos_q, cfg.rope_theta)
    kr = O.rope(K, pos_k, cfg.rope_theta)
    grp = q.shape[1] // hkv
    lo, hi = part * nk // n_parts, (part + 1) * nk // n_parts
    o = np.zeros(q.shape, np.float64)
    lse = np.full(q.shape[:2], -np.inf)
    for h in range(q.shape[1]):
        g = h // grp
        sc = qr[:, h, :] @ kr[lo:hi, g, :].T / np.sqrt(d)                  # [nq, hi-lo]
        sc = np.where(pos_k[None, lo:hi] <= pos_q[:, None], sc, -np.inf)
        m = sc.max(axis=1, keepdims=True)
        ok = np.isfinite(m[:, 0])
        pr = np.where(ok[:, None], np.exp(sc - np.where(ok[:, None], m, 0.0)), 0.0)
        l = pr.sum(axis=1)
        o[ok, h, :] = (pr @ V[lo:hi, g, :])[ok] / l[ok, None]
        lse[ok, h] = (m[ok, 0] + np.log(l[ok])) / np.log(2.0)
    return o, lse


def _worker_context(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = _small_cfg()
    t = 6
    o, lse = _partial_attend(cfg, 1, t, rank, world)          # this rank's key range only
    o_all, l_all = gather_partials(torch.from_numpy(o), torch.from_numpy(lse))
    merged = merge_partials(o_all, l_all)
    if rank == 0:
        out_q.put(merged.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_context_split_partials_merge_to_unsharded_oracle():
    """P3: each rank attends over its contiguous range of the context keys;
    the all-gathered (O_r, lse_r) merge to the full attention (PAPER.md:637 softmax is
    invariant to how its key set is partitioned)."""
    merged = _run(_worker_context)
    ref = _oracle_attend(_small_cfg(), 1, 6)
    assert merged.shape == ref.shape
    assert np.abs(merged - ref).max() < 1e-12


@pytest.mark.parametrize("n_parts", [1, 3, 5])
def test_partial_merge_single_process(n_parts):
    cfg = _small_cfg()
    parts = [_partial_attend(cfg, 2, 7, r, n_parts) for r in range(n_parts)]
    merged = merge_partials(torch.from_numpy(np.stack([p[0] for p in parts])),
                            torch.from_numpy(np.stack([p[1] for p in parts])))
    assert np.abs(merged.numpy() - _oracle_attend(cfg, 2, 7)).max() < 1e-12


def _worker_peer_outputs(rank, world, port, out_q):
    """PeerOutputs handle exchange (P2 fused all-gather, two buffers per rank) with a stand-in
    IPC layer: rank r's buffer b has handle b"r<r>b<b>" with offset 16*r + b; opening it
    yields base 10**6*(r+1) + 1000*b."""
    from paper_2605_01858_b200.dist import PeerOutputs
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    opened, closed, made = [], [], []

    def handle(t):
        b = len(made)
        made.append(t)
        return b"r%db%d" % (rank, b), 16 * rank + b

    def open_(dev, hd):
        opened.append(hd)
        r, b = (int(x) for x in hd[1:].split(b"b"))
        return 10 ** 6 * (r + 1) + 1000 * b

    peers = PeerOutputs((2, 3), torch.float32, "cpu", ipc=(handle, open_, lambda dev, p: closed.append(p)))
    ok = len(peers.locals) == 2 and peers.local is peers.locals[0]
    for b in range(2):
        want = [peers.locals[b].data_ptr() if r == rank else 10 ** 6 * (r + 1) + 1000 * b + 16 * r + b
                for r in range(world)]
        ok = ok and peers.ptrs[b] == want
    ok = ok and sorted(opened) == sorted(b"r%db%d" % (r, b) for r in range(world) if r != rank for b in range(2))
    peers.close()
    ok = ok and sorted(closed) == sorted(10 ** 6 * (r + 1) + 1000 * b for r in range(world) if r != rank
                                         for b in range(2))
    out_q.put((rank, ok))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_peer_outputs_exchange_rank_order(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_peer_outputs, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert all(ok for _, ok in res), res
