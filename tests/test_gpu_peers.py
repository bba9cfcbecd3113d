"""GPU checks of the fused all-gather epilogue of the KV-head split (P2, SURVEY §8(e) and
NEXT-4 item C3): dscache_attend_peers stores every output row from the attention kernel
into each rank's gathered-O buffer.

The GPU box has one GPU, so the "ranks" here share cuda:0: in one process two handles
(KV-head halves) write into two local buffers, and across two processes the buffers are
mapped with CUDA IPC (dscache_ipc_handle / dscache_ipc_open) exactly as on an NVSwitch
node.  No kernel waits on another: each rank's kernel only stores, and the readers wait on
a host barrier after their stream drained.  Results are compared with the unsharded fp64
oracle (bf16 bar of BASELINE.json north_star)."""
import os
import socket

import numpy as np
import pytest
import torch

import dscache_synth as synth
from oracle import dscache_oracle as O
from oracle.workload import StreamInputs, step_schedule
from tests.gpu_harness import assert_close
from paper_2605_01858_b200 import dscache as D
from paper_2605_01858_b200.dist import kv_head_partition

pytestmark = pytest.mark.gpu


def _shard_stream(cfg, heads, t_last, dev, rnd_seed=7):
    """Handle holding KV heads [kv_lo, kv_lo+kv_n) of every (stream, layer), fed frames 0..t_last
    (stream 0 / layer 0 from the seeded generator, the rest random), and the step-t_last query
    tensors of the shard.  Returns (handle, q, k_self, v_self)."""
    kv_lo, kv_n, q_lo, q_n = heads
    lcfg = cfg.replace(num_q_heads=q_n, num_kv_heads=kv_n)
    h = D.DSCache.from_config(lcfg, kv_head_offset=kv_lo)
    S, N = cfg.num_streams, cfg.num_layers
    g = torch.Generator(device=dev)
    g.manual_seed(rnd_seed)

    def batch(x00, n, nh, lo):
        t = (torch.randn((S, N, n, nh, cfg.head_dim), device=dev, generator=g) * cfg.scale).to(cfg.torch_dtype)
        t[0, 0] = x00[:, lo:lo + nh].to(dev)
        return t.contiguous()

    A, tpf = cfg.sink_tokens, cfg.tokens_per_frame
    sk, sv = synth.sink_kv(cfg, 0, 0)
    h.append_frame(batch(sk, A, kv_n, kv_lo), batch(sv, A, kv_n, kv_lo))
    for t in range(t_last + 1):
        fk, fv = synth.frame_kv(cfg, 0, 0, t)
        h.append_frame(batch(fk, tpf, kv_n, kv_lo), batch(fv, tpf, kv_n, kv_lo))
    q, ks, vs = synth.query_qkv(cfg, 0, 0, t_last)
    return (h, batch(q, cfg.query_tokens, q_n, q_lo), batch(ks, cfg.query_tokens, kv_n, kv_lo),
            batch(vs, cfg.query_tokens, kv_n, kv_lo))


def _oracle_full(cfg, t):
    inp = StreamInputs(cfg, 0, 0)
    q, ks, vs = inp.query(t)
    return O.attend_output(step_schedule(cfg, t), inp.sink(), inp.frame_kv, q, ks, vs, cfg.rope_theta)


@pytest.mark.parametrize("name,world,t", [("c2", 2, 40), ("c2", 4, 3), ("c5", 2, 9), ("c5", 4, 40)])
def test_attend_peers_all_ranks_in_one_process(lib, name, world, t):
    # c2: few work items -> split-KV + combine kernel epilogue; c5: 64 streams x 4 layers ->
    # the tcgen05 kernel's own epilogue writes the peers
    cfg = synth.CONFIGS[name]
    dev = torch.device("cuda", 0)
    Hq = cfg.num_q_heads
    shape = (cfg.num_streams, cfg.num_layers, cfg.query_tokens, Hq, cfg.head_dim)
    bufs = [torch.full(shape, float("nan"), dtype=cfg.torch_dtype, device=dev) for _ in range(world)]
    handles = []
    for r in range(world):
        heads = kv_head_partition(Hq, cfg.num_kv_heads, world, r)
        h, q, ks, vs = _shard_stream(cfg, heads, t, dev, rnd_seed=7 + r)
        h.attend_peers(q, ks, vs, bufs, Hq, heads[2])
        handles.append(h)
        # the plain attend of the same shard: the peer rows must be the same bits
        o_local = h.attend(q, ks, vs)
        torch.cuda.synchronize()
        for b in bufs:
            assert torch.equal(b[:, :, :, heads[2]:heads[2] + heads[3]], o_local)
    torch.cuda.synchronize()
    ref = _oracle_full(cfg, t)
    for b in bufs:
        assert not torch.isnan(b.float()).any()
        assert torch.equal(b, bufs[0])
        assert_close(b[0, 0].float().cpu(), ref, cfg.dtype, f"{name} peers world={world}")
    for h in handles:
        h.close()


def test_attend_peers_argument_errors(lib):
    import ctypes
    cfg = synth.CONFIGS["c2"]
    dev = torch.device("cuda", 0)
    h, q, ks, vs = _shard_stream(cfg, kv_head_partition(cfg.num_q_heads, cfg.num_kv_heads, 2, 0), 2, dev)
    buf = torch.empty((1, 1, cfg.query_tokens, cfg.num_q_heads, cfg.head_dim), dtype=cfg.torch_dtype, device=dev)
    with pytest.raises(D.DSCacheError):
        h.attend_peers(q, ks, vs, [buf] * 9, cfg.num_q_heads, 0)                 # > 8 peers
    with pytest.raises(D.DSCacheError):
        h.attend_peers(q, ks, vs, [buf], cfg.num_q_heads, cfg.num_q_heads - 1)  # head range outside hq_total
    arr = (ctypes.c_void_p * 1)(None)
    assert D._lib.dscache_attend_peers(h._h, 0, 1, ctypes.c_void_p(q.data_ptr()), ctypes.c_void_p(ks.data_ptr()),
                                       ctypes.c_void_p(vs.data_ptr()), cfg.query_tokens, arr, 1, cfg.num_q_heads, 0,
                                       None) == D.E_ARG                          # null peer pointer
    torch.cuda.synchronize()
    h.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _ipc_worker(rank, world, port, t, out_q):
    import torch.distributed as dist
    from paper_2605_01858_b200.dist import PeerOutputs, kv_split_attend_fused
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = synth.CONFIGS["c2"]
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        heads = kv_head_partition(cfg.num_q_heads, cfg.num_kv_heads, world, rank)
        h, q, ks, vs = _shard_stream(cfg, heads, t, dev, rnd_seed=11 + rank)
        shape = (1, 1, cfg.query_tokens, cfg.num_q_heads, cfg.head_dim)
        peers = PeerOutputs(shape, cfg.torch_dtype, dev)
        peers.local.fill_(float("nan"))
        torch.cuda.synchronize()
        dist.barrier()
        full = kv_split_attend_fused(h, q, ks, vs, peers, cfg.num_q_heads, heads[2])
        ref = _oracle_full(cfg, t)
        got = full[0, 0].float().cpu()
        ok = not torch.isnan(got).any().item()
        ma, rl = assert_close(got, ref, cfg.dtype, f"ipc rank {rank}") if ok else (float("nan"), float("nan"))
        dist.barrier()
        peers.close()
        h.close()
        out_q.put((rank, ok, ma, rl))
    except Exception as e:   # report instead of hanging the parent
        out_q.put((rank, False, repr(e), None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_attend_peers_across_processes_cuda_ipc(lib, world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, 40, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    for (rank, ok, ma, rl) in res:
        assert ok, f"rank {rank}: {ma}"
    assert all(p.exitcode == 0 for p in procs)


def _async_gather_worker(port, out_q):
    """One NCCL rank on cuda:0 (world 1): AsyncHeadGather's side-stream gather after attends
    on a compute stream, 3 steps over 2 rotating O slots."""
    import torch.distributed as dist
    from paper_2605_01858_b200.dist import AsyncHeadGather
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    cfg = synth.CONFIGS["c2"]
    heads = kv_head_partition(cfg.num_q_heads, cfg.num_kv_heads, 1, 0)
    h, q, ks, vs = _shard_stream(cfg, heads, 20, dev)
    comp = torch.cuda.Stream(dev)
    g = AsyncHeadGather(tuple(q.shape), q.dtype, dev, nbuf=2)
    outs = []
    with torch.cuda.stream(comp):
        for _ in range(3):
            o = g.slot(comp)
            h.attend(q, ks, vs, o, stream=comp)
            outs.append(g.launch(comp))
        g.wait(comp)
    comp.synchronize()
    ref = h.attend(q, ks, vs)
    torch.cuda.synchronize()
    out_q.put([float((x - ref).abs().max()) for x in outs])
    dist.destroy_process_group()
    h.close()


def test_async_head_gather_side_stream_nccl(lib):
    import multiprocessing as mp
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_async_gather_worker, args=(port, q))
    p.start()
    diffs = q.get(timeout=300)
    p.join(timeout=60)
    assert p.exitcode == 0
    assert all(d == 0.0 for d in diffs), diffs   # the gather of one rank is its own output, bit for bit
