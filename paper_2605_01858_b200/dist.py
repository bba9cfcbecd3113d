"""Multi-GPU plumbing of the hot path (one process per GPU, torch.distributed).

Two partitions, both from the north_star:

* P1 -- independent streams: rank r holds streams [r*S/G, (r+1)*S/G) in its own
  DSCache handle.  Streams share nothing, so the data path has no collective.
* P2 -- KV-head groups of one stream: rank r holds KV heads
  [r*Hkv/G, (r+1)*Hkv/G) and their Hq/Hkv query heads each.  Attention is
  independent per KV head; the only exchange is an all-gather of the attend
  output O, gathered head-major so no permute is needed on the wire.
* P3 -- context parallelism of one stream: every rank holds the
  stream's cache and computes the attend over 1/G of its keys (dscache_attend_partial);
  the partials (O_r, lse_r) are all-gathered and merged (dscache_combine_partials).
  Softmax attention is invariant to how its key set is split, so the merge is exact up
  to rounding; G = 8 works for Hkv = 4, where P2 cannot.

P2 has two gather paths: the NCCL all-gather of O (gather_heads; AsyncHeadGather runs it on
a side stream overlapped with the next step's kernels) and the
fused all-gather epilogue (PeerOutputs + kv_split_attend_fused): every rank's
gathered-O buffer is mapped into every other rank through CUDA IPC, and the attention
kernel's epilogue stores each output row straight into all of them over NVLink, so no
collective runs on the data path -- only a barrier before the buffers are read.

The collective backend is whatever the process group was created with: NCCL
over NVLink on the GPU box, gloo on CPU for the multi-process tests.
"""
from __future__ import annotations

from typing import Tuple

import torch


def stream_partition(num_streams: int, world: int, rank: int) -> Tuple[int, int]:
    """[lo, hi) streams of `rank` -- contiguous, sizes differ by at most one."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    lo = rank * num_streams // world
    hi = (rank + 1) * num_streams // world
    return lo, hi


def kv_head_partition(num_q_heads: int, num_kv_heads: int, world: int, rank: int):
    """(kv_lo, kv_count, q_lo, q_count) of `rank`.  Needs Hkv % world == 0 (the
    GQA group of a KV head never straddles ranks)."""
    if num_kv_heads % world:
        raise ValueError(f"Hkv={num_kv_heads} is not divisible by world={world}")
    grp = num_q_heads // num_kv_heads
    kv_count = num_kv_heads // world
    kv_lo = rank * kv_count
    return kv_lo, kv_count, kv_lo * grp, kv_count * grp


def head_major(o: torch.Tensor) -> torch.Tensor:
    """[S][N][n_q][Hq_local][d] -> contiguous [Hq_local][S][N][n_q][d] (one local copy
    on the sender so the gathered buffer is contiguous per rank's head block)."""
    return o.permute(3, 0, 1, 2, 4).contiguous()


def gather_heads(o_local: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather the head-sharded attend outputs of every rank (P2).

    o_local: [S][N][n_q][Hq_local][d] on this rank.  Returns [S][N][n_q][Hq][d]
    with rank r's heads at [r*Hq_local, (r+1)*Hq_local), i.e. global head order."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    hm = head_major(o_local)                                   # [Hl][S][N][q][d]
    out = torch.empty((world,) + tuple(hm.shape), dtype=hm.dtype, device=hm.device)
    if hasattr(dist, "all_gather_into_tensor") and dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, hm, group=group)
    else:
        dist.all_gather(list(out.unbind(0)), hm, group=group)
    full = out.reshape((world * hm.shape[0],) + tuple(hm.shape[1:]))   # [Hq][S][N][q][d]
    return full.permute(1, 2, 3, 0, 4)


class AsyncHeadGather:
    """P2's all-gather of O on a side stream, overlapped with the next step's kernels.

    `nbuf` O slots rotate: step i's attend writes `slot()` (= slot i % nbuf), `launch()`
    records an event on the compute stream and runs the head-major all-gather of that slot
    on the side stream (NCCL waits for the side stream, which waits for the event), and the
    attend of step i + nbuf -- which overwrites the slot -- first waits for that gather's
    completion event.  `launch()` returns the gathered [S][N][n_q][Hq][d] tensor, valid once
    `wait(stream)` has made `stream` wait for it.  On CPU tensors (gloo tests) everything
    runs synchronously in the same order."""

    def __init__(self, local_shape, dtype, device, group=None, nbuf: int = 2):
        self.group, self.nbuf, self.i = group, nbuf, 0
        self.device = torch.device(device)
        self.slots = [torch.empty(local_shape, dtype=dtype, device=self.device) for _ in range(nbuf)]
        self.cuda = self.device.type == "cuda"
        self.side = torch.cuda.Stream(self.device) if self.cuda else None
        self.ready = [torch.cuda.Event() for _ in range(nbuf)] if self.cuda else None
        self.done = [torch.cuda.Event() for _ in range(nbuf)] if self.cuda else None
        self.used = [False] * nbuf
        self.out = [None] * nbuf

    def slot(self, stream=None) -> torch.Tensor:
        """The O buffer of this step; `stream` (the compute stream) waits until the gather
        that last read it has finished."""
        b = self.i % self.nbuf
        if self.cuda and self.used[b]:
            (stream or torch.cuda.current_stream(self.device)).wait_event(self.done[b])
        return self.slots[b]

    def launch(self, stream=None) -> torch.Tensor:
        b = self.i % self.nbuf
        if self.cuda:
            st = stream or torch.cuda.current_stream(self.device)
            self.ready[b].record(st)
            self.side.wait_event(self.ready[b])
            with torch.cuda.stream(self.side):
                self.out[b] = gather_heads(self.slots[b], self.group)
            self.done[b].record(self.side)
        else:
            self.out[b] = gather_heads(self.slots[b], self.group)
        self.used[b] = True
        self.i += 1
        return self.out[b]

    def wait(self, stream=None):
        """Make `stream` wait for every gather launched so far."""
        if self.cuda:
            (stream or torch.cuda.current_stream(self.device)).wait_stream(self.side)


def merge_partials(o_parts: torch.Tensor, lse_parts: torch.Tensor) -> torch.Tensor:
    """Reference merge of key-split partials (any backend, any dtype): o_parts [n][..., d],
    lse_parts [n][...] (log2-sum-exp) -> sum_r 2^(lse_r - M) O_r / sum_r 2^(lse_r - M)."""
    m = lse_parts.max(dim=0).values
    w = torch.exp2(lse_parts - m)
    w = torch.where(torch.isfinite(lse_parts), w, torch.zeros_like(w))
    return (w.unsqueeze(-1) * o_parts).sum(0) / w.sum(0).unsqueeze(-1)


def gather_partials(o_part: torch.Tensor, lse_part: torch.Tensor, group=None):
    """All-gather every rank's (O_part, lse_part) -> ([G][...], [G][...]) in rank order."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    o_all = torch.empty((world,) + tuple(o_part.shape), dtype=o_part.dtype, device=o_part.device)
    l_all = torch.empty((world,) + tuple(lse_part.shape), dtype=lse_part.dtype, device=lse_part.device)
    if hasattr(dist, "all_gather_into_tensor") and dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(o_all, o_part.contiguous(), group=group)
        dist.all_gather_into_tensor(l_all, lse_part.contiguous(), group=group)
    else:
        dist.all_gather(list(o_all.unbind(0)), o_part.contiguous(), group=group)
        dist.all_gather(list(l_all.unbind(0)), lse_part.contiguous(), group=group)
    return o_all, l_all


def context_parallel_attend(dsc, q, k_self, v_self, group=None, **kw) -> torch.Tensor:
    """P3: rank r attends over key range r of G (DSCache.attend_partial), the partials are
    all-gathered over `group` (NCCL on the GPU box) and merged on every rank with the
    library's combine kernel.  Returns O like DSCache.attend."""
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    o_part, lse = dsc.attend_partial(q, k_self, v_self, rank, world, **kw)
    o_all, l_all = gather_partials(o_part, lse, group)
    return dsc.combine_partials(o_all, l_all)


class PeerOutputs:
    """Gathered-O buffers of every rank, mapped into this process (P2 fused all-gather).

    Each rank allocates `nbuf` (default 2) buffers [S][N][n_q][Hq][d] of its own (`locals`);
    the CUDA IPC handles (plus offsets inside the allocations) are exchanged with
    all_gather_object over `group`, and every peer's buffers are opened on this rank's device.
    `ptrs[b]` lists buffer b's device pointers in rank order (this rank's own in its slot).
    Steps alternate buffers (kv_split_attend_fused): a step's output stays valid while the
    next step runs, and no rank's stores of step i+1 can land in a buffer a peer is still
    reading from step i (the write-after-read hazard of a single buffer).
    `ipc` = (handle, open, close) functions, the library's by default (injectable for CPU tests)."""

    def __init__(self, shape, dtype, device, group=None, ipc=None, nbuf: int = 2):
        import torch.distributed as dist
        from . import dscache as D
        self.get_handle, self.open, self.close_fn = ipc or (D.ipc_handle, D.ipc_open, D.ipc_close)
        self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        self.device = torch.device(device)
        self.group = group
        self.locals = [torch.empty(shape, dtype=dtype, device=self.device) for _ in range(nbuf)]
        self.step = 0
        mine = [self.get_handle(t) for t in self.locals]
        allh = [None] * self.world
        dist.all_gather_object(allh, mine, group=group)
        self.ptrs, self._opened = [[] for _ in range(nbuf)], []
        for r, handles in enumerate(allh):
            for b, (handle, offset) in enumerate(handles):
                if r == self.rank:
                    self.ptrs[b].append(self.locals[b].data_ptr())
                else:
                    base = self.open(self.device.index or 0, handle)
                    self._opened.append(base)
                    self.ptrs[b].append(base + offset)

    @property
    def local(self):
        """The buffer the next step writes."""
        return self.locals[self.step % len(self.locals)]

    def close(self):
        for base in self._opened:
            self.close_fn(self.device.index or 0, base)
        self._opened = []


def stores_complete(group=None, device=None):
    """Every rank's kernels enqueued so far on its current stream (including their peer
    stores) have completed.  NCCL: a stream-ordered all_reduce of one element, no host sync
    (it can only finish once every rank's stream has reached it); other backends: drain the
    stream, then a host barrier."""
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        flag = torch.zeros(1, dtype=torch.int32, device=device)
        dist.all_reduce(flag, group=group)
    else:
        torch.cuda.current_stream(device).synchronize()
        dist.barrier(group)


def kv_split_attend_fused(dsc, q, k_self, v_self, peers: PeerOutputs, hq_total: int, head_offset: int,
                          group=None, **kw) -> torch.Tensor:
    """P2 with the fused all-gather epilogue: this rank's heads are written by its attention
    kernel into every rank's copy of the step's gathered O (buffer step % nbuf); once every
    rank's stores are complete (stores_complete: stream-ordered on NCCL) it holds the full
    [S][N][n_q][Hq][d] output.  The returned tensor stays valid until the call after next."""
    b = peers.step % len(peers.locals)
    out = peers.locals[b]
    dsc.attend_peers(q, k_self, v_self, peers.ptrs[b], hq_total, head_offset, **kw)
    stores_complete(group if group is not None else peers.group, peers.device)
    peers.step += 1
    return out
