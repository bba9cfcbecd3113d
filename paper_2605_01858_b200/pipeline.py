"""Host-fed streaming steps: the serving path when a step's inputs arrive in (pinned) host
memory and its answer must return to the host.

`HostStepPipeline.submit` enqueues one streaming step -- the H2D copies of the frame K/V,
the instant queries and the query chunk, `DSCache.step` (append + build_instant + attend,
one fused tcgen05 launch), and the D2H copy of the answer O -- on three CUDA streams
with a `depth`-slot ring of device buffers, so step i+1's H2D (PCIe, host -> device)
overlaps step i's kernels and step i-1's D2H (the other PCIe direction).  Everything is
stream-ordered: the call returns at once; `synchronize()` (or the event of `submit`)
marks completion.  Slot reuse is guarded by events (the H2D of step i waits for the
kernels of step i-depth to finish reading the slot; the kernels of step i wait for the
D2H of step i-depth to finish reading its O).  Plumbing only: every step of the hot
path runs in the library's kernels.
"""
from __future__ import annotations

import torch


class HostStepPipeline:
    def __init__(self, dsc, n_q: int, depth: int = 2, layer_begin: int = 0, layer_count=None):
        c = dsc.cfg
        self.dsc, self.depth, self.lb = dsc, depth, layer_begin
        self.lc = c.num_layers - layer_begin if layer_count is None else layer_count
        dev, dt = dsc.device, dsc.torch_dtype
        S, N, tpf, Hkv, Hq, d = c.num_streams, self.lc, c.tokens_per_frame, c.num_kv_heads, c.num_q_heads, c.head_dim
        C = dsc.state(layer_begin)["instant_capacity"]   # C = l_I * tpf, from the library

        def e(*shape):
            return torch.empty(shape, dtype=dt, device=dev)
        # q_inst / O_inst are flat per slot: a step with C_t < C instant rows (warm-up) uses the
        # first S*N*C_t*Hq*d elements as a contiguous [S][N][C_t][Hq][d] view -- no temporary
        # is ever created outside the pipeline's own streams
        self.slots = [dict(k=e(S, N, tpf, Hkv, d), v=e(S, N, tpf, Hkv, d), qi=e(S * N * C * Hq * d),
                           q=e(S, N, n_q, Hq, d), ks=e(S, N, n_q, Hkv, d), vs=e(S, N, n_q, Hkv, d),
                           oi=e(S * N * C * Hq * d), o=e(S, N, n_q, Hq, d)) for _ in range(depth)]
        self.h2d, self.compute, self.d2h = (torch.cuda.Stream(dev) for _ in range(3))
        ev = lambda: [torch.cuda.Event() for _ in range(depth)]   # noqa: E731
        self.loaded, self.in_free, self.computed, self.out_free = ev(), ev(), ev(), ev()
        self.i = 0

    def submit(self, hk, hv, hqi, hq, hks, hvs, ho, o_inst_host=None):
        """One step from pinned host tensors ([S][N][..] as DSCache.step) into `ho` (pinned,
        [S][N][n_q][Hq][d]).  q_inst may cover C_t < C rows only before the buffer is full:
        it is copied into the first hqi.shape[2] rows of the slot.  Returns the event that
        completes when `ho` holds the answer."""
        s = self.i % self.depth
        b = self.slots[s]
        n_inst = hqi.shape[2]
        S, N, _, Hq, d = hqi.shape
        qi = b["qi"][:S * N * n_inst * Hq * d].view(S, N, n_inst, Hq, d)
        oi = b["oi"][:S * N * n_inst * Hq * d].view(S, N, n_inst, Hq, d)
        self.h2d.wait_event(self.in_free[s])
        with torch.cuda.stream(self.h2d):
            b["k"].copy_(hk, non_blocking=True)
            b["v"].copy_(hv, non_blocking=True)
            qi.copy_(hqi, non_blocking=True)
            b["q"].copy_(hq, non_blocking=True)
            b["ks"].copy_(hks, non_blocking=True)
            b["vs"].copy_(hvs, non_blocking=True)
            self.loaded[s].record(self.h2d)
        self.compute.wait_event(self.loaded[s])
        self.compute.wait_event(self.out_free[s])
        self.dsc.step(b["k"], b["v"], qi, b["q"], b["ks"], b["vs"], o_inst=oi, o=b["o"], layer_begin=self.lb,
                      layer_count=self.lc, stream=self.compute)
        self.in_free[s].record(self.compute)
        self.computed[s].record(self.compute)
        self.d2h.wait_event(self.computed[s])
        with torch.cuda.stream(self.d2h):
            ho.copy_(b["o"], non_blocking=True)
            if o_inst_host is not None:
                o_inst_host.copy_(oi, non_blocking=True)
            self.out_free[s].record(self.d2h)
        self.i += 1
        return self.out_free[s]

    def synchronize(self):
        for st in (self.h2d, self.compute, self.d2h):
            st.synchronize()
