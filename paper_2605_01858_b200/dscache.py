"""Thin ctypes binding of libdscache.so (include/dscache.h).

Argument marshalling only: every step of the hot path runs in the library's
sm_100a kernels.  There is no CPU or PyTorch fallback -- if the library is
missing, :func:`load_library` raises.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
# DSCACHE_LIB selects a tuning variant built by _build.build_variant (same ABI)
LIB_PATH = os.environ.get("DSCACHE_LIB") or os.path.join(_PKG, "libdscache.so")

OK, E_ARG, E_CONFIG, E_POS_OVERFLOW, E_STATE, E_CUDA, E_OOM = 0, -1, -2, -3, -4, -5, -6
STATUS_NAMES = {0: "OK", -1: "E_ARG", -2: "E_CONFIG", -3: "E_POS_OVERFLOW", -4: "E_STATE", -5: "E_CUDA",
                -6: "E_OOM"}
DTYPE_BF16, DTYPE_FP32 = 0, 1
ROPE_SPLIT_HALF, ROPE_ADJACENT = 0, 1
IMPL_AUTO, IMPL_TC, IMPL_SIMT = 0, 1, 2
INSTANT_RING, INSTANT_EXTERNAL = 0, 1


class DSCacheError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class Config(ctypes.Structure):
    _fields_ = [("num_streams", ctypes.c_int32), ("num_layers", ctypes.c_int32),
                ("num_q_heads", ctypes.c_int32), ("num_kv_heads", ctypes.c_int32),
                ("head_dim", ctypes.c_int32), ("kv_head_offset", ctypes.c_int32),
                ("tokens_per_frame", ctypes.c_int32), ("sink_tokens", ctypes.c_int32),
                ("past_frames", ctypes.c_int32), ("instant_frames", ctypes.c_int32),
                ("max_query_tokens", ctypes.c_int32), ("max_position", ctypes.c_int32),
                ("rope_theta", ctypes.c_double), ("rope_style", ctypes.c_int32),
                ("dtype", ctypes.c_int32), ("device", ctypes.c_int32), ("attn_impl", ctypes.c_int32),
                ("instant_source", ctypes.c_int32)]


class State(ctypes.Structure):
    _fields_ = [("frames_seen", ctypes.c_int64), ("last_evicted_frame", ctypes.c_int64),
                ("sink_filled", ctypes.c_int32), ("past_tokens", ctypes.c_int32),
                ("instant_tokens", ctypes.c_int32), ("ring_slots", ctypes.c_int32),
                ("tail_slot", ctypes.c_int32), ("instant_slot", ctypes.c_int32),
                ("max_key_id", ctypes.c_int32), ("max_query_id", ctypes.c_int32),
                ("next_instant_tokens", ctypes.c_int32), ("instant_capacity", ctypes.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


EXPORTS = ["dscache_create", "dscache_destroy", "dscache_append_frame", "dscache_build_instant",
           "dscache_append_past", "dscache_build_instant_ext", "dscache_attend_ext", "dscache_decode_ext",
           "dscache_attend", "dscache_update_attend", "dscache_decode", "dscache_build_instant_newest",
           "dscache_instant_approx_rows", "dscache_build_instant_approx", "dscache_decode_sampled", "dscache_step", "dscache_get_state", "dscache_copy_ring", "dscache_copy_sink",
           "dscache_restore_ring", "dscache_restore_sink", "dscache_set_state",
           "dscache_set_debug", "dscache_debug_len", "dscache_set_trace", "dscache_profile", "dscache_profile_read",
           "dscache_attn_impl", "dscache_watchdog_read", "dscache_last_error", "dscache_attend_partial", "dscache_combine_partials",
           "dscache_build_instant_boost", "dscache_attend_boost", "dscache_attend_peers",
           "dscache_ipc_handle", "dscache_ipc_open", "dscache_ipc_close"]

_lib = None


def load_library(path: str = LIB_PATH):
    """Load libdscache.so (once).  Raises if it is missing: no fallback exists."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is missing; build it with `python -m paper_2605_01858_b200._build` "
                           "(or __graft_entry__.build()).  There is no CPU fallback.")
    lib = ctypes.CDLL(path)
    P, I32, I64, D = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    sig = {
        "dscache_create": ([ctypes.POINTER(Config), ctypes.POINTER(P)], I32),
        "dscache_destroy": ([P], I32),
        "dscache_append_frame": ([P, I32, I32, P, P, I32, P], I32),
        "dscache_build_instant": ([P, I32, I32, P, P, P], I32),
        "dscache_attend": ([P, I32, I32, P, P, P, I32, P, P], I32),
        "dscache_update_attend": ([P, I32, I32, P, P, I32, P], I32),
        "dscache_decode": ([P, I32, I32, P, P, P, I32, I32, P, P], I32),
        "dscache_decode_sampled": ([P, I32, I32, P, P, P, I32, I32, I32, P, P], I32),
        "dscache_build_instant_newest": ([P, I32, I32, P, P, P], I32),
        "dscache_instant_approx_rows": ([P, I32, I32, I32, P, ctypes.POINTER(ctypes.c_int32)], I32),
        "dscache_build_instant_approx": ([P, I32, I32, I32, P, I32, P, P], I32),
        "dscache_step": ([P, I32, I32, P, P, P, P, P, P, P, I32, P, P], I32),
        "dscache_get_state": ([P, I32, ctypes.POINTER(State)], I32),
        "dscache_copy_ring": ([P, I32, I32, P, P], I32),
        "dscache_copy_sink": ([P, I32, I32, P, P], I32),
        "dscache_restore_ring": ([P, I32, I32, P, P], I32),
        "dscache_restore_sink": ([P, I32, I32, P, P], I32),
        "dscache_set_state": ([P, I32, I64, I32], I32),
        "dscache_set_debug": ([P, P, P, I32], I32),
        "dscache_debug_len": ([P], I32),
        "dscache_set_trace": ([P, P, I32], I32),
        "dscache_profile": ([P, I32], I32),
        "dscache_profile_read": ([P, ctypes.POINTER(D), ctypes.POINTER(D), ctypes.POINTER(I64),
                                  ctypes.POINTER(I64), ctypes.POINTER(I64), I32], I32),
        "dscache_attn_impl": ([P, I32], I32),
        "dscache_watchdog_read": ([P, I32], I32),
        "dscache_attend_partial": ([P, I32, I32, P, P, P, I32, I32, I32, P, P, P], I32),
        "dscache_combine_partials": ([P, I32, I64, P, P, P, P], I32),
        "dscache_build_instant_boost": ([P, I32, I32, P, P, P, I32, P, P], I32),
        "dscache_attend_boost": ([P, I32, I32, P, P, P, I32, P, P, I32, P, P], I32),
        "dscache_append_past": ([P, I32, I32, P, P, I32, P], I32),
        "dscache_build_instant_ext": ([P, I32, I32, P, P, P, P, P], I32),
        "dscache_attend_ext": ([P, I32, I32, P, P, P, I32, P, P, P, P], I32),
        "dscache_decode_ext": ([P, I32, I32, P, P, P, I32, I32, P, P, P, P], I32),
        "dscache_attend_peers": ([P, I32, I32, P, P, P, I32, ctypes.POINTER(P), I32, I32, I32, P], I32),
        "dscache_ipc_handle": ([P, P, ctypes.POINTER(I64)], I32),
        "dscache_ipc_open": ([I32, P, ctypes.POINTER(P)], I32),
        "dscache_ipc_close": ([I32, P], I32),
        "dscache_last_error": ([], ctypes.c_char_p),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def _check(status: int):
    if status != OK:
        raise DSCacheError(status, _lib.dscache_last_error().decode())


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream_ptr(stream) -> ctypes.c_void_p:
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def ipc_handle(t: torch.Tensor):
    """(64-byte CUDA IPC handle of the allocation holding t, byte offset of t inside it)."""
    load_library()
    buf = ctypes.create_string_buffer(64)
    off = ctypes.c_int64()
    _check(_lib.dscache_ipc_handle(ctypes.c_void_p(t.data_ptr()), buf, ctypes.byref(off)))
    return buf.raw, int(off.value)


def ipc_open(device: int, handle: bytes) -> int:
    """Map another process's IPC handle on `device`; returns the allocation base (int):
    add the exporter's offset."""
    load_library()
    out = ctypes.c_void_p()
    _check(_lib.dscache_ipc_open(int(device), ctypes.create_string_buffer(bytes(handle), 64), ctypes.byref(out)))
    return int(out.value)


def ipc_close(device: int, ptr: int):
    load_library()
    _check(_lib.dscache_ipc_close(int(device), ctypes.c_void_p(ptr)))


class DSCache:
    """One handle = S streams x N layers x Hkv KV heads of DSCache state on one GPU."""

    def __init__(self, *, num_streams: int, num_layers: int, num_q_heads: int, num_kv_heads: int,
                 head_dim: int, tokens_per_frame: int, sink_tokens: int, past_frames: int,
                 instant_frames: int, max_query_tokens: int, rope_theta: float,
                 max_position: int = 32768, dtype: str = "bf16", rope_style: int = ROPE_SPLIT_HALF,
                 device: int = 0, kv_head_offset: int = 0, attn_impl: int = IMPL_AUTO,
                 instant_source: int = INSTANT_RING):
        lib = load_library()
        self.torch_dtype = torch.bfloat16 if dtype == "bf16" else torch.float32
        self.cfg = Config(num_streams, num_layers, num_q_heads, num_kv_heads, head_dim, kv_head_offset,
                          tokens_per_frame, sink_tokens, past_frames, instant_frames, max_query_tokens,
                          max_position, float(rope_theta), rope_style,
                          DTYPE_BF16 if dtype == "bf16" else DTYPE_FP32, device, attn_impl, instant_source)
        self.device = torch.device("cuda", device)
        h = ctypes.c_void_p()
        _check(lib.dscache_create(ctypes.byref(self.cfg), ctypes.byref(h)))
        self._h = h
        self.R = self.state(0)["ring_slots"]   # from the library (it owns the layout)

    @classmethod
    def from_config(cls, cfg, device: int = 0, **kw):
        """From a dscache_synth.StreamConfig-like object (attribute names as in the ABI)."""
        args = dict(num_streams=cfg.num_streams, num_layers=cfg.num_layers, num_q_heads=cfg.num_q_heads,
                    num_kv_heads=cfg.num_kv_heads, head_dim=cfg.head_dim,
                    tokens_per_frame=cfg.tokens_per_frame, sink_tokens=cfg.sink_tokens,
                    past_frames=cfg.past_frames, instant_frames=cfg.instant_frames,
                    max_query_tokens=cfg.query_tokens, rope_theta=cfg.rope_theta,
                    max_position=cfg.max_position, dtype=cfg.dtype, device=device)
        args.update(kw)
        return cls(**args)

    # ------------------------------------------------------------------ lifecycle
    def close(self):
        if getattr(self, "_h", None):
            _check(_lib.dscache_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ------------------------------------------------------------------ checks
    def _t(self, t: torch.Tensor, name: str, shape=None) -> torch.Tensor:
        if not isinstance(t, torch.Tensor) or t.device != self.device:
            raise ValueError(f"{name} must be a CUDA tensor on {self.device}")
        if t.dtype != self.torch_dtype:
            raise ValueError(f"{name} must be {self.torch_dtype}, got {t.dtype}")
        if not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
        if shape is not None and tuple(t.shape) != tuple(shape):
            raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")
        return t

    def _layers(self, layer_begin, layer_count):
        return layer_begin, (self.cfg.num_layers - layer_begin if layer_count is None else layer_count)

    # ------------------------------------------------------------------ hot path
    def append_frame(self, k: torch.Tensor, v: torch.Tensor, layer_begin: int = 0,
                     layer_count: Optional[int] = None, stream=None):
        """k, v: [S][layer_count][n][Hkv][d] (n = A for the sink, tpf for frames)."""
        lb, lc = self._layers(layer_begin, layer_count)
        c = self.cfg
        self._t(k, "k"); self._t(v, "v", k.shape)
        if k.dim() != 5 or k.shape[0] != c.num_streams or k.shape[1] != lc or k.shape[3] != c.num_kv_heads \
                or k.shape[4] != c.head_dim:
            raise ValueError(f"k has shape {tuple(k.shape)}, expected [S, {lc}, n, Hkv, d]")
        _check(_lib.dscache_append_frame(self._h, lb, lc, _ptr(k), _ptr(v), int(k.shape[2]),
                                         _stream_ptr(stream)))

    def build_instant(self, q_inst: torch.Tensor, o_inst: Optional[torch.Tensor] = None, layer_begin: int = 0,
                      layer_count: Optional[int] = None, stream=None) -> torch.Tensor:
        """q_inst: [S][layer_count][C_t][Hq][d] -> O_inst (same shape)."""
        lb, lc = self._layers(layer_begin, layer_count)
        c = self.cfg
        C_t = self.state(lb)["instant_tokens"]
        shape = (c.num_streams, lc, C_t, c.num_q_heads, c.head_dim)
        self._t(q_inst, "q_inst", shape)
        if o_inst is None:
            o_inst = torch.empty(shape, dtype=self.torch_dtype, device=self.device)
        self._t(o_inst, "o_inst", shape)
        _check(_lib.dscache_build_instant(self._h, lb, lc, _ptr(q_inst), _ptr(o_inst), _stream_ptr(stream)))
        return o_inst

    def attend(self, q: torch.Tensor, k_self: torch.Tensor, v_self: torch.Tensor,
               o: Optional[torch.Tensor] = None, layer_begin: int = 0, layer_count: Optional[int] = None,
               stream=None) -> torch.Tensor:
        """q: [S][lc][n_q][Hq][d], k_self/v_self: [S][lc][n_q][Hkv][d] -> O [S][lc][n_q][Hq][d]."""
        lb, lc = self._layers(layer_begin, layer_count)
        c = self.cfg
        n_q = int(q.shape[2])
        self._t(q, "q", (c.num_streams, lc, n_q, c.num_q_heads, c.head_dim))
        self._t(k_self, "k_self", (c.num_streams, lc, n_q, c.num_kv_heads, c.head_dim))
        self._t(v_self, "v_self", k_self.shape)
        if o is None:
            o = torch.empty(q.shape, dtype=self.torch_dtype, device=self.device)
        self._t(o, "o", q.shape)
        _check(_lib.dscache_attend(self._h, lb, lc, _ptr(q), _ptr(k_self), _ptr(v_self), n_q, _ptr(o),
                                   _stream_ptr(stream)))
        return o

    def build_instant_boost(self, q_inst: torch.Tensor, k_boost: torch.Tensor, v_boost: torch.Tensor,
                            o_inst: Optional[torch.Tensor] = None, layer_begin: int = 0,
                            layer_count: Optional[int] = None, stream=None) -> torch.Tensor:
        """Instant cache with the newest frame re-encoded:
        k_boost/v_boost [S][lc][n_boost][Hkv][d] replace the newest frame's ring K/V;
        q_inst [S][lc][C_t - tpf + n_boost][Hq][d] -> O_inst (same shape)."""
        lb, lc = self._layers(layer_begin, layer_count)
        c = self.cfg
        n_boost = int(k_boost.shape[2])
        self._t(k_boost, "k_boost", (c.num_streams, lc, n_boost, c.num_kv_heads, c.head_dim))
        self._t(v_boost, "v_boost", k_boost.shape)
        C_t = self.state(lb)["instant_tokens"]
        shape = (c.num_streams, lc, C_t - c.tokens_per_frame + n_boost, c.num_q_heads, c.head_dim)
        self._t(q_inst, "q_inst", shape)
        if o_inst is None:
            o_inst = torch.empty(shape, dtype=self.torch_dtype, device=self.device)
        self._t(o_inst, "o_inst", shape)
        _check(_lib.dscache_build_instant_boost(self._h, lb, lc, _ptr(q_inst), _ptr(k_boost), _ptr(v_boost), n_boost,
                                                _ptr(o_inst), _stream_ptr(stream)))
        return o_inst

    def attend_boost(self, q: torch.Tensor, k_self: torch.Tensor, v_self: torch.Tensor, k_boost: torch.Tensor,
                     v_boost: torch.Tensor, o: Optional[torch.Tensor] = None, layer_begin: int = 0,
                     layer_count: Optional[int] = None, stream=None) -> torch.Tensor:
        """attend() over a final cache whose newest instant frame is the boosted re-encoding."""
        lb, lc = self._layers(layer_begin, layer_count)
        c = self.cfg
        n_q, n_boost = int(q.shape[2]), int(k_boost.shape[2])
        self._t(q, "q", (c.num_streams, lc, n_q, c.num_q_heads, c.head_dim))
        self._t(k_self, "k_self", (c.num_streams, lc, n_q, c.num_kv_heads, c.head_dim))
        self._t(v_self, "v_self", k_self.shape)
        self._t(k_boost, "k_boost", (c.num_streams, lc, n_boost, c.num_kv_heads, c.head_dim))
        self._t(v_boost, "v_boost", k_boost.shape)
        if o is None:
            o = torch.empty(q.shape, dtype=self.torch_dtype, device=self.device)
        self._t(o, "o", q.shape)
        _check(_lib.dscache_attend_boost(self._h, lb, lc, _ptr(q), _ptr(k_self), _ptr(v_self), n_q, _ptr(k_boost),
                                         _ptr(v_boost), n_boost, _ptr(o), _stream_ptr(stream)))
        return o

    # ------------------------------------------------------------------ real-model mode (NEXT-1)
    def append_past(self, k_past: Optional[torch.Tensor], v_past: Optional[torch.Tensor], layer_begin: int = 0,
                    layer_count: Optional[int] = None, stream=None):
        """Advance to the next step; once a frame leaves the buffer, store its Eq. 5 K/V
        ([S][lc][tpf][Hkv][d]; None while nothing leaves)."""
        lb, lc = self._layers(layer_begin, layer_count)
        c = self.cfg
        n = 0
        if k_past is not None:
            n = int(k_past.shape[2])
            self._t(k_past, "k_past", (c.num_streams, lc, n, c.num_kv_heads, c.head_dim))
            self._t(v_past, "v_past", k_past.shape)
        _check(_lib.dscache_append_past(self._h, lb, lc, _ptr(k_past), _ptr(v_past), n, _stream_ptr(stream)))

    def build_instant_ext(self, q_inst: torch.Tensor, k_inst: torch.Tensor, v_inst: torch.Tensor,
                          o_inst: Optional[torch.Tensor] = None, layer_begin: int = 0,
                          layer_count: Optional[int] = None, stream=None) -> torch.Tensor:
        """Eq. 7 with the caller's instant K/V ([S][lc][C_t][Hkv][d])."""
        lb, lc = self._layers(layer_begin, layer_count)
        c = self.cfg
        C_t = self.state(lb)["instant_tokens"]
        self._t(q_inst, "q_inst", (c.num_streams, lc, C_t, c.num_q_heads, c.head_dim))
        self._t(k_inst, "k_inst", (c.num_streams, lc, C_t, c.num_kv_heads, c.head_dim))
        self._t(v_inst, "v_inst", k_inst.shape)
        if o_inst is None:
            o_inst = torch.empty(q_inst.shape, dtype=self.torch_dtype, device=self.device)
        self._t(o_inst, "o_inst", q_inst.shape)
        _check(_lib.dscache_build_instant_ext(self._h, lb, lc, _ptr(q_inst), _ptr(k_inst), _ptr(v_inst), _ptr(o_inst),
                                              _stream_ptr(stream)))
        return o_inst

    def attend_ext(self, q: torch.Tensor, k_self: torch.Tensor, v_self: torch.Tensor, k_inst: torch.Tensor,
                   v_inst: torch.Tensor, o: Optional[torch.Tensor] = None, layer_begin: int = 0,
                   layer_count: Optional[int] = None, stream=None) -> torch.Tensor:
        """Eq. 8 over [sink | past (ring) | caller instant K/V | self]."""
        lb, lc = self._layers(layer_begin, layer_count)
        c = self.cfg
        n_q = int(q.shape[2])
        C_t = self.state(lb)["instant_tokens"]
        self._t(q, "q", (c.num_streams, lc, n_q, c.num_q_heads, c.head_dim))
        self._t(k_self, "k_self", (c.num_streams, lc, n_q, c.num_kv_heads, c.head_dim))
        self._t(v_self, "v_self", k_self.shape)
        self._t(k_inst, "k_inst", (c.num_streams, lc, C_t, c.num_kv_heads, c.head_dim))
        self._t(v_inst, "v_inst", k_inst.shape)
        if o is None:
            o = torch.empty(q.shape, dtype=self.torch_dtype, device=self.device)
        self._t(o, "o", q.shape)
        _check(_lib.dscache_attend_ext(self._h, lb, lc, _ptr(q), _ptr(k_self), _ptr(v_self), n_q, _ptr(k_inst),
                                       _ptr(v_inst), _ptr(o), _stream_ptr(stream)))
        return o

    def decode_ext(self, q: torch.Tensor, k_self: torch.Tensor, v_self: torch.Tensor, k_inst: torch.Tensor,
                   v_inst: torch.Tensor, o: Optional[torch.Tensor] = None, layer_begin: int = 0,
                   layer_count: Optional[int] = None, stream=None) -> torch.Tensor:
        """Decode over [sink | past (ring) | caller instant K/V | self]: q = the last n_q of the
        n_self self tokens (real-model mode)."""
        lb, lc = self._layers(layer_begin, layer_count)
        c = self.cfg
        n_q, n_self = int(q.shape[2]), int(k_self.shape[2])
        C_t = self.state(lb)["instant_tokens"]
        self._t(q, "q", (c.num_streams, lc, n_q, c.num_q_heads, c.head_dim))
        self._t(k_self, "k_self", (c.num_streams, lc, n_self, c.num_kv_heads, c.head_dim))
        self._t(v_self, "v_self", k_self.shape)
        self._t(k_inst, "k_inst", (c.num_streams, lc, C_t, c.num_kv_heads, c.head_dim))
        self._t(v_inst, "v_inst", k_inst.shape)
        if o is None:
            o = torch.empty(q.shape, dtype=self.torch_dtype, device=self.device)
        self._t(o, "o", q.shape)
        _check(_lib.dscache_decode_ext(self._h, lb, lc, _ptr(q), _ptr(k_self), _ptr(v_self), n_self, n_q,
                                       _ptr(k_inst), _ptr(v_inst), _ptr(o), _stream_ptr(stream)))
        return o

    def attend_peers(self, q: torch.Tensor, k_self: torch.Tensor, v_self: torch.Tensor, peer_ptrs, hq_total: int,
                     head_offset: int, layer_begin: int = 0, layer_count: Optional[int] = None, stream=None):
        """Fused all-gather epilogue (P2): this handle's attend rows are stored by the kernel into
        every gathered-O buffer in `peer_ptrs` (device pointers as ints, or tensors on this
        device), bf16 [S][lc][n_q][hq_total][d], q head h at head_offset + h."""
        lb, lc = self._layers(layer_begin, layer_count)
        c = self.cfg
        n_q = int(q.shape[2])
        self._t(q, "q", (c.num_streams, lc, n_q, c.num_q_heads, c.head_dim))
        self._t(k_self, "k_self", (c.num_streams, lc, n_q, c.num_kv_heads, c.head_dim))
        self._t(v_self, "v_self", k_self.shape)
        ptrs = []
        for x in peer_ptrs:
            if isinstance(x, torch.Tensor):
                self._t(x, "peer O", (c.num_streams, lc, n_q, hq_total, c.head_dim))
                x = x.data_ptr()
            ptrs.append(int(x))
        arr = (ctypes.c_void_p * max(len(ptrs), 1))(*ptrs)
        _check(_lib.dscache_attend_peers(self._h, lb, lc, _ptr(q), _ptr(k_self), _ptr(v_self), n_q, arr, len(ptrs),
                                         int(hq_total), int(head_offset), _stream_ptr(stream)))

    def attend_partial(self, q: torch.Tensor, k_self: torch.Tensor, v_self: torch.Tensor, part: int, n_parts: int,
                       layer_begin: int = 0, layer_count: Optional[int] = None, stream=None):
        """Part `part` of `n_parts` of the attend's keys (context parallelism):
        returns (O_part fp32 [S][lc][n_q][Hq][d], lse_part fp32 [S][lc][n_q][Hq])."""
        lb, lc = self._layers(layer_begin, layer_count)
        c = self.cfg
        n_q = int(q.shape[2])
        self._t(q, "q", (c.num_streams, lc, n_q, c.num_q_heads, c.head_dim))
        self._t(k_self, "k_self", (c.num_streams, lc, n_q, c.num_kv_heads, c.head_dim))
        self._t(v_self, "v_self", k_self.shape)
        o_part = torch.empty(q.shape, dtype=torch.float32, device=self.device)
        lse = torch.empty(q.shape[:-1], dtype=torch.float32, device=self.device)
        _check(_lib.dscache_attend_partial(self._h, lb, lc, _ptr(q), _ptr(k_self), _ptr(v_self), n_q, part, n_parts,
                                           _ptr(o_part), _ptr(lse), _stream_ptr(stream)))
        return o_part, lse

    def combine_partials(self, o_parts: torch.Tensor, lse_parts: torch.Tensor, stream=None) -> torch.Tensor:
        """o_parts [n][..., d] fp32, lse_parts [n][...] fp32 -> merged O (bf16, shape o_parts[0])."""
        if o_parts.dtype != torch.float32 or lse_parts.dtype != torch.float32:
            raise TypeError("partials must be fp32")
        if not (o_parts.is_contiguous() and lse_parts.is_contiguous()):
            raise ValueError("partials must be contiguous")
        n = int(o_parts.shape[0])
        rows = lse_parts[0].numel()
        if o_parts[0].numel() != rows * self.cfg.head_dim:
            raise ValueError("o_parts / lse_parts shapes disagree")
        o = torch.empty(o_parts.shape[1:], dtype=torch.bfloat16, device=self.device)
        _check(_lib.dscache_combine_partials(self._h, n, rows, _ptr(o_parts), _ptr(lse_parts), _ptr(o),
                                             _stream_ptr(stream)))
        return o

    def step(self, k: torch.Tensor, v: torch.Tensor, q_inst: torch.Tensor, q: torch.Tensor, k_self: torch.Tensor,
             v_self: torch.Tensor, o_inst: Optional[torch.Tensor] = None, o: Optional[torch.Tensor] = None,
             layer_begin: int = 0, layer_count: Optional[int] = None, stream=None):
        """append_frame(k, v) + build_instant(q_inst) + attend(q, k_self, v_self) in one call
        (one fused tcgen05 launch for the two attentions).  Returns (O_inst, O)."""
        lb, lc = self._layers(layer_begin, layer_count)
        c = self.cfg
        fshape = (c.num_streams, lc, c.tokens_per_frame, c.num_kv_heads, c.head_dim)
        self._t(k, "k", fshape); self._t(v, "v", fshape)
        C_t = self.state(lb)["next_instant_tokens"]   # the library's closed form (C_{t+1})
        ishape = (c.num_streams, lc, C_t, c.num_q_heads, c.head_dim)
        self._t(q_inst, "q_inst", ishape)
        if o_inst is None:
            o_inst = torch.empty(ishape, dtype=self.torch_dtype, device=self.device)
        self._t(o_inst, "o_inst", ishape)
        n_q = int(q.shape[2])
        self._t(q, "q", (c.num_streams, lc, n_q, c.num_q_heads, c.head_dim))
        self._t(k_self, "k_self", (c.num_streams, lc, n_q, c.num_kv_heads, c.head_dim))
        self._t(v_self, "v_self", k_self.shape)
        if o is None:
            o = torch.empty(q.shape, dtype=self.torch_dtype, device=self.device)
        self._t(o, "o", q.shape)
        _check(_lib.dscache_step(self._h, lb, lc, _ptr(k), _ptr(v), _ptr(q_inst), _ptr(o_inst), _ptr(q),
                                 _ptr(k_self), _ptr(v_self), n_q, _ptr(o), _stream_ptr(stream)))
        return o_inst, o

    def build_instant_newest(self, q_new: torch.Tensor, o_new: Optional[torch.Tensor] = None,
                             layer_begin: int = 0, layer_count: Optional[int] = None, stream=None) -> torch.Tensor:
        """Approximate instant cache (NEXT-3): only the newest frame's instant rows."""
        lb, lc = self._layers(layer_begin, layer_count)
        c = self.cfg
        shape = (c.num_streams, lc, c.tokens_per_frame, c.num_q_heads, c.head_dim)
        self._t(q_new, "q_new", shape)
        if o_new is None:
            o_new = torch.empty(shape, dtype=self.torch_dtype, device=self.device)
        self._t(o_new, "o_new", shape)
        _check(_lib.dscache_build_instant_newest(self._h, lb, lc, _ptr(q_new), _ptr(o_new), _stream_ptr(stream)))
        return o_new

    def approx_ring(self, layer_count: Optional[int] = None) -> torch.Tensor:
        """A row ring for build_instant_approx: [S][lc][C][Hq][d], frame f at rows (f mod l_I)*tpf."""
        c = self.cfg
        lc = c.num_layers if layer_count is None else layer_count
        C = self.state(0)["instant_capacity"]   # C = l_I * tpf, from the library
        return torch.zeros((c.num_streams, lc, C, c.num_q_heads, c.head_dim),
                           dtype=self.torch_dtype, device=self.device)

    def approx_rows(self, o_ring: torch.Tensor, period: int, layer_begin: int = 0,
                    layer_count: Optional[int] = None) -> int:
        """Query rows the next build_instant_approx takes: C_t on a refresh, tpf otherwise."""
        lb, lc = self._layers(layer_begin, layer_count)
        n = ctypes.c_int32()
        _check(_lib.dscache_instant_approx_rows(self._h, lb, lc, int(period), _ptr(o_ring), ctypes.byref(n)))
        return n.value

    def build_instant_approx(self, q_rows: torch.Tensor, o_ring: torch.Tensor, period: int, layer_begin: int = 0,
                             layer_count: Optional[int] = None, stream=None) -> torch.Tensor:
        """Approximate instant cache (NEXT-3): refresh every `period` steps, otherwise only the
        newest frame's rows; o_ring [S][lc][C][Hq][d] is updated in place (see approx_ring)."""
        lb, lc = self._layers(layer_begin, layer_count)
        c = self.cfg
        n = int(q_rows.shape[2])
        self._t(q_rows, "q_rows", (c.num_streams, lc, n, c.num_q_heads, c.head_dim))
        self._t(o_ring, "o_ring", (c.num_streams, lc, self.state(lb)["instant_capacity"], c.num_q_heads,
                                   c.head_dim))
        _check(_lib.dscache_build_instant_approx(self._h, lb, lc, int(period), _ptr(q_rows), n, _ptr(o_ring),
                                                 _stream_ptr(stream)))
        return o_ring

    def decode(self, q: torch.Tensor, k_self: torch.Tensor, v_self: torch.Tensor, o: Optional[torch.Tensor] = None,
               layer_begin: int = 0, layer_count: Optional[int] = None, stream=None,
               past_stride: int = 1) -> torch.Tensor:
        """Decode (NEXT-2): q [S][lc][n_q][Hq][d] = the last n_q tokens of the self segment
        k_self/v_self [S][lc][n_self][Hkv][d] (query chunk + generated tokens).  past_stride > 1
        keeps every past_stride-th past frame (zeta_decode)."""
        lb, lc = self._layers(layer_begin, layer_count)
        c = self.cfg
        n_q, n_self = int(q.shape[2]), int(k_self.shape[2])
        self._t(q, "q", (c.num_streams, lc, n_q, c.num_q_heads, c.head_dim))
        self._t(k_self, "k_self", (c.num_streams, lc, n_self, c.num_kv_heads, c.head_dim))
        self._t(v_self, "v_self", k_self.shape)
        if o is None:
            o = torch.empty(q.shape, dtype=self.torch_dtype, device=self.device)
        self._t(o, "o", q.shape)
        _check(_lib.dscache_decode_sampled(self._h, lb, lc, _ptr(q), _ptr(k_self), _ptr(v_self), n_self, n_q,
                                           int(past_stride), _ptr(o), _stream_ptr(stream)))
        return o

    def update_attend(self, q_upd: torch.Tensor, o_upd: Optional[torch.Tensor] = None,
                      active_frames: Optional[int] = None, layer_begin: int = 0,
                      layer_count: Optional[int] = None, stream=None) -> torch.Tensor:
        """Eq. 5 cumulative-update attention of the frame leaving the buffer.
        q_upd: [S][lc][tpf][Hq][d]; active_frames = l_L (default l_U)."""
        lb, lc = self._layers(layer_begin, layer_count)
        c = self.cfg
        shape = (c.num_streams, lc, c.tokens_per_frame, c.num_q_heads, c.head_dim)
        self._t(q_upd, "q_upd", shape)
        if o_upd is None:
            o_upd = torch.empty(shape, dtype=self.torch_dtype, device=self.device)
        self._t(o_upd, "o_upd", shape)
        l_L = c.past_frames if active_frames is None else int(active_frames)
        _check(_lib.dscache_update_attend(self._h, lb, lc, _ptr(q_upd), _ptr(o_upd), l_L, _stream_ptr(stream)))
        return o_upd

    # ------------------------------------------------------------------ introspection
    def state(self, layer: int = 0) -> dict:
        st = State()
        _check(_lib.dscache_get_state(self._h, layer, ctypes.byref(st)))
        return st.as_dict()

    def copy_ring(self, stream_idx: int, layer: int):
        c = self.cfg
        shape = (c.num_kv_heads, self.R, c.head_dim)
        k = torch.empty(shape, dtype=self.torch_dtype)
        v = torch.empty(shape, dtype=self.torch_dtype)
        _check(_lib.dscache_copy_ring(self._h, stream_idx, layer, _ptr(k), _ptr(v)))
        return k, v

    def copy_sink(self, stream_idx: int, layer: int):
        c = self.cfg
        shape = (c.num_kv_heads, c.sink_tokens, c.head_dim)
        k = torch.empty(shape, dtype=self.torch_dtype)
        v = torch.empty(shape, dtype=self.torch_dtype)
        _check(_lib.dscache_copy_sink(self._h, stream_idx, layer, _ptr(k), _ptr(v)))
        return k, v

    # ------------------------------------------------------------------ checkpoint / resume
    def restore_ring(self, stream_idx: int, layer: int, k: torch.Tensor, v: torch.Tensor):
        """Upload a ring snapshot ([Hkv][R][d] host tensors, as copy_ring returns them)."""
        c = self.cfg
        shape = (c.num_kv_heads, self.R, c.head_dim)
        for t in (k, v):
            if tuple(t.shape) != shape or t.dtype != self.torch_dtype or t.is_cuda or not t.is_contiguous():
                raise ValueError(f"ring snapshot must be contiguous host {self.torch_dtype} {shape}")
        _check(_lib.dscache_restore_ring(self._h, stream_idx, layer, _ptr(k), _ptr(v)))

    def restore_sink(self, stream_idx: int, layer: int, k: torch.Tensor, v: torch.Tensor):
        """Upload a sink snapshot ([Hkv][A][d] host tensors, as copy_sink returns them)."""
        c = self.cfg
        shape = (c.num_kv_heads, c.sink_tokens, c.head_dim)
        for t in (k, v):
            if tuple(t.shape) != shape or t.dtype != self.torch_dtype or t.is_cuda or not t.is_contiguous():
                raise ValueError(f"sink snapshot must be contiguous host {self.torch_dtype} {shape}")
        _check(_lib.dscache_restore_sink(self._h, stream_idx, layer, _ptr(k), _ptr(v)))

    def set_state(self, layer: int, frames_seen: int, sink_filled: int):
        _check(_lib.dscache_set_state(self._h, layer, int(frames_seen), int(sink_filled)))

    def snapshot(self) -> bytes:
        """The whole streaming state as one flat little-endian blob (checkpoint.pack)."""
        from . import checkpoint
        c = self.cfg
        counters = [(self.state(l)["frames_seen"], self.state(l)["sink_filled"]) for l in range(c.num_layers)]
        slabs = {}
        for s in range(c.num_streams):
            for l in range(c.num_layers):
                slabs[(s, l)] = self.copy_sink(s, l) + self.copy_ring(s, l)
        return checkpoint.pack(c, self.R, counters, slabs)

    def restore(self, blob: bytes):
        """Resume from snapshot(): the config must match this handle's field for field."""
        from . import checkpoint
        counters, slabs = checkpoint.unpack(blob, self.cfg, self.R)
        c = self.cfg
        for s in range(c.num_streams):
            for l in range(c.num_layers):
                sk, sv, rk, rv = slabs[(s, l)]
                self.restore_sink(s, l, sk, sv)
                self.restore_ring(s, l, rk, rv)
        for l, (f, sf) in enumerate(counters):
            self.set_state(l, f, sf)

    def debug_len(self) -> int:
        return int(_lib.dscache_debug_len(self._h))

    def set_debug(self, build_pos: Optional[torch.Tensor] = None, attend_pos: Optional[torch.Tensor] = None,
                  poison: bool = False):
        need = self.cfg.num_streams * self.cfg.num_layers * self.debug_len()
        for t in (build_pos, attend_pos):
            if t is not None and (t.dtype != torch.int32 or t.device != self.device or t.numel() < need):
                raise ValueError("debug buffers must be int32 CUDA tensors of num_streams*num_layers*debug_len() "
                                 "entries ([S][N][debug_len])")
        self._dbg = (build_pos, attend_pos)   # keep alive
        _check(_lib.dscache_set_debug(self._h, _ptr(build_pos), _ptr(attend_pos), int(bool(poison))))

    def set_trace(self, buf: Optional[torch.Tensor], ntrace_cta: int = 1):
        """buf: int64 CUDA tensor of ntrace_cta*32*1024 entries (v7 FA_TRACE layout; None = off)."""
        if buf is not None and (buf.dtype != torch.int64 or buf.numel() < ntrace_cta * 32 * 1024):
            raise ValueError("trace buffer must be int64 with ntrace_cta*32*1024 entries")
        self._trace = buf
        _check(_lib.dscache_set_trace(self._h, _ptr(buf), int(ntrace_cta)))

    def profile(self, enable: bool = True):
        _check(_lib.dscache_profile(self._h, int(enable)))

    def profile_read(self, reset: bool = True) -> dict:
        mb, ma = ctypes.c_double(), ctypes.c_double()
        nb, na, nl = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _check(_lib.dscache_profile_read(self._h, ctypes.byref(mb), ctypes.byref(ma), ctypes.byref(nb),
                                         ctypes.byref(na), ctypes.byref(nl), int(reset)))
        return {"ms_build": mb.value, "ms_attend": ma.value, "n_build": nb.value, "n_attend": na.value,
                "kernel_launches": nl.value}

    def attn_impl(self) -> dict:
        names = {IMPL_TC: "tcgen05", IMPL_SIMT: "simt"}
        return {"build_instant": names.get(_lib.dscache_attn_impl(self._h, 0)),
                "attend": names.get(_lib.dscache_attn_impl(self._h, 1))}


def watchdog_records():
    """Debug: the tcgen05 kernel's watchdog records (DSC_WATCHDOG=1), as a list of
    (cta, warp, barrier index, parity, clock); readable after a trapped kernel."""
    buf = (ctypes.c_uint64 * 257)()
    if _lib.dscache_watchdog_read(buf, 257) != 0:
        return None
    n = min(int(buf[0]), 64)
    return [(int(buf[1 + 4 * i]), int(buf[2 + 4 * i]), int(buf[3 + 4 * i]) >> 32, int(buf[3 + 4 * i]) & 0xFFFFFFFF,
             int(buf[4 + 4 * i])) for i in range(n)]
