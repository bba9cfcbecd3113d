"""DSCache fp64 CPU oracle -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import or execute anything under ``oracle/``.  The
CUDA path (``paper_2605_01858_b200``) never imports it, and this file imports
nothing from the CUDA path: the two share only the seeded input generator
``dscache_synth`` (which holds no arithmetic of the method).

What it computes (per stream s, per layer r; everything in float64):

* the buffer / cumulative-cache schedule, simulated literally as the FIFO lists
  of Eq. 3 and Eq. 5-6, with text K/V
  never entering U;
* the instant cache build I = phi(B, C_a) (Eq. 7): each
  instant token attends to the sink and to the instant tokens before it, with
  consecutive position ids from 0;
* the final attention over [C_a, U, I] (Eq. 8) plus the query
  chunk itself, again with consecutive position ids from 0 (PAPER.md:236,
  Eq. 2);
* the resolution-boosted newest frame: the instant cache
  and the final attention with the buffer's newest input re-encoded;
* the real-model mode: Eq. 7 / Eq. 8 with the step's instant K/V supplied
  by the caller and U holding each frame's Eq. 5 K/V (instant_cache_output_ext,
  attend_output_ext; the Eq. 5 attention is cumulative_update_output over those K/V);
* the approximate instant cache: full Eq. 7 rebuilds
  every `period` steps, the newest frame's rows alone in between, older rows reused
  (instant_cache_output_approx);
* decoding over C_{t+1}: the last tokens of [query chunk | generated
  tokens] attend over [C_a, U, I, self], optionally with U sampled at a
  frame stride (decode_output_sampled);
* the cumulative-update attention inside phi(X_{t-l_I}, [C_a, zeta(U_{t-1})]) of
  Eq. 5: the input leaving the buffer attends to the sink, the
  newest l_L frames of U_{t-1} and itself;
* position-agnostic encoding (Def. 4.1): keys are kept raw and
  RoPE f(., m) is applied at use time;
* softmax attention a_ij = softmax(Q_i K_j / sqrt(D)), with D read
  as the head dimension (reading Q8).

Readings of points where the paper is silent: split-half
RoPE with theta_i = base^(-2i/d) (Q7; adjacent pairs available), 1/sqrt(head_dim)
scale (Q8), causal masking by position id (Q9), GQA head map g = h // (Hq/Hkv)
(Q10), whole-frame FIFO eviction (Q11), order append -> build -> attend with the
newest frame already in the instant window (Q12).

Pins (tests/test_oracle_pins.py, all ``-m "not gpu"``): RoPE closed forms and
group/shift invariances, the Eq. 3/6 FIFO against an independently derived
closed form and hand-derived golden values, Q = 0 closed forms (mean of visible
V, mean of position ids), single-key identity, pure-Python brute force on tiny
streams, torch SDPA (fp64) as a library routine for the attention core, the
Proposition with absolute ids, the l_I = 0 / l_U = 0
reductions and the decoupling of Eq. 7.  No
function here is "parity unpinned".
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, List, Sequence, Tuple

import numpy as np

SPLIT_HALF = 0   # pairs (i, i + d/2)   -- DESIGN.md reading Q7 (Qwen2 / LLaVA-OV convention)
ADJACENT = 1     # pairs (2i, 2i + 1)   -- SPEC.md:142 convention, kept as an option


# ---------------------------------------------------------------------------
# RoPE  f(x, m)   ("applies positional encoding using contiguous
# position IDs starting from m"; relative property)
# ---------------------------------------------------------------------------
def rope_frequencies(head_dim: int, theta: float) -> np.ndarray:
    """theta_i = base^(-2i/d), i < d/2."""
    i = np.arange(head_dim // 2, dtype=np.float64)
    return theta ** (-2.0 * i / head_dim)


def rope(x: np.ndarray, positions: np.ndarray, theta: float, style: int = SPLIT_HALF) -> np.ndarray:
    """Rotate the last axis of x (shape [n, ..., d]) by the position of its row.

    positions has shape [n]; every pair (a, b) of coordinates is rotated by the
    angle position * theta_i:  (a, b) -> (a cos - b sin, a sin + b cos).
    """
    x = np.asarray(x, dtype=np.float64)
    d = x.shape[-1]
    ang = np.asarray(positions, dtype=np.float64)[:, None] * rope_frequencies(d, theta)[None, :]
    ang = ang.reshape((ang.shape[0],) + (1,) * (x.ndim - 2) + (d // 2,))
    c, s = np.cos(ang), np.sin(ang)
    if style == SPLIT_HALF:
        a, b = x[..., : d // 2], x[..., d // 2:]
        return np.concatenate([a * c - b * s, a * s + b * c], axis=-1)
    a, b = x[..., 0::2], x[..., 1::2]
    out = np.empty_like(x)
    out[..., 0::2] = a * c - b * s
    out[..., 1::2] = a * s + b * c
    return out


# ---------------------------------------------------------------------------
# Softmax attention  (Eq. in App. B):  a_ij = softmax(Q_i K_j / sqrt(D))
# ---------------------------------------------------------------------------
def softmax_attention(q: np.ndarray, k: np.ndarray, v: np.ndarray, visible: np.ndarray) -> np.ndarray:
    """q [nq, d], k [nk, d], v [nk, dv], visible [nq, nk] bool -> [nq, dv] (fp64).

    Rows with no visible key return 0 (never happens on the DSCache path: every
    query sees at least itself).
    """
    d = q.shape[-1]
    if q.shape[0] == 0 or k.shape[0] == 0:   # an empty attention (e.g. no instant cache: l_I = 0)
        return np.zeros((q.shape[0], v.shape[-1]), np.float64)
    s = (q @ k.T) / math.sqrt(d)
    s = np.where(visible, s, -np.inf)
    m = np.max(s, axis=1, keepdims=True)
    m = np.where(np.isfinite(m), m, 0.0)
    p = np.where(visible, np.exp(s - m), 0.0)
    den = p.sum(axis=1, keepdims=True)
    den = np.where(den > 0, den, 1.0)
    return (p / den) @ v


def gqa_attention(q: np.ndarray, pos_q: np.ndarray, k_raw: np.ndarray, v: np.ndarray,
                  pos_k: np.ndarray, theta: float, style: int = SPLIT_HALF) -> np.ndarray:
    """Position-agnostic GQA attention (Def. 4.1): raw keys rotated at use time.

    q [nq, Hq, d]; k_raw, v [nk, Hkv, d]; query i sees key j iff pos_k[j] <= pos_q[i]
    (causal in position-id order, reading Q9).  Query head h reads KV head
    h // (Hq/Hkv) (reading Q10).  Returns [nq, Hq, d] float64.
    """
    nq, hq, d = q.shape
    hkv = k_raw.shape[1]
    grp = hq // hkv
    qr = rope(q, pos_q, theta, style)
    kr = rope(k_raw, pos_k, theta, style)
    vis = np.asarray(pos_k)[None, :] <= np.asarray(pos_q)[:, None]
    out = np.zeros((nq, hq, v.shape[-1]), dtype=np.float64)
    for h in range(hq):
        g = h // grp
        out[:, h, :] = softmax_attention(qr[:, h, :], kr[:, g, :], np.asarray(v[:, g, :], np.float64), vis)
    return out


# ---------------------------------------------------------------------------
# Buffer / cumulative-cache schedule, literally as FIFO lists (Eq. 3, 5, 6)
# ---------------------------------------------------------------------------
@dataclass
class StepSchedule:
    t: int
    instant_frames: List[int]           # B_t (Eq. 3), oldest first
    past_frames: List[int]              # U_t (Eq. 5-6), oldest first
    evicted: List[int] = field(default_factory=list)   # frames dropped from U at step t (Eq. 6)
    tokens_per_frame: int = 0
    sink_tokens: int = 0

    @property
    def C_t(self) -> int:
        return len(self.instant_frames) * self.tokens_per_frame

    @property
    def P_t(self) -> int:
        return len(self.past_frames) * self.tokens_per_frame


def schedule_fifo(t: int, instant_frames: int, past_frames: int, tokens_per_frame: int,
                  sink_tokens: int) -> StepSchedule:
    """Replay Eq. 3 / Eq. 5 / Eq. 6 as list operations for frames 0..t.

    Eq. 3: push X_t into B; when B already held l_I inputs the
    oldest X_{t-l_I} leaves B.  Eq. 5: the evicted input is
    appended to U.  Eq. 6: U keeps its newest l_U frames
    (whole frames, reading Q11).  Text K/V never enter U, so only
    frames are tracked.
    """
    B: List[int] = []
    U: List[int] = []
    evicted_now: List[int] = []
    for f in range(t + 1):
        evicted_now = []
        B.append(f)
        if len(B) > instant_frames:          # |B_{t-1}| == l_I case of Eq. 3
            U.append(B.pop(0))               # Eq. 5: U_t = [U_{t-1}, phi(X_{t-l_I}, ...)]
        while len(U) > past_frames:          # Eq. 6: FIFO along the sequence axis
            evicted_now.append(U.pop(0))
    return StepSchedule(t, list(B), list(U), evicted_now, tokens_per_frame, sink_tokens)


def ring_slots(frame: int, tokens_per_frame: int, instant_frames: int, past_frames: int) -> np.ndarray:
    """Contracted ring layout (reading Q17): token j of frame f
    lives in slot (f*tpf + j) mod R with R = (l_U + l_I + 1) * tpf."""
    R = (past_frames + instant_frames + 1) * tokens_per_frame
    return (frame * tokens_per_frame + np.arange(tokens_per_frame)) % R


# ---------------------------------------------------------------------------
# The two attentions of one step
# ---------------------------------------------------------------------------
FrameFn = Callable[[int], Tuple[np.ndarray, np.ndarray]]    # f -> (k [tpf,Hkv,d], v [tpf,Hkv,d])


def _cat(parts: Sequence[np.ndarray], hkv: int, d: int) -> np.ndarray:
    parts = [np.asarray(p, np.float64) for p in parts]
    if not parts:
        return np.zeros((0, hkv, d), np.float64)
    return np.concatenate(parts, axis=0)


def instant_cache_output(sched: StepSchedule, sink: Tuple[np.ndarray, np.ndarray], frame_kv: FrameFn,
                         q_inst: np.ndarray, theta: float, style: int = SPLIT_HALF) -> np.ndarray:
    """I_{t} = phi(B_t, C_a)  (Eq. 7): the instant tokens attend to the
    sink and to the buffer only -- never to U.

    Context [C_a | B_t] gets consecutive ids 0 .. A + C_t - 1; the
    query of instant token i is at id A + i and sees keys with id <= A + i.
    q_inst [C_t, Hq, d] -> O_inst [C_t, Hq, d].
    """
    sk, sv = sink
    hkv, d = sk.shape[1], sk.shape[2]
    ks = _cat([sk] + [frame_kv(f)[0] for f in sched.instant_frames], hkv, d)
    vs = _cat([sv] + [frame_kv(f)[1] for f in sched.instant_frames], hkv, d)
    A = sk.shape[0]
    pos_k = np.arange(ks.shape[0])
    pos_q = A + np.arange(q_inst.shape[0])
    return gqa_attention(np.asarray(q_inst, np.float64), pos_q, ks, vs, pos_k, theta, style)


def attend_output(sched: StepSchedule, sink: Tuple[np.ndarray, np.ndarray], frame_kv: FrameFn,
                  q: np.ndarray, k_self: np.ndarray, v_self: np.ndarray, theta: float,
                  style: int = SPLIT_HALF) -> np.ndarray:
    """Inference on C_{t} = [C_a, U_t, I_t] (Eq. 8) plus the query
    chunk's own K/V (used, then discarded: PAPER.md:212, 699).

    Keys in [sink | past | instant | self] order get ids 0..; the
    query tokens start at A + P_t + C_t (Eq. 2's l_A + l_W once the window is
    full, reading Q5) and are causal among themselves.
    q [nq, Hq, d], k_self/v_self [nq, Hkv, d] -> O [nq, Hq, d].
    """
    sk, sv = sink
    hkv, d = sk.shape[1], sk.shape[2]
    frames = list(sched.past_frames) + list(sched.instant_frames)
    ks = _cat([sk] + [frame_kv(f)[0] for f in frames] + [k_self], hkv, d)
    vs = _cat([sv] + [frame_kv(f)[1] for f in frames] + [v_self], hkv, d)
    L_ctx = ks.shape[0] - q.shape[0]
    pos_k = np.arange(ks.shape[0])
    pos_q = L_ctx + np.arange(q.shape[0])
    return gqa_attention(np.asarray(q, np.float64), pos_q, ks, vs, pos_k, theta, style)


def instant_cache_output_boosted(sched: StepSchedule, sink: Tuple[np.ndarray, np.ndarray], frame_kv: FrameFn,
                                 q_inst: np.ndarray, k_boost: np.ndarray, v_boost: np.ndarray, theta: float,
                                 style: int = SPLIT_HALF) -> np.ndarray:
    """I_t = phi(B_t, C_a) with the newest buffer input temporarily re-encoded at a higher
    resolution, "without modifying the buffer itself" (Table
    "spa" PAPER.md:719-749).  The context is [C_a | B_t minus its newest
    frame | re-encoded newest frame (n_boost tokens)] with consecutive ids 0..;
    query i sits at id A + i and sees ids <= A + i (Eq. 7 otherwise unchanged).
    q_inst [C_t - tpf + n_boost, Hq, d], k_boost/v_boost [n_boost, Hkv, d] -> same rows as q_inst."""
    sk, sv = sink
    hkv, d = sk.shape[1], sk.shape[2]
    older = list(sched.instant_frames)[:-1]
    ks = _cat([sk] + [frame_kv(f)[0] for f in older] + [k_boost], hkv, d)
    vs = _cat([sv] + [frame_kv(f)[1] for f in older] + [v_boost], hkv, d)
    A = sk.shape[0]
    pos_k = np.arange(ks.shape[0])
    pos_q = A + np.arange(q_inst.shape[0])
    return gqa_attention(np.asarray(q_inst, np.float64), pos_q, ks, vs, pos_k, theta, style)


def attend_output_boosted(sched: StepSchedule, sink: Tuple[np.ndarray, np.ndarray], frame_kv: FrameFn,
                          q: np.ndarray, k_self: np.ndarray, v_self: np.ndarray, k_boost: np.ndarray,
                          v_boost: np.ndarray, theta: float, style: int = SPLIT_HALF) -> np.ndarray:
    """Eq. 8 over [C_a, U_t, I_t] where I_t was built from the re-encoded
    newest frame (instant_cache_output_boosted): the instant segment holds the older instant
    frames and then the n_boost re-encoded tokens (reading Q22), followed by the
    query chunk; ids consecutive from 0, causal inside the chunk."""
    sk, sv = sink
    hkv, d = sk.shape[1], sk.shape[2]
    frames = list(sched.past_frames) + list(sched.instant_frames)[:-1]
    ks = _cat([sk] + [frame_kv(f)[0] for f in frames] + [k_boost, k_self], hkv, d)
    vs = _cat([sv] + [frame_kv(f)[1] for f in frames] + [v_boost, v_self], hkv, d)
    L_ctx = ks.shape[0] - q.shape[0]
    pos_k = np.arange(ks.shape[0])
    pos_q = L_ctx + np.arange(q.shape[0])
    return gqa_attention(np.asarray(q, np.float64), pos_q, ks, vs, pos_k, theta, style)


def instant_cache_output_ext(sched: StepSchedule, sink: Tuple[np.ndarray, np.ndarray], k_inst: np.ndarray,
                             v_inst: np.ndarray, q_inst: np.ndarray, theta: float, style: int = SPLIT_HALF) -> np.ndarray:
    """Eq. 7 in the real-model mode: I = phi(B_t, C_a) where the buffer tokens'
    K/V are the caller's (k_inst, v_inst [C_t, Hkv, d], the step's instant K/V).
    Context [C_a | instant tokens] with ids 0..; query i at A + i, causal."""
    sk, sv = sink
    hkv, d = sk.shape[1], sk.shape[2]
    ks = _cat([sk, k_inst], hkv, d)
    vs = _cat([sv, v_inst], hkv, d)
    pos_k = np.arange(ks.shape[0])
    pos_q = sk.shape[0] + np.arange(q_inst.shape[0])
    return gqa_attention(np.asarray(q_inst, np.float64), pos_q, ks, vs, pos_k, theta, style)


def attend_output_ext(sched: StepSchedule, sink: Tuple[np.ndarray, np.ndarray], past_kv: FrameFn,
                      k_inst: np.ndarray, v_inst: np.ndarray, q: np.ndarray, k_self: np.ndarray, v_self: np.ndarray,
                      theta: float, style: int = SPLIT_HALF) -> np.ndarray:
    """Eq. 8 in the real-model mode: C_t = [C_a, U_t, I_t] where U_t's frames
    carry the K/V of their Eq. 5 update (past_kv(f)) and I_t is the step's
    instant K/V (k_inst, v_inst) -- a frame in the instant window is NOT read from U.
    Plus the self segment's K/V (the query chunk, and while decoding the tokens generated so
    far: PAPER.md:128); q are its LAST q.shape[0] tokens; ids contiguous from 0, causal."""
    sk, sv = sink
    hkv, d = sk.shape[1], sk.shape[2]
    ks = _cat([sk] + [past_kv(f)[0] for f in sched.past_frames] + [k_inst, k_self], hkv, d)
    vs = _cat([sv] + [past_kv(f)[1] for f in sched.past_frames] + [v_inst, v_self], hkv, d)
    L_ctx = ks.shape[0] - q.shape[0]
    pos_k = np.arange(ks.shape[0])
    pos_q = L_ctx + np.arange(q.shape[0])
    return gqa_attention(np.asarray(q, np.float64), pos_q, ks, vs, pos_k, theta, style)


def instant_cache_output_approx(t_last: int, period: int, instant_frames: int, past_frames: int,
                                tokens_per_frame: int, sink: Tuple[np.ndarray, np.ndarray], frame_kv: FrameFn,
                                q_at: Callable[[int, int], np.ndarray], theta: float, style: int = SPLIT_HALF,
                                capture: Sequence[int] = ()):
    """Approximate instant cache ("an extra periodically refreshed cache for
    recent frames, enabling reuse of buffer-frame caches"; DESIGN.md reading
    Q23), replayed from step 0 to t_last in the paper's order:

    * step s is a refresh when s mod period == 0: every buffer frame's instant rows are
      rebuilt, i.e. Eq. 7 (instant_cache_output) at step s with the step's C_s queries;
    * otherwise only the newest frame's rows are computed -- the last tpf rows of Eq. 7 at
      step s (its tokens at ids A + C_s - tpf + j over [C_a | B_s]) -- and every other buffer
      frame keeps the rows it already had;
    * a frame leaving the buffer (Eq. 3) drops its rows.

    q_at(s, C_s) -> the C_s instant queries of step s, oldest first (a non-refresh step reads
    only its last tpf).  Returns {s: rows [C_s, Hq, d] of B_s, oldest frame first} for s in
    capture (default: t_last only)."""
    tpf = tokens_per_frame
    sk, sv = sink
    A = sk.shape[0]
    hkv, d = sk.shape[1], sk.shape[2]
    capture = set(capture) if capture else {t_last}
    rows = {}
    out = {}
    for s in range(t_last + 1):
        sch = schedule_fifo(s, instant_frames, past_frames, tpf, A)
        q = np.asarray(q_at(s, sch.C_t), np.float64)
        if s % period == 0:
            o = instant_cache_output(sch, sink, frame_kv, q, theta, style)
            for k, f in enumerate(sch.instant_frames):
                rows[f] = o[k * tpf:(k + 1) * tpf]
        else:
            ks = _cat([sk] + [frame_kv(f)[0] for f in sch.instant_frames], hkv, d)
            vs = _cat([sv] + [frame_kv(f)[1] for f in sch.instant_frames], hkv, d)
            pos_q = A + sch.C_t - tpf + np.arange(tpf)
            rows[s] = gqa_attention(q[sch.C_t - tpf:], pos_q, ks, vs, np.arange(ks.shape[0]), theta, style)
        for f in list(rows):
            if f not in sch.instant_frames:
                del rows[f]
        if s in capture:
            out[s] = np.concatenate([rows[f] for f in sch.instant_frames])
    return out


def decode_output(sched: StepSchedule, sink: Tuple[np.ndarray, np.ndarray], frame_kv: FrameFn,
                  q_last: np.ndarray, k_self: np.ndarray, v_self: np.ndarray, theta: float,
                  style: int = SPLIT_HALF) -> np.ndarray:
    """Decoding over C_{t+1}: the self segment (query chunk followed by the
    tokens generated so far; n_self tokens, used then discarded PAPER.md:212) extends the
    context [sink | past | instant] with consecutive ids; q_last are the
    queries of its last n_q tokens, causal.  q_last [n_q, Hq, d] -> [n_q, Hq, d]."""
    sk, sv = sink
    hkv, d = sk.shape[1], sk.shape[2]
    frames = list(sched.past_frames) + list(sched.instant_frames)
    ks = _cat([sk] + [frame_kv(f)[0] for f in frames] + [k_self], hkv, d)
    vs = _cat([sv] + [frame_kv(f)[1] for f in frames] + [v_self], hkv, d)
    pos_k = np.arange(ks.shape[0])
    pos_q = ks.shape[0] - q_last.shape[0] + np.arange(q_last.shape[0])
    return gqa_attention(np.asarray(q_last, np.float64), pos_q, ks, vs, pos_k, theta, style)


def decode_output_sampled(sched: StepSchedule, sink: Tuple[np.ndarray, np.ndarray], frame_kv: FrameFn,
                          q_last: np.ndarray, k_self: np.ndarray, v_self: np.ndarray, stride: int, theta: float,
                          style: int = SPLIT_HALF) -> np.ndarray:
    """Decoding over a sampled cumulative cache ("sample the cumulative KV cache
    at 0.5 FPS during decoding"; reading Q24): of U_t (oldest first) keep every
    stride-th frame counting back from the newest, then decode exactly as decode_output over
    [sink | kept past | instant | self] with ids consecutive from 0."""
    U = list(sched.past_frames)
    kept = U[::-1][::stride][::-1]
    sampled = StepSchedule(sched.t, list(sched.instant_frames), kept, list(sched.evicted), sched.tokens_per_frame,
                           sched.sink_tokens)
    return decode_output(sampled, sink, frame_kv, q_last, k_self, v_self, theta, style)


def cumulative_update_output(t: int, instant_frames: int, past_frames: int, active_frames: int,
                             sink: Tuple[np.ndarray, np.ndarray], frame_kv: FrameFn, q_upd: np.ndarray,
                             theta: float, tokens_per_frame: int, style: int = SPLIT_HALF) -> np.ndarray:
    """The attention inside phi(X_{t-l_I}, [C_a, zeta(U_{t-1})]) of Eq. 5.

    At step t the input X_{t-l_I} leaves the buffer (Eq. 3) and its tokens attend to the
    sink C_a, to zeta(U_{t-1}) -- "the most recent l_L KV caches" of the cumulative cache
    before this update (l_L = active_frames frames) -- and to themselves,
    causally.  Ids are consecutive from 0 over that active cache: sink
    0..A-1, zeta(U) from A, the frame's token i at A + |zeta(U)| + i.  Requires t >= l_I.
    q_upd [tpf, Hq, d] -> [tpf, Hq, d].
    """
    if t < instant_frames:
        raise ValueError("no input has left the buffer before step l_I")
    prev = schedule_fifo(t - 1, instant_frames, past_frames, tokens_per_frame, sink[0].shape[0]) if t >= 1 else None
    U_prev = list(prev.past_frames) if prev is not None else []
    zeta = U_prev[len(U_prev) - min(active_frames, len(U_prev)):] if active_frames > 0 else []
    e = t - instant_frames
    sk, sv = sink
    hkv, d = sk.shape[1], sk.shape[2]
    ks = _cat([sk] + [frame_kv(f)[0] for f in zeta] + [frame_kv(e)[0]], hkv, d)
    vs = _cat([sv] + [frame_kv(f)[1] for f in zeta] + [frame_kv(e)[1]], hkv, d)
    pos_k = np.arange(ks.shape[0])
    pos_q = ks.shape[0] - tokens_per_frame + np.arange(tokens_per_frame)
    return gqa_attention(np.asarray(q_upd, np.float64), pos_q, ks, vs, pos_k, theta, style)


def position_ids(sched: StepSchedule, n_query: int):
    """All ids one step applies: (build key ids, build query ids,
    attend key ids, attend query ids), as int64 arrays."""
    A, C, P = sched.sink_tokens, sched.C_t, sched.P_t
    build_k = np.arange(A + C)
    build_q = A + np.arange(C)
    attend_k = np.arange(A + P + C + n_query)
    attend_q = A + P + C + np.arange(n_query)
    return build_k, build_q, attend_k, attend_q
