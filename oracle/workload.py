"""Drive the oracle on a BASELINE.json workload -- TEST INFRASTRUCTURE ONLY.

Draws inputs from ``dscache_synth`` (the shared seeded generator), widens them
to float64 (reading Q15: the oracle consumes the *rounded* inputs), and calls
the step functions of ``dscache_oracle``.  Random access to any step t: the
schedule is replayed from Eq. 3/5/6 and only the frames in the window are drawn.
"""
from __future__ import annotations

from functools import lru_cache

import numpy as np

import dscache_synth as synth
from .dscache_oracle import (SPLIT_HALF, attend_output, instant_cache_output, ring_slots,
                             schedule_fifo, StepSchedule)


def f64(x) -> np.ndarray:
    return x.double().numpy()


def step_schedule(cfg, t: int) -> StepSchedule:
    return schedule_fifo(t, cfg.instant_frames, cfg.past_frames, cfg.tokens_per_frame, cfg.sink_tokens)


class StreamInputs:
    """Seeded inputs of one (stream, layer) of a config, as fp64 numpy arrays."""

    def __init__(self, cfg, stream: int, layer: int):
        self.cfg, self.stream, self.layer = cfg, stream, layer
        self.frame_kv = lru_cache(maxsize=512)(self._frame_kv)

    def sink(self):
        k, v = synth.sink_kv(self.cfg, self.stream, self.layer)
        return f64(k), f64(v)

    def _frame_kv(self, f: int):
        k, v = synth.frame_kv(self.cfg, self.stream, self.layer, f)
        return f64(k), f64(v)

    def instant_q(self, t: int, n: int):
        return f64(synth.instant_q(self.cfg, self.stream, self.layer, t, n))

    def query(self, t: int, n_q=None):
        return tuple(f64(x) for x in synth.query_qkv(self.cfg, self.stream, self.layer, t, n_q))


def oracle_step(cfg, stream: int, layer: int, t: int, inputs: StreamInputs | None = None,
                style: int = SPLIT_HALF, n_q=None):
    """(schedule, O_inst [C_t,Hq,d], O [q,Hq,d]) at step t for one (stream, layer)."""
    inp = inputs or StreamInputs(cfg, stream, layer)
    sch = step_schedule(cfg, t)
    sink = inp.sink()
    o_inst = instant_cache_output(sch, sink, inp.frame_kv, inp.instant_q(t, sch.C_t), cfg.rope_theta, style)
    q, ks, vs = inp.query(t, n_q)
    o = attend_output(sch, sink, inp.frame_kv, q, ks, vs, cfg.rope_theta, style)
    return sch, o_inst, o


def expected_ring(cfg, sched: StepSchedule, inputs: StreamInputs):
    """{slot -> (k [Hkv,d], v [Hkv,d])} for every token held in the window at the
    schedule's step (past + instant frames), per the contracted slot map."""
    out = {}
    for f in list(sched.past_frames) + list(sched.instant_frames):
        k, v = inputs.frame_kv(f)
        for j, s in enumerate(ring_slots(f, cfg.tokens_per_frame, cfg.instant_frames, cfg.past_frames)):
            out[int(s)] = (k[j], v[j])
    return out
