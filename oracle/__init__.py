"""fp64 CPU oracle for the DSCache hot path -- TEST INFRASTRUCTURE ONLY.

Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  See dscache_oracle.py's header.
"""
from .dscache_oracle import *  # noqa: F401,F403
from .dscache_oracle import (SPLIT_HALF, ADJACENT, StepSchedule, rope, rope_frequencies,  # noqa: F401
                             softmax_attention, gqa_attention, schedule_fifo, ring_slots,
                             instant_cache_output, attend_output, position_ids,
                             cumulative_update_output, decode_output)
