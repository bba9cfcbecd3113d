"""Which (kv head, m-block) rows of the c2 attend are wrong (debug of the per-CTA work lists)."""
import numpy as np
import torch
import dscache_synth as synth
from oracle import dscache_oracle as O
from oracle.workload import StreamInputs, step_schedule
from tests.gpu_harness import run_stream

cfg = synth.CONFIGS["c2"]
t = 40
res = run_stream(cfg, [t], [(0, 0)])
g_inst, g_o = res[t][(0, 0)]
inp = StreamInputs(cfg, 0, 0)
q, ks, vs = inp.query(t)
ref = O.attend_output(step_schedule(cfg, t), inp.sink(), inp.frame_kv, q, ks, vs, cfg.rope_theta)
g = g_o.float().numpy()
grp = cfg.num_q_heads // cfg.num_kv_heads
err = np.abs(g - ref).max(axis=2)          # [n_q, Hq]
for kv in range(cfg.num_kv_heads):
    for mb in range(2):
        rows = [(i, kv * grp + j) for i in range(cfg.query_tokens) for j in range(grp)]
        rows = rows[mb * 256:(mb + 1) * 256]
        e = max(err[i, h] for i, h in rows) if rows else 0
        print(f"kv {kv} mb {mb}: max abs {e:.3e}")
