import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import dscache_synth as synth
from oracle import dscache_oracle as O
from oracle.workload import StreamInputs
from tests.gpu_harness import run_stream, errors
from paper_2605_01858_b200 import dscache as D
cfg = synth.CONFIGS["c2"].replace(instant_frames=0, tokens_per_frame=128, past_frames=6, num_frames=12)
for impl in (D.IMPL_AUTO, D.IMPL_SIMT):
    steps = [2, 5, 6, 7, 8, 11]
    res = run_stream(cfg, steps, [(0, 0)], update_lL=6, impl=impl)
    for t in steps:
        inp = StreamInputs(cfg, 0, 0)
        qu = synth.update_q(cfg, 0, 0, t).double().numpy()
        ref = O.cumulative_update_output(t, 0, 6, 6, inp.sink(), inp.frame_kv, qu, cfg.rope_theta, 128)
        g = res["upd"][t][(0, 0)]
        print(impl, t, "rel", errors(g, ref)[1], "row errs (first tokens):", [round(errors(g[i:i+1], ref[i:i+1])[1], 3) for i in (0, 1, 64, 127)])
