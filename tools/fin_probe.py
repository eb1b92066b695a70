"""Times K4 (+ the mix) of tiny renders: how long one CTA takes to mix a channel (mixfin.cuh).
usage: [RSG_FUSED_MIX=0] python tools/fin_probe.py [n_utt]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1712_03439_b200 import roomsim as rs, scenes

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1
ctx = rs.Context(0)
ctx.set_profiling(True)
for seed in ([int(a) for a in sys.argv[2].split(",")] if len(sys.argv) > 2 else (1, 2, 3)):
    b = scenes.config4(n_utt=n, seed=seed)
    sig = torch.from_numpy(b.signals).cuda()
    dout = torch.zeros(max(b.out_total, 1), dtype=torch.float32, device="cuda")
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = rs.render_batch(b, ctx=ctx, device_signals_ptr=sig.data_ptr(), device_out_ptr=dout.data_ptr())
        e1.record()
        torch.cuda.synchronize()
    st = ctx.stage_times()
    print(f"seed {seed}: {b.n_pairs} pairs, samples/channel {int(r.out_len.mean())}, render {e0.elapsed_time(e1):.3f} ms, "
          f"ola {st['ola']:.3f} ms, gain_mix {st['gain_mix']:.3f} ms, fused {ctx.mix_counts()}")
