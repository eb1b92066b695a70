"""Renders one workload in a fresh process and saves what it produced (GPU tests).

The library reads its tuning overrides (RSG_CHUNK_PAIRS, RSG_IP, ...) once per
process, so tests that compare renders under different overrides run each one
through this script:

    python tests/render_worker.py <config> <n_utt> <seed> <host|device> <out.npz> [utt,utt,...]

The optional last argument renders only those utterances of the config batch
(``SceneBatch.subset``: same scenes, same signals).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    cfg, n_utt, seed, mode, path = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], sys.argv[5]
    from paper_1712_03439_b200 import roomsim as rs, scenes

    b = scenes.CONFIGS[cfg](n_utt=n_utt, seed=seed)
    if len(sys.argv) > 6:
        b = b.subset([int(u) for u in sys.argv[6].split(",")])
    ctx = rs.Context(0)
    if mode == "host":
        r = rs.render_batch(b, ctx=ctx)
        out = r.out
    else:
        import torch

        sig = torch.from_numpy(b.signals).cuda()
        dout = torch.zeros(max(b.out_total, 1), dtype=torch.float32, device="cuda")
        r = rs.render_batch(b, ctx=ctx, device_signals_ptr=sig.data_ptr(), device_out_ptr=dout.data_ptr())
        torch.cuda.synchronize()
        out = dout.cpu().numpy()[: b.out_total]
    np.savez(path, out=out.view(np.uint32), out_len=r.out_len, gains=r.gains, power=r.power,
             layout=r.layout.view(np.uint8), mix_counts=np.array(ctx.mix_counts(), dtype=np.int64))
    ctx.close()


if __name__ == "__main__":
    main()
