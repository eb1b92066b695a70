"""One small invocation of every device kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck) under each K4 variant selected by the environment
(RSG_OLA2, RSG_IP + RSG_IP_FORCE, RSG_LARGE_MIN, ...):

    compute-sanitizer --tool memcheck python tools/sanitize_case.py

K1 (both launch classes), K2, K3, K4, gains + mix (host and device buffers), the FFT seam,
the FP64 direct convolution, the signal generator (plan and one-shot) and the log-Mel
kernel.  Prints one line; exits nonzero on a library error.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_1712_03439_b200 import roomsim as rs, scenes

    ctx = rs.Context(0)
    b = scenes.config3(n_utt=3, seed=5)
    r = rs.render_batch(b, ctx=ctx)  # host buffers
    sig = torch.from_numpy(b.signals).cuda()
    out = torch.zeros(b.out_total, dtype=torch.float32, device="cuda")
    rs.render_batch(b, ctx=ctx, device_signals_ptr=sig.data_ptr(), device_out_ptr=out.data_ptr())
    b5 = scenes.config5(n_utt=1, seed=6)
    b5.max_taps[:] = 4000  # short RIRs, still N = 32768 forced
    rs.render_batch(b5, ctx=ctx)
    rng = np.random.default_rng(3)
    for n in (8, 256, 4096, 65536):
        x, h = rng.standard_normal(3 * n + 5), rng.standard_normal(max(1, n // 2 - 1))
        rs.convolve_ola(x, h, n, ctx=ctx)
        rs.CudaRealFft(n, ctx=ctx).forward(x[:n])
    rs.convolve_direct(rng.standard_normal(700), rng.standard_normal(90), ctx=ctx)
    sp = rs.sampler_spec(scenes.spec_config4(4))
    bb = rs.sample_batch(sp, 4, seed=4)
    dev = torch.empty(bb.total_samples, dtype=torch.float32, device="cuda")
    rs.generate_signals(sp, bb, seed=4, device_ptr=dev.data_ptr())
    plan = rs.SignalPlan(sp, bb, seed=4)
    plan.generate(dev.data_ptr(), epoch=1)
    torch.cuda.synchronize()
    J = np.diff(b.mic_begin)
    ch_off = np.concatenate([b.out_off[u] + np.arange(J[u]) * b.out_stride[u] for u in range(b.n_utt)])
    ch_len = np.repeat(r.out_len, J)
    S = np.array([rs.logmel_shape(int(n))[1] for n in ch_len], np.int64)
    f_off = np.concatenate([[0], np.cumsum(S * 512)[:-1]]).astype(np.int64)
    feat = torch.empty(max(int(S.sum()) * 512, 1), dtype=torch.float32, device="cuda")
    rs.logmel_device(out.data_ptr(), ch_off, ch_len, feat.data_ptr(), f_off, ctx=ctx)
    torch.cuda.synchronize()
    ctx.close()
    print("sanitize case ok:", {k: v for k, v in os.environ.items() if k.startswith("RSG_")})


if __name__ == "__main__":
    main()
