"""On-device scene sampling and signal generation == the host fixture generator, bit for
bit, and a render fed by device-generated signals."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SPEC_WEIGHTS = (0.15, 0.35, 0.30, 0.20)


def _dev(a, torch):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("cfg,weights", [("config4", SPEC_WEIGHTS), ("config5", None), ("config2", None)])
def test_device_scenes_equal_host(rs, cfg, weights):
    import torch
    from paper_1712_03439_b200 import scenes

    spec = getattr(scenes, "spec_" + cfg)()
    sp = rs.sampler_spec(spec, weights=weights)
    n = 1000
    host = rs.sample_batch(sp, n, seed=77, first_utt=5, epoch=2)
    L = rs.load_library()
    I_d = torch.zeros(n, dtype=torch.int32, device="cuda")
    rs._check(L.rs_sampler_counts_device(C.byref(sp), 77, 5, n, 2, I_d.data_ptr(), None))
    I_h = np.diff(host.src_begin).astype(np.int32)
    assert np.array_equal(I_d.cpu().numpy(), I_h)
    sb = _dev(host.src_begin, torch)
    J = sp.mic_count
    outs = dict(room=torch.zeros(n, 3, dtype=torch.float64, device="cuda"),
                refl=torch.zeros(n, dtype=torch.float64, device="cuda"),
                order=torch.zeros(n, dtype=torch.int32, device="cuda"),
                taps=torch.zeros(n, dtype=torch.int64, device="cuda"),
                src=torch.zeros(host.n_src, 3, dtype=torch.float64, device="cuda"),
                mic=torch.zeros(n * J, 3, dtype=torch.float64, device="cuda"),
                snr=torch.zeros(host.n_src, dtype=torch.float64, device="cuda"),
                nx=torch.zeros(n, dtype=torch.int64, device="cuda"))
    rs._check(L.rs_sample_scenes_device(C.byref(sp), 77, 5, n, 2, sb.data_ptr(),
                                        *[t.data_ptr() for t in outs.values()], None))
    torch.cuda.synchronize()
    want = [host.room_dims, host.reflection, host.image_order, host.max_taps, host.src_pos, host.mic_pos,
            host.snr_db, host.sig_len[host.src_begin[:-1]]]
    for (k, got), w in zip(outs.items(), want):
        g = got.cpu().numpy()
        assert np.array_equal(g.view(np.uint8), np.ascontiguousarray(w, g.dtype).view(np.uint8)), k


def test_device_signals_equal_host(rs):
    import torch
    from paper_1712_03439_b200 import scenes

    sp = rs.sampler_spec(scenes.spec_config4())
    b = rs.sample_batch(sp, 12, seed=8, first_utt=100)
    host = rs.generate_signals(sp, b, seed=8, first_utt=100)
    dev = torch.zeros(b.total_samples, dtype=torch.float32, device="cuda")
    rs.generate_signals(sp, b, seed=8, first_utt=100, device_ptr=dev.data_ptr())
    torch.cuda.synchronize()
    assert np.array_equal(dev.cpu().numpy().view(np.uint32), host.view(np.uint32))


def test_render_from_device_generated_signals(rs, ctx, port):
    """Epoch loop: scenes sampled, signals generated in HBM, rendered there — equal to the
    host-generated fixture rendered by the oracle."""
    import torch
    from paper_1712_03439_b200 import scenes

    sp = rs.sampler_spec(scenes.spec_config4(), weights=SPEC_WEIGHTS)
    b = rs.sample_batch(sp, 3, seed=12, eta_db=20.0, plan_rule=scenes.PLAN_POW2_TWICE)
    sig = torch.zeros(b.total_samples, dtype=torch.float32, device="cuda")
    rs.generate_signals(sp, b, seed=12, device_ptr=sig.data_ptr())
    out = torch.zeros(b.out_total, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    g = rs.render_batch(b, ctx=ctx, device_signals_ptr=sig.data_ptr(), device_out_ptr=out.data_ptr())
    b.signals = rs.generate_signals(sp, b, seed=12)
    o_out, o_len, o_lay, o_gain, o_pow = port.render_batch(b, threads=8)
    assert (g.out_len == o_len).all()
    np.testing.assert_allclose(g.gains, o_gain, rtol=1e-5)
    go = out.cpu().numpy()
    for u in range(b.n_utt):
        for j in range(int(b.mic_begin[u + 1] - b.mic_begin[u])):
            a = b.channel(go, u, j, o_len[u])
            w = b.channel(o_out, u, j, o_len[u])
            assert np.abs(a - w).max() <= 1e-5 * np.abs(w).max()


def test_signal_plan_epochs_and_subsets(rs):
    """rs_signal_plan (the table built once, one launch per epoch) equals the host generator
    for several epochs, on a full batch and on a non-contiguous subset (shards keep their
    utterance ids), including sources whose length is not a multiple of 4 (tail quads)."""
    import torch
    from paper_1712_03439_b200 import scenes

    sp = rs.sampler_spec(scenes.spec_config4())
    b = rs.sample_batch(sp, 40, seed=21, first_utt=7)
    b.sig_len = b.sig_len.copy()
    b.sig_len[::3] -= np.arange(b.sig_len[::3].size) % 4  # ragged tails
    b.sig_off = scenes.signal_offsets(b.sig_len)
    sub = b.subset([3, 11, 12, 30, 39])
    for batch in (b, sub):
        plan = rs.SignalPlan(sp, batch, seed=21)
        dev = torch.full((batch.total_samples,), float("nan"), dtype=torch.float32, device="cuda")
        for ep in (0, 3):
            plan.generate(dev.data_ptr(), epoch=ep)
            torch.cuda.synchronize()
            host = rs.generate_signals(sp, batch, seed=21, epoch=ep)
            d = dev.cpu().numpy()
            for o, n in zip(batch.sig_off, batch.sig_len):
                assert np.array_equal(d[o:o + n].view(np.uint32), host[o:o + n].view(np.uint32))
        plan.close()
    # the subset's samples are the full batch's (keyed by the global utterance ids)
    full = rs.generate_signals(sp, b, seed=21)
    part = rs.generate_signals(sp, sub, seed=21)
    for k, u in enumerate([3, 11, 12, 30, 39]):
        s_full, s_sub = b.src_begin[u], sub.src_begin[k]
        n = int(b.sig_len[s_full])
        assert np.array_equal(full[b.sig_off[s_full]:b.sig_off[s_full] + n],
                              part[sub.sig_off[s_sub]:sub.sig_off[s_sub] + n])


def test_k4_breakdown_rows(rs):
    """Profiling level 2: per-(N, variant) rows whose flops sum to the render's K4 flops."""
    from paper_1712_03439_b200 import scenes

    c = rs.Context(0)
    b = scenes.config3(n_utt=6, seed=55)
    c.set_profiling(2)
    rs.render_batch(b, ctx=c)
    rows = c.k4_breakdown()
    t = c.last_timing()
    assert rows and sum(r["pairs"] for r in rows) == b.n_pairs
    assert abs(sum(r["flops"] for r in rows) - t["ola_flops"]) <= 1e-6 * t["ola_flops"]
    assert all(r["ms"] > 0 for r in rows)
    c.close()
