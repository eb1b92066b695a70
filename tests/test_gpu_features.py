"""log-Mel front end (features.cu) against the numpy restatement oracle/logmel.py."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(rs, ctx, chans):
    import torch

    lens = np.array([c.size for c in chans], np.int64)
    offs = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int64)
    S = np.array([rs.logmel_shape(n)[1] for n in lens], np.int64)
    foff = np.concatenate([[0], np.cumsum(S * 512)[:-1]]).astype(np.int64)
    wave = torch.from_numpy(np.concatenate(chans).astype(np.float32)).cuda()
    feat = torch.full((max(int(S.sum()) * 512, 1),), float("nan"), dtype=torch.float32, device="cuda")
    rs.logmel_device(wave.data_ptr(), offs, lens, feat.data_ptr(), foff, ctx=ctx)
    f = feat.cpu().numpy()
    return [f[o:o + s * 512].reshape(s, 512) for o, s in zip(foff, S)]


def _check(got, want):
    assert got.shape == want.shape
    if got.size == 0:
        return
    assert np.isfinite(got).all()
    live = want > np.log(1e-6)  # filters with energy: log agreement
    assert np.abs(got - want)[live].max() <= 2e-3
    dead = want <= np.log(1e-8)  # empty filters sit on the floor
    if dead.any():
        assert np.abs(got - want)[dead].max() <= 1.0


def test_logmel_random_channels(rs, ctx):
    from oracle import logmel as L

    rng = np.random.default_rng(3)
    chans = [rng.standard_normal(n) * 0.1 for n in (512, 511, 1000, 16000, 48017, 160 * 9 + 512)]
    chans.append(np.sin(2 * np.pi * 1000.0 * np.arange(16000) / 16000.0))  # a 1 kHz tone
    for g, x in zip(_run(rs, ctx, chans), chans):
        _check(g, L.logmel(x.astype(np.float32)))


def test_logmel_of_a_render(rs, ctx, port):
    from oracle import logmel as L
    from paper_1712_03439_b200 import scenes

    b = scenes.config3(n_utt=2, seed=41)
    g = rs.render_batch(b, ctx=ctx)
    chans = [b.channel(g.out, u, j, g.out_len[u]).copy() for u in range(b.n_utt) for j in range(2)]
    for got, x in zip(_run(rs, ctx, chans), chans):
        _check(got, L.logmel(x))
    assert rs.logmel_shape(100)[1] == 0 and rs.logmel_shape(512 + 3 * 160)[1] == 1


def test_render_to_wav_roundtrip(rs, ctx, tmp_path):
    from paper_1712_03439_b200 import audio_io as aio
    from paper_1712_03439_b200 import scenes

    b = scenes.config3(n_utt=2, seed=43)
    g = rs.render_batch(b, ctx=ctx)
    paths = aio.write_render(b, g, str(tmp_path / "utt"), "float32")
    for u, p in enumerate(paths):
        x, fs = aio.read_wav(p, expect_rate=16000)
        assert x.shape == (2, g.out_len[u])
        for j in range(2):
            assert np.array_equal(x[j].astype(np.float32), b.channel(g.out, u, j, g.out_len[u]))


def test_fused_mix_logmel_matches_separate(rs, ctx):
    """rs_render_features_device (log-Mel fused into the mix) gives the same waveforms and
    bit-identical features as the render followed by rs_logmel_device — and without an
    output buffer the waveforms are never written."""
    import torch

    from paper_1712_03439_b200 import scenes

    b = scenes.config4(n_utt=6, seed=47)
    sig = torch.from_numpy(b.signals).cuda()
    out = torch.zeros(b.out_total, dtype=torch.float32, device="cuda")
    r = rs.render_batch(b, ctx=ctx, device_signals_ptr=sig.data_ptr(), device_out_ptr=out.data_ptr())
    foff, ftot = rs.feature_layout(b)
    J = np.diff(b.mic_begin)
    ch_off = np.concatenate([b.out_off[u] + np.arange(J[u]) * b.out_stride[u] for u in range(b.n_utt)])
    ch_len = np.repeat(r.out_len, J)
    sep = torch.full((max(ftot, 1),), float("nan"), dtype=torch.float32, device="cuda")
    rs.logmel_device(out.data_ptr(), ch_off, ch_len, sep.data_ptr(), foff, ctx=ctx)
    out2 = torch.full((b.out_total,), float("nan"), dtype=torch.float32, device="cuda")
    fused = torch.full((max(ftot, 1),), float("nan"), dtype=torch.float32, device="cuda")
    r2 = rs.render_features(b, device_signals_ptr=sig.data_ptr(), feat_ptr=fused.data_ptr(), feat_off=foff,
                            device_out_ptr=out2.data_ptr(), ctx=ctx)
    fused_only = torch.full((max(ftot, 1),), float("nan"), dtype=torch.float32, device="cuda")
    rs.render_features(b, device_signals_ptr=sig.data_ptr(), feat_ptr=fused_only.data_ptr(), feat_off=foff, ctx=ctx)
    torch.cuda.synchronize()
    assert (r2.out_len == r.out_len).all() and (r2.gains == r.gains).all()
    assert (out2.cpu().numpy().view(np.uint32) == out.cpu().numpy().view(np.uint32)).all()
    S = np.array([rs.logmel_shape(int(n))[1] for n in ch_len], np.int64)
    a, c, d = sep.cpu().numpy(), fused.cpu().numpy(), fused_only.cpu().numpy()
    for o, s_ in zip(foff, S):
        seg = slice(o, o + s_ * 512)
        assert np.isfinite(a[seg]).all()
        assert (a[seg].view(np.uint32) == c[seg].view(np.uint32)).all()
        assert (a[seg].view(np.uint32) == d[seg].view(np.uint32)).all()
