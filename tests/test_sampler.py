"""The scene sampler / signal generator (SPEC.md:141-192 contract):
host fixture generator checks on CPU (the device mirror is checked bit for bit in
tests/test_gpu_sampler.py)."""
import math

import numpy as np
import pytest

from paper_1712_03439_b200 import roomsim as rs
from paper_1712_03439_b200 import scenes

SPEC_WEIGHTS = (0.15, 0.35, 0.30, 0.20)  # SPEC.md:151-158 defaults, mean 1.55


def spec4(**kw):
    return rs.sampler_spec(scenes.spec_config4(), **kw)


def fields(b):
    return (b.src_begin, b.room_dims, b.reflection, b.image_order, b.max_taps, b.src_pos, b.mic_pos,
            b.snr_db, b.sig_len)


def same(a, b):
    return all(np.array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8))
               for x, y in zip(fields(a), fields(b)))


def test_pure_function_of_seed_utterance_epoch():
    sp = spec4(weights=SPEC_WEIGHTS)
    a = rs.sample_batch(sp, 40, seed=9)
    b = rs.sample_batch(sp, 40, seed=9)
    assert same(a, b)
    # batch order / batch boundaries never matter
    c = rs.sample_batch(sp, 5, seed=9, first_utt=17)
    assert same(c, a.subset(range(17, 22)))
    # another epoch re-samples every utterance
    d = rs.sample_batch(sp, 100, seed=9, epoch=1)
    e = rs.sample_batch(sp, 100, seed=9, epoch=0)
    assert not np.any(np.all(d.room_dims == e.room_dims, axis=1))


def test_noise_count_mean():
    sp = spec4(weights=SPEC_WEIGHTS)
    n = np.zeros(100_000, np.int32)
    lib = rs.load_library()
    import ctypes as C
    rs._check(lib.rs_sampler_counts(C.byref(sp), 3, 0, n.size, 0, rs._ptr(n)))
    noises = n - 1
    assert set(np.unique(noises)) <= {0, 1, 2, 3}
    assert abs(noises.mean() - 1.55) <= 0.02


@pytest.mark.parametrize("mode", ["refl", "t60", "circle"])
def test_support(mode):
    base = scenes.spec_config4() if mode != "t60" else scenes.spec_config5()
    if mode == "circle":
        base = scenes.spec_config5()
        base.t60_range = None
    sp = rs.sampler_spec(base, weights=SPEC_WEIGHTS if mode == "refl" else None)
    b = rs.sample_batch(sp, 500, seed=21)
    lo, hi = np.array(base.dim_lo), np.array(base.dim_hi)
    assert (b.room_dims >= lo).all() and (b.room_dims <= hi).all()
    c = base.min_wall_clearance
    room_s = np.repeat(b.room_dims, np.diff(b.src_begin), axis=0)
    assert (b.src_pos >= c).all() and (b.src_pos <= room_s - c).all()
    room_m = np.repeat(b.room_dims, np.diff(b.mic_begin), axis=0)
    assert (b.mic_pos >= c - 1e-12).all() and (b.mic_pos <= room_m - c + 1e-12).all()
    V = np.prod(b.room_dims, axis=1)
    S = 2 * (b.room_dims[:, 0] * b.room_dims[:, 1] + b.room_dims[:, 0] * b.room_dims[:, 2]
             + b.room_dims[:, 1] * b.room_dims[:, 2])
    t60 = 0.161 * V / (-S * np.log(b.reflection ** 2))
    if mode == "t60":
        # r = exp(-0.0805 V / (S T60)) for T60 ~ U(t60_range): Eyring inverts it
        assert (t60 >= base.t60_range[0] - 1e-9).all() and (t60 <= base.t60_range[1] + 1e-9).all()
    else:
        lo_r, hi_r = base.refl_range
        assert (b.reflection >= lo_r).all() and (b.reflection <= hi_r).all()
        assert (t60 <= base.t60_max * (1 + 1e-12)).all()
    K = np.ceil(343.0 * t60 / np.linalg.norm(b.room_dims, axis=1))
    assert (np.abs(K - b.image_order) <= 1).all() and (K == b.image_order).mean() > 0.999
    horizon = np.ceil(t60 * 16000.0)
    assert (np.abs(horizon - b.max_taps) <= 1).all()
    secs = b.sig_len[b.src_begin[:-1]] / 16000.0
    assert (secs >= base.seconds_range[0] - 1e-4).all() and (secs <= base.seconds_range[1] + 1e-4).all()
    snr = np.delete(b.snr_db, b.src_begin[:-1])
    assert (snr >= base.snr_range_db[0]).all() and (snr <= base.snr_range_db[1]).all()
    if mode == "circle":  # 8 mics on a 5 cm circle around a common centre
        m = b.mic_pos.reshape(b.n_utt, base.mic_count, 3)
        ctr = m.mean(axis=1, keepdims=True)
        np.testing.assert_allclose(np.linalg.norm(m - ctr, axis=2), base.mic_radius, rtol=1e-9)


def test_signals_moments_and_determinism():
    sp = spec4()
    b = rs.sample_batch(sp, 6, seed=4)
    x = rs.generate_signals(sp, b, seed=4)
    assert x.dtype == np.float32 and x.size == b.total_samples
    assert abs(float(x.mean())) < 1e-3 and abs(float(x.std()) - 0.1) < 1e-3
    k = float(((x.astype(np.float64) / x.std()) ** 4).mean())
    assert abs(k - 3.0) < 0.05  # Gaussian kurtosis
    assert np.array_equal(x, rs.generate_signals(sp, b, seed=4))
    from scipy import stats

    ks = stats.kstest(x[:1_000_000].astype(np.float64) / 0.1, "norm")
    assert ks.statistic < 1.95 / math.sqrt(1_000_000)  # KS at the 0.1% level
    # one source's samples do not depend on the batch it is generated in
    c = b.subset([3])
    y = rs.generate_signals(sp, c, seed=4, first_utt=3)
    s0 = int(b.src_begin[3])
    o, n = int(b.sig_off[s0]), int(b.sig_len[s0])
    assert np.array_equal(y[:n], x[o:o + n])


def test_spec_errors():
    base = scenes.spec_config4()
    base.dim_lo = (0.8, 3.0, 2.5)  # 0.8 m cannot hold 0.5 m clearance on both sides
    with pytest.raises(rs.ConfigError):
        rs.sample_batch(rs.sampler_spec(base), 2, seed=1)
    with pytest.raises(rs.ConfigError):
        rs.sample_batch(spec4(weights=[0.0, 0.0]), 2, seed=1)
