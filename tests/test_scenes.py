"""Seeded scene sampler (SPEC.md:141-192 contract; fixture generator)."""
import numpy as np

from paper_1712_03439_b200 import scenes


def test_determinism_and_epochs():
    spec = scenes.spec_config2(seed=3)
    a = scenes.sample_scene(spec, 17, epoch=1)
    b = scenes.sample_scene(spec, 17, epoch=1)
    assert (a.room == b.room).all() and (a.src == b.src).all() and a.n_samples == b.n_samples
    diff = sum(not np.array_equal(scenes.sample_scene(spec, u, 1).room, scenes.sample_scene(spec, u, 2).room)
               for u in range(100))
    assert diff == 100


def test_support_and_clearance():
    for spec in (scenes.spec_config2(), scenes.spec_config4(), scenes.spec_config5()):
        for u in range(200):
            s = scenes.sample_scene(spec, u)
            c = spec.min_wall_clearance
            assert (s.src >= c - 1e-12).all() and (s.src <= s.room - c + 1e-12).all()
            assert (s.mic >= c - 1e-12).all() and (s.mic <= s.room - c + 1e-12).all()
            if spec.t60_range is None:
                assert s.t60 <= spec.t60_max
                assert spec.refl_range[0] <= s.refl <= spec.refl_range[1]
            else:
                assert spec.t60_range[0] <= s.t60 <= spec.t60_range[1]
            assert s.order == int(np.ceil(343.0 * s.t60 / np.linalg.norm(s.room)))
            assert s.horizon == int(np.ceil(s.t60 * 16000))


def test_mic_geometry():
    s = scenes.sample_scene(scenes.spec_config2(), 5)
    assert abs(np.linalg.norm(s.mic[0] - s.mic[1]) - 0.071) < 1e-12
    s = scenes.sample_scene(scenes.spec_config5(), 5)
    c = s.mic.mean(0)
    assert np.allclose(np.linalg.norm(s.mic - c, axis=1), 0.05)


def test_batch_layout_and_subset():
    b = scenes.config3(n_utt=5, seed=9)
    assert b.n_pairs == int((np.diff(b.src_begin) * np.diff(b.mic_begin)).sum())
    assert b.total_samples == b.signals.size
    s = b.subset([3, 1])
    assert s.n_utt == 2 and (s.room_dims[0] == b.room_dims[3]).all()
    o = b.sig_off[b.src_begin[3]]
    assert (s.signals[: s.sig_len[0]] == b.signals[o: o + s.sig_len[0]]).all()
    assert (b.out_off[1:] == np.cumsum(b.out_stride * np.diff(b.mic_begin))[:-1]).all()
