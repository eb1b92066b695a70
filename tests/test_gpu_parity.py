"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Bars (BASELINE.json north_star):
  * RIR taps (FP64), cut indices, truncated lengths, N / L / B: bit-exact;
  * waveforms: max|gpu - oracle| <= 1e-5 * peak|oracle| per utterance (FP32);
  * achieved SNR within 1e-6 dB.
"""
import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

WAVE_TOL = 1e-5  # relative to each utterance's peak, written per north_star


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def rel_err(got, want):
    return np.abs(np.asarray(got, np.float64) - want).max() / max(np.abs(want).max(), 1e-300)


# ---- K1 / K2 ------------------------------------------------------------------------
def test_rir_single_tap(rs, ctx):
    h = rs.synthesize_rir([5, 5, 5], 0.5, 0, [1, 1, 1], [2, 1, 1], ctx=ctx)
    assert h.size == 48 and h[47] == 1.0 and not h[:47].any()


def test_rir_bitexact_random(rs, ctx, port):
    rng = np.random.default_rng(10)
    for t in range(60):
        room = rng.uniform([3, 3, 2.5], [10, 8, 6])
        src, mic = rng.uniform(0.5, room - 0.5), rng.uniform(0.5, room - 0.5)
        k, r = int(rng.integers(0, 18)), rng.uniform(0.2, 0.95)
        mt = int(rng.choice([0, 700, 4000, 20000]))
        want = port.synthesize_rir(room, r, k, src, mic, max_taps=mt)
        got = rs.synthesize_rir(room, r, k, src, mic, max_taps=mt, ctx=ctx)
        assert got.size == want.size, t
        assert (bits(got) == bits(want)).all(), t


def test_rir_bitexact_long_sliced(rs, ctx, port):
    # K large enough that the RIR exceeds one K1 slice (12288 bins)
    room, src, mic = [10.0, 8.0, 6.0], [1.1, 2.0, 1.3], [2.9, 1.0, 1.7]
    want = port.synthesize_rir(room, 0.9, 30, src, mic, max_taps=30000)
    got = rs.synthesize_rir(room, 0.9, 30, src, mic, max_taps=30000, ctx=ctx)
    assert want.size > 12288 and (bits(got) == bits(want)).all()


def test_truncate_bitexact(rs, ctx, port):
    rng = np.random.default_rng(11)
    for _ in range(50):
        n = int(rng.integers(1, 20000))
        h = rng.random(n) * np.exp(-rng.random() * 12 * np.linspace(0, 1, n))
        for eta in (5.0, 20.0, 60.0):
            a = port.truncate_rir(h, eta)
            b = rs.truncate_rir(h, eta, ctx=ctx)
            assert (a[1], a[0].size, a[2]) == (b[1], b[0].size, b[2])
    t, nc, _ = rs.truncate_rir(0.9 ** np.arange(60), 20, ctx=ctx)
    assert nc == 21


def test_errors(rs, ctx):
    with pytest.raises(rs.PlacementError):
        rs.synthesize_rir([5, 5, 5], 0.5, 2, [0, 1, 1], [2, 2, 2], ctx=ctx)
    with pytest.raises(rs.ConfigError):
        rs.synthesize_rir([5, 5, 5], 1.5, 2, [1, 1, 1], [2, 2, 2], ctx=ctx)
    with pytest.raises(rs.GeometryError):
        rs.synthesize_rir([5, 5, 5], 0.5, 0, [1, 1, 1], [1, 1, 1], ctx=ctx)
    with pytest.raises(rs.PlanError):
        rs.convolve_ola(np.ones(10), np.ones(8), 4, ctx=ctx)
    with pytest.raises(rs.DegenerateInputError):
        rs.convolve_ola(np.ones(0), np.ones(8), 16, ctx=ctx)
    with pytest.raises(rs.DegenerateInputError):
        rs.truncate_rir(np.zeros(10), 20, ctx=ctx)


# ---- FFT seam ---------------------------------------------------------------------
@pytest.mark.parametrize("n", [2 ** k for k in range(1, 16)] + [2 ** 16, 2 ** 18, 2 ** 20])
def test_rfft_engine(rs, ctx, port, n):
    rng = np.random.default_rng(n)
    eng = rs.CudaRealFft(n, ctx=ctx)
    assert eng.spectrum_size() == n // 2 + 1
    x = rng.standard_normal((3, n))
    got = eng.forward(x)
    for i in range(3):
        want = port.rfft_forward(x[i])
        assert np.abs(got[i] - want).max() <= 1e-5 * np.abs(want).max() + 1e-6
    back = eng.inverse(got)
    assert np.abs(back - x).max() <= 1e-5 * np.abs(x).max()
    for i in range(3):
        want = port.rfft_inverse(got[i], n)
        assert np.abs(back[i] - want).max() <= 1e-5 * np.abs(want).max()


# ---- K3 + K4 single pair ----------------------------------------------------------------
def test_convolve_kats(rs, ctx):
    np.testing.assert_allclose(rs.convolve_ola([1, 2, 3], [1], 2, ctx=ctx), [1, 2, 3], atol=1e-6)
    np.testing.assert_allclose(rs.convolve_ola([1, 1], [1, 1], 2, ctx=ctx), [1, 2, 1], atol=1e-6)
    np.testing.assert_allclose(rs.convolve_ola([2, 0, -1], [0.5, 0.25], 4, ctx=ctx),
                               [1, 0.5, -0.5, -0.25], atol=1e-6)
    np.testing.assert_allclose(rs.convolve_full_fft([1, 2, 3], [1], ctx=ctx), [1, 2, 3], atol=1e-6)
    assert np.abs(rs.convolve_ola(np.zeros(50), np.ones(5), 8, ctx=ctx)).max() == 0


def test_convolve_random_vs_oracle(rs, ctx, port):
    rng = np.random.default_rng(12)
    for _ in range(120):
        nx, nh = int(rng.integers(1, 6000)), int(rng.integers(1, 700))
        x, h = rng.standard_normal(nx), rng.standard_normal(nh)
        lo = max(1, (nh - 1).bit_length())
        n = 1 << int(rng.integers(lo, min(16, lo + 5)))
        want = port.convolve_ola(x, h, n)
        got = rs.convolve_ola(x, h, n, ctx=ctx)
        assert got.size == want.size
        assert rel_err(got, want) <= WAVE_TOL, (nx, nh, n)


def test_ola_block_boundaries(rs, ctx, port):
    rng = np.random.default_rng(13)
    h = rng.standard_normal(8)
    for nx in (9, 17, 18, 16, 1, 2, 900):
        x = rng.standard_normal(nx)
        assert rel_err(rs.convolve_ola(x, h, 16, ctx=ctx), port.convolve_ola(x, h, 16)) <= WAVE_TOL
    x, h = rng.standard_normal(777), rng.standard_normal(64)
    assert rel_err(rs.convolve_ola(x, h, 64, ctx=ctx), port.convolve_ola(x, h, 64)) <= WAVE_TOL  # L=1


@pytest.mark.parametrize("n", [2 ** k for k in range(1, 21)])
def test_every_fft_size(rs, ctx, port, n):
    # N <= 32768: one CTA per transform (K4); N >= 65536: the four-step path (large.cu)
    rng = np.random.default_rng(100 + n)
    nh = max(1, n // 2 - 3) if n > 2 else 1
    nx = 5 * n + 7 if n <= 65536 else 2 * n + 7
    x, h = rng.standard_normal(nx), rng.standard_normal(nh)
    assert rel_err(rs.convolve_ola(x, h, n, ctx=ctx), port.convolve_ola(x, h, n)) <= WAVE_TOL


def test_full_fft_long_signal(rs, ctx, port):
    # one-block filtering of a 20 s signal: N = 2^19 through the four-step path
    rng = np.random.default_rng(14)
    x, h = rng.standard_normal(320000), rng.standard_normal(9000) * np.exp(-np.arange(9000) / 2000)
    got = rs.convolve_full_fft(x, h, ctx=ctx)
    assert rel_err(got, port.convolve_full_fft(x, h)) <= WAVE_TOL


def test_two_stream_k4_all_sizes():
    """Run the two-stream K4 (ola2.cu) at every size it supports (RSG_OLA2) in a fresh
    process: single pairs long enough for several runs per item, and a render."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import numpy as np, oracle\n"
        "from paper_1712_03439_b200 import roomsim as rs, scenes\n"
        "ctx = rs.Context(0); port = oracle.port(); rng = np.random.default_rng(8); worst = 0.0\n"
        "for k in range(5, 13):\n"
        "    n = 2 ** k\n"
        "    for nh in (1, n // 4 + 1, n // 2, n - 3):\n"
        "        x, h = rng.standard_normal(40 * n + 13), rng.standard_normal(max(nh, 1))\n"
        "        want = port.convolve_ola(x, h, n); got = rs.convolve_ola(x, h, n, ctx=ctx)\n"
        "        worst = max(worst, float(np.abs(got - want).max() / np.abs(want).max()))\n"
        "b = scenes.config4(n_utt=3, seed=31)\n"
        "g = rs.render_batch(b, ctx=ctx); o = port.render_batch(b, threads=8)\n"
        "assert np.allclose(g.gains, o[3], rtol=1e-5), (g.gains, o[3])\n"
        "assert np.allclose(g.power, o[4], rtol=1e-5), (g.power, o[4])\n"
        "for u in range(b.n_utt):\n"
        "    for j in range(int(b.mic_begin[u + 1] - b.mic_begin[u])):\n"
        "        a_ = b.channel(g.out, u, j, g.out_len[u]); w_ = b.channel(o[0], u, j, o[1][u])\n"
        "        worst = max(worst, float(np.abs(a_ - w_).max() / np.abs(w_).max()))\n"
        "print(worst)\n")
    env = dict(os.environ, RSG_OLA2="5,12")
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert float(r.stdout.strip().splitlines()[-1]) <= WAVE_TOL


@pytest.mark.parametrize("env,sizes", [
    ({"RSG_IP": "9,14", "RSG_IP_FORCE": "1"}, (10, 11, 12, 13, 14, 15)),  # in-place K4 (big.cu), every size
    ({"RSG_IP": "0,0"}, (10, 11, 12, 13)),  # in-place K4 off: ola_small_kernel up to M = 4096, four-step above
])
def test_k4_variants(env, sizes):
    """Opt-in K4 variants in a fresh process (their selection is read once per process):
    single pairs with several runs per item at every N_h regime, and a render."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import numpy as np, oracle\n"
        "from paper_1712_03439_b200 import roomsim as rs, scenes\n"
        "ctx = rs.Context(0); port = oracle.port(); rng = np.random.default_rng(9); worst = 0.0\n"
        f"for k in {tuple(sizes)!r}:\n"
        "    n = 2 ** k\n"
        "    for nh in (1, n // 4 + 1, n // 2, n - 3):\n"
        "        x, h = rng.standard_normal(23 * n + 13), rng.standard_normal(max(nh, 1))\n"
        "        want = port.convolve_ola(x, h, n); got = rs.convolve_ola(x, h, n, ctx=ctx)\n"
        "        worst = max(worst, float(np.abs(got - want).max() / np.abs(want).max()))\n"
        "b = scenes.config3(n_utt=4, seed=33)\n"
        "g = rs.render_batch(b, ctx=ctx); o = port.render_batch(b, threads=8)\n"
        "assert np.allclose(g.power, o[4], rtol=1e-5), (g.power, o[4])\n"
        "for u in range(b.n_utt):\n"
        "    for j in range(int(b.mic_begin[u + 1] - b.mic_begin[u])):\n"
        "        a_ = b.channel(g.out, u, j, g.out_len[u]); w_ = b.channel(o[0], u, j, o[1][u])\n"
        "        worst = max(worst, float(np.abs(a_ - w_).max() / np.abs(w_).max()))\n"
        "print(worst)\n")
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=dict(os.environ, **env),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert float(r.stdout.strip().splitlines()[-1]) <= WAVE_TOL


@pytest.mark.parametrize("n", [4096, 8192])
def test_two_blocks_per_transform_k4(rs, ctx, port, n):
    """ola_ipc_kernel (big.cu): blocks 2j and 2j + 1 of a pair share one complex N-point
    transform.  Odd and even block counts, one block, N_h from 1 to the largest carry that
    fits, signals that end inside the first / second block of a transform, and runs long
    enough to be split into several work items (recomputed overlap blocks)."""
    rng = np.random.default_rng(n)
    for nh in (1, 2, 57, n // 8 + 1, n // 4 + 3, n // 2, n // 2 + 401):
        L = n - nh + 1
        for nx in (1, L - 1, L, L + 1, 2 * L, 2 * L + 1, 3 * L - 5, 7 * L + 13, 150 * L + 77):
            x, h = rng.standard_normal(nx), rng.standard_normal(nh) * np.exp(-np.arange(nh) / max(nh / 4, 1))
            want = port.convolve_ola(x, h, n)
            got = rs.convolve_ola(x, h, n, ctx=ctx)
            assert got.shape == want.shape
            assert rel_err(got, want) <= WAVE_TOL, (n, nh, nx)


@pytest.mark.parametrize("env", [{"RSG_IPC": "0,0"}, {"RSG_REBLOCK": "0"}, {"RSG_REBLOCK": "0", "RSG_IPC": "0,0"}])
def test_render_with_reference_blocking_and_without_ipc(env):
    """The render with the executed block size = the reference's plan (RSG_REBLOCK=0) and
    with the two-blocks-per-transform K4 off (RSG_IPC=0,0), in fresh processes: both
    against the reference port, and identical layouts."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import numpy as np, oracle\n"
        "from paper_1712_03439_b200 import roomsim as rs, scenes\n"
        "ctx = rs.Context(0); port = oracle.port(); worst = 0.0\n"
        "for b in (scenes.config4(n_utt=6, seed=41), scenes.config3(n_utt=4, seed=42), scenes.config2(n_utt=2, seed=43)):\n"
        "    g = rs.render_batch(b, ctx=ctx); o = port.render_batch(b, threads=8)\n"
        "    for f in ('rir_keep', 'cutoff', 'fft_size', 'block_len', 'n_blocks'):\n"
        "        assert (g.layout[f] == o[2][f]).all(), f\n"
        "    assert np.allclose(g.gains, o[3], rtol=1e-5); assert np.allclose(g.power, o[4], rtol=1e-5)\n"
        "    for u in range(b.n_utt):\n"
        "        for j in range(int(b.mic_begin[u + 1] - b.mic_begin[u])):\n"
        "            a_ = b.channel(g.out, u, j, g.out_len[u]); w_ = b.channel(o[0], u, j, o[1][u])\n"
        "            worst = max(worst, float(np.abs(a_ - w_).max() / np.abs(w_).max()))\n"
        "print(worst)\n")
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=dict(os.environ, **env),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert float(r.stdout.strip().splitlines()[-1]) <= WAVE_TOL


def test_four_step_path_small_sizes(tmp_path):
    """Route every size >= 2^7 through the four-step path (RSG_LARGE_MIN) in a fresh
    process and check it against the oracle at sizes where K4 normally runs."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import numpy as np, oracle\n"
        "from paper_1712_03439_b200 import roomsim as rs\n"
        "ctx = rs.Context(0); port = oracle.port(); rng = np.random.default_rng(7); worst = 0.0\n"
        "for k in range(7, 17):\n"
        "    n = 2 ** k\n"
        "    for nh in (1, n // 4 + 1, n // 2 - 3, n - 5):\n"
        "        x, h = rng.standard_normal(3 * n + 11), rng.standard_normal(max(nh, 1))\n"
        "        want = port.convolve_ola(x, h, n); got = rs.convolve_ola(x, h, n, ctx=ctx)\n"
        "        worst = max(worst, float(np.abs(got - want).max() / np.abs(want).max()))\n"
        "print(worst)\n")
    env = dict(os.environ, RSG_LARGE_MIN="6")
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert float(r.stdout.strip().splitlines()[-1]) <= WAVE_TOL


def test_config1(rs, ctx, port):
    from paper_1712_03439_b200 import scenes

    x, h, n = scenes.config1()
    assert rs.ola_block_count(x.size, h.size, n) == 20 and n - h.size + 1 == 4097
    got = rs.convolve_ola(x.astype(np.float64), h, n, ctx=ctx)
    want = port.convolve_ola(x.astype(np.float64), h, n)
    assert rel_err(got, want) <= WAVE_TOL
    t = ctx.last_timing()
    assert t["launches"] >= 1  # K4 alone at N = 8192: ola_ipc_kernel transforms the RIR itself (no K3 launch)


# ---- the batched render -------------------------------------------------------------
def _render_both(rs, ctx, port, b):
    g = rs.render_batch(b, ctx=ctx)
    o_out, o_len, o_lay, o_gain, o_pow = port.render_batch(b, threads=8)
    return g, (o_out, o_len, o_lay, o_gain, o_pow)


def _check_render(b, g, o):
    o_out, o_len, o_lay, o_gain, o_pow = o
    assert (g.out_len == o_len).all()
    for f in ("rir_len", "rir_keep", "cutoff", "fft_size", "block_len", "n_blocks", "out_len"):
        assert (g.layout[f] == o_lay[f]).all(), f
    np.testing.assert_allclose(g.gains, o_gain, rtol=1e-5)
    np.testing.assert_allclose(g.power, o_pow, rtol=1e-5)
    J = np.diff(b.mic_begin)
    for u in range(b.n_utt):
        want = np.concatenate([b.channel(o_out, u, j, o_len[u]) for j in range(J[u])])
        got = np.concatenate([b.channel(g.out, u, j, o_len[u]) for j in range(J[u])])
        assert rel_err(got, want) <= WAVE_TOL, u
        # tail beyond out_len is zero-filled
        for j in range(J[u]):
            o = int(b.out_off[u] + j * b.out_stride[u])
            assert not g.out[o + o_len[u]: o + b.out_stride[u]].any()


def test_render_config3_subset(rs, ctx, port):
    from paper_1712_03439_b200 import scenes

    b = scenes.config3(n_utt=6, seed=21)
    g, o = _render_both(rs, ctx, port, b)
    _check_render(b, g, o)


def test_render_config4_subset(rs, ctx, port):
    from paper_1712_03439_b200 import scenes

    b = scenes.config4(n_utt=4, seed=22)
    g, o = _render_both(rs, ctx, port, b)
    _check_render(b, g, o)


def test_mix_epilogue_edges(rs, ctx, port):
    """The mix in the K4 epilogue (mixfin.cuh) at its edges: utterances with more sources than it
    caches (10 > 8: mix_kernel mixes them), channels that do not start on 16-byte boundaries
    (scalar stores), and the per-context toggle — same bytes with the epilogue on and off."""
    import dataclasses

    from paper_1712_03439_b200 import scenes

    wide = scenes.make_batch(dataclasses.replace(scenes.spec_config4(33), num_noises=9), 3, eta_db=20.0,
                             plan_rule=scenes.PLAN_POW2_TWICE, name="wide")
    g, o = _render_both(rs, ctx, port, wide)
    _check_render(wide, g, o)
    assert ctx.mix_counts() == (0, int(np.diff(wide.mic_begin).sum()))

    b = scenes.config4(n_utt=5, seed=34)
    base = type(b)

    class OddStrides(base):
        out_stride = property(lambda self: base.out_stride.fget(self) + 1)

    b.__class__ = OddStrides
    assert (b.out_stride % 4 != 0).any()
    g, o = _render_both(rs, ctx, port, b)
    _check_render(b, g, o)
    fused, total = ctx.mix_counts()
    assert fused == total > 0
    try:
        ctx.set_fused_mix(0)
        g0 = rs.render_batch(b, ctx=ctx)
        assert ctx.mix_counts() == (0, total)
    finally:
        ctx.set_fused_mix(-1)
    assert (g0.out.view(np.uint32) == g.out.view(np.uint32)).all()
    assert (g0.gains.view(np.uint64) == g.gains.view(np.uint64)).all()


def test_render_config2_subset(rs, ctx, port):
    from paper_1712_03439_b200 import scenes

    b = scenes.config2(n_utt=4, seed=23)
    g, o = _render_both(rs, ctx, port, b)
    _check_render(b, g, o)


def test_render_forced_65536(rs, ctx, port):
    # the batched render through the four-step path (N = 65536, M = 32768)
    from paper_1712_03439_b200 import scenes

    b = scenes.config3(n_utt=2, seed=25)
    b.plan_rule, b.forced_fft_size = scenes.PLAN_FORCED, 65536
    g, o = _render_both(rs, ctx, port, b)
    assert (g.layout["fft_size"] == 65536).all()
    _check_render(b, g, o)


def test_render_config5_subset(rs, ctx, port):
    from paper_1712_03439_b200 import scenes

    b = scenes.config5(n_utt=1, seed=24)
    g, o = _render_both(rs, ctx, port, b)
    assert (g.layout["fft_size"] == 32768).all()
    _check_render(b, g, o)


def test_render_kats(rs, ctx):
    """SPEC.md:354-355 with K = 0, d = 1 m (a single unit tap at 47)."""
    from paper_1712_03439_b200 import scenes

    x = np.random.default_rng(5).standard_normal(1000).astype(np.float32)

    def batch(n_src):
        return scenes.SceneBatch(
            src_begin=np.array([0, n_src]), mic_begin=np.array([0, 1]),
            room_dims=np.array([[5.0, 5.0, 5.0]]), reflection=np.array([0.5]),
            sample_rate=np.array([16000.0]), speed_of_sound=np.array([343.0]),
            image_order=np.array([0], np.int32), max_taps=np.array([0]),
            src_pos=np.tile([1.0, 1.0, 1.0], (n_src, 1)), mic_pos=np.array([[2.0, 1.0, 1.0]]),
            snr_db=np.zeros(n_src), sig_off=np.zeros(n_src, np.int64), sig_len=np.full(n_src, 1000),
            signals=x, plan_rule=scenes.PLAN_CHOOSE)

    b = batch(1)
    r = rs.render_batch(b, ctx=ctx)
    y = b.channel(r.out, 0, 0, r.out_len[0])
    assert r.out_len[0] == 1047
    assert np.abs(y[47:] - x).max() <= WAVE_TOL * np.abs(x).max()
    assert np.abs(y[:47]).max() <= WAVE_TOL * np.abs(x).max()
    b = batch(2)
    r = rs.render_batch(b, ctx=ctx)
    y = b.channel(r.out, 0, 0, r.out_len[0])
    assert r.gains[1] == pytest.approx(1.0, rel=1e-12)
    assert np.abs(y[47:] - 2 * x).max() <= WAVE_TOL * 2 * np.abs(x).max()


def test_snr_fidelity(rs, ctx):
    """10 log10(P_target / P_scaled_noise) = snr within 1e-6 dB."""
    from paper_1712_03439_b200 import scenes

    b = scenes.config3(n_utt=3, seed=31)
    r = rs.render_batch(b, ctx=ctx)
    pb = b.pair_begin
    for u in range(b.n_utt):
        I, J = int(np.diff(b.src_begin)[u]), int(np.diff(b.mic_begin)[u])
        for j in range(J):
            t = rs.last_pair_signal(pb[u] + j, 1 << 22, ctx=ctx).astype(np.float64)
            pt = np.mean(t * t)
            for i in range(1, I):
                p = pb[u] + i * J + j
                n = rs.last_pair_signal(p, 1 << 22, ctx=ctx).astype(np.float64) * r.gains[p]
                snr = 10 * math.log10(pt / np.mean(n * n))
                assert abs(snr - b.snr_db[b.src_begin[u] + i]) <= 1e-6


def test_determinism(rs, ctx):
    from paper_1712_03439_b200 import scenes

    b = scenes.config4(n_utt=8, seed=41)
    a = rs.render_batch(b, ctx=ctx).out.copy()
    c = rs.render_batch(b, ctx=ctx).out.copy()
    assert (a.view(np.uint32) == c.view(np.uint32)).all()


def test_device_mode_matches_host(rs, ctx):
    import torch

    from paper_1712_03439_b200 import scenes

    b = scenes.config4(n_utt=5, seed=42)
    host = rs.render_batch(b, ctx=ctx)
    sig = torch.from_numpy(b.signals).cuda()
    out = torch.zeros(b.out_total, dtype=torch.float32, device="cuda")
    dev = rs.render_batch(b, ctx=ctx, device_signals_ptr=sig.data_ptr(), device_out_ptr=out.data_ptr())
    torch.cuda.synchronize()
    assert (out.cpu().numpy().view(np.uint32) == host.out.view(np.uint32)).all()
    assert (dev.layout == host.layout).all()


def test_render_errors(rs, ctx):
    from paper_1712_03439_b200 import scenes

    b = scenes.config3(n_utt=2, seed=51)
    b.src_pos[1] = [0.0, 1.0, 1.0]
    with pytest.raises(rs.PlacementError):
        rs.render_batch(b, ctx=ctx)
    b = scenes.config3(n_utt=2, seed=51)
    b.plan_rule, b.forced_fft_size = scenes.PLAN_FORCED, 16
    with pytest.raises(rs.PlanError):
        rs.render_batch(b, ctx=ctx)


@pytest.mark.parametrize("cfg,n_utt,seed", [("config5", 1, 24), ("config4", 4, 26), ("config2", 4, 33)])
def test_render_rirs_bit_exact(rs, ctx, port, cfg, n_utt, seed):
    """Every pair's RIR as the batched render synthesized it (K1, through its launch
    classes: the 128- / 512-thread lattices, the sliced and the one-CTA long RIRs) equals
    the reference synthesize_rir (room_model.hpp:141-174) bit for bit."""
    from paper_1712_03439_b200 import scenes

    b = getattr(scenes, cfg)(n_utt=n_utt, seed=seed)
    g = rs.render_batch(b, ctx=ctx)
    I, J = np.diff(b.src_begin), np.diff(b.mic_begin)
    checked = 0
    for u in range(b.n_utt):
        for i in range(I[u]):
            for j in range(J[u]):
                p = int(b.pair_begin[u] + i * J[u] + j)
                want = port.synthesize_rir(b.room_dims[u], float(b.reflection[u]), int(b.image_order[u]),
                                           b.src_pos[b.src_begin[u] + i], b.mic_pos[b.mic_begin[u] + j],
                                           fs=float(b.sample_rate[u]), c0=float(b.speed_of_sound[u]),
                                           max_taps=int(b.max_taps[u]))
                assert want.size == g.layout["rir_len"][p], (p, want.size)
                if b.eta_db > 0:  # the render keeps the truncated RIR (room_model.hpp:203-213)
                    want = port.truncate_rir(want, b.eta_db)[0]
                got = rs.last_pair_rir(p, want.size + 8, ctx=ctx)
                assert got.size == want.size == g.layout["rir_keep"][p], (p, got.size, want.size)
                assert (got.view(np.uint64) == want.view(np.uint64)).all(), p
                checked += 1
    assert checked == b.n_pairs


def test_k1_match_fold_variant():
    """The 512-thread K1 classes with the match_any fold forced (RSG_K1_FOLD / _S = 0; the
    default there is the ordered-claims fold) in a fresh process: single RIRs (one slice and
    sliced) and every pair of a config-5 and a config-4 render, bit for bit."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import numpy as np, oracle\n"
        "from paper_1712_03439_b200 import roomsim as rs, scenes\n"
        "ctx = rs.Context(0); port = oracle.port(); rng = np.random.default_rng(12)\n"
        "u64 = lambda a: np.ascontiguousarray(a, np.float64).view(np.uint64)\n"
        "for t in range(12):\n"
        "    room = rng.uniform([3, 3, 2.5], [10, 8, 6]); k = int(rng.integers(0, 30))\n"
        "    src, mic = rng.uniform(0.5, room - 0.5), rng.uniform(0.5, room - 0.5)\n"
        "    want = port.synthesize_rir(room, 0.9, k, src, mic, max_taps=30000)\n"
        "    got = rs.synthesize_rir(room, 0.9, k, src, mic, max_taps=30000, ctx=ctx)\n"
        "    assert (u64(got) == u64(want)).all(), t\n"
        "n = 0\n"
        "for b in (scenes.config5(n_utt=1, seed=27), scenes.config4(n_utt=3, seed=28)):\n"
        "    g = rs.render_batch(b, ctx=ctx); I, J = np.diff(b.src_begin), np.diff(b.mic_begin)\n"
        "    for u in range(b.n_utt):\n"
        "        for i in range(I[u]):\n"
        "            for j in range(J[u]):\n"
        "                p = int(b.pair_begin[u] + i * J[u] + j)\n"
        "                w = port.synthesize_rir(b.room_dims[u], float(b.reflection[u]), int(b.image_order[u]),\n"
        "                    b.src_pos[b.src_begin[u] + i], b.mic_pos[b.mic_begin[u] + j], fs=float(b.sample_rate[u]),\n"
        "                    c0=float(b.speed_of_sound[u]), max_taps=int(b.max_taps[u]))\n"
        "                if b.eta_db > 0: w = port.truncate_rir(w, b.eta_db)[0]\n"
        "                got = rs.last_pair_rir(p, w.size + 8, ctx=ctx)\n"
        "                assert got.size == w.size and (u64(got) == u64(w)).all(), p\n"
        "                n += 1\n"
        "print(n)\n")
    env = dict(os.environ, RSG_K1_FOLD="0", RSG_K1_FOLD_S="0")
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert int(r.stdout.strip().splitlines()[-1]) > 20


def test_render_error_order_matches_reference(rs, ctx):
    """The first error of a render is the one the reference meets first: utterance
    order, then pair order; per pair RoomConfig::validate and the placements inside
    synthesize_rir, then geometry, then the convolution's own checks."""
    import oracle
    from paper_1712_03439_b200 import scenes

    ref = oracle.reference() if oracle.reference_available() else oracle.port()
    codes = {rs.PlacementError: 1, rs.GeometryError: 2, rs.DegenerateInputError: 3, rs.PlanError: 4,
             rs.ConfigError: 5}

    def run_both(b):
        try:
            rs.render_batch(b, ctx=ctx)
            got = 0
        except rs.Error as e:
            got = codes[type(e)]
        try:
            ref.render_batch(b)
            want = 0
        except oracle.OracleError as e:
            want = e.code
        return got, want

    cases = []
    b = scenes.config3(n_utt=3, seed=81)       # utt 0 pair (1, *): placement; utt 1: bad room
    b.src_pos[b.src_begin[0] + 1] = [0.0, 1.0, 1.0]
    b.reflection[1] = 1.5
    cases.append((b, 1))
    b = scenes.config3(n_utt=3, seed=81)       # utt 1: bad room before utt 2's placement error
    b.reflection[1] = 1.5
    b.mic_pos[b.mic_begin[2]] = [-1.0, 1.0, 1.0]
    cases.append((b, 5))
    b = scenes.config3(n_utt=2, seed=82)       # mic on the source (geometry) beats its empty signal
    b.image_order[1] = 0
    s = b.src_begin[1]
    b.mic_pos[b.mic_begin[1]] = b.src_pos[s]
    b.sig_len = b.sig_len.copy()
    b.sig_len[s] = 0
    cases.append((b, 2))
    b = scenes.config3(n_utt=2, seed=83)       # an empty signal alone: DegenerateInputError
    b.sig_len = b.sig_len.copy()
    b.sig_len[b.src_begin[1] + 1] = 0
    cases.append((b, 3))
    for k, (b, want_code) in enumerate(cases):
        got, want = run_both(b)
        assert got == want == want_code, (k, got, want)
