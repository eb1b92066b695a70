"""Pins the CPU oracle (oracle/roomsim_oracle.c) — CPU only.

(a) SPEC.md known-answer tests (the reference has no test suite; SPEC's
    examples and acceptance criteria are its de-facto KATs);
(b) bit-exact agreement with the reference itself, compiled from
    /root/reference by oracle/Makefile into oracle/_ref (skipped where that
    build is absent, e.g. on the GPU box);
(c) the committed golden fixtures in tests/golden/ (made from oracle/_ref by
    tests/golden/make_golden.py).
"""
import math
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden.npz")


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


# ---- SPEC room_model KATs ---------------------------------------------------------
def test_image_count_and_lattice(port):
    assert port.virtual_source_count(8) == 4913
    for k in range(0, 11):
        assert port.virtual_source_count(k) == (2 * k + 1) ** 3
    pos, g = port.enumerate_images([5, 5, 5], 0.5, 0, [1, 1, 1])
    assert pos.shape == (1, 3) and (pos[0] == [1, 1, 1]).all() and g[0] == 0
    pos, g = port.enumerate_images([3, 4, 5], 0.5, 1, [1, 1, 1])
    assert pos.shape[0] == 27  # index (-1,0,0) -> (-1,1,1), g=1
    idx = (0 * 3 + 1) * 3 + 1  # nx=-1, ny=0, nz=0 in nx->ny->nz order
    assert (pos[idx] == [-1, 1, 1]).all() and g[idx] == 1


def test_single_tap(port):
    # K=0, d = 1 m -> h[47] = 1.0 (ceil(16000/343) = 47)
    h = port.synthesize_rir([5, 5, 5], 0.5, 0, [1, 1, 1], [2, 1, 1])
    assert h.size == 48 and h[47] == 1.0 and not h[:47].any()


def test_k1_bruteforce(port):
    # equals an independent brute-force sum over all 27 images
    room, src, mic, r = [3.0, 4.0, 5.0], [1.0, 2.0, 2.0], [2.0, 2.0, 2.0], 0.5
    pos, g = port.enumerate_images(room, r, 1, src)
    d = np.sqrt(((pos - np.array(mic)) ** 2).sum(1))
    delay = np.ceil(d * 16000.0 / 343.0).astype(int)
    want = np.zeros(delay.max() + 1)
    for dl, gg, dd in zip(delay, g, d):
        want[dl] += r ** gg / dd
    got = port.synthesize_rir(room, r, 1, src, mic)
    np.testing.assert_allclose(got, want, rtol=1e-15, atol=0)


def test_threshold_cut_truncate(port):
    assert port.power_threshold(np.array([0.0, 1.0, 0.5]), 20) == pytest.approx(0.01, rel=1e-15)
    assert port.power_threshold(np.array([2.0]), 10) == pytest.approx(0.4, rel=1e-15)
    h = 0.9 ** np.arange(60)
    assert port.cutoff_index(h, port.power_threshold(h, 20)) == 21
    assert port.cutoff_index(np.array([1.0, 0, 0]), 0.5) == 0
    t, nc, _ = port.truncate_rir(np.array([1, 0.5, 0.001, 0.0005]), 20)
    assert nc == 1 and list(t) == [1, 0.5, 0.001]
    h = np.random.default_rng(0).random(100)
    assert (port.truncate_rir(h, 200)[0] == h).all()


def test_truncation_properties(port):
    rng = np.random.default_rng(1)
    for _ in range(100):
        h = rng.random(rng.integers(5, 400)) * np.exp(-np.linspace(0, 8, 1)[0] * rng.random())
        h *= np.exp(-rng.random() * 10 * np.linspace(0, 1, h.size))
        n1 = port.truncate_rir(h, 10)[1]
        n2 = port.truncate_rir(h, 30)[1]
        assert n1 <= n2
        th = port.power_threshold(h, 20)
        nc = port.cutoff_index(h, th)
        assert (h[nc + 1:] ** 2 < th).all()


def test_errors(port):
    import oracle

    with pytest.raises(oracle.OracleError) as e:
        port.synthesize_rir([5, 5, 5], 0.5, 2, [0, 1, 1], [2, 2, 2])
    assert e.value.code == 1
    with pytest.raises(oracle.OracleError) as e:
        port.synthesize_rir([5, 5, 5], 1.5, 2, [1, 1, 1], [2, 2, 2])
    assert e.value.code == 5
    with pytest.raises(oracle.OracleError) as e:  # mic on the source: d = 0
        port.synthesize_rir([5, 5, 5], 0.5, 0, [1, 1, 1], [1, 1, 1])
    assert e.value.code == 2
    with pytest.raises(oracle.OracleError) as e:
        port.convolve_ola(np.ones(10), np.ones(8), 4)
    assert e.value.code == 4


# ---- SPEC convolution KATs -----------------------------------------------------------
def test_costs_and_plan(port):
    # SPEC.md:254, :263, :273, :283, acceptance 1
    assert port.cost_direct(2.55, 2, 116991, 3893) == pytest.approx(2.3228e9, rel=1e-4)
    assert port.cost_full_fft(2.55, 2, 116991, 3893, 2 ** 17) == pytest.approx(69520588.8, rel=1e-12)
    assert port.cost_ola(2.55, 2, 116991, 3893, 2 ** 14) == pytest.approx(50803507.2, rel=1e-12)
    s, n, c = port.choose_plan(2.55, 2, 116991, 3893)
    assert (s, n) == (2, 2 ** 14) and c == pytest.approx(50803507.2, rel=1e-12)
    assert port.cost_direct(1, 1, 1, 1) == 1 and port.cost_direct(2, 2, 10, 5) == 200
    assert port.cost_full_fft(1, 1, 1, 1, 2) == 16 and port.cost_full_fft(1, 2, 2, 2, 4) == 112
    assert port.cost_ola(1, 1, 1, 1, 2) == 16 and port.cost_ola(1, 1, 100, 1, 4) == 1016
    assert port.ola_block_count(116991, 3893, 2 ** 14) == 10
    # config 1 layout: L = 4097 (convolution.hpp:230), B = 20
    assert port.ola_block_count(80000, 4096, 8192) == 20


def test_plan_optimality(port):
    rng = np.random.default_rng(2)
    for _ in range(200):
        nx, nh = int(rng.integers(1, 300000)), int(rng.integers(1, 20000))
        s, n, c = port.choose_plan(1, 1, nx, nh)
        cand = []
        m = 1 << max(1, (max(nh, 2) - 1).bit_length())
        top = 1 << max(1, (nx + nh - 2).bit_length())
        while m <= top:
            cand.append(port.cost_ola(1, 1, nx, nh, m))
            m <<= 1
        full = port.cost_full_fft(1, 1, nx, nh, top)
        assert c == min(min(cand), full)


def test_convolution_kats(port):
    np.testing.assert_allclose(port.convolve_direct([1, 2, 3], [1]), [1, 2, 3])
    np.testing.assert_allclose(port.convolve_direct([1, 1], [1, 1]), [1, 2, 1])
    np.testing.assert_allclose(port.convolve_direct([2, 0, -1], [0.5, 0.25]), [1, 0.5, -0.5, -0.25])
    np.testing.assert_allclose(port.convolve_full_fft([1, 2, 3], [1]), [1, 2, 3], atol=1e-12)
    assert np.abs(port.convolve_ola(np.zeros(50), np.ones(5), 8)).max() == 0


def test_oracle_equivalence(port):
    # SPEC.md:288 / acceptance 2: 200 random pairs, full and OLA vs direct
    rng = np.random.default_rng(3)
    for _ in range(200):
        nx, nh = int(rng.integers(1, 2000)), int(rng.integers(1, 256))
        x, h = rng.standard_normal(nx), rng.standard_normal(nh)
        d = port.convolve_direct(x, h)
        tol = 1e-9 * (1 + np.abs(d).max())
        assert np.abs(port.convolve_full_fft(x, h) - d).max() <= tol
        n = 1 << int(rng.integers(max(1, (nh - 1).bit_length()), 13))
        assert np.abs(port.convolve_ola(x, h, n) - d).max() <= tol


def test_ola_block_boundaries(port):
    rng = np.random.default_rng(4)
    h = rng.standard_normal(8)
    for nx in (9, 17, 18, 16, 1, 2):  # L = 9 at N = 16: divisible, off by one
        x = rng.standard_normal(nx)
        d = port.convolve_direct(x, h)
        assert np.abs(port.convolve_ola(x, h, 16) - d).max() <= 1e-12
    x = rng.standard_normal(37)
    h = rng.standard_normal(16)
    d = port.convolve_direct(x, h)
    assert np.abs(port.convolve_ola(x, h, 16) - d).max() <= 1e-12  # L = 1


def test_gain_kats(port):
    assert port.compute_gain(2.0, 2.0, 0.0) == 1.0
    assert port.compute_gain(2.0, 2.0, 20.0) == pytest.approx(0.1, rel=1e-15)
    rng = np.random.default_rng(5)
    for _ in range(20):
        pt, pn, snr = rng.random() + 0.1, rng.random() + 0.1, rng.uniform(0, 30)
        a = port.compute_gain(pt, pn, snr)
        assert abs(10 * math.log10(pt / (a * a * pn)) - snr) <= 1e-9


# ---- agreement with the compiled reference -------------------------------------------
def test_port_matches_reference_rirs(port, ref):
    rng = np.random.default_rng(6)
    for _ in range(40):
        room = rng.uniform([3, 3, 2.5], [10, 8, 6])
        src, mic = rng.uniform(0.5, room - 0.5), rng.uniform(0.5, room - 0.5)
        k, r = int(rng.integers(0, 9)), rng.uniform(0.2, 0.9)
        mt = int(rng.choice([0, 500, 3000]))
        a = port.synthesize_rir(room, r, k, src, mic, max_taps=mt)
        b = ref.synthesize_rir(room, r, k, src, mic, max_taps=mt)
        assert (bits(a) == bits(b)).all()
        for eta in (10.0, 20.0, 37.5):
            ta, na, pa = port.truncate_rir(a, eta)
            tb, nb, pb = ref.truncate_rir(b, eta)
            assert (na, ta.size) == (nb, tb.size) and pa == pb


def test_port_matches_reference_fft_conv_plan(port, ref):
    rng = np.random.default_rng(7)
    for n in [2 ** k for k in range(1, 16)]:
        x = rng.standard_normal(n)
        fa, fb = port.rfft_forward(x), ref.rfft_forward(x)
        assert (bits(fa.view(np.float64)) == bits(fb.view(np.float64))).all()
        assert (bits(port.rfft_inverse(fa, n)) == bits(ref.rfft_inverse(fb, n))).all()
    for _ in range(50):
        nx, nh = int(rng.integers(1, 5000)), int(rng.integers(1, 600))
        x, h = rng.standard_normal(nx), rng.standard_normal(nh)
        assert port.choose_plan(1, 1, nx, nh) == ref.choose_plan(1, 1, nx, nh)
        n = port.choose_plan(1, 1, nx, nh)[1]
        assert (bits(port.convolve_ola(x, h, n)) == bits(ref.convolve_ola(x, h, n))).all()
        assert (bits(port.convolve_full_fft(x, h)) == bits(ref.convolve_full_fft(x, h))).all()


def test_port_matches_reference_render(port, ref):
    from paper_1712_03439_b200 import scenes

    b = scenes.config3(n_utt=2, seed=11)
    oa = port.render_batch(b)
    ob = ref.render_batch(b)
    for x, y in zip(oa, ob):
        if x.dtype.names:
            for f in x.dtype.names:
                assert (x[f] == y[f]).all(), f
        else:
            assert (np.asarray(x).view(np.uint8) == np.asarray(y).view(np.uint8)).all()


# ---- golden fixtures (from oracle/_ref, tests/golden/make_golden.py) ---------------------
@pytest.fixture(scope="module")
def golden():
    if not os.path.exists(GOLDEN):
        pytest.skip("golden fixtures not generated")
    return np.load(GOLDEN, allow_pickle=False)


def test_port_matches_golden(port, golden):
    from tests.golden import cases

    for i, c in enumerate(cases.RIR_CASES):
        h = port.synthesize_rir(c["room"], c["r"], c["K"], c["src"], c["mic"], max_taps=c["max_taps"])
        assert (bits(h) == golden[f"rir_{i}"].view(np.uint64)).all(), i
        t, nc, th = port.truncate_rir(h, 20.0)
        assert nc == int(golden[f"nc_{i}"]) and th == float(golden[f"pth_{i}"])
    for i, (nx, nh) in enumerate(cases.PLAN_CASES):
        s, n, c = port.choose_plan(1, 1, nx, nh)
        assert (s, n, c) == tuple(golden["plans"][i][:2].astype(int)) + (golden["plan_costs"][i],)
    x, h, n = cases.ola_case()
    y = port.convolve_ola(x, h, n)
    assert (bits(y) == golden["ola"].view(np.uint64)).all()
