"""GPU parity at BASELINE scale and render invariance (VERDICT r01 "do this" #1).

* The full config-4 workload (4096 utterances, 49,152 pairs) through the chunked
  pipeline in device mode (16,384-pair chunks) and host mode (6,144-pair chunks, the
  C/2, C/4, C/4 tail split, signal uploads two chunks ahead): the two modes return
  the same bytes, and a deterministic subsample — every 64th utterance plus the
  first and last utterance of every chunk of both modes — matches the reference
  itself (oracle/_ref: the unmodified reference headers compiled) within the
  north-star bars.
* Config 2 at its full 128 utterances and config 5 at 16 utterances against the
  reference.
* Invariance: a render's bytes do not depend on the chunk size (RSG_CHUNK_PAIRS),
  the buffer mode or which other utterances share the batch (SPEC.md:472:
  results must not depend on the degree of parallelism).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WAVE_TOL = 1e-5  # relative to each utterance's peak (north_star)
LAYOUT_FIELDS = ("rir_len", "rir_keep", "cutoff", "fft_size", "block_len", "n_blocks", "out_len")


def chunk_ranges(pairs_per_utt, chunk_pairs, host):
    """Utterance ranges of the render's chunks (mirror of api.cu render_impl)."""
    total = int(np.sum(pairs_per_utt))
    ranges, u0, pairs, done = [], 0, 0, 0

    def target():
        rem = total - done
        if not host:
            return chunk_pairs
        if rem > chunk_pairs:
            return min(chunk_pairs, rem - chunk_pairs)
        return max(rem // 2, chunk_pairs // 4) if rem > chunk_pairs // 4 else rem

    want = target()
    for u, p in enumerate(pairs_per_utt):
        pairs += int(p)
        if pairs >= want or u + 1 == len(pairs_per_utt):
            ranges.append((u0, u + 1))
            u0, done, pairs = u + 1, done + pairs, 0
            want = target()
    return ranges


def checker():
    import oracle

    return oracle.reference() if oracle.reference_available() else oracle.port()


def compare_subset(full, g_out, g_len, g_lay, g_gain, g_pow, ids, want):
    """Utterances `ids` of a GPU render of `full` against a CPU render `want` of full.subset(ids)."""
    o_out, o_len, o_lay, o_gain, o_pow = want
    sub = full.subset(ids)
    pb_full, pb_sub = full.pair_begin, sub.pair_begin
    J = np.diff(full.mic_begin)
    worst = 0.0
    for k, u in enumerate(ids):
        assert g_len[u] == o_len[k], u
        gp = np.arange(pb_full[u], pb_full[u + 1])
        sp = np.arange(pb_sub[k], pb_sub[k + 1])
        for f in LAYOUT_FIELDS:
            assert (g_lay[f][gp] == o_lay[f][sp]).all(), (u, f)
        np.testing.assert_allclose(g_gain[gp], o_gain[sp], rtol=1e-5)
        np.testing.assert_allclose(g_pow[gp], o_pow[sp], rtol=1e-5)
        got = np.concatenate([full.channel(g_out, u, j, g_len[u]) for j in range(J[u])]).astype(np.float64)
        ref = np.concatenate([sub.channel(o_out, k, j, o_len[k]) for j in range(J[u])])
        err = np.abs(got - ref).max() / np.abs(ref).max()
        assert err <= WAVE_TOL, (u, err)
        worst = max(worst, err)
    return worst


def test_config4_full_scale_device_and_host():
    """BASELINE config 4 at full size: device vs host mode bytes, and a subsample vs the reference."""
    import torch

    from paper_1712_03439_b200 import roomsim as rs, scenes

    seed = 4
    b = scenes.config4(n_utt=4096, seed=seed, signals=False)
    spec = rs.sampler_spec(scenes.spec_config4(seed))
    ctx = rs.Context(0)
    sig = torch.empty(b.total_samples, dtype=torch.float32, device="cuda")
    rs.generate_signals(spec, b, seed=seed, device_ptr=sig.data_ptr())
    dout = torch.zeros(b.out_total, dtype=torch.float32, device="cuda")
    d = rs.render_batch(b, ctx=ctx, device_signals_ptr=sig.data_ptr(), device_out_ptr=dout.data_ptr())
    torch.cuda.synchronize()
    dev_out = dout.cpu().numpy()
    del dout
    # host mode: pinned host buffers, per-chunk H2D / D2H inside the call
    h_sig = torch.empty(b.total_samples, dtype=torch.float32, pin_memory=True)
    h_sig.copy_(sig)
    del sig
    h_out = torch.zeros(b.out_total, dtype=torch.float32, pin_memory=True)
    b.signals = h_sig.numpy()
    h = rs.render_batch(b, ctx=ctx, out=h_out.numpy())
    host_out = h_out.numpy()
    assert (host_out.view(np.uint32) == dev_out.view(np.uint32)).all()
    assert (h.layout == d.layout).all()
    assert (h.gains.view(np.uint64) == d.gains.view(np.uint64)).all()
    assert (h.power.view(np.uint64) == d.power.view(np.uint64)).all()
    # subsample: every 64th utterance + first / last utterance of every chunk of both modes
    ppu = b.pairs_per_utt
    ids = set(range(0, b.n_utt, 64)) | {b.n_utt - 1}
    for host_mode, cp in ((False, 16384), (True, 6144)):  # api.cu kChunkPairsDevice / kChunkPairsHost
        rng_ = chunk_ranges(ppu, cp, host_mode)
        assert len(rng_) >= (3 if not host_mode else 8), rng_
        for u0, u1 in rng_:
            ids |= {u0, u1 - 1}
    ids = np.array(sorted(ids), np.int64)
    sub = b.subset(ids)
    sub.signals = rs.generate_signals(spec, sub, seed=seed)  # host generator, keyed by utterance id
    # the subset's signals are the full batch's (bit-exact host/device generator)
    for k, u in enumerate(ids[:8]):
        s0 = b.src_begin[u]
        o, n = int(b.sig_off[s0]), int(b.sig_len[s0])
        so = int(sub.sig_off[sub.src_begin[k]])
        assert (sub.signals[so: so + n].view(np.uint32) == b.signals[o: o + n].view(np.uint32)).all()
    want = checker().render_batch(sub, threads=os.cpu_count() or 8)
    worst = compare_subset(b, dev_out, d.out_len, d.layout, d.gains, d.power, ids, want)
    # the subset rendered alone on the GPU gives the full batch's bytes (batch composition)
    s_out = rs.render_batch(sub, ctx=ctx)
    J = np.diff(b.mic_begin)
    for k, u in enumerate(ids):
        for j in range(J[u]):
            a_ = b.channel(dev_out, u, j, d.out_len[u])
            c_ = sub.channel(s_out.out, k, j, s_out.out_len[k])
            assert (a_.view(np.uint32) == c_.view(np.uint32)).all(), (u, j)
    print(f"config 4 full scale: {ids.size} utterances checked, worst {worst:.2e}")
    ctx.close()


@pytest.mark.parametrize("cfg,n_utt,seed", [("config2", 128, 2), ("config5", 16, 5), ("config3", 128, 3)])
def test_full_configs_vs_reference(rs, ctx, cfg, n_utt, seed):
    from paper_1712_03439_b200 import scenes

    b = scenes.CONFIGS[cfg](n_utt=n_utt, seed=seed)
    g = rs.render_batch(b, ctx=ctx)
    ids = np.arange(b.n_utt)
    want = checker().render_batch(b, threads=os.cpu_count() or 8)
    compare_subset(b, g.out, g.out_len, g.layout, g.gains, g.power, ids, want)


def _worker(tmp_path, tag, env, cfg, n_utt, seed, mode, ids=None):
    path = str(tmp_path / f"{tag}.npz")
    cmd = [sys.executable, os.path.join(ROOT, "tests", "render_worker.py"), cfg, str(n_utt), str(seed), mode, path]
    if ids is not None:
        cmd.append(",".join(str(int(u)) for u in ids))
    r = subprocess.run(cmd, cwd=ROOT, env=dict(os.environ, **env), capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    return dict(np.load(path))


def test_render_invariance(tmp_path):
    """Same bytes whatever the chunk size (chunk boundaries everywhere with 7 pairs),
    the buffer mode or the batch composition; the 7-pair render also against the
    reference."""
    from paper_1712_03439_b200 import scenes

    cfg, n, seed = "config3", 24, 71
    base = _worker(tmp_path, "base", {}, cfg, n, seed, "host")
    runs = {
        "chunk7_host": _worker(tmp_path, "c7h", {"RSG_CHUNK_PAIRS": "7"}, cfg, n, seed, "host"),
        "chunk7_dev": _worker(tmp_path, "c7d", {"RSG_CHUNK_PAIRS": "7"}, cfg, n, seed, "device"),
        "chunk50_dev": _worker(tmp_path, "c50d", {"RSG_CHUNK_PAIRS": "50"}, cfg, n, seed, "device"),
        "default_dev": _worker(tmp_path, "dd", {}, cfg, n, seed, "device"),
        # K1 over the whole RIR instead of the prefix the cut can keep (synth_bound.cu)
        "full_synth": _worker(tmp_path, "fs", {"RSG_SYNTH_CUT": "0"}, cfg, n, seed, "host"),
        # every channel through mix_kernel instead of the K4 epilogue (mixfin.cuh)
        "mix_kernel": _worker(tmp_path, "mk", {"RSG_FUSED_MIX": "0"}, cfg, n, seed, "device"),
    }
    for k, r in runs.items():
        for f in ("out", "out_len", "layout"):
            assert (r[f] == base[f]).all(), (k, f)
        for f in ("gains", "power"):
            assert (r[f].view(np.uint64) == base[f].view(np.uint64)).all(), (k, f)
    # composition: utterances 3, 10, 17 rendered alone
    ids = np.array([3, 10, 17])
    alone = _worker(tmp_path, "alone", {}, cfg, n, seed, "host", ids)
    b = scenes.CONFIGS[cfg](n_utt=n, seed=seed, signals=False)
    sub = b.subset(ids)
    full_out = base["out"]
    J = np.diff(b.mic_begin)
    for k, u in enumerate(ids):
        for j in range(J[u]):
            a_ = b.channel(full_out, u, j, base["out_len"][u])
            c_ = sub.channel(alone["out"], k, j, alone["out_len"][k])
            assert (a_ == c_).all(), (u, j)
        gp = np.arange(b.pair_begin[u], b.pair_begin[u + 1])
        sp = np.arange(sub.pair_begin[k], sub.pair_begin[k + 1])
        assert (alone["gains"][sp].view(np.uint64) == base["gains"][gp].view(np.uint64)).all()
    # and the 7-pair chunked render against the reference
    import oracle  # noqa: F401

    from paper_1712_03439_b200 import roomsim as rs

    bs = scenes.CONFIGS[cfg](n_utt=n, seed=seed)
    want = checker().render_batch(bs, threads=os.cpu_count() or 8)
    r = runs["chunk7_host"]
    lay = r["layout"].view(rs.LAYOUT_DTYPE)
    compare_subset(bs, r["out"].view(np.float32), r["out_len"], lay, r["gains"], r["power"],
                   np.arange(bs.n_utt), want)


@pytest.mark.parametrize("cfg,n,seed", [("config4", 48, 5), ("config5", 3, 9), ("config3", 40, 13)])
def test_fused_mix_matches_mix_kernel(tmp_path, cfg, n, seed):
    """The mix inside the K4 launches (the last work item of a channel mixes it, mixfin.cuh)
    and mix_kernel give the same bytes; the epilogue really ran (mix_counts)."""
    for mode in ("device", "host"):
        fused = _worker(tmp_path, f"f{mode}", {}, cfg, n, seed, mode)
        plain = _worker(tmp_path, f"p{mode}", {"RSG_FUSED_MIX": "0"}, cfg, n, seed, mode)
        small = _worker(tmp_path, f"s{mode}", {"RSG_CHUNK_PAIRS": "30"}, cfg, n, seed, mode)
        assert plain["mix_counts"][0] == 0 and plain["mix_counts"][1] > 0
        assert fused["mix_counts"][0] > 0.5 * fused["mix_counts"][1], fused["mix_counts"]
        for r in (plain, small):
            for f in ("out", "out_len", "layout"):
                assert (r[f] == fused[f]).all(), (mode, f)
            for f in ("gains", "power"):
                assert (r[f].view(np.uint64) == fused[f].view(np.uint64)).all(), (mode, f)


def test_concurrent_contexts(rs):
    """Renders from two host threads, one context each, running at once (a stream of batches with
    two in flight, bench.py `two_in_flight`): the same bytes as one at a time.  The two workloads
    need different shared-memory sizes from the same kernels (K1 slices, K4 carries)."""
    import threading

    from paper_1712_03439_b200 import scenes

    batches = [scenes.config4(n_utt=24, seed=61), scenes.config5(n_utt=2, seed=62), scenes.config3(n_utt=40, seed=63)]
    solo = rs.Context(0)
    want = [rs.render_batch(b, ctx=solo) for b in batches]
    solo.close()
    errs, got = [], {}

    def work(tid):
        try:
            c = rs.Context(0)
            for rep in range(4):
                for k in range(len(batches)):
                    i = (k + tid) % len(batches)
                    got[(tid, i)] = rs.render_batch(batches[i], ctx=c)
            c.close()
        except Exception as e:  # noqa: BLE001
            errs.append(repr(e))

    ths = [threading.Thread(target=work, args=(t,)) for t in range(2)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    assert not errs, errs
    for (tid, i), g in got.items():
        assert (g.out.view(np.uint32) == want[i].out.view(np.uint32)).all(), (tid, i)
        assert (g.gains.view(np.uint64) == want[i].gains.view(np.uint64)).all(), (tid, i)
        assert (g.layout == want[i].layout).all(), (tid, i)


def test_four_step_for_carries_that_do_not_fit(rs, ctx, port):
    """N = 32768 with N_h ~ 30000: the in-place K4's carry does not fit in shared memory,
    so the pair takes the four-step path (large.cu); also inside a render."""
    from paper_1712_03439_b200 import scenes

    rng = np.random.default_rng(91)
    for nh in (20000, 30000, 32000):
        x, h = rng.standard_normal(5 * 32768 + 77), rng.standard_normal(nh) * np.exp(-np.arange(nh) / 8000.0)
        got = rs.convolve_ola(x, h, 32768, ctx=ctx)
        want = port.convolve_ola(x, h, 32768)
        assert np.abs(got - want).max() <= WAVE_TOL * np.abs(want).max(), nh
    b = scenes.config5(n_utt=1, seed=93)
    b.max_taps[:] = 30000  # untruncated RIRs of ~30k taps at N = 32768
    b.image_order[:] = np.maximum(b.image_order, 40)
    g = rs.render_batch(b, ctx=ctx)
    assert (g.layout["rir_keep"] > 24000).all()
    want = checker().render_batch(b, threads=os.cpu_count() or 8)
    compare_subset(b, g.out, g.out_len, g.layout, g.gains, g.power, np.arange(b.n_utt), want)


def test_convolve_dispatch(rs, ctx):
    """roomsim::convolve (convolution.hpp:258-271) through rs_convolve for all three
    strategies against the reference: direct bit-exact (FP64), FFT strategies FP32."""
    ref = checker()
    rng = np.random.default_rng(92)
    for t in range(8):
        nx, nh = int(rng.integers(1, 9000)), int(rng.integers(1, 900))
        x, h = rng.standard_normal(nx), rng.standard_normal(nh)
        d = rs.convolve(x, h, rs.plan_for(1, 1, nx, nh, rs.DIRECT), ctx=ctx)
        assert (d.view(np.uint64) == ref.convolve_direct(x, h).view(np.uint64)).all(), t
        assert (rs.convolve_direct(x, h, ctx=ctx).view(np.uint64) == d.view(np.uint64)).all()
        f = rs.convolve(x, h, rs.plan_for(1, 1, nx, nh, rs.FULL_FFT), ctx=ctx)
        want = ref.convolve_full_fft(x, h)
        assert f.size == want.size and np.abs(f - want).max() <= WAVE_TOL * np.abs(want).max()
        p = rs.plan_for(1, 1, nx, nh, rs.OVERLAP_ADD)
        o = rs.convolve(x, h, p, ctx=ctx)
        want = ref.convolve_ola(x, h, p.fft_size)
        assert o.size == want.size and np.abs(o - want).max() <= WAVE_TOL * np.abs(want).max()
    with pytest.raises(rs.PlanError):
        rs.convolve(np.ones(10), np.ones(3), rs.ConvolutionPlan(rs.OVERLAP_ADD, None), ctx=ctx)
    with pytest.raises(rs.DegenerateInputError):
        rs.convolve(np.ones(0), np.ones(3), rs.ConvolutionPlan(rs.DIRECT), ctx=ctx)


@pytest.mark.parametrize("eta", [3.0, 20.0, 45.0, 80.0])
def test_truncation_any_eta(rs, ctx, eta):
    """K1 + K2 at shallow and deep cuts: cut indices, kept taps (bit-exact against the
    reference synthesize_rir + truncate_rir) and the renders."""
    from paper_1712_03439_b200 import scenes

    b = scenes.config3(n_utt=6, seed=int(eta) + 100)
    b.eta_db = eta
    g = rs.render_batch(b, ctx=ctx)
    ref = checker()
    want = ref.render_batch(b, threads=os.cpu_count() or 8)
    compare_subset(b, g.out, g.out_len, g.layout, g.gains, g.power, np.arange(b.n_utt), want)
    I, J = np.diff(b.src_begin), np.diff(b.mic_begin)
    for u in range(b.n_utt):
        for i in range(I[u]):
            for j in range(J[u]):
                p = int(b.pair_begin[u] + i * J[u] + j)
                full = ref.synthesize_rir(b.room_dims[u], float(b.reflection[u]), int(b.image_order[u]),
                                          b.src_pos[b.src_begin[u] + i], b.mic_pos[b.mic_begin[u] + j],
                                          max_taps=int(b.max_taps[u]))
                kept = ref.truncate_rir(full, eta)[0]
                got = rs.last_pair_rir(p, kept.size + 8, ctx=ctx)
                assert got.size == kept.size and (got.view(np.uint64) == kept.view(np.uint64)).all(), (p, eta)
