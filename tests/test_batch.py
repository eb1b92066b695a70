"""cmd_batch: manifest parsing on CPU; the GPU runs — determinism under
parallelism, the empty manifest, a failing record among five, and parity of a rendered
record against the reference."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _write_manifest(path, header, records):
    with open(path, "w") as f:
        if header is not None:
            f.write(json.dumps(header) + "\n")
        for r in records:
            f.write(json.dumps(r) + "\n")


def _inputs(tmp_path, n, seed=5):
    from paper_1712_03439_b200 import audio_io

    rng = np.random.default_rng(seed)
    recs = []
    for k in range(n):
        p = tmp_path / "in" / f"u{k:02d}.wav"
        p.parent.mkdir(exist_ok=True)
        audio_io.write_wav(rng.standard_normal(int(rng.integers(8000, 40000))) * 0.1, str(p), "float32")
        recs.append({"utterance_id": f"spk/u{k:02d}", "input": str(p), "output": str(tmp_path / "OUT" / f"u{k:02d}.wav")})
    return recs


def test_parse_manifest(tmp_path):
    from paper_1712_03439_b200 import batch, roomsim

    p = tmp_path / "m.jsonl"
    _write_manifest(p, {"spec": "config4", "seed": 9, "epoch": 3, "eta_db": 10.0},
                    [{"utterance_id": "a", "input": "x.wav", "output": "y.wav"},
                     {"utterance_id": "b", "input": "x2.wav", "output": "y2.wav", "noises": ["n.wav"]}])
    m = batch.parse_manifest(str(p))
    assert (m.spec, m.seed, m.epoch, m.eta_db) == ("config4", 9, 3, 10.0)
    assert [r.utterance_id for r in m.records] == ["a", "b"] and m.records[1].noises == ("n.wav",)
    _write_manifest(p, None, [{"utterance_id": "a", "input": "x", "output": "y"},
                              {"utterance_id": "a", "input": "x", "output": "z"}])
    with pytest.raises(roomsim.ConfigError, match="duplicate"):
        batch.parse_manifest(str(p))
    _write_manifest(p, None, [{"utterance_id": "a", "input": "", "output": "y"}])
    with pytest.raises(roomsim.ConfigError):
        batch.parse_manifest(str(p))
    p.write_text("{not json\n")
    with pytest.raises(roomsim.ConfigError):
        batch.parse_manifest(str(p))
    p.write_text("")
    assert batch.parse_manifest(str(p)).records == []


def test_scenes_are_keyed_by_utterance_id():
    from paper_1712_03439_b200 import scenes

    spec = scenes.spec_config2(2)
    a = scenes.sample_scene(spec, "spk/u01", 0)
    b = scenes.sample_scene(spec, "spk/u01", 0)
    c = scenes.sample_scene(spec, "spk/u01", 1)
    assert np.array_equal(a.room, b.room) and np.array_equal(a.src, b.src)
    assert not np.array_equal(a.room, c.room)


def _run(manifest, *extra):
    r = subprocess.run([sys.executable, "-m", "paper_1712_03439_b200.batch", str(manifest)] + list(extra),
                       cwd=ROOT, capture_output=True, text=True, timeout=900)
    summary = json.loads(r.stdout.strip().splitlines()[-1]) if r.stdout.strip() else None
    return r, summary


@pytest.mark.gpu
def test_batch_parallelism_and_errors(tmp_path):
    recs = _inputs(tmp_path, 20)
    header = {"spec": "config3", "seed": 4, "epoch": 1}
    m = tmp_path / "m.jsonl"
    _write_manifest(m, header, recs)
    outs = {}
    for P, bs in ((1, 256), (2, 3)):
        for r_ in recs:
            r_["output"] = str(tmp_path / f"out{P}" / os.path.basename(r_["input"]))
        _write_manifest(m, header, recs)
        r, s = _run(m, "--parallelism", str(P), "--batch-utts", str(bs))
        assert r.returncode == 0, r.stderr[-2000:]
        assert s["count"] == 20 and s["processed"] == 20 and s["failures"] == 0
        outs[P] = [open(r_["output"], "rb").read() for r_ in recs]
    assert outs[1] == outs[2]  # identical output bytes for parallelism 1 vs 8
    # empty manifest: success, zero processed
    e = tmp_path / "empty.jsonl"
    e.write_text("")
    r, s = _run(e)
    assert r.returncode == 0 and s["count"] == 0 and s["processed"] == 0
    # one unreadable input among 5: 4 succeed, nonzero exit, failure named
    five = _inputs(tmp_path, 5, seed=6)
    five[2]["input"] = str(tmp_path / "does_not_exist.wav")
    _write_manifest(m, header, five)
    r, s = _run(m, "--parallelism", "2")
    assert r.returncode != 0 and s["processed"] == 4 and s["failed"] == [five[2]["utterance_id"]]
    assert five[2]["utterance_id"] in r.stderr


@pytest.mark.gpu
def test_batch_output_matches_reference(tmp_path):
    """A record rendered by cmd_batch equals the reference render of the same scene."""
    import oracle
    from paper_1712_03439_b200 import audio_io, batch

    recs = _inputs(tmp_path, 3, seed=7)
    m = tmp_path / "m.jsonl"
    _write_manifest(m, {"spec": "config3", "seed": 4, "epoch": 0}, recs)
    r, s = _run(m)
    assert r.returncode == 0, r.stderr[-2000:]
    man = batch.parse_manifest(str(m))
    b, ok, failed = batch.build_batch(man, man.records, eta_db=20.0)
    assert len(ok) == 3 and not failed
    ref = oracle.reference() if oracle.reference_available() else oracle.port()
    o_out, o_len, *_ = ref.render_batch(b, threads=8)
    for u, rec in enumerate(man.records):
        got, _ = audio_io.read_wav(rec.output)
        want = np.stack([b.channel(o_out, u, j, o_len[u]) for j in range(got.shape[0])])
        assert got.shape == want.shape
        assert np.abs(got - want).max() <= 1e-5 * np.abs(want).max()
