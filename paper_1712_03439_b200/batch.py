"""cmd_batch: dataset noisification from a JSON-lines manifest (SURVEY.md §8f
row 3), on top of the batched GPU render.

    python -m paper_1712_03439_b200.batch MANIFEST [--epoch E] [--parallelism P] [--eta-db D]
                                                   [--batch-utts B] [--format float32|pcm16]

Manifest (JSON lines; SPEC.md:392-395 ``Manifest``): an optional header line with the global
``SamplerSpec`` reference and defaults, then one record per utterance::

    {"spec": "config3", "seed": 2, "epoch": 0, "eta_db": 20.0, "noise": "synthetic"}
    {"utterance_id": "spk1/utt001", "input": "in/utt001.wav", "output": "out/utt001.wav"}
    {"utterance_id": "spk1/utt002", "input": "in/utt002.wav", "output": "out/utt002.wav",
     "noises": ["noise/babble.wav", "noise/car.wav"]}

Each record's scene (room, reflection, placements, SNRs) is ``sample_scene(spec,
utterance_id, epoch)`` — a pure function of (seed, utterance id, epoch).
The record's input WAV (mono, 16 kHz) is the target; the noise sources take the record's
``noises`` WAVs in order (cycled, trimmed or zero-padded to the target's length) or, by
default, synthetic N(0, 0.1) noise keyed by (seed, utterance id, epoch, source).  The output is
one J-channel WAV per record.

Records are rendered in GPU batches through ``rs_render_batch``; ``--parallelism P`` runs P
worker processes (one CUDA context each, records dealt round-robin).  A render's bytes do not
depend on the batch composition (the K4 variant and power partials are per-pair functions,
power.cuh), so the outputs are identical for every P and batch size.
Unreadable or invalid records are logged and skipped; the exit status is nonzero if any
record failed.  The last line is a JSON summary: count, failures, wall time, mean ms per
utterance.
"""
from __future__ import annotations

import argparse
import dataclasses
import hashlib
import json
import os
import sys
import time
from typing import Optional

import numpy as np


@dataclasses.dataclass
class Record:
    utterance_id: str
    input: str
    output: str
    noises: tuple = ()


@dataclasses.dataclass
class Manifest:
    records: list
    spec: str = "config3"
    seed: int = 2
    epoch: int = 0
    eta_db: Optional[float] = None  # None: the spec's config default
    noise: str = "synthetic"


def parse_manifest(path: str) -> Manifest:
    """JSON lines: an optional header (has no "utterance_id"), then records.  Raises
    ConfigError on a malformed line, a missing field or a duplicate utterance id."""
    from .roomsim import ConfigError

    m = Manifest(records=[])
    seen = set()
    with open(path) as f:
        for ln, line in enumerate(f, 1):
            line = line.strip()
            if not line:
                continue
            try:
                d = json.loads(line)
            except json.JSONDecodeError as e:
                raise ConfigError(f"{path}:{ln}: not JSON ({e})") from e
            if "utterance_id" not in d:
                if m.records:
                    raise ConfigError(f"{path}:{ln}: header after the first record")
                m.spec = str(d.get("spec", m.spec))
                m.seed = int(d.get("seed", m.seed))
                m.epoch = int(d.get("epoch", m.epoch))
                m.eta_db = d.get("eta_db", m.eta_db)
                m.noise = str(d.get("noise", m.noise))
                continue
            uid, inp, out = str(d["utterance_id"]), d.get("input"), d.get("output")
            if not inp or not out:
                raise ConfigError(f"{path}:{ln}: record needs non-empty input and output paths")
            if uid in seen:
                raise ConfigError(f"{path}:{ln}: duplicate utterance_id {uid!r}")
            seen.add(uid)
            m.records.append(Record(uid, str(inp), str(out), tuple(d.get("noises", ()))))
    return m


def _spec(name: str, seed: int):
    from . import scenes

    fn = getattr(scenes, "spec_" + name, None) or (scenes.spec_config2 if name == "config3" else None)
    if fn is None:
        from .roomsim import ConfigError

        raise ConfigError(f"unknown sampler spec {name!r}")
    return fn(seed)


def _plan(name: str):
    from . import scenes

    # the config's FFT-size rule and default truncation (scenes.CONFIGS)
    b = scenes.CONFIGS.get(name, scenes.config3)(n_utt=1, signals=False)
    return b.plan_rule, b.forced_fft_size, b.eta_db


def _noise_signal(seed: int, uid: str, epoch: int, src: int, n: int) -> np.ndarray:
    key = hashlib.blake2b(f"{seed}/noise/{uid}/{epoch}/{src}".encode(), digest_size=16).digest()
    g = np.random.Generator(np.random.Philox(key=int.from_bytes(key, "little")))
    return g.standard_normal(n, dtype=np.float32) * np.float32(0.1)


def _fit(x: np.ndarray, n: int) -> np.ndarray:
    """x cycled / trimmed to n samples."""
    if x.size == 0:
        return np.zeros(n, np.float32)
    reps = -(-n // x.size)
    return np.tile(x, reps)[:n].astype(np.float32)


def build_batch(m: Manifest, recs: list, eta_db: float):
    """A SceneBatch of `recs` (scenes from the sampler, signals from the WAVs); returns
    (batch, records that failed to load as (record, message))."""
    from . import audio_io, scenes

    spec = _spec(m.spec, m.seed)
    plan_rule, forced, _ = _plan(m.spec)
    ok, failed, sigs, scs = [], [], [], []
    for r in recs:
        try:
            x, rate = audio_io.read_wav(r.input, expect_rate=16000)
            if x.shape[0] != 1:
                raise audio_io.FormatError(f"{r.input}: input must be mono, has {x.shape[0]} channels")
            target = x[0].astype(np.float32)
            if target.size == 0:
                raise audio_io.FormatError(f"{r.input}: empty audio")
            sc = scenes.sample_scene(spec, r.utterance_id, m.epoch)
            I = sc.src.shape[0]
            src = [target]
            for i in range(1, I):
                if r.noises:
                    nx_, _ = audio_io.read_wav(r.noises[(i - 1) % len(r.noises)], expect_rate=16000)
                    src.append(_fit(nx_[0].astype(np.float32), target.size))
                else:
                    src.append(_noise_signal(m.seed, r.utterance_id, m.epoch, i, target.size))
        except Exception as e:  # per-record failure: logged by the caller, the batch goes on
            failed.append((r, f"{type(e).__name__}: {e}"))
            continue
        ok.append(r)
        scs.append(sc)
        sigs.extend(src)
    if not ok:
        return None, ok, failed
    I = np.array([s.src.shape[0] for s in scs])
    J = np.array([s.mic.shape[0] for s in scs])
    lens = np.array([s.size for s in sigs], np.int64)
    offs = scenes.signal_offsets(lens)
    buf = np.zeros(int((offs + lens).max()), np.float32)
    for o, x in zip(offs, sigs):
        buf[o : o + x.size] = x
    b = scenes.SceneBatch(
        src_begin=np.concatenate([[0], np.cumsum(I)]).astype(np.int64),
        mic_begin=np.concatenate([[0], np.cumsum(J)]).astype(np.int64),
        room_dims=np.stack([s.room for s in scs]), reflection=np.array([s.refl for s in scs]),
        sample_rate=np.full(len(scs), scenes.FS), speed_of_sound=np.full(len(scs), scenes.C0),
        image_order=np.array([s.order for s in scs], np.int32), max_taps=np.array([s.horizon for s in scs], np.int64),
        src_pos=np.concatenate([s.src for s in scs]), mic_pos=np.concatenate([s.mic for s in scs]),
        snr_db=np.concatenate([s.snr_db for s in scs]),
        sig_off=offs, sig_len=lens, signals=buf, eta_db=eta_db, plan_rule=plan_rule,
        forced_fft_size=forced, name="manifest", seed=m.seed)
    return b, ok, failed


def run_records(m: Manifest, recs: list, *, eta_db: float, batch_utts: int, fmt: str, device: int = 0,
                log=sys.stderr):
    """Render and write `recs`; returns (processed, failures as (utterance_id, message))."""
    from . import audio_io, roomsim

    ctx = roomsim.Context(device)
    done, failures = 0, []
    try:
        for k in range(0, len(recs), batch_utts):
            b, ok, failed = build_batch(m, recs[k:k + batch_utts], eta_db)
            for r, msg in failed:
                print(f"[cmd_batch] FAILED {r.utterance_id}: {msg}", file=log, flush=True)
                failures.append((r.utterance_id, msg))
            if b is None:
                continue
            try:
                res = roomsim.render_batch(b, ctx=ctx)
            except roomsim.Error:
                # isolate the failing record(s): render one by one
                res = None
            if res is None:
                for u, r in enumerate(ok):
                    try:
                        sb = b.subset([u])
                        rr = roomsim.render_batch(sb, ctx=ctx)
                        _write(audio_io, sb, rr, 0, r, fmt)
                        done += 1
                    except Exception as e:
                        msg = f"{type(e).__name__}: {e}"
                        print(f"[cmd_batch] FAILED {r.utterance_id}: {msg}", file=log, flush=True)
                        failures.append((r.utterance_id, msg))
                continue
            for u, r in enumerate(ok):
                try:
                    _write(audio_io, b, res, u, r, fmt)
                    done += 1
                except Exception as e:
                    msg = f"{type(e).__name__}: {e}"
                    print(f"[cmd_batch] FAILED {r.utterance_id}: {msg}", file=log, flush=True)
                    failures.append((r.utterance_id, msg))
    finally:
        ctx.close()
    return done, failures


def _write(audio_io, b, res, u: int, r: Record, fmt: str) -> None:
    J = int(b.mic_begin[u + 1] - b.mic_begin[u])
    chans = np.stack([b.channel(res.out, u, j, res.out_len[u]) for j in range(J)])
    d = os.path.dirname(os.path.abspath(r.output))
    os.makedirs(d, exist_ok=True)
    audio_io.write_wav(chans, r.output, fmt, 16000)


def _worker(rank: int, world: int, argv: list, q) -> None:
    a = _args(argv)
    m = parse_manifest(a.manifest)
    if a.epoch is not None:
        m.epoch = a.epoch
    eta = a.eta_db if a.eta_db is not None else (m.eta_db if m.eta_db is not None else _plan(m.spec)[2])
    recs = m.records[rank::world]
    done, failures = run_records(m, recs, eta_db=float(eta), batch_utts=a.batch_utts, fmt=a.format)
    q.put((done, failures))


def _args(argv=None):
    ap = argparse.ArgumentParser(prog="python -m paper_1712_03439_b200.batch")
    ap.add_argument("manifest")
    ap.add_argument("--epoch", type=int, default=None, help="overrides the manifest header's epoch")
    ap.add_argument("--parallelism", type=int, default=1, help="worker processes (GPU contexts)")
    ap.add_argument("--eta-db", type=float, default=None, help="RIR cut; 0 = none (default: manifest / spec)")
    ap.add_argument("--batch-utts", type=int, default=256, help="utterances per GPU render")
    ap.add_argument("--format", choices=["float32", "pcm16"], default="float32")
    return ap.parse_args(argv)


def main(argv=None) -> int:
    argv = list(sys.argv[1:] if argv is None else argv)
    a = _args(argv)
    t0 = time.perf_counter()
    try:
        m = parse_manifest(a.manifest)
    except Exception as e:
        print(f"[cmd_batch] invalid manifest: {type(e).__name__}: {e}", file=sys.stderr)
        return 2
    done, failures = 0, []
    if m.records:
        import multiprocessing as mp

        P = max(1, min(a.parallelism, len(m.records)))
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        procs = [ctx.Process(target=_worker, args=(r, P, argv, q)) for r in range(P)]
        for p in procs:
            p.start()
        for _ in procs:
            d, f = q.get()
            done += d
            failures += f
        for p in procs:
            p.join()
            if p.exitcode != 0:
                failures.append(("<worker>", f"worker exited with {p.exitcode}"))
    wall = time.perf_counter() - t0
    summary = {"count": len(m.records), "processed": done, "failures": len(failures),
               "failed": sorted(u for u, _ in failures), "wall_s": wall,
               "mean_ms_per_utterance": 1e3 * wall / len(m.records) if m.records else 0.0}
    print(json.dumps(summary), flush=True)
    return 1 if failures else 0


if __name__ == "__main__":
    sys.exit(main())
