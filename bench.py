#!/usr/bin/env python3
"""Benchmark of the room-simulation hot path (BASELINE.json metric).

Metric: simulated audio-seconds per second (Σ_utterances N_x / 16 kHz; the
target's duration, counted once per utterance) for BASELINE config 4: 4096
utterances x (1 target + 5 noises) x 2 mics, image-method RIRs truncated at
-20 dB, N = bit_ceil(2 N_h), synth -> cut -> OLA -> SNR mix all on device.

  python bench.py [--gpus N --steps K --warmup W]          # our CUDA path
  python bench.py --impl reference [...]                    # the reference's CPU path
  python bench.py --gpus 2 --dry-run                        # CPU: spawn/shard/reduce only

Our arm prints `value` (inputs resident in HBM, CUDA events on the launching
stream, max over ranks), `e2e` (host pinned buffers through the C-ABI with
H2D/D2H in the timed region), the OLA kernel's `roofline` (with a per-size
breakdown), the reference CPU `cpu_baseline` (rank 0, N = 1, bounded sample),
`parity` (that sample rendered on the GPU against the reference), `clocks` and
`gpu_launches`.

Multi-GPU: one process per GPU — torchrun's ranks, or, when WORLD_SIZE is
unset and --gpus N > 1, N processes spawned here (127.0.0.1 rendezvous).
Utterances are sharded with no collective on the data path: "scaling":
"strong" by default (the config's 4096 utterances LPT-partitioned over the
ranks by predicted work), "weak" on request (every rank renders
its own set of utterance ids).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "simulated audio-sec/sec"
UNIT = "audio-s/s"


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="config4", choices=["config2", "config3", "config4", "config5"])
    ap.add_argument("--utterances", type=int, default=0, help="total (strong) or per GPU (weak); 0 = config default")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="strong",
                    help="strong (default): the config's utterances sharded over the GPUs (BASELINE config 4: "
                         "4096 utterances over 1/2/4/8 B200); weak: every GPU renders its own set")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU only (gloo): spawn / shard / max-over-ranks logic without rendering")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--gather", action="store_true",
                    help="after the timed region: gather every rank's mixed outputs on rank 0 (NCCL; optional, "
                         "not on the render path)")
    ap.add_argument("--no-breakdown", action="store_true",
                    help="skip the diagnostic renders after the timed region (per-size K4, K4 without the mix epilogue)")
    ap.add_argument("--cpu-sample-utts", type=int, default=0)
    ap.add_argument("--seed", type=int, default=4)
    return ap.parse_args(argv)


DEFAULT_UTTS = {"config2": 128, "config3": 128, "config4": 4096, "config5": 512}


# ---- the workload and its shards ------------------------------------------------
def n_config(args) -> int:
    return args.utterances or DEFAULT_UTTS[args.config]


def full_batch(args, signals=False, first_utt=0):
    from paper_1712_03439_b200 import scenes

    return scenes.CONFIGS[args.config](n_utt=n_config(args), seed=args.seed, signals=signals, first_utt=first_utt)


def rank_batch(args, rank, world):
    """The scenes rank `rank` renders: its LPT shard of the workload (strong) or its
    own block of utterance ids (weak).  Returns (batch, total utterances of the job)."""
    from paper_1712_03439_b200 import shard

    n = n_config(args)
    if args.scaling == "weak":
        return full_batch(args, first_utt=rank * n), n * world
    b, _ = shard.shard_batch(full_batch(args), rank, world)
    return b, n


def workload_config(args, world):
    """The `config` object both arms print (same keys, same values)."""
    from paper_1712_03439_b200 import scenes

    b = scenes.CONFIGS[args.config](n_utt=1, seed=args.seed, signals=False)
    n = n_config(args)
    return {"workload": args.config, "utterances": n * world if args.scaling == "weak" else n,
            "scaling": args.scaling, "seed": args.seed, "eta_db": b.eta_db,
            "fft_rule": {0: "choose_plan", 1: f"forced {b.forced_fft_size}", 2: "bit_ceil(2*N_h)"}[b.plan_rule]}


# ---- clocks (sampled during the timed region) -----------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # the timed region is a few hundred ms: start it only once sampling runs
            t0 = time.perf_counter()
            while not self.lines and time.perf_counter() - t0 < 5.0:
                time.sleep(0.01)
            self.skip = len(self.lines)  # samples before the timed region
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines[getattr(self, "skip", 0):] or self.lines[-1:]:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---- CPU reference runs -------------------------------------------------------
def cpu_sample(args, want: int):
    """Deterministic subsample of the whole workload (every k-th utterance) with host
    N(0, 0.1) signals: what the CPU baseline renders (and the GPU, for `parity`)."""
    full = full_batch(args)
    k = max(1, full.n_utt // max(want, 1))
    ids = np.arange(0, full.n_utt, k)[:want]
    sub = full.subset(ids)
    g = np.random.Generator(np.random.Philox(key=99))
    sub.signals = g.standard_normal(sub.total_samples, dtype=np.float32) * np.float32(0.1)
    return sub, k


def run_cpu_reference(sub, threads: int, tuned: bool = True):
    """The reference (oracle/_ref: the unmodified reference headers, compiled) renders
    `sub` on `threads` host threads; the C restatement if that build is absent."""
    import oracle

    kind = "reference" if oracle.reference_available() else "port"
    lib = oracle.reference() if kind == "reference" else oracle.port()
    if kind == "reference":
        lib.lib.ref_set_malloc_tuning(1 if tuned else 0)
    t0 = time.perf_counter()
    res = lib.render_batch(sub, threads=threads)
    dt = time.perf_counter() - t0
    return sub.audio_seconds / dt, dt, kind, res


def reference_arm(args, rank, world):
    """--impl reference: the reference's own CPU path (oracle/_ref) on all host cores,
    on our arm's config / metric / unit; each step renders a bounded deterministic
    sample of the workload.  Rank 0 alone runs it."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    # each step ~3-5 s of the host's cores: the whole K+W run stays within minutes
    want = args.cpu_sample_utts or max(16, 24 * threads)
    sub, k = cpu_sample(args, want)
    for _ in range(args.warmup):
        run_cpu_reference(sub, threads)
    secs = []
    kind = None
    for _ in range(args.steps):
        _, dt, kind, _ = run_cpu_reference(sub, threads)
        secs.append(dt)
    value = float(sub.audio_seconds * args.steps / sum(secs))
    sample = (f"{sub.n_utt} of {n_config(args)} {args.config} utterances (every {k}th, "
              f"{sub.audio_seconds:.1f} audio-s, {sub.n_pairs} pairs) per step")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(secs) / args.steps,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: seeded N(0,0.1) signals, sampled image-method rooms",
        "config": workload_config(args, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample,
                         "note": "reference radix-2 CPU path (FFTW3 unavailable); malloc mmap_threshold=64MiB"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def dry_run(args, rank, world):
    """CPU check of the multi-rank plumbing (gloo): every rank builds its shard; rank 0
    checks the union covers every utterance exactly once and prints the shards."""
    import torch
    import torch.distributed as dist

    from paper_1712_03439_b200 import shard

    b, total = rank_batch(args, rank, world)
    ids = [int(u) for u in b.ids]
    w = shard.predicted_work(b)
    mine = (ids, float(b.audio_seconds), int(b.n_pairs), float(w.sum()), float(w.max()) if w.size else 0.0)
    got = [None] * world
    if world > 1:
        dist.all_gather_object(got, mine)
    else:
        got = [mine]
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)  # stands in for a rank's step time
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        allids = sorted(u for g in got for u in g[0])
        want = list(range(total))
        line = {"dry_run": True, "n_gpus": world, "scaling": args.scaling, "config": workload_config(args, world),
                "shard_utterances": [len(g[0]) for g in got], "shard_pairs": [g[2] for g in got],
                "shard_audio_seconds": [round(g[1], 3) for g in got],
                "shard_predicted_work": [g[3] for g in got], "max_utterance_work": max(g[4] for g in got),
                "covers_every_utterance_once": allids == want, "max_over_ranks": float(t[0])}
        print(json.dumps(line), flush=True)


# ---- our arm ---------------------------------------------------------------------
def ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_1712_03439_b200 import roomsim, scenes

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    batch, total_utts = rank_batch(args, rank, world)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1000 + rank)
    signals = torch.randn(max(batch.total_samples, 1), generator=gen, device=dev, dtype=torch.float32).mul_(0.1)
    out = torch.empty(max(batch.out_total, 1), device=dev, dtype=torch.float32)
    stream = torch.cuda.current_stream(dev)
    ctx = roomsim.Context(local_rank)
    ctx.set_stream(stream.cuda_stream)
    ctx.set_profiling(True)

    last = [None]

    def step():
        # the result arrays (layouts, gains, powers) of the previous step are reused
        last[0] = roomsim.render_batch(batch, ctx=ctx, device_signals_ptr=signals.data_ptr(),
                                       device_out_ptr=out.data_ptr(), result=last[0])
        return last[0]

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(vals):
        t = torch.tensor(vals, device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return [float(v) for v in t]

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    clk = ClockSampler(local_rank)
    clk.start()
    barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ola_ms, flops, launches = 0.0, 0.0, 0
    stages = {}
    e0.record(stream)
    for _ in range(args.steps):
        step()
        t = ctx.last_timing()
        ola_ms += t["ola_ms"]
        flops += t["ola_flops"]
        launches += t["launches"]
        for k, v in ctx.stage_times().items():
            stages[k] = stages.get(k, 0.0) + v / args.steps
    e1.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    clocks = clk.stop()
    ms = e0.elapsed_time(e1) / args.steps
    alg_bytes = ctx.last_timing()["alg_bytes"]
    mix_fused, mix_channels = ctx.mix_counts()
    ms_max, ola_ms_max = max_over_ranks([ms, ola_ms / args.steps])
    aud = torch.tensor([batch.audio_seconds, batch.n_pairs], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(aud, op=dist.ReduceOp.SUM)
    total_audio, total_pairs = float(aud[0]), int(aud[1])
    value = total_audio / (ms_max / 1e3)

    # ---- optional final gather of the mixed outputs on rank 0 (north star: NCCL only here) -----
    gather = None
    if args.gather:
        from paper_1712_03439_b200 import shard

        res = step()
        torch.cuda.synchronize(dev)
        barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        got = shard.gather_outputs(out, batch.ids, res.out_len)
        g1.record(stream)
        torch.cuda.synchronize(dev)
        ms_g = max_over_ranks([g0.elapsed_time(g1)])[0]
        if rank == 0:
            gather = {"ms": ms_g, "bytes": int(sum(4 * o.numel() for _, _, o in got)), "ranks": len(got),
                      "utterances": int(sum(len(i) for i, _, _ in got)),
                      "what": "shard.gather_outputs: every rank's output buffer, utterance ids and lengths to "
                              "rank 0 (torch.distributed gather over NCCL), after the timed region"}
        del got

    # ---- two renders in flight (steady-state stream of batches: the paper's on-the-fly data
    # generation) — a second context on its own streams and buffers renders the same batch into a
    # second output buffer from a second host thread, so one render's fill time (host preparation,
    # K1, the wait for the RIR summary, planning) hides under the other's K4.  Not the headline:
    # `value` above is one render at a time.  Host-timed between device synchronizations (every
    # render call returns after its device work). -----------------------------------------------
    in_flight2 = None
    if not args.no_breakdown:
        import threading

        ctx2 = roomsim.Context(local_rank)
        out2 = torch.empty(max(batch.out_total, 1), device=dev, dtype=torch.float32)
        n_each = max(2, args.steps // 2)

        errs = []

        def stream_of_batches(c, o, n, res):
            try:
                for _ in range(n):
                    res[0] = roomsim.render_batch(batch, ctx=c, device_signals_ptr=signals.data_ptr(),
                                                  device_out_ptr=o.data_ptr(), result=res[0])
            except Exception as e:  # noqa: BLE001 - reported below
                errs.append(repr(e))

        for c, o in ((ctx, out), (ctx2, out2)):  # warm both contexts' buffers
            stream_of_batches(c, o, 2, [None])
        torch.cuda.synchronize(dev)
        barrier()
        ths = [threading.Thread(target=stream_of_batches, args=(c, o, n_each, [None]))
               for c, o in ((ctx, out), (ctx2, out2))]
        t0 = time.perf_counter()
        for th in ths:
            th.start()
        for th in ths:
            th.join()
        torch.cuda.synchronize(dev)
        if errs:
            raise RuntimeError("two_in_flight: " + "; ".join(errs))
        ms2 = max_over_ranks([(time.perf_counter() - t0) * 1e3 / (2 * n_each)])[0]
        in_flight2 = {"value": total_audio / (ms2 / 1e3), "unit": UNIT, "ms_per_render": ms2,
                      "renders": 2 * n_each,
                      "what": "two contexts, two host threads, each rendering the batch n times back to back: "
                              "steady-state throughput of a stream of batches; host-timed"}
        ctx2.close()
        del out2

    # ---- per-size K4 breakdown: one diagnostic render with the K4 launches serialized and
    # timed one by one (outside the timed region) --------------------------------------
    k4_sizes, k4_alone = None, None
    try:
        if args.no_breakdown:
            raise AttributeError
        ctx.set_profiling(2)
        step()
        k4_sizes = ctx.k4_breakdown()
        ctx.set_profiling(True)
        # and one with every channel through mix_kernel: K4 alone, the mix alone
        ctx.set_fused_mix(0)
        step()
        st_plain = ctx.stage_times()
        k4_alone = {"ola_ms": st_plain["ola"], "mix_ms": st_plain["gain_mix"],
                    "flops": ctx.last_timing()["ola_flops"]}
        ctx.set_fused_mix(-1)
    except AttributeError:
        pass

    # ---- e2e: host pinned buffers through rs_render_batch (H2D + D2H inside) ----
    e2e = None
    if not args.no_e2e:
        h_sig = torch.empty(max(batch.total_samples, 1), dtype=torch.float32, pin_memory=True)
        h_sig.copy_(signals)
        h_out = torch.empty(max(batch.out_total, 1), dtype=torch.float32, pin_memory=True)
        batch.signals = h_sig.numpy()
        hout = h_out.numpy()
        roomsim.render_batch(batch, ctx=ctx, out=hout)  # warm
        barrier()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        e0.record(stream)
        for _ in range(args.steps):
            roomsim.render_batch(batch, ctx=ctx, out=hout)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        wall = (time.perf_counter() - t0) / args.steps * 1e3
        ev = e0.elapsed_time(e1) / args.steps
        te = max_over_ranks([max(wall, ev)])[0]
        e2e = {"value": total_audio / (te / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(4 * batch.total_samples), "d2h_bytes_per_step": int(4 * batch.out_total),
               "ms_per_step": te, "what": "rs_render_batch with pinned host signals/outputs: per-chunk H2D of the "
                                          "signals and D2H of the mixed channels inside the timed region"}
        batch.signals = None

    # ---- epoch loop: source signals generated in HBM (rs_generate_signals, SURVEY.md §8f
    # row 1) + the render, per step; no host staging of the 12.6 GB of inputs ----------------
    epoch_loop = None
    if not args.no_e2e:
        spec = roomsim.sampler_spec(getattr(scenes, "spec_" + args.config)(args.seed))
        gen_plan = roomsim.SignalPlan(spec, batch, seed=args.seed)  # per-batch tables, built once
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

        def epoch_step(ep):
            g0.record(stream)
            gen_plan.generate(signals.data_ptr(), epoch=ep, stream=stream.cuda_stream)
            g1.record(stream)
            return step()

        epoch_step(0)
        barrier()
        torch.cuda.synchronize(dev)
        e0.record(stream)
        for k in range(args.steps):
            epoch_step(k + 1)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        gen_ms = g0.elapsed_time(g1)
        ms_ep = max_over_ranks([e0.elapsed_time(e1) / args.steps])[0]
        epoch_loop = {"value": total_audio / (ms_ep / 1e3), "unit": UNIT, "ms_per_step": ms_ep,
                      "signal_gen_ms": gen_ms,
                      "what": "per step: N(0, 0.1) source signals generated in HBM by rs_generate_signals "
                              "(Philox, bit-exact with the host fixture generator) + rs_render_batch_device; "
                              "scene metadata from the host sampler; no host<->device staging of samples"}

    # ---- log-Mel front end on the rendered channels -----------------
    logmel = None
    if not args.no_e2e:
        res = step()
        J = np.diff(batch.mic_begin)
        ch_off = np.concatenate([batch.out_off[u] + np.arange(J[u]) * batch.out_stride[u] for u in range(batch.n_utt)])
        ch_len = np.repeat(res.out_len, J)
        S = np.array([roomsim.logmel_shape(int(n))[1] for n in ch_len], np.int64)
        f_off = np.concatenate([[0], np.cumsum(S * 512)[:-1]]).astype(np.int64)
        feat = torch.empty(max(int(S.sum()) * 512, 1), dtype=torch.float32, device=dev)
        roomsim.logmel_device(out.data_ptr(), ch_off, ch_len, feat.data_ptr(), f_off, ctx=ctx)  # warm
        lm_ms = 0.0
        for _ in range(args.steps):
            roomsim.logmel_device(out.data_ptr(), ch_off, ch_len, feat.data_ptr(), f_off, ctx=ctx)
            lm_ms += ctx.last_timing()["ola_ms"]
        frames = int(sum(3 * (s_ - 1) + 4 for s_ in S if s_ > 0))
        # the render with the log-Mel fused into the mix, waveforms never written (features only)
        foff, ftot = roomsim.feature_layout(batch)
        fused = torch.empty(max(ftot, 1), dtype=torch.float32, device=dev)
        fstep = lambda: roomsim.render_features(batch, device_signals_ptr=signals.data_ptr(),  # noqa: E731
                                                feat_ptr=fused.data_ptr(), feat_off=foff, ctx=ctx)
        fstep()
        barrier()
        torch.cuda.synchronize(dev)
        e0.record(stream)
        for _ in range(args.steps):
            fstep()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ms_f = max_over_ranks([e0.elapsed_time(e1) / args.steps])[0]
        # features and waveforms: the mix in the K4 epilogue, the log-Mel reading the channels back
        wstep = lambda: roomsim.render_features(batch, device_signals_ptr=signals.data_ptr(),  # noqa: E731
                                                feat_ptr=fused.data_ptr(), feat_off=foff,
                                                device_out_ptr=out.data_ptr(), ctx=ctx)
        wstep()
        barrier()
        torch.cuda.synchronize(dev)
        e0.record(stream)
        for _ in range(args.steps):
            wstep()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ms_w = max_over_ranks([e0.elapsed_time(e1) / args.steps])[0]
        logmel = {"ms_per_step": lm_ms / args.steps, "channels": int(ch_len.size), "frames": frames,
                  "stacked_vectors": int(S.sum()),
                  "frames_per_s": frames / (lm_ms / args.steps / 1e3) if lm_ms > 0 else None,
                  "what": "128 log-Mel, 32 ms Hann / 10 ms hop, 125-7500 Hz, 4-frame stacks every 3rd "
                          "(PAPER.md:452-460) of every rendered channel; device-timed kernel",
                  "fused_render_features": {
                      "ms_per_step": ms_f, "value": total_audio / (ms_f / 1e3), "unit": UNIT,
                      "vs_render_plus_logmel_ms": ms_max + lm_ms / args.steps,
                      "what": "rs_render_features_device: the whole render with the log-Mel computed inside the "
                              "mix kernel from shared memory; waveforms not written (features only)"},
                  "render_features_with_waveforms": {
                      "ms_per_step": ms_w, "value": total_audio / (ms_w / 1e3), "unit": UNIT,
                      "what": "rs_render_features_device with an output buffer: waveforms mixed in the K4 "
                              "epilogue, the log-Mel kernel reads them back; features bit-identical"}}
        del feat, fused

    # ---- roofline of the OLA filter kernels (K4) -------------------------------------
    props = torch.cuda.get_device_properties(dev)
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except Exception:
        pass
    sm_max = float(peaks.get("sm_max_mhz") or clocks.get("sm_max_mhz") or 1965.0)
    fp32_peak = props.multi_processor_count * 128 * 2 * sm_max * 1e6 / 1e12  # TFLOP/s
    per_step_flops = flops / args.steps
    achieved = per_step_flops / (ola_ms / args.steps / 1e3) / 1e12 if ola_ms > 0 else None
    hbm = float(peaks.get("hbm_gbs") or 6543.1)
    traffic, traffic_src = None, None
    try:  # K4 DRAM bytes per render, from the committed ncu launch list of this workload
        with open(os.path.join(ROOT, "profiles", "k4_traffic.json")) as f:
            tj = json.load(f)
        if tj.get("workload") == args.config and tj.get("utterances_per_rank") == batch.n_utt:
            traffic, traffic_src = tj["dram_bytes_per_render"], tj["source"] + "; " + tj["note"]
    except Exception:
        pass
    ser = None
    if k4_sizes:
        for r in k4_sizes:
            r["tflops"] = r["flops"] / (r["ms"] / 1e3) / 1e12 if r["ms"] > 0 else None
            r["frac"] = r["tflops"] / fp32_peak if r["tflops"] else None
            r["exec_frac"] = r["exec_flops"] / (r["ms"] / 1e3) / 1e12 / fp32_peak if r["ms"] > 0 else None
        ms_ser = sum(r["ms"] for r in k4_sizes)
        if ms_ser > 0:
            ser = {"ms": ms_ser,
                   "frac": sum(r["flops"] for r in k4_sizes) / (ms_ser / 1e3) / 1e12 / fp32_peak,
                   "exec_frac": sum(r["exec_flops"] for r in k4_sizes) / (ms_ser / 1e3) / 1e12 / fp32_peak}
    roofline = {
        "bound": "fp32", "achieved": achieved, "peak": fp32_peak, "unit": "TFLOP/s",
        "frac": achieved / fp32_peak if achieved else None, "traffic": traffic,
        "traffic_unit": "DRAM bytes per step (all K4 launches)", "traffic_source": traffic_src,
        "kernel": "K4 (ola_ipc_kernel<N>, ola_ip_kernel<M>, ola_small_kernel<M>, ola2_kernel<N>, four-step stages), "
                  "all FFT sizes of one render, with the SNR-scaled mix in the launches' epilogue",
        "ola_ms_per_step": ola_ms / args.steps,
        "alg_flops_per_step": per_step_flops,
        "alg_bytes_per_step": alg_bytes,
        "hbm_time_ms": alg_bytes / (hbm * 1e9) * 1e3,
        "peak_source": f"derived: {props.multi_processor_count} SMs x 128 FP32 lanes x 2 x {sm_max:.0f} MHz "
                       "(sm_max_mhz of MEASURED_PEAKS.json); FFT flops = 5 N log2 N per real transform",
        "flops_note": "achieved / frac count the REFERENCE plan's flops, (2B+1) 5 N log2 N with N = the "
                      "reference's FFT size (SURVEY.md 8d); the device executes each pair's overlap-add at the "
                      "block size that minimises its modelled time (DESIGN.md 4: re-blocking), reported as "
                      "exec_flops / exec_frac per executed size in by_size",
        "serialized": ser,
        "without_epilogue": None if not k4_alone else {
            "ola_ms": k4_alone["ola_ms"], "mix_kernel_ms": k4_alone["mix_ms"],
            "frac": k4_alone["flops"] / (k4_alone["ola_ms"] / 1e3) / 1e12 / fp32_peak if k4_alone["ola_ms"] > 0 else None,
            "note": "one extra render with rs_ctx_set_fused_mix(0): K4 without the mix epilogue and the mix "
                    "kernel it replaces; in the timed region the last work item of every output channel mixes "
                    "it inside the K4 launches (mixfin.cuh), so ola_ms_per_step and frac above include the mix"},
        "by_size": k4_sizes,
        "by_size_note": "one extra render with the K4 launches serialized, each timed with CUDA events; rows "
                        "are keyed by the EXECUTED fft_size; `frac` = the rows' reference-plan flops / time / "
                        "peak, `exec_frac` = the executed plan's; the headline frac is the timed region's "
                        "concurrent launches (K4 event windows per chunk, which also see the tail of the "
                        "first chunks' K1 on the other stream); `serialized` sums the rows",
    }

    cpu, parity = None, None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        want = args.cpu_sample_utts or max(32, 64 * threads)  # ~10 s of the host's cores
        sub, k = cpu_sample(args, want)
        # glibc's default malloc first (SURVEY.md §8d asks for both; mallopt cannot be undone
        # within the process): a quarter of the sample, so the baseline leg stays within seconds
        sub_u = sub.subset(np.arange(0, sub.n_utt, 4))
        v_u, dt_u, _, _ = run_cpu_reference(sub_u, threads, tuned=False)
        v, dt, kind, ref_res = run_cpu_reference(sub, threads)
        cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": kind,
               "sample": f"{sub.n_utt} of {n_config(args)} {args.config} utterances (every {k}th), "
                         f"{sub.audio_seconds:.1f} audio-s, {dt:.1f} s wall",
               "note": "reference radix-2 CPU path (FFTW3 unavailable); malloc mmap_threshold=64MiB",
               "value_default_malloc": v_u,
               "default_malloc_sample": f"every 4th utterance of the sample ({sub_u.n_utt}), {dt_u:.1f} s wall"}
        # the same sample through our path: layouts bit-exact, waveforms within 1e-5 of the peak
        g = roomsim.render_batch(sub, ctx=ctx)
        o_out, o_len, o_lay, o_gain, o_pow = ref_res
        lay_ok = all(bool((g.layout[f] == o_lay[f]).all()) for f in
                     ("rir_len", "rir_keep", "cutoff", "fft_size", "block_len", "n_blocks", "out_len"))
        J = np.diff(sub.mic_begin)
        worst = 0.0
        for u in range(sub.n_utt):
            w_ = np.concatenate([sub.channel(o_out, u, j, o_len[u]) for j in range(J[u])])
            g_ = np.concatenate([sub.channel(g.out, u, j, o_len[u]) for j in range(J[u])]).astype(np.float64)
            worst = max(worst, float(np.abs(g_ - w_).max() / np.abs(w_).max()))
        parity = {"checked_against": kind, "utterances": sub.n_utt, "pairs": sub.n_pairs,
                  "layouts_bit_exact": lay_ok, "max_rel_wave_err": worst,
                  "max_rel_gain_err": float(np.max(np.abs(g.gains - o_gain) / np.abs(o_gain))),
                  "pass": bool(lay_ok and worst <= 1e-5)}

    if rank == 0:
        cfg = workload_config(args, world)
        cfg.update({"pairs": total_pairs, "audio_seconds": total_audio,
                    "per_rank": {"utterances": batch.n_utt, "pairs": batch.n_pairs},
                    "l2": "inputs (%.1f GB per GPU) >> L2 (126 MB): no flush needed" % (4 * batch.total_samples / 1e9)})
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f32",
            "data": "synthetic: seeded N(0,0.1) fp32 signals, sampled image-method rooms",
            "config": cfg, "roofline": roofline, "cpu_baseline": cpu, "parity": parity, "e2e": e2e,
            "epoch_loop": epoch_loop, "logmel": logmel, "gpu_launches": launches, "clocks": clocks,
            "stage_ms": {k: round(v, 3) for k, v in stages.items()},
            # output channels mixed inside the K4 launches (the last work item of a channel mixes it)
            "mix": {"fused_channels": mix_fused, "channels": mix_channels},
            "two_in_flight": in_flight2, "gather": gather,
        }
        print(json.dumps(line), flush=True)
    ctx.close()


def _free_port() -> int:
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    return port


def run_rank(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one process per GPU "
                 f"(torchrun --nproc-per-node {args.gpus}) or leave WORLD_SIZE unset to spawn here")
    if args.impl == "reference":
        reference_arm(args, rank, world)
        return
    import torch
    import torch.distributed as dist

    if world > 1:
        if args.dry_run:
            dist.init_process_group("gloo", rank=rank, world_size=world)
        else:
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        if args.dry_run:
            dry_run(args, rank, world)
        else:
            ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            dist.destroy_process_group()


def _spawned(local_rank, argv, world, port):
    os.environ.update(RANK=str(local_rank), LOCAL_RANK=str(local_rank), WORLD_SIZE=str(world),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    run_rank(parse(argv))


def main():
    argv = sys.argv[1:]
    args = parse(argv)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        if args.impl == "reference":  # rank 0 alone runs the CPU reference: no processes to spawn
            os.environ.update(RANK="0", LOCAL_RANK="0", WORLD_SIZE=str(args.gpus))
            reference_arm(args, 0, args.gpus)
            return
        import torch.multiprocessing as mp

        mp.spawn(_spawned, args=(argv, args.gpus, _free_port()), nprocs=args.gpus, join=True)
        return
    run_rank(args)


if __name__ == "__main__":
    main()
