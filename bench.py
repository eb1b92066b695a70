#!/usr/bin/env python3
"""Benchmark of the room-simulation hot path (BASELINE.json metric).

Metric: simulated audio-seconds per second (Σ_utterances N_x / 16 kHz; the
target's duration, counted once per utterance) for BASELINE config 4: 4096
utterances x (1 target + 5 noises) x 2 mics, image-method RIRs truncated at
-20 dB, N = bit_ceil(2 N_h), synth -> cut -> OLA -> SNR mix all on device.

  python bench.py [--gpus N --steps K --warmup W]          # our CUDA path
  python bench.py --impl reference [...]                    # the reference's CPU path

Our arm prints `value` (inputs resident in HBM, CUDA events on the launching
stream, max over ranks), `e2e` (host pinned buffers through the C-ABI with
H2D/D2H in the timed region), the OLA kernel's `roofline`, the reference
CPU `cpu_baseline` (rank 0, N = 1, bounded sample), `clocks` and
`gpu_launches`.  Multi-GPU: one process per GPU (torchrun), utterances sharded
with no collective on the data path ("scaling": "weak" by default: every
rank renders its own 4096 utterances).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "simulated audio-sec/sec"
UNIT = "audio-s/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="config4", choices=["config2", "config3", "config4", "config5"])
    ap.add_argument("--utterances", type=int, default=0, help="per GPU (weak) or total (strong); 0 = config default")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-utts", type=int, default=0)
    ap.add_argument("--seed", type=int, default=4)
    return ap.parse_args()


DEFAULT_UTTS = {"config2": 128, "config3": 128, "config4": 4096, "config5": 512}


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
def cpu_sample(batch_fn, n_utt: int, want: int):
    """Deterministic subsample of the workload (every k-th utterance), host signals."""
    from paper_1712_03439_b200 import scenes

    k = max(1, n_utt // max(want, 1))
    ids = np.arange(0, n_utt, k)[:want]
    full = batch_fn(signals=False)
    sub = full.subset(ids)
    sub.signals = np.empty(sub.total_samples, np.float32)
    g = np.random.Generator(np.random.Philox(key=99))
    sub.signals[:] = g.standard_normal(sub.total_samples, dtype=np.float32) * np.float32(0.1)
    return sub, k


def run_cpu_reference(sub, threads: int):
    import oracle

    kind = "reference" if oracle.reference_available() else "port"
    lib = oracle.reference() if kind == "reference" else oracle.port()
    if kind == "reference":
        lib.lib.ref_set_malloc_tuning(1)
    t0 = time.perf_counter()
    lib.render_batch(sub, threads=threads)
    dt = time.perf_counter() - t0
    return sub.audio_seconds / dt, dt, kind


def reference_arm(args, rank, world):
    """--impl reference: the reference's own CPU path (oracle/_ref) on the host cores."""
    if rank != 0:
        return
    from paper_1712_03439_b200 import scenes

    n_utt = args.utterances or DEFAULT_UTTS[args.config]
    threads = os.cpu_count() or 1
    # each step ~3-5 s of the host's cores: the whole K+W run stays within minutes
    want = args.cpu_sample_utts or max(16, 24 * threads)
    fn = lambda signals=False: scenes.CONFIGS[args.config](n_utt=n_utt, seed=args.seed, signals=signals)  # noqa: E731
    sub, k = cpu_sample(fn, n_utt, want)
    for _ in range(args.warmup):
        run_cpu_reference(sub, threads)
    vals, secs = [], []
    kind = None
    for _ in range(args.steps):
        v, dt, kind = run_cpu_reference(sub, threads)
        vals.append(v)
        secs.append(dt)
    value = float(sub.audio_seconds * args.steps / sum(secs))
    sample = (f"{sub.n_utt} of {n_utt} {args.config} utterances (every {k}th, "
              f"{sub.audio_seconds:.1f} audio-s, {sub.n_pairs} pairs) per step")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(secs) / args.steps,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": args.config, "utterances": n_utt},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample,
                         "note": "reference radix-2 CPU path (FFTW3 unavailable); malloc mmap_threshold=64MiB"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---- our arm ---------------------------------------------------------------------
def ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_1712_03439_b200 import roomsim, scenes, shard

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    n_cfg = args.utterances or DEFAULT_UTTS[args.config]
    if args.scaling == "weak":
        batch = scenes.CONFIGS[args.config](n_utt=n_cfg, seed=args.seed, signals=False, first_utt=rank * n_cfg)
    else:
        full = scenes.CONFIGS[args.config](n_utt=n_cfg, seed=args.seed, signals=False)
        batch, _ = shard.shard_batch(full, rank, world)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1000 + rank)
    signals = torch.randn(max(batch.total_samples, 1), generator=gen, device=dev, dtype=torch.float32).mul_(0.1)
    out = torch.empty(max(batch.out_total, 1), device=dev, dtype=torch.float32)
    stream = torch.cuda.current_stream(dev)
    ctx = roomsim.Context(local_rank)
    ctx.set_stream(stream.cuda_stream)
    ctx.set_profiling(True)

    def step():
        return roomsim.render_batch(batch, ctx=ctx, device_signals_ptr=signals.data_ptr(),
                                    device_out_ptr=out.data_ptr())

    def barrier():
        if world > 1:
            dist.barrier()

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
        res = step()
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
    t = torch.tensor([ms, ola_ms / args.steps], device=dev, dtype=torch.float64)
    aud = torch.tensor([batch.audio_seconds], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(aud, op=dist.ReduceOp.SUM)
    ms_max, ola_ms_max = float(t[0]), float(t[1])
    total_audio = float(aud[0])
    value = total_audio / (ms_max / 1e3)

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
        te = torch.tensor([max(wall, ev)], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": total_audio / (float(te[0]) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(4 * batch.total_samples), "d2h_bytes_per_step": int(4 * batch.out_total),
               "ms_per_step": float(te[0])}
        batch.signals = None

    # ---- epoch loop: source signals generated in HBM (rs_generate_signals, SURVEY.md §8f
    # row 1) + the render, per step; no host staging of the 12.6 GB of inputs ----------------
    epoch_loop = None
    if not args.no_e2e and args.config != "config1":
        spec = roomsim.sampler_spec(getattr(scenes, "spec_" + args.config)(args.seed))
        gen_ms = 0.0
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        def epoch_step(ep):
            g0.record(stream)
            roomsim.generate_signals(spec, batch, seed=args.seed, epoch=ep, first_utt=rank * n_cfg,
                                     device_ptr=signals.data_ptr(), stream=stream.cuda_stream)
            g1.record(stream)
            return step()
        epoch_step(0)
        barrier()
        torch.cuda.synchronize(dev)
        e0.record(stream)
        for k in range(args.steps):
            epoch_step(k + 1)
            torch.cuda.synchronize(dev)
            gen_ms += g0.elapsed_time(g1)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ms_ep = e0.elapsed_time(e1) / args.steps
        te = torch.tensor([ms_ep], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        epoch_loop = {"value": total_audio / (float(te[0]) / 1e3), "unit": UNIT, "ms_per_step": float(te[0]),
                      "signal_gen_ms": gen_ms / args.steps,
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
        logmel = {"ms_per_step": lm_ms / args.steps, "channels": int(ch_len.size), "frames": frames,
                  "stacked_vectors": int(S.sum()),
                  "frames_per_s": frames / (lm_ms / args.steps / 1e3) if lm_ms > 0 else None,
                  "what": "128 log-Mel, 32 ms Hann / 10 ms hop, 125-7500 Hz, 4-frame stacks every 3rd "
                          "(PAPER.md:452-460) of every rendered channel; device-timed kernel"}

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
    if args.config == "config4" and n_cfg == DEFAULT_UTTS["config4"]:
        try:  # K4 DRAM bytes per render, from the committed ncu launch list of this workload
            with open(os.path.join(ROOT, "profiles", "r01_k4_traffic.json")) as f:
                tj = json.load(f)
            traffic, traffic_src = tj["dram_bytes_per_render"], tj["source"] + "; " + tj["note"]
        except Exception:
            pass
    roofline = {
        "bound": "fp32", "achieved": achieved, "peak": fp32_peak, "unit": "TFLOP/s",
        "frac": achieved / fp32_peak if achieved else None, "traffic": traffic,
        "traffic_unit": "DRAM bytes per step (all K4 launches)", "traffic_source": traffic_src,
        "kernel": "K4 (ola_small_kernel<M>, ola_ip_kernel<M>, ola2_kernel<N>, four-step stages), all FFT sizes of one render",
        "ola_ms_per_step": ola_ms / args.steps,
        "alg_flops_per_step": per_step_flops,
        "alg_bytes_per_step": alg_bytes,
        "hbm_time_ms": alg_bytes / (hbm * 1e9) * 1e3,
        "peak_source": f"derived: {props.multi_processor_count} SMs x 128 FP32 lanes x 2 x {sm_max:.0f} MHz "
                       "(sm_max_mhz of MEASURED_PEAKS.json); FFT flops = 5 N log2 N per real transform",
    }

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        want = args.cpu_sample_utts or max(32, 64 * threads)  # ~10 s of the host's cores
        fn = lambda signals=False: scenes.CONFIGS[args.config](n_utt=n_cfg, seed=args.seed, signals=signals)  # noqa: E731
        sub, k = cpu_sample(fn, n_cfg, want)
        v, dt, kind = run_cpu_reference(sub, threads)
        cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": kind,
               "sample": f"{sub.n_utt} of {n_cfg} {args.config} utterances (every {k}th), "
                         f"{sub.audio_seconds:.1f} audio-s, {dt:.1f} s wall",
               "note": "reference radix-2 CPU path (FFTW3 unavailable)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f32",
            "data": "synthetic: seeded N(0,0.1) fp32 signals, sampled image-method rooms",
            "config": {"workload": args.config, "utterances_per_gpu" if args.scaling == "weak" else "utterances": n_cfg,
                       "pairs_per_gpu": batch.n_pairs, "audio_seconds_total": total_audio,
                       "eta_db": batch.eta_db, "fft_rule": {0: "choose_plan", 1: f"forced {batch.forced_fft_size}",
                                                             2: "bit_ceil(2*N_h)"}[batch.plan_rule],
                       "l2": "inputs (%.1f GB/GPU) >> L2 (126 MB): no flush needed" % (4 * batch.total_samples / 1e9)},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "epoch_loop": epoch_loop, "logmel": logmel,
            "gpu_launches": launches, "clocks": clocks,
            "stage_ms": {k: round(v, 3) for k, v in stages.items()},
        }
        print(json.dumps(line), flush=True)
    ctx.close()


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        reference_arm(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    ours(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
