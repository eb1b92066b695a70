"""Seeded scene sampler and the BASELINE.json workload configs (host side).

The reference specifies a `config_sampler` but ships no
code for it; this module restates its contract — every scene is a pure
function of (seed, utterance_id, epoch), derived by hashing so batch order
never matters — and fixes the distributions of BASELINE.json
configs 2-5.  It produces a ``SceneBatch`` in the SoA layout
of ``rs_scene_batch`` (include/roomsim_gpu.h) that both the CUDA path and
the CPU checkers consume, so they see identical inputs.

Fixture decisions:
  * rooms U(3-10 x 3-8 x 2.5-6 m), r ~ U(0.2, 0.9), resampled while the
    Eyring T60 = 0.161 V / (-S ln r^2) exceeds 0.9 s;
  * image order K = ceil(c0 T60 / ||L||_2), RIR cut to the T60 horizon
    ceil(T60 fs) (the RIR length "set to the T60 horizon");
  * sources and the mic array >= 0.5 m from every wall; 2 mics 7.1 cm apart
     on a random horizontal axis, or an 8-mic circle;
  * signals i.i.d. N(0, 0.1) float32 (0.1 is the standard deviation),
    one N_x per utterance shared by all its sources; SNR ~ U(0, 30) dB.
"""
from __future__ import annotations

import dataclasses
import hashlib
import math
from typing import Optional

import numpy as np

FS = 16000.0
C0 = 343.0

PLAN_CHOOSE, PLAN_FORCED, PLAN_POW2_TWICE = 0, 1, 2


@dataclasses.dataclass
class SamplerSpec:
    """SPEC.md:146-158 SamplerSpec, extended with the BASELINE config knobs."""

    dim_lo: tuple = (3.0, 3.0, 2.5)
    dim_hi: tuple = (10.0, 8.0, 6.0)
    refl_range: tuple = (0.2, 0.9)
    t60_max: float = 0.9
    t60_range: Optional[tuple] = None  # if set: sample T60, solve r from Eyring
    num_noises: int = 3
    snr_range_db: tuple = (0.0, 30.0)
    mic_count: int = 2
    mic_spacing: float = 0.071   # line array (J = 2)
    mic_radius: float = 0.0      # > 0: circular array of mic_count mics
    min_wall_clearance: float = 0.5
    seconds_range: tuple = (2.0, 10.0)
    seed: int = 1


def _rng(seed: int, utt: int, epoch: int) -> np.random.Generator:
    h = hashlib.blake2b(f"{seed}/{utt}/{epoch}".encode(), digest_size=16).digest()
    return np.random.Generator(np.random.Philox(key=int.from_bytes(h, "little")))


def t60_eyring(dims, r: float) -> float:
    """Eyring T60 = 0.161 V / (-S ln(r^2)) (harness only)."""
    lx, ly, lz = dims
    V = lx * ly * lz
    S = 2.0 * (lx * ly + lx * lz + ly * lz)
    return 0.161 * V / (-S * math.log(r * r))


@dataclasses.dataclass
class Scene:
    room: np.ndarray      # (3,)
    refl: float
    order: int
    t60: float
    horizon: int          # ceil(T60 fs)
    src: np.ndarray       # (I, 3), row 0 = target
    mic: np.ndarray       # (J, 3)
    snr_db: np.ndarray    # (I,), entry 0 unused
    n_samples: int        # N_x shared by the utterance's sources


def sample_scene(spec: SamplerSpec, utt: int, epoch: int = 0) -> Scene:
    """SPEC.md:161-169 sample_scene: a pure function of (seed, utt, epoch)."""
    g = _rng(spec.seed, utt, epoch)
    lo, hi = np.array(spec.dim_lo), np.array(spec.dim_hi)
    while True:
        room = g.uniform(lo, hi)
        if spec.t60_range is not None:
            t60 = float(g.uniform(*spec.t60_range))
            V = float(np.prod(room))
            S = 2.0 * (room[0] * room[1] + room[0] * room[2] + room[1] * room[2])
            refl = math.exp(-0.0805 * V / (S * t60))
            if not (0.0 < refl < 1.0):
                continue
        else:
            refl = float(g.uniform(*spec.refl_range))
            t60 = t60_eyring(room, refl)
            if t60 > spec.t60_max:
                continue
        break
    order = int(math.ceil(C0 * t60 / float(np.linalg.norm(room))))
    horizon = int(math.ceil(t60 * FS))
    c = spec.min_wall_clearance
    I = 1 + spec.num_noises
    src = g.uniform(c, room - c, size=(I, 3))
    # Mic array: centre far enough from walls that every element keeps clearance.
    ext = spec.mic_radius if spec.mic_radius > 0 else spec.mic_spacing / 2.0
    centre = g.uniform([c + ext, c + ext, c], [room[0] - c - ext, room[1] - c - ext, room[2] - c])
    phi = float(g.uniform(0.0, 2.0 * math.pi))
    if spec.mic_radius > 0:
        ang = phi + 2.0 * math.pi * np.arange(spec.mic_count) / spec.mic_count
        mic = centre + spec.mic_radius * np.stack([np.cos(ang), np.sin(ang), np.zeros_like(ang)], 1)
    else:
        off = np.array([math.cos(phi), math.sin(phi), 0.0]) * spec.mic_spacing / 2.0
        mic = np.stack([centre - off, centre + off])[: spec.mic_count]
    snr = np.concatenate([[0.0], g.uniform(*spec.snr_range_db, size=I - 1)])
    secs = float(g.uniform(*spec.seconds_range))
    n = int(round(secs * FS))
    return Scene(room, refl, order, t60, horizon, src, mic, snr, n)


@dataclasses.dataclass
class SceneBatch:
    """Host SoA mirror of rs_scene_batch (include/roomsim_gpu.h)."""

    src_begin: np.ndarray
    mic_begin: np.ndarray
    room_dims: np.ndarray
    reflection: np.ndarray
    sample_rate: np.ndarray
    speed_of_sound: np.ndarray
    image_order: np.ndarray
    max_taps: np.ndarray
    src_pos: np.ndarray
    mic_pos: np.ndarray
    snr_db: np.ndarray
    sig_off: np.ndarray
    sig_len: np.ndarray
    signals: Optional[np.ndarray]   # float32; None when generated on device
    eta_db: float = 0.0
    plan_rule: int = PLAN_CHOOSE
    forced_fft_size: int = 0
    name: str = ""
    seed: int = 1
    utt_ids: Optional[np.ndarray] = None  # global utterance ids (sampler keys); None: 0..n_utt-1

    @property
    def n_utt(self) -> int:
        return int(self.room_dims.shape[0])

    @property
    def ids(self) -> np.ndarray:
        """Global utterance id of every utterance of the batch (what the samplers key on)."""
        return np.arange(self.n_utt, dtype=np.int64) if self.utt_ids is None else np.asarray(self.utt_ids, np.int64)

    @property
    def n_src(self) -> int:
        return int(self.src_pos.shape[0])

    @property
    def pairs_per_utt(self) -> np.ndarray:
        return np.diff(self.src_begin) * np.diff(self.mic_begin)

    @property
    def n_pairs(self) -> int:
        return int(self.pairs_per_utt.sum())

    @property
    def pair_begin(self) -> np.ndarray:
        return np.concatenate([[0], np.cumsum(self.pairs_per_utt)]).astype(np.int64)

    @property
    def total_samples(self) -> int:
        """Extent of the signal buffer (sources start on 16-byte boundaries: `signal_offsets`)."""
        return int((self.sig_off + self.sig_len).max()) if self.sig_len.size else 0

    @property
    def audio_seconds(self) -> float:
        """Σ_utterances N_x / fs — the target's duration, counted once per utterance."""
        return float(self.sig_len[self.src_begin[:-1]].astype(np.float64).sum() / FS)

    @property
    def out_stride(self) -> np.ndarray:
        """Channel stride per utterance: an upper bound on max_ij(N_x + N_h - 1), rounded up to
        whole quads so every channel starts on a 16-byte boundary (float4 stores in the mix)."""
        nx_max = np.maximum.reduceat(self.sig_len, self.src_begin[:-1])
        cap = np.where(self.max_taps > 0, self.max_taps, self._lattice_bound())
        return ((nx_max + cap - 1 + 3) // 4 * 4).astype(np.int64)

    def _lattice_bound(self) -> np.ndarray:
        ext = (self.image_order[:, None] + 2.0) * self.room_dims
        return np.ceil(np.linalg.norm(ext, axis=1) * self.sample_rate / self.speed_of_sound).astype(np.int64) + 4

    @property
    def out_off(self) -> np.ndarray:
        per = self.out_stride * np.diff(self.mic_begin)
        return np.concatenate([[0], np.cumsum(per)[:-1]]).astype(np.int64)

    @property
    def out_total(self) -> int:
        return int((self.out_stride * np.diff(self.mic_begin)).sum())

    def channel(self, out: np.ndarray, u: int, j: int, length: int) -> np.ndarray:
        o = int(self.out_off[u] + j * self.out_stride[u])
        return out[o : o + int(length)]

    def as_struct(self, struct_cls, signals_ptr: Optional[int] = None):
        """Fill a ctypes rs_scene_batch; returns (struct, keepalive list)."""
        keep = []

        def ptr(a, dt):
            a = np.ascontiguousarray(a, dtype=dt)
            keep.append(a)
            return a.ctypes.data

        s = struct_cls()
        s.n_utt = self.n_utt
        s.src_begin = ptr(self.src_begin, np.int64)
        s.mic_begin = ptr(self.mic_begin, np.int64)
        s.room_dims = ptr(self.room_dims, np.float64)
        s.reflection = ptr(self.reflection, np.float64)
        s.sample_rate = ptr(self.sample_rate, np.float64)
        s.speed_of_sound = ptr(self.speed_of_sound, np.float64)
        s.image_order = ptr(self.image_order, np.int32)
        s.max_taps = ptr(self.max_taps, np.int64)
        s.src_pos = ptr(self.src_pos, np.float64)
        s.mic_pos = ptr(self.mic_pos, np.float64)
        s.snr_db = ptr(self.snr_db, np.float64)
        s.sig_off = ptr(self.sig_off, np.int64)
        s.sig_len = ptr(self.sig_len, np.int64)
        if signals_ptr is not None:
            s.signals = signals_ptr
        else:
            s.signals = ptr(self.signals, np.float32)
        s.eta_db = float(self.eta_db)
        s.plan_rule = int(self.plan_rule)
        s.forced_fft_size = int(self.forced_fft_size)
        return s, keep

    def subset(self, utts) -> "SceneBatch":
        """A batch holding only utterances `utts` (signals re-packed if present)."""
        utts = np.asarray(utts, dtype=np.int64)
        sb, mb = [0], [0]
        srcs, mics = [], []
        for u in utts:
            s0, s1 = self.src_begin[u], self.src_begin[u + 1]
            m0, m1 = self.mic_begin[u], self.mic_begin[u + 1]
            srcs.extend(range(s0, s1))
            mics.extend(range(m0, m1))
            sb.append(sb[-1] + (s1 - s0))
            mb.append(mb[-1] + (m1 - m0))
        srcs = np.asarray(srcs, np.int64)
        lens = self.sig_len[srcs]
        offs = signal_offsets(lens)
        sig = None
        if self.signals is not None:
            sig = np.zeros(int((offs + lens).max()) if len(srcs) else 0, np.float32)
            for o_new, o, n in zip(offs, self.sig_off[srcs], lens):
                sig[o_new : o_new + n] = self.signals[o : o + n]
        return dataclasses.replace(
            self,
            src_begin=np.asarray(sb, np.int64),
            mic_begin=np.asarray(mb, np.int64),
            room_dims=self.room_dims[utts],
            reflection=self.reflection[utts],
            sample_rate=self.sample_rate[utts],
            speed_of_sound=self.speed_of_sound[utts],
            image_order=self.image_order[utts],
            max_taps=self.max_taps[utts],
            src_pos=self.src_pos[srcs],
            mic_pos=self.mic_pos[np.asarray(mics, np.int64)],
            snr_db=self.snr_db[srcs],
            sig_off=offs,
            sig_len=lens.astype(np.int64),
            signals=sig,
            utt_ids=self.ids[utts],
        )


def signal_offsets(lens) -> np.ndarray:
    """Offsets of consecutive sources in one signal buffer, each rounded up to a multiple of
    4 samples (16 bytes): vector loads and stores of a source start aligned."""
    lens = np.asarray(lens, np.int64)
    padded = (lens + 3) // 4 * 4
    return np.concatenate([[0], np.cumsum(padded)[:-1]]).astype(np.int64) if lens.size else np.zeros(0, np.int64)


def make_batch(spec: SamplerSpec, n_utt: int, *, epoch: int = 0, first_utt: int = 0,
               eta_db: float = 0.0, plan_rule: int = PLAN_CHOOSE, forced_fft_size: int = 0,
               signals: bool = True, name: str = "") -> SceneBatch:
    scenes = [sample_scene(spec, first_utt + u, epoch) for u in range(n_utt)]
    I = np.array([s.src.shape[0] for s in scenes])
    J = np.array([s.mic.shape[0] for s in scenes])
    nx = np.repeat([s.n_samples for s in scenes], I).astype(np.int64)
    off = signal_offsets(nx)
    b = SceneBatch(
        src_begin=np.concatenate([[0], np.cumsum(I)]).astype(np.int64),
        mic_begin=np.concatenate([[0], np.cumsum(J)]).astype(np.int64),
        room_dims=np.stack([s.room for s in scenes]).astype(np.float64),
        reflection=np.array([s.refl for s in scenes], np.float64),
        sample_rate=np.full(n_utt, FS),
        speed_of_sound=np.full(n_utt, C0),
        image_order=np.array([s.order for s in scenes], np.int32),
        max_taps=np.array([s.horizon for s in scenes], np.int64),
        src_pos=np.concatenate([s.src for s in scenes]).astype(np.float64),
        mic_pos=np.concatenate([s.mic for s in scenes]).astype(np.float64),
        snr_db=np.concatenate([s.snr_db for s in scenes]).astype(np.float64),
        sig_off=off,
        sig_len=nx,
        signals=None,
        eta_db=eta_db,
        plan_rule=plan_rule,
        forced_fft_size=forced_fft_size,
        name=name,
        seed=spec.seed,
        utt_ids=first_utt + np.arange(n_utt, dtype=np.int64),
    )
    if signals:
        b.signals = host_signals(b, spec.seed, epoch, first_utt)
    return b


def host_signals(b: SceneBatch, seed: int, epoch: int = 0, first_utt: int = 0) -> np.ndarray:
    """i.i.d. N(0, 0.1) float32 per source, keyed by (seed, utterance, source)."""
    out = np.zeros(b.total_samples, np.float32)
    for u in range(b.n_utt):
        for s in range(b.src_begin[u], b.src_begin[u + 1]):
            g = _rng(seed ^ 0x5EED, (first_utt + u) * 64 + int(s - b.src_begin[u]), epoch)
            n = int(b.sig_len[s])
            o = int(b.sig_off[s])
            out[o : o + n] = g.standard_normal(n, dtype=np.float32) * np.float32(0.1)
    return out


# ---- BASELINE.json configs ---------------------------------------------------

def config1(seed: int = 1):
    """Config 1: one 5 s N(0, 0.1) signal, one 4096-tap RIR (unit tap at 0,
    exponentially decaying Gaussian noise with T60 = 0.3 s), N = 8192."""
    g = np.random.Generator(np.random.Philox(key=seed))
    x = (g.standard_normal(80000, dtype=np.float32) * np.float32(0.1))
    n = np.arange(4096)
    h = g.standard_normal(4096) * 10.0 ** (-3.0 * n / (FS * 0.3))
    h[0] = 1.0
    return x, h.astype(np.float64), 8192


def spec_config2(seed: int = 2) -> SamplerSpec:
    return SamplerSpec(seed=seed, num_noises=3, mic_count=2, seconds_range=(2.0, 10.0))


def config2(n_utt: int = 128, seed: int = 2, signals: bool = True, first_utt: int = 0):
    return make_batch(spec_config2(seed), n_utt, plan_rule=PLAN_CHOOSE, signals=signals,
                      first_utt=first_utt, name="config2")


def config3(n_utt: int = 128, seed: int = 2, signals: bool = True, first_utt: int = 0):
    return make_batch(spec_config2(seed), n_utt, eta_db=20.0, plan_rule=PLAN_POW2_TWICE,
                      signals=signals, first_utt=first_utt, name="config3")


def spec_config4(seed: int = 4) -> SamplerSpec:
    return SamplerSpec(seed=seed, num_noises=5, mic_count=2, seconds_range=(1.0, 15.0))


def config4(n_utt: int = 4096, seed: int = 4, signals: bool = True, first_utt: int = 0):
    return make_batch(spec_config4(seed), n_utt, eta_db=20.0, plan_rule=PLAN_POW2_TWICE,
                      signals=signals, first_utt=first_utt, name="config4")


def spec_config5(seed: int = 5) -> SamplerSpec:
    return SamplerSpec(seed=seed, dim_lo=(10.0, 8.0, 3.5), dim_hi=(20.0, 15.0, 6.0),
                       t60_range=(0.9, 1.2), num_noises=7, mic_count=8, mic_radius=0.05,
                       seconds_range=(10.0, 10.0))


def config5(n_utt: int = 512, seed: int = 5, signals: bool = True, first_utt: int = 0):
    return make_batch(spec_config5(seed), n_utt, plan_rule=PLAN_FORCED, forced_fft_size=32768,
                      signals=signals, first_utt=first_utt, name="config5")


CONFIGS = {"config2": config2, "config3": config3, "config4": config4, "config5": config5}
