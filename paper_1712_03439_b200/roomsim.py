"""Python mirror of the reference ``roomsim`` C++ API over the CUDA C-ABI.

Names, argument meaning and error behaviour follow the reference headers
(/root/reference/proj/include/roomsim/*.hpp) so parity tests read like the
reference's own: ``synthesize_rir`` (room_model.hpp:141), ``truncate_rir``
(:203), ``power_threshold``/``cutoff_index`` (:177/:188), ``cost_*``,
``plan_for``, ``choose_plan`` (convolution.hpp:89-161), ``convolve_ola``
(:219), ``convolve_full_fft`` (:182), ``convolve`` (:258), the
``RealFftEngine`` concept (fft.hpp:38-49) as ``CudaRealFft``, and SPEC
``render`` as ``render_batch``.  Errors raise the classes of
roomsim/errors.hpp:22-68.

Every compute call runs on the GPU through ``_lib/libroomsim_gpu.so``; there
is no CPU fallback — importing on a machine without the built library raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ROOMSIM_LIB") or os.path.join(_HERE, "_lib", "libroomsim_gpu.so")

DIRECT, FULL_FFT, OVERLAP_ADD = 0, 1, 2
PLAN_CHOOSE, PLAN_FORCED, PLAN_POW2_TWICE = 0, 1, 2


# ---- error taxonomy (roomsim/errors.hpp:22-68) --------------------------------
class Error(RuntimeError):
    """roomsim::Error"""


class PlacementError(Error):
    pass


class GeometryError(Error):
    pass


class DegenerateInputError(Error):
    pass


class PlanError(Error):
    pass


class ConfigError(Error):
    pass


class FormatError(Error):
    pass


class IoError(Error):
    pass


class DeviceError(Error):
    """CUDA / allocation failure (no reference analogue)."""


class UnsupportedError(Error):
    """Size outside what the device kernels implement."""


_CODES = {1: PlacementError, 2: GeometryError, 3: DegenerateInputError, 4: PlanError,
          5: ConfigError, 6: FormatError, 7: IoError, 16: DeviceError, 17: DeviceError,
          18: UnsupportedError}


class RsSceneBatch(C.Structure):
    _fields_ = [
        ("n_utt", C.c_int64), ("src_begin", C.c_void_p), ("mic_begin", C.c_void_p),
        ("room_dims", C.c_void_p), ("reflection", C.c_void_p), ("sample_rate", C.c_void_p),
        ("speed_of_sound", C.c_void_p), ("image_order", C.c_void_p), ("max_taps", C.c_void_p),
        ("src_pos", C.c_void_p), ("mic_pos", C.c_void_p), ("snr_db", C.c_void_p),
        ("sig_off", C.c_void_p), ("sig_len", C.c_void_p), ("signals", C.c_void_p),
        ("eta_db", C.c_double), ("plan_rule", C.c_int32), ("forced_fft_size", C.c_int64),
    ]


LAYOUT_DTYPE = np.dtype([("rir_len", np.int64), ("rir_keep", np.int64), ("cutoff", np.int64),
                         ("fft_size", np.int64), ("block_len", np.int64), ("n_blocks", np.int64),
                         ("out_len", np.int64), ("strategy", np.int32), ("flags", np.int32)])

# Every symbol include/roomsim_gpu.h declares (checked by tests/test_abi.py).
ABI_SYMBOLS = [
    "rs_last_error", "rs_version", "rs_ctx_create", "rs_ctx_destroy", "rs_ctx_set_stream",
    "rs_ctx_synchronize", "rs_ctx_last_timing", "rs_ctx_mix_counts", "rs_ctx_set_fused_mix", "rs_ctx_stage_times", "rs_ctx_set_profiling",
    "rs_ctx_k4_breakdown", "rs_cost_direct",
    "rs_cost_full_fft", "rs_cost_ola", "rs_ola_block_count", "rs_plan_for", "rs_choose_plan",
    "rs_rfft_forward", "rs_rfft_inverse", "rs_synthesize_rir", "rs_truncate_rir",
    "rs_convolve_ola", "rs_convolve_full_fft", "rs_convolve_direct", "rs_convolve", "rs_batch_num_pairs",
    "rs_render_batch", "rs_render_batch_device", "rs_last_pair_signal", "rs_last_pair_rir",
    "rs_sampler_counts", "rs_sample_scenes", "rs_sampler_counts_device", "rs_sample_scenes_device",
    "rs_generate_signals_host", "rs_generate_signals", "rs_signal_plan_create", "rs_signal_plan_generate",
    "rs_signal_plan_destroy", "rs_logmel_shape", "rs_logmel_device", "rs_render_features_device",
]


class RsSamplerSpec(C.Structure):
    _fields_ = [
        ("dim_lo", C.c_double * 3), ("dim_hi", C.c_double * 3), ("refl_lo", C.c_double),
        ("refl_hi", C.c_double), ("t60_max", C.c_double), ("t60_lo", C.c_double), ("t60_hi", C.c_double),
        ("snr_lo", C.c_double), ("snr_hi", C.c_double), ("mic_spacing", C.c_double),
        ("mic_radius", C.c_double), ("clearance", C.c_double), ("sec_lo", C.c_double),
        ("sec_hi", C.c_double), ("fs", C.c_double), ("c0", C.c_double), ("signal_std", C.c_double),
        ("num_noises", C.c_int32), ("mic_count", C.c_int32), ("n_weights", C.c_int32), ("pad_", C.c_int32),
        ("weights", C.c_double * 8),
    ]

_lib = None


def load_library() -> C.CDLL:
    """Load the CUDA library (raises if it was not built: no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built (run `make` / __graft_entry__.build())")
    L = C.CDLL(LIB_PATH)
    d, sz, i64, vp = C.c_double, C.c_size_t, C.c_int64, C.c_void_p
    dp = C.POINTER(C.c_double)
    szp = C.POINTER(C.c_size_t)
    sig = {
        "rs_last_error": (C.c_char_p, []),
        "rs_version": (C.c_char_p, []),
        "rs_ctx_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
        "rs_ctx_destroy": (C.c_int, [vp]),
        "rs_ctx_set_stream": (C.c_int, [vp, vp]),
        "rs_ctx_synchronize": (C.c_int, [vp]),
        "rs_ctx_last_timing": (C.c_int, [vp, dp, dp, dp, C.POINTER(i64)]),
        "rs_ctx_mix_counts": (C.c_int, [vp, C.POINTER(i64), C.POINTER(i64)]),
        "rs_ctx_set_fused_mix": (C.c_int, [vp, C.c_int]),
        "rs_ctx_set_profiling": (C.c_int, [vp, C.c_int]),
        "rs_ctx_stage_times": (C.c_int, [vp, dp, C.c_int, dp]),
        "rs_ctx_k4_breakdown": (C.c_int, [vp, C.c_int, vp, vp, vp, vp, vp, vp]),
        "rs_cost_direct": (d, [d, d, sz, sz]),
        "rs_cost_full_fft": (d, [d, d, sz, sz, sz]),
        "rs_cost_ola": (d, [d, d, sz, sz, sz]),
        "rs_ola_block_count": (sz, [sz, sz, sz]),
        "rs_plan_for": (C.c_int, [d, d, sz, sz, C.c_int, C.POINTER(C.c_int), szp, dp]),
        "rs_choose_plan": (C.c_int, [d, d, sz, sz, C.POINTER(C.c_int), szp, dp]),
        "rs_rfft_forward": (C.c_int, [vp, sz, sz, vp, vp]),
        "rs_rfft_inverse": (C.c_int, [vp, sz, sz, vp, vp]),
        "rs_synthesize_rir": (C.c_int, [vp, vp, d, d, d, C.c_int, vp, vp, i64, vp, sz, szp]),
        "rs_truncate_rir": (C.c_int, [vp, vp, sz, d, szp, szp, dp]),
        "rs_convolve_ola": (C.c_int, [vp, vp, sz, vp, sz, sz, vp]),
        "rs_convolve_full_fft": (C.c_int, [vp, vp, sz, vp, sz, vp]),
        "rs_convolve_direct": (C.c_int, [vp, vp, sz, vp, sz, vp]),
        "rs_convolve": (C.c_int, [vp, vp, sz, vp, sz, C.c_int, sz, vp]),
        "rs_batch_num_pairs": (i64, [vp]),
        "rs_render_batch": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, vp, vp]),
        "rs_render_batch_device": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, vp, vp]),
        "rs_last_pair_signal": (C.c_int, [vp, i64, vp, sz, szp]),
        "rs_last_pair_rir": (C.c_int, [vp, i64, vp, sz, szp]),
        "rs_sampler_counts": (C.c_int, [vp, C.c_uint64, i64, i64, i64, vp]),
        "rs_sample_scenes": (C.c_int, [vp, C.c_uint64, i64, i64, i64] + [vp] * 9),
        "rs_sampler_counts_device": (C.c_int, [vp, C.c_uint64, i64, i64, i64, vp, vp]),
        "rs_sample_scenes_device": (C.c_int, [vp, C.c_uint64, i64, i64, i64] + [vp] * 10),
        "rs_generate_signals_host": (C.c_int, [vp, C.c_uint64, i64, i64, vp, vp, vp, vp, vp]),
        "rs_generate_signals": (C.c_int, [vp, C.c_uint64, i64, i64, vp, vp, vp, vp, vp, vp]),
        "rs_signal_plan_create": (C.c_int, [vp, C.c_uint64, i64, vp, vp, vp, vp, C.POINTER(vp)]),
        "rs_signal_plan_generate": (C.c_int, [vp, i64, vp, vp]),
        "rs_signal_plan_destroy": (C.c_int, [vp]),
        "rs_logmel_shape": (C.c_int, [i64, C.POINTER(i64), C.POINTER(i64)]),
        "rs_logmel_device": (C.c_int, [vp, vp, i64, vp, vp, vp, vp]),
        "rs_render_features_device": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _check(st: int) -> None:
    if st != 0:
        msg = load_library().rs_last_error().decode()
        raise _CODES.get(st, Error)(msg)


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


# ---- planner (host side; exact mirror of convolution.hpp) ----------------------
@dataclass
class ConvolutionPlan:
    """roomsim::ConvolutionPlan (convolution.hpp:64-68)."""

    strategy: int = DIRECT
    fft_size: Optional[int] = None
    predicted_cost: float = 0.0


def cost_direct(I, J, nx, nh) -> float:
    v = load_library().rs_cost_direct(I, J, nx, nh)
    if np.isnan(v):
        _check(5)
    return v


def cost_full_fft(I, J, nx, nh, n) -> float:
    v = load_library().rs_cost_full_fft(I, J, nx, nh, n)
    if np.isnan(v):
        raise (PlanError if "FFT" in load_library().rs_last_error().decode() else ConfigError)(
            load_library().rs_last_error().decode())
    return v


def cost_ola(I, J, nx, nh, n) -> float:
    v = load_library().rs_cost_ola(I, J, nx, nh, n)
    if np.isnan(v):
        raise (PlanError if "FFT" in load_library().rs_last_error().decode() else ConfigError)(
            load_library().rs_last_error().decode())
    return v


def ola_block_count(nx, nh, n) -> int:
    return int(load_library().rs_ola_block_count(nx, nh, n))


def plan_for(I, J, nx, nh, strategy) -> ConvolutionPlan:
    s, n, c = C.c_int(), C.c_size_t(), C.c_double()
    _check(load_library().rs_plan_for(I, J, nx, nh, strategy, C.byref(s), C.byref(n), C.byref(c)))
    return ConvolutionPlan(s.value, n.value if s.value != DIRECT else None, c.value)


def choose_plan(I, J, nx, nh) -> ConvolutionPlan:
    s, n, c = C.c_int(), C.c_size_t(), C.c_double()
    _check(load_library().rs_choose_plan(I, J, nx, nh, C.byref(s), C.byref(n), C.byref(c)))
    return ConvolutionPlan(s.value, n.value if s.value != DIRECT else None, c.value)


# ---- device context -------------------------------------------------------------
class Context:
    """rs_ctx: one device, one stream, one arena.  Not shareable across threads."""

    def __init__(self, device: int = 0):
        L = load_library()
        h = C.c_void_p()
        _check(L.rs_ctx_create(int(device), C.byref(h)))
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            load_library().rs_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_handle: int) -> None:
        _check(load_library().rs_ctx_set_stream(self.h, C.c_void_p(stream_handle)))

    def set_profiling(self, on) -> None:
        """True/1: event timing of the stages; 2: also the per-(size, variant) K4
        breakdown (K4 launches serialized — a diagnostic render, not a timed one)."""
        _check(load_library().rs_ctx_set_profiling(self.h, int(on)))

    K4_VARIANTS = ("ola_small", "ola_ip", "ola2", "four_step", "ola_ipc")

    def k4_breakdown(self) -> list:
        """Rows of the last render at profiling level 2: executed N, variant, pairs, algorithmic
        flops (reference plan), ms, flops of the executed plan."""
        L = load_library()
        n = L.rs_ctx_k4_breakdown(self.h, 0, None, None, None, None, None, None)
        if n < 0:
            _check(-n)
        lg = np.zeros(n, np.int32)
        var = np.zeros(n, np.int32)
        pairs = np.zeros(n, np.int64)
        fl = np.zeros(n)
        ms = np.zeros(n)
        ef = np.zeros(n)
        L.rs_ctx_k4_breakdown(self.h, n, _ptr(lg), _ptr(var), _ptr(pairs), _ptr(fl), _ptr(ms), _ptr(ef))
        return [{"fft_size": 1 << int(lg[i]), "kernel": self.K4_VARIANTS[int(var[i])], "pairs": int(pairs[i]),
                 "flops": float(fl[i]), "ms": float(ms[i]), "exec_flops": float(ef[i])} for i in np.argsort(-fl)]

    def synchronize(self) -> None:
        _check(load_library().rs_ctx_synchronize(self.h))

    STAGES = ("synth", "cut", "plan_gap", "spectrum", "ola", "gain_mix")

    def stage_times(self) -> dict:
        """Device ms per stage of the last render (profiling on) + host planner ms."""
        arr = (C.c_double * 6)()
        hp = C.c_double()
        _check(load_library().rs_ctx_stage_times(self.h, arr, 6, C.byref(hp)))
        d = {k: arr[i] for i, k in enumerate(self.STAGES)}
        d["host_plan_ms"] = hp.value
        return d

    def last_timing(self):
        ms, fl, by = C.c_double(), C.c_double(), C.c_double()
        n = C.c_int64()
        _check(load_library().rs_ctx_last_timing(self.h, C.byref(ms), C.byref(fl), C.byref(by), C.byref(n)))
        return {"ola_ms": ms.value, "ola_flops": fl.value, "alg_bytes": by.value, "launches": n.value}

    def set_fused_mix(self, on: int):
        """1 / 0: the K4 epilogue mixes the channels it can / mix_kernel mixes all; -1: process default."""
        _check(load_library().rs_ctx_set_fused_mix(self.h, int(on)))

    def mix_counts(self):
        """(channels of the last render mixed by the K4 epilogue, all its channels)."""
        a, b = C.c_int64(), C.c_int64()
        _check(load_library().rs_ctx_mix_counts(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value


_default: Optional[Context] = None


def default_context() -> Context:
    global _default
    if _default is None:
        _default = Context(0)
    return _default


# ---- room model ------------------------------------------------------------------
def synthesize_rir(room, reflection, image_order, src, mic, *, sample_rate=16000.0,
                   speed_of_sound=343.0, max_taps=0, ctx: Optional[Context] = None) -> np.ndarray:
    """roomsim::synthesize_rir (room_model.hpp:141-174), FP64 bit-exact on device."""
    ctx = ctx or default_context()
    room = np.ascontiguousarray(room, np.float64)
    src = np.ascontiguousarray(src, np.float64)
    mic = np.ascontiguousarray(mic, np.float64)
    ext = (abs(int(image_order)) + 2) * room
    cap = int(np.ceil(np.sqrt((ext ** 2).sum()) * sample_rate / speed_of_sound)) + 4
    if max_taps:
        cap = min(cap, int(max_taps))
    out = np.zeros(max(cap, 1))
    n = C.c_size_t()
    _check(load_library().rs_synthesize_rir(ctx.h, _ptr(room), float(reflection), float(sample_rate),
                                            float(speed_of_sound), int(image_order), _ptr(src), _ptr(mic),
                                            int(max_taps), _ptr(out), out.size, C.byref(n)))
    return out[: n.value].copy()


def truncate_rir(h, eta_db, ctx: Optional[Context] = None):
    """roomsim::truncate_rir (room_model.hpp:203-213) -> (taps, n_c, p_th)."""
    ctx = ctx or default_context()
    h = np.ascontiguousarray(h, np.float64)
    keep, nc, th = C.c_size_t(), C.c_size_t(), C.c_double()
    _check(load_library().rs_truncate_rir(ctx.h, _ptr(h), h.size, float(eta_db), C.byref(keep),
                                          C.byref(nc), C.byref(th)))
    return h[: keep.value].copy(), nc.value, th.value


def power_threshold(h, eta_db, ctx: Optional[Context] = None) -> float:
    return truncate_rir(h, eta_db, ctx)[2]


# ---- FFT engine seam (fft.hpp:38-49) ------------------------------------------------
class CudaRealFft:
    """RealFftEngine on the device: forward -> N/2+1 bins, inverse includes 1/N."""

    def __init__(self, size: int, ctx: Optional[Context] = None):
        if size < 2 or size & (size - 1):
            raise PlanError("FFT size must be a power of two >= 2")
        self._n = int(size)
        self.ctx = ctx or default_context()

    def size(self) -> int:
        return self._n

    def spectrum_size(self) -> int:
        return self._n // 2 + 1

    def forward(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64).reshape(-1, self._n)
        out = np.zeros((x.shape[0], 2 * self.spectrum_size()))
        _check(load_library().rs_rfft_forward(self.ctx.h, self._n, x.shape[0], _ptr(x), _ptr(out)))
        res = out[:, 0::2] + 1j * out[:, 1::2]
        return res[0] if res.shape[0] == 1 else res

    def inverse(self, spec: np.ndarray) -> np.ndarray:
        spec = np.asarray(spec, np.complex128).reshape(-1, self.spectrum_size())
        inp = np.zeros((spec.shape[0], 2 * self.spectrum_size()))
        inp[:, 0::2] = spec.real
        inp[:, 1::2] = spec.imag
        out = np.zeros((spec.shape[0], self._n))
        _check(load_library().rs_rfft_inverse(self.ctx.h, self._n, spec.shape[0], _ptr(inp), _ptr(out)))
        return out[0] if out.shape[0] == 1 else out


# ---- convolution ---------------------------------------------------------------------
def _conv(fn, x, h, *extra, ctx=None):
    ctx = ctx or default_context()
    x = np.ascontiguousarray(x, np.float64)
    h = np.ascontiguousarray(h, np.float64)
    out = np.zeros(max(x.size + h.size - 1, 1))
    _check(fn(ctx.h, _ptr(x), x.size, _ptr(h), h.size, *extra, _ptr(out)))
    return out[: x.size + h.size - 1]


def convolve_ola(x, h, fft_size, ctx: Optional[Context] = None) -> np.ndarray:
    """roomsim::convolve_ola (convolution.hpp:219-255)."""
    return _conv(load_library().rs_convolve_ola, x, h, int(fft_size), ctx=ctx)


def convolve_full_fft(x, h, ctx: Optional[Context] = None) -> np.ndarray:
    """roomsim::convolve_full_fft (convolution.hpp:182-212)."""
    return _conv(load_library().rs_convolve_full_fft, x, h, ctx=ctx)


def convolve_direct(x, h, ctx: Optional[Context] = None) -> np.ndarray:
    """roomsim::convolve_direct (convolution.hpp:164-179): FP64 on the device, bit-exact."""
    return _conv(load_library().rs_convolve_direct, x, h, ctx=ctx)


def convolve(x, h, plan: ConvolutionPlan, ctx: Optional[Context] = None) -> np.ndarray:
    """roomsim::convolve (convolution.hpp:258-271)."""
    return _conv(load_library().rs_convolve, x, h, int(plan.strategy), int(plan.fft_size or 0), ctx=ctx)


# ---- batched render --------------------------------------------------
@dataclass
class RenderResult:
    out: object               # host np.float32 array or device tensor
    out_len: np.ndarray       # [n_utt]
    layout: np.ndarray        # [n_pairs] LAYOUT_DTYPE
    gains: np.ndarray         # [n_pairs] alpha_ij
    power: np.ndarray         # [n_pairs] mean power of each reverberant pair signal


def render_batch(batch, *, ctx: Optional[Context] = None, out: Optional[np.ndarray] = None,
                 device_signals_ptr: Optional[int] = None, device_out_ptr: Optional[int] = None,
                 result: Optional[RenderResult] = None) -> RenderResult:
    """Render a ``scenes.SceneBatch``.

    ``result``: a RenderResult of an earlier render of a batch of the same shape, whose
    layout / gain / power arrays are overwritten and returned (no per-call allocation).

    Host mode (default): signals/out are host arrays, H2D/D2H inside the call.
    Device mode: pass ``device_signals_ptr`` and ``device_out_ptr`` (e.g. torch
    ``data_ptr()``); nothing large crosses PCIe."""
    ctx = ctx or default_context()
    L = load_library()
    device = device_signals_ptr is not None
    b, keep = batch.as_struct(RsSceneBatch, signals_ptr=device_signals_ptr)
    # the output layout of a batch (numpy reductions over its utterances: ~0.4 ms at 4096
    # utterances, idle GPU time between renders) is derived once per batch object
    key = (id(batch.sig_len), id(batch.src_begin), id(batch.mic_begin), id(batch.max_taps), id(batch.room_dims),
           id(batch.image_order), int(batch.sig_len.sum()), int(np.asarray(batch.max_taps).sum()),
           int(np.asarray(batch.image_order).sum()), float(np.asarray(batch.room_dims).sum()))
    memo = getattr(batch, "_rs_layout_memo", None)
    if memo is None or memo[0] != key:
        memo = (key, np.ascontiguousarray(batch.out_off, np.int64), np.ascontiguousarray(batch.out_stride, np.int64),
                int(batch.n_pairs), int(batch.n_utt), int(batch.out_total))
        try:
            batch._rs_layout_memo = memo
        except AttributeError:
            pass
    _, out_off, out_stride, n_pairs, n_utt, out_total = memo
    if result is not None and result.layout.shape == (n_pairs,) and result.out_len.shape == (n_utt,):
        out_len, layout, gains, power = result.out_len, result.layout, result.gains, result.power
    else:
        out_len = np.zeros(n_utt, np.int64)
        layout = np.zeros(n_pairs, LAYOUT_DTYPE)
        gains = np.zeros(n_pairs)
        power = np.zeros(n_pairs)
    if device:
        assert device_out_ptr is not None
        st = L.rs_render_batch_device(ctx.h, C.byref(b), C.c_void_p(device_out_ptr), _ptr(out_off),
                                      _ptr(out_stride), _ptr(out_len), _ptr(layout), _ptr(gains), _ptr(power))
        res_out = None
    else:
        if out is None:
            out = np.zeros(out_total, np.float32)
        st = L.rs_render_batch(ctx.h, C.byref(b), _ptr(out), _ptr(out_off), _ptr(out_stride),
                               _ptr(out_len), _ptr(layout), _ptr(gains), _ptr(power))
        res_out = out
    del keep
    _check(st)
    return RenderResult(res_out, out_len, layout, gains, power)


def last_pair_signal(pair: int, cap: int, ctx: Optional[Context] = None) -> np.ndarray:
    ctx = ctx or default_context()
    out = np.zeros(cap, np.float32)
    n = C.c_size_t()
    _check(load_library().rs_last_pair_signal(ctx.h, int(pair), _ptr(out), cap, C.byref(n)))
    return out[: n.value]


def last_pair_rir(pair: int, cap: int, ctx: Optional[Context] = None) -> np.ndarray:
    ctx = ctx or default_context()
    out = np.zeros(cap)
    n = C.c_size_t()
    _check(load_library().rs_last_pair_rir(ctx.h, int(pair), _ptr(out), cap, C.byref(n)))
    return out[: n.value]


# ---- scene sampler and signal generator ----------
def sampler_spec(spec, *, weights=None, signal_std: float = 0.1, fs: float = 16000.0,
                 c0: float = 343.0) -> RsSamplerSpec:
    """An rs_sampler_spec from a ``scenes.SamplerSpec`` (``weights``: categorical
    noise-count weights over 0..len-1 noises; None keeps ``spec.num_noises`` fixed)."""
    s = RsSamplerSpec()
    s.dim_lo[:] = list(spec.dim_lo)
    s.dim_hi[:] = list(spec.dim_hi)
    s.refl_lo, s.refl_hi = spec.refl_range
    s.t60_max = spec.t60_max
    s.t60_lo, s.t60_hi = spec.t60_range if spec.t60_range is not None else (0.0, 0.0)
    s.snr_lo, s.snr_hi = spec.snr_range_db
    s.mic_spacing, s.mic_radius, s.clearance = spec.mic_spacing, spec.mic_radius, spec.min_wall_clearance
    s.sec_lo, s.sec_hi = spec.seconds_range
    s.fs, s.c0, s.signal_std = fs, c0, signal_std
    s.num_noises, s.mic_count = spec.num_noises, spec.mic_count
    w = list(weights or [])
    s.n_weights = len(w)
    s.weights[: len(w)] = w
    return s


def sample_batch(spec: RsSamplerSpec, n_utt: int, *, seed: int, first_utt: int = 0, epoch: int = 0,
                 eta_db: float = 0.0, plan_rule: int = 0, forced_fft_size: int = 0):
    """Scenes of utterances first_utt.. from the library's host sampler (the fixture
    generator) as a ``scenes.SceneBatch`` without signals."""
    from . import scenes as sc

    L = load_library()
    I = np.zeros(n_utt, np.int32)
    _check(L.rs_sampler_counts(C.byref(spec), seed, first_utt, n_utt, epoch, _ptr(I)))
    src_begin = np.concatenate([[0], np.cumsum(I)]).astype(np.int64)
    n_src, J = int(src_begin[-1]), int(spec.mic_count)
    room = np.zeros((n_utt, 3)); refl = np.zeros(n_utt); order = np.zeros(n_utt, np.int32)
    taps = np.zeros(n_utt, np.int64); src = np.zeros((n_src, 3)); mic = np.zeros((n_utt * J, 3))
    snr = np.zeros(n_src); nx = np.zeros(n_utt, np.int64)
    _check(L.rs_sample_scenes(C.byref(spec), seed, first_utt, n_utt, epoch, _ptr(src_begin), _ptr(room),
                              _ptr(refl), _ptr(order), _ptr(taps), _ptr(src), _ptr(mic), _ptr(snr), _ptr(nx)))
    sig_len = np.repeat(nx, I).astype(np.int64)
    return sc.SceneBatch(
        src_begin=src_begin, mic_begin=(np.arange(n_utt + 1) * J).astype(np.int64), room_dims=room,
        reflection=refl, sample_rate=np.full(n_utt, spec.fs), speed_of_sound=np.full(n_utt, spec.c0),
        image_order=order, max_taps=taps, src_pos=src, mic_pos=mic, snr_db=snr,
        sig_off=sc.signal_offsets(sig_len), sig_len=sig_len,
        signals=None, eta_db=eta_db, plan_rule=plan_rule, forced_fft_size=forced_fft_size, seed=seed,
        utt_ids=first_utt + np.arange(n_utt, dtype=np.int64))


def _signal_meta(batch, first_utt: Optional[int]):
    """(global utterance id, source index within it) of every source of ``batch``: the
    generator's keys.  ``first_utt`` given: utterances first_utt.. (a contiguous batch);
    else the batch's own ids (``SceneBatch.ids``: subsets and shards keep theirs)."""
    I = np.diff(batch.src_begin)
    ids = (np.arange(batch.n_utt, dtype=np.int64) + first_utt) if first_utt is not None else batch.ids
    utt = np.repeat(ids, I).astype(np.int64)
    local = (np.arange(batch.n_src) - np.repeat(batch.src_begin[:-1], I)).astype(np.int32)
    return utt, local


def generate_signals(spec: RsSamplerSpec, batch, *, seed: int, first_utt: Optional[int] = None, epoch: int = 0,
                     device_ptr: Optional[int] = None, stream: int = 0) -> Optional[np.ndarray]:
    """Synthetic N(0, std^2) source signals of ``batch``: on the host (returns the array)
    or straight into device memory at ``device_ptr`` (returns None).  Keyed by each
    source's global utterance id (``batch.ids`` unless ``first_utt`` is given), so a
    subset or a shard gets the same samples as the full batch."""
    L = load_library()
    utt, local = _signal_meta(batch, first_utt)
    off = np.ascontiguousarray(batch.sig_off, np.int64)
    ln = np.ascontiguousarray(batch.sig_len, np.int64)
    if device_ptr is None:
        out = np.zeros(max(batch.total_samples, 1), np.float32)
        _check(L.rs_generate_signals_host(C.byref(spec), seed, epoch, batch.n_src, _ptr(utt), _ptr(local),
                                          _ptr(off), _ptr(ln), _ptr(out)))
        return out
    _check(L.rs_generate_signals(C.byref(spec), seed, epoch, batch.n_src, _ptr(utt), _ptr(local), _ptr(off),
                                 _ptr(ln), device_ptr, stream or None))
    return None


class SignalPlan:
    """rs_signal_plan: the generator table of a fixed batch on the device, built once;
    ``generate(ptr, epoch)`` is then one kernel launch (no host work, no sync)."""

    def __init__(self, spec: RsSamplerSpec, batch, *, seed: int, first_utt: Optional[int] = None):
        L = load_library()
        utt, local = _signal_meta(batch, first_utt)
        off = np.ascontiguousarray(batch.sig_off, np.int64)
        ln = np.ascontiguousarray(batch.sig_len, np.int64)
        h = C.c_void_p()
        _check(L.rs_signal_plan_create(C.byref(spec), seed, batch.n_src, _ptr(utt), _ptr(local), _ptr(off),
                                       _ptr(ln), C.byref(h)))
        self.h = h

    def generate(self, device_ptr: int, *, epoch: int = 0, stream: int = 0) -> None:
        _check(load_library().rs_signal_plan_generate(self.h, int(epoch), C.c_void_p(device_ptr),
                                                      C.c_void_p(stream or None)))

    def close(self):
        if getattr(self, "h", None):
            load_library().rs_signal_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---- log-Mel front end ---------------------------
def logmel_shape(n_samples: int):
    """(frames, stacked 512-element vectors) of an n-sample 16 kHz channel."""
    F, S = C.c_int64(), C.c_int64()
    _check(load_library().rs_logmel_shape(int(n_samples), C.byref(F), C.byref(S)))
    return F.value, S.value


def logmel_device(wave_ptr: int, chan_off, chan_len, feat_ptr: int, feat_off,
                  ctx: Optional[Context] = None) -> None:
    """Stacked log-Mel features of device channels into device memory (see roomsim_gpu.h)."""
    ctx = ctx or default_context()
    co = np.ascontiguousarray(chan_off, np.int64)
    cl = np.ascontiguousarray(chan_len, np.int64)
    fo = np.ascontiguousarray(feat_off, np.int64)
    _check(load_library().rs_logmel_device(ctx.h, wave_ptr, co.size, _ptr(co), _ptr(cl), feat_ptr, _ptr(fo)))


def feature_layout(batch):
    """(per-channel offsets, total floats) of a features buffer sized from the channel
    capacities (out_stride), channels utterance-major then mic."""
    J = np.diff(batch.mic_begin)
    caps = np.repeat(batch.out_stride, J)
    S = np.array([logmel_shape(int(n))[1] for n in caps], np.int64)
    off = np.concatenate([[0], np.cumsum(S * 512)[:-1]]).astype(np.int64) if S.size else np.zeros(0, np.int64)
    return off, int((S * 512).sum())


def render_features(batch, *, device_signals_ptr: int, feat_ptr: int, feat_off, device_out_ptr: Optional[int] = None,
                    ctx: Optional[Context] = None) -> RenderResult:
    """The render with the log-Mel fused into the mix (rs_render_features_device); with
    device_out_ptr None the waveforms are not written."""
    ctx = ctx or default_context()
    L = load_library()
    b, keep = batch.as_struct(RsSceneBatch, signals_ptr=device_signals_ptr)
    out_off = np.ascontiguousarray(batch.out_off, np.int64)
    out_stride = np.ascontiguousarray(batch.out_stride, np.int64)
    out_len = np.zeros(batch.n_utt, np.int64)
    layout = np.zeros(batch.n_pairs, LAYOUT_DTYPE)
    gains = np.zeros(batch.n_pairs)
    power = np.zeros(batch.n_pairs)
    fo = np.ascontiguousarray(feat_off, np.int64)
    st = L.rs_render_features_device(ctx.h, C.byref(b), C.c_void_p(device_out_ptr), _ptr(out_off), _ptr(out_stride),
                                     _ptr(out_len), _ptr(layout), _ptr(gains), _ptr(power), C.c_void_p(feat_ptr),
                                     _ptr(fo))
    del keep
    _check(st)
    return RenderResult(None, out_len, layout, gains, power)
