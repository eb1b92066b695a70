"""TEST INFRASTRUCTURE ONLY — ctypes access to the CPU checkers.

Two libraries with identical signatures:
  * ``port()``      -> oracle/_build/libroomsim_oracle.so, the plain-C
                       restatement of the reference path (roomsim_oracle.c);
  * ``reference()`` -> oracle/_ref/libroomsim_ref.so, the reference headers
                       themselves compiled from /root/reference (ref_driver.cpp).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this
package.  The product (paper_1712_03439_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libroomsim_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libroomsim_ref.so")

RS_DIRECT, RS_FULL_FFT, RS_OVERLAP_ADD = 0, 1, 2

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_sz = C.c_size_t
_szp = C.POINTER(C.c_size_t)


class RsSceneBatch(C.Structure):
    """Mirror of rs_scene_batch (include/roomsim_gpu.h)."""

    _fields_ = [
        ("n_utt", C.c_int64),
        ("src_begin", C.c_void_p),
        ("mic_begin", C.c_void_p),
        ("room_dims", C.c_void_p),
        ("reflection", C.c_void_p),
        ("sample_rate", C.c_void_p),
        ("speed_of_sound", C.c_void_p),
        ("image_order", C.c_void_p),
        ("max_taps", C.c_void_p),
        ("src_pos", C.c_void_p),
        ("mic_pos", C.c_void_p),
        ("snr_db", C.c_void_p),
        ("sig_off", C.c_void_p),
        ("sig_len", C.c_void_p),
        ("signals", C.c_void_p),
        ("eta_db", C.c_double),
        ("plan_rule", C.c_int32),
        ("forced_fft_size", C.c_int64),
    ]


class RsPairLayout(C.Structure):
    _fields_ = [
        ("rir_len", C.c_int64),
        ("rir_keep", C.c_int64),
        ("cutoff", C.c_int64),
        ("fft_size", C.c_int64),
        ("block_len", C.c_int64),
        ("n_blocks", C.c_int64),
        ("out_len", C.c_int64),
        ("strategy", C.c_int32),
        ("flags", C.c_int32),
    ]


LAYOUT_DTYPE = np.dtype(
    [
        ("rir_len", np.int64),
        ("rir_keep", np.int64),
        ("cutoff", np.int64),
        ("fft_size", np.int64),
        ("block_len", np.int64),
        ("n_blocks", np.int64),
        ("out_len", np.int64),
        ("strategy", np.int32),
        ("flags", np.int32),
    ]
)
assert LAYOUT_DTYPE.itemsize == C.sizeof(RsPairLayout)


def build() -> None:
    """Compile the checkers (make -C oracle); _ref only where /root/reference exists."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class _Lib:
    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.path = path
        self.lib = C.CDLL(path)
        self.p = prefix
        L, p = self.lib, prefix
        sig = {
            "last_error": (C.c_char_p, []),
            "virtual_source_count": (_sz, [C.c_int]),
            "enumerate_images": (C.c_int, [_dp, C.c_double, C.c_double, C.c_double, C.c_int, _dp, _dp, _ip, _sz]),
            "synthesize_rir": (C.c_int, [_dp, C.c_double, C.c_double, C.c_double, C.c_int, _dp, _dp, C.c_int64, _dp, _sz, _szp]),
            "power_threshold": (C.c_int, [_dp, _sz, C.c_double, C.POINTER(C.c_double)]),
            "cutoff_index": (C.c_int, [_dp, _sz, C.c_double, _szp]),
            "truncate_rir": (C.c_int, [_dp, _sz, C.c_double, _szp, _szp, C.POINTER(C.c_double)]),
            "cost_direct": (C.c_double, [C.c_double, C.c_double, _sz, _sz]),
            "cost_full_fft": (C.c_double, [C.c_double, C.c_double, _sz, _sz, _sz]),
            "cost_ola": (C.c_double, [C.c_double, C.c_double, _sz, _sz, _sz]),
            "ola_block_count": (_sz, [_sz, _sz, _sz]),
            "plan_for": (C.c_int, [C.c_double, C.c_double, _sz, _sz, C.c_int, C.POINTER(C.c_int), _szp, C.POINTER(C.c_double)]),
            "choose_plan": (C.c_int, [C.c_double, C.c_double, _sz, _sz, C.POINTER(C.c_int), _szp, C.POINTER(C.c_double)]),
            "rfft_forward": (C.c_int, [_sz, _dp, _dp]),
            "rfft_inverse": (C.c_int, [_sz, _dp, _dp]),
            "convolve_direct": (C.c_int, [_dp, _sz, _dp, _sz, _dp]),
            "convolve_full_fft": (C.c_int, [_dp, _sz, _dp, _sz, _dp]),
            "convolve_ola": (C.c_int, [_dp, _sz, _dp, _sz, _sz, _dp]),
            "mean_power": (C.c_int, [_dp, _sz, C.POINTER(C.c_double)]),
            "compute_gain": (C.c_int, [C.c_double, C.c_double, C.c_double, C.POINTER(C.c_double)]),
            "render_batch": (C.c_int, [C.POINTER(RsSceneBatch), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, p + name)
            f.restype = res
            f.argtypes = args
            setattr(self, name + "_raw", f)
        if prefix == "ref_":
            L.ref_hardware_concurrency.restype = C.c_int
            L.ref_set_malloc_tuning.restype = C.c_int
            L.ref_set_malloc_tuning.argtypes = [C.c_int]

    def _check(self, st: int) -> None:
        if st != 0:
            raise OracleError(st, self.last_error_raw().decode())

    # ---- room model ------------------------------------------------------
    def virtual_source_count(self, order: int) -> int:
        return int(self.virtual_source_count_raw(order))

    def enumerate_images(self, room, refl, order, src, fs=16000.0, c0=343.0):
        V = self.virtual_source_count(order)
        pos = np.zeros(3 * V)
        g = np.zeros(V, dtype=np.int32)
        self._check(self.enumerate_images_raw(np.asarray(room, float), refl, fs, c0, order,
                                              np.asarray(src, float), pos, g, V))
        return pos.reshape(V, 3), g

    def synthesize_rir(self, room, refl, order, src, mic, fs=16000.0, c0=343.0, max_taps=0,
                       cap=None):
        room = np.asarray(room, float)
        if cap is None:
            ext = (abs(order) + 2) * room
            cap = int(np.ceil(np.sqrt((ext ** 2).sum()) * fs / c0)) + 4
            if max_taps:
                cap = min(cap, int(max_taps))
        out = np.zeros(max(cap, 1))
        n = C.c_size_t(0)
        self._check(self.synthesize_rir_raw(room, refl, fs, c0, order, np.asarray(src, float),
                                            np.asarray(mic, float), int(max_taps), out, cap,
                                            C.byref(n)))
        return out[: n.value].copy()

    def power_threshold(self, h, eta):
        v = C.c_double()
        h = np.ascontiguousarray(h, float)
        self._check(self.power_threshold_raw(h, h.size, eta, C.byref(v)))
        return v.value

    def cutoff_index(self, h, th):
        v = C.c_size_t()
        h = np.ascontiguousarray(h, float)
        self._check(self.cutoff_index_raw(h, h.size, th, C.byref(v)))
        return v.value

    def truncate_rir(self, h, eta):
        h = np.ascontiguousarray(h, float)
        keep, nc, th = C.c_size_t(), C.c_size_t(), C.c_double()
        self._check(self.truncate_rir_raw(h, h.size, eta, C.byref(keep), C.byref(nc), C.byref(th)))
        return h[: keep.value].copy(), nc.value, th.value

    # ---- planner ---------------------------------------------------------
    def cost_direct(self, I, J, nx, nh):
        return self.cost_direct_raw(I, J, nx, nh)

    def cost_full_fft(self, I, J, nx, nh, n):
        return self.cost_full_fft_raw(I, J, nx, nh, n)

    def cost_ola(self, I, J, nx, nh, n):
        return self.cost_ola_raw(I, J, nx, nh, n)

    def ola_block_count(self, nx, nh, n):
        return int(self.ola_block_count_raw(nx, nh, n))

    def plan_for(self, I, J, nx, nh, strategy):
        s, n, c = C.c_int(), C.c_size_t(), C.c_double()
        self._check(self.plan_for_raw(I, J, nx, nh, strategy, C.byref(s), C.byref(n), C.byref(c)))
        return s.value, n.value, c.value

    def choose_plan(self, I, J, nx, nh):
        s, n, c = C.c_int(), C.c_size_t(), C.c_double()
        self._check(self.choose_plan_raw(I, J, nx, nh, C.byref(s), C.byref(n), C.byref(c)))
        return s.value, n.value, c.value

    # ---- FFT / convolution ---------------------------------------------
    def rfft_forward(self, x):
        x = np.ascontiguousarray(x, float)
        out = np.zeros(2 * (x.size // 2 + 1))
        self._check(self.rfft_forward_raw(x.size, x, out))
        return out[0::2] + 1j * out[1::2]

    def rfft_inverse(self, spec, n):
        s = np.zeros(2 * (n // 2 + 1))
        s[0::2] = np.real(spec)
        s[1::2] = np.imag(spec)
        out = np.zeros(n)
        self._check(self.rfft_inverse_raw(n, s, out))
        return out

    def _conv(self, fn, x, h, *extra):
        x = np.ascontiguousarray(x, float)
        h = np.ascontiguousarray(h, float)
        out = np.zeros(max(x.size + h.size - 1, 1))
        self._check(fn(x, x.size, h, h.size, *extra, out))
        return out[: x.size + h.size - 1]

    def convolve_direct(self, x, h):
        return self._conv(self.convolve_direct_raw, x, h)

    def convolve_full_fft(self, x, h):
        return self._conv(self.convolve_full_fft_raw, x, h)

    def convolve_ola(self, x, h, n):
        return self._conv(self.convolve_ola_raw, x, h, n)

    def mean_power(self, v):
        v = np.ascontiguousarray(v, float)
        p = C.c_double()
        self._check(self.mean_power_raw(v, v.size, C.byref(p)))
        return p.value

    def compute_gain(self, pt, pn, snr):
        a = C.c_double()
        self._check(self.compute_gain_raw(pt, pn, snr, C.byref(a)))
        return a.value

    # ---- batch render ----------------------------------------------------
    def render_batch(self, scene, threads: int = 1):
        """Render a ``paper_1712_03439_b200.scenes.SceneBatch`` on the CPU.

        Returns (out[float64], out_len, layout[LAYOUT_DTYPE], gains, power)."""
        b, keep = scene.as_struct(RsSceneBatch)
        out = np.zeros(scene.out_total)
        out_len = np.zeros(scene.n_utt, np.int64)
        layout = np.zeros(scene.n_pairs, LAYOUT_DTYPE)
        gains = np.zeros(scene.n_pairs)
        power = np.zeros(scene.n_pairs)
        out_off = np.ascontiguousarray(scene.out_off, np.int64)  # keep alive across the call
        out_stride = np.ascontiguousarray(scene.out_stride, np.int64)
        st = self.render_batch_raw(C.byref(b), out.ctypes.data, out_off.ctypes.data,
                                   out_stride.ctypes.data, out_len.ctypes.data,
                                   layout.ctypes.data, gains.ctypes.data, power.ctypes.data,
                                   int(threads))
        del keep
        self._check(st)
        return out, out_len, layout, gains, power


_cache: dict = {}


def port() -> _Lib:
    if "port" not in _cache:
        if not os.path.exists(PORT_SO):
            build()
        _cache["port"] = _Lib(PORT_SO, "orc_")
    return _cache["port"]


def reference_available() -> bool:
    if not os.path.exists(REF_SO):
        try:
            build()
        except Exception:
            return False
    return os.path.exists(REF_SO)


def reference() -> _Lib:
    if "ref" not in _cache:
        if not reference_available():
            raise FileNotFoundError(REF_SO)
        _cache["ref"] = _Lib(REF_SO, "ref_")
    return _cache["ref"]
