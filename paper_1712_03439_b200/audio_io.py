"""WAV reader / writer for the rendered channels (SPEC.md:397-421 `audio_io`; SURVEY.md §8f
row 3, the data format on the output side of the path).  The reference specifies the
contract but ships no code for it.

* read_wav: RIFF/WAVE, PCM 16-bit (mapped to [-1, 1) by / 32768) or IEEE float 32-bit
  (passed through); channels preserved -> float64 array [channels, frames].
* write_wav: pcm16 rounds to nearest with ties away from zero and saturates out-of-range
  samples (returned as a counter); float32 is lossless.  Non-finite samples are an error.
* Canonical rate 16 kHz; other rates are rejected by `read_wav(..., expect_rate=16000)`.
"""
from __future__ import annotations

import os
import struct

import numpy as np

from .roomsim import ConfigError, FormatError, IoError

_PCM, _FLOAT = 1, 3


def read_wav(path: str, expect_rate: int | None = None):
    """-> (samples float64 [channels, frames], sample_rate)."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError as e:
        raise IoError(f"cannot read {path}: {e}") from e
    if len(data) < 12 or data[:4] != b"RIFF" or data[8:12] != b"WAVE":
        raise FormatError("not a RIFF/WAVE file")
    pos, fmt, raw = 12, None, None
    while pos + 8 <= len(data):
        cid, size = data[pos:pos + 4], struct.unpack_from("<I", data, pos + 4)[0]
        body = data[pos + 8:pos + 8 + size]
        if cid == b"fmt ":
            if len(body) < 16:
                raise FormatError("malformed fmt chunk")
            fmt = struct.unpack_from("<HHIIHH", body, 0)
        elif cid == b"data":
            if len(body) < size:
                raise FormatError("truncated data chunk")
            raw = body
        pos += 8 + size + (size & 1)
    if fmt is None or raw is None:
        raise FormatError("missing fmt or data chunk")
    tag, ch, rate, _, align, bits = fmt
    if ch < 1 or align != ch * bits // 8:
        raise FormatError("inconsistent channel count / block alignment")
    if expect_rate is not None and rate != expect_rate:
        raise ConfigError(f"sample rate {rate} Hz, expected {expect_rate} Hz (no resampling)")
    if len(raw) % align:
        raise FormatError("data chunk is not a whole number of frames")
    if tag == _PCM and bits == 16:
        x = np.frombuffer(raw, "<i2").astype(np.float64) / 32768.0
    elif tag == _FLOAT and bits == 32:
        x = np.frombuffer(raw, "<f4").astype(np.float64)
    else:
        raise FormatError(f"unsupported codec {tag} / {bits}-bit (PCM 16 or float 32)")
    return x.reshape(-1, ch).T.copy(), rate


def write_wav(samples, path: str, fmt: str = "float32", rate: int = 16000) -> int:
    """Write [channels, frames] (or [frames]) samples; returns the pcm16 saturation count."""
    x = np.atleast_2d(np.asarray(samples, np.float64))
    if not np.isfinite(x).all():
        raise ConfigError("non-finite samples")
    ch, n = x.shape
    inter = x.T.reshape(-1)
    clipped = 0
    if fmt == "pcm16":
        q = np.sign(inter) * np.floor(np.abs(inter) * 32768.0 + 0.5)  # nearest, ties away from 0
        clipped = int(((q > 32767) | (q < -32768)).sum())
        payload = np.clip(q, -32768, 32767).astype("<i2").tobytes()
        tag, bits = _PCM, 16
    elif fmt == "float32":
        payload = inter.astype("<f4").tobytes()
        tag, bits = _FLOAT, 32
    else:
        raise ConfigError(f"unknown format {fmt!r} (pcm16 or float32)")
    align = ch * bits // 8
    hdr = b"RIFF" + struct.pack("<I", 36 + len(payload)) + b"WAVE"
    hdr += b"fmt " + struct.pack("<IHHIIHH", 16, tag, ch, rate, rate * align, align, bits)
    hdr += b"data" + struct.pack("<I", len(payload))
    try:
        with open(path, "wb") as f:
            f.write(hdr + payload)
    except OSError as e:
        raise IoError(f"cannot write {path}: {e}") from e
    return clipped


def write_render(batch, result, prefix: str, fmt: str = "float32") -> list:
    """One multichannel WAV per utterance of a render (`render_batch` result)."""
    paths = []
    J = np.diff(batch.mic_begin)
    for u in range(batch.n_utt):
        chans = np.stack([batch.channel(result.out, u, j, result.out_len[u]) for j in range(J[u])])
        p = f"{prefix}{u:06d}.wav"
        write_wav(chans, p, fmt, int(batch.sample_rate[u]))
        paths.append(os.path.abspath(p))
    return paths
