"""audio_io: the SPEC examples and error contract."""
import struct

import numpy as np
import pytest

from paper_1712_03439_b200 import audio_io as aio
from paper_1712_03439_b200 import roomsim as rs


def test_pcm16_value_mapping(tmp_path):
    p = tmp_path / "a.wav"
    raw = np.array([16384, -32768, 32767, 0], "<i2").tobytes()
    hdr = b"RIFF" + struct.pack("<I", 36 + len(raw)) + b"WAVE"
    hdr += b"fmt " + struct.pack("<IHHIIHH", 16, 1, 1, 16000, 32000, 2, 16) + b"data" + struct.pack("<I", len(raw))
    p.write_bytes(hdr + raw)
    x, fs = aio.read_wav(str(p), expect_rate=16000)
    assert fs == 16000 and x.shape == (1, 4)
    assert x[0, 0] == 0.5 and x[0, 1] == -1.0  # 16384 / 32768


def test_float32_roundtrip_bit_identical(tmp_path):
    x = (np.random.default_rng(1).standard_normal((2, 1001)) * 0.3).astype(np.float32)
    p = str(tmp_path / "f.wav")
    aio.write_wav(x, p, "float32")
    y, _ = aio.read_wav(p)
    assert np.array_equal(y.astype(np.float32).view(np.uint32), x.view(np.uint32))


def test_pcm16_roundtrip_quantization_bound(tmp_path):
    x = np.random.default_rng(2).uniform(-1, 1 - 2 ** -15, (3, 5000))
    p = str(tmp_path / "q.wav")
    assert aio.write_wav(x, p, "pcm16") == 0
    y, _ = aio.read_wav(p)
    assert np.abs(y - x).max() <= 2.0 ** -15
    # ties away from zero, saturation counted
    assert aio.write_wav(np.array([0.5 / 32768, -0.5 / 32768, 1.5, -2.0]), p, "pcm16") == 2
    y, _ = aio.read_wav(p)
    assert y[0, 0] == 1 / 32768 and y[0, 1] == -1 / 32768 and y[0, 2] == 32767 / 32768 and y[0, 3] == -1.0


def test_errors(tmp_path):
    p = tmp_path / "bad.wav"
    p.write_bytes(b"RIFF\x00\x00\x00\x00WAVEjunk")
    with pytest.raises(rs.FormatError):
        aio.read_wav(str(p))
    with pytest.raises(rs.IoError):
        aio.read_wav(str(tmp_path / "missing.wav"))
    with pytest.raises(rs.ConfigError):
        aio.write_wav(np.array([np.nan]), str(tmp_path / "n.wav"))
    good = str(tmp_path / "g.wav")
    aio.write_wav(np.zeros(10), good, "float32", rate=8000)
    with pytest.raises(rs.ConfigError):
        aio.read_wav(good, expect_rate=16000)
    data = open(good, "rb").read()
    open(good, "wb").write(data[:-6])  # truncated data chunk
    with pytest.raises(rs.FormatError):
        aio.read_wav(good)
