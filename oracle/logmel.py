"""CPU restatement (numpy, FP64) of the log-Mel front end described in PAPER.md:452-460 —
test infrastructure only, the checker of paper_1712_03439_b200/csrc/features.cu.

The paper fixes: 128 log-Mel features, 32 ms window, 10 ms frame interval, Mel
filterbank cut-offs 125 Hz and 7500 Hz, four frames stacked (128 x 4 = 512) and the
stacked sequence down-sampled by three.  The unstated details are fixed here and in
features.cu alike: 16 kHz audio, periodic Hann window, 512-point FFT, power spectrum,
HTK mel scale 2595 log10(1 + f/700) with 130 equally spaced edges, unnormalised
triangles, natural log with floor 1e-10, stacked vector t = frames 3t .. 3t+3.
"""
import numpy as np

FRAME, HOP, MELS = 512, 160, 128


def shape(n):
    F = 1 + (n - FRAME) // HOP if n >= FRAME else 0
    return F, ((F - 4) // 3 + 1 if F >= 4 else 0)


def filterbank():
    mel = lambda f: 2595.0 * np.log10(1.0 + f / 700.0)  # noqa: E731
    hz = lambda m: 700.0 * (10.0 ** (m / 2595.0) - 1.0)  # noqa: E731
    edge = hz(mel(125.0) + (mel(7500.0) - mel(125.0)) * np.arange(130) / 129.0)
    f = np.arange(257) * 16000.0 / FRAME
    fb = np.zeros((MELS, 257))
    for m in range(MELS):
        up = (f > edge[m]) & (f <= edge[m + 1])
        dn = (f > edge[m + 1]) & (f < edge[m + 2])
        fb[m, up] = (f[up] - edge[m]) / (edge[m + 1] - edge[m])
        fb[m, dn] = (edge[m + 2] - f[dn]) / (edge[m + 2] - edge[m + 1])
    return fb


def logmel(x):
    """Stacked features [n_stacked, 512] of one 16 kHz channel."""
    x = np.asarray(x, np.float64)
    F, S = shape(x.size)
    if S == 0:
        return np.zeros((0, 4 * MELS))
    win = 0.5 - 0.5 * np.cos(2 * np.pi * np.arange(FRAME) / FRAME)
    idx = np.arange(FRAME)[None, :] + HOP * np.arange(F)[:, None]
    spec = np.abs(np.fft.rfft(x[idx] * win, axis=1)) ** 2
    lm = np.log(np.maximum(spec @ filterbank().T, 1e-10))
    t = np.arange(S)
    return np.concatenate([lm[3 * t + c] for c in range(4)], axis=1)
