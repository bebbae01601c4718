"""Host model of the external product's rounding margin.

Negacyclic products of four random gadget-digit polynomials (|d| <= 2^8,
PARAM_128's Bg = 2^9) with four random 32-bit key polynomials, through the
folded FP64 FFT (numpy), summed in the frequency domain and inverse
transformed -- once with the full 32-bit key words (v5) and once with the
balanced low 16-bit half (the split key of v3).  Prints the worst
|x - rint(x)| of each over TRIALS x 2 x 1024 rounded values."""
import sys

import numpy as np

N, M = 1024, 512
TRIALS = int(sys.argv[1]) if len(sys.argv) > 1 else 200
tw = np.exp(1j * np.pi * np.arange(M) / N)


def fold(a):
    return (a[..., :M] + 1j * a[..., M:]) * tw


def unfold(z):
    z = z / tw
    return np.concatenate([z.real, z.imag], axis=-1)


rng = np.random.default_rng(1)
worst_full = worst_lo = 0.0
for _ in range(TRIALS):
    D = rng.integers(-256, 256, size=(4, N)).astype(np.float64)
    K = rng.integers(-2 ** 31, 2 ** 31, size=(2, 4, N)).astype(np.int64)  # [component][row]
    FD = np.fft.fft(fold(D), axis=-1)
    for c in range(2):
        R = unfold(np.fft.ifft((FD * np.fft.fft(fold(K[c].astype(np.float64)), axis=-1)).sum(0)))
        worst_full = max(worst_full, float(np.abs(R - np.rint(R)).max()))
        lo = ((K[c] + 2 ** 15) % 2 ** 16) - 2 ** 15
        RL = unfold(np.fft.ifft((FD * np.fft.fft(fold(lo.astype(np.float64)), axis=-1)).sum(0)))
        worst_lo = max(worst_lo, float(np.abs(RL - np.rint(RL)).max()))
print(f"{TRIALS} trials: one key image (v5) worst {worst_full:.4g}, split-key half (v3) worst {worst_lo:.4g}")
