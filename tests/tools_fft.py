"""Test helper: numpy inverse of the engine's native FFT-domain key layout
(index maps of csrc/fft.cuh, replayed by tools/fft_model.py)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
from fft_model import freq_index, geometry  # noqa: E402


def native_inverse_poly(fft_flat, n, l, N):
    """[i][c][h][s][r][lane] complex (scaled 1/M) -> (n, 2l, 2, N) int64 = lo + 2^16 hi."""
    M, P, L, _ = geometry(N)
    R = 2 * l
    arr = fft_flat.reshape(n, 2, 2, P, R, L)           # i c h s r lane
    K = freq_index(N)                                   # [lane][slot] -> k
    Z = np.zeros((n, 2, R, 2, M), complex)              # i c r h k
    for lane in range(L):
        for s in range(P):
            Z[..., K[lane, s]] = arr[:, :, :, s, :, lane].transpose(0, 1, 3, 2)
    m = np.arange(M)
    # forward used kernel e^{+2 pi i mk/M} and the key is pre-scaled by 1/M, so
    # sum_k Z_k e^{-2 pi i mk/M} (numpy's forward fft) recovers z exactly
    z = np.fft.fft(Z, axis=-1)
    v = z * np.exp(-1j * np.pi * m / N)
    halves = np.rint(np.concatenate([v.real, v.imag], axis=-1)).astype(np.int64)  # (n,2,R,2,N)
    val = halves[:, :, :, 0, :] + (halves[:, :, :, 1, :] << 16)                   # (n,2,R,N)
    return val.transpose(0, 2, 1, 3)                                               # (n,R,2,N)
