"""NumPy model of the warp FFT used by the blind-rotation kernel.

Design check only (not product, not oracle): it replays, lane by lane, the exact
index maps of csrc/fft.cuh -- in-thread DIF DFT-P, lane twiddle, smem transpose,
in-thread DFT-P, lane-pair radix-2 -- and the mirrored inverse, so the layout
can be validated on the CPU before the CUDA code runs on a B200.
M = N/2 complex points, P = sqrt(M/2) values per lane, L = 2P lanes.
"""
import numpy as np


def bitrev(x, bits):
    r = 0
    for _ in range(bits):
        r = (r << 1) | (x & 1)
        x >>= 1
    return r


def dif(x, sign):
    """In-place radix-2 DIF on the last axis; output in bit-reversed order."""
    x = x.copy()
    P = x.shape[-1]
    ln = P
    while ln >= 2:
        h = ln // 2
        for st in range(0, P, ln):
            for j in range(h):
                a = x[..., st + j].copy()
                b = x[..., st + j + h].copy()
                x[..., st + j] = a + b
                x[..., st + j + h] = (a - b) * np.exp(sign * 2j * np.pi * j / ln)
        ln //= 2
    return x


def dit(x, sign):
    """In-place radix-2 DIT on the last axis; bit-reversed input, natural output."""
    x = x.copy()
    P = x.shape[-1]
    ln = 2
    while ln <= P:
        h = ln // 2
        for st in range(0, P, ln):
            for j in range(h):
                a = x[..., st + j].copy()
                b = x[..., st + j + h] * np.exp(sign * 2j * np.pi * j / ln)
                x[..., st + j] = a + b
                x[..., st + j + h] = a - b
        ln *= 2
    return x


def geometry(N):
    M = N // 2
    P = int(round((M // 2) ** 0.5))
    assert 2 * P * P == M
    return M, P, 2 * P, P.bit_length() - 1


def forward(z):
    """z: (M,) complex natural order -> (L, P) native layout [lane][slot]."""
    M = z.shape[0]
    _, P, L, lp = geometry(2 * M)
    x = np.array([[z[L * m1 + l] for m1 in range(P)] for l in range(L)])  # lane l, slot m1
    x = dif(x, +1)                                                        # x[l][bitrev(k1)]
    for l in range(L):
        for k1 in range(P):
            x[l, bitrev(k1, lp)] *= np.exp(2j * np.pi * l * k1 / M)
    # transpose: (m2=l, k1) -> lane 2*k1 + (l&1), slot l>>1
    y = np.zeros((L, P), complex)
    for l in range(L):
        for k1 in range(P):
            y[2 * k1 + (l & 1), l >> 1] = x[l, bitrev(k1, lp)]
    u = dif(y, +1)                                                        # u[lane][bitrev(c)]
    X = np.zeros((L, P), complex)
    w = lambda c: np.exp(2j * np.pi * c / (2 * P))
    for lane in range(L):
        b = lane & 1
        partner = lane ^ 1
        for j in range(P // 2):
            clo, chi = j, j + P // 2
            send_p = u[partner, bitrev(clo, lp)] if (partner & 1) else u[partner, bitrev(chi, lp)]
            recv = send_p
            u0 = recv if b else u[lane, bitrev(clo, lp)]
            u1 = u[lane, bitrev(chi, lp)] if b else recv
            c = chi if b else clo
            t = u1 * w(c)
            X[lane, j] = u0 + t
            X[lane, j + P // 2] = u0 - t
    return X


def freq_index(N):
    """k(lane, slot) for the native layout."""
    M, P, L, lp = geometry(N)
    K = np.zeros((L, P), int)
    for lane in range(L):
        k1, b = lane >> 1, lane & 1
        for s in range(P):
            c = b * (P // 2) + (s % (P // 2))
            d = s // (P // 2)
            K[lane, s] = k1 + P * (c + P * d)
    return K


def inverse(X):
    """(L, P) native layout -> (M,) natural order, scaled by M (not divided)."""
    L, P = X.shape
    M = L * P
    lp = P.bit_length() - 1
    w = lambda c: np.exp(2j * np.pi * c / (2 * P))
    u = np.zeros((L, P), complex)
    for lane in range(L):
        b = lane & 1
        partner = lane ^ 1
        for j in range(P // 2):
            clo, chi = j, j + P // 2
            S = X[lane, j] + X[lane, j + P // 2]
            D = (X[lane, j] - X[lane, j + P // 2]) * np.conj(w(chi if b else clo))
            Sp = X[partner, j] + X[partner, j + P // 2]
            Dp = (X[partner, j] - X[partner, j + P // 2]) * np.conj(w(chi if (partner & 1) else clo))
            recv = Sp if (partner & 1) else Dp
            u[lane, bitrev(clo, lp)] = recv if b else S
            u[lane, bitrev(chi, lp)] = D if b else recv
    y = dit(u, -1)                                                         # y[lane][a]
    x = np.zeros((L, P), complex)
    for lane in range(L):
        k1, b = lane >> 1, lane & 1
        for a in range(P):
            x[b + 2 * a, bitrev(k1, lp)] = y[lane, a]
    for l in range(L):
        for k1 in range(P):
            x[l, bitrev(k1, lp)] *= np.exp(-2j * np.pi * l * k1 / M)
    x = dit(x, -1)                                                         # x[l][m1]
    z = np.zeros(M, complex)
    for l in range(L):
        for m1 in range(P):
            z[L * m1 + l] = x[l, m1]
    return z


def negacyclic_fold(a):
    N = a.shape[0]
    M = N // 2
    m = np.arange(M)
    return (a[:M] + 1j * a[M:]) * np.exp(1j * np.pi * m / N)


def negacyclic_unfold(z):
    M = z.shape[0]
    N = 2 * M
    m = np.arange(M)
    v = z * np.exp(-1j * np.pi * m / N)
    return np.concatenate([v.real, v.imag])


def check(N, trials=3):
    M, P, L, _ = geometry(N)
    rng = np.random.default_rng(N)
    K = freq_index(N)
    assert sorted(K.ravel()) == list(range(M))
    for _ in range(trials):
        z = rng.standard_normal(M) + 1j * rng.standard_normal(M)
        X = forward(z)
        ref = np.array([np.sum(z * np.exp(2j * np.pi * np.arange(M) * k / M)) for k in range(M)])
        assert np.allclose(X, ref[K]), "forward layout mismatch"
        back = inverse(X) / M
        assert np.allclose(back, z), "inverse mismatch"
        # negacyclic product of integer polys through the layout
        a = rng.integers(-256, 256, N).astype(float)
        b = rng.integers(-2**15, 2**15, N).astype(float)
        prod = inverse(forward(negacyclic_fold(a)) * forward(negacyclic_fold(b))) / M
        got = np.rint(negacyclic_unfold(prod)).astype(np.int64)
        full = np.convolve(a.astype(np.int64), b.astype(np.int64))
        want = full[:N] - np.concatenate([full[N:], [0]])
        assert np.array_equal(got, want), "negacyclic product mismatch"
    print(f"N={N}: P={P} L={L} ok")


if __name__ == "__main__":
    for N in (64, 256, 1024):
        check(N, trials=1 if N == 1024 else 3)
