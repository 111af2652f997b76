"""numpy model of the 16-points-per-lane K3 transform (N = 1024, 64 lanes per
pair): radix-16 over r per class, exchange E, radix-16 over c' per (k1, c0),
exchange F, radix-4 over c0, natural C, post with 8 k per lane.  Also checks
the shared-memory bank pattern of every access."""
import numpy as np

N = 1024; n = N - 1; Q = 64; L = 64
s = np.sqrt(2.0 / N); h = s / 2
al = s / 2 * np.sin(np.pi * np.arange(N) / N) + s / 4
W = lambda M, e: np.exp(-2j * np.pi * e / M)
ES, FS = 68, 19
pc = lambda k: k + (k >> 3) + 2 * (k >> 6)


def conflicts(addr_lists):
    """addr_lists: per lane the 16-byte unit index of one warp-wide access;
    returns the max conflict degree over the 4 quarter-warp phases."""
    worst = 1
    for ph in range(4):
        units = [a % 8 for a in addr_lists[8 * ph: 8 * ph + 8]]
        worst = max(worst, max(units.count(u) for u in set(units)))
    return worst


def model(A, B):
    x = lambda R, j: 0.0 if j == 0 or j == N else R[j - 1]
    Bc = np.zeros((16, Q), complex)   # B_c[k1]
    for t in range(L):
        v = np.zeros(16, complex)
        for r in range(16):
            j = t + Q * r
            if j:
                v[r] = (al[j] * x(A, j) + (al[j] - h) * x(A, N - j)) + 1j * (al[j] * x(B, j) + (al[j] - h) * x(B, N - j))
        Bc[:, t] = np.fft.fft(v) * W(N, t * np.arange(16))
    H = np.zeros((16, 4, 16), complex)   # [k1][c0][k2']
    for lam in range(64):
        k1, c0 = lam >> 2, lam & 3
        g = np.array([Bc[k1, c0 + 4 * cp] for cp in range(16)])
        H[k1, c0] = np.fft.fft(g) * W(64, c0 * np.arange(16))
    C = np.zeros(N, complex)
    for lam in range(64):
        k1, c0 = lam >> 2, lam & 3
        for i in range(4):
            k2p = 4 * c0 + i
            out = np.fft.fft(H[k1, :, k2p])
            for k3 in range(4):
                C[k1 + 16 * (k2p + 16 * k3)] = out[k3]
    ref = np.fft.fft([0] + [(al[j] * x(A, j) + (al[j] - h) * x(A, N - j)) + 1j * (al[j] * x(B, j) + (al[j] - h) * x(B, N - j)) for j in range(1, N)])
    assert np.allclose(C, ref)
    return C


rng = np.random.default_rng(0)
model(rng.standard_normal(n), rng.standard_normal(n))
print("math ok")
# bank conflicts per access pattern (per warp: lanes 0..31 of the team, and 32..63)
for wbase in (0, 32):
    lanes = range(wbase, wbase + 32)
    pats = {
        "E write": [[k1 * ES + t for t in lanes] for k1 in range(16)],
        "E read": [[(lam >> 2) * ES + (lam & 3) + 4 * cp for lam in lanes] for cp in range(16)],
        "F write": [[lam * FS + k2 + ((k2 >> 2) & 3) for lam in lanes] for k2 in range(16)],
        "F read": [[((lam >> 2) * 4 + c0p) * FS + 4 * (lam & 3) + i + (lam & 3) for lam in lanes] for c0p in range(4) for i in range(4)],
        "C write": [[pc((lam >> 2) + 16 * (4 * (lam & 3) + i + 16 * k3)) for lam in lanes] for i in range(4) for k3 in range(4)],
        "C read own": [[pc(8 * t + i) for t in lanes] for i in range(9)],
        "C read mirror": [[pc(N - 8 * t - i) if 8 * t + i else 0 for t in lanes] for i in range(9)],
    }
    print(wbase, {k: max(conflicts(a) for a in v) for k, v in pats.items()})
print("units", pc(N - 1) + 1, 16 * ES, 64 * FS)
