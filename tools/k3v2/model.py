"""Lane-level numpy model of the K3v2 real-symmetric DST-I (one row pair),
mirroring the CUDA kernel's data movement: class-pair loads, radix-16 pass,
exchange, radix-32 + cross-lane radix-R3, natural-order C, post (mirror +
scan).  Validates index arithmetic against the orthonormal DST-I."""
import numpy as np


def dst_ref(x):
    n = x.shape[-1]
    N = n + 1
    j = np.arange(1, n + 1)
    S = np.sin(np.pi * np.outer(j, j) / N) * np.sqrt(2.0 / N)
    return x @ S


def model(A, B):
    n = A.shape[0]
    N = n + 1
    Q = N // 16          # classes
    L = Q // 2           # lanes per pair
    s = np.sqrt(2.0 / N)
    h = 0.5 * s
    al = s / 2 * np.sin(np.pi * np.arange(N) / N) + s / 4
    x = lambda R, j: 0.0 if j == 0 or j == N else R[j - 1]
    W = lambda M, e: np.exp(-2j * np.pi * e / M)
    # ---- pass 1: lane t holds classes c1 = t, c2 = Q - t (lane 0: 0 and Q/2)
    B1 = {}   # B_c[k1]
    for t in range(L):
        classes = (0, Q // 2) if t == 0 else (t, Q - t)
        for c in classes:
            v = np.zeros(16, complex)
            for r in range(16):
                j = c + Q * r
                if j == 0:
                    continue
                ya = al[j] * x(A, j) + (al[j] - h) * x(A, N - j)
                yb = al[j] * x(B, j) + (al[j] - h) * x(B, N - j)
                v[r] = ya + 1j * yb
            Aout = np.fft.fft(v)
            B1[c] = Aout * W(N, c * np.arange(16))
    # ---- stage 2: lane (k1, c0), R3 = Q/32 (Q >= 64) else R3 = 1
    R3 = max(1, Q // 32)
    C = np.zeros(N, complex)
    for k1 in range(16):
        G = np.zeros((R3, 32), complex)
        for c0 in range(R3):
            vals = np.array([B1[c0 + R3 * cp][k1] for cp in range(Q // R3)])
            G[c0] = np.fft.fft(vals)     # over c' -> k2'
        for k2p in range(Q // R3):
            H = np.array([W(Q, c0 * k2p) * G[c0][k2p] for c0 in range(R3)])
            out = np.fft.fft(H)          # over c0 -> k3
            for k3 in range(R3):
                C[k1 + 16 * (k2p + (Q // R3) * k3)] = out[k3]
    assert np.allclose(C, np.fft.fft(np.array([0] + [al[j] * x(A, j) + (al[j] - h) * x(A, N - j) + 1j * (al[j] * x(B, j) + (al[j] - h) * x(B, N - j)) for j in range(1, N)])))
    # ---- post: lane t owns k in [16t, 16t + 16]
    XA = np.zeros(N)
    XB = np.zeros(N)
    tot = []
    lane = []
    for t in range(L):
        ea, eb, da, db = [], [], [], []
        for i in range(17):
            k = 16 * t + i
            c = C[k % N]
            c2 = 0.0 if k == 0 else C[N - k]
            ea.append(c2.imag - c.imag)
            eb.append(c.real - c2.real)
            da.append(c.real + c2.real)
            db.append(c.imag + c2.imag)
        Sa = np.cumsum(da[:16])
        Sb = np.cumsum(db[:16])
        lane.append((ea, eb, Sa, Sb))
        tot.append((Sa[-1], Sb[-1]))
    pa = pb = 0.0
    for t in range(L):
        ea, eb, Sa, Sb = lane[t]
        for i in range(16):
            XA[32 * t + 2 * i] = Sa[i] + pa
            XB[32 * t + 2 * i] = Sb[i] + pb
            XA[32 * t + 2 * i + 1] = ea[i + 1]
            XB[32 * t + 2 * i + 1] = eb[i + 1]
        pa += tot[t][0]
        pb += tot[t][1]
    return XA[:n], XB[:n]


if __name__ == "__main__":
    rng = np.random.default_rng(0)
    for N in (512, 1024, 2048):
        n = N - 1
        A, B = rng.standard_normal(n), rng.standard_normal(n)
        XA, XB = model(A, B)
        ra, rb = dst_ref(A), dst_ref(B)
        print(N, np.abs(XA - ra).max(), np.abs(XB - rb).max())
