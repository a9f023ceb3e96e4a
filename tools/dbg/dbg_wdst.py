import ctypes, sys
import numpy as np, torch, scipy.fft as sf
L = ctypes.CDLL(sys.argv[1])
for N in (256, 1024):
    wl = 16 if N == 256 else 64
    wt = np.zeros((2 * N + 64, 2))
    for l in range(N): wt[l] = (np.cos(np.pi * l / N), np.sin(np.pi * l / N))
    for k2 in range(N // wl):
        for l in range(wl):
            ang = 2 * np.pi * ((l * k2) % N) / N
            wt[N + k2 * wl + l] = (np.cos(ang), -np.sin(ang))
    for k in range(64): wt[2 * N + k] = (np.cos(2 * np.pi * k / 64), -np.sin(2 * np.pi * k / 64))
    npairs = 5
    x = np.random.default_rng(0).standard_normal((npairs, 2, N)); x[:, :, 0] = 0
    ti = torch.tensor(x, device="cuda"); to = torch.zeros_like(ti); tw = torch.tensor(wt, device="cuda")
    rc = L.dbg_dst(N, ctypes.c_void_p(ti.data_ptr()), ctypes.c_void_p(to.data_ptr()), ctypes.c_void_p(tw.data_ptr()), npairs)
    got = to.cpu().numpy()
    want = np.zeros_like(x); want[:, :, 1:] = sf.dst(x[:, :, 1:], type=1, axis=-1) / 2
    print(N, "rc", rc, "max err", np.abs(got - want).max(), "max |want|", np.abs(want).max())
    if np.abs(got - want).max() > 1e-9:
        e = np.abs(got - want)[0, 0]; print(" first bad idx", np.nonzero(e > 1e-9)[0][:10])
