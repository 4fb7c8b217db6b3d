"""TMA gather4 vs LDG gathers (diagnostics; tools/tma_gather.cu).
usage: python tools/tma_gather.py [--c4]"""
import ctypes, os, subprocess, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
so = os.path.join(ROOT, "build", "libtg.so")
src = os.path.join(ROOT, "tools", "tma_gather.cu")
os.makedirs(os.path.dirname(so), exist_ok=True)
if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a",
                           "-O3", "-shared", "-Xcompiler", "-fPIC", "-o", so, src])
L = ctypes.CDLL(so)
L.tg_run.restype = ctypes.c_float
L.tg_run.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                     ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int,
                     ctypes.c_int]
L.tg_fill.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64]
dev = torch.device("cuda:0")

sets = []
n = 1 << 24
m = 263431078 // 128 * 128
col = torch.empty(m + 128, dtype=torch.int32, device=dev)
L.tg_fill(m, col.data_ptr(), n, 7)
sets.append(("uniform n=2^24", n, m, col))
if "--c4" in sys.argv:
    import fjgen
    p = fjgen.config(4)
    c = torch.from_numpy(p.col).to(dev)
    rows = torch.repeat_interleave(torch.arange(p.n, device=dev, dtype=torch.int32),
                                   torch.from_numpy(np.diff(p.row_ptr)).to(dev))
    _, idx = torch.sort(c, stable=True)
    ocol = torch.empty(p.m + 128, dtype=torch.int32, device=dev)
    ocol[: p.m] = rows[idx]
    ocol[p.m:] = 0
    sets.append(("C4 pull stream", p.n, p.m // 128 * 128, ocol))
    del c, rows, idx

for name, n, m, col in sets:
    x = torch.rand(n + 4, dtype=torch.float64, device=dev)
    def run(mode, cps=4, thr=256, tw=0, frac=0.0, promo=0, reps=7):
        return L.tg_run(mode, m, col.data_ptr(), x.data_ptr(), n, cps, thr, tw, frac, promo, reps)
    print(f"{name}: m={m} n={n}", flush=True)
    t0 = run(0)
    print(f"  LDG 4x256                        {t0:.3f} ms  ({m / t0 / 1e6:.1f} G gathers/s)", flush=True)
    for cps, thr in ((1, 256), (1, 128), (2, 128), (3, 128)):
        for promo in (0, 2):
            t = run(1, cps, thr, promo=promo)
            print(f"  TMA {cps}x{thr} promo={promo}               {t:.3f} ms  ({m / t / 1e6:.1f} G/s)", flush=True)
    for tw in (1, 2):
        for frac in (0.2, 0.3, 0.4, 0.5):
            t = run(2, 4, 256, tw, frac)
            print(f"  hybrid 4x256 tma_warps={tw} frac={frac:.1f}  {t:.3f} ms  ({m / t / 1e6:.1f} G/s)",
                  flush=True)
    del x
