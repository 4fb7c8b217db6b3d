"""Gather ceilings on config 4's pull CSR (diagnostics): scalar vs 128-bit
stream loads, and the H most popular columns served from shared memory.
usage: python tools/gather_bench.py [CID]"""
import ctypes, os, subprocess, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import fjgen  # noqa: E402
so = os.path.join(ROOT, "build", "libgb.so")
src = os.path.join(ROOT, "tools", "gather_bench.cu")
os.makedirs(os.path.dirname(so), exist_ok=True)
if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a",
                           "-O3", "-shared", "-Xcompiler", "-fPIC", "-o", so, src])
L = ctypes.CDLL(so)
L.gb_run.restype = ctypes.c_float
L.gb_run.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64] + [ctypes.c_void_p] * 3 + \
    [ctypes.c_int] * 5
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 4
p = fjgen.config(cid)
dev = torch.device("cuda:0")
col = torch.from_numpy(p.col).to(dev)
rows = torch.repeat_interleave(torch.arange(p.n, device=dev, dtype=torch.int32),
                               torch.from_numpy(np.diff(p.row_ptr)).to(dev))
key, idx = torch.sort(col, stable=True)
ocol = rows[idx].contiguous()            # pull-CSR columns, rows by u
w = None if p.w is None else torch.from_numpy(p.w).to(dev)[idx].contiguous()
m = (p.m // 4) * 4
cnt = torch.bincount(ocol.long(), minlength=p.n)
order = torch.argsort(cnt, descending=True, stable=True)
newid = torch.empty_like(order)
newid[order] = torch.arange(p.n, device=dev)
rcol = newid[ocol.long()].int().contiguous()          # columns relabelled by popularity
x = torch.rand(p.n, dtype=torch.float64, device=dev)
cum = torch.cumsum(cnt[order].double(), 0) / p.m
wp = 0 if w is None else w.data_ptr()


def run(vec, hot, c, H=0, thr=256, carve=-1, extra=0, reps=10):
    return L.gb_run(vec, hot, m, c.data_ptr(), wp, x.data_ptr(), H, thr, carve, reps, extra)


print(f"{p.name}: m={p.m}")
for name, c in (("raw ids", ocol), ("popularity ids", rcol)):
    for vec in (1, 4):
        print(f"  {name:15s} vec{vec} no hot 4x256       {run(vec, 0, c):.3f} ms", flush=True)
import math
for extra in (0, 32768):
    for H in (4096, 8192, 12288, 16384, 20480):
        need = H * 8 + extra
        cov = float(cum[H - 1])
        for carve in (math.ceil(100 * (need + 2048) / (228 * 1024)), 100):
            if carve > 100:
                continue
            ts = [run(4, 1, rcol, H, 1024, carve, extra) for _ in range(3)]
            print(f"  hot H={H:6d} ({cov:.3f} of arcs) extra={extra // 1024:3d}KB carve={carve:3d}%: "
                  + " ".join(f"{t:.3f}" for t in ts) + " ms", flush=True)
for carve in (0, 25, 50, 75, 100):
    ts = [run(4, 0, rcol, 0, 256, carve, 0) for _ in range(3)]
    print(f"  no hot 4x256 carve={carve:3d}%: " + " ".join(f"{t:.3f}" for t in ts) + " ms", flush=True)
    ts = [run(4, 0, rcol, 0, 1024, carve, 0) for _ in range(3)]
    print(f"  no hot 1x1024 carve={carve:3d}%: " + " ".join(f"{t:.3f}" for t in ts) + " ms", flush=True)

# ---- arc order inside 256-arc tiles: rows of ≤ 256 arcs, layout-like order
# (length class descending, id), each consecutive 256-arc chunk sorted by column
if os.environ.get("GB_TILESORT"):
    deg = torch.from_numpy(np.diff(p.row_ptr)).to(dev)          # pull row lengths: out-degree
    odeg = torch.bincount(col.long(), minlength=p.n)             # out-row length of u
    short = (odeg > 0) & (odeg <= 256)
    cls = torch.clamp(torch.ceil(torch.log2(odeg.clamp(min=1).double())).long(), 0, 8)
    key = (8 - cls) * p.n + torch.arange(p.n, device=dev)
    order = torch.argsort(torch.where(short, key, torch.full_like(key, 1 << 62)))
    order = order[: int(short.sum())]
    # arcs of the short rows in that row order
    ostart = torch.zeros(p.n + 1, dtype=torch.long, device=dev)
    ostart[1:] = torch.cumsum(odeg, 0)
    lens = odeg[order]
    starts = ostart[order]
    seg = torch.repeat_interleave(torch.arange(len(order), device=dev), lens)
    off = torch.arange(int(lens.sum()), device=dev) - torch.repeat_interleave(torch.cumsum(lens, 0) - lens, lens)
    arcs = starts[seg] + off
    tcol = rcol[arcs].contiguous()                               # popularity ids, tile order
    ms = (len(tcol) // 256) * 256
    tcol = tcol[:ms].contiguous()
    chunk = torch.arange(ms, device=dev) // 256
    sc = tcol[torch.argsort(chunk * p.n + tcol.long())].contiguous()
    mm = ms
    def run2(c, reps=10):
        return L.gb_run(1, 0, mm, c.data_ptr(), 0, x.data_ptr(), 0, 256, -1, reps, 0)
    print(f"  short-row arcs {ms}: tile order {run2(tcol):.3f} ms, tile-sorted {run2(sc):.3f} ms", flush=True)
