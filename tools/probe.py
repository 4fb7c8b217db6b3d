"""Bandwidth probes of the sweep's access pattern on config 4 (diagnostics)."""
import ctypes, os, subprocess, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import fjgen
so = os.path.join(ROOT, "tools", "libprobe.so")
if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(os.path.join(ROOT, "tools", "microbench.cu")):
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a",
                           "-O3", "-shared", "-Xcompiler", "-fPIC", "-o", so,
                           os.path.join(ROOT, "tools", "microbench.cu")])
L = ctypes.CDLL(so)
L.fj_probe.restype = ctypes.c_float
L.fj_probe.argtypes = [ctypes.c_int, ctypes.c_int64] + [ctypes.c_void_p] * 4 + [ctypes.c_int, ctypes.c_int]
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 4
p = fjgen.config(cid)
dev = torch.device("cuda:0")
col = torch.from_numpy(p.col).to(dev)
rows = torch.repeat_interleave(torch.arange(p.n, device=dev, dtype=torch.int32),
                               torch.from_numpy(np.diff(p.row_ptr)).to(dev))
key, idx = torch.sort(col, stable=True)
ocol = rows[idx].contiguous()            # out-CSR columns (u's targets), rows by u
w = None if p.w is None else torch.from_numpy(p.w).to(dev)[idx].contiguous()
z = torch.rand(p.n, dtype=torch.float64, device=dev)
zf = z.float()
m = p.m
for bps in (4, 8):
    for mode, name in [(0, "stream col+w"), (1, "gather z fp64"), (2, "w*z fp64 (spmv)"), (3, "w*z fp32")]:
        ms = L.fj_probe(mode, m, ocol.data_ptr(), 0 if w is None else w.data_ptr(), z.data_ptr(),
                        zf.data_ptr(), 5, bps)
        stream_bytes = m * (4 + (4 if w is not None else 0))
        print(f"{p.name} blocks/SM={bps} {name:18s} {ms:7.3f} ms  stream {stream_bytes/ms/1e6:7.0f} GB/s  "
              f"arcs/s {m/ms/1e6:7.1f} G", flush=True)

# relabelling experiments: the gathered target ids under several node orders
indeg = torch.bincount(ocol.long(), minlength=p.n)
outdeg = torch.from_numpy(np.bincount(p.col, minlength=p.n)).to(dev)
def cls(L):
    c = torch.zeros_like(L)
    for t in [0, 4, 8, 16, 32, 64, 256, 2048]:
        c += (L > t).long()
    return c
orders = {
    "layout(class desc,id)": torch.argsort(-cls(outdeg) * p.n * 4 + torch.arange(p.n, device=dev), stable=True),
    "in-degree desc": torch.argsort(-indeg, stable=True),
    "random": torch.randperm(p.n, device=dev),
}
for name, perm in orders.items():
    rank = torch.empty_like(perm)
    rank[perm] = torch.arange(p.n, device=dev)
    oc2 = rank[ocol.long()].int().contiguous()
    ms = L.fj_probe(2, m, oc2.data_ptr(), 0 if w is None else w.data_ptr(), z.data_ptr(),
                    zf.data_ptr(), 5, 4)
    print(f"{p.name} relabel {name:24s} spmv fp64 {ms:7.3f} ms  arcs/s {m/ms/1e6:7.1f} G", flush=True)

L.fj_probe_k.restype = ctypes.c_float
L.fj_probe_k.argtypes = [ctypes.c_int, ctypes.c_int64] + [ctypes.c_void_p] * 3 + [ctypes.c_int]
for K in (2, 4, 8):
    zk = torch.rand(p.n * K, dtype=torch.float64, device=dev)
    ms = L.fj_probe_k(K, m, ocol.data_ptr(), 0 if w is None else w.data_ptr(), zk.data_ptr(), 5)
    print(f"{p.name} K={K} spmv fp64 {ms:7.3f} ms  arcs/s {m/ms/1e6:7.1f} G  EU/s {K*m/ms/1e6:7.1f} G", flush=True)
