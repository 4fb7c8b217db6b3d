"""A/B timing of libfj builds (FJ_LIB_PATH) on full configs (diagnostics).

usage: python tools/ab.py CIDS OMEGA LIB [LIB ...]   e.g. tools/ab.py 2,4 1.0 a.so b.so
Each (config, lib) runs in a fresh process; configs are cached under /tmp."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import os, sys, numpy as np, torch
sys.path.insert(0, %r)
import fjgen, paper_2507_14864_b200 as fj
cid, om, reps = int(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3])
path = f"/tmp/fjcache/c{cid}.npz"
if os.path.exists(path):
    d = np.load(path, allow_pickle=True)
    rp, col, w, s, directed = d["rp"], d["col"], (d["w"] if d["w"].size else None), d["s"], bool(d["directed"])
else:
    p = fjgen.config(cid)
    os.makedirs("/tmp/fjcache", exist_ok=True)
    np.savez(path, rp=p.row_ptr, col=p.col, w=(p.w if p.w is not None else np.zeros(0, np.float32)), s=p.s, directed=p.directed)
    rp, col, w, s, directed = p.row_ptr, p.col, p.w, p.s, p.directed
dev = torch.device("cuda:0")
T = lambda a: None if a is None else torch.from_numpy(a).to(dev)
g = fj.Graph(len(rp) - 1, T(rp), T(col), T(w), directed=directed)
st_ = T(s); z = torch.empty(len(rp) - 1, dtype=torch.float32, device=dev)
res = []
for r in range(reps):
    st = fj.solve(g, st_, z, 1e-6, om, raise_on_numeric=False, max_sweeps=4000)
    res.append((st.solve_ms, st.sweeps, st.sweep_ms / max(1, st.sweeps), st.cert_ratio, st.status))
res.sort()
t = res[len(res) // 2]
print(f"{t[0]:8.1f} ms  {t[1]:4d} sweeps  {t[2]:.4f} ms/sweep  cert {t[3]:.4f} status {t[4]}  all " + " ".join(f"{x[0]:.1f}/{x[1]}" for x in res))
''' % ROOT
cids = [int(c) for c in sys.argv[1].split(",")]
om = sys.argv[2]
libs = sys.argv[3:]
reps = os.environ.get("AB_REPS", "5")
for cid in cids:
    for lib in libs:
        env = dict(os.environ, FJ_LIB_PATH=os.path.abspath(lib))
        try:
            out = subprocess.run([sys.executable, "-c", code, str(cid), om, reps], env=env,
                                 capture_output=True, text=True, timeout=240)
        except subprocess.TimeoutExpired:
            print(f"C{cid} w={om} {lib:45s} TIMEOUT", flush=True)
            continue
        print(f"C{cid} w={om} {lib:45s}", out.stdout.strip(), out.stderr[-400:] if out.returncode else "",
              flush=True)
