"""Per-sweep time with warp units (1), warp tiles (2) or both (3) skipped (FJ_DBG_SKIP), diagnostics.
usage: python tools/skip_all.py CID [CID ...]"""
import os, sys, subprocess
ROOT = "/root/repo" if os.path.exists("/root/repo") else "."
code = r'''
import sys, torch
sys.path.insert(0, ".")
import fjgen, paper_2507_14864_b200 as fj
dev = torch.device("cuda:0")
p = fjgen.config(int(sys.argv[1]))
g = fj.Graph(p.n, torch.from_numpy(p.row_ptr).to(dev), torch.from_numpy(p.col).to(dev), None if p.w is None else torch.from_numpy(p.w).to(dev), directed=p.directed)
s = torch.from_numpy(p.s).to(dev); z = torch.empty(p.n, dtype=torch.float32, device=dev)
for r in range(2):
    st = fj.solve(g, s, z, 1e-6, 1.0, max_sweeps=100, certify=False, raise_on_numeric=False)
print(f"{st.sweep_ms / st.sweeps:.4f}")
'''
for cid in sys.argv[1:]:
    for skip in ["0", "1", "2", "3"]:
        out = subprocess.run([sys.executable, "-c", code, cid], env=dict(os.environ, FJ_DBG_SKIP=skip), capture_output=True, text=True)
        print(f"C{cid} skip {skip}: ms/sweep {out.stdout.strip()} {out.stderr[-200:] if out.returncode else ''}", flush=True)
