import os, sys, subprocess, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, numpy as np, torch
sys.path.insert(0, "%s")
import fjgen, paper_2507_14864_b200 as fj
dev = torch.device("cuda:0")
p = fjgen.config(4)
g = fj.Graph(p.n, torch.from_numpy(p.row_ptr).to(dev), torch.from_numpy(p.col).to(dev), torch.from_numpy(p.w).to(dev), directed=True)
s = torch.from_numpy(p.s).to(dev); z = torch.empty(p.n, dtype=torch.float32, device=dev)
for r in range(2):
    st = fj.solve(g, s, z, 1e-6, 1.0, max_sweeps=60, certify=False, raise_on_numeric=False)
print(st.sweep_ms / st.sweeps)
''' % ROOT
for skip in ["0", "1", "2"]:
    env = dict(os.environ, FJ_DBG_SKIP=skip)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print("skip", skip, "ms/sweep", out.stdout.strip()[-30:], out.stderr[-300:] if out.returncode else "")
