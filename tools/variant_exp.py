"""Time the C4 sweep with several diagnostic builds of libfj (FJ_LIB_PATH)."""
import os, sys, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, numpy as np, torch
sys.path.insert(0, "%s")
import fjgen, paper_2507_14864_b200 as fj
dev = torch.device("cuda:0")
p = fjgen.config(int(sys.argv[1]))
g = fj.Graph(p.n, torch.from_numpy(p.row_ptr).to(dev), torch.from_numpy(p.col).to(dev), None if p.w is None else torch.from_numpy(p.w).to(dev), directed=p.directed)
s = torch.from_numpy(p.s).to(dev); z = torch.empty(p.n, dtype=torch.float32, device=dev)
for r in range(2):
    st = fj.solve(g, s, z, 1e-6, 1.0, raise_on_numeric=False)
print(f"{st.solve_ms:.1f} ms, {st.sweeps} sweeps, {st.sweep_ms/st.sweeps:.3f} ms/sweep, cert {st.cert_ratio:.4f}")
''' % ROOT
libs = sys.argv[2:] if len(sys.argv) > 2 else ["paper_2507_14864_b200/libfj.so"]
for lib in libs:
    env = dict(os.environ, FJ_LIB_PATH=os.path.join(ROOT, lib))
    out = subprocess.run([sys.executable, "-c", code, sys.argv[1]], env=env, capture_output=True, text=True)
    print(f"{lib:40s}", out.stdout.strip(), out.stderr[-300:] if out.returncode else "", flush=True)
