"""Per-sweep cost of the COLORED schedule with and without work (diagnostics)."""
import os, sys, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, torch
sys.path.insert(0, "%s")
import fjgen, paper_2507_14864_b200 as fj
dev = torch.device("cuda:0")
p = fjgen.config(int(sys.argv[1]))
g = fj.Graph(p.n, torch.from_numpy(p.row_ptr).to(dev), torch.from_numpy(p.col).to(dev), None if p.w is None else torch.from_numpy(p.w).to(dev), directed=p.directed)
s = torch.from_numpy(p.s).to(dev); z = torch.empty(p.n, dtype=torch.float32, device=dev)
for r in range(2):
    st = fj.solve(g, s, z, 1e-6, 1.4, method="colored", max_sweeps=40, certify=False, raise_on_numeric=False)
print(f"colors {st.colors} {st.sweep_ms/st.sweeps:.3f} ms/sweep")
''' % ROOT
for cid in sys.argv[1:]:
    for skip in ["0", "3"]:
        env = dict(os.environ, FJ_DBG_SKIP=skip)
        out = subprocess.run([sys.executable, "-c", code, cid], env=env, capture_output=True, text=True)
        print("config", cid, "skip", skip, out.stdout.strip(), out.stderr[-200:] if out.returncode else "", flush=True)
