"""Throughput of fj_solve_batch vs k single solves on a config (diagnostics)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fjgen, paper_2507_14864_b200 as fj
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 4
dev = torch.device("cuda:0")
p = fjgen.config(cid)
n = p.n
g = fj.Graph(n, torch.from_numpy(p.row_ptr).to(dev), torch.from_numpy(p.col).to(dev),
             None if p.w is None else torch.from_numpy(p.w).to(dev), directed=p.directed)
cols = [p.s, fjgen.exponential(n, 21), fjgen.pareto(n, 22), fjgen.uniform(n, 23),
        fjgen.uniform(n, 24), fjgen.exponential(n, 26), fjgen.pareto(n, 27), fjgen.beta25(n, 28)]
om = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
z = torch.empty(n, dtype=torch.float32, device=dev)
single_ms, single_eu = 0.0, 0
for r in range(4):
    s = torch.from_numpy(cols[r]).to(dev)
    fj.solve(g, s, z, 1e-6, om, raise_on_numeric=False)
    st = fj.solve(g, s, z, 1e-6, om, raise_on_numeric=False)
    single_ms += st.solve_ms
    single_eu += st.edge_updates
    print(f"{p.name} single r={r}: {st.solve_ms:.1f} ms sweeps {st.sweeps} EU {st.edge_updates:.3e}", flush=True)
for k in (2, 4, 8):
    S = torch.from_numpy(np.ascontiguousarray(np.stack(cols[:k], 1).astype(np.float32)).ravel()).to(dev)
    Z = torch.empty(n * k, dtype=torch.float32, device=dev)
    fj.solve_batch(g, S, Z, k, 1e-6, om, raise_on_numeric=False)
    st = fj.solve_batch(g, S, Z, k, 1e-6, om, raise_on_numeric=False)
    print(f"{p.name} w={om} batch k={k}: {st.solve_ms:.1f} ms sweeps {st.sweeps} "
          f"{st.sweep_ms / max(1, st.sweeps):.3f} ms/sweep EU {st.edge_updates:.3e} "
          f"EU/s {st.edge_updates/st.solve_ms/1e6:.1f} G cert {st.cert_ratio:.3f} status {st.status}",
          flush=True)
print(f"4 singles: {single_ms:.1f} ms EU/s {single_eu/single_ms/1e6:.1f} G")
