"""One batched solve (k opinion vectors) on a config, for ncu (diagnostics):
python tools/batch_one.py CID K [OMEGA]"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fjgen, paper_2507_14864_b200 as fj  # noqa: E402
cid, k = int(sys.argv[1]), int(sys.argv[2])
om = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
dev = torch.device("cuda:0")
p = fjgen.config(cid)
n = p.n
g = fj.Graph(n, torch.from_numpy(p.row_ptr).to(dev), torch.from_numpy(p.col).to(dev),
             None if p.w is None else torch.from_numpy(p.w).to(dev), directed=p.directed)
cols = [p.s, fjgen.exponential(n, 21), fjgen.pareto(n, 22), fjgen.uniform(n, 23),
        fjgen.uniform(n, 24), fjgen.exponential(n, 26), fjgen.pareto(n, 27), fjgen.beta25(n, 28)][:k]
S = torch.from_numpy(np.ascontiguousarray(np.stack(cols, 1).astype(np.float32)).ravel()).to(dev)
Z = torch.empty(n * k, dtype=torch.float32, device=dev)
st = fj.solve_batch(g, S, Z, k, 1e-6, om)
print(f"{p.name} k={k} w={om}: {st.solve_ms:.1f} ms sweeps {st.sweeps} "
      f"{st.sweep_ms / max(1, st.sweeps):.3f} ms/sweep EU/s {st.edge_updates / st.solve_ms / 1e6:.1f} G")
