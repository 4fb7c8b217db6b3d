"""Relaxations and edge updates per sweep (diagnostics): cumulative counts of
solves capped at k sweeps (ASYNC, certificate off), differenced."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fjgen  # noqa: E402
import paper_2507_14864_b200 as fj  # noqa: E402
dev = torch.device("cuda:0")
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 4
step = int(sys.argv[2]) if len(sys.argv) > 2 else 10
p = fjgen.config(cid)
g = fj.Graph(p.n, torch.from_numpy(p.row_ptr).to(dev), torch.from_numpy(p.col).to(dev),
             None if p.w is None else torch.from_numpy(p.w).to(dev), directed=p.directed)
s = torch.from_numpy(p.s).to(dev)
z = torch.empty(p.n, dtype=torch.float32, device=dev)
full = fj.solve(g, s, z, 1e-6, 1.0, method="async")
print(f"C{cid}: {full.sweeps} sweeps, {full.relaxations} relaxations, EU {full.edge_updates}")
prev_r = prev_e = 0
for k in list(range(step, full.sweeps, step)) + [full.sweeps]:
    st = fj.solve(g, s, z, 1e-6, 1.0, method="async", max_sweeps=k, certify=False,
                  raise_on_numeric=False)
    r, e = st.relaxations, st.edge_updates
    print(f"sweeps {k - step + 1:4d}-{k:4d}: relaxed rows/sweep {(r - prev_r) / step / p.n:.4f} of n, "
          f"edge updates/sweep {(e - prev_e) / step / p.m:.4f} of m", flush=True)
    prev_r, prev_e = r, e
