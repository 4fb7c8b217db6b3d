import os, sys, numpy as np, torch
os.environ["FJ_DEBUG"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fjgen, paper_2507_14864_b200 as fj
dev = torch.device("cuda:0")
for cid in [int(x) for x in sys.argv[1].split(",")]:
    p = fjgen.config(cid)
    g = fj.Graph(p.n, torch.from_numpy(p.row_ptr).to(dev), torch.from_numpy(p.col).to(dev),
                 None if p.w is None else torch.from_numpy(p.w).to(dev), directed=p.directed)
    s = torch.from_numpy(p.s).to(dev); z = torch.empty(p.n, dtype=torch.float32, device=dev)
    print("config", cid, flush=True); sys.stderr.flush()
    st = fj.solve(g, s, z, 1e-6, 1.3, max_sweeps=3, raise_on_numeric=False)
    print("colors", st.colors, "ms/sweep", st.sweep_ms / max(1, st.sweeps), flush=True)
    g.close()
