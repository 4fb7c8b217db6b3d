"""Wall time of the pieces of one bench step on config 4 (diagnostics): graph create,
solve, measures, close, each synchronised.  usage: python tools/step_time.py"""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fjgen
import paper_2507_14864_b200 as fj
dev = torch.device("cuda:0")
p = fjgen.config(4)
rp, col = torch.from_numpy(p.row_ptr).to(dev), torch.from_numpy(p.col).to(dev)
w = torch.from_numpy(p.w).to(dev); s = torch.from_numpy(p.s).to(dev)
z = torch.empty(p.n, dtype=torch.float32, device=dev)
def T():
    torch.cuda.synchronize(); return time.time()
for r in range(6):
    t0 = T(); g = fj.Graph(p.n, rp, col, w, directed=p.directed)
    t1 = T(); st = fj.solve(g, s, z, 1e-6, 1.0)
    t2 = T(); m = fj.measures(g, z)
    t3 = T(); g.close()
    t4 = T()
    print(f"create {1e3*(t1-t0):.1f} solve {1e3*(t2-t1):.1f} (dev {st.solve_ms:.1f}, sweeps {st.sweeps}) measures {1e3*(t3-t2):.1f} close {1e3*(t4-t3):.1f} total {1e3*(t4-t0):.1f}", flush=True)
