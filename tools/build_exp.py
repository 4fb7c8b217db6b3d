"""Graph-build phase times (FJ_DEBUG marks) on a config (diagnostics)."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fjgen  # noqa: E402
import paper_2507_14864_b200 as fj  # noqa: E402
dev = torch.device("cuda:0")
p = fjgen.config(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
rp, col = torch.from_numpy(p.row_ptr).to(dev), torch.from_numpy(p.col).to(dev)
w = None if p.w is None else torch.from_numpy(p.w).to(dev)
for r in range(4):
    torch.cuda.synchronize()
    t0 = time.time()
    g = fj.Graph(p.n, rp, col, w, directed=p.directed)
    torch.cuda.synchronize()
    t1 = time.time()
    g.close()
    print(f"create {1e3 * (t1 - t0):.1f} ms", flush=True)
