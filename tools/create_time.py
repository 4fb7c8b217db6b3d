"""fj_graph_create wall time (device-resident inputs, synchronised) on full
configs (diagnostics): python tools/create_time.py CID [CID ...]"""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fjgen  # noqa: E402
import paper_2507_14864_b200 as fj  # noqa: E402
dev = torch.device("cuda:0")
for cid in [int(c) for c in sys.argv[1:]]:
    p = fjgen.config(cid)
    rp, col = torch.from_numpy(p.row_ptr).to(dev), torch.from_numpy(p.col).to(dev)
    w = None if p.w is None else torch.from_numpy(p.w).to(dev)
    ts = []
    for r in range(5):
        torch.cuda.synchronize()
        t0 = time.time()
        g = fj.Graph(p.n, rp, col, w, directed=p.directed)
        torch.cuda.synchronize()
        ts.append(1e3 * (time.time() - t0))
        g.close()
    ts.sort()
    print(f"C{cid} {p.name}: create {ts[len(ts) // 2]:.1f} ms (min {ts[0]:.1f})", flush=True)
