"""Wall time of a first COLORED solve on C3 (coloring + layout + solve), diagnostics."""
import sys, time, torch
sys.path.insert(0, ".")
import fjgen, paper_2507_14864_b200 as fj
dev = torch.device("cuda:0")
p = fjgen.config(3)
rp, col = torch.from_numpy(p.row_ptr).to(dev), torch.from_numpy(p.col).to(dev)
s = torch.from_numpy(p.s).to(dev); z = torch.empty(p.n, dtype=torch.float32, device=dev)
for r in range(3):
    g = fj.Graph(p.n, rp, col, None, directed=False)
    torch.cuda.synchronize(); t0 = time.time()
    st = fj.solve(g, s, z, 1e-6, 1.6)
    torch.cuda.synchronize(); t1 = time.time()
    print(f"first colored solve incl. coloring: {1e3*(t1-t0):.1f} ms (solve {st.solve_ms:.1f} ms)", flush=True)
    g.close()
