import sys, json, numpy as np, torch
sys.path.insert(0,'/root/repo')
import fjgen, paper_2507_14864_b200 as fj
dev=torch.device('cuda:0')
for shrink in [1,0]:
    p=fjgen.config(3, shrink=shrink)
    g=fj.Graph(p.n, torch.from_numpy(p.row_ptr).to(dev), torch.from_numpy(p.col).to(dev), None, directed=False)
    s=torch.from_numpy(p.s).to(dev); z=torch.empty(p.n,dtype=torch.float32,device=dev)
    for om in [1.4,1.6]:
        for ms in [300,1000,3000]:
            st=fj.solve(g,s,z,1e-6,om,max_sweeps=ms,raise_on_numeric=False)
            print(shrink, om, ms, st.status, st.reason, st.sweeps, st.relaxations, st.cert_ratio, round(st.solve_ms,1), flush=True)
    g.close()
