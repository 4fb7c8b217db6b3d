"""One C4 (or CID) solve capped at MAXSW sweeps, for ncu captures of k_sweep / k_sweep_sh.
usage: python tools/shadow_prof.py CID SHADOW [MAXSW]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import fjgen  # noqa: E402
import paper_2507_14864_b200 as fj  # noqa: E402

cid, sh = int(sys.argv[1]), int(sys.argv[2])
maxsw = int(sys.argv[3]) if len(sys.argv) > 3 else 40
dev = torch.device("cuda:0")
T = lambda a: None if a is None else torch.from_numpy(a).to(dev)  # noqa: E731
p = fjgen.config(cid)
n = len(p.row_ptr) - 1
g = fj.Graph(n, T(p.row_ptr), T(p.col), T(p.w), directed=p.directed)
z = torch.empty(n, dtype=torch.float32, device=dev)
st = fj.solve(g, T(p.s), z, 1e-6, 1.0, raise_on_numeric=False, max_sweeps=maxsw, shadow=sh,
              certify=False)
print(st)
