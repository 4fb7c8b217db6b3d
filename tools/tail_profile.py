"""Relaxations per sweep in the tail of a solve, slices vs tiles (diagnostics):
solves capped at k sweeps (certificate off), cumulative counts differenced.
usage: python tools/tail_profile.py CID [SHADOW]"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fjgen  # noqa: E402
import paper_2507_14864_b200 as fj  # noqa: E402
dev = torch.device("cuda:0")
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 4
shadow = int(sys.argv[2]) if len(sys.argv) > 2 else 0
p = fjgen.config(cid)
g = fj.Graph(p.n, torch.from_numpy(p.row_ptr).to(dev), torch.from_numpy(p.col).to(dev),
             None if p.w is None else torch.from_numpy(p.w).to(dev), directed=p.directed)
s = torch.from_numpy(p.s).to(dev)
z = torch.empty(p.n, dtype=torch.float32, device=dev)
for sl in (0, 1):
    full = [fj.solve(g, s, z, 1e-6, 1.0, method="async", slices=sl, shadow=shadow).sweeps for _ in range(5)]
    print(f"C{cid} slices={sl} shadow={shadow}: sweeps of 5 solves {full}")
    prev = 0
    ks = list(range(20, 200, 20)) + list(range(200, max(full) + 1, 5))
    for k in ks:
        st = fj.solve(g, s, z, 1e-6, 1.0, method="async", max_sweeps=k, certify=False,
                      raise_on_numeric=False, slices=sl, shadow=shadow)
        if st.sweeps < k:
            print(f"  ended at {st.sweeps}")
            break
        print(f"  sweeps ..{k:4d}: relaxations {st.relaxations - prev:12d}  total {st.relaxations}", flush=True)
        prev = st.relaxations
