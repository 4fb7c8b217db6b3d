"""COLORED schedule with the tail-color merge (reading R23): time-to-ε and
sweeps for several fj_opts.tail_frac settings against ASYNC ω = 1 (diagnostics).

usage: python tools/tail_exp.py CID [CID ...]
env: TAIL_FRACS (comma list, default 0,0.002,0.01,0.03)
"""
import os, sys, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, torch
sys.path.insert(0, "%s")
import fjgen, paper_2507_14864_b200 as fj
dev = torch.device("cuda:0")
cid = int(sys.argv[1]); eps = float(sys.argv[2]); omegas = [float(x) for x in sys.argv[3].split(",")]
frac = float(sys.argv[4])
p = fjgen.config(cid)
g = fj.Graph(p.n, torch.from_numpy(p.row_ptr).to(dev), torch.from_numpy(p.col).to(dev), None if p.w is None else torch.from_numpy(p.w).to(dev), directed=p.directed)
s = torch.from_numpy(p.s).to(dev); z = torch.empty(p.n, dtype=torch.float32, device=dev)
for om in omegas:
    meth = "async" if om == 1.0 else "colored"
    best = None
    for r in range(3):
        st = fj.solve(g, s, z, eps, om, method=meth, raise_on_numeric=False, tail_frac=frac)
        if best is None or st.solve_ms < best.solve_ms: best = st
    st = best
    print(f"  {meth:8s} omega {om:.2f} phases {st.colors:4d} sweeps {st.sweeps:5d} solve {st.solve_ms:8.2f} ms  {st.sweep_ms/max(st.sweeps,1):.3f} ms/sweep  cert {st.cert_ratio:.3f} status {st.status}", flush=True)
''' % ROOT
for cid in sys.argv[1:]:
    eps = "1e-6"
    for frac in os.environ.get("TAIL_FRACS", "0,0.002,0.01,0.03").split(","):
        oms = "1.0,1.2,1.4,1.6" if frac == "0" else "1.2,1.4,1.6"
        out = subprocess.run([sys.executable, "-c", code, cid, eps, oms, frac],
                             capture_output=True, text=True, timeout=900)
        print(f"config {cid} tail_frac={frac}", flush=True)
        print(out.stdout.rstrip(), out.stderr[-400:] if out.returncode else "", flush=True)
