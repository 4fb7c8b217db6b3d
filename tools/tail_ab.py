"""Active-set tail (k_sweep_tail) settings on full configs (diagnostics).

The kernel this drove (FJ_TAIL_EU / FJ_TAIL_INNER) was measured and removed
(DESIGN.md §8 tuning log, profiles/r01_sweep_profile.txt); kept as the record
of the experiment.  Against the current library every setting runs the same
code.
usage: python tools/tail_ab.py CID [CID ...]"""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, torch
sys.path.insert(0, "%s")
import fjgen, paper_2507_14864_b200 as fj
dev = torch.device("cuda:0")
p = fjgen.config(int(sys.argv[1]))
g = fj.Graph(p.n, torch.from_numpy(p.row_ptr).to(dev), torch.from_numpy(p.col).to(dev), None if p.w is None else torch.from_numpy(p.w).to(dev), directed=p.directed)
s = torch.from_numpy(p.s).to(dev); z = torch.empty(p.n, dtype=torch.float32, device=dev)
best = None
for r in range(3):
    st = fj.solve(g, s, z, 1e-6, 1.0, method="async")
    best = st if best is None or st.solve_ms < best.solve_ms else best
st = best
print(f"{st.solve_ms:7.1f} ms  full sweeps {st.sweeps:4d}  tail sweeps {st.phases - st.sweeps:4d}  EU {st.edge_updates/p.m:.0f}m  cert {st.cert_ratio:.3f}")
''' % ROOT
settings = [("off", {"FJ_TAIL_EU": "0"}), ("0.35/4", {}), ("0.2/4", {"FJ_TAIL_EU": "0.2"}),
            ("0.5/4", {"FJ_TAIL_EU": "0.5"}), ("0.35/2", {"FJ_TAIL_INNER": "2"}),
            ("0.35/8", {"FJ_TAIL_INNER": "8"})]
for cid in sys.argv[1:]:
    for name, env in settings:
        out = subprocess.run([sys.executable, "-c", code, cid], env=dict(os.environ, **env),
                             capture_output=True, text=True)
        print(f"C{cid} tail {name:7s}: {out.stdout.strip()} {out.stderr[-300:] if out.returncode else ''}",
              flush=True)
