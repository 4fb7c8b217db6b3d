"""Repeat seeded fuzz cases (tests/test_gpu_fuzz.draw) with one method; report certificate failures (diagnostics)."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, oracle, fjgen
import paper_2507_14864_b200 as fj
from tests.test_gpu_fuzz import draw
seeds = [int(x) for x in sys.argv[1].split(",")]
reps = int(sys.argv[2])
meth = sys.argv[3] if len(sys.argv) > 3 else "push"
os.environ["FJ_PUSH_COMPACT"] = "1"
for seed in seeds:
    fam, rp, col, w, s, directed, eps, rng = draw(seed)
    n = len(rp) - 1
    div = int(rng.integers(1, 64))
    os.environ["FJ_PUSH_SPARSE_DIV"] = str(div)
    omega = 1.0 if rng.random() < 0.4 else float(rng.uniform(1.05, 1.9))
    s32 = np.asarray(s, np.float32)
    bad = 0
    for r in range(reps):
        g = fj.Graph(n, rp, col, w, directed=directed)
        z = np.empty(n, np.float32); zp = np.empty(n, np.float64)
        st = fj.solve(g, s32, z, eps, omega, method=meth, zprime_out=zp, raise_on_numeric=False)
        g.close()
        if st.status != 0:
            if not (omega > 1.0 and st.reason in (1, 2)): bad += 1; print("status", st)
            continue
        c = oracle.certificate(rp, col, w, s, zp, eps)[0]
        if not c <= 1.0:
            g2 = fj.Graph(n, rp, col, w, directed=directed)
            z2 = np.empty(n, np.float32); zp2 = np.empty(n, np.float64)
            fj.solve(g2, s32, z2, eps, 1.0, method="async", zprime_out=zp2)
            g2.close()
            d = np.abs(zp - zp2) / np.abs(zp2).max()
            bi = np.nonzero(d > 1e-4)[0]
            indeg = np.diff(rp)
            outdeg = np.bincount(col, minlength=n)
            print("  differing nodes", len(bi), bi[:10], "zp", zp[bi[:5]], "ref", zp2[bi[:5]],
                  "indeg", indeg[bi[:10]], "outdeg", outdeg[bi[:10]])
            bad += 1
            if bad < 3: print(seed, "cert", c, st)
    print(seed, fam, n, "omega", round(omega, 3), "div", div, "bad", bad, "of", reps, flush=True)
