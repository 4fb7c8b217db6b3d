#!/usr/bin/env python
"""Run the five BASELINE.json configs (or a subset) through the C-ABI on the
GPU, for a list of ω and methods, and record per-solve stats.  With --certify
the oracle's compensated fp64 certificate (oracle/, test infrastructure) is
applied to every GPU ẑ' and the oracle measures are computed on the GPU z.

    python tests/harness/run_configs.py --configs 1,2,3,4,5 --certify --out gpurun_out/configs.jsonl
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--shrink", type=int, default=0)
    ap.add_argument("--omegas", default=None, help="override: comma list")
    ap.add_argument("--methods", default="auto")
    ap.add_argument("--certify", action="store_true")
    ap.add_argument("--oracle", action="store_true", help="also run the full oracle FIFO (slow)")
    ap.add_argument("--repeat", type=int, default=2)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()

    import torch

    import fjgen
    import paper_2507_14864_b200 as fj
    dev = torch.device("cuda:0")
    out = open(a.out, "a") if a.out else None
    for cid in [int(c) for c in a.configs.split(",")]:
        t0 = time.time()
        prob = fjgen.config(cid, shrink=a.shrink)
        tgen = time.time() - t0
        omegas = [float(x) for x in a.omegas.split(",")] if a.omegas else \
            fjgen.CONFIG_SOLVE[cid]["omegas"]
        eps = fjgen.CONFIG_SOLVE[cid]["eps"]
        rp = torch.from_numpy(prob.row_ptr).to(dev)
        col = torch.from_numpy(prob.col).to(dev)
        w = None if prob.w is None else torch.from_numpy(prob.w).to(dev)
        s = torch.from_numpy(prob.s).to(dev)
        z = torch.empty(prob.n, dtype=torch.float32, device=dev)
        zp = torch.empty(prob.n, dtype=torch.float64, device=dev)
        torch.cuda.synchronize()
        t0 = time.time()
        g = fj.Graph(prob.n, rp, col, w, directed=prob.directed)
        torch.cuda.synchronize()
        tcreate = time.time() - t0
        info = g.info()
        refs = {}

        def oracle_ref(om):
            """The oracle's z at the same ε: at the same ω on undirected graphs,
            at ω = 1 on directed ones (reading R11)."""
            import oracle
            ro = 1.0 if prob.directed else om
            if ro not in refs:
                refs[ro] = oracle.solve(prob.row_ptr, prob.col, prob.w, prob.s, eps, ro)
            return ro, refs[ro]

        for method in a.methods.split(","):
            for om in omegas:
                ref = None
                if a.oracle:
                    ref_omega, ref = oracle_ref(om)
                best = None
                for r in range(a.repeat):
                    st = fj.solve(g, s, z, eps, om, method=method, zprime_out=zp,
                                  raise_on_numeric=False)
                    best = st if best is None or st.solve_ms < best.solve_ms else best
                st = best
                rec = {"config": cid, "name": prob.name, "n": prob.n, "m": prob.m,
                       "directed": prob.directed, "omega": om, "method": method, "eps": eps,
                       "status": st.status, "reason": st.reason, "sweeps": st.sweeps,
                       "phases": st.phases, "colors": st.colors,
                       "relaxations": st.relaxations, "edge_updates": st.edge_updates,
                       "solve_ms": st.solve_ms, "sweep_ms": st.sweep_ms, "cert_ms": st.cert_ms,
                       "gpu_cert_ratio": st.cert_ratio, "cert_rounds": st.cert_rounds,
                       "eu_per_s": st.edge_updates / (st.solve_ms / 1e3) if st.solve_ms else None,
                       "gen_s": tgen, "create_s": tcreate, "info": info}
                if st.status == 0:
                    m = fj.measures(g, z)
                    rec.update(P=m["P"], D=m["D"])
                if a.certify and st.status == 0:
                    import oracle
                    zph = zp.cpu().numpy()
                    zh = z.cpu().numpy()
                    t1 = time.time()
                    ratio, _ = oracle.certificate(prob.row_ptr, prob.col, prob.w, prob.s, zph, eps)
                    om_ = oracle.measures(prob.row_ptr, prob.col, prob.w, zh.astype(np.float64),
                                          directed=prob.directed)
                    rec.update(oracle_cert_ratio=ratio, oracle_cert_s=time.time() - t1,
                               P_rel=abs(m["P"] - om_["P"]) / abs(om_["P"]),
                               D_rel=abs(m["D"] - om_["D"]) / abs(om_["D"]))
                    if ref is not None:
                        rel = np.abs(zh - ref.z) / np.maximum(np.abs(ref.z), 1e-5)
                        omr = oracle.measures(prob.row_ptr, prob.col, prob.w, ref.z,
                                              directed=prob.directed)
                        rec.update(z_rel_vs_oracle=float(rel.max()),
                                   P_rel_vs_oracle=abs(m["P"] - omr["P"]) / abs(omr["P"]),
                                   D_rel_vs_oracle=abs(m["D"] - omr["D"]) / abs(omr["D"]),
                                   oracle_s=ref.seconds, oracle_touched=ref.touched,
                                   oracle_pushes=ref.pushes, oracle_omega=ref_omega,
                                   oracle_status=ref.status)
                line = json.dumps(rec)
                print(line, flush=True)
                if out:
                    out.write(line + "\n")
                    out.flush()
        g.close()
        del rp, col, w, s, z, zp
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
