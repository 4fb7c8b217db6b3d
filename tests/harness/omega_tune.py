"""Tuned ω of reading R10 for the full configs, computed by the ORACLE only:
the paper's heuristic — walk ω from 1.95 down to 1.00 in steps of
0.05, keep the ω with the fewest updates (FIFO pops of ImprovedBLISOR),
diverging points cost +∞, ties to the smaller ω (oracle.omega_sweep).

Writes one JSON line per config to profiles/r02_oracle_omega_tune.jsonl; the
`tuned` values in fjgen.CONFIG_SOLVE are copied from that file (a stored value
written by a committed script that calls only oracle/).

usage: python tests/harness/omega_tune.py CID [CID ...]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import fjgen  # noqa: E402
import oracle  # noqa: E402

out = os.path.join(ROOT, "profiles", "r02_oracle_omega_tune.jsonl")
for arg in sys.argv[1:]:
    cid = int(arg)
    p = fjgen.config(cid)
    eps = fjgen.CONFIG_SOLVE[cid]["eps"]
    t0 = time.time()
    best, table = oracle.omega_sweep(p.row_ptr, p.col, p.w, p.s, eps)
    rec = {"config": cid, "name": p.name, "n": p.n, "m": p.m, "eps": eps, "tuned_omega": best,
           "table": [[om, (None if c == float("inf") else int(c)), st] for om, c, st in table],
           "oracle_wall_s": round(time.time() - t0, 1),
           "rule": "argmin FIFO pops over 1.95:-0.05:1.00, +inf on divergence, ties to smaller omega "
                   "(P:488, reading R10); runs above the best count so far are pruned"}
    with open(out, "a") as f:
        f.write(json.dumps(rec) + "\n")
    print(json.dumps({k: rec[k] for k in ("config", "name", "tuned_omega", "oracle_wall_s")}),
          flush=True)
