"""Time the oracle (paper's FIFO ImprovedBLISOR, fp64, one host core) at a given
ω on full configs — the CPU baseline SURVEY §8(d) asks for at the best ω.
usage: python tests/harness/oracle_sor_time.py CID:OMEGA [CID:OMEGA ...]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import fjgen  # noqa: E402
import oracle  # noqa: E402
for arg in sys.argv[1:]:
    cid, om = arg.split(":")
    p = fjgen.config(int(cid))
    t0 = time.time()
    r = oracle.solve(p.row_ptr, p.col, p.w, p.s, 1e-6, float(om))
    dt = time.time() - t0
    print(json.dumps({"config": int(cid), "name": p.name, "omega": float(om), "status": r.status,
                      "seconds": r.seconds, "wall_s": dt, "pushes": r.pushes,
                      "edge_updates": r.touched, "edge_updates_per_s": r.touched / r.seconds}),
          flush=True)
