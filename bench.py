#!/usr/bin/env python
"""Benchmark of the FJ hot path on B200 (BASELINE.json metric: edge-updates/s
and time-to-ε on R-MAT-24, achieved HBM GB/s vs peak).

One STEP = one pass of every §8(a) row over the config-4 workload (directed
weighted R-MAT-24, s ~ Beta(2,5), ε = 1e-6) with inputs resident in HBM:
fj_graph_create (a1) → fj_solve_ex (a2–a6) → fj_measures (a7) → destroy.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--omega 1.0] [--impl reference]

N > 1 (torchrun): independent replicas, one per GPU (the default; one C4 solve
fits one B200), or with --mode sharded ONE problem split over the
ranks by fj_shard_* over NCCL (row f4, strong scaling).  Rank 0 prints one
JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "edge-updates/s (time-to-eps on R-MAT-24; achieved HBM GB/s vs peak)"
UNIT = "edge-updates/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--shrink", type=int, default=0, help="smaller size of the same recipe (dev only)")
    ap.add_argument("--omega", type=float, default=1.0)
    ap.add_argument("--method", default="auto")
    ap.add_argument("--eps", type=float, default=1e-6)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sweep", action="store_true",
                    help="skip the per-omega time-to-eps table of the config (untimed)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--mode", default="replicas", choices=["replicas", "sharded"],
                    help="N>1: independent replicas (default) or ONE problem sharded over the "
                         "ranks with fj_shard_* over NCCL (row f4; strong scaling)")
    ap.add_argument("--out", default=None, help="also write the JSON line here")
    return ap.parse_args()


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return None


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return None
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > i + 2 and r[i + 2].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        # torchrun pins OMP_NUM_THREADS=1; the input generator (OpenMP, runs
        # before the timed region) gets an even share of the host cores instead
        os.environ["OMP_NUM_THREADS"] = str(max(1, (os.cpu_count() or 1) // world))
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl" if args.impl == "ours" else "gloo")
    return world, rank, local


def max_over_ranks(value: float, world: int, device=None) -> float:
    """Max of `value` over all ranks (device time is the max over ranks)."""
    if world <= 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64,
                     device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, world: int, device=None) -> float:
    """Sum of `value` over all ranks (work units every rank processed)."""
    if world <= 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64,
                     device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def config_dict(prob, args, extra=None):
    d = {"workload": f"config{args.config}:{prob.name}", "n": prob.n, "m": prob.m,
         "eps": args.eps, "omega": args.omega, "directed": prob.directed,
         "weighted": prob.w is not None, "opinions": prob.meta.get("kind"),
         "seed": prob.meta.get("seed"),
         "l2": "inputs larger than L2 (CSR > 126 MB), no flush needed",
         "parallelism": "replicas" if args.gpus > 1 else "single-gpu"}
    if extra:
        d.update(extra)
    return d


# ------------------------------------------------------------ reference arm
#: the oracle's full C4 time-to-ε (ImprovedBLI, FIFO, fp64, one core) from the
#: round-2 full-size parity run (profiles/r02_full_parity.md)
ORACLE_FULL_C4 = {"time_to_eps_s": 843.8, "edge_updates_per_s": 6.45e7,
                  "source": "profiles/r02_full_parity.md (config 4, omega 1.0, one host core "
                            "of the GPU box, round 2)"}
#: scale reduction of the CPU sample: config 4's recipe at R-MAT scale 20
#: (shrink 2), a complete solve to ε in 23–46 s on one core depending on the
#: host.  A smaller graph caches better, so its edge-update rate is an upper
#: bound of the full-size rate (GPU box, round 2: 1.15e8 at scale 20 against
#: 6.45e7 for the full C4 solve): the sample flatters the CPU, and the
#: full-size time-to-ε is quoted beside it
SAMPLE_SHRINK = 2


def oracle_full_solve(args, shrink):
    """One complete ImprovedBLI solve (Alg. 2+1, FIFO, fp64) of the bench
    config's recipe at a reduced scale: the whole algorithm, start to ε."""
    import fjgen
    import oracle
    p = fjgen.config(args.config, shrink=shrink)
    r = oracle.solve(p.row_ptr, p.col, p.w, p.s, args.eps, 1.0)
    return p, r


def run_reference(args, prob, world, rank):
    """The oracle (fp64 FIFO ImprovedBLI, single thread) timed on the host
    cores.  Each timed step is a COMPLETE solve to ε of the config-4 recipe at
    R-MAT scale 20 (representative of the full solve: all of its phases, the
    same edge-update rate as the full-size run); warm-up steps use scale 16."""
    if rank != 0:
        return None  # rank 0 alone runs the CPU reference
    times, eus = [], []
    for i in range(args.warmup + args.steps):
        p, r = oracle_full_solve(args, max(args.shrink, SAMPLE_SHRINK if i >= args.warmup else 4))
        assert r.status == 0
        if i >= args.warmup:
            times.append(r.seconds)
            eus.append(r.touched)
    v = sum(eus) / sum(times)
    sample = (f"complete ImprovedBLI solves (Alg. 2+1, FIFO, fp64, to eps={args.eps}) of the "
              f"config-{args.config} recipe at reduced size ({p.name}, n={p.n}, m={p.m}), "
              f"{statistics.mean(times):.1f} s each")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * statistics.mean(times), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (fjgen seeded R-MAT, Beta(2,5) opinions)",
            "config": config_dict(prob, args, {"omega": 1.0}),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": sample, "full_size_time_to_eps": ORACLE_FULL_C4},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    return line


def cpu_baseline(prob, args):
    p, r = oracle_full_solve(args, max(args.shrink, SAMPLE_SHRINK))
    return {"value": r.touched / r.seconds, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"one complete ImprovedBLI solve (Alg. 2+1, FIFO, fp64, to eps={args.eps}) "
                      f"of the config-{args.config} recipe at reduced size ({p.name}, n={p.n}, "
                      f"m={p.m}): {r.pushes} pops, {r.touched} edge updates, {r.seconds:.1f} s",
            "full_size_time_to_eps": ORACLE_FULL_C4}


# ----------------------------------------------------------------- our arm
def algorithmic_bytes(st, weighted: bool, empty_rows: int):
    """SURVEY §8(d)'s algorithmic bytes of the sweep kernel:
    per edge-update (an arc of a relaxed row, P:488's "updates" × their arcs)
    col 4 + gathered ẑ_j 4 (+ w 4 weighted) = 8 / 12 B; per relaxation the
    row's state: row_ptr 8 + s 4 + ẑ_i read 8 + ẑ_i write 8 (+ 1+d 8
    weighted) = 28 / 36 B.  Rows solved exactly at init (no arcs) move nothing."""
    per_eu = 12 if weighted else 8
    per_relax = 36 if weighted else 28
    swept_relax = st.relaxations - empty_rows
    return st.edge_updates * per_eu + swept_relax * per_relax


def streamed_bytes(st, weighted: bool, empty_rows: int):
    """What the sweep kernels actually stream per solve: every arc of every
    sweep (col 4 + w 4 weighted), one gathered ẑ_j per arc counted at its useful
    size (4 B from the shadow in shadow sweeps, 8 B fp64 in the others), every
    evaluated row's state (s 4 + ẑ_i 8 + 1+d 8 weighted) and one 8-byte write
    (+ 4 for the shadow) per relaxation."""
    shf = st.shadow_sweeps / max(1, st.sweeps)
    per_arc = (8 if weighted else 4) + 4 * shf + 8 * (1 - shf)
    per_row = 20 if weighted else 12
    return (st.arcs_read * per_arc + st.rows_read * per_row
            + (8 + 4 * shf) * (st.relaxations - empty_rows))


def lib_fingerprint():
    """sha256 (16 hex) of the SASS of the loaded libfj.so (cuobjdump, source paths
    dropped): ties an ncu capture to its machine code.  The .so bytes themselves
    differ between checkouts (-lineinfo records the build path)."""
    import hashlib
    import paper_2507_14864_b200 as fj
    return sass_fingerprint(fj.LIB_PATH)


def sass_fingerprint(path):
    import hashlib
    try:
        out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True,
                             timeout=120).stdout
    except Exception:
        return None
    keep = [ln for ln in out.splitlines() if ln and "identifier" not in ln and
            not ln.startswith("Fatbin")]
    return hashlib.sha256("\n".join(keep).encode()).hexdigest()[:16] if keep else None


def run_ours(args, prob, world, rank, local):
    import torch

    import paper_2507_14864_b200 as fj
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream(dev)
    rp = torch.from_numpy(prob.row_ptr).to(dev)
    col = torch.from_numpy(prob.col).to(dev)
    w = None if prob.w is None else torch.from_numpy(prob.w).to(dev)
    s = torch.from_numpy(prob.s).to(dev)
    z = torch.empty(prob.n, dtype=torch.float32, device=dev)
    torch.cuda.synchronize()

    def step():
        g = fj.Graph(prob.n, rp, col, w, directed=prob.directed)
        st = fj.solve(g, s, z, args.eps, args.omega, method=args.method)
        m = fj.measures(g, z)
        g.close()
        return st, m

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    launches0 = fj.lib().fj_kernel_launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stats = []
    with Clocks(local) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            stats.append(step())
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = fj.lib().fj_kernel_launches() - launches0
    ms = max_over_ranks(ev0.elapsed_time(ev1), world, dev)
    eu_rank = sum(st.edge_updates for st, _ in stats)
    value = sum_over_ranks(eu_rank, world, dev) / (ms / 1e3)
    st0, m0 = stats[-1]
    solve_ms = statistics.median(st.solve_ms for st, _ in stats)
    sweep_ms = statistics.median(st.sweep_ms for st, _ in stats)

    # roofline of the dominant kernel (k_sweep), CUDA events on the graph stream
    pk = peaks()
    peak = pk["hbm_gbs"] if pk else 6650.0
    g = fj.Graph(prob.n, rp, col, w, directed=prob.directed)
    empty_rows = g.info()["empty_rows"]
    g.close()
    ab = algorithmic_bytes(st0, prob.w is not None, empty_rows)
    sb = streamed_bytes(st0, prob.w is not None, empty_rows)
    achieved = ab / (st0.sweep_ms / 1e3) / 1e9
    traffic = None
    traffic_src = None
    prof = os.path.join(ROOT, "profiles", "ncu_sweep_traffic.json")
    if os.path.exists(prof):
        try:
            # ncu's dram bytes per sweep of its captured launch × this launch's
            # sweeps — only if the capture was taken on this very build
            tj = json.load(open(prof))
            fp = lib_fingerprint()
            if fp and tj.get("sass_sha16") == fp and args.config == tj.get("config", 4):
                # (the capture is the first sweep launch: the shadow sweeps when the solve
                # uses them, ≈ 95 % of all sweeps; the fp64 tail is counted at that rate)
                traffic = tj["dram_bytes_per_sweep"] * st0.sweeps
                traffic_src = tj.get("source")
        except Exception:
            traffic = None

    # practical roofline: the sweep's memory pattern without its arithmetic
    # (fj_gather_probe: stream every arc, gather one fp64 per arc), timed live
    g = fj.Graph(prob.n, rp, col, w, directed=prob.directed)
    probe_ms = fj.gather_probe(g, 10)
    g.close()
    sweep_per = st0.sweep_ms / max(st0.sweeps, 1)
    ceiling = {"probe_ms_per_pass": probe_ms, "sweep_ms_per_sweep": sweep_per,
               "frac": probe_ms / sweep_per,
               "note": "fj_gather_probe over the same layout: every arc's col+w streamed and "
                       "one fp64 gathered per arc; frac = probe / sweep time (1 = at the gather "
                       "ceiling; above 1 when the sweeps gather from the 4-byte shadow, which the "
                       "8-byte probe does not)"}

    # f2: the same graph with k = 4 opinion vectors in one batched solve
    batched = None
    if not args.no_sweep:
        # f2: the same graph with k = 4 and k = 8 opinion vectors in one solve
        import fjgen
        g = fj.Graph(prob.n, rp, col, w, directed=prob.directed)
        cols = [prob.s, fjgen.exponential(prob.n, 21), fjgen.pareto(prob.n, 22),
                fjgen.uniform(prob.n, 23), fjgen.uniform(prob.n, 24),
                fjgen.exponential(prob.n, 26), fjgen.pareto(prob.n, 27), fjgen.beta25(prob.n, 28)]
        batched = []
        for k in (4, 8):
            S = torch.from_numpy(np.ascontiguousarray(np.stack(cols[:k], 1).astype(np.float32))
                                 .ravel()).to(dev)
            Z = torch.empty(prob.n * k, dtype=torch.float32, device=dev)
            fj.solve_batch(g, S, Z, k, args.eps, args.omega)
            stb = fj.solve_batch(g, S, Z, k, args.eps, args.omega)
            batched.append({"k": k, "opinions": "Beta(2,5), Exp, Pareto, U[0,1] (+ U, Exp, Pareto, "
                                                "Beta(2,5) of other seeds at k = 8)",
                            "time_to_eps_s": stb.solve_ms / 1e3, "sweeps": stb.sweeps,
                            "ms_per_sweep": stb.sweep_ms / max(1, stb.sweeps),
                            "edge_updates": stb.edge_updates,
                            "edge_updates_per_s": stb.edge_updates / (stb.solve_ms / 1e3),
                            "cert_ratio": stb.cert_ratio})
            del S, Z
        g.close()

    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, prob, fj, torch, dev, stream, world)
    omega_table = None
    if not args.no_sweep:
        omega_table = run_omega_table(args, prob, fj, torch, rp, col, w, s, z)

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (fjgen seeded R-MAT-24 weights U(0,1], Beta(2,5) opinions)",
            "config": config_dict(prob, args, {"method": args.method}),
            "time_to_eps_s": solve_ms / 1e3,
            "sweep_kernel_ms": sweep_ms,
            "step_breakdown": {"solve_ms": solve_ms, "sweeps": st0.sweeps,
                               "shadow_sweeps": st0.shadow_sweeps, "shadow_ms": st0.shadow_ms,
                               "frontier_rounds": st0.frontier_rounds,
                               "frontier_pushes": st0.frontier_pushes,
                               "frontier_ms": st0.frontier_ms,
                               "relaxations": st0.relaxations, "edge_updates": st0.edge_updates,
                               "cert_ratio": st0.cert_ratio, "colors": st0.colors,
                               "polarization": m0["P"], "disagreement": m0["D"]},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs" if pk else "fallback 6.65 TB/s",
                         "kernel": "k_sweep_sh (persistent sweeps: warp units + row slices, shadow "
                                   "gathers) + the frontier phase (k_pass<CERT> residuals, k_front) "
                                   "+ any fp64 k_sweep tail; every launch of the sweep stage timed "
                                   "together"
                         if st0.shadow_sweeps else "k_sweep (persistent sweeps: warp units + row "
                                                   "slices) + the frontier phase",
                         "algorithmic_bytes_per_launch": ab,
                         "bytes_model": "SURVEY 8(d): 12 B per edge-update (col, w, gathered z_j) "
                                        "+ 36 B per relaxation (row_ptr, s, z_i r/w, 1+d)",
                         "streamed_bytes_per_launch": sb,
                         "streamed_gbs": sb / (st0.sweep_ms / 1e3) / 1e9,
                         "traffic_source": traffic_src, "sass_sha16": lib_fingerprint()},
            "gather_ceiling": ceiling,
            "batched": batched,
            "omega_sweep": omega_table,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "e2e": e2e}
    return line


def run_sharded(args, prob, world, rank, local):
    """--mode sharded: one config-4 problem split over the ranks (row f4).
    Each rank transposes the generated in-CSR to the out-CSR on its GPU
    (torch, plumbing only), keeps its arc-balanced slice resident in HBM, and a
    step is fj_shard_create + connect + solve + measures + destroy over NCCL."""
    import torch

    import paper_2507_14864_b200 as fj
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream(dev)
    n = prob.n
    rp = torch.from_numpy(prob.row_ptr).to(dev)
    colt = torch.from_numpy(prob.col).to(dev).long()
    order = torch.sort(colt, stable=True).indices
    v = torch.repeat_interleave(torch.arange(n, device=dev), torch.diff(rp))
    ocol = v[order].int()
    ow = None if prob.w is None else torch.from_numpy(prob.w).to(dev)[order]
    orp = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    orp[1:] = torch.cumsum(torch.bincount(colt, minlength=n), 0)
    del colt, order, v, rp
    begin = fj.shard_plan(orp.cpu().numpy(), world)
    a, b = begin[rank], begin[rank + 1]
    k0, k1 = int(orp[a]), int(orp[b])
    srp = (orp[a:b + 1] - k0).contiguous()
    scol = ocol[k0:k1].contiguous()
    sw = None if ow is None else ow[k0:k1].contiguous()
    del ocol, ow, orp
    s = torch.from_numpy(prob.s[a:b].copy()).to(dev)
    z = torch.empty(b - a, dtype=torch.float32, device=dev)
    if world > 1:
        import torch.distributed as dist
        box = [fj.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        uid = box[0]
    else:
        uid = fj.comm_unique_id()
    comm = fj.Comm.nccl(uid, rank, world)
    torch.cuda.synchronize()

    def step():
        sh = fj.Shard(comm, rank, n, begin, srp, scol, sw, directed=prob.directed)
        fj.shard_connect([sh])
        st = fj.shard_solve([sh], [s], [z], args.eps, args.omega)
        m = fj.shard_measures([sh], [z])
        sh.close()
        return st, m

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    launches0 = fj.lib().fj_kernel_launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stats = []
    with Clocks(local) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            stats.append(step())
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = fj.lib().fj_kernel_launches() - launches0
    ms = max_over_ranks(ev0.elapsed_time(ev1), world, dev)
    eu = sum(st.edge_updates for st, _ in stats)  # already summed over the ranks
    st0, m0 = stats[-1]
    pk = peaks()
    peak = pk["hbm_gbs"] if pk else 6650.0
    # §8(d) bytes of this rank's share (edge updates and relaxations are
    # all-reduced totals; rows without arcs are ignored here)
    ab = algorithmic_bytes(st0, prob.w is not None, 0) / world
    achieved = ab / (st0.sweep_ms / 1e3) / 1e9
    comm.close()
    return {"metric": METRIC, "value": eu / (ms / 1e3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (fjgen seeded R-MAT-24 weights U(0,1], Beta(2,5) opinions)",
            "config": config_dict(prob, args, {"method": "sharded-async",
                                               "parallelism": f"shard{world}",
                                               "begin": [int(x) for x in begin]}),
            "time_to_eps_s": statistics.median(st.solve_ms for st, _ in stats) / 1e3,
            "sweep_kernel_ms": statistics.median(st.sweep_ms for st, _ in stats),
            "step_breakdown": {"sweeps": st0.sweeps, "relaxations": st0.relaxations,
                               "edge_updates": st0.edge_updates, "cert_ratio": st0.cert_ratio,
                               "polarization": m0["P"], "disagreement": m0["D"]},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None,
                         "kernel": "k_sweep + per-sweep exchange (rank 0's shard)",
                         "algorithmic_bytes_per_launch": ab},
            "gpu_launches": int(launches), "clocks": clk.summary(),
            "e2e": None, "e2e_note": "not measured in --mode sharded"}


def run_omega_table(args, prob, fj, torch, rp, col, w, s, z):
    """Time-to-ε per ω of the config's list (BASELINE config 4: SOR ω swept
    over {1.0, 1.2, 1.4, 1.6, 1.8}); outside the timed steps, graph built once,
    median of 3 solves, diverging ω reported as such."""
    import fjgen
    omegas = fjgen.CONFIG_SOLVE.get(args.config, {}).get("omegas", [args.omega])
    g = fj.Graph(prob.n, rp, col, w, directed=prob.directed)
    rows = []
    for om in omegas:
        runs = [fj.solve(g, s, z, args.eps, om, method=args.method, raise_on_numeric=False)
                for _ in range(3)]
        st = sorted(runs, key=lambda r: r.solve_ms)[1]
        rows.append({"omega": om, "status": "ok" if st.status == 0 else "diverged/numeric",
                     "time_to_eps_s": st.solve_ms / 1e3 if st.status == 0 else None,
                     "sweeps": st.sweeps, "edge_updates": st.edge_updates,
                     "edge_updates_per_s": st.edge_updates / (st.solve_ms / 1e3),
                     "cert_ratio": st.cert_ratio})
    g.close()
    torch.cuda.synchronize()
    return rows


def run_e2e(args, prob, fj, torch, dev, stream, world):
    """Same metric through the C-ABI with HOST buffers: the H2D copy of the
    step's inputs (pinned) and the D2H read of z and the measures are inside
    the timed region (the library stages host pointers itself)."""
    rp = torch.from_numpy(prob.row_ptr).pin_memory()
    col = torch.from_numpy(prob.col).pin_memory()
    w = None if prob.w is None else torch.from_numpy(prob.w).pin_memory()
    s = torch.from_numpy(prob.s).pin_memory()
    z = torch.empty(prob.n, dtype=torch.float32).pin_memory()
    sptr = ctypes_stream(stream)

    def step():
        g = fj.Graph(prob.n, rp, col, w, directed=prob.directed, stream=sptr)
        st = fj.solve(g, s, z, args.eps, args.omega, method=args.method)
        fj.measures(g, z)
        g.close()
        return st

    step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eu = 0
    k = max(1, min(args.steps, 3))
    for _ in range(k):
        eu += step().edge_updates
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    h2d = prob.row_ptr.nbytes + prob.col.nbytes + (0 if prob.w is None else prob.w.nbytes) + \
        prob.s.nbytes
    d2h = 4 * prob.n + 32
    dt = max_over_ranks(dt, world, dev)
    return {"value": sum_over_ranks(eu, world, dev) / dt, "unit": UNIT,
            "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "steps": k,
            "note": "wall clock around blocking C-ABI calls with pinned host buffers"}


def ctypes_stream(stream):
    import ctypes
    return ctypes.c_void_p(stream.cuda_stream)


def main():
    args = parse()
    world, rank, local = dist_setup(args)
    import fjgen
    prob = fjgen.config(args.config, shrink=args.shrink)
    if args.impl == "reference":
        line = run_reference(args, prob, world, rank)
    elif args.mode == "sharded":
        line = run_sharded(args, prob, world, rank, local)
    else:
        line = run_ours(args, prob, world, rank, local)
        if rank == 0 and not args.no_cpu:
            line["cpu_baseline"] = cpu_baseline(prob, args)
    if rank == 0 and line is not None:
        txt = json.dumps(line)
        print(txt, flush=True)
        if args.out:
            with open(args.out, "w") as f:
                f.write(txt + "\n")
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
