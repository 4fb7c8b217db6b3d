"""A/B of fj_solve_batch builds on one config (diagnostics): FJ_LIB_PATH per run."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for lib in sys.argv[2:]:
    env = dict(os.environ, FJ_LIB_PATH=os.path.join(ROOT, lib))
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "batch_exp.py"), sys.argv[1]],
                         env=env, capture_output=True, text=True)
    for line in out.stdout.splitlines():
        if "batch" in line:
            print(f"{lib:32s} {line}", flush=True)
    if out.returncode:
        print(lib, out.stderr[-400:])
