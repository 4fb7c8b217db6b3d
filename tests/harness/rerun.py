"""Call one GPU test function many times in one process and report failures
(diagnostics for rare flakes).  usage: rerun.py module func param reps"""
import sys, os, traceback, inspect
sys.path.insert(0, os.getcwd())
import importlib, torch
mod = importlib.import_module(sys.argv[1])
fn = getattr(mod, sys.argv[2])
params = sys.argv[3].split(",")
reps = int(sys.argv[4])
dev = torch.device("cuda:0")
for prm in params:
    fails = 0
    for r in range(reps):
        try:
            kw = {}
            sig = inspect.signature(fn).parameters
            if "dev" in sig: kw["dev"] = dev
            if "name" in sig: kw["name"] = prm
            if "cid" in sig: kw["cid"] = int(prm)
            fn(**kw)
        except Exception:
            fails += 1
            if fails <= 2: traceback.print_exc()
    print(sys.argv[2], prm, "fails", fails, "of", reps, flush=True)
