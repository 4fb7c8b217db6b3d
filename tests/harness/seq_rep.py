"""Full-size property tests followed by warm-start tests in one process (diagnostics: history-dependent flakes)."""
import sys, os, traceback
sys.path.insert(0, os.getcwd())
import torch
from tests import test_gpu_parity as T
dev = torch.device("cuda:0")
fails = 0
for rnd in range(3):
    for cid in (2, 3, 4, 5):
        T.test_full_size_config_properties(dev, cid)
    for name in ["er2000", "rmat12w", "lattice64", "er2000", "rmat12w", "lattice64"]:
        try:
            T.test_warm_start_resume(dev, name)
        except Exception:
            fails += 1
            traceback.print_exc()
    print("round", rnd, "fails", fails, flush=True)
