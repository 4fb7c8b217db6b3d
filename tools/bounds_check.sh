#!/bin/bash
# Device-side bounds checks of the sweep / frontier kernels (diagnostics; compute-sanitizer is
# closed on the GPU pool): builds libfj with -DFJ_BOUNDS (FJ_CHECK traps on a bad slot, column
# or list entry) and runs the tiny GPU tests that cover row slices, hub pieces and the
# frontier phase under it.  usage: tools/bounds_check.sh   (on the GPU box)
set -u
mkdir -p gpurun_out tools/libs_bounds
python - <<'PY'
import sys
sys.path.insert(0, ".")
from paper_2507_14864_b200 import build as b
print(b.build(out="tools/libs_bounds/libfj.so", defines=("FJ_BOUNDS",)))
PY
FJ_LIB_PATH=$PWD/tools/libs_bounds/libfj.so python -m pytest tests/test_gpu_parity.py -m gpu -q \
  -k "row_walks or row_slices or frontier_phase or tiny_async or tiny_colored or shadow or star or hub" \
  2>&1 | tail -5
