"""Refresh profiles/ncu_sweep_traffic.json from an ncu capture of k_sweep on
the CURRENT build (bench.py uses it only when sass_sha16 matches the loaded
libfj.so).  Run on the GPU box:

    ncu --set full --clock-control none --import-source on -k regex:k_sweep -c 1 \\
        -o gpurun_out/prof_X python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --no-sweep
    python tools/ncu_traffic.py gpurun_out/prof_X.ncu-rep SWEEPS_IN_LAUNCH

SWEEPS_IN_LAUNCH: the sweeps of the captured launch (bench's step_breakdown)."""
import csv, hashlib, io, json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep, sweeps = sys.argv[1], int(sys.argv[2])
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
def get(name):
    i = hdr.index(name)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ms": 1, "us": 1e-3,
             "ns": 1e-6, "s": 1e3}[units[i]]
    return float(vals[i].replace(",", "")) * scale
rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
lib = os.path.join(ROOT, "paper_2507_14864_b200", "libfj.so")
sys.path.insert(0, ROOT)
from bench import sass_fingerprint  # noqa: E402
sha = sass_fingerprint(lib)
out = {"kernel": vals[hdr.index("Kernel Name")], "config": 4, "source": os.path.basename(rep),
       "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
       "sweeps_in_launch": sweeps, "dram_bytes_per_sweep": (rd + wr) / sweeps,
       "duration_ms": get("gpu__time_duration.sum"), "sass_sha16": sha}
json.dump(out, open(os.path.join(ROOT, "profiles", "ncu_sweep_traffic.json"), "w"), indent=1)
print(json.dumps(out))
