"""Per-kernel summary of one timed bench step from an ncu launch list (diagnostics).
usage: python tools/launch_summary.py LAUNCHES.csv [STEP_INDEX=2] — steps start at k_validate_rowptr
(the first kernel of fj_graph_create); with --steps 2 --warmup 1 index 2 is the last timed step."""
import csv
import sys
from collections import OrderedDict

path = sys.argv[1]
step = int(sys.argv[2]) if len(sys.argv) > 2 else 2
rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
hdr = rows[0]
ik, im, iv, iu = (hdr.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
L = []
for r in rows[1:]:
    if r[im] != "gpu__time_duration.sum":
        continue
    v = float(r[iv].replace(",", ""))
    v *= {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}.get(r[iu], 1e-6)
    L.append((r[ik], v))
starts = [i for i, (k, _) in enumerate(L) if "k_validate_rowptr" in k]
a = starts[step]
b = starts[step + 1] if step + 1 < len(starts) else len(L)
seg = L[a:b]
tot = sum(v for _, v in seg)
agg = OrderedDict()
for k, v in seg:
    name = k.split("(")[0].replace("fj::", "")
    c = agg.setdefault(name, [0, 0.0])
    c[0] += 1
    c[1] += v
print(f"# One timed step (launches {a}..{b - 1} of the list: graph create -> solve -> measures): "
      f"{len(seg)} launches, {tot:.2f} ms summed (cold-cache, serialised)")
print(f"{'kernel':48s} {'launches':>8s} {'ms':>10s} {'share':>7s}")
for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:48]:48s} {n:8d} {v:10.3f} {100 * v / tot:6.2f}%")
