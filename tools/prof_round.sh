#!/bin/bash
# Profiles of the current build on the GPU box (diagnostics): the bench's
# ncu launch list, one `ncu --set full` capture of k_sweep (source-level
# counters), and the traffic file bench.py reads.  usage: tools/prof_round.sh TAG
set -u
TAG=${1:-x}
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-cpu \
  > gpurun_out/launches_$TAG.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_sweep -c 1 \
  -o gpurun_out/prof_$TAG -f python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --no-sweep \
  > gpurun_out/prof_$TAG.log 2>&1
SW=$(python - "$TAG" <<'PY'
import json, sys
for line in open(f"gpurun_out/prof_{sys.argv[1]}.log"):
    if line.startswith("{"):
        b = json.loads(line)["step_breakdown"]
        print(b.get("shadow_sweeps") or b["sweeps"])  # sweeps of the captured (first) launch
PY
)
python tools/ncu_traffic.py gpurun_out/prof_$TAG.ncu-rep "$SW" > gpurun_out/traffic_$TAG.json 2>&1
cp profiles/ncu_sweep_traffic.json gpurun_out/ncu_sweep_traffic_$TAG.json
python tools/ncu_summary.py gpurun_out/prof_$TAG.ncu-rep > gpurun_out/ncu_summary_$TAG.txt 2>&1
ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv > gpurun_out/source_$TAG.csv 2>&1
ls -la gpurun_out
