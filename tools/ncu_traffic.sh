#!/bin/bash
# One compute() under ncu with time + DRAM bytes per kernel -> per-stage traffic (profiles/traffic.json)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
SIZE=${1:-512}; KIND=${2:-gnoise}
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --profile-from-start off --csv --log-file gpurun_out/traffic_${SIZE}_${KIND}.csv \
  python tools/profile_compute.py ${SIZE} ${KIND} > gpurun_out/traffic_${SIZE}_${KIND}.log 2>&1
python tools/stage_traffic.py gpurun_out/traffic_${SIZE}_${KIND}.csv gpurun_out/traffic_${SIZE}_${KIND}.json
