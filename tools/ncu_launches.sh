#!/bin/bash
# Per-kernel launch list (gpu__time_duration) of one compute() -> gpurun_out/launches_<tag>.txt
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
SIZE=${1:-512}; KIND=${2:-gnoise}; TAG=${3:-${SIZE}_${KIND}}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches_${TAG}.csv python tools/profile_compute.py ${SIZE} ${KIND} > gpurun_out/ncu_${TAG}.log 2>&1
python tools/ncu_summary.py gpurun_out/launches_${TAG}.csv > gpurun_out/launches_${TAG}.txt 2>&1
cat gpurun_out/launches_${TAG}.txt
