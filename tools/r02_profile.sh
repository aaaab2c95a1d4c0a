#!/bin/bash
# Round-2 evidence run on one B200 (scratch -> gpurun_out/): bench line, per-kernel launch
# list (ncu gpu__time_duration), per-stage DRAM traffic, ncu --set full of the top kernels.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r02}
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches_${TAG}.csv python tools/profile_compute.py 512 gnoise > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/launches_${TAG}.csv > gpurun_out/launches_${TAG}.txt 2>&1
bash tools/ncu_traffic.sh 512 gnoise > /dev/null 2>&1
TAG=full_${TAG} REGEX="k_gradient|k_count|k_walk|k_reach|k_rewrite|k_succ_table|k_compact_crit3|k_jump_all" COUNT=12 \
  NCU_TIMEOUT=1500 bash tools/ncu_full.sh > /dev/null 2>&1
ls -la gpurun_out/
