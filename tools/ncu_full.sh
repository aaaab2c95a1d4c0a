#!/bin/bash
# ncu --set full capture of the top kernels of one compute() at 512^3 gnoise (scratch -> gpurun_out/).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-full}
REGEX=${REGEX:-"k_kahn_persistent|k_origin_dests|k_gradient|k_bfs_persistent|k_source_write"}
timeout ${NCU_TIMEOUT:-1500} ncu --set full --clock-control none --import-source on --profile-from-start off \
  --kernel-name "regex:${REGEX}" --launch-count ${COUNT:-8} -f -o gpurun_out/${TAG} \
  python tools/profile_compute.py ${SIZE:-512} ${KIND:-gnoise} > gpurun_out/${TAG}.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${TAG}.log
tail -5 gpurun_out/${TAG}.log
ls -la gpurun_out/
