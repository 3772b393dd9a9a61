#!/bin/bash
# Profiling of the auxiliary workloads (under gpurun): for each of cfg3 (voxel
# map), lidar, cfg4 (IESKF update) and window (maintain), the per-kernel
# device time, DRAM bytes and warp instructions of every kernel inside the
# bench's timed region (NVTX range lsb_timed), plus one `ncu --set full`
# capture of that workload's top kernel.
# usage: bash tools/gpu_prof_aux.sh TAG
TAG=${1:-r02c}
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
NCU=/usr/local/cuda/bin/ncu
MET=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum
declare -A STEPS=([cfg3]=10 [lidar]=3 [cfg4]=2 [window]=10)
declare -A TOP=([cfg3]=k_acc_fold [lidar]=k_lidar_rows [cfg4]=k_pose_rows [window]=k_win_mark)
for W in ${WL:-cfg3 lidar cfg4 window}; do
  timeout 900 $NCU --metrics $MET --clock-control none --nvtx --nvtx-include "lsb_timed/" --csv \
    --log-file gpurun_out/aux_${TAG}_$W.csv python bench.py --config $W --steps ${STEPS[$W]} --warmup 1 \
    --no-cpu-baseline > gpurun_out/aux_${TAG}_$W.log 2>&1
  timeout 900 $NCU --set full --clock-control none --import-source on --nvtx --nvtx-include "lsb_timed/" \
    -k regex:${TOP[$W]} -c 1 -o gpurun_out/prof_${TAG}_${W}_${TOP[$W]} python bench.py --config $W \
    --steps ${STEPS[$W]} --warmup 1 --no-cpu-baseline > gpurun_out/prof_${TAG}_$W.log 2>&1
done
ls gpurun_out | grep $TAG
