#!/bin/bash
TAG=${1:-r01}
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
NCU=/usr/local/cuda/bin/ncu
timeout 300 python tools/debug_optimize.py > gpurun_out/debug_opt_$TAG.log 2>&1
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
  > gpurun_out/ncu_bench_$TAG.log 2>&1
for K in ${KERNELS:-k_blend_bwd k_blend_fwd}; do
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:$K -s 12 -c 1 \
    -o gpurun_out/prof_${TAG}_$K python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
    > gpurun_out/ncu_${K}_$TAG.log 2>&1
done
cat gpurun_out/debug_opt_$TAG.log; grep -E "passed|failed|FAILED" gpurun_out/pytest_gpu_$TAG.log | tail -12
