#!/bin/bash
# Profiling session: ncu launch list of a short bench + full captures.
TAG=${1:-r01}
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
NCU=/usr/local/cuda/bin/ncu
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
  > gpurun_out/ncu_bench_$TAG.log 2>&1
for K in k_blend_bwd k_blend_fwd k_preprocess k_tile_sort k_chain; do
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:$K -s 12 -c 1 \
    -o gpurun_out/prof_${TAG}_$K python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
    > gpurun_out/ncu_${K}_$TAG.log 2>&1
done
tail -3 gpurun_out/pytest_gpu_$TAG.log; ls -la gpurun_out
