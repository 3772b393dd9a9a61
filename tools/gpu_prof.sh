#!/bin/bash
# One profiling session (under gpurun): the bench line, the launch list of a
# short bench run, and one `ncu --set full` capture per kernel in $KERNELS.
# usage: KERNELS="k_blend_bwd k_blend_fwd" bash tools/gpu_prof.sh TAG [bench args]
TAG=${1:-r01}
shift
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
NCU=/usr/local/cuda/bin/ncu
timeout 600 python bench.py "$@" > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline "$@" \
  > gpurun_out/ncu_bench_$TAG.log 2>&1
for K in ${KERNELS:-k_blend_fused k_pre_count k_pre_emit k_chain}; do
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:"(^|:)$K\$" -s 12 -c 1 \
    -o gpurun_out/prof_${TAG}_$K python bench.py --steps 2 --warmup 3 --no-cpu-baseline "$@" \
    > gpurun_out/ncu_${K}_$TAG.log 2>&1
done
tail -c 1500 gpurun_out/bench_$TAG.json
