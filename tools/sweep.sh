#!/bin/bash
# A/B sweep of library variants: bench.py per variant (kernel split only).
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
TAG=${1:-sweep}
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
tail -2 gpurun_out/pytest_gpu_$TAG.log
for so in paper_2501_08672_b200/libsplat_b200*.so; do
  LSB_SO=$PWD/$so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/sweep_$(basename $so).json 2>&1
  python -c "
import json,sys
d=json.loads(open('gpurun_out/sweep_$(basename $so).json').read().strip().splitlines()[-1])
print('$(basename $so)', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['kernel_ms_per_step'].items()})"
done
