#!/bin/bash
# A/B sweep of library variants: bench.py per variant (step time + kernel split).
# usage (under gpurun): bash tools/sweep.sh TAG [bench args]
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
TAG=${1:-sweep}
shift
for so in paper_2501_08672_b200/libsplat_b200*.so; do
  LSB_SO=$PWD/$so timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/sweep_${TAG}_$(basename $so).json 2>&1
  python -c "
import json,sys
d=json.loads(open('gpurun_out/sweep_${TAG}_$(basename $so).json').read().strip().splitlines()[-1])
print('$(basename $so)', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],3), {k: round(v,3) for k,v in d['kernel_ms_per_step'].items()})"
done
