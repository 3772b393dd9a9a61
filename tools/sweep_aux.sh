#!/bin/bash
# A/B of library variants on the auxiliary workloads (cfg3, window, lidar, cfg4): ms per unit.
# usage (under gpurun): bash tools/sweep_aux.sh TAG [configs]
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
TAG=${1:-aux}
CFGS=${2:-"cfg3 window lidar cfg4"}
for so in paper_2501_08672_b200/libsplat_b200*.so; do
  for c in $CFGS; do
    LSB_SO=$PWD/$so timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/sweepaux_${TAG}_${c}_$(basename $so).json 2>&1
    python -c "
import json
d=json.loads(open('gpurun_out/sweepaux_${TAG}_${c}_$(basename $so).json').read().strip().splitlines()[-1])
print('$(basename $so)', '$c', round(d['ms_per_step'],4), d['unit'], round(d['value'],3))" 2>&1 | tail -1
  done
done
