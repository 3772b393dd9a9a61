#!/bin/bash
# Compile blend.cu alone (register / spill report) and dump the fused kernel's SASS to /tmp/fused.sass.
# usage: bash tools/cc_blend.sh [-DFLAG=..]
R=/root/repo
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I $R/include -Xptxas -v \
  --expt-relaxed-constexpr "$@" -c $R/paper_2501_08672_b200/csrc/blend.cu -o /tmp/blend.o 2>&1 | grep -A2 "k_blend_fused" | grep -E "registers|spill"
cuobjdump -sass -fun '_ZN3lsb13k_blend_fusedILb1EEEvNS_2WsENS_9BlendArgsENS_8LossArgsE' /tmp/blend.o | grep -E "^\s+/\*[0-9a-f]{4}\*/" | sed 's@/\* 0x[0-9a-f]* \*/@@' > /tmp/fused.sass
wc -l < /tmp/fused.sass
