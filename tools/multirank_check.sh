#!/bin/bash
# N>1 bench paths on a one-GPU box: every rank on cuda:0 (LSB_BENCH_SHARE_GPU),
# gloo for the exchange (NCCL refuses two ranks on one GPU).  Checks that the
# torchrun launches exit 0 and print one JSON line; the times are not a
# scaling measurement (the ranks share one GPU).
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1 LSB_BENCH_SHARE_GPU=1 LSB_BENCH_BACKEND=gloo
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 2 4; do
  for C in target cfg2 cfg3 window lidar cfg4; do
    timeout 600 $TR --nproc-per-node $N --master-port $((29500 + N)) bench.py --gpus $N --steps 5 --warmup 3 \
      --config $C --no-cpu-baseline > gpurun_out/mr_${C}_$N.json 2> gpurun_out/mr_${C}_$N.err
    echo "N=$N $C rc=$? $(tail -c 300 gpurun_out/mr_${C}_$N.json)"
  done
  timeout 600 $TR --nproc-per-node $N --master-port $((29600 + N)) bench.py --impl reference --gpus $N --steps 2 \
    --warmup 3 > gpurun_out/mr_ref_$N.json 2> gpurun_out/mr_ref_$N.err
  echo "N=$N reference rc=$? $(tail -c 300 gpurun_out/mr_ref_$N.json)"
done
