#!/usr/bin/env bash
# --sharded at N = 1 (single-rank NCCL communicators) next to the single-GPU graph, c3 and c5
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in ${CONFIGS:-c3 c5}; do
  timeout 600 python bench.py --config $c --sharded --steps 5 --warmup 3 > gpurun_out/sharded_$c.json 2> gpurun_out/sharded_$c.err; echo "sharded $c rc=$?"
  tail -c 1500 gpurun_out/sharded_$c.json; tail -5 gpurun_out/sharded_$c.err
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --config c2 --sharded --steps 5 --warmup 3 > gpurun_out/sharded_c2_torchrun.json 2> gpurun_out/sharded_c2_torchrun.err; echo "torchrun rc=$?"
tail -c 600 gpurun_out/sharded_c2_torchrun.json
