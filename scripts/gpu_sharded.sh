#!/usr/bin/env bash
# GPU round-trip for the native sharded pipeline tests
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharded_native.py -x -q ${PYTEST_ARGS:-} > gpurun_out/sharded.log 2>&1; echo "rc=$?" >> gpurun_out/sharded.log
tail -40 gpurun_out/sharded.log
