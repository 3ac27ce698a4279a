#!/usr/bin/env bash
# rebuild liblramm_cuda.so and the sytrd phase-trace probe
set -e
cd "$(dirname "$0")/.."
python paper_2405_16917_b200/build.py >/dev/null
cd scripts
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I../include sytrd_probe.cu -o sytrd_probe \
  -L../paper_2405_16917_b200 -llramm_cuda -Xlinker -rpath -Xlinker '$ORIGIN/../paper_2405_16917_b200' 2>&1 | grep -i error || true
echo rebuilt
