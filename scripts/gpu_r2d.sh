#!/usr/bin/env bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python scripts/e2e_timeline.py 3 3 > gpurun_out/e2e_timeline_3.txt 2>&1; tail -60 gpurun_out/e2e_timeline_3.txt
python scripts/prof_c4.py > gpurun_out/prof_c4.txt 2>&1; tail -45 gpurun_out/prof_c4.txt
