#!/usr/bin/env bash
cd "$(dirname "$0")/.."
for args in "8192 544 8192 f64" "8192 544 8192 f64 row" "8192 544 8192 i32" "8192 544 8192 f32" "8192 512 8192 f64 row" "8192 256 8192 f64 row" "8192 8192 512 f32" "4096 272 4096 f64 row" "131072 1056 8192 f64"; do
  python scripts/igemm_once.py $args 2>&1 | tail -1
done
