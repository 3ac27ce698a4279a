#!/usr/bin/env bash
# Round-2 final evidence: bench lines c1..c5 (default = c3 with CPU baseline + accuracy), the
# reference arm, the sharded path at N = 1, the ncu launch list of the default bench command and
# one full ncu capture of the c3 sketch GEMM (each ncu pass only after the plain command exited 0).
cd "$(dirname "$0")/.."
O=gpurun_out/r02f
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
timeout 1200 python bench.py --steps 10 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err; echo "c3 rc=$?"
for c in c1 c2 c4 c5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; echo "$c rc=$?"
done
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > $O/bench_reference_c3.json 2> $O/bench_reference_c3.err; echo "reference rc=$?"
timeout 600 python bench.py --sharded --steps 10 --warmup 3 --no-cpu-baseline --no-accuracy > $O/bench_sharded_c3_n1.json 2> $O/bench_sharded.err; echo "sharded rc=$?"
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-accuracy > $O/plain_bench.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled \
  -k 'regex:lramm::' -c 1200 --csv --log-file $O/ncu_launches_c3.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-accuracy > $O/ncu_launch_run.log 2>&1
echo "ncu launches rc=$?"
python scripts/launch_summary.py $O/ncu_launches_c3.csv > $O/ncu_launches_c3_summary.txt 2>&1; head -12 $O/ncu_launches_c3_summary.txt
timeout 300 python scripts/igemm_once.py 8192 544 8192 f64 row > $O/plain_igemm.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:igemm_tn_kernel -s 3 -c 1 \
  -o $O/ncu_igemm_c3 -f python scripts/igemm_once.py 8192 544 8192 f64 row > $O/ncu_igemm.log 2>&1
echo "igemm ncu rc=$?"
python scripts/ncu_summary.py $O/ncu_igemm_c3.ncu-rep "igemm_tn_kernel<3,0,0> 8192x544x8192 -> f64, row/col scales (c3 sketch shape)" > $O/ncu_igemm_c3.txt 2>&1; head -40 $O/ncu_igemm_c3.txt
