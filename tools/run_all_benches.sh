#!/bin/bash
# Every bench workload at its defaults + the reference arm + the C5-q2b launch list (one gpurun call).
set -x
mkdir -p gpurun_out/r
for p in "C5-q2b default" "C2 c2_q2b" "C3-complex c3_complex" "C3-rotate c3_rotate" "C4 c4_betae" "C5-betae c5_betae" "C5-q2b-bw c5q2b_bw" "C4-bw c4_bw"; do
  set -- $p
  timeout 600 python bench.py --workload $1 > gpurun_out/r/r1_bench_$2.json 2> gpurun_out/r/$2.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r/r1_bench_reference_arm.json 2> gpurun_out/r/ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r/r1_launches_c5q2b_final.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-sampler > /dev/null 2>&1
ls -la gpurun_out/r
