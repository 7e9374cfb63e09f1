#!/bin/bash
# Every bench workload at its defaults + the reference arm + the C5-q2b launch list + per-stage DRAM
# traffic of the main workloads + full ncu captures of the top kernels (one gpurun call).
#   bash tools/run_all_benches.sh r2   -> gpurun_out/r/<tag>_*
TAG=${1:-r2}
set -x
mkdir -p gpurun_out/r
for p in "C5-q2b default" "C2 c2_q2b" "C3-complex c3_complex" "C3-rotate c3_rotate" "C4 c4_betae" "C5-betae c5_betae" "C5-q2b-bw c5q2b_bw" "C4-bw c4_bw"; do
  set -- $p
  timeout 600 python bench.py --workload $1 > gpurun_out/r/${TAG}_bench_$2.json 2> gpurun_out/r/${TAG}_$2.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r/${TAG}_bench_reference_arm.json 2> gpurun_out/r/${TAG}_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r/${TAG}_launches_c5q2b.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-sampler > /dev/null 2>&1
for W in C5-q2b C5-betae C5-q2b-bw C4 C2 C3-complex C3-rotate C4-bw; do
  timeout 600 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv --log-file gpurun_out/r/traffic_$W.csv python tools/step_traffic.py --workload $W > /dev/null 2>&1
done
timeout 600 ncu --profile-from-start off --clock-control none --set full --import-source on --kernel-name-base demangled -k "regex:pair_bwd_kernel<kg::MBox>" -c 1 -o gpurun_out/r/${TAG}_pairbwd_full python tools/step_traffic.py --workload C5-q2b > /dev/null 2>&1
timeout 600 ncu --profile-from-start off --clock-control none --set full --import-source on --kernel-name-base demangled -k "regex:pair_fwd_kernel<kg::MBox, \(int\)1>" -c 1 -o gpurun_out/r/${TAG}_pairfwd_full python tools/step_traffic.py --workload C5-q2b > /dev/null 2>&1
timeout 600 ncu --profile-from-start off --clock-control none --set full --import-source on -k regex:sparse_adam_fused -c 2 -o gpurun_out/r/${TAG}_sparse_full python tools/step_traffic.py --workload C5-q2b > /dev/null 2>&1
timeout 600 ncu --profile-from-start off --clock-control none --set full --import-source on --kernel-name-base demangled -k "regex:gemm_tf32x3_tma_kernel<\(int\)160" -c 1 -o gpurun_out/r/${TAG}_gemm160_full python tools/step_traffic.py --workload C5-betae > /dev/null 2>&1
for R in gpurun_out/r/${TAG}_*_full.ncu-rep; do
  ncu -i $R --page raw --csv > ${R%.ncu-rep}_raw.csv 2>/dev/null
done
ls -la gpurun_out/r
