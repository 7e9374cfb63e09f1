#!/bin/bash
# GPU tests, C5-q2b and C5-q2b-bw bench lines, and isolated (ncu, clocks not locked) durations
# + DRAM bytes of the fused sparse-Adam kernel -> gpurun_out/<tag>_*
TAG=${1:-r2}
python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.txt 2>&1; tail -2 gpurun_out/${TAG}_gpu_tests.txt
python bench.py --no-sampler --no-cpu-baseline > gpurun_out/${TAG}_bench_c5.json 2>&1
python bench.py --workload C5-q2b-bw --no-sampler --no-cpu-baseline --steps 180 > gpurun_out/${TAG}_bench_bw.json 2>&1
for W in C5-q2b C5-q2b-bw; do
  timeout 300 ncu --profile-from-start off --clock-control none -k regex:'sparse_adam|dense_adam|rel_reduce|seg_piece' \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
    --log-file gpurun_out/${TAG}_sa_$W.csv python tools/step_traffic.py --workload $W > /dev/null 2>&1
done
