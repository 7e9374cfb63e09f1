#!/bin/bash
# Per-stage DRAM traffic of every workload under ncu -> gpurun_out/traffic_<W>.csv (then: python tools/step_traffic.py --parse gpurun_out/traffic_*.csv)
for W in C5-q2b C2 C3-complex C3-rotate C4 C5-betae C5-q2b-bw C4-bw; do
  timeout 600 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv --log-file gpurun_out/traffic_$W.csv python tools/step_traffic.py --workload $W > gpurun_out/tr_$W.log 2>&1
  tail -1 gpurun_out/tr_$W.log
done
