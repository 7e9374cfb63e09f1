#!/bin/bash
# Host-tier measurements (profiles/r1_bench_c5q2b_g2shard_host_tier.json): theta_E tables in pinned host memory.
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "host_tier or pageable" 2>&1 | tail -3
python bench.py --steps 300 --warmup 10 --host-tier ent_v --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/b_host_v.json
python bench.py --steps 200 --warmup 10 --shard-of 2 --host-tier ent_v --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/b_shard2_host_v.json
