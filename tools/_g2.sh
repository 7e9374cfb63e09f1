timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "host_tier or pageable" 2>&1 | tail -3
python bench.py --steps 300 --warmup 10 --host-tier ent_v --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/b_host_v.json
python bench.py --steps 200 --warmup 10 --shard-of 2 --host-tier ent_v --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/b_shard2_host_v.json
