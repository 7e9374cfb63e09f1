timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for i in 1; do python bench.py --workload C4 --steps 200 --warmup 10 2>&1 | tail -1 > gpurun_out/b_C4_r$i.json; done
python bench.py --workload C5-q2b --steps 200 --warmup 10 2>&1 | tail -1 > gpurun_out/b_C5-q2b_def.json
