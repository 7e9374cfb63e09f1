timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for wl in C4 C5-q2b; do
python bench.py --workload $wl --steps 200 --warmup 10 2>&1 | tail -1 > gpurun_out/b_${wl}_def.json
done
