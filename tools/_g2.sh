for dv in 8 16 1000; do
KG_SPLITK_DIV=$dv python bench.py --workload C5-q2b --steps 300 --warmup 10 2>&1 | tail -1 > gpurun_out/b_q_$dv.json
KG_SPLITK_DIV=$dv python bench.py --workload C4 --steps 200 --warmup 10 2>&1 | tail -1 > gpurun_out/b_c4_$dv.json
done
timeout 600 ncu --set full --import-source on -k regex:pair_bwd -c 1 -o gpurun_out/pair_bwd_f2 python tools/step_probe.py C5-q2b 2i 2 > /dev/null 2>&1
