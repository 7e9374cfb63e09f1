cp paper_2110_14890_b200/libkg.so variants/libkg_8.so
for w in 4 8 12 16; do cp variants/libkg_$w.so paper_2110_14890_b200/libkg.so; timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/gemm_w$w.csv python tools/gemm_probe.py > /dev/null 2>&1; done
