"""Key metrics of `ncu --page raw --csv` exports (one kernel each):  python tools/ncu_key.py file..."""
import csv
import sys

KEYS = [("gpu__time_duration.sum", "us"), ("launch__grid_size", ""), ("launch__registers_per_thread", "regs"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "% warps active"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "% issue active"),
        ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "% FMA pipe"),
        ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "% ALU pipe"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "% tensor pipe"),
        ("smsp__inst_executed.sum", "warp inst"), ("dram__bytes_read.sum", "DRAM read"),
        ("dram__bytes_write.sum", "DRAM write"), ("sm__cycles_active.avg", "SM active cycles"),
        ("sm__cycles_elapsed.avg", "SM elapsed cycles")]
for f in sys.argv[1:]:
    rows = list(csv.reader(open(f)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        print(f"{f}: {d.get('Kernel Name', '')[:70]}")
        for k, lab in KEYS:
            if k in d:
                print(f"  {lab or k:18s} {d[k]} {u.get(k, '')}")
