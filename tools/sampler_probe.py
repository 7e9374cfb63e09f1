"""Host throughput of the native sampler (queries/s) per structure and for the pipeline."""
import sys, time, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import kggen
from paper_2110_14890_b200.sampler import KGSampler, Pipeline

shape = sys.argv[1] if len(sys.argv) > 1 else "FB400k"
t = time.time(); kg = kggen.make_kg(*kggen.KG_SHAPES[shape], seed=0); t_gen = time.time() - t
t = time.time(); smp = KGSampler(kg); t_idx = time.time() - t
print(f"{shape}: |E|={smp.n_edges} roots={smp.n_roots} gen {t_gen:.1f}s index {t_idx:.1f}s threads {smp.n_threads}")
M, K = 512, 1024
for s in kggen.ALL_STRUCTURES:
    t = time.time(); b = smp.sample(s, M, K, seed=0, step=1, n_threads=1); dt = time.time() - t
    bits = kggen.unpack_mask(b["mask"], K)
    print(f"  {s:4s} 1 thread {M/dt:9.0f} q/s  attempts {b['attempts'].mean():.2f}  masked-out {(~bits).mean():.4f}")
p = Pipeline(smp, kggen.STRUCTURES, M, K, seed=0)
for _ in range(4): p.next()
t = time.time(); n = 36
for _ in range(n): p.next()
dt = time.time() - t
print(f"pipeline ({os.cpu_count()} cpus): {n*M/dt:.0f} q/s")
