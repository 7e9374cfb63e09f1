// sparse_probe.cu -- the fused segment-reduce + sparse-Adam kernel (k_adam.cu) timed alone on
// the bench's id streams (a12 + a13).  Built with k_adam.cu and k_dedup.cu into a small .so
// (tools/sparse_probe.py builds and drives it); ids come from kggen batches, the tables are
// a theta_E shard of the workload's size, so the rows are random HBM rows as in the step.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../paper_2110_14890_b200/csrc/kg_launch.h"

namespace kg {
int64_t g_launches = 0;
}

extern "C" {
// ids [L] int64 device; outputs into the given device buffers
int probe_dedup(const int64_t *ids, int L, int end_bit, int64_t *uniq, int32_t *inv, int32_t *perm, int32_t *seg,
                int32_t *U, int32_t *sinv, int32_t *hrow, void *stream) {
  kg::launch_dedup(ids, nullptr, L, end_bit, uniq, inv, perm, seg, U, (cudaStream_t)stream, sinv, hrow);
  return (int)cudaGetLastError();
}

int probe_sparse(const int64_t *uniq, const int32_t *seg, const int32_t *perm, const int32_t *sinv, const int32_t *hrow,
                 const int32_t *U,
                 int L, const float *OG, float *PS, int32_t *cnt, int d, float *ent, float *m, float *v,
                 const float *lr, const float *bc, const int *flags, int early, void *stream) {
  kg::launch_sparse_adam(uniq, seg, perm, sinv, hrow, U, L, OG, PS, cnt, d, 1, ent, m, v, nullptr, lr, 0.9, 0.999, 1e-8,
                         bc, flags, 1, (cudaStream_t)stream, -1, early);
  return (int)cudaGetLastError();
}
}

