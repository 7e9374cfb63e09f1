// Driver of tools/gemm_trace.py: launch_gemm_tc from a -DKG_GEMM_TRACE build of k_gemm.cu.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../paper_2110_14890_b200/csrc/kg_launch.h"

namespace kg {
int64_t g_launches = 0;
}
extern "C" int trace_gemm(int ta, int tb, int M, int N, int K, const float *A, int lda, const float *B, int ldb,
                          float *Cm, int ldc, float *P, long long pcap, int force, void *st) {
  kg::GemmArgs g;
  g.A = A; g.B = B; g.C = Cm; g.M = M; g.N = N; g.K = K; g.lda = lda; g.ldb = ldb; g.ldc = ldc;
  g.a_mn = ta != 0; g.b_mn = tb != 0; g.drain = true; g.force = force;
  return kg::launch_gemm_tc(g, P, pcap, (cudaStream_t)st) ? 1 : 0;
}
