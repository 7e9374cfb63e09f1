// k_dedup.cu -- index dedup / segment sort (SURVEY K-new-1).
//
// PAPER.md §4.2: the gradients of theta_E^{V_q}, theta_E^{N} and
// theta_E^{A} are scattered "into a single continuous memory, due to the
// potential overlap among the sets V_q, N_q and A_q".  Here: one CTA sorts the
// L = M*n_anchor + M + K occurrence ids (stable LSD radix sort of (id,
// position) pairs in shared memory), flags segment heads, scans them, and
// writes the distinct ids ascending, the inverse map, the sorted positions and
// the segment starts.  The sparse-Adam kernel then sums each segment in
// ascending position order: a fixed order, no atomics on hot rows.
#include <cub/block/block_discontinuity.cuh>
#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_scan.cuh>

#include "kg_common.cuh"
#include "kg_launch.h"

namespace kg {

constexpr int kDedupThreads = 1024;

template <int ITEMS>
__global__ void __launch_bounds__(kDedupThreads) dedup_kernel(const int64_t *ids64, const int32_t *ids32, int L,
                                                              int end_bit, int64_t *uniq, int32_t *inv,
                                                              int32_t *perm, int32_t *seg, int32_t *U_out,
                                                              int32_t *sinv, int32_t *hrow) {
  KG_GRID_DEP_WAIT();
  using Sort = cub::BlockRadixSort<uint32_t, kDedupThreads, ITEMS, uint32_t>;
  using Disc = cub::BlockDiscontinuity<uint32_t, kDedupThreads>;
  using Scan = cub::BlockScan<int, kDedupThreads>;
  union Temp {
    typename Sort::TempStorage sort;
    typename Disc::TempStorage disc;
    typename Scan::TempStorage scan;
  };
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Temp &temp = *reinterpret_cast<Temp *>(smem_raw);

  const uint32_t pad = (end_bit >= 32) ? 0xFFFFFFFFu : ((1u << end_bit) - 1u);
  uint32_t keys[ITEMS], vals[ITEMS];
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    const int p = threadIdx.x * ITEMS + it;   // blocked arrangement
    uint32_t k = pad;
    if (p < L) k = ids64 ? (uint32_t)ids64[p] : (uint32_t)ids32[p];
    keys[it] = k;
    vals[it] = (uint32_t)p;
  }
  // stable: equal keys keep ascending positions; padding (p >= L) sorts last
  Sort(temp.sort).Sort(keys, vals, 0, end_bit);
  __syncthreads();

  int head[ITEMS], tail[ITEMS];
  Disc(temp.disc).FlagHeadsAndTails(head, tail, keys, cub::Inequality());
  __syncthreads();
#pragma unroll
  for (int it = 0; it < ITEMS; ++it)
    if ((int)vals[it] >= L) head[it] = 0;
  int excl[ITEMS], total;
  Scan(temp.scan).ExclusiveSum(head, excl, total);
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    const int s = threadIdx.x * ITEMS + it;
    if ((int)vals[it] >= L) continue;
    const int u = excl[it] + head[it] - 1;
    perm[s] = (int32_t)vals[it];
    inv[vals[it]] = u;
    if (sinv) sinv[s] = u;   // sorted position -> distinct index (= inv[perm[s]])
    if (head[it]) {
      uniq[u] = (int64_t)keys[it];
      seg[u] = s;
      // the single occurrence of a segment of length 1, else -1 (the next position is
      // padding, p >= L, or another key)
      if (hrow) hrow[u] = (tail[it] || s + 1 >= L) ? (int32_t)vals[it] : -1;
    }
  }
  if (threadIdx.x == 0) {
    seg[total] = L;
    *U_out = total;
  }
}

int dedup_capacity() { return kDedupThreads * 32; }

template <int ITEMS>
static void run_dedup(const int64_t *ids64, const int32_t *ids32, int L, int end_bit, int64_t *uniq, int32_t *inv,
                      int32_t *perm, int32_t *seg, int32_t *U_out, int32_t *sinv, int32_t *hrow,
                      cudaStream_t st) {
  using Sort = cub::BlockRadixSort<uint32_t, kDedupThreads, ITEMS, uint32_t>;
  using Disc = cub::BlockDiscontinuity<uint32_t, kDedupThreads>;
  using Scan = cub::BlockScan<int, kDedupThreads>;
  size_t bytes = sizeof(typename Sort::TempStorage);
  if (sizeof(typename Disc::TempStorage) > bytes) bytes = sizeof(typename Disc::TempStorage);
  if (sizeof(typename Scan::TempStorage) > bytes) bytes = sizeof(typename Scan::TempStorage);
  // per-template attribute, set once (a function-local static: thread-safe initialisation, the
  // handles of several host threads may launch concurrently)
  static const bool configured =
      cudaFuncSetAttribute(dedup_kernel<ITEMS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) == cudaSuccess;
  (void)configured;
  { dedup_kernel<ITEMS><<<1, kDedupThreads, bytes, st>>>(ids64, ids32, L, end_bit, uniq, inv, perm, seg, U_out, sinv, hrow); ++g_launches; }
}

void launch_dedup(const int64_t *ids64, const int32_t *ids32, int L, int end_bit, int64_t *uniq, int32_t *inv,
                  int32_t *perm, int32_t *seg, int32_t *U_out, cudaStream_t st, int32_t *sinv, int32_t *hrow) {
  if (end_bit < 1) end_bit = 1;
  if (L <= kDedupThreads * 4) run_dedup<4>(ids64, ids32, L, end_bit, uniq, inv, perm, seg, U_out, sinv, hrow, st);
  else if (L <= kDedupThreads * 8) run_dedup<8>(ids64, ids32, L, end_bit, uniq, inv, perm, seg, U_out, sinv, hrow, st);
  else if (L <= kDedupThreads * 16) run_dedup<16>(ids64, ids32, L, end_bit, uniq, inv, perm, seg, U_out, sinv, hrow, st);
  else run_dedup<32>(ids64, ids32, L, end_bit, uniq, inv, perm, seg, U_out, sinv, hrow, st);
}

}  // namespace kg
