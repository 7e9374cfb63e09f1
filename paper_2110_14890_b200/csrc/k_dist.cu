// k_dist.cu -- row-sharded theta_E across ranks: routing kernels
// for the request / row / gradient exchange around the NCCL calls of kg_api.cu.
//
// PAPER.md §4.1: one worker per GPU; the paper keeps theta_E in host
// memory with hogwild updates; this build row-shards theta_E and its
// Adam state over the GPUs (owner(id) = id % G, local row = id / G) and keeps
// the update synchronous (reading A18).  Every order below is a fixed function
// of the inputs (deterministic merges, no atomics).
#include <cstdio>

#include "kg_common.cuh"
#include "kg_launch.h"

namespace kg {

constexpr int kPartThreads = 1024;

// Stable partition of the distinct ids (ascending) by owner: send_ids[pos] = uniq[u]
// with pos = offset[owner] + (rank of u among the ids of that owner); send_pos[u] = pos;
// counts[o] = number of distinct ids owned by o.  One CTA; per-thread contiguous
// ranges keep the order stable.  cap > 0: fixed-capacity buckets instead (offset[o] =
// o * cap, the caller pre-fills send_ids with -1 = empty slot); an id ranked >= cap in its
// bucket is not sent and flags[1] = 2 marks the step as not applicable (bucket overflow).
__global__ void __launch_bounds__(kPartThreads) owner_partition_kernel(const int64_t *uniq, const int32_t *U_dev,
                                                                       int G, int64_t *send_ids, int32_t *send_pos,
                                                                       int32_t *counts, int cap, int *flags) {
  KG_GRID_DEP_WAIT();
  __shared__ int32_t s_cnt[kMaxWorld][kPartThreads];
  __shared__ int32_t s_base[kMaxWorld + 1];
  const int U = *U_dev, t = threadIdx.x;
  const int per = (U + kPartThreads - 1) / kPartThreads;
  const int b = t * per, e = min(U, b + per);
  int c[kMaxWorld];
#pragma unroll
  for (int o = 0; o < kMaxWorld; ++o) c[o] = 0;
  for (int u = b; u < e; ++u) {
    const int o = (int)(uniq[u] % G);
#pragma unroll
    for (int q = 0; q < kMaxWorld; ++q) c[q] += (q == o);
  }
#pragma unroll
  for (int o = 0; o < kMaxWorld; ++o) s_cnt[o][t] = c[o];
  __syncthreads();
  if (t < G) {   // exclusive scan over threads for owner t (serial, fixed order)
    int run = 0;
    for (int k = 0; k < kPartThreads; ++k) {
      const int v = s_cnt[t][k];
      s_cnt[t][k] = run;
      run += v;
    }
    counts[t] = run;
    s_base[t + 1] = run;
  }
  __syncthreads();
  if (t == 0) {
    s_base[0] = 0;
    if (cap > 0) {
      for (int o = 0; o <= G; ++o) s_base[o] = o * cap;
    } else {
      for (int o = 1; o <= G; ++o) s_base[o] += s_base[o - 1];
    }
  }
  __syncthreads();
  int run[kMaxWorld];
#pragma unroll
  for (int o = 0; o < kMaxWorld; ++o) run[o] = (o < G) ? s_base[o] + s_cnt[o][t] : 0;
  for (int u = b; u < e; ++u) {
    const int o = (int)(uniq[u] % G);
    int pos = 0;
#pragma unroll
    for (int q = 0; q < kMaxWorld; ++q)
      if (q == o) pos = run[q]++;
    if (cap > 0 && pos >= (o + 1) * cap) {   // bucket overflow: the step will not be applied
      flags[1] = 2;
      pos = o * cap;
    } else {
      send_ids[pos] = uniq[u];
    }
    send_pos[u] = pos;
  }
}

void launch_owner_partition(const int64_t *uniq, const int32_t *U_dev, int G, int64_t *send_ids, int32_t *send_pos,
                            int32_t *counts, cudaStream_t st, int cap, int *flags) {
  { owner_partition_kernel<<<1, kPartThreads, 0, st>>>(uniq, U_dev, G, send_ids, send_pos, counts, cap, flags); ++g_launches; }
}

// rows[p] = send_pos[inv[p]]: the occurrence's row in the received (owner-grouped) row buffer.
__global__ void occ_rows_kernel(const int32_t *inv, const int32_t *send_pos, int L, int64_t *rows) {
  KG_GRID_DEP_WAIT();
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < L) rows[p] = send_pos[inv[p]];
}
void launch_occ_rows(const int32_t *inv, const int32_t *send_pos, int L, int64_t *rows, cudaStream_t st) {
  if (L > 0) { occ_rows_kernel<<<(L + 255) / 256, 256, 0, st>>>(inv, send_pos, L, rows); ++g_launches; }
}

// Owner side: out[i] = theta_E[ids[i] / G] (rows requested by the peers, in receive order).
__global__ void gather_owned_kernel(const float *ent, const int64_t *ids, int n, int G, int d4, float4 *out) {
  KG_GRID_DEP_WAIT();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)n * d4) return;
  const int i = (int)(e / d4), c = (int)(e - (int64_t)i * d4);
  const int64_t id = ids[i];
  if (id < 0) return;   // empty bucket slot
  out[e] = reinterpret_cast<const float4 *>(ent)[(id / G) * d4 + c];
}
void launch_gather_owned(const float *ent, const int64_t *ids, int n, int G, int d, float *out, cudaStream_t st) {
  const int64_t m = (int64_t)n * (d / 4);
  if (m > 0) {
    gather_owned_kernel<<<(int)((m + 255) / 256), 256, 0, st>>>(ent, ids, n, G, d / 4, reinterpret_cast<float4 *>(out));
    ++g_launches;
  }
}

// out[send_pos[u]] = G[u] (merged row gradients in send order).
__global__ void reorder_rows_kernel(const float4 *Gu, const int32_t *send_pos, const int32_t *U_dev, int d4,
                                    float4 *out) {
  KG_GRID_DEP_WAIT();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int u = (int)(e / d4), c = (int)(e - (int64_t)u * d4);
  if (u >= *U_dev) return;
  out[(int64_t)send_pos[u] * d4 + c] = Gu[e];
}
void launch_reorder_rows(const float *Gu, const int32_t *send_pos, const int32_t *U_dev, int Lmax, int d, float *out,
                         cudaStream_t st) {
  const int64_t m = (int64_t)Lmax * (d / 4);
  if (m > 0) {
    reorder_rows_kernel<<<(int)((m + 255) / 256), 256, 0, st>>>(reinterpret_cast<const float4 *>(Gu), send_pos, U_dev,
                                                                d / 4, reinterpret_cast<float4 *>(out));
    ++g_launches;
  }
}

// keys[i] = ids[i] / G (owner-local rows of the received ids, for the owner-side merge);
// empty bucket slots (id < 0) get the key `empty` (one past the last local row).
__global__ void local_rows_kernel(const int64_t *ids, int n, int G, int64_t *keys, int64_t empty) {
  KG_GRID_DEP_WAIT();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) keys[i] = ids[i] < 0 ? empty : ids[i] / G;
}
void launch_local_rows(const int64_t *ids, int n, int G, int64_t *keys, cudaStream_t st, int64_t empty) {
  if (n > 0) { local_rows_kernel<<<(n + 255) / 256, 256, 0, st>>>(ids, n, G, keys, empty); ++g_launches; }
}

// ---------------------------------------------------------------- peer-memory exchange
// KG_XCHG=p2p: the ranks' theta_E shards and owner-side receive buffers are
// mapped into every rank (CUDA IPC over NVLink / NVSwitch; in-process for the loopback test
// hook), so the row exchange needs no NCCL call: a rank READS the rows it needs straight from
// the owners' shards into its bucket-ordered row buffer (the same layout the NCCL path
// receives), and WRITES its merged row gradients straight into the owners' receive buckets;
// two flag barriers per step order these one-sided accesses against the owners' updates.

// X[send_pos[u]] = theta_E^{owner(id)}[id / G] for the distinct ids u of this rank.
__global__ void p2p_gather_kernel(const PeerPtrs *__restrict__ pp, const int64_t *uniq, const int32_t *U_dev,
                                  const int32_t *send_pos, int G, int d4, float4 *X) {
  KG_GRID_DEP_WAIT();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int u = (int)(e / d4), c = (int)(e - (int64_t)u * d4);
  if (u >= *U_dev) return;
  const int64_t id = uniq[u];
  const float4 *src = reinterpret_cast<const float4 *>(pp->ent[id % G]);
  X[(int64_t)send_pos[u] * d4 + c] = src[(id / G) * d4 + c];
}
void launch_p2p_gather(const PeerPtrs *pp, const int64_t *uniq, const int32_t *U_dev, const int32_t *send_pos, int G,
                       int Lmax, int d, float *X, cudaStream_t st) {
  const int64_t m = (int64_t)Lmax * (d / 4);
  if (m > 0) {
    p2p_gather_kernel<<<(int)((m + 255) / 256), 256, 0, st>>>(pp, uniq, U_dev, send_pos, G, d / 4,
                                                              reinterpret_cast<float4 *>(X));
    ++g_launches;
  }
}

// Bucket o of this rank (ids, -1 = empty slot, and the gradient rows of the filled slots) into
// owner o's receive buffers at [me][0 .. cap): the layout the NCCL path's receive produces.
__global__ void p2p_push_kernel(const PeerPtrs *__restrict__ pp, const int64_t *send_ids, const float4 *Gsend, int G,
                                int me, int cap, int d4) {
  KG_GRID_DEP_WAIT();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t slot = e / d4;
  if (slot >= (int64_t)G * cap) return;
  const int c = (int)(e - slot * d4), o = (int)(slot / cap), k = (int)(slot - (int64_t)o * cap);
  const int64_t id = send_ids[slot], dst = (int64_t)me * cap + k;
  if (c == 0) pp->rids[o][dst] = id;
  if (id >= 0) reinterpret_cast<float4 *>(pp->grecv[o])[dst * d4 + c] = Gsend[slot * d4 + c];
  __threadfence_system();
}
void launch_p2p_push(const PeerPtrs *pp, const int64_t *send_ids, const float *Gsend, int G, int me, int cap, int d,
                     cudaStream_t st) {
  const int64_t m = (int64_t)G * cap * (d / 4);
  if (m > 0) {
    p2p_push_kernel<<<(int)((m + 255) / 256), 256, 0, st>>>(pp, send_ids, reinterpret_cast<const float4 *>(Gsend), G,
                                                            me, cap, d / 4);
    ++g_launches;
  }
}

// All-rank barrier on flags in peer memory: epoch e = ++(*epoch) (identical on every rank:
// every rank passes the same barriers in the same order), release-store e into flag `me` of
// every rank, then acquire-spin until all G flags of this rank reach e.  A peer that does not
// arrive within 20 s sets flags[1] = 3 (the step is reported failed) instead of hanging.
__global__ void p2p_barrier_kernel(const PeerPtrs *__restrict__ pp, unsigned long long *mine,
                                   unsigned long long *epoch, int G, int me, int *flags) {
  KG_GRID_DEP_WAIT();
  if (threadIdx.x != 0) return;
  const unsigned long long e = *epoch + 1;
  *epoch = e;
  __threadfence_system();
  for (int o = 0; o < G; ++o)
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(pp->flags[o] + me), "l"(e) : "memory");
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int o = 0; o < G; ++o) {
    while (true) {
      unsigned long long v, now;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(mine + o) : "memory");
      if (v >= e) break;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (now - t0 > 20000000000ull) {
        // flags[0] too: every update kernel queued after this barrier (the owner's sparse Adam)
        // checks flags[0] only, so none of them applies a stale bucket
        flags[1] = 3;
        flags[0] |= 2;
        printf("kg p2p barrier timeout: rank %d epoch %llu waiting on rank %d (flag %llu)\n", me, e, o, v);
        return;
      }
      __nanosleep(256);
    }
  }
}
void launch_p2p_barrier(const PeerPtrs *pp, unsigned long long *mine, unsigned long long *epoch, int G, int me,
                        int *flags, cudaStream_t st) {
  { p2p_barrier_kernel<<<1, 32, 0, st>>>(pp, mine, epoch, G, me, flags); ++g_launches; }
}

// Dense relation gradient (for the all-reduce): gfull[s*R*w + r*w + c] = RGU[u][s*w + c]
// for the relations used by this rank (the caller zeroes the relation part first).
__global__ void scatter_rel_kernel(const float *RGU, const int64_t *runiq, const int32_t *rU, int R, int w, int nseg,
                                   float *gfull) {
  KG_GRID_DEP_WAIT();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int dr = w * nseg;
  const int u = (int)(e / dr), c = (int)(e - (int64_t)u * dr);
  if (u >= *rU) return;
  const int s = c / w, cc = c - s * w;
  gfull[(int64_t)s * R * w + runiq[u] * w + cc] = RGU[e];
}
void launch_scatter_rel(const float *RGU, const int64_t *runiq, const int32_t *rU, int Lrmax, int R, int w, int nseg,
                        float *gfull, cudaStream_t st) {
  const int64_t m = (int64_t)Lrmax * w * nseg;
  if (m > 0) {
    scatter_rel_kernel<<<(int)((m + 255) / 256), 256, 0, st>>>(RGU, runiq, rU, R, w, nseg, gfull);
    ++g_launches;
  }
}

}  // namespace kg
