// kg_api.cu -- host implementation of the C-ABI in include/kg.h.
//
// Owns the handle: validation, the static per-structure DAG plans (SURVEY
// App. A.3), the device workspace, pinned staging, cuBLAS, and the order in
// which the sm_100a kernels of k_*.cu are enqueued for one training step
// (§4.1, §4.2, §4.3).
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>
#include <mutex>
#include <condition_variable>
#include <atomic>
#include <chrono>
#include <vector>

#include "../../include/kg.h"
#include <nvtx3/nvToolsExt.h>
#include "kg_launch.h"

using namespace kg;

namespace kg {
int64_t g_launches = 0;
}

namespace {

// ------------------------------------------------------------------ NCCL (world > 1 only)
// NCCL is resolved at run time (dlopen) so that single-GPU use has no NCCL
// dependency and so that the library binds to the NCCL that torch already
// loaded (RTLD_NOLOAD) instead of a second, different copy.
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t *, ncclConfig_t *) = nullptr;   // optional
  ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
};
// ------------------------------------------------------------------ loopback communicator
// Test hook (KG_NCCL=loopback): the NCCL calls of step_dist for ranks that are threads of
// ONE process sharing ONE device (the pool gives one GPU; NCCL refuses two ranks per GPU).
// Every collective is a barrier-synchronised exchange of device buffers with cudaMemcpyAsync
// between the ranks' streams (cross-stream events), reductions in rank order by a kernel --
// the same data movement NCCL performs, so the routing kernels and the protocol of
// step_dist run on the GPU end to end (tests/test_dist_loopback_gpu.py).  Not a transport.
namespace loop {
struct Op {
  bool send;
  const void *sbuf;
  void *rbuf;
  size_t bytes;
  int peer;
};
struct Shared {
  int world = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  int64_t gen = 0;
  std::vector<std::vector<Op>> posts;        // per rank: its sends of the current exchange
  std::vector<cudaEvent_t> ev_ready, ev_done;
  std::vector<std::vector<void *>> ptrs;     // share_ptrs
};
struct Comm {
  Shared *s;
  int rank;
  void *tmp = nullptr;
  size_t tmp_bytes = 0;
};
std::mutex g_reg_mu;
std::vector<std::pair<std::string, Shared *>> g_reg;
thread_local std::vector<std::pair<Comm *, Op>> t_group;
thread_local int t_depth = 0;
thread_local cudaStream_t t_stream = nullptr;
thread_local Comm *t_comm = nullptr;   // the calling rank's communicator (an empty group still joins)

void barrier(Shared *s) {
  std::unique_lock<std::mutex> lk(s->mu);
  const int64_t g = s->gen;
  if (++s->arrived == s->world) {
    s->arrived = 0;
    ++s->gen;
    s->cv.notify_all();
  } else {
    s->cv.wait(lk, [&] { return s->gen != g; });
  }
}

// one exchange: every rank posts its sends, then copies what it receives, then waits for the
// peers' copies out of its buffers before its stream may overwrite them
ncclResult_t exchange(Comm *c, const std::vector<Op> &ops, cudaStream_t st) {
  Shared *s = c->s;
  const int me = c->rank;
  if (cudaEventRecord(s->ev_ready[me], st) != cudaSuccess) return ncclUnhandledCudaError;
  {
    std::lock_guard<std::mutex> lk(s->mu);
    s->posts[me].clear();
    for (auto &o : ops)
      if (o.send) s->posts[me].push_back(o);
  }
  barrier(s);
  std::vector<int> taken(s->world, 0);
  for (auto &o : ops) {
    if (o.send) continue;
    const auto &src = s->posts[o.peer];
    int k = -1, seen = 0;
    for (size_t i = 0; i < src.size(); ++i)
      if (src[i].peer == me && seen++ == taken[o.peer]) { k = (int)i; break; }
    if (k < 0 || src[k].bytes != o.bytes) return ncclInvalidUsage;
    ++taken[o.peer];
    if (cudaStreamWaitEvent(st, s->ev_ready[o.peer], 0) != cudaSuccess ||
        cudaMemcpyAsync(o.rbuf, src[k].sbuf, o.bytes, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      return ncclUnhandledCudaError;
  }
  if (cudaEventRecord(s->ev_done[me], st) != cudaSuccess) return ncclUnhandledCudaError;
  barrier(s);
  for (int p = 0; p < s->world; ++p)
    if (p != me && cudaStreamWaitEvent(st, s->ev_done[p], 0) != cudaSuccess) return ncclUnhandledCudaError;
  barrier(s);
  return ncclSuccess;
}

size_t type_size(ncclDataType_t t) {
  switch (t) {
    case ncclInt8: case ncclUint8: return 1;
    case ncclFloat16: case ncclBfloat16: return 2;
    case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
    default: return 8;
  }
}

ncclResult_t GetUniqueId(ncclUniqueId *id) {
  static std::atomic<uint64_t> ctr{1};
  std::memset(id, 0, sizeof(*id));
  const uint64_t v = ctr++ ^ (uint64_t)std::chrono::steady_clock::now().time_since_epoch().count();
  std::memcpy(id->internal, &v, sizeof(v));
  return ncclSuccess;
}
ncclResult_t CommInitRank(ncclComm_t *comm, int world, ncclUniqueId id, int rank) {
  const std::string key(id.internal, sizeof(id.internal));
  Shared *s = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    for (auto &e : g_reg)
      if (e.first == key) s = e.second;
    if (!s) {
      s = new Shared();
      s->world = world;
      s->posts.resize(world);
      s->ev_ready.resize(world);
      s->ev_done.resize(world);
      for (int r = 0; r < world; ++r)
        if (cudaEventCreateWithFlags(&s->ev_ready[r], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&s->ev_done[r], cudaEventDisableTiming) != cudaSuccess)
          return ncclUnhandledCudaError;
      g_reg.emplace_back(key, s);
    }
  }
  if (s->world != world || rank < 0 || rank >= world) return ncclInvalidArgument;
  Comm *c = new Comm{s, rank};
  t_comm = c;
  *comm = reinterpret_cast<ncclComm_t>(c);
  return ncclSuccess;
}
// a second communicator over the same ranks (its own exchange state), e.g. for a collective on
// another stream; t_comm (the rank's main communicator) is left as it is
ncclResult_t CommSplit(ncclComm_t parent, int color, int key, ncclComm_t *out, ncclConfig_t *) {
  Comm *p = reinterpret_cast<Comm *>(parent);
  char buf[64];
  std::snprintf(buf, sizeof(buf), "split:%p:%d", (void *)p->s, color);
  const std::string k(buf);
  Shared *s = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    for (auto &e : g_reg)
      if (e.first == k) s = e.second;
    if (!s) {
      s = new Shared();
      s->world = p->s->world;
      s->posts.resize(s->world);
      s->ev_ready.resize(s->world);
      s->ev_done.resize(s->world);
      for (int r = 0; r < s->world; ++r)
        if (cudaEventCreateWithFlags(&s->ev_ready[r], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&s->ev_done[r], cudaEventDisableTiming) != cudaSuccess)
          return ncclUnhandledCudaError;
      g_reg.emplace_back(k, s);
    }
  }
  (void)key;
  *out = reinterpret_cast<ncclComm_t>(new Comm{s, p->rank});
  return ncclSuccess;
}
ncclResult_t CommDestroy(ncclComm_t comm) {
  Comm *c = reinterpret_cast<Comm *>(comm);
  if (c->tmp) cudaFree(c->tmp);
  delete c;
  return ncclSuccess;
}
ncclResult_t GroupStart() {
  ++t_depth;
  return ncclSuccess;
}
ncclResult_t GroupEnd() {
  if (--t_depth > 0) return ncclSuccess;
  if (t_group.empty()) return t_comm ? exchange(t_comm, {}, t_stream) : ncclSuccess;
  Comm *c = t_group.front().first;
  std::vector<Op> ops;
  for (auto &e : t_group) ops.push_back(e.second);
  t_group.clear();
  return exchange(c, ops, t_stream);
}
ncclResult_t p2p(bool send, const void *sb, void *rb, size_t count, ncclDataType_t t, int peer, ncclComm_t comm,
                 cudaStream_t st) {
  Comm *c = reinterpret_cast<Comm *>(comm);
  Op o{send, sb, rb, count * type_size(t), peer};
  t_stream = st;
  t_comm = c;
  if (t_depth > 0) {
    t_group.emplace_back(c, o);
    return ncclSuccess;
  }
  return exchange(c, {o}, st);
}
ncclResult_t Send(const void *b, size_t n, ncclDataType_t t, int peer, ncclComm_t comm, cudaStream_t st) {
  return p2p(true, b, nullptr, n, t, peer, comm, st);
}
ncclResult_t Recv(void *b, size_t n, ncclDataType_t t, int peer, ncclComm_t comm, cudaStream_t st) {
  return p2p(false, nullptr, b, n, t, peer, comm, st);
}
ncclResult_t AllGather(const void *sb, void *rb, size_t n, ncclDataType_t t, ncclComm_t comm, cudaStream_t st) {
  Comm *c = reinterpret_cast<Comm *>(comm);
  const size_t bytes = n * type_size(t);
  std::vector<Op> ops;
  for (int p = 0; p < c->s->world; ++p) {
    ops.push_back(Op{true, sb, nullptr, bytes, p});
    ops.push_back(Op{false, nullptr, static_cast<char *>(rb) + p * bytes, bytes, p});
  }
  return exchange(c, ops, st);
}
template <class T, bool MAX>
__global__ void reduce_ranks_kernel(const T *tmp, int world, size_t n, T *out) {
  const size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (e >= n) return;
  T v = tmp[e];
  for (int r = 1; r < world; ++r) v = MAX ? (tmp[r * n + e] > v ? tmp[r * n + e] : v) : v + tmp[r * n + e];
  out[e] = v;
}
ncclResult_t AllReduce(const void *sb, void *rb, size_t n, ncclDataType_t t, ncclRedOp_t op, ncclComm_t comm,
                       cudaStream_t st) {
  Comm *c = reinterpret_cast<Comm *>(comm);
  const int W = c->s->world;
  const size_t bytes = n * type_size(t);
  if (c->tmp_bytes < W * bytes) {   // (world > 1 steps are not graph-captured)
    // stream-ordered: cudaFree / cudaMalloc may synchronise the device, which would wait for a
    // peer rank's spinning p2p barrier kernel (same context here) while that rank waits for us
    if (c->tmp) cudaFreeAsync(c->tmp, st);
    if (cudaMallocAsync(&c->tmp, W * bytes, st) != cudaSuccess) return ncclSystemError;
    c->tmp_bytes = W * bytes;
  }
  ncclResult_t r = AllGather(sb, c->tmp, n, t, comm, st);   // every rank's input, in rank order
  if (r != ncclSuccess) return r;
  const int g = (int)((n + 255) / 256);
  if (op != ncclSum && op != ncclMax) return ncclInvalidArgument;
  const bool mx = op == ncclMax;
  switch (t) {
    case ncclFloat32:
      if (mx) reduce_ranks_kernel<float, true><<<g, 256, 0, st>>>((const float *)c->tmp, W, n, (float *)rb);
      else reduce_ranks_kernel<float, false><<<g, 256, 0, st>>>((const float *)c->tmp, W, n, (float *)rb);
      break;
    case ncclFloat64:
      if (mx) reduce_ranks_kernel<double, true><<<g, 256, 0, st>>>((const double *)c->tmp, W, n, (double *)rb);
      else reduce_ranks_kernel<double, false><<<g, 256, 0, st>>>((const double *)c->tmp, W, n, (double *)rb);
      break;
    case ncclInt32:
      if (mx) reduce_ranks_kernel<int, true><<<g, 256, 0, st>>>((const int *)c->tmp, W, n, (int *)rb);
      else reduce_ranks_kernel<int, false><<<g, 256, 0, st>>>((const int *)c->tmp, W, n, (int *)rb);
      break;
    default:
      return ncclInvalidArgument;
  }
  return cudaGetLastError() == cudaSuccess ? ncclSuccess : ncclUnhandledCudaError;
}
const char *GetErrorString(ncclResult_t) { return "loopback communicator error"; }
// host all-gather of the ranks' buffer addresses (the peer-memory exchange's "mapping" when the
// ranks are threads of one process on one device)
std::vector<void *> share_ptrs(ncclComm_t comm, const std::vector<void *> &mine) {
  Comm *c = reinterpret_cast<Comm *>(comm);
  Shared *s = c->s;
  {
    std::lock_guard<std::mutex> lk(s->mu);
    s->ptrs.resize(s->world);
    s->ptrs[c->rank] = mine;
  }
  barrier(s);
  std::vector<void *> all;
  for (int r = 0; r < s->world; ++r) all.insert(all.end(), s->ptrs[r].begin(), s->ptrs[r].end());
  barrier(s);
  return all;
}
}  // namespace loop
bool loopback_nccl() {
  const char *e = std::getenv("KG_NCCL");
  return e && std::string(e) == "loopback";
}

NcclApi load_nccl() {
  NcclApi api;
  if (const char *e = std::getenv("KG_NCCL")) {
    if (std::string(e) == "loopback") {
      api.GetUniqueId = loop::GetUniqueId;
      api.CommInitRank = loop::CommInitRank;
      api.CommDestroy = loop::CommDestroy;
      api.CommSplit = loop::CommSplit;
      api.AllGather = loop::AllGather;
      api.AllReduce = loop::AllReduce;
      api.Send = loop::Send;
      api.Recv = loop::Recv;
      api.GroupStart = loop::GroupStart;
      api.GroupEnd = loop::GroupEnd;
      api.GetErrorString = loop::GetErrorString;
      api.ok = true;
      return api;
    }
  }
  void *lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
#ifdef KG_NCCL_PATH
  if (!lib) lib = dlopen(KG_NCCL_PATH, RTLD_NOW | RTLD_GLOBAL);
#endif
  if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!lib) return api;
  bool all = true;
  auto get = [&](auto &fp, const char *name) {
    fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(lib, name));
    all = all && fp;
  };
  get(api.GetUniqueId, "ncclGetUniqueId");
  get(api.CommInitRank, "ncclCommInitRank");
  get(api.CommDestroy, "ncclCommDestroy");
  get(api.AllGather, "ncclAllGather");
  get(api.AllReduce, "ncclAllReduce");
  get(api.Send, "ncclSend");
  get(api.Recv, "ncclRecv");
  get(api.GroupStart, "ncclGroupStart");
  get(api.GroupEnd, "ncclGroupEnd");
  get(api.GetErrorString, "ncclGetErrorString");
  api.ok = all;
  api.CommSplit = reinterpret_cast<decltype(api.CommSplit)>(dlsym(lib, "ncclCommSplit"));   // NCCL >= 2.18
  return api;
}
// resolved once, thread-safely (function-local static): the ranks of the loopback test are
// threads that create their handles concurrently
const NcclApi &nccl() {
  static const NcclApi api = load_nccl();
  return api;
}

// ------------------------------------------------------------------ plans
struct PNode {
  int type;       // 0 projection, 1 intersection, 2 negation (input = `in`)
  int in;         // projection input node (-1: anchor slot)
  int anchor;     // anchor slot (when in == -1)
  int rel;        // relation slot (execution order, A21)
  int ins[3];
  int nin;
};
struct Plan {
  int gs[6], ge[6];   // projection group [gs, ge) of each projection node
  int na, nr, nn, nout, nproj;
  PNode n[6];
  int outs[2];
  int inter;      // index of the intersection node or -1
};

PNode P(int in, int anchor, int rel) { return PNode{0, in, anchor, rel, {0, 0, 0}, 0}; }
PNode I2(int a, int b) { return PNode{1, -1, -1, -1, {a, b, 0}, 2}; }
PNode I3(int a, int b, int c) { return PNode{1, -1, -1, -1, {a, b, c}, 3}; }
PNode Ng(int in) { return PNode{2, in, -1, -1, {0, 0, 0}, 0}; }

Plan make_plan(int s) {
  Plan p{};
  p.inter = -1;
  auto set = [&](std::initializer_list<PNode> nodes, std::initializer_list<int> outs, int na, int nr) {
    p.nn = 0;
    for (auto &x : nodes) p.n[p.nn++] = x;
    p.nout = 0;
    for (int o : outs) p.outs[p.nout++] = o;
    p.na = na;
    p.nr = nr;
  };
  switch (s) {
    case KG_1P: set({P(-1, 0, 0)}, {0}, 1, 1); break;
    case KG_2P: set({P(-1, 0, 0), P(0, -1, 1)}, {1}, 1, 2); break;
    case KG_3P: set({P(-1, 0, 0), P(0, -1, 1), P(1, -1, 2)}, {2}, 1, 3); break;
    case KG_2I: set({P(-1, 0, 0), P(-1, 1, 1), I2(0, 1)}, {2}, 2, 2); break;
    case KG_3I: set({P(-1, 0, 0), P(-1, 1, 1), P(-1, 2, 2), I3(0, 1, 2)}, {3}, 3, 3); break;
    case KG_IP: set({P(-1, 0, 0), P(-1, 1, 1), I2(0, 1), P(2, -1, 2)}, {3}, 2, 3); break;
    // projections of the same depth are consecutive nodes (one batched MLP for BetaE)
    case KG_PI: set({P(-1, 0, 0), P(-1, 1, 2), P(0, -1, 1), I2(2, 1)}, {3}, 2, 3); break;
    case KG_2U: set({P(-1, 0, 0), P(-1, 1, 1)}, {0, 1}, 2, 2); break;
    case KG_UP: set({P(-1, 0, 0), P(-1, 1, 1), P(0, -1, 2), P(1, -1, 2)}, {2, 3}, 2, 3); break;
    case KG_2IN: set({P(-1, 0, 0), P(-1, 1, 1), Ng(1), I2(0, 2)}, {3}, 2, 2); break;
    case KG_3IN: set({P(-1, 0, 0), P(-1, 1, 1), P(-1, 2, 2), Ng(2), I3(0, 1, 3)}, {4}, 3, 3); break;
    case KG_INP: set({P(-1, 0, 0), P(-1, 1, 1), Ng(1), I2(0, 2), P(3, -1, 2)}, {4}, 2, 3); break;
    case KG_PIN: set({P(-1, 0, 0), P(-1, 1, 2), P(0, -1, 1), Ng(1), I2(2, 3)}, {4}, 2, 3); break;
    case KG_PNI: set({P(-1, 0, 0), P(-1, 1, 2), P(0, -1, 1), Ng(2), I2(3, 1)}, {4}, 2, 3); break;
  }
  // groups of consecutive, mutually independent projection nodes [gs, ge)
  for (int i = 0; i < p.nn;) {
    if (p.n[i].type != 0) { ++i; continue; }
    int j = i + 1;
    while (j < p.nn && p.n[j].type == 0 && p.n[j].in < i) ++j;
    for (int k = i; k < j; ++k) { p.gs[k] = i; p.ge[k] = j; }
    i = j;
  }
  p.nproj = 0;
  for (int i = 0; i < p.nn; ++i) {
    if (p.n[i].type == 0) p.nproj++;
    else if (p.n[i].type == 1) p.inter = i;
  }
  return p;
}

int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

struct Seg {
  std::string name;
  int64_t off, n;
  int rows, cols;
  float lo, hi;
};

struct Arena {
  char *base = nullptr;
  size_t off = 0;
  template <class T>
  T *take(int64_t n) {
    off = (size_t)align_up((int64_t)off, 256);
    T *p = base ? reinterpret_cast<T *>(base + off) : nullptr;
    off += (size_t)std::max<int64_t>(n, 1) * sizeof(T);
    return p;
  }
};

}  // namespace

struct kg_handle {
  kg_config cfg{};
  std::string err;
  bool broken = false, bound = false;
  int kind = 0, d = 0, m = 0, H = 0, R = 0, world = 1, rank = 0;
  int sk = 0;            // projection / scoring kind: the base model of an -m variant (A27), else kind
  int qnorm = 0;         // query normalisation after projection / intersection: 0 none, 1 L2, 2 Re and Im (A27)
  bool deepset = false;  // GQE DeepSet intersection (GQE and the -m variants)
  int64_t n_ent = 0, shard = 0;
  int dq = 0, dr = 0, ent_bits = 1, rel_bits = 1;
  std::vector<Seg> segs;
  int64_t dense_size = 0, w_off = 0;
  kg_tables t{};
  cudaStream_t st = nullptr;
  int device = 0;

  // workspace
  char *ws = nullptr;
  size_t ws_bytes = 0;
  int Mx = 0, Kx = 0, Cx = 0, Lx = 0, Lrx = 0, Kpx = 0;
  int64_t *b_anchors = nullptr, *b_answers = nullptr, *b_negs = nullptr;
  int32_t *b_rels = nullptr;
  uint32_t *b_mask = nullptr;
  int64_t *ids = nullptr, *rows = nullptr, *uniq = nullptr;
  int32_t *inv = nullptr, *perm = nullptr, *seg = nullptr, *Udev = nullptr, *bad = nullptr;
  int32_t *rocc = nullptr, *rinv = nullptr, *rperm = nullptr, *rseg = nullptr, *rU = nullptr;
  int64_t *runiq = nullptr;
  int32_t *rel_seg_map = nullptr;
  int64_t *rel_stamp = nullptr;
  float *OG = nullptr, *RG = nullptr, *RGU = nullptr, *Gc = nullptr, *gdense = nullptr, *PS = nullptr, *PSr = nullptr;
  int32_t *pcnt = nullptr, *ocnt = nullptr, *sinv = nullptr, *osinv = nullptr, *hrow = nullptr,
          *ohrow = nullptr;
  // pre-split weight planes of the MLP weights used as GEMM B operands (refreshed at the start of
  // every DAG forward, on a side stream): lo (W's layout), t = W^T, tlo = lo^T
  struct WPlanes { std::string name; float *lo = nullptr, *t = nullptr, *tlo = nullptr; };
  std::vector<WPlanes> wpl;
  cudaEvent_t ev_wsplit = nullptr, ev_wsplit_t = nullptr;   // lo planes / transposed planes refreshed
  bool wsplit_issued = false;                               // this step's transposed planes are on their way
  float *Q = nullptr, *dQ = nullptr, *C = nullptr, *Dmin = nullptr, *Dpos = nullptr, *loss_part = nullptr,
        *loss_pos = nullptr;
  float *F = nullptr, *Cv = nullptr, *QP = nullptr, *Cq = nullptr;
  double *loss_dev = nullptr;
  int *flags = nullptr;
  int64_t *t_dev = nullptr;
  float *bc = nullptr;
  float *nval[6] = {}, *ngrad[6] = {};
  float *stack_v = nullptr, *stack_g = nullptr;
  float *qn = nullptr;   // [6 nodes][Mx][2] norms of the -m query normalisation
  int host_tier = 0;     // bit i: theta_E table i (ent, ent_m, ent_v) is pinned host memory
  float *T[12] = {};
  int8_t *amin = nullptr;
  float *pXT = nullptr, *pH1T = nullptr, *pH2T = nullptr;   // BetaE MLP inputs transposed ([cols][rows]) for dW
  cudaEvent_t ev_xt = nullptr;
  float *pX = nullptr, *pH1 = nullptr, *pH2 = nullptr, *pZp1 = nullptr, *pdZ = nullptr, *pdH2 = nullptr,
        *pdH1 = nullptr, *pZ = nullptr, *pdX = nullptr;
  float *Dscore = nullptr;
  float *gsP = nullptr, *gsP2 = nullptr, *gsP3 = nullptr;   // GEMM split-K scratch (st / st3 / st5)
  int64_t gsP_cap = 0;
  float *Dpart = nullptr, *partQ = nullptr, *partV = nullptr, *Cpart = nullptr, *Csum = nullptr;
  float *Eg = nullptr;     // dot-product scorers: the pool's rows, contiguous (GEMM operand)
  bool score_bf16 = false;  // kg_config.score_precision == KG_SCORE_BF16
  bool gemm_lowp = false;   // the GEMMs being enqueued take bf16-rounded operands (scoring, bf16 mode)
  int64_t cap_D = 0, cap_Q = 0, cap_V = 0;
  cudaStream_t st2 = nullptr, st_cap = nullptr, st3 = nullptr, st4 = nullptr;
  // st5: the DAG backward's weight gradients (dW = dY^T X, bias column sums) -- they feed only the
  // dense Adam, so they run beside the dX chain; w_used: st5 joined the step, ev_wjoin its end
  cudaStream_t st5 = nullptr;
  cudaEvent_t ev_wjoin = nullptr, ev_bent = nullptr;   // ev_bent: BetaE pool features done (st3)
  bool w_used = false;
  cudaEvent_t ev_rel = nullptr, ev_loss = nullptr, ev_early = nullptr;
  cudaEvent_t ev_i1 = nullptr, ev_i2 = nullptr;   // fork / join of the two Q2B intersection branches
  cudaEvent_t ev_fork = nullptr, ev_fork2 = nullptr, ev_join = nullptr;
  float *lr_dev = nullptr;
  int64_t *stamp_dev = nullptr;
  struct GraphEntry {
    int structure, M, K, flags, kernels, gemms, pdl_edges;
    cudaGraphExec_t exec;
  };
  std::vector<GraphEntry> graphs;
  bool use_graphs = true;
  bool gemm_drain = true, use_pdl = true;
  int side = 0;   // the stream the GEMMs are enqueued on: 0 st, 1 st3, 2 st5 (split-K scratch)
  // row-sharded exchange (world > 1, k_dist.cu)
  ncclComm_t comm = nullptr;
  ncclComm_t comm2 = nullptr;  // world > 1: the dense all-reduce's own communicator (on st2, overlapped)
  const float *ent_src = nullptr;       // rows read by the step: theta_E (world 1) or the received rows
  float *gfull = nullptr;               // dense dL/dtheta_D [dense_size] (weights part = gdense)
  int64_t *send_ids = nullptr, *recv_ids = nullptr, *recv_keys = nullptr, *ouniq = nullptr;
  int cap = 0;             // bucket capacity per owner (ids) of the fixed-capacity exchange
  bool buckets = true;     // fixed-capacity exchange (no host round trip); KG_DIST_BUCKETS=0: exact counts
  bool p2p = false;        // KG_XCHG=p2p: row exchange over peer memory (one-sided), no NCCL for rows
  PeerPtrs *pp = nullptr;  // device copy of the mapped peer addresses (workspace)
  unsigned long long *p2p_flags = nullptr, *p2p_epoch = nullptr;   // barrier flags [kMaxWorld], epoch
  std::vector<void *> ipc_opened;   // peer allocations mapped with cudaIpcOpenMemHandle
  bool dist_graph = true;  // capture world > 1 steps (NCCL only); KG_DIST_GRAPH=0: eager
  int32_t *send_pos = nullptr, *counts = nullptr, *all_counts = nullptr, *oinv = nullptr, *operm = nullptr,
          *oseg = nullptr, *oU = nullptr;
  float *Xin = nullptr, *send_rows = nullptr, *Gsend = nullptr, *Grecv = nullptr, *PSo = nullptr;
  int32_t *h_counts = nullptr;           // pinned [G*G]
  int flag_key() const { return apply | (keep_grads << 1) | (timing << 2); }

  // pinned staging (double-buffered) + host mirrors of the step results
  char *pin[2] = {nullptr, nullptr};
  size_t pin_bytes = 0;
  cudaEvent_t pin_ev[2] = {nullptr, nullptr};
  int pin_cur = 0;
  struct HostOut {       // = the device result block (loss, flags, U, t at 0 / 8 / 16 / 24)
    double loss;
    int flags[2];
    int32_t U;
    int64_t t;
  } *hout = nullptr;      // [2]: two steps' results may be in flight (pipelined host loop)
  char *resdev = nullptr;
  cudaEvent_t step_done = nullptr, res_ev[2] = {nullptr, nullptr};
  int res_next = 0, res_pending = 0;             // ring of the two result slots
  int res_kernels[2] = {0, 0}, res_gemms[2] = {0, 0};

  int64_t stamp = 0;
  int apply = 1, keep_grads = 0, timing = 0;
  cudaEvent_t sev[12] = {};
  bool side_timed = false;
  int64_t launches0 = 0;
  int last_kernels = 0, last_gemms = 0, gemm_count = 0;
  int last_M = 0, last_K = 0, last_U_valid = 0;
  bool step_pending = false;
};

namespace {

kg_status fail(kg_handle *h, kg_status s, const std::string &msg) {
  if (h) {
    h->err = msg;
    if (s == KG_ECUDA || s == KG_ENCCL) h->broken = true;
  }
  return s;
}

#define CK(call)                                                                               \
  do {                                                                                         \
    cudaError_t e_ = (call);                                                                   \
    if (e_ != cudaSuccess)                                                                     \
      return fail(h, KG_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));            \
  } while (0)
#define NCK(call)                                                                                \
  do {                                                                                           \
    ncclResult_t r_ = (call);                                                                    \
    if (r_ != ncclSuccess) return fail(h, KG_ENCCL, std::string(#call) + ": " + nccl().GetErrorString(r_)); \
  } while (0)
bool single_hop(int k) { return k == KG_TRANSE || k == KG_ROTATE || k == KG_DISTMULT || k == KG_COMPLEX; }
int base_kind(int k) {
  return k == KG_ROTATE_M ? KG_ROTATE : (k == KG_DISTMULT_M ? KG_DISTMULT : (k == KG_COMPLEX_M ? KG_COMPLEX : k));
}
int bits_for(int64_t n) {
  int b = 1;
  while (b < 31 && ((int64_t)1 << b) < n) ++b;
  return b;
}

// theta_D layout -- identical to kggen.dense_layout.
void build_layout(kg_handle *h) {
  const int d = h->d, R = h->R, H = h->H, m = h->m;
  const double rho = ((double)h->cfg.gamma + 2.0) / (double)d;
  const double w = 1.0 / std::sqrt((double)d);
  auto add = [&](const char *name, int rows, int cols, double lo, double hi) {
    Seg s{name, 0, (int64_t)rows * cols, rows, cols, (float)lo, (float)hi};
    h->segs.push_back(s);
  };
  const int k = h->sk;   // an -m variant keeps its base model's relation table (A27)
  if (k == KG_GQE || k == KG_TRANSE || k == KG_DISTMULT || k == KG_COMPLEX) add("rel", R, d, -rho, rho);
  else if (k == KG_Q2B) { add("rel_center", R, d, -rho, rho); add("rel_offset", R, d, 0.0, rho); }
  else if (k == KG_BETAE) add("rel", R, d, -rho, rho);
  else if (k == KG_ROTATE) add("rel_phase", R, m, -M_PI, M_PI);
  const size_t nrel = h->segs.size();
  if (h->deepset) {
    add("ds_W1", d, d, -w, w); add("ds_b1", 1, d, -w, w); add("ds_W2", d, d, -w, w); add("ds_b2", 1, d, -w, w);
  } else if (k == KG_Q2B) {
    add("att_W1", d, d, -w, w); add("att_b1", 1, d, -w, w); add("att_W2", d, d, -w, w); add("att_b2", 1, d, -w, w);
    add("off_W1", d, d, -w, w); add("off_b1", 1, d, -w, w); add("off_W2", d, d, -w, w); add("off_b2", 1, d, -w, w);
  } else if (k == KG_BETAE) {
    const double w1 = 1.0 / std::sqrt(2.0 * d), wh = 1.0 / std::sqrt((double)H);
    add("prj_W1", H, 2 * d, -w1, w1); add("prj_b1", 1, H, -w1, w1);
    add("prj_W2", H, H, -wh, wh); add("prj_b2", 1, H, -wh, wh);
    add("prj_W0", d, H, -wh, wh); add("prj_b0", 1, d, -wh, wh);
    add("att_U1", d, d, -w, w); add("att_c1", 1, d, -w, w); add("att_U2", m, d, -w, w); add("att_c2", 1, m, -w, w);
  }
  int64_t off = 0;
  for (size_t i = 0; i < h->segs.size(); ++i) {
    h->segs[i].off = off;
    off += h->segs[i].n;
    if (i + 1 == nrel) h->w_off = off;
  }
  h->dense_size = off;
}

const Seg *seg_of(const kg_handle *h, const char *name) {
  for (auto &s : h->segs)
    if (s.name == name) return &s;
  return nullptr;
}
float *dp(kg_handle *h, const char *name) { return h->t.dense + seg_of(h, name)->off; }
const kg_handle::WPlanes *wplanes(const kg_handle *h, const char *name) {
  for (auto &w : h->wpl)
    if (w.name == name) return &w;
  return nullptr;
}
// forward operand: B = W [out][in] (K-major) with its lo plane
const float *wlo(const kg_handle *h, const char *name) { const auto *w = wplanes(h, name); return w ? w->lo : nullptr; }
// backward operand of dX = dY W: W^T [in][out] (K-major, ld = out) and its lo plane
const float *wt(const kg_handle *h, const char *name) { return wplanes(h, name)->t; }
const float *wtlo(const kg_handle *h, const char *name) { return wplanes(h, name)->tlo; }
float *gp(kg_handle *h, const char *name) { return h->gdense + (seg_of(h, name)->off - h->w_off); }

void carve(kg_handle *h, Arena &A) {
  const int Mx = h->Mx, Kx = h->Kx, d = h->d, dq = h->dq, H = h->H;
  const int NQ = 2 * Mx;
  h->b_anchors = A.take<int64_t>(3 * Mx);
  h->b_rels = A.take<int32_t>(3 * Mx);
  h->b_answers = A.take<int64_t>(Mx);
  h->b_negs = A.take<int64_t>(std::max(Kx, h->Cx));
  h->b_mask = A.take<uint32_t>((int64_t)Mx * ((Kx + 31) / 32));
  h->ids = A.take<int64_t>(h->Lx);
  h->rows = A.take<int64_t>(h->Lx);
  h->uniq = A.take<int64_t>(h->Lx);
  h->inv = A.take<int32_t>(h->Lx);
  h->perm = A.take<int32_t>(h->Lx);
  h->sinv = A.take<int32_t>(h->Lx);
  h->hrow = A.take<int32_t>(h->Lx);
  h->seg = A.take<int32_t>(h->Lx + 1);
  {
    // the step's scalar results, contiguous so that one D2H copies them (layout = HostOut)
    char *res = reinterpret_cast<char *>(A.take<int64_t>(4));
    h->resdev = res;
    h->loss_dev = reinterpret_cast<double *>(res);
    h->flags = reinterpret_cast<int *>(res + 8);
    h->Udev = reinterpret_cast<int32_t *>(res + 16);
    h->t_dev = reinterpret_cast<int64_t *>(res + 24);
  }
  h->bad = A.take<int32_t>(1);
  h->rocc = A.take<int32_t>(h->Lrx);
  h->runiq = A.take<int64_t>(h->Lrx);
  h->rinv = A.take<int32_t>(h->Lrx);
  h->rperm = A.take<int32_t>(h->Lrx);
  h->rseg = A.take<int32_t>(h->Lrx + 1);
  h->rU = A.take<int32_t>(1);
  h->rel_seg_map = A.take<int32_t>(h->R);
  h->rel_stamp = A.take<int64_t>(h->R);
  h->RG = A.take<float>((int64_t)h->Lrx * h->dr);
  h->RGU = A.take<float>((int64_t)h->Lrx * h->dr);
  h->OG = A.take<float>((int64_t)h->Lx * d);
  h->Gc = A.take<float>((int64_t)h->Lx * d);
  h->PS = A.take<float>((int64_t)h->Lx * d);
  h->pcnt = A.take<int32_t>((int64_t)h->Lx * 16);   // piece arrival counters of the fused sparse Adam (self-resetting)
  h->PSr = A.take<float>((int64_t)h->Lrx * h->dr);
  h->gfull = A.take<float>(h->dense_size);
  h->gdense = h->gfull + h->w_off;
  h->Q = A.take<float>((int64_t)NQ * dq);
  h->dQ = A.take<float>((int64_t)NQ * dq);
  h->C = A.take<float>((int64_t)NQ * h->Kpx);
  h->Dmin = A.take<float>((int64_t)Mx * Kx);
  h->Dpos = A.take<float>(Mx);
  h->loss_part = A.take<float>(Mx);
  {
    const int64_t KK = std::max(h->Kpx, (int)align_up(std::max(h->Cx, 1), 4));
    const int64_t one = 2LL * Mx * KK;
    int64_t ks = std::max<int64_t>(1, std::min<int64_t>(8, (64LL << 20) / std::max<int64_t>(one, 1)));
    h->cap_D = one * ks;
    h->cap_Q = 2LL * Mx * dq * std::max<int64_t>(1, (std::max(Kx, h->Cx) + 63) / 64);   // one dQ partial per >= 64 pool entries
    h->cap_V = (int64_t)std::max(Kx, h->Cx) * d * 8;
    h->Dpart = A.take<float>(h->cap_D);
    h->partQ = A.take<float>(h->cap_Q);
    h->partV = A.take<float>(h->cap_V);
    h->Cpart = A.take<float>(8LL * std::max(Kx, h->Cx));
    h->Csum = A.take<float>(NQ);
    if (h->sk == KG_DISTMULT || h->sk == KG_COMPLEX) h->Eg = A.take<float>((int64_t)Kx * d);   // pool rows, gathered
  }
  h->loss_pos = A.take<float>(Mx);
  if (h->kind == KG_BETAE) {
    h->F = A.take<float>((int64_t)std::max(Kx, h->Cx) * 9 * h->m);
    h->Cv = A.take<float>(std::max(Kx, h->Cx));
    h->QP = A.take<float>((int64_t)NQ * d);
    h->Cq = A.take<float>(NQ);
  }
  h->lr_dev = A.take<float>(4);
  h->stamp_dev = A.take<int64_t>(1);
  h->bc = A.take<float>(2);
  for (int i = 0; i < 6; ++i) {
    h->nval[i] = A.take<float>((int64_t)Mx * dq);
    h->ngrad[i] = A.take<float>((int64_t)Mx * dq);
  }
  h->qn = A.take<float>((int64_t)6 * 2 * Mx);   // per-node query norms (A27)
  if (!single_hop(h->kind)) {
    h->stack_v = A.take<float>((int64_t)3 * Mx * dq);
    h->stack_g = A.take<float>((int64_t)3 * Mx * dq);
    for (int i = 0; i < 12; ++i) h->T[i] = A.take<float>((int64_t)3 * Mx * d);
    h->amin = A.take<int8_t>((int64_t)Mx * d);
  }
  if (h->kind == KG_BETAE) {
    const int64_t P = 4 * (int64_t)Mx;
    h->pX = A.take<float>(P * 2 * d);
    h->pH1 = A.take<float>(P * H);
    h->pH2 = A.take<float>(P * H);
    h->pXT = A.take<float>(align_up(P, 4) * 2 * d);
    h->pH1T = A.take<float>(align_up(P, 4) * H);
    h->pH2T = A.take<float>(align_up(P, 4) * H);
    h->pZp1 = A.take<float>(P * d);
    h->pdZ = A.take<float>(P * d);
    h->pdH2 = A.take<float>(P * H);
    h->pdH1 = A.take<float>(P * H);
    h->pZ = A.take<float>(P * d);
    h->pdX = A.take<float>(P * 2 * d);
  }
  h->Dscore = A.take<float>((int64_t)Mx * std::max(h->Cx, 1));
  {
    const int64_t wide = std::max<int64_t>({(int64_t)H, 2LL * d, (int64_t)dq});
    const int64_t tall = std::max<int64_t>({4LL * Mx, (int64_t)H, 2LL * d});
    h->gsP_cap = std::min<int64_t>(16LL << 20, 8LL * 4 * Mx * wide);
    h->gsP = A.take<float>(h->gsP_cap);
    h->gsP2 = A.take<float>(h->gsP_cap);
    h->gsP3 = A.take<float>(h->gsP_cap);
  }
  {
    static const char *kWNames[] = {"prj_W1", "prj_W2", "prj_W0", "ds_W1", "ds_W2", "off_W1", "off_W2",
                                    "att_W1", "att_W2", "att_U1", "att_U2"};
    h->wpl.clear();
    for (const char *n : kWNames) {
      const Seg *sg = seg_of(h, n);
      if (!sg) continue;
      kg_handle::WPlanes w;
      w.name = n;
      w.lo = A.take<float>(sg->n);
      w.t = A.take<float>(sg->n);
      w.tlo = A.take<float>(sg->n);
      h->wpl.push_back(w);
    }
  }
  if (h->world > 1) {
    const int64_t GL = (int64_t)h->world * h->Lx;
    // fixed-capacity exchange buckets: twice the mean share of distinct ids per
    // owner + 256, at most all of them
    h->cap = (int)std::min<int64_t>(h->Lx, 2 * ((h->Lx + h->world - 1) / h->world) + 256);
    const int64_t SL = std::max<int64_t>(h->Lx, (int64_t)h->world * h->cap);
    h->send_ids = A.take<int64_t>(SL);
    h->send_pos = A.take<int32_t>(h->Lx);
    h->counts = A.take<int32_t>(kMaxWorld);
    h->all_counts = A.take<int32_t>(kMaxWorld * kMaxWorld);
    h->recv_ids = A.take<int64_t>(GL);
    h->recv_keys = A.take<int64_t>(GL);
    h->ouniq = A.take<int64_t>(GL);
    h->oinv = A.take<int32_t>(GL);
    h->operm = A.take<int32_t>(GL);
    h->osinv = A.take<int32_t>(GL);
    h->ohrow = A.take<int32_t>(GL);
    h->oseg = A.take<int32_t>(GL + 1);
    h->oU = A.take<int32_t>(1);
    h->Xin = A.take<float>(SL * d);
    h->send_rows = A.take<float>(GL * d);
    h->Gsend = A.take<float>(SL * d);
    h->Grecv = A.take<float>(GL * d);
    h->PSo = A.take<float>(GL * d);
    h->ocnt = A.take<int32_t>(GL * 16);
    h->pp = reinterpret_cast<PeerPtrs *>(A.take<char>(sizeof(PeerPtrs)));
    h->p2p_flags = A.take<unsigned long long>(kMaxWorld + 1);
    h->p2p_epoch = h->p2p_flags ? h->p2p_flags + kMaxWorld : nullptr;
  }
}

// Row-major GEMM: C[m x n] = op(A) op(B) + beta C, op(A) is [m x k]; tb: B given as [n x k].
// Every contraction of the DAG runs on the tcgen05 3xTF32 kernel (k_gemm.cu; drained
// accumulation, see kg_create); the side stream has its own split-K scratch.
kg_status gemm(kg_handle *h, bool ta, bool tb, int m, int n, int k, const float *A, int lda, const float *B, int ldb,
               float beta, float *C, int ldc, const float *bias = nullptr, int relu = 0, float alpha = 1.f,
               const float *B_lo = nullptr, bool tb_t = false, const float *mask = nullptr) {
  if (m <= 0 || n <= 0) return KG_OK;
  // the tensor-core kernel reads either operand layout directly ([k][m] / [k][n] = MN-major)
  GemmArgs g;
  g.A = A; g.B = B; g.C = C; g.M = m; g.N = n; g.K = k; g.lda = lda; g.ldb = ldb; g.ldc = ldc; g.beta = beta;
  g.bias = bias; g.relu = relu; g.a_mn = ta; g.b_mn = !tb; g.drain = h->gemm_drain && !h->gemm_lowp;
  g.lowp = h->gemm_lowp;
  g.alpha = alpha;
  if (B_lo) CK(cudaStreamWaitEvent(h->st, tb_t ? h->ev_wsplit_t : h->ev_wsplit, 0));   // this step's planes (st3)
  g.B_lo = B_lo;
  g.mask = mask;
  float *scr = h->side == 2 ? h->gsP3 : h->side == 1 ? h->gsP2 : h->gsP;
  if (k <= 0 || !launch_gemm_tc(g, scr, h->gsP_cap, h->st))
    return fail(h, KG_EUNSUPPORTED, "tensor-core GEMM: operands must be 16-byte aligned with ld % 4 == 0 and K > 0 "
                                    "(and cuTensorMapEncodeTiled available)");
  h->gemm_count++;
  return KG_OK;
}
// Y = X W^T (X [m][k] with ld lda, W [n][k]) as raw split-K partial products in the stream's
// split-K scratch (*P, [splits][m][n]); returns the split count, 0 on failure.  The consumer
// kernel (k_dag.cu *_red) sums the splits, adds the bias and pools (fused epilogue).
int gemm_raw(kg_handle *h, int m, int n, int k, const float *A, int lda, const float *B, int ldb, const float **P) {
  GemmArgs g;
  g.A = A; g.B = B; g.M = m; g.N = n; g.K = k; g.lda = lda; g.ldb = ldb; g.ldc = n;
  g.drain = h->gemm_drain && !h->gemm_lowp;
  float *scr = h->side == 2 ? h->gsP3 : h->side == 1 ? h->gsP2 : h->gsP;
  const int s = launch_gemm_tc_raw(g, scr, h->gsP_cap, h->st);
  if (s > 0) h->gemm_count++;
  *P = scr;
  return s;
}
#define GR(var, ...)                                                                           \
  do {                                                                                         \
    var = gemm_raw(h, __VA_ARGS__);                                                            \
    if (var <= 0) return fail(h, KG_EUNSUPPORTED, "tensor-core GEMM (raw partials) not launched"); \
  } while (0)
// Run the following GEMMs / kernels on another stream (restored on scope exit).
// The side stream gets its own cuBLAS handle (own workspace) and its own tensor-core GEMM
// split-K scratch, so the two branches cannot race on scratch memory.
struct OnStream {
  kg_handle *h;
  cudaStream_t prev;
  int prev_side;
  OnStream(kg_handle *hh, cudaStream_t s, int which = 1) : h(hh), prev(hh->st), prev_side(hh->side) {
    h->st = s;
    h->side = which;
  }
  ~OnStream() {
    h->st = prev;
    h->side = prev_side;
  }
};
// Programmatic dependent launch inside the step graph: every edge between two of this
// library's kernels (they all begin with griddepcontrol.wait, KG_GRID_DEP_WAIT) becomes a
// programmatic edge, so the downstream grid is launched as the upstream one drains instead of
// after it has completed; the wait keeps the data dependence.  Edges touching kernels of
// other modules (cuBLAS, NCCL) and event nodes are kept as they are.
bool ours(cudaGraphNode_t n) {
  cudaGraphNodeType t;
  if (cudaGraphNodeGetType(n, &t) != cudaSuccess || t != cudaGraphNodeTypeKernel) return false;
  cudaKernelNodeParams kp;
  if (cudaGraphKernelNodeGetParams(n, &kp) != cudaSuccess || !kp.func) { cudaGetLastError(); return false; }
  Dl_info info;
  return dladdr(kp.func, &info) && info.dli_fname && std::strstr(info.dli_fname, "libkg") != nullptr;
}
int make_programmatic(cudaGraph_t g) {
  size_t n = 0;
  if (cudaGraphGetEdges_v2(g, nullptr, nullptr, nullptr, &n) != cudaSuccess || n == 0) return 0;
  std::vector<cudaGraphNode_t> from(n), to(n);
  std::vector<cudaGraphEdgeData> ed(n);
  if (cudaGraphGetEdges_v2(g, from.data(), to.data(), ed.data(), &n) != cudaSuccess) return 0;
  int converted = 0;
  for (size_t i = 0; i < n; ++i) {
    if (ed[i].type != cudaGraphDependencyTypeDefault || ed[i].from_port != 0) continue;
    if (!ours(from[i]) || !ours(to[i])) continue;   // library kernels on both ends (not cuBLAS / NCCL)
    if (cudaGraphRemoveDependencies_v2(g, &from[i], &to[i], &ed[i], 1) != cudaSuccess) { cudaGetLastError(); continue; }
    cudaGraphEdgeData e{};
    e.from_port = cudaGraphKernelNodePortProgrammatic;
    e.type = cudaGraphDependencyTypeProgrammatic;
    if (cudaGraphAddDependencies_v2(g, &from[i], &to[i], &e, 1) != cudaSuccess) {
      cudaGetLastError();
      cudaGraphAddDependencies_v2(g, &from[i], &to[i], &ed[i], 1);   // restore the plain edge
      continue;
    }
    ++converted;
  }
  return converted;
}

// the lowest stream priority (the early dense-Adam stream yields the SMs to the scoring kernels)
int kLowPriority() {
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  return lo;
}
kg_status fork(kg_handle *h, cudaStream_t from, cudaStream_t to) {
  CK(cudaEventRecord(h->ev_i1, from));
  CK(cudaStreamWaitEvent(to, h->ev_i1, 0));
  return KG_OK;
}
kg_status join(kg_handle *h, cudaStream_t from, cudaStream_t to) {
  CK(cudaEventRecord(h->ev_i2, from));
  CK(cudaStreamWaitEvent(to, h->ev_i2, 0));
  return KG_OK;
}

// Weight gradients on st5 (off the dX chain): wfork(from) makes st5 wait for everything enqueued
// on `from` so far; the GEMMs enqueued inside a WOn scope go to st5 with its own split-K scratch.
kg_status wfork(kg_handle *h, cudaStream_t from) {
  h->w_used = true;
  return fork(h, from, h->st5);
}
struct WOn : OnStream {
  explicit WOn(kg_handle *hh) : OnStream(hh, hh->st5, 2) {}
};
// end of the DAG backward's st5 work: the stream that runs the dense Adam waits for ev_wjoin
kg_status wjoin(kg_handle *h, cudaStream_t to) {
  if (!h->w_used) return KG_OK;
  h->w_used = false;
  CK(cudaEventRecord(h->ev_wjoin, h->st5));
  CK(cudaStreamWaitEvent(to, h->ev_wjoin, 0));
  return KG_OK;
}

#define G(...)                                   \
  do {                                           \
    kg_status s_ = gemm(h, __VA_ARGS__);         \
    if (s_ != KG_OK) return s_;                  \
  } while (0)
#define WF(from)                                 \
  do {                                           \
    kg_status s_ = wfork(h, from);               \
    if (s_ != KG_OK) return s_;                  \
  } while (0)

struct StepBufs {
  Plan plan;
  int M, K, Kp, NQ;
  float *val[6], *grad[6];
};

// -------------------------------------------------------------- forward DAG
// The transposed pre-split planes of the MLP weights (W^T and its lo plane, the K-major B
// operand of the backward's dX = dY W): one launch per step, issued where it interferes least --
// at the start of a local step on the low-priority stream (st4, concurrent with the gathers and
// the DAG forward), else on st3 at the start of the DAG backward.  The dX GEMMs wait ev_wsplit_t.
bool needs_wplanes(const kg_handle *h, const Plan &p) { return !h->wpl.empty() && (h->kind == KG_BETAE || p.inter >= 0); }
kg_status issue_wplanes(kg_handle *h, cudaStream_t from, cudaStream_t on) {
  WSplitJobs J;
  for (auto &w : h->wpl) {
    const Seg *sg = seg_of(h, w.name.c_str());
    J.j[J.n++] = WSplitJob{h->t.dense + sg->off, w.lo, w.t, w.tlo, sg->rows, sg->cols};
  }
  kg_status fs = fork(h, from, on);
  if (fs) return fs;
  launch_wsplit(J, 1, on);
  CK(cudaEventRecord(h->ev_wsplit_t, on));
  h->wsplit_issued = true;
  return KG_OK;
}

kg_status dag_forward(kg_handle *h, StepBufs &S) {
  const Plan &p = S.plan;
  const int M = S.M, d = h->d, dq = h->dq, m = h->m, HH = h->H;
  cudaStream_t st = h->st;
  const float *ent = h->ent_src;
  int u = 0;
  for (int ni = 0; ni < p.nn; ++ni) {
    const PNode &nd = p.n[ni];
    if (nd.type == 0 && h->kind == KG_BETAE) {
      // one MLP over the rows of all projections of the group (same weights, A9)
      const int nj = p.ge[ni], GM = (nj - ni) * M;
      float *X = h->pX + (int64_t)u * M * 2 * d, *H1 = h->pH1 + (int64_t)u * M * HH, *H2 = h->pH2 + (int64_t)u * M * HH;
      for (int k = ni; k < nj; ++k) {
        const PNode &nk = p.n[k];
        const int64_t *arows = nk.in < 0 ? h->rows + (int64_t)nk.anchor * M : nullptr;
        launch_betae_proj_in(M, d, nk.in < 0 ? nullptr : S.val[nk.in], arows, ent, h->rocc + (int64_t)(u + k - ni) * M,
                             1, dp(h, "rel"), X + (int64_t)(k - ni) * M * 2 * d, st);
      }
      G(false, true, GM, HH, 2 * d, X, 2 * d, dp(h, "prj_W1"), 2 * d, 0.f, H1, HH, dp(h, "prj_b1"), 1);
      G(false, true, GM, HH, HH, H1, HH, dp(h, "prj_W2"), HH, 0.f, H2, HH, dp(h, "prj_b2"), 1);
      {
        const float *P = nullptr;
        int sp = 0;
        GR(sp, GM, d, HH, H2, HH, dp(h, "prj_W0"), HH, &P);   // Z, its epilogue fused below
        OutPtrs op{};
        for (int k = ni; k < nj; ++k) op.p[k - ni] = S.val[k];
        launch_betae_proj_out_red(P, sp, dp(h, "prj_b0"), GM, M, d, h->pZp1 + (int64_t)u * M * d, op, st);
      }
      u += nj - ni;
      ni = nj - 1;
      continue;
    }
    if (nd.type == 0) {
      const int64_t *arows = nd.in < 0 ? h->rows + (int64_t)nd.anchor * M : nullptr;
      const float *in = nd.in < 0 ? nullptr : S.val[nd.in];
      const int32_t *rel = h->rocc + (int64_t)u * M;
      {
        const float *relA = nullptr, *relB = nullptr;
        if (h->kind == KG_Q2B) { relA = dp(h, "rel_center"); relB = dp(h, "rel_offset"); }
        else if (h->sk == KG_ROTATE) relA = dp(h, "rel_phase");
        else relA = dp(h, "rel");
        launch_proj_fwd(h->sk, M, d, in, dq, arows, ent, rel, 1, relA, relB, S.val[ni], st);
        if (h->qnorm) launch_qnorm_fwd(S.val[ni], M, d, h->qnorm, h->qn + (int64_t)ni * 2 * h->Mx, st);   // A27
      }
      ++u;
    } else if (nd.type == 2) {
      launch_neg_fwd(S.val[nd.in], (int64_t)M * d, S.val[ni], st);   // N(q) = 1/q (Table 1)
    } else {
      const int n = nd.nin, NR = n * M;
      float *out = S.val[ni];
      float **T = h->T;
      const float *P = nullptr;
      int sp = 0;
      if (h->deepset) {
        GR(sp, NR, d, d, h->stack_v, d, dp(h, "ds_W1"), d, &P);
        launch_mean_red(P, sp, dp(h, "ds_b1"), n, M, d, T[0], T[1], st);              // H, Mn
        G(false, true, M, d, d, T[1], d, dp(h, "ds_W2"), d, 0.f, out, d, dp(h, "ds_b2"), 0);
        if (h->qnorm) launch_qnorm_fwd(out, M, d, h->qnorm, h->qn + (int64_t)ni * 2 * h->Mx, st);   // A27
      } else if (h->kind == KG_Q2B) {
        // the center-attention and offset-DeepSet branches are independent: second stream
        kg_status fs = fork(h, st, h->st3);
        if (fs) return fs;
        {
          OnStream os(h, h->st3);
          const float *P3 = nullptr;
          int sp3 = 0;
          GR(sp3, NR, d, d, h->stack_v + d, 2 * d, dp(h, "off_W1"), d, &P3);
          launch_mean_red(P3, sp3, dp(h, "off_b1"), n, M, d, T[3], T[4], h->st3);                  // Ho, Mo
          GR(sp3, M, d, d, T[4], d, dp(h, "off_W2"), d, &P3);
          launch_q2b_off_red(P3, sp3, dp(h, "off_b2"), h->stack_v, n, M, d, T[6], h->amin, out, h->st3);  // sig, amin, offset
        }
        G(false, true, NR, d, d, h->stack_v, 2 * d, dp(h, "att_W1"), d, 0.f, T[0], d, dp(h, "att_b1"), 1);  // Hc
        GR(sp, NR, d, d, T[0], d, dp(h, "att_W2"), d, &P);
        launch_q2b_att_red(P, sp, dp(h, "att_b2"), h->stack_v, n, M, d, T[2], out, st);        // a, center
        if ((fs = join(h, h->st3, st)) != KG_OK) return fs;
      } else if (h->kind == KG_BETAE) {
        G(false, true, NR, d, d, h->stack_v, d, dp(h, "att_U1"), d, 0.f, T[0], d, dp(h, "att_c1"), 1);     // Hs
        GR(sp, NR, m, d, T[0], d, dp(h, "att_U2"), d, &P);
        launch_beta_att_red(P, sp, dp(h, "att_c2"), h->stack_v, n, M, d, T[2], out, st);      // w, out
      }
    }
  }
  if (h->kind == KG_BETAE && p.nproj > 0) {
    // the MLP layers' inputs transposed ([cols][rows], ld = rows rounded up to 4) for the weight
    // gradients dW = dY^T X of the backward: K-major B operands instead of MN-major ones the
    // GEMM's split warps would transpose; on the low-priority stream, during the scoring
    const int NR = p.nproj * M, ldT = (int)align_up(NR, 4);
    kg_status fs = fork(h, st, h->st4);
    if (fs) return fs;
    launch_transpose(h->pX, NR, 2 * d, 2 * d, h->pXT, ldT, h->st4);
    launch_transpose(h->pH1, NR, HH, HH, h->pH1T, ldT, h->st4);
    launch_transpose(h->pH2, NR, HH, HH, h->pH2T, ldT, h->st4);
    CK(cudaEventRecord(h->ev_xt, h->st4));
  }
  return KG_OK;
}

// -------------------------------------------------------------- backward DAG
kg_status dag_backward(kg_handle *h, StepBufs &S, bool defer_wjoin = false) {
  const Plan &p = S.plan;
  if (needs_wplanes(h, p) && !h->wsplit_issued) {
    kg_status ws = issue_wplanes(h, h->st, h->st3);
    if (ws) return ws;
  }
  h->wsplit_issued = false;   // consumed by this backward (the next step issues its own)
  const int M = S.M, d = h->d, dq = h->dq, m = h->m, HH = h->H;
  cudaStream_t st = h->st;
  const float *ent = h->ent_src;
  // projection-use index of each node
  int use[6], u = 0;
  for (int ni = 0; ni < p.nn; ++ni) use[ni] = p.n[ni].type == 0 ? u++ : -1;
  // (BetaE's projection-MLP weight gradients issued group by group on st5, beside the dX chain of
  // the earlier groups, measured slower: C5-betae 3p 0.709 -> 0.810 ms -- the concurrent GEMMs
  // slow the chain more than they overlap; they run once after it, over all groups)
  for (int ni = p.nn - 1; ni >= 0; --ni) {
    const PNode &nd = p.n[ni];
    if (nd.type == 0 && h->kind == KG_BETAE) {
      // the group [gs, ge) ends here: its output gradients are complete (consumers come later)
      const int n0 = p.gs[ni], u0 = use[n0], GM = (ni + 1 - n0) * M;
      float *dZ = h->pdZ + (int64_t)u0 * M * d, *dH2 = h->pdH2 + (int64_t)u0 * M * HH,
            *dH1 = h->pdH1 + (int64_t)u0 * M * HH;
      for (int k = n0; k <= ni; ++k)
        launch_betae_proj_dz(S.grad[k], h->pZp1 + (int64_t)use[k] * M * d, M, d, h->pdZ + (int64_t)use[k] * M * d, st);
      G(false, true, GM, HH, d, dZ, d, wt(h, "prj_W0"), d, 0.f, dH2, HH, nullptr, 0, 1.f, wtlo(h, "prj_W0"), true,
        h->pH2 + (int64_t)u0 * M * HH);   // ReLU backward folded into the GEMM's combine
      G(false, true, GM, HH, HH, dH2, HH, wt(h, "prj_W2"), HH, 0.f, dH1, HH, nullptr, 0, 1.f, wtlo(h, "prj_W2"), true,
        h->pH1 + (int64_t)u0 * M * HH);
      G(false, true, GM, 2 * d, HH, dH1, HH, wt(h, "prj_W1"), HH, 0.f, h->pdX, 2 * d, nullptr, 0, 1.f, wtlo(h, "prj_W1"), true);
      for (int k = n0; k <= ni; ++k) {
        const PNode &nk = p.n[k];
        const int64_t *arows = nk.in < 0 ? h->rows + (int64_t)nk.anchor * M : nullptr;
        float *din = nk.in < 0 ? h->OG + (int64_t)nk.anchor * M * d : S.grad[nk.in];
        launch_betae_split(h->pdX + (int64_t)(k - n0) * M * 2 * d, M, d, arows, ent, din, nk.in < 0 ? d : dq,
                           h->RG + (int64_t)use[k] * M * h->dr, st);
      }
      ni = n0;   // the loop's --ni moves past the group
      continue;
    }
    if (nd.type == 0) {
      const int uu = use[ni];
      const int64_t *arows = nd.in < 0 ? h->rows + (int64_t)nd.anchor * M : nullptr;
      const float *in = nd.in < 0 ? nullptr : S.val[nd.in];
      float *din = nd.in < 0 ? h->OG + (int64_t)nd.anchor * M * d : S.grad[nd.in];
      const int64_t din_ld = nd.in < 0 ? d : dq;
      const int32_t *rel = h->rocc + (int64_t)uu * M;
      float *drel = h->RG + (int64_t)uu * M * h->dr;
      {
        const float *relA = nullptr, *relB = nullptr;
        if (h->kind == KG_Q2B) { relA = dp(h, "rel_center"); relB = dp(h, "rel_offset"); }
        else if (h->sk == KG_ROTATE) relA = dp(h, "rel_phase");
        else relA = dp(h, "rel");
        if (h->qnorm) launch_qnorm_bwd(S.grad[ni], S.val[ni], M, d, h->qnorm, h->qn + (int64_t)ni * 2 * h->Mx, st);
        launch_proj_bwd(h->sk, M, d, S.grad[ni], in, dq, arows, ent, rel, 1, relA, relB, S.val[ni], din, din_ld,
                        drel, st);
      }
    } else if (nd.type == 2) {
      launch_neg_bwd(S.grad[ni], S.val[nd.in], (int64_t)M * d, S.grad[nd.in], st);   // d(1/x) = -dx / x^2
    } else {
      const int n = nd.nin, NR = n * M;
      const float *gout = S.grad[ni];
      float **T = h->T;
      if (h->deepset) {
        // T0 = H, T1 = Mn (forward);  T7 = dMn, T8 = dH
        if (h->qnorm) launch_qnorm_bwd(S.grad[ni], S.val[ni], M, d, h->qnorm, h->qn + (int64_t)ni * 2 * h->Mx, st);
        WF(st);
        { WOn w(h); G(true, false, d, d, M, gout, d, T[1], d, 0.f, gp(h, "ds_W2"), d); }
        G(false, true, M, d, d, gout, d, wt(h, "ds_W2"), d, 0.f, T[7], d, nullptr, 0, 1.f, wtlo(h, "ds_W2"), true);
        launch_gqe_inter_dh(T[7], T[0], n, M, d, T[8], st);
        WF(st);
        {
          WOn w(h);
          G(true, false, d, d, NR, T[8], d, h->stack_v, d, 0.f, gp(h, "ds_W1"), d);
          ColsumJobs cj;
          cj.add(gout, M, d, d, gp(h, "ds_b2"));
          cj.add(T[8], NR, d, d, gp(h, "ds_b1"));
          launch_colsum_multi(cj, h->st5);
        }
        G(false, true, NR, d, d, T[8], d, wt(h, "ds_W1"), d, 0.f, h->stack_g, d, nullptr, 0, 1.f, wtlo(h, "ds_W1"), true);
      } else if (h->kind == KG_Q2B) {
        // forward: T0 Hc, T1 Lg, T2 a, T3 Ho, T4 Mo, T5 Z, T6 sig.  backward: T7 dLg, T8 dHc, T9 dZ, T10 dMo, T11 dHo
        // offset branch on the second stream (writes the offset half of stack_g only)
        kg_status fs = fork(h, st, h->st3);
        if (fs) return fs;
        {
          OnStream os(h, h->st3);
          cudaStream_t s3 = h->st3;
          launch_q2b_off_bwd(h->stack_v, T[6], h->amin, gout, n, M, d, T[9], h->stack_g, s3);
          WF(s3);
          { WOn w(h); G(true, false, d, d, M, T[9], d, T[4], d, 0.f, gp(h, "off_W2"), d); }
          G(false, true, M, d, d, T[9], d, wt(h, "off_W2"), d, 0.f, T[10], d, nullptr, 0, 1.f, wtlo(h, "off_W2"), true);
          launch_gqe_inter_dh(T[10], T[3], n, M, d, T[11], s3);
          WF(s3);
          { WOn w(h); G(true, false, d, d, NR, T[11], d, h->stack_v + d, 2 * d, 0.f, gp(h, "off_W1"), d); }
          G(false, true, NR, d, d, T[11], d, wt(h, "off_W1"), d, 1.f, h->stack_g + d, 2 * d, nullptr, 0, 1.f, wtlo(h, "off_W1"), true);
        }
        launch_q2b_att_bwd(h->stack_v, T[2], gout, n, M, d, T[7], h->stack_g, st);
        WF(st);
        { WOn w(h); G(true, false, d, d, NR, T[7], d, T[0], d, 0.f, gp(h, "att_W2"), d); }
        G(false, true, NR, d, d, T[7], d, wt(h, "att_W2"), d, 0.f, T[8], d, nullptr, 0, 1.f, wtlo(h, "att_W2"), true,
          T[0]);
        WF(st);
        {
          // st5 already waits for the offset branch's dZ / dHo (forked from st3 above, enqueued first)
          WOn w(h);
          G(true, false, d, d, NR, T[8], d, h->stack_v, 2 * d, 0.f, gp(h, "att_W1"), d);
          ColsumJobs cj;
          cj.add(T[7], NR, d, d, gp(h, "att_b2"));
          cj.add(T[8], NR, d, d, gp(h, "att_b1"));
          cj.add(T[9], M, d, d, gp(h, "off_b2"));
          cj.add(T[11], NR, d, d, gp(h, "off_b1"));
          launch_colsum_multi(cj, h->st5);
        }
        G(false, true, NR, d, d, T[8], d, wt(h, "att_W1"), d, 1.f, h->stack_g, 2 * d, nullptr, 0, 1.f, wtlo(h, "att_W1"), true);
        if ((fs = join(h, h->st3, st)) != KG_OK) return fs;
      } else if (h->kind == KG_BETAE) {
        // forward: T0 Hs, T1 Lg, T2 w.  backward: T7 dLg, T8 dHs
        launch_beta_att_bwd(h->stack_v, T[2], gout, n, M, d, T[7], h->stack_g, st);
        WF(st);
        { WOn w(h); G(true, false, m, d, NR, T[7], m, T[0], d, 0.f, gp(h, "att_U2"), d); }
        G(false, true, NR, d, m, T[7], m, wt(h, "att_U2"), m, 0.f, T[8], d, nullptr, 0, 1.f, wtlo(h, "att_U2"), true,
          T[0]);
        WF(st);
        {
          WOn w(h);
          G(true, false, d, d, NR, T[8], d, h->stack_v, d, 0.f, gp(h, "att_U1"), d);
          ColsumJobs cj;
          cj.add(T[7], NR, m, m, gp(h, "att_c2"));
          cj.add(T[8], NR, d, d, gp(h, "att_c1"));
          launch_colsum_multi(cj, h->st5);
        }
        G(false, true, NR, d, d, T[8], d, wt(h, "att_U1"), d, 1.f, h->stack_g, d, nullptr, 0, 1.f, wtlo(h, "att_U1"), true);
      }
    }
  }
  if (h->kind == KG_BETAE) {
    // projection-MLP weight gradients over all projection uses at once (A9)
    const int NR = p.nproj * M, ldT = (int)align_up(NR, 4);
    WF(st);
    WOn w(h);
    CK(cudaStreamWaitEvent(h->st5, h->ev_xt, 0));   // the transposed inputs (DAG forward, st4)
    G(true, true, d, HH, NR, h->pdZ, d, h->pH2T, ldT, 0.f, gp(h, "prj_W0"), HH);
    G(true, true, HH, HH, NR, h->pdH2, HH, h->pH1T, ldT, 0.f, gp(h, "prj_W2"), HH);
    G(true, true, HH, 2 * d, NR, h->pdH1, HH, h->pXT, ldT, 0.f, gp(h, "prj_W1"), 2 * d);
    ColsumJobs cj;
    cj.add(h->pdZ, NR, d, d, gp(h, "prj_b0"));
    cj.add(h->pdH2, NR, HH, HH, gp(h, "prj_b2"));
    cj.add(h->pdH1, NR, HH, HH, gp(h, "prj_b1"));
    launch_colsum_multi(cj, h->st5);
  }
  // the weight gradients on st5 join `st` here, or (defer_wjoin) the caller joins them into
  // the stream of the dense Adam (wjoin)
  if (!defer_wjoin) return wjoin(h, st);
  return KG_OK;
}

// Assign node value / gradient buffers for the current M (outputs -> Q / dQ slices,
// intersection inputs -> stack slices).
void assign_buffers(kg_handle *h, StepBufs &S) {
  const Plan &p = S.plan;
  const int64_t Md = (int64_t)S.M * h->dq;
  for (int ni = 0; ni < p.nn; ++ni) { S.val[ni] = h->nval[ni]; S.grad[ni] = h->ngrad[ni]; }
  if (p.inter >= 0)
    for (int k = 0; k < p.n[p.inter].nin; ++k) {
      S.val[p.n[p.inter].ins[k]] = h->stack_v + k * Md;
      S.grad[p.n[p.inter].ins[k]] = h->stack_g + k * Md;
    }
  for (int t = 0; t < p.nout; ++t) { S.val[p.outs[t]] = h->Q + t * Md; S.grad[p.outs[t]] = h->dQ + t * Md; }
}

kg_status check_state(kg_handle *h) {
  if (!h) return KG_EINVAL;
  if (h->broken) return fail(h, KG_ESTATE, "handle is in an error state: " + h->err);
  if (!h->bound) return fail(h, KG_ESTATE, "kg_bind has not been called");
  return KG_OK;
}

// Validate a batch and stage host inputs into the workspace (H2D on the bound stream).
kg_status ingest(kg_handle *h, const kg_batch *b, bool train, const Plan &plan, float lr = 0.f) {
  const int M = b->M, K = train ? b->K : 0, na = plan.na, nr = plan.nr;
  const int W = (K + 31) / 32;
  if (M < 1 || M > h->Mx) return fail(h, KG_EINVAL, "M out of range [1, max_M]");
  if (K < 0 || K > h->Kx) return fail(h, KG_EINVAL, "K out of range [0, max_K]");
  if (!b->anchors || !b->relations) return fail(h, KG_EINVAL, "null anchors / relations");
  if (train && (!b->answers || (K > 0 && (!b->negatives || !b->mask))))
    return fail(h, KG_EINVAL, "null answers / negatives / mask");
  const size_t sz_a = (size_t)M * na * 8, sz_r = (size_t)M * nr * 4, sz_ans = train ? (size_t)M * 8 : 0,
               sz_n = (size_t)K * 8, sz_m = (size_t)M * W * 4;
  if (b->on_device) {
    if (train) {   // step scalars (lr, stamp) through the pinned staging buffer
      const int cur = h->pin_cur;
      h->pin_cur ^= 1;
      CK(cudaEventSynchronize(h->pin_ev[cur]));
      char *p = h->pin[cur];
      std::memcpy(p, &lr, sizeof(float));
      std::memcpy(p + 8, &h->stamp, sizeof(int64_t));
      CK(cudaMemcpyAsync(h->lr_dev, p, sizeof(float), cudaMemcpyHostToDevice, h->st));
      CK(cudaMemcpyAsync(h->stamp_dev, p + 8, sizeof(int64_t), cudaMemcpyHostToDevice, h->st));
      CK(cudaEventRecord(h->pin_ev[cur], h->st));
    }
    CK(cudaMemcpyAsync(h->b_anchors, b->anchors, sz_a, cudaMemcpyDeviceToDevice, h->st));
    CK(cudaMemcpyAsync(h->b_rels, b->relations, sz_r, cudaMemcpyDeviceToDevice, h->st));
    if (train) {
      CK(cudaMemcpyAsync(h->b_answers, b->answers, sz_ans, cudaMemcpyDeviceToDevice, h->st));
      if (K > 0) {
        CK(cudaMemcpyAsync(h->b_negs, b->negatives, sz_n, cudaMemcpyDeviceToDevice, h->st));
        CK(cudaMemcpyAsync(h->b_mask, b->mask, sz_m, cudaMemcpyDeviceToDevice, h->st));
      }
    }
    return KG_OK;
  }
  // host inputs: validate here (EINVAL before anything is enqueued)
  for (int64_t i = 0; i < (int64_t)M * na; ++i)
    if (b->anchors[i] < 0 || b->anchors[i] >= h->n_ent) return fail(h, KG_EINVAL, "anchor id out of range");
  for (int64_t i = 0; i < (int64_t)M * nr; ++i)
    if (b->relations[i] < 0 || b->relations[i] >= h->R) return fail(h, KG_EINVAL, "relation id out of range");
  if (train) {
    for (int i = 0; i < M; ++i)
      if (b->answers[i] < 0 || b->answers[i] >= h->n_ent) return fail(h, KG_EINVAL, "answer id out of range");
    for (int j = 0; j < K; ++j)
      if (b->negatives[j] < 0 || b->negatives[j] >= h->n_ent) return fail(h, KG_EINVAL, "negative id out of range");
  }
  const size_t total = sz_a + sz_r + sz_ans + sz_n + sz_m + 7 * 256;
  if (total > h->pin_bytes) return fail(h, KG_EINVAL, "batch exceeds staging capacity");
  const int cur = h->pin_cur;
  h->pin_cur ^= 1;
  CK(cudaEventSynchronize(h->pin_ev[cur]));   // the H2D that last read this buffer has finished
  char *p = h->pin[cur];
  size_t off = 0;
  auto put = [&](const void *src, size_t n, void *dst) -> kg_status {
    if (!n) return KG_OK;
    std::memcpy(p + off, src, n);
    CK(cudaMemcpyAsync(dst, p + off, n, cudaMemcpyHostToDevice, h->st));
    off = (size_t)align_up((int64_t)(off + n), 256);
    return KG_OK;
  };
  kg_status s;
  if (train) {
    if ((s = put(&lr, sizeof(float), h->lr_dev)) != KG_OK) return s;
    if ((s = put(&h->stamp, sizeof(int64_t), h->stamp_dev)) != KG_OK) return s;
  }
  if ((s = put(b->anchors, sz_a, h->b_anchors)) != KG_OK) return s;
  if ((s = put(b->relations, sz_r, h->b_rels)) != KG_OK) return s;
  if (train) {
    if ((s = put(b->answers, sz_ans, h->b_answers)) != KG_OK) return s;
    if ((s = put(b->negatives, sz_n, h->b_negs)) != KG_OK) return s;
    if ((s = put(b->mask, sz_m, h->b_mask)) != KG_OK) return s;
  }
  CK(cudaEventRecord(h->pin_ev[cur], h->st));
  return KG_OK;
}

void mark(kg_handle *h, int i, cudaStream_t s = nullptr) {
  if (!h->timing) return;
  // external: inside a stream capture this becomes an event-record node of the graph; outside a
  // capture (world > 1, KG_NO_GRAPH) the flag is not allowed and a plain record is used
  cudaStream_t st = s ? s : h->st;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  if (cs == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(h->sev[i], st, cudaEventRecordExternal);
  else cudaEventRecord(h->sev[i], st);
}

// Result of the step in ring slot `slot` (waits for it); stage times are those of the last
// step issued (stage timing is meant for synchronous steps).
kg_status read_result(kg_handle *h, kg_step_info *info, int slot) {
  CK(cudaEventSynchronize(h->res_ev[slot]));
  const kg_handle::HostOut &o = h->hout[slot];
  if (info) {
    info->loss = o.loss;
    info->n_touched = o.U;
    info->step = o.t;
    info->kernels = h->res_kernels[slot];
    info->gemms = h->res_gemms[slot];
    for (int i = 0; i < 10; ++i) info->stage_ms[i] = 0.f;
    if (h->timing) {
      for (int i = 0; i < 7; ++i) CK(cudaEventElapsedTime(&info->stage_ms[i], h->sev[i], h->sev[i + 1]));
      CK(cudaEventElapsedTime(&info->stage_ms[7], h->sev[0], h->sev[7]));
      if (h->side_timed) {
        CK(cudaEventElapsedTime(&info->stage_ms[8], h->sev[8], h->sev[9]));
        if (h->apply) CK(cudaEventElapsedTime(&info->stage_ms[9], h->sev[10], h->sev[11]));
      }
    }
  }
  if (o.flags[1] == 3)
    return fail(h, KG_ESTATE, "peer-memory exchange: a rank did not reach the step barrier within 20 s (theta_E "
                              "not updated; a dense update already under way may have run; handle unusable)");
  if (o.flags[1] == 2)
    return fail(h, KG_EINVAL, "row exchange bucket overflow (the batch's distinct ids concentrate on one owner beyond "
                              "the fixed capacity); step not applied -- KG_DIST_BUCKETS=0 exchanges exact counts");
  if (o.flags[1]) return fail(h, KG_EINVAL, "an id or relation of the (device) batch was out of range; step not applied");
  if (o.flags[0]) return fail(h, KG_ENONFINITE, "non-finite loss; step not applied");
  return KG_OK;
}
// the latest step (drains every pending result)
kg_status read_latest(kg_handle *h, kg_step_info *info) {
  const int slot = (h->res_next + 1) & 1;      // the slot written last
  h->res_pending = 0;
  h->step_pending = false;
  return read_result(h, info, slot);
}

}  // namespace

namespace {
// KG_XCHG=p2p (collective, at kg_bind): every rank's theta_E shard, receive buckets and barrier
// flags mapped into every rank -- CUDA IPC handles all-gathered over NCCL (the shard's handle
// is that of its allocation, plus the offset; the workspace has the same layout on every rank),
// or the plain addresses for the in-process loopback ranks.
kg_status map_peers(kg_handle *h) {
  const int G = h->world, me = h->rank;
  PeerPtrs hp{};
  if (loopback_nccl()) {
    const std::vector<void *> all = loop::share_ptrs(h->comm, {h->t.ent, h->recv_ids, h->Grecv, h->p2p_flags});
    for (int o = 0; o < G; ++o) {
      hp.ent[o] = static_cast<const float *>(all[4 * o]);
      hp.rids[o] = static_cast<int64_t *>(all[4 * o + 1]);
      hp.grecv[o] = static_cast<float *>(all[4 * o + 2]);
      hp.flags[o] = static_cast<unsigned long long *>(all[4 * o + 3]);
    }
  } else {
    struct Rec {
      cudaIpcMemHandle_t ent, ws;
      int64_t ent_off;
    } rec{};
    using AddrRange = CUresult (*)(CUdeviceptr *, size_t *, CUdeviceptr);
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return fail(h, KG_EUNSUPPORTED, "KG_XCHG=p2p: cuMemGetAddressRange unavailable");
    CUdeviceptr base = 0;
    size_t bytes = 0;
    if (reinterpret_cast<AddrRange>(fn)(&base, &bytes, (CUdeviceptr)h->t.ent) != CUDA_SUCCESS)
      return fail(h, KG_EUNSUPPORTED, "KG_XCHG=p2p: theta_E allocation not found");
    rec.ent_off = (int64_t)((CUdeviceptr)h->t.ent - base);
    if (cudaIpcGetMemHandle(&rec.ent, (void *)base) != cudaSuccess || cudaIpcGetMemHandle(&rec.ws, h->ws) != cudaSuccess) {
      cudaGetLastError();
      return fail(h, KG_EUNSUPPORTED, "KG_XCHG=p2p: no IPC handle for theta_E / the workspace (e.g. a VMM allocation)");
    }
    char *d = nullptr;
    CK(cudaMalloc(&d, sizeof(Rec) * (G + 1)));
    CK(cudaMemcpy(d, &rec, sizeof(Rec), cudaMemcpyHostToDevice));
    NCK(nccl().AllGather(d, d + sizeof(Rec), sizeof(Rec), ncclInt8, h->comm, h->st));
    std::vector<Rec> all(G);
    CK(cudaMemcpyAsync(all.data(), d + sizeof(Rec), sizeof(Rec) * G, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    cudaFree(d);
    const char *wsb = static_cast<const char *>(h->ws);
    for (int o = 0; o < G; ++o) {
      char *ent_base = nullptr, *ws_o = nullptr;
      if (o == me) {
        ent_base = reinterpret_cast<char *>(base);
        ws_o = static_cast<char *>(h->ws);
      } else {
        if (cudaIpcOpenMemHandle(reinterpret_cast<void **>(&ent_base), all[o].ent, cudaIpcMemLazyEnablePeerAccess) !=
                cudaSuccess ||
            cudaIpcOpenMemHandle(reinterpret_cast<void **>(&ws_o), all[o].ws, cudaIpcMemLazyEnablePeerAccess) !=
                cudaSuccess) {
          cudaGetLastError();
          return fail(h, KG_EUNSUPPORTED, "KG_XCHG=p2p: cudaIpcOpenMemHandle failed (peers not on one node?)");
        }
        h->ipc_opened.push_back(ent_base);
        h->ipc_opened.push_back(ws_o);
      }
      hp.ent[o] = reinterpret_cast<const float *>(ent_base + all[o].ent_off);
      hp.rids[o] = reinterpret_cast<int64_t *>(ws_o + (reinterpret_cast<const char *>(h->recv_ids) - wsb));
      hp.grecv[o] = reinterpret_cast<float *>(ws_o + (reinterpret_cast<const char *>(h->Grecv) - wsb));
      hp.flags[o] = reinterpret_cast<unsigned long long *>(ws_o + (reinterpret_cast<const char *>(h->p2p_flags) - wsb));
    }
  }
  CK(cudaMemcpy(h->pp, &hp, sizeof(hp), cudaMemcpyHostToDevice));
  return KG_OK;
}
}  // namespace

// ====================================================================== ABI
extern "C" {

kg_status kg_create(const kg_config *cfg, kg_handle **out) {
  if (!cfg || !out) return KG_EINVAL;
  *out = nullptr;
  const kg_config &c = *cfg;
  if (c.kind < KG_GQE || c.kind > KG_COMPLEX_M) return KG_EINVAL;
  if (c.dim < 8 || c.dim > 2048 || c.dim % 8) return KG_EINVAL;
  if (c.n_entities < 1 || c.n_entities >= ((int64_t)1 << 31) || c.n_relations < 1) return KG_EINVAL;
  if (c.kind == KG_BETAE && (c.hidden < 8 || c.hidden % 8)) return KG_EINVAL;
  if (c.max_M < 1 || c.max_K < 0 || c.max_cand < 0) return KG_EINVAL;
  if (c.world < 1 || c.rank < 0 || c.rank >= c.world) return KG_EINVAL;
  if (!(c.gamma == c.gamma) || !(c.beta1 >= 0.0 && c.beta1 < 1.0) || !(c.beta2 >= 0.0 && c.beta2 < 1.0) ||
      !(c.eps > 0.0))
    return KG_EINVAL;
  const int Lx = 3 * c.max_M + c.max_M + std::max(c.max_K, c.max_cand);
  if (Lx > dedup_capacity()) return KG_EINVAL;
  if (c.world > kMaxWorld || (c.world > 1 && !c.nccl_id)) return KG_EINVAL;
  if ((int64_t)c.world * Lx > dedup_capacity()) return KG_EINVAL;
  if (c.score_precision != KG_SCORE_FP32 && c.score_precision != KG_SCORE_BF16) return KG_EINVAL;
  if (c.score_precision == KG_SCORE_BF16 && base_kind(c.kind) != KG_DISTMULT && base_kind(c.kind) != KG_COMPLEX)
    return KG_EUNSUPPORTED;   // bf16 scoring only for the dot-product scorers

  kg_handle *h = new kg_handle();
  h->cfg = c;
  h->kind = c.kind; h->d = c.dim; h->m = c.dim / 2; h->R = c.n_relations; h->n_ent = c.n_entities;
  h->sk = base_kind(c.kind);
  h->qnorm = c.kind == KG_DISTMULT_M ? 1 : (c.kind == KG_COMPLEX_M ? 2 : 0);
  h->deepset = c.kind == KG_GQE || c.kind >= KG_ROTATE_M;
  h->H = c.kind == KG_BETAE ? c.hidden : 0;
  h->world = c.world; h->rank = c.rank;
  h->shard = (c.n_entities + c.world - 1) / c.world;
  h->dq = c.kind == KG_Q2B ? 2 * c.dim : c.dim;
  h->dr = c.kind == KG_Q2B ? 2 * c.dim : (h->sk == KG_ROTATE ? c.dim / 2 : c.dim);
  h->ent_bits = bits_for(c.n_entities);
  h->rel_bits = bits_for(c.n_relations);
  h->Mx = c.max_M; h->Kx = std::max(c.max_K, 1); h->Cx = c.max_cand;
  h->Lx = Lx; h->Lrx = 4 * c.max_M; h->Kpx = (int)align_up(std::max(c.max_K, 1), 64);
  build_layout(h);

  if (cudaGetDevice(&h->device) != cudaSuccess) { delete h; return KG_ECUDA; }
  Arena A;
  carve(h, A);
  h->ws_bytes = A.off;
  if (cudaMalloc(&h->ws, h->ws_bytes) != cudaSuccess) { delete h; return KG_ENOMEM; }
  A = Arena{h->ws, 0};
  carve(h, A);
  const int W = (h->Kx + 31) / 32;
  h->pin_bytes = (size_t)h->Mx * 3 * 8 + (size_t)h->Mx * 3 * 4 + (size_t)h->Mx * 8 + (size_t)h->Kx * 8 +
                 (size_t)h->Mx * W * 4 + 8 * 256;
  for (int i = 0; i < 2; ++i) {
    if (cudaMallocHost(&h->pin[i], h->pin_bytes) != cudaSuccess) { kg_destroy(h); return KG_ENOMEM; }
    if (cudaEventCreateWithFlags(&h->pin_ev[i], cudaEventDisableTiming) != cudaSuccess) { kg_destroy(h); return KG_ECUDA; }
  }
  if (cudaMallocHost(&h->hout, 2 * sizeof(kg_handle::HostOut)) != cudaSuccess) { kg_destroy(h); return KG_ENOMEM; }
  std::memset(h->hout, 0, 2 * sizeof(kg_handle::HostOut));
  if (cudaEventCreateWithFlags(&h->step_done, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->res_ev[0], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->res_ev[1], cudaEventDisableTiming) != cudaSuccess) { kg_destroy(h); return KG_ECUDA; }
  for (int i = 0; i < 12; ++i)
    if (cudaEventCreate(&h->sev[i]) != cudaSuccess) { kg_destroy(h); return KG_ECUDA; }
  if (cudaStreamCreateWithFlags(&h->st2, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&h->st_cap, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&h->st3, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&h->st5, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_wjoin, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_bent, cudaEventDisableTiming) != cudaSuccess ||
      cudaStreamCreateWithPriority(&h->st4, cudaStreamNonBlocking, kLowPriority()) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_rel, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_loss, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_early, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_i1, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_i2, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_fork2, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_wsplit, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_wsplit_t, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_xt, cudaEventDisableTiming) != cudaSuccess) { kg_destroy(h); return KG_ECUDA; }
  if (c.world > 1) {
    ncclUniqueId id;
    std::memcpy(&id, c.nccl_id, sizeof(id));
    if (!nccl().ok || nccl().CommInitRank(&h->comm, c.world, id, c.rank) != ncclSuccess) { kg_destroy(h); return KG_ENCCL; }
    if (cudaMallocHost(&h->h_counts, sizeof(int32_t) * kMaxWorld * kMaxWorld) != cudaSuccess) { kg_destroy(h); return KG_ENOMEM; }
    // the dL/dtheta_D all-reduce runs on a second stream, overlapped with
    // the row-gradient exchange and the owners' sparse Adam -- on a communicator of its own
    // (collectives of one communicator must not run concurrently); KG_DIST_OVERLAP=0: serial
    const char *ov = std::getenv("KG_DIST_OVERLAP");
    if (!(ov && ov[0] == '0') && nccl().CommSplit &&
        nccl().CommSplit(h->comm, 0, c.rank, &h->comm2, nullptr) != ncclSuccess)
      h->comm2 = nullptr;
  }
  if (const char *e = std::getenv("KG_NO_GRAPH")) h->use_graphs = !(e[0] == '1');
  if (const char *e = std::getenv("KG_PDL")) h->use_pdl = !(e[0] == '0');
  if (const char *e = std::getenv("KG_DIST_BUCKETS")) h->buckets = !(e[0] == '0');
  if (const char *e = std::getenv("KG_XCHG")) h->p2p = c.world > 1 && h->buckets && std::string(e) == "p2p";
  // zeroed before any rank can reach a barrier (a synchronous copy: the steps run on non-blocking
  // streams, which do not order against the legacy stream of a plain cudaMemset)
  static const unsigned long long zeros[kMaxWorld + 1] = {};
  if (h->p2p_flags && cudaMemcpy(h->p2p_flags, zeros, sizeof(zeros), cudaMemcpyHostToDevice) != cudaSuccess) {
    kg_destroy(h);
    return KG_ECUDA;
  }
  h->score_bf16 = c.score_precision == KG_SCORE_BF16;
  if (const char *e = std::getenv("KG_DIST_GRAPH")) h->dist_graph = !(e[0] == '0');
  if (const char *e = std::getenv("KG_NCCL")) if (std::string(e) == "loopback") h->dist_graph = false;
  // DAG contractions (reading A24): the hand-written tcgen05 3xTF32 kernel
  // (k_gemm.cu) in its drained form: TMEM accumulates 4 k-blocks at a time and the chunks are
  // summed in fp32 registers -- a long TMEM accumulation carries 15-25x SGEMM's error
  // (tools/gemm_precision.py), which BetaE's full-size gradients (K = 800 / 1600 contractions
  // feeding differences of digammas) amplify past the 1e-5 bar; drained, the error is SGEMM's.
  // GQE / Q2B would pass undrained too (1 % faster); one accurate path is kept for all.
  h->gemm_drain = true;
  // device scalars
  if (cudaMemset(h->ws, 0, h->ws_bytes) != cudaSuccess) { kg_destroy(h); return KG_ECUDA; }
  if (cudaMemset(h->rel_stamp, 0xff, sizeof(int64_t) * h->R) != cudaSuccess) { kg_destroy(h); return KG_ECUDA; }
  *out = h;
  return KG_OK;
}

int64_t kg_shard_rows(const kg_handle *h) { return h ? h->shard : -1; }
int64_t kg_dense_size(const kg_handle *h) { return h ? h->dense_size : -1; }
int64_t kg_workspace_size(const kg_handle *h) { return h ? (int64_t)h->ws_bytes : -1; }

kg_status kg_bind(kg_handle *h, const kg_tables *t, void *stream) {
  if (!h || !t) return KG_EINVAL;
  if (h->broken) return fail(h, KG_ESTATE, "handle is in an error state: " + h->err);
  if (!t->ent || !t->ent_m || !t->ent_v || !t->dense || !t->dense_m || !t->dense_v)
    return fail(h, KG_EINVAL, "null table pointer");
  const void *ps[6] = {t->ent, t->ent_m, t->ent_v, t->dense, t->dense_m, t->dense_v};
  for (const void *p : ps)
    if ((uintptr_t)p % 16) return fail(h, KG_EINVAL, "table pointers must be 16-byte aligned");
  // theta_E tables may live in device memory or in pinned host memory (the host tier of
  // SURVEY §8(f) f4): the kernels then read / write the rows zero-copy through
  // their device-visible address.  Anything else (pageable host memory) is rejected.
  kg_tables tt = *t;
  float **ents[3] = {&tt.ent, &tt.ent_m, &tt.ent_v};
  h->host_tier = 0;
  for (int i = 0; i < 6; ++i) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, ps[i]) != cudaSuccess) {
      cudaGetLastError();
      return fail(h, KG_EINVAL, "table pointer is not CUDA-visible memory");
    }
    if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) continue;
    if (a.type == cudaMemoryTypeHost && i < 3 && a.devicePointer) {
      *ents[i] = static_cast<float *>(a.devicePointer);
      h->host_tier |= 1 << i;
      continue;
    }
    return fail(h, KG_EINVAL, i < 3 ? "theta_E tables must be device or pinned host memory"
                                    : "theta_D tables must be device memory");
  }
  const bool rebind = h->bound;
  if (rebind && h->p2p)   // the peers mapped this rank's shard and buckets at the first bind
    return fail(h, KG_ESTATE, "KG_XCHG=p2p: kg_bind may be called once (peers hold the mapped tables)");
  if (rebind) {
    // the cached step graphs baked the old table pointers and stream into their kernel
    // arguments: finish what is in flight, then drop them (recaptured on the next step)
    CK(cudaStreamSynchronize(h->st));
    for (auto &g : h->graphs) cudaGraphExecDestroy(g.exec);
    h->graphs.clear();
  }
  h->t = tt;
  h->st = (cudaStream_t)stream;
  if (h->p2p) {
    if (h->host_tier) return fail(h, KG_EUNSUPPORTED, "KG_XCHG=p2p needs theta_E in device memory");
    kg_status s = map_peers(h);
    if (s != KG_OK) return s;
  }
  h->bound = true;
  return KG_OK;
}

kg_status kg_init_params(kg_handle *h, uint64_t seed) {
  kg_status s = check_state(h);
  if (s) return s;
  const double rho = ((double)h->cfg.gamma + 2.0) / (double)h->d;
  launch_init_rows(h->t.ent, h->shard, h->d, h->rank, h->world, seed, 0, (float)-rho, (float)rho, h->st);
  for (size_t i = 0; i < h->segs.size(); ++i)
    launch_init_flat(h->t.dense + h->segs[i].off, h->segs[i].n, seed, 1 + i, h->segs[i].lo, h->segs[i].hi, h->st);
  // moments start at 0 (A23); a host-tier table is written by a kernel through its mapped address
  float *mv[2] = {h->t.ent_m, h->t.ent_v};
  for (int i = 0; i < 2; ++i) {
    if (h->host_tier & (2 << i)) launch_init_flat(mv[i], h->shard * h->d, 0, 0, 0.f, 0.f, h->st);
    else CK(cudaMemsetAsync(mv[i], 0, sizeof(float) * h->shard * h->d, h->st));
  }
  CK(cudaMemsetAsync(h->t.dense_m, 0, sizeof(float) * h->dense_size, h->st));
  CK(cudaMemsetAsync(h->t.dense_v, 0, sizeof(float) * h->dense_size, h->st));
  CK(cudaMemsetAsync(h->t_dev, 0, sizeof(int64_t), h->st));
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(h->st));
  return KG_OK;
}

}  // extern "C"

namespace {

// a8-a10 for the dot-product scorers (DistMult / ComplEx and their -m variants; SURVEY §8(a)
// a8: "a tcgen05 dense contraction only for dot-product scorers"): with the pool's rows
// gathered into Eg [K][d], S = Q Eg^T is one GEMM (D = -S, A13; the pair epilogue applies the
// DNF min and Eq. 1 on it), and the backward is two: dQ += -C Eg, dV = -C^T Q (alpha = -1,
// written straight into the gradient buffers).  The other scorers (L1 / box / Beta-KL / RotatE) stay on the CUDA-core pair kernels.
// bf16 score mode for the GEMMs enqueued in a scope (the scoring contractions only)
struct LowpScope {
  kg_handle *h;
  LowpScope(kg_handle *hh, bool on) : h(hh) { h->gemm_lowp = on; }
  ~LowpScope() { h->gemm_lowp = false; }
};
bool gemm_scoring(const kg_handle *h) { return h->sk == KG_DISTMULT || h->sk == KG_COMPLEX; }
kg_status score_forward(kg_handle *h, ScoreArgs &sa, int nout, bool train, const int64_t *neg_rows,
                        const std::function<void()> &between = {}) {
  if (!gemm_scoring(h)) {
    launch_pair_fwd(h->sk, sa, nout, train, h->st, between);
    return KG_OK;
  }
  if (between) between();
  launch_gather_rows(h->Eg, h->ent_src, neg_rows, sa.K, h->d, h->st);
  sa.KS = 1;
  LowpScope lp(h, train && h->score_bf16);
  G(false, true, sa.NQ, sa.K, h->d, sa.Q, h->d, h->Eg, h->d, 0.f, sa.Dpart, sa.Kp);
  launch_pair_epi(h->sk, sa, nout, train, h->st);
  return KG_OK;
}
kg_status score_backward(kg_handle *h, ScoreArgs &sa, cudaStream_t st2) {
  if (!gemm_scoring(h)) {
    launch_pair_bwd(h->sk, sa, h->st, st2);
    return KG_OK;
  }
  LowpScope lp(h, h->score_bf16);
  // straight into the gradient buffers (no combine pass): dQ += -C Eg on top of the positive
  // term, the pool rows' raw gradients dV = -C^T Q (rows of d, the layout of OG)
  G(false, false, sa.NQ, h->d, sa.K, sa.C, sa.Kp, h->Eg, h->d, 1.f, sa.dQ, h->d, nullptr, 0, -1.f);
  G(true, false, sa.K, h->d, sa.NQ, sa.C, sa.Kp, sa.Q, h->d, 0.f, sa.dV, h->d, nullptr, 0, -1.f);
  return KG_OK;
}

// Everything of one step after ingest: enqueued on h->st (directly, or while
// h->st is a capturing stream -- the sequence is then replayed as a CUDA graph).
kg_status enqueue_step(kg_handle *h, StepBufs &S) {
  kg_status s;
  const Plan &p = S.plan;
  const int M = S.M, K = S.K, d = h->d, na = p.na, nr = p.nr;
  const int L = na * M + M + K, Lr = p.nproj * M;
  cudaStream_t st = h->st;
  h->ent_src = h->t.ent;
  h->side_timed = true;
  mark(h, 0);
  // a2: ids (fused gather indices) on the main stream; dedup of entities and relations
  // on the side stream -- only the sparse update at the end needs them
  CK(cudaMemsetAsync(h->flags, 0, 2 * sizeof(int), st));
  Slots4 sl{{0, 0, 0, 0}};
  {
    int u = 0;
    for (int ni = 0; ni < p.nn; ++ni)
      if (p.n[ni].type == 0) sl.s[u++] = p.n[ni].rel;
  }
  launch_ids_rel(h->b_anchors, na, M, h->b_answers, M, h->b_negs, K, h->world, h->ids, h->rows, h->n_ent, h->b_rels,
                 nr, sl, p.nproj, h->R, h->rocc, h->flags + 1, st);
  if (needs_wplanes(h, p) && (s = issue_wplanes(h, st, h->st4)) != KG_OK) return s;
  const int64_t *neg_rows = h->rows + (int64_t)na * M + M;
  if (h->kind == KG_BETAE && K > 0) {
    // the pool's Beta features (digamma / trigamma planes) depend only on the gathered rows:
    // on st3 beside the DAG forward, joined before the scoring
    if ((s = fork(h, st, h->st3)) != KG_OK) return s;
    launch_beta_entity(h->ent_src, neg_rows, K, h->m, h->F, h->Cv, h->st3);
    CK(cudaEventRecord(h->ev_bent, h->st3));
  }
  CK(cudaEventRecord(h->ev_fork, st));
  CK(cudaStreamWaitEvent(h->st2, h->ev_fork, 0));
  launch_dedup(h->ids, nullptr, L, h->ent_bits, h->uniq, h->inv, h->perm, h->seg, h->Udev, h->st2, h->sinv, h->hrow);
  launch_dedup(nullptr, h->rocc, Lr, h->rel_bits, h->runiq, h->rinv, h->rperm, h->rseg, h->rU, h->st2);
  CK(cudaEventRecord(h->ev_rel, h->st2));

  // a4-a7: fused gather + DAG forward
  mark(h, 1);
  assign_buffers(h, S);
  if ((s = dag_forward(h, S)) != KG_OK) return s;
  mark(h, 2);

  // a8-a10: scoring, Eq. 1, scoring backward
  const int U = (h->sk == KG_BETAE || h->sk == KG_ROTATE || h->sk == KG_COMPLEX) ? h->m : d;
  const float scale = 1.f / (float)((double)M * h->world);
  if (h->kind == KG_BETAE) {
    // the query's Beta features (QP, Cq) and then the positive term on st3 beside pair_fwd
    // (which reads only Q and the pool features); the pair epilogue joins st3
    if ((s = fork(h, st, h->st3)) != KG_OK) return s;
    launch_beta_query(h->Q, S.NQ, h->m, h->QP, h->Cq, h->st3);
    if (K > 0) CK(cudaStreamWaitEvent(st, h->ev_bent, 0));   // pool features (st3, before the fork)
  }
  PosArgs pa;
  pa.M = M; pa.U = U; pa.d = d; pa.ent = h->ent_src; pa.ans_rows = h->rows + (int64_t)na * M; pa.Q = h->Q;
  pa.alpha = h->cfg.box_alpha; pa.gamma = h->cfg.gamma; pa.scale = scale; pa.Cq = h->Cq; pa.QP = h->QP;
  pa.loss_pos = h->loss_pos; pa.Dpos = h->Dpos; pa.dQ = h->dQ; pa.dV = h->OG + (int64_t)na * M * d;
  // the positive term (D+, its adjoint and gradients: per query): BetaE's (digamma / lgamma
  // per unit) beside the pool scoring on st3; the light ones in order (run beside pair_fwd they
  // slowed it more than they took: C5-q2b scoring forward 57 -> 62 us)
  // (pair kernels: on st3 beside the pair epilogue, forked once pair_fwd is enqueued -- beside
  // pair_fwd itself it slowed that kernel more than it saved)
  const bool pos_side = h->kind == KG_BETAE;   // st3 already forked (beta_query)
  const bool pos_between = !pos_side && !gemm_scoring(h) && K > 0;
  if (!pos_between) launch_pos(h->sk, pa, p.nout, pos_side ? h->st3 : st);
  kg_status sb = KG_OK;
  auto pos_beside_epi = [&]() {
    sb = fork(h, st, h->st3);
    launch_pos(h->sk, pa, p.nout, h->st3);
  };
  auto join_before_epi = [&]() { sb = join(h, h->st3, st); };   // BetaE: QP / Cq / loss_pos (st3)
  ScoreArgs sa;
  sa.Q = h->Q; sa.NQ = S.NQ; sa.M = M; sa.K = K; sa.Kp = S.Kp; sa.U = U; sa.d = d;
  if (h->kind == KG_BETAE) { sa.E = h->F; sa.eidx = nullptr; sa.estride = 9LL * h->m; }
  else { sa.E = h->ent_src; sa.eidx = neg_rows; sa.estride = d; }
  sa.mask = h->b_mask; sa.W = (K + 31) / 32; sa.Cq = h->Cq; sa.Cv = h->Cv; sa.QP = h->QP;
  sa.gamma = h->cfg.gamma; sa.alpha = h->cfg.box_alpha; sa.scale = scale;
  sa.C = h->C; sa.Dmin = h->keep_grads ? h->Dmin : nullptr; sa.loss_part = h->loss_part; sa.dQ = h->dQ;   // D only for kg_last_grads
  sa.Dpart = h->Dpart; sa.partQ = h->partQ; sa.partV = h->partV; sa.Cpart = h->Cpart; sa.Csum = h->Csum;
  sa.cap_D = h->cap_D; sa.cap_Q = h->cap_Q; sa.cap_V = h->cap_V;
  sa.dV = h->OG + (int64_t)(na * M + M) * d;
  const int njt = K > 0 ? 1 : 0;
  if (K > 0 && (s = score_forward(h, sa, p.nout, true, neg_rows,
                                  pos_between ? std::function<void()>(pos_beside_epi)
                                  : pos_side  ? std::function<void()>(join_before_epi)
                                              : std::function<void()>())) != KG_OK)
    return s;
  if (sb != KG_OK) return sb;
  if ((pos_side || pos_between) && (s = join(h, h->st3, st)) != KG_OK) return s;
  // Eq. 1's loss, the step's fate (flags) and Adam's bias corrections: one CTA on st3, off the
  // scoring backward's path (only the updates need it: the early dense Adam waits for ev_loss,
  // the sparse update joins st3 before it)
  // (measured neutral against the in-order launch: C5-q2b 1.561M / 1.562M, C3-complex 8.98M / 9.01M)
  cudaStream_t slf = h->st3;
  if ((s = fork(h, st, h->st3)) != KG_OK) return s;
  launch_loss_finalize(h->loss_pos, h->loss_part, M, njt, 1.0 / ((double)M * h->world), h->loss_dev, h->flags,
                       h->t_dev, h->bc, h->cfg.beta1, h->cfg.beta2, h->apply, slf);
  CK(cudaEventRecord(h->ev_loss, slf));
  mark(h, 3);
  // a14 (first part): the relation rows this step does not use take their Adam update with
  // g = 0 (A17) as soon as the step's fate (flags, bias corrections) is known -- a 300 MB
  // stream overlapped with the ALU-bound scoring backward; the used rows follow at the end.
  if (h->apply) {
    CK(cudaStreamWaitEvent(h->st4, h->ev_loss, 0));
    CK(cudaStreamWaitEvent(h->st4, h->ev_rel, 0));
    mark(h, 10, h->st4);
    launch_rel_stamp(h->runiq, h->rU, Lr, h->rel_seg_map, h->rel_stamp, h->stamp_dev, h->st4);
    const Seg &r = h->segs[0];
    const int nseg = h->kind == KG_Q2B ? 2 : 1;
    launch_dense_adam_rel(h->t.dense + r.off, h->t.dense_m + r.off, h->t.dense_v + r.off, h->R, r.cols, nseg,
                          h->RGU, h->rel_seg_map, h->rel_stamp, h->stamp_dev, h->lr_dev, h->cfg.beta1,
                          h->cfg.beta2, h->cfg.eps, h->bc, h->flags, h->st4, /*untouched_only=*/1);
    mark(h, 11, h->st4);
    CK(cudaEventRecord(h->ev_early, h->st4));
  }
  if (K > 0) {
    // dV (pool rows) on the side stream, concurrently with dQ and the DAG backward
    CK(cudaEventRecord(h->ev_fork2, st));
    CK(cudaStreamWaitEvent(h->st2, h->ev_fork2, 0));
  }
  if (K > 0 && (s = score_backward(h, sa, h->st2)) != KG_OK) return s;
  CK(cudaEventRecord(h->ev_join, h->st2));
  mark(h, 4);

  // a11: DAG backward (its weight gradients join the dense Adam's stream below)
  if ((s = dag_backward(h, S, /*defer_wjoin=*/true)) != KG_OK) return s;
  if (p.inter < 0 && h->kind != KG_BETAE && h->w_off < h->dense_size)
    CK(cudaMemsetAsync(h->gdense, 0, sizeof(float) * (h->dense_size - h->w_off), st));
  if (p.inter < 0 && h->kind == KG_BETAE) {   // attention weights unused by this structure
    const Seg *a = seg_of(h, "att_U1");
    CK(cudaMemsetAsync(h->gdense + (a->off - h->w_off), 0, sizeof(float) * (h->dense_size - a->off), st));
  }

  // a12-a14: the sparse update (segment reduce + sparse Adam, latency-bound random rows) on
  // the main stream, concurrently with the relation-row reduce and the dense Adam over
  // theta_D (a streaming, HBM-bound pass) on the side stream; joined before the outputs.
  // Stage 5-6 = the sparse path, stage 6-7 = what the dense path adds after it.
  CK(cudaStreamWaitEvent(st, h->ev_join, 0));
  CK(cudaStreamWaitEvent(st, h->ev_loss, 0));   // loss_finalize (st3): flags, bias corrections
  mark(h, 5);
  CK(cudaEventRecord(h->ev_fork2, st));
  CK(cudaStreamWaitEvent(h->st2, h->ev_fork2, 0));
  {
    cudaStream_t s2 = h->st2;
    mark(h, 8, s2);
    launch_rel_reduce(h->rseg, h->rperm, h->rinv, h->rU, Lr, h->RG, h->PSr, h->dr, h->RGU, s2);
    const double b1 = h->cfg.beta1, b2 = h->cfg.beta2, eps = h->cfg.eps;
    const float *lr = h->lr_dev;
    if (h->apply) {
      CK(cudaStreamWaitEvent(s2, h->ev_early, 0));
      // the relation rows used by this step: segs[0] (and segs[1] for Q2B: rel_offset right after)
      const Seg &r = h->segs[0];
      const int nseg = h->kind == KG_Q2B ? 2 : 1;
      launch_dense_adam_rel_touched(h->t.dense + r.off, h->t.dense_m + r.off, h->t.dense_v + r.off, h->R, r.cols,
                                    nseg, h->RGU, h->runiq, h->rU, Lr, lr, b1, b2, eps, h->bc, h->flags, s2);
    }
    // only the operator weights' Adam needs the weight gradients of st5 (the relation rows' do not)
    if ((s = wjoin(h, s2)) != KG_OK) return s;
    if (h->apply)
      launch_dense_adam(h->t.dense + h->w_off, h->t.dense_m + h->w_off, h->t.dense_v + h->w_off, h->gdense,
                        h->dense_size - h->w_off, lr, b1, b2, eps, h->bc, h->flags, s2);
    mark(h, 9, s2);
    CK(cudaEventRecord(h->ev_join, s2));
  }
  if (h->apply || h->keep_grads)
    launch_sparse_adam(h->uniq, h->seg, h->perm, h->sinv, h->hrow, h->Udev, L, h->OG, h->PS, h->pcnt, d, h->world, h->t.ent, h->t.ent_m,
                       h->t.ent_v, h->keep_grads ? h->Gc : nullptr, h->lr_dev, h->cfg.beta1, h->cfg.beta2,
                       h->cfg.eps, h->bc, h->flags, h->apply, st, -1, /*early=*/1);
  mark(h, 6);
  CK(cudaStreamWaitEvent(st, h->ev_join, 0));
  mark(h, 7);
  CK(cudaGetLastError());
  return KG_OK;
}


// One step with theta_E row-sharded over G ranks (reading A18):
// requests of the distinct ids go to their owners, owners return the rows, the
// step runs on the received rows, merged row gradients go back to the owners,
// which sum the contributions of all ranks in (source rank, position) order and
// apply Adam; dL/dtheta_D (relations + weights) is all-reduced and every rank
// applies the same dense Adam.  Collective: all ranks call it with the same
// structure, M and K.
kg_status step_dist(kg_handle *h, StepBufs &S) {
  kg_status s;
  const Plan &p = S.plan;
  const int M = S.M, K = S.K, d = h->d, na = p.na, nr = p.nr, G = h->world, me = h->rank;
  const int L = na * M + M + K, Lr = p.nproj * M;
  cudaStream_t st = h->st;
  h->side_timed = false;
  mark(h, 0);
  CK(cudaMemsetAsync(h->flags, 0, 2 * sizeof(int), st));
  launch_ids_concat(h->b_anchors, na, M, h->b_answers, M, h->b_negs, K, G, h->ids, h->rows, h->flags + 1, h->n_ent,
                    st);
  Slots4 sl{{0, 0, 0, 0}};
  {
    int u = 0;
    for (int ni = 0; ni < p.nn; ++ni)
      if (p.n[ni].type == 0) sl.s[u++] = p.n[ni].rel;
  }
  launch_rel_occ(h->b_rels, M, nr, sl, p.nproj, h->R, h->rocc, h->flags + 1, st);
  launch_dedup(h->ids, nullptr, L, h->ent_bits, h->uniq, h->inv, h->perm, h->seg, h->Udev, st, h->sinv, h->hrow);
  launch_dedup(nullptr, h->rocc, Lr, h->rel_bits, h->runiq, h->rinv, h->rperm, h->rseg, h->rU, st);
  // a3: route the distinct ids to their owners (owner = id % G).  Buckets: every rank sends
  // `cap` slots to every owner (empty slots = -1), so no size is read on the host and the
  // step needs no host round trip; otherwise exact counts are all-gathered and read first.
  const int cap = h->buckets ? h->cap : 0;
  std::vector<int64_t> so(G + 1, 0), ro(G + 1, 0);   // send / receive offsets (rows)
  if (cap > 0) {
    CK(cudaMemsetAsync(h->send_ids, 0xff, sizeof(int64_t) * G * cap, st));
    launch_owner_partition(h->uniq, h->Udev, G, h->send_ids, h->send_pos, h->counts, st, cap, h->flags);
    for (int o = 0; o <= G; ++o) so[o] = ro[o] = (int64_t)o * cap;
  } else {
    launch_owner_partition(h->uniq, h->Udev, G, h->send_ids, h->send_pos, h->counts, st);
    NCK(nccl().AllGather(h->counts, h->all_counts, kMaxWorld, ncclInt32, h->comm, st));
    CK(cudaMemcpyAsync(h->h_counts, h->all_counts, sizeof(int32_t) * kMaxWorld * G, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int o = 0; o < G; ++o) {
      so[o + 1] = so[o] + h->h_counts[me * kMaxWorld + o];
      ro[o + 1] = ro[o] + h->h_counts[o * kMaxWorld + me];
    }
  }
  const int Rtot = (int)ro[G];
  if (h->p2p) {
    // one-sided: every owner's previous update (and init) is done once all ranks pass the
    // barrier; then the rows are read straight from the owners' shards into bucket order
    launch_p2p_barrier(h->pp, h->p2p_flags, h->p2p_epoch, G, me, h->flags, st);
    launch_p2p_gather(h->pp, h->uniq, h->Udev, h->send_pos, G, L, d, h->Xin, st);
  } else {
    NCK(nccl().GroupStart());
    for (int o = 0; o < G; ++o) {
      if (so[o + 1] > so[o]) NCK(nccl().Send(h->send_ids + so[o], so[o + 1] - so[o], ncclInt64, o, h->comm, st));
      if (ro[o + 1] > ro[o]) NCK(nccl().Recv(h->recv_ids + ro[o], ro[o + 1] - ro[o], ncclInt64, o, h->comm, st));
    }
    NCK(nccl().GroupEnd());
    launch_gather_owned(h->t.ent, h->recv_ids, Rtot, G, d, h->send_rows, st);
    NCK(nccl().GroupStart());
    for (int o = 0; o < G; ++o) {
      if (ro[o + 1] > ro[o]) NCK(nccl().Send(h->send_rows + ro[o] * d, (ro[o + 1] - ro[o]) * d, ncclFloat32, o, h->comm, st));
      if (so[o + 1] > so[o]) NCK(nccl().Recv(h->Xin + so[o] * d, (so[o + 1] - so[o]) * d, ncclFloat32, o, h->comm, st));
    }
    NCK(nccl().GroupEnd());
  }
  launch_occ_rows(h->inv, h->send_pos, L, h->rows, st);
  h->ent_src = h->Xin;

  // a4-a10 on the received rows (as for one rank)
  mark(h, 1);
  assign_buffers(h, S);
  if ((s = dag_forward(h, S)) != KG_OK) return s;
  mark(h, 2);
  const int U = (h->sk == KG_BETAE || h->sk == KG_ROTATE || h->sk == KG_COMPLEX) ? h->m : d;
  const int64_t *neg_rows = h->rows + (int64_t)na * M + M;
  const float scale = 1.f / (float)((double)M * G);
  if (h->kind == KG_BETAE) {
    launch_beta_query(h->Q, S.NQ, h->m, h->QP, h->Cq, st);
    launch_beta_entity(h->ent_src, neg_rows, K, h->m, h->F, h->Cv, st);
  }
  PosArgs pa;
  pa.M = M; pa.U = U; pa.d = d; pa.ent = h->ent_src; pa.ans_rows = h->rows + (int64_t)na * M; pa.Q = h->Q;
  pa.alpha = h->cfg.box_alpha; pa.gamma = h->cfg.gamma; pa.scale = scale; pa.Cq = h->Cq; pa.QP = h->QP;
  pa.loss_pos = h->loss_pos; pa.Dpos = h->Dpos; pa.dQ = h->dQ; pa.dV = h->OG + (int64_t)na * M * d;
  launch_pos(h->sk, pa, p.nout, st);
  ScoreArgs sa;
  sa.Q = h->Q; sa.NQ = S.NQ; sa.M = M; sa.K = K; sa.Kp = S.Kp; sa.U = U; sa.d = d;
  if (h->kind == KG_BETAE) { sa.E = h->F; sa.eidx = nullptr; sa.estride = 9LL * h->m; }
  else { sa.E = h->ent_src; sa.eidx = neg_rows; sa.estride = d; }
  sa.mask = h->b_mask; sa.W = (K + 31) / 32; sa.Cq = h->Cq; sa.Cv = h->Cv; sa.QP = h->QP;
  sa.gamma = h->cfg.gamma; sa.alpha = h->cfg.box_alpha; sa.scale = scale;
  sa.C = h->C; sa.Dmin = h->keep_grads ? h->Dmin : nullptr; sa.loss_part = h->loss_part; sa.dQ = h->dQ;   // D only for kg_last_grads
  sa.Dpart = h->Dpart; sa.partQ = h->partQ; sa.partV = h->partV; sa.Cpart = h->Cpart; sa.Csum = h->Csum;
  sa.cap_D = h->cap_D; sa.cap_Q = h->cap_Q; sa.cap_V = h->cap_V;
  sa.dV = h->OG + (int64_t)(na * M + M) * d;
  if (K > 0 && (s = score_forward(h, sa, p.nout, true, neg_rows)) != KG_OK) return s;
  // global loss = sum over ranks of the (1/(M G))-scaled local sums (A18); one finite check for all
  launch_loss_finalize(h->loss_pos, h->loss_part, M, K > 0 ? 1 : 0, 1.0 / ((double)M * G), h->loss_dev, h->flags,
                       h->t_dev, h->bc, h->cfg.beta1, h->cfg.beta2, h->apply, st, /*check=*/0);
  NCK(nccl().AllReduce(h->loss_dev, h->loss_dev, 1, ncclFloat64, ncclSum, h->comm, st));
  NCK(nccl().AllReduce(h->flags + 1, h->flags + 1, 1, ncclInt32, ncclMax, h->comm, st));
  launch_loss_check(h->loss_dev, h->flags, h->t_dev, h->bc, h->cfg.beta1, h->cfg.beta2, h->apply, st);
  mark(h, 3);
  if (K > 0 && (s = score_backward(h, sa, st)) != KG_OK) return s;
  mark(h, 4);
  if ((s = dag_backward(h, S)) != KG_OK) return s;
  if (p.inter < 0 && h->kind != KG_BETAE && h->w_off < h->dense_size)
    CK(cudaMemsetAsync(h->gdense, 0, sizeof(float) * (h->dense_size - h->w_off), st));
  if (p.inter < 0 && h->kind == KG_BETAE) {
    const Seg *a = seg_of(h, "att_U1");
    CK(cudaMemsetAsync(h->gdense + (a->off - h->w_off), 0, sizeof(float) * (h->dense_size - a->off), st));
  }
  mark(h, 5);
  // a14, first half: the dense dL/dtheta_D of this rank (relation reduce + scatter); with a second
  // communicator its all-reduce and the dense Adam run on st2 while st exchanges the row
  // gradients and the owners apply sparse Adam
  launch_rel_reduce(h->rseg, h->rperm, h->rinv, h->rU, Lr, h->RG, h->PSr, h->dr, h->RGU, st);
  CK(cudaMemsetAsync(h->gfull, 0, sizeof(float) * h->w_off, st));
  launch_scatter_rel(h->RGU, h->runiq, h->rU, Lr, h->R, h->segs[0].cols, h->kind == KG_Q2B ? 2 : 1, h->gfull, st);
  const bool overlap = h->comm2 != nullptr;
  if (overlap) {
    if ((s = fork(h, st, h->st2)) != KG_OK) return s;
    NCK(nccl().AllReduce(h->gfull, h->gfull, h->dense_size, ncclFloat32, ncclSum, h->comm2, h->st2));
    if (h->apply)
      launch_dense_adam(h->t.dense, h->t.dense_m, h->t.dense_v, h->gfull, h->dense_size, h->lr_dev, h->cfg.beta1,
                        h->cfg.beta2, h->cfg.eps, h->bc, h->flags, h->st2);
  }
  // a12: merged row gradients of this rank (distinct-id order) -> send order -> owners
  launch_sparse_adam(h->uniq, h->seg, h->perm, h->sinv, h->hrow, h->Udev, L, h->OG, h->PS, h->pcnt, d, 1, h->t.ent, h->t.ent_m,
                     h->t.ent_v, h->Gc, h->lr_dev, h->cfg.beta1, h->cfg.beta2, h->cfg.eps, h->bc, h->flags,
                     /*apply=*/0, st);
  launch_reorder_rows(h->Gc, h->send_pos, h->Udev, L, d, h->Gsend, st);
  if (h->p2p) {
    // one-sided: ids + gradient rows straight into the owners' receive buckets, then a barrier
    // (every rank's writes into this rank's buckets are complete)
    launch_p2p_push(h->pp, h->send_ids, h->Gsend, G, me, cap, d, st);
    launch_p2p_barrier(h->pp, h->p2p_flags, h->p2p_epoch, G, me, h->flags, st);
  } else {
    NCK(nccl().GroupStart());
    for (int o = 0; o < G; ++o) {
      if (so[o + 1] > so[o]) NCK(nccl().Send(h->Gsend + so[o] * d, (so[o + 1] - so[o]) * d, ncclFloat32, o, h->comm, st));
      if (ro[o + 1] > ro[o]) NCK(nccl().Recv(h->Grecv + ro[o] * d, (ro[o + 1] - ro[o]) * d, ncclFloat32, o, h->comm, st));
    }
    NCK(nccl().GroupEnd());
  }
  // a13 at the owner: merge the contributions of all ranks (fixed order) + sparse Adam on local rows
  // empty bucket slots carry the key `shard` (one past the last local row), skipped by the update
  launch_local_rows(h->recv_ids, Rtot, G, h->recv_keys, st, h->shard);
  launch_dedup(h->recv_keys, nullptr, Rtot, bits_for(h->shard + 1), h->ouniq, h->oinv, h->operm, h->oseg, h->oU, st,
               h->osinv, h->ohrow);
  if (h->apply)
    launch_sparse_adam(h->ouniq, h->oseg, h->operm, h->osinv, h->ohrow, h->oU, Rtot, h->Grecv, h->PSo, h->ocnt, d, 1, h->t.ent,
                       h->t.ent_m, h->t.ent_v, nullptr, h->lr_dev, h->cfg.beta1, h->cfg.beta2, h->cfg.eps, h->bc,
                       h->flags, 1, st, /*skip_key=*/h->shard);
  mark(h, 6);
  // a14, second half: all-reduce -> dense Adam (identical on every rank)
  if (overlap) {
    if ((s = join(h, h->st2, st)) != KG_OK) return s;
  } else {
    NCK(nccl().AllReduce(h->gfull, h->gfull, h->dense_size, ncclFloat32, ncclSum, h->comm, st));
    if (h->apply)
      launch_dense_adam(h->t.dense, h->t.dense_m, h->t.dense_v, h->gfull, h->dense_size, h->lr_dev, h->cfg.beta1,
                        h->cfg.beta2, h->cfg.eps, h->bc, h->flags, st);
  }
  mark(h, 7);
  CK(cudaGetLastError());
  return KG_OK;
}


// Per-call device buffers of the untimed paths (kg_score / kg_eval / kg_gather_rows with
// world > 1), freed in stream order when the call returns.
struct CallBufs {
  kg_handle *h;
  std::vector<void *> p;
  explicit CallBufs(kg_handle *hh) : h(hh) {}
  template <class T> T *get(int64_t n) {
    void *q = nullptr;
    if (cudaMallocAsync(&q, sizeof(T) * (size_t)std::max<int64_t>(n, 1), h->st) != cudaSuccess) return nullptr;
    p.push_back(q);
    return static_cast<T *>(q);
  }
  ~CallBufs() {
    for (void *q : p) cudaFreeAsync(q, h->st);
  }
};

// Rows of arbitrary global ids from their owners (owner = id % G, local row id / G; SURVEY
// §8(b) "collective ... gathering rows from their owners"), collective over the ranks: every
// rank calls it, each with its own n >= 0 ids (host), and receives tab's rows in id order in
// d_out [n][d] (device).  Exact counts are all-gathered first (these are not the captured
// training step; one host round trip per phase).  Leaves the stream synchronised.
kg_status fetch_rows(kg_handle *h, const int64_t *ids, int64_t n, const float *tab, float *d_out, CallBufs &B) {
  const int G = h->world, me = h->rank, d = h->d;
  cudaStream_t st = h->st;
  std::vector<int64_t> send, pos;                // requests grouped by owner, their positions in ids
  std::vector<int64_t> so(G + 1, 0), ro(G + 1, 0);
  send.reserve(n);
  pos.reserve(n);
  for (int o = 0; o < G; ++o) {
    for (int64_t i = 0; i < n; ++i)
      if (ids[i] % G == o) { send.push_back(ids[i]); pos.push_back(i); }
    so[o + 1] = (int64_t)send.size();
  }
  std::vector<int32_t> cnt(kMaxWorld, 0);
  for (int o = 0; o < G; ++o) cnt[o] = (int32_t)(so[o + 1] - so[o]);
  CK(cudaMemcpyAsync(h->counts, cnt.data(), sizeof(int32_t) * kMaxWorld, cudaMemcpyHostToDevice, st));
  NCK(nccl().AllGather(h->counts, h->all_counts, kMaxWorld, ncclInt32, h->comm, st));
  CK(cudaMemcpyAsync(h->h_counts, h->all_counts, sizeof(int32_t) * kMaxWorld * G, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (int o = 0; o < G; ++o) ro[o + 1] = ro[o] + h->h_counts[o * kMaxWorld + me];
  const int64_t S = so[G], R = ro[G];
  int64_t *d_send = B.get<int64_t>(S), *d_recv = B.get<int64_t>(R), *d_pos = B.get<int64_t>(S);
  float *rows_out = B.get<float>(R * d), *rows_in = B.get<float>(S * d);
  if (!d_send || !d_recv || !d_pos || !rows_out || !rows_in) return fail(h, KG_ENOMEM, "fetch_rows buffers");
  if (S) CK(cudaMemcpyAsync(d_send, send.data(), sizeof(int64_t) * S, cudaMemcpyHostToDevice, st));
  if (S) CK(cudaMemcpyAsync(d_pos, pos.data(), sizeof(int64_t) * S, cudaMemcpyHostToDevice, st));
  NCK(nccl().GroupStart());
  for (int o = 0; o < G; ++o) {
    if (so[o + 1] > so[o]) NCK(nccl().Send(d_send + so[o], so[o + 1] - so[o], ncclInt64, o, h->comm, st));
    if (ro[o + 1] > ro[o]) NCK(nccl().Recv(d_recv + ro[o], ro[o + 1] - ro[o], ncclInt64, o, h->comm, st));
  }
  NCK(nccl().GroupEnd());
  // owner side: the requested global ids -> local rows -> row copies
  std::vector<int64_t> req(R);
  if (R) CK(cudaMemcpyAsync(req.data(), d_recv, sizeof(int64_t) * R, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (int64_t i = 0; i < R; ++i) req[i] /= G;
  if (R) {
    CK(cudaMemcpyAsync(d_recv, req.data(), sizeof(int64_t) * R, cudaMemcpyHostToDevice, st));
    launch_gather_rows(rows_out, tab, d_recv, (int)R, d, st);
  }
  NCK(nccl().GroupStart());
  for (int o = 0; o < G; ++o) {
    if (ro[o + 1] > ro[o]) NCK(nccl().Send(rows_out + ro[o] * d, (ro[o + 1] - ro[o]) * d, ncclFloat32, o, h->comm, st));
    if (so[o + 1] > so[o]) NCK(nccl().Recv(rows_in + so[o] * d, (so[o + 1] - so[o]) * d, ncclFloat32, o, h->comm, st));
  }
  NCK(nccl().GroupEnd());
  if (S) launch_scatter_rows(d_out, rows_in, d_pos, (int)S, d, st);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(st));
  return KG_OK;
}

}  // namespace

// NVTX ranges on the host side of the public calls (enqueue, capture, H2D staging); the
// device work of a step is one graph launch, its stage boundaries are the stage events.
struct NvtxRange {
  explicit NvtxRange(const char *n) { nvtxRangePushA(n); }
  ~NvtxRange() { nvtxRangePop(); }
};

extern "C" {

kg_status kg_step(kg_handle *h, const kg_batch *b, float lr, kg_step_info *info) {
  NvtxRange range("kg_step");
  kg_status s = check_state(h);
  if (s) return s;
  if (!b) return fail(h, KG_EINVAL, "null batch");
  if (b->structure < KG_1P || b->structure > KG_PNI) return fail(h, KG_EINVAL, "bad structure");
  if (single_hop(h->kind) && b->structure != KG_1P)
    return fail(h, KG_EUNSUPPORTED, "single-hop models accept only 1p (Table 2, P:L55)");
  if (b->structure >= KG_2IN && h->kind != KG_BETAE)
    return fail(h, KG_EUNSUPPORTED, "negation structures need BetaE (Table 1 'Negation' column)");
  if (!(lr > 0.f)) return fail(h, KG_EINVAL, "lr must be > 0");
  StepBufs S;
  S.plan = make_plan(b->structure);
  const Plan &p = S.plan;
  S.M = b->M; S.K = b->K; S.Kp = (int)align_up(std::max(b->K, 1), 64); S.NQ = p.nout * b->M;
  h->stamp++;
  {
    NvtxRange r2("kg_step: ingest (H2D staging)");
    if ((s = ingest(h, b, true, p, lr)) != KG_OK) return s;
  }
  h->last_M = S.M; h->last_K = S.K;
  // world > 1 is captured too when its exchange has fixed sizes (buckets) and the
  // communicator is NCCL (the loopback test communicator synchronises on the host)
  const bool graph_ok = h->use_graphs && (h->world == 1 || (h->buckets && h->dist_graph));
  if (!graph_ok) {
    const int64_t l0 = g_launches;
    h->gemm_count = 0;
    if ((s = h->world > 1 ? step_dist(h, S) : enqueue_step(h, S)) != KG_OK) return s;
    h->last_kernels = (int)(g_launches - l0);
    h->last_gemms = h->gemm_count;
  } else if (h->use_graphs) {
    bool eager_done = false;   // world > 1 whose capture failed: ran eagerly instead
    kg_handle::GraphEntry *g = nullptr;
    for (auto &e : h->graphs)
      if (e.structure == b->structure && e.M == S.M && e.K == S.K && e.flags == h->flag_key()) { g = &e; break; }
    if (!g) {
      // capture once per (structure, M, K, flags) on the internal stream, then replay
      cudaStream_t user = h->st;
      h->st = h->st_cap;
      const int64_t l0 = g_launches;
      h->gemm_count = 0;
      NvtxRange r3("kg_step: graph capture + instantiate");
      CK(cudaStreamBeginCapture(h->st_cap, cudaStreamCaptureModeThreadLocal));
      s = h->world > 1 ? step_dist(h, S) : enqueue_step(h, S);
      cudaGraph_t graph = nullptr;
      cudaError_t ce = cudaStreamEndCapture(h->st_cap, &graph);
      h->st = user;
      if (h->world > 1 && (s != KG_OK || ce != cudaSuccess)) {
        // the collectives could not be captured: this and later steps run eagerly
        if (graph) cudaGraphDestroy(graph);
        cudaGetLastError();
        h->dist_graph = false;
        const int64_t l0e = g_launches;
        h->gemm_count = 0;
        if ((s = step_dist(h, S)) != KG_OK) return s;
        h->last_kernels = (int)(g_launches - l0e);
        h->last_gemms = h->gemm_count;
        eager_done = true;
      }
      if (!eager_done) {
      if (s != KG_OK) { if (graph) cudaGraphDestroy(graph); return s; }
      if (ce != cudaSuccess) return fail(h, KG_ECUDA, std::string("stream capture: ") + cudaGetErrorString(ce));
      kg_handle::GraphEntry e{};
      e.structure = b->structure; e.M = S.M; e.K = S.K; e.flags = h->flag_key();
      e.kernels = (int)(g_launches - l0);
      e.gemms = h->gemm_count;
      if (h->use_pdl) e.pdl_edges = make_programmatic(graph);
      ce = cudaGraphInstantiate(&e.exec, graph, 0);
      cudaGraphDestroy(graph);
      if (ce != cudaSuccess) return fail(h, KG_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(ce));
      if (h->graphs.size() >= 64) { cudaGraphExecDestroy(h->graphs.front().exec); h->graphs.erase(h->graphs.begin()); }
      h->graphs.push_back(e);
      g = &h->graphs.back();
      }
    }
    if (!eager_done) {
      CK(cudaGraphLaunch(g->exec, h->st));
      h->last_kernels = g->kernels;
      h->last_gemms = g->gemms;
    }
  } else {
    const int64_t l0 = g_launches;
    h->gemm_count = 0;
    if ((s = enqueue_step(h, S)) != KG_OK) return s;
    h->last_kernels = (int)(g_launches - l0);
    h->last_gemms = h->gemm_count;
  }
  {
    // the step's scalar results into its ring slot (one D2H), outside the replayed graph
    const int slot = h->res_next;
    h->res_next ^= 1;
    CK(cudaMemcpyAsync(&h->hout[slot], h->resdev, sizeof(kg_handle::HostOut), cudaMemcpyDeviceToHost, h->st));
    CK(cudaEventRecord(h->res_ev[slot], h->st));
    h->res_kernels[slot] = h->last_kernels;
    h->res_gemms[slot] = h->last_gemms;
    h->res_pending = std::min(2, h->res_pending + 1);   // a third unread step drops the oldest
  }
  CK(cudaEventRecord(h->step_done, h->st));
  h->step_pending = true;
  h->last_U_valid = 1;
  if (info) return read_latest(h, info);
  return KG_OK;
}

kg_status kg_sync(kg_handle *h, kg_step_info *info) {
  kg_status s = check_state(h);
  if (s) return s;
  return read_latest(h, info);
}

kg_status kg_result(kg_handle *h, kg_step_info *info) {
  kg_status s = check_state(h);
  if (s) return s;
  if (h->res_pending == 0) return fail(h, KG_ESTATE, "no unread step result");
  const int slot = (h->res_next + 2 - h->res_pending) & 1;   // the oldest unread slot
  --h->res_pending;
  if (h->res_pending == 0) h->step_pending = false;
  return read_result(h, info, slot);
}

// Validate a query batch for kg_score / kg_eval and compute its embeddings into h->Q
// (ingest, relation occurrences, DAG forward); n_cand candidate ids (device, in b_negs)
// get their rows in h->rows after the anchors.
// Forward DAG of the queries; with world > 1 the rows of the anchors and the n_cand candidates
// (already in b_negs) are first fetched from their owners (collective) into a per-call buffer,
// and rows[] indexes that buffer.
static kg_status embed_queries(kg_handle *h, const kg_batch *q, StepBufs &S, int n_cand, CallBufs &B) {
  if (q->structure < KG_1P || q->structure > KG_PNI) return fail(h, KG_EINVAL, "bad structure");
  if (single_hop(h->kind) && q->structure != KG_1P) return fail(h, KG_EUNSUPPORTED, "single-hop models accept only 1p");
  if (q->structure >= KG_2IN && h->kind != KG_BETAE)
    return fail(h, KG_EUNSUPPORTED, "negation structures need BetaE (Table 1 'Negation' column)");
  S.plan = make_plan(q->structure);
  kg_batch qb = *q;
  kg_status s;
  if ((s = ingest(h, &qb, false, S.plan)) != KG_OK) return s;
  h->ent_src = h->t.ent;
  const Plan &p = S.plan;
  const int M = q->M, na = p.na, nr = p.nr;
  S.M = M; S.K = n_cand; S.Kp = n_cand; S.NQ = p.nout * M;
  cudaStream_t st = h->st;
  CK(cudaMemsetAsync(h->flags, 0, 2 * sizeof(int), st));
  launch_ids_concat(h->b_anchors, na, M, nullptr, 0, h->b_negs, n_cand, h->world, h->ids, h->rows, h->flags + 1,
                    h->n_ent, st);
  Slots4 sl{{0, 0, 0, 0}};
  {
    int u = 0;
    for (int ni = 0; ni < p.nn; ++ni)
      if (p.n[ni].type == 0) sl.s[u++] = p.n[ni].rel;
  }
  launch_rel_occ(h->b_rels, M, nr, sl, p.nproj, h->R, h->rocc, h->flags + 1, st);
  if (h->world > 1) {
    const int64_t L = (int64_t)na * M + n_cand;
    std::vector<int64_t> ids(L), iota(L);
    CK(cudaMemcpyAsync(ids.data(), h->ids, sizeof(int64_t) * L, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int64_t i = 0; i < L; ++i) iota[i] = i;
    float *X = B.get<float>(L * h->d);
    if (!X) return fail(h, KG_ENOMEM, "score row buffer");
    kg_status s;
    if ((s = fetch_rows(h, ids.data(), L, h->t.ent, X, B)) != KG_OK) return s;
    CK(cudaMemcpyAsync(h->rows, iota.data(), sizeof(int64_t) * L, cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));   // iota is a host temporary
    h->ent_src = X;
  }
  assign_buffers(h, S);
  return dag_forward(h, S);
}

kg_status kg_score(kg_handle *h, const kg_batch *q, const int64_t *cand, int32_t n_cand, float *out_dist) {
  NvtxRange range("kg_score");
  kg_status s = check_state(h);
  if (s) return s;
  if (!q || !cand || !out_dist) return fail(h, KG_EINVAL, "null argument");
  if (n_cand < 1 || n_cand > h->Cx) return fail(h, KG_EINVAL, "n_cand out of range [1, max_cand]");
  for (int c = 0; c < n_cand; ++c)
    if (cand[c] < 0 || cand[c] >= h->n_ent) return fail(h, KG_EINVAL, "candidate id out of range");
  cudaStream_t st = h->st;
  // candidates share the negative slot of the workspace
  CK(cudaMemcpyAsync(h->b_negs, cand, sizeof(int64_t) * n_cand, cudaMemcpyHostToDevice, st));
  StepBufs S;
  CallBufs B(h);
  if ((s = embed_queries(h, q, S, n_cand, B)) != KG_OK) return s;
  const Plan &p = S.plan;
  const int M = q->M, d = h->d, na = p.na;
  const int U = (h->sk == KG_BETAE || h->sk == KG_ROTATE || h->sk == KG_COMPLEX) ? h->m : d;
  const int64_t *cand_rows = h->rows + (int64_t)na * M;
  if (h->kind == KG_BETAE) {
    launch_beta_query(h->Q, S.NQ, h->m, h->QP, h->Cq, st);
    launch_beta_entity(h->ent_src, cand_rows, n_cand, h->m, h->F, h->Cv, st);
  }
  ScoreArgs sa;
  sa.Q = h->Q; sa.NQ = S.NQ; sa.M = M; sa.K = n_cand; sa.Kp = n_cand; sa.U = U; sa.d = d;
  if (h->kind == KG_BETAE) { sa.E = h->F; sa.eidx = nullptr; sa.estride = 9LL * h->m; }
  else { sa.E = h->ent_src; sa.eidx = cand_rows; sa.estride = d; }
  sa.Cq = h->Cq; sa.Cv = h->Cv; sa.alpha = h->cfg.box_alpha; sa.Dmin = h->Dscore; sa.ldo = n_cand;
  sa.Dpart = h->Dpart; sa.cap_D = h->cap_D;
  launch_pair_fwd(h->sk, sa, p.nout, false, st);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out_dist, h->Dscore, sizeof(float) * (size_t)M * n_cand, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return KG_OK;
}

kg_status kg_score_each(kg_handle *h, const kg_batch *q, const int64_t *cand, int32_t n_cand, float *out_dist) {
  NvtxRange range("kg_score_each");
  kg_status s = check_state(h);
  if (s) return s;
  if (!q || !cand || !out_dist) return fail(h, KG_EINVAL, "null argument");
  const int M = q->M;
  if (M < 1 || M > h->Mx) return fail(h, KG_EINVAL, "M out of range [1, max_M]");
  if (n_cand < 1 || (int64_t)n_cand * M > (1LL << 31)) return fail(h, KG_EINVAL, "n_cand out of range");
  const int64_t nc = (int64_t)M * n_cand;
  for (int64_t k = 0; k < nc; ++k)
    if (cand[k] < 0 || cand[k] >= h->n_ent) return fail(h, KG_EINVAL, "candidate id out of range");
  StepBufs S;
  CallBufs B(h);
  if ((s = embed_queries(h, q, S, 0, B)) != KG_OK) return s;
  cudaStream_t st = h->st;
  const float *ent = h->ent_src;
  std::vector<int64_t> pos_ids;
  if (h->world > 1) {   // the candidate rows from their owners (collective), read by position
    float *X = B.get<float>(nc * h->d);
    if (!X) return fail(h, KG_ENOMEM, "score row buffer");
    if ((s = fetch_rows(h, cand, nc, h->t.ent, X, B)) != KG_OK) return s;
    pos_ids.resize(nc);
    for (int64_t i = 0; i < nc; ++i) pos_ids[i] = i;
    cand = pos_ids.data();
    ent = X;
  }
  int64_t *d_cand = nullptr;
  float *d_out = nullptr;
  CK(cudaMallocAsync(&d_cand, sizeof(int64_t) * nc, st));
  CK(cudaMallocAsync(&d_out, sizeof(float) * nc, st));
  CK(cudaMemcpyAsync(d_cand, cand, sizeof(int64_t) * nc, cudaMemcpyHostToDevice, st));
  EvalArgs a;
  a.Q = h->Q; a.ent = ent; a.negatives = d_cand; a.metrics = d_out;
  a.M = M; a.d = h->d; a.U = (h->sk == KG_BETAE || h->sk == KG_ROTATE || h->sk == KG_COMPLEX) ? h->m : h->d;
  a.n_neg = n_cand; a.alpha = h->cfg.box_alpha;
  launch_score_each(h->sk, a, S.plan.nout, st);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out_dist, d_out, sizeof(float) * nc, cudaMemcpyDeviceToHost, st));
  CK(cudaFreeAsync(d_cand, st));
  CK(cudaFreeAsync(d_out, st));
  CK(cudaStreamSynchronize(st));
  return KG_OK;
}

kg_status kg_eval(kg_handle *h, const kg_batch *q, const int64_t *ans_off, const int64_t *ans_ids, int32_t n_neg,
                  const int64_t *negatives, int32_t *ranks, float *metrics) {
  NvtxRange range("kg_eval");
  kg_status s = check_state(h);
  if (s) return s;
  if (!q || !ans_off || !ans_ids || !ranks || !metrics || n_neg < 0 || (n_neg > 0 && !negatives))
    return fail(h, KG_EINVAL, "null argument");
  const int M = q->M;
  if (M < 1 || M > h->Mx) return fail(h, KG_EINVAL, "M out of range [1, max_M]");
  if (ans_off[0] != 0) return fail(h, KG_EINVAL, "ans_off[0] must be 0");
  int64_t max_ans = 0;
  for (int i = 0; i < M; ++i) {
    const int64_t n = ans_off[i + 1] - ans_off[i];
    if (n < 1) return fail(h, KG_EINVAL, "every query needs at least one missing answer");
    max_ans = std::max(max_ans, n);
  }
  const int64_t n_ans = ans_off[M];
  if ((max_ans + n_neg) * 4 > 200 * 1024) return fail(h, KG_EINVAL, "answers + negatives per query exceed 51200");
  for (int64_t k = 0; k < n_ans; ++k)
    if (ans_ids[k] < 0 || ans_ids[k] >= h->n_ent) return fail(h, KG_EINVAL, "answer id out of range");
  for (int64_t k = 0; k < (int64_t)M * n_neg; ++k)
    if (negatives[k] < 0 || negatives[k] >= h->n_ent) return fail(h, KG_EINVAL, "negative id out of range");
  StepBufs S;
  CallBufs B(h);
  if ((s = embed_queries(h, q, S, 0, B)) != KG_OK) return s;
  cudaStream_t st = h->st;
  // world > 1: the answer and negative rows come from their owners (collective); the kernel
  // then reads them by position in the fetched buffer
  const float *ent = h->ent_src;
  std::vector<int64_t> pos_ids;
  if (h->world > 1) {
    const int64_t nc = n_ans + (int64_t)M * n_neg;
    std::vector<int64_t> all(nc);
    std::copy(ans_ids, ans_ids + n_ans, all.begin());
    if (n_neg > 0) std::copy(negatives, negatives + (int64_t)M * n_neg, all.begin() + n_ans);
    float *X = B.get<float>(nc * h->d);
    if (!X) return fail(h, KG_ENOMEM, "eval row buffer");
    if ((s = fetch_rows(h, all.data(), nc, h->t.ent, X, B)) != KG_OK) return s;
    pos_ids.resize(nc);
    for (int64_t i = 0; i < nc; ++i) pos_ids[i] = i;
    ans_ids = pos_ids.data();
    negatives = pos_ids.data() + n_ans;
    ent = X;
  }
  // per-call buffers (the evaluation path is not part of the captured training step)
  int64_t *d_off = nullptr, *d_ans = nullptr, *d_neg = nullptr;
  int32_t *d_ranks = nullptr;
  float *d_met = nullptr;
  CK(cudaMallocAsync(&d_off, sizeof(int64_t) * (M + 1), st));
  CK(cudaMallocAsync(&d_ans, sizeof(int64_t) * n_ans, st));
  CK(cudaMallocAsync(&d_neg, sizeof(int64_t) * std::max<int64_t>(1, (int64_t)M * n_neg), st));
  CK(cudaMallocAsync(&d_ranks, sizeof(int32_t) * n_ans, st));
  CK(cudaMallocAsync(&d_met, sizeof(float) * 4 * M, st));
  CK(cudaMemcpyAsync(d_off, ans_off, sizeof(int64_t) * (M + 1), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_ans, ans_ids, sizeof(int64_t) * n_ans, cudaMemcpyHostToDevice, st));
  if (n_neg > 0) CK(cudaMemcpyAsync(d_neg, negatives, sizeof(int64_t) * M * n_neg, cudaMemcpyHostToDevice, st));
  EvalArgs a;
  a.Q = h->Q; a.ent = ent; a.ans_off = d_off; a.ans_ids = d_ans; a.negatives = d_neg;
  a.M = M; a.d = h->d; a.U = (h->sk == KG_BETAE || h->sk == KG_ROTATE || h->sk == KG_COMPLEX) ? h->m : h->d;
  a.n_neg = n_neg; a.max_ans = (int)max_ans; a.alpha = h->cfg.box_alpha; a.ranks = d_ranks; a.metrics = d_met;
  launch_eval(h->sk, a, S.plan.nout, st);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(ranks, d_ranks, sizeof(int32_t) * n_ans, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(metrics, d_met, sizeof(float) * 4 * M, cudaMemcpyDeviceToHost, st));
  CK(cudaFreeAsync(d_off, st));
  CK(cudaFreeAsync(d_ans, st));
  CK(cudaFreeAsync(d_neg, st));
  CK(cudaFreeAsync(d_ranks, st));
  CK(cudaFreeAsync(d_met, st));
  CK(cudaStreamSynchronize(st));
  return KG_OK;
}

static float *table_of(kg_handle *h, int which) {
  return which == 0 ? h->t.ent : (which == 1 ? h->t.ent_m : (which == 2 ? h->t.ent_v : nullptr));
}

kg_status kg_read_rows(kg_handle *h, int32_t which, const int64_t *ids, int32_t n, float *out) {
  kg_status s = check_state(h);
  if (s) return s;
  float *tab = table_of(h, which);
  if (!tab || !ids || !out || n < 0) return fail(h, KG_EINVAL, "bad argument");
  std::vector<int64_t> rows(n);
  for (int i = 0; i < n; ++i) {
    if (ids[i] < 0 || ids[i] >= h->n_ent || ids[i] % h->world != h->rank) return fail(h, KG_EINVAL, "id not owned");
    rows[i] = ids[i] / h->world;
  }
  if (n == 0) return KG_OK;
  int64_t *drows = nullptr;
  float *buf = nullptr;
  CK(cudaMalloc(&drows, sizeof(int64_t) * n));
  CK(cudaMalloc(&buf, sizeof(float) * (size_t)n * h->d));
  CK(cudaMemcpyAsync(drows, rows.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice, h->st));
  launch_gather_rows(buf, tab, drows, n, h->d, h->st);
  CK(cudaMemcpyAsync(out, buf, sizeof(float) * (size_t)n * h->d, cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  cudaFree(drows);
  cudaFree(buf);
  return KG_OK;
}

kg_status kg_gather_rows(kg_handle *h, int32_t which, const int64_t *ids, int32_t n, float *out) {
  kg_status s = check_state(h);
  if (s) return s;
  float *tab = table_of(h, which);
  if (!tab || (n > 0 && (!ids || !out)) || n < 0) return fail(h, KG_EINVAL, "bad argument");
  for (int i = 0; i < n; ++i)
    if (ids[i] < 0 || ids[i] >= h->n_ent) return fail(h, KG_EINVAL, "id out of range");
  if (h->world == 1) return n ? kg_read_rows(h, which, ids, n, out) : KG_OK;
  CallBufs B(h);
  float *X = B.get<float>((int64_t)n * h->d);
  if (!X) return fail(h, KG_ENOMEM, "gather buffer");
  if ((s = fetch_rows(h, ids, n, tab, X, B)) != KG_OK) return s;
  if (n) CK(cudaMemcpyAsync(out, X, sizeof(float) * (size_t)n * h->d, cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  return KG_OK;
}

kg_status kg_write_rows(kg_handle *h, int32_t which, const int64_t *ids, int32_t n, const float *in) {
  kg_status s = check_state(h);
  if (s) return s;
  float *tab = table_of(h, which);
  if (!tab || !ids || !in || n < 0) return fail(h, KG_EINVAL, "bad argument");
  std::vector<int64_t> rows(n);
  for (int i = 0; i < n; ++i) {
    if (ids[i] < 0 || ids[i] >= h->n_ent || ids[i] % h->world != h->rank) return fail(h, KG_EINVAL, "id not owned");
    rows[i] = ids[i] / h->world;
  }
  if (n == 0) return KG_OK;
  int64_t *drows = nullptr;
  float *buf = nullptr;
  CK(cudaMalloc(&drows, sizeof(int64_t) * n));
  CK(cudaMalloc(&buf, sizeof(float) * (size_t)n * h->d));
  CK(cudaMemcpyAsync(drows, rows.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice, h->st));
  CK(cudaMemcpyAsync(buf, in, sizeof(float) * (size_t)n * h->d, cudaMemcpyHostToDevice, h->st));
  launch_scatter_rows(tab, buf, drows, n, h->d, h->st);
  CK(cudaStreamSynchronize(h->st));
  cudaFree(drows);
  cudaFree(buf);
  return KG_OK;
}

kg_status kg_read_dense(kg_handle *h, int32_t which, float *out) {
  kg_status s = check_state(h);
  if (s) return s;
  float *p = which == 0 ? h->t.dense : (which == 1 ? h->t.dense_m : (which == 2 ? h->t.dense_v : nullptr));
  if (!p || !out) return fail(h, KG_EINVAL, "bad argument");
  CK(cudaMemcpyAsync(out, p, sizeof(float) * h->dense_size, cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  return KG_OK;
}

kg_status kg_write_dense(kg_handle *h, int32_t which, const float *in) {
  kg_status s = check_state(h);
  if (s) return s;
  float *p = which == 0 ? h->t.dense : (which == 1 ? h->t.dense_m : (which == 2 ? h->t.dense_v : nullptr));
  if (!p || !in) return fail(h, KG_EINVAL, "bad argument");
  CK(cudaMemcpyAsync(p, in, sizeof(float) * h->dense_size, cudaMemcpyHostToDevice, h->st));
  CK(cudaStreamSynchronize(h->st));
  return KG_OK;
}

kg_status kg_last_grads(kg_handle *h, int64_t *uniq, float *grad_rows, float *grad_dense, int32_t cap,
                        int32_t *n_uniq, float *d_pos, float *d_neg) {
  kg_status s = check_state(h);
  if (s) return s;
  if (!h->last_U_valid) return fail(h, KG_ESTATE, "no step has run");
  CK(cudaStreamSynchronize(h->st));
  int32_t U = 0, rU = 0;
  CK(cudaMemcpy(&U, h->Udev, sizeof(int32_t), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&rU, h->rU, sizeof(int32_t), cudaMemcpyDeviceToHost));
  if (n_uniq) *n_uniq = U;
  if ((uniq || grad_rows) && U > cap) return fail(h, KG_EINVAL, "cap < number of touched rows");
  if (uniq) CK(cudaMemcpy(uniq, h->uniq, sizeof(int64_t) * U, cudaMemcpyDeviceToHost));
  if (grad_rows) {
    if (!h->keep_grads) return fail(h, KG_ESTATE, "enable gradient capture with kg_set_apply(h, flags | 2)");
    CK(cudaMemcpy(grad_rows, h->Gc, sizeof(float) * (size_t)U * h->d, cudaMemcpyDeviceToHost));
  }
  if (grad_dense) {
    std::memset(grad_dense, 0, sizeof(float) * h->dense_size);
    if (h->dense_size > h->w_off)
      CK(cudaMemcpy(grad_dense + h->w_off, h->gdense, sizeof(float) * (h->dense_size - h->w_off),
                    cudaMemcpyDeviceToHost));
    std::vector<int64_t> ru(rU);
    std::vector<float> rg((size_t)rU * h->dr);
    CK(cudaMemcpy(ru.data(), h->runiq, sizeof(int64_t) * rU, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(rg.data(), h->RGU, sizeof(float) * rg.size(), cudaMemcpyDeviceToHost));
    for (int k = 0; k < rU; ++k) {
      const int64_t r = ru[k];
      if (h->kind == KG_Q2B) {
        const Seg *c = seg_of(h, "rel_center"), *o = seg_of(h, "rel_offset");
        std::memcpy(grad_dense + c->off + r * h->d, &rg[(size_t)k * h->dr], sizeof(float) * h->d);
        std::memcpy(grad_dense + o->off + r * h->d, &rg[(size_t)k * h->dr + h->d], sizeof(float) * h->d);
      } else {
        const Seg &s0 = h->segs[0];
        std::memcpy(grad_dense + s0.off + r * s0.cols, &rg[(size_t)k * h->dr], sizeof(float) * s0.cols);
      }
    }
  }
  if (d_pos) CK(cudaMemcpy(d_pos, h->Dpos, sizeof(float) * h->last_M, cudaMemcpyDeviceToHost));
  if (d_neg && h->last_K > 0)
    CK(cudaMemcpy(d_neg, h->Dmin, sizeof(float) * (size_t)h->last_M * h->last_K, cudaMemcpyDeviceToHost));
  return KG_OK;
}

kg_status kg_set_apply(kg_handle *h, int32_t flags) {
  if (!h) return KG_EINVAL;
  h->apply = flags & 1;
  h->keep_grads = (flags >> 1) & 1;
  h->timing = (flags >> 2) & 1;
  return KG_OK;
}

const char *kg_last_error(const kg_handle *h) { return h ? h->err.c_str() : "null handle"; }

kg_status kg_test_gemm(int32_t ta, int32_t tb, int32_t M, int32_t N, int32_t K, const float *A, int32_t lda,
                       const float *B, int32_t ldb, float *C, int32_t ldc, const float *bias, int32_t relu, float beta,
                       void *stream) {
  if (!A || !B || !C || M < 0 || N < 0 || K < 1) return KG_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  GemmArgs g;
  g.A = A; g.B = B; g.C = C; g.bias = bias; g.M = M; g.N = N; g.K = K; g.lda = lda; g.ldb = ldb; g.ldc = ldc;
  g.relu = relu & 1; g.beta = beta; g.a_mn = ta != 0; g.b_mn = tb != 0; g.drain = (relu & 2) != 0;
  g.force = (relu >> 2) & 63;   // tile experiments (tools/gemm_tiles.py, tools/gemm_events.py)
  const int reps = std::max(1, relu >> 8);   // back-to-back launches (event timing, tools/gemm_events.py)
  if (!gemm_tc_accepts(g)) return KG_EINVAL;   // 16-byte aligned operands with ld % 4 == 0
  float *sP = nullptr;
  const int64_t pcap = 8LL * std::max(M, 1) * std::max(N, 1);
  if (cudaMalloc(&sP, sizeof(float) * pcap) != cudaSuccess) return KG_ENOMEM;
  bool launched = true;
  for (int r = 0; r < reps && launched; ++r) launched = launch_gemm_tc(g, sP, pcap, st);
  const cudaError_t e = cudaStreamSynchronize(st);
  cudaFree(sP);
  if (!launched) return KG_EUNSUPPORTED;   // tensor map encoding failed
  if (e != cudaSuccess) return KG_ECUDA;
  return cudaGetLastError() == cudaSuccess ? KG_OK : KG_ECUDA;
}

kg_status kg_get_step(kg_handle *h, int64_t *t) {
  kg_status s = check_state(h);
  if (s) return s;
  if (!t) return fail(h, KG_EINVAL, "null pointer");
  CK(cudaStreamSynchronize(h->st));
  h->step_pending = false;
  CK(cudaMemcpy(t, h->t_dev, sizeof(int64_t), cudaMemcpyDeviceToHost));
  return KG_OK;
}

kg_status kg_set_step(kg_handle *h, int64_t t) {
  kg_status s = check_state(h);
  if (s) return s;
  if (t < 0) return fail(h, KG_EINVAL, "negative step");
  CK(cudaStreamSynchronize(h->st));
  h->step_pending = false;
  CK(cudaMemcpy(h->t_dev, &t, sizeof(int64_t), cudaMemcpyHostToDevice));
  return KG_OK;
}

kg_status kg_nccl_unique_id(void *out) {
  if (!out) return KG_EINVAL;
  ncclUniqueId id;
  if (!nccl().ok || nccl().GetUniqueId(&id) != ncclSuccess) return KG_ENCCL;
  std::memcpy(out, &id, sizeof(id));
  return KG_OK;
}

void kg_destroy(kg_handle *h) {
  if (!h) return;
  if (h->st) cudaStreamSynchronize(h->st);
  else cudaDeviceSynchronize();
  if (h->st2) { cudaStreamSynchronize(h->st2); cudaStreamDestroy(h->st2); }
  if (h->st_cap) cudaStreamDestroy(h->st_cap);
  if (h->st3) { cudaStreamSynchronize(h->st3); cudaStreamDestroy(h->st3); }
  if (h->st4) { cudaStreamSynchronize(h->st4); cudaStreamDestroy(h->st4); }
  if (h->st5) { cudaStreamSynchronize(h->st5); cudaStreamDestroy(h->st5); }
  if (h->ev_wjoin) cudaEventDestroy(h->ev_wjoin);
  if (h->ev_bent) cudaEventDestroy(h->ev_bent);
  if (h->ev_i1) cudaEventDestroy(h->ev_i1);
  if (h->ev_i2) cudaEventDestroy(h->ev_i2);
  for (auto &g : h->graphs) cudaGraphExecDestroy(g.exec);
  if (h->ev_fork2) cudaEventDestroy(h->ev_fork2);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  for (int i = 0; i < 2; ++i) {
    if (h->pin[i]) cudaFreeHost(h->pin[i]);
    if (h->pin_ev[i]) cudaEventDestroy(h->pin_ev[i]);
  }
  if (h->hout) cudaFreeHost(h->hout);
  if (h->step_done) cudaEventDestroy(h->step_done);
  for (int i = 0; i < 2; ++i)
    if (h->res_ev[i]) cudaEventDestroy(h->res_ev[i]);
  for (int i = 0; i < 12; ++i)
    if (h->sev[i]) cudaEventDestroy(h->sev[i]);
  if (h->ev_rel) cudaEventDestroy(h->ev_rel);
  if (h->ev_loss) cudaEventDestroy(h->ev_loss);
  if (h->ev_early) cudaEventDestroy(h->ev_early);
  for (void *p : h->ipc_opened) cudaIpcCloseMemHandle(p);
  if (h->comm2) nccl().CommDestroy(h->comm2);
  if (h->comm) nccl().CommDestroy(h->comm);
  if (h->h_counts) cudaFreeHost(h->h_counts);
  if (h->ws) cudaFree(h->ws);
  delete h;
}

}  // extern "C"
