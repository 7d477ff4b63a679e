// TEST backend of fo::Comm (comm.h): W ranks of one process on ONE GPU.
//
// A single-GPU box cannot run NCCL with two ranks (one device per rank), so
// without this the library's multi-rank data path (the RS / A2A receive
// buffers, the per-group calls on the comm stream, the last group on the
// caller stream, the sequential schedules) would first run on real peers at
// the driver's round-end scaling bench.  fo_loopback_create makes a group of W
// in-process ranks on one device; fo_ctx_create_loopback gives each rank a
// context whose communication calls are small kernels:
//
//   1. publish: block 0 writes (src, dst, count, p2p descriptors) into the
//      rank's mailbox slot of this call (slot = call number mod RING);
//   2. arrive: every CTA of every rank adds 1 to the slot's arrive counter
//      (release) and waits until all W*G CTAs of the call arrived (acquire) —
//      the point where every rank's data (written by its GEMM, earlier in its
//      stream order) is visible;
//   3. move the data with plain loads / stores through the other ranks'
//      mailbox pointers (same address space): AllReduce — rank r sums chunk r
//      of the range over all ranks (fp32, rank order, one bf16 rounding) and
//      writes it into EVERY rank's buffer (each element is touched by one
//      rank only, so in-place is safe); ReduceScatter / AllGather — rank r
//      fills its own receive buffer; grouped send/recv — rank r copies each
//      of its receives from the matching send of the peer (k-th receive from
//      s = k-th send from s to r, counts must match: NCCL's pairing);
//   4. depart: the same barrier again, so no rank moves on (e.g. its next
//      GEMM overwriting the send buffer) while another still reads from it.
//
// Mismatched call sequences (a hang with NCCL) are detected instead: a count
// or pairing mismatch, or a barrier not reached within kTimeoutNs, records an
// error code and traps (the process's CUDA context dies loudly; tests run it
// in a subprocess).  All ranks must call in the same order, as with NCCL.
// Not CUDA-graph capturable (descriptors are written by the host at issue).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <ctime>
#include <cstring>
#include <memory>
#include <mutex>
#include <vector>

#include "comm.h"
#include "common.h"
#include "kernels.h"

namespace fo {

namespace {

constexpr int kRing = 64;           // mailbox / descriptor slots per rank
constexpr int kMaxDesc = 8192;      // p2p descriptors per (slot, rank)
// CTAs per loopback call and rank: every CTA of a call on every rank must be
// resident at once (they meet at the barrier), so W * ctas stays at 128
// (beside the ranks' GEMMs, which leave no registers for these kernels on
// their SMs)
inline int lb_ctas(int world) { return world >= 32 ? 4 : (128 / world > 32 ? 32 : 128 / world); }
constexpr unsigned long long kTimeoutNs = 20ull * 1000 * 1000 * 1000;

enum LbKind : int { LB_ALLREDUCE = 0, LB_REDUCESCATTER = 1, LB_ALLGATHER = 2, LB_P2P = 3 };

struct LbDesc {
  int kind;  // 0 send, 1 recv
  int peer;
  void* ptr;
  long long count;
};

struct LbMail {
  const void* src;
  void* dst;
  long long count;
  int kind;
  int ndesc;
  const LbDesc* desc;
};

struct LbArgs {
  int kind, rank, world, slot;
  unsigned target;           // W * ctas * (uses of this slot so far, this one included)
  const void* src;
  void* dst;
  long long count;
  int ndesc;
  const LbDesc* desc;        // pinned host, mapped
  LbMail* mail;              // device [kRing][world]
  unsigned* ctr;             // device [kRing][2] arrive / depart (monotone)
  int* err;                  // device: first error code
  const int* abort_flag;     // pinned host, mapped: set by abort()
  int trace;                 // FO_LOOPBACK_TRACE=2: per-call phase times from CTA 0
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void red_release(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned long long now_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ void fail_trap(int* err, int code) {
  printf("loopback communicator: schedule mismatch / timeout (code %d, block %d) - trapping\n", code, blockIdx.x);
  atomicCAS(err, 0, code);
  __threadfence_system();
  __trap();
}

// every CTA: arrive, then wait for all W*G CTAs of the call
__device__ void barrier(const LbArgs& a, unsigned* c) {
  __syncthreads();
  if (threadIdx.x == 0) {
    red_release(c, 1u);
    const unsigned long long t0 = now_ns();
    while ((int)(ld_acquire(c) - a.target) < 0) {
      if (*(volatile const int*)a.abort_flag) break;  // (host-mapped: one PCIe read per spin, thread 0 only)
      if (now_ns() - t0 > kTimeoutNs) {
        printf("loopback rank %d kind %d slot %d: barrier %s counter %u target %u (waiting since t=%llu ms)\n",
               a.rank, a.kind, a.slot, (c == a.ctr + (size_t)a.slot * 2) ? "arrive" : "depart", ld_acquire(c),
               a.target, (t0 / 1000000ull) % 1000000ull);
        fail_trap(a.err, 1000 + a.kind);
      }
      __nanosleep(256);
    }
  }
  __syncthreads();
}

__device__ __forceinline__ float b2f(unsigned short v) { return __uint_as_float((unsigned)v << 16); }
__device__ __forceinline__ unsigned short f2b(float f) {  // round to nearest even (finite values)
  unsigned u = __float_as_uint(f);
  if ((u & 0x7f800000u) == 0x7f800000u) return (unsigned short)(u >> 16 | ((u & 0xffff) ? 0x40 : 0));
  u += 0x7fffu + ((u >> 16) & 1u);
  return (unsigned short)(u >> 16);
}

// grid-wide copy of n bf16: 16-byte vectors, 4 in flight per thread, when aligned
__device__ void lb_copy(unsigned short* __restrict__ dst, const unsigned short* __restrict__ src, long long n,
                        long long tid, long long nthr) {
  if (n % 8 == 0 && !(reinterpret_cast<uintptr_t>(dst) & 15) && !(reinterpret_cast<uintptr_t>(src) & 15)) {
    const long long step = 8 * nthr;
    for (long long e0 = 8 * tid; e0 < n; e0 += 4 * step) {
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (e0 + u * step < n) v[u] = *reinterpret_cast<const uint4*>(src + e0 + u * step);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (e0 + u * step < n) *reinterpret_cast<uint4*>(dst + e0 + u * step) = v[u];
    }
  } else {
    for (long long e = tid; e < n; e += nthr) dst[e] = src[e];
  }
}

__global__ void __launch_bounds__(256) lb_kernel(const LbArgs a) {
  LbMail* mail = a.mail + (size_t)a.slot * a.world;
  unsigned* ctr = a.ctr + (size_t)a.slot * 2;
  const unsigned long long t_start = (a.trace && threadIdx.x == 0) ? now_ns() : 0ull;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    LbMail m;
    m.src = a.src;
    m.dst = a.dst;
    m.count = a.count;
    m.kind = a.kind;
    m.ndesc = a.ndesc;
    m.desc = a.desc;
    mail[a.rank] = m;
    __threadfence();
  }
  barrier(a, ctr + 0);
  const unsigned long long t_arrived = (a.trace && threadIdx.x == 0) ? now_ns() : 0ull;
  {
    __shared__ int s_abort;
    if (threadIdx.x == 0) s_abort = *(volatile const int*)a.abort_flag;
    __syncthreads();
    if (s_abort) return;
  }
  // every rank must be in the same kind of call with the same count
  if (threadIdx.x == 0 && blockIdx.x == 0)
    for (int q = 0; q < a.world; ++q) {
      const LbMail mq = mail[q];
      if (mq.kind != a.kind || (a.kind != LB_P2P && mq.count != a.count)) fail_trap(a.err, 2000 + q);
    }
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nthr = (long long)gridDim.x * blockDim.x;
  const int W = a.world;
  // 16-byte vectors (8 bf16) when every pointer and the count allow it
  auto al16 = [](const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; };
  if (a.kind == LB_ALLREDUCE || a.kind == LB_REDUCESCATTER) {
    const bool ar = a.kind == LB_ALLREDUCE;
    // the ranks' pointers, once (the mailbox is global memory the stores
    // below might alias, so the compiler would reload it every element)
    __shared__ const unsigned short* s_src[64];
    __shared__ unsigned short* s_dst[64];
    if (threadIdx.x < W) {
      s_src[threadIdx.x] = reinterpret_cast<const unsigned short*>(mail[threadIdx.x].src);
      s_dst[threadIdx.x] = reinterpret_cast<unsigned short*>(mail[threadIdx.x].dst);
    }
    __syncthreads();
    // AllReduce: rank r reduces chunk r of the range into EVERY rank's buffer;
    // ReduceScatter: rank r reduces block r of the sources into its own buffer
    const long long lo = ar ? a.count * a.rank / W : 0, hi = ar ? a.count * (a.rank + 1) / W : a.count;
    const long long soff = ar ? 0 : a.count * a.rank;
    unsigned short* mydst = reinterpret_cast<unsigned short*>(a.dst);
    bool vec = (a.count % 8 == 0) && (lo % 8 == 0) && (hi % 8 == 0) && al16(mydst);
    for (int q = 0; q < W && vec; ++q) vec = al16(s_src[q]) && (ar ? al16(s_dst[q]) : true);
    if (vec) {
      constexpr int U = 4;  // vectors per thread in flight
      const long long step = 8 * nthr;
      for (long long e0 = lo + 8 * tid; e0 < hi; e0 += U * step) {
        float acc[U][8];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[u][i] = 0.f;
        for (int q = 0; q < W; ++q) {
          uint4 v[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const long long e = e0 + u * step;
            if (e < hi) v[u] = *reinterpret_cast<const uint4*>(s_src[q] + soff + e);
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const unsigned short* h = reinterpret_cast<const unsigned short*>(&v[u]);
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[u][i] += b2f(h[i]);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const long long e = e0 + u * step;
          if (e >= hi) continue;
          uint4 o;
          unsigned short* ho = reinterpret_cast<unsigned short*>(&o);
#pragma unroll
          for (int i = 0; i < 8; ++i) ho[i] = f2b(acc[u][i]);
          if (ar) {
            for (int q = 0; q < W; ++q) *reinterpret_cast<uint4*>(s_dst[q] + e) = o;
          } else {
            *reinterpret_cast<uint4*>(mydst + e) = o;
          }
        }
      }
    } else {
      for (long long e = lo + tid; e < hi; e += nthr) {
        float acc = 0.f;
        for (int q = 0; q < W; ++q) acc += b2f(s_src[q][soff + e]);
        const unsigned short v = f2b(acc);
        if (ar) {
          for (int q = 0; q < W; ++q) s_dst[q][e] = v;
        } else {
          mydst[e] = v;
        }
      }
    }
  } else if (a.kind == LB_ALLGATHER) {
    for (int q = 0; q < W; ++q)
      lb_copy(reinterpret_cast<unsigned short*>(a.dst) + q * a.count,
              reinterpret_cast<const unsigned short*>(mail[q].src), a.count, tid, nthr);
  } else {
    // every receive of mine: the matching send of the peer (k-th receive
    // from s = k-th send from s to me, counts equal), copied by all CTAs
    for (int i = 0; i < a.ndesc; ++i) {
      const LbDesc d = a.desc[i];
      if (d.kind != 1) continue;
      int k = 0;
      for (int t = 0; t < i; ++t) k += (a.desc[t].kind == 1 && a.desc[t].peer == d.peer);
      const LbMail ms = mail[d.peer];
      long long found = -1;
      for (int t = 0, seen = 0; t < ms.ndesc; ++t) {
        const LbDesc sd = ms.desc[t];
        if (sd.kind == 0 && sd.peer == a.rank) {
          if (seen == k) {
            found = t;
            break;
          }
          ++seen;
        }
      }
      if (found < 0 || ms.desc[found].count != d.count) {
        if (threadIdx.x == 0) fail_trap(a.err, 3000 + d.peer);
        return;
      }
      lb_copy(reinterpret_cast<unsigned short*>(d.ptr), reinterpret_cast<const unsigned short*>(ms.desc[found].ptr),
              d.count, tid, nthr);
    }
    // every send of mine must be received by its peer (else the peer's
    // receive list is short: NCCL would hang)
    if (blockIdx.x == 0 && threadIdx.x == 0)
      for (int q = 0; q < W; ++q) {
        if (q == a.rank) continue;
        int sends = 0, recvs = 0;
        for (int t = 0; t < a.ndesc; ++t) sends += (a.desc[t].kind == 0 && a.desc[t].peer == q);
        const LbMail mq = mail[q];
        for (int t = 0; t < mq.ndesc; ++t) recvs += (mq.desc[t].kind == 1 && mq.desc[t].peer == a.rank);
        if (sends != recvs) fail_trap(a.err, 4000 + q);
      }
  }
  __threadfence();
  const unsigned long long t_moved = (a.trace && threadIdx.x == 0) ? now_ns() : 0ull;
  barrier(a, ctr + 1);
  if (a.trace && threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1))
    printf("[lb] rank %d cta %d kind %d count %lld: arrive %.1f us, move %.1f us, depart %.1f us\n", a.rank,
           blockIdx.x, a.kind, a.count, (t_arrived - t_start) / 1e3, (t_moved - t_arrived) / 1e3,
           (now_ns() - t_moved) / 1e3);
}

}  // namespace

// ---------------------------------------------------------------- shared group state
struct LoopbackGroup {
  int device = 0, world = 1;
  LbMail* mail = nullptr;   // device
  unsigned* ctr = nullptr;  // device
  int* err = nullptr;       // device
  int* abort_flag = nullptr;  // pinned mapped host
  LbDesc* arena = nullptr;  // pinned mapped host [kRing][world][kMaxDesc]
  int members = 0;
  std::mutex mu;
};

namespace {

unsigned long long wall_ms() {  // same clock domain as %globaltimer (ns since the epoch), in ms mod 1e6
  timespec ts;
  clock_gettime(CLOCK_REALTIME, &ts);
  return ((unsigned long long)ts.tv_sec * 1000ull + ts.tv_nsec / 1000000) % 1000000ull;
}

struct LoopbackComm final : Comm {
  LoopbackGroup* g;
  int r;
  unsigned long long seq = 0;
  bool in_group = false;
  cudaStream_t group_stream = nullptr;
  std::vector<LbDesc> pending;
  cudaEvent_t slot_done[kRing] = {};
  bool trace_ = false;
  int trace_level_ = 0;
  LoopbackComm(LoopbackGroup* g_, int r_) : g(g_), r(r_) {
    const char* t = getenv("FO_LOOPBACK_TRACE");
    trace_level_ = t ? atoi(t) : 0;
    trace_ = trace_level_ == 1;
  }
  ~LoopbackComm() override {
    for (auto& e : slot_done)
      if (e) cudaEventDestroy(e);
    std::lock_guard<std::mutex> lk(g->mu);
    --g->members;
  }
  int rank() const override { return r; }
  int world() const override { return g->world; }

  // the slot of the next call; its previous use (kRing calls ago, whose peers
  // have all been issued by now) must be finished before its descriptors are
  // overwritten
  int next_slot(unsigned* target) {
    const int slot = (int)(seq % kRing);
    *target = (unsigned)(g->world * lb_ctas(g->world)) * (unsigned)(seq / kRing + 1);
    ++seq;
    if (slot_done[slot]) {
      cudaError_t e = cudaEventSynchronize(slot_done[slot]);
      if (e != cudaSuccess) fail(FO_ERR_CUDA, "loopback: %s", cudaGetErrorString(e));
    }
    return slot;
  }
  void launch(int kind, const void* src, void* dst, long long count, const std::vector<LbDesc>* desc,
              cudaStream_t s) {
    LbArgs a{};
    unsigned target = 0;
    a.slot = next_slot(&target);
    a.target = target;
    a.kind = kind;
    a.rank = r;
    a.world = g->world;
    a.src = src;
    a.dst = dst;
    a.count = count;
    a.mail = g->mail;
    a.ctr = g->ctr;
    a.err = g->err;
    a.abort_flag = g->abort_flag;
    a.trace = trace_level_ >= 2;
    if (desc) {
      if ((int)desc->size() > kMaxDesc) fail(FO_ERR_UNSUPPORTED, "loopback: %zu p2p calls in one group", desc->size());
      LbDesc* slot_desc = g->arena + ((size_t)a.slot * g->world + r) * kMaxDesc;
      if (!desc->empty()) std::memcpy(slot_desc, desc->data(), sizeof(LbDesc) * desc->size());
      a.desc = slot_desc;
      a.ndesc = (int)desc->size();
    }
    if (trace_)
      fprintf(stderr, "[loopback] t=%llu ms rank %d call %llu slot %d kind %d count %lld ndesc %d stream %p\n",
              wall_ms(), r, seq - 1, a.slot, kind, count, a.ndesc, (void*)s);
    lb_kernel<<<lb_ctas(g->world), 256, 0, s>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) fail(FO_ERR_CUDA, "loopback launch: %s", cudaGetErrorString(e));
    count_launch();
    if (!slot_done[a.slot]) {
      e = cudaEventCreateWithFlags(&slot_done[a.slot], cudaEventDisableTiming);
      if (e != cudaSuccess) fail(FO_ERR_CUDA, "loopback: %s", cudaGetErrorString(e));
    }
    e = cudaEventRecord(slot_done[a.slot], s);
    if (e != cudaSuccess) fail(FO_ERR_CUDA, "loopback: %s", cudaGetErrorString(e));
  }
  void allreduce(const void* send, void* recv, size_t count, cudaStream_t s) override {
    if (send != recv) {  // out of place: copy first, then reduce in place
      cudaError_t e = cudaMemcpyAsync(recv, send, 2 * count, cudaMemcpyDeviceToDevice, s);
      if (e != cudaSuccess) fail(FO_ERR_CUDA, "loopback: %s", cudaGetErrorString(e));
    }
    launch(LB_ALLREDUCE, recv, recv, (long long)count, nullptr, s);
  }
  void reducescatter(const void* send, void* recv, size_t recvcount, cudaStream_t s) override {
    launch(LB_REDUCESCATTER, send, recv, (long long)recvcount, nullptr, s);
  }
  void allgather(const void* send, void* recv, size_t sendcount, cudaStream_t s) override {
    launch(LB_ALLGATHER, send, recv, (long long)sendcount, nullptr, s);
  }
  void group_start() override {
    if (in_group) fail(FO_ERR_STATE, "loopback: nested group");
    in_group = true;
    group_stream = nullptr;
    pending.clear();
  }
  void group_end(cudaStream_t s) override {
    if (!in_group) fail(FO_ERR_STATE, "loopback: group_end without group_start");
    in_group = false;
    if (group_stream && group_stream != s) fail(FO_ERR_UNSUPPORTED, "loopback: one stream per group");
    // an empty group is a matched call too (every rank issues the same groups)
    launch(LB_P2P, nullptr, nullptr, 0, &pending, s);
    pending.clear();
  }
  void p2p(int kind, void* buf, size_t count, int peer, cudaStream_t s) {
    if (peer < 0 || peer >= g->world || peer == r) fail(FO_ERR_INVALID_ARG, "loopback: bad peer %d", peer);
    if (group_stream && group_stream != s) fail(FO_ERR_UNSUPPORTED, "loopback: one stream per group");
    group_stream = s;
    pending.push_back(LbDesc{kind, peer, buf, (long long)count});
  }
  void send(const void* buf, size_t count, int peer, cudaStream_t s) override {
    const bool solo = !in_group;
    if (solo) group_start();
    p2p(0, const_cast<void*>(buf), count, peer, s);
    if (solo) group_end(s);
  }
  void recv(void* buf, size_t count, int peer, cudaStream_t s) override {
    const bool solo = !in_group;
    if (solo) group_start();
    p2p(1, buf, count, peer, s);
    if (solo) group_end(s);
  }
  void abort() override { *(volatile int*)g->abort_flag = 1; }
};

}  // namespace

Comm* make_loopback_comm(LoopbackGroup* g, int rank) {
  std::lock_guard<std::mutex> lk(g->mu);
  ++g->members;
  return new LoopbackComm(g, rank);
}

LoopbackGroup* loopback_create(int device, int world) {
  if (world < 1 || world > 64) fail(FO_ERR_INVALID_ARG, "loopback world %d (1..64)", world);
  // With lazy module loading the first launch of a kernel may wait for the
  // kernels already running — here another rank's call spinning at the
  // barrier for this rank: a deadlock NCCL's one-process-per-GPU never sees.
  {
    typedef CUresult (*GetModeFn)(CUmoduleLoadingMode*);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CUmoduleLoadingMode mode = CU_MODULE_EAGER_LOADING;
    if (cudaGetDriverEntryPoint("cuModuleGetLoadingMode", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess && fn)
      reinterpret_cast<GetModeFn>(fn)(&mode);
    if (mode == CU_MODULE_LAZY_LOADING)
      fail(FO_ERR_UNSUPPORTED,
           "the loopback communicator needs eager module loading: set CUDA_MODULE_LOADING=EAGER before CUDA starts");
  }
  auto* g = new LoopbackGroup();
  g->device = device;
  g->world = world;
  auto ck = [&](cudaError_t e) {
    if (e != cudaSuccess) fail(FO_ERR_CUDA, "loopback_create: %s", cudaGetErrorString(e));
  };
  try {
    ck(cudaSetDevice(device));
    ck(cudaMalloc(&g->mail, sizeof(LbMail) * kRing * world));
    ck(cudaMemset(g->mail, 0, sizeof(LbMail) * kRing * world));
    ck(cudaMalloc(&g->ctr, sizeof(unsigned) * kRing * 2));
    ck(cudaMemset(g->ctr, 0, sizeof(unsigned) * kRing * 2));
    ck(cudaMalloc(&g->err, sizeof(int)));
    ck(cudaMemset(g->err, 0, sizeof(int)));
    ck(cudaHostAlloc(&g->abort_flag, sizeof(int), cudaHostAllocMapped));
    *g->abort_flag = 0;
    ck(cudaHostAlloc(&g->arena, sizeof(LbDesc) * (size_t)kRing * world * kMaxDesc, cudaHostAllocMapped));
  } catch (...) {
    loopback_destroy(g);
    throw;
  }
  return g;
}

void loopback_destroy(LoopbackGroup* g) {
  if (!g) return;
  if (g->mail) cudaFree(g->mail);
  if (g->ctr) cudaFree(g->ctr);
  if (g->err) cudaFree(g->err);
  if (g->abort_flag) cudaFreeHost(g->abort_flag);
  if (g->arena) cudaFreeHost(g->arena);
  delete g;
}

int loopback_members(LoopbackGroup* g) {
  std::lock_guard<std::mutex> lk(g->mu);
  return g->members;
}

int loopback_world(LoopbackGroup* g) { return g->world; }
int loopback_device(LoopbackGroup* g) { return g->device; }

}  // namespace fo
