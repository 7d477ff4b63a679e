// Runtime: NCCL context, device plan state, and the overlapped op
// (PAPER.md:297 fig:framework, PAPER.md:555 two-stream orchestration).
//
// fo_run on the caller stream `s`:
//   1. reset the P group counters (counting table)
//   2. fork: record E0 on s; the comm stream waits on E0
//   3. s: persistent tcgen05 GEMM with the reorder+signal epilogue
//   4. comm stream, for each group j: cuStreamWaitValue32(counter_j >= |G_j|)
//      (a front-end wait, no SM spent — replaces the paper's spinning signal
//      kernel) then the NCCL call on group j's contiguous range
//      — except the last group (FO_OPT_LAST_GROUP_IN_ORDER, default): its
//      collective follows the GEMM on s itself (stream order; s first waits for
//      the comm stream's earlier collectives)
//   5. post-communication reorder (+ fused add / RMSNorm): per group on the
//      post stream, or once after the last collective
//   6. join: s waits for the comm / post streams
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <climits>
#include <thread>
#include <cstring>
#include <mutex>
#include <vector>

#include "comm.h"
#include "kernels.h"
#include "runtime.h"

struct fo_ctx_s {
  int device = 0;
  bool aborted = false;                // the watchdog (fo_plan_sync) aborted the communicator
  int rank = 0, world = 1;
  fo::Comm* comm = nullptr;            // NCCL (owned or borrowed) or the test loopback
  cudaStream_t comm_stream = nullptr;
  cudaStream_t post_stream = nullptr;  // per-group post-reorder, chained to each group's collective
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_post_join = nullptr;
  std::vector<cudaEvent_t> ev_group;   // one per wave group (grown on demand)
  // fo_run_host: chunked H2D of A and per-group D2H of out on their own streams
  cudaStream_t h2d_stream[2] = {nullptr, nullptr}, d2h_stream = nullptr;
  cudaEvent_t ev_h2d_fork = nullptr, ev_h2d_join[2] = {nullptr, nullptr}, ev_d2h_join = nullptr;
  std::vector<cudaEvent_t> ev_d2h;     // group j's output final (grown on demand)
  // NCCL buffer registration (fo_ctx_config.buffers): 0 plain cudaMalloc,
  // 1 ncclMemAlloc + ncclCommRegister, 2 ncclMemAlloc + window registration
  int mem_mode = 0;
  std::vector<fo_plan_s*> reg_plans;   // plans whose buffers are registered with this context's comm
  struct UserBuf {
    void* ptr;
    size_t bytes;
    void* handle;                      // ncclCommRegister handle
    ncclWindow_t win;
  };
  std::vector<UserBuf> user_bufs;      // fo_mem_alloc
};

namespace fo {

#define FO_CUDA(x)                                                                          \
  do {                                                                                      \
    cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess) fail(FO_ERR_CUDA, "%s: %s (%s:%d)", #x, cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)

#define FO_NCCL(x)                                                                          \
  do {                                                                                      \
    ncclResult_t r_ = (x);                                                                  \
    if (r_ != ncclSuccess) fail(FO_ERR_NCCL, "%s: %s (%s:%d)", #x, ncclGetErrorString(r_), __FILE__, __LINE__); \
  } while (0)

// CTAs that run (and signal) one tile: a CTA pair for 256-row tiles
static inline int ctas_per_tile(int BM) { return BM == 256 ? 2 : 1; }

typedef CUresult (*WaitValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*WriteValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

static WriteValue32Fn write_value_fn() {
  static WriteValue32Fn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<WriteValue32Fn>(ptr);
  });
  return fn;
}

static WaitValue32Fn wait_value_fn() {
  static WaitValue32Fn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<WaitValue32Fn>(ptr);
  });
  return fn;
}

// ---- NCCL backend of fo::Comm (comm.h)
struct NcclComm final : Comm {
  ncclComm_t c;
  int r, w;
  bool owns;
  NcclComm(ncclComm_t c_, int r_, int w_, bool o) : c(c_), r(r_), w(w_), owns(o) {}
  ~NcclComm() override {
    if (c && owns) ncclCommDestroy(c);
  }
  int rank() const override { return r; }
  int world() const override { return w; }
  ncclComm_t nccl() const override { return c; }
  void allreduce(const void* send, void* recv, size_t count, cudaStream_t s) override {
    FO_NCCL(ncclAllReduce(send, recv, count, ncclBfloat16, ncclSum, c, s));
  }
  void reducescatter(const void* send, void* recv, size_t recvcount, cudaStream_t s) override {
    FO_NCCL(ncclReduceScatter(send, recv, recvcount, ncclBfloat16, ncclSum, c, s));
  }
  void allgather(const void* send, void* recv, size_t sendcount, cudaStream_t s) override {
    FO_NCCL(ncclAllGather(send, recv, sendcount, ncclBfloat16, c, s));
  }
  void group_start() override { FO_NCCL(ncclGroupStart()); }
  void group_end(cudaStream_t) override { FO_NCCL(ncclGroupEnd()); }
  void send(const void* buf, size_t count, int peer, cudaStream_t s) override {
    FO_NCCL(ncclSend(buf, count, ncclBfloat16, peer, c, s));
  }
  void recv(void* buf, size_t count, int peer, cudaStream_t s) override {
    FO_NCCL(ncclRecv(buf, count, ncclBfloat16, peer, c, s));
  }
  void abort() override {
    // a borrowed communicator is its owner's to abort; drop it either way
    if (c && owns) ncclCommAbort(c);
    c = nullptr;
  }
};

Comm* make_nccl_comm(ncclComm_t comm, int rank, int world, bool owns) { return new NcclComm(comm, rank, world, owns); }

template <class T>
static T* upload(const std::vector<T>& v) {
  if (v.empty()) return nullptr;
  T* d = nullptr;
  FO_CUDA(cudaMalloc(&d, sizeof(T) * v.size()));
  FO_CUDA(cudaMemcpy(d, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
  return d;
}

// Undo the NCCL registration of a plan's send / receive buffers (the
// registering context's communicator must still be alive).
static void deregister_plan(fo_plan_s* p) {
  fo_ctx_s* c = p->reg_ctx;
  if (!c) return;
  ncclComm_t comm = c->comm ? c->comm->nccl() : nullptr;
  if (comm) {
    for (void* h : {p->reg_send, p->reg_recv})
      if (h) ncclCommDeregister(comm, h);
    for (ncclWindow_t w : {p->win_send, p->win_recv})
      if (w) ncclCommWindowDeregister(comm, w);
  }
  p->reg_send = p->reg_recv = nullptr;
  p->win_send = p->win_recv = nullptr;
  auto& v = c->reg_plans;
  v.erase(std::remove(v.begin(), v.end(), p), v.end());
  p->reg_ctx = nullptr;
}

void release_device(fo_plan_s* p) {
  if (p->device < 0) return;
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(p->device);
  deregister_plan(p);
  if (p->d_recv == p->d_send) p->d_recv = nullptr;  // aliased at world 1
  if (p->nccl_mem) {  // send / receive buffers from ncclMemAlloc
    for (void*& b : {std::ref(p->d_send), std::ref(p->d_recv)})
      if (b) {
        ncclMemFree(b);
        b = nullptr;
      }
  }
  for (cudaEvent_t& e : p->ev_set_done)
    if (e) {
      cudaEventDestroy(e);
      e = nullptr;
    }
  for (void* ptr : {(void*)p->d_order, (void*)p->d_pos_of_tile, (void*)p->d_group_of_pos, (void*)p->d_gpos,
                    (void*)p->d_row_slot, (void*)p->d_src_row, (void*)p->d_counters, p->d_send, p->d_recv,
                    p->d_rowmajor, (void*)p->d_recv_dst, p->h_A, p->h_Bt, p->h_out, p->h_res, p->h_gamma,
                    p->h_A2, p->h_out2,
                    (void*)p->d_ws, (void*)p->d_a_ready, (void*)p->d_wave, (void*)p->d_rs_info,
                    (void*)p->d_seg, (void*)p->d_wseg})
    if (ptr) cudaFree(ptr);
  cudaSetDevice(cur);
  p->device = -1;
}

static void ensure_device(fo_plan_s* p) {
  int dev = 0;
  FO_CUDA(cudaGetDevice(&dev));
  if (p->device == dev) return;
  if (p->device >= 0) fail(FO_ERR_STATE, "plan bound to device %d, used on %d", p->device, dev);
  const PlanHost& h = p->host;
  if (!gemm_shape_supported(h.BM, h.BN))
    fail(FO_ERR_UNSUPPORTED, "tile %dx%d not compiled into this build", h.BM, h.BN);
  int sms = 0;
  FO_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (h.S * ctas_per_tile(h.BM) > sms)
    fail(FO_ERR_INVALID_ARG, "workers=%d x %d CTAs exceeds the %d SMs (waves would not be resident)", h.S,
         ctas_per_tile(h.BM), sms);
  if (h.BM == 64 && (h.mn_major || p->tail_split_req > 1 || p->tail_split_req < 0))
    fail(FO_ERR_UNSUPPORTED, "64-row tiles (tcgen05 M=64): K-major operands and no tail split");
  p->free_sms = sms - h.S * ctas_per_tile(h.BM);
  int major = 0, minor = 0;
  FO_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  FO_CUDA(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev));
  if (major != 10 || minor != 0) fail(FO_ERR_UNSUPPORTED, "sm_%d%d device; this build targets sm_100a", major, minor);
  p->device = dev;
  p->d_order = upload(h.order);
  p->d_pos_of_tile = upload(h.pos_of_tile);
  p->d_group_of_pos = upload(h.group_of_pos);
  p->d_gpos = upload(h.gpos);
  p->d_row_slot = upload(h.row_slot);
  if (h.coll == FO_REDUCESCATTER) {
    // per position: {first position, size} of its group; ROWBAND (R40):
    // {first tile-row, tile-rows} of its band
    std::vector<int2> info(h.tiles);
    for (int q = 0; q < h.tiles; ++q) {
      const int g = h.group_of_pos[q];
      info[q] = h.banded() ? make_int2((int)h.band_rows[2 * g], (int)(h.band_rows[2 * g + 1] - h.band_rows[2 * g]))
                           : make_int2(h.gpos[g], h.gpos[g + 1] - h.gpos[g]);
    }
    p->d_rs_info = upload(info);
  }
  p->d_src_row = upload(h.src_row);
  p->d_recv_dst = upload(h.recv_dst);
  // ---- tail split: the R tiles of the last partial wave are split along K
  // over the workers of that wave.  f >= 2: each into f equal K-slices on
  // consecutive workers (R*f <= S); stream-K (-2): their R*KB k-blocks dealt
  // out evenly to the workers in contiguous ranges (at most 4 parts per tile).
  // -3 (DP + suffix helpers, for a last wave of more than S/2 tiles): every
  // tail tile's worker runs k-blocks [0, x) and the S - R idle workers run the
  // suffixes [x, KB) of consecutive tail tiles, x chosen so the busiest helper
  // (ceil(R / (S-R)) suffixes) ends with the owners: the owners stay in
  // k-lockstep (the operand panels stay shared in L2, unlike stream-K) and
  // the wave takes x instead of KB k-blocks.
  // The host lists every worker's K-ranges; the range starting at k-block 0
  // owns the tile (it is its worker's last, the others' first segment, so no
  // owner ever waits on a worker that is itself waiting).
  {
    const int KB = (int)(h.K / 64);
    const int R = h.tiles - (h.T - 1) * h.S;
    int f = p->tail_split_req;
    const bool streamk = (f == -2) && R > 0 && KB >= 2 && R < h.S;
    const bool suffix = (f == -3) && R > 0 && KB >= 4 && 2 * R > h.S && R < h.S;
    if (f == -1) {  // auto: never more slices than k-blocks; no split when under 2
      f = (R > 0 && 2 * R <= h.S) ? std::min(std::min(4, h.S / R), KB) : 1;
      if (f < 2) f = 1;
    }
    if (f > 1 && (R * f > h.S || f > KB))
      fail(FO_ERR_INVALID_ARG, "tail split %d: %d tail tiles x %d slices exceed S=%d or k-blocks=%d", f, R, f, h.S, KB);
    std::vector<GemmSeg> segs;
    std::vector<int32_t> wseg(h.S + 1, 0);
    int nslots = 0;
    const int tail0 = (h.T - 1) * h.S;
    if (streamk || suffix || f > 1) {
      // pieces[w] = (tile, kb0, kb1) of worker w, in global k order
      std::vector<std::vector<std::array<int, 3>>> pieces(h.S);
      if (streamk) {
        const long total = (long)R * KB;
        long L = (total + h.S - 1) / h.S;
        L = std::max<long>(L, (KB + 3) / 4);  // at most ~4 parts per tile
        for (int w = 0; w < h.S; ++w) {
          long g0 = (long)w * L, g1 = std::min(total, g0 + L);
          while (g0 < g1) {
            const int r = (int)(g0 / KB), kb0 = (int)(g0 % KB);
            const int kb1 = (int)std::min<long>(KB, kb0 + (g1 - g0));
            pieces[w].push_back({r, kb0, kb1});
            g0 += kb1 - kb0;
          }
        }
      } else if (suffix) {
        const int H = h.S - R;
        const int per = (R + H - 1) / H;          // suffixes of the busiest helper
        const int y = std::max(1, KB / (1 + per));  // suffix length: x = KB - y ~ per * y
        const int x = KB - y;
        for (int r = 0; r < R; ++r) pieces[r].push_back({r, 0, x});
        for (int hh = 0, r = 0; hh < H; ++hh)
          for (int c = 0; c < R / H + (hh < R % H ? 1 : 0); ++c, ++r) pieces[R + hh].push_back({r, x, KB});
      } else {
        for (int r = 0; r < R; ++r)
          for (int sl = 0; sl < f; ++sl) pieces[r * f + sl].push_back({r, sl * KB / f, (sl + 1) * KB / f});
      }
      // parts per tile and their slots (the non-owner parts of a tile take
      // consecutive slots in k order)
      std::vector<int> nparts(R, 0), first_slot(R, -1);
      for (int w = 0; w < h.S; ++w)
        for (auto& pc : pieces[w]) ++nparts[pc[0]];
      // f-slices also reserve one slot per tile for the owner's own partial
      // (the distributed fold, R34)
      for (int r = 0; r < R; ++r) {
        first_slot[r] = nslots;
        nslots += nparts[r] - 1 + ((streamk || suffix) ? 0 : 1);
      }
      std::vector<int> next_idx(R, 0);
      std::vector<int> next_slot = first_slot;
      for (int w = 0; w < h.S; ++w) {
        wseg[w] = (int)segs.size();
        for (auto& pc : pieces[w]) {
          GemmSeg sg{};
          sg.pos = tail0 + pc[0];
          sg.kb0 = pc[1];
          sg.kb1 = pc[2];
          sg.tt = pc[0];
          sg.nparts = nparts[pc[0]];
          sg.idx = pc[1] == 0 ? 0 : ++next_idx[pc[0]];
          if (sg.nparts == 1) {
            sg.role = 0;
          } else if (pc[1] == 0) {
            sg.role = 1;
            sg.slot = first_slot[pc[0]];
          } else {
            sg.role = 2;
            sg.slot = next_slot[pc[0]]++;
          }
          segs.push_back(sg);
        }
      }
      wseg[h.S] = (int)segs.size();
    }
    const bool split = !segs.empty();
    p->split = split ? std::max(2, f) : 1;
    p->tail_pos = split ? tail0 : h.tiles;
    p->units = split ? tail0 + (int)segs.size() : h.tiles;
    const int cg = ctas_per_tile(h.BM);
    p->dist_fold = split && !streamk && !suffix;
    p->ctr_words = h.P + (split ? R * cg * (p->dist_fold ? 2 : 1) : 0);
    if (split) {
      p->d_seg = upload(segs);
      p->d_wseg = upload(wseg);
      if (nslots > 0) FO_CUDA(cudaMalloc(&p->d_ws, sizeof(float) * (size_t)nslots * h.BM * h.BN));
    }
  }
  FO_CUDA(cudaMalloc(&p->d_wave, sizeof(uint32_t) * (size_t)h.T));
  FO_CUDA(cudaMemset(p->d_wave, 0, sizeof(uint32_t) * (size_t)h.T));
  FO_CUDA(cudaMalloc(&p->d_counters, sizeof(uint32_t) * p->ctr_words));
  FO_CUDA(cudaMemset(p->d_counters, 0, sizeof(uint32_t) * p->ctr_words));
  p->d_flags = p->d_counters + h.P;
  // banded plans reduce in place in the output (AR; RS at one rank) or
  // scatter straight into it (RS): no send buffer resp. no receive buffer
  const bool need_send = !(h.coll == FO_NOCOMM || (h.coll == FO_ALLREDUCE && h.banded()) ||
                           (h.coll == FO_REDUCESCATTER && h.banded() && h.world == 1));
  // the buffers NCCL reads and writes: plain device memory, or (a context
  // configured for registration) ncclMemAlloc'd so NCCL can register them
  // for zero-copy / NVLS
  p->nccl_mem = p->mem_mode > 0;
  auto alloc = [&](void** b, size_t bytes) {
    if (p->nccl_mem) FO_NCCL(ncclMemAlloc(b, bytes));
    else FO_CUDA(cudaMalloc(b, bytes));
  };
  if (need_send && h.send_elems) alloc(&p->d_send, 2 * h.send_elems);
  if ((h.coll == FO_REDUCESCATTER || h.coll == FO_ALLTOALL) && h.recv_elems && !h.banded()) {
    // one rank: the receive layout ([group][source 0]) is the send layout, so
    // the collective runs in place (no copy)
    if (h.world == 1) p->d_recv = p->d_send;
    else alloc(&p->d_recv, 2 * h.recv_elems);
  }
}

// Bind a plan to the context it first runs with (its buffers are allocated for
// that context's registration mode) and register its send / receive buffers
// with the context's communicator.  Window registration is collective: every
// rank's first run of the plan (itself collective) performs it.
static void bind_ctx(fo_ctx_s* c, fo_plan_s* p) {
  if (p->device < 0) p->mem_mode = c->comm && c->comm->nccl() ? c->mem_mode : 0;
  ensure_device(p);
  if (p->mem_mode == 0 || p->reg_ctx == c) return;
  if (p->reg_ctx) fail(FO_ERR_STATE, "plan's buffers are registered with another context");
  ncclComm_t comm = c->comm ? c->comm->nccl() : nullptr;
  if (!comm) return;
  const PlanHost& h = p->host;
  const bool sym = p->mem_mode == 2 && h.coll != FO_ALLTOALL;  // equal sizes on every rank
  auto reg = [&](void* b, size_t bytes, void** handle, ncclWindow_t* win) {
    if (!b || !bytes) return;
    if (p->mem_mode == 2) FO_NCCL(ncclCommWindowRegister(comm, b, bytes, win, sym ? NCCL_WIN_COLL_SYMMETRIC : 0));
    else FO_NCCL(ncclCommRegister(comm, b, bytes, handle));
  };
  reg(p->d_send, 2 * (size_t)h.send_elems, &p->reg_send, &p->win_send);
  if (p->d_recv != p->d_send) reg(p->d_recv, 2 * (size_t)h.recv_elems, &p->reg_recv, &p->win_recv);
  p->reg_ctx = c;
  c->reg_plans.push_back(p);
}

static bool is_rmsnorm(int post) { return post == FO_POST_ADD_RMSNORM || post == FO_POST_ADD_RMSNORM_RESIDUAL; }

static GemmArgs gemm_args(fo_plan_s* p, const void* A, const void* Bt, void* dst, int mode, bool signal) {
  const PlanHost& h = p->host;
  GemmArgs a{};
  a.A = A;
  a.Bt = Bt;
  a.mn_major = h.mn_major;
  a.dst = dst;
  a.M = h.M;
  a.N = h.N;
  a.K = h.K;
  a.BM = h.BM;
  a.BN = h.BN;
  a.Mt = h.Mt;
  a.Nt = h.Nt;
  a.tiles = h.tiles;
  a.workers = h.S;
  a.mode = mode;
  a.ldc = h.N;
  a.order = p->d_order;
  a.group_of_pos = p->d_group_of_pos;
  a.gpos = p->d_gpos;
  a.row_slot = p->d_row_slot;
  a.rs_info = p->d_rs_info;
  a.counters = signal ? p->d_counters : nullptr;
  a.h = h.h;
  a.h_log2 = 0;
  while ((1 << a.h_log2) < h.h) ++a.h_log2;
  a.tile_ts = nullptr;
  a.tail_pos = p->tail_pos;
  a.split = p->split;
  a.seg = p->d_seg;
  a.wseg = p->d_wseg;
  a.workspace = p->d_ws;
  a.flags = p->d_flags;
  a.dist_fold = p->dist_fold && p->dist_fold_opt;
  a.done = p->dist_fold ? p->d_flags + (h.tiles - p->tail_pos) * ctas_per_tile(h.BM) : nullptr;
  if (p->a_staged_run) {
    a.a_ready = p->d_a_ready + (size_t)p->host_set * p->a_chunks;
    a.a_epoch = p->a_epoch;
    a.a_chunk_rows = p->a_chunk_rows;
  }
  a.multicast = p->multicast;
  // auto (-1): on for long K, where a wave's panels are long enough for the
  // reversal to matter (measured: -12% HBM reads and -1.4% time at 4096^2 x
  // 14336; within noise or slightly slower at 16 k-blocks)
  a.k_snake = p->k_snake < 0 ? (h.K / 64 >= 64) : p->k_snake;
  a.tma_store_ok = p->tma_store;
  if (p->wave_sync && p->split == 1 && h.T > 1) {
    a.wave_ctr = p->d_wave;
    a.wave_epoch = p->gemm_launches;
  }
  return a;
}

// Epilogue mode + destination of the overlapped GEMM for this plan.
static int epi_mode(const PlanHost& h) {
  switch (h.coll) {
    case FO_ALLREDUCE: return h.layout == FO_LAYOUT_ROWBAND ? EPI_ROWMAJOR : EPI_SLOT;
    case FO_REDUCESCATTER: return h.banded() ? EPI_RS_BAND : EPI_RS;
    case FO_ALLTOALL: return EPI_A2A;
    default: return EPI_ROWMAJOR;
  }
}

static void run_gemm(fo_plan_s* p, const void* A, const void* Bt, void* dst, int mode, bool signal,
                     cudaStream_t s, unsigned long long* tile_ts = nullptr) {
  if (p->host.tiles == 0) return;  // an All-to-All source with no rows (R45): nothing to compute or signal
  if (!A || !Bt || !dst) fail(FO_ERR_INVALID_ARG, "null device pointer");
  GemmArgs a = gemm_args(p, A, Bt, dst, mode, signal);
  if (p->swiglu && mode == EPI_ROWMAJOR) {  // FO_OPT_GEMM_SWIGLU: C is [m, n/2] = silu(gate) * up
    if (p->host.BN != 256 || p->host.coll != FO_NOCOMM || p->host.post != FO_POST_NONE)
      fail(FO_ERR_UNSUPPORTED, "the SwiGLU epilogue needs a no-comm plan, tile_n 256 and post none");
    a.mode = EPI_SWIGLU;
    a.ldc = p->host.N / 2;
  }
  a.tile_ts = tile_ts;
  FO_CUDA(launch_gemm(a, s));
  ++p->gemm_launches;  // every launch of the plan's GEMM advances the wave counters once
}

static void run_post(fo_plan_s* p, int map, const void* src, void* out, const void* residual, const void* gamma,
                     cudaStream_t s) {
  const PlanHost& h = p->host;
  if (h.post != FO_POST_NONE && !residual) fail(FO_ERR_INVALID_ARG, "post op needs a residual");
  if (is_rmsnorm(h.post) && !gamma) fail(FO_ERR_INVALID_ARG, "RMSNorm needs gamma");
  PostArgs a{};
  a.map = map;
  a.op = h.post;
  a.src = src;
  a.out = out;
  a.residual = residual;
  a.gamma = gamma;
  a.rows = h.out_rows;
  a.N = h.N;
  a.BM = h.BM;
  a.BN = h.BN;
  a.Nt = h.Nt;
  a.h = h.h;
  a.pos_of_tile = p->d_pos_of_tile;
  a.src_row = p->d_src_row;
  a.eps = h.eps;
  a.bulk_ok = p->post_bulk;  // the whole-output pass runs after the GEMM
  FO_CUDA(launch_post(a, s));
}

static int post_map(const PlanHost& h) {
  switch (h.coll) {
    case FO_ALLREDUCE: return h.layout == FO_LAYOUT_ROWBAND ? POSTMAP_IDENTITY : POSTMAP_SLOT;
    case FO_REDUCESCATTER: return h.banded() ? POSTMAP_IDENTITY : POSTMAP_RS;
    case FO_ALLTOALL: return h.layout == FO_LAYOUT_ROWBAND ? POSTMAP_IDENTITY : POSTMAP_A2A;
    default: return POSTMAP_IDENTITY;
  }
}

// Each CTA signals once per tile it finishes; a 256-row tile is finished by a
// CTA pair, so group j completes at |G_j| * tile_m/128 signals.
static cuuint32_t signal_target(const PlanHost& h, int j) {
  return (cuuint32_t)(h.group_tiles(j) * ctas_per_tile(h.BM));
}

// Trigger: block the comm stream until group j's counter
// reaches its target — a front-end stream wait (no SM) or the paper's
// signaling kernel (a 1-warp spin on an acquire load).
static void stream_wait(fo_plan_s* p, WaitValue32Fn wait, cudaStream_t cs, int j) {
  // FO_OPT_DEBUG_STALL_GROUP: one more signal than the GEMM will ever send
  const cuuint32_t target = signal_target(p->host, j) + (j == p->debug_stall_group ? 1u : 0u);
  if (p->wait_kernel) {
    FO_CUDA(launch_wait(p->d_counters + j, target, cs));
    return;
  }
  CUresult r = wait(reinterpret_cast<CUstream>(cs), reinterpret_cast<CUdeviceptr>(p->d_counters + j), target,
                    CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) fail(FO_ERR_CUDA, "cuStreamWaitValue32 failed (%d)", (int)r);
}

// Per-group post-reorder (H11b) applies to the non-identity maps
// when the fused op is elementwise per element (none / residual add); RMSNorm
// needs whole rows and runs once after the last group.
// Per-group post kernels run while the persistent GEMM still holds its S
// workers.  With FO_OPT_POST_SM_PARTITION they request more dynamic shared
// memory than a GEMM CTA leaves free on its SM (>= 12 KB of 228 KB), which
// keeps them on the SMs the GEMM left free — the SM partition Alg. 1 assumes
// — instead of co-residing with GEMM CTAs.  Default off:
// measured, the confined fused RMSNorm falls behind the GEMM
// (profiles/r01_predictor_check.txt).
constexpr int kPartitionSmem = 24 * 1024;

// AR / RS ROWBAND with a fused op: every group is a band of complete rows, so
// the op (residual add, RMSNorm over whole rows) can run on the band right
// after the band's AllReduce / ReduceScatter.
static bool band_post(const PlanHost& h) { return h.banded() && h.post != FO_POST_NONE; }

static bool use_group_post(const fo_plan_s* p) {
  const PlanHost& h = p->host;
  if (p->group_post == 0) return false;
  if (band_post(h)) return true;
  const int map = post_map(h);
  return map != POSTMAP_IDENTITY && (h.post == FO_POST_NONE || h.post == FO_POST_ADD);
}

// `after_gemm`: the pass is ordered after the GEMM kernel (the last group on
// the caller stream), so it may use the bulk-staged RMSNorm.
static void run_group_post(fo_plan_s* p, int j, const void* src, void* out, const void* residual,
                           const void* gamma, cudaStream_t s, bool after_gemm = false) {
  const PlanHost& h = p->host;
  if (h.post != FO_POST_NONE && !residual) fail(FO_ERR_INVALID_ARG, "post op needs a residual");
  if (band_post(h)) {
    // in place on the band's output rows [r0*R, r1*R) of out (== src); R =
    // BM (AR) or h (RS: the band's rows that landed on this rank)
    if (is_rmsnorm(h.post) && !gamma) fail(FO_ERR_INVALID_ARG, "RMSNorm needs gamma");
    const int64_t R = h.band_out_rows();
    const int64_t row0 = h.band_rows[2 * j] * R, rows = (h.band_rows[2 * j + 1] - h.band_rows[2 * j]) * R;
    PostArgs a{};
    a.map = POSTMAP_IDENTITY;
    a.op = h.post;
    a.src = reinterpret_cast<const char*>(src) + 2 * row0 * h.N;
    a.out = reinterpret_cast<char*>(out) + 2 * row0 * h.N;
    a.residual = reinterpret_cast<const char*>(residual) + 2 * row0 * h.N;
    a.gamma = gamma;
    a.rows = rows;
    a.N = h.N;
    a.BM = h.BM;
    a.BN = h.BN;
    a.Nt = h.Nt;
    a.h = h.h;
    a.eps = h.eps;
    a.smem_pad = p->post_sm_partition ? kPartitionSmem : 0;
    a.bulk_ok = after_gemm ? p->post_bulk : 0;
    FO_CUDA(launch_post(a, s));
    return;
  }
  GroupPostArgs a{};
  a.map = post_map(h);
  a.op = h.post;
  a.src = src;
  a.out = out;
  a.residual = residual;
  a.N = h.N;
  a.BN = h.BN;
  a.Nt = h.Nt;
  a.R = (h.coll == FO_REDUCESCATTER) ? h.h : h.BM;
  a.pos_begin = h.gpos[j];
  a.pos_end = h.gpos[j + 1];
  a.order = p->d_order;
  if (h.coll == FO_ALLTOALL) {
    const int W = h.world;
    a.sub_begin = h.recv_off[(size_t)j * W];
    a.sub_end = (j + 1 < h.P) ? h.recv_off[(size_t)(j + 1) * W] : h.recv_elems / h.BN;
  }
  a.recv_dst = p->d_recv_dst;
  a.grid_cap = 0;  // default: 4 blocks per SM (warp kernel) / one per SM (bulk kernel)
  a.smem_pad = p->post_sm_partition ? kPartitionSmem : 0;
  FO_CUDA(launch_group_post(a, s));
}

// Execute calls [b, e) of a schedule (PlanHost::calls / seq_calls, the
// fo_plan_export_calls contract) on stream `cs`.  bufs: FO_BUF_SEND, _RECV,
// _OUT, _SCRATCH base pointers.
static void exec_calls(fo_ctx_s* c, const std::vector<fo_comm_call>& calls, size_t b, size_t e, void* const bufs[4],
                       cudaStream_t cs) {
  auto at = [&](int buf, int64_t off) -> char* {
    if (buf < 0 || buf > 3 || !bufs[buf]) fail(FO_ERR_STATE, "schedule names buffer %d, which this run does not have", buf);
    return reinterpret_cast<char*>(bufs[buf]) + 2 * off;
  };
  for (size_t i = b; i < e; ++i) {
    const fo_comm_call& k = calls[i];
    switch (k.kind) {
      case FO_CALL_ALLREDUCE:
        c->comm->allreduce(at(k.src_buf, k.src_off), at(k.dst_buf, k.dst_off), (size_t)k.count, cs);
        break;
      case FO_CALL_REDUCESCATTER:
        c->comm->reducescatter(at(k.src_buf, k.src_off), at(k.dst_buf, k.dst_off), (size_t)k.count, cs);
        break;
      case FO_CALL_SEND:
        c->comm->send(at(k.src_buf, k.src_off), (size_t)k.count, k.peer, cs);
        break;
      case FO_CALL_RECV:
        c->comm->recv(at(k.dst_buf, k.dst_off), (size_t)k.count, k.peer, cs);
        break;
      case FO_CALL_LOCAL_COPY: {
        char* src = at(k.src_buf, k.src_off);
        char* dst = at(k.dst_buf, k.dst_off);
        if (src != dst) FO_CUDA(cudaMemcpyAsync(dst, src, 2 * (size_t)k.count, cudaMemcpyDeviceToDevice, cs));
        break;
      }
      case FO_CALL_GROUP_START:
        c->comm->group_start();
        break;
      case FO_CALL_GROUP_END:
        c->comm->group_end(cs);
        break;
      default:
        fail(FO_ERR_STATE, "unknown schedule call kind %d", k.kind);
    }
  }
}

// The collective of group j ("Once the j-th number reaches
// |G_j|, the communication of G_j starts"): the plan's calls of group j on
// the run's send / receive buffers.
static void group_collective(fo_ctx_s* c, fo_plan_s* p, int j, void* send, void* recv, void* out, cudaStream_t cs) {
  const PlanHost& h = p->host;
  void* const bufs[4] = {send, recv, out, nullptr};
  exec_calls(c, h.calls, (size_t)h.call_begin[j], (size_t)h.call_begin[j + 1], bufs, cs);
}

}  // namespace fo

using namespace fo;

extern "C" {

fo_status fo_device_sm_count(int32_t device, int32_t* sm_count) {
  return guard([&] {
    if (!sm_count) fail(FO_ERR_INVALID_ARG, "null argument");
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) n = 0;
    *sm_count = n;
  });
}

// streams and events of a context (both constructors)
static void init_streams(fo_ctx_s* c) {
  int lo = 0, hi = 0;
  FO_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  // highest priority for the communication stream
  FO_CUDA(cudaStreamCreateWithPriority(&c->comm_stream, cudaStreamNonBlocking, hi));
  // post-reorder one step below the collectives (pending NCCL CTAs are
  // scheduled first), still above default-priority work
  FO_CUDA(cudaStreamCreateWithPriority(&c->post_stream, cudaStreamNonBlocking, hi < lo ? hi + 1 : hi));
  FO_CUDA(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
  FO_CUDA(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  FO_CUDA(cudaEventCreateWithFlags(&c->ev_post_join, cudaEventDisableTiming));
  for (int i = 0; i < 2; ++i) FO_CUDA(cudaEventCreateWithFlags(&c->ev_h2d_join[i], cudaEventDisableTiming));
  FO_CUDA(cudaEventCreateWithFlags(&c->ev_h2d_fork, cudaEventDisableTiming));
  FO_CUDA(cudaEventCreateWithFlags(&c->ev_d2h_join, cudaEventDisableTiming));
}

// the copy streams of fo_run_host, created on first use (a context that
// never stages host buffers holds only its comm and post streams)
static void ensure_host_streams(fo_ctx_s* c) {
  if (c->d2h_stream) return;
  for (int i = 0; i < 2; ++i) FO_CUDA(cudaStreamCreateWithFlags(&c->h2d_stream[i], cudaStreamNonBlocking));
  FO_CUDA(cudaStreamCreateWithFlags(&c->d2h_stream, cudaStreamNonBlocking));
}

fo_status fo_get_unique_id(uint8_t uid[128]) {
  return guard([&] {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    FO_NCCL(ncclGetUniqueId(&id));
    std::memcpy(uid, &id, 128);
  });
}

fo_status fo_ctx_create_config(int32_t device, int32_t rank, int32_t world, const uint8_t uid[128],
                               const fo_ctx_config* config, fo_ctx* out) {
  return guard([&] {
    if (!uid || !out || world < 1 || rank < 0 || rank >= world) fail(FO_ERR_INVALID_ARG, "bad arguments");
    fo_ctx_config k{};
    if (config) k = *config;
    if (k.nccl_max_ctas < 0 || k.nccl_min_ctas < 0 || k.nvls_ctas < 0 || k.cta_policy < 0 || k.cta_policy > 2 ||
        k.buffers < 0 || k.buffers > 2)
      fail(FO_ERR_INVALID_ARG, "bad fo_ctx_config");
    FO_CUDA(cudaSetDevice(device));
    auto* c = new fo_ctx_s();
    c->device = device;
    c->rank = rank;
    c->world = world;
    c->mem_mode = k.buffers;
    try {
      ncclUniqueId id;
      std::memcpy(&id, uid, 128);
      ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
      cfg.blocking = 1;
      if (k.nccl_max_ctas > 0) {
        cfg.maxCTAs = k.nccl_max_ctas;
        cfg.minCTAs = k.nccl_min_ctas > 0 ? std::min(k.nccl_min_ctas, k.nccl_max_ctas) : 1;
      } else if (k.nccl_min_ctas > 0) {
        cfg.minCTAs = k.nccl_min_ctas;
      }
      if (k.cta_policy > 0) cfg.CTAPolicy = k.cta_policy == 1 ? NCCL_CTA_POLICY_EFFICIENCY : NCCL_CTA_POLICY_ZERO;
      if (k.nvls_ctas > 0) cfg.nvlsCTAs = k.nvls_ctas;
      ncclComm_t comm = nullptr;
      FO_NCCL(ncclCommInitRankConfig(&comm, world, id, rank, &cfg));
      c->comm = make_nccl_comm(comm, rank, world, true);
      init_streams(c);
    } catch (...) {
      delete c->comm;
      delete c;
      throw;
    }
    *out = c;
  });
}

fo_status fo_ctx_create(int32_t device, int32_t rank, int32_t world, const uint8_t uid[128], int32_t nccl_max_ctas,
                        fo_ctx* out) {
  fo_ctx_config k{};
  k.nccl_max_ctas = nccl_max_ctas;
  return fo_ctx_create_config(device, rank, world, uid, &k, out);
}

fo_status fo_ctx_create_from_comm(int32_t device, void* nccl_comm, fo_ctx* out) {
  return guard([&] {
    if (!nccl_comm || !out) fail(FO_ERR_INVALID_ARG, "null argument");
    ncclComm_t comm = static_cast<ncclComm_t>(nccl_comm);
    int count = 0, rank = 0, cudev = -1;
    FO_NCCL(ncclCommCount(comm, &count));
    FO_NCCL(ncclCommUserRank(comm, &rank));
    FO_NCCL(ncclCommCuDevice(comm, &cudev));
    if (cudev != device) fail(FO_ERR_INVALID_ARG, "communicator is on device %d, not %d", cudev, device);
    FO_CUDA(cudaSetDevice(device));
    auto* c = new fo_ctx_s();
    c->device = device;
    c->rank = rank;
    c->world = count;
    c->comm = make_nccl_comm(comm, rank, count, false);
    try {
      init_streams(c);
    } catch (...) {
      delete c->comm;
      delete c;
      throw;
    }
    *out = c;
  });
}

fo_status fo_loopback_create(int32_t device, int32_t world, void** group) {
  return guard([&] {
    if (!group) fail(FO_ERR_INVALID_ARG, "null argument");
    *group = loopback_create(device, world);
  });
}

fo_status fo_loopback_destroy(void* group) {
  return guard([&] {
    if (!group) return;
    auto* g = static_cast<LoopbackGroup*>(group);
    if (loopback_members(g)) fail(FO_ERR_STATE, "loopback group still has %d contexts", loopback_members(g));
    loopback_destroy(g);
  });
}

fo_status fo_ctx_create_loopback(void* group, int32_t rank, fo_ctx* out) {
  return guard([&] {
    if (!group || !out) fail(FO_ERR_INVALID_ARG, "null argument");
    auto* g = static_cast<LoopbackGroup*>(group);
    if (rank < 0 || rank >= loopback_world(g)) fail(FO_ERR_INVALID_ARG, "rank %d of %d", rank, loopback_world(g));
    FO_CUDA(cudaSetDevice(loopback_device(g)));
    auto* c = new fo_ctx_s();
    c->device = loopback_device(g);
    c->rank = rank;
    c->world = loopback_world(g);
    try {
      c->comm = make_loopback_comm(g, rank);
      init_streams(c);
    } catch (...) {
      delete c->comm;
      delete c;
      throw;
    }
    *out = c;
  });
}

fo_status fo_ctx_create_emulated(int32_t device, int32_t rank, int32_t world, double link_gbps, double latency_us,
                                 int32_t ctas, fo_ctx* out) {
  return guard([&] {
    if (!out) fail(FO_ERR_INVALID_ARG, "null argument");
    if (world < 1 || rank < 0 || rank >= world) fail(FO_ERR_INVALID_ARG, "rank %d of %d", rank, world);
    if (!(link_gbps > 0) || latency_us < 0 || ctas < 1 || ctas > 1024)
      fail(FO_ERR_INVALID_ARG, "link_gbps > 0, latency_us >= 0, 1 <= ctas <= 1024");
    FO_CUDA(cudaSetDevice(device));
    auto* c = new fo_ctx_s();
    c->device = device;
    c->rank = rank;
    c->world = world;
    try {
      c->comm = make_emulated_comm(rank, world, link_gbps, latency_us, ctas);
      init_streams(c);
    } catch (...) {
      delete c->comm;
      delete c;
      throw;
    }
    *out = c;
  });
}

fo_status fo_ctx_destroy(fo_ctx c) {
  return guard([&] {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->comm_stream) cudaStreamSynchronize(c->comm_stream);
    cudaDeviceSynchronize();
    while (!c->reg_plans.empty()) deregister_plan(c->reg_plans.back());
    for (auto& b : c->user_bufs) {
      ncclComm_t comm = c->comm ? c->comm->nccl() : nullptr;
      if (comm && b.handle) ncclCommDeregister(comm, b.handle);
      if (comm && b.win) ncclCommWindowDeregister(comm, b.win);
      ncclMemFree(b.ptr);
    }
    c->user_bufs.clear();
    delete c->comm;
    c->comm = nullptr;
    if (c->post_stream) cudaStreamSynchronize(c->post_stream);
    if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
    if (c->post_stream) cudaStreamDestroy(c->post_stream);
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    if (c->ev_post_join) cudaEventDestroy(c->ev_post_join);
    for (cudaEvent_t e : c->ev_group) cudaEventDestroy(e);
    for (cudaStream_t st : {c->h2d_stream[0], c->h2d_stream[1], c->d2h_stream})
      if (st) {
        cudaStreamSynchronize(st);
        cudaStreamDestroy(st);
      }
    for (cudaEvent_t e : {c->ev_h2d_fork, c->ev_h2d_join[0], c->ev_h2d_join[1], c->ev_d2h_join})
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : c->ev_d2h) cudaEventDestroy(e);
    delete c;
  });
}

// Rows [r0, r1) of the output that are final once group j is done — defined
// when every group is a band of whole tile-rows that lands row-major in the
// output (AR / RS ROWBAND); false otherwise.
static bool group_out_rows(const PlanHost& h, int j, int64_t* r0, int64_t* r1) {
  if (!h.banded()) return false;
  if ((int)h.band_rows.size() < 2 * h.P) return false;
  *r0 = (int64_t)h.band_rows[2 * j] * h.band_out_rows();
  *r1 = (int64_t)h.band_rows[2 * j + 1] * h.band_out_rows();
  return true;
}

// fo_run_host: copy group j's final output rows to the host as soon as the
// group is done (stream `done` = where its last op ran), overlapping the
// device->host transfer with the remaining groups.
static void group_d2h(fo_ctx c, fo_plan p, int j, const void* out, cudaStream_t done) {
  const PlanHost& h = p->host;
  int64_t r0 = 0, r1 = 0;
  if (!group_out_rows(h, j, &r0, &r1)) return;
  while ((int)c->ev_d2h.size() <= j) {
    cudaEvent_t e;
    FO_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->ev_d2h.push_back(e);
  }
  FO_CUDA(cudaEventRecord(c->ev_d2h[j], done));
  FO_CUDA(cudaStreamWaitEvent(c->d2h_stream, c->ev_d2h[j], 0));
  const size_t off = 2 * (size_t)(r0 * h.N), bytes = 2 * (size_t)((r1 - r0) * h.N);
  FO_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(p->d2h_host) + off, reinterpret_cast<const char*>(out) + off,
                          bytes, cudaMemcpyDeviceToHost, c->d2h_stream));
}

fo_status fo_run(fo_ctx c, fo_plan p, const void* A, const void* Bt, void* out, const void* residual,
                 const void* gamma, void* stream) {
  return guard([&] {
    if (!c || !p) fail(FO_ERR_INVALID_ARG, "null argument");
    const PlanHost& h = p->host;
    // an All-to-All rank that receives no rows (or a combine with no tokens)
    // has an empty output and may pass NULL (R45)
    if (!out && !(h.coll == FO_ALLTOALL && (p->combine ? p->combine->tokens == 0 : h.out_rows == 0)))
      fail(FO_ERR_INVALID_ARG, "null argument");
    if (h.world != c->world || h.rank != c->rank) fail(FO_ERR_STATE, "plan rank/world do not match the context");
    if (c->aborted) fail(FO_ERR_STATE, "context aborted by the watchdog (fo_plan_sync timed out)");
    bind_ctx(c, p);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    WaitValue32Fn wait = wait_value_fn();
    if (!wait) fail(FO_ERR_UNSUPPORTED, "cuStreamWaitValue32 unavailable");
    // the GEMM writes the output itself for no-comm and in-place banded
    // plans (AR ROWBAND; RS ROWBAND at one rank), else the send buffer; a
    // banded RS scatters into the output, so every banded plan's
    // post-communication data is `out`
    const bool rowband = (h.coll == FO_NOCOMM) || h.banded();
    const bool gemm_out = (h.coll == FO_NOCOMM) || (h.banded() && (h.coll == FO_ALLREDUCE || h.world == 1));
    // A2A ROWBAND (R41): the groups' rows are received straight into `out`
    // (the output layout), except under the MoE combine, whose `out` is the
    // combined tokens: then into the library's receive buffer; at one rank
    // send, receive and output layouts coincide
    const bool a2a_band = h.coll == FO_ALLTOALL && h.layout == FO_LAYOUT_ROWBAND;
    void* recv_buf = (a2a_band && !p->combine) ? out : p->d_recv;
    void* send_buf = (a2a_band && !p->combine && h.world == 1) ? out : p->d_send;
    void* gemm_dst = gemm_out ? out : send_buf;
    // a single group issued in stream order (R32) waits on no counter: the GEMM
    // then neither signals nor needs the counting table reset
    const bool counted = !(p->last_in_order && h.coll != FO_NOCOMM && h.P == 1);
    // 1. counting table reset (every run starts from zero)
    if (counted || p->split > 1) FO_CUDA(cudaMemsetAsync(p->d_counters, 0, sizeof(uint32_t) * p->ctr_words, s));
    // 2. fork (nothing to fork when the single group runs on s)
    if (counted) {
      FO_CUDA(cudaEventRecord(c->ev_fork, s));
      FO_CUDA(cudaStreamWaitEvent(c->comm_stream, c->ev_fork, 0));
    }
    // 3. GEMM with reorder + signal epilogue
    run_gemm(p, A, Bt, gemm_dst, epi_mode(h), counted, s, p->trace_tile_ts);
    const bool gpost = use_group_post(p) && !p->combine;
    const void* post_src = (h.coll == FO_ALLREDUCE) ? (rowband ? out : p->d_send) : (rowband ? out : recv_buf);
    // 4. per-group wait + collective; the per-group post-reorder runs on the
    //    post stream, chained to its group's collective by an event, so the
    //    next group's collective never queues behind a reorder
    while ((int)c->ev_group.size() < h.P) {
      cudaEvent_t e;
      FO_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      c->ev_group.push_back(e);
    }
    // the last group in stream order (FO_OPT_LAST_GROUP_IN_ORDER): its
    // collective follows the GEMM on s — the kernel boundary already orders
    // every tile's stores, so no counter wait (and no wait-release latency)
    // sits on the layer's critical path; s first waits for the comm stream's
    // earlier collectives so the communicator sees the same call order
    const bool last_on_s = p->last_in_order && h.coll != FO_NOCOMM;
    cudaStream_t tail = last_on_s ? s : c->comm_stream;
    if (h.coll != FO_NOCOMM) {
      for (int j = 0; j < h.P; ++j) {
        const bool on_s = last_on_s && j == h.P - 1;
        cudaStream_t cs = on_s ? s : c->comm_stream;
        if (on_s) {
          if (h.P > 1) {
            FO_CUDA(cudaEventRecord(c->ev_join, c->comm_stream));
            FO_CUDA(cudaStreamWaitEvent(s, c->ev_join, 0));
          }
        } else {
          stream_wait(p, wait, cs, j);
        }
        if (p->trace_group_ts) FO_CUDA(launch_timestamp(p->trace_group_ts + 2 * j, cs));
        group_collective(c, p, j, send_buf, recv_buf, out, cs);
        cudaStream_t ps = cs;
        if (gpost) {
          if (!on_s) {
            FO_CUDA(cudaEventRecord(c->ev_group[j], cs));
            FO_CUDA(cudaStreamWaitEvent(c->post_stream, c->ev_group[j], 0));
            ps = c->post_stream;
          }
          run_group_post(p, j, post_src, out, residual, gamma, ps, on_s);
        }
        if (p->trace_group_ts) FO_CUDA(launch_timestamp(p->trace_group_ts + 2 * j + 1, ps));
        if (p->d2h_host) group_d2h(c, p, j, out, ps);
      }
    } else {
      // no communication: the comm stream only has to see the GEMM finish
      for (int j = 0; j < h.P; ++j) {
        stream_wait(p, wait, c->comm_stream, j);
        if (p->d2h_host) group_d2h(c, p, j, out, c->comm_stream);
      }
    }
    // 5. post-communication reorder (+ fused op) when not done per group
    const int map = post_map(h);
    if (p->combine) {
      CombineArgs ca = *p->combine;
      ca.src = post_src;
      FO_CUDA(launch_combine(ca, tail));
    } else if (!gpost && (map != POSTMAP_IDENTITY || h.post != FO_POST_NONE)) {
      run_post(p, map, post_src, out, residual, gamma, tail);
    }
    // 6. join (with the last group on s, s already waited for the comm stream)
    if (!last_on_s) {
      FO_CUDA(cudaEventRecord(c->ev_join, c->comm_stream));
      FO_CUDA(cudaStreamWaitEvent(s, c->ev_join, 0));
    }
    if (gpost && h.coll != FO_NOCOMM && !(last_on_s && h.P == 1)) {
      FO_CUDA(cudaEventRecord(c->ev_post_join, c->post_stream));
      FO_CUDA(cudaStreamWaitEvent(s, c->ev_post_join, 0));
    }
    if (p->d2h_host) {
      FO_CUDA(cudaEventRecord(c->ev_d2h_join, c->d2h_stream));
      FO_CUDA(cudaStreamWaitEvent(s, c->ev_d2h_join, 0));
    }
  });
}

static bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();  // clear: plain host memory
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Chunking of a host-staged A: ~FO_OPT_HOST_CHUNKS (8) chunks of whole tile-rows, copied in the
// order the tile order first needs them.
static void plan_a_chunks(fo_plan p) {
  const PlanHost& h = p->host;
  if (p->a_chunks) return;
  p->a_chunk_rows = (int)((h.Mt + p->a_chunk_target - 1) / p->a_chunk_target);
  p->a_chunks = (int)((h.Mt + p->a_chunk_rows - 1) / p->a_chunk_rows);
  std::vector<int64_t> first(p->a_chunks, INT64_MAX);
  for (int64_t pos = 0; pos < h.tiles; ++pos) {
    const int ch = (int)((h.order[pos] / h.Nt) / p->a_chunk_rows);
    first[ch] = std::min(first[ch], pos);
  }
  p->a_chunk_order.resize(p->a_chunks);
  for (int i = 0; i < p->a_chunks; ++i) p->a_chunk_order[i] = i;
  std::stable_sort(p->a_chunk_order.begin(), p->a_chunk_order.end(),
                   [&](int x, int y) { return first[x] < first[y]; });
  FO_CUDA(cudaMalloc(&p->d_a_ready, sizeof(uint32_t) * 2 * p->a_chunks));   // one flag set per staging set
  FO_CUDA(cudaMemset(p->d_a_ready, 0, sizeof(uint32_t) * 2 * p->a_chunks));
}

fo_status fo_run_host(fo_ctx c, fo_plan p, const void* A, const void* Bt, void* out, const void* residual,
                      const void* gamma, void* stream) {
  struct Transient {  // the per-call pipelining state never outlives the call
    fo_plan p;
    ~Transient() {
      p->a_staged_run = false;
      p->d2h_host = nullptr;
    }
  };
  return guard([&] {
    if (!c || !p || !A || !Bt || !out) fail(FO_ERR_INVALID_ARG, "null argument");
    bind_ctx(c, p);
    FO_CUDA(cudaSetDevice(c->device));
    ensure_host_streams(c);
    const PlanHost& h = p->host;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const size_t a_bytes = 2 * (size_t)(h.M * h.K), b_bytes = 2 * (size_t)(h.N * h.K);
    // the SwiGLU epilogue writes C as [m, n/2]
    const size_t o_bytes = 2 * (size_t)(h.out_rows * (p->swiglu ? h.N / 2 : h.N));
    // host operands are staged through library-owned device buffers; operands
    // that already live on the device (e.g. resident weights) are used in place
    auto stage = [&](const void* src, void*& buf, size_t bytes) -> const void* {
      if (!src) return nullptr;
      if (is_device_ptr(src)) return src;
      if (!buf) FO_CUDA(cudaMalloc(&buf, bytes));
      FO_CUDA(cudaMemcpyAsync(buf, src, bytes, cudaMemcpyHostToDevice, s));
      return buf;
    };
    Transient guard_state{p};
    WriteValue32Fn write = write_value_fn();
    const bool a_host = !is_device_ptr(A);
    // pipelined A: chunked copies on the H2D stream, each released to the GEMM
    // producer by a stream write of this run's epoch (PAPER.md:368's
    // signal/wait, applied to the input side); needs K-major A
    const bool pipe_a = a_host && (p->host_pipeline & 1) && write && !(h.mn_major & 1);
    // two staging sets (bit 2): this call uses set b, the previous call the
    // other one, so this call's H2D only has to wait for the call before the
    // previous one (the last user of set b) and overlaps the previous call's
    // GEMM, collectives and D2H
    const bool two_sets = pipe_a && (p->host_pipeline & 4);
    p->host_set = two_sets ? (p->host_set ^ 1) : 0;
    const int b = p->host_set;
    void*& stA = (b == 0) ? p->h_A : p->h_A2;
    void*& stO = (b == 0) ? p->h_out : p->h_out2;
    const void* dA = nullptr;
    if (pipe_a) {
      plan_a_chunks(p);
      if (!stA) FO_CUDA(cudaMalloc(&stA, a_bytes));
      ++p->a_epoch;
      // the copies may overwrite the staging only after its last user's GEMM
      // (one staging set: the work already on `s`; two sets: the call that
      // last used set b); they are enqueued BEFORE the GEMM that waits on
      // them, so no hardware-queue aliasing can order the GEMM ahead of the
      // copies it waits for
      if (two_sets) {
        if (!p->ev_set_done[b]) {
          FO_CUDA(cudaEventCreateWithFlags(&p->ev_set_done[b], cudaEventDisableTiming));
          FO_CUDA(cudaEventRecord(p->ev_set_done[b], s));
        }
        for (int i = 0; i < 2; ++i) FO_CUDA(cudaStreamWaitEvent(c->h2d_stream[i], p->ev_set_done[b], 0));
      } else {
        FO_CUDA(cudaEventRecord(c->ev_h2d_fork, s));
        for (int i = 0; i < 2; ++i) FO_CUDA(cudaStreamWaitEvent(c->h2d_stream[i], c->ev_h2d_fork, 0));
      }
      // chunks alternate between two copy streams so one chunk's release
      // write never leaves the copy engine idle before the next chunk
      const size_t row_bytes = 2 * (size_t)h.K;
      for (size_t i = 0; i < p->a_chunk_order.size(); ++i) {
        const int ch = p->a_chunk_order[i];
        cudaStream_t cs = c->h2d_stream[i & 1];
        const int64_t r0 = (int64_t)ch * p->a_chunk_rows * h.BM;
        const int64_t r1 = std::min<int64_t>(h.M, r0 + (int64_t)p->a_chunk_rows * h.BM);
        FO_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(stA) + r0 * row_bytes,
                                reinterpret_cast<const char*>(A) + r0 * row_bytes, (r1 - r0) * row_bytes,
                                cudaMemcpyHostToDevice, cs));
        CUresult r = write(reinterpret_cast<CUstream>(cs),
                           reinterpret_cast<CUdeviceptr>(p->d_a_ready + (size_t)b * p->a_chunks + ch), p->a_epoch, 0);
        if (r != CUDA_SUCCESS) fail(FO_ERR_CUDA, "cuStreamWriteValue32 failed (%d)", (int)r);
      }
      for (int i = 0; i < 2; ++i) FO_CUDA(cudaEventRecord(c->ev_h2d_join[i], c->h2d_stream[i]));
      p->a_staged_run = true;
      dA = stA;
    } else {
      dA = stage(A, p->h_A, a_bytes);
    }
    const void* dB = stage(Bt, p->h_Bt, b_bytes);
    const void* dR = stage(residual, p->h_res, o_bytes);
    const void* dG = stage(gamma, p->h_gamma, 2 * (size_t)h.N);
    const bool out_dev = is_device_ptr(out);
    if (!out_dev && !stO) FO_CUDA(cudaMalloc(&stO, o_bytes));
    void* dO = out_dev ? out : stO;
    int64_t r0 = 0, r1 = 0;
    // per-group D2H only when each group's rows are final after its own
    // stream work (a post pass deferred to the end would rewrite them)
    const bool pipe_out = !out_dev && (p->host_pipeline & 2) && group_out_rows(h, 0, &r0, &r1) &&
                          (h.post == FO_POST_NONE || use_group_post(p));
    if (pipe_out) p->d2h_host = out;
    fo_status st = fo_run(c, p, dA, dB, dO, dR, dG, stream);
    if (st != FO_OK) throw Error(st, fo_last_error());
    if (pipe_a)
      for (int i = 0; i < 2; ++i) FO_CUDA(cudaStreamWaitEvent(s, c->ev_h2d_join[i], 0));
    if (!out_dev && !pipe_out) FO_CUDA(cudaMemcpyAsync(out, dO, o_bytes, cudaMemcpyDeviceToHost, s));
    // FO_POST_ADD_RMSNORM_RESIDUAL updates the residual in place: a host
    // residual gets its staged copy back
    if (residual && dR != residual && h.post == FO_POST_ADD_RMSNORM_RESIDUAL)
      FO_CUDA(cudaMemcpyAsync(const_cast<void*>(residual), dR, o_bytes, cudaMemcpyDeviceToHost, s));
    if (two_sets) FO_CUDA(cudaEventRecord(p->ev_set_done[b], s));  // set b free once this call is done
  });
}

fo_status fo_run_sequential(fo_ctx c, fo_plan p, const void* A, const void* Bt, void* out, const void* residual,
                            const void* gamma, void* stream) {
  return guard([&] {
    if (!c || !p) fail(FO_ERR_INVALID_ARG, "null argument");
    if (!out && !(p->host.coll == FO_ALLTOALL && p->host.out_rows == 0)) fail(FO_ERR_INVALID_ARG, "null argument");
    if (c->aborted) fail(FO_ERR_STATE, "context aborted by the watchdog (fo_plan_sync timed out)");
    const PlanHost& h = p->host;
    if (h.world != c->world || h.rank != c->rank) fail(FO_ERR_STATE, "plan rank/world do not match the context");
    bind_ctx(c, p);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int64_t MN = h.M * h.N;
    if (p->split > 1) FO_CUDA(cudaMemsetAsync(p->d_counters, 0, sizeof(uint32_t) * p->ctr_words, s));
    // the same GEMM writing row-major C (in place into out for AR / no-comm,
    // into a scratch C for RS / A2A), then the plan's sequential schedule:
    // one full-size collective (fo_plan_export_calls schedule 1)
    void* C = out;
    if (h.coll == FO_REDUCESCATTER || h.coll == FO_ALLTOALL) {
      if (!p->d_rowmajor) FO_CUDA(cudaMalloc(&p->d_rowmajor, 2 * MN));
      C = p->d_rowmajor;
    }
    run_gemm(p, A, Bt, C, EPI_ROWMAJOR, false, s);
    void* const bufs[4] = {nullptr, nullptr, out, p->d_rowmajor};
    exec_calls(c, h.seq_calls, 0, h.seq_calls.size(), bufs, s);
    if (h.post != FO_POST_NONE) run_post(p, POSTMAP_IDENTITY, out, out, residual, gamma, s);
  });
}

// ---- RS follow-on (NEXT f2): AllGather of the block-cyclic
// local outputs, then the row exchange (fused with the plan's elementwise op)
static void run_rowexchange(fo_plan_s* p, const void* gathered, void* out, const void* residual, const void* gamma,
                            cudaStream_t s) {
  const PlanHost& h = p->host;
  PostArgs a{};
  a.map = POSTMAP_ROWX;
  a.op = h.post;
  a.src = gathered;
  a.out = out;
  a.residual = residual;
  a.gamma = gamma;
  a.rows = h.M;
  a.N = h.N;
  a.BM = h.BM;
  a.BN = h.BN;
  a.Nt = h.Nt;
  a.h = h.h;
  a.eps = h.eps;
  a.bulk_ok = p->post_bulk;
  if (h.post != FO_POST_NONE && !residual) fail(FO_ERR_INVALID_ARG, "post op needs a residual");
  if (is_rmsnorm(h.post) && !gamma) fail(FO_ERR_INVALID_ARG, "RMSNorm needs gamma");
  FO_CUDA(launch_post(a, s));
}

fo_status fo_rowexchange_stage(fo_plan p, const void* gathered, void* out, const void* residual, const void* gamma,
                               void* stream) {
  return guard([&] {
    if (!p || !gathered || !out) fail(FO_ERR_INVALID_ARG, "null argument");
    if (p->host.coll != FO_REDUCESCATTER) fail(FO_ERR_INVALID_ARG, "row exchange follows a ReduceScatter plan");
    ensure_device(p);
    run_rowexchange(p, gathered, out, residual, gamma, reinterpret_cast<cudaStream_t>(stream));
  });
}

fo_status fo_run_allgather(fo_ctx c, fo_plan p, const void* local, void* out, const void* residual,
                           const void* gamma, int32_t row_exchange, void* stream) {
  return guard([&] {
    if (!c || !p || !local || !out) fail(FO_ERR_INVALID_ARG, "null argument");
    if (c->aborted) fail(FO_ERR_STATE, "context aborted by the watchdog (fo_plan_sync timed out)");
    const PlanHost& h = p->host;
    if (h.coll != FO_REDUCESCATTER) fail(FO_ERR_INVALID_ARG, "AllGather follow-on needs a ReduceScatter plan");
    if (h.world != c->world || h.rank != c->rank) fail(FO_ERR_STATE, "plan rank/world do not match the context");
    bind_ctx(c, p);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const size_t local_elems = (size_t)(h.out_rows * h.N);
    if (!row_exchange) {
      // row order not needed downstream: gather straight into out
      c->comm->allgather(local, out, local_elems, s);
      if (h.post != FO_POST_NONE) {
        PostArgs a{};
        a.map = POSTMAP_IDENTITY;
        a.op = h.post;
        a.src = out;
        a.out = out;
        a.residual = residual;
        a.gamma = gamma;
        a.rows = h.M;
        a.N = h.N;
        a.BM = h.BM;
        a.BN = h.BN;
        a.Nt = h.Nt;
        a.h = h.h;
        a.eps = h.eps;
        a.bulk_ok = p->post_bulk;
        if (!residual) fail(FO_ERR_INVALID_ARG, "post op needs a residual");
        FO_CUDA(launch_post(a, s));
      }
      return;
    }
    if (!p->d_rowmajor) FO_CUDA(cudaMalloc(&p->d_rowmajor, 2 * (size_t)(h.M * h.N)));
    c->comm->allgather(local, p->d_rowmajor, local_elems, s);
    run_rowexchange(p, p->d_rowmajor, out, residual, gamma, s);
  });
}

fo_status fo_gemm_stage(fo_plan p, const void* A, const void* Bt, void* send, void* stream) {
  return guard([&] {
    if (!p) fail(FO_ERR_INVALID_ARG, "null plan");
    ensure_device(p);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    FO_CUDA(cudaMemsetAsync(p->d_counters, 0, sizeof(uint32_t) * p->ctr_words, s));
    run_gemm(p, A, Bt, send, epi_mode(p->host), true, s);
  });
}

fo_status fo_gemm_stage_timed(fo_plan p, const void* A, const void* Bt, void* send, unsigned long long* tile_ts,
                              void* stream) {
  return guard([&] {
    if (!p) fail(FO_ERR_INVALID_ARG, "null plan");
    ensure_device(p);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    FO_CUDA(cudaMemsetAsync(p->d_counters, 0, sizeof(uint32_t) * p->ctr_words, s));
    run_gemm(p, A, Bt, send, epi_mode(p->host), true, s, tile_ts);
  });
}

fo_status fo_group_post_stage(fo_plan p, int32_t j, const void* recv, void* out, const void* residual,
                              void* stream) {
  return guard([&] {
    if (!p || !recv || !out) fail(FO_ERR_INVALID_ARG, "null argument");
    const PlanHost& h = p->host;
    if (j < 0 || j >= h.P) fail(FO_ERR_INVALID_ARG, "group %d out of range", j);
    const int map = post_map(h);
    if (map == POSTMAP_IDENTITY || !(h.post == FO_POST_NONE || h.post == FO_POST_ADD))
      fail(FO_ERR_UNSUPPORTED, "per-group post pass needs a slot / RS / A2A layout and post none or add");
    ensure_device(p);
    run_group_post(p, j, recv, out, residual, nullptr, reinterpret_cast<cudaStream_t>(stream));
  });
}

fo_status fo_post_stage(fo_plan p, const void* recv, void* out, const void* residual, const void* gamma,
                        void* stream) {
  return guard([&] {
    if (!p || !recv || !out) fail(FO_ERR_INVALID_ARG, "null argument");
    ensure_device(p);
    run_post(p, post_map(p->host), recv, out, residual, gamma, reinterpret_cast<cudaStream_t>(stream));
  });
}

// MoE combine arguments (R31), validated against the plan.
static CombineArgs combine_args(fo_plan p, const void* recv, void* out, const int32_t* idx, const float* w,
                                int32_t topk, int64_t tokens, const void* residual) {
  const PlanHost& h = p->host;
  if (h.coll != FO_ALLTOALL) fail(FO_ERR_INVALID_ARG, "the MoE combine follows an All-to-All plan");
  if (h.post != FO_POST_NONE) fail(FO_ERR_INVALID_ARG, "the combine replaces the plan's post op (use post=none)");
  if (topk < 1 || topk > 64 || tokens < 0) fail(FO_ERR_INVALID_ARG, "topk must be 1..64 and tokens >= 0");
  if (tokens > 0 && (!out || !idx || !w)) fail(FO_ERR_INVALID_ARG, "null argument");
  CombineArgs a{};
  a.src = recv;
  a.out = out;
  a.residual = residual;
  a.idx = idx;
  a.w = w;
  a.topk = topk;
  a.tokens = tokens;
  a.N = h.N;
  a.a2a_rows = h.out_rows;
  a.BN = h.BN;
  a.Nt = (int)h.Nt;
  a.src_row = p->d_src_row;
  return a;
}

fo_status fo_combine_stage(fo_plan p, const void* recv, void* out, const int32_t* idx, const float* w,
                           int32_t topk, int64_t tokens, const void* residual, void* stream) {
  return guard([&] {
    if (!p || (!recv && p->host.recv_elems)) fail(FO_ERR_INVALID_ARG, "null argument");
    ensure_device(p);
    FO_CUDA(launch_combine(combine_args(p, recv, out, idx, w, topk, tokens, residual),
                           reinterpret_cast<cudaStream_t>(stream)));
  });
}

fo_status fo_run_combine(fo_ctx c, fo_plan p, const void* A, const void* Bt, void* out, const int32_t* idx,
                         const float* w, int32_t topk, int64_t tokens, const void* residual, void* stream) {
  struct Transient {
    fo_plan p;
    ~Transient() { p->combine = nullptr; }
  };
  return guard([&] {
    if (!c || !p || (!out && tokens > 0)) fail(FO_ERR_INVALID_ARG, "null argument");
    ensure_device(p);
    const CombineArgs ca = combine_args(p, nullptr, out, idx, w, topk, tokens, residual);
    Transient t{p};
    p->combine = &ca;
    fo_status st = fo_run(c, p, A, Bt, out, nullptr, nullptr, stream);
    if (st != FO_OK) throw Error(st, fo_last_error());
  });
}

// Debug watchdog (H8): wait for the plan's last run on `stream` with a
// timeout.  On timeout the communicator is aborted (in-flight NCCL kernels
// exit), every counter of the plan is forced past any target so pending
// stream waits / spin kernels release and the streams drain, and the context
// refuses further runs.
fo_status fo_plan_sync(fo_ctx c, fo_plan p, void* stream, int64_t timeout_ms) {
  return guard([&] {
    if (!c || !p) fail(FO_ERR_INVALID_ARG, "null argument");
    if (timeout_ms < 0) fail(FO_ERR_INVALID_ARG, "timeout_ms must be >= 0");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    cudaEvent_t ev = nullptr;
    FO_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    struct EvGuard {
      cudaEvent_t e;
      ~EvGuard() { cudaEventDestroy(e); }
    } eg{ev};
    FO_CUDA(cudaEventRecord(ev, s));
    auto drained = [&](int64_t ms) {
      const auto t0 = std::chrono::steady_clock::now();
      while (true) {
        const cudaError_t q = cudaEventQuery(ev);
        if (q == cudaSuccess) return true;
        if (q != cudaErrorNotReady) fail(FO_ERR_CUDA, "cudaEventQuery: %s", cudaGetErrorString(q));
        if (std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(ms)) return false;
        std::this_thread::sleep_for(std::chrono::microseconds(200));
      }
    };
    if (drained(timeout_ms)) return;
    c->aborted = true;
    // 1. release the trigger waits: every counter past any target (from a
    //    fresh non-blocking stream; the stuck streams cannot run a memset)
    if (p->d_counters) {
      cudaStream_t rescue = nullptr;
      FO_CUDA(cudaStreamCreateWithFlags(&rescue, cudaStreamNonBlocking));
      FO_CUDA(cudaMemsetAsync(p->d_counters, 0x3f, sizeof(uint32_t) * p->ctr_words, rescue));
      cudaStreamSynchronize(rescue);
      cudaStreamDestroy(rescue);
    }
    // 2. the released NCCL calls either complete (peers present) or, still
    //    stuck after another timeout, are killed by aborting the communicator
    //    (ncclCommAbort makes in-flight NCCL kernels exit)
    const bool done = drained(std::max<int64_t>(timeout_ms, 1000));
    if (c->comm) c->comm->abort();
    if (!done) drained(std::max<int64_t>(timeout_ms, 1000));
    fail(FO_ERR_TIMEOUT, "plan run did not finish within %lld ms: waits released, communicator aborted",
         (long long)timeout_ms);
  });
}

fo_status fo_mem_alloc(fo_ctx c, int64_t bytes, void** ptr) {
  return guard([&] {
    if (!c || !ptr || bytes <= 0) fail(FO_ERR_INVALID_ARG, "bad arguments");
    FO_CUDA(cudaSetDevice(c->device));
    fo_ctx_s::UserBuf b{};
    b.bytes = (size_t)bytes;
    FO_NCCL(ncclMemAlloc(&b.ptr, b.bytes));
    ncclComm_t comm = c->comm ? c->comm->nccl() : nullptr;
    try {
      if (comm && c->mem_mode == 1) FO_NCCL(ncclCommRegister(comm, b.ptr, b.bytes, &b.handle));
      if (comm && c->mem_mode == 2) FO_NCCL(ncclCommWindowRegister(comm, b.ptr, b.bytes, &b.win, NCCL_WIN_COLL_SYMMETRIC));
    } catch (...) {
      ncclMemFree(b.ptr);
      throw;
    }
    c->user_bufs.push_back(b);
    *ptr = b.ptr;
  });
}

fo_status fo_mem_free(fo_ctx c, void* ptr) {
  return guard([&] {
    if (!c || !ptr) fail(FO_ERR_INVALID_ARG, "null argument");
    auto& v = c->user_bufs;
    auto it = std::find_if(v.begin(), v.end(), [&](const fo_ctx_s::UserBuf& b) { return b.ptr == ptr; });
    if (it == v.end()) fail(FO_ERR_INVALID_ARG, "pointer not from fo_mem_alloc on this context");
    FO_CUDA(cudaSetDevice(c->device));
    FO_CUDA(cudaDeviceSynchronize());
    ncclComm_t comm = c->comm ? c->comm->nccl() : nullptr;
    if (comm && it->handle) FO_NCCL(ncclCommDeregister(comm, it->handle));
    if (comm && it->win) FO_NCCL(ncclCommWindowDeregister(comm, it->win));
    FO_NCCL(ncclMemFree(it->ptr));
    v.erase(it);
  });
}

fo_status fo_plan_prepare(fo_ctx c, fo_plan p, int32_t what) {
  return guard([&] {
    if (!p) fail(FO_ERR_INVALID_ARG, "null plan");
    if (what < 0 || what > 3) fail(FO_ERR_INVALID_ARG, "what must be a mask of 1 | 2");
    if (c) bind_ctx(c, p);
    else ensure_device(p);
    const PlanHost& h = p->host;
    if ((what & 1) && (h.coll == FO_REDUCESCATTER || h.coll == FO_ALLTOALL) && !p->d_rowmajor)
      FO_CUDA(cudaMalloc(&p->d_rowmajor, 2 * (size_t)(h.M * h.N)));
    if (what & 2) {
      const size_t a_bytes = 2 * (size_t)(h.M * h.K), o_bytes = 2 * (size_t)(h.out_rows * h.N);
      if (!(h.mn_major & 1)) plan_a_chunks(p);
      for (void** b : {&p->h_A, &p->h_A2})
        if (!*b) FO_CUDA(cudaMalloc(b, a_bytes));
      for (void** b : {&p->h_out, &p->h_out2})
        if (!*b) FO_CUDA(cudaMalloc(b, o_bytes));
    }
    FO_CUDA(cudaDeviceSynchronize());
  });
}

fo_status fo_plan_read_counters(fo_plan p, uint32_t* counters) {
  return guard([&] {
    if (!p || !counters) fail(FO_ERR_INVALID_ARG, "null argument");
    if (p->device < 0) fail(FO_ERR_STATE, "plan has no device state yet");
    FO_CUDA(cudaDeviceSynchronize());
    FO_CUDA(cudaMemcpy(counters, p->d_counters, sizeof(uint32_t) * p->host.P, cudaMemcpyDeviceToHost));
  });
}

fo_status fo_plan_gemm_cluster(fo_plan p, int32_t* cluster_ctas) {
  return guard([&] {
    if (!p || !cluster_ctas) fail(FO_ERR_INVALID_ARG, "null argument");
    ensure_device(p);
    GemmArgs a = gemm_args(p, nullptr, nullptr, nullptr, EPI_ROWMAJOR, false);
    *cluster_ctas = gemm_multicast_used(a) ? 4 : ctas_per_tile(p->host.BM);
  });
}

int64_t fo_kernel_launch_count(void) { return launch_count(); }

fo_status fo_ctx_time_collective(fo_ctx c, int32_t coll, int64_t bytes, int32_t iters, double* avg_us,
                                 double* busbw_gbps) {
  return guard([&] {
    if (!c || !avg_us || bytes <= 0 || iters < 1) fail(FO_ERR_INVALID_ARG, "bad arguments");
    if (c->aborted) fail(FO_ERR_STATE, "context aborted by the watchdog (fo_plan_sync timed out)");
    FO_CUDA(cudaSetDevice(c->device));
    const int W = c->world;
    const size_t count = (size_t)(bytes / 2 / W) * W;  // bf16 elements, divisible by world
    if (count == 0) fail(FO_ERR_INVALID_ARG, "message too small");
    // the buffers the context's plans would use: registered ones when the
    // context registers (the curve then includes NVLS / zero-copy paths)
    void *a = nullptr, *b = nullptr;
    ncclComm_t comm = c->comm ? c->comm->nccl() : nullptr;
    const bool reg = c->mem_mode > 0 && comm;
    void *ha = nullptr, *hb = nullptr;
    ncclWindow_t wa = nullptr, wb = nullptr;
    if (reg) {
      FO_NCCL(ncclMemAlloc(&a, 2 * count));
      FO_NCCL(ncclMemAlloc(&b, 2 * count));
      if (c->mem_mode == 2) {
        FO_NCCL(ncclCommWindowRegister(comm, a, 2 * count, &wa, NCCL_WIN_COLL_SYMMETRIC));
        FO_NCCL(ncclCommWindowRegister(comm, b, 2 * count, &wb, NCCL_WIN_COLL_SYMMETRIC));
      } else {
        FO_NCCL(ncclCommRegister(comm, a, 2 * count, &ha));
        FO_NCCL(ncclCommRegister(comm, b, 2 * count, &hb));
      }
    } else {
      FO_CUDA(cudaMalloc(&a, 2 * count));
      FO_CUDA(cudaMalloc(&b, 2 * count));
    }
    FO_CUDA(cudaMemset(a, 0, 2 * count));
    FO_CUDA(cudaDeviceSynchronize());
    cudaStream_t cs = c->comm_stream;
    auto once = [&] {
      switch (coll) {
        case FO_ALLREDUCE:
          c->comm->allreduce(a, a, count, cs);
          break;
        case FO_REDUCESCATTER:
          c->comm->reducescatter(a, b, count / W, cs);
          break;
        case FO_ALLTOALL: {
          const size_t per = count / W;
          c->comm->group_start();
          for (int d = 0; d < W; ++d) {
            c->comm->send(reinterpret_cast<char*>(a) + 2 * per * d, per, d, cs);
            c->comm->recv(reinterpret_cast<char*>(b) + 2 * per * d, per, d, cs);
          }
          c->comm->group_end(cs);
          break;
        }
        default:
          fail(FO_ERR_INVALID_ARG, "unknown collective %d", coll);
      }
    };
    cudaEvent_t e0, e1;
    FO_CUDA(cudaEventCreate(&e0));
    FO_CUDA(cudaEventCreate(&e1));
    for (int i = 0; i < 2; ++i) once();
    FO_CUDA(cudaEventRecord(e0, cs));
    for (int i = 0; i < iters; ++i) once();
    FO_CUDA(cudaEventRecord(e1, cs));
    FO_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    FO_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    *avg_us = 1e3 * ms / iters;
    // bus bandwidth, nccl-tests convention: AllReduce 2(n-1)/n S, ReduceScatter
    // and All-to-All (n-1)/n S, over the message's total bytes S
    if (busbw_gbps) {
      const double S = 2.0 * (double)count, n = (double)W;
      const double factor = (coll == FO_ALLREDUCE) ? 2.0 * (n - 1) / n : (n - 1) / n;
      *busbw_gbps = (*avg_us > 0) ? S * factor / (*avg_us * 1e-6) / 1e9 : 0.0;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (reg) {
      for (void* h : {ha, hb})
        if (h) ncclCommDeregister(comm, h);
      for (ncclWindow_t w : {wa, wb})
        if (w) ncclCommWindowDeregister(comm, w);
      ncclMemFree(a);
      ncclMemFree(b);
    } else {
      cudaFree(a);
      cudaFree(b);
    }
  });
}

fo_status fo_plan_set_debug(fo_plan p, unsigned long long* tile_ts, unsigned long long* group_ts,
                            int32_t group_post) {
  return guard([&] {
    if (!p) fail(FO_ERR_INVALID_ARG, "null plan");
    if (group_post < -1 || group_post > 1) fail(FO_ERR_INVALID_ARG, "group_post must be -1, 0 or 1");
    p->trace_tile_ts = tile_ts;
    p->trace_group_ts = group_ts;
    p->group_post = group_post;
  });
}

fo_status fo_plan_set_option(fo_plan p, int32_t option, int64_t value) {
  return guard([&] {
    if (!p) fail(FO_ERR_INVALID_ARG, "null plan");
    switch (option) {
      case FO_OPT_GROUP_POST:
        if (value < -1 || value > 1) fail(FO_ERR_INVALID_ARG, "group_post must be -1, 0 or 1");
        p->group_post = (int)value;
        break;
      case FO_OPT_POST_SM_PARTITION:
        if (value < 0 || value > 1) fail(FO_ERR_INVALID_ARG, "post_sm_partition must be 0 or 1");
        p->post_sm_partition = (int)value;
        break;
      case FO_OPT_TAIL_SPLIT:
        if (value < -3 || value > 16) fail(FO_ERR_INVALID_ARG, "tail_split must be -3..16");
        if (p->device >= 0) fail(FO_ERR_STATE, "tail_split must be set before the plan's first run");
        p->tail_split_req = (int)value;
        break;
      case FO_OPT_WAIT_KERNEL:
        if (value < 0 || value > 1) fail(FO_ERR_INVALID_ARG, "wait_kernel must be 0 or 1");
        p->wait_kernel = (int)value;
        break;
      case FO_OPT_HOST_CHUNKS:
        if (value < 1 || value > 4096) fail(FO_ERR_INVALID_ARG, "host_chunks must be 1..4096");
        if (p->a_chunks) fail(FO_ERR_STATE, "host_chunks must be set before the first fo_run_host");
        p->a_chunk_target = (int)value;
        break;
      case FO_OPT_HOST_PIPELINE:
        if (value < 0 || value > 7) fail(FO_ERR_INVALID_ARG, "host_pipeline must be 0..7");
        p->host_pipeline = (int)value;
        break;
      case FO_OPT_DIST_FOLD:
        if (value < 0 || value > 1) fail(FO_ERR_INVALID_ARG, "dist_fold must be 0 or 1");
        p->dist_fold_opt = (int)value;
        break;
      case FO_OPT_GEMM_SWIGLU:
        if (value < 0 || value > 1) fail(FO_ERR_INVALID_ARG, "gemm_swiglu must be 0 or 1");
        if (value && (p->host.coll != FO_NOCOMM || p->host.BN != 256 || p->host.BM == 64 || p->host.post != FO_POST_NONE))
          fail(FO_ERR_UNSUPPORTED, "the SwiGLU epilogue needs a no-comm plan with tile_n 256 and post none");
        p->swiglu = (int)value;
        break;
      case FO_OPT_DEBUG_STALL_GROUP:
        if (value < -1 || value >= p->host.P) fail(FO_ERR_INVALID_ARG, "debug_stall_group must be -1..P-1");
        p->debug_stall_group = (int)value;
        break;
      case FO_OPT_MULTICAST:
        if (value < 0 || value > 1) fail(FO_ERR_INVALID_ARG, "multicast must be 0 or 1");
        p->multicast = (int)value;
        break;
      case FO_OPT_WAVE_SYNC:
        if (value < 0 || value > 1) fail(FO_ERR_INVALID_ARG, "wave_sync must be 0 or 1");
        p->wave_sync = (int)value;
        break;
      case FO_OPT_TMA_STORE:
        if (value < 0 || value > 1) fail(FO_ERR_INVALID_ARG, "tma_store must be 0 or 1");
        p->tma_store = (int)value;
        break;
      case FO_OPT_POST_BULK:
        if (value < 0 || value > 1) fail(FO_ERR_INVALID_ARG, "post_bulk must be 0 or 1");
        p->post_bulk = (int)value;
        break;
      case FO_OPT_K_SNAKE:
        if (value < -1 || value > 1) fail(FO_ERR_INVALID_ARG, "k_snake must be -1, 0 or 1");
        p->k_snake = (int)value;
        break;
      case FO_OPT_LAST_GROUP_IN_ORDER:
        if (value < 0 || value > 1) fail(FO_ERR_INVALID_ARG, "last_group_in_order must be 0 or 1");
        p->last_in_order = (int)value;
        break;
      default:
        fail(FO_ERR_INVALID_ARG, "unknown option %d", option);
    }
  });
}

fo_status fo_plan_fill_buffers(fo_plan p, uint16_t pattern, void* stream) {
  return guard([&] {
    if (!p) fail(FO_ERR_INVALID_ARG, "null plan");
    ensure_device(p);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (p->d_send) FO_CUDA(launch_fill_u16(p->d_send, p->host.send_elems, pattern, s));
    if (p->d_recv) FO_CUDA(launch_fill_u16(p->d_recv, p->host.recv_elems, pattern, s));
  });
}

}  // extern "C"
