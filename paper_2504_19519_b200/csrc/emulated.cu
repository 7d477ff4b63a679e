// EVALUATION backend of fo::Comm (comm.h): one process acting as rank `rank`
// of a `world`-rank tensor-parallel group whose NVLink collectives are
// emulated on this GPU (fo_ctx_create_emulated).  NOT a communicator: no data
// leaves the GPU and the results are not the collective's (below).
//
// Why: the build boxes have one B200, so the overlapped op has only ever run
// against a 1-rank NCCL call that moves nothing.  Alg. 1's predictor
// and the overlap machinery (signals, stream waits, the
// per-group calls, the last group in stream order) are validated by the paper
// against real collectives whose duration grows with the group's bytes
// (PAPER.md:625-647).  This backend gives every call that shape: a kernel of
// `ctas` CTAs (512 threads) on the communication stream that
//   1. moves the call's LOCAL HBM traffic (reads the send range, writes the
//      receive range, as a rank's NCCL kernels do), and
//   2. does not finish before latency_us + bus_bytes / link_gbps after it
//      started (%globaltimer), bus_bytes in the nccl-tests convention per rank:
//      AllReduce 2(n-1)/n x bytes, ReduceScatter / AllGather (n-1)/n x the full
//      buffer, grouped send/recv max(bytes sent, bytes received).
// It occupies SMs the persistent GEMM leaves free, like NCCL's kernels, and
// its stream / event / wait structure is the real one.
//
// Results: AllReduce leaves the rank's own partial (as if the other ranks
// contributed zeros), ReduceScatter delivers the rank's own chunk,
// AllGather replicates the rank's part into every slot, receives are zeroed.
// Timing only — tools/predictor_check.py --emulate, never the bench value.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "comm.h"
#include "common.h"
#include "kernels.h"

namespace fo {

namespace {

// dst[j] = src[j % n_src] for j < n_dst (16-byte vectors; src null: zeros),
// plus a read-only sweep of rd[0 .. n_rd) (the send data a reduction reads);
// then spin until `dur_ns` after the CTA started (the CTAs of a call start
// together on the SMs the GEMM leaves free).  Each thread keeps EMU_UNROLL
// 16-byte loads in flight (64 KB per CTA), like a collective's copy loop, so
// a few CTAs move the call's bytes at the link rate instead of at the rate
// one load per thread allows.
constexpr int EMU_THREADS = 512;
constexpr int EMU_UNROLL = 8;

__global__ void __launch_bounds__(EMU_THREADS) fo_emu_link_kernel(const uint4* rd, int64_t n_rd, const uint4* src,
                                                                  int64_t n_src, uint4* dst, int64_t n_dst,
                                                                  unsigned long long dur_ns) {
  unsigned long long t0, now;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t span = (int64_t)gridDim.x * blockDim.x;  // consecutive threads -> consecutive vectors
  uint32_t acc = 0;
  for (int64_t base = 0; base < n_rd; base += span * EMU_UNROLL) {
    uint4 v[EMU_UNROLL];
#pragma unroll
    for (int u = 0; u < EMU_UNROLL; ++u) {
      const int64_t i = base + u * span + tid;
      v[u] = i < n_rd ? __ldcs(rd + i) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < EMU_UNROLL; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  for (int64_t base = 0; base < n_dst; base += span * EMU_UNROLL) {
    uint4 v[EMU_UNROLL];
#pragma unroll
    for (int u = 0; u < EMU_UNROLL; ++u) {
      const int64_t j = base + u * span + tid;
      v[u] = (src && j < n_dst) ? __ldcs(src + (j % n_src)) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < EMU_UNROLL; ++u) {
      const int64_t j = base + u * span + tid;
      if (j < n_dst) __stcs(dst + j, v[u]);
    }
  }
  if (acc == 0x9e3779b9u && n_rd < 0) dst[0] = make_uint4(acc, 0, 0, 0);  // keeps the read sweep (never true)
  if (threadIdx.x == 0) {
    while (true) {
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (now >= t0 + dur_ns) break;
      __nanosleep(256);
    }
  }
  __syncthreads();
}

struct EmuComm : Comm {
  int r, w, ctas;
  double gbps, lat_us;
  struct P2P {
    bool send;
    void* buf;
    size_t count;
  };
  std::vector<P2P> pending;
  bool in_group = false;

  EmuComm(int rank, int world, double link_gbps, double latency_us, int c)
      : r(rank), w(world), ctas(c), gbps(link_gbps), lat_us(latency_us) {}
  int rank() const override { return r; }
  int world() const override { return w; }

  unsigned long long wire_ns(double bus_bytes) const {
    return (unsigned long long)((lat_us * 1e3) + bus_bytes / gbps);  // GB/s = bytes/ns
  }
  void launch(const void* rd, size_t rd_bytes, const void* src, size_t src_bytes, void* dst, size_t dst_bytes,
              double bus_bytes, cudaStream_t s) {
    fo_emu_link_kernel<<<ctas, EMU_THREADS, 0, s>>>(static_cast<const uint4*>(rd), (int64_t)(rd_bytes / 16),
                                            static_cast<const uint4*>(src), (int64_t)(src_bytes / 16),
                                            static_cast<uint4*>(dst), (int64_t)(dst_bytes / 16), wire_ns(bus_bytes));
    count_launch();
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) fail(FO_ERR_CUDA, "emulated link launch: %s", cudaGetErrorString(e));
  }
  void allreduce(const void* send, void* recv, size_t count, cudaStream_t s) override {
    const double b = 2.0 * count;
    launch(nullptr, 0, send, 2 * count, recv, 2 * count, 2.0 * (w - 1) / w * b, s);
  }
  void reducescatter(const void* send, void* recv, size_t recvcount, cudaStream_t s) override {
    const char* own = static_cast<const char*>(send) + 2 * (size_t)r * recvcount;
    launch(send, 2 * recvcount * (size_t)w, own, 2 * recvcount, recv, 2 * recvcount,
           (double)(w - 1) * 2.0 * recvcount, s);
  }
  void allgather(const void* send, void* recv, size_t sendcount, cudaStream_t s) override {
    launch(nullptr, 0, send, 2 * sendcount, recv, 2 * sendcount * (size_t)w, (double)(w - 1) * 2.0 * sendcount, s);
  }
  void group_start() override {
    in_group = true;
    pending.clear();
  }
  void group_end(cudaStream_t s) override {
    double sent = 0, recvd = 0;
    for (const P2P& p : pending) (p.send ? sent : recvd) += 2.0 * p.count;
    // the traffic of every send (read) and receive (write), then one wire-time wait
    for (const P2P& p : pending) {
      if (p.send) launch(p.buf, 2 * p.count, nullptr, 0, nullptr, 0, 0.0, s);
      else launch(nullptr, 0, nullptr, 0, p.buf, 2 * p.count, 0.0, s);
    }
    if (!pending.empty()) launch(nullptr, 0, nullptr, 0, nullptr, 0, std::max(sent, recvd), s);
    pending.clear();
    in_group = false;
  }
  void send(const void* buf, size_t count, int, cudaStream_t s) override {
    if (!in_group) {
      group_start();
      pending.push_back({true, const_cast<void*>(buf), count});
      group_end(s);
      return;
    }
    pending.push_back({true, const_cast<void*>(buf), count});
  }
  void recv(void* buf, size_t count, int, cudaStream_t s) override {
    if (!in_group) {
      group_start();
      pending.push_back({false, buf, count});
      group_end(s);
      return;
    }
    pending.push_back({false, buf, count});
  }
  void abort() override {}
};

}  // namespace

Comm* make_emulated_comm(int rank, int world, double link_gbps, double latency_us, int ctas) {
  return new EmuComm(rank, world, link_gbps, latency_us, ctas);
}

}  // namespace fo
