// Communicator backends behind a context.  Every communication call of the
// data path goes through this interface, and fo_run / fo_run_sequential issue
// exactly the calls of the plan's schedule (PlanHost::calls / seq_calls,
// exported by fo_plan_export_calls).
//
//  * NcclComm     — the product backend: ncclAllReduce / ncclReduceScatter /
//                   ncclAllGather / ncclSend / ncclRecv on a
//                   library-owned or borrowed communicator.
//  * LoopbackComm — TEST backend (fo_loopback_create / fo_ctx_create_loopback):
//                   W ranks of one process on ONE GPU, each rank's calls run
//                   as small kernels that meet the other ranks' calls at a
//                   device-side barrier and move the data with plain loads and
//                   stores.  It lets a single-GPU box run fo_run end to end at
//                   world 2/4/8 (streams, stream waits, call order, offsets,
//                   counts, peers) against the oracle.
//  * EmuComm      — EVALUATION backend (fo_ctx_create_emulated): one rank whose
//                   collectives take the time NVLink would (bytes / link
//                   bandwidth + latency) and move their local HBM traffic on
//                   the SMs the GEMM leaves free; it validates Alg. 1's
//                   predictor and the overlap schedule on one GPU.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstddef>

namespace fo {

struct Comm {
  virtual ~Comm() {}
  virtual int rank() const = 0;
  virtual int world() const = 0;
  // bf16 sum, in place allowed (send == recv)
  virtual void allreduce(const void* send, void* recv, size_t count, cudaStream_t s) = 0;
  // recv[count] = sum over ranks of send[rank*count ...]
  virtual void reducescatter(const void* send, void* recv, size_t recvcount, cudaStream_t s) = 0;
  // recv[q*count ...] = rank q's send[count]
  virtual void allgather(const void* send, void* recv, size_t sendcount, cudaStream_t s) = 0;
  virtual void group_start() = 0;
  virtual void group_end(cudaStream_t s) = 0;  // s: the stream of the group's calls
  virtual void send(const void* buf, size_t count, int peer, cudaStream_t s) = 0;
  virtual void recv(void* buf, size_t count, int peer, cudaStream_t s) = 0;
  // the watchdog: make in-flight calls exit (the communicator is unusable afterwards)
  virtual void abort() = 0;
  // the NCCL communicator, or nullptr (loopback)
  virtual ncclComm_t nccl() const { return nullptr; }
};

// NCCL backend; owns (destroys / may abort) the communicator iff `owns`.
Comm* make_nccl_comm(ncclComm_t comm, int rank, int world, bool owns);

// Loopback test backend (loopback.cu): a group of `world` in-process ranks on
// one device; every rank's context gets make_loopback_comm(group, rank).
struct LoopbackGroup;
LoopbackGroup* loopback_create(int device, int world);
void loopback_destroy(LoopbackGroup* g);
int loopback_members(LoopbackGroup* g);
int loopback_world(LoopbackGroup* g);
int loopback_device(LoopbackGroup* g);
Comm* make_loopback_comm(LoopbackGroup* g, int rank);

// Emulated-link EVALUATION backend (emulated.cu): rank `rank` of `world` whose
// collectives are kernels moving the call's local HBM traffic for at least
// latency_us + bus bytes / link_gbps (timing only; results are not the
// collective's).
Comm* make_emulated_comm(int rank, int world, double link_gbps, double latency_us, int ctas);

}  // namespace fo
