// Runtime objects behind the opaque C handles.
#pragma once

#include <cstdint>
#include <vector>

#include "kernels.h"
#include "plan.h"

#include <nccl.h>

struct fo_ctx_s;

struct fo_plan_s {
  fo::PlanHost host;
  // ---- device state (created lazily on first device use)
  int device = -1;
  int32_t* d_order = nullptr;
  int32_t* d_pos_of_tile = nullptr;
  int32_t* d_group_of_pos = nullptr;
  int32_t* d_gpos = nullptr;
  int32_t* d_row_slot = nullptr;
  int2* d_rs_info = nullptr;        // RS: per position {group's first position, group size}
  int32_t* d_src_row = nullptr;
  uint32_t* d_counters = nullptr;
  void* d_send = nullptr;  // pre-reordered send buffer (bf16), library-owned
  void* d_recv = nullptr;  // receive buffer (RS / A2A)
  void* d_rowmajor = nullptr;  // sequential baseline scratch (RS / A2A row-major C)
  // ---- NCCL buffer registration (fo_ctx_config.buffers of the first context)
  int mem_mode = 0;            // 0 plain, 1 ncclMemAlloc + ncclCommRegister, 2 + window registration
  bool nccl_mem = false;       // d_send / d_recv came from ncclMemAlloc
  fo_ctx_s* reg_ctx = nullptr; // context whose communicator holds the registrations
  void *reg_send = nullptr, *reg_recv = nullptr;
  ncclWindow_t win_send = nullptr, win_recv = nullptr;
  int32_t* d_recv_dst = nullptr;  // A2A received subtoken -> output position
  // ---- device staging for fo_run_host (lazily allocated)
  void* h_A = nullptr;
  void* h_Bt = nullptr;
  void* h_out = nullptr;
  void* h_res = nullptr;
  void* h_gamma = nullptr;
  // ---- fo_run_host pipelining (FO_OPT_HOST_PIPELINE): A copied in chunks of
  // a_chunk_rows tile-rows, each followed by a release write of the run's
  // epoch into d_a_ready[chunk]; the GEMM producer waits per tile-row
  int host_pipeline = 7;                          // bit 0: chunked A, bit 1: per-group D2H, bit 2: 2 staging sets
  void* h_A2 = nullptr;                           // second A / out staging set (bit 2: consecutive
  void* h_out2 = nullptr;                         //   calls alternate, so call i+1's H2D overlaps call i)
  int host_set = 0;                               // staging set of the next fo_run_host
  cudaEvent_t ev_set_done[2] = {nullptr, nullptr};  // last call on set b finished (its staging is free)
  uint32_t* d_a_ready = nullptr;
  uint32_t a_epoch = 0;
  int a_chunk_target = 8;                         // FO_OPT_HOST_CHUNKS
  int a_chunk_rows = 0, a_chunks = 0;
  std::vector<int> a_chunk_order;                 // chunks in order of first use
  bool a_staged_run = false;                      // transient: this fo_run's GEMM waits on d_a_ready
  void* d2h_host = nullptr;                       // transient: per-group D2H of out (AR ROWBAND) to here
  const fo::CombineArgs* combine = nullptr;       // transient: fo_run_combine replaces the A2A post pass
  // ---- debug / evidence hooks (fo_plan_set_debug)
  unsigned long long* trace_tile_ts = nullptr;   // device [tiles]
  unsigned long long* trace_group_ts = nullptr;  // device [2P]: wait released, group done
  int group_post = -1;                            // -1 auto, 0 off, 1 on
  int wait_kernel = 0;                            // 0 cuStreamWaitValue32, 1 spin-wait kernel
  int last_in_order = 1;                          // last group's collective on the caller stream after the GEMM
  int post_sm_partition = 0;                      // FO_OPT_POST_SM_PARTITION
  int free_sms = 0;                               // SMs the persistent GEMM leaves free (set by ensure_device)
  int tail_split_req = 0;                         // FO_OPT_TAIL_SPLIT: 0/1 off, >=2 slices, -1 auto, -2 stream-K
  // ---- resolved tail split (set by ensure_device)
  int split = 1, tail_pos = 0, units = 0;
  int dist_fold = 0;                              // f-slice split: distributed fold possible
  int dist_fold_opt = 1;                          // FO_OPT_DIST_FOLD
  float* d_ws = nullptr;                          // fp32 partials of the split tail
  fo::GemmSeg* d_seg = nullptr;                   // the split tail's K-ranges by worker
  int32_t* d_wseg = nullptr;                      // [S+1] per-worker segment offsets
  uint32_t* d_flags = nullptr;                    // = d_counters + P (one allocation, reset together)
  int ctr_words = 0;                              // P + tail flags
  // ---- wave alignment of the persistent producers (FO_OPT_WAVE_SYNC)
  int wave_sync = 0;
  int multicast = 0;                              // FO_OPT_MULTICAST (measured slower: off)
  int k_snake = -1;                               // FO_OPT_K_SNAKE (-1 auto: K >= 64 k-blocks)
  int tma_store = 1;                              // FO_OPT_TMA_STORE
  int post_bulk = 1;                              // FO_OPT_POST_BULK
  int debug_stall_group = -1;                     // FO_OPT_DEBUG_STALL_GROUP (watchdog test)
  int swiglu = 0;                                 // FO_OPT_GEMM_SWIGLU (no-comm GEMM epilogue)
  uint32_t* d_wave = nullptr;                     // [T] monotone per-wave issue counters
  uint32_t gemm_launches = 0;                     // launches of this plan's GEMM so far (wave epoch)
};

namespace fo {
void release_device(fo_plan_s* p);
}
