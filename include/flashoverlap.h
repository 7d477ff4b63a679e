/*
 * flashoverlap.h — C ABI of the B200-native FlashOverlap hot path
 * (arXiv 2504.19519, "Efficient and Adaptable Overlapping for Computation and
 * Communication via Signaling and Reordering").
 *
 * The library runs ONE tensor-parallel GEMM  C = A · Btᵀ as a
 * single persistent tcgen05 kernel whose epilogue stores every finished tile
 * into a pre-communication-reordered buffer and bumps a per-wave-group counter
 * (signaling; reordering).  A
 * communication stream waits on each counter (cuStreamWaitValue32, no SM
 * spent) and issues a plain NCCL AllReduce / ReduceScatter / All-to-All on the
 * group's contiguous range.  A post-communication reorder
 * kernel restores row-major order, optionally fused with residual-add and
 * RMSNorm.  Alg. 1 is exposed as
 * fo_tune_search / fo_tune_predict.
 *
 * Conventions
 *  - Matrices are bf16, row-major, contiguous.  A is [m, k] (K-major); Bt is
 *    [n, k] (the nn.Linear weight layout, K-major); C is [m, n].
 *  - "device" pointers are CUDA device addresses on the context's device.
 *    "host" pointers are ordinary CPU memory, read during the call only
 *    (the library copies what it keeps).
 *  - Streams are passed as void* (a cudaStream_t); NULL is the legacy stream.
 *  - Tiles: tile id t = i*nt + j (tile-row i, tile-column j).  Execution
 *    position p in [0, tiles): the persistent kernel runs the tile
 *    tile_order[p] as the p-th unit; worker w of S runs positions w, w+S, ...
 *    so position p belongs to wave floor(p/S) and to the wave
 *    group containing that wave.
 *  - Every function returns fo_status; nothing is thrown across the ABI.
 *    On a non-OK status fo_last_error() returns a thread-local message.
 *
 * Ownership: the caller owns A, Bt, out, residual, gamma and every buffer it
 * passes; they must stay valid until the stream reaches the end of the op.
 * The library owns contexts (NCCL communicator, streams, events) and plans
 * (device tables, the communication buffer, the counting table); the
 * matching *_destroy releases them.
 */
#ifndef FLASHOVERLAP_H_
#define FLASHOVERLAP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FO_OK = 0,
  FO_ERR_INVALID_ARG = 1, /* non-permutation order, sum(group_waves) != T, zero group, row_dst out of range, NULL */
  FO_ERR_SHAPE = 2,       /* m % tile_m, n % tile_n, k % 64, tile_m % world (RS) */
  FO_ERR_UNSUPPORTED = 3, /* tile shape not compiled, layout not applicable, no sm_100 device */
  FO_ERR_CUDA = 4,
  FO_ERR_NCCL = 5,
  FO_ERR_OOM = 6,
  FO_ERR_TIMEOUT = 7,
  FO_ERR_STATE = 8        /* plan used with a mismatched context, etc. */
} fo_status;

/* Which collective follows the GEMM. */
typedef enum {
  FO_ALLREDUCE = 0,     /* TP row-parallel linear; every rank gets sum_r C_r           */
  FO_REDUCESCATTER = 1, /* TP + sequence parallel; rank k gets rows R_k of sum_r C_r    */
  FO_ALLTOALL = 2,      /* EP combine; row g of C goes to rank row_dst[g]               */
  FO_NOCOMM = 3         /* plain GEMM writing row-major C (sequential baseline, tuner)  */
} fo_coll;

/* AllReduce / ReduceScatter / All-to-All buffer layout (H11a, R40, R41). */
typedef enum {
  FO_LAYOUT_SLOT = 0,    /* paper: AR: tile at position p -> contiguous slot p (tile_m*tile_n elems, row-major);
                            RS: subtile k of every tile of a group -> chunk k of the group */
  FO_LAYOUT_ROWBAND = 1, /* every group is a band of whole tile-rows.  AR: the epilogue writes C in place and
                            both reorders are the identity.  RS (bands must also be ascending in group order):
                            chunk k of a band holds the k-th subtile rows of its tiles as complete rows, so the
                            ReduceScatter of the band lands the rank's block-cyclic rows R_k directly in `out`
                            (no receive buffer, no post-communication reorder).  A2A (every source's bands
                            ascending, decided from the census descriptors so all ranks agree): pools hold complete
                            rows in source-row order and each group's rows from a source are received straight
                            into their output rows (R41) */
  FO_LAYOUT_AUTO = 2     /* ROWBAND when legal, else SLOT; with swizzle 0 the default order prefers panel heights
                            whose panels end on the group boundaries (AR and RS; ROWBAND asked for explicitly:
                            any collective) */
} fo_ar_layout;

/* Elementwise op fused into the post-communication reorder (R12). */
typedef enum {
  FO_POST_NONE = 0,
  FO_POST_ADD = 1,          /* out = x + residual                                   */
  FO_POST_ADD_RMSNORM = 2,  /* y = x + residual; out = y / sqrt(mean(y^2) + eps) * gamma */
  FO_POST_ADD_RMSNORM_RESIDUAL = 3  /* as ADD_RMSNORM, and y (bf16) is written back into the residual
                                       buffer in place — the next layer's residual stream (the fused
                                       add + RMSNorm of a pre-norm transformer block) */
} fo_post;

typedef struct fo_ctx_s* fo_ctx;
typedef struct fo_plan_s* fo_plan;

/* One rank's view of the overlapped layer.  All pointers are HOST pointers,
 * read during fo_plan_create only. */
typedef struct {
  int32_t coll;          /* fo_coll */
  int32_t ar_layout;     /* fo_ar_layout (AllReduce, ReduceScatter, All-to-All; ignored for no-comm) */
  int64_t m, n, k;       /* this rank's GEMM: A [m,k], Bt [n,k], C [m,n]; k = K/world for TP;
                            m = 0 only for an All-to-All source with no rows (an expert
                            no token was routed to: no GEMM, P empty groups, whose
                            group_waves are all 0; R45) */
  int32_t tile_m;        /* 64 or 128 (one CTA, tcgen05.mma M=64 / M=128; 64: K-major operands, no tail split)
                            or 256 (cta_group::2 CTA pair) */
  int32_t tile_n;        /* 64, 128 or 256 */
  int32_t workers;       /* S >= 1 = concurrent tile workers = wave width (grid of the persistent GEMM) */
  const int32_t* tile_order; /* [tiles] permutation of tile ids, or NULL => default swizzle */
  int32_t swizzle;       /* default order: row-panels of `swizzle` tile-rows, column-major inside (R1);
                            0 = auto: the panel height minimising the tile-rows + tile-columns the waves touch,
                            summed over all waves (the operand panels streamed from HBM; R25), or the Hilbert
                            order when that is 5% lower (and no band layout needs panels); -1 = a generalized
                            Hilbert curve over the tile grid (R44) */
  int32_t num_groups;    /* P */
  const int32_t* group_waves; /* [P] wave counts, sum == T = ceil(tiles / S); NULL => one group;
                                 all 0 when m == 0 (All-to-All) */
  const int32_t* row_dst;     /* All-to-All: [m] destination rank of each output row (may be NULL when m == 0) */
  int32_t post;          /* fo_post */
  float eps;             /* RMSNorm epsilon */
  int32_t a_mn_major;    /* 0: A is [m, k] row-major (K-major); 1: A is stored [k, m] row-major (M-major),
                            e.g. dY of a weight-gradient GEMM dW = dY^T X (NEXT f4) */
  int32_t b_mn_major;    /* 0: Bt is [n, k] row-major (K-major); 1: stored [k, n] row-major (N-major), e.g. X.
                            MN-major operands need tile_n >= 128 */
} fo_plan_desc;

typedef struct {
  int32_t rank, world;
  int32_t mt, nt, tiles;
  int32_t workers;       /* S actually used */
  int32_t waves;         /* T */
  int32_t num_groups;    /* P */
  int32_t ar_layout;     /* resolved layout (ROWBAND for no-comm) */
  int32_t rs_subtile_rows; /* h = tile_m / world (ReduceScatter) */
  int64_t send_elems;    /* elements of the pre-reordered send buffer */
  int64_t recv_elems;    /* elements of the receive layout (AR: == send; RS ROWBAND: it is `out` itself) */
  int64_t out_rows, out_cols; /* shape of `out` expected by fo_run */
} fo_plan_info;

/* ---------------------------------------------------------------- library */
const char* fo_last_error(void);
const char* fo_version(void);
/* Number of SMs of `device` (0 if no device); for choosing workers. */
fo_status fo_device_sm_count(int32_t device, int32_t* sm_count);

/* ---------------------------------------------------------------- plan (host only, no GPU needed) */
/* Build the host-side plan of rank `rank` in a `world`-rank group.
 * peers: All-to-All only — peers[s] is rank s's descriptor (peers[rank] may be
 * `self`); every rank must use the same number of groups P.  The caller
 * gathers the peer descriptors (e.g. torch.distributed all_gather_object);
 * this is the "census" of the A2A receive layout.  Ignored
 * (may be NULL) for AllReduce / ReduceScatter / no-comm.
 * No CUDA call is made; device state is created lazily by the first run. */
fo_status fo_plan_create(const fo_plan_desc* self, int32_t rank, int32_t world,
                         const fo_plan_desc* const* peers, fo_plan* out);
fo_status fo_plan_destroy(fo_plan plan);
fo_status fo_plan_get_info(fo_plan plan, fo_plan_info* info);
/* Group j: execution positions [pos_begin, pos_end) and send-buffer element
 * range [elem_begin, elem_end) (AR / RS; for A2A the element range spans the
 * group's part of pool 0..world-1 and is informational). */
fo_status fo_plan_group(fo_plan plan, int32_t j, int32_t* pos_begin, int32_t* pos_end,
                        int64_t* elem_begin, int64_t* elem_end);
/* Parity exports (host arrays, caller-allocated):
 *  order[tiles]                 execution order (tile id at position p)
 *  send_map[m*n]                send-buffer element index of C[r][c] (index r*n + c)
 *  recv_map[out_rows*out_cols]  receive-buffer element index read for out[r][c]
 *  a2a_send_cnt[P*world], a2a_recv_cnt[P*world]  subtokens per (group, peer) */
fo_status fo_plan_export_order(fo_plan plan, int32_t* order);
fo_status fo_plan_export_send_map(fo_plan plan, int64_t* send_map);
fo_status fo_plan_export_recv_map(fo_plan plan, int64_t* recv_map);
fo_status fo_plan_export_a2a_counts(fo_plan plan, int64_t* a2a_send_cnt, int64_t* a2a_recv_cnt);

/* ---------------------------------------------------------------- communication schedule
 * The exact list of communication calls a plan issues ("Once the
 * j-th number reaches |G_j|, the communication of G_j starts"
 * NCCL AllReduce / ReduceScatter / send-recv All-to-All; PAPER.md:381-392 the
 * contiguous per-group ranges).  fo_run and fo_run_sequential execute THESE
 * calls, in this order, on the communicator (no other communication call is
 * made on the data path), so a host-only test can check every offset, count
 * and peer against the oracle, and that all ranks' schedules match, without a
 * GPU.  Buffers are named, offsets and counts are in bf16 ELEMENTS:
 *   FO_BUF_SEND    the plan's library-owned pre-reordered send buffer
 *                  (info.send_elems)
 *   FO_BUF_RECV    the plan's library-owned receive buffer (info.recv_elems;
 *                  at world 1 it is the send buffer itself)
 *   FO_BUF_OUT     the caller's `out` of fo_run / fo_run_sequential
 *   FO_BUF_SCRATCH the sequential baseline's row-major C [m, n] (RS / A2A)
 * Call semantics (NCCL's, bf16, sum):
 *   ALLREDUCE      in place: buf src_buf, elements [src_off, src_off+count)
 *   REDUCESCATTER  send src_buf[src_off, src_off + world*count), receive
 *                  dst_buf[dst_off, dst_off + count)  (count = NCCL recvcount)
 *   SEND / RECV    point-to-point with `peer`, count elements from src_buf at
 *                  src_off (SEND) / into dst_buf at dst_off (RECV); only inside
 *                  a GROUP_START ... GROUP_END bracket; sends and receives of
 *                  one (source, destination) pair match in order
 *   LOCAL_COPY     count elements src_buf[src_off..] -> dst_buf[dst_off..] on
 *                  this rank (the All-to-All self part; skipped when source and
 *                  destination coincide)
 * `group` is the wave group the call belongs to (-1 for the sequential
 * schedule).  schedule 0 = fo_run, 1 = fo_run_sequential.  capacity = entries
 * `calls` can hold; *ncalls receives the schedule length (calls may be NULL to
 * query it; FO_ERR_INVALID_ARG if capacity is too small).  Host only. */
typedef enum { FO_CALL_ALLREDUCE = 0, FO_CALL_REDUCESCATTER = 1, FO_CALL_SEND = 2, FO_CALL_RECV = 3,
               FO_CALL_LOCAL_COPY = 4, FO_CALL_GROUP_START = 5, FO_CALL_GROUP_END = 6 } fo_call_kind;
typedef enum { FO_BUF_NONE = -1, FO_BUF_SEND = 0, FO_BUF_RECV = 1, FO_BUF_OUT = 2, FO_BUF_SCRATCH = 3 } fo_buf;
typedef struct {
  int32_t kind;      /* fo_call_kind */
  int32_t group;     /* wave group j, -1 in the sequential schedule */
  int32_t peer;      /* SEND / RECV: the other rank; else -1 */
  int32_t src_buf;   /* fo_buf */
  int32_t dst_buf;   /* fo_buf */
  int32_t reserved;
  int64_t src_off;   /* elements */
  int64_t dst_off;   /* elements */
  int64_t count;     /* elements (NCCL's count argument) */
} fo_comm_call;
fo_status fo_plan_export_calls(fo_plan plan, int32_t schedule, fo_comm_call* calls, int32_t capacity,
                               int32_t* ncalls);

/* ---------------------------------------------------------------- context (one per process / GPU) */
/* NCCL unique id (128 bytes) made on one rank and broadcast by the caller. */
fo_status fo_get_unique_id(uint8_t uid[128]);
/* Create the library's NCCL communicator (rank of world) on `device` plus a
 * highest-priority communication stream.  nccl_max_ctas > 0
 * caps NCCL's CTAs (ncclConfig_t.maxCTAs) so they fit the SMs the persistent
 * GEMM leaves free; 0 = NCCL default.  Collective over the ranks. */
fo_status fo_ctx_create(int32_t device, int32_t rank, int32_t world, const uint8_t uid[128],
                        int32_t nccl_max_ctas, fo_ctx* out);
/* Communicator configuration of fo_ctx_create_config (all 0 = NCCL defaults,
 * plain buffers; fo_ctx_create(..., max) = {max, 0, 0, 0, 0}).
 *   nccl_max_ctas / nccl_min_ctas  ncclConfig_t.maxCTAs / minCTAs: the CTAs
 *       NCCL may use, sized to the SMs the persistent GEMM leaves free
 *       (R18);
 *   cta_policy  ncclConfig_t.CTAPolicy: 0 default, 1 NCCL_CTA_POLICY_EFFICIENCY
 *       (fewest CTAs that keep the bandwidth), 2 NCCL_CTA_POLICY_ZERO;
 *   nvls_ctas   ncclConfig_t.nvlsCTAs (CTAs of the NVLS in-switch reduction);
 *   buffers     0: plans allocate their send / receive buffers with
 *       cudaMalloc; 1: with ncclMemAlloc, registered with the communicator
 *       (ncclCommRegister: zero-copy / NVLS-capable buffers);
 *       2: ncclMemAlloc + ncclCommWindowRegister (NCCL_WIN_COLL_SYMMETRIC for
 *       AllReduce / ReduceScatter plans, whose buffers have the same size on
 *       every rank).  A plan's buffers are allocated and registered for the
 *       context it first runs with (collective: every rank's first run of the
 *       plan); running it with another context is FO_ERR_STATE.  The
 *       registrations are released by fo_plan_destroy or fo_ctx_destroy,
 *       whichever comes first. */
typedef struct {
  int32_t nccl_max_ctas;
  int32_t nccl_min_ctas;
  int32_t cta_policy;
  int32_t nvls_ctas;
  int32_t buffers;
} fo_ctx_config;
fo_status fo_ctx_create_config(int32_t device, int32_t rank, int32_t world, const uint8_t uid[128],
                               const fo_ctx_config* config, fo_ctx* out);
/* Device memory for a caller buffer NCCL will read / write (the `out` of a
 * ROWBAND plan: AllReduce reduces it in place, ReduceScatter and the A2A
 * receives write it): ncclMemAlloc, registered with
 * the context's communicator per its `buffers` mode (none for mode 0).
 * fo_mem_free deregisters and frees (synchronises the device).  Window
 * registration (mode 2) is collective: every rank allocates the same size in
 * the same order. */
fo_status fo_mem_alloc(fo_ctx ctx, int64_t bytes, void** ptr);
fo_status fo_mem_free(fo_ctx ctx, void* ptr);
/* Create a context on an EXISTING NCCL communicator (an ncclComm_t passed as
 * void*, e.g. torch's ProcessGroupNCCL::_comm_ptr()): rank and world are read
 * from it (ncclCommUserRank / ncclCommCount); it must live on `device`
 * (ncclCommCuDevice), else FO_ERR_INVALID_ARG.  The communicator is BORROWED:
 * fo_ctx_destroy does not destroy it and the fo_plan_sync watchdog does not
 * abort it (it returns FO_ERR_TIMEOUT and the context stays unusable, aborting
 * is the owner's call).  The caller keeps it alive until fo_ctx_destroy, and
 * NCCL calls it issues on other streams are ordered against the library's only
 * by the caller.  Local (not collective); the NCCL config (maxCTAs) is the
 * owner's. */
fo_status fo_ctx_create_from_comm(int32_t device, void* nccl_comm, fo_ctx* out);
fo_status fo_ctx_destroy(fo_ctx ctx);
/* TEST BACKEND — W ranks of one process on ONE GPU.  A box with one GPU
 * cannot run NCCL with two ranks, so these make the library's multi-rank data
 * path (fo_run / fo_run_sequential / fo_run_allgather at world > 1: receive
 * buffers, per-group calls on the comm stream, the last group on the caller
 * stream, the plan's schedule) run for real on one device.
 * fo_loopback_create: a group of `world` in-process ranks on `device` (host
 * object `*group`).  fo_ctx_create_loopback: rank `rank`'s context in that
 * group (its own comm / post streams, like fo_ctx_create); its communication
 * calls are small kernels that meet the other ranks' calls at a device-side
 * barrier and move the data with loads / stores (AllReduce: fp32 sum in rank
 * order, one bf16 rounding).  The caller issues every rank's calls from its
 * threads in any interleaving, each rank in the same order as with NCCL.
 * A call sequence that differs between ranks (a hang with NCCL) or a barrier
 * not reached within 20 s traps the device (the CUDA context is lost) instead
 * of hanging.  Needs eager module loading (CUDA_MODULE_LOADING=EAGER before
 * CUDA starts; else FO_ERR_UNSUPPORTED): a lazily loaded kernel's first launch
 * may wait for running kernels, i.e. for another rank's call at its barrier.
 * Prepare every plan (fo_plan_prepare) before the ranks issue: an allocation
 * in one rank must not wait on another rank's call.  Not CUDA-graph capturable.  fo_loopback_destroy fails with
 * FO_ERR_STATE while contexts of the group exist.  Not for production use. */
fo_status fo_loopback_create(int32_t device, int32_t world, void** group);
fo_status fo_loopback_destroy(void* group);
fo_status fo_ctx_create_loopback(void* group, int32_t rank, fo_ctx* out);

/* EVALUATION BACKEND — an emulated NVLink group on ONE GPU (not a
 * communicator).  The context acts as rank `rank` of `world`; each of its
 * collectives is a kernel of `ctas` CTAs (512 threads) on the comm stream that
 * moves the call's local HBM traffic (reads the send range, writes the receive
 * range) and lasts at least latency_us + bus_bytes / link_gbps, bus_bytes per
 * rank in the nccl-tests convention (AllReduce 2(n-1)/n x bytes; ReduceScatter
 * and AllGather (n-1)/n x the full buffer; a grouped send/recv max(sent,
 * received) bytes).  Results are NOT the collective's: AllReduce leaves the
 * rank's own partial, ReduceScatter delivers its own chunk, AllGather
 * replicates its part, receives are zeroed.  It lets one B200 validate Alg. 1's
 * predictor and the overlap schedule against collectives
 * whose duration grows with the group's bytes (tools/predictor_check.py
 * --emulate).  FO_ERR_INVALID_ARG for world < 1, rank out of range,
 * link_gbps <= 0, latency_us < 0 or ctas outside 1..1024.  Not for production
 * use; never a benchmark value. */
fo_status fo_ctx_create_emulated(int32_t device, int32_t rank, int32_t world, double link_gbps, double latency_us,
                                 int32_t ctas, fo_ctx* out);

/* Offline stage of the tuner ("the bandwidth curve is sampled
 * with multiple dense points"): average latency of one `coll` (AllReduce in
 * place, ReduceScatter, or equal-split All-to-All) of `bytes` total message
 * bytes on the context's own communicator and comm stream (its CTA cap and
 * buffer registration included), and (busbw_gbps, may be NULL) the bus
 * bandwidth in the nccl-tests convention: AllReduce 2(n-1)/n x bytes,
 * ReduceScatter / All-to-All (n-1)/n x bytes, per second.  Collective;
 * synchronises the host (tuning only). */
fo_status fo_ctx_time_collective(fo_ctx ctx, int32_t coll, int64_t bytes, int32_t iters, double* avg_us,
                                 double* busbw_gbps);

/* ---------------------------------------------------------------- the overlapped op */
/* MoE combine fused into the All-to-All post-reorder (R31; the A2A
 * "transfer[s] the processed data back to the original GPUs after expert
 * computation"; the post-reorder fused into the following
 * elementwise kernel).  On the token-owning rank:
 *   out[t] = sum_{i<topk} w[t*topk+i] * X[idx[t*topk+i]]  (+ residual[t])
 * where X is this rank's standard A2A output (the rows fo_run would write,
 * grouped by source rank ascending, then source row ascending) — read straight
 * from the receive buffer through the plan's map, never materialised (a
 * ROWBAND plan receives in the output layout into the library's buffer).
 *   plan: an FO_ALLTOALL plan with post = FO_POST_NONE;
 *   idx  device int32 [tokens, topk]: row of X for each (token, slot); a value
 *        < 0 or >= info.out_rows is a dropped slot (contributes nothing);
 *   w    device float [tokens, topk]: combine weights (e.g. the softmax over
 *        the token's top-k router logits);
 *   out  device bf16 [tokens, n]; residual device bf16 [tokens, n] or NULL.
 * Accumulation in fp32 in slot order, one bf16 rounding.
 * fo_run_combine = fo_run with the post pass replaced by the combine (runs
 * once after the last group's exchange: a token's slots arrive in different
 * groups); fo_combine_stage = the combine alone on a given receive buffer
 * (single-GPU stage access for multi-rank parity).  Errors:
 * FO_ERR_INVALID_ARG for a non-A2A plan, post != none, topk outside 1..64. */
fo_status fo_run_combine(fo_ctx ctx, fo_plan plan, const void* A, const void* Bt, void* out, const int32_t* idx,
                         const float* w, int32_t topk, int64_t tokens, const void* residual, void* stream);
fo_status fo_combine_stage(fo_plan plan, const void* recv, void* out, const int32_t* idx, const float* w,
                           int32_t topk, int64_t tokens, const void* residual, void* stream);

/* Overlapped GEMM + collective (+ post-reorder, + fused elementwise), stream
 * ordered on `stream` and host-asynchronous.  Collective: every rank calls it
 * with matching plans in the same order.  A plan must not run concurrently
 * with itself.
 *   A [m,k], Bt [n,k]: device bf16.
 *   out: device bf16 [info.out_rows, info.out_cols]:
 *     AR  -> [m, n] row-major, identical on every rank;
 *     RS  -> [m/world, n]: local row l = global row floor(l/h)*tile_m + rank*h + l%h (h = tile_m/world);
 *     A2A -> [sum_s cnt(s->rank), n]: rows grouped by source rank ascending, then source row ascending
 *       (may be NULL when no row is routed to this rank; A and Bt may be NULL when m == 0, R45);
 *     NOCOMM -> [m, n].
 *   residual (FO_POST_ADD*): device bf16, same shape as out; gamma (RMSNorm): device bf16 [n].
 * Internals: counters reset, GEMM on the caller stream, per group a
 * stream-side wait (counter >= |G_j|) then the NCCL call on the comm stream,
 * post-reorder (none for ROWBAND plans: the AR reduces `out` in place, the RS
 * and the A2A receives write `out` directly, so `out` is written by NCCL),
 * join back to `stream`; the last group's collective follows
 * the GEMM on `stream` itself (FO_OPT_LAST_GROUP_IN_ORDER, default), and a
 * single group then needs no counters, signals or fork at all (GEMM ->
 * collective).  Errors: FO_ERR_STATE when the plan's rank/world differ from
 * the context's; FO_ERR_CUDA / FO_ERR_NCCL wrap failed launches or calls. */
fo_status fo_run(fo_ctx ctx, fo_plan plan, const void* A, const void* Bt, void* out,
                 const void* residual, const void* gamma, void* stream);
/* fo_run with HOST buffers (same shapes as fo_run): stream-ordered
 * host->device copies of A, Bt (+ residual, gamma) into library-owned device
 * staging, the overlapped op, and the device->host copy of `out`, all on
 * `stream` (host-asynchronous when the host buffers are page-locked; the
 * caller synchronises the stream before reading `out`).  Any operand that is
 * already a device pointer (e.g. resident weights Bt) is used in place and
 * not copied.  This is the end-to-end entry point bench.py's `e2e` number is
 * measured through. */
fo_status fo_run_host(fo_ctx ctx, fo_plan plan, const void* A, const void* Bt, void* out,
                      const void* residual, const void* gamma, void* stream);
/* Non-overlapped baseline: the SAME GEMM kernel writing row-major C, then ONE
 * full-size NCCL call, then the fused elementwise op as its own pass:
 *   AR  -> ncclAllReduce in place on out [m, n] (same result as fo_run);
 *   RS  -> ncclReduceScatter of row-major C: out [m/world, n] holds the
 *          CONTIGUOUS global rows [rank*m/world, (rank+1)*m/world) (NCCL's
 *          standard layout; fo_run's block-cyclic R_k is the paper's,
 *          both are valid ReduceScatters of the same sum);
 *   A2A -> one grouped send/recv: every maximal run of consecutive rows with
 *          the same destination is one message (one per peer when row_dst is
 *          sorted, the usual MoE layout); out as fo_run's.
 * The calls are fo_plan_export_calls(plan, 1, ...). */
fo_status fo_run_sequential(fo_ctx ctx, fo_plan plan, const void* A, const void* Bt, void* out,
                            const void* residual, const void* gamma, void* stream);

/* RS follow-on (NEXT f2): AllGather of every rank's local RS
 * output `local` [m/world, n] (block-cyclic rows R_k, device bf16) into
 * `out` [m, n].  row_exchange != 0: the rank-major gather is permuted back to
 * the standard row order by a kernel that also applies the plan's elementwise
 * op (residual / gamma as in fo_run, now [m, n] / [n]); row_exchange == 0:
 * gathered rows stay rank-major ("if the row order has no impact on
 * subsequent processing, the exchange step can be safely eliminated").
 * Collective; `plan` must be the ReduceScatter plan that produced `local`. */
fo_status fo_run_allgather(fo_ctx ctx, fo_plan plan, const void* local, void* out, const void* residual,
                           const void* gamma, int32_t row_exchange, void* stream);

/* ---------------------------------------------------------------- stages (tests, single GPU, no NCCL) */
/* Run only the GEMM with this plan's pre-reorder epilogue into a caller
 * device buffer `send` of info.send_elems bf16 (the counting table is bumped
 * as in fo_run).  Lets one GPU exercise every rank's epilogue of a
 * multi-rank plan. */
fo_status fo_gemm_stage(fo_plan plan, const void* A, const void* Bt, void* send, void* stream);
/* As fo_gemm_stage, and also write %globaltimer (ns) into the device array
 * tile_ts[tiles] at the moment each execution position signals (wave
 * pattern evidence, the analogue of PAPER.md:230 fig:wave). */
fo_status fo_gemm_stage_timed(fo_plan plan, const void* A, const void* Bt, void* send,
                              unsigned long long* tile_ts, void* stream);
/* Run only wave group j's post-communication reorder (the per-group pass of
 * fo_run: slot / RS / A2A layouts, post none or add) from a caller device
 * receive buffer of info.recv_elems bf16; the rows of group j in `out` are
 * written.  FO_ERR_UNSUPPORTED for other layouts / ops. */
fo_status fo_group_post_stage(fo_plan plan, int32_t j, const void* recv, void* out, const void* residual,
                              void* stream);
/* Run only the post-communication reorder (+ fused op) from a caller device
 * receive buffer of info.recv_elems bf16. */
fo_status fo_post_stage(fo_plan plan, const void* recv, void* out, const void* residual,
                        const void* gamma, void* stream);
/* The row exchange alone, from a caller-provided rank-major gathered buffer
 * [m, n] (what ncclAllGather of the ranks' RS outputs delivers). */
fo_status fo_rowexchange_stage(fo_plan plan, const void* gathered, void* out, const void* residual,
                               const void* gamma, void* stream);
/* CTAs per thread-block cluster the plan's GEMM launches with on the current
 * device: 1 (128-row tiles), 2 (CTA pair, 256-row tiles) or 4 (two pairs with
 * TMA multicast, FO_OPT_MULTICAST).  Binds the plan to the device like a run. */
fo_status fo_plan_gemm_cluster(fo_plan plan, int32_t* cluster_ctas);
/* Debug watchdog (a hang from mismatched plans across ranks, a lost signal):
 * wait up to timeout_ms for everything enqueued on `stream` (fo_run joins
 * all of its streams into it) to finish.  FO_OK when it does.  Otherwise
 * every counter of the plan is forced past any target so the pending trigger
 * waits release, the context's NCCL communicator is aborted (ncclCommAbort:
 * NCCL kernels still stuck on absent peers exit), the streams drain, the
 * context refuses further runs (FO_ERR_STATE; destroy it and create a new
 * one; the run's output is undefined), and FO_ERR_TIMEOUT is returned.
 * Host-blocking; not graph-capturable. */
fo_status fo_plan_sync(fo_ctx ctx, fo_plan plan, void* stream, int64_t timeout_ms);
/* Bind the plan to the current device (and, ctx != NULL, to that context: its
 * buffer registration, as on a first fo_run) and allocate, now, the device state its
 * runs would otherwise allocate on first use: tables, counters, the send /
 * receive buffers (always), the row-major scratch of fo_run_sequential /
 * fo_run_allgather for RS / A2A plans (what & 1), and the staging buffers of
 * fo_run_host for a host A and a host out (what & 2).  After it no run of the
 * plan allocates (CUDA-graph capture; multi-rank issue where one rank's
 * allocation must not wait on another rank's in-flight collective).
 * Synchronises the device. */
fo_status fo_plan_prepare(fo_ctx ctx, fo_plan plan, int32_t what);
/* Copy the plan's P counters to host (synchronises the device). */
fo_status fo_plan_read_counters(fo_plan plan, uint32_t* counters);
/* Debug / evidence hooks (tests, tools; never needed for correct use):
 *  tile_ts  device uint64[tiles] or NULL: fo_run records %globaltimer (ns)
 *           when each execution position signals (PAPER.md:230 fig:wave);
 *  group_ts device uint64[2P] or NULL: fo_run records %globaltimer on the
 *           comm stream right after group j's wait is released (2j) and after
 *           its collective + per-group post-reorder (2j+1) — causality and
 *           overlap evidence;
 *  group_post -1 auto (default), 0 off, 1 on: run the post-communication
 *           reorder per group right after its collective (only for non-identity
 *           maps with op none/add; RMSNorm always runs once at the end). */
fo_status fo_plan_set_debug(fo_plan plan, unsigned long long* tile_ts, unsigned long long* group_ts,
                            int32_t group_post);
/* Plan options (run-time knobs; defaults shown):
 *  FO_OPT_GROUP_POST  -1 auto | 0 off | 1 on — as group_post above
 *  FO_OPT_WAIT_KERNEL  0 — trigger = cuStreamWaitValue32 (front-end wait, no SM)
 *                      1 — trigger = the paper's signaling kernel:
 *                          a 1-warp kernel spinning on an acquire load
 *  FO_OPT_TAIL_SPLIT   0 — off; f >= 2 — the R tiles of the last partial wave are
 *                      split into f K-slices run by otherwise idle workers of that
 *                      wave (needs R*f <= S); the slice-0 owner adds the fp32
 *                      partials in its epilogue and signals as usual; -1 — auto
 *                      (f = min(4, S/R, k-blocks) when 2R <= S and that is >= 2;
 *                      else no split); -2 — stream-K tail: the tail's R x k-blocks
 *                      dealt out evenly to the S workers in contiguous K-ranges
 *                      (measured slower than -1, R34); -3 — DP + suffix
 *                      helpers for a last wave of R > S/2 tiles (e.g. a one-wave
 *                      GEMM of 64 tiles on 74 pairs): each tail tile's own worker
 *                      runs k-blocks [0, x), the S-R idle workers run the suffixes
 *                      [x, KB) of consecutive tail tiles, x = KB - KB/(1 +
 *                      ceil(R/(S-R))) (R43; correct, measured slower than
 *                      the plain grid, profiles/r02_suffix_probe.txt).  Works with
 *                      every epilogue mode.  Set before the first run.
 *  FO_OPT_POST_SM_PARTITION 0 — per-group post kernels may co-reside with GEMM CTAs;
 *                      1 — they request padding shared memory so they only run on
 *                      the SMs the persistent GEMM leaves free (Alg. 1's SM split)
 *  FO_OPT_HOST_PIPELINE 7 — bit 0: fo_run_host copies a host A in ~8 chunks of
 *                      whole tile-rows on its own stream, each chunk released to
 *                      the GEMM by a stream write the TMA producer waits on (the
 *                      GEMM starts on the first chunk); bit 1: (AR / RS ROWBAND)
 *                      each group's output rows are copied to the host right after its
 *                      collective; bit 2 (with bit 0): two device staging sets
 *                      used by alternate calls, so a call's H2D overlaps the
 *                      previous call's GEMM, collectives and D2H; 0 — whole-
 *                      buffer copies before / after
 *  FO_OPT_HOST_CHUNKS  8 — target number of A chunks (whole tile-rows each) for
 *                      bit 0 above; set before the plan's first fo_run_host
 *  FO_OPT_LAST_GROUP_IN_ORDER 1 — the last group's collective (and its post
 *                      pass) is issued on the caller stream right after the GEMM:
 *                      the kernel boundary orders every tile's stores before it,
 *                      so the last group needs no counter wait and its
 *                      wait-release latency leaves the critical path (the
 *                      caller stream first waits for the comm stream's earlier
 *                      collectives: same call order on the communicator);
 *                      0 — every group triggered by its counter on the comm
 *                      stream (PAPER.md:368 applied to all groups)
 *  FO_OPT_WAVE_SYNC    0 — free-running persistent workers (default);
 *                      1 — the persistent GEMM keeps its waves aligned (the
 *                      hardware-scheduled waves of PAPER.md:235): a worker issues
 *                      no load of its wave-(w+1) tile before every worker has
 *                      issued the last load of its wave-w tile, so workers never
 *                      drift into different operand panels and one wave's panels
 *                      are read from HBM once (L2 reuse; less HBM power, higher
 *                      clocks under the power cap); a scheduling constraint only,
 *                      results are identical; ignored with a tail split.
 *                      Measured: halves HBM reads of long-K many-wave GEMMs
 *                      under ncu, no wall-clock change in interleaved timing
 *                      (profiles/r01_wave_sync.txt), hence off by default
 *  FO_OPT_MULTICAST    0 — independent CTA pairs (default);
 *                      1 — 256-row (CTA-pair) tiles with K-major operands, an even
 *                      S and no tail split run as clusters of two pairs when all
 *                      S/2 clusters fit on the device: the pairs run consecutive
 *                      execution positions in lockstep and a shared A tile-row
 *                      or B tile-column is loaded once per cluster and
 *                      TMA-multicast to both pairs (17% fewer L2 sectors);
 *                      results are identical.  Measured 12-20% slower: the
 *                      shared stage-release barriers couple the two pairs'
 *                      pipelines (profiles/r01_multicast.txt), hence off
 *  FO_OPT_DEBUG_STALL_GROUP -1 — off; j — TEST ONLY: group j's trigger waits for
 *                      one more signal than the GEMM sends, so the run never
 *                      finishes (exercises the fo_plan_sync watchdog)
 *  FO_OPT_GEMM_SWIGLU  0 — off; 1 — (no-comm plans, tile_n 256, post none)
 *                      the GEMM's epilogue applies the SwiGLU of an MLP: with the
 *                      weight rows interleaved in blocks of 128 (gate 0..127, up
 *                      0..127, gate 128..255, up 128..255, ...), tile column block
 *                      j writes C[:, 128j .. 128j+128) = silu(gate) * up from the
 *                      fp32 accumulators (one bf16 rounding); C is [m, n/2]
 *  FO_OPT_DIST_FOLD    1 (default) — with an f-slice tail split, the K-slices of a
 *                      split tile reduce it together: 64-column chunk c is summed
 *                      and stored by slice c % f, each slice publishing the fp32
 *                      partials of the chunks it does not own; 0 — the slice
 *                      starting at k-block 0 folds every chunk (the SwiGLU
 *                      epilogue and the stream-K tail always fold this way).
 *                      Slices wait on each other, which is safe because every
 *                      slice is its worker's last unit and all workers are
 *                      co-resident (workers x CTAs <= SMs is enforced)
 *  FO_OPT_K_SNAKE      -1 (default) — auto: 1 when K >= 64 k-blocks (4096), else 0;
 *                      0 — every tile runs its k-blocks first to last; 1 — a
 *                      worker's odd units (its odd waves) run them last to first,
 *                      so a wave starts on the k-slices of the operand panels the
 *                      previous wave read last, which are still in L2 (fewer
 *                      HBM re-reads of the panels consecutive waves share); the
 *                      fp32 accumulation order of those tiles is reversed.
 *                      Measured (profiles/r02_ksnake.txt): 4096^2 x 14336, S=74 +
 *                      split tail: HBM reads 598 -> 526 MB, 292.9 -> 288.9 us
 *  FO_OPT_TMA_STORE    1 (default) — whole tiles written to row-major C or to AR
 *                      slots leave the epilogue as TMA stores (one 64-column box
 *                      per warp from the 128B-swizzled staging buffer); with
 *                      counters the signalling warp waits for the stores'
 *                      completion (cp.async.bulk.wait_group 0 + async-proxy
 *                      fence) before its release add; 0 — 16-byte st.global from
 *                      the staging buffer (always used for the RS slot and A2A
 *                      layouts, RS bands with h < 32 and split-tail tiles; RS
 *                      ROWBAND with h >= 32 uses TMA stores too)
 *  FO_OPT_POST_BULK    1 (default) — an add + RMSNorm pass ordered after the GEMM
 *                      (the whole-output pass, fo_run_sequential's, the stage
 *                      entry points', the last band's) stages its rows in shared
 *                      memory by bulk copies, 2-4 rows per block in flight; 0 —
 *                      the register kernel (always used beside the GEMM); both
 *                      give the same bits */
typedef enum { FO_OPT_GROUP_POST = 0, FO_OPT_WAIT_KERNEL = 1, FO_OPT_TAIL_SPLIT = 2,
               FO_OPT_POST_SM_PARTITION = 3, FO_OPT_HOST_PIPELINE = 4, FO_OPT_HOST_CHUNKS = 5,
               FO_OPT_LAST_GROUP_IN_ORDER = 6, FO_OPT_WAVE_SYNC = 7, FO_OPT_MULTICAST = 8,
               FO_OPT_DEBUG_STALL_GROUP = 10, FO_OPT_GEMM_SWIGLU = 11,
               FO_OPT_DIST_FOLD = 12, FO_OPT_K_SNAKE = 13, FO_OPT_TMA_STORE = 14,
               FO_OPT_POST_BULK = 15 } fo_option;
fo_status fo_plan_set_option(fo_plan plan, int32_t option, int64_t value);
/* Fill the library-owned send/receive buffers of the plan with a bf16 bit
 * pattern on `stream` (poison for the memory-ordering stress test). */
fo_status fo_plan_fill_buffers(fo_plan plan, uint16_t pattern, void* stream);
/* Number of kernels the library launched since load (for gpu_launches). */
int64_t fo_kernel_launch_count(void);

/* ---------------------------------------------------------------- tuner (Alg. 1, host only) */
/* Predicted latency (us) of partition `groups[0..P)`:
 *   duration_us  GEMM duration at wave width S; T = ceil(tiles/S)
 *   tile_bytes   message bytes per tile (tile_m*tile_n*2)
 *   curve        npts samples (bytes, GB/s), bytes strictly increasing;
 *                linear interpolation in log2(bytes), clamped (R15). */
fo_status fo_tune_predict(const int32_t* groups, int32_t P, double duration_us, int32_t tiles,
                          int32_t S, double tile_bytes, const double* curve_bytes,
                          const double* curve_gbps, int32_t npts, double* predicted_us);
/* Alg. 1 search.  prune: 0 = enumerate all 2^(T-1)
 * partitions, 1 = enumerate those with |G_1| <= s1 and |G_P| <= sp
 * (PAPER.md:446); ties -> fewer groups, then lexicographically smaller
 * (R16).  2 / 3 = exact argmin of the same predictor by an O(T^2)
 * dynamic program (R24) without / with the caps; used automatically
 * (with the caps iff prune == 1) when T > 20, where enumeration is
 * infeasible.  out_groups must hold T entries. */
fo_status fo_tune_search(double duration_us, int32_t tiles, int32_t S, double tile_bytes,
                         const double* curve_bytes, const double* curve_gbps, int32_t npts,
                         int32_t s1, int32_t sp, int32_t prune, int32_t* out_groups,
                         int32_t* out_num_groups, double* predicted_us);

/* A2A imbalance extension of Alg. 1 (NEXT f3; R26):
 * `ranks` GPUs share one partition of T waves; durations[r] is rank r's GEMM
 * duration, wave_bytes[r*T + w] the A2A bytes rank r sends in wave w.  The
 * accumulated latencies are maxed across GPUs after every step. */
fo_status fo_tune_predict_multi(const int32_t* groups, int32_t P, int32_t ranks, int32_t T,
                                const double* durations, const double* wave_bytes,
                                const double* curve_bytes, const double* curve_gbps, int32_t npts,
                                double* predicted_us);
fo_status fo_tune_search_multi(int32_t ranks, int32_t T, const double* durations, const double* wave_bytes,
                               const double* curve_bytes, const double* curve_gbps, int32_t npts,
                               int32_t s1, int32_t sp, int32_t prune, int32_t* out_groups,
                               int32_t* out_num_groups, double* predicted_us);

#ifdef __cplusplus
}
#endif
#endif /* FLASHOVERLAP_H_ */
