// Launch interface of the sm_100a kernels (host <-> device structs).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace fo {

// Epilogue store mode = the pre-communication reordering.
enum EpiMode : int {
  EPI_ROWMAJOR = 0,  // C row-major with row stride ldc (no-comm, AR ROWBAND)
  EPI_SLOT = 1,      // AR: tile at position p -> slot p (BM*BN contiguous, row-major)
  EPI_RS = 2,        // RS: subtile k of the tile -> chunk k of its group
  EPI_A2A = 3,       // A2A: row a of the tile -> its destination pool slot
  EPI_SWIGLU = 4,    // no-comm, BN = 256: tile columns [0,128) gate, [128,256) up (interleaved
                     // weight rows); writes silu(gate) * up to C[:, tj*128 .. +128), row stride ldc
  EPI_RS_BAND = 5    // RS ROWBAND (R40): row a of tile-row i (band [r0, r0+B)) -> row
                     // r0*BM + ((a/h)*B + i - r0)*h + a%h of a row-major [M, ldc] buffer
};

// One K-range of a split tail tile (host-built table, see fo_gemm's my_unit):
// role 1 = owner (the range starting at k-block 0; folds nparts-1 partials
// from workspace slots slot.. in), role 2 = part (publishes to slot `slot`).
struct GemmSeg {
  int pos, kb0, kb1, role, slot, nparts, tt;
  int idx;  // participant index of the tile in k order (0 = owner)
};

struct GemmArgs {
  const void* A;      // [M, K] bf16 row-major (K-major) or [K, M] (mn_major bit 0)
  const void* Bt;     // [N, K] bf16 row-major (K-major) or [K, N] (mn_major bit 1)
  int mn_major;       // bit 0: A is M-major, bit 1: Bt is N-major
  void* dst;          // bf16 destination (C or the send buffer)
  int64_t M, N, K;
  int BM, BN;
  int Mt, Nt, tiles;
  int workers;        // grid size S
  int mode;           // EpiMode
  int64_t ldc;        // EPI_ROWMAJOR row stride
  const int32_t* order;        // [tiles] device
  const int32_t* group_of_pos; // [tiles] device
  const int32_t* gpos;         // [P+1] device
  const int32_t* row_slot;     // [tiles*BM] device (A2A)
  const int2* rs_info;         // [tiles] device (RS): {first position, size} of the position's group
                               // (EPI_RS_BAND: {first tile-row, tile-rows} of its band)
  uint32_t* counters;          // [P] device, may be null
  int h;                       // RS subtile rows (tile_m / world, a power of two)
  int h_log2;
  unsigned long long* tile_ts; // optional [tiles] device: %globaltimer at signal
  // ---- tail split (split-K of the last partial wave across idle workers)
  int tail_pos;                // first execution position of the split tail (= tiles: no split)
  int split;                   // > 1: the tail is split (segments below); 1: no split
  const GemmSeg* seg;          // [segments] the tail's K-ranges, grouped by worker
  const int32_t* wseg;         // [S + 1] worker w's segments: seg[wseg[w] .. wseg[w+1])
  float* workspace;            // fp32 partials [slots][TM][BN]
  uint32_t* flags;             // [(tiles - tail_pos) * CG] partial-ready counts (reset with the counters)
  // distributed fold (f-slice split, every participant's last unit): 64-column
  // chunk c of a split tile is reduced and stored by participant c % nparts;
  // each participant publishes the chunks it does not own (the owner into
  // slot + nparts - 1), and the last one to store signals the tile (`done`)
  int dist_fold;
  uint32_t* done;              // [(tiles - tail_pos) * CG] participants finished (reset with the counters)
  // ---- host-staged A (fo_run_host pipelining): A arrives in chunks of
  // a_chunk_rows tile-rows; the producer loads a tile's A only once
  // a_ready[ti / a_chunk_rows] has reached a_epoch (null: A is resident)
  const uint32_t* a_ready;
  uint32_t a_epoch;
  int a_chunk_rows;
  // ---- wave alignment (FO_OPT_WAVE_SYNC): each CTA's producer adds 1 to
  // wave_ctr[w] after issuing its wave-w tile's last load and issues no load
  // of wave w+1 before wave w's count reached its target for this launch;
  // counters only grow (launch `wave_epoch` of this plan expects
  // (wave_epoch+1) * CG * |wave w| ), null = off
  uint32_t* wave_ctr;
  uint32_t wave_epoch;
  // ---- TMA multicast across clusters of two CTA pairs (FO_OPT_MULTICAST)
  int multicast;
  // ---- FO_OPT_K_SNAKE: a worker's odd units run their k-blocks last to first,
  // so a wave starts on the k-slices of the operand panels the previous wave
  // read last (still in L2)
  int k_snake;
  // ---- epilogue stores: tma_store_ok (runtime: FO_OPT_TMA_STORE) lets the
  // launcher use TMA stores for whole tiles in EPI_ROWMAJOR / EPI_SLOT;
  // tma_store is set by the launcher when it built the destination map
  int tma_store_ok;
  int tma_store;
};

enum PostMode : int {
  POSTMAP_IDENTITY = 0,
  POSTMAP_SLOT = 1,
  POSTMAP_RS = 2,
  POSTMAP_A2A = 3,
  POSTMAP_ROWX = 4  // RS follow-on: rank-major AllGather of block-cyclic rows -> standard row order
};

struct PostArgs {
  int map;                 // PostMode
  int op;                  // fo_post
  const void* src;         // receive buffer (bf16)
  void* out;               // [rows, N] bf16
  const void* residual;    // [rows, N] bf16 or null
  const void* gamma;       // [N] bf16 or null
  int64_t rows, N;
  int BM, BN, Nt, h;
  const int32_t* pos_of_tile;  // device
  const int32_t* src_row;      // device (A2A)
  float eps;
  int smem_pad;                // dynamic smem (bytes, unused) requested per block: > the SM's
                               // smem left beside a live GEMM CTA keeps the kernel off the GEMM's SMs
  int bulk_ok;                 // add + RMSNorm may stage rows in smem by bulk copies (launches that do
                               // not run beside the persistent GEMM)
};

// Post-reorder of ONE wave group's data right after its collective (DESIGN.md
// H11b): AR-slot / RS move whole per-position blocks of R rows x BN
// (R = BM for AR, h for RS) from src + p*R*BN to out tile (i, jc); A2A moves
// the group's received subtokens [sub_begin, sub_end) through recv_dst.
struct GroupPostArgs {
  int map;                 // POSTMAP_SLOT / POSTMAP_RS / POSTMAP_A2A
  int op;                  // FO_POST_NONE or FO_POST_ADD
  const void* src;
  void* out;
  const void* residual;
  int64_t N;
  int BN, Nt, R;
  int pos_begin, pos_end;          // positions of the group (SLOT / RS)
  const int32_t* order;            // device
  int64_t sub_begin, sub_end;      // received subtokens of the group (A2A)
  const int32_t* recv_dst;         // device
  int grid_cap;                    // max blocks (0 = default)
  int smem_pad;                    // as PostArgs::smem_pad
};

// Returns a cudaError_t-compatible code (0 = success).
// MoE top-k combine fused into the A2A post-reorder (R31):
// out[t] = sum_i w[t*k+i] * a2a_out[idx[t*k+i]] (+ residual[t]), where row r of
// the standard A2A output is read straight from the receive buffer through
// src_row (no intermediate [rows, N] buffer); fp32 accumulation, one bf16 rounding.
struct CombineArgs {
  const void* src;           // receive buffer (bf16 subtokens)
  void* out;                 // [tokens, N] bf16
  const void* residual;      // [tokens, N] bf16 or null
  const int32_t* idx;        // [tokens, topk] device; < 0 or >= a2a_rows: dropped slot
  const float* w;            // [tokens, topk] device
  int topk;
  int64_t tokens, N, a2a_rows;
  int BN, Nt;
  const int32_t* src_row;    // [a2a_rows, Nt] device (plan)
};

cudaError_t launch_gemm(const GemmArgs& a, cudaStream_t stream);
cudaError_t launch_combine(const CombineArgs& a, cudaStream_t stream);
cudaError_t launch_post(const PostArgs& a, cudaStream_t stream);
cudaError_t launch_group_post(const GroupPostArgs& a, cudaStream_t stream);
cudaError_t launch_timestamp(unsigned long long* dst, cudaStream_t stream);
cudaError_t launch_wait(const uint32_t* counter, uint32_t target, cudaStream_t stream);
cudaError_t launch_fill_u16(void* dst, int64_t count, uint16_t value, cudaStream_t stream);
bool gemm_shape_supported(int BM, int BN);
bool gemm_multicast_used(const GemmArgs& a);  // the launch would use clusters of two pairs
void count_launch();
int64_t launch_count();

}  // namespace fo
