// Host-side plan: the integer math of the method for one rank (no CUDA).
//
// Tile grid, execution order / block swizzle (PAPER.md:237-238,
// 378), waves and wave groups,
// and the pre/post-communication index maps for AllReduce, ReduceScatter and
// All-to-All.  Readings R1-R9 of DESIGN.md apply.
#pragma once

#include <cstdint>
#include <vector>

#include "common.h"

namespace fo {

struct PlanHost {
  // ---- descriptor (copied)
  int coll = FO_NOCOMM;
  int layout = FO_LAYOUT_SLOT;  // resolved AR / RS layout
  int64_t M = 0, N = 0, K = 0;
  int BM = 128, BN = 128;
  int S = 0;                    // wave width (0 until resolved against a device)
  int post = FO_POST_NONE;
  float eps = 1e-5f;
  int rank = 0, world = 1;
  int mn_major = 0;             // bit 0: A M-major, bit 1: Bt N-major

  // ---- O1-O3
  int Mt = 0, Nt = 0, tiles = 0, T = 0, P = 0;
  std::vector<int32_t> order;        // [tiles] tile id at position p
  std::vector<int32_t> pos_of_tile;  // [tiles] inverse
  std::vector<int32_t> group_waves;  // [P]
  std::vector<int32_t> gpos;         // [P+1] position boundaries
  std::vector<int32_t> group_of_pos; // [tiles]
  int h = 0;                         // RS subtile rows

  // ---- A2A
  std::vector<int32_t> row_dst;          // [M]
  std::vector<int64_t> pool_base;        // [world+1] subtoken offset of pool d in the send buffer
  std::vector<int64_t> send_cnt;         // [P*world] subtokens of group j to peer d
  std::vector<int64_t> send_start;       // [P*world] start (within pool d) of group j
  std::vector<int32_t> row_slot;         // [tiles*BM] send-buffer subtoken index of (position p, row a); -1 never
  std::vector<int64_t> recv_cnt;         // [P*world] subtokens of group j from source s
  std::vector<int64_t> recv_off;         // [P*world] receive-buffer subtoken offset, layout [group][source]
  std::vector<int32_t> src_row;          // [out_rows*Nt] receive-buffer subtoken index for out row r, col block j
  std::vector<int32_t> recv_dst;         // [recv subtokens] out_row*Nt + col block of each received subtoken
  std::vector<int64_t> src_base;         // [world+1] first output row of each source

  int64_t out_rows = 0;
  int64_t send_elems = 0, recv_elems = 0;

  std::vector<int64_t> band_rows;       // AR / RS ROWBAND: [2P] tile-row band (r0, r1) of each group

  // ---- communication schedules (fo_plan_export_calls): what fo_run /
  // fo_run_sequential issue on the communicator, in order
  std::vector<fo_comm_call> calls;      // overlapped, grouped by wave group
  std::vector<int32_t> call_begin;      // [P+1] calls of group j = [call_begin[j], call_begin[j+1])
  std::vector<fo_comm_call> seq_calls;  // sequential baseline

  // AllReduce / ReduceScatter with every group a band of whole tile-rows
  // (H11a, R40): no post-communication reorder.
  bool banded() const { return (coll == FO_ALLREDUCE || coll == FO_REDUCESCATTER) && layout == FO_LAYOUT_ROWBAND; }
  // Output rows per tile-row of a banded plan (AR: BM; RS: the h rows of each
  // tile-row that land on this rank).
  int band_out_rows() const { return coll == FO_REDUCESCATTER ? h : BM; }

  // Group j's element range in the AR/RS send buffer (ROWBAND: its row band of C).
  int64_t group_elem_begin(int j) const {
    if (banded()) return band_rows[2 * j] * BM * N;
    return (int64_t)gpos[j] * BM * BN;
  }
  int64_t group_elem_end(int j) const {
    if (banded()) return band_rows[2 * j + 1] * BM * N;
    return (int64_t)gpos[j + 1] * BM * BN;
  }
  int group_tiles(int j) const { return gpos[j + 1] - gpos[j]; }

  int64_t send_index(int64_t r, int64_t c) const;  // C[r][c] -> send buffer
  int64_t recv_index(int64_t r, int64_t c) const;  // out[r][c] <- receive buffer
};

// Default order of DESIGN.md R1: row-panels of s tile-rows, column-major inside.
std::vector<int32_t> default_order(int Mt, int Nt, int s);
// swizzle == -1 (R44): a generalized Hilbert curve over the tile grid.
std::vector<int32_t> hilbert_order(int Mt, int Nt);
// swizzle == 0: the panel height minimising the tile-rows + tile-columns one
// wave of S touches (the operand panels that must be L2-resident together).
int auto_swizzle(int Mt, int Nt, int S);

// Validate + build.  `sm_count` resolves workers == 0 (pass 0 if unknown: then
// workers must be given explicitly).
PlanHost build_plan(const fo_plan_desc& self, int rank, int world,
                    const fo_plan_desc* const* peers, int sm_count);

// The overlapped and sequential communication schedules of a built plan
// (peers: the A2A census descriptors, as for build_plan).
void build_schedules(PlanHost& p, const fo_plan_desc& self, const fo_plan_desc* const* peers);

}  // namespace fo
