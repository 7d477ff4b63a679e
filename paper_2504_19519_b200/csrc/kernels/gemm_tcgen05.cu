// Persistent warp-specialised tcgen05 bf16 GEMM for sm_100a whose epilogue
// performs FlashOverlap's pre-communication reordering and group signaling.
//
//   C[M,N] = A[M,K] · Bt[N,K]^T,   bf16 in, fp32 accumulate (TMEM), bf16 out.
//
// Method: the main loop is an unmodified GEMM (PAPER.md:241-242,
// 394 "involving only the epilogue without interrupting the main loop"); the
// epilogue stores each finished tile straight into the reordered send buffer
// and then atomically adds 1 to the counter of the tile's
// wave group ("The j-th number in the counting table is
// atomically added by 1 when a tile in G_j is finished").
//
// B200 design:
//  - grid = S persistent CTAs (S = wave width); CTA w runs execution positions
//    w, w+S, w+2S, ...  so position p is in wave floor(p/S) by construction.
//  - warp 0: TMA producer (128B-swizzled K-major boxes, mbarrier ring of ST
//    stages); warp 1: single-thread tcgen05.mma issuer (M=128, N=BN, K=16)
//    accumulating in TMEM; warp 2: TMEM allocator; warps 4-7: epilogue.
//  - two TMEM accumulator stages so the epilogue of tile i overlaps the main
//    loop of tile i+1.
//  - epilogue: tcgen05.ld (32 lanes x 32 cols) -> bf16 RNE -> per-warp smem
//    staging -> coalesced 16-byte stores to the mode's destination rows; a
//    named barrier over the 4 epilogue warps, then ONE red.release.gpu add on
//    the group counter (release orders all the tile's stores before it).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>

#include "../kernels.h"

namespace fo {
namespace {

constexpr int BM = 128;                     // rows per CTA (a CTA pair covers 256)
constexpr int BK = 64;                      // 64 bf16 = 128 B = one swizzle row
constexpr int EPI_COLS = 64;                // columns staged per epilogue chunk
// Epilogue staging: per warp 32 rows x 128 B (one 64-column bf16 chunk), the
// 16-byte chunks of row r at position x ^ (r & 7) — the TMA 128-byte swizzle,
// so the buffer is both a bank-conflict-free transpose stage for the 16-byte
// st.global path and the source box of a SWIZZLE_128B TMA store.
constexpr int EPI_ROW = EPI_COLS * 2;
constexpr int EPI_WARP_BYTES = 32 * EPI_ROW;
constexpr int EPI_BYTES = 4 * EPI_WARP_BYTES;
constexpr int NUM_THREADS = 256;

// CG = CTA group size: 1 -> tile 128 x BN on one SM; 2 -> tile 256 x BN on a
// CTA pair (tcgen05 cta_group::2): each CTA stages its 128 rows of A and
// BN/2 rows of B, the leader issues M=256 MMAs, each CTA's TMEM holds its
// 128 accumulator rows.
// RB = accumulator rows per CTA: 128, or 64 (cta_group::1 only: tcgen05.mma
// M=64, whose D rows 16q..16q+15 sit in TMEM lanes 32q..32q+15 — the
// "half subpartition" layout — so each epilogue warp owns 16 rows).
template <int BN, int CG, int RB = 128>
struct Cfg {
  static constexpr int A_STAGE = RB * BK * 2;            // A rows staged per CTA
  static constexpr int B_ROWS = BN / CG;                 // B rows staged per CTA
  static constexpr int B_STAGE_BYTES = B_ROWS * BK * 2;
  static constexpr int STAGE_BYTES = A_STAGE + B_STAGE_BYTES;
  static constexpr int BUDGET = 232448 - 1024 - EPI_BYTES - 256;
  static constexpr int STAGES = (BUDGET / STAGE_BYTES) > 8 ? 8 : (BUDGET / STAGE_BYTES);
  static constexpr int TMEM_COLS = 2 * BN;  // two fp32 accumulator stages
  static constexpr int BAR_BYTES = 8 * (2 * STAGES + 6) + 16;
  static constexpr int SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + EPI_BYTES + BAR_BYTES;
  static_assert(SMEM_BYTES <= 232448, "shared memory budget");
  static_assert(TMEM_COLS == 128 || TMEM_COLS == 256 || TMEM_COLS == 512, "TMEM alloc power of 2");
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
  } while (!ok);
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// setup barrier of a cluster: what other CTAs need from this one before
// their first remote operation is its mbarrier initialisation, already
// released to the cluster by fence.mbarrier_init; the TMEM address slot is
// CTA-local (bar.sync orders it).  So the cluster arrive can be relaxed.
__device__ __forceinline__ void cluster_setup_sync() {
  __syncthreads();
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// shared::cluster address of the same object in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_shared(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}

// arrive on a barrier of another CTA of the cluster.  Default semantics
// (.release.cta): the only data ordered by it are TMEM reads, already ordered
// by tcgen05.wait::ld + tcgen05.fence::before_thread_sync; .release.cluster
// would add a MEMBAR.GPU that waits for the warp's outstanding global stores.
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

// one lane of a converged warp (elect.sync)
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// 2-SM TMA: data lands in this CTA's smem, the transaction bytes are counted
// on the leader CTA's mbarrier (cluster address).
__device__ __forceinline__ void tma_load_2d_2sm(void* dst, const CUtensorMap* map, int x, int y, uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(x), "r"(y)
      : "memory");
}

// 2-SM TMA multicast (cluster of CTA pairs): the box lands at the same smem
// offset in every CTA of `mask`; each destination's transaction bytes are
// counted on the barrier at this offset in the destination's pair leader
// (peer bit of the barrier address cleared, the CUTLASS SM100 2-SM form).
__device__ __forceinline__ void tma_load_2d_2sm_mc(void* dst, const CUtensorMap* map, int x, int y, const void* bar,
                                                   uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%4, %5}], [%2], %3;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & 0xFEFFFFFFu), "h"(mask), "r"(x), "r"(y)
      : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// UMMA shared-memory descriptor: K-major, 128-byte swizzle, 8-row core groups
// 1024 B apart (SBO), LBO unused for swizzled K-major (=1), version 1 (sm_100).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// UMMA descriptor for an MN-major operand staged as 64x64 TMA boxes (64
// MN-elements = one 128-byte swizzled row per k): 8-k-row core groups are
// 1024 B apart (SBO), consecutive 64-element MN chunks (boxes) 8192 B apart
// (LBO); a K=16 step advances 2 core groups = 2048 B.
__device__ __forceinline__ uint64_t sw128_mn_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)(8192 >> 4) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// Instruction descriptor, kind::f16: D fp32, A/B bf16, N>>3, M>>4; MJ bit 0 /
// bit 1 = A / B is MN-major (else K-major).
template <int M, int N, int MJ>
__device__ __forceinline__ constexpr uint32_t idesc_bf16() {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(MJ & 1) << 15) | ((uint32_t)((MJ >> 1) & 1) << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// The four K=16 MMAs of one 64-wide k-block from ONE elected lane of a
// converged warp: descriptors step by da / db (16-byte units) per MMA; the
// first accumulates into D unless `acc` is 0.  One elect and one operand
// transfer to uniform registers per k-block instead of per MMA.
template <int CG>
__device__ __forceinline__ void umma_kblock(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t da, uint32_t db,
                                            uint32_t idesc, uint32_t acc) {
  static_assert(BK == 64, "four K=16 steps per k-block");
#define FO_UMMA_CG(cg)                                                                          \
  asm volatile(                                                                                 \
      "{\n\t.reg .pred e, p, t;\n\t.reg .b64 a1, a2, a3, b1, b2, b3, sa, sb;\n\t"         \
      "elect.sync _|e, 0xffffffff;\n\t"                                                       \
      "setp.ne.b32 p, %4, 0;\n\t"                                                             \
      "setp.eq.u32 t, 0, 0;\n\t"                                                              \
      "cvt.u64.u32 sa, %5;\n\t"                                                               \
      "cvt.u64.u32 sb, %6;\n\t"                                                               \
      "add.s64 a1, %1, sa;\n\tadd.s64 a2, a1, sa;\n\tadd.s64 a3, a2, sa;\n\t"             \
      "add.s64 b1, %2, sb;\n\tadd.s64 b2, b1, sb;\n\tadd.s64 b3, b2, sb;\n\t"             \
      "@e tcgen05.mma.cta_group::" #cg ".kind::f16 [%0], %1, %2, %3, p;\n\t"                  \
      "@e tcgen05.mma.cta_group::" #cg ".kind::f16 [%0], a1, b1, %3, t;\n\t"                  \
      "@e tcgen05.mma.cta_group::" #cg ".kind::f16 [%0], a2, b2, %3, t;\n\t"                  \
      "@e tcgen05.mma.cta_group::" #cg ".kind::f16 [%0], a3, b3, %3, t;\n\t}" ::"r"(d_tmem),  \
      "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(da), "r"(db))
  if constexpr (CG == 1) {
    FO_UMMA_CG(1);
  } else {
    FO_UMMA_CG(2);
  }
#undef FO_UMMA_CG
}

// MMA completion -> mbarrier arrive; for a pair, multicast to the barrier at
// the same offset in the CTAs of `mask` (the pair itself, or every CTA of a
// cluster of pairs whose smem stages the pair's loads also fill).
template <int CG>
__device__ __forceinline__ void umma_commit(uint64_t* bar, uint16_t mask = 0x3) {
  if constexpr (CG == 1) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
  } else {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
  }
}

#define FO_R8(i) "=r"(v[i]), "=r"(v[i + 1]), "=r"(v[i + 2]), "=r"(v[i + 3]), "=r"(v[i + 4]), "=r"(v[i + 5]), "=r"(v[i + 6]), "=r"(v[i + 7])
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : FO_R8(0), FO_R8(8), FO_R8(16), FO_R8(24)
      : "r"(taddr));
}
#undef FO_R8

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ uint32_t pack_bf16(uint32_t lo, uint32_t hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(lo), __uint_as_float(hi));
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ void red_release_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// staging addresses (swizzled, see EPI_ROW)
__device__ __forceinline__ uint4* stg_at(uint8_t* stg, int r, int x) {
  return reinterpret_cast<uint4*>(stg + r * EPI_ROW + ((x ^ (r & 7)) << 4));
}

// TMA store of a 64-column x `rows`-row box from swizzled shared memory
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(x), "r"(y)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint32_t atom_add_acq_rel(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// The work of one worker: its k-th unit.  Units of the first tail_pos
// positions are whole tiles (worker w runs positions w, w+S, ...); with a
// split tail the worker then runs its segments of the tail tiles, listed by
// the host in p.seg[p.wseg[w] .. p.wseg[w+1]) — a K-range of one tail tile
// and its role: 0 whole tile, 1 owner (the K-range starting at k-block 0:
// folds the other parts' fp32 partials in, writes and signals the tile),
// 2 part (publishes its fp32 partial to workspace slot `slot`).
struct Unit {
  int pos, kb0, kb1, role, slot, nparts, tt, idx;
};

__device__ __forceinline__ int unit_count(const GemmArgs& p, int worker, int nworkers) {
  const int nreg = (p.tail_pos > worker) ? (p.tail_pos - worker + nworkers - 1) / nworkers : 0;
  return nreg + (p.seg ? p.wseg[worker + 1] - p.wseg[worker] : 0);
}

__device__ __forceinline__ Unit my_unit(const GemmArgs& p, int worker, int nworkers, int k, int KB) {
  const int nreg = (p.tail_pos > worker) ? (p.tail_pos - worker + nworkers - 1) / nworkers : 0;
  Unit r;
  if (k < nreg) {
    r.pos = worker + k * nworkers;
    r.kb0 = 0;
    r.kb1 = KB;
    r.role = 0;
    r.slot = 0;
    r.nparts = 1;
    r.tt = 0;
    r.idx = 0;
  } else {
    const GemmSeg sg = p.seg[p.wseg[worker] + (k - nreg)];
    r.pos = sg.pos;
    r.kb0 = sg.kb0;
    r.kb1 = sg.kb1;
    r.role = sg.role;
    r.slot = sg.slot;
    r.nparts = sg.nparts;
    r.tt = sg.tt;
    r.idx = sg.idx;
  }
  return r;
}

// RS ROWBAND (R40): buffer row of row `a` of tile-row `ti` in the
// band of tile-rows [r0, r0 + B): subtile k = a / h goes to chunk k of the band
// (rows [r0*TM + k*B*h, +B*h)), tile-row by tile-row.
template <int TM>
__device__ __forceinline__ int64_t rs_band_row(const GemmArgs& p, int ti, int a, int r0, int B) {
  const int k = a >> p.h_log2, a2 = a & (p.h - 1);
  return (int64_t)r0 * TM + ((int64_t)(k * B + (ti - r0)) << p.h_log2) + a2;
}

// Destination of row `a` (0..TM-1) of the TM x BN tile at position `pos` =
// (ti, tj); `rs_ps` / `rs_G` = first position and size of the tile's group
// (RS) and `a2a_slot` = row_slot[pos*TM + a] (A2A), loaded by the caller one
// tile ahead.
template <int TM, int BN>
__device__ __forceinline__ __nv_bfloat16* row_dst(const GemmArgs& p, int pos, int ti, int tj, int a, int rs_ps,
                                                  int rs_G, int a2a_slot) {
  __nv_bfloat16* base = reinterpret_cast<__nv_bfloat16*>(p.dst);
  switch (p.mode) {
    case EPI_ROWMAJOR:
      return base + ((int64_t)ti * TM + a) * p.ldc + (int64_t)tj * BN;
    case EPI_SLOT:  // slot pos, row-major
      return base + ((int64_t)pos * TM + a) * BN;
    case EPI_RS: {  // subtile k = a / h goes to chunk k of the group (h = 2^h_log2)
      const int k = a >> p.h_log2, a2 = a & (p.h - 1);
      return base + ((int64_t)rs_ps * TM + (((k * rs_G + (pos - rs_ps)) << p.h_log2) + a2)) * BN;
    }
    case EPI_RS_BAND:  // DESIGN.md R40: band [rs_ps, rs_ps + rs_G) of tile-rows, chunk k = its k-th subtile rows
      return base + rs_band_row<TM>(p, ti, a, rs_ps, rs_G) * p.ldc + (int64_t)tj * BN;
    default:  // EPI_A2A: row -> slot in its destination pool (row_slot, prefetched)
      return base + (int64_t)a2a_slot * BN;
  }
}

// One persistent worker = one CTA (CG=1) or one CTA pair (CG=2).  Worker w of
// S = gridDim.x/CG runs positions w, w+S, ... (wave floor(p/S)).
// MJ: operand majorness (bit 0: A is [K, M] M-major, bit 1: Bt is [K, N]
// N-major — the weight-gradient dW = dY^T X layout); 0 = both K-major.
// MC: CTA pairs per cluster.  MC = 2 (K-major, no tail split, even S): the
// two pairs of a cluster run consecutive execution positions p, p^1 in
// lockstep; when the two tiles share their A tile-row (or B tile-column), each
// CTA loads half of its share of that operand and TMA-multicasts it to the
// CTA at the same half of the other pair, so the operand crosses L2 once for
// both tiles (tmA2 / tmB2: maps with half-height boxes).
template <int BN, int CG, int MJ, int MC, int RB = 128>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    fo_gemm_tcgen05_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                           const __grid_constant__ CUtensorMap tmA2, const __grid_constant__ CUtensorMap tmB2,
                           const __grid_constant__ CUtensorMap tmC, const GemmArgs p) {
  using C = Cfg<BN, CG, RB>;
  constexpr int ST = C::STAGES;
  constexpr int TM = RB * CG;  // tile rows
  constexpr int A_STAGE_BYTES = C::A_STAGE;
  constexpr int RPW = RB / 4;  // accumulator rows per epilogue warp (TMEM lanes 32q .. 32q + RPW - 1)
  static_assert(RB == 128 || (RB == 64 && CG == 1 && MJ == 0 && MC == 1), "64-row tiles: one CTA, K-major");
  static_assert(!(MJ & 2) || (C::B_ROWS % 64 == 0), "MN-major B needs 64-row chunks");
  static_assert(MC == 1 || (CG == 2 && MJ == 0), "multicast clusters: CTA pairs, K-major operands");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                                   // ST x 16 KB
  uint8_t* sB = smem + ST * A_STAGE_BYTES;              // ST x (BN/CG)*128 B
  uint8_t* sEpi = smem + ST * C::STAGE_BYTES;           // 4 warps x 32 rows x pitch
  uint64_t* full = reinterpret_cast<uint64_t*>(sEpi + EPI_BYTES);
  uint64_t* empty = full + ST;
  uint64_t* tfull = empty + ST;
  uint64_t* tempty = tfull + 2;
  uint64_t* lte_go = tempty + 2;    // shared last-tile epilogue: accumulator ready for warps 0-3
  uint64_t* lte_done = tempty + 3;  // ... and warps 0-3's stores complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 4);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t crank = (CG * MC == 1) ? 0u : cluster_rank();
  const uint32_t half = (CG == 1) ? 0u : (crank & 1u);  // this CTA's half of the pair's tile
  const uint32_t pic = crank >> 1;                      // pair index inside the cluster (MC = 2)
  const uint32_t lead_rank = crank & ~1u;               // the pair's leader CTA
  const bool leader = (half == 0);
  const uint16_t pair_mask = (uint16_t)(0x3u << (2 * pic));
  const int worker = blockIdx.x / CG;
  const int nworkers = gridDim.x / CG;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    if (p.tma_store) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmC)) : "memory");
    if constexpr (MC == 2) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA2)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB2)) : "memory");
    }
  }
  // Producer prologue (K-major, no multicast, a regular first unit, A
  // resident): the first tile's row is read now and its first k-blocks are
  // loaded right after the setup sync, in straight-line code — the main
  // loop's first TMA otherwise issues ~1 us after the sync (the table load,
  // then the loop's cold code path; profiles/r02_epilogue_ab.txt)
  const bool pro = MJ == 0 && MC == 1 && p.tail_pos > worker && !p.a_ready;
  int t_pro = 0;
  if (pro && warp == 0 && lane == 0) t_pro = p.order[worker];  // consumed after the setup
  if (warp == 3 && lane == 0) {
    // warm L2 with the table entries the producer needs for its first TMA
    // (cold after an L2 flush) while the setup below runs; non-blocking
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p.order + worker));
    if (p.seg) asm volatile("prefetch.global.L2 [%0];" ::"l"(p.wseg + worker));
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], MC);  // MC = 2: both pairs' MMAs release a stage (their loads fill each other's)
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 4 * CG);  // one arrive per epilogue warp of each CTA of the group
    }
    mbar_init(lte_go, 1);
    mbar_init(lte_done, 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    if constexpr (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"((uint32_t)C::TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"((uint32_t)C::TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  if constexpr (CG * MC == 1) __syncthreads(); else cluster_setup_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int KB = (int)(p.K / BK);
  constexpr int NC = BN / EPI_COLS;  // 64-column epilogue chunks per tile
  // Shared last-tile epilogue: a worker's last unit has no successor whose
  // MMAs hide its epilogue, and one warp per SM sub-partition stages its
  // chunks serially (~0.5 us per 64-column chunk: TMEM load, bf16 pack,
  // staging, store issue), so warps 0-3 — producer, MMA issuer, TMEM
  // allocator, idle, all done by then — take the upper half of its chunks
  // (measured: the last signal ~1 us earlier on one-wave shapes,
  // profiles/r02_epilogue_ab.txt).  Whole tiles with the TMA-store epilogue
  // only (split-tile parts/owners and SwiGLU keep the 4-warp path; so do
  // multicast clusters: a partner's loads may still land in this CTA's
  // stages, which warps 0-3 reuse as staging).  Whether the last unit is a
  // whole tile is decided where it is needed (a split plan's segment table
  // is cold here: reading it now would delay every warp's start).
  const bool lte = MC == 1 && NC >= 2 && p.tma_store && p.mode != EPI_SWIGLU;
  // one TMA box store of chunk c of rows [r0, r0 + RPW) of a tile staged in
  // `s`: row-major C, AR slot or RS band (h >= RPW: consecutive buffer rows)
  auto tma_chunk = [&](const uint8_t* s, int c, int pos, int ti, int tj, int r0, int2 rs) {
    if (p.mode == EPI_SLOT) tma_store_2d(&tmC, s, c * EPI_COLS, pos * TM + r0);
    else if (p.mode == EPI_RS_BAND)
      tma_store_2d(&tmC, s, tj * BN + c * EPI_COLS, (int)rs_band_row<TM>(p, ti, r0, rs.x, rs.y));
    else tma_store_2d(&tmC, s, tj * BN + c * EPI_COLS, ti * TM + r0);
    bulk_commit();
  };

  if (warp == 0) {
    // ======================= TMA producer (every CTA loads its own A rows and B rows)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int kk_pro = 0;  // unit 0's k-blocks already issued by the prologue
      if (pro) {
        const int ti = t_pro / p.Nt, tj = t_pro - ti * p.Nt;
        const int arow = ti * TM + (int)half * RB, brow = tj * BN + (int)half * C::B_ROWS;
        kk_pro = min(ST, KB);
        for (int s0 = 0; s0 < kk_pro; ++s0) {  // fresh stages: no empty wait
          if (leader) mbar_arrive_expect_tx(&full[s0], CG * C::STAGE_BYTES);
          if constexpr (CG == 1) {
            tma_load_2d(sA + s0 * A_STAGE_BYTES, &tmA, s0 * BK, arow, &full[s0]);
            tma_load_2d(sB + s0 * C::B_STAGE_BYTES, &tmB, s0 * BK, brow, &full[s0]);
          } else {
            const uint32_t fb = mapa_shared(&full[s0], lead_rank);
            tma_load_2d_2sm(sA + s0 * A_STAGE_BYTES, &tmA, s0 * BK, arow, fb);
            tma_load_2d_2sm(sB + s0 * C::B_STAGE_BYTES, &tmB, s0 * BK, brow, fb);
          }
        }
        stage = kk_pro % ST;
        phase = (kk_pro == ST) ? 1u : 0u;
      }
      int ready_chunk = -1;
      // the first regular unit's tile is loaded independently of the segment
      // table, so the two loads overlap
      const bool reg0 = p.tail_pos > worker;
      const int t_first = reg0 ? p.order[worker] : 0;
      const int nu = unit_count(p, worker, nworkers);
      for (int k = 0; k < nu; ++k) {
        const Unit un = my_unit(p, worker, nworkers, k, KB);
        const int u = un.pos;  // == worker + k*S without a split tail (multicast / wave sync)
        const int t = (k == 0 && reg0) ? t_first : p.order[un.pos];
        const int ti = t / p.Nt, tj = t - ti * p.Nt;
        if (p.a_ready && ti / p.a_chunk_rows != ready_chunk) {
          // host-staged A: wait until this tile-row's chunk has landed (the
          // copy stream's release write follows the chunk's H2D copy), then
          // order the generic-proxy acquire before the async-proxy TMA reads
          ready_chunk = ti / p.a_chunk_rows;
          while ((int32_t)(ld_acquire(p.a_ready + ready_chunk) - p.a_epoch) < 0) __nanosleep(128);
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        const int arow = ti * TM + (int)half * RB;
        const int brow = tj * BN + (int)half * C::B_ROWS;
        // multicast partner: the other pair of the cluster runs position u^1
        bool mcA = false, mcB = false;
        uint16_t mc_mask = 0;
        if constexpr (MC == 2) {
          if ((u ^ 1) < p.tiles) {
            const int t2 = p.order[u ^ 1];
            const int ti2 = t2 / p.Nt;
            mcA = (ti2 == ti);
            mcB = (t2 - ti2 * p.Nt == tj);
            mc_mask = (uint16_t)((1u << half) | (1u << (2 + half)));
          }
        }
        const int wave = k;  // wave sync runs without a split tail: unit k = wave k
        if (p.wave_ctr && wave > 0) {
          // keep the waves aligned: no load of wave w before every CTA of
          // wave w-1 has issued its last one (cyclic compare: monotone counters)
          const uint32_t size = (uint32_t)min(nworkers, p.tiles - (wave - 1) * nworkers) * CG;
          const uint32_t target = (p.wave_epoch + 1u) * size;
          while ((int32_t)(ld_acquire(p.wave_ctr + wave - 1) - target) < 0) __nanosleep(64);
        }
        const bool rev = p.k_snake && (k & 1);
        for (int kk = un.kb0 + (k == 0 ? kk_pro : 0); kk < un.kb1; ++kk) {
          const int kb = rev ? un.kb0 + un.kb1 - 1 - kk : kk;
          mbar_wait(&empty[stage], phase ^ 1);
          // K-major operand: one box [rows, 64 k]; MN-major operand: 64x64
          // boxes [64 k, 64 mn], one per 64-row chunk, 8 KB apart
          auto load = [&](void* dst, const CUtensorMap* map, int rows0, int nrows) {
            const bool mn = (map == &tmA) ? (MJ & 1) : (MJ & 2);
            if (!mn) {
              if constexpr (CG == 1) tma_load_2d(dst, map, kb * BK, rows0, &full[stage]);
              else tma_load_2d_2sm(dst, map, kb * BK, rows0, mapa_shared(&full[stage], lead_rank));
            } else {
              for (int h = 0; h < nrows / 64; ++h) {
                uint8_t* d = reinterpret_cast<uint8_t*>(dst) + h * 8192;
                if constexpr (CG == 1) tma_load_2d(d, map, rows0 + 64 * h, kb * BK, &full[stage]);
                else tma_load_2d_2sm(d, map, rows0 + 64 * h, kb * BK, mapa_shared(&full[stage], lead_rank));
              }
            }
          };
          // a pair's two CTAs' bytes are all counted on the leader's full barrier
          if (leader) mbar_arrive_expect_tx(&full[stage], CG * C::STAGE_BYTES);
          if constexpr (MC == 2) {
            // shared operand: this CTA loads rows [pic*h, pic*h + h) of its half
            // and multicasts them to the same half of both pairs
            if (mcA)
              tma_load_2d_2sm_mc(sA + stage * A_STAGE_BYTES + pic * (A_STAGE_BYTES / 2), &tmA2, kb * BK,
                                 arow + (int)pic * (RB / 2), &full[stage], mc_mask);
            else
              tma_load_2d_2sm(sA + stage * A_STAGE_BYTES, &tmA, kb * BK, arow, mapa_shared(&full[stage], lead_rank));
            if (mcB)
              tma_load_2d_2sm_mc(sB + stage * C::B_STAGE_BYTES + pic * (C::B_STAGE_BYTES / 2), &tmB2, kb * BK,
                                 brow + (int)pic * (C::B_ROWS / 2), &full[stage], mc_mask);
            else
              tma_load_2d_2sm(sB + stage * C::B_STAGE_BYTES, &tmB, kb * BK, brow, mapa_shared(&full[stage], lead_rank));
          } else {
            load(sA + stage * A_STAGE_BYTES, &tmA, arow, RB);
            load(sB + stage * C::B_STAGE_BYTES, &tmB, brow, C::B_ROWS);
          }
          if (++stage == ST) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (p.wave_ctr) atomicAdd(p.wave_ctr + wave, 1u);
      }
    }
  } else if (warp == 1) {
    // ======================= MMA issuer (leader CTA): the whole warp runs the
    // loop (warp-uniform operands stay in uniform registers), one elected lane
    // issues each tcgen05.mma / commit
    if (leader) {
      constexpr uint32_t idesc = idesc_bf16<TM, BN, MJ>();
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t aphase = 0;
      const int nu = unit_count(p, worker, nworkers);
      for (int k = 0; k < nu; ++k) {
        const Unit un = my_unit(p, worker, nworkers, k, KB);
        const int u = un.pos;
        mbar_wait(&tempty[acc], aphase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
        for (int kb = un.kb0; kb < un.kb1; ++kb) {  // (order-free here: the producer decides which k-block)
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(sA + stage * A_STAGE_BYTES);
          const uint32_t sb = smem_u32(sB + stage * C::B_STAGE_BYTES);
          // per K=16 step: K-major +32 bytes along K inside the 128-byte swizzle
          // row (+2 in the >>4 address field); MN-major +2 core groups of 8
          // k-rows (+2048 B = +128); the field never carries (smem < 256 KB)
          umma_kblock<CG>(d_tmem, (MJ & 1) ? sw128_mn_desc(sa) : sw128_desc(sa),
                          (MJ & 2) ? sw128_mn_desc(sb) : sw128_desc(sb), (MJ & 1) ? 128u : 2u, (MJ & 2) ? 128u : 2u,
                          idesc, kb != un.kb0 ? 1u : 0u);
          // frees the smem stage when these MMAs retire: in both CTAs of the
          // pair; with a multicast partner in all four CTAs (count 2 each), and
          // alone (partner done) twice in the pair's own CTAs
          if (elect_one()) {
            if constexpr (MC == 2) {
              if ((u ^ 1) < p.tiles) {
                umma_commit<CG>(&empty[stage], 0xF);
              } else {
                umma_commit<CG>(&empty[stage], pair_mask);
                umma_commit<CG>(&empty[stage], pair_mask);
              }
            } else {
              umma_commit<CG>(&empty[stage]);
            }
          }
          __syncwarp();
          if (++stage == ST) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (elect_one()) umma_commit<CG>(&tfull[acc], pair_mask);  // accumulator ready for the pair's epilogues
        __syncwarp();
        if (++acc == 2) {
          acc = 0;
          aphase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    // ======================= epilogue: reorder-store + signal (this CTA's 128 rows)
    const int q = warp - 4;  // TMEM lane quarter: warp (4+q) may access lanes 32q..32q+31
    uint8_t* stg = sEpi + q * EPI_WARP_BYTES;
    const uint32_t tempty_leader0 = (CG == 1) ? 0u : mapa_shared(&tempty[0], lead_rank);
    int acc = 0;
    uint32_t aphase = 0;
    // destination-table entries of the next tile (RS: group start / size of
    // the position; A2A: this lane's 8 row slots), loaded one tile ahead
    int2 nx_rs = make_int2(0, 0);
    int32_t nx_slot[8];
#pragma unroll
    for (int it = 0; it < 8; ++it) nx_slot[it] = 0;
    static_assert(RPW == 32 || RPW == 16, "rows per epilogue warp");
    auto prefetch_dst = [&](int npos) {
      if (p.mode == EPI_RS || p.mode == EPI_RS_BAND) {
        nx_rs = p.rs_info[npos];
      } else if (p.mode == EPI_A2A) {
#pragma unroll
        for (int it = 0; it < RPW / 4; ++it)
          nx_slot[it] = p.row_slot[(int64_t)npos * TM + (int)half * RB + q * RPW + it * 4 + (lane >> 3)];
      }
    };
    const int nu = unit_count(p, worker, nworkers);
    if (nu > 0) prefetch_dst(my_unit(p, worker, nworkers, 0, KB).pos);
    for (int k = 0; k < nu; ++k) {
      const Unit un = my_unit(p, worker, nworkers, k, KB);
      const int pos = un.pos;
      const int t = p.order[pos];
      const int ti = t / p.Nt, tj = t - ti * p.Nt;
      const bool owner = (un.role == 1), part = (un.role == 2);  // split tail tile roles
      const int tt = un.tt;  // tail tile index (flags)
      const int row = (int)half * RB + q * RPW + lane;  // this thread's accumulator row in the tile (lane < RPW)
      // this lane's 8 destination rows of the tile (rows it*4 + lane/8 of the
      // warp's 32-row quarter), resolved once per tile from table entries
      // loaded during the previous tile (no memory latency here: at short K
      // the epilogue is on the critical path)
      __nv_bfloat16* drow[8];
      const int2 cur_rs = nx_rs;  // this tile's RS group / band (nx_rs moves on to the next tile)
#pragma unroll
      for (int it = 0; it < RPW / 4; ++it)
        drow[it] = row_dst<TM, BN>(p, pos, ti, tj, (int)half * RB + q * RPW + it * 4 + (lane >> 3), nx_rs.x, nx_rs.y,
                                   nx_slot[it]) +
                   (lane & 7) * 8;
      mbar_wait(&tfull[acc], aphase);
      const bool lte_tile = lte && k == nu - 1 && un.role == 0;
      if (lte_tile && q == 0 && lane == 0) mbar_arrive(lte_go);  // accumulator ready: wake warps 0-3
      if (k + 1 < nu) prefetch_dst(my_unit(p, worker, nworkers, k + 1, KB).pos);
      tc_fence_after();
      if (p.dist_fold && p.mode != EPI_SWIGLU && (owner || part)) {
        // distributed fold of a split tile (f-slices: every slice is its
        // worker's last unit, so slices may wait on each other): slice `me`
        // reduces and stores the 64-column chunks c with c % f == me and
        // publishes the fp32 partials of the others to its own slot
        const int f = un.nparts, me = un.idx;
        const int base = owner ? un.slot : un.slot - me + 1;  // the tile's first slot
        auto pslot = [&](int j) { return j == 0 ? base + f - 1 : base + j - 1; };
        auto release_tmem = [&]() {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if constexpr (CG == 1) mbar_arrive(&tempty[acc]);
            else mbar_arrive_cluster(tempty_leader0 + 8u * acc);
          }
        };
        const bool has_own = me < NC;
        // the worker's previous tile may have left TMA stores reading the staging
        if (p.tma_store) {
          if (lane == 0) bulk_wait_read0();
          __syncwarp();
        }
#pragma unroll 1
        for (int c = 0; c < NC; ++c) {
          if (c % f == me) continue;
          uint32_t v[64];
          const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + c * EPI_COLS);
          tmem_ld32(taddr, v);
          tmem_ld32(taddr + 32, v + 32);
          tmem_wait_ld();
          float4* w = reinterpret_cast<float4*>(p.workspace + (int64_t)pslot(me) * TM * BN) + (int64_t)c * 16 * TM + row;
#pragma unroll
          for (int x = 0; x < 16; ++x)
            w[x * TM] = make_float4(__uint_as_float(v[4 * x]), __uint_as_float(v[4 * x + 1]),
                                    __uint_as_float(v[4 * x + 2]), __uint_as_float(v[4 * x + 3]));
        }
        if (!has_own) release_tmem();
        // published -> count it; then wait for every slice's partials
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (q == 0 && lane == 0) {
          uint32_t* fl = p.flags + tt * CG + half;
          red_release_add(fl, 1u);
          while (ld_acquire(fl) < (uint32_t)f) __nanosleep(32);
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        const int last_own = has_own ? me + ((NC - 1 - me) / f) * f : -1;
#pragma unroll 1
        for (int c = me; c < NC; c += f) {
          uint32_t v[64];
          const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + c * EPI_COLS);
          tmem_ld32(taddr, v);
          tmem_ld32(taddr + 32, v + 32);
          tmem_wait_ld();
          if (c == last_own) release_tmem();
          // the other slices' partials in k order (deterministic)
          for (int j = 0; j < f; ++j) {
            if (j == me) continue;
            const float4* w =
                reinterpret_cast<const float4*>(p.workspace + (int64_t)pslot(j) * TM * BN) + (int64_t)c * 16 * TM + row;
#pragma unroll
            for (int x = 0; x < 16; ++x) {
              const float4 fv = w[x * TM];
              v[4 * x] = __float_as_uint(__uint_as_float(v[4 * x]) + fv.x);
              v[4 * x + 1] = __float_as_uint(__uint_as_float(v[4 * x + 1]) + fv.y);
              v[4 * x + 2] = __float_as_uint(__uint_as_float(v[4 * x + 2]) + fv.z);
              v[4 * x + 3] = __float_as_uint(__uint_as_float(v[4 * x + 3]) + fv.w);
            }
          }
#pragma unroll
          for (int x = 0; x < 8; ++x) {
            uint4 o;
            o.x = pack_bf16(v[8 * x + 0], v[8 * x + 1]);
            o.y = pack_bf16(v[8 * x + 2], v[8 * x + 3]);
            o.z = pack_bf16(v[8 * x + 4], v[8 * x + 5]);
            o.w = pack_bf16(v[8 * x + 6], v[8 * x + 7]);
            *stg_at(stg, lane, x) = o;
          }
          __syncwarp();
#pragma unroll
          for (int it = 0; it < RPW / 4; ++it) {
            const int r = it * 4 + (lane >> 3);
            const uint4 o = *stg_at(stg, r, lane & 7);
            *reinterpret_cast<uint4*>(drow[it] + c * EPI_COLS) = o;
          }
          __syncwarp();
        }
        // the last slice to finish its chunks signals the tile (acq_rel: the
        // other slices' stores, released by their increments, precede ours)
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (q == 0 && lane == 0) {
          if (atom_add_acq_rel(p.done + tt * CG + half, 1u) == (uint32_t)(f - 1)) {
            if (p.counters) red_release_add(&p.counters[p.group_of_pos[pos]], 1u);
            if (p.tile_ts && leader) p.tile_ts[pos] = globaltimer();
          }
        }
        if (++acc == 2) {
          acc = 0;
          aphase ^= 1;
        }
        continue;
      }
      if (owner) {
        // owner of a split tile: wait until the other parts' partials of this
        // CTA's rows are published (acquire), then fold them in below
        if (q == 0 && lane == 0) {
          const uint32_t* f = p.flags + tt * CG + half;
          while (ld_acquire(f) < (uint32_t)(un.nparts - 1)) __nanosleep(32);
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
      if constexpr (BN == 256) {
        if (p.mode == EPI_SWIGLU && !part) {  // a split tile's parts publish fp32 partials below
          // fused SwiGLU (the MLP's activation): gate columns [0,128) and up
          // columns [128,256) of the accumulator, 32 output columns per step,
          // silu(g) * u in fp32, one bf16 rounding; 8 rows x 64 B per store
#pragma unroll 1
          for (int c2 = 0; c2 < 4; ++c2) {
            uint32_t g[32], up[32];
            const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + 32 * c2);
            tmem_ld32(taddr, g);
            tmem_ld32(taddr + 128, up);
            tmem_wait_ld();
            if (owner) {
              // fold in the parts' partials of columns [32c2, +32) (gate) and
              // [128 + 32c2, +32) (up): chunk c2/2 resp. 2 + c2/2, float4s 8(c2%2)..
              for (int sl = 0; sl < un.nparts - 1; ++sl) {
                const float4* w = reinterpret_cast<const float4*>(p.workspace + (int64_t)(un.slot + sl) * TM * BN);
#pragma unroll
                for (int x = 0; x < 8; ++x) {
                  const float4 fg = w[((int64_t)(c2 >> 1) * 16 + 8 * (c2 & 1) + x) * TM + row];
                  const float4 fu = w[((int64_t)(2 + (c2 >> 1)) * 16 + 8 * (c2 & 1) + x) * TM + row];
                  g[4 * x] = __float_as_uint(__uint_as_float(g[4 * x]) + fg.x);
                  g[4 * x + 1] = __float_as_uint(__uint_as_float(g[4 * x + 1]) + fg.y);
                  g[4 * x + 2] = __float_as_uint(__uint_as_float(g[4 * x + 2]) + fg.z);
                  g[4 * x + 3] = __float_as_uint(__uint_as_float(g[4 * x + 3]) + fg.w);
                  up[4 * x] = __float_as_uint(__uint_as_float(up[4 * x]) + fu.x);
                  up[4 * x + 1] = __float_as_uint(__uint_as_float(up[4 * x + 1]) + fu.y);
                  up[4 * x + 2] = __float_as_uint(__uint_as_float(up[4 * x + 2]) + fu.z);
                  up[4 * x + 3] = __float_as_uint(__uint_as_float(up[4 * x + 3]) + fu.w);
                }
              }
            }
            if (c2 == 3) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) {
                if constexpr (CG == 1) mbar_arrive(&tempty[acc]);
                else mbar_arrive_cluster(tempty_leader0 + 8u * acc);
              }
            }
#pragma unroll
            for (int x = 0; x < 4; ++x) {
              float o[8];
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                const float gv = __uint_as_float(g[8 * x + e]);
                o[e] = gv / (1.f + __expf(-gv)) * __uint_as_float(up[8 * x + e]);
              }
              uint4 w;
              w.x = pack_bf16(__float_as_uint(o[0]), __float_as_uint(o[1]));
              w.y = pack_bf16(__float_as_uint(o[2]), __float_as_uint(o[3]));
              w.z = pack_bf16(__float_as_uint(o[4]), __float_as_uint(o[5]));
              w.w = pack_bf16(__float_as_uint(o[6]), __float_as_uint(o[7]));
              *stg_at(stg, lane, x) = w;
            }
            __syncwarp();
#pragma unroll
            for (int it = 0; it < 4; ++it) {
              const int r = it * 8 + (lane >> 2);
              const uint4 w = *stg_at(stg, r, lane & 3);
              __nv_bfloat16* d = reinterpret_cast<__nv_bfloat16*>(p.dst) +
                                 ((int64_t)ti * TM + (int)half * RB + q * 32 + r) * p.ldc + (int64_t)tj * 128 +
                                 32 * c2 + (lane & 3) * 8;
              *reinterpret_cast<uint4*>(d) = w;
            }
            __syncwarp();
          }
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (q == 0 && lane == 0) {
            if (p.counters) red_release_add(&p.counters[p.group_of_pos[pos]], 1u);
            if (p.tile_ts && leader) p.tile_ts[pos] = globaltimer();
          }
          if (++acc == 2) {
            acc = 0;
            aphase ^= 1;
          }
          continue;
        }
      }
      const int c_end = lte_tile ? NC / 2 : NC;  // the shared last tile: chunks [NC/2, NC) go to warps 0-3
#pragma unroll 1
      for (int c = 0; c < c_end; ++c) {
        uint32_t v[64];
        const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + c * EPI_COLS);
        tmem_ld32(taddr, v);
        tmem_ld32(taddr + 32, v + 32);
        tmem_wait_ld();
        if (c == c_end - 1) {
          // accumulator fully read: hand the TMEM stage back to the MMA warp
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if constexpr (CG == 1) mbar_arrive(&tempty[acc]);
            else mbar_arrive_cluster(tempty_leader0 + 8u * acc);
          }
        }
        // partial slot layout [chunk c][float4 x][tile row][4]: for a fixed x the
        // warp's 32 rows are 32 consecutive float4 — coalesced stores and loads
        if (part) {
          // part of a split tile: publish fp32 partials of this thread's row
          float4* w = reinterpret_cast<float4*>(p.workspace + (int64_t)un.slot * TM * BN) + (int64_t)c * 16 * TM + row;
#pragma unroll
          for (int x = 0; x < 16; ++x)
            w[x * TM] = make_float4(__uint_as_float(v[4 * x]), __uint_as_float(v[4 * x + 1]),
                                    __uint_as_float(v[4 * x + 2]), __uint_as_float(v[4 * x + 3]));
          continue;
        }
        if (owner) {
          // the parts' partials in part order (deterministic), slots slot..slot+nparts-2
          for (int sl = 0; sl < un.nparts - 1; ++sl) {
            const float4* w = reinterpret_cast<const float4*>(p.workspace + (int64_t)(un.slot + sl) * TM * BN) +
                              (int64_t)c * 16 * TM + row;
#pragma unroll
            for (int x = 0; x < 16; ++x) {
              const float4 f = w[x * TM];
              v[4 * x] = __float_as_uint(__uint_as_float(v[4 * x]) + f.x);
              v[4 * x + 1] = __float_as_uint(__uint_as_float(v[4 * x + 1]) + f.y);
              v[4 * x + 2] = __float_as_uint(__uint_as_float(v[4 * x + 2]) + f.z);
              v[4 * x + 3] = __float_as_uint(__uint_as_float(v[4 * x + 3]) + f.w);
            }
          }
        }
        // TMA store (row-major C / AR slot / RS bands, whole tiles): the
        // staging buffer must be read out by the previous chunk's store (also
        // the previous tile's, for an owner's 16-byte path) before it is
        // refilled.  (A second staging buffer per warp, letting chunk c fill
        // one while chunk c-1's store reads the other, measured no faster:
        // profiles/r02_epilogue_ab.txt)
        const bool tma = p.tma_store && !owner;
        if (p.tma_store) {
          if (lane == 0) bulk_wait_read0();
          __syncwarp();
        }
        // stage row `lane` (this thread's TMEM lane) as bf16
        if (lane < RPW) {
#pragma unroll
          for (int x = 0; x < 8; ++x) {
            uint4 w;
            w.x = pack_bf16(v[8 * x + 0], v[8 * x + 1]);
            w.y = pack_bf16(v[8 * x + 2], v[8 * x + 3]);
            w.z = pack_bf16(v[8 * x + 4], v[8 * x + 5]);
            w.w = pack_bf16(v[8 * x + 6], v[8 * x + 7]);
            *stg_at(stg, lane, x) = w;
          }
        }
        if (tma) {
          // the warp's RPW rows x 64 columns as one box (generic-proxy smem
          // writes made visible to the async proxy first)
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) tma_chunk(stg, c, pos, ti, tj, (int)half * RB + q * RPW, cur_rs);
          continue;
        }
        __syncwarp();
        // coalesced copy-out: each instruction moves 4 rows x 128 B
#pragma unroll
        for (int it = 0; it < RPW / 4; ++it) {
          const int r = it * 4 + (lane >> 3);
          const int ch = lane & 7;
          const uint4 w = *stg_at(stg, r, ch);
          *reinterpret_cast<uint4*>(drow[it] + c * EPI_COLS) = w;
        }
        __syncwarp();
      }
      if (part) {
        // partials of this CTA's rows stored -> one release increment of the tile's flag
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (q == 0 && lane == 0) red_release_add(p.flags + tt * CG + half, 1u);
        if (++acc == 2) {
          acc = 0;
          aphase ^= 1;
        }
        continue;
      }
      // all 128 epilogue threads of this CTA finished their stores -> one
      // release add (a pair signals twice per tile: counters count half tiles);
      // TMA stores are complete (not just read out) and ordered before the
      // release by the async-proxy fence
      if (p.tma_store && !owner && p.counters && lane == 0) {
        bulk_wait_all();
        asm volatile("fence.proxy.async.global;" ::: "memory");
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (q == 0 && lane == 0) {
        // the shared last tile: warps 0-3's stores are complete too (their
        // release arrivals, acquired here, precede this thread's release)
        if (lte_tile) mbar_wait(lte_done, 0);
        if (p.counters) red_release_add(&p.counters[p.group_of_pos[pos]], 1u);
        if (p.tile_ts && leader) p.tile_ts[pos] = globaltimer();
      }
      if (++acc == 2) {
        acc = 0;
        aphase ^= 1;
      }
    }
  }
  const int nu_all = (lte && warp < 4) ? unit_count(p, worker, nworkers) : 0;
  const Unit last = nu_all > 0 ? my_unit(p, worker, nworkers, nu_all - 1, KB) : Unit{};
  if (nu_all > 0 && last.role == 0) {
    // ======================= shared last-tile epilogue, warps 0-3 (TMEM lane
    // quarter = warp): chunks [NC/2, NC) of the worker's last tile, staged in
    // the idle A stages — every MMA, hence every load, has completed once
    // the accumulator is ready (lte_go: the epilogue warps saw tfull)
    static_assert(ST * A_STAGE_BYTES >= 4 * EPI_WARP_BYTES, "staging for warps 0-3 fits the A stages");
    __syncwarp();
    const int q = warp;
    const int k = nu_all - 1;
    const int pos = last.pos;
    const int t = p.order[pos];
    const int ti = t / p.Nt, tj = t - ti * p.Nt;
    const int2 rs = (p.mode == EPI_RS_BAND) ? p.rs_info[pos] : make_int2(0, 0);
    uint8_t* hstg = sA + q * EPI_WARP_BYTES;
    mbar_wait(lte_go, 0);
    tc_fence_after();
#pragma unroll 1
    for (int c = NC / 2; c < NC; ++c) {
      uint32_t v[64];
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)((k & 1) * BN + c * EPI_COLS);
      tmem_ld32(taddr, v);
      tmem_ld32(taddr + 32, v + 32);
      tmem_wait_ld();
      if (c > NC / 2) {
        if (lane == 0) bulk_wait_read0();
        __syncwarp();
      }
      if (lane < RPW) {
#pragma unroll
        for (int x = 0; x < 8; ++x) {
          uint4 w;
          w.x = pack_bf16(v[8 * x + 0], v[8 * x + 1]);
          w.y = pack_bf16(v[8 * x + 2], v[8 * x + 3]);
          w.z = pack_bf16(v[8 * x + 4], v[8 * x + 5]);
          w.w = pack_bf16(v[8 * x + 6], v[8 * x + 7]);
          *stg_at(hstg, lane, x) = w;
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) tma_chunk(hstg, c, pos, ti, tj, (int)half * RB + q * RPW, rs);
    }
    if (lane == 0) {
      bulk_wait_all();
      asm volatile("fence.proxy.async.global;" ::: "memory");
      mbar_arrive(lte_done);
    }
    tc_fence_before();
    __syncwarp();
  }
  if (warp >= 4 && lane == 0 && p.tma_store) bulk_wait_all();  // the staging must outlive the stores
  tc_fence_before();
  if constexpr (CG * MC == 1) __syncthreads(); else cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    if constexpr (CG == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"((uint32_t)C::TMEM_COLS)
                   : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"((uint32_t)C::TMEM_COLS)
                   : "memory");
  }
}

// ------------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  return fn;
}

// 2-D bf16 map with 128B swizzle.  K-major operand [rows, K]: box [box_rows, 64 k].
// MN-major operand stored [K, rows]: box [64 k, 64 rows].
bool make_map(CUtensorMap* m, const void* base, int64_t rows, int64_t K, int box_rows, bool mn_major) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(K * 2)};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  if (mn_major) {
    dims[0] = (cuuint64_t)rows;
    dims[1] = (cuuint64_t)K;
    strides[0] = (cuuint64_t)(rows * 2);
    box[0] = 64;
    box[1] = (cuuint32_t)BK;
  }
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN, int CG, int MJ, int MC, int RB = 128>
cudaError_t launch_cfg(const GemmArgs& a, cudaStream_t stream) {
  using C = Cfg<BN, CG, RB>;
  static std::atomic<uint64_t> attr_set{0};  // one bit per device (the attribute is per device context)
  auto kern = fo_gemm_tcgen05_kernel<BN, CG, MJ, MC, RB>;
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (!(attr_set.load() & bit)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr_set.fetch_or(bit);
  }
  CUtensorMap mA, mB, mA2, mB2;
  if (!make_map(&mA, a.A, a.M, a.K, RB, MJ & 1) || !make_map(&mB, a.Bt, a.N, a.K, C::B_ROWS, MJ & 2))
    return cudaErrorInvalidValue;
  if (MC == 2) {
    if (!make_map(&mA2, a.A, a.M, a.K, RB / 2, false) || !make_map(&mB2, a.Bt, a.N, a.K, C::B_ROWS / 2, false))
      return cudaErrorInvalidValue;
  } else {
    mA2 = mA;
    mB2 = mB;
  }
  // TMA-store epilogue for whole tiles into row-major C, AR slots or RS
  // bands (when a warp's rows stay inside one subtile, h >= rows per warp):
  // the destination as a 2-D bf16 tensor, box = 64 columns x one warp's rows
  GemmArgs g = a;
  CUtensorMap mC = mA;
  g.tma_store = 0;
  const bool tma_mode = a.mode == EPI_ROWMAJOR || a.mode == EPI_SLOT || (a.mode == EPI_RS_BAND && a.h >= RB / 4);
  if (tma_mode && !(reinterpret_cast<uintptr_t>(a.dst) & 15) && (a.mode == EPI_SLOT || (a.ldc * 2) % 16 == 0) &&
      a.tma_store_ok) {
    const int64_t rows = a.mode == EPI_SLOT ? (int64_t)a.tiles * RB * CG : a.M;
    const int64_t cols = a.mode == EPI_SLOT ? BN : a.N;
    const int64_t pitch = a.mode == EPI_SLOT ? BN : a.ldc;
    EncodeTiledFn enc = get_encode();
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)(pitch * 2)};
    cuuint32_t box[2] = {(cuuint32_t)EPI_COLS, (cuuint32_t)(RB / 4)};
    cuuint32_t estr[2] = {1, 1};
    if (enc && enc(&mC, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a.dst, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
      g.tma_store = 1;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(a.workers * CG);
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.dynamicSmemBytes = C::SMEM_BYTES;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG * MC;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, mA, mB, mA2, mB2, mC, g);
  count_launch();
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// Clusters of two CTA pairs resident at once for this configuration (per
// device, cached): a persistent grid of S pairs may use them only if all S/2
// clusters fit.
template <int BN>
int max_pair_clusters() {
  static std::atomic<int> cache[64];
  int dev = 0;
  cudaGetDevice(&dev);
  int v = cache[dev & 63].load();
  if (v) return v;
  using C = Cfg<BN, 2>;
  auto kern = fo_gemm_tcgen05_kernel<BN, 2, 0, 2>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(4);
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.dynamicSmemBytes = C::SMEM_BYTES;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 4;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
    cudaGetLastError();
    n = -1;
  }
  cache[dev & 63].store(n ? n : -1);
  return n ? n : -1;
}

std::atomic<int64_t> g_launches{0};

}  // namespace

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
int64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

bool gemm_shape_supported(int bm, int bn) {
  return (bm == 64 || bm == 128 || bm == 256) && (bn == 64 || bn == 128 || bn == 256);
}

template <int BN, int CG>
cudaError_t launch_mj(const GemmArgs& a, cudaStream_t stream) {
  switch (a.mn_major) {
    case 0:
      if constexpr (CG == 2) {
        // TMA multicast across clusters of two pairs (FO_OPT_MULTICAST): even S,
        // no tail split, every cluster resident
        if (a.multicast && a.workers % 2 == 0 && a.split == 1 && max_pair_clusters<BN>() >= a.workers / 2)
          return launch_cfg<BN, CG, 0, 2>(a, stream);
      }
      return launch_cfg<BN, CG, 0, 1>(a, stream);
    case 1: return launch_cfg<BN, CG, 1, 1>(a, stream);
    case 2: return launch_cfg<BN, CG, 2, 1>(a, stream);
    case 3: return launch_cfg<BN, CG, 3, 1>(a, stream);
  }
  return cudaErrorInvalidValue;
}

bool gemm_multicast_used(const GemmArgs& a) {
  if (!(a.BM == 256 && a.mn_major == 0 && a.multicast && a.workers % 2 == 0 && a.split == 1)) return false;
  switch (a.BN) {
    case 64: return false;
    case 128: return max_pair_clusters<128>() >= a.workers / 2;
    case 256: return max_pair_clusters<256>() >= a.workers / 2;
  }
  return false;
}

cudaError_t launch_gemm(const GemmArgs& a, cudaStream_t stream) {
  if (a.mn_major && a.BN == 64) return cudaErrorInvalidValue;  // MN-major needs >= 64-row B chunks per CTA
  if (a.BM == 64) {
    // tcgen05.mma M=64 (one CTA): K-major operands, no split tail / SwiGLU
    if (a.mn_major || a.split > 1 || a.mode == EPI_SWIGLU) return cudaErrorInvalidValue;
    switch (a.BN) {
      case 64: return launch_cfg<64, 1, 0, 1, 64>(a, stream);
      case 128: return launch_cfg<128, 1, 0, 1, 64>(a, stream);
      case 256: return launch_cfg<256, 1, 0, 1, 64>(a, stream);
    }
  } else if (a.BM == 128) {
    switch (a.BN) {
      case 64: return launch_cfg<64, 1, 0, 1>(a, stream);
      case 128: return launch_mj<128, 1>(a, stream);
      case 256: return launch_mj<256, 1>(a, stream);
    }
  } else if (a.BM == 256) {
    switch (a.BN) {
      case 64: return launch_cfg<64, 2, 0, 1>(a, stream);
      case 128: return launch_mj<128, 2>(a, stream);
      case 256: return launch_mj<256, 2>(a, stream);
    }
  }
  return cudaErrorInvalidValue;
}

}  // namespace fo
