// Post-communication reorder with an optional fused residual
// add / RMSNorm (R12), for sm_100a.
//
// One warp per output row.  Lane l handles the 16-byte chunks l, l+32, ... of
// the row; chunk c covers columns [8c, 8c+8) which all lie in tile-column
// jc = 8c / BN, so its source is one contiguous 16-byte run of the receive
// buffer:
//   IDENTITY  src row-major [rows, N]                 (AR ROWBAND / no-comm)
//   SLOT      (pos_of_tile[i*Nt+jc]*BM + r%BM)*BN + b (AR)
//   RS        (pos_of_tile[(r/h)*Nt+jc]*h + r%h)*BN + b
//   A2A       src_row[r*Nt+jc]*BN + b
// Reads are 16-byte vector loads (consecutive lanes read consecutive chunks of
// a BN-wide contiguous run), writes are fully coalesced row segments, so the
// kernel is HBM-bound at 2 x bytes(out) (+ residual).
#include <atomic>

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "../../../include/flashoverlap.h"
#include "../kernels.h"

namespace fo {
namespace {

// Per-row source description: chunk c of row r (columns 8c..8c+7, tile-column
// jc = 8c >> log2(BN)) starts at element  tbl[jc] * tscale + roff + (8c & (BN-1)).
struct RowSrc {
  const int32_t* tbl;  // per tile-column table row (pos_of_tile / src_row), or null for identity
  int64_t tscale;      // elements per table unit
  int64_t roff;        // element offset of this row inside the unit
};

template <int MAP>
__device__ __forceinline__ RowSrc row_src(const PostArgs& p, int64_t r) {
  RowSrc s;
  if (MAP == POSTMAP_IDENTITY) {
    s.tbl = nullptr;
    s.tscale = 0;
    s.roff = r * p.N;
  } else if (MAP == POSTMAP_ROWX) {
    // PAPER.md:390 row exchange: global row r = (l/h)*BM + k*h + l%h came from
    // rank k's local row l, i.e. row k*(M/n) + l of the rank-major gather
    const int64_t n = p.BM / p.h, rows_per_rank = p.rows / n;
    const int64_t k = (r % p.BM) / p.h, l = (r / p.BM) * p.h + r % p.h;
    s.tbl = nullptr;
    s.tscale = 0;
    s.roff = (k * rows_per_rank + l) * p.N;
  } else if (MAP == POSTMAP_SLOT) {  // slot of tile (r/BM, jc), row r%BM
    s.tbl = p.pos_of_tile + (r / p.BM) * p.Nt;
    s.tscale = (int64_t)p.BM * p.BN;
    s.roff = (r % p.BM) * p.BN;
  } else if (MAP == POSTMAP_RS) {    // receive row q*h + r%h
    s.tbl = p.pos_of_tile + (r / p.h) * p.Nt;
    s.tscale = (int64_t)p.h * p.BN;
    s.roff = (r % p.h) * p.BN;
  } else {                           // A2A subtoken
    s.tbl = p.src_row + r * p.Nt;
    s.tscale = p.BN;
    s.roff = 0;
  }
  return s;
}

template <int MAP>
__device__ __forceinline__ int64_t chunk_src(const RowSrc& s, int64_t col, int lbn, int bn_mask) {
  if (MAP == POSTMAP_IDENTITY || MAP == POSTMAP_ROWX) return s.roff + col;
  return (int64_t)__ldg(s.tbl + (col >> lbn)) * s.tscale + s.roff + (col & bn_mask);
}

__device__ __forceinline__ uint4 ld_stream(const void* ptr) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(ptr));
  return v;
}

__device__ __forceinline__ uint4 ld_coherent(const void* ptr) { return *reinterpret_cast<const uint4*>(ptr); }

__device__ __forceinline__ void st_stream(void* ptr, const uint4& v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(ptr), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

__device__ __forceinline__ void unpack8(const uint4& v, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}

__device__ __forceinline__ uint4 pack8(const float* f) {
  uint4 v;
  uint32_t* w = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
    w[i] = *reinterpret_cast<uint32_t*>(&h);
  }
  return v;
}

constexpr int UNROLL = 4;
constexpr int SEG_CHUNKS = 32 * UNROLL;  // 16-byte chunks per work unit (2 KB)

// Copy / residual-add: work unit = (row, 2 KB segment) so that outputs with
// few rows (RS: M/n rows) still fill every SM.  One warp per unit; lane l
// moves chunks l, l+32, l+64, l+96 with UNROLL independent loads in flight.
template <int MAP, int OP>
__global__ void __launch_bounds__(256) fo_post_reorder_kernel(const PostArgs p, int lbn) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t chunks = p.N >> 3;
  const int64_t upr = (chunks + SEG_CHUNKS - 1) / SEG_CHUNKS;  // units per row
  const int64_t units = p.rows * upr;
  const int bn_mask = p.BN - 1;
  const __nv_bfloat16* src = reinterpret_cast<const __nv_bfloat16*>(p.src);
  __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(p.out);
  const __nv_bfloat16* res = reinterpret_cast<const __nv_bfloat16*>(p.residual);
  const bool inplace = (p.src == p.out);
  for (int64_t u = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); u < units; u += warps) {
    const int64_t r = u / upr;
    const int64_t c0 = (u - r * upr) * SEG_CHUNKS;
    const RowSrc rs = row_src<MAP>(p, r);
    __nv_bfloat16* orow = out + r * p.N;
    const __nv_bfloat16* rrow = res ? res + r * p.N : nullptr;
    if (c0 + SEG_CHUNKS <= chunks) {
      uint4 v[UNROLL];
#pragma unroll
      for (int k = 0; k < UNROLL; ++k) {
        const __nv_bfloat16* sp = src + chunk_src<MAP>(rs, 8 * (c0 + lane + 32 * k), lbn, bn_mask);
        v[k] = inplace ? ld_coherent(sp) : ld_stream(sp);
      }
      if (OP == FO_POST_ADD) {
        uint4 w[UNROLL];
#pragma unroll
        for (int k = 0; k < UNROLL; ++k) w[k] = ld_stream(rrow + 8 * (c0 + lane + 32 * k));
#pragma unroll
        for (int k = 0; k < UNROLL; ++k) {
          float x[8], y[8];
          unpack8(v[k], x);
          unpack8(w[k], y);
#pragma unroll
          for (int i = 0; i < 8; ++i) x[i] += y[i];
          v[k] = pack8(x);
        }
      }
#pragma unroll
      for (int k = 0; k < UNROLL; ++k) st_stream(orow + 8 * (c0 + lane + 32 * k), v[k]);
    } else {
      for (int64_t c = c0 + lane; c < chunks; c += 32) {
        const __nv_bfloat16* sp = src + chunk_src<MAP>(rs, 8 * c, lbn, bn_mask);
        uint4 v = inplace ? ld_coherent(sp) : ld_stream(sp);
        if (OP == FO_POST_ADD) {
          float x[8], y[8];
          unpack8(v, x);
          unpack8(ld_stream(rrow + 8 * c), y);
#pragma unroll
          for (int i = 0; i < 8; ++i) x[i] += y[i];
          v = pack8(x);
        }
        st_stream(orow + 8 * c, v);
      }
    }
  }
}

// Residual add + RMSNorm: one THREADS-thread block per row, the whole row held
// in registers (MAXC chunks of 8 per thread, N <= 8*THREADS*MAXC), single pass
// over HBM: read x (through the map) and residual once, write out once.
// Rows of up to 8192 columns (<= 4 chunks per thread) prefetch the block's
// next row (PF below) on a grid of resident blocks that loop over rows:
// 9-16% faster than a block per row without the prefetch
// (profiles/r01_post_reorder_probe.txt); a cluster of blocks per row with a
// DSMEM reduction was slower.
// RES: also write y = x + residual (bf16) back into the residual buffer (the
// residual stream of a pre-norm block); each row's residual is read before
// its own write, by the same thread, so in place is safe.
template <int MAP, int MAXC, int THREADS, bool RES>
__global__ void __launch_bounds__(THREADS) fo_post_rmsnorm_kernel(const PostArgs p, int lbn) {
  constexpr int WARPS = THREADS / 32;
  // rows of up to 4 chunks per thread also prefetch the block's next row while
  // reducing / writing the current one: without it every resident block
  // alternates a load phase and a reduce + store phase in step with the
  // others, leaving HBM idle in between
  constexpr bool PF = MAXC <= 4;
  __shared__ float red[WARPS];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t chunks = p.N >> 3;
  const int bn_mask = p.BN - 1;
  const __nv_bfloat16* src = reinterpret_cast<const __nv_bfloat16*>(p.src);
  __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(p.out);
  const __nv_bfloat16* gam = reinterpret_cast<const __nv_bfloat16*>(p.gamma);
  uint4 xv[MAXC], rv[MAXC];
  auto load_row = [&](int64_t r, uint4* xo, uint4* ro) {
    const RowSrc rs = row_src<MAP>(p, r);
    const __nv_bfloat16* rrow = reinterpret_cast<const __nv_bfloat16*>(p.residual) + r * p.N;
#pragma unroll
    for (int i = 0; i < MAXC; ++i) {
      const int64_t c = tid + THREADS * i;
      if (c < chunks) {
        xo[i] = ld_coherent(src + chunk_src<MAP>(rs, 8 * c, lbn, bn_mask));
        ro[i] = ld_stream(rrow + 8 * c);
      }
    }
  };
  if (PF && blockIdx.x < p.rows) load_row(blockIdx.x, xv, rv);
  for (int64_t r = blockIdx.x; r < p.rows; r += gridDim.x) {
    const __nv_bfloat16* rrow = reinterpret_cast<const __nv_bfloat16*>(p.residual) + r * p.N;
    __nv_bfloat16* orow = out + r * p.N;
    uint4 xn[MAXC], rn[MAXC];
    if (PF) {
      if (r + gridDim.x < p.rows) load_row(r + gridDim.x, xn, rn);
    } else {
      load_row(r, xv, rv);
    }
    // y = x + residual is recomputed from the packed inputs in the second
    // phase (identical fp32 ops) instead of being held: fewer registers, more
    // rows in flight per SM
    float ss = 0.f;
#pragma unroll
    for (int i = 0; i < MAXC; ++i) {
      const int64_t c = tid + THREADS * i;
      if (c < chunks) {
        float x[8], q[8];
        unpack8(xv[i], x);
        unpack8(rv[i], q);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float y = x[k] + q[k];
          ss += y * y;
        }
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (lane == 0) red[warp] = ss;
    __syncthreads();
    float tot = 0.f;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) tot += red[w];
    __syncthreads();  // red[] reused by the next row
    const float rstd = rsqrtf(tot / (float)p.N + p.eps);
#pragma unroll
    for (int i = 0; i < MAXC; ++i) {
      const int64_t c = tid + THREADS * i;
      if (c < chunks) {
        float x[8], q[8], g[8];
        unpack8(xv[i], x);
        unpack8(rv[i], q);
        unpack8(ld_coherent(gam + 8 * c), g);
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] += q[k];
        if (RES) st_stream(const_cast<__nv_bfloat16*>(rrow) + 8 * c, pack8(x));
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = x[k] * rstd * g[k];
        st_stream(orow + 8 * c, pack8(x));
      }
    }
    if (PF) {
#pragma unroll
      for (int i = 0; i < MAXC; ++i) {
        xv[i] = xn[i];
        rv[i] = rn[i];
      }
    }
  }
}

// Residual add + RMSNorm with the rows staged in shared memory by bulk copies
// (cp.async.bulk, the TMA's linear mode): for launches that do not share the
// GPU with the persistent GEMM (the final / sequential / stage post pass; its
// shared memory keeps it off SMs a GEMM CTA holds).  Warp 0 keeps `stages`
// rows per block in flight (x through the map — one copy per BN-wide run, or
// the whole row for identity maps — and the residual row), so the bytes in
// flight per SM are set by shared memory, not by registers: the register
// kernel above holds ~2 rows per block and reaches 0.63-0.72 of the HBM copy
// bandwidth on 4096-8192-column rows (profiles/r02_post_probe.txt).  Each
// thread reads its CPT 16-byte chunks of a row from shared memory once, the
// block reduces the sum of squares, and warp 0 refills the slot for the
// block's row `stages` ahead before the normalised row is written.
namespace bulkcp {
__device__ __forceinline__ uint32_t smem_u32(const void* ptr) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(ptr));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
}  // namespace bulkcp

constexpr int BULK_THREADS = 256;

template <int MAP, int CPT, bool RES>
__global__ void __launch_bounds__(BULK_THREADS) fo_post_rmsnorm_bulk_kernel(const PostArgs p, int lbn, int stages) {
  extern __shared__ __align__(128) uint8_t bsm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int WARPS = BULK_THREADS / 32;
  const int64_t N = p.N;
  const int chunks = (int)(N >> 3);
  const uint32_t row_bytes = (uint32_t)(N * 2);
  uint8_t* slots = bsm;  // [stages][x row | residual row]
  uint64_t* full = reinterpret_cast<uint64_t*>(bsm + (size_t)stages * 2 * row_bytes);
  float* red = reinterpret_cast<float*>(full + stages);  // [2][WARPS], alternating rows
  const __nv_bfloat16* src = reinterpret_cast<const __nv_bfloat16*>(p.src);
  const __nv_bfloat16* res = reinterpret_cast<const __nv_bfloat16*>(p.residual);
  __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(p.out);
  const __nv_bfloat16* gam = reinterpret_cast<const __nv_bfloat16*>(p.gamma);
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) bulkcp::mbar_init(&full[s], 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  const int Nt = (int)(N >> lbn);
  const uint32_t run_bytes = (uint32_t)(p.BN * 2);
  // warp 0: stage row r into slot s (x through the map, the residual row)
  auto issue = [&](int64_t r, int s) {
    uint8_t* xs = slots + (size_t)s * 2 * row_bytes;
    const RowSrc rs = row_src<MAP>(p, r);
    if (lane == 0) bulkcp::mbar_expect_tx(&full[s], 2 * row_bytes);
    __syncwarp();
    if (MAP == POSTMAP_IDENTITY || MAP == POSTMAP_ROWX) {
      if (lane == 0) bulkcp::g2s(xs, src + rs.roff, row_bytes, &full[s]);
    } else {
      for (int jc = lane; jc < Nt; jc += 32)
        bulkcp::g2s(xs + (size_t)jc * run_bytes, src + (int64_t)__ldg(rs.tbl + jc) * rs.tscale + rs.roff, run_bytes,
                    &full[s]);
    }
    if (lane == 1) bulkcp::g2s(xs + row_bytes, res + r * N, row_bytes, &full[s]);
  };
  const int64_t step = gridDim.x;
  if (warp == 0)
    for (int s = 0; s < stages; ++s) {
      const int64_t r = blockIdx.x + s * step;
      if (r < p.rows) issue(r, s);
    }
  uint4 gv[CPT];
#pragma unroll
  for (int i = 0; i < CPT; ++i) {
    const int c = tid + BULK_THREADS * i;
    if (c < chunks) gv[i] = *reinterpret_cast<const uint4*>(gam + 8 * (int64_t)c);
  }
  int s = 0, it = 0;
  uint32_t phase = 0;
  for (int64_t r = blockIdx.x; r < p.rows; r += step, ++it) {
    bulkcp::mbar_wait(&full[s], phase);
    const uint4* xs = reinterpret_cast<const uint4*>(slots + (size_t)s * 2 * row_bytes);
    const uint4* rsd = reinterpret_cast<const uint4*>(slots + (size_t)s * 2 * row_bytes + row_bytes);
    float y[CPT][8];
    float ss = 0.f;
#pragma unroll
    for (int i = 0; i < CPT; ++i) {
      const int c = tid + BULK_THREADS * i;
      if (c < chunks) {
        float q[8];
        unpack8(xs[c], y[i]);
        unpack8(rsd[c], q);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          y[i][k] += q[k];
          ss += y[i][k] * y[i][k];
        }
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    float* rb = red + (it & 1) * WARPS;
    if (lane == 0) rb[warp] = ss;
    __syncthreads();  // every thread's smem reads of slot s are done, the partial sums are in
    if (warp == 0) {
      const int64_t rn = r + (int64_t)stages * step;
      if (rn < p.rows) issue(rn, s);
    }
    float tot = 0.f;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) tot += rb[w];
    const float rstd = rsqrtf(tot / (float)N + p.eps);
    __nv_bfloat16* orow = out + r * N;
#pragma unroll
    for (int i = 0; i < CPT; ++i) {
      const int c = tid + BULK_THREADS * i;
      if (c < chunks) {
        if (RES) st_stream(const_cast<__nv_bfloat16*>(res) + r * N + 8 * c, pack8(y[i]));
        float g[8], o[8];
        unpack8(gv[i], g);
#pragma unroll
        for (int k = 0; k < 8; ++k) o[k] = y[i][k] * rstd * g[k];
        st_stream(orow + 8 * c, pack8(o));
      }
    }
    if (++s == stages) {
      s = 0;
      phase ^= 1;
    }
  }
}

// Fallback for very wide rows (N > 16384): warp per row, two passes (the
// second read hits L2).
template <int MAP, bool RES>
__global__ void __launch_bounds__(256) fo_post_rmsnorm_wide_kernel(const PostArgs p, int lbn) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t chunks = p.N >> 3;
  const int bn_mask = p.BN - 1;
  const __nv_bfloat16* src = reinterpret_cast<const __nv_bfloat16*>(p.src);
  __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(p.out);
  const __nv_bfloat16* gam = reinterpret_cast<const __nv_bfloat16*>(p.gamma);
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < p.rows; r += warps) {
    const RowSrc rs = row_src<MAP>(p, r);
    const __nv_bfloat16* rrow = reinterpret_cast<const __nv_bfloat16*>(p.residual) + r * p.N;
    float ss = 0.f;
    for (int64_t c = lane; c < chunks; c += 32) {
      float x[8], y[8];
      unpack8(ld_coherent(src + chunk_src<MAP>(rs, 8 * c, lbn, bn_mask)), x);
      unpack8(ld_coherent(rrow + 8 * c), y);
#pragma unroll
      for (int i = 0; i < 8; ++i) ss += (x[i] + y[i]) * (x[i] + y[i]);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    const float rstd = rsqrtf(ss / (float)p.N + p.eps);
    for (int64_t c = lane; c < chunks; c += 32) {
      float x[8], y[8], g[8];
      unpack8(ld_coherent(src + chunk_src<MAP>(rs, 8 * c, lbn, bn_mask)), x);
      unpack8(ld_coherent(rrow + 8 * c), y);
      unpack8(ld_coherent(gam + 8 * c), g);
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] += y[i];
      if (RES) st_stream(const_cast<__nv_bfloat16*>(rrow) + 8 * c, pack8(x));
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = x[i] * rstd * g[i];
      st_stream(out + r * p.N + 8 * c, pack8(x));
    }
  }
}

// Per-group post-reorder.  Unit = one warp x 32 chunks (512 B) of the group's
// contiguous received data; reads are fully contiguous, each 16-byte chunk is
// written to its row of the output tile.
template <int MAP, int OP>
__global__ void __launch_bounds__(256) fo_post_group_kernel(const GroupPostArgs p, int lbn) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int cpr = p.BN >> 3;  // chunks per BN-wide row segment
  int64_t c_begin, c_end;
  if (MAP == POSTMAP_A2A) {
    c_begin = p.sub_begin * cpr;
    c_end = p.sub_end * cpr;
  } else {
    c_begin = (int64_t)p.pos_begin * p.R * cpr;
    c_end = (int64_t)p.pos_end * p.R * cpr;
  }
  const __nv_bfloat16* src = reinterpret_cast<const __nv_bfloat16*>(p.src);
  __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(p.out);
  const __nv_bfloat16* res = reinterpret_cast<const __nv_bfloat16*>(p.residual);
  for (int64_t c = c_begin + ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32 + lane; c < c_end;
       c += warps * 32) {
    int64_t dst;
    const int64_t seg = c / cpr;               // BN-wide row segment index in the receive buffer
    const int b = (int)(c - seg * cpr) * 8;
    if (MAP == POSTMAP_A2A) {
      const int32_t d = __ldg(p.recv_dst + seg);
      const int64_t orow = d / p.Nt;
      dst = orow * p.N + (int64_t)(d - orow * p.Nt) * p.BN + b;
    } else {
      const int64_t pos = seg / p.R;
      const int a = (int)(seg - pos * p.R);
      const int t = __ldg(p.order + pos);
      const int ti = t / p.Nt, tj = t - ti * p.Nt;
      dst = ((int64_t)ti * p.R + a) * p.N + (int64_t)tj * p.BN + b;
    }
    uint4 v = ld_stream(src + 8 * c);
    if (OP == FO_POST_ADD) {
      float x[8], y[8];
      unpack8(v, x);
      unpack8(ld_stream(res + dst), y);
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] += y[i];
      v = pack8(x);
    }
    st_stream(out + dst, v);
  }
}

__global__ void fo_timestamp_kernel(unsigned long long* dst) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *dst = t;
}

// The paper's signaling kernel: spin until the group counter
// reaches its target (cyclic comparison, like CU_STREAM_WAIT_VALUE_GEQ), with
// acquire semantics so the following stream work sees the group's data.
__global__ void fo_wait_kernel(const uint32_t* ctr, uint32_t target) {
  if (threadIdx.x == 0) {
    uint32_t v;
    while (true) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
      if ((int32_t)(v - target) >= 0) break;
      __nanosleep(64);
    }
  }
}

__global__ void fo_fill_u16_kernel(uint16_t* dst, int64_t n, uint16_t v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = v;
}

// Host-side per-device caches below are written by whichever thread gets
// there first (the loopback backend issues every rank from its own thread);
// each value is idempotent, so relaxed atomics suffice.
int num_sms() {
  static std::atomic<int> cache[64];  // per device
  int dev = 0;
  cudaGetDevice(&dev);
  int n = cache[dev & 63].load(std::memory_order_relaxed);
  if (!n) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (!n) n = 148;
    cache[dev & 63].store(n, std::memory_order_relaxed);
  }
  return n;
}

// Grid of the prefetching row kernel: the blocks that are resident at once
// (occupancy per SM x SMs, cached per instantiation and device), so every
// block loops over several rows and its next-row prefetch overlaps the
// current row instead of the block retiring after one row.
template <int MAP, int MAXC, int THREADS, bool RES>
int resident_grid(int smem) {
  static std::atomic<int> cache[64][2];  // [device][smem != 0] -> blocks per SM
  int dev = 0;
  cudaGetDevice(&dev);
  int v = cache[dev & 63][smem != 0].load(std::memory_order_relaxed);
  if (!v) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, fo_post_rmsnorm_kernel<MAP, MAXC, THREADS, RES>, THREADS,
                                                      smem) != cudaSuccess || v < 1) {
      cudaGetLastError();
      v = 1;
    }
    cache[dev & 63][smem != 0].store(v, std::memory_order_relaxed);
  }
  return v * num_sms();
}

// The bulk-staged kernel: stages per block from a ~100 KB budget (two blocks
// per SM at 8192 columns), grid = the resident blocks; returns false when it
// does not apply (rows wider than 16384 columns, unaligned buffers).
template <int MAP, bool RES, int CPT>
bool launch_rmsnorm_bulk_cpt(const PostArgs& a, int lbn, cudaStream_t stream) {
  const size_t slot = 4 * (size_t)a.N;
  const int stages = (int)std::max<size_t>(2, std::min<size_t>(4, (100u << 10) / slot));
  const int smem = (int)(stages * slot + stages * 8 + 2 * 8 * sizeof(float));
  auto kern = fo_post_rmsnorm_bulk_kernel<MAP, CPT, RES>;
  static std::atomic<int> attr_dev_mask{0};  // per device bit: the dynamic-smem attribute is set
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr_dev_mask.load(std::memory_order_relaxed) & (1 << (dev & 31)))) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 << 10) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    attr_dev_mask.fetch_or(1 << (dev & 31), std::memory_order_relaxed);
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, BULK_THREADS, smem) != cudaSuccess || per_sm < 1) {
    cudaGetLastError();
    return false;
  }
  const int grid = (int)std::min<int64_t>(a.rows, (int64_t)per_sm * num_sms());
  kern<<<grid, BULK_THREADS, smem, stream>>>(a, lbn, stages);
  return true;
}

template <int MAP, bool RES>
bool launch_rmsnorm_bulk(const PostArgs& a, int lbn, cudaStream_t stream) {
  const int64_t chunks = a.N / 8;
  auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  if (!a.bulk_ok || !al16(a.src) || !al16(a.residual) || !al16(a.gamma) || a.BN < 8) return false;
  // measured (profiles/r02_post_probe.txt): ahead only where many rows per
  // block keep the ring full — 8192^2: 1.00 vs 0.97 of the copy bandwidth on
  // whole rows, 0.79 vs 0.72 through the slot map; at 4096^2 and below the
  // prologue dominates and the register kernel is 5-15% faster
  if (a.rows * a.N * 2 < (int64_t(64) << 20)) return false;
  if (chunks <= BULK_THREADS) return launch_rmsnorm_bulk_cpt<MAP, RES, 1>(a, lbn, stream);
  if (chunks <= 2 * BULK_THREADS) return launch_rmsnorm_bulk_cpt<MAP, RES, 2>(a, lbn, stream);
  if (chunks <= 4 * BULK_THREADS) return launch_rmsnorm_bulk_cpt<MAP, RES, 4>(a, lbn, stream);
  if (chunks <= 8 * BULK_THREADS) return launch_rmsnorm_bulk_cpt<MAP, RES, 8>(a, lbn, stream);
  return false;
}

// Both kernels give each thread the chunks c = tid + 256 i (the register
// kernel's 128-thread configuration only below 129 chunks, where the extra
// warps of the bulk kernel hold none) and sum in the same order, so a per-band
// pass beside the GEMM and a whole-output pass after it agree bit for bit.
template <int MAP, bool RES>
cudaError_t launch_rmsnorm(const PostArgs& a, int lbn, cudaStream_t stream) {
  const int64_t chunks = a.N / 8;
  if (launch_rmsnorm_bulk<MAP, RES>(a, lbn, stream)) return cudaGetLastError();
  const int grid = (int)std::min<int64_t>(a.rows, (int64_t)num_sms() * 16);
  auto pgrid = [&](int resident) { return (int)std::min<int64_t>(a.rows, resident); };
  if (chunks <= 128)
    fo_post_rmsnorm_kernel<MAP, 1, 128, RES>
        <<<pgrid(resident_grid<MAP, 1, 128, RES>(a.smem_pad)), 128, a.smem_pad, stream>>>(a, lbn);
  else if (chunks <= 256)  // 256 threads x 1 chunk: the bulk kernel's chunk -> thread map (same fp32 sum order)
    fo_post_rmsnorm_kernel<MAP, 1, 256, RES>
        <<<pgrid(resident_grid<MAP, 1, 256, RES>(a.smem_pad)), 256, a.smem_pad, stream>>>(a, lbn);
  else if (chunks <= 512)
    fo_post_rmsnorm_kernel<MAP, 2, 256, RES>
        <<<pgrid(resident_grid<MAP, 2, 256, RES>(a.smem_pad)), 256, a.smem_pad, stream>>>(a, lbn);
  else if (chunks <= 1024)
    fo_post_rmsnorm_kernel<MAP, 4, 256, RES>
        <<<pgrid(resident_grid<MAP, 4, 256, RES>(a.smem_pad)), 256, a.smem_pad, stream>>>(a, lbn);
  else if (chunks <= 2048) fo_post_rmsnorm_kernel<MAP, 8, 256, RES><<<grid, 256, a.smem_pad, stream>>>(a, lbn);
  else {
    const int g2 = (int)std::min<int64_t>((a.rows + 7) / 8, (int64_t)num_sms() * 8);
    fo_post_rmsnorm_wide_kernel<MAP, RES><<<g2, 256, a.smem_pad, stream>>>(a, lbn);
  }
  return cudaGetLastError();
}

template <int MAP>
cudaError_t launch_map(const PostArgs& a, int lbn, cudaStream_t stream) {
  const int64_t chunks = a.N / 8;
  if (a.op == FO_POST_ADD_RMSNORM) return launch_rmsnorm<MAP, false>(a, lbn, stream);
  if (a.op == FO_POST_ADD_RMSNORM_RESIDUAL) return launch_rmsnorm<MAP, true>(a, lbn, stream);
  const int64_t units = a.rows * ((chunks + SEG_CHUNKS - 1) / SEG_CHUNKS);
  const int grid = (int)std::min<int64_t>((units + 7) / 8, (int64_t)num_sms() * 16);
  if (a.op == FO_POST_ADD) fo_post_reorder_kernel<MAP, FO_POST_ADD><<<grid, 256, a.smem_pad, stream>>>(a, lbn);
  else fo_post_reorder_kernel<MAP, FO_POST_NONE><<<grid, 256, a.smem_pad, stream>>>(a, lbn);
  return cudaGetLastError();
}

// MoE combine: work unit = (token, 2 KB column segment), one warp; for each of
// the token's k slots the warp gathers the slot's row segment from the
// receive buffer (16-B loads, UNROLL in flight per lane) and accumulates
// w * x in fp32; one bf16 rounding at the end (after the optional residual).
__global__ void __launch_bounds__(256) fo_combine_kernel(const CombineArgs p, int lbn) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t chunks = p.N >> 3;
  const int64_t upr = (chunks + SEG_CHUNKS - 1) / SEG_CHUNKS;
  const int64_t units = p.tokens * upr;
  const int bn_mask = p.BN - 1;
  const __nv_bfloat16* src = reinterpret_cast<const __nv_bfloat16*>(p.src);
  __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(p.out);
  const __nv_bfloat16* res = reinterpret_cast<const __nv_bfloat16*>(p.residual);
  for (int64_t u = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); u < units; u += warps) {
    const int64_t t = u / upr;
    const int64_t c0 = (u - t * upr) * SEG_CHUNKS;
    float acc[UNROLL][8];
#pragma unroll
    for (int k = 0; k < UNROLL; ++k)
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[k][e] = 0.f;
    // the residual's loads go out first and land while the slots are gathered
    uint4 rv[UNROLL];
    if (res) {
#pragma unroll
      for (int k = 0; k < UNROLL; ++k) {
        const int64_t c = c0 + lane + 32 * k;
        if (c < chunks) rv[k] = ld_stream(res + t * p.N + 8 * c);
      }
    }
    for (int i = 0; i < p.topk; ++i) {
      const int64_t r = __ldg(p.idx + t * p.topk + i);
      if (r < 0 || r >= p.a2a_rows) continue;  // dropped slot
      const float wt = __ldg(p.w + t * p.topk + i);
      const int32_t* tbl = p.src_row + r * p.Nt;
      uint4 v[UNROLL];
#pragma unroll
      for (int k = 0; k < UNROLL; ++k) {
        const int64_t c = c0 + lane + 32 * k;
        if (c < chunks) {
          const int64_t col = 8 * c;
          v[k] = ld_stream(src + (int64_t)__ldg(tbl + (col >> lbn)) * p.BN + (col & bn_mask));
        }
      }
#pragma unroll
      for (int k = 0; k < UNROLL; ++k) {
        if (c0 + lane + 32 * k < chunks) {
          float f[8];
          unpack8(v[k], f);
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[k][e] = fmaf(wt, f[e], acc[k][e]);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < UNROLL; ++k) {
      const int64_t c = c0 + lane + 32 * k;
      if (c >= chunks) continue;
      if (res) {
        float f[8];
        unpack8(rv[k], f);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[k][e] += f[e];
      }
      st_stream(out + t * p.N + 8 * c, pack8(acc[k]));
    }
  }
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

constexpr int CMB_SEG_COLS = SEG_CHUNKS * 8;  // columns per work unit (1024)
constexpr int CMB_TBL_REGS = 4;               // table entries per lane: topk x tiles-per-segment <= 128
constexpr int CMB_ASYNC_MAX_BUF = 3;          // more slots (+ residual) per unit: the register kernel

// MoE combine, async-copy pipeline (R31b).  Same work unit, same
// lane -> chunk map and the same fp32 accumulation order as fo_combine_kernel
// (bit-identical results), but the gathers go through cp.async (LDGSTS) into a
// per-warp, two-stage shared-memory buffer [stage][slot (+ residual)][2 KB]:
// while unit u is accumulated from shared memory, unit u+1's k row segments
// (and its residual) are in flight without holding registers, and unit u+2's
// (row, weight) pairs are being loaded.  The slot -> source-row table entries a
// unit needs (topk x tiles-per-segment) are loaded once per unit, one per lane,
// and broadcast with shuffles, so no per-slot chain of dependent loads sits
// on the issue path.  Each lane reads back exactly the chunks it copied, so
// cp.async.wait_group alone orders the copy before the read.
__global__ void __launch_bounds__(256) fo_combine_async_kernel(const CombineArgs p, int lbn, int nbuf) {
  extern __shared__ uint4 cmb_smem[];
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  const int64_t warps = (int64_t)gridDim.x * wpb;
  const int64_t chunks = p.N >> 3;
  const int64_t upr = (chunks + SEG_CHUNKS - 1) / SEG_CHUNKS;
  const int64_t units = p.tokens * upr;
  const int bn_mask = p.BN - 1;
  const int topk = p.topk;
  const int tps = lbn >= 10 ? 1 : (CMB_SEG_COLS >> lbn);  // tile columns per unit
  const int ents = topk * tps;
  const __nv_bfloat16* src = reinterpret_cast<const __nv_bfloat16*>(p.src);
  __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(p.out);
  const __nv_bfloat16* res = reinterpret_cast<const __nv_bfloat16*>(p.residual);
  uint4* buf = cmb_smem + (int64_t)(threadIdx.x >> 5) * 2 * nbuf * SEG_CHUNKS;

  // lane i < topk: slot i's receive row (-1 when dropped) and weight
  auto load_meta = [&](int64_t uu, int& r, float& wt) {
    r = -1;
    wt = 0.f;
    if (uu < units && lane < topk) {
      const int64_t t = uu / upr;
      r = __ldg(p.idx + t * topk + lane);
      wt = __ldg(p.w + t * topk + lane);
      if (r < 0 || r >= p.a2a_rows) r = -1;
    }
  };
  // start unit uu's copies into stage `st` (always commits a group, possibly
  // empty, so every lane's wait_group count stays uniform)
  auto issue = [&](int64_t uu, int r_l, int st) {
    if (uu < units) {
      const int64_t t = uu / upr;
      const int64_t c0 = (uu - t * upr) * SEG_CHUNKS;
      const int64_t jt0 = (8 * c0) >> lbn;  // first tile column of the unit
      int tv[CMB_TBL_REGS];
#pragma unroll
      for (int q = 0; q < CMB_TBL_REGS; ++q) {
        const int e = lane + 32 * q;
        const int slot = e / tps;
        const int rr = __shfl_sync(0xffffffffu, r_l, slot < topk ? slot : 0);
        const int64_t jc = jt0 + (e - slot * tps);
        tv[q] = (e < ents && rr >= 0 && jc < p.Nt) ? __ldg(p.src_row + (int64_t)rr * p.Nt + jc) : 0;
      }
      uint4* sb = buf + st * nbuf * SEG_CHUNKS;
      for (int i = 0; i < topk; ++i) {
        const int rr = __shfl_sync(0xffffffffu, r_l, i);
#pragma unroll
        for (int k = 0; k < UNROLL; ++k) {
          const int64_t c = c0 + lane + 32 * k;
          const int64_t col = 8 * c;
          const int e = i * tps + (int)((col >> lbn) - jt0);
          int tval = 0;
#pragma unroll
          for (int q = 0; q < CMB_TBL_REGS; ++q) {
            const int v = __shfl_sync(0xffffffffu, tv[q], e & 31);
            if (q == (e >> 5)) tval = v;
          }
          if (rr >= 0 && c < chunks)
            cp_async16(sb + i * SEG_CHUNKS + lane + 32 * k, src + (int64_t)tval * p.BN + (col & bn_mask));
        }
      }
      if (res) {
#pragma unroll
        for (int k = 0; k < UNROLL; ++k) {
          const int64_t c = c0 + lane + 32 * k;
          if (c < chunks) cp_async16(sb + topk * SEG_CHUNKS + lane + 32 * k, res + t * p.N + 8 * c);
        }
      }
    }
    cp_async_commit();
  };

  int64_t u = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5);
  int r_cur, r_nxt;
  float w_cur, w_nxt;
  load_meta(u, r_cur, w_cur);
  issue(u, r_cur, 0);
  load_meta(u + warps, r_nxt, w_nxt);
  int st = 0;
  for (; u < units; u += warps) {
    issue(u + warps, r_nxt, st ^ 1);
    int r_n2;
    float w_n2;
    load_meta(u + 2 * warps, r_n2, w_n2);
    cp_async_wait<1>();  // this lane's copies of unit u have landed
    const int64_t t = u / upr;
    const int64_t c0 = (u - t * upr) * SEG_CHUNKS;
    const uint4* sb = buf + st * nbuf * SEG_CHUNKS;
    float acc[UNROLL][8];
#pragma unroll
    for (int k = 0; k < UNROLL; ++k)
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[k][e] = 0.f;
    for (int i = 0; i < topk; ++i) {
      const int rr = __shfl_sync(0xffffffffu, r_cur, i);
      const float wt = __shfl_sync(0xffffffffu, w_cur, i);
      if (rr < 0) continue;  // dropped slot
#pragma unroll
      for (int k = 0; k < UNROLL; ++k) {
        if (c0 + lane + 32 * k < chunks) {
          float f[8];
          unpack8(sb[i * SEG_CHUNKS + lane + 32 * k], f);
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[k][e] = fmaf(wt, f[e], acc[k][e]);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < UNROLL; ++k) {
      const int64_t c = c0 + lane + 32 * k;
      if (c >= chunks) continue;
      if (res) {
        float f[8];
        unpack8(sb[topk * SEG_CHUNKS + lane + 32 * k], f);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[k][e] += f[e];
      }
      st_stream(out + t * p.N + 8 * c, pack8(acc[k]));
    }
    r_cur = r_nxt;
    w_cur = w_nxt;
    r_nxt = r_n2;
    w_nxt = w_n2;
    st ^= 1;
  }
  cp_async_wait<0>();
}

}  // namespace

cudaError_t launch_combine(const CombineArgs& a, cudaStream_t stream) {
  if (a.tokens <= 0) return cudaSuccess;
  if (a.N % 8 || (a.BN & (a.BN - 1)) || a.topk < 1) return cudaErrorInvalidValue;
  int lbn = 0;
  while ((1 << lbn) < a.BN) ++lbn;
  const int64_t units = a.tokens * ((a.N / 8 + SEG_CHUNKS - 1) / SEG_CHUNKS);
  const int tps = lbn >= 10 ? 1 : (CMB_SEG_COLS >> lbn);
  const int nbuf = a.topk + (a.residual ? 1 : 0);
  const int per_warp = 2 * nbuf * SEG_CHUNKS * 16;  // two stages of (topk [+1]) 2 KB segments
  // the async pipeline needs 16 warps per SM (two 8-warp blocks) to beat the
  // register kernel, i.e. at most three 2 KB buffers per stage: top-1/top-2
  // (+ residual) (profiles/r02_combine_probe.txt)
  if (nbuf <= CMB_ASYNC_MAX_BUF && a.topk * tps <= 32 * CMB_TBL_REGS) {
    const int wpb = std::max(1, std::min(8, (112 * 1024) / per_warp));
    const int smem = wpb * per_warp;
    static std::atomic<int> attr_dev_mask{0};  // per device bit: the dynamic-smem attribute is set (112 KB cap)
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (!(attr_dev_mask.load(std::memory_order_relaxed) & (1 << (dev & 31)))) {
      e = cudaFuncSetAttribute(fo_combine_async_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024);
      if (e != cudaSuccess) return e;
      attr_dev_mask.fetch_or(1 << (dev & 31), std::memory_order_relaxed);
    }
    static std::atomic<int> occ_cache[32][CMB_ASYNC_MAX_BUF + 1];  // resident blocks per SM by (device, nbuf)
    int occ = occ_cache[dev & 31][nbuf].load(std::memory_order_relaxed);
    if (occ == 0) {
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fo_combine_async_kernel, 32 * wpb, smem);
      if (e != cudaSuccess) return e;
      occ_cache[dev & 31][nbuf].store(occ, std::memory_order_relaxed);
    }
    const int64_t blocks = (units + wpb - 1) / wpb;
    const int grid = (int)std::min<int64_t>(blocks, (int64_t)num_sms() * std::max(1, occ));
    fo_combine_async_kernel<<<grid, 32 * wpb, smem, stream>>>(a, lbn, nbuf);
  } else {
    const int grid = (int)std::min<int64_t>((units + 7) / 8, (int64_t)num_sms() * 16);
    fo_combine_kernel<<<grid, 256, 0, stream>>>(a, lbn);
  }
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_group_post(const GroupPostArgs& a, cudaStream_t stream) {
  if (a.BN & (a.BN - 1)) return cudaErrorInvalidValue;
  int lbn = 0;
  while ((1 << lbn) < a.BN) ++lbn;
  const int64_t cpr = a.BN / 8;
  const int64_t chunks = (a.map == POSTMAP_A2A) ? (a.sub_end - a.sub_begin) * cpr
                                                 : (int64_t)(a.pos_end - a.pos_begin) * a.R * cpr;
  if (chunks <= 0) return cudaSuccess;
  const int cap = a.grid_cap > 0 ? a.grid_cap : num_sms() * 4;
  const int grid = (int)std::min<int64_t>((chunks + 255) / 256, cap);
  switch (a.map * 4 + a.op) {
    case POSTMAP_SLOT * 4 + FO_POST_NONE: fo_post_group_kernel<POSTMAP_SLOT, FO_POST_NONE><<<grid, 256, a.smem_pad, stream>>>(a, lbn); break;
    case POSTMAP_SLOT * 4 + FO_POST_ADD: fo_post_group_kernel<POSTMAP_SLOT, FO_POST_ADD><<<grid, 256, a.smem_pad, stream>>>(a, lbn); break;
    case POSTMAP_RS * 4 + FO_POST_NONE: fo_post_group_kernel<POSTMAP_RS, FO_POST_NONE><<<grid, 256, a.smem_pad, stream>>>(a, lbn); break;
    case POSTMAP_RS * 4 + FO_POST_ADD: fo_post_group_kernel<POSTMAP_RS, FO_POST_ADD><<<grid, 256, a.smem_pad, stream>>>(a, lbn); break;
    case POSTMAP_A2A * 4 + FO_POST_NONE: fo_post_group_kernel<POSTMAP_A2A, FO_POST_NONE><<<grid, 256, a.smem_pad, stream>>>(a, lbn); break;
    case POSTMAP_A2A * 4 + FO_POST_ADD: fo_post_group_kernel<POSTMAP_A2A, FO_POST_ADD><<<grid, 256, a.smem_pad, stream>>>(a, lbn); break;
    default: return cudaErrorInvalidValue;
  }
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_timestamp(unsigned long long* dst, cudaStream_t stream) {
  fo_timestamp_kernel<<<1, 1, 0, stream>>>(dst);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_wait(const uint32_t* counter, uint32_t target, cudaStream_t stream) {
  fo_wait_kernel<<<1, 32, 0, stream>>>(counter, target);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_fill_u16(void* dst, int64_t count, uint16_t value, cudaStream_t stream) {
  if (count <= 0) return cudaSuccess;
  const int grid = (int)std::min<int64_t>((count + 255) / 256, (int64_t)num_sms() * 8);
  fo_fill_u16_kernel<<<grid, 256, 0, stream>>>(reinterpret_cast<uint16_t*>(dst), count, value);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_post(const PostArgs& a, cudaStream_t stream) {
  if (a.rows <= 0) return cudaSuccess;
  if (a.N % 8 || (a.BN & (a.BN - 1))) return cudaErrorInvalidValue;
  int lbn = 0;
  while ((1 << lbn) < a.BN) ++lbn;
  cudaError_t e;
  switch (a.map) {
    case POSTMAP_SLOT: e = launch_map<POSTMAP_SLOT>(a, lbn, stream); break;
    case POSTMAP_RS: e = launch_map<POSTMAP_RS>(a, lbn, stream); break;
    case POSTMAP_A2A: e = launch_map<POSTMAP_A2A>(a, lbn, stream); break;
    case POSTMAP_ROWX: e = launch_map<POSTMAP_ROWX>(a, lbn, stream); break;
    default: e = launch_map<POSTMAP_IDENTITY>(a, lbn, stream); break;
  }
  count_launch();
  return e;
}

}  // namespace fo
