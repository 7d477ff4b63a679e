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
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "../../../include/flashoverlap.h"
#include "../kernels.h"

namespace fo {
namespace {

__device__ __forceinline__ int64_t src_offset(const PostArgs& p, int64_t r, int64_t col) {
  const int jc = (int)(col / p.BN), b = (int)(col - (int64_t)jc * p.BN);
  switch (p.map) {
    case POSTMAP_IDENTITY:
      return r * p.N + col;
    case POSTMAP_SLOT:
      return ((int64_t)p.pos_of_tile[(r / p.BM) * p.Nt + jc] * p.BM + r % p.BM) * p.BN + b;
    case POSTMAP_RS:
      return ((int64_t)p.pos_of_tile[(r / p.h) * p.Nt + jc] * p.h + r % p.h) * p.BN + b;
    default:
      return (int64_t)p.src_row[r * p.Nt + jc] * p.BN + b;
  }
}

__device__ __forceinline__ uint4 ldg16(const void* ptr) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(ptr));
  return v;
}

__device__ __forceinline__ uint4 ldg16_coherent(const void* ptr) {
  return *reinterpret_cast<const uint4*>(ptr);
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

template <int OP>
__global__ void __launch_bounds__(256) fo_post_reorder_kernel(const PostArgs p) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t chunks = p.N / 8;
  const char* src = reinterpret_cast<const char*>(p.src);
  char* out = reinterpret_cast<char*>(p.out);
  const char* res = reinterpret_cast<const char*>(p.residual);
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < p.rows; r += warps) {
    if (OP == FO_POST_ADD_RMSNORM) {
      // pass 1: sum of squares of y = x + residual (fp32)
      float ss = 0.f;
      for (int64_t c = lane; c < chunks; c += 32) {
        float x[8], y[8];
        unpack8(ldg16_coherent(src + 2 * src_offset(p, r, 8 * c)), x);
        unpack8(ldg16(res + 2 * (r * p.N + 8 * c)), y);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float t = x[i] + y[i];
          ss += t * t;
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      const float rstd = rsqrtf(ss / (float)p.N + p.eps);
      const char* gam = reinterpret_cast<const char*>(p.gamma);
      // pass 2 (re-read hits L2): out = y * rstd * gamma
      for (int64_t c = lane; c < chunks; c += 32) {
        float x[8], y[8], g[8];
        unpack8(ldg16_coherent(src + 2 * src_offset(p, r, 8 * c)), x);
        unpack8(ldg16(res + 2 * (r * p.N + 8 * c)), y);
        unpack8(ldg16(gam + 2 * (8 * c)), g);
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = (x[i] + y[i]) * rstd * g[i];
        *reinterpret_cast<uint4*>(out + 2 * (r * p.N + 8 * c)) = pack8(x);
      }
    } else {
#pragma unroll 4
      for (int64_t c = lane; c < chunks; c += 32) {
        const char* sp = src + 2 * src_offset(p, r, 8 * c);
        uint4 v = (p.src == p.out) ? ldg16_coherent(sp) : ldg16(sp);
        if (OP == FO_POST_ADD) {
          float x[8], y[8];
          unpack8(v, x);
          unpack8(ldg16(res + 2 * (r * p.N + 8 * c)), y);
#pragma unroll
          for (int i = 0; i < 8; ++i) x[i] += y[i];
          v = pack8(x);
        }
        *reinterpret_cast<uint4*>(out + 2 * (r * p.N + 8 * c)) = v;
      }
    }
  }
}

int g_num_sms = 0;

}  // namespace

cudaError_t launch_post(const PostArgs& a, cudaStream_t stream) {
  if (a.rows <= 0) return cudaSuccess;
  if (a.N % 8) return cudaErrorInvalidValue;
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (!g_num_sms) g_num_sms = 148;
  }
  const int64_t blocks_needed = (a.rows + 7) / 8;  // 8 warps (rows) per block
  const int grid = (int)std::min<int64_t>(blocks_needed, (int64_t)g_num_sms * 8);
  switch (a.op) {
    case FO_POST_ADD: fo_post_reorder_kernel<FO_POST_ADD><<<grid, 256, 0, stream>>>(a); break;
    case FO_POST_ADD_RMSNORM: fo_post_reorder_kernel<FO_POST_ADD_RMSNORM><<<grid, 256, 0, stream>>>(a); break;
    default: fo_post_reorder_kernel<FO_POST_NONE><<<grid, 256, 0, stream>>>(a); break;
  }
  count_launch();
  return cudaGetLastError();
}

}  // namespace fo
