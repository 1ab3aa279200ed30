// Llama block glue for cooperative execution: RMSNorm, rotary embedding,
// SiLU-gated product.  Memory-bound; 16-byte vector accesses, fp32 math,
// one rounding to bf16 per output.  The GEMMs live in gemm_tcgen05.cu.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/blitz.h"
#include "common.cuh"

namespace bz {
namespace llama {

__device__ __forceinline__ float warp_sum(float v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// y[r] = x[r] * rsqrt(mean(x[r]^2) + eps) * w ; one CTA per row, d % 8 == 0
__global__ void __launch_bounds__(256) k_rmsnorm(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ w,
                                                 __nv_bfloat16* __restrict__ y, int d, int ldx, int ldy, float eps) {
  __shared__ float part[8];
  pdl_trigger();
  pdl_wait();
  const int row = blockIdx.x;
  const uint4* xr = reinterpret_cast<const uint4*>(x + static_cast<int64_t>(row) * ldx);
  const uint4* wr = reinterpret_cast<const uint4*>(w);
  uint4* yr = reinterpret_cast<uint4*>(y + static_cast<int64_t>(row) * ldy);
  const int nv = d / 8;
  float ss = 0.f;
  for (int i = threadIdx.x; i < nv; i += blockDim.x) {
    uint4 v = xr[i];
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float2 f = __bfloat1622float2(h[j]);
      ss += f.x * f.x + f.y * f.y;
    }
  }
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? part[threadIdx.x] : 0.f;
    v = warp_sum(v);
    if (threadIdx.x == 0) part[0] = rsqrtf(v / d + eps);
  }
  __syncthreads();
  const float inv = part[0];
  for (int i = threadIdx.x; i < nv; i += blockDim.x) {
    uint4 v = xr[i], g = wr[i], o;
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
    const __nv_bfloat162* gw = reinterpret_cast<const __nv_bfloat162*>(&g);
    __nv_bfloat162* out = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float2 f = __bfloat1622float2(h[j]);
      float2 s = __bfloat1622float2(gw[j]);
      out[j] = __floats2bfloat162_rn(f.x * inv * s.x, f.y * inv * s.y);
    }
    yr[i] = o;
  }
}

// In-place rotary embedding (rotate-half convention) on the q and k heads of a
// fused qkv row: [q heads | k heads | v heads], head_dim hd.
__global__ void k_rope(__nv_bfloat16* qkv, const int32_t* __restrict__ pos, int n_rot_heads, int hd, int ld,
                       float log2_theta) {
  pdl_trigger();
  pdl_wait();
  const int row = blockIdx.x;
  const int half = hd / 2;
  const float p = static_cast<float>(pos[row]);
  __nv_bfloat16* base = qkv + static_cast<int64_t>(row) * ld;
  for (int idx = threadIdx.x; idx < n_rot_heads * half; idx += blockDim.x) {
    const int h = idx / half, i = idx % half;
    // inv_freq_i = theta^(-2i/hd)
    const float inv_freq = exp2f(-log2_theta * (2.0f * i) / hd);
    float sn, cs;
    sincosf(p * inv_freq, &sn, &cs);
    __nv_bfloat16* hp = base + h * hd;
    const float a = __bfloat162float(hp[i]);
    const float b = __bfloat162float(hp[i + half]);
    hp[i] = __float2bfloat16_rn(a * cs - b * sn);
    hp[i + half] = __float2bfloat16_rn(b * cs + a * sn);
  }
}

// act[r, j] = silu(gu[r, j]) * gu[r, ffn + j]
__global__ void k_silu_mul(const __nv_bfloat16* __restrict__ gu, __nv_bfloat16* __restrict__ act, int ffn, int ldg,
                           int lda) {
  pdl_trigger();
  pdl_wait();
  const int row = blockIdx.y;
  const __nv_bfloat162* g = reinterpret_cast<const __nv_bfloat162*>(gu + static_cast<int64_t>(row) * ldg);
  const __nv_bfloat162* u = reinterpret_cast<const __nv_bfloat162*>(gu + static_cast<int64_t>(row) * ldg + ffn);
  __nv_bfloat162* o = reinterpret_cast<__nv_bfloat162*>(act + static_cast<int64_t>(row) * lda);
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < ffn / 2; j += gridDim.x * blockDim.x) {
    float2 a = __bfloat1622float2(g[j]);
    float2 b = __bfloat1622float2(u[j]);
    const float sa = a.x / (1.f + __expf(-a.x));
    const float sb = a.y / (1.f + __expf(-a.y));
    o[j] = __floats2bfloat162_rn(sa * b.x, sb * b.y);
  }
}

}  // namespace llama
}  // namespace bz

using namespace bz;

extern "C" int bz_rmsnorm(const void* x, const void* w, void* y, int rows, int d, int ldx, int ldy, float eps,
                          void* stream) {
  if (!x || !w || !y || rows < 0 || d % 8 || ldx % 8 || ldy % 8) return bz_fail(BZ_EINVAL, "rmsnorm: bad args");
  if (rows == 0) return BZ_OK;
  cudaError_t e = launch_pdl(PDL_GLUE, llama::k_rmsnorm, dim3(rows), dim3(256), 0, static_cast<cudaStream_t>(stream),
                             static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(w),
                             static_cast<__nv_bfloat16*>(y), d, ldx, ldy, eps);
  if (e != cudaSuccess) return bz_fail_cuda(e, "bz_rmsnorm");
  return bz_check_launch("bz_rmsnorm");
}

extern "C" int bz_rope(void* qkv, const int32_t* positions, int rows, int n_rot_heads, int head_dim, int ld,
                       float theta, void* stream) {
  if (!qkv || !positions || head_dim % 2 || rows < 0) return bz_fail(BZ_EINVAL, "rope: bad args");
  if (rows == 0) return BZ_OK;
  cudaError_t e = launch_pdl(PDL_GLUE, llama::k_rope, dim3(rows), dim3(256), 0, static_cast<cudaStream_t>(stream),
                             static_cast<__nv_bfloat16*>(qkv), positions, n_rot_heads, head_dim, ld, log2f(theta));
  if (e != cudaSuccess) return bz_fail_cuda(e, "bz_rope");
  return bz_check_launch("bz_rope");
}

extern "C" int bz_silu_mul(const void* gu, void* act, int rows, int ffn, int ldg, int lda, void* stream) {
  if (!gu || !act || ffn % 2 || rows < 0) return bz_fail(BZ_EINVAL, "silu_mul: bad args");
  if (rows == 0) return BZ_OK;
  dim3 grid((ffn / 2 + 255) / 256, rows);
  cudaError_t e = launch_pdl(PDL_GLUE, llama::k_silu_mul, grid, dim3(256), 0, static_cast<cudaStream_t>(stream),
                             static_cast<const __nv_bfloat16*>(gu), static_cast<__nv_bfloat16*>(act), ffn, ldg, lda);
  if (e != cudaSuccess) return bz_fail_cuda(e, "bz_silu_mul");
  return bz_check_launch("bz_silu_mul");
}

const void* bz::module_anchor_llama() { return reinterpret_cast<const void*>(llama::k_rmsnorm); }
