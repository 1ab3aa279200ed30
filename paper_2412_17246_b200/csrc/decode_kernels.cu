// KV-cache decode for the cooperative executor's decode steps (and for a
// prefill instance flipped to decode, livescale.py:512-544).
//
// Both kernels read the decode position from DEVICE memory, so one CUDA graph
// of a whole decode step replays for every position (no host work per token):
//
//   bz_rope_append      rotate q in place; rotate k and write k, v of the
//                       newest token into the cache at position *pos
//   bz_decode_attention softmax(q K[0..*pos]^T / sqrt(hd)) V, split over the
//                       context in chunk-token pieces (flash-decoding), then
//                       one combine pass; GQA groups share the K/V reads.
//
// Cache layout: [rows, n_kv, s_max, hd] bf16 (row = sequence), so one
// (sequence, kv head) is a contiguous [s_max, hd] panel.  HBM-bound: every
// cached K/V byte of the attended prefix is read once per step.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>
#include <stdlib.h>

#include "../../include/blitz.h"
#include "common.cuh"

namespace bz {
namespace decode {

constexpr int CHUNK = 256;      // max context tokens per partial CTA (64..256, see chunk_for)
constexpr int THREADS = 128;
constexpr int MAX_SPLITS = 64;  // context chunks the combine pass stages

__device__ __forceinline__ float4 lds4(const float* p) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(smem_u32(p)));
  return v;
}

// same rotation as llama_kernels.cu k_rope (rotate-half, theta^(-2i/hd)), so a
// decoded token's q/k match what the prefill path computes at that position
__device__ __forceinline__ void rotate_pair(float a, float b, float p, int i, int hd, float log2_theta, float& ra,
                                            float& rb) {
  const float inv_freq = exp2f(-log2_theta * (2.0f * i) / hd);
  float sn, cs;
  sincosf(p * inv_freq, &sn, &cs);
  ra = a * cs - b * sn;
  rb = b * cs + a * sn;
}

// grid (rows, n_heads + n_kv), hd/2 threads: block (r, h < n_heads) rotates q
// head h in place; block (r, n_heads + g) rotates k head g into the cache and
// copies v head g.
__global__ void k_rope_append(__nv_bfloat16* qkv, int ld, int n_heads, int n_kv, int hd, float log2_theta,
                              __nv_bfloat16* kc, __nv_bfloat16* vc, int64_t s_max, const int32_t* __restrict__ pos,
                              int pos_stride) {
  pdl_wait();
  const int row = blockIdx.x, head = blockIdx.y, i = threadIdx.x;
  const int half = hd / 2;
  if (i >= half) return;
  const int p = pos[row * pos_stride];   // one position for the batch (stride 0) or one per row
  if (p < 0 || p >= s_max) {  // full cache: never write past the panel (the host raises first)
    pdl_trigger();
    return;
  }
  const float pf = static_cast<float>(p);
  __nv_bfloat16* base = qkv + static_cast<int64_t>(row) * ld;
  float ra, rb;
  if (head < n_heads) {
    __nv_bfloat16* hp = base + head * hd;
    rotate_pair(__bfloat162float(hp[i]), __bfloat162float(hp[i + half]), pf, i, hd, log2_theta, ra, rb);
    hp[i] = __float2bfloat16_rn(ra);
    hp[i + half] = __float2bfloat16_rn(rb);
    pdl_trigger();
    return;
  }
  const int g = head - n_heads;
  const __nv_bfloat16* kp = base + (n_heads + g) * hd;
  const __nv_bfloat16* vp = base + (n_heads + n_kv + g) * hd;
  const int64_t off = ((static_cast<int64_t>(row) * n_kv + g) * s_max + p) * hd;
  rotate_pair(__bfloat162float(kp[i]), __bfloat162float(kp[i + half]), pf, i, hd, log2_theta, ra, rb);
  kc[off + i] = __float2bfloat16_rn(ra);
  kc[off + i + half] = __float2bfloat16_rn(rb);
  vc[off + i] = vp[i];
  vc[off + i + half] = vp[i + half];
  pdl_trigger();
}

// One CTA = (sequence, kv head, context chunk).  Writes, for each of the G query
// heads of the group, the chunk's max m, sum l and unnormalised o[HD].  The
// score pass reads one K row per thread (q re-read from shared memory as
// float4s); the PV pass reads 8 columns of a V row per thread (HD/8 threads
// cover a row, THREADS/(HD/8) rows at a time).
template <int HD, int G>
__global__ void __launch_bounds__(THREADS) k_decode_partial(const __nv_bfloat16* __restrict__ q, int ldq,
                                                            const __nv_bfloat16* __restrict__ kc,
                                                            const __nv_bfloat16* __restrict__ vc, int n_heads,
                                                            int n_kv, int64_t s_max, const int32_t* __restrict__ pos,
                                                            int pos_stride, float* __restrict__ ws, int nsplit,
                                                            int chunk, float scale) {
  constexpr int VEC = HD / 8;            // uint4 per row
  constexpr int LANES = THREADS / VEC;   // rows per PV sweep
  constexpr int KCH = G >= 4 ? 4 : VEC;  // K-row uint4s held at once (register budget)
  constexpr int PV_UNROLL = G >= 4 ? 1 : 4;
  __shared__ __align__(16) float qs[G][HD];
  __shared__ float sc[G][CHUNK];
  __shared__ float red[LANES][G][HD];
  __shared__ float stat_m[G], stat_l[G];

  pdl_wait();
  const int split = blockIdx.x;
  const int bg = blockIdx.y;
  const int b = bg / n_kv, g = bg % n_kv;
  // attended prefix of this sequence: one position for the batch or one per row; never past the panel
  const int len = static_cast<int>(tmin<int64_t>(static_cast<int64_t>(pos[b * pos_stride]) + 1, s_max));
  const int c0 = split * chunk;
  const int n = min(chunk, len - c0);
  const int tid = threadIdx.x;
  const int64_t stride = HD + 2;
  float* out0 = ws + ((static_cast<int64_t>(b) * n_heads + g * G) * nsplit + split) * stride;

  if (n <= 0) {  // chunk beyond the attended prefix (graph-replayed grid covers s_max)
    pdl_trigger();
    if (tid < G) {
      float* o = out0 + static_cast<int64_t>(tid) * nsplit * stride;
      o[HD] = -CUDART_INF_F;
      o[HD + 1] = 0.f;
    }
    return;
  }
  for (int idx = tid; idx < G * HD; idx += THREADS) {
    const int j = idx / HD, d = idx % HD;
    qs[j][d] = __bfloat162float(q[static_cast<int64_t>(b) * ldq + (g * G + j) * HD + d]) * scale;
  }
  __syncthreads();

  const int64_t panel = (static_cast<int64_t>(b) * n_kv + g) * s_max + c0;
  const uint4* kbase = reinterpret_cast<const uint4*>(kc + panel * HD);
  const uint4* vbase = reinterpret_cast<const uint4*>(vc + panel * HD);
  for (int t = tid; t < n; t += THREADS) {
    float acc[G];
#pragma unroll
    for (int j = 0; j < G; ++j) acc[j] = 0.f;
#pragma unroll
    for (int v0 = 0; v0 < VEC; v0 += KCH) {
      uint4 row[KCH];
#pragma unroll
      for (int v = 0; v < KCH; ++v) row[v] = kbase[static_cast<int64_t>(t) * VEC + v0 + v];
#pragma unroll
      for (int v = 0; v < KCH; ++v) {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&row[v]);
        float f[8];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 x = __bfloat1622float2(h[e]);
          f[2 * e] = x.x;
          f[2 * e + 1] = x.y;
        }
        const int d = (v0 + v) * 8;
#pragma unroll
        for (int j = 0; j < G; ++j) {
          // re-read q from shared memory per row (volatile: not hoisted into G*HD registers)
          const float4 a = lds4(&qs[j][d]), c = lds4(&qs[j][d + 4]);
          acc[j] += f[0] * a.x + f[1] * a.y + f[2] * a.z + f[3] * a.w + f[4] * c.x + f[5] * c.y + f[6] * c.z +
                    f[7] * c.w;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < G; ++j) sc[j][t] = acc[j];
  }
  __syncthreads();

  // per head: max, exp, sum (warp w handles heads w, w + 4, ...)
  const int warp = tid >> 5, lane = tid & 31;
  for (int j = warp; j < G; j += THREADS / 32) {
    float m = -CUDART_INF_F;
    for (int t = lane; t < n; t += 32) m = fmaxf(m, sc[j][t]);
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float l = 0.f;
    for (int t = lane; t < n; t += 32) {
      const float e = __expf(sc[j][t] - m);
      sc[j][t] = e;
      l += e;
    }
    for (int o = 16; o; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
    if (lane == 0) {
      stat_m[j] = m;
      stat_l[j] = l;
    }
  }
  __syncthreads();

  const int cv = tid % VEC, tl = tid / VEC;
  float acc[G][8];
#pragma unroll
  for (int j = 0; j < G; ++j)
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[j][e] = 0.f;
#pragma unroll PV_UNROLL
  for (int t = tl; t < n; t += LANES) {
    const uint4 x = vbase[static_cast<int64_t>(t) * VEC + cv];
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&x);
    float f[8];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 v2 = __bfloat1622float2(h[e]);
      f[2 * e] = v2.x;
      f[2 * e + 1] = v2.y;
    }
#pragma unroll
    for (int j = 0; j < G; ++j) {
      const float p = sc[j][t];
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[j][e] += p * f[e];
    }
  }
#pragma unroll
  for (int j = 0; j < G; ++j)
#pragma unroll
    for (int e = 0; e < 8; ++e) red[tl][j][cv * 8 + e] = acc[j][e];
  pdl_trigger();  // K/V streamed: the combine may launch
  __syncthreads();
  for (int idx = tid; idx < G * HD; idx += THREADS) {
    const int j = idx / HD, d = idx % HD;
    float s = 0.f;
#pragma unroll
    for (int r = 0; r < LANES; ++r) s += red[r][j][d];
    float* o = out0 + static_cast<int64_t>(j) * nsplit * stride;
    o[d] = s;
    if (d == 0) {
      o[HD] = stat_m[j];
      o[HD + 1] = stat_l[j];
    }
  }
}

// out[b, h*HD + d] = sum_s w_s o_s[d] / sum_s w_s l_s,  w_s = exp(m_s - max m)
// (the split weights are staged in shared memory once, then every thread's
// column loop issues independent loads)
template <int HD>
__global__ void k_decode_combine(const float* __restrict__ ws, int nsplit, __nv_bfloat16* __restrict__ out, int ldo,
                                 int n_heads) {
  __shared__ float wgt[MAX_SPLITS];
  __shared__ float inv_den;
  pdl_trigger();
  pdl_wait();
  const int bh = blockIdx.x;
  const int b = bh / n_heads, h = bh % n_heads;
  const int64_t stride = HD + 2;
  const float* base = ws + static_cast<int64_t>(bh) * nsplit * stride;
  if (threadIdx.x < 32) {
    float m = -CUDART_INF_F;
    for (int s = threadIdx.x; s < nsplit; s += 32)
      if (base[s * stride + HD + 1] > 0.f) m = fmaxf(m, base[s * stride + HD]);
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float den = 0.f;
    for (int s = threadIdx.x; s < nsplit; s += 32) {
      const float l = base[s * stride + HD + 1];
      const float w = l > 0.f ? __expf(base[s * stride + HD] - m) : 0.f;
      wgt[s] = w;
      den += w * l;
    }
    for (int o = 16; o; o >>= 1) den += __shfl_xor_sync(0xffffffffu, den, o);
    if (threadIdx.x == 0) inv_den = 1.f / den;
  }
  __syncthreads();
  for (int d = threadIdx.x; d < HD; d += blockDim.x) {
    float num = 0.f;
#pragma unroll 8
    for (int s = 0; s < nsplit; ++s) {
      const float w = wgt[s];
      num += w != 0.f ? w * base[s * stride + d] : 0.f;  // empty chunks never wrote o
    }
    out[static_cast<int64_t>(b) * ldo + h * HD + d] = __float2bfloat16_rn(num * inv_den);
  }
}

template <int HD, int G>
static cudaError_t launch_partial(dim3 grid, cudaStream_t s, const __nv_bfloat16* q, int ldq,
                                  const __nv_bfloat16* kc, const __nv_bfloat16* vc, int n_heads, int n_kv,
                                  int64_t s_max, const int32_t* pos, int pos_stride, float* ws, int nsplit, int chunk,
                                  float scale) {
  return launch_pdl(PDL_ATTN, k_decode_partial<HD, G>, grid, dim3(THREADS), 0, s, q, ldq, kc, vc, n_heads, n_kv, s_max, pos,
                    pos_stride, ws, nsplit, chunk, scale);
}

template <int HD>
static int attention(int group, int rows, dim3 grid, cudaStream_t s, const __nv_bfloat16* q, int ldq,
                     const __nv_bfloat16* kc, const __nv_bfloat16* vc, int n_heads, int n_kv, int64_t s_max,
                     const int32_t* pos, int pos_stride, float* ws, int nsplit, int chunk, float scale,
                     __nv_bfloat16* out, int ldo) {
  cudaError_t e;
  switch (group) {
    case 1:
      e = launch_partial<HD, 1>(grid, s, q, ldq, kc, vc, n_heads, n_kv, s_max, pos, pos_stride, ws, nsplit, chunk,
                                  scale);
      break;
    case 2:
      e = launch_partial<HD, 2>(grid, s, q, ldq, kc, vc, n_heads, n_kv, s_max, pos, pos_stride, ws, nsplit, chunk,
                                  scale);
      break;
    case 4:
      e = launch_partial<HD, 4>(grid, s, q, ldq, kc, vc, n_heads, n_kv, s_max, pos, pos_stride, ws, nsplit, chunk,
                                  scale);
      break;
    case 8:
      e = launch_partial<HD, 8>(grid, s, q, ldq, kc, vc, n_heads, n_kv, s_max, pos, pos_stride, ws, nsplit, chunk,
                                  scale);
      break;
    default:
      return bz_fail(BZ_EINVAL, "decode_attention: heads per kv head must be 1, 2, 4 or 8");
  }
  if (e != cudaSuccess) return bz_fail_cuda(e, "bz_decode_attention (partial)");
  e = launch_pdl(PDL_ATTN, k_decode_combine<HD>, dim3(rows * n_heads), dim3(HD), 0, s, ws, nsplit, out, ldo, n_heads);
  if (e != cudaSuccess) return bz_fail_cuda(e, "bz_decode_attention (combine)");
  return bz_check_launch("bz_decode_attention");
}

// context tokens per CTA: 128 (256 only when 64 chunks of 128 cannot hold s_max), shrunk
// to 64 while the grid is under four waves of the 148 SMs.  Measured on 7B blocks, KV
// 1024 (scripts/decode_breakdown.py, us per block): batch 1 chunk 64/128/256 = 96.4 /
// 97.6 / 104.1, batch 4 109.4 / 106.3 / 112.0, batch 16 154.2 / 151.9 / 158.3.
static int chunk_for(int rows, int n_kv, int64_t s_max) {
  if (const char* e = getenv("BZ_DECODE_CHUNK")) {  // A/B measurements: 64, 128 or 256
    const int c = atoi(e);
    if (c == 64 || c == 128 || c == 256) return c;
  }
  int chunk = s_max > static_cast<int64_t>(MAX_SPLITS) * 128 ? CHUNK : 128;
  while (chunk > 64 && static_cast<int64_t>(rows) * n_kv * ((s_max + chunk - 1) / chunk) < 4 * 148 &&
         (s_max + chunk / 2 - 1) / (chunk / 2) <= MAX_SPLITS)  // never more chunks than the combine stages
    chunk /= 2;
  return chunk;
}
static int nsplit_for(int rows, int n_kv, int64_t s_max) {
  const int chunk = chunk_for(rows, n_kv, s_max);
  return static_cast<int>((s_max + chunk - 1) / chunk);
}

}  // namespace decode
}  // namespace bz

using namespace bz;

static int64_t workspace_bytes(int rows, int n_heads, int n_kv, int head_dim, int64_t s_max) {
  return static_cast<int64_t>(rows) * n_heads * decode::nsplit_for(rows, n_kv, s_max) * (head_dim + 2) * 4;
}

extern "C" int bz_decode_workspace_bytes(int rows, int n_heads, int n_kv, int head_dim, int64_t s_max,
                                         int64_t* bytes) {
  if (!bytes || rows < 0 || n_heads <= 0 || n_kv <= 0 || head_dim <= 0 || s_max <= 0)
    return bz_fail(BZ_EINVAL, "decode_workspace_bytes: bad args");
  *bytes = workspace_bytes(rows, n_heads, n_kv, head_dim, s_max);
  return BZ_OK;
}

static int rope_append(void* qkv, int ld, int rows, int n_heads, int n_kv, int head_dim, float theta, void* k_cache,
                       void* v_cache, int64_t s_max, const int32_t* pos, int pos_stride, void* stream) {
  if (!qkv || !k_cache || !v_cache || !pos || rows < 0 || n_heads <= 0 || n_kv <= 0 || head_dim % 2 ||
      n_heads % n_kv || s_max <= 0 || head_dim > 2048)
    return bz_fail(BZ_EINVAL, "rope_append: bad args");
  if (rows == 0) return BZ_OK;
  const int threads = (head_dim / 2 + 31) / 32 * 32;
  cudaError_t e = launch_pdl(PDL_GLUE, decode::k_rope_append, dim3(rows, n_heads + n_kv), dim3(threads), 0,
                             static_cast<cudaStream_t>(stream), static_cast<__nv_bfloat16*>(qkv), ld, n_heads, n_kv,
                             head_dim, log2f(theta), static_cast<__nv_bfloat16*>(k_cache),
                             static_cast<__nv_bfloat16*>(v_cache), s_max, pos, pos_stride);
  if (e != cudaSuccess) return bz_fail_cuda(e, "bz_rope_append");
  return bz_check_launch("bz_rope_append");
}

extern "C" int bz_rope_append(void* qkv, int ld, int rows, int n_heads, int n_kv, int head_dim, float theta,
                              void* k_cache, void* v_cache, int64_t s_max, const int32_t* pos, void* stream) {
  return rope_append(qkv, ld, rows, n_heads, n_kv, head_dim, theta, k_cache, v_cache, s_max, pos, 0, stream);
}

extern "C" int bz_rope_append_rows(void* qkv, int ld, int rows, int n_heads, int n_kv, int head_dim, float theta,
                                   void* k_cache, void* v_cache, int64_t s_max, const int32_t* pos, void* stream) {
  return rope_append(qkv, ld, rows, n_heads, n_kv, head_dim, theta, k_cache, v_cache, s_max, pos, 1, stream);
}

static int decode_attention(const void* q, int ldq, const void* k_cache, const void* v_cache, int rows, int n_heads,
                            int n_kv, int head_dim, int64_t s_max, const int32_t* pos, int pos_stride, void* out,
                            int ldo, void* workspace, int64_t ws_bytes, void* stream) {
  if (!q || !k_cache || !v_cache || !pos || !out || !workspace || rows < 0 || n_heads <= 0 || n_kv <= 0 ||
      n_heads % n_kv || s_max <= 0 || ldq % 8)
    return bz_fail(BZ_EINVAL, "decode_attention: bad args");
  if (head_dim != 64 && head_dim != 128) return bz_fail(BZ_EINVAL, "decode_attention: head_dim must be 64 or 128");
  if (rows == 0) return BZ_OK;
  if (ws_bytes < workspace_bytes(rows, n_heads, n_kv, head_dim, s_max))
    return bz_fail(BZ_EINVAL, "decode_attention: workspace too small");
  const int chunk = decode::chunk_for(rows, n_kv, s_max);
  const int nsplit = decode::nsplit_for(rows, n_kv, s_max);
  if (nsplit > decode::MAX_SPLITS)
    return bz_fail(BZ_EINVAL, "decode_attention: s_max above 64 chunks of 256 tokens (16384)");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const float scale = 1.0f / sqrtf(static_cast<float>(head_dim));
  const dim3 grid(nsplit, rows * n_kv);
  float* ws = static_cast<float*>(workspace);
  const auto* qb = static_cast<const __nv_bfloat16*>(q);
  const auto* kb = static_cast<const __nv_bfloat16*>(k_cache);
  const auto* vb = static_cast<const __nv_bfloat16*>(v_cache);
  auto* ob = static_cast<__nv_bfloat16*>(out);
  const int group = n_heads / n_kv;
  if (head_dim == 128)
    return decode::attention<128>(group, rows, grid, s, qb, ldq, kb, vb, n_heads, n_kv, s_max, pos, pos_stride, ws, nsplit,
                                  chunk, scale, ob, ldo);
  return decode::attention<64>(group, rows, grid, s, qb, ldq, kb, vb, n_heads, n_kv, s_max, pos, pos_stride, ws, nsplit, chunk,
                               scale, ob, ldo);
}

extern "C" int bz_decode_attention(const void* q, int ldq, const void* k_cache, const void* v_cache, int rows,
                                   int n_heads, int n_kv, int head_dim, int64_t s_max, const int32_t* pos, void* out,
                                   int ldo, void* workspace, int64_t ws_bytes, void* stream) {
  return decode_attention(q, ldq, k_cache, v_cache, rows, n_heads, n_kv, head_dim, s_max, pos, 0, out, ldo, workspace,
                          ws_bytes, stream);
}

extern "C" int bz_decode_attention_rows(const void* q, int ldq, const void* k_cache, const void* v_cache, int rows,
                                        int n_heads, int n_kv, int head_dim, int64_t s_max, const int32_t* pos,
                                        void* out, int ldo, void* workspace, int64_t ws_bytes, void* stream) {
  return decode_attention(q, ldq, k_cache, v_cache, rows, n_heads, n_kv, head_dim, s_max, pos, 1, out, ldo, workspace,
                          ws_bytes, stream);
}

const void* bz::module_anchor_decode() { return reinterpret_cast<const void*>(decode::k_rope_append); }
