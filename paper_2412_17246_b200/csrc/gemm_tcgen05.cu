// Persistent warp-specialised bf16 GEMM for sm_100a: TMA -> smem ring ->
// tcgen05.mma (accumulator in TMEM, double-buffered) -> tcgen05.ld epilogue.
//
//   C[M, N] (bf16, row-major) = A[M, K] (bf16, row-major) . B[N, K]^T
//
// B is a weight in torch Linear layout [out_features, in_features], so both
// operands are K-major and one kernel serves every projection of a Llama block
// (qkv, o, gate/up, down, lm_head).  This is the dense contraction of the
// cooperative (ZigZag) execution path -- the reference stands it in with the
// token-linear cost model ModelSpec.prefill_ms (parampool.py:58-62).
//
// Roles (8 warps): w0 = TMA producer, w1 = MMA issuer (one elected lane),
// w2 = TMEM allocator, w4..w7 = epilogue (TMEM lane quarter = warp % 4).
// Tiles: 128 x 256 x 64, 4-stage smem ring (48 KiB/stage), 2 x 256 TMEM
// columns so the epilogue of tile i overlaps the MMAs of tile i+1.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>
#include <stdlib.h>

#include "../../include/blitz.h"
#include "common.cuh"
#include "tc_primitives.cuh"

namespace bz {
namespace gemm {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 B = one swizzle-128B row
constexpr int UMMA_K = 16;
constexpr int A_BYTES = BM * BK * 2;  // 16 KiB
constexpr int THREADS = 256;
constexpr int SMEM_LIMIT = 232448;    // 227 KiB dynamic shared memory per CTA

// Single-CTA tiles: the width N is a template parameter (32 .. 256); the smem
// ring depth is chosen at launch from the bytes one stage really carries (a
// skinny A stage holds only ceil8(M) rows), up to MAX_STAGES, so a narrow
// weight tile still keeps ~128 KB of loads in flight per SM.
constexpr int MAX_STAGES = 32;
constexpr int BAR_BYTES = (2 * MAX_STAGES + 4) * 8 + 16;  // full/empty ring, acc full/empty, TMEM slot, flag
// OCC = CTAs per SM.  OCC = 2 (skinny decode GEMMs, BN <= 128): half the shared
// memory and at most 256 TMEM columns per CTA, so the next GEMM's CTA (launched
// early by PDL) is resident beside this one and streams its first weight stages
// while this one drains -- with one 227 KiB CTA per SM consecutive GEMMs cannot overlap.
constexpr int SMEM_LIMIT_OCC2 = 115712;  // 2 x (113 KiB + 1 KiB reserved) = 228 KiB per SM
template <int BN_, int OCC_ = 1>
struct Cfg {
  static constexpr int BN = BN_;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int ACC_COLS = BN;  // fp32 accumulator columns per buffer
  static constexpr int TMEM_COLS = 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;
  static constexpr int SMEM_BYTES = OCC_ == 1 ? SMEM_LIMIT : SMEM_LIMIT_OCC2;
  static_assert(BN % 32 == 0 && BN <= 256, "tile N");
  static_assert(OCC_ == 1 || (OCC_ == 2 && TMEM_COLS <= 256), "two CTAs per SM share 512 TMEM columns");
};
// ring stages for one A stage of a_stage bytes (multiple of 1024) and B_BYTES
__host__ __device__ constexpr int ring_stages(int a_stage, int b_bytes, int limit = SMEM_LIMIT) {
  return (limit - 1024 - BAR_BYTES) / (a_stage + b_bytes) < MAX_STAGES ? (limit - 1024 - BAR_BYTES) / (a_stage + b_bytes)
                                                                      : MAX_STAGES;
}

using namespace bz::tc;

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

struct Params {
  __nv_bfloat16* C;
  const __nv_bfloat16* R;  // optional residual added in the epilogue (same layout as C)
  int M, N, K, ldc, ldr;
  int m_tiles, n_tiles;
  uint32_t* signal;  // optional: +1 (release, system scope) per CTA when its tiles are stored
  // Stream-K (skinny M <= 128, e.g. decode, where tiles < SMs): the tiles x
  // K-blocks iteration space is cut into equal contiguous ranges, one per CTA,
  // so every SM streams the same weight bytes.  A range covers at most two
  // partial tiles (its head and tail); a partial writes fp32 to its CTA's slot
  // ws[cta][0 = head | 1 = tail][M][BN] and bumps counters[tile]; the last
  // contributor sums the slots (+ residual) into C and resets the counter, so
  // the workspace stays zeroed between calls.  streamk == 0: whole tiles,
  // round-robin over a persistent grid.
  float* ws;
  int* counters;
  int streamk, sk_per, sk_total;
  int a_bytes;   // bytes of one A stage actually loaded (M < 128: only ceil8(M) rows)
  int a_stage;   // smem stride of the A ring (a_bytes rounded up to the 1024-B swizzle atom)
  int stages;    // ring depth (single-CTA kernel)
  int b_static;  // B is not written by in-flight predecessors: prefetch it before pdl_wait
  int c_f32;     // C is fp32 (BZ_GEMM_C_F32: logits keep the accumulator's precision)
  // split-K of the pair kernel (few tiles, long K): unit = (tile, K slice); slices
  // store fp32 partials to ws[slice][M][N], k_splitk_reduce adds them into C
  int ksplit, kb_slice;
  int kc_nomma;  // diagnostic (BZ_GEMM_KC_NOMMA): the K-chunked kernel streams B without MMAs
};

// The (tile, k0, k1) segments one CTA processes, in order; identical for the
// producer, MMA and epilogue roles.
struct SegIter {
  int i, end, next_tile, k_blocks, num_tiles;
  bool sk;
  __device__ SegIter(const Params& p, int kb, int tiles)
      : k_blocks(kb), num_tiles(tiles), sk(p.streamk != 0) {
    i = static_cast<int>(blockIdx.x) * p.sk_per;
    end = min(i + p.sk_per, p.sk_total);
    next_tile = blockIdx.x;
  }
  __device__ bool next(int& tile, int& k0, int& k1) {
    if (sk) {
      if (i >= end) return false;
      tile = i / k_blocks;
      k0 = i % k_blocks;
      k1 = min(k_blocks, k0 + (end - i));
      i += k1 - k0;
      return true;
    }
    if (next_tile >= num_tiles) return false;
    tile = next_tile;
    k0 = 0;
    k1 = k_blocks;
    next_tile += gridDim.x;
    return true;
  }
};

// bf16 store of a 32-column accumulator chunk (+ optional residual) for one row
// (columns at or beyond `lim` -- the end of C or of a tile narrower than a
// multiple of 32 -- are not written)
__device__ __forceinline__ void store_chunk(const Params& p, int row, int col, const uint32_t (&r)[32], int lim) {
  if (p.c_f32) {
    // fp32 C (+ bf16 residual): the accumulator as is, 16-byte stores
    float* of = reinterpret_cast<float*>(p.C) + static_cast<int64_t>(row) * p.ldc + col;
    const __nv_bfloat16* rs = p.R ? p.R + static_cast<int64_t>(row) * p.ldr + col : nullptr;
    if (col + 32 <= lim) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float4 v = make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]), __uint_as_float(r[4 * q + 2]),
                               __uint_as_float(r[4 * q + 3]));
        if (rs) {
          v.x += __bfloat162float(rs[4 * q]), v.y += __bfloat162float(rs[4 * q + 1]);
          v.z += __bfloat162float(rs[4 * q + 2]), v.w += __bfloat162float(rs[4 * q + 3]);
        }
        reinterpret_cast<float4*>(of)[q] = v;
      }
    } else {
      for (int j = 0; j < 32; ++j)
        if (col + j < lim) of[j] = __uint_as_float(r[j]) + (rs ? __bfloat162float(rs[j]) : 0.f);
    }
    return;
  }
  __nv_bfloat16* out = p.C + static_cast<int64_t>(row) * p.ldc + col;
  const __nv_bfloat16* res = p.R ? p.R + static_cast<int64_t>(row) * p.ldr + col : nullptr;
  if (col + 32 <= lim) {
    uint32_t w[16];
    if (res) {
      uint32_t x[16];
      if ((reinterpret_cast<uintptr_t>(res) & 31) == 0) {
        // two 256-bit loads of the residual row segment
#pragma unroll
        for (int h = 0; h < 2; ++h)
          asm volatile("ld.global.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                       : "=r"(x[8 * h]), "=r"(x[8 * h + 1]), "=r"(x[8 * h + 2]), "=r"(x[8 * h + 3]),
                         "=r"(x[8 * h + 4]), "=r"(x[8 * h + 5]), "=r"(x[8 * h + 6]), "=r"(x[8 * h + 7])
                       : "l"(res + 16 * h));
      } else {
        const uint4* rv = reinterpret_cast<const uint4*>(res);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint4 v = rv[q];
          x[4 * q] = v.x, x[4 * q + 1] = v.y, x[4 * q + 2] = v.z, x[4 * q + 3] = v.w;
        }
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&x[j]));
        w[j] = pack_bf16(__uint_as_float(r[2 * j]) + f.x, __uint_as_float(r[2 * j + 1]) + f.y);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) w[j] = pack_bf16(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1]));
    }
    if ((reinterpret_cast<uintptr_t>(out) & 31) == 0) {
      // two 256-bit stores: each request fills whole 32-byte L2 sectors
#pragma unroll
      for (int h = 0; h < 2; ++h)
        asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(out + 16 * h), "r"(w[8 * h]),
                     "r"(w[8 * h + 1]), "r"(w[8 * h + 2]), "r"(w[8 * h + 3]), "r"(w[8 * h + 4]), "r"(w[8 * h + 5]),
                     "r"(w[8 * h + 6]), "r"(w[8 * h + 7])
                     : "memory");
    } else {
      uint4* o = reinterpret_cast<uint4*>(out);
#pragma unroll
      for (int q = 0; q < 4; ++q) o[q] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      if (col + j < lim) {
        float v = __uint_as_float(r[j]);
        if (res) v += __bfloat162float(res[j]);
        out[j] = __float2bfloat16_rn(v);
      }
    }
  }
}

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

__device__ __forceinline__ float* sk_slot(const Params& p, int cta, int slot, int bn) {
  return p.ws + (static_cast<int64_t>(cta) * 2 + slot) * p.M * bn;
}

// Last contributor of a stream-K tile: C[tile] = bf16(sum of the contributors'
// slots + R).  Contributor c's segment of tile t sits in its head slot iff c's
// range starts inside t.  The 128 epilogue threads sweep the [M][bn] slots as
// flat float4 arrays (coalesced), eight float4s per thread per pass and two
// contributors per round, so each pass keeps 16 independent L2 loads in flight.
__device__ __forceinline__ void streamk_fixup(const Params& p, int tile, int n0, int bn, int k_blocks, int et) {
  constexpr int U = 8;  // float4s per thread per pass: 2 x 8 independent L2 loads in flight
  const int first = tile * k_blocks / p.sk_per, last = ((tile + 1) * k_blocks - 1) / p.sk_per;
  const int q_row = bn / 4;  // float4s per slot row
  const int n4 = p.M * q_row;
  for (int f0 = et; f0 < n4; f0 += U * 128) {
    float4 acc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int c = first; c <= last; c += 2) {
      const bool two = c + 1 <= last;
      const float4* s0 =
          reinterpret_cast<const float4*>(sk_slot(p, c, c * p.sk_per >= tile * k_blocks ? 0 : 1, bn));
      const float4* s1 = reinterpret_cast<const float4*>(
          sk_slot(p, two ? c + 1 : c, (c + 1) * p.sk_per >= tile * k_blocks ? 0 : 1, bn));
      float4 v0[U], v1[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int f = f0 + u * 128;
        v0[u] = f < n4 ? __ldcg(s0 + f) : make_float4(0.f, 0.f, 0.f, 0.f);
        v1[u] = (two && f < n4) ? __ldcg(s1 + f) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        acc[u].x += v0[u].x + v1[u].x;
        acc[u].y += v0[u].y + v1[u].y;
        acc[u].z += v0[u].z + v1[u].z;
        acc[u].w += v0[u].w + v1[u].w;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int f = f0 + u * 128;
      if (f >= n4) break;
      const int row = f / q_row, col = n0 + (f % q_row) * 4;
      if (col >= p.N) continue;
      float4 v = acc[u];
      if (p.R) {
        const uint2 rv = *reinterpret_cast<const uint2*>(p.R + static_cast<int64_t>(row) * p.ldr + col);
        const float2 r0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&rv.x));
        const float2 r1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&rv.y));
        v.x += r0.x, v.y += r0.y, v.z += r1.x, v.w += r1.y;
      }
      if (p.c_f32)
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(p.C) + static_cast<int64_t>(row) * p.ldc + col) = v;
      else
        *reinterpret_cast<uint2*>(p.C + static_cast<int64_t>(row) * p.ldc + col) =
            make_uint2(pack_bf16(v.x, v.y), pack_bf16(v.z, v.w));
    }
  }
}

template <int BN_, int OCC_>
__global__ void __launch_bounds__(THREADS, OCC_)
    k_gemm_bf16(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b, Params p) {
  using C = Cfg<BN_, OCC_>;
  constexpr int BN = C::BN, B_BYTES = C::B_BYTES;
  constexpr int ACC_COLS = C::ACC_COLS, TMEM_COLS = C::TMEM_COLS;
  const int STAGES = p.stages, A_STAGE = p.a_stage;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // ring: STAGES x A (A_STAGE bytes each) | STAGES x B | barriers.  A skinny A
  // stage holds only the rows that exist; the 128-row MMA reads past them into
  // later stages (stale rows, never stored).
  uint8_t* sa = smem;
  uint8_t* sb = smem + STAGES * A_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(sb + STAGES * B_BYTES);
  uint64_t* empty = full + MAX_STAGES;
  uint64_t* acc_full = empty + STAGES;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  volatile int* last_contrib = reinterpret_cast<volatile int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_tiles = p.m_tiles * p.n_tiles;
  const int k_blocks = (p.K + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&map_a);
    prefetch_tmap(&map_b);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 4);  // one arrive per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer ----
      // Prologue: with a static B (weights) the first stages' B tiles are issued
      // before pdl_wait, overlapping the predecessor kernel; A (activations)
      // follows once the predecessor's writes are visible.
      SegIter seg(p, k_blocks, num_tiles);
      int tile, k0, k1, pre = 0, pre_k0 = 0, pre_m0 = 0;
      bool have = seg.next(tile, k0, k1);
      if (p.b_static && have) {
        pre_m0 = (tile % p.m_tiles) * BM;
        pre_k0 = k0;
        pre = min(STAGES, k1 - k0);
        for (int i = 0; i < pre; ++i) {
          mbar_expect_tx(&full[i], p.a_bytes + B_BYTES);
          tma_load_2d(sb + i * B_BYTES, &map_b, (k0 + i) * BK, (tile / p.m_tiles) * BN, &full[i]);
        }
      }
      pdl_wait();
      for (int i = 0; i < pre; ++i) tma_load_2d(sa + i * A_STAGE, &map_a, (pre_k0 + i) * BK, pre_m0, &full[i]);
      uint32_t stage = pre % STAGES, phase = pre == STAGES ? 1u : 0u;
      for (int skip = pre; have; have = seg.next(tile, k0, k1), skip = 0) {
        const int m0 = (tile % p.m_tiles) * BM;
        const int n0 = (tile / p.m_tiles) * BN;
        for (int kb = k0 + skip; kb < k1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], p.a_bytes + B_BYTES);
          tma_load_2d(sa + stage * A_STAGE, &map_a, kb * BK, m0, &full[stage]);
          tma_load_2d(sb + stage * B_BYTES, &map_b, kb * BK, n0, &full[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      // every load is issued: let the next kernel launch during the drain
      pdl_trigger();
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---- MMA issuer ----
      pdl_wait();
      constexpr uint32_t idesc = instr_desc_bf16(BM, BN);
      SegIter seg(p, k_blocks, num_tiles);
      int tile, k0, k1;
      uint32_t stage = 0, phase = 0;
      for (int it = 0; seg.next(tile, k0, k1); ++it) {
        const int buf = it & 1;
        const uint32_t use = static_cast<uint32_t>(it >> 1);
        mbar_wait(&acc_empty[buf], (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + buf * ACC_COLS;
        for (int kb = k0; kb < k1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t da = umma_desc_sw128(smem_u32(sa + stage * A_STAGE));
          const uint64_t db = umma_desc_sw128(smem_u32(sb + stage * B_BYTES));
#pragma unroll
          for (int k = 0; k < BK / UMMA_K; ++k) {
            // +32 B along K inside the swizzle atom = +2 in the encoded address
            umma_bf16(d, da + 2 * k, db + 2 * k, idesc, (kb != k0 || k != 0) ? 1u : 0u);
          }
          umma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&acc_full[buf]);
      }
    }
  } else if (warp >= 4) {
    // ---- epilogue: TMEM -> registers -> bf16 -> global ----
    pdl_wait();  // reads the residual and writes C / the stream-K workspace
    const int quarter = warp & 3;
    const int et = threadIdx.x - 128;  // epilogue thread 0..127
    SegIter seg(p, k_blocks, num_tiles);
    int tile, k0, k1;
    for (int it = 0; seg.next(tile, k0, k1); ++it) {
      const int buf = it & 1;
      const uint32_t use = static_cast<uint32_t>(it >> 1);
      const int m0 = (tile % p.m_tiles) * BM;
      const int n0 = (tile / p.m_tiles) * BN;
      const bool partial = k0 != 0 || k1 != k_blocks;
      // head slot iff this CTA's range starts inside the tile
      const int slot = static_cast<int>(blockIdx.x) * p.sk_per >= tile * k_blocks ? 0 : 1;
      mbar_wait(&acc_full[buf], use & 1);
      tc_fence_after();
      const int row = m0 + quarter * 32 + lane;
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + buf * ACC_COLS;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(taddr + c, r);
        if (row >= p.M) continue;
        if (partial) {
          // the slot is [M][BN] fp32, 32-byte aligned: 256-bit stores of 8 columns
          float* dst = sk_slot(p, blockIdx.x, slot, BN) + row * BN + c;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (n0 + c + 8 * q < p.N)
              asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst + 8 * q), "r"(r[8 * q]),
                           "r"(r[8 * q + 1]), "r"(r[8 * q + 2]), "r"(r[8 * q + 3]), "r"(r[8 * q + 4]),
                           "r"(r[8 * q + 5]), "r"(r[8 * q + 6]), "r"(r[8 * q + 7])
                           : "memory");
        } else {
          store_chunk(p, row, n0 + c, r, p.N);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[buf]);
      if (partial) {
        const int contributors =
            ((tile + 1) * k_blocks - 1) / p.sk_per - tile * k_blocks / p.sk_per + 1;
        __threadfence();
        epi_bar();
        if (et == 0) *last_contrib = atomicAdd(&p.counters[tile], 1) == contributors - 1;
        epi_bar();
        if (*last_contrib) {
          __threadfence();
          streamk_fixup(p, tile, n0, BN, k_blocks, et);
          if (et == 0) p.counters[tile] = 0;
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(TMEM_COLS));
  }
  if (p.signal != nullptr && threadIdx.x == 0) {
    // fused hand-off: C may be a peer (NVLink) mapping; publish this CTA's tiles
    // (with stream-K, every fix-up this CTA performed is complete here)
    __threadfence_system();
    asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(p.signal) : "memory");
  }
}

// ===========================================================================
// Decode-shaped (M <= 16) whole-tile variant with K-chunked stages: a stage is one 3-D
// TMA box {64 k, rows, KCH k-blocks} of A and of B (KCH 64-wide 128B-swizzled tiles
// side by side), so a narrow weight tile (BN = 32) still moves 32 KiB per TMA op and
// per pipeline step.  With the 2-D layout a 32-row tile paid the per-k-block ring step
// (~270 ns) every 4 KiB, so narrow tiles were slow and decode relied on wide tiles
// plus stream-K (and its fix-up tail).  Here every CTA owns whole BN-row tiles over all
// of K -- no partials, no fix-up -- and BN is chosen to give each SM about one tile.
// Roles as k_gemm_bf16: w0 TMA, w1 MMA, w2 TMEM allocator, w4..w7 epilogue.
template <int BN_>
__global__ void __launch_bounds__(THREADS, 1)
    k_gemm_skinny_kc(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b, Params p,
                     int kch, int a_rows) {
  constexpr int BN = BN_;
  constexpr int ACC_COLS = BN;
  constexpr int TMEM_COLS = 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;
  const int STAGES = p.stages;
  const int A_STG = kch * a_rows * 128, B_STG = kch * BN * 128;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;                                   // STAGES x A_STG (1024-B multiples)
  uint8_t* sb = smem + STAGES * A_STG;                  // STAGES x B_STG
  uint64_t* full = reinterpret_cast<uint64_t*>(sb + STAGES * B_STG);
  uint64_t* empty = full + MAX_STAGES;
  uint64_t* acc_full = empty + MAX_STAGES;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k_blocks = (p.K + BK - 1) / BK;
  const int nks = (k_blocks + kch - 1) / kch;           // stages per tile
  const int n_tiles = p.n_tiles;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&map_a);
    prefetch_tmap(&map_b);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // the first tile's first stages of B (weights) go out before pdl_wait, overlapping
      // the predecessor; A (activations) follows once its writes are visible
      const int pre = (p.b_static && static_cast<int>(blockIdx.x) < n_tiles) ? min(STAGES, nks) : 0;
      for (int i = 0; i < pre; ++i) {
        mbar_expect_tx(&full[i], A_STG + B_STG);
        tma_load_3d(sb + i * B_STG, &map_b, 0, static_cast<int>(blockIdx.x) * BN, i * kch, &full[i]);
      }
      pdl_wait();
      for (int i = 0; i < pre; ++i) tma_load_3d(sa + i * A_STG, &map_a, 0, 0, i * kch, &full[i]);
      uint32_t stage = pre % STAGES, phase = pre == STAGES ? 1u : 0u;
      for (int tile = blockIdx.x, skip = pre; tile < n_tiles; tile += gridDim.x, skip = 0) {
        for (int ks = skip; ks < nks; ++ks) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], A_STG + B_STG);
          tma_load_3d(sa + stage * A_STG, &map_a, 0, 0, ks * kch, &full[stage]);
          tma_load_3d(sb + stage * B_STG, &map_b, 0, tile * BN, ks * kch, &full[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      pdl_trigger();
    }
  } else if (warp == 1) {
    if (lane == 0) {
      pdl_wait();
      constexpr uint32_t idesc = instr_desc_bf16(BM, BN);
      uint32_t stage = 0, phase = 0;
      for (int tile = blockIdx.x, it = 0; tile < n_tiles; tile += gridDim.x, ++it) {
        const int buf = it & 1;
        const uint32_t use = static_cast<uint32_t>(it >> 1);
        mbar_wait(&acc_empty[buf], (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + buf * ACC_COLS;
        for (int ks = 0; ks < nks; ++ks) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const int subs = p.kc_nomma ? 0 : min(kch, k_blocks - ks * kch);
          for (int sub = 0; sub < subs; ++sub) {
            const uint64_t da = umma_desc_sw128(smem_u32(sa + stage * A_STG + sub * a_rows * 128));
            const uint64_t db = umma_desc_sw128(smem_u32(sb + stage * B_STG + sub * BN * 128));
#pragma unroll
            for (int k = 0; k < BK / UMMA_K; ++k)
              umma_bf16(d, da + 2 * k, db + 2 * k, idesc, (ks != 0 || sub != 0 || k != 0) ? 1u : 0u);
          }
          umma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&acc_full[buf]);
      }
    }
  } else if (warp >= 4) {
    pdl_wait();  // reads the residual and writes C
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    for (int tile = blockIdx.x, it = 0; tile < n_tiles; tile += gridDim.x, ++it) {
      const int buf = it & 1;
      const uint32_t use = static_cast<uint32_t>(it >> 1);
      mbar_wait(&acc_full[buf], use & 1);
      tc_fence_after();
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + buf * ACC_COLS;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(taddr + c, r);
        if (row < p.M) store_chunk(p, row, tile * BN + c, r, p.N);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[buf]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(TMEM_COLS));
  }
  if (p.signal != nullptr && threadIdx.x == 0) {
    __threadfence_system();
    asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(p.signal) : "memory");
  }
}

// ===========================================================================
// CTA-pair variant (cta_group::2): a cluster of two CTAs computes a 256 x BN
// tile.  CTA r loads A rows [128r, 128r+128) and B rows [r*BN/2, (r+1)*BN/2)
// of the pair tile; the leader (r = 0) issues tcgen05.mma.cta_group::2 M=256,
// which reads A from both CTAs' shared memory and B from both halves, and
// writes 128 accumulator lanes x BN columns into each CTA's TMEM.  Per SM the
// smem fill per K step drops from (128 + BN) rows to (128 + BN/2) rows.

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa_cta(uint32_t smem_addr, uint32_t cta) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr), "r"(cta));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// both CTAs load into their own smem; completion bytes go to the leader's barrier
__device__ __forceinline__ void tma_load_2d_pair(void* smem, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  const uint32_t leader_bar = smem_u32(bar) & 0xFEFFFFFFu;
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(smem_u32(smem)),
      "l"(map), "r"(c0), "r"(c1), "r"(leader_bar)
      : "memory");
}
__device__ __forceinline__ void umma_bf16_pair(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// arrive on the same-offset barrier of both CTAs when the leader's MMAs complete
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(static_cast<uint16_t>(0x3))
      : "memory");
}

// A pair tile is 256 rows x (NSUB * BN) columns: NSUB independent M256xBN
// accumulators, each fed by the same A stage, so NSUB = 2 halves the A bytes per
// MAC (the smem feed, not the MMA, bounds this kernel: with loads elided it runs
// at 1.9 PFLOP/s).  TMEM holds two tiles (double-buffered epilogue) when
// 2 * NSUB * BN <= 512 columns, else one.
template <int BN_, int NSUB_ = 1>
struct CfgPair {
  static constexpr int BN = BN_;
  static constexpr int NSUB = NSUB_;
  static constexpr int TILE_N = BN * NSUB;
  static constexpr int B_SUB = (BN / 2) * BK * 2;    // this CTA's half of one sub-tile's B
  static constexpr int B_BYTES = NSUB * B_SUB;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES_FIT = (SMEM_LIMIT - 2048) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_FIT > 8 ? 8 : STAGES_FIT;
  static constexpr int ACC_BUFS = 2 * TILE_N <= 512 ? 2 : 1;
  static constexpr int TMEM_COLS = ACC_BUFS * TILE_N <= 256 ? 256 : 512;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
  static_assert(BN % 16 == 0 && (BN / 2) % 8 == 0 && BN <= 256 && BN >= 64, "tile N");
  static_assert(ACC_BUFS * TILE_N <= 512, "TMEM");
};

// 32 fp32 columns of one row of a split-K partial (columns at or beyond `lim` skipped)
__device__ __forceinline__ void store_partial(float* row_base, int col, const uint32_t (&r)[32], int lim) {
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (col + 8 * q < lim)
      asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(row_base + col + 8 * q), "r"(r[8 * q]),
                   "r"(r[8 * q + 1]), "r"(r[8 * q + 2]), "r"(r[8 * q + 3]), "r"(r[8 * q + 4]), "r"(r[8 * q + 5]),
                   "r"(r[8 * q + 6]), "r"(r[8 * q + 7])
                   : "memory");
}

// C = bf16(sum of the K-slice partials + R): 8 columns (two 256-bit loads per slice,
// one 16-byte store) per thread; the fused hand-off signal is raised here.
__global__ void __launch_bounds__(256) k_splitk_reduce(const float* __restrict__ ws, int ksplit, int M, int N,
                                                       __nv_bfloat16* C, int ldc, const __nv_bfloat16* R, int ldr,
                                                       uint32_t* signal) {
  pdl_wait();
  pdl_trigger();
  const int g8 = N / 8;
  const int64_t groups = static_cast<int64_t>(M) * g8;
  const int64_t plane = static_cast<int64_t>(M) * N;
  for (int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; g < groups;
       g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int row = static_cast<int>(g / g8), col = static_cast<int>(g % g8) * 8;
    const float* src = ws + static_cast<int64_t>(row) * N + col;
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int sl = 0; sl < ksplit; ++sl) {
      const float4 a = __ldcg(reinterpret_cast<const float4*>(src + sl * plane));
      const float4 b = __ldcg(reinterpret_cast<const float4*>(src + sl * plane) + 1);
      acc[0] += a.x, acc[1] += a.y, acc[2] += a.z, acc[3] += a.w;
      acc[4] += b.x, acc[5] += b.y, acc[6] += b.z, acc[7] += b.w;
    }
    if (R) {
      const uint4 rv = *reinterpret_cast<const uint4*>(R + static_cast<int64_t>(row) * ldr + col);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&rv);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(h[j]);
        acc[2 * j] += f.x;
        acc[2 * j + 1] += f.y;
      }
    }
    *reinterpret_cast<uint4*>(C + static_cast<int64_t>(row) * ldc + col) =
        make_uint4(pack_bf16(acc[0], acc[1]), pack_bf16(acc[2], acc[3]), pack_bf16(acc[4], acc[5]),
                   pack_bf16(acc[6], acc[7]));
  }
  if (signal != nullptr) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(signal) : "memory");
    }
  }
}

// p.m_tiles counts 256-row pair tiles here
template <int BN_, int NSUB_>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    k_gemm_bf16_pair(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b, Params p) {
  using C = CfgPair<BN_, NSUB_>;
  constexpr int BN = C::BN, NSUB = C::NSUB, TILE_N = C::TILE_N, STAGES = C::STAGES;
  constexpr int B_SUB = C::B_SUB, B_BYTES = C::B_BYTES, STAGE_BYTES = C::STAGE_BYTES;
  constexpr int ACC_BUFS = C::ACC_BUFS, TMEM_COLS = C::TMEM_COLS;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;
  uint8_t* sb = smem + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cluster = blockIdx.x >> 1;
  const int clusters = gridDim.x >> 1;
  const int num_tiles = p.m_tiles * p.n_tiles;
  const int num_units = num_tiles * p.ksplit;
  const int k_blocks = (p.K + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&map_a);
    prefetch_tmap(&map_b);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 8);  // 4 epilogue warps x 2 CTAs (leader's copy is used)
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      pdl_wait();
      uint32_t stage = 0, phase = 0;
      for (int unit = cluster; unit < num_units; unit += clusters) {
        const int tile = unit % num_tiles;
        const int m0 = (tile % p.m_tiles) * (2 * BM) + static_cast<int>(rank) * BM;
        const int n0 = (tile / p.m_tiles) * TILE_N + static_cast<int>(rank) * (BN / 2);
        const int kb0 = (unit / num_tiles) * p.kb_slice, kb1 = min(k_blocks, kb0 + p.kb_slice);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (leader) mbar_expect_tx(&full[stage], 2 * STAGE_BYTES);
          tma_load_2d_pair(sa + stage * A_BYTES, &map_a, kb * BK, m0, &full[stage]);
#pragma unroll
          for (int j = 0; j < NSUB; ++j)
            tma_load_2d_pair(sb + stage * B_BYTES + j * B_SUB, &map_b, kb * BK, n0 + j * BN, &full[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      pdl_trigger();
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      pdl_wait();
      constexpr uint32_t idesc = instr_desc_bf16(2 * BM, BN);
      uint32_t stage = 0, phase = 0;
      int it = 0;
      for (int unit = cluster; unit < num_units; unit += clusters, ++it) {
        const int buf = it % ACC_BUFS;
        const uint32_t use = static_cast<uint32_t>(it / ACC_BUFS);
        const int kb0 = (unit / num_tiles) * p.kb_slice, kb1 = min(k_blocks, kb0 + p.kb_slice);
        mbar_wait(&acc_empty[buf], (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + buf * TILE_N;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t da = umma_desc_sw128(smem_u32(sa + stage * A_BYTES));
#pragma unroll
          for (int k = 0; k < BK / UMMA_K; ++k) {
#pragma unroll
            for (int j = 0; j < NSUB; ++j) {
              const uint64_t db = umma_desc_sw128(smem_u32(sb + stage * B_BYTES + j * B_SUB));
              umma_bf16_pair(d + j * BN, da + 2 * k, db + 2 * k, idesc, (kb != kb0 || k != 0) ? 1u : 0u);
            }
          }
          umma_commit_pair(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_pair(&acc_full[buf]);
      }
    }
  } else if (warp >= 4) {
    pdl_wait();
    const int quarter = warp & 3;
    const uint32_t leader_acc_empty0 = mapa_cta(smem_u32(&acc_empty[0]), 0);
    int it = 0;
    for (int unit = cluster; unit < num_units; unit += clusters, ++it) {
      const int tile = unit % num_tiles;
      const int buf = it % ACC_BUFS;
      const uint32_t use = static_cast<uint32_t>(it / ACC_BUFS);
      const int m0 = (tile % p.m_tiles) * (2 * BM) + static_cast<int>(rank) * BM;
      const int n0 = (tile / p.m_tiles) * TILE_N;
      mbar_wait(&acc_full[buf], use & 1);
      tc_fence_after();
      const int row = m0 + quarter * 32 + lane;
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + buf * TILE_N;
      const int lim = min(p.N, n0 + TILE_N);
#pragma unroll 1
      for (int c = 0; c < TILE_N; c += 64) {
        // two 32-column loads in flight, then store both
        uint32_t r0[32], r1[32];
        tmem_ld_32x32b_x32_async(taddr + c, r0);
        if (c + 32 < TILE_N) tmem_ld_32x32b_x32_async(taddr + c + 32, r1);
        tmem_wait_ld(r0);
        tmem_wait_ld(r1);
        if (row >= p.M) continue;
        if (p.ksplit > 1) {
          // fp32 partial of this K slice (reduced by k_splitk_reduce)
          float* dst = p.ws + (static_cast<int64_t>(unit / num_tiles) * p.M + row) * p.N;
          store_partial(dst, n0 + c, r0, lim);
          if (c + 32 < TILE_N) store_partial(dst, n0 + c + 32, r1, lim);
        } else {
          if (n0 + c < p.N) store_chunk(p, row, n0 + c, r0, lim);
          if (c + 32 < TILE_N && n0 + c + 32 < p.N) store_chunk(p, row, n0 + c + 32, r1, lim);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(leader_acc_empty0 + buf * 8);
    }
  }

  tc_fence_before();
  cluster_sync_all();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(TMEM_COLS));
  }
  if (p.signal != nullptr && p.ksplit == 1 && threadIdx.x == 0) {
    __threadfence_system();
    asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(p.signal) : "memory");
  }
}

// workspace = [stream-K tile counters (int32, zero between calls): a FIXED header |
//              stream-K per-CTA head/tail slots, or the pair kernel's split-K partials]
// The header is never written by anything but the counters' own atomics and resets:
// split-K partials used to start at offset 0 and clobbered the counters, so the next
// stream-K GEMM on the same workspace (a decode step after a split-K prefill) summed
// garbage.  Stream-K runs only with fewer tiles than SMs, so 1024 counters suffice.
constexpr int64_t kCounterHeader = 4096;
static int64_t counters_bytes(int tiles) { return tiles * 4 <= kCounterHeader ? 0 : INT64_MAX / 4; }

// BZ_GEMM_STREAMK=0|1 forces stream-K off/on (when feasible); unset: cost model
static int streamk_override() {
  static int v = -2;
  if (v == -2) {
    const char* e = getenv("BZ_GEMM_STREAMK");
    v = e ? atoi(e) : -1;
  }
  return v;
}

// Skinny weight streaming on B200 (scripts/skinny_bench.py, profiles/r1_skinny_gemm.txt):
// a CTA retires one 64-deep K block (4 single-CTA MMAs issued from shared
// memory) in ~270 ns whatever the tile width up to 128 (~330 ns at 256): the
// MMA floor, not the bytes, paces a narrow tile; the chip pulls ~5.5 TB/s of
// weight tiles; stream-K costs ~5 us (partial write, fence, counter, slot sum
// on the critical path) plus ~0.09 us per row of A at width 128, growing as
// width^1.5.
constexpr double SKINNY_CHIP_BPS = 5.5e12, SKINNY_KBLOCK_S = 270e-9;
constexpr double SKINNY_FIXUP_US = 5.0, SKINNY_FIXUP_US_PER_ROW128 = 0.09;

static double kblock_s(int bn) { return SKINNY_KBLOCK_S * (bn > 200 ? bn / 200.0 : 1.0); }

struct SkinnyPlan {
  int bn;
  int sk_per;  // K blocks per CTA under stream-K; 0 = whole tiles
};

// Tile width and schedule for M <= 128 (one row of tiles): the fastest predicted
// of {32 .. 256} x {whole tiles, stream-K}.
static SkinnyPlan plan_skinny(int M, int N, int K, int ctas, int64_t ws_bytes, int only_bn, int max_bn = 256) {
  const int widths[5] = {256, 192, 128, 64, 32};
  const int k_blocks = (K + BK - 1) / BK;
  const double chip = 2.0 * N * K / SKINNY_CHIP_BPS;
  const int force = streamk_override();
  SkinnyPlan plain{only_bn ? only_bn : 128, 0}, sk{0, 0};
  double t_plain = 1e30, t_sk = 1e30;
  for (int bn : widths) {  // widest first: a narrower tile must win by 2 %
    if ((only_bn && bn != only_bn) || bn > max_bn) continue;
    const int tiles = (N + bn - 1) / bn;
    const double waves = static_cast<double>((tiles + ctas - 1) / ctas);
    const double run = waves * k_blocks * kblock_s(bn);
    const double t = chip > run ? chip : run;
    if (t < 0.98 * t_plain) {
      t_plain = t;
      plain = {bn, 0};
    }
    if (ws_bytes <= 0 || tiles >= ctas) continue;
    int per = (tiles * k_blocks + ctas - 1) / ctas;
    if (per < 4) per = 4;
    if (per >= k_blocks) continue;
    const int used = (tiles * k_blocks + per - 1) / per;
    if (counters_bytes(tiles) + static_cast<int64_t>(used) * 2 * M * bn * 4 > ws_bytes) continue;
    const double sk_run = per * kblock_s(bn);
    const double wide = bn / 128.0;
    const double ts = (chip > sk_run ? chip : sk_run) +
                      (SKINNY_FIXUP_US + SKINNY_FIXUP_US_PER_ROW128 * M * wide * sqrt(wide)) * 1e-6;
    if (ts < 0.98 * t_sk) {
      t_sk = ts;
      sk = {bn, per};
    }
  }
  if (sk.bn && (force == 1 || (force != 0 && t_sk < t_plain))) return sk;
  return plain;
}

static int encode_kmajor(CUtensorMap* map, const void* ptr, int rows, int k, int ld, int box_rows) {
  const DriverApi* d = driver_api();
  if (!d) return BZ_ECUDA;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(k), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(BK), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t elem[2] = {1, 1};
  CUresult r = d->cuTensorMapEncodeTiled(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims,
                                         strides, box, elem, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return bz_fail_cu(r, "cuTensorMapEncodeTiled");
  return BZ_OK;
}

// BZ_GEMM_BN=32|64|128|192|256 pins the tile width (tests/benchmarks); 0 = automatic
static int bn_override() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BZ_GEMM_BN");
    v = e ? atoi(e) : 0;
    if (v != 32 && v != 64 && v != 128 && v != 192 && v != 240 && v != 256) v = 0;
  }
  return v;
}

// Tile width for a problem: maximise (useful columns / padded columns) x
// (tiles / (waves x SMs)) x a small per-width efficiency prior.
static int pick_bn(int M, int N, int ctas) {
  const int widths[3] = {256, 192, 128};
  const double prior[3] = {1.0, 0.985, 0.95};
  int best = 256;
  double best_score = -1.0;
  const int mt = (M + BM - 1) / BM;
  for (int i = 0; i < 3; ++i) {
    const int bn = widths[i];
    const int nt = (N + bn - 1) / bn;
    const long tiles = static_cast<long>(mt) * nt;
    const long waves = (tiles + ctas - 1) / ctas;
    const double fill = static_cast<double>(tiles) / static_cast<double>(waves * ctas);
    const double cols = static_cast<double>(N) / (static_cast<double>(nt) * bn);
    const double score = fill * cols * prior[i];
    if (score > best_score + 1e-9) {
      best_score = score;
      best = bn;
    }
  }
  return best;
}

template <int BN_, int OCC_ = 1>
static int launch(const CUtensorMap& ma, const void* B, int N, int K, int ldb, Params p, int max_ctas, int sk_per,
                  cudaStream_t stream, int* ctas_out) {
  using Cf = Cfg<BN_, OCC_>;
  CUtensorMap mb;
  if (int rc = encode_kmajor(&mb, B, N, K, ldb, BN_)) return rc;
  p.n_tiles = (N + BN_ - 1) / BN_;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int cap = max_ctas > 0 ? tmin(max_ctas, sms) : sms;
  const int k_blocks = (K + BK - 1) / BK;
  const int tiles = p.m_tiles * p.n_tiles;
  int grid = tiles < cap ? tiles : cap;
  if (sk_per > 0) {
    p.streamk = 1;
    p.sk_per = sk_per;
    p.sk_total = tiles * k_blocks;
    grid = (p.sk_total + sk_per - 1) / sk_per;   // p.counters / p.ws split in gemm_impl
  }
  static bool attr_set[64] = {};
  p.a_stage = (p.a_bytes + 1023) / 1024 * 1024;
  p.stages = ring_stages(p.a_stage, Cf::B_BYTES, Cf::SMEM_BYTES);
  if (dev < 64 && !attr_set[dev]) {
    cudaError_t e =
        cudaFuncSetAttribute(k_gemm_bf16<BN_, OCC_>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::SMEM_BYTES);
    if (e != cudaSuccess) return bz_fail_cuda(e, "gemm smem attribute");
    attr_set[dev] = true;
  }
  cudaError_t e =
      launch_pdl(PDL_GEMM, k_gemm_bf16<BN_, OCC_>, dim3(grid), dim3(THREADS), Cf::SMEM_BYTES, stream, ma, mb, p);
  if (e != cudaSuccess) return bz_fail_cuda(e, "bz_gemm_bf16 launch");
  if (ctas_out) *ctas_out = grid;
  return bz_check_launch("bz_gemm_bf16");
}

template <int BN_, int NSUB_>
static int launch_pair(const CUtensorMap& ma, const void* B, int N, int K, int ldb, Params p, int max_ctas,
                       int ksplit, cudaStream_t stream, int* ctas_out) {
  using Cf = CfgPair<BN_, NSUB_>;
  CUtensorMap mb;
  if (int rc = encode_kmajor(&mb, B, N, K, ldb, BN_ / 2)) return rc;
  p.n_tiles = (N + Cf::TILE_N - 1) / Cf::TILE_N;
  const int k_blocks = (K + BK - 1) / BK;
  p.kb_slice = (k_blocks + ksplit - 1) / ksplit;
  p.ksplit = (k_blocks + p.kb_slice - 1) / p.kb_slice;   // no empty slice
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int cap = (max_ctas > 0 ? tmin(max_ctas, sms) : sms) / 2;
  int clusters = p.m_tiles * p.n_tiles * p.ksplit;
  if (clusters > cap) clusters = cap;
  if (clusters < 1) clusters = 1;
  static bool attr_set[64] = {};
  if (dev < 64 && !attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(k_gemm_bf16_pair<BN_, NSUB_>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Cf::SMEM_BYTES);
    if (e != cudaSuccess) return bz_fail_cuda(e, "gemm pair smem attribute");
    attr_set[dev] = true;
  }
  cudaError_t e = launch_pdl(PDL_GEMM, k_gemm_bf16_pair<BN_, NSUB_>, dim3(2 * clusters), dim3(THREADS),
                             Cf::SMEM_BYTES, stream, ma, mb, p);
  if (e != cudaSuccess) return bz_fail_cuda(e, "bz_gemm_bf16 (pair) launch");
  if (ctas_out) *ctas_out = 2 * clusters;
  if (p.ksplit > 1) {
    const int64_t groups = static_cast<int64_t>(p.M) * (N / 8);
    const int blocks = static_cast<int>(tmin<int64_t>((groups + 255) / 256, 4 * sms));
    e = launch_pdl(PDL_GEMM, k_splitk_reduce, dim3(blocks), dim3(256), 0, stream, static_cast<const float*>(p.ws),
                   p.ksplit, p.M, N, p.C, p.ldc, p.R, p.ldr, p.signal);
    if (e != cudaSuccess) return bz_fail_cuda(e, "bz_gemm_bf16 (split-K reduce) launch");
    if (ctas_out) *ctas_out = blocks;
  }
  return bz_check_launch("bz_gemm_bf16 (pair)");
}

// ===========================================================================
// Decode GEMMs (M <= 16) with the operands swapped: D^T[n][m] = W[n, :] . X[m, :].
// A 128-row weight tile is the MMA's M operand and the (zero-padded) 16 token rows
// are its N, so one tcgen05.mma consumes 4 KiB of weights; with the tokens as M a
// 128 x 32 instruction consumed 1 KiB and the MMA issue rate, not HBM, bounded the
// narrow tiles decode needs for chip fill (profiles/r2_fused_decode.txt: K-chunked
// BN = 32 streams 5.6-6.6 TB/s without its MMAs, half that with them).  A cluster
// of S CTAs splits K of one tile; the S fp32 partials meet in distributed shared
// memory (no workspace, no fix-up pass) and rank r stores rows [r*128/S, (r+1)*128/S).
// One (tile, K range) per CTA; grid = tiles x S <= SMs.
constexpr int SW_ROWS = 128, SW_TOK = 16, SW_KCH = 2;

__device__ __forceinline__ float ld_cluster_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
  return v;
}

// C[m][n] (+ R[m][n]) for one element of the transposed accumulator
__device__ __forceinline__ void store_swapped(const Params& p, int m, int n, float v) {
  if (n >= p.N) return;
  if (p.R) v += __bfloat162float(p.R[static_cast<int64_t>(m) * p.ldr + n]);
  if (p.c_f32)
    reinterpret_cast<float*>(p.C)[static_cast<int64_t>(m) * p.ldc + n] = v;
  else
    p.C[static_cast<int64_t>(m) * p.ldc + n] = __float2bfloat16_rn(v);
}

template <int S>
__global__ void __cluster_dims__(S, 1, 1) __launch_bounds__(THREADS, 1)
    k_gemm_swap(const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_x, Params p) {
  constexpr int W_STG = SW_KCH * SW_ROWS * 128, X_STG = SW_KCH * SW_TOK * 128;
  const int STAGES = p.stages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sw = smem;                                   // STAGES x W_STG
  uint8_t* sx = smem + STAGES * W_STG;                  // STAGES x X_STG
  float* red = reinterpret_cast<float*>(sx + STAGES * X_STG);  // [SW_TOK][SW_ROWS] fp32 partial
  uint64_t* full = reinterpret_cast<uint64_t*>(red + SW_TOK * SW_ROWS);
  uint64_t* empty = full + MAX_STAGES;
  uint64_t* acc_full = empty + MAX_STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = S == 1 ? 0 : static_cast<int>(cluster_ctarank());
  const int tile = blockIdx.x / S;
  const int k_blocks = p.K / BK;
  const int chunks = (k_blocks + SW_KCH - 1) / SW_KCH;
  const int c0 = rank * chunks / S, nks = (rank + 1) * chunks / S - c0;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&map_w);
    prefetch_tmap(&map_x);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&acc_full[0], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // weights are static: the first stages go out before pdl_wait, overlapping the
      // predecessor; the activations follow once its writes are visible
      const int pre = p.b_static ? min(STAGES, nks) : 0;
      for (int i = 0; i < pre; ++i) {
        mbar_expect_tx(&full[i], W_STG + X_STG);
        tma_load_3d(sw + i * W_STG, &map_w, 0, tile * SW_ROWS, (c0 + i) * SW_KCH, &full[i]);
      }
      pdl_wait();
      for (int i = 0; i < pre; ++i) tma_load_3d(sx + i * X_STG, &map_x, 0, 0, (c0 + i) * SW_KCH, &full[i]);
      uint32_t stage = pre % STAGES, phase = pre == STAGES ? 1u : 0u;
      for (int ks = pre; ks < nks; ++ks) {
        mbar_wait(&empty[stage], phase ^ 1);
        mbar_expect_tx(&full[stage], W_STG + X_STG);
        tma_load_3d(sw + stage * W_STG, &map_w, 0, tile * SW_ROWS, (c0 + ks) * SW_KCH, &full[stage]);
        tma_load_3d(sx + stage * X_STG, &map_x, 0, 0, (c0 + ks) * SW_KCH, &full[stage]);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      pdl_trigger();
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = instr_desc_bf16(SW_ROWS, SW_TOK);
      uint32_t stage = 0, phase = 0;
      for (int ks = 0; ks < nks; ++ks) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const int subs = min(SW_KCH, k_blocks - (c0 + ks) * SW_KCH);
        for (int sub = 0; sub < subs; ++sub) {
          const uint64_t da = umma_desc_sw128(smem_u32(sw + stage * W_STG + sub * SW_ROWS * 128));
          const uint64_t db = umma_desc_sw128(smem_u32(sx + stage * X_STG + sub * SW_TOK * 128));
#pragma unroll
          for (int k = 0; k < BK / UMMA_K; ++k)
            umma_bf16(tmem_base, da + 2 * k, db + 2 * k, idesc, (ks != 0 || sub != 0 || k != 0) ? 1u : 0u);
        }
        umma_commit(&empty[stage]);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      umma_commit(&acc_full[0]);
    }
  } else if (warp >= 4) {
    pdl_wait();  // reads the residual and writes C
    const int row = (warp & 3) * 32 + lane;  // TMEM lane = weight row of the tile
    mbar_wait(&acc_full[0], 0);
    tc_fence_after();
    uint32_t r[32];  // columns 0..15 = tokens
    tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>((warp & 3) * 32) << 16), r);
    if (S == 1) {
      for (int m = 0; m < p.M; ++m) store_swapped(p, m, tile * SW_ROWS + row, __uint_as_float(r[m]));
    } else {
#pragma unroll
      for (int m = 0; m < SW_TOK; ++m) red[m * SW_ROWS + row] = __uint_as_float(r[m]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem_base));
  }
  if (S > 1) {
    cluster_sync_all();  // every rank's partial is in its shared memory
    const int r0 = rank * SW_ROWS / S, per = (rank + 1) * SW_ROWS / S - r0;
    for (int idx = threadIdx.x; idx < per * p.M; idx += THREADS) {
      const int m = idx / per, j = r0 + idx % per;
      const uint32_t a = smem_u32(red + m * SW_ROWS + j);
      float v = 0.f;
#pragma unroll
      for (int q = 0; q < S; ++q) v += ld_cluster_f32(mapa_cta(a, q));  // fixed order: deterministic
      store_swapped(p, m, tile * SW_ROWS + j, v);
    }
    cluster_sync_all();  // no rank leaves while a peer still reads its partial
  }
  if (p.signal != nullptr && threadIdx.x == 0) {
    __threadfence_system();
    asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(p.signal) : "memory");
  }
}

// 3-D view {64 k, rows, K / 64} of a K-major [rows, K] bf16 operand (K % 64 == 0): one box
// {64, box_rows, kch} is kch 128B-swizzled [box_rows x 64] tiles side by side
static int encode_kc3d(CUtensorMap* map, const void* ptr, int rows, int k, int ld, int box_rows, int kch) {
  const DriverApi* d = driver_api();
  if (!d) return BZ_ECUDA;
  cuuint64_t dims[3] = {64, static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(k / 64)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld) * 2, 128};
  cuuint32_t box[3] = {64, static_cast<cuuint32_t>(box_rows), static_cast<cuuint32_t>(kch)};
  cuuint32_t elem[3] = {1, 1, 1};
  CUresult r = d->cuTensorMapEncodeTiled(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims,
                                         strides, box, elem, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return bz_fail_cu(r, "cuTensorMapEncodeTiled (3-D)");
  return BZ_OK;
}

// BZ_GEMM_KC=0 turns the K-chunked decode kernel off (A/B checks); default on for M <= 16
static int kc_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BZ_GEMM_KC");
    v = e ? (atoi(e) != 0) : 1;
  }
  return v;
}

template <int BN_>
static int launch_kc(const void* A, const void* B, int M, int N, int K, int lda, int ldb, Params p, int max_ctas,
                     cudaStream_t stream, int* ctas_out) {
  const int a_rows = (M + 7) / 8 * 8;
  int kch = 32768 / (BN_ * 128);  // ~32 KiB of weights per stage
  kch = kch < 1 ? 1 : kch > 8 ? 8 : kch;
  CUtensorMap ma, mb;
  if (int rc = encode_kc3d(&ma, A, M, K, lda, a_rows, kch)) return rc;
  if (int rc = encode_kc3d(&mb, B, N, K, ldb, BN_, kch)) return rc;
  p.m_tiles = 1;
  p.n_tiles = (N + BN_ - 1) / BN_;
  const int stage_bytes = kch * (a_rows + BN_) * 128;
  const int stages = (SMEM_LIMIT - 1024 - BAR_BYTES) / stage_bytes;
  p.stages = stages < MAX_STAGES ? stages : MAX_STAGES;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int cap = max_ctas > 0 ? tmin(max_ctas, sms) : sms;
  const int grid = p.n_tiles < cap ? p.n_tiles : cap;
  static bool attr_set[64] = {};
  if (dev < 64 && !attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(k_gemm_skinny_kc<BN_>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_LIMIT);
    if (e != cudaSuccess) return bz_fail_cuda(e, "gemm (K-chunked) smem attribute");
    attr_set[dev] = true;
  }
  cudaError_t e = launch_pdl(PDL_GEMM, k_gemm_skinny_kc<BN_>, dim3(grid), dim3(THREADS), SMEM_LIMIT, stream, ma, mb,
                             p, kch, a_rows);
  if (e != cudaSuccess) return bz_fail_cuda(e, "bz_gemm_bf16 (K-chunked) launch");
  if (ctas_out) *ctas_out = grid;
  return bz_check_launch("bz_gemm_bf16 (K-chunked)");
}

// BZ_GEMM_SWAP=0 turns the swapped decode kernel off (A/B checks); default on
static int swap_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BZ_GEMM_SWAP");
    v = e ? (atoi(e) != 0) : 1;
  }
  return v;
}

template <int S>
static int launch_swap(const void* A, const void* B, int M, int N, int K, int lda, int ldb, Params p,
                       cudaStream_t stream, int* ctas_out) {
  CUtensorMap mw, mx;
  if (int rc = encode_kc3d(&mw, B, N, K, ldb, SW_ROWS, SW_KCH)) return rc;
  if (int rc = encode_kc3d(&mx, A, M, K, lda, SW_TOK, SW_KCH)) return rc;
  p.n_tiles = (N + SW_ROWS - 1) / SW_ROWS;
  const int stage_bytes = SW_KCH * (SW_ROWS + SW_TOK) * 128;
  const int fixed = 1024 + SW_TOK * SW_ROWS * 4 + BAR_BYTES;
  int stages = (SMEM_LIMIT - fixed) / stage_bytes;
  if (const char* e = getenv("BZ_GEMM_SWAP_STAGES")) stages = tmin(stages, atoi(e) > 0 ? atoi(e) : 1);
  p.stages = tmin(stages, MAX_STAGES);
  const int smem = fixed + p.stages * stage_bytes;
  int dev = 0;
  cudaGetDevice(&dev);
  static bool attr_set[64] = {};
  if (dev < 64 && !attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(k_gemm_swap<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_LIMIT);
    if (e != cudaSuccess) return bz_fail_cuda(e, "gemm (swapped) smem attribute");
    attr_set[dev] = true;
  }
  const int grid = p.n_tiles * S;
  cudaError_t e = launch_pdl(PDL_GEMM, k_gemm_swap<S>, dim3(grid), dim3(THREADS), smem, stream, mw, mx, p);
  if (e != cudaSuccess) return bz_fail_cuda(e, "bz_gemm_bf16 (swapped) launch");
  if (ctas_out) *ctas_out = grid;
  return bz_check_launch("bz_gemm_bf16 (swapped)");
}

// BZ_GEMM_OCC=2 runs skinny (M <= 128) GEMMs two CTAs per SM (BN <= 128, half the smem
// ring); default one: at decode batch 1..64 the pair measured 5-10 % slower per 7B block
// (profiles/r2_gemm_occ2.txt)
static int occ_override() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BZ_GEMM_OCC");
    v = e ? atoi(e) : 0;
    if (v != 1 && v != 2) v = 0;
  }
  return v;
}

// BZ_GEMM_PAIR=0 forces single-CTA tiles, =1 forces CTA pairs; default: pairs when M >= 256
static int pair_override() {
  static int v = -2;
  if (v == -2) {
    const char* e = getenv("BZ_GEMM_PAIR");
    v = e ? atoi(e) : -1;
  }
  return v;
}

// BZ_GEMM_PAIR_SPLIT=0 disables the pair kernel's split-K (A/B checks); unset: model
static int split_override() {
  static int v = -2;
  if (v == -2) {
    const char* e = getenv("BZ_GEMM_PAIR_SPLIT");
    v = e ? atoi(e) : -1;
  }
  return v;
}

// BZ_GEMM_NSUB=1|2 pins the pair kernel's sub-tiles per A stage (tests); 0 = model
static int nsub_override() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BZ_GEMM_NSUB");
    v = e ? atoi(e) : 0;
    if (v != 1 && v != 2) v = 0;
  }
  return v;
}

// Pair-kernel tile choice from measured per-K-block times (scripts/gemm_bench.py
// with BZ_GEMM_BN / BZ_GEMM_NSUB pinned, 7B block shapes at 2000 tokens; see
// profiles/r1_gemm_pair_configs.txt).  The kernel is bound by the smem feed (with
// its loads elided it runs at 1.9 PFLOP/s), so wider tiles pay less per MAC;
// NSUB = 2 (one TMEM buffer) additionally exposes ~3.8 us of epilogue per tile
// (two TMEM loads in flight per epilogue warp).  Minimise waves x (K blocks x t_kb + exposed).
struct PairPlan {
  int bn, nsub;
  double kb_s, tile_s;
  int ksplit;
  double t = 0.0;  // predicted seconds
};
static PairPlan plan_pair(int m_tiles, int M, int N, int K, int clusters, int only_bn, int only_nsub,
                          int64_t ws_bytes) {
  const PairPlan cands[6] = {{256, 1, 0.368e-6, 0.0, 1},
                             {256, 2, 0.685e-6, 3.8e-6, 1},
                             {240, 1, 0.368e-6, 0.0, 1},  // measured: no faster per K block than 256
                             {192, 1, 0.332e-6, 0.0, 1},
                             {192, 2, 0.600e-6, 3.8e-6, 1},
                             {128, 1, 0.356e-6, 0.0, 1}};  // measured at M = 384-512 (r1_gemm_small_m.txt)
  const int splits[6] = {1, 2, 3, 4, 6, 8};
  const int k_blocks = (K + BK - 1) / BK;
  PairPlan best = cands[0];
  double best_t = 1e30;
  for (const PairPlan& c : cands) {
    if ((only_bn && c.bn != only_bn) || (only_nsub && c.nsub != only_nsub)) continue;
    const int tile_n = c.bn * c.nsub;
    const long tiles = static_cast<long>(m_tiles) * ((N + tile_n - 1) / tile_n);
    for (int sp : splits) {
      if (split_override() > 0 && sp != split_override()) continue;  // pinned (tests, sweeps)
      // split K only to fill the chip (few tiles), into a workspace that holds the partials
      if (sp > 1 && (tiles * sp > clusters || static_cast<int64_t>(sp) * M * N * 4 > ws_bytes ||
                     k_blocks / sp < 8 || split_override() == 0))
        continue;
      const double waves = static_cast<double>((tiles * sp + clusters - 1) / clusters);
      const double slice = static_cast<double>((k_blocks + sp - 1) / sp);
      // partials written by the GEMM and read back by the reduce pass, bf16 written,
      // ~3 us of launch and tail; a split must win by 10 % (the model is rough)
      const double reduce = sp > 1 ? 3e-6 + (8.0 * sp + 2.0) * M * N / 5.0e12 : 0.0;
      const double t = (waves * (slice * c.kb_s + c.tile_s) + reduce) * (sp > 1 ? 1.1 : 1.0);
      if (t < best_t) {
        best_t = t;
        best = c;
        best.ksplit = sp;
        best.t = t;
      }
    }
  }
  return best;
}

// The single-CTA kernel's 128-row tiles fill the chip better when M is not a
// multiple of 256 (e.g. 384 rows: 3 x 48 = 144 tiles of 128 x 256 in one wave vs
// 96 pair tiles in two); per SM it retires a K block of a 128 x BN tile in the
// same ~time as the pair kernel's share.  Returns the predicted seconds and width.
static double single_tile_time(int M, int N, int K, int ctas, int* bn_out) {
  const int widths[3] = {256, 192, 128};
  const double kb_s[3] = {0.368e-6, 0.332e-6, 0.312e-6};
  const int k_blocks = (K + BK - 1) / BK;
  double best = 1e30;
  for (int i = 0; i < 3; ++i) {
    const long tiles = static_cast<long>((M + BM - 1) / BM) * ((N + widths[i] - 1) / widths[i]);
    const double t = static_cast<double>((tiles + ctas - 1) / ctas) * k_blocks * kb_s[i];
    if (t < best) {
      best = t;
      *bn_out = widths[i];
    }
  }
  return best;
}

static int gemm_impl(const void* A, const void* B, void* C, const void* residual, int M, int N, int K, int lda,
                     int ldb, int ldc, int ldr, int max_ctas, unsigned flags, void* workspace, int64_t ws_bytes,
                     uint32_t* signal, int* ctas_out, void* stream) {
  if (!A || !B || !C || M <= 0 || N <= 0 || K <= 0) return bz_fail(BZ_EINVAL, "gemm: bad shape");
  // K tails are zero-filled by TMA (out-of-bounds box columns), so only the
  // 16-byte stride/alignment rules of the tensor maps constrain K.
  if (K % 8 || lda % 8 || ldb % 8 || ldc % 8 || (residual && ldr % 8) || N % 8)
    return bz_fail(BZ_EINVAL, "gemm: K, N and leading dims must be multiples of 8");
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B) | reinterpret_cast<uintptr_t>(C) |
       reinterpret_cast<uintptr_t>(residual)) & 15)
    return bz_fail(BZ_EINVAL, "gemm: operands (and the residual) must be 16-byte aligned");
  // skinny A: load only the rows that exist (8-row swizzle atoms); the rows of
  // the 128-row MMA beyond them read stale smem and are never stored
  const bool c_f32 = (flags & BZ_GEMM_C_F32) != 0;
  if (c_f32 && (reinterpret_cast<uintptr_t>(C) & 15))
    return bz_fail(BZ_EINVAL, "gemm: fp32 C must be 16-byte aligned");
  const int po = pair_override();
  // fp32 C is a single-CTA epilogue feature (logit heads: M = sequences)
  bool pair = !c_f32 && (po == 1 || (po == -1 && M >= 2 * BM));
  int single_bn = 0;
  if (pair && po == -1 && bn_override() == 0) {
    // a pair plan against single-CTA tiles (chip fill), using the pair model's constants
    const int ctas_all = max_ctas > 0 ? tmin(max_ctas, 148) : 148;
    const PairPlan pp = plan_pair((M + 2 * BM - 1) / (2 * BM), M, N, K, ctas_all / 2, 0, nsub_override(),
                                  (workspace && !(reinterpret_cast<uintptr_t>(workspace) & 15) &&
                                   ws_bytes > kCounterHeader) ? ws_bytes - kCounterHeader : 0);
    const double ts = single_tile_time(M, N, K, ctas_all, &single_bn);
    if (ts < pp.t) pair = false;
  }
  const int a_box = (!pair && M < BM) ? (M + 7) / 8 * 8 : BM;
  CUtensorMap ma;
  if (int rc = encode_kmajor(&ma, A, M, K, lda, a_box)) return rc;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int ctas = max_ctas > 0 ? tmin(max_ctas, sms) : sms;
  Params p;
  p.C = static_cast<__nv_bfloat16*>(C);
  p.R = static_cast<const __nv_bfloat16*>(residual);
  p.M = M;
  p.N = N;
  p.K = K;
  p.ldc = ldc;
  p.ldr = ldr;
  p.m_tiles = (M + BM - 1) / BM;
  p.n_tiles = 0;
  p.signal = signal;
  p.ws = static_cast<float*>(workspace);
  p.counters = nullptr;
  p.streamk = 0;
  p.sk_per = 1;
  p.sk_total = 0;
  p.ksplit = 1;
  p.kb_slice = (K + BK - 1) / BK;
  p.a_bytes = a_box * BK * 2;
  p.b_static = (flags & BZ_GEMM_B_STATIC) ? 1 : 0;
  p.c_f32 = c_f32 ? 1 : 0;
  p.kc_nomma = 0;
  if (!workspace || (reinterpret_cast<uintptr_t>(workspace) & 15) || ws_bytes <= kCounterHeader) {
    ws_bytes = 0;
  } else {
    p.counters = static_cast<int*>(workspace);
    p.ws = reinterpret_cast<float*>(static_cast<char*>(workspace) + kCounterHeader);
    ws_bytes -= kCounterHeader;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int forced = bn_override();
  if (pair) {
    p.m_tiles = (M + 2 * BM - 1) / (2 * BM);
    const PairPlan pp = plan_pair(p.m_tiles, M, N, K, ctas / 2, forced, nsub_override(), ws_bytes);
    const int sp = pp.ksplit;
    switch (pp.bn * 10 + pp.nsub) {
      case 1281:
        return launch_pair<128, 1>(ma, B, N, K, ldb, p, max_ctas, sp, s, ctas_out);
      case 1921:
        return launch_pair<192, 1>(ma, B, N, K, ldb, p, max_ctas, sp, s, ctas_out);
      case 1922:
        return launch_pair<192, 2>(ma, B, N, K, ldb, p, max_ctas, sp, s, ctas_out);
      case 2562:
        return launch_pair<256, 2>(ma, B, N, K, ldb, p, max_ctas, sp, s, ctas_out);
      case 2401:
        return launch_pair<240, 1>(ma, B, N, K, ldb, p, max_ctas, sp, s, ctas_out);
      default:
        return launch_pair<256, 1>(ma, B, N, K, ldb, p, max_ctas, sp, s, ctas_out);
    }
  }
  SkinnyPlan plan{forced ? forced : (single_bn ? single_bn : pick_bn(M, N, ctas)), 0};
  // decode shapes: 128-row weight tiles as the MMA's M, K split over a cluster of S
  // CTAs (tiles x S <= SMs, at least two 2-k-block chunks per rank)
  const int sw_tiles = (N + SW_ROWS - 1) / SW_ROWS;
  if (M <= SW_TOK && K % 64 == 0 && swap_enabled() && !forced && sw_tiles <= ctas) {
    const int chunks = (K / BK + SW_KCH - 1) / SW_KCH;
    int S = 1;
    while (S < 8 && sw_tiles * (S + 1) <= ctas && chunks >= 2 * (S + 1)) ++S;
    if (const char* e = getenv("BZ_GEMM_SWAP_S")) S = tmin(atoi(e) > 1 ? atoi(e) : 1, 8);
    switch (S) {
      case 1:
        return launch_swap<1>(A, B, M, N, K, lda, ldb, p, s, ctas_out);
      case 2:
        return launch_swap<2>(A, B, M, N, K, lda, ldb, p, s, ctas_out);
      case 3:
        return launch_swap<3>(A, B, M, N, K, lda, ldb, p, s, ctas_out);
      case 4:
        return launch_swap<4>(A, B, M, N, K, lda, ldb, p, s, ctas_out);
      case 5:
        return launch_swap<5>(A, B, M, N, K, lda, ldb, p, s, ctas_out);
      case 6:
        return launch_swap<6>(A, B, M, N, K, lda, ldb, p, s, ctas_out);
      case 7:
        return launch_swap<7>(A, B, M, N, K, lda, ldb, p, s, ctas_out);
      default:
        return launch_swap<8>(A, B, M, N, K, lda, ldb, p, s, ctas_out);
    }
  }
  // wider decode GEMMs (more 128-row tiles than SMs): whole tiles of about one per SM
  // over K-chunked stages (no stream-K)
  if (M <= 16 && K % 64 == 0 && kc_enabled() && !forced) {
    const int widths[7] = {32, 64, 96, 128, 160, 192, 256};
    int bn = 256;
    for (int w : widths)
      if ((N + w - 1) / w <= ctas) {
        bn = w;
        break;
      }
    if (const char* e = getenv("BZ_GEMM_KC_BN")) bn = atoi(e);
    if (const char* e = getenv("BZ_GEMM_KC_NOMMA")) p.kc_nomma = atoi(e);
    // a tile narrower than 128 is MMA-issue bound here (the swapped kernel covers those
    // shapes); such plans stay on the stream-K path
    if (bn >= 128 || getenv("BZ_GEMM_KC_BN")) switch (bn) {
      case 32:
        return launch_kc<32>(A, B, M, N, K, lda, ldb, p, max_ctas, s, ctas_out);
      case 64:
        return launch_kc<64>(A, B, M, N, K, lda, ldb, p, max_ctas, s, ctas_out);
      case 96:
        return launch_kc<96>(A, B, M, N, K, lda, ldb, p, max_ctas, s, ctas_out);
      case 128:
        return launch_kc<128>(A, B, M, N, K, lda, ldb, p, max_ctas, s, ctas_out);
      case 160:
        return launch_kc<160>(A, B, M, N, K, lda, ldb, p, max_ctas, s, ctas_out);
      case 192:
        return launch_kc<192>(A, B, M, N, K, lda, ldb, p, max_ctas, s, ctas_out);
      default:
        return launch_kc<256>(A, B, M, N, K, lda, ldb, p, max_ctas, s, ctas_out);
    }
  }
  const bool occ2 = M <= BM && occ_override() == 2 && forced <= 128;
  if (M <= BM) {
    plan = plan_skinny(M, N, K, ctas, ws_bytes, forced, occ2 ? 128 : 256);
  }
  if (occ2) {
    switch (plan.bn) {
      case 32:
        return launch<32, 2>(ma, B, N, K, ldb, p, max_ctas, plan.sk_per, s, ctas_out);
      case 64:
        return launch<64, 2>(ma, B, N, K, ldb, p, max_ctas, plan.sk_per, s, ctas_out);
      default:
        return launch<128, 2>(ma, B, N, K, ldb, p, max_ctas, plan.sk_per, s, ctas_out);
    }
  }
  switch (plan.bn) {
    case 32:
      return launch<32>(ma, B, N, K, ldb, p, max_ctas, plan.sk_per, s, ctas_out);
    case 64:
      return launch<64>(ma, B, N, K, ldb, p, max_ctas, plan.sk_per, s, ctas_out);
    case 128:
      return launch<128>(ma, B, N, K, ldb, p, max_ctas, plan.sk_per, s, ctas_out);
    case 192:
      return launch<192>(ma, B, N, K, ldb, p, max_ctas, plan.sk_per, s, ctas_out);
    default:
      return launch<256>(ma, B, N, K, ldb, p, max_ctas, plan.sk_per, s, ctas_out);
  }
}

}  // namespace gemm
}  // namespace bz

using namespace bz;

extern "C" int bz_gemm_bf16(const void* A, const void* B, void* C, const void* residual, int M, int N, int K,
                            int lda, int ldb, int ldc, int ldr, int max_ctas, void* stream) {
  return gemm::gemm_impl(A, B, C, residual, M, N, K, lda, ldb, ldc, ldr, max_ctas, 0u, nullptr, 0, nullptr,
                         nullptr, stream);
}

extern "C" int bz_gemm_bf16_signal(const void* A, const void* B, void* C, const void* residual, int M, int N,
                                   int K, int lda, int ldb, int ldc, int ldr, int max_ctas, uint32_t* signal,
                                   int* ctas_out, void* stream) {
  if (!signal || !ctas_out) return bz_fail(BZ_EINVAL, "gemm_signal: signal and ctas_out required");
  return gemm::gemm_impl(A, B, C, residual, M, N, K, lda, ldb, ldc, ldr, max_ctas, 0u, nullptr, 0, signal,
                         ctas_out, stream);
}

extern "C" int bz_gemm_bf16_ex(const void* A, const void* B, void* C, const void* residual, int M, int N, int K,
                               int lda, int ldb, int ldc, int ldr, int max_ctas, unsigned flags, void* workspace,
                               int64_t workspace_bytes, uint32_t* signal, int* ctas_out, void* stream) {
  if (signal && !ctas_out) return bz_fail(BZ_EINVAL, "gemm_ex: a signal needs ctas_out");
  return gemm::gemm_impl(A, B, C, residual, M, N, K, lda, ldb, ldc, ldr, max_ctas, flags, workspace,
                         workspace_bytes, signal, ctas_out, stream);
}

const void* bz::module_anchor_gemm() { return reinterpret_cast<const void*>(gemm::k_splitk_reduce); }
