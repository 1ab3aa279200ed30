// Causal flash attention for the prefill of a Llama block on sm_100a tensor cores.
//
// The reference stands the whole forward in with ModelSpec.prefill_ms
// (parampool.py:58-62); with the projections on tcgen05 GEMMs (gemm_tcgen05.cu)
// this is the block's other contraction: softmax(Q K^T / sqrt(hd)) V per head,
// causal, GQA (query head h reads kv head h / (H / KV)).
//
//   in : qkv  [B*S, ld]  bf16, row = token, [q heads | k heads | v heads] (RoPE applied)
//        V is read in place: its tiles [128 keys x hd] are the B operand of O += P V in
//        MN-major form (hd contiguous), so no transpose pass and no workspace
//   out: attn [B*S, ldo] bf16, head h at columns [h*hd, (h+1)*hd) -- the o-projection's A
//
// One CTA = two adjacent 128-row query tiles A, B of one (sequence, head): every K / V
// tile it loads feeds two independent softmax streams, and the tensor core works on
// one tile while the other tile's softmax runs (FA4-style ping-pong).  Keys come in
// tiles of 128.  TMEM lane = query row of a tile.
//   w0      TMA producer: Q_A, Q_B once; K_j / V^T_j into 2-deep rings
//   w1      MMA issuer (one lane), per tile X in (A, B): O_X += P_X(j) V_j with P read
//           straight from TMEM (tcgen05.mma A-operand in tensor memory), then
//           S_X(j+1) = Q_X K_{j+1}^T into the same TMEM columns
//   w2..w5  softmax of A, w6..w9 softmax of B (thread = query row): S_X(j) from TMEM,
//           causal mask on the diagonal tile only, running max in the log2 domain,
//           P = exp2(s log2e / sqrt(hd) - m) packed to bf16 and stored back into the
//           first half of S_X's columns (no shared memory traffic for P).  The max is
//           only raised when it grows by more than 2^8 (P <= 256, exact in fp32 /
//           bf16); only then is O rescaled in TMEM (ld, scale, st), warp-uniformly --
//           S_X(j) completing implies O_X += P_X(j-1) V_{j-1} completed (tcgen05 ops
//           execute in issue order), so the rescale needs no extra wait.
//   epilogue: O / l, bf16 rows of the o-projection input.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "../../include/blitz.h"
#include "common.cuh"
#include "tc_primitives.cuh"

namespace bz {
namespace attn {

using namespace bz::tc;

constexpr int BQ = 128;       // query rows per tile (= TMEM lanes)
constexpr int BKV = 128;      // keys per tile
constexpr int THREADS = 320;  // w0 TMA, w1 MMA + TMEM allocator, w2..w5 softmax A, w6..w9 softmax B
constexpr int STAGES = 2;     // K and V rings

template <int HD>
struct Cfg {
  static constexpr int KA = HD / 64;               // 64-wide swizzle atoms along hd
  static constexpr int ROW_ATOM = 128 * 128;       // 128 rows x 128 B
  static constexpr int Q_BYTES = KA * ROW_ATOM;    // one query tile
  static constexpr int K_BYTES = KA * ROW_ATOM;    // 128 keys x hd
  static constexpr int V_BYTES = KA * ROW_ATOM;    // 128 keys x hd, as loaded (hd contiguous)
  static constexpr int BAR_BYTES = 256;   // 18 barriers + the TMEM address
  static constexpr int SMEM = 1024 + 2 * Q_BYTES + STAGES * (K_BYTES + V_BYTES) + BAR_BYTES;
  // TMEM: S_A at [0, 128), S_B at [128, 256) -- P_X (bf16 pairs) in the first 64 columns
  // of S_X once S_X is in registers -- then O_A, O_B (HD columns each)
  static constexpr int S_COL = 0;
  static constexpr int O_COL = 2 * BKV;
  static constexpr int TMEM_COLS = 512;
  static_assert(HD == 64 || HD == 128, "head dim");
  static_assert(SMEM <= 232448, "smem");
};

struct Args {
  __nv_bfloat16* out;
  int ldo;
  int S;          // tokens per sequence
  int H, KV;      // query heads, kv heads
  int q_col0;     // column of q head 0 in qkv (0)
  int k_col0;     // column of k head 0 (H * hd)
  int v_col0;     // column of v head 0 ((H + KV) * hd)
  int B;          // sequences
  float scale_log2;  // log2(e) / sqrt(hd)
};

__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 2^x on the FMA / ALU pipes for x <= 8 (x = -inf gives ~1e-38): round x to the
// nearest integer n with the 1.5 * 2^23 trick, 2^(x - n) by a degree-3 Taylor
// polynomial on [-0.5, 0.5] (relative error < 8e-4, below bf16 2^-9 half-ulp),
// then add n to the exponent field.
__device__ __forceinline__ float ex2_fma(float x) {
  x = fmaxf(x, -126.0f);
  const float t = x + 12582912.0f;
  const float f = x - (t - 12582912.0f);
  float p = fmaf(f, 0.0555041087f, 0.240226507f);
  p = fmaf(f, p, 0.693147181f);
  p = fmaf(f, p, 1.0f);
  const int n = __float_as_int(t) - 0x4B400000;
  return __int_as_float(__float_as_int(p) + (n << 23));
}
__device__ __forceinline__ float max3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ void tmem_st_32x32b_x16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st_32x32b_x32(uint32_t taddr, const uint32_t (&r)[32]) {
  tmem_st_32x32b_x16(taddr, r);
  tmem_st_32x32b_x16(taddr + 16, r + 16);
}
// D[tmem] (+)= A[tmem] . B[smem]: the A operand (M = 128 lanes x K = 16 bf16, two per
// 32-bit column) is read from tensor memory
__device__ __forceinline__ void umma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc,
                                             uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

constexpr float kRescale = 8.0f;  // raise the running max only when it grows by > 2^8

// MN-major, 128B-swizzled operand: rows of 128 B run along K (8-row atoms SBO apart),
// the 64-element row is contiguous along M/N and the next 64 of M/N are LBO away
__device__ __forceinline__ uint64_t umma_desc_mn_sw128(uint32_t smem_addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}

// Timeline probe (scripts/attn_trace.cu compiles this file with BZ_ATTN_TRACE): CTA 0's
// softmax warps and MMA thread stamp %globaltimer at their waits and arrivals.
#ifdef BZ_ATTN_TRACE
__device__ unsigned long long g_trace[4096];
__device__ __forceinline__ void trace(int slot) {
  if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && slot < 4096) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_trace[slot] = t;
  }
}
#define BZ_TRACE(slot) trace(slot)
#else
#define BZ_TRACE(slot)
#endif

template <int HD>
__global__ void __launch_bounds__(THREADS, 1)
    k_flash_prefill(const __grid_constant__ CUtensorMap map_q, Args a) {
  using C = Cfg<HD>;
  constexpr int KA = C::KA;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sq = smem;                              // [2 tiles]
  uint8_t* sk = sq + 2 * C::Q_BYTES;               // [STAGES]
  uint8_t* sv = sk + STAGES * C::K_BYTES;          // [STAGES]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sv + STAGES * C::V_BYTES);
  uint64_t* q_full = bars;          // 1
  uint64_t* k_full = bars + 1;      // [2]
  uint64_t* k_empty = bars + 3;     // [2]
  uint64_t* v_full = bars + 5;      // [2]
  uint64_t* v_empty = bars + 7;     // [2]
  uint64_t* s_full = bars + 9;      // [tile]  S_X(j) in TMEM
  uint64_t* p_full = bars + 11;     // [tile]  P_X(j) in TMEM (and O_X rescaled)
  uint64_t* pv_done = bars + 13;    // [tile]  O_X += P_X(j) V_j complete
  uint64_t* q_empty = bars + 15;    // 1       the item's last S issued: Q smem reusable
  uint64_t* o_free = bars + 16;     // [tile]  the epilogue has read O_X out of TMEM
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 18);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_qt = (a.S + BQ - 1) / BQ;
  const int n_pairs = (n_qt + 1) / 2;
  const int per_pair = a.H * a.B;
  const int n_items = n_pairs * per_pair;
  // Persistent CTAs over work items (one query-tile pair of one (sequence, head)),
  // items ordered longest first and dealt in snake order (round k even: c + k G, odd:
  // (k + 1) G - 1 - c), so every CTA's total is close to the longest item.  Every role
  // walks the same item list; barrier phases run on across items.
  const int G = static_cast<int>(gridDim.x), c = static_cast<int>(blockIdx.x);
  auto item_at = [&](int k) -> int { return (k & 1) ? (k + 1) * G - 1 - c : c + k * G; };
  struct Item { int s0, qt_a, nj_a, nj, h, g, row0; };
  auto decode = [&](int i) {
    Item it;
    const int pair = n_pairs - 1 - i / per_pair;
    const int rem = i % per_pair;
    it.h = rem % a.H;
    const int b = rem / a.H;
    it.g = it.h / (a.H / a.KV);
    it.s0 = pair * 2 * BQ;
    it.qt_a = 2 * pair;
    it.nj_a = it.qt_a + 1;
    it.nj = it.qt_a + 2;
    it.row0 = b * a.S;
    return it;
  };

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&map_q);
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 4);
      mbar_init(&pv_done[i], 1);
      mbar_init(&o_free[i], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer ----
      pdl_wait();  // q/k/v were written by the predecessor (qkv GEMM + RoPE)
      int gk = 0;  // running K/V tile count (ring stage = gk & 1)
      for (int k = 0, i; (i = item_at(k)) < n_items && i >= 0; ++k) {
        const Item it = decode(i);
        mbar_wait(q_empty, (k & 1) ^ 1);
        mbar_expect_tx(q_full, 2 * C::Q_BYTES);
        for (int t = 0; t < 2; ++t)
          for (int ka = 0; ka < KA; ++ka)
            tma_load_2d(sq + t * C::Q_BYTES + ka * C::ROW_ATOM, &map_q, a.q_col0 + it.h * HD + ka * 64,
                        it.row0 + it.s0 + t * BQ, q_full);
        for (int j = 0; j < it.nj; ++j, ++gk) {
          const int st = gk & 1, ph = ((gk >> 1) & 1) ^ 1;
          mbar_wait(&k_empty[st], ph);
          mbar_expect_tx(&k_full[st], C::K_BYTES);
          for (int ka = 0; ka < KA; ++ka)
            tma_load_2d(sk + st * C::K_BYTES + ka * C::ROW_ATOM, &map_q, a.k_col0 + it.g * HD + ka * 64,
                        it.row0 + j * BKV, &k_full[st]);
          mbar_wait(&v_empty[st], ph);
          mbar_expect_tx(&v_full[st], C::V_BYTES);
          for (int ka = 0; ka < KA; ++ka)
            tma_load_2d(sv + st * C::V_BYTES + ka * C::ROW_ATOM, &map_q, a.v_col0 + it.g * HD + ka * 64,
                        it.row0 + j * BKV, &v_full[st]);
        }
      }
      pdl_trigger();
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---- MMA issuer ----
      constexpr uint32_t idesc_s = instr_desc_bf16(BQ, BKV);
      constexpr uint32_t idesc_o = instr_desc_bf16(BQ, HD) | (1u << 16);   // B (V) MN-major
      auto issue_s = [&](int t, int st) {   // S_t = Q_t K^T from ring stage st
        const uint32_t d = tmem + C::S_COL + t * BKV;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint64_t da = umma_desc_sw128(smem_u32(sq + t * C::Q_BYTES + (kk >> 2) * C::ROW_ATOM)) + 2 * (kk & 3);
          const uint64_t db = umma_desc_sw128(smem_u32(sk + st * C::K_BYTES + (kk >> 2) * C::ROW_ATOM)) + 2 * (kk & 3);
          umma_bf16(d, da, db, idesc_s, kk > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[t]);
      };
      auto issue_pv = [&](int t, int st, bool first) {  // O_t (+)= P_t V, P from TMEM
        const uint32_t d = tmem + C::O_COL + t * HD;
        const uint32_t pa = tmem + C::S_COL + t * BKV;
#pragma unroll
        for (int kk = 0; kk < BKV / 16; ++kk) {
          // 16 keys = two 8-key swizzle atoms along K (2048 B); the hd halves 64..127
          // are the next TMA box (LBO = one 128-row atom)
          const uint64_t db = umma_desc_mn_sw128(smem_u32(sv + st * C::V_BYTES) + kk * 2048, C::ROW_ATOM, 1024);
          umma_bf16_ts(d, pa + kk * 8, db, idesc_o, (!first || kk > 0) ? 1u : 0u);
        }
        umma_commit(&pv_done[t]);
      };
      int gk = 0;              // running K/V tile count
      int up[2] = {0, 0};      // P(j) uses per tile (p_full phases)
      for (int k = 0, i; (i = item_at(k)) < n_items && i >= 0; ++k) {
        const Item it = decode(i);
        mbar_wait(q_full, k & 1);
        mbar_wait(&k_full[gk & 1], (gk >> 1) & 1);
        tc_fence_after();
        issue_s(0, gk & 1);
        issue_s(1, gk & 1);
        umma_commit(&k_empty[gk & 1]);
        for (int j = 0; j < it.nj; ++j) {
          const int g0 = gk + j, st = g0 & 1;
          mbar_wait(&v_full[st], (g0 >> 1) & 1);
          const bool more = j + 1 < it.nj;
          if (more) mbar_wait(&k_full[(g0 + 1) & 1], ((g0 + 1) >> 1) & 1);
          for (int t = 0; t < 2; ++t) {
            if (t == 0 && j >= it.nj_a) continue;          // tile A is done after its diagonal
            BZ_TRACE(2048 + 8 * j + 2 * t);
            mbar_wait(&p_full[t], up[t] & 1);
            BZ_TRACE(2048 + 8 * j + 2 * t + 1);
            ++up[t];
            // the previous item's epilogue must have read O_t before it is overwritten
            if (j == 0) mbar_wait(&o_free[t], (k & 1) ^ 1);
            tc_fence_after();
            issue_pv(t, st, j == 0);
            if (more && !(t == 0 && j + 1 >= it.nj_a)) issue_s(t, (g0 + 1) & 1);
          }
          umma_commit(&v_empty[st]);
          if (more) umma_commit(&k_empty[(g0 + 1) & 1]);
          if (j + 2 == it.nj) umma_commit(q_empty);  // S_B(nj-1) was the item's last S
        }
        gk += it.nj;
      }
    }
  } else {
    // ---- softmax of tile t (thread = query row r) ----
    const int t = (warp - 2) >> 2;           // 0 = A, 1 = B
    const int quarter = warp & 3;            // TMEM lane quarter (hardware: warp id % 4)
    const int r = quarter * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    const uint32_t s_addr = tmem + lane_off + C::S_COL + t * BKV;
    const uint32_t o_addr = tmem + lane_off + C::O_COL + t * HD;
    int us = 0;                              // S / P uses of this tile (phases)
    for (int k = 0, i; (i = item_at(k)) < n_items && i >= 0; ++k) {
      const Item it = decode(i);
      const int qpos = it.s0 + t * BQ + r;   // query position in its sequence
      const int my_nj = t == 0 ? it.nj_a : it.nj;
      const int diag = it.qt_a + t;
      float m = -INFINITY;                   // running max in use (log2 domain)
      float l = 0.f;                         // row sum relative to m
      for (int j = 0; j < my_nj; ++j, ++us) {
        if (lane == 0 && quarter == 2 && k == 0) BZ_TRACE(1024 * t + 4 * j);
        mbar_wait(&s_full[t], us & 1);
        if (lane == 0 && quarter == 2 && k == 0) BZ_TRACE(1024 * t + 4 * j + 1);
        tc_fence_after();
        uint32_t v[4][32];
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) tmem_ld_32x32b_x32_async(s_addr + 32 * cc, v[cc]);
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) tmem_wait_ld(v[cc]);
        if (j == diag) {  // causal mask: keys after this query get -inf
          const int key0 = j * BKV;
#pragma unroll
          for (int cc = 0; cc < 4; ++cc)
#pragma unroll
            for (int q = 0; q < 32; ++q)
              if (key0 + 32 * cc + q > qpos) v[cc][q] = __float_as_uint(-INFINITY);
        }
        // row max: four independent FMNMX3 chains (latency, not throughput, bounds them)
        float mxc[4];
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          mxc[cc] = -INFINITY;
#pragma unroll
          for (int q = 0; q < 32; q += 2)
            mxc[cc] = max3(mxc[cc], __uint_as_float(v[cc][q]), __uint_as_float(v[cc][q + 1]));
        }
        const float mx = fmaxf(fmaxf(mxc[0], mxc[1]), fmaxf(mxc[2], mxc[3])) * a.scale_log2;
        // raise the max only when it grows by more than 2^kRescale: O and l are then
        // scaled by 2^(m_old - m_new).  tcgen05.ld/st are warp-collective, so the warp
        // rescales whenever any of its rows must (alpha = 1 on the others).  O holds
        // P(j-1) V_{j-1} already: S(j) was issued after that MMA.
        const bool raise = mx > m + kRescale;
        if (__any_sync(0xffffffffu, raise)) {
          const float alpha = raise ? ex2(m - mx) : 1.f;   // 0 on the first tile
          if (j > 0) {
#pragma unroll
            for (int cc = 0; cc < HD; cc += 32) {
              uint32_t o[32];
              tmem_ld_32x32b_x32(o_addr + cc, o);
#pragma unroll
              for (int q = 0; q < 32; ++q) o[q] = __float_as_uint(__uint_as_float(o[q]) * alpha);
              tmem_st_32x32b_x32(o_addr + cc, o);
            }
          }
          l *= alpha;
          if (raise) m = mx;
        }
        // P = exp2(s * scale - m) as bf16 pairs into the first 64 columns of S_t; eight
        // partial sums (short FADD chains).  (Moving a quarter of the exponentials to the
        // FMA pipe with ex2_fma was measured 7 % slower: MUFU is not the limiter.)
        float sum[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) sum[q] = 0.f;
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          uint32_t w[16];
#pragma unroll
          for (int q = 0; q < 32; q += 2) {
            const float p0 = ex2(fmaf(__uint_as_float(v[cc][q]), a.scale_log2, -m));
            const float p1 = ex2(fmaf(__uint_as_float(v[cc][q + 1]), a.scale_log2, -m));
            sum[(q >> 1) & 7] += p0 + p1;
            w[q >> 1] = pack2(p0, p1);
          }
          tmem_st_32x32b_x16(s_addr + 16 * cc, w);
        }
        l += ((sum[0] + sum[1]) + (sum[2] + sum[3])) + ((sum[4] + sum[5]) + (sum[6] + sum[7]));
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[t]);
        if (lane == 0 && quarter == 2 && k == 0) BZ_TRACE(1024 * t + 4 * j + 2);
      }
      // ---- epilogue: O / l -> bf16; O is handed back to the MMA once read ----
      mbar_wait(&pv_done[t], (us - 1) & 1);
      tc_fence_after();
      const float inv = 1.f / l;
      uint32_t o[HD / 32][32];
#pragma unroll
      for (int cc = 0; cc < HD / 32; ++cc) tmem_ld_32x32b_x32_async(o_addr + 32 * cc, o[cc]);
#pragma unroll
      for (int cc = 0; cc < HD / 32; ++cc) tmem_wait_ld(o[cc]);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_free[t]);
      if (qpos < a.S) {
        __nv_bfloat16* dst = a.out + static_cast<int64_t>(it.row0 + qpos) * a.ldo + it.h * HD;
#pragma unroll
        for (int q = 0; q < HD; q += 8) {
          const float* f = reinterpret_cast<const float*>(&o[q >> 5][q & 31]);
          *reinterpret_cast<uint4*>(dst + q) =
              make_uint4(pack2(f[0] * inv, f[1] * inv), pack2(f[2] * inv, f[3] * inv),
                         pack2(f[4] * inv, f[5] * inv), pack2(f[6] * inv, f[7] * inv));
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::TMEM_COLS));
  }
}

static int encode(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld_elems, int box_cols,
                  int box_rows) {
  const DriverApi* d = driver_api();
  if (!d) return BZ_ECUDA;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld_elems) * 2};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t elem[2] = {1, 1};
  CUresult r = d->cuTensorMapEncodeTiled(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims,
                                         strides, box, elem, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return bz_fail_cu(r, "attention: cuTensorMapEncodeTiled");
  return BZ_OK;
}

template <int HD>
static int launch(const void* qkv, int ld, int B, int S, int H, int KV, void* out, int ldo, cudaStream_t s) {
  using C = Cfg<HD>;
  CUtensorMap mq;
  const int cols = (H + 2 * KV) * HD;
  if (int rc = encode(&mq, qkv, static_cast<int64_t>(B) * S, cols, ld, 64, BQ)) return rc;   // Q, K and V tiles
  int dev = 0;
  cudaGetDevice(&dev);
  static bool attr_set[64] = {};
  if (dev < 64 && !attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(k_flash_prefill<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return bz_fail_cuda(e, "attention smem attribute");
    attr_set[dev] = true;
  }
  Args a;
  a.out = static_cast<__nv_bfloat16*>(out);
  a.ldo = ldo;
  a.S = S;
  a.H = H;
  a.KV = KV;
  a.q_col0 = 0;
  a.k_col0 = H * HD;
  a.v_col0 = (H + KV) * HD;
  a.scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(HD));
  a.B = B;
  const int n_qt = (S + BQ - 1) / BQ;
  const int items = (n_qt + 1) / 2 * H * B;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e = launch_pdl(PDL_ATTN, k_flash_prefill<HD>, dim3(items < sms ? items : sms), dim3(THREADS), C::SMEM,
                             s, mq, a);
  if (e != cudaSuccess) return bz_fail_cuda(e, "attention launch");
  return bz_check_launch("bz_prefill_attention");
}

}  // namespace attn
}  // namespace bz

using namespace bz;

extern "C" int bz_prefill_attention_workspace_bytes(int B, int S, int KV, int head_dim, int64_t* bytes) {
  if (!bytes || B < 1 || S < 1 || KV < 1 || (head_dim != 64 && head_dim != 128))
    return bz_fail(BZ_EINVAL, "prefill attention workspace: bad sizes");
  *bytes = 0;   // V is read in place (MN-major operand); kept for ABI stability
  return BZ_OK;
}

extern "C" int bz_prefill_attention(const void* qkv, int ld, int B, int S, int n_heads, int n_kv, int head_dim,
                                    void* /*workspace*/, int64_t /*workspace_bytes*/, void* out, int ldo, void* stream) {
  if (!qkv || !out || B < 1 || S < 1 || n_kv < 1 || n_heads % n_kv)
    return bz_fail(BZ_EINVAL, "prefill attention: bad arguments");
  if (head_dim != 64 && head_dim != 128) return bz_fail(BZ_EINVAL, "prefill attention: head_dim must be 64 or 128");
  if (ld % 8 || ldo % 8 || (reinterpret_cast<uintptr_t>(qkv) & 15) || (reinterpret_cast<uintptr_t>(out) & 15))
    return bz_fail(BZ_EINVAL, "prefill attention: 16-byte aligned pointers and leading dims required");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (head_dim == 128) return attn::launch<128>(qkv, ld, B, S, n_heads, n_kv, out, ldo, s);
  return attn::launch<64>(qkv, ld, B, S, n_heads, n_kv, out, ldo, s);
}

const void* bz::module_anchor_attention() { return reinterpret_cast<const void*>(attn::k_flash_prefill<128>); }
