// Whole decode step in ONE persistent kernel for small batches (1..4 sequences):
// every block of [first, last) -- rmsnorm, qkv, RoPE + KV append, attention,
// o-proj + residual, rmsnorm, gate/up + SiLU, down + residual -- without a kernel
// boundary.  Decode at batch 1 is a weight stream (7B: 404 MB per block, 0.3 MFLOP
// per MB), so the kernel is organised around keeping HBM busy:
//
//   * warp 8 of every CTA is a producer that streams THIS CTA's fixed slice of each
//     weight matrix (16-row units) through a ring of 16 KiB shared-memory slots with
//     3-D TMA tensor copies (16 rows x 512 k, 128B-swizzled, L2 evict-first), block
//     after block, never waiting for activations -- weights do not depend on them, so
//     the stream runs straight through every phase boundary and grid barrier;
//   * warps 0..7 consume slots: one warp owns a 16-row unit and forms its rows . x
//     products with warp-level tensor-core MMAs (mma.sync m16n8k16, weights as the
//     16-row A operand via ldmatrix, the 1..4 sequences as the n=8 B operand, fp32
//     accumulators): 8 instructions per 256 weights.  A CUDA-core dot product (FFMA2)
//     needed ~30 and left the warps latency-bound below the HBM rate.  (tcgen05 would
//     need a 128-row tile and TMEM for a 1..4-column product; at this arithmetic
//     intensity the legacy warp MMA is not the bound.)
//   * phases that need the whole previous result are separated by a grid barrier
//     (5 per block); the per-CTA inputs (rmsnorm of the residual, the attention
//     combine) are recomputed redundantly by every CTA into shared memory, which
//     costs L2 reads instead of extra barriers.
//
// The separate-kernel path (decode_block: 4 tcgen05 GEMMs + 6 glue kernels per
// block) pays each GEMM's ramp and stream-K tail: 106 us per 7B block at batch 1
// (0.60 of HBM); here the stream only pauses when the ring is full.
//
// Numerics follow the separate-kernel path rounding for rounding: h, qkv, RoPE'd
// q/k, attention output, o, h2, gate, up, act and the block output are rounded to
// bf16 exactly where those kernels store bf16; only the fp32 summation order differs.
//
// Reference: the decode step the reference models as decode_step_ms
// (parampool.py:58-62) and runs on a mutated prefill instance (livescale.py:512-544).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>
#include <stdlib.h>

#include "../../include/blitz.h"
#include "common.cuh"
#include "tc_primitives.cuh"

namespace bz {
namespace fused {

using namespace bz::tc;

constexpr int CW = 8;                     // consumer (compute) warps
constexpr int CT = CW * 32;               // consumer threads
constexpr int THREADS = CT + 32;          // + one producer warp
constexpr int SLOT = 16384;               // bytes per ring slot
constexpr int MAX_SLOTS = 16;
constexpr int MAX_ROWS = 4;               // sequences per step
constexpr int UROWS = 16;                 // weight rows per unit (one m16 MMA tile)
constexpr int SLOT_K = 512;               // k per slot: 8 x 64-element swizzle rows
constexpr int GMAX = 8;                   // query heads per kv head
constexpr int CHUNK_MAX = 512;            // context tokens per attention item
constexpr int NSPLIT_CAP = 256;           // context chunks per (sequence, head)
constexpr int MAX_BLOCKS = 48;           // per launch (tensor maps live in the 32 KB parameter space)
constexpr int SMEM_MAX = 232448;
constexpr uint64_t SPIN_NS = 4000000000ull;  // grid-barrier timeout (a missing CTA = a bug)

struct Block {
  const __nv_bfloat16 *attn_norm, *wqkv, *wo, *ffn_norm, *wgu, *wdown;
  __nv_bfloat16 *kc, *vc;
};

// tensor maps per block: wqkv, wo, wgu (gate rows then up rows), wdown -- each viewed as
// 3-D {64 k, rows, k / 64} so one copy brings 16 rows x 512 k as 8 swizzled 2 KiB tiles
enum { TM_QKV, TM_O, TM_GU, TM_DOWN, TM_N };

struct Params {
  CUtensorMap tm[MAX_BLOCKS][TM_N];
  Block blk[MAX_BLOCKS];
  int n_blocks, d, H, KV, ffn, nqkv, ldx;
  float log2_theta, eps, scale;
  int64_t s_max;
  const int32_t* pos;
  int pos_stride;
  __nv_bfloat16* x;        // [rows, ldx] hidden in / out
  unsigned* bar;           // [0] arrivals, [1] generation, [2] error
  __nv_bfloat16* qkv;      // [rows, nqkv]
  __nv_bfloat16* o;        // [rows, d]
  __nv_bfloat16* act;      // [rows, ffn]
  float* part;             // [rows * H, NSPLIT_CAP, hd]  unnormalised o of each context chunk
  float* pml;              // [rows * H, NSPLIT_CAP, 2]   its (max, sum)
  int nslot;
  int nomath;              // diagnostics (BZ_FUSED_NOMATH=1): consume slots without the dot products
  int region_bytes;        // activation / attention scratch region
  uint64_t* trace;         // optional: %globaltimer per CTA per event (bz_decode_fused_set_trace)
};

// trace events per block (consumer thread 0 unless noted)
enum { EV_START, EV_NORM1, EV_QKV, EV_BAR1, EV_ATTN, EV_BAR2, EV_COMB, EV_O, EV_BAR3, EV_NORM2, EV_GU, EV_BAR4,
       EV_ACT, EV_DOWN, EV_PROD_QKV, EV_PROD_O, EV_PROD_GU, EV_PROD_DOWN, EV_A_Q, EV_A_S, EV_A_SM, EV_A_PV, EV_N };
__device__ __forceinline__ void trace_ev(const Params& p, int l, int ev);

// ---- small PTX helpers ------------------------------------------------------------------
__device__ __forceinline__ void named_sync() { asm volatile("bar.sync 1, %0;" ::"n"(CT) : "memory"); }
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ float bf_lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf_hi(uint32_t v) { return __uint_as_float(v & 0xffff0000u); }
__device__ __forceinline__ float bf16r(float v) { return __bfloat162float(__float2bfloat16_rn(v)); }
__device__ __forceinline__ void unpack8(const uint4& v, float (&f)[8]) {
  f[0] = bf_lo(v.x), f[1] = bf_hi(v.x), f[2] = bf_lo(v.y), f[3] = bf_hi(v.y);
  f[4] = bf_lo(v.z), f[5] = bf_hi(v.z), f[6] = bf_lo(v.w), f[7] = bf_hi(v.w);
}
__device__ __forceinline__ void tma_load_3d(void* smem, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar,
                                            uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, "
      "%4}], [%5], %6;" ::"r"(smem_u32(smem)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void ldmatrix_x4(uint32_t addr, uint32_t (&a)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3])
               : "r"(addr));
}
__device__ __forceinline__ void mma_bf16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Grid barrier over the co-resident grid (cooperative launch): bar[0] counts arrivals
// over the whole launch (zeroed by the host before it), so barrier i completes when it
// reaches (i + 1) * grid -- one fire-and-forget release-add per CTA and a poll, no
// read-modify-write round trip on the critical path.  Bounded spin: a timeout raises
// bar[2] and every later barrier returns at once (wrong results, never a hung GPU).
__device__ void grid_sync(const Params& p, unsigned& epoch) {
  named_sync();
  ++epoch;
  if (threadIdx.x == 0) {
    if (*reinterpret_cast<volatile unsigned*>(p.bar + 2) == 0) {
      __threadfence();
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p.bar) : "memory");
      const unsigned target = epoch * gridDim.x;
      if (ld_acquire(p.bar) < target) {
        const uint64_t t0 = gtimer();
        while (ld_acquire(p.bar) < target) {
          if (gtimer() - t0 > SPIN_NS) {
            atomicExch(p.bar + 2, 1u);
            break;
          }
        }
      }
    }
    __threadfence();
  }
  named_sync();
}

// ---- weight phases ----------------------------------------------------------------------
// 0: qkv (n = nqkv, k = d)   1: o-proj (d, d)   2: gate|up (ffn, d; two row groups: gate
// rows r and up rows ffn + r of one unit land in consecutive slots)   3: down (d, ffn).
// A unit is 16 rows x all of k (ks slots of 512 k); CTA c owns units [u0, u1).
struct WPhase {
  int map, n, k, ks, groups, up, u0, u1;
};

__device__ __forceinline__ WPhase wphase(const Params& p, int ph) {
  WPhase w;
  w.map = ph;
  w.groups = 1;
  w.up = 0;
  if (ph == 0) {
    w.n = p.nqkv, w.k = p.d;
  } else if (ph == 1) {
    w.n = p.d, w.k = p.d;
  } else if (ph == 2) {
    w.n = p.ffn, w.k = p.d, w.groups = 2, w.up = p.ffn;
  } else {
    w.n = p.d, w.k = p.ffn;
  }
  w.ks = (w.k + SLOT_K - 1) / SLOT_K;
  const int units = (w.n + UROWS - 1) / UROWS;
  w.u0 = static_cast<int>(static_cast<int64_t>(units) * blockIdx.x / gridDim.x);
  w.u1 = static_cast<int>(static_cast<int64_t>(units) * (blockIdx.x + 1) / gridDim.x);
  return w;
}

__device__ __forceinline__ void trace_ev(const Params& p, int l, int ev) {
  if (p.trace) p.trace[(static_cast<int64_t>(blockIdx.x) * p.n_blocks + l) * EV_N + ev] = gtimer();
}

struct Ring {
  uint8_t* slots;
  uint64_t* full;
  uint64_t* empty;
  volatile uint32_t* issued;
  int nslot;
};

// Walks this CTA's weight slots in stream order: blocks -> phases -> waves of up to CW
// units (one per consumer warp) -> row groups -> k slots -> the wave's units, so the CW
// warps of a wave consume their units' slots side by side.
struct ChunkIter {
  WPhase w;
  int l, ph, w0, nw, g, j, i;
  bool done;
  __device__ void init(const Params& p) {
    l = 0, ph = 0, done = false;
    w = wphase(p, 0);
    start_wave(w.u0);
    settle(p);
  }
  __device__ void start_wave(int u) {
    w0 = u, nw = min(CW, w.u1 - u), g = 0, j = 0, i = 0;
  }
  __device__ void settle(const Params& p) {
    while (!done && w0 >= w.u1) {
      if (++ph == 4) {
        ph = 0;
        if (++l == p.n_blocks) {
          done = true;
          return;
        }
      }
      w = wphase(p, ph);
      start_wave(w.u0);
    }
  }
  __device__ void advance(const Params& p) {
    if (++i < nw) return;
    i = 0;
    if (++j < w.ks) return;
    j = 0;
    if (++g < w.groups) return;
    start_wave(w0 + nw);
    settle(p);
  }
  __device__ int unit() const { return w0 + i; }
};

// Context split of this step's attention (same on every CTA and role: pos is read-only
// during the kernel): about one (sequence, kv head, chunk) item per CTA.
__device__ __forceinline__ void attn_split(const Params& p, int rows, int& nsplit, int& chunk) {
  int maxlen = 0;
  for (int b = 0; b < rows; ++b)
    maxlen = max(maxlen, static_cast<int>(tmin<int64_t>(static_cast<int64_t>(p.pos[b * p.pos_stride]) + 1, p.s_max)));
  const int want = max(1, static_cast<int>(gridDim.x) / (rows * p.KV));
  chunk = (maxlen + want - 1) / want;
  chunk = max(32, (chunk + 31) / 32 * 32);
  if (chunk > CHUNK_MAX) chunk = CHUNK_MAX;
  nsplit = max(1, (maxlen + chunk - 1) / chunk);  // <= NSPLIT_CAP (host checks s_max)
}

template <int HD>
__device__ void prefetch_kv(const Params& p, const Block& blk, int rows, int nsplit, int chunk);

// Producer: lane 0 of warp CW streams every weight slot of this CTA in the fixed order,
// and on entering a block's weights pulls that block's attention K/V chunks into L2.
// (Prefetching further ahead into L2 while the ring is full measured slower at every
// depth: the extra L2 requests slow the streaming phases more than they save.)
template <int NB, int HD>
__device__ void produce(const Params& p, const Ring& ring) {
  int nsplit, chunk;
  attn_split(p, NB, nsplit, chunk);
  prefetch_kv<HD>(p, p.blk[0], NB, nsplit, chunk);
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  ChunkIter ld;
  ld.init(p);
  uint32_t q = 0;
  while (!ld.done) {
    const int s = static_cast<int>(q % ring.nslot);
    const uint32_t lap = q / ring.nslot;
    if (lap) mbar_wait(&ring.empty[s], (lap - 1) & 1);
    mbar_expect_tx(&ring.full[s], SLOT);  // out-of-range k / rows arrive as zeros, full box
    tma_load_3d(ring.slots + static_cast<size_t>(s) * SLOT, &p.tm[ld.l][ld.w.map], 0,
                ld.unit() * UROWS + ld.g * ld.w.up, ld.j * (SLOT_K / 64), &ring.full[s], pol);
    *ring.issued = ++q;
    const int l = ld.l, ph = ld.ph;
    ld.advance(p);
    if (ld.done || ld.l != l || ld.ph != ph) trace_ev(p, l, EV_PROD_QKV + ph);
    if (!ld.done && ld.l != l) prefetch_kv<HD>(p, p.blk[ld.l], NB, nsplit, chunk);
  }
}

// One slot (16 rows x 512 k, 8 swizzled 2 KiB tiles) into the unit's accumulators:
// per 16 k an ldmatrix.x4 of the weights (A), the sequences' x as B (thread (g, t) holds
// x[g][k + 2t .. +1] and x[g][k + 2t + 8 .. +9]; columns g >= NB are zero), one MMA.
// Two accumulator sets alternate for two independent chains.
template <int NB>
__device__ __forceinline__ void slot_mma(uint32_t slot, const __nv_bfloat16* act, int act_ld, int k_base, int k,
                                         int lane, float (&c0)[4], float (&c1)[4]) {
  const int r = lane & 15, hi = lane >> 4, gq = lane >> 2, t2 = (lane & 3) * 2;
  const bool bcol = gq < NB;
  const __nv_bfloat16* xrow = act + (bcol ? gq : 0) * act_ld + t2;
  const uint32_t rowoff = slot + r * 128;
#pragma unroll
  for (int kh = 0; kh < SLOT_K / 64; ++kh) {
    const int k64 = k_base + kh * 64;
    if (k64 >= k) break;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      uint32_t a[4];
      ldmatrix_x4(rowoff + kh * 2048 + (((ks * 2 + hi) ^ (r & 7)) << 4), a);
      const int kk = k64 + ks * 16;
      const uint32_t b0 = bcol ? *reinterpret_cast<const uint32_t*>(xrow + kk) : 0u;
      const uint32_t b1 = bcol ? *reinterpret_cast<const uint32_t*>(xrow + kk + 8) : 0u;
      if (ks & 1)
        mma_bf16(c1, a, b0, b1);
      else
        mma_bf16(c0, a, b0, b1);
    }
  }
}

// All slots of row group g of the unit this warp owns in a wave (slot q0 + (g * ks + j) *
// nw + i for k slot j).  c = the sum of the two MMA chains: thread (g, t) holds rows
// g, g + 8 x sequences 2t, 2t + 1.
template <int NB>
__device__ __forceinline__ void unit_group(const Params& p, const WPhase& w, uint32_t q0, int nw, int i, int g,
                                           const Ring& ring, const __nv_bfloat16* act, int act_ld, int lane,
                                           float (&c)[4]) {
  float c1[4] = {0.f, 0.f, 0.f, 0.f};
  c[0] = c[1] = c[2] = c[3] = 0.f;
  for (int j = 0; j < w.ks; ++j) {
    const uint32_t q = q0 + static_cast<uint32_t>((g * w.ks + j) * nw + i);
    const int s = static_cast<int>(q % ring.nslot);
    while (*ring.issued <= q) {
    }
    mbar_wait(&ring.full[s], (q / ring.nslot) & 1);
    if (!p.nomath)
      slot_mma<NB>(smem_u32(ring.slots + static_cast<size_t>(s) * SLOT), act, act_ld, j * SLOT_K, w.k, lane, c, c1);
    __syncwarp();
    if (lane == 0) mbar_arrive(&ring.empty[s]);
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) c[k] += c1[k];
}

// Consumer side of one weight phase: in each wave of up to CW units, warp i owns unit
// w0 + i; `act` is the phase input [NB][act_ld] bf16 in shared memory.  Each thread
// writes its own (row, sequence) outputs -- no cross-lane reduction.
template <int NB>
__device__ void consume(const Params& p, const WPhase& w, int ph, uint32_t& q, const Ring& ring,
                        const __nv_bfloat16* act, int act_ld) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, t2 = (lane & 3) * 2;
  for (int w0 = w.u0; w0 < w.u1; w0 += CW) {
    const int nw = min(CW, w.u1 - w0);
    const uint32_t q0 = q;
    q += static_cast<uint32_t>(w.groups * w.ks * nw);
    if (warp >= nw) continue;
    const int u = w0 + warp;
    float cg[4], cu[4];
    unit_group<NB>(p, w, q0, nw, warp, 0, ring, act, act_ld, lane, cg);
    if (w.groups == 2) unit_group<NB>(p, w, q0, nw, warp, 1, ring, act, act_ld, lane, cu);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int row = u * UROWS + gq + (k >> 1) * 8;
      const int b = t2 + (k & 1);
      if (b >= NB || row >= w.n) continue;
      const float v0 = cg[k];
      if (ph == 0) {
        p.qkv[static_cast<int64_t>(b) * p.nqkv + row] = __float2bfloat16_rn(v0);
      } else if (ph == 1) {
        const float res = __bfloat162float(p.x[static_cast<int64_t>(b) * p.ldx + row]);
        p.o[static_cast<int64_t>(b) * p.d + row] = __float2bfloat16_rn(v0 + res);
      } else if (ph == 2) {
        const float gt = bf16r(v0), up = bf16r(cu[k]);
        p.act[static_cast<int64_t>(b) * p.ffn + row] = __float2bfloat16_rn(gt / (1.f + __expf(-gt)) * up);
      } else {
        const float res = __bfloat162float(p.o[static_cast<int64_t>(b) * p.d + row]);
        p.x[static_cast<int64_t>(b) * p.ldx + row] = __float2bfloat16_rn(v0 + res);
      }
    }
  }
}

// ---- per-CTA staging of a phase input into shared memory -------------------------------
// act[b][:] = bf16(src[b] * rsqrt(mean(src[b]^2) + eps) * w)   (k_rmsnorm's formula)
template <int NB>
__device__ void stage_norm(const Params& p, const __nv_bfloat16* src, int ld, const __nv_bfloat16* w,
                           __nv_bfloat16* act, float* red) {
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int n8 = p.d / 8;
  float ss[NB];
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    ss[b] = 0.f;
    const uint4* xr = reinterpret_cast<const uint4*>(src + static_cast<int64_t>(b) * ld);
    for (int i = t; i < n8; i += CT) {
      float f[8];
      unpack8(xr[i], f);
#pragma unroll
      for (int e = 0; e < 8; ++e) ss[b] = fmaf(f[e], f[e], ss[b]);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) ss[b] += __shfl_xor_sync(0xffffffffu, ss[b], o);
    if (lane == 0) red[b * CW + warp] = ss[b];
  }
  named_sync();
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    float tot = 0.f;
#pragma unroll
    for (int i = 0; i < CW; ++i) tot += red[b * CW + i];
    const float inv = rsqrtf(tot / p.d + p.eps);
    const uint4* xr = reinterpret_cast<const uint4*>(src + static_cast<int64_t>(b) * ld);
    const uint4* wr = reinterpret_cast<const uint4*>(w);
    uint4* out = reinterpret_cast<uint4*>(act + b * p.d);
    for (int i = t; i < n8; i += CT) {
      float f[8], g[8];
      unpack8(xr[i], f);
      unpack8(wr[i], g);
      uint4 v;
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
      for (int e = 0; e < 4; ++e)
        h[e] = __floats2bfloat162_rn(f[2 * e] * inv * g[2 * e], f[2 * e + 1] * inv * g[2 * e + 1]);
      out[i] = v;
    }
  }
  named_sync();
}

// act[b][h*HD + d] = combine of the attention partials (k_decode_combine's formula).
// Fast path: the (max, sum) of every (sequence, head, chunk) staged in shared memory,
// split weights formed once per (sequence, head), then every thread combines float4
// column groups with all of its partial loads in flight at once.
template <int NB, int HD>
__device__ void stage_combine(const Params& p, int nsplit, __nv_bfloat16* act, float* sm) {
  const int t = threadIdx.x;
  const int pairs = NB * p.H;
  const int ps = pairs * nsplit;
  if (2 * ps + pairs <= CW * NSPLIT_CAP) {
    float* wgt = sm;           // [pairs][nsplit]: m, then the split weight
    float* ll = sm + ps;       // [pairs][nsplit]: l
    float* inv = sm + 2 * ps;  // [pairs]
    for (int i = t; i < ps; i += CT) {
      const int bh = i / nsplit, sp = i % nsplit;
      const float2 ml = *reinterpret_cast<const float2*>(p.pml + (static_cast<int64_t>(bh) * NSPLIT_CAP + sp) * 2);
      wgt[i] = ml.x;
      ll[i] = ml.y;
    }
    named_sync();
    for (int bh = t; bh < pairs; bh += CT) {
      float m = -CUDART_INF_F;
      for (int sp = 0; sp < nsplit; ++sp)
        if (ll[bh * nsplit + sp] > 0.f) m = fmaxf(m, wgt[bh * nsplit + sp]);
      float den = 0.f;
      for (int sp = 0; sp < nsplit; ++sp) {
        const float l = ll[bh * nsplit + sp];
        const float wv = l > 0.f ? __expf(wgt[bh * nsplit + sp] - m) : 0.f;
        wgt[bh * nsplit + sp] = wv;
        den += wv * l;
      }
      inv[bh] = 1.f / den;
    }
    named_sync();
    constexpr int QPH = HD / 4;   // float4 groups per head
    const int ng = NB * p.d / 4;
    const float4* part4 = reinterpret_cast<const float4*>(p.part);
    // each thread: column groups gi = t + u*CT; all (group, split) loads of a round of
    // up to 16 issued before any is used
    for (int g0 = t; g0 < ng; g0 += 4 * CT) {
      float4 acc[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int s0 = 0; s0 < nsplit; s0 += 4) {
        float4 ov[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int gi = g0 + u * CT;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int sp = s0 + k;
            ov[u][k] = (gi < ng && sp < nsplit)
                           ? part4[(static_cast<int64_t>(gi / QPH) * NSPLIT_CAP + sp) * QPH + gi % QPH]
                           : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int gi = g0 + u * CT;
          if (gi >= ng) break;
          const int bh = gi / QPH;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int sp = s0 + k;
            if (sp >= nsplit) break;
            const float wv = wgt[bh * nsplit + sp];
            if (wv != 0.f) {  // an empty chunk's stale o is masked by its zero weight
              acc[u].x = fmaf(wv, ov[u][k].x, acc[u].x);
              acc[u].y = fmaf(wv, ov[u][k].y, acc[u].y);
              acc[u].z = fmaf(wv, ov[u][k].z, acc[u].z);
              acc[u].w = fmaf(wv, ov[u][k].w, acc[u].w);
            }
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int gi = g0 + u * CT;
        if (gi >= ng) break;
        const float iv = inv[gi / QPH];
        __nv_bfloat162* dst = reinterpret_cast<__nv_bfloat162*>(act + gi * 4);
        dst[0] = __floats2bfloat162_rn(acc[u].x * iv, acc[u].y * iv);
        dst[1] = __floats2bfloat162_rn(acc[u].z * iv, acc[u].w * iv);
      }
    }
    named_sync();
    return;
  }
  // long contexts x many heads: one warp per (sequence, head)
  const int warp = t >> 5, lane = t & 31;
  float* wgt = sm + warp * NSPLIT_CAP;
  for (int bh = warp; bh < pairs; bh += CW) {
    const float* ml = p.pml + static_cast<int64_t>(bh) * NSPLIT_CAP * 2;
    const float* base = p.part + static_cast<int64_t>(bh) * NSPLIT_CAP * HD;
    float m = -CUDART_INF_F;
    for (int sp = lane; sp < nsplit; sp += 32)
      if (ml[2 * sp + 1] > 0.f) m = fmaxf(m, ml[2 * sp]);
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float den = 0.f;
    for (int sp = lane; sp < nsplit; sp += 32) {
      const float l = ml[2 * sp + 1];
      const float wv = l > 0.f ? __expf(ml[2 * sp] - m) : 0.f;
      wgt[sp] = wv;
      den += wv * l;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) den += __shfl_xor_sync(0xffffffffu, den, o);
    __syncwarp();
    const float inv_den = 1.f / den;
    for (int dd = lane; dd < HD; dd += 32) {
      float num = 0.f;
      for (int sp = 0; sp < nsplit; ++sp) {
        const float wv = wgt[sp];
        num += wv != 0.f ? wv * base[sp * HD + dd] : 0.f;
      }
      act[bh * HD + dd] = __float2bfloat16_rn(num * inv_den);
    }
    __syncwarp();
  }
  named_sync();
}

// ---- attention phase ---------------------------------------------------------------------
// Item (b, kv head g, split): the G query heads of the group over context tokens
// [split*chunk, +chunk) of sequence b, flash-decoding partials (m, l, o) into p.part.
// The newest token (position pos_b) is RoPE'd from the qkv row and written into the
// cache by the item whose chunk holds it, before the item reads its chunk (CTA
// barrier: the same CTA's global writes are visible to its later loads).  One CTA per
// SM runs the item, so every K row is fetched whole (VEC independent 16-byte loads per
// thread) and the P.V pass keeps PV_U rows in flight per thread.
template <int HD>
__device__ void attention(const Params& p, const Block& blk, int rows, int nsplit, int chunk, uint8_t* scratch,
                          int layer) {
  constexpr int HALF = HD / 2, VEC = HD / 8, LANES = CT / VEC, PV_U = 12;
  const int G = p.H / p.KV;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  float* qs = reinterpret_cast<float*>(scratch);   // [G][HD]
  float* sc = qs + G * HD;                          // [G][CHUNK_MAX]
  float* red = sc + G * CHUNK_MAX;                  // [CW][G][HD]
  float* stat = red + CW * G * HD;                  // m[GMAX], l[GMAX]
  const int items = rows * p.KV * nsplit;
  for (int it = blockIdx.x; it < items; it += gridDim.x) {
    const int b = it / (p.KV * nsplit), g = (it / nsplit) % p.KV, split = it % nsplit;
    const int pb = p.pos[b * p.pos_stride];
    const int len = static_cast<int>(tmin<int64_t>(static_cast<int64_t>(pb) + 1, p.s_max));
    const int c0 = split * chunk;
    const int n = min(chunk, len - c0);
    const int64_t slot0 = (static_cast<int64_t>(b) * p.H + g * G) * NSPLIT_CAP + split;  // head j: + j * NSPLIT_CAP
    if (n <= 0) {
      if (t < G) *reinterpret_cast<float2*>(p.pml + (slot0 + t * NSPLIT_CAP) * 2) = make_float2(-CUDART_INF_F, 0.f);
      continue;
    }
    const __nv_bfloat16* row = p.qkv + static_cast<int64_t>(b) * p.nqkv;
    const float pf = static_cast<float>(pb);
    // q heads of the group: RoPE, bf16 (as k_rope_append stores them), * 1/sqrt(hd)
    for (int idx = t; idx < G * HALF; idx += CT) {
      const int j = idx / HALF, i = idx % HALF;
      const __nv_bfloat16* hp = row + (g * G + j) * HD;
      const float inv_freq = exp2f(-p.log2_theta * (2.0f * i) / HD);
      float sn, cs;
      sincosf(pf * inv_freq, &sn, &cs);
      const float a = __bfloat162float(hp[i]), c = __bfloat162float(hp[i + HALF]);
      qs[j * HD + i] = bf16r(a * cs - c * sn) * p.scale;
      qs[j * HD + i + HALF] = bf16r(c * cs + a * sn) * p.scale;
    }
    const int64_t panel = (static_cast<int64_t>(b) * p.KV + g) * p.s_max;
    if (pb >= c0 && pb < c0 + n) {  // the newest token's k (RoPE'd) and v into the cache
      const __nv_bfloat16* kp = row + (p.H + g) * HD;
      const __nv_bfloat16* vp = row + (p.H + p.KV + g) * HD;
      __nv_bfloat16* kdst = blk.kc + (panel + pb) * HD;
      __nv_bfloat16* vdst = blk.vc + (panel + pb) * HD;
      for (int i = t; i < HALF; i += CT) {
        const float inv_freq = exp2f(-p.log2_theta * (2.0f * i) / HD);
        float sn, cs;
        sincosf(pf * inv_freq, &sn, &cs);
        const float a = __bfloat162float(kp[i]), c = __bfloat162float(kp[i + HALF]);
        kdst[i] = __float2bfloat16_rn(a * cs - c * sn);
        kdst[i + HALF] = __float2bfloat16_rn(c * cs + a * sn);
        vdst[i] = vp[i];
        vdst[i + HALF] = vp[i + HALF];
      }
    }
    named_sync();
    const bool tr = p.trace && t == 0 && it == static_cast<int>(blockIdx.x);
    if (tr) trace_ev(p, layer, EV_A_Q);
    // scores: VEC lanes per context token (one coalesced K row per lane group), SU rows
    // per lane group in flight, lane-group reduction by shuffles
    const uint4* kbase = reinterpret_cast<const uint4*>(blk.kc + (panel + c0) * HD);
    const uint4* vbase = reinterpret_cast<const uint4*>(blk.vc + (panel + c0) * HD);
    {
      constexpr int RPW = 32 / VEC, SU = 12;
      const int sub = lane / VEC, li = lane % VEC;
      for (int base = warp * RPW; base < n; base += CW * RPW * SU) {  // warp-uniform trip count
        uint4 kr[SU];
#pragma unroll
        for (int u = 0; u < SU; ++u) {
          const int tt = base + sub + u * CW * RPW;
          kr[u] = tt < n ? kbase[static_cast<int64_t>(tt) * VEC + li] : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < SU; ++u) {
          const int tt = base + sub + u * CW * RPW;
          float f[8];
          unpack8(kr[u], f);
#pragma unroll
          for (int j = 0; j < GMAX; ++j) {
            if (j >= G) break;
            const float4 q0 = *reinterpret_cast<const float4*>(qs + j * HD + li * 8);
            const float4 q1 = *reinterpret_cast<const float4*>(qs + j * HD + li * 8 + 4);
            float a = f[0] * q0.x;
            a = fmaf(f[1], q0.y, a);
            a = fmaf(f[2], q0.z, a);
            a = fmaf(f[3], q0.w, a);
            a = fmaf(f[4], q1.x, a);
            a = fmaf(f[5], q1.y, a);
            a = fmaf(f[6], q1.z, a);
            a = fmaf(f[7], q1.w, a);
#pragma unroll
            for (int o = VEC / 2; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
            if (li == 0 && tt < n) sc[j * CHUNK_MAX + tt] = a;
          }
        }
      }
    }
    named_sync();
    if (tr) trace_ev(p, layer, EV_A_S);
    for (int j = warp; j < G; j += CW) {
      float m = -CUDART_INF_F;
      for (int tt = lane; tt < n; tt += 32) m = fmaxf(m, sc[j * CHUNK_MAX + tt]);
#pragma unroll
      for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      float l = 0.f;
      for (int tt = lane; tt < n; tt += 32) {
        const float e = __expf(sc[j * CHUNK_MAX + tt] - m);
        sc[j * CHUNK_MAX + tt] = e;
        l += e;
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
      if (lane == 0) {
        stat[j] = m;
        stat[GMAX + j] = l;
      }
    }
    named_sync();
    if (tr) trace_ev(p, layer, EV_A_SM);
    // P.V: thread (token lane tl, 8-column group cv), PV_U V rows in flight (coalesced rows)
    const int cv = t % VEC, tl = t / VEC;
    float acc[GMAX][8];
#pragma unroll
    for (int j = 0; j < GMAX; ++j)
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[j][e] = 0.f;
    for (int t0 = tl; t0 < n; t0 += LANES * PV_U) {
      uint4 vr[PV_U];
#pragma unroll
      for (int u = 0; u < PV_U; ++u) {
        const int tt = t0 + u * LANES;
        vr[u] = tt < n ? vbase[static_cast<int64_t>(tt) * VEC + cv] : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < PV_U; ++u) {
        const int tt = t0 + u * LANES;
        if (tt >= n) break;
        float f[8];
        unpack8(vr[u], f);
#pragma unroll
        for (int j = 0; j < GMAX; ++j) {
          if (j >= G) break;
          const float pr = sc[j * CHUNK_MAX + tt];
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[j][e] = fmaf(pr, f[e], acc[j][e]);
        }
      }
    }
    // lanes of a warp that share cv: xor over the token-lane bits, then one row per warp
#pragma unroll
    for (int j = 0; j < GMAX; ++j) {
      if (j >= G) break;
#pragma unroll
      for (int e = 0; e < 8; ++e)
#pragma unroll
        for (int o = VEC; o < 32; o <<= 1) acc[j][e] += __shfl_xor_sync(0xffffffffu, acc[j][e], o);
    }
    if (lane < VEC) {
#pragma unroll
      for (int j = 0; j < GMAX; ++j) {
        if (j >= G) break;
#pragma unroll
        for (int e = 0; e < 8; ++e) red[(warp * G + j) * HD + cv * 8 + e] = acc[j][e];
      }
    }
    named_sync();
    if (tr) trace_ev(p, layer, EV_A_PV);
    for (int idx = t; idx < G * HD; idx += CT) {
      const int j = idx / HD, dd = idx % HD;
      float s = 0.f;
#pragma unroll
      for (int w = 0; w < CW; ++w) s += red[(w * G + j) * HD + dd];
      const int64_t slot = slot0 + static_cast<int64_t>(j) * NSPLIT_CAP;
      p.part[slot * HD + dd] = s;
      if (dd == 0) *reinterpret_cast<float2*>(p.pml + slot * 2) = make_float2(stat[j], stat[GMAX + j]);
    }
    named_sync();
  }
}

// Thread 0: pull this CTA's attention chunks of K and V into L2 at the start of the
// block, so the attention phase (after the qkv phase) reads them at L2 latency.
template <int HD>
__device__ void prefetch_kv(const Params& p, const Block& blk, int rows, int nsplit, int chunk) {
  const int items = rows * p.KV * nsplit;
  for (int it = blockIdx.x; it < items; it += gridDim.x) {
    const int b = it / (p.KV * nsplit), g = (it / nsplit) % p.KV, split = it % nsplit;
    const int len = static_cast<int>(tmin<int64_t>(static_cast<int64_t>(p.pos[b * p.pos_stride]) + 1, p.s_max));
    const int c0 = split * chunk;
    const int n = min(chunk, len - c0);
    if (n <= 0) continue;
    const int64_t row0 = (static_cast<int64_t>(b) * p.KV + g) * p.s_max + c0;
    const char* kp = reinterpret_cast<const char*>(blk.kc + row0 * HD);
    const char* vp = reinterpret_cast<const char*>(blk.vc + row0 * HD);
    const uint32_t bytes = static_cast<uint32_t>(n) * HD * 2;
    for (uint32_t off = 0; off < bytes; off += 32768) {
      const uint32_t sz = min(32768u, bytes - off);
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(kp + off), "r"(sz) : "memory");
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(vp + off), "r"(sz) : "memory");
    }
  }
}

__host__ __device__ constexpr int attn_scratch_bytes(int G, int HD) {
  return 4 * (G * HD + G * CHUNK_MAX + CW * G * HD + 2 * GMAX);
}

// ---- the kernel ---------------------------------------------------------------------------
template <int NB, int HD>
__global__ void __launch_bounds__(THREADS, 1) k_decode_fused(const __grid_constant__ Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 128B-swizzled TMA tiles need 1024-byte aligned slots
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  Ring ring;
  ring.nslot = p.nslot;
  ring.slots = smem;
  ring.full = reinterpret_cast<uint64_t*>(smem + static_cast<size_t>(p.nslot) * SLOT);
  ring.empty = ring.full + MAX_SLOTS;
  ring.issued = reinterpret_cast<volatile uint32_t*>(ring.empty + MAX_SLOTS);
  float* red = reinterpret_cast<float*>(ring.empty + MAX_SLOTS + 2);      // [MAX_ROWS][CW]
  float* wgt = red + MAX_ROWS * CW;                                        // [CW][NSPLIT_CAP]
  uint8_t* region = reinterpret_cast<uint8_t*>(wgt + CW * NSPLIT_CAP);     // act / attention scratch
  __nv_bfloat16* act = reinterpret_cast<__nv_bfloat16*>(region);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < MAX_SLOTS; ++s) {
      mbar_init(&ring.full[s], 1);
      mbar_init(&ring.empty[s], 1);
    }
    *ring.issued = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == CW) {
    if (lane == 0) produce<NB, HD>(p, ring);
    return;
  }

  int nsplit, chunk;
  attn_split(p, NB, nsplit, chunk);

  uint32_t q = 0;
  unsigned epoch = 0;
  for (int l = 0; l < p.n_blocks; ++l) {
    const Block& blk = p.blk[l];
    if (l) grid_sync(p, epoch);  // previous block's output complete everywhere
    const bool tr = p.trace && threadIdx.x == 0;
    if (tr) trace_ev(p, l, EV_START);
    stage_norm<NB>(p, p.x, p.ldx, blk.attn_norm, act, red);
    if (tr) trace_ev(p, l, EV_NORM1);
    consume<NB>(p, wphase(p, 0), 0, q, ring, act, p.d);
    if (tr) trace_ev(p, l, EV_QKV);
    grid_sync(p, epoch);
    if (tr) trace_ev(p, l, EV_BAR1);
    attention<HD>(p, blk, NB, nsplit, chunk, region, l);
    if (tr) trace_ev(p, l, EV_ATTN);
    grid_sync(p, epoch);
    if (tr) trace_ev(p, l, EV_BAR2);
    stage_combine<NB, HD>(p, nsplit, act, wgt);
    if (tr) trace_ev(p, l, EV_COMB);
    consume<NB>(p, wphase(p, 1), 1, q, ring, act, p.d);
    if (tr) trace_ev(p, l, EV_O);
    grid_sync(p, epoch);
    if (tr) trace_ev(p, l, EV_BAR3);
    stage_norm<NB>(p, p.o, p.d, blk.ffn_norm, act, red);
    if (tr) trace_ev(p, l, EV_NORM2);
    consume<NB>(p, wphase(p, 2), 2, q, ring, act, p.d);
    if (tr) trace_ev(p, l, EV_GU);
    grid_sync(p, epoch);
    if (tr) trace_ev(p, l, EV_BAR4);
    {  // act (global, [NB][ffn]) -> shared memory
      const int n8 = NB * p.ffn / 8;
      const uint4* src = reinterpret_cast<const uint4*>(p.act);
      uint4* dst = reinterpret_cast<uint4*>(act);
      for (int i = threadIdx.x; i < n8; i += CT) dst[i] = src[i];
      named_sync();
    }
    if (tr) trace_ev(p, l, EV_ACT);
    consume<NB>(p, wphase(p, 3), 3, q, ring, act, p.ffn);
    if (tr) trace_ev(p, l, EV_DOWN);
  }
}

template <int NB, int HD>
static cudaError_t launch(const Params& p, int grid, int smem, cudaStream_t s) {
  static bool attr_set[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(k_decode_fused<NB, HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_MAX);
    if (e != cudaSuccess) return e;
    attr_set[dev] = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // every CTA resident: the grid barriers need it
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_decode_fused<NB, HD>, p);
}

static uint64_t* g_trace = nullptr;
static int64_t g_trace_bytes = 0;

static int64_t align256(int64_t v) { return (v + 255) / 256 * 256; }

struct WsLayout {
  int64_t qkv, o, act, part, pml, total;
};
static WsLayout ws_layout(int rows, int d, int n_heads, int n_kv, int head_dim, int ffn) {
  WsLayout w;
  const int64_t nqkv = static_cast<int64_t>(n_heads + 2 * n_kv) * head_dim;
  w.qkv = 256;
  w.o = w.qkv + align256(rows * nqkv * 2);
  w.act = w.o + align256(static_cast<int64_t>(rows) * d * 2);
  w.part = w.act + align256(static_cast<int64_t>(rows) * ffn * 2);
  w.pml = w.part + static_cast<int64_t>(rows) * n_heads * NSPLIT_CAP * head_dim * 4;
  w.total = w.pml + static_cast<int64_t>(rows) * n_heads * NSPLIT_CAP * 2 * 4;
  return w;
}

}  // namespace fused
}  // namespace bz

using namespace bz;

extern "C" int bz_decode_fused_workspace_bytes(int rows, int d, int n_heads, int n_kv, int head_dim, int ffn,
                                               int64_t* bytes) {
  if (!bytes || rows <= 0 || d <= 0 || n_heads <= 0 || n_kv <= 0 || head_dim <= 0 || ffn <= 0)
    return bz_fail(BZ_EINVAL, "decode_fused_workspace_bytes: bad args");
  *bytes = fused::ws_layout(rows, d, n_heads, n_kv, head_dim, ffn).total;
  return BZ_OK;
}

// 3-D view {64 k, rows, k / 64} of a [rows, k] bf16 weight: one box {64, 16, 8} is 16 rows
// x 512 k, stored as 8 consecutive 128B-swizzled [16 x 64] tiles.
static int encode_w3d(CUtensorMap* map, const void* w, int rows, int k) {
  const DriverApi* d = driver_api();
  if (!d) return BZ_ECUDA;
  cuuint64_t dims[3] = {64, static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(k / 64)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(k) * 2, 128};
  cuuint32_t box[3] = {64, fused::UROWS, fused::SLOT_K / 64};
  cuuint32_t elem[3] = {1, 1, 1};
  CUresult r = d->cuTensorMapEncodeTiled(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(w), dims, strides,
                                         box, elem, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return bz_fail_cu(r, "decode_fused: cuTensorMapEncodeTiled");
  return BZ_OK;
}

extern "C" int bz_decode_fused(const bz_decode_block* blocks, int n_blocks, void* x, int ldx, int rows, int d,
                               int n_heads, int n_kv, int head_dim, int ffn, float rope_theta, float eps,
                               int64_t s_max, const int32_t* pos, int pos_stride, void* workspace, int64_t ws_bytes,
                               int max_ctas, void* stream) {
  using namespace fused;
  if (!blocks || n_blocks <= 0 || !x || !pos || !workspace || rows <= 0 || d <= 0 || ffn <= 0)
    return bz_fail(BZ_EINVAL, "decode_fused: bad args");
  if (rows > MAX_ROWS) return bz_fail(BZ_EINVAL, "decode_fused: at most 4 sequences per step");
  if (head_dim != 64 && head_dim != 128) return bz_fail(BZ_EINVAL, "decode_fused: head_dim must be 64 or 128");
  if (n_kv <= 0 || n_heads % n_kv || n_heads / n_kv > GMAX)
    return bz_fail(BZ_EINVAL, "decode_fused: heads per kv head must divide and be <= 8");
  if (d % 64 || ffn % 64 || ldx % 8 || d != n_heads * head_dim)
    return bz_fail(BZ_EINVAL, "decode_fused: d and ffn multiples of 64, ldx of 8, d == n_heads * head_dim");
  if (s_max <= 0 || s_max > static_cast<int64_t>(NSPLIT_CAP) * CHUNK_MAX)
    return bz_fail(BZ_EINVAL, "decode_fused: s_max must be in [1, 131072]");
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(workspace)) & 15)
    return bz_fail(BZ_EINVAL, "decode_fused: x and workspace must be 16-byte aligned");
  const WsLayout wl = ws_layout(rows, d, n_heads, n_kv, head_dim, ffn);
  if (ws_bytes < wl.total) return bz_fail(BZ_EINVAL, "decode_fused: workspace too small");
  static thread_local Params p;  // ~28 KB: not on the stack
  p.d = d;
  p.H = n_heads;
  p.KV = n_kv;
  p.ffn = ffn;
  p.nqkv = (n_heads + 2 * n_kv) * head_dim;
  p.ldx = ldx;
  p.log2_theta = log2f(rope_theta);
  p.eps = eps;
  p.scale = 1.0f / sqrtf(static_cast<float>(head_dim));
  p.s_max = s_max;
  p.pos = pos;
  p.pos_stride = pos_stride;
  p.x = static_cast<__nv_bfloat16*>(x);
  char* ws = static_cast<char*>(workspace);
  p.bar = reinterpret_cast<unsigned*>(ws);
  p.qkv = reinterpret_cast<__nv_bfloat16*>(ws + wl.qkv);
  p.o = reinterpret_cast<__nv_bfloat16*>(ws + wl.o);
  p.act = reinterpret_cast<__nv_bfloat16*>(ws + wl.act);
  p.part = reinterpret_cast<float*>(ws + wl.part);
  p.pml = reinterpret_cast<float*>(ws + wl.pml);
  // shared memory: ring | barriers | norm + combine scratch | activation / attention region
  const int kmax = d > ffn ? d : ffn;
  const int scratch = attn_scratch_bytes(n_heads / n_kv, head_dim);
  const int region = (rows * kmax * 2 > scratch ? rows * kmax * 2 : scratch + 15) / 16 * 16;
  const int fixed = 2 * MAX_SLOTS * 8 + 16 + (MAX_ROWS * CW + CW * NSPLIT_CAP) * 4 + region + 1024;
  int nslot = (SMEM_MAX - fixed) / SLOT;
  if (nslot > MAX_SLOTS) nslot = MAX_SLOTS;
  if (nslot < 4) return bz_fail(BZ_EINVAL, "decode_fused: activations leave too little shared memory for the ring");
  p.nslot = nslot;
  p.region_bytes = region;
  p.trace = nullptr;
  {
    const char* e = getenv("BZ_FUSED_NOMATH");
    p.nomath = e && atoi(e) == 1;
  }
  const int smem = nslot * SLOT + fixed;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = max_ctas > 0 && max_ctas < sms ? max_ctas : sms;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // blocks in launches of up to MAX_BLOCKS (the tensor maps travel in the parameters)
  for (int first = 0; first < n_blocks; first += MAX_BLOCKS) {
    const int nb = n_blocks - first < MAX_BLOCKS ? n_blocks - first : MAX_BLOCKS;
    for (int l = 0; l < nb; ++l) {
      const bz_decode_block& b = blocks[first + l];
      if (!b.attn_norm || !b.wqkv || !b.wo || !b.ffn_norm || !b.wgu || !b.wdown || !b.k_cache || !b.v_cache)
        return bz_fail(BZ_EINVAL, "decode_fused: null block pointer");
      const uintptr_t align = reinterpret_cast<uintptr_t>(b.attn_norm) | reinterpret_cast<uintptr_t>(b.wqkv) |
                              reinterpret_cast<uintptr_t>(b.wo) | reinterpret_cast<uintptr_t>(b.ffn_norm) |
                              reinterpret_cast<uintptr_t>(b.wgu) | reinterpret_cast<uintptr_t>(b.wdown);
      if (align & 15) return bz_fail(BZ_EINVAL, "decode_fused: weights must be 16-byte aligned");
      p.blk[l] = {static_cast<const __nv_bfloat16*>(b.attn_norm), static_cast<const __nv_bfloat16*>(b.wqkv),
                  static_cast<const __nv_bfloat16*>(b.wo),        static_cast<const __nv_bfloat16*>(b.ffn_norm),
                  static_cast<const __nv_bfloat16*>(b.wgu),       static_cast<const __nv_bfloat16*>(b.wdown),
                  static_cast<__nv_bfloat16*>(b.k_cache),         static_cast<__nv_bfloat16*>(b.v_cache)};
      if (int rc = encode_w3d(&p.tm[l][TM_QKV], b.wqkv, p.nqkv, d)) return rc;
      if (int rc = encode_w3d(&p.tm[l][TM_O], b.wo, d, d)) return rc;
      if (int rc = encode_w3d(&p.tm[l][TM_GU], b.wgu, 2 * ffn, d)) return rc;
      if (int rc = encode_w3d(&p.tm[l][TM_DOWN], b.wdown, d, ffn)) return rc;
    }
    p.n_blocks = nb;
    if (g_trace && g_trace_bytes >= static_cast<int64_t>(grid) * nb * EV_N * 8) p.trace = g_trace;
    // the barrier words: arrivals must start at 0; the error flag reports this launch
    cudaError_t e = cudaMemsetAsync(ws, 0, 16, s);
    if (e != cudaSuccess) return bz_fail_cuda(e, "decode_fused: barrier reset");
    switch (rows * 1000 + head_dim) {
      case 1128: e = launch<1, 128>(p, grid, smem, s); break;
      case 2128: e = launch<2, 128>(p, grid, smem, s); break;
      case 3128: e = launch<3, 128>(p, grid, smem, s); break;
      case 4128: e = launch<4, 128>(p, grid, smem, s); break;
      case 1064: e = launch<1, 64>(p, grid, smem, s); break;
      case 2064: e = launch<2, 64>(p, grid, smem, s); break;
      case 3064: e = launch<3, 64>(p, grid, smem, s); break;
      default: e = launch<4, 64>(p, grid, smem, s); break;
    }
    if (e != cudaSuccess) return bz_fail_cuda(e, "bz_decode_fused launch");
  }
  return bz_check_launch("bz_decode_fused");
}

extern "C" int bz_decode_fused_status(const void* workspace, int* timed_out, void* stream) {
  if (!workspace || !timed_out) return bz_fail(BZ_EINVAL, "decode_fused_status: bad args");
  unsigned v = 0;
  cudaError_t e = cudaMemcpyAsync(&v, static_cast<const char*>(workspace) + 8, 4, cudaMemcpyDeviceToHost,
                                  static_cast<cudaStream_t>(stream));
  if (e == cudaSuccess) e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return bz_fail_cuda(e, "decode_fused_status");
  *timed_out = v != 0;
  return BZ_OK;
}

extern "C" int bz_decode_fused_set_trace(void* buf, int64_t bytes) {
  fused::g_trace = static_cast<uint64_t*>(buf);
  fused::g_trace_bytes = buf ? bytes : 0;
  return BZ_OK;
}
