// sm_100a data-plane kernels: layer-tiled weight multicast, host staging,
// layer-readiness tracking, payload generation and fingerprints.
//
// What the reference models as arithmetic, these kernels do with bytes:
//   k_push_tiles      chain-edge store-and-forward (planner.py:240-244: a node
//                     forwards each unit as soon as it has received it)
//   k_multicast_tiles NVLink fan-out (planner.py:245-253) as one NVLS
//                     multimem.st stream replicated by the NVSwitch
//   k_stage_tiles     mem<h> -> gpu pcie source edge (topology.py:174-176)
//   k_track_layers    LayerLoaded(k) events (simcore.py:727-733, 752-763)
//
// Unit of pipelining = one tile (a few hundred KB of one layer).  Each CTA
// owns tiles blockIdx.x, blockIdx.x + gridDim.x, ... so tiles complete in
// roughly ascending order and a relay's chain fill costs one tile per hop.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <vector>

#include "../../include/blitz.h"
#include "common.cuh"

namespace bz {

// ---------------------------------------------------------------------------
// memory-order helpers
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void mc_st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("multimem.st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// streaming 16-byte loads: immutable sources may use the non-coherent path;
// relayed tiles were written by a peer GPU during this kernel -> coherent loads.  Both
// ask L2 for 256-byte fetches: a relay that PULLS reads its upstream through NVLink,
// where 32-byte sector requests cost round trips (1->4 chain: 581 vs 692 GB/s without)
template <bool kCoherent>
__device__ __forceinline__ int4 ld16(const int4* p) {
  int4 r;
  if (kCoherent)
    asm volatile("ld.global.L1::no_allocate.L2::256B.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
  else
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
  return r;
}
__device__ __forceinline__ void st16(int4* p, const int4& v) {
  asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}
// weak multicast store (plain STG.E.128 on the multicast VA); ordering to the
// tile flag comes from the CTA barrier + fence.sys + release flag store
__device__ __forceinline__ void mc_st16(int4* p, const int4& v) {
  asm volatile("multimem.st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p),
               "f"(__int_as_float(v.x)), "f"(__int_as_float(v.y)), "f"(__int_as_float(v.z)),
               "f"(__int_as_float(v.w))
               : "memory");
}

// Bounded spin: a wait that outlives the budget gives up and counts a timeout
// in g_wait_timeouts (read by bz_wait_timeouts) instead of hanging the GPU.
__device__ unsigned long long g_wait_timeouts = 0;
__constant__ uint64_t c_spin_budget_ns = 30ull * 1000 * 1000 * 1000;

__device__ __forceinline__ bool spin_until_geq(const uint32_t* p, uint32_t v) {
  if (ld_acquire_sys(p) >= v) return true;
  const uint64_t t0 = globaltimer();
  while (ld_acquire_sys(p) < v) {
    __nanosleep(64);
    if (globaltimer() - t0 > c_spin_budget_ns) {
      atomicAdd(&g_wait_timeouts, 1ull);
      return false;
    }
  }
  return true;
}

// wait (thread 0) for an upstream tile flag, then release the CTA.  Returns false
// (uniformly across the CTA) if the wait timed out: the caller must then neither
// copy the tile nor release its downstream flag, so every GPU below a dead relay
// times out too instead of publishing stale bytes as loaded.
__device__ __forceinline__ bool wait_tile(const uint32_t* flags, int t, uint32_t epoch) {
  __shared__ int ok;
  if (threadIdx.x == 0) ok = spin_until_geq(flags + t, epoch);
  __syncthreads();
  const bool r = ok != 0;
  __syncthreads();  // `ok` is rewritten by the next tile's wait
  return r;
}

// Epoch whose copy-engine relay gate timed out on this device: the flag kernel
// behind that gate then withholds the downstream release (same rule as wait_tile).
__device__ uint32_t g_poisoned_epoch = 0;

constexpr int kThreads = 512;
constexpr int kUnroll = 8;

struct PushArgs {
  const int4* src;
  int4* dst[BZ_MAX_DST];
  uint32_t* flags[BZ_MAX_DST];
  int ndst;
  const uint32_t* wait_flags;
  const int64_t* tile_off;
  const int32_t* ids;  // optional tile list: entries [t0, t1) of it name the tiles
  uint32_t* notify;    // optional: also raise notify[t] (the puller below's upstream flags)
  int t0, t1;
  uint32_t epoch;
};

// Copy one tile [b, e) (in 16-byte words) from src to every destination.
// kMC: destinations are multicast VAs (multimem.st).
template <bool kCoherent, bool kMC, int U = kUnroll>
__device__ __forceinline__ void copy_tile(const int4* __restrict__ src, int4* const* dst, int ndst,
                                          int64_t b, int64_t e) {
  const int64_t step = blockDim.x;
  int64_t i = b + threadIdx.x;
  for (; i + (U - 1) * step < e; i += U * step) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ld16<kCoherent>(src + i + u * step);
    for (int d = 0; d < ndst; ++d) {
      int4* o = dst[d];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (kMC)
          mc_st16(o + i + u * step, v[u]);
        else
          st16(o + i + u * step, v[u]);
      }
    }
  }
  for (; i < e; i += step) {
    int4 v = ld16<kCoherent>(src + i);
    for (int d = 0; d < ndst; ++d) {
      if (kMC)
        mc_st16(dst[d] + i, v);
      else
        st16(dst[d] + i, v);
    }
  }
}

// 256-bit variant (sm_100 LDG/STG.E.ENL2.256): half the memory instructions per byte
struct __align__(32) v8u32 {
  uint32_t v[8];
};
template <bool kCoherent>
__device__ __forceinline__ v8u32 ld32(const v8u32* p) {
  v8u32 r;
  if (kCoherent)
    asm volatile("ld.global.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]), "=r"(r.v[5]),
                   "=r"(r.v[6]), "=r"(r.v[7])
                 : "l"(p));
  else
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]), "=r"(r.v[5]),
                   "=r"(r.v[6]), "=r"(r.v[7])
                 : "l"(p));
  return r;
}
__device__ __forceinline__ void st32(v8u32* p, const v8u32& x) {
  asm volatile("st.global.L1::no_allocate.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(x.v[0]),
               "r"(x.v[1]), "r"(x.v[2]), "r"(x.v[3]), "r"(x.v[4]), "r"(x.v[5]), "r"(x.v[6]), "r"(x.v[7])
               : "memory");
}

// tile [b, e) in 32-byte words
template <bool kCoherent>
__device__ __forceinline__ void copy_tile32(const v8u32* __restrict__ src, int4* const* dst, int ndst, int64_t b,
                                            int64_t e) {
  constexpr int U = 4;
  const int64_t step = blockDim.x;
  int64_t i = b + threadIdx.x;
  for (; i + (U - 1) * step < e; i += U * step) {
    v8u32 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ld32<kCoherent>(src + i + u * step);
    for (int d = 0; d < ndst; ++d) {
      v8u32* o = reinterpret_cast<v8u32*>(dst[d]);
#pragma unroll
      for (int u = 0; u < U; ++u) st32(o + i + u * step, v[u]);
    }
  }
  for (; i < e; i += step) {
    v8u32 v = ld32<kCoherent>(src + i);
    for (int d = 0; d < ndst; ++d) st32(reinterpret_cast<v8u32*>(dst[d]) + i, v);
  }
}

template <bool kRelay>
__global__ void __launch_bounds__(kThreads) k_push_tiles32(PushArgs a) {
  for (int t = a.t0 + blockIdx.x; t < a.t1; t += gridDim.x) {
    if (kRelay && !wait_tile(a.wait_flags, t, a.epoch)) continue;
    const int64_t ob = a.tile_off[t], oe = a.tile_off[t + 1];
    if ((ob | oe) & 31)  // a tile not on 32-byte boundaries: 16-byte path (no dropped tail)
      copy_tile<kRelay, false>(a.src, a.dst, a.ndst, ob >> 4, oe >> 4);
    else
      copy_tile32<kRelay>(reinterpret_cast<const v8u32*>(a.src), a.dst, a.ndst, ob >> 5, oe >> 5);
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      for (int d = 0; d < a.ndst; ++d) st_release_sys(a.flags[d] + t, a.epoch);
    }
  }
}

template <bool kRelay>
__global__ void __launch_bounds__(kThreads) k_push_tiles(PushArgs a) {
  for (int i = a.t0 + blockIdx.x; i < a.t1; i += gridDim.x) {
    const int t = a.ids ? __ldg(a.ids + i) : i;
    if (kRelay && !wait_tile(a.wait_flags, t, a.epoch)) continue;
    const int64_t b = a.tile_off[t] >> 4, e = a.tile_off[t + 1] >> 4;
    copy_tile<kRelay, false>(a.src, a.dst, a.ndst, b, e);
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      for (int d = 0; d < a.ndst; ++d) st_release_sys(a.flags[d] + t, a.epoch);
      if (a.notify) st_release_sys(a.notify + t, a.epoch);
    }
  }
}

template <bool kRelay, int U>
__global__ void __launch_bounds__(kThreads) k_multicast_tiles(PushArgs a) {
  for (int t = a.t0 + blockIdx.x; t < a.t1; t += gridDim.x) {
    if (kRelay && !wait_tile(a.wait_flags, t, a.epoch)) continue;
    const int64_t b = a.tile_off[t] >> 4, e = a.tile_off[t + 1] >> 4;
    copy_tile<kRelay, true, U>(a.src, a.dst, 1, b, e);
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      mc_st_release_sys(a.flags[0] + t, a.epoch);
    }
  }
}

// ---------------------------------------------------------------------------
// TMA bulk-copy engine: one elected thread per CTA streams a tile through a
// ring of shared-memory stages: cp.async.bulk global->smem (mbarrier
// complete_tx), then cp.async.bulk smem->global for every destination.
constexpr int kTmaStages = 4;
constexpr int kTmaChunk = 32 * 1024;  // bytes per stage

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"(smem_u32(smem)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

template <bool kRelay>
__global__ void __launch_bounds__(32) k_push_tiles_tma(PushArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kTmaStages * kTmaChunk);
  if (threadIdx.x != 0) return;
  for (int s = 0; s < kTmaStages; ++s) mbar_init(&bars[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const char* src = reinterpret_cast<const char*>(a.src);
  uint32_t first = 0;  // running use count of the slot ring (slot = use % kTmaStages)
  for (int t = a.t0 + blockIdx.x; t < a.t1; t += gridDim.x) {
    if (kRelay) {
      if (!spin_until_geq(a.wait_flags + t, a.epoch)) continue;  // never forward stale bytes
      // relayed bytes arrived through the generic proxy; TMA reads via the async proxy
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    const int64_t b = a.tile_off[t], e = a.tile_off[t + 1];
    const int n = static_cast<int>((e - b + kTmaChunk - 1) / kTmaChunk);
    auto chunk_bytes = [&](int c) {
      return static_cast<uint32_t>(tmin<int64_t>(kTmaChunk, e - b - int64_t(c) * kTmaChunk));
    };
    auto load = [&](int c) {
      const uint32_t slot = (first + c) % kTmaStages;
      const uint32_t nb = chunk_bytes(c);
      mbar_expect_tx(&bars[slot], nb);
      bulk_g2s(smem + slot * kTmaChunk, src + b + int64_t(c) * kTmaChunk, nb, &bars[slot]);
    };
    for (int c = 0; c < n && c < kTmaStages; ++c) load(c);
    for (int c = 0; c < n; ++c) {
      const uint32_t g = first + c, slot = g % kTmaStages;
      mbar_wait(&bars[slot], (g / kTmaStages) & 1);
      const uint32_t nb = chunk_bytes(c);
      for (int d = 0; d < a.ndst; ++d)
        bulk_s2g(reinterpret_cast<char*>(a.dst[d]) + b + int64_t(c) * kTmaChunk, smem + slot * kTmaChunk, nb);
      bulk_commit();
      // refill the slot of chunk c-1 with chunk c+S-1 once chunk c-1's stores have read it
      const int nxt = c + kTmaStages - 1;
      if (c >= 1 && nxt < n) {
        bulk_wait_read<1>();
        load(nxt);
      }
    }
    first += n;
    bulk_wait_all();
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __threadfence_system();
    for (int d = 0; d < a.ndst; ++d) st_release_sys(a.flags[d] + t, a.epoch);
  }
}

// ---------------------------------------------------------------------------
__global__ void k_set_flags(uint32_t* flags, int t0, int t1, uint32_t epoch, int relay) {
  if (relay && *reinterpret_cast<volatile uint32_t*>(&g_poisoned_epoch) == epoch) return;
  int t = t0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (t < t1) st_release_sys(flags + t, epoch);
}

__global__ void __launch_bounds__(32) k_track_layers(const uint32_t* flags, const int32_t* layer_tile,
                                                     int nlayers, uint32_t epoch, uint32_t* loaded,
                                                     uint64_t* stamps) {
  const int lane = threadIdx.x;
  for (int k = 0; k < nlayers; ++k) {
    bool ok = true;
    for (int t = layer_tile[k] + lane; t < layer_tile[k + 1] && ok; t += 32) ok = spin_until_geq(flags + t, epoch);
    // a timed-out tile: layer k is not loaded -- stop publishing (gated compute
    // and the host both see the timeout rather than stale weights)
    if (!__all_sync(0xffffffffu, ok)) return;
    if (lane == 0) {
      stamps[k] = globaltimer();
      __threadfence_system();
      st_release_sys(loaded, static_cast<uint32_t>(k + 1));
    }
    __syncwarp();
  }
}

__global__ void k_publish_layer(uint32_t* loaded, uint32_t value, uint64_t* stamp) {
  if (stamp) *stamp = globaltimer();
  __threadfence_system();
  st_release_sys(loaded, value);
}

__global__ void k_wait_flag(const uint32_t* flag, uint32_t value) { spin_until_geq(flag, value); }

// one warp: every flag in [t0, t1) >= epoch (gate in front of a copy-engine relay)
__global__ void __launch_bounds__(32) k_wait_range(const uint32_t* flags, int t0, int t1, uint32_t epoch) {
  bool ok = true;
  for (int t = t0 + threadIdx.x; t < t1 && ok; t += 32) ok = spin_until_geq(flags + t, epoch);
  if (!ok) atomicExch(&g_poisoned_epoch, epoch);
}

// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__global__ void k_fill_random(uint64_t* dst, uint64_t nwords, uint64_t seed) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (uint64_t w = 2 * i; w + 1 < nwords; w += 2 * stride) {
    ulonglong2 v;
    v.x = splitmix64(seed + w);
    v.y = splitmix64(seed + w + 1);
    *reinterpret_cast<ulonglong2*>(dst + w) = v;
  }
  if ((nwords & 1) && i == 0) dst[nwords - 1] = splitmix64(seed + nwords - 1);
}

// Fingerprint of a tile: sum over its 8-byte words of splitmix64(word ^ splitmix64(index)),
// index relative to the tile start -- order independent, position sensitive.
__global__ void __launch_bounds__(256) k_tile_fingerprints(const uint64_t* base, const int64_t* tile_off,
                                                           int t0, int t1, uint64_t* out) {
  __shared__ uint64_t part[8];
  for (int t = t0 + blockIdx.x; t < t1; t += gridDim.x) {
    const int64_t b = tile_off[t] >> 3, e = tile_off[t + 1] >> 3;
    uint64_t acc = 0;
    for (int64_t i = b + threadIdx.x; i < e; i += blockDim.x)
      acc += splitmix64(base[i] ^ splitmix64(static_cast<uint64_t>(i - b)));
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint64_t s = 0;
      for (int w = 0; w < int(blockDim.x >> 5); ++w) s += part[w];
      out[t - t0] = s;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kThreads) k_handoff(const int4* __restrict__ src, int4* dst, int64_t n16,
                                                      uint32_t* flag) {
  const int64_t per = (n16 + gridDim.x - 1) / gridDim.x;
  const int64_t b = tmin<int64_t>(n16, per * blockIdx.x), e = tmin<int64_t>(n16, b + per);
  int4* const outs[1] = {dst};
  copy_tile<true, false>(src, outs, 1, b, e);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(flag) : "memory");
  }
}

// n_panels equal strided panels: copy the first `n16` 16-byte words of panel q
// (src + q * stride16) to dst + q * dst_stride16.  dst may be a peer mapping.
// Used to consolidate the KV prefix of a cooperative pair onto the new instance.
__global__ void __launch_bounds__(kThreads) k_copy_panels(const int4* __restrict__ src, int4* dst, int64_t n_panels,
                                                          int64_t src_stride16, int64_t dst_stride16, int64_t n16) {
  const int64_t total = n_panels * n16;
  const int64_t per = (total + gridDim.x - 1) / gridDim.x;
  const int64_t b = tmin<int64_t>(total, per * blockIdx.x), e = tmin<int64_t>(total, b + per);
  for (int64_t w = b + threadIdx.x; w < e; w += kThreads * 4) {
    int4 v[4];
    int64_t q[4], r[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = w + u * kThreads;
      q[u] = i / n16;
      r[u] = i - q[u] * n16;
      if (i < e) v[u] = ld16<false>(src + q[u] * src_stride16 + r[u]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (w + u * kThreads < e) st16(dst + q[u] * dst_stride16 + r[u], v[u]);
  }
}

}  // namespace bz

// ===========================================================================
// C ABI
using namespace bz;

static int fill_push_args(PushArgs& a, const void* src, void* const* dst, uint32_t* const* dst_flags,
                          int ndst, const uint32_t* wait_flags, const int64_t* tile_off, int t0, int t1,
                          uint32_t epoch) {
  if (!src || ndst < 1 || ndst > BZ_MAX_DST || !tile_off || t0 < 0 || t1 < t0)
    return bz_fail(BZ_EINVAL, "push: bad arguments");
  a.src = static_cast<const int4*>(src);
  for (int d = 0; d < BZ_MAX_DST; ++d) {
    a.dst[d] = d < ndst ? static_cast<int4*>(dst[d]) : nullptr;
    a.flags[d] = d < ndst ? dst_flags[d] : nullptr;
  }
  a.ndst = ndst;
  a.wait_flags = wait_flags;
  a.tile_off = tile_off;
  a.ids = nullptr;
  a.notify = nullptr;
  a.t0 = t0;
  a.t1 = t1;
  a.epoch = epoch;
  return BZ_OK;
}

// Pull: k_push_tiles launched on the RECEIVING GPU with the sender's slab (through the
// peer mapping) as src.  (A pull-only kernel with the destination count fixed at one let
// ptxas interleave the non-coherent loads with the stores -- ~3 NVLink reads in flight
// per thread, 589 vs 782 GB/s at 64 CTAs; copy_tile's runtime destination loop keeps
// all U loads ahead of the stores.)
extern "C" int bz_pull_tiles(const void* src, void* dst, uint32_t* dst_flags, const uint32_t* wait_flags,
                             uint32_t* notify_flags, const int64_t* tile_off, int t0, int t1, uint32_t epoch,
                             int nctas, void* stream) {
  void* dsts[1] = {dst};
  uint32_t* flags[1] = {dst_flags};
  PushArgs a;
  int rc = fill_push_args(a, src, dsts, flags, 1, wait_flags, tile_off, t0, t1, epoch);
  if (rc) return rc;
  if (!dst || !dst_flags) return bz_fail(BZ_EINVAL, "pull: destination and flags required");
  a.notify = notify_flags;
  if (t1 == t0) return BZ_OK;
  const int grid = nctas > 0 ? min(nctas, t1 - t0) : min(64, t1 - t0);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (wait_flags)
    k_push_tiles<true><<<grid, kThreads, 0, s>>>(a);
  else
    k_push_tiles<false><<<grid, kThreads, 0, s>>>(a);
  return bz_check_launch("bz_pull_tiles");
}

extern "C" int bz_push_tiles(const void* src, void* const* dst, uint32_t* const* dst_flags, int ndst,
                             const uint32_t* wait_flags, const int64_t* tile_off, int t0, int t1,
                             uint32_t epoch, int nctas, int engine, void* stream) {
  PushArgs a;
  int rc = fill_push_args(a, src, dst, dst_flags, ndst, wait_flags, tile_off, t0, t1, epoch);
  if (rc) return rc;
  if (t1 == t0) return BZ_OK;
  const int grid = nctas > 0 ? min(nctas, t1 - t0) : min(32, t1 - t0);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (engine == 1) {
    const int smem = kTmaStages * kTmaChunk + kTmaStages * 8;
    auto kern = wait_flags ? k_push_tiles_tma<true> : k_push_tiles_tma<false>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<grid, 32, smem, s>>>(a);
  } else if (engine == 2) {
    // 256-bit path: needs 32-byte aligned bases and tile offsets (slabs are 256-B aligned)
    uintptr_t align = reinterpret_cast<uintptr_t>(src);
    for (int d = 0; d < ndst; ++d) align |= reinterpret_cast<uintptr_t>(dst[d]);
    if (align & 31) return bz_fail(BZ_EINVAL, "push (256-bit): bases must be 32-byte aligned");
    if (wait_flags)
      k_push_tiles32<true><<<grid, kThreads, 0, s>>>(a);
    else
      k_push_tiles32<false><<<grid, kThreads, 0, s>>>(a);
  } else if (wait_flags) {
    k_push_tiles<true><<<grid, kThreads, 0, s>>>(a);
  } else {
    k_push_tiles<false><<<grid, kThreads, 0, s>>>(a);
  }
  return bz_check_launch("bz_push_tiles");
}

// Push an arbitrary list of tiles (ids[0..n)), each gated on this GPU's own
// flag when wait_flags is given: a striped host load pushes the pieces this GPU
// staged to every other member of its NVLink group, layer by layer.
extern "C" int bz_push_tile_list(const void* src, void* const* dst, uint32_t* const* dst_flags, int ndst,
                                 const uint32_t* wait_flags, const int64_t* tile_off, const int32_t* ids, int n,
                                 uint32_t epoch, int nctas, void* stream) {
  PushArgs a;
  int rc = fill_push_args(a, src, dst, dst_flags, ndst, wait_flags, tile_off, 0, n, epoch);
  if (rc) return rc;
  if (n == 0) return BZ_OK;
  if (!ids) return bz_fail(BZ_EINVAL, "push_tile_list: null tile list");
  a.ids = ids;
  const int grid = nctas > 0 ? min(nctas, n) : min(32, n);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (wait_flags)
    k_push_tiles<true><<<grid, kThreads, 0, s>>>(a);
  else
    k_push_tiles<false><<<grid, kThreads, 0, s>>>(a);
  return bz_check_launch("bz_push_tile_list");
}

extern "C" int bz_multicast_tiles(const void* src, void* mc_dst, uint32_t* mc_flags, const uint32_t* wait_flags,
                                  const int64_t* tile_off, int t0, int t1, uint32_t epoch, int nctas,
                                  void* stream) {
  PushArgs a;
  void* dsts[1] = {mc_dst};
  uint32_t* flags[1] = {mc_flags};
  int rc = fill_push_args(a, src, dsts, flags, 1, wait_flags, tile_off, t0, t1, epoch);
  if (rc) return rc;
  if (t1 == t0) return BZ_OK;
  const int grid = nctas > 0 ? min(nctas, t1 - t0) : min(32, t1 - t0);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // stores in flight per thread (multimem.st.v4 = 16 B each); BZ_MC_UNROLL selects
  // 4 / 8 (default) / 16 for sweeps (scripts/nvlink_probe.py)
  const char* env = getenv("BZ_MC_UNROLL");
  const int unroll = env ? atoi(env) : 8;
  auto kern = wait_flags ? k_multicast_tiles<true, 8> : k_multicast_tiles<false, 8>;
  if (unroll == 4) kern = wait_flags ? k_multicast_tiles<true, 4> : k_multicast_tiles<false, 4>;
  if (unroll == 16) kern = wait_flags ? k_multicast_tiles<true, 16> : k_multicast_tiles<false, 16>;
  kern<<<grid, kThreads, 0, s>>>(a);
  return bz_check_launch("bz_multicast_tiles");
}

extern "C" int bz_stage_tiles_ce(const void* host_src, void* dst, uint32_t* dst_flags,
                                 const int64_t* tile_off_host, int t0, int t1, int tiles_per_copy,
                                 uint32_t epoch, void* stream) {
  if (!host_src || !dst || !dst_flags || !tile_off_host || t0 < 0 || t1 < t0 || tiles_per_copy < 1)
    return bz_fail(BZ_EINVAL, "stage_ce: bad arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (int t = t0; t < t1; t += tiles_per_copy) {
    const int te = min(t1, t + tiles_per_copy);
    const int64_t b = tile_off_host[t], e = tile_off_host[te];
    cudaError_t err = cudaMemcpyAsync(static_cast<char*>(dst) + b, static_cast<const char*>(host_src) + b,
                                      static_cast<size_t>(e - b), cudaMemcpyHostToDevice, s);
    if (err != cudaSuccess) return bz_fail_cuda(err, "stage_ce memcpy");
    k_set_flags<<<(te - t + 127) / 128, 128, 0, s>>>(dst_flags, t, te, epoch, 0);
  }
  return bz_check_launch("bz_stage_tiles_ce");
}

// Chain hop on the copy engines: no SM moves bytes (the SMs stay with the
// cooperating instance's GEMMs).  Per group of tiles: [relay: one-warp gate on
// the group's upstream flags] -> cudaMemcpyAsync into the peer mapping -> flag
// kernel (system-scope release into the peer's flag array).
//
// With a `flag_stream` the flag kernels run there, each behind an event recorded
// after its group's copy: the copy stream then carries only copies (and relay
// gates), so the copy engine streams back to back instead of idling for a kernel
// launch between groups.
// per host thread: a record + wait pair is enqueued back to back by one thread, so
// another thread's calls can never re-record an event between them
static cudaEvent_t pooled_event(int dev, size_t i) {
  static thread_local std::vector<cudaEvent_t> pool[64];
  auto& v = pool[dev < 64 ? dev : 63];
  while (v.size() <= i) {
    cudaEvent_t e;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
    v.push_back(e);
  }
  return v[i];
}

static int push_ce(const void* src, void* dst, uint32_t* dst_flags, const uint32_t* wait_flags,
                   const int64_t* tile_off_host, int t0, int t1, int tiles_per_copy, uint32_t epoch, void* stream,
                   void* flag_stream, void* gate_stream = nullptr) {
  if (!src || !dst || !dst_flags || !tile_off_host || t0 < 0 || t1 < t0 || tiles_per_copy < 1)
    return bz_fail(BZ_EINVAL, "push_ce: bad arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaStream_t fs = static_cast<cudaStream_t>(flag_stream);
  cudaStream_t gs = static_cast<cudaStream_t>(gate_stream);
  int dev = 0;
  cudaGetDevice(&dev);
  const int ngroups = (t1 - t0 + tiles_per_copy - 1) / tiles_per_copy;
  if (wait_flags && gs) {
    // relay gates on their own stream, enqueued ahead: the copy stream only waits on
    // events between copies (no kernel in the copy engine's way)
    cudaEvent_t start = pooled_event(dev, 2 * ngroups + 1);
    if (!start) return bz_fail(BZ_ECUDA, "push_ce: event pool");
    cudaEventRecord(start, s);
    cudaStreamWaitEvent(gs, start, 0);
    for (int g = 0; g < ngroups; ++g) {
      const int t = t0 + g * tiles_per_copy, te = min(t1, t + tiles_per_copy);
      k_wait_range<<<1, 32, 0, gs>>>(wait_flags, t, te, epoch);
      cudaEvent_t ev = pooled_event(dev, ngroups + 1 + g);
      if (!ev) return bz_fail(BZ_ECUDA, "push_ce: event pool");
      cudaEventRecord(ev, gs);
    }
  }
  size_t group = 0;
  for (int t = t0; t < t1; t += tiles_per_copy, ++group) {
    const int te = min(t1, t + tiles_per_copy);
    if (wait_flags && gs)
      cudaStreamWaitEvent(s, pooled_event(dev, ngroups + 1 + group), 0);
    else if (wait_flags)
      k_wait_range<<<1, 32, 0, s>>>(wait_flags, t, te, epoch);
    const int64_t b = tile_off_host[t], e = tile_off_host[te];
    cudaError_t err = cudaMemcpyAsync(static_cast<char*>(dst) + b, static_cast<const char*>(src) + b,
                                      static_cast<size_t>(e - b), cudaMemcpyDeviceToDevice, s);
    if (err != cudaSuccess) return bz_fail_cuda(err, "push_ce memcpy");
    if (fs) {
      cudaEvent_t ev = pooled_event(dev, group);
      if (!ev) return bz_fail(BZ_ECUDA, "push_ce: event pool");
      cudaEventRecord(ev, s);
      cudaStreamWaitEvent(fs, ev, 0);
      k_set_flags<<<(te - t + 127) / 128, 128, 0, fs>>>(dst_flags, t, te, epoch, wait_flags != nullptr);
    } else {
      k_set_flags<<<(te - t + 127) / 128, 128, 0, s>>>(dst_flags, t, te, epoch, wait_flags != nullptr);
    }
  }
  if (fs) {  // the copy stream's completion implies the flags: join the flag stream back
    cudaEvent_t ev = pooled_event(dev, group);
    if (!ev) return bz_fail(BZ_ECUDA, "push_ce: event pool");
    cudaEventRecord(ev, fs);
    cudaStreamWaitEvent(s, ev, 0);
  }
  return bz_check_launch("bz_push_tiles_ce");
}

extern "C" int bz_push_tiles_ce(const void* src, void* dst, uint32_t* dst_flags, const uint32_t* wait_flags,
                                const int64_t* tile_off_host, int t0, int t1, int tiles_per_copy, uint32_t epoch,
                                void* stream) {
  return push_ce(src, dst, dst_flags, wait_flags, tile_off_host, t0, t1, tiles_per_copy, epoch, stream, nullptr);
}

extern "C" int bz_push_tiles_ce2(const void* src, void* dst, uint32_t* dst_flags, const uint32_t* wait_flags,
                                 const int64_t* tile_off_host, int t0, int t1, int tiles_per_copy, uint32_t epoch,
                                 void* stream, void* flag_stream) {
  if (!flag_stream) return bz_fail(BZ_EINVAL, "push_ce2: flag_stream required");
  return push_ce(src, dst, dst_flags, wait_flags, tile_off_host, t0, t1, tiles_per_copy, epoch, stream, flag_stream);
}

extern "C" int bz_push_tiles_ce_gated(const void* src, void* dst, uint32_t* dst_flags, const uint32_t* wait_flags,
                                      const int64_t* tile_off_host, int t0, int t1, int tiles_per_copy,
                                      uint32_t epoch, void* stream, void* flag_stream, void* gate_stream) {
  if (!flag_stream || !gate_stream) return bz_fail(BZ_EINVAL, "push_ce_gated: flag and gate streams required");
  return push_ce(src, dst, dst_flags, wait_flags, tile_off_host, t0, t1, tiles_per_copy, epoch, stream, flag_stream,
                 gate_stream);
}

extern "C" int bz_stage_tiles_sm(const void* host_src, void* dst, uint32_t* dst_flags, const int64_t* tile_off,
                                 int t0, int t1, uint32_t epoch, int nctas, void* stream) {
  void* dsts[1] = {dst};
  uint32_t* flags[1] = {dst_flags};
  PushArgs a;
  int rc = fill_push_args(a, host_src, dsts, flags, 1, nullptr, tile_off, t0, t1, epoch);
  if (rc) return rc;
  if (t1 == t0) return BZ_OK;
  const int grid = nctas > 0 ? min(nctas, t1 - t0) : min(16, t1 - t0);
  k_push_tiles<false><<<grid, kThreads, 0, static_cast<cudaStream_t>(stream)>>>(a);
  return bz_check_launch("bz_stage_tiles_sm");
}

extern "C" int bz_track_layers(const uint32_t* flags, const int32_t* layer_tile, int nlayers, uint32_t epoch,
                               uint32_t* loaded, uint64_t* stamps, void* stream) {
  if (!flags || !layer_tile || nlayers < 1 || !loaded || !stamps) return bz_fail(BZ_EINVAL, "track: bad args");
  k_track_layers<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(flags, layer_tile, nlayers, epoch, loaded,
                                                                   stamps);
  return bz_check_launch("bz_track_layers");
}

extern "C" int bz_publish_layer(uint32_t* loaded, uint32_t value, uint64_t* stamp, void* stream) {
  k_publish_layer<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(loaded, value, stamp);
  return bz_check_launch("bz_publish_layer");
}

extern "C" int bz_wait_layer(const uint32_t* loaded, uint32_t k, void* stream) {
  const DriverApi* d = driver_api();
  if (!d) return BZ_ECUDA;
  CUresult r = d->cuStreamWaitValue32(static_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(loaded), k,
                                      CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) return bz_fail_cu(r, "cuStreamWaitValue32");
  return BZ_OK;
}

extern "C" int bz_wait_timeouts(uint64_t* count, uint64_t budget_ns) {
  unsigned long long v = 0;
  cudaError_t e = cudaMemcpyFromSymbol(&v, g_wait_timeouts, sizeof(v));
  if (e != cudaSuccess) return bz_fail_cuda(e, "read wait timeouts");
  *count = v;
  if (budget_ns) {
    e = cudaMemcpyToSymbol(c_spin_budget_ns, &budget_ns, sizeof(budget_ns));
    if (e != cudaSuccess) return bz_fail_cuda(e, "set spin budget");
  }
  return BZ_OK;
}

extern "C" int bz_wait_flag_kernel(const uint32_t* flag, uint32_t value, void* stream) {
  k_wait_flag<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(flag, value);
  return bz_check_launch("bz_wait_flag_kernel");
}

extern "C" int bz_fill_random(void* dst, uint64_t bytes, uint64_t seed, void* stream) {
  if (!dst || (bytes & 15)) return bz_fail(BZ_EINVAL, "fill_random: dst must be 16-byte sized");
  const uint64_t nwords = bytes >> 3;
  int grid = static_cast<int>(tmin<uint64_t>(148 * 8, (nwords / 2 + 255) / 256 + 1));
  k_fill_random<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<uint64_t*>(dst), nwords, seed);
  return bz_check_launch("bz_fill_random");
}

extern "C" int bz_tile_fingerprints(const void* base, const int64_t* tile_off, int t0, int t1, uint64_t* out,
                                    void* stream) {
  if (!base || !tile_off || !out || t1 < t0) return bz_fail(BZ_EINVAL, "fingerprints: bad args");
  if (t1 == t0) return BZ_OK;
  int grid = min(t1 - t0, 148 * 4);
  k_tile_fingerprints<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<const uint64_t*>(base),
                                                                          tile_off, t0, t1, out);
  return bz_check_launch("bz_tile_fingerprints");
}

extern "C" int bz_handoff(const void* src, void* dst, uint64_t bytes, uint32_t* flag, uint32_t /*value*/,
                          int nctas, void* stream) {
  if (!src || !dst || !flag || (bytes & 15)) return bz_fail(BZ_EINVAL, "handoff: bad args");
  const int grid = nctas > 0 ? nctas : 16;
  k_handoff<<<grid, kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const int4*>(src), static_cast<int4*>(dst), static_cast<int64_t>(bytes >> 4), flag);
  return bz_check_launch("bz_handoff");
}

extern "C" int bz_copy_panels(const void* src, void* dst, int64_t n_panels, int64_t src_stride, int64_t dst_stride,
                              int64_t panel_bytes, int nctas, void* stream) {
  if (!src || !dst || n_panels < 0 || panel_bytes < 0 || ((src_stride | dst_stride | panel_bytes) & 15) ||
      (reinterpret_cast<uintptr_t>(src) & 15) || (reinterpret_cast<uintptr_t>(dst) & 15))
    return bz_fail(BZ_EINVAL, "copy_panels: 16-byte aligned pointers, strides and sizes required");
  if (n_panels == 0 || panel_bytes == 0) return BZ_OK;
  const int grid = nctas > 0 ? nctas : 64;
  k_copy_panels<<<grid, kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const int4*>(src), static_cast<int4*>(dst), n_panels, src_stride >> 4, dst_stride >> 4,
      panel_bytes >> 4);
  return bz_check_launch("bz_copy_panels");
}

const void* bz::module_anchor_dataplane() { return reinterpret_cast<const void*>(k_set_flags); }
