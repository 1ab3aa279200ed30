/* blitz.h -- C ABI of libblitz.so, the sm_100a live-autoscaling data plane.
 *
 * Plain pointers, sizes and stream handles; no torch types.  Every entry point
 * returns 0 on success or a negative BZ_E* code, with a message available from
 * bz_last_error() (thread-local).  Nothing here falls back to the CPU: a CUDA
 * failure is returned to the caller, which raises.
 *
 * The reference (/root/reference/pkg/src/scalesim) has NO native layer -- it
 * models these mechanisms as arithmetic.  Each entry point names the modeled
 * item it realises:
 *   weight slabs + peer mesh     <- the pre-established NVLink/RDMA connection pool
 *                                   (SURVEY.md §5 "communication backend")
 *   bz_push_tiles                <- a chain edge's store-and-forward transfer
 *                                   (planner.py:240-244 PlanEdge hop; simcore.py:690-703)
 *   bz_pull_tiles                <- the same hop out of a live source into a leaf, run by
 *                                   the receiving GPU (the source spends no SM)
 *   bz_push_tiles_ce2 / _ce_gated <- the hop on the copy engines (a relay chain; the live pair)
 *   bz_multicast_tiles           <- ScalePlan.nvlink_fanout intra-host broadcast
 *                                   (planner.py:86-87, 245-253)
 *   bz_stage_tiles_ce / _sm      <- mem<h> -> gpu pcie source edge; autoscaler.baseline_load_time
 *                                   (topology.py:174-176; autoscaler.py:102-117)
 *   bz_track_layers              <- per-layer LayerLoaded(k) events
 *                                   (simcore.py:727-733, 752-763; livescale.py:458-468)
 *   bz_wait_layer                <- gating execution of layer k on its arrival
 *   bz_gemm_bf16                 <- the per-layer prefill cost model ModelSpec.prefill_ms
 *                                   (parampool.py:58-62): the real layer GEMMs
 *
 * Memory model.  A slab is one VMM allocation (cuMemCreate, POSIX-FD
 * shareable) holding a model shard laid out layer by layer, followed by a
 * u32 tile-flag array.  Tiles never straddle layers.  flag[t] >= epoch means
 * tile t of this slab holds the bytes of transfer `epoch`.
 */
#ifndef BLITZ_H
#define BLITZ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  BZ_OK = 0,
  BZ_ECUDA = -1,    /* CUDA runtime/driver error */
  BZ_EINVAL = -2,   /* bad arguments */
  BZ_ESYS = -3,     /* OS error (pidfd, fd passing) */
  BZ_EUNSUP = -4    /* device lacks the feature (e.g. NVLS multicast) */
};

#define BZ_MAX_DST 8

const char* bz_last_error(void);
int bz_version(void);

/* ---- devices ------------------------------------------------------------ */
int bz_device_count(int* n);
int bz_device_caps(int dev, int* multicast, int* posix_fd, int* fabric, int* sm_count);
/* Enable peer access from `dev` to every other visible device (the "connection pool"). */
int bz_enable_peer_mesh(int dev);

/* ---- weight slabs (VMM) ------------------------------------------------------- */
typedef struct {
  uint64_t ptr;        /* device VA of the mapping in this process */
  uint64_t bytes;      /* mapped size (rounded to granularity) */
  uint64_t handle;     /* CUmemGenericAllocationHandle */
  int dev;             /* device the memory lives on */
  int fd;              /* exported POSIX fd (owner) or imported fd, -1 if none */
} bz_slab;

/* Physical allocation on `dev`, mapped RW for `dev`.  Rounded up to the
 * multicast granularity so it can be bound into a multicast object. */
int bz_slab_create(int dev, uint64_t bytes, bz_slab* out);
/* Export as a POSIX fd (stored in out->fd). */
int bz_slab_export(bz_slab* slab);
/* Import a peer process's slab: (owner_pid, owner_fd) come from bz_slab_export
 * in that process; mapped RW for `local_dev`, giving a peer VA over NVLink. */
int bz_slab_import(int local_dev, int owner_pid, int owner_fd, uint64_t bytes, bz_slab* out);
int bz_slab_free(bz_slab* slab);

/* ---- NVLS multicast ----------------------------------------------------------- */
typedef struct {
  uint64_t handle;     /* CUmemGenericAllocationHandle of the multicast object */
  uint64_t mc_ptr;     /* VA of the multicast mapping in this process (0 until mapped) */
  uint64_t bytes;
  int fd;
} bz_mc;

int bz_mc_granularity(int dev, int ndev, uint64_t* min_gran, uint64_t* rec_gran);
int bz_mc_create(int ndev, uint64_t bytes, bz_mc* out);         /* root; exports fd */
int bz_mc_import(int owner_pid, int owner_fd, uint64_t bytes, bz_mc* out);
int bz_mc_add_device(bz_mc* mc, int dev);
int bz_mc_bind(bz_mc* mc, int dev, const bz_slab* slab, uint64_t slab_offset,
               uint64_t mc_offset, uint64_t bytes);
int bz_mc_map(bz_mc* mc, int dev);
int bz_mc_free(bz_mc* mc, int dev, uint64_t bound_bytes);
/* Unbind `dev`'s memory from the object without releasing it (a process that
 * bound slabs on several of its GPUs unbinds each before bz_mc_free). */
int bz_mc_unbind(bz_mc* mc, int dev, uint64_t bound_bytes);

/* ---- tile transfer kernels ---------------------------------------------------- */
/* Tile table: tile t covers bytes [tile_off[t], tile_off[t+1]) of a slab
 * (device array of ntiles+1 int64, 16-byte aligned offsets).
 *
 * bz_push_tiles: copy tiles [t0, t1) from `src` to each of the ndst
 * destination bases (peer VAs or local), then publish dst_flags[d][t] = epoch
 * with a system-scope release.  If wait_flags != NULL the tile is forwarded
 * only after wait_flags[t] >= epoch (store-and-forward relay of a chain hop).
 * engine: 0 = 16-byte vector LD/ST, 1 = TMA bulk copy (cp.async.bulk). */
int bz_push_tiles(const void* src, void* const* dst, uint32_t* const* dst_flags, int ndst,
                  const uint32_t* wait_flags, const int64_t* tile_off, int t0, int t1,
                  uint32_t epoch, int nctas, int engine, void* stream);

/* bz_pull_tiles: the receiving GPU's SMs copy tiles [t0, t1) from `src` (the sender's
 * slab through this GPU's peer mapping) into the local `dst`, raising dst_flags[t] =
 * epoch (system-scope release); with wait_flags (e.g. a relaying sender's flags through
 * the peer mapping) tile t is read only after wait_flags[t] >= epoch; notify_flags
 * (nullable) receives the same release.  The realisation of a source -> leaf PlanEdge
 * hop (planner.py:240-244): NVLink reads carry less protocol than writes, 781 GB/s vs
 * 717 for a push (profiles/r2_pull_probe_n2.txt), and the source spends no SM. */
int bz_pull_tiles(const void* src, void* dst, uint32_t* dst_flags, const uint32_t* wait_flags,
                  uint32_t* notify_flags, const int64_t* tile_off, int t0, int t1, uint32_t epoch, int nctas,
                  void* stream);

/* bz_push_tile_list: bz_push_tiles over an explicit tile list ids[0..n) (device
 * int32), 16-byte vector engine.  Striped host-cache load: every member of a
 * host-fed NVLink group stages its piece of each layer over its own PCIe link
 * and forwards that piece to the other members (the mem<h> -> rep pcie edge plus
 * ScalePlan.nvlink_fanout, planner.py:86-87, 245-253, realised over all the
 * group's host links). */
int bz_push_tile_list(const void* src, void* const* dst, uint32_t* const* dst_flags, int ndst,
                      const uint32_t* wait_flags, const int64_t* tile_off, const int32_t* ids, int n,
                      uint32_t epoch, int nctas, void* stream);

/* bz_push_tiles_ce: the same hop on the copy engines (one destination): per
 * group of `tiles_per_copy` tiles, [relay: one-warp gate until wait_flags of the
 * group >= epoch] -> cudaMemcpyAsync into the peer VA -> release of dst_flags.
 * tile_off_host is a host copy of the tile table.  Keeps the SMs for compute. */
int bz_push_tiles_ce(const void* src, void* dst, uint32_t* dst_flags, const uint32_t* wait_flags,
                     const int64_t* tile_off_host, int t0, int t1, int tiles_per_copy, uint32_t epoch,
                     void* stream);
/* The same with the flag releases on `flag_stream` (each behind an event after its
 * group's copy), so `stream` carries only copies (+ relay gates) and the copy engine
 * runs back to back; `stream` joins `flag_stream` at the end. */
int bz_push_tiles_ce2(const void* src, void* dst, uint32_t* dst_flags, const uint32_t* wait_flags,
                      const int64_t* tile_off_host, int t0, int t1, int tiles_per_copy, uint32_t epoch,
                      void* stream, void* flag_stream);

/* The same with a relay's gates (one-warp waits on wait_flags per copy group, bounded
 * spin with the usual timeout / poison rule) enqueued ahead on `gate_stream`: `stream`
 * waits on one event per group instead of a kernel, so the copy engine does not idle
 * behind gate launches. */
int bz_push_tiles_ce_gated(const void* src, void* dst, uint32_t* dst_flags, const uint32_t* wait_flags,
                           const int64_t* tile_off_host, int t0, int t1, int tiles_per_copy, uint32_t epoch,
                           void* stream, void* flag_stream, void* gate_stream);

/* bz_multicast_tiles: one multimem.st stream into the multicast VA `mc_dst`
 * (bound to every receiver's slab); flags go through `mc_flags` (the
 * multicast VA of the receivers' flag arrays). */
int bz_multicast_tiles(const void* src, void* mc_dst, uint32_t* mc_flags,
                       const uint32_t* wait_flags, const int64_t* tile_off, int t0, int t1,
                       uint32_t epoch, int nctas, void* stream);

/* Host staging from pinned memory. _ce: copy engine, one cudaMemcpyAsync per
 * group of `tiles_per_copy` tiles followed by a flag update; _sm: a kernel that
 * reads the mapped host buffer (zero-copy) with 16-byte loads. */
int bz_stage_tiles_ce(const void* host_src, void* dst, uint32_t* dst_flags,
                      const int64_t* tile_off_host, int t0, int t1, int tiles_per_copy,
                      uint32_t epoch, void* stream);
int bz_stage_tiles_sm(const void* host_src, void* dst, uint32_t* dst_flags,
                      const int64_t* tile_off, int t0, int t1, uint32_t epoch, int nctas,
                      void* stream);

/* ---- layer readiness ---------------------------------------------------------------- */
/* One-warp tracker: for k = 0..nlayers-1 in order, waits until every tile of
 * layer k (tiles [layer_tile[k], layer_tile[k+1])) has flag >= epoch, then
 * publishes loaded[0] = k+1 (release, monotone) and stamps[k] = %globaltimer ns. */
int bz_track_layers(const uint32_t* flags, const int32_t* layer_tile, int nlayers,
                    uint32_t epoch, uint32_t* loaded, uint64_t* stamps, void* stream);
/* In-stream publish (producer on this GPU, e.g. copy-engine staging): after the
 * preceding work in `stream`, stamp[0] = %globaltimer, then *loaded = value. */
int bz_publish_layer(uint32_t* loaded, uint32_t value, uint64_t* stamp, void* stream);
/* Stream gate: blocks `stream` until *loaded >= k (cuStreamWaitValue32 GEQ). */
int bz_wait_layer(const uint32_t* loaded, uint32_t k, void* stream);
/* Device gate kernel variant of the same (spins with ld.acquire.sys). */
int bz_wait_flag_kernel(const uint32_t* flag, uint32_t value, void* stream);
/* Every device-side wait is bounded: after `budget` ns it gives up and counts a
 * timeout.  Returns the count for the current device (synchronous); a non-zero
 * budget_ns replaces the budget (default 30 s). */
int bz_wait_timeouts(uint64_t* count, uint64_t budget_ns);

/* ---- payload + verification ---------------------------------------------------------- */
/* Deterministic random bits: 64-bit word i = splitmix64(seed + i). */
int bz_fill_random(void* dst, uint64_t bytes, uint64_t seed, void* stream);
/* Per-tile 64-bit fingerprints of [tile_off[t], tile_off[t+1]) into out[t - t0]. */
int bz_tile_fingerprints(const void* base, const int64_t* tile_off, int t0, int t1,
                         uint64_t* out, void* stream);
/* Plain copy of a small buffer into a peer/local buffer followed by a release
 * flag store (activation handoff of cooperative execution). */
int bz_handoff(const void* src, void* dst, uint64_t bytes, uint32_t* flag, uint32_t value,
               int nctas, void* stream);
/* Copy the first panel_bytes of each of n_panels panels (src + q*src_stride ->
 * dst + q*dst_stride; dst may be a peer mapping).  KV consolidation after a
 * cooperative prefill: the source's [T_i, L) KV prefixes move to the new
 * instance (simcore.py:462-514 as real NVLink bytes). */
int bz_copy_panels(const void* src, void* dst, int64_t n_panels, int64_t src_stride, int64_t dst_stride,
                   int64_t panel_bytes, int nctas, void* stream);

/* ---- tensor-core GEMM (tcgen05 + TMEM + TMA) ----------------------------------------- */
/* The dense contraction the reference models as ModelSpec.prefill_ms /
 * decode_step_ms (parampool.py:58-62) and scales by max(k, L-k)/L for a live pair
 * (simcore.py:408-417): every projection of a Llama block on a cooperating instance.
 * C[M,N] = A[M,K] . B[N,K]^T (+ residual[M,N]), all bf16 row-major, fp32 accumulate in
 * TMEM.  B is a Linear weight [out, in].  K % 8 == 0 (tails zero-filled by TMA), N % 8 == 0,
 * leading dims % 8 == 0,
 * 16-byte aligned pointers.  residual may be NULL.  max_ctas <= 0: one CTA per SM. */
int bz_gemm_bf16(const void* A, const void* B, void* C, const void* residual, int M, int N, int K,
                 int lda, int ldb, int ldc, int ldr, int max_ctas, void* stream);
/* Fused GEMM -> hand-off: same GEMM, C may be a peer (NVLink) mapping of the
 * receiving instance's buffer; every CTA, after storing its tiles, adds 1 to
 * *signal with a system-scope release.  *ctas_out = number of CTAs launched, so
 * the receiver gates on (*signal >= previous + ctas_out) (bz_wait_layer). */
int bz_gemm_bf16_signal(const void* A, const void* B, void* C, const void* residual, int M, int N,
                        int K, int lda, int ldb, int ldc, int ldr, int max_ctas, uint32_t* signal,
                        int* ctas_out, void* stream);
/* General form.  With a caller-owned fp32 workspace (16-byte aligned) a skinny
 * problem (M <= 128 and fewer tiles than SMs, e.g. a decode step's M = batch
 * rows) runs stream-K: the tiles x K-blocks space is cut into equal ranges, one
 * per CTA; tiles shared by two or more CTAs are summed in fp32 (plus the
 * residual) by their last contributor.  workspace = NULL disables it.
 * Decode shapes (M <= 16, K % 64 == 0) take neither: when the 128-row weight
 * tiles fit the SMs the weights are the MMA's M operand and K is split over a
 * thread-block cluster summed in distributed shared memory (BZ_GEMM_SWAP=0 off),
 * else whole tiles of >= 128 rows stream K-chunked (BZ_GEMM_KC=0 off); neither
 * uses the workspace.
 * signal/ctas_out as in bz_gemm_bf16_signal.  All compute kernels are launched
 * with programmatic dependent launch (set-up overlaps the previous kernel;
 * BZ_PDL=0 disables).  The workspace must be zero-filled before its first use
 * (it holds per-tile arrival counters, which every call leaves at zero) and must
 * not be shared by GEMMs running concurrently. */
#define BZ_GEMM_C_F32 2u    /* C is fp32 (ldc in floats): the accumulator is stored unrounded (logit heads);
                               single-CTA tiles only */
#define BZ_GEMM_B_STATIC 1u /* B is not written by kernels still in flight on the stream (weights):
                               its first tiles may load before the predecessor kernel completes */
int bz_gemm_bf16_ex(const void* A, const void* B, void* C, const void* residual, int M, int N, int K,
                    int lda, int ldb, int ldc, int ldr, int max_ctas, unsigned flags, void* workspace,
                    int64_t workspace_bytes, uint32_t* signal, int* ctas_out, void* stream);

/* ---- Llama block glue (bf16 in/out, fp32 math) ---------------------------------------- */
/* y = x * rsqrt(mean(x^2) + eps) * w per row; d % 8 == 0. */
int bz_rmsnorm(const void* x, const void* w, void* y, int rows, int d, int ldx, int ldy, float eps,
               void* stream);
/* In-place rotate-half RoPE on the first n_rot_heads heads of each row of a fused
 * [q | k | v] projection; positions[rows] int32. */
int bz_rope(void* qkv, const int32_t* positions, int rows, int n_rot_heads, int head_dim, int ld,
            float theta, void* stream);
/* act[:, j] = silu(gu[:, j]) * gu[:, ffn + j]. */
int bz_silu_mul(const void* gu, void* act, int rows, int ffn, int ldg, int lda, void* stream);

/* ---- prefill attention (csrc/attention_tcgen05.cu) -------------------------------------
 * Causal softmax(Q K^T / sqrt(hd)) V for B sequences of S tokens on tcgen05 tensor
 * cores (TMEM accumulators, TMA-fed), GQA (n_heads % n_kv == 0), hd 64 or 128.
 * qkv: [B*S, ld] bf16 rows [q heads | k heads | v heads] with RoPE applied; out:
 * [B*S, ldo] bf16, head h at columns [h*hd, (h+1)*hd).  V is read in place as an MN-major
 * MMA operand; the workspace arguments are kept for ABI stability (0 bytes needed). */
int bz_prefill_attention_workspace_bytes(int B, int S, int n_kv, int head_dim, int64_t* bytes);
int bz_prefill_attention(const void* qkv, int ld, int B, int S, int n_heads, int n_kv, int head_dim,
                         void* workspace, int64_t workspace_bytes, void* out, int ldo, void* stream);

/* ---- KV-cache decode (csrc/decode_kernels.cu) -------------------------------------------
 * The decode position is read from device memory (*pos, int32), so a captured
 * decode step replays for every position.  Cache layout [rows, n_kv, s_max, hd]
 * bf16.  Replaces the reference's decode cost line ModelSpec.decode_step_ms
 * (parampool.py:61-62) for a prefill instance flipped to decode by
 * mutate_prefill_to_decode (livescale.py:512-536) and for cooperative decode. */
/* Rotate q (in place) and k of each row's fused [q | k | v] projection at
 * position *pos, and write k, v into the caches at that position. */
int bz_rope_append(void* qkv, int ld, int rows, int n_heads, int n_kv, int head_dim, float theta,
                   void* k_cache, void* v_cache, int64_t s_max, const int32_t* pos, void* stream);
/* Continuous batching: the same with one position per row, pos[rows] (each sequence
 * of the batch at its own length; a row at or past s_max is skipped). */
int bz_rope_append_rows(void* qkv, int ld, int rows, int n_heads, int n_kv, int head_dim, float theta,
                        void* k_cache, void* v_cache, int64_t s_max, const int32_t* pos, void* stream);
/* Bytes of workspace bz_decode_attention needs for these sizes. */
int bz_decode_workspace_bytes(int rows, int n_heads, int n_kv, int head_dim, int64_t s_max, int64_t* bytes);
/* out[r, h*hd:(h+1)*hd] = softmax(q_h K[0..*pos]^T / sqrt(hd)) V over each row's
 * cached prefix (GQA: head h reads kv head h / (n_heads / n_kv), 1/2/4/8 heads per kv head);
 * hd 64 or 128. */
int bz_decode_attention(const void* q, int ldq, const void* k_cache, const void* v_cache, int rows, int n_heads,
                        int n_kv, int head_dim, int64_t s_max, const int32_t* pos, void* out, int ldo,
                        void* workspace, int64_t workspace_bytes, void* stream);
/* ... with one position per row, pos[rows] (attended prefix pos[r] + 1 tokens). */
int bz_decode_attention_rows(const void* q, int ldq, const void* k_cache, const void* v_cache, int rows,
                             int n_heads, int n_kv, int head_dim, int64_t s_max, const int32_t* pos, void* out,
                             int ldo, void* workspace, int64_t workspace_bytes, void* stream);

/* ---- fused small-batch decode (csrc/decode_fused.cu) ------------------------------------
 * A whole decode step over n_blocks blocks in ONE persistent cooperative kernel
 * (1..4 sequences): per block rmsnorm -> qkv -> RoPE + KV append -> attention ->
 * o-proj + residual -> rmsnorm -> gate/up + SiLU -> down + residual, with each CTA
 * streaming its slice of every weight through shared memory (3-D TMA, 16-row units)
 * into warp tensor-core MMAs, and grid barriers between phases; d and ffn multiples of
 * 64; blocks beyond 48 run as further launches.  Same math and bf16 rounding points as bz_rmsnorm / bz_gemm_bf16 /
 * bz_rope_append(_rows) / bz_decode_attention(_rows) / bz_silu_mul.
 * x: [rows, ldx] bf16 hidden state, updated in place to the last block's output.
 * pos_stride 0: one device position for the batch (pos[0]); 1: one per row.
 * Workspace (bz_decode_fused_workspace_bytes) must be zeroed once before first use.
 * Per block (device pointers, the slab's tensor views): attn_norm [d], wqkv
 * [(n_heads + 2 n_kv) hd, d], wo [d, d], ffn_norm [d], wgu [2 ffn, d] (gate rows, then
 * up rows), wdown [d, ffn], caches [rows, n_kv, s_max, hd]. */
typedef struct bz_decode_block {
  const void* attn_norm;
  const void* wqkv;
  const void* wo;
  const void* ffn_norm;
  const void* wgu;
  const void* wdown;
  void* k_cache;
  void* v_cache;
} bz_decode_block;
int bz_decode_fused_workspace_bytes(int rows, int d, int n_heads, int n_kv, int head_dim, int ffn, int64_t* bytes);
int bz_decode_fused(const bz_decode_block* blocks, int n_blocks, void* x, int ldx, int rows, int d, int n_heads,
                    int n_kv, int head_dim, int ffn, float rope_theta, float eps, int64_t s_max, const int32_t* pos,
                    int pos_stride, void* workspace, int64_t workspace_bytes, int max_ctas, void* stream);
/* *timed_out = 1 if the last bz_decode_fused on this workspace hit its grid-barrier
 * timeout (a CTA never became resident); synchronises the stream. */
int bz_decode_fused_status(const void* workspace, int* timed_out, void* stream);
/* Diagnostics: while buf is set (device memory, >= grid * n_blocks * 22 * 8 bytes), every
 * bz_decode_fused launch stores a %globaltimer stamp per CTA, block and phase event
 * (scripts/fused_trace.py reads them); NULL turns it off. */
int bz_decode_fused_set_trace(void* buf, int64_t bytes);

/* ---- misc ------------------------------------------------------------------------------ */
int bz_sm_count(int dev, int* n);

/* Load every libblitz kernel into dev's context (returns how many).  CUDA lazy
 * loading would otherwise load a kernel at its first launch, which may wait for
 * the device to drain -- a deadlock if a resident gate/tracker kernel waits on
 * that launch.  Called once per device by the Python layer. */
int bz_preload_kernels(int dev, int* nloaded);

#ifdef __cplusplus
}
#endif
#endif /* BLITZ_H */
