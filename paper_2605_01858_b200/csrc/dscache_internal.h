// Internal launch parameters shared by the host bookkeeping (dscache_api.cu) and
// the sm_100a kernels.  Product code only; nothing here is visible through the ABI.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

// DSC_CHECK=1 builds (scripts/gpu_checked.sh): device-side bounds checks on every global
// address the kernels form (rows of the ring / sink / self / Q / O / workspaces, TMA boxes),
// trapping with the failing site -- the in-house substitute for compute-sanitizer, which is
// closed on the GPU pool.  Off (compiled out) in the product library.
#ifndef DSC_CHECK
#define DSC_CHECK 0
#endif
#if DSC_CHECK
#include <cstdio>
#define DSC_ASSERT(cond, what)                                                                         \
  do {                                                                                                \
    if (!(cond)) {                                                                                    \
      printf("DSC_CHECK failed: %s (%s:%d) block %d thread %d\n", what, __FILE__, __LINE__, (int)blockIdx.x, \
             (int)threadIdx.x);                                                                       \
      __trap();                                                                                       \
    }                                                                                                 \
  } while (0)
#else
#define DSC_ASSERT(cond, what) \
  do {                         \
  } while (0)
#endif

namespace dsc {

constexpr int kTileN = 128;   // keys per K/V tile of the tcgen05 kernel (N of QK^T, K of PV)
constexpr int kTileM = 128;   // query rows per Q tile (tcgen05 M)
constexpr int kMirror = 128;  // ring rows after slot R-1 mirroring slots [0, 128): a 128-row tile never wraps
constexpr int kMaxPeers = 8;  // fused all-gather epilogue: destinations of every O row

// One attention launch (build_instant or attend) over P = S * layer_count problems.
// Keys of problem p, kv head g, in logical order L = 0, 1, ...:
//   [0, A)                  sink rows           (position L)
//   [A, A + ring_count)     ring slots (ring_start + L - A) mod R   (position L)
//   [A+ring_count, +n_self) self rows            (position L)
// Query row i (i < n_q) of q head h sits at position q_pos0 + i and sees key L iff
// L <= q_pos0 + i.  Ids are contiguous from 0.
// A work item of the v7 kernel decoded on the host (sched.cu): what every role needs of it,
// so the kernel's roles do no index arithmetic per item.  flags: bit 0 = item of the second
// launch block (pb), bits 8.. = kv head g.
struct ItemRec {
  int pp, head_row, m0, t_begin, n_tiles, cnt, flags, sp;
};

struct AttnParams {
  // problems
  int P, S, layer_count, layer_begin, N_total;
  int Hq, Hkv, grp, d;
  // queries / outputs: [P][n_q][Hq][d]
  const void* q;
  void* o;
  int n_q;
  int q_pos0;
  // keys
  const void* sink_k; const void* sink_v;   // [S][N][Hkv][A][d]
  int A;
  const void* ring_k; const void* ring_v;   // [S][N][Hkv][Rp][d]: slots [0, R) + mirror of slots [0, 128)
  int R, Rp;                                 // ring slots, rows per head (R + kMirror)
  int ring_start, ring_count;
  // SIMT kernel only: the past sampled at a frame stride (decode_sampled off the decode kernel):
  // ring keys [0, kept*tpf) are kept past frames (newest-anchored), then the instant window
  int past_stride, stride_tpf, stride_past_frames, stride_kept_frames;
  const void* self_k; const void* self_v;   // [P][n_self][Hkv][d]
  int n_self;
  // rope
  const float2* rope;                        // [npos][d/2] (cos, sin)
  const float4* rope_pairs;                  // [npos][d/4] (cos f, cos f+1, sin f, sin f+1), f = 2j
  int rope_style;
  float scale_log2;                          // log2(e) / sqrt(d)
  // split-KV (attend): partial (O/l, log2-sum-exp) per split
  int n_splits, tiles_per_split;
  int split_only;                            // >= 0: compute only this split; its partial goes to ws_o/ws_lse slot 0
  float* ws_o;                               // [n_splits][P][n_q][Hq][d]
  float* ws_lse;                             // [n_splits][P][n_q][Hq]
  // tcgen05 kernel work decomposition
  int n_mblocks;                             // ceil(n_q * grp / (2 * kTileM)): 256-row m-blocks
  // debug export (K7); null = off.  Layout [dbg_A sink ids | dbg_R ring-slot ids | dbg_M self ids |
  // query ids], indexed with the RING geometry (dbg_A, dbg_R) even when the launch reads a
  // staging buffer (staged build: A = 0, R = staging rows)
  int* dbg_pos; int dbg_M; int dbg_A, dbg_R;
  int dbg_len;                               // entries per problem: the buffer is [S][N][dbg_len], kv head 0
  // per-CTA event timeline (FA_TRACE profiling builds); null = off.  [ntrace_cta][32][1024] clock64
  long long* trace; int ntrace_cta;
  int dtype;                                 // 0 bf16, 1 fp32
  // fused all-gather epilogue (P2 over peer memory): n_peers > 0 stores O row
  // (pp, i, h) to EVERY peer_o[j] (bf16 [P][n_q][o_hq][d]) at head o_head_off + h instead
  // of to o; peer_o are device pointers mapped in this process (local, P2P or CUDA IPC)
  void* peer_o[kMaxPeers];
  int n_peers, o_hq, o_head_off;
  // ring-ordered output (approximate instant cache, NEXT-3): o_rows > 0 stores query row i of
  // problem pp at row pp * o_rows + (i + o_rot) mod o_rows of o (o_rot < o_rows, n_q <= o_rows)
  int o_rows, o_rot;
  // CTA b of the tcgen05 kernel runs the host-decoded items item_recs[item_off[b] .. item_off[b+1])
  // in order (set by its launcher from the handle's item-table cache)
  const int* item_off;
  const ItemRec* item_recs;
  // staged build (tcgen05 path): the keys are rows [0, ring_count) of the per-step staging
  // buffers [S*N*Hkv][Rp][d] holding sink ++ instant window with K ALREADY rotated at ids
  // 0..ring_count-1 (stage_instant_kernel); A = 0, ring_start = 0, no K rotation in-kernel
  int staged;
  // TMA descriptors of the K / V rings viewed as [S*N*Hkv*Rp rows][128] bf16, box 64 x kTileN, SW128
  CUtensorMap tmap_k;
  CUtensorMap tmap_v;
  // the pair kernel's K half-tiles: the same K rows, box 64 columns x 64 rows
  CUtensorMap tmap_k64;
};

// Memory-bound decode: n_q * grp <= 16 query rows of one
// (problem, kv head) over the logical keys [sink A | kept past | instant | self], ids 0.. in
// that order.  The past is sampled at a frame stride anchored at its newest frame
// (zeta_decode; stride 1 keeps every frame): kept frame kk (0 = oldest kept)
// is past frame j = past_frames - 1 - stride * (kept_frames - 1 - kk), tokens at ring slots
// (past_start + j * tpf + tok) mod R.  Instant token u is slot (inst_start + u) mod R.
struct DecodeParams {
  int P, layer_count, layer_begin, N_total, Hq, Hkv, grp;
  const void* q; void* o; int n_q;             // [P][n_q][Hq][d]
  const void* sink_k; const void* sink_v; int A;
  const void* ring_k; const void* ring_v; int R, Rp;
  int past_start, tpf, past_frames, stride, kept_frames;
  int inst_start, inst_count;
  const void* self_k; const void* self_v; int n_self;   // [P][n_self][Hkv][d]
  const void* inst_k; const void* inst_v;      // real-model mode: the instant keys [P][inst_count][Hkv][d], else null
  int q_pos0;                                  // id of query row 0 (its token is self token n_self - n_q)
  int n_keys;                                  // A + kept_frames * tpf + inst_count + n_self
  const float4* rope_pairs;
  float scale_log2;
  int n_splits, tiles_per_split;               // key range split in 128-key tiles
  float* ws_o; float* ws_lse;                  // [n_splits][P*n_q*Hq][d], [n_splits][P*n_q*Hq]
  int* counters;                               // per-call tickets, one per (problem, kv head), zeroed
  int* dbg_pos; int dbg_len, dbg_A, dbg_R, dbg_M;   // debug id export (kv head 0), null = off
  // TMA descriptors of the K / V rings ([S*N*Hkv*Rp rows][128] bf16, box 64 x 128, SW128):
  // 128-key tiles that are one consecutive ring run load with four TMA boxes
  CUtensorMap tmap_k, tmap_v;
};
cudaError_t launch_decode(const DecodeParams& p, cudaStream_t st);

struct AppendParams {
  const void* k; const void* v;              // [S][lc][n][Hkv][d]
  void* dst_k; void* dst_v;                  // ring [S][N][Hkv][Rp][d] or sink [S][N][Hkv][A][d]
  int S, layer_count, layer_begin, N_total, Hkv, n, rows_dst;  // rows_dst = Rp or A
  int mirror_R;                              // ring: slot s < kMirror is also written to row R + s; 0 = sink
  int slot0;                                 // destination row of token 0
  int row_bytes;                             // d * elem
  // eviction poison (debug): slots [poison_slot0, +n) of every head, -1 = off
  int poison_slot0;
  int elem_bytes;
};

// One step's instant-cache keys, staged once per (stream, layer, kv head) instead of once
// per m-block: row i < A is sink row i, row i >= A is ring slot (inst_start + i - A) mod R;
// K rows are rotated at id i (split-half RoPE, pair table), V rows copied.
struct StageParams {
  const void* sink_k; const void* sink_v;    // [S][N][Hkv][A][d]
  const void* ring_k; const void* ring_v;    // [S][N][Hkv][Rp_ring][d]
  void* stage_k; void* stage_v;              // [S][N][Hkv][rows_stage][d]
  const float4* rope_pairs;
  int S, layer_count, layer_begin, N_total, Hkv, A, R, Rp_ring, inst_start, rows, rows_stage;
  // resolution boost (NEXT-4): rows >= A + n_older come from the caller's re-encoded newest
  // frame boost_k/v [S][layer_count][rows - A - n_older][Hkv][d] instead of the ring; null = off
  const void* boost_k; const void* boost_v;
  int n_older;
  // debug export (set_debug): the build key ids applied, [S][N][dbg_len] at [A + slot] / [row]
  int* dbg_pos; int dbg_len;
};

// kernels (launchers return cudaGetLastError())
cudaError_t launch_stage_instant(const StageParams& p, cudaStream_t st);
cudaError_t launch_rope_table(float2* table, int npos, int d, double theta, cudaStream_t st);
cudaError_t launch_append(const AppendParams& p, cudaStream_t st);
cudaError_t launch_attn_simt(const AttnParams& p, cudaStream_t st);
cudaError_t launch_combine(const AttnParams& p, cudaStream_t st);
// O (bf16 [rows][d]) = merge of n fp32 partials o_parts [n][rows][d] with log2-sum-exps lse [n][rows]
cudaError_t launch_combine_partials(int n, long long rows, int d, const float* o_parts, const float* lse, void* o,
                                    cudaStream_t st);
// the tcgen05 attention kernel (attn_fa.cu): one persistent launch over the items of pa and
// then those of *pb (a fused step: attend + build_instant of the same handle); per-CTA item
// tables come from the handle's cache
struct SchedCache;
SchedCache* sched_cache_new();
void sched_cache_free(SchedCache* c);
// per-CTA lists of host-decoded items (list-scheduled where that beats the stride by > 2%);
// *off = device [grid + 1] offsets, return = device records; nullptr on failure
using ItemDecoder = ItemRec (*)(const AttnParams& p, int local, int isb);
const ItemRec* item_table(SchedCache* cache, const AttnParams& pa, const AttnParams* pb, long long na, long long nb,
                          unsigned grid, ItemDecoder dec, const int** off, cudaStream_t st);
cudaError_t launch_attn_fa(const AttnParams& pa, const AttnParams* pb, SchedCache* cache, cudaStream_t st);
int attn_fa_smem_bytes();
int fa_watchdog_read(unsigned long long* out, int n);   // debug record (DSC_WATCHDOG=1)
// K/V tensor map: [rows][128] bf16, box 64 columns x box_rows rows, SW128
cudaError_t make_kv_tmap(CUtensorMap* map, void* base, unsigned long long rows, int box_rows);

}  // namespace dsc
