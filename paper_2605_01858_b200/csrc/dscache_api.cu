// Host side of the C ABI (include/dscache.h): validation, the closed-form
// eviction / position-id bookkeeping, and kernel launches.
//
// Per layer r the host keeps one int64 counter (frames appended).  At step t
// (frame t appended) with l_I = instant_frames, l_U = past_frames:
//   instant frames  [max(0, t-l_I+1), t]          C_t = min(t+1, l_I) * tpf      (Eq. 3)
//   past frames     [max(0, t-l_I-l_U+1), t-l_I]  P_t = min(max(t+1-l_I,0), l_U) * tpf (Eq. 5-6)
//   evicted at t    frame t - l_I - l_U (if >= 0)                               (Eq. 6)
//   ring slot of token j of frame f = (f*tpf + j) mod R,  R = (l_U + l_I + 1) * tpf
// Ids are contiguous from 0 over [sink | past | instant | query].
// No device bytes move on eviction.
#include "../../include/dscache.h"
#include "dscache_internal.h"

#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

// DSC_SPLIT_DIV: the attend's key splits target num_sms / DSC_SPLIT_DIV work items when its
// (problem, kv head, m-block) items cannot fill the SMs
// DSC_STAGE_MIN: the build is staged when it has at least DSC_STAGE_MIN * num_sms items
#ifndef DSC_STAGE_MIN
#define DSC_STAGE_MIN 1LL   // v8: 1 measured c4 +4.5 % vs 2, c2 / c3 / c5 unchanged (profiles/r2c/ab_ogrp_stage.txt)
#endif
#ifndef DSC_SPLIT_DIV
// v8 (two-SM clusters, num_sms / 2 of them): 4 = 37 items measured best vs 2 (74): c2 +3.5 %,
// c4 +4.6 %, context split +6.7 %, kvsplit +1.3 %, c5 0; 6 / 8 lose 3-18 % except kvsplit
// (+3 %) (profiles/r2c/ab_split_div_*.txt).  v7 (single-SM CTAs) measured 2 best.
#define DSC_SPLIT_DIV 4
#endif

namespace {

thread_local std::string g_err;

dscache_status fail(dscache_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

#define DSC_CUDA(call)                                                                     \
  do {                                                                                     \
    cudaError_t _e = (call);                                                               \
    if (_e != cudaSuccess)                                                                 \
      return fail(DSCACHE_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e));     \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

struct Schedule {
  int64_t t;          // newest frame index (frames_seen - 1)
  int C_t, P_t;
  int ring_start;     // slot of the oldest window token (past, or instant if no past)
  int inst_start;     // slot of the oldest instant token
  int64_t evicted;    // frame dropped at this step, -1 if none
};

}  // namespace

struct dscache_s {
  dscache_config cfg;
  int W, C, R, Rp, elem, npos;   // Rp = R + kMirror rows per head
  void* ring_k = nullptr;
  void* ring_v = nullptr;
  void* sink_k = nullptr;
  void* sink_v = nullptr;
  float2* rope = nullptr;
  void* bstage_k = nullptr;  // staged boosted build: sink ++ older instant ++ boosted frame (grown on demand)
  void* bstage_v = nullptr;
  int bstage_rows = 0;
  CUtensorMap tmap_bk{}, tmap_bv{}, tmap_bk64{};
  std::vector<int64_t> frames;
  std::vector<int> sink_filled;
  std::vector<int64_t> last_evicted;
  // approximate instant cache (NEXT-3): per layer, the step of the last approximate build, its
  // period, and the (o_ring, layer_count) of that call at its layer_begin
  std::vector<int64_t> approx_last;
  std::vector<int> approx_period;
  std::vector<const void*> approx_ring;
  std::vector<int> approx_lc;
  int* dbg_build = nullptr;
  int* dbg_attend = nullptr;
  int poison = 0;
  long long* trace = nullptr;
  int ntrace = 0;
  int impl_build = DSCACHE_IMPL_SIMT, impl_attend = DSCACHE_IMPL_SIMT;
  int num_sms = 148;
  dsc::SchedCache* sched = nullptr;   // per-CTA item tables of the tcgen05 kernel, owned by the handle
  CUtensorMap tmap_k{}, tmap_v{}, tmap_k64{};
  // staged build (tcgen05): per-step copy of sink ++ instant window, K pre-rotated
  void* stage_k = nullptr;
  void* stage_v = nullptr;
  int stage_rows = 0;          // A + C
  CUtensorMap tmap_sk{}, tmap_sv{}, tmap_sk64{};
  // profiling
  int prof = 0;
  struct Ev { cudaEvent_t a, b; int kind; };
  std::vector<Ev> pending;
  std::vector<cudaEvent_t> pool;
  double ms[2] = {0, 0};
  int64_t n[2] = {0, 0};
  int64_t launches = 0;

  Schedule schedule(int layer) const {
    Schedule s{};
    const int tpf = cfg.tokens_per_frame, lI = cfg.instant_frames, lU = cfg.past_frames;
    s.t = frames[layer] - 1;
    const int64_t t = s.t;
    s.C_t = (int)(std::min<int64_t>(t + 1, lI) * tpf);
    s.P_t = (int)(std::min<int64_t>(std::max<int64_t>(t + 1 - lI, 0), lU) * tpf);
    const int64_t f0 = std::max<int64_t>(0, t - lI - lU + 1);
    const int64_t fi = std::max<int64_t>(0, t - lI + 1);
    s.ring_start = (int)((f0 * tpf) % R);
    s.inst_start = (int)((fi * tpf) % R);
    s.evicted = (t - lI - lU >= 0) ? t - lI - lU : -1;
    return s;
  }

  cudaEvent_t take_event() {
    if (!pool.empty()) { cudaEvent_t e = pool.back(); pool.pop_back(); return e; }
    cudaEvent_t e; cudaEventCreate(&e); return e;
  }
};

namespace {

dscache_status check_layers(dscache_t h, int lb, int lc) {
  if (!h) return fail(DSCACHE_E_ARG, "null handle");
  if (lc < 1 || lb < 0 || lb + lc > h->cfg.num_layers)
    return fail(DSCACHE_E_ARG, "layer range [" + std::to_string(lb) + ", +" + std::to_string(lc) +
                                   ") outside [0, " + std::to_string(h->cfg.num_layers) + ")");
  for (int l = lb + 1; l < lb + lc; ++l)
    if (h->frames[l] != h->frames[lb] || h->sink_filled[l] != h->sink_filled[lb])
      return fail(DSCACHE_E_STATE, "layers of the range are not at the same step");
  return DSCACHE_OK;
}

dscache_status need_mode(dscache_t h, int mode, const char* what) {
  if (!h) return fail(DSCACHE_E_ARG, "null handle");
  if (h->cfg.instant_source != mode)
    return fail(DSCACHE_E_CONFIG, std::string(what) + (mode == DSCACHE_INSTANT_EXTERNAL
                                                           ? " needs instant_source = DSCACHE_INSTANT_EXTERNAL"
                                                           : " reads the ring's instant frames: not in the "
                                                             "external-instant (real-model) mode"));
  return DSCACHE_OK;
}

bool tc_eligible(const dscache_config& c) {
  return c.dtype == DSCACHE_DTYPE_BF16 && c.head_dim == 128 && c.rope_style == DSCACHE_ROPE_SPLIT_HALF;
}

void fill_common(dscache_t h, dsc::AttnParams& p, int lb, int lc) {
  const dscache_config& c = h->cfg;
  p.S = c.num_streams; p.layer_count = lc; p.layer_begin = lb; p.N_total = c.num_layers;
  p.P = c.num_streams * lc;
  p.Hq = c.num_q_heads; p.Hkv = c.num_kv_heads; p.grp = c.num_q_heads / c.num_kv_heads; p.d = c.head_dim;
  p.sink_k = h->sink_k; p.sink_v = h->sink_v; p.A = c.sink_tokens;
  p.ring_k = h->ring_k; p.ring_v = h->ring_v; p.R = h->R; p.Rp = h->Rp;
  p.rope = h->rope; p.rope_style = c.rope_style;
  p.rope_pairs = reinterpret_cast<const float4*>(h->rope + (size_t)h->npos * (c.head_dim / 2));
  p.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)c.head_dim));
  p.dtype = c.dtype;
  p.dbg_M = std::max(h->C, c.max_query_tokens);
  p.dbg_A = c.sink_tokens; p.dbg_R = h->R;
  p.dbg_len = c.sink_tokens + h->R + 2 * p.dbg_M;
  p.tmap_k = h->tmap_k; p.tmap_v = h->tmap_v; p.tmap_k64 = h->tmap_k64;
  p.staged = 0;
  p.trace = h->trace; p.ntrace_cta = h->ntrace;
  p.n_splits = 1; p.tiles_per_split = 1 << 30; p.split_only = -1;
}

// Per-call scratch, stream-ordered (cudaMallocAsync / cudaFreeAsync on the call's stream):
// calls for different layer ranges may run on different streams concurrently, so no
// scratch is shared between calls (a per-handle workspace was).
struct StreamScratch {
  void* ptr = nullptr;
  cudaStream_t st = nullptr;
  ~StreamScratch() { if (ptr) cudaFreeAsync(ptr, st); }
  bool alloc(size_t bytes, cudaStream_t s) {
    st = s;
    if (cudaMallocAsync(&ptr, bytes, s) != cudaSuccess) { cudaGetLastError(); ptr = nullptr; return false; }
    return true;
  }
};

// split-KV attend: the fp32 partials [splits][rows][d] + log2-sum-exps [splits][rows]
dscache_status alloc_ws(dsc::AttnParams& p, StreamScratch& ws, cudaStream_t st) {
  if (p.n_splits <= 1 || p.split_only >= 0 || p.ws_o) return DSCACHE_OK;
  const size_t rows = (size_t)p.P * p.n_q * p.Hq;
  if (!ws.alloc((size_t)p.n_splits * rows * (p.d + 1) * sizeof(float), st))
    return fail(DSCACHE_E_OOM, "split-KV workspace allocation failed");
  p.ws_o = static_cast<float*>(ws.ptr);
  p.ws_lse = p.ws_o + (size_t)p.n_splits * rows * p.d;
  return DSCACHE_OK;
}

// the tcgen05 attention launch (pb: the build items of a fused step)
cudaError_t launch_tc(dscache_t h, const dsc::AttnParams& pa, const dsc::AttnParams* pb, cudaStream_t st) {
  return dsc::launch_attn_fa(pa, pb, h->sched, st);
}

dscache_status run_attention(dscache_t h, dsc::AttnParams& p, int impl, int kind, cudaStream_t st) {
  StreamScratch ws;
  dscache_status ss = alloc_ws(p, ws, st);
  if (ss != DSCACHE_OK) return ss;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (h->prof) { e0 = h->take_event(); e1 = h->take_event(); cudaEventRecord(e0, st); }
  cudaError_t e;
  if (impl == DSCACHE_IMPL_TC) e = launch_tc(h, p, nullptr, st);
  else e = dsc::launch_attn_simt(p, st);
  h->launches++;
  if (e == cudaSuccess && p.n_splits > 1 && p.split_only < 0) { e = dsc::launch_combine(p, st); h->launches++; }
  if (h->prof) {
    cudaEventRecord(e1, st);
    h->pending.push_back({e0, e1, kind});
  }
  if (e != cudaSuccess) return fail(DSCACHE_E_CUDA, std::string("attention launch: ") + cudaGetErrorString(e));
  return DSCACHE_OK;
}

}  // namespace

namespace {
// NVTX range around every public call that launches work (SURVEY §5 tracing): named after
// the C entry point, visible in Nsight Systems / ncu --nvtx; a no-op without a tool.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

extern "C" {

const char* dscache_last_error(void) { return g_err.c_str(); }

dscache_status dscache_create(const dscache_config* cfg, dscache_t* out) {
  if (!cfg || !out) return fail(DSCACHE_E_ARG, "null config or output pointer");
  *out = nullptr;
  const dscache_config& c = *cfg;
  if (c.num_streams < 1 || c.num_layers < 1 || c.num_q_heads < 1 || c.num_kv_heads < 1)
    return fail(DSCACHE_E_CONFIG, "S, N, Hq, Hkv must be >= 1");
  if (c.num_q_heads % c.num_kv_heads) return fail(DSCACHE_E_CONFIG, "Hq must be a multiple of Hkv");
  if (c.head_dim != 64 && c.head_dim != 128) return fail(DSCACHE_E_CONFIG, "head_dim must be 64 or 128");
  if (c.tokens_per_frame < 1 || c.sink_tokens < 0 || c.past_frames < 0 || c.instant_frames < 0 ||
      c.max_query_tokens < 1 || c.max_position < 1)
    return fail(DSCACHE_E_CONFIG, "tpf >= 1, A/l_U/l_I >= 0, q_max >= 1, max_position >= 1 required");
  if (c.past_frames + c.instant_frames < 1)
    return fail(DSCACHE_E_CONFIG, "l_U + l_I must be >= 1 (the newest frame must be held)");
  if (c.dtype != DSCACHE_DTYPE_BF16 && c.dtype != DSCACHE_DTYPE_FP32) return fail(DSCACHE_E_CONFIG, "dtype");
  if (c.rope_style != DSCACHE_ROPE_SPLIT_HALF && c.rope_style != DSCACHE_ROPE_ADJACENT)
    return fail(DSCACHE_E_CONFIG, "rope_style");
  if (c.instant_source != DSCACHE_INSTANT_RING && c.instant_source != DSCACHE_INSTANT_EXTERNAL)
    return fail(DSCACHE_E_CONFIG, "instant_source");
  if (!(c.rope_theta > 1.0)) return fail(DSCACHE_E_CONFIG, "rope_theta must be > 1");
  const int64_t W = (int64_t)c.past_frames * c.tokens_per_frame, C = (int64_t)c.instant_frames * c.tokens_per_frame;
  // largest id any attention applies: attend A+W+C+q_max-1, update attention (Eq. 5) A+W+tpf-1
  const int64_t span = c.sink_tokens + W + std::max<int64_t>(C + c.max_query_tokens, c.tokens_per_frame);
  if (span > c.max_position)
    return fail(DSCACHE_E_POS_OVERFLOW, "A+W+max(C+q_max,tpf) = " + std::to_string(span) + " exceeds max_position " +
                                            std::to_string(c.max_position));
  if (c.attn_impl == DSCACHE_IMPL_TC && !tc_eligible(c))
    return fail(DSCACHE_E_CONFIG, "tcgen05 kernel needs bf16, d=128, split-half RoPE");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || c.device < 0 || c.device >= ndev) {
    cudaGetLastError();
    return fail(DSCACHE_E_CUDA, "no CUDA device " + std::to_string(c.device));
  }
  DeviceGuard dg(c.device);

  dscache_s* h = new dscache_s();
  h->cfg = c;
  h->W = (int)W; h->C = (int)C;
  h->R = (int)(W + C + c.tokens_per_frame);
  h->Rp = h->R + dsc::kMirror;
  h->elem = c.dtype == DSCACHE_DTYPE_BF16 ? 2 : 4;
  h->npos = c.max_position;   // RoPE table covers every id < max_position (decode ids grow per token)
  h->frames.assign(c.num_layers, 0);
  h->sink_filled.assign(c.num_layers, c.sink_tokens == 0 ? 1 : 0);
  h->approx_last.assign(c.num_layers, -1);
  h->approx_period.assign(c.num_layers, 0);
  h->approx_ring.assign(c.num_layers, nullptr);
  h->approx_lc.assign(c.num_layers, 0);
  h->last_evicted.assign(c.num_layers, -1);
  cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, c.device);
  h->sched = dsc::sched_cache_new();
  if (c.attn_impl == DSCACHE_IMPL_SIMT) {
    h->impl_build = h->impl_attend = DSCACHE_IMPL_SIMT;
  } else {
    h->impl_build = tc_eligible(c) ? DSCACHE_IMPL_TC : DSCACHE_IMPL_SIMT;
    h->impl_attend = h->impl_build;
  }

  const size_t heads = (size_t)c.num_streams * c.num_layers * c.num_kv_heads;
  const size_t ring_bytes = heads * h->Rp * c.head_dim * h->elem;
  const size_t sink_bytes = heads * std::max(c.sink_tokens, 1) * c.head_dim * h->elem;
  const size_t rope_bytes = 2 * (size_t)h->npos * (c.head_dim / 2) * sizeof(float2);   // float2 + pair-packed copy
  auto oom = [&](const char* what) {
    cudaGetLastError();
    dscache_destroy(h);
    return fail(DSCACHE_E_OOM, std::string("cudaMalloc failed for ") + what);
  };
  if (cudaMalloc(&h->ring_k, ring_bytes) != cudaSuccess) return oom("ring K");
  if (cudaMalloc(&h->ring_v, ring_bytes) != cudaSuccess) return oom("ring V");
  if (cudaMalloc(&h->sink_k, sink_bytes) != cudaSuccess) return oom("sink K");
  if (cudaMalloc(&h->sink_v, sink_bytes) != cudaSuccess) return oom("sink V");
  if (cudaMalloc(&h->rope, rope_bytes) != cudaSuccess) return oom("rope table");
  cudaError_t e = cudaMemset(h->ring_k, 0, ring_bytes);
  if (e == cudaSuccess) e = cudaMemset(h->ring_v, 0, ring_bytes);
  if (e == cudaSuccess) e = cudaMemset(h->sink_k, 0, sink_bytes);
  if (e == cudaSuccess) e = cudaMemset(h->sink_v, 0, sink_bytes);
  if (e == cudaSuccess) e = dsc::launch_rope_table(h->rope, h->npos, c.head_dim, c.rope_theta, 0);
  if (e == cudaSuccess && (h->impl_build == DSCACHE_IMPL_TC || h->impl_attend == DSCACHE_IMPL_TC)) {
    const unsigned long long rows = (unsigned long long)heads * h->Rp;
    e = dsc::make_kv_tmap(&h->tmap_k, h->ring_k, rows, dsc::kTileN);
    if (e == cudaSuccess) e = dsc::make_kv_tmap(&h->tmap_k64, h->ring_k, rows, dsc::kTileN / 2);
    if (e == cudaSuccess) e = dsc::make_kv_tmap(&h->tmap_v, h->ring_v, rows, dsc::kTileN);
  }
  if (e == cudaSuccess && h->impl_build == DSCACHE_IMPL_TC && h->C > 0) {
    h->stage_rows = c.sink_tokens + h->C;
    const size_t sb = heads * h->stage_rows * c.head_dim * h->elem;
    if (cudaMalloc(&h->stage_k, sb) != cudaSuccess || cudaMalloc(&h->stage_v, sb) != cudaSuccess) return oom("staging");
    e = cudaMemset(h->stage_k, 0, sb);
    if (e == cudaSuccess) e = cudaMemset(h->stage_v, 0, sb);
    if (e == cudaSuccess) e = dsc::make_kv_tmap(&h->tmap_sk, h->stage_k, (unsigned long long)heads * h->stage_rows, dsc::kTileN);
    if (e == cudaSuccess)
      e = dsc::make_kv_tmap(&h->tmap_sk64, h->stage_k, (unsigned long long)heads * h->stage_rows, dsc::kTileN / 2);
    if (e == cudaSuccess) e = dsc::make_kv_tmap(&h->tmap_sv, h->stage_v, (unsigned long long)heads * h->stage_rows, dsc::kTileN);
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    std::string m = cudaGetErrorString(e);
    dscache_destroy(h);
    return fail(DSCACHE_E_CUDA, "create: " + m);
  }
  *out = h;
  return DSCACHE_OK;
}

dscache_status dscache_destroy(dscache_t h) {
  if (!h) return fail(DSCACHE_E_ARG, "null handle");
  DeviceGuard dg(h->cfg.device);
  cudaDeviceSynchronize();
  for (auto& ev : h->pending) { cudaEventDestroy(ev.a); cudaEventDestroy(ev.b); }
  for (auto e : h->pool) cudaEventDestroy(e);
  cudaFree(h->ring_k); cudaFree(h->ring_v); cudaFree(h->sink_k); cudaFree(h->sink_v);
  cudaFree(h->rope);
  cudaFree(h->stage_k); cudaFree(h->stage_v);
  cudaFree(h->bstage_k); cudaFree(h->bstage_v);
  dsc::sched_cache_free(h->sched);
  delete h;
  return DSCACHE_OK;
}

dscache_status dscache_append_frame(dscache_t h, int32_t lb, int32_t lc, const void* k, const void* v,
                                    int32_t n_tokens, void* stream) {
  NvtxRange nvtx_("dscache_append_frame");
  dscache_status s = check_layers(h, lb, lc);
  if (s != DSCACHE_OK) return s;
  if (!k || !v) return fail(DSCACHE_E_ARG, "null k/v");
  const dscache_config& c = h->cfg;
  DeviceGuard dg(c.device);
  cudaStream_t st = (cudaStream_t)stream;
  dsc::AppendParams p{};
  p.k = k; p.v = v;
  p.S = c.num_streams; p.layer_count = lc; p.layer_begin = lb; p.N_total = c.num_layers; p.Hkv = c.num_kv_heads;
  p.row_bytes = c.head_dim * h->elem; p.elem_bytes = h->elem; p.n = n_tokens; p.poison_slot0 = -1;
  p.mirror_R = 0;
  if (!h->sink_filled[lb]) {
    if (n_tokens != c.sink_tokens)
      return fail(DSCACHE_E_ARG, "first append of a layer must carry the " + std::to_string(c.sink_tokens) +
                                     " sink tokens, got " + std::to_string(n_tokens));
    p.dst_k = h->sink_k; p.dst_v = h->sink_v; p.rows_dst = c.sink_tokens; p.slot0 = 0;
    DSC_CUDA(dsc::launch_append(p, st));
    h->launches++;
    for (int l = lb; l < lb + lc; ++l) h->sink_filled[l] = 1;
    return DSCACHE_OK;
  }
  if (c.instant_source != DSCACHE_INSTANT_RING)
    return fail(DSCACHE_E_CONFIG, "external-instant (real-model) mode: frames enter the ring via dscache_append_past");
  if (n_tokens != c.tokens_per_frame)
    return fail(DSCACHE_E_ARG, "frame append must carry tokens_per_frame = " + std::to_string(c.tokens_per_frame) +
                                   " tokens, got " + std::to_string(n_tokens));
  const int64_t f = h->frames[lb];
  p.dst_k = h->ring_k; p.dst_v = h->ring_v; p.rows_dst = h->Rp; p.mirror_R = h->R;
  p.slot0 = (int)((f * c.tokens_per_frame) % h->R);
  const int64_t ev = f - c.instant_frames - c.past_frames;
  if (h->poison && ev >= 0) p.poison_slot0 = (int)((ev * c.tokens_per_frame) % h->R);
  DSC_CUDA(dsc::launch_append(p, st));
  h->launches++;
  for (int l = lb; l < lb + lc; ++l) { h->frames[l] = f + 1; h->last_evicted[l] = ev >= 0 ? ev : -1; }
  return DSCACHE_OK;
}

namespace {
// Parameters of build_instant (Eq. 7): the C_t instant tokens attend causally over
// [sink | instant window].  *empty is set when l_I = 0 (nothing to build).
dscache_status prep_build(dscache_t h, int32_t lb, int32_t lc, const void* q_inst, void* o_inst, dsc::AttnParams& p,
                          bool* empty, dsc::StageParams* stage) {
  *empty = false;
  dscache_status s = check_layers(h, lb, lc);
  if (s != DSCACHE_OK) return s;
  if (!h->sink_filled[lb] || h->frames[lb] < 1)
    return fail(DSCACHE_E_STATE, "build_instant before the sink and the first frame were appended");
  const Schedule sc = h->schedule(lb);
  if (sc.C_t == 0) { *empty = true; return DSCACHE_OK; }   // l_I = 0: the instant cache is empty
  if (!q_inst || !o_inst) return fail(DSCACHE_E_ARG, "null q_inst/o_inst");
  p = dsc::AttnParams{};
  fill_common(h, p, lb, lc);
  p.q = q_inst; p.o = o_inst; p.n_q = sc.C_t; p.q_pos0 = h->cfg.sink_tokens;
  p.ring_start = sc.inst_start; p.ring_count = sc.C_t;
  p.self_k = p.self_v = nullptr; p.n_self = 0;
  p.dbg_pos = h->dbg_build;
  p.n_mblocks = (p.n_q * p.grp + 2 * dsc::kTileM - 1) / (2 * dsc::kTileM);
  // tcgen05 build: stage sink ++ instant window once per (stream, layer, head) with K
  // rotated at the build ids 0.. (the window is re-read by every m-block; rotating it once
  // instead of per m-block removes the RoPE work from the build items).  The debug id
  // export records ids where the kernel rotates, so debug runs keep the ring path.
  // Small launches (fewer build items than two waves of SMs, e.g. one stream x one layer)
  // are latency-bound: the extra staging launch costs more than the RoPE it saves there.
  const long long build_items = (long long)p.P * p.Hkv * p.n_mblocks;
  if (h->impl_build == DSCACHE_IMPL_TC && h->stage_k && build_items >= DSC_STAGE_MIN * h->num_sms) {
    dsc::StageParams sp{};
    sp.sink_k = h->sink_k; sp.sink_v = h->sink_v; sp.ring_k = h->ring_k; sp.ring_v = h->ring_v;
    sp.stage_k = h->stage_k; sp.stage_v = h->stage_v; sp.rope_pairs = p.rope_pairs;
    sp.S = p.S; sp.layer_count = lc; sp.layer_begin = lb; sp.N_total = p.N_total; sp.Hkv = p.Hkv;
    sp.A = p.A; sp.R = h->R; sp.Rp_ring = h->Rp; sp.inst_start = sc.inst_start;
    sp.rows = p.A + sc.C_t; sp.rows_stage = h->stage_rows;
    sp.dbg_pos = h->dbg_build; sp.dbg_len = p.dbg_len;   // the staging kernel applies the build key ids
    *stage = sp;
    p.staged = 1;
    p.A = 0; p.ring_start = 0; p.ring_count = sp.rows; p.R = h->stage_rows; p.Rp = h->stage_rows;
    p.tmap_k = h->tmap_sk; p.tmap_v = h->tmap_sv; p.tmap_k64 = h->tmap_sk64;
  }
  return DSCACHE_OK;
}
}  // namespace

dscache_status dscache_build_instant(dscache_t h, int32_t lb, int32_t lc, const void* q_inst, void* o_inst,
                                     void* stream) {
  NvtxRange nvtx_("dscache_build_instant");
  if (h && h->cfg.instant_source != DSCACHE_INSTANT_RING) return need_mode(h, DSCACHE_INSTANT_RING, "build_instant");
  dsc::AttnParams p{};
  dsc::StageParams sp{};
  bool empty = false;
  dscache_status s = prep_build(h, lb, lc, q_inst, o_inst, p, &empty, &sp);
  if (s != DSCACHE_OK || empty) return s;
  DeviceGuard dg(h->cfg.device);
  if (p.staged) {
    DSC_CUDA(dsc::launch_stage_instant(sp, (cudaStream_t)stream));
    h->launches++;
  }
  return run_attention(h, p, h->impl_build, 0, (cudaStream_t)stream);
}

namespace {
// Parameters of the newest frame's Eq. 7 rows: its tpf queries attend causally over [sink |
// instant window] at ids A + C_t - tpf + j (the rows of build_instant a causal mask makes
// independent of the other instant queries).
dscache_status prep_newest(dscache_t h, int32_t lb, int32_t lc, const void* q_new, void* o_new, dsc::AttnParams& p) {
  dscache_status s = check_layers(h, lb, lc);
  if (s != DSCACHE_OK) return s;
  if (!h->sink_filled[lb] || h->frames[lb] < 1)
    return fail(DSCACHE_E_STATE, "newest-frame build before the sink and the first frame were appended");
  if (h->cfg.instant_frames < 1) return fail(DSCACHE_E_CONFIG, "l_I = 0: there is no instant cache");
  if (!q_new || !o_new) return fail(DSCACHE_E_ARG, "null q/o");
  const Schedule sc = h->schedule(lb);
  const int tpf = h->cfg.tokens_per_frame;
  p = dsc::AttnParams{};
  fill_common(h, p, lb, lc);
  p.q = q_new; p.o = o_new; p.n_q = tpf;
  p.q_pos0 = h->cfg.sink_tokens + sc.C_t - tpf;   // the newest frame's tokens are the last tpf instant ids
  p.ring_start = sc.inst_start; p.ring_count = sc.C_t;
  p.self_k = p.self_v = nullptr; p.n_self = 0;
  p.dbg_pos = nullptr;
  p.n_mblocks = (p.n_q * p.grp + 2 * dsc::kTileM - 1) / (2 * dsc::kTileM);
  return DSCACHE_OK;
}

// Approximate instant cache (NEXT-3, reading Q23): a refresh rebuilds every buffer
// frame's rows; between refreshes only the newest frame's rows are built.  A step refreshes
// when t is a multiple of the period or when the rows in o_ring are not the previous step's
// (first call, a skipped step, another period, another buffer or layer range).
bool approx_refresh(dscache_t h, int32_t lb, int32_t lc, int32_t period, const void* o_ring, int64_t t) {
  if (t % period == 0) return true;
  if (h->approx_ring[lb] != o_ring || h->approx_lc[lb] != lc) return true;
  for (int l = lb; l < lb + lc; ++l)
    if (h->approx_last[l] != t - 1 || h->approx_period[l] != period) return true;
  return false;
}
}  // namespace

dscache_status dscache_build_instant_newest(dscache_t h, int32_t lb, int32_t lc, const void* q_new, void* o_new,
                                            void* stream) {
  NvtxRange nvtx_("dscache_build_instant_newest");
  if (h && h->cfg.instant_source != DSCACHE_INSTANT_RING) return need_mode(h, DSCACHE_INSTANT_RING, "build_instant_newest");
  dsc::AttnParams p{};
  dscache_status s = prep_newest(h, lb, lc, q_new, o_new, p);
  if (s != DSCACHE_OK) return s;
  DeviceGuard dg(h->cfg.device);
  return run_attention(h, p, h->impl_build, 0, (cudaStream_t)stream);
}

dscache_status dscache_instant_approx_rows(dscache_t h, int32_t lb, int32_t lc, int32_t period, const void* o_ring,
                                           int32_t* n_rows) {
  dscache_status s = need_mode(h, DSCACHE_INSTANT_RING, "instant_approx_rows");
  if (s == DSCACHE_OK) s = check_layers(h, lb, lc);
  if (s != DSCACHE_OK) return s;
  if (!n_rows) return fail(DSCACHE_E_ARG, "null n_rows");
  if (period < 1) return fail(DSCACHE_E_ARG, "period must be >= 1");
  if (!h->sink_filled[lb] || h->frames[lb] < 1)
    return fail(DSCACHE_E_STATE, "approximate build before the sink and the first frame were appended");
  if (h->cfg.instant_frames < 1) return fail(DSCACHE_E_CONFIG, "l_I = 0: there is no instant cache");
  const int64_t t = h->frames[lb] - 1;
  *n_rows = approx_refresh(h, lb, lc, period, o_ring, t) ? h->schedule(lb).C_t : h->cfg.tokens_per_frame;
  return DSCACHE_OK;
}

dscache_status dscache_build_instant_approx(dscache_t h, int32_t lb, int32_t lc, int32_t period, const void* q_rows,
                                            int32_t n_rows, void* o_ring, void* stream) {
  NvtxRange nvtx_("dscache_build_instant_approx");
  int32_t need = 0;
  dscache_status s = dscache_instant_approx_rows(h, lb, lc, period, o_ring, &need);
  if (s != DSCACHE_OK) return s;
  if (n_rows != need)
    return fail(DSCACHE_E_ARG, "approximate build at this step takes " + std::to_string(need) + " query rows (" +
                                   (need == h->cfg.tokens_per_frame && need != h->schedule(lb).C_t ? "newest frame" : "refresh") +
                                   "), got " + std::to_string(n_rows));
  if (!q_rows || !o_ring) return fail(DSCACHE_E_ARG, "null q_rows/o_ring");
  const dscache_config& c = h->cfg;
  const int64_t t = h->frames[lb] - 1;
  const int tpf = c.tokens_per_frame, lI = c.instant_frames;
  const bool refresh = approx_refresh(h, lb, lc, period, o_ring, t);
  DeviceGuard dg(c.device);
  dsc::AttnParams p{};
  if (refresh) {
    // every buffer frame f in max(0, t-l_I+1)..t: row i (frame b + i/tpf) lands at ring row
    // ((b + i/tpf) mod l_I) * tpf + i mod tpf = (i + (b mod l_I) * tpf) mod C
    dsc::StageParams sp{};
    bool empty = false;
    s = prep_build(h, lb, lc, q_rows, o_ring, p, &empty, &sp);
    if (s != DSCACHE_OK) return s;
    const int64_t b = t - lI + 1 > 0 ? t - lI + 1 : 0;
    p.o_rows = h->C; p.o_rot = (int)(b % lI) * tpf;
    if (p.staged) {
      DSC_CUDA(dsc::launch_stage_instant(sp, (cudaStream_t)stream));
      h->launches++;
    }
  } else {
    s = prep_newest(h, lb, lc, q_rows, o_ring, p);
    if (s != DSCACHE_OK) return s;
    p.o_rows = h->C; p.o_rot = (int)(t % lI) * tpf;
  }
  s = run_attention(h, p, h->impl_build, 0, (cudaStream_t)stream);
  if (s != DSCACHE_OK) return s;
  for (int l = lb; l < lb + lc; ++l) { h->approx_last[l] = t; h->approx_period[l] = period; }
  h->approx_ring[lb] = o_ring; h->approx_lc[lb] = lc;
  return DSCACHE_OK;
}

namespace {
// Attention of n_q query rows over [sink | past | instant | self], where the self segment
// holds n_self >= n_q transient tokens (the query chunk, and during decode the tokens
// generated so far) and the queries are its last n_q tokens.
// ring_drop: tokens left out at the newest end of the window (the boosted newest frame's
// ring slots, whose keys the caller supplies re-encoded inside the self segment instead)
dscache_status prep_attend(dscache_t h, int32_t lb, int32_t lc, const void* q, const void* k_self,
                           const void* v_self, int32_t n_self, int32_t n_q, void* o, bool dbg, dsc::AttnParams& p,
                           int ring_drop = 0) {
  dscache_status s = check_layers(h, lb, lc);
  if (s != DSCACHE_OK) return s;
  if (!h->sink_filled[lb] || h->frames[lb] < 1)
    return fail(DSCACHE_E_STATE, "attend before the sink and the first frame were appended");
  if (n_q < 1 || n_q > n_self) return fail(DSCACHE_E_ARG, "need 1 <= n_q <= n_self");
  if (!q || !k_self || !v_self || !o) return fail(DSCACHE_E_ARG, "null q/k_self/v_self/o");
  const Schedule sc = h->schedule(lb);
  if ((int64_t)h->cfg.sink_tokens + sc.P_t + sc.C_t - ring_drop + n_self > h->cfg.max_position)
    return fail(DSCACHE_E_POS_OVERFLOW, "A + P_t + C_t + n_self exceeds max_position");
  p = dsc::AttnParams{};
  fill_common(h, p, lb, lc);
  p.q = q; p.o = o; p.n_q = n_q;
  p.ring_start = sc.ring_start; p.ring_count = sc.P_t + sc.C_t - ring_drop;
  p.q_pos0 = h->cfg.sink_tokens + p.ring_count + (n_self - n_q);
  p.self_k = k_self; p.self_v = v_self; p.n_self = n_self;
  p.dbg_pos = dbg ? h->dbg_attend : nullptr;
  p.n_mblocks = (p.n_q * p.grp + 2 * dsc::kTileM - 1) / (2 * dsc::kTileM);
  const int impl = h->impl_attend;
  if (impl == DSCACHE_IMPL_TC) {
    // split the key range when (problem, kv head, m-block) work items cannot fill the SMs
    // sink/self tiles + logical window tiles (see tc_common.cuh tile_segments)
    const int BN = dsc::kTileN;
    const int tiles = std::max(1, (p.A + n_self + BN - 1) / BN + (p.ring_count + BN - 1) / BN);
    const int items = p.P * p.Hkv * p.n_mblocks;
    int splits = 1;
    if (items < h->num_sms) {
      splits = std::min((h->num_sms / DSC_SPLIT_DIV + items - 1) / items, std::max(1, tiles / 4));
    }
    if (splits > 1) {
      p.tiles_per_split = (tiles + splits - 1) / splits;
      splits = (tiles + p.tiles_per_split - 1) / p.tiles_per_split;
    }
    p.n_splits = splits;   // the workspace is allocated per call on its stream (alloc_ws)
  }
  return DSCACHE_OK;
}

dscache_status attend_common(dscache_t h, int32_t lb, int32_t lc, const void* q, const void* k_self,
                             const void* v_self, int32_t n_self, int32_t n_q, void* o, void* stream, bool dbg) {
  dsc::AttnParams p{};
  dscache_status s = prep_attend(h, lb, lc, q, k_self, v_self, n_self, n_q, o, dbg, p);
  if (s != DSCACHE_OK) return s;
  DeviceGuard dg(h->cfg.device);
  return run_attention(h, p, h->impl_attend, 1, (cudaStream_t)stream);
}
}  // namespace

dscache_status dscache_attend(dscache_t h, int32_t lb, int32_t lc, const void* q, const void* k_self,
                              const void* v_self, int32_t n_q, void* o, void* stream) {
  NvtxRange nvtx_("dscache_attend");
  if (h && h->cfg.instant_source != DSCACHE_INSTANT_RING) return need_mode(h, DSCACHE_INSTANT_RING, "attend");
  if (h && (n_q < 1 || n_q > h->cfg.max_query_tokens))
    return fail(DSCACHE_E_ARG, "n_q must be in [1, max_query_tokens]");
  return attend_common(h, lb, lc, q, k_self, v_self, n_q, n_q, o, stream, true);
}

namespace {
// The memory-bound decode kernel (decode.cu) serves bf16, d = 128, split-half RoPE and up to
// 16 query rows (n_q * Hq/Hkv) per kv head; anything else runs through the attention kernel.
bool decode_kernel_ok(dscache_t h, int n_q) {
  return tc_eligible(h->cfg) && n_q * (h->cfg.num_q_heads / h->cfg.num_kv_heads) <= 16;
}

dscache_status run_decode(dscache_t h, int32_t lb, int32_t lc, const void* q, const void* k_self, const void* v_self,
                          int32_t n_self, int32_t n_q, int32_t stride, void* o, cudaStream_t st,
                          const void* k_inst = nullptr, const void* v_inst = nullptr) {
  dscache_status s = check_layers(h, lb, lc);
  if (s != DSCACHE_OK) return s;
  if (!h->sink_filled[lb] || h->frames[lb] < 1)
    return fail(DSCACHE_E_STATE, "decode before the sink and the first frame were appended");
  if (n_q < 1 || n_q > n_self) return fail(DSCACHE_E_ARG, "need 1 <= n_q <= n_self");
  if (!q || !k_self || !v_self || !o) return fail(DSCACHE_E_ARG, "null q/k_self/v_self/o");
  const dscache_config& c = h->cfg;
  const Schedule sc = h->schedule(lb);
  const int tpf = c.tokens_per_frame;
  // (real-model mode: the ring holds the same past; the C_t instant keys come from k_inst)
  const int past_frames = sc.P_t / tpf;
  const int kept = (past_frames + stride - 1) / stride;
  const int64_t n_keys = (int64_t)c.sink_tokens + (int64_t)kept * tpf + sc.C_t + n_self;
  if (n_keys > c.max_position) return fail(DSCACHE_E_POS_OVERFLOW, "A + kept past + C_t + n_self exceeds max_position");
  DeviceGuard dg(c.device);
  dsc::DecodeParams p{};
  p.P = c.num_streams * lc; p.layer_count = lc; p.layer_begin = lb; p.N_total = c.num_layers;
  p.Hq = c.num_q_heads; p.Hkv = c.num_kv_heads; p.grp = c.num_q_heads / c.num_kv_heads;
  p.q = q; p.o = o; p.n_q = n_q;
  p.sink_k = h->sink_k; p.sink_v = h->sink_v; p.A = c.sink_tokens;
  p.ring_k = h->ring_k; p.ring_v = h->ring_v; p.R = h->R; p.Rp = h->Rp;
  p.past_start = sc.ring_start; p.tpf = tpf; p.past_frames = past_frames; p.stride = stride; p.kept_frames = kept;
  p.inst_start = sc.inst_start; p.inst_count = sc.C_t;
  p.self_k = k_self; p.self_v = v_self; p.n_self = n_self;
  p.inst_k = k_inst; p.inst_v = v_inst;
  p.n_keys = (int)n_keys;
  p.q_pos0 = (int)(n_keys - n_q);
  p.rope_pairs = reinterpret_cast<const float4*>(h->rope + (size_t)h->npos * (c.head_dim / 2));
  p.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)c.head_dim));
  p.dbg_pos = h->dbg_attend;
  p.tmap_k = h->tmap_k; p.tmap_v = h->tmap_v;
  p.dbg_M = std::max(h->C, c.max_query_tokens); p.dbg_A = c.sink_tokens; p.dbg_R = h->R;
  p.dbg_len = c.sink_tokens + h->R + 2 * p.dbg_M;
  // one wave of CTAs: split each (problem, kv head)'s keys when there are fewer of them than
  // SMs, keeping at least one 16-key warp tile per warp in every split
  const int units = p.P * p.Hkv;
  const int tiles = (int)((n_keys + 127) / 128);
  int splits = 1;
  if (units < h->num_sms) splits = std::max(1, std::min((h->num_sms + units - 1) / units, tiles));
  p.tiles_per_split = (tiles + splits - 1) / splits;
  splits = (tiles + p.tiles_per_split - 1) / p.tiles_per_split;
  p.n_splits = splits;
  StreamScratch ws;
  if (splits > 1) {
    // per-call workspace: the partials, their log2-sum-exps and one zeroed ticket per
    // (problem, kv head), so concurrent decodes on different streams share nothing
    const size_t rows = (size_t)p.P * n_q * c.num_q_heads;
    const size_t fl = (size_t)splits * rows * (c.head_dim + 1);
    if (!ws.alloc(fl * sizeof(float) + (size_t)units * sizeof(int), st))
      return fail(DSCACHE_E_OOM, "decode split-KV workspace");
    p.ws_o = static_cast<float*>(ws.ptr);
    p.ws_lse = p.ws_o + (size_t)splits * rows * c.head_dim;
    p.counters = reinterpret_cast<int*>(p.ws_o + fl);
    if (cudaMemsetAsync(p.counters, 0, (size_t)units * sizeof(int), st) != cudaSuccess)
      return fail(DSCACHE_E_CUDA, "decode tickets");
  }
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (h->prof) { e0 = h->take_event(); e1 = h->take_event(); cudaEventRecord(e0, st); }
  cudaError_t e = dsc::launch_decode(p, st);
  h->launches++;
  if (h->prof) {
    cudaEventRecord(e1, st);
    h->pending.push_back({e0, e1, 1});
  }
  if (e != cudaSuccess) return fail(DSCACHE_E_CUDA, std::string("decode launch: ") + cudaGetErrorString(e));
  return DSCACHE_OK;
}
}  // namespace

dscache_status dscache_decode(dscache_t h, int32_t lb, int32_t lc, const void* q, const void* k_self,
                              const void* v_self, int32_t n_self, int32_t n_q, void* o, void* stream) {
  return dscache_decode_sampled(h, lb, lc, q, k_self, v_self, n_self, n_q, 1, o, stream);
}

dscache_status dscache_decode_sampled(dscache_t h, int32_t lb, int32_t lc, const void* q, const void* k_self,
                                      const void* v_self, int32_t n_self, int32_t n_q, int32_t past_stride, void* o,
                                      void* stream) {
  NvtxRange nvtx_("dscache_decode_sampled");
  if (h && h->cfg.instant_source != DSCACHE_INSTANT_RING) return need_mode(h, DSCACHE_INSTANT_RING, "decode");
  if (!h) return fail(DSCACHE_E_ARG, "null handle");
  if (past_stride < 1) return fail(DSCACHE_E_ARG, "past_stride must be >= 1");
  if (decode_kernel_ok(h, n_q) && h->impl_attend == DSCACHE_IMPL_TC)
    return run_decode(h, lb, lc, q, k_self, v_self, n_self, n_q, past_stride, o, (cudaStream_t)stream);
  if (past_stride == 1) return attend_common(h, lb, lc, q, k_self, v_self, n_self, n_q, o, stream, false);
  // sampled past off the decode kernel (fp32, d = 64, adjacent RoPE, or > 16 query rows):
  // the SIMT kernel with the stride's slot map
  dsc::AttnParams p{};
  dscache_status s = prep_attend(h, lb, lc, q, k_self, v_self, n_self, n_q, o, false, p);
  if (s != DSCACHE_OK) return s;
  const Schedule sc = h->schedule(lb);
  const int tpf = h->cfg.tokens_per_frame;
  const int past_frames = sc.P_t / tpf, kept = (past_frames + past_stride - 1) / past_stride;
  p.past_stride = past_stride; p.stride_tpf = tpf; p.stride_past_frames = past_frames; p.stride_kept_frames = kept;
  p.ring_count = kept * tpf + sc.C_t;
  p.q_pos0 = h->cfg.sink_tokens + p.ring_count + (n_self - n_q);
  p.n_splits = 1; p.tiles_per_split = 1 << 30;
  DeviceGuard dg(h->cfg.device);
  return run_attention(h, p, DSCACHE_IMPL_SIMT, 1, (cudaStream_t)stream);
}

namespace {
// Eq. 7 over [sink | ring_older instant tokens of the ring (from the oldest instant slot) |
// n_inst caller tokens (k_inst, v_inst: [S][lc][n_inst][Hkv][d])]: the ring_older + n_inst
// queries at ids A + i, causal.  Serves the resolution boost (ring_older = C_t - tpf: the
// newest frame re-encoded) and the real-model mode (ring_older = 0: every instant K/V from
// the caller).
dscache_status build_with_inst(dscache_t h, int32_t lb, int32_t lc, const void* q_inst, const void* k_inst,
                               const void* v_inst, int32_t n_inst, int ring_older, void* o_inst, cudaStream_t st) {
  const Schedule sc = h->schedule(lb);
  if ((int64_t)h->cfg.sink_tokens + ring_older + n_inst > h->cfg.max_position)
    return fail(DSCACHE_E_POS_OVERFLOW, "A + instant tokens exceeds max_position");
  DeviceGuard dg(h->cfg.device);
  // keys: sink | ring window of the older instant frames | caller tokens as the self
  // segment (ids A + ring_older + j); queries: ids A + i over [older | caller tokens]
  dsc::AttnParams p{};
  fill_common(h, p, lb, lc);
  p.q = q_inst; p.o = o_inst; p.n_q = ring_older + n_inst; p.q_pos0 = h->cfg.sink_tokens;
  p.ring_start = sc.inst_start; p.ring_count = ring_older;
  p.self_k = k_inst; p.self_v = v_inst; p.n_self = n_inst;
  p.dbg_pos = nullptr;
  p.n_mblocks = (p.n_q * p.grp + 2 * dsc::kTileM - 1) / (2 * dsc::kTileM);
  const long long build_items = (long long)p.P * p.Hkv * p.n_mblocks;
  if (h->impl_build == DSCACHE_IMPL_TC && build_items >= 2LL * h->num_sms) {
    // staged as the plain build: [sink | older instant | caller tokens] once per (stream,
    // layer, kv head), K rotated at ids 0.., read by TMA (the caller tokens otherwise go
    // through the per-item sink/self loads)
    const int rows = h->cfg.sink_tokens + ring_older + n_inst;
    if (rows > h->bstage_rows) {
      cudaFree(h->bstage_k); cudaFree(h->bstage_v);
      h->bstage_k = h->bstage_v = nullptr; h->bstage_rows = 0;
      const size_t heads = (size_t)h->cfg.num_streams * h->cfg.num_layers * h->cfg.num_kv_heads;
      const size_t sb = heads * rows * h->cfg.head_dim * h->elem;
      if (cudaMalloc(&h->bstage_k, sb) != cudaSuccess || cudaMalloc(&h->bstage_v, sb) != cudaSuccess) {
        cudaGetLastError();
        return fail(DSCACHE_E_OOM, "instant staging allocation failed");
      }
      DSC_CUDA(dsc::make_kv_tmap(&h->tmap_bk, h->bstage_k, (unsigned long long)heads * rows, dsc::kTileN));
      DSC_CUDA(dsc::make_kv_tmap(&h->tmap_bk64, h->bstage_k, (unsigned long long)heads * rows, dsc::kTileN / 2));
      DSC_CUDA(dsc::make_kv_tmap(&h->tmap_bv, h->bstage_v, (unsigned long long)heads * rows, dsc::kTileN));
      h->bstage_rows = rows;
    }
    dsc::StageParams sp{};
    sp.sink_k = h->sink_k; sp.sink_v = h->sink_v; sp.ring_k = h->ring_k; sp.ring_v = h->ring_v;
    sp.stage_k = h->bstage_k; sp.stage_v = h->bstage_v; sp.rope_pairs = p.rope_pairs;
    sp.S = p.S; sp.layer_count = lc; sp.layer_begin = lb; sp.N_total = p.N_total; sp.Hkv = p.Hkv;
    sp.A = p.A; sp.R = h->R; sp.Rp_ring = h->Rp; sp.inst_start = sc.inst_start;
    sp.rows = rows; sp.rows_stage = h->bstage_rows;
    sp.boost_k = k_inst; sp.boost_v = v_inst; sp.n_older = ring_older;
    DSC_CUDA(dsc::launch_stage_instant(sp, st));
    h->launches++;
    p.staged = 1;
    p.A = 0; p.ring_start = 0; p.ring_count = rows; p.R = h->bstage_rows; p.Rp = h->bstage_rows;
    p.self_k = p.self_v = nullptr; p.n_self = 0;
    p.tmap_k = h->tmap_bk; p.tmap_v = h->tmap_bv; p.tmap_k64 = h->tmap_bk64;
  }
  return run_attention(h, p, h->impl_build, 0, st);
}

// Eq. 8 over [sink | ring window minus its newest ring_drop tokens | n_inst caller tokens |
// self (n_q)]: the [caller tokens | self] keys are gathered into per-call stream-ordered
// scratch [P][n_inst + n_q][Hkv][d] and passed as the self segment.
// n_self >= n_q: the self segment holds n_self tokens (the query chunk, plus during decoding
// the tokens generated so far) and the queries are its last n_q (n_self = n_q for an attend).
dscache_status attend_with_inst(dscache_t h, int32_t lb, int32_t lc, const void* q, const void* k_self,
                                const void* v_self, int32_t n_q, const void* k_inst, const void* v_inst,
                                int32_t n_inst, int ring_drop, void* o, cudaStream_t st, int32_t n_self = -1) {
  if (n_self < 0) n_self = n_q;
  const dscache_config& c = h->cfg;
  const size_t row = (size_t)c.num_kv_heads * c.head_dim * h->elem;      // one token of one problem
  const size_t P = (size_t)c.num_streams * lc;
  const size_t need = P * (size_t)(n_inst + n_self) * row;
  DeviceGuard dg(c.device);
  StreamScratch bk, bv;
  if (!bk.alloc(need, st) || !bv.alloc(need, st)) return fail(DSCACHE_E_OOM, "instant gather scratch allocation failed");
  dsc::AttnParams p{};
  dscache_status s = prep_attend(h, lb, lc, q, bk.ptr, bv.ptr, n_inst + n_self, n_q, o, false, p, ring_drop);
  if (s != DSCACHE_OK) return s;
  // self segment [caller tokens | self tokens] per problem: [P][n_inst + n_self][Hkv][d]
  const size_t pitch = (size_t)(n_inst + n_self) * row;
  if (n_inst > 0) {
    DSC_CUDA(cudaMemcpy2DAsync(bk.ptr, pitch, k_inst, n_inst * row, n_inst * row, P, cudaMemcpyDeviceToDevice, st));
    DSC_CUDA(cudaMemcpy2DAsync(bv.ptr, pitch, v_inst, n_inst * row, n_inst * row, P, cudaMemcpyDeviceToDevice, st));
  }
  DSC_CUDA(cudaMemcpy2DAsync((char*)bk.ptr + n_inst * row, pitch, k_self, n_self * row, n_self * row, P,
                             cudaMemcpyDeviceToDevice, st));
  DSC_CUDA(cudaMemcpy2DAsync((char*)bv.ptr + n_inst * row, pitch, v_self, n_self * row, n_self * row, P,
                             cudaMemcpyDeviceToDevice, st));
  return run_attention(h, p, h->impl_attend, 1, st);
}

}  // namespace

dscache_status dscache_build_instant_boost(dscache_t h, int32_t lb, int32_t lc, const void* q_inst,
                                           const void* k_boost, const void* v_boost, int32_t n_boost, void* o_inst,
                                           void* stream) {
  NvtxRange nvtx_("dscache_build_instant_boost");
  dscache_status s = need_mode(h, DSCACHE_INSTANT_RING, "build_instant_boost");
  if (s == DSCACHE_OK) s = check_layers(h, lb, lc);
  if (s != DSCACHE_OK) return s;
  if (!h->sink_filled[lb] || h->frames[lb] < 1)
    return fail(DSCACHE_E_STATE, "build_instant_boost before the sink and the first frame were appended");
  if (h->cfg.instant_frames < 1) return fail(DSCACHE_E_CONFIG, "l_I = 0: there is no instant cache");
  if (!q_inst || !k_boost || !v_boost || !o_inst) return fail(DSCACHE_E_ARG, "null q_inst/k_boost/v_boost/o_inst");
  if (n_boost < 1) return fail(DSCACHE_E_ARG, "n_boost must be >= 1");
  const int older = h->schedule(lb).C_t - h->cfg.tokens_per_frame;   // instant tokens before the newest frame
  return build_with_inst(h, lb, lc, q_inst, k_boost, v_boost, n_boost, older, o_inst, (cudaStream_t)stream);
}

dscache_status dscache_attend_boost(dscache_t h, int32_t lb, int32_t lc, const void* q, const void* k_self,
                                    const void* v_self, int32_t n_q, const void* k_boost, const void* v_boost,
                                    int32_t n_boost, void* o, void* stream) {
  NvtxRange nvtx_("dscache_attend_boost");
  dscache_status s = need_mode(h, DSCACHE_INSTANT_RING, "attend_boost");
  if (s != DSCACHE_OK) return s;
  if (n_q < 1 || n_q > h->cfg.max_query_tokens) return fail(DSCACHE_E_ARG, "n_q must be in [1, max_query_tokens]");
  if (h->cfg.instant_frames < 1) return fail(DSCACHE_E_CONFIG, "l_I = 0: there is no instant frame to boost");
  if (!k_boost || !v_boost || !k_self || !v_self) return fail(DSCACHE_E_ARG, "null k/v pointers");
  if (n_boost < 1) return fail(DSCACHE_E_ARG, "n_boost must be >= 1");
  s = check_layers(h, lb, lc);
  if (s != DSCACHE_OK) return s;
  return attend_with_inst(h, lb, lc, q, k_self, v_self, n_q, k_boost, v_boost, n_boost, h->cfg.tokens_per_frame, o,
                          (cudaStream_t)stream);
}

dscache_status dscache_append_past(dscache_t h, int32_t lb, int32_t lc, const void* k, const void* v,
                                   int32_t n_tokens, void* stream) {
  NvtxRange nvtx_("dscache_append_past");
  dscache_status s = need_mode(h, DSCACHE_INSTANT_EXTERNAL, "append_past");
  if (s == DSCACHE_OK) s = check_layers(h, lb, lc);
  if (s != DSCACHE_OK) return s;
  if (!h->sink_filled[lb]) return fail(DSCACHE_E_STATE, "append_past before the sink was appended");
  const dscache_config& c = h->cfg;
  const int64_t t = h->frames[lb];                  // the step this call advances to
  const int64_t leave = t - c.instant_frames;       // frame leaving the buffer at step t (Eq. 3)
  const int need = leave >= 0 ? c.tokens_per_frame : 0;
  if (n_tokens != need)
    return fail(DSCACHE_E_ARG, "append_past at step " + std::to_string(t) + " must carry " + std::to_string(need) +
                                   " tokens (the Eq. 5 K/V of frame t - l_I), got " + std::to_string(n_tokens));
  DeviceGuard dg(c.device);
  if (need > 0) {
    if (!k || !v) return fail(DSCACHE_E_ARG, "null k_past/v_past");
    dsc::AppendParams p{};
    p.k = k; p.v = v;
    p.S = c.num_streams; p.layer_count = lc; p.layer_begin = lb; p.N_total = c.num_layers; p.Hkv = c.num_kv_heads;
    p.row_bytes = c.head_dim * h->elem; p.elem_bytes = h->elem; p.n = n_tokens; p.poison_slot0 = -1;
    p.dst_k = h->ring_k; p.dst_v = h->ring_v; p.rows_dst = h->Rp; p.mirror_R = h->R;
    p.slot0 = (int)((leave * c.tokens_per_frame) % h->R);
    const int64_t ev = t - c.instant_frames - c.past_frames;   // Eq. 6: same closed form
    if (h->poison && ev >= 0) p.poison_slot0 = (int)((ev * c.tokens_per_frame) % h->R);
    DSC_CUDA(dsc::launch_append(p, (cudaStream_t)stream));
    h->launches++;
  }
  const int64_t ev = t - c.instant_frames - c.past_frames;
  for (int l = lb; l < lb + lc; ++l) { h->frames[l] = t + 1; h->last_evicted[l] = ev >= 0 ? ev : -1; }
  return DSCACHE_OK;
}

dscache_status dscache_build_instant_ext(dscache_t h, int32_t lb, int32_t lc, const void* q_inst, const void* k_inst,
                                         const void* v_inst, void* o_inst, void* stream) {
  NvtxRange nvtx_("dscache_build_instant_ext");
  dscache_status s = need_mode(h, DSCACHE_INSTANT_EXTERNAL, "build_instant_ext");
  if (s == DSCACHE_OK) s = check_layers(h, lb, lc);
  if (s != DSCACHE_OK) return s;
  if (!h->sink_filled[lb] || h->frames[lb] < 1)
    return fail(DSCACHE_E_STATE, "build_instant_ext before the sink and the first step");
  const int C_t = h->schedule(lb).C_t;
  if (C_t == 0) return DSCACHE_OK;                  // l_I = 0: no instant cache
  if (!q_inst || !k_inst || !v_inst || !o_inst) return fail(DSCACHE_E_ARG, "null q_inst/k_inst/v_inst/o_inst");
  return build_with_inst(h, lb, lc, q_inst, k_inst, v_inst, C_t, 0, o_inst, (cudaStream_t)stream);
}

dscache_status dscache_attend_ext(dscache_t h, int32_t lb, int32_t lc, const void* q, const void* k_self,
                                  const void* v_self, int32_t n_q, const void* k_inst, const void* v_inst, void* o,
                                  void* stream) {
  NvtxRange nvtx_("dscache_attend_ext");
  dscache_status s = need_mode(h, DSCACHE_INSTANT_EXTERNAL, "attend_ext");
  if (s != DSCACHE_OK) return s;
  if (n_q < 1 || n_q > h->cfg.max_query_tokens) return fail(DSCACHE_E_ARG, "n_q must be in [1, max_query_tokens]");
  s = check_layers(h, lb, lc);
  if (s != DSCACHE_OK) return s;
  if (!h->sink_filled[lb] || h->frames[lb] < 1) return fail(DSCACHE_E_STATE, "attend_ext before the sink and the first step");
  if (!k_self || !v_self) return fail(DSCACHE_E_ARG, "null k_self/v_self");
  const int C_t = h->schedule(lb).C_t;
  if (C_t > 0 && (!k_inst || !v_inst)) return fail(DSCACHE_E_ARG, "null k_inst/v_inst");
  // the ring holds only past frames in this mode: its window minus the C_t instant tokens
  return attend_with_inst(h, lb, lc, q, k_self, v_self, n_q, k_inst, v_inst, C_t, C_t, o, (cudaStream_t)stream);
}

dscache_status dscache_decode_ext(dscache_t h, int32_t lb, int32_t lc, const void* q, const void* k_self,
                                  const void* v_self, int32_t n_self, int32_t n_q, const void* k_inst,
                                  const void* v_inst, void* o, void* stream) {
  NvtxRange nvtx_("dscache_decode_ext");
  dscache_status s = need_mode(h, DSCACHE_INSTANT_EXTERNAL, "decode_ext");
  if (s != DSCACHE_OK) return s;
  if (n_q < 1 || n_q > n_self) return fail(DSCACHE_E_ARG, "need 1 <= n_q <= n_self");
  s = check_layers(h, lb, lc);
  if (s != DSCACHE_OK) return s;
  if (!h->sink_filled[lb] || h->frames[lb] < 1) return fail(DSCACHE_E_STATE, "decode_ext before the sink and the first step");
  if (!q || !k_self || !v_self || !o) return fail(DSCACHE_E_ARG, "null q/k_self/v_self/o");
  const int C_t = h->schedule(lb).C_t;
  if (C_t > 0 && (!k_inst || !v_inst)) return fail(DSCACHE_E_ARG, "null k_inst/v_inst");
  if (C_t > 0 && decode_kernel_ok(h, n_q) && h->impl_attend == DSCACHE_IMPL_TC)   // the memory-bound decode kernel
    return run_decode(h, lb, lc, q, k_self, v_self, n_self, n_q, 1, o, (cudaStream_t)stream, k_inst, v_inst);
  return attend_with_inst(h, lb, lc, q, k_self, v_self, n_q, k_inst, v_inst, C_t, C_t, o, (cudaStream_t)stream, n_self);
}

dscache_status dscache_attend_partial(dscache_t h, int32_t lb, int32_t lc, const void* q, const void* k_self,
                                      const void* v_self, int32_t n_q, int32_t part, int32_t n_parts, float* o_part,
                                      float* lse_part, void* stream) {
  NvtxRange nvtx_("dscache_attend_partial");
  if (h && h->cfg.instant_source != DSCACHE_INSTANT_RING) return need_mode(h, DSCACHE_INSTANT_RING, "attend_partial");
  if (!h) return fail(DSCACHE_E_ARG, "null handle");
  if (n_q < 1 || n_q > h->cfg.max_query_tokens) return fail(DSCACHE_E_ARG, "n_q must be in [1, max_query_tokens]");
  if (n_parts < 1 || part < 0 || part >= n_parts) return fail(DSCACHE_E_ARG, "need 0 <= part < n_parts");
  if (!o_part || !lse_part) return fail(DSCACHE_E_ARG, "null o_part/lse_part");
  if (h->impl_attend != DSCACHE_IMPL_TC)
    return fail(DSCACHE_E_CONFIG, "attend_partial runs on the tcgen05 path (bf16, d=128, split-half RoPE)");
  dsc::AttnParams p{};
  dscache_status s = prep_attend(h, lb, lc, q, k_self, v_self, n_q, n_q, /*o*/ o_part, false, p);
  if (s != DSCACHE_OK) return s;
  // the key tiles of every item (sink/self tiles, then logical window tiles), cut into n_parts
  // contiguous ranges; part `part` is computed here
  const int BN = dsc::kTileN;
  const int tiles = (p.A + n_q + BN - 1) / BN + (p.ring_count + BN - 1) / BN;
  const int tps = (tiles + n_parts - 1) / n_parts;
  if ((long long)(n_parts - 1) * tps >= tiles)
    return fail(DSCACHE_E_ARG, "n_parts = " + std::to_string(n_parts) + " leaves a part without keys (" +
                                   std::to_string(tiles) + " key tiles)");
  p.n_splits = n_parts; p.tiles_per_split = tps; p.split_only = part;
  p.ws_o = o_part; p.ws_lse = lse_part;
  DeviceGuard dg(h->cfg.device);
  return run_attention(h, p, h->impl_attend, 1, (cudaStream_t)stream);
}

dscache_status dscache_attend_peers(dscache_t h, int32_t lb, int32_t lc, const void* q, const void* k_self,
                                    const void* v_self, int32_t n_q, void* const* peer_o, int32_t n_peers,
                                    int32_t hq_total, int32_t head_offset, void* stream) {
  NvtxRange nvtx_("dscache_attend_peers");
  if (h && h->cfg.instant_source != DSCACHE_INSTANT_RING) return need_mode(h, DSCACHE_INSTANT_RING, "attend_peers");
  if (!h) return fail(DSCACHE_E_ARG, "null handle");
  if (n_q < 1 || n_q > h->cfg.max_query_tokens) return fail(DSCACHE_E_ARG, "n_q must be in [1, max_query_tokens]");
  if (!peer_o || n_peers < 1 || n_peers > dsc::kMaxPeers)
    return fail(DSCACHE_E_ARG, "need 1 <= n_peers <= " + std::to_string(dsc::kMaxPeers) + " destination buffers");
  for (int i = 0; i < n_peers; ++i)
    if (!peer_o[i]) return fail(DSCACHE_E_ARG, "null peer_o[" + std::to_string(i) + "]");
  if (head_offset < 0 || head_offset + h->cfg.num_q_heads > hq_total)
    return fail(DSCACHE_E_ARG, "head_offset + Hq must be <= hq_total");
  if (h->impl_attend != DSCACHE_IMPL_TC)
    return fail(DSCACHE_E_CONFIG, "attend_peers runs on the tcgen05 path (bf16, d=128, split-half RoPE)");
  dsc::AttnParams p{};
  dscache_status s = prep_attend(h, lb, lc, q, k_self, v_self, n_q, n_q, peer_o[0], false, p);
  if (s != DSCACHE_OK) return s;
  for (int i = 0; i < n_peers; ++i) p.peer_o[i] = peer_o[i];
  p.n_peers = n_peers; p.o_hq = hq_total; p.o_head_off = head_offset;
  DeviceGuard dg(h->cfg.device);
  return run_attention(h, p, h->impl_attend, 1, (cudaStream_t)stream);
}

dscache_status dscache_ipc_handle(const void* dev_ptr, void* handle_out, int64_t* offset_out) {
  if (!dev_ptr || !handle_out || !offset_out) return fail(DSCACHE_E_ARG, "null pointer");
  // the handle names the whole allocation; report where dev_ptr sits inside it
  using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static GetRange get_range = nullptr;
  if (!get_range) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    DSC_CUDA(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !fn) return fail(DSCACHE_E_CUDA, "cuMemGetAddressRange unavailable");
    get_range = reinterpret_cast<GetRange>(fn);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (get_range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
    return fail(DSCACHE_E_CUDA, "cuMemGetAddressRange failed (not a device allocation?)");
  cudaIpcMemHandle_t hd;
  DSC_CUDA(cudaIpcGetMemHandle(&hd, reinterpret_cast<void*>(base)));
  std::memcpy(handle_out, &hd, sizeof(hd));
  *offset_out = (int64_t)(reinterpret_cast<CUdeviceptr>(dev_ptr) - base);
  return DSCACHE_OK;
}

dscache_status dscache_ipc_open(int32_t device, const void* handle, void** dev_ptr_out) {
  if (!handle || !dev_ptr_out) return fail(DSCACHE_E_ARG, "null pointer");
  DeviceGuard dg(device);
  cudaIpcMemHandle_t hd;
  std::memcpy(&hd, handle, sizeof(hd));
  DSC_CUDA(cudaIpcOpenMemHandle(dev_ptr_out, hd, cudaIpcMemLazyEnablePeerAccess));
  return DSCACHE_OK;
}

dscache_status dscache_ipc_close(int32_t device, void* dev_ptr) {
  if (!dev_ptr) return fail(DSCACHE_E_ARG, "null pointer");
  DeviceGuard dg(device);
  DSC_CUDA(cudaIpcCloseMemHandle(dev_ptr));
  return DSCACHE_OK;
}

dscache_status dscache_combine_partials(dscache_t h, int32_t n_parts, int64_t rows, const float* o_parts,
                                        const float* lse_parts, void* o, void* stream) {
  NvtxRange nvtx_("dscache_combine_partials");
  if (!h) return fail(DSCACHE_E_ARG, "null handle");
  if (n_parts < 1 || rows < 1 || !o_parts || !lse_parts || !o) return fail(DSCACHE_E_ARG, "bad combine arguments");
  if (h->cfg.dtype != DSCACHE_DTYPE_BF16 || h->cfg.head_dim != 128)
    return fail(DSCACHE_E_CONFIG, "combine_partials writes bf16 rows of d = 128");
  DeviceGuard dg(h->cfg.device);
  DSC_CUDA(dsc::launch_combine_partials(n_parts, rows, h->cfg.head_dim, o_parts, lse_parts, o, (cudaStream_t)stream));
  h->launches++;
  return DSCACHE_OK;
}

dscache_status dscache_step(dscache_t h, int32_t lb, int32_t lc, const void* k_frame, const void* v_frame,
                            const void* q_inst, void* o_inst, const void* q, const void* k_self, const void* v_self,
                            int32_t n_q, void* o, void* stream) {
  NvtxRange nvtx_("dscache_step");
  if (h && h->cfg.instant_source != DSCACHE_INSTANT_RING) return need_mode(h, DSCACHE_INSTANT_RING, "step");
  if (!h) return fail(DSCACHE_E_ARG, "null handle");
  if (n_q < 1 || n_q > h->cfg.max_query_tokens) return fail(DSCACHE_E_ARG, "n_q must be in [1, max_query_tokens]");
  dscache_status cs = check_layers(h, lb, lc);
  if (cs != DSCACHE_OK) return cs;
  if (!h->sink_filled[lb]) return fail(DSCACHE_E_STATE, "step before the sink was appended");
  dscache_status s = dscache_append_frame(h, lb, lc, k_frame, v_frame, h->cfg.tokens_per_frame, stream);
  if (s != DSCACHE_OK) return s;
  dsc::AttnParams pb{}, pa{};
  dsc::StageParams sp{};
  bool empty = false;
  s = prep_build(h, lb, lc, q_inst, o_inst, pb, &empty, &sp);
  if (s != DSCACHE_OK) return s;
  s = prep_attend(h, lb, lc, q, k_self, v_self, n_q, n_q, o, true, pa);
  if (s != DSCACHE_OK) return s;
  DeviceGuard dg(h->cfg.device);
  cudaStream_t st = (cudaStream_t)stream;
  if (!empty && pb.staged) {
    DSC_CUDA(dsc::launch_stage_instant(sp, st));
    h->launches++;
  }
  if (empty || h->impl_build != DSCACHE_IMPL_TC || h->impl_attend != DSCACHE_IMPL_TC) {
    if (!empty) {
      s = run_attention(h, pb, h->impl_build, 0, st);
      if (s != DSCACHE_OK) return s;
    }
    return run_attention(h, pa, h->impl_attend, 1, st);
  }
  // one persistent tcgen05 launch: the attend items (longest) first, then the build items
  StreamScratch ws;
  s = alloc_ws(pa, ws, st);
  if (s != DSCACHE_OK) return s;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (h->prof) { e0 = h->take_event(); e1 = h->take_event(); cudaEventRecord(e0, st); }
  cudaError_t e = launch_tc(h, pa, &pb, st);
  h->launches++;
  if (e == cudaSuccess && pa.n_splits > 1) { e = dsc::launch_combine(pa, st); h->launches++; }
  if (h->prof) {
    cudaEventRecord(e1, st);
    h->pending.push_back({e0, e1, 1});
  }
  if (e != cudaSuccess) return fail(DSCACHE_E_CUDA, std::string("fused step launch: ") + cudaGetErrorString(e));
  return DSCACHE_OK;
}

dscache_status dscache_update_attend(dscache_t h, int32_t lb, int32_t lc, const void* q_upd, void* o_upd,
                                     int32_t active_frames, void* stream) {
  NvtxRange nvtx_("dscache_update_attend");
  dscache_status s = check_layers(h, lb, lc);
  if (s != DSCACHE_OK) return s;
  const dscache_config& c = h->cfg;
  if (!h->sink_filled[lb] || h->frames[lb] < 1)
    return fail(DSCACHE_E_STATE, "update_attend before the sink and the first frame were appended");
  if (active_frames < 0) return fail(DSCACHE_E_ARG, "active_frames must be >= 0");
  const int64_t t = h->frames[lb] - 1;
  const int64_t e = t - c.instant_frames;               // the input leaving the buffer at step t
  if (e < 0) return fail(DSCACHE_E_STATE, "no input has left the buffer yet (step < l_I)");
  if (!q_upd || !o_upd) return fail(DSCACHE_E_ARG, "null q_upd/o_upd");
  DeviceGuard dg(c.device);
  // U_{t-1} holds min(e, l_U) frames (e - min(e,l_U) .. e-1); zeta = the newest nz of them
  const int64_t nz = std::min<int64_t>({(int64_t)active_frames, (int64_t)c.past_frames, e});
  dsc::AttnParams p{};
  fill_common(h, p, lb, lc);
  p.q = q_upd; p.o = o_upd; p.n_q = c.tokens_per_frame;
  p.ring_start = (int)(((e - nz) * c.tokens_per_frame) % h->R);
  p.ring_count = (int)((nz + 1) * c.tokens_per_frame);
  p.q_pos0 = c.sink_tokens + (int)(nz * c.tokens_per_frame);
  p.self_k = p.self_v = nullptr; p.n_self = 0;
  p.dbg_pos = nullptr;
  p.n_mblocks = (p.n_q * p.grp + 2 * dsc::kTileM - 1) / (2 * dsc::kTileM);
  return run_attention(h, p, h->impl_build, 0, (cudaStream_t)stream);
}

dscache_status dscache_get_state(dscache_t h, int32_t layer, dscache_state* out) {
  if (!h || !out) return fail(DSCACHE_E_ARG, "null handle/output");
  if (layer < 0 || layer >= h->cfg.num_layers) return fail(DSCACHE_E_ARG, "layer out of range");
  dscache_state st{};
  st.frames_seen = h->frames[layer];
  st.sink_filled = h->sink_filled[layer];
  st.ring_slots = h->R;
  st.last_evicted_frame = h->last_evicted[layer];
  if (h->frames[layer] > 0) {
    Schedule sc = h->schedule(layer);
    st.past_tokens = sc.P_t; st.instant_tokens = sc.C_t;
    st.tail_slot = sc.ring_start; st.instant_slot = sc.inst_start;
  }
  st.max_key_id = h->cfg.sink_tokens + st.past_tokens + st.instant_tokens - 1;
  st.next_instant_tokens =
      (int32_t)(std::min<int64_t>(h->frames[layer] + 1, h->cfg.instant_frames) * h->cfg.tokens_per_frame);
  st.instant_capacity = h->C;
  st.max_query_id = st.max_key_id + h->cfg.max_query_tokens;
  *out = st;
  return DSCACHE_OK;
}

// rows per head [rows] copied out of a device layout with `pitch_rows` rows per head
static dscache_status copy_rows(dscache_t h, int s_idx, int layer, const void* dk, const void* dv, int rows,
                                int pitch_rows, void* kh, void* vh) {
  if (!h || !kh || !vh) return fail(DSCACHE_E_ARG, "null argument");
  const dscache_config& c = h->cfg;
  if (s_idx < 0 || s_idx >= c.num_streams || layer < 0 || layer >= c.num_layers)
    return fail(DSCACHE_E_ARG, "stream/layer out of range");
  DeviceGuard dg(c.device);
  const size_t row_bytes = (size_t)c.head_dim * h->elem;
  const size_t off = ((size_t)s_idx * c.num_layers + layer) * c.num_kv_heads * pitch_rows * row_bytes;
  DSC_CUDA(cudaDeviceSynchronize());
  DSC_CUDA(cudaMemcpy2D(kh, rows * row_bytes, (const char*)dk + off, pitch_rows * row_bytes, rows * row_bytes,
                        c.num_kv_heads, cudaMemcpyDeviceToHost));
  DSC_CUDA(cudaMemcpy2D(vh, rows * row_bytes, (const char*)dv + off, pitch_rows * row_bytes, rows * row_bytes,
                        c.num_kv_heads, cudaMemcpyDeviceToHost));
  return DSCACHE_OK;
}

dscache_status dscache_copy_ring(dscache_t h, int32_t s_idx, int32_t layer, void* kh, void* vh) {
  if (!h) return fail(DSCACHE_E_ARG, "null handle");
  return copy_rows(h, s_idx, layer, h->ring_k, h->ring_v, h->R, h->Rp, kh, vh);
}

dscache_status dscache_copy_sink(dscache_t h, int32_t s_idx, int32_t layer, void* kh, void* vh) {
  if (!h) return fail(DSCACHE_E_ARG, "null handle");
  if (h->cfg.sink_tokens == 0) return DSCACHE_OK;
  return copy_rows(h, s_idx, layer, h->sink_k, h->sink_v, h->cfg.sink_tokens, h->cfg.sink_tokens, kh, vh);
}

// rows per head [rows] uploaded into a device layout with `pitch_rows` rows per head (inverse
// of copy_rows); mirror = also write slots [0, min(rows, kMirror)) to rows [rows, rows + ...)
static dscache_status upload_rows(dscache_t h, int s_idx, int layer, void* dk, void* dv, int rows, int pitch_rows,
                                  bool mirror, const void* kh, const void* vh) {
  if (!h || !kh || !vh) return fail(DSCACHE_E_ARG, "null argument");
  const dscache_config& c = h->cfg;
  if (s_idx < 0 || s_idx >= c.num_streams || layer < 0 || layer >= c.num_layers)
    return fail(DSCACHE_E_ARG, "stream/layer out of range");
  DeviceGuard dg(c.device);
  const size_t row_bytes = (size_t)c.head_dim * h->elem;
  const size_t off = ((size_t)s_idx * c.num_layers + layer) * c.num_kv_heads * pitch_rows * row_bytes;
  DSC_CUDA(cudaDeviceSynchronize());   // no kernel of any stream may still read the rows replaced
  for (int which = 0; which < 2; ++which) {
    char* dst = (char*)(which ? dv : dk) + off;
    const void* src = which ? vh : kh;
    DSC_CUDA(cudaMemcpy2D(dst, pitch_rows * row_bytes, src, rows * row_bytes, rows * row_bytes, c.num_kv_heads,
                          cudaMemcpyHostToDevice));
    const int nm = std::min(rows, dsc::kMirror);
    if (mirror && nm > 0)
      DSC_CUDA(cudaMemcpy2D(dst + rows * row_bytes, pitch_rows * row_bytes, src, rows * row_bytes, nm * row_bytes,
                            c.num_kv_heads, cudaMemcpyHostToDevice));
  }
  DSC_CUDA(cudaDeviceSynchronize());
  return DSCACHE_OK;
}

dscache_status dscache_restore_ring(dscache_t h, int32_t s_idx, int32_t layer, const void* kh, const void* vh) {
  if (!h) return fail(DSCACHE_E_ARG, "null handle");
  return upload_rows(h, s_idx, layer, h->ring_k, h->ring_v, h->R, h->Rp, true, kh, vh);
}

dscache_status dscache_restore_sink(dscache_t h, int32_t s_idx, int32_t layer, const void* kh, const void* vh) {
  if (!h) return fail(DSCACHE_E_ARG, "null handle");
  if (h->cfg.sink_tokens == 0) return DSCACHE_OK;
  return upload_rows(h, s_idx, layer, h->sink_k, h->sink_v, h->cfg.sink_tokens, h->cfg.sink_tokens, false, kh, vh);
}

dscache_status dscache_set_state(dscache_t h, int32_t layer, int64_t frames_seen, int32_t sink_filled) {
  if (!h) return fail(DSCACHE_E_ARG, "null handle");
  const dscache_config& c = h->cfg;
  if (layer < 0 || layer >= c.num_layers) return fail(DSCACHE_E_ARG, "layer out of range");
  if (frames_seen < 0 || (sink_filled != 0 && sink_filled != 1))
    return fail(DSCACHE_E_ARG, "frames_seen must be >= 0 and sink_filled 0 or 1");
  if (c.sink_tokens == 0 && !sink_filled) return fail(DSCACHE_E_STATE, "A = 0: the sink is always filled");
  if (frames_seen > 0 && !sink_filled) return fail(DSCACHE_E_STATE, "frames cannot precede the sink");
  // ids stay below max_position for any frames_seen: create bounded A + W + max(C + q_max, tpf)
  h->frames[layer] = frames_seen;
  h->sink_filled[layer] = sink_filled;
  const int64_t ev = frames_seen - 1 - c.instant_frames - c.past_frames;   // dropped at the latest append (Eq. 6)
  h->last_evicted[layer] = ev >= 0 ? ev : -1;
  h->approx_last[layer] = -1;   // the approximate cache's reuse chain restarts with a refresh
  h->approx_ring[layer] = nullptr;
  return DSCACHE_OK;
}

int32_t dscache_debug_len(dscache_t h) {
  if (!h) return 0;
  return h->cfg.sink_tokens + h->R + 2 * std::max(h->C, h->cfg.max_query_tokens);   // per problem
}

dscache_status dscache_set_debug(dscache_t h, int32_t* build_pos, int32_t* attend_pos, int32_t poison) {
  if (!h) return fail(DSCACHE_E_ARG, "null handle");
  h->dbg_build = build_pos; h->dbg_attend = attend_pos; h->poison = poison;
  return DSCACHE_OK;
}

dscache_status dscache_set_trace(dscache_t h, int64_t* buf, int32_t ntrace_cta) {
  if (!h) return fail(DSCACHE_E_ARG, "null handle");
  if (buf && ntrace_cta < 1) return fail(DSCACHE_E_ARG, "ntrace_cta must be >= 1");
  h->trace = reinterpret_cast<long long*>(buf);
  h->ntrace = buf ? ntrace_cta : 0;
  return DSCACHE_OK;
}

dscache_status dscache_profile(dscache_t h, int32_t enable) {
  if (!h) return fail(DSCACHE_E_ARG, "null handle");
  h->prof = enable;
  return DSCACHE_OK;
}

dscache_status dscache_profile_read(dscache_t h, double* ms_build, double* ms_attend, int64_t* n_build,
                                    int64_t* n_attend, int64_t* kernel_launches, int32_t reset) {
  if (!h) return fail(DSCACHE_E_ARG, "null handle");
  DeviceGuard dg(h->cfg.device);
  for (auto& ev : h->pending) {
    DSC_CUDA(cudaEventSynchronize(ev.b));
    float ms = 0.f;
    DSC_CUDA(cudaEventElapsedTime(&ms, ev.a, ev.b));
    h->ms[ev.kind] += ms;
    h->n[ev.kind] += 1;
    h->pool.push_back(ev.a); h->pool.push_back(ev.b);
  }
  h->pending.clear();
  if (ms_build) *ms_build = h->ms[0];
  if (ms_attend) *ms_attend = h->ms[1];
  if (n_build) *n_build = h->n[0];
  if (n_attend) *n_attend = h->n[1];
  if (kernel_launches) *kernel_launches = h->launches;
  if (reset) { h->ms[0] = h->ms[1] = 0; h->n[0] = h->n[1] = 0; h->launches = 0; }
  return DSCACHE_OK;
}

int32_t dscache_watchdog_read(uint64_t* out, int32_t n) {
  if (!out || n < 1) return -1;
  return dsc::fa_watchdog_read(reinterpret_cast<unsigned long long*>(out), n);
}

int32_t dscache_attn_impl(dscache_t h, int32_t which) {
  if (!h) return -1;
  return which == 0 ? h->impl_build : h->impl_attend;
}

}  // extern "C"
