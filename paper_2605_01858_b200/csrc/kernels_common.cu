// sm_100a kernels of the DSCache hot path other than the tcgen05 attention:
//   K1 append/evict  -- 16-byte vector copy of a frame's raw K/V into ring slots
//                       (f*tpf + j) mod R; eviction is a host pointer move, the
//                       optional debug poison overwrites the evicted frame's slots
//   K2 rope table    -- (cos, sin)(p * theta_i) in fp64, rounded to fp32, indexed by id
//   K6 SIMT attention-- fp32 FFMA flash attention (online softmax, warp shuffles) with
//                       RoPE on load; serves the fp32 configs and ineligible shapes
//   K5 combine       -- merges split-KV partials (O_s / l_s, log2-sum-exp) into O
#include "dscache_internal.h"

#include <cuda_bf16.h>
#include <cstdint>
#include <algorithm>

namespace dsc {

// ------------------------------------------------------------------ K2 RoPE table
// theta_i = base^(-2i/d) (reading Q7); the angle p*theta_i is formed in
// fp64 so the table is exact to fp32 rounding at every id (< 3e-8 abs).
__global__ void rope_table_kernel(float2* __restrict__ t, int npos, int d, double theta) {
  const int half = d / 2;
  const long long total = (long long)npos * half;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int f = (int)(idx % half);
    const long long pos = idx / half;
    const double inv = pow(theta, -2.0 * (double)f / (double)d);
    double s, c;
    sincos((double)pos * inv, &s, &c);
    t[idx] = make_float2((float)c, (float)s);
  }
}

// Same angles, pair-packed for f32x2 math: entry (pos, j) = (cos f, cos f+1, sin f, sin f+1)
// with f = 2j, so a float4 load yields the cos and sin of two adjacent frequencies.
__global__ void rope_table_pairs_kernel(float4* __restrict__ t, int npos, int d, double theta) {
  const int pairs = d / 4;
  const long long total = (long long)npos * pairs;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(idx % pairs);
    const long long pos = idx / pairs;
    double s0, c0, s1, c1;
    sincos((double)pos * pow(theta, -2.0 * (double)(2 * j) / (double)d), &s0, &c0);
    sincos((double)pos * pow(theta, -2.0 * (double)(2 * j + 1) / (double)d), &s1, &c1);
    t[idx] = make_float4((float)c0, (float)c1, (float)s0, (float)s1);
  }
}

cudaError_t launch_rope_table(float2* table, int npos, int d, double theta, cudaStream_t st) {
  const long long total = (long long)npos * (d / 2);
  int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 16);
  rope_table_kernel<<<blocks, 256, 0, st>>>(table, npos, d, theta);
  // the pair-packed copy lives right after the float2 table (same byte size)
  rope_table_pairs_kernel<<<blocks, 256, 0, st>>>(reinterpret_cast<float4*>(table + total), npos, d, theta);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ K1 append / evict
__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// blockIdx.y: 0 = K, 1 = V.  Each thread moves 4 independent 16-byte chunks per
// iteration (4 loads in flight before the stores).  Source [S][lc][n][Hkv][d] is
// read fully coalesced; destination rows are 256-byte contiguous per (head, slot).
__global__ void __launch_bounds__(256) append_kernel(AppendParams p) {
  const int cpr = p.row_bytes >> 4;
  const long long total = (long long)p.S * p.layer_count * p.n * p.Hkv * cpr;
  const uint4* __restrict__ src = reinterpret_cast<const uint4*>(blockIdx.y ? p.v : p.k);
  uint4* __restrict__ dst = reinterpret_cast<uint4*>(blockIdx.y ? p.dst_v : p.dst_k);
  const long long stride = (long long)gridDim.x * blockDim.x;
  // destination chunk of source chunk idx; *mirror = the chunk's mirror copy (ring slot
  // s < kMirror is also stored at row R + s), -1 if none
  auto dst_index = [&](long long idx, long long* mirror) -> long long {
    const int c = (int)(idx % cpr);
    long long r = idx / cpr;
    const int g = (int)(r % p.Hkv); r /= p.Hkv;
    const int j = (int)(r % p.n); r /= p.n;
    const int l = (int)(r % p.layer_count);
    const long long s = r / p.layer_count;
    const long long head = ((s * p.N_total + p.layer_begin + l) * p.Hkv + g) * p.rows_dst;
    const int slot = p.slot0 + j;
    DSC_ASSERT(slot >= 0 && slot < (p.mirror_R > 0 ? p.mirror_R : p.rows_dst) && s < p.S, "append destination row");
    *mirror = (p.mirror_R > 0 && slot < kMirror) ? (head + p.mirror_R + slot) * cpr + c : -1;
    return (head + slot) * cpr + c;
  };
  auto put = [&](long long idx, uint4 v) {
    long long mi;
    dst[dst_index(idx, &mi)] = v;
    if (mi >= 0) dst[mi] = v;
  };
  long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; idx + 3 * stride < total; idx += 4 * stride) {
    uint4 a = ld_stream(src + idx), b = ld_stream(src + idx + stride);
    uint4 c = ld_stream(src + idx + 2 * stride), d = ld_stream(src + idx + 3 * stride);
    put(idx, a);
    put(idx + stride, b);
    put(idx + 2 * stride, c);
    put(idx + 3 * stride, d);
  }
  for (; idx < total; idx += stride) put(idx, ld_stream(src + idx));

  if (p.poison_slot0 >= 0) {
    // sentinel = 1e30 (finite): bf16 0x714A, fp32 0x7149F2CA
    const uint32_t w = p.elem_bytes == 2 ? 0x714A714Au : 0x7149F2CAu;
    const uint4 pv = make_uint4(w, w, w, w);
    for (long long i2 = blockIdx.x * (long long)blockDim.x + threadIdx.x; i2 < total; i2 += stride) {
      const int c = (int)(i2 % cpr);
      long long r = i2 / cpr;
      const int g = (int)(r % p.Hkv); r /= p.Hkv;
      const int j = (int)(r % p.n); r /= p.n;
      const int l = (int)(r % p.layer_count);
      const long long s = r / p.layer_count;
      const long long head = ((s * p.N_total + p.layer_begin + l) * p.Hkv + g) * p.rows_dst;
      const int slot = p.poison_slot0 + j;
      dst[(head + slot) * cpr + c] = pv;
      if (p.mirror_R > 0 && slot < kMirror) dst[(head + p.mirror_R + slot) * cpr + c] = pv;
    }
  }
}

cudaError_t launch_append(const AppendParams& p, cudaStream_t st) {
  const long long total = (long long)p.S * p.layer_count * p.n * p.Hkv * (p.row_bytes >> 4);
  int blocks = (int)std::min<long long>((total + 1023) / 1024, 148 * 8);
  if (blocks < 1) blocks = 1;
  append_kernel<<<dim3(blocks, 2), 256, 0, st>>>(p);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ K8 instant-window staging
// One thread per (head, staged row, 8-frequency chunk c8): K chunk c8 (cols 8c8..8c8+7) and
// its split-half partner (cols 64+8c8..) rotated at id = row with the fp64-built pair table
// (y_f = x_f cos - x_{f+64} sin, y_{f+64} = x_f sin + x_{f+64} cos, Def. 4.1
// applied at the build's ids), rounded to bf16; the V row's two 16-byte chunks
// are copied alongside.
__device__ __forceinline__ float2 bfp(uint32_t w) {
  return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u));
}
__device__ __forceinline__ uint32_t pk_bf16(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__global__ void __launch_bounds__(256) stage_instant_kernel(StageParams p) {
  const long long total = (long long)p.S * p.layer_count * p.Hkv * p.rows * 8;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int c8 = (int)(idx & 7);
    long long r = idx >> 3;
    const int row = (int)(r % p.rows); r /= p.rows;
    const int g = (int)(r % p.Hkv); r /= p.Hkv;
    const int l = (int)(r % p.layer_count);
    const long long s = r / p.layer_count;
    const long long head = (s * p.N_total + p.layer_begin + l) * p.Hkv + g;
    const uint4 *sk, *sv;
    if (row < p.A) {
      sk = reinterpret_cast<const uint4*>(p.sink_k) + (head * p.A + row) * 16;
      sv = reinterpret_cast<const uint4*>(p.sink_v) + (head * p.A + row) * 16;
    } else if (p.boost_k != nullptr && row >= p.A + p.n_older) {
      const int nb = p.rows - p.A - p.n_older;
      const long long br = ((s * p.layer_count + l) * nb + (row - p.A - p.n_older)) * p.Hkv + g;
      sk = reinterpret_cast<const uint4*>(p.boost_k) + br * 16;
      sv = reinterpret_cast<const uint4*>(p.boost_v) + br * 16;
    } else {
      int slot = p.inst_start + row - p.A;
      if (slot >= p.R) slot -= p.R;
      sk = reinterpret_cast<const uint4*>(p.ring_k) + (head * p.Rp_ring + slot) * 16;
      sv = reinterpret_cast<const uint4*>(p.ring_v) + (head * p.Rp_ring + slot) * 16;
    }
    DSC_ASSERT(row < p.rows_stage && s < p.S, "stage destination row");
    uint4* dk = reinterpret_cast<uint4*>(p.stage_k) + (head * p.rows_stage + row) * 16;
    uint4* dv = reinterpret_cast<uint4*>(p.stage_v) + (head * p.rows_stage + row) * 16;
    const uint4 lo = sk[c8], hi = sk[c8 + 8];
    const float4* t = p.rope_pairs + (long long)row * 32 + 4 * c8;
    const uint32_t lw[4] = {lo.x, lo.y, lo.z, lo.w}, hw[4] = {hi.x, hi.y, hi.z, hi.w};
    uint32_t ol[4], oh[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float4 cs = t[j];   // (cos f, cos f+1, sin f, sin f+1), f = 8c8 + 2j
      const float2 a = bfp(lw[j]), b = bfp(hw[j]);
      ol[j] = pk_bf16(a.x * cs.x - b.x * cs.z, a.y * cs.y - b.y * cs.w);
      oh[j] = pk_bf16(a.x * cs.z + b.x * cs.x, a.y * cs.w + b.y * cs.y);
    }
    dk[c8] = make_uint4(ol[0], ol[1], ol[2], ol[3]);
    dk[c8 + 8] = make_uint4(oh[0], oh[1], oh[2], oh[3]);
    // debug export: the build id this K row was rotated at, by sink row / ring slot (kv head 0)
    if (p.dbg_pos && g == 0 && c8 == 0 && p.boost_k == nullptr) {
      int* const dbgp = p.dbg_pos + (s * p.N_total + p.layer_begin + l) * p.dbg_len;
      int slot = p.inst_start + row - p.A;
      if (slot >= p.R) slot -= p.R;
      dbgp[row < p.A ? row : p.A + slot] = row;
    }
    dv[c8] = sv[c8];
    dv[c8 + 8] = sv[c8 + 8];
  }
}

cudaError_t launch_stage_instant(const StageParams& p, cudaStream_t st) {
  const long long total = (long long)p.S * p.layer_count * p.Hkv * p.rows * 8;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 16);
  stage_instant_kernel<<<std::max(blocks, 1), 256, 0, st>>>(p);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ K6 SIMT attention
template <typename T> __device__ __forceinline__ float to_f(T x);
template <> __device__ __forceinline__ float to_f<float>(float x) { return x; }
template <> __device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }
template <typename T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }

// Lane `lane` holds E = D/32 elements.  Split-half: element e_k = lane + 32k, pairs
// (k, k+E/2) with frequency lane + 32k.  Adjacent: element 2(lane+32m)+b for k = 2m+b,
// pairs (2m, 2m+1) with frequency lane + 32m.  Either way both members of a pair are
// in the same lane, so the rotation needs no shuffles.
template <int D>
__device__ __forceinline__ int elem_of(int lane, int k, int style) {
  return style == 0 ? lane + 32 * k : 2 * (lane + 32 * (k >> 1)) + (k & 1);
}

template <int D>
__device__ __forceinline__ void rotate(float (&x)[D / 32], const float2* __restrict__ rope, int pos, int lane,
                                       int style) {
  constexpr int E = D / 32;
  const float2* row = rope + (long long)pos * (D / 2);
  if (style == 0) {
#pragma unroll
    for (int k = 0; k < E / 2; ++k) {
      const float2 cs = row[lane + 32 * k];
      const float a = x[k], b = x[k + E / 2];
      x[k] = a * cs.x - b * cs.y;
      x[k + E / 2] = a * cs.y + b * cs.x;
    }
  } else {
#pragma unroll
    for (int m = 0; m < E / 2; ++m) {
      const float2 cs = row[lane + 32 * m];
      const float a = x[2 * m], b = x[2 * m + 1];
      x[2 * m] = a * cs.x - b * cs.y;
      x[2 * m + 1] = a * cs.y + b * cs.x;
    }
  }
}

// One warp per (problem, query row i, q head h).  Keys in logical order L, id L;
// visible iff L <= q_pos0 + i (AttnParams).  Online softmax in fp32 with expf.
template <typename T, int D>
__global__ void __launch_bounds__(128) attn_simt_kernel(AttnParams p) {
  constexpr int E = D / 32;
  const int lane = threadIdx.x & 31;
  const long long wg = blockIdx.x * 4ll + (threadIdx.x >> 5);
  const long long total = (long long)p.P * p.n_q * p.Hq;
  if (wg >= total) return;
  const int h = (int)(wg % p.Hq);
  const int i = (int)((wg / p.Hq) % p.n_q);
  const int pp = (int)(wg / ((long long)p.Hq * p.n_q));
  const int s = pp / p.layer_count, l = pp % p.layer_count;
  const int g = h / p.grp;
  const long long head_row = ((long long)s * p.N_total + p.layer_begin + l) * p.Hkv + g;
  const T* __restrict__ Q = reinterpret_cast<const T*>(p.q);
  const T* __restrict__ SK = reinterpret_cast<const T*>(p.sink_k);
  const T* __restrict__ SV = reinterpret_cast<const T*>(p.sink_v);
  const T* __restrict__ RK = reinterpret_cast<const T*>(p.ring_k);
  const T* __restrict__ RV = reinterpret_cast<const T*>(p.ring_v);
  const T* __restrict__ XK = reinterpret_cast<const T*>(p.self_k);
  const T* __restrict__ XV = reinterpret_cast<const T*>(p.self_v);

  const int qpos = p.q_pos0 + i;
  float q[E];
  const T* qrow = Q + (((long long)pp * p.n_q + i) * p.Hq + h) * D;
#pragma unroll
  for (int k = 0; k < E; ++k) q[k] = to_f(qrow[elem_of<D>(lane, k, p.rope_style)]);
  rotate<D>(q, p.rope, qpos, lane, p.rope_style);
  const float scale = rsqrtf((float)D);

  // debug export: every problem, q head 0, block [s * N_total + layer] of the buffer
  const bool dbg = p.dbg_pos && g == 0 && h == 0;
  int* const dbgp = dbg ? p.dbg_pos + (head_row / p.Hkv) * p.dbg_len : nullptr;
  if (dbg && lane == 0) dbgp[p.dbg_A + p.dbg_R + p.dbg_M + i] = qpos;
  const bool dbg_keys = dbg && i == p.n_q - 1;

  const int n_keys = p.A + p.ring_count + p.n_self;
  const int last = min(qpos, n_keys - 1);
  float m = -INFINITY, lsum = 0.f, acc[E];
#pragma unroll
  for (int k = 0; k < E; ++k) acc[k] = 0.f;
  for (int L = 0; L <= last; ++L) {
    const T *kr, *vr;
    if (L < p.A) {
      kr = SK + (head_row * p.A + L) * D; vr = SV + (head_row * p.A + L) * D;
      if (dbg_keys && lane == 0) dbgp[L] = L;
    } else if (L < p.A + p.ring_count) {
      const int x = L - p.A;
      int slot;
      if (p.past_stride > 1) {
        const int kept = p.stride_kept_frames * p.stride_tpf;
        if (x < kept) {
          const int kk = x / p.stride_tpf, tok = x - kk * p.stride_tpf;
          const int j = p.stride_past_frames - 1 - p.past_stride * (p.stride_kept_frames - 1 - kk);
          slot = (p.ring_start + j * p.stride_tpf + tok) % p.R;
        } else {
          slot = (p.ring_start + p.stride_past_frames * p.stride_tpf + (x - kept)) % p.R;
        }
      } else {
        slot = p.ring_start + x;
        if (slot >= p.R) slot -= p.R;
      }
      DSC_ASSERT(slot >= 0 && slot < p.R, "simt ring slot");
      kr = RK + (head_row * p.Rp + slot) * D; vr = RV + (head_row * p.Rp + slot) * D;
      if (dbg_keys && lane == 0) dbgp[p.dbg_A + slot] = L;
    } else {
      const int j = L - p.A - p.ring_count;
      DSC_ASSERT(j < p.n_self, "simt self row");
      kr = XK + (((long long)pp * p.n_self + j) * p.Hkv + g) * D;
      vr = XV + (((long long)pp * p.n_self + j) * p.Hkv + g) * D;
      if (dbg_keys && lane == 0) dbgp[p.dbg_A + p.dbg_R + j] = L;
    }
    float kx[E], vx[E];
#pragma unroll
    for (int k = 0; k < E; ++k) {
      const int e = elem_of<D>(lane, k, p.rope_style);
      kx[k] = to_f(kr[e]);
      vx[k] = to_f(vr[e]);
    }
    rotate<D>(kx, p.rope, L, lane, p.rope_style);
    float dot = 0.f;
#pragma unroll
    for (int k = 0; k < E; ++k) dot = fmaf(q[k], kx[k], dot);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    const float sc = dot * scale;
    const float mn = fmaxf(m, sc);
    const float corr = expf(m - mn);
    const float pw = expf(sc - mn);
    lsum = lsum * corr + pw;
#pragma unroll
    for (int k = 0; k < E; ++k) acc[k] = fmaf(acc[k], corr, pw * vx[k]);
    m = mn;
  }
  const float inv = lsum > 0.f ? 1.f / lsum : 0.f;
  int oi = i + p.o_rot;
  if (p.o_rows > 0 && oi >= p.o_rows) oi -= p.o_rows;
  T* orow = reinterpret_cast<T*>(p.o) + (((long long)pp * (p.o_rows > 0 ? p.o_rows : p.n_q) + oi) * p.Hq + h) * D;
#pragma unroll
  for (int k = 0; k < E; ++k) orow[elem_of<D>(lane, k, p.rope_style)] = from_f<T>(acc[k] * inv);
}

cudaError_t launch_attn_simt(const AttnParams& p, cudaStream_t st) {
  const long long warps = (long long)p.P * p.n_q * p.Hq;
  const int blocks = (int)((warps + 3) / 4);
  if (p.dtype == 1) {
    if (p.d == 64) attn_simt_kernel<float, 64><<<blocks, 128, 0, st>>>(p);
    else attn_simt_kernel<float, 128><<<blocks, 128, 0, st>>>(p);
  } else {
    if (p.d == 64) attn_simt_kernel<__nv_bfloat16, 64><<<blocks, 128, 0, st>>>(p);
    else attn_simt_kernel<__nv_bfloat16, 128><<<blocks, 128, 0, st>>>(p);
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------ K5 split-KV combine
// O = sum_s 2^(lse_s - M) O_s / sum_s 2^(lse_s - M), M = max_s lse_s (log2 domain).
// One warp per output row; lanes own 4 consecutive features (d = 128).
__global__ void __launch_bounds__(128) combine_kernel(AttnParams p) {
  const int lane = threadIdx.x & 31;
  const long long row = blockIdx.x * 4ll + (threadIdx.x >> 5);
  const long long rows = (long long)p.P * p.n_q * p.Hq;
  if (row >= rows) return;
  float M = -INFINITY;
  for (int s = 0; s < p.n_splits; ++s) M = fmaxf(M, p.ws_lse[s * rows + row]);
  float den = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int s = 0; s < p.n_splits; ++s) {
    const float lse = p.ws_lse[s * rows + row];
    const float w = (lse == -INFINITY) ? 0.f : exp2f(lse - M);
    den += w;
    const float4 o = reinterpret_cast<const float4*>(p.ws_o + (s * rows + row) * p.d)[lane];
    acc.x = fmaf(w, o.x, acc.x); acc.y = fmaf(w, o.y, acc.y);
    acc.z = fmaf(w, o.z, acc.z); acc.w = fmaf(w, o.w, acc.w);
  }
  const float inv = den > 0.f ? 1.f / den : 0.f;
  __nv_bfloat162 a = __floats2bfloat162_rn(acc.x * inv, acc.y * inv);
  __nv_bfloat162 b = __floats2bfloat162_rn(acc.z * inv, acc.w * inv);
  uint2 out;
  out.x = *reinterpret_cast<uint32_t*>(&a);
  out.y = *reinterpret_cast<uint32_t*>(&b);
  if (p.n_peers > 0) {   // fused all-gather epilogue: row (pp, i, h) to every peer at head o_head_off + h
    const long long h = row % p.Hq, pi = row / p.Hq;
    const long long prow = pi * p.o_hq + p.o_head_off + h;
    for (int r = 0; r < p.n_peers; ++r)
      reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(p.peer_o[r]) + prow * p.d)[lane] = out;
    return;
  }
  reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(p.o) + row * p.d)[lane] = out;
}

cudaError_t launch_combine_partials(int n, long long rows, int d, const float* o_parts, const float* lse, void* o,
                                    cudaStream_t st) {
  AttnParams p{};
  p.P = 1; p.n_q = (int)rows; p.Hq = 1; p.d = d; p.n_splits = n;
  p.ws_o = const_cast<float*>(o_parts); p.ws_lse = const_cast<float*>(lse); p.o = o;
  return launch_combine(p, st);
}

cudaError_t launch_combine(const AttnParams& p, cudaStream_t st) {
  const long long rows = (long long)p.P * p.n_q * p.Hq;
  combine_kernel<<<(int)((rows + 3) / 4), 128, 0, st>>>(p);
  return cudaGetLastError();
}

}  // namespace dsc
