// Memory-bound decode attention ("autoregressive decoding is
// performed using the KV cache C_{t+1}"), with the optional 0.5-FPS sampling of the
// cumulative cache during decoding (zeta_decode; reading Q24).
//
// One CTA = one (problem, kv head, key split); its n_q * grp <= 16 query rows (every q head
// of the GQA group, every query token) form ONE m16 tile, so each K/V byte is read from HBM
// once per kv head and feeds all grp q heads.  The key range is cut into 16-key warp tiles;
// each of the 8 warps streams its own tiles through a private 3-stage cp.async ring
// (8 KB per stage: 16 rows of K and of V, 16-byte chunks XOR-swizzled by row), so the main
// loop has no CTA-wide barrier.  Per warp tile:
//   * K is rotated by R(j), j = key - n0 (0..15), in the mma B fragments (registers), from
//     a 16-row table slice that stays in L1;
//   * the queries are rotated by R(m - n0) straight into mma.sync A fragments, so
//     (R(m - n0) q) . (R(j) k) = (R(m) q) . (R(n0 + j) k) -- the use-time RoPE of
//     Def. 4.1 without a per-key trip to the full position table;
//   * S = Q K^T (16 x 16 x 128) and O += P V (16 x 128 x 16) on mma.sync.m16n8k16 bf16 with
//     fp32 accumulation (the work is a 16-row GEMV pair, HBM-bound; tcgen05's 128-row M
//     would be 7/128 used at n_q = 1), online softmax in the log2 domain per warp.
// The 8 warps' (m, l, O) merge in shared memory; with several key splits the CTAs write
// normalised partials + log2-sum-exp and the LAST CTA of the (problem, kv head) -- an
// atomic ticket -- merges them, so a decode step is one launch.
#include <cuda_bf16.h>
#include <cstdint>

#include "dscache_internal.h"

namespace dsc {
namespace {

constexpr int kWarps = 8;
constexpr int kKeys = 16;                        // keys per warp tile
constexpr int kStages = 3;
constexpr int kRowBytes = 256;                   // d = 128 bf16
constexpr int kTabBytes = 2 * 512;               // RoPE rows R(m - n0) of query tokens 0, 1
constexpr int kStageBytes = 2 * kKeys * kRowBytes + kTabBytes;   // K, V, then the q table rows
constexpr int kWarpBytes = kStages * kStageBytes;
constexpr int kSmemBytes = kWarps * kWarpBytes;      // 216 KB; the merge reuses it

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void cp16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void ldsm4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void ldsm4t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
               "{%0,%1,%2,%3};"
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pk(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float2 unpk(uint32_t w) {
  return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u));
}
// byte offset of 16-byte chunk c of row r inside a [16][256 B] tile (chunk XOR row swizzle:
// the 8 rows an ldmatrix phase reads land in 8 distinct bank groups)
__device__ __forceinline__ uint32_t swz(int r, int c) { return (uint32_t)(r * kRowBytes + ((c ^ (r & 7)) << 4)); }

// source row of logical key x of (problem pp, head row hr): [sink | kept past | instant | self]
__device__ __forceinline__ long long key_row(const DecodeParams& p, int pp, long long hr, int g, int x, int& kind,
                                             int& slot) {
  if (x < p.A) { kind = 0; slot = x; return hr * p.A + x; }
  x -= p.A;
  const int past = p.kept_frames * p.tpf;
  if (x < past + p.inst_count) {
    int off;
    if (p.stride == 1 || x >= past) {
      // every past frame kept: past and instant are one contiguous ring run from past_start
      off = x < past ? p.past_start + x : p.inst_start + (x - past);
    } else {
      const int kk = x / p.tpf, tok = x - kk * p.tpf;
      const int j = p.past_frames - 1 - p.stride * (p.kept_frames - 1 - kk);
      off = p.past_start + j * p.tpf + tok;
    }
    if (off >= p.R) off -= p.R;                    // off < 2R: start < R, run length <= R
    kind = 1; slot = off;
    return hr * p.Rp + off;
  }
  x -= past + p.inst_count;
  kind = 2; slot = x;
  return ((long long)pp * p.n_self + x) * p.Hkv + g;
}

__global__ void __launch_bounds__(kWarps * 32, 1) decode_kernel(const DecodeParams p) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int split = blockIdx.x % p.n_splits;
  const int unit = blockIdx.x / p.n_splits;
  const int g = unit % p.Hkv, pp = unit / p.Hkv;
  const int s = pp / p.layer_count, l = pp % p.layer_count;
  const long long hr = ((long long)s * p.N_total + p.layer_begin + l) * p.Hkv + g;   // head row
  const __nv_bfloat16* Q = reinterpret_cast<const __nv_bfloat16*>(p.q);
  const int rows = p.n_q * p.grp;                 // <= 16
  const int wt_total = (p.n_keys + kKeys - 1) / kKeys;
  const int wt0 = split * p.wtiles_per_split;
  const int wt1 = min(wt_total, wt0 + p.wtiles_per_split);
  int* const dbgp = (p.dbg_pos && g == 0) ? p.dbg_pos + (hr / p.Hkv) * p.dbg_len : nullptr;

  // raw queries of this lane's fragment rows (g8 = lane/4 and g8 + 8), k-step kk dims
  // 16kk + {2t, 2t+1, 2t+8, 2t+9}; row r = qi * grp + hh
  const int g8 = lane >> 2, t4 = lane & 3;
  float qf[2][8][4];
  int qpos[2], qrow[2];   // query id and query token index of the lane's two fragment rows
#pragma unroll
  for (int h2 = 0; h2 < 2; ++h2) {
    const int r = g8 + 8 * h2;
    const bool valid = r < rows;
    const int qi = valid ? r / p.grp : 0, hh = valid ? r % p.grp : 0;
    qpos[h2] = valid ? p.q_pos0 + qi : -1;
    qrow[h2] = qi;
    const __nv_bfloat16* qr = Q + (((long long)pp * p.n_q + qi) * p.Hq + g * p.grp + hh) * 128;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const float2 a = valid ? unpk(*reinterpret_cast<const uint32_t*>(qr + 16 * kk + 2 * t4)) : make_float2(0.f, 0.f);
      const float2 b = valid ? unpk(*reinterpret_cast<const uint32_t*>(qr + 16 * kk + 2 * t4 + 8)) : make_float2(0.f, 0.f);
      qf[h2][kk][0] = a.x; qf[h2][kk][1] = a.y; qf[h2][kk][2] = b.x; qf[h2][kk][3] = b.y;
    }
  }
  const bool two_halves = rows > 8;
  if (dbgp && split == 0 && warp == 0 && lane < p.n_q) dbgp[p.dbg_A + p.dbg_R + p.dbg_M + lane] = p.q_pos0 + lane;

  // per-warp cp.async ring: lanes 2r, 2r+1 load key r of the warp tile, lane parity picking
  // the even / odd 16-byte chunks, so each copy instruction covers whole 32-byte sectors of
  // 16 rows; one source-row lookup per lane per tile
  unsigned char* wbuf = smem + warp * kWarpBytes;
  const uint32_t wbase = smem_u32(wbuf);
  const __nv_bfloat16* SK = reinterpret_cast<const __nv_bfloat16*>(p.sink_k);
  const __nv_bfloat16* SV = reinterpret_cast<const __nv_bfloat16*>(p.sink_v);
  const __nv_bfloat16* RK = reinterpret_cast<const __nv_bfloat16*>(p.ring_k);
  const __nv_bfloat16* RV = reinterpret_cast<const __nv_bfloat16*>(p.ring_v);
  const __nv_bfloat16* XK = reinterpret_cast<const __nv_bfloat16*>(p.self_k);
  const __nv_bfloat16* XV = reinterpret_cast<const __nv_bfloat16*>(p.self_v);
  const int lr = lane >> 1, lhalf = lane & 1;
  auto issue = [&](int it, int stage) {
    const int wt = wt0 + warp + it * kWarps;
    if (wt < wt1) {
      const uint32_t sb = wbase + stage * kStageBytes;
      const int x = wt * kKeys + lr;
      const bool valid = x < p.n_keys;
      int kind = 0, slot = 0;
      const long long row = valid ? key_row(p, pp, hr, g, x, kind, slot) : 0;
      const __nv_bfloat16* ks = (kind == 0 ? SK : kind == 1 ? RK : XK) + row * 128;
      const __nv_bfloat16* vs = (kind == 0 ? SV : kind == 1 ? RV : XV) + row * 128;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int c = 2 * j + lhalf;
        cp16(sb + swz(lr, c), ks + 8 * c, valid);
        cp16(sb + kKeys * kRowBytes + swz(lr, c), vs + 8 * c, valid);
      }
      if (dbgp && valid && lhalf == 0)
        dbgp[kind == 0 ? slot : kind == 1 ? p.dbg_A + slot : p.dbg_A + p.dbg_R + slot] = x;
      // the table rows that rotate query tokens 0 and 1 for this tile, prefetched with it
#pragma unroll
      for (int qd = 0; qd < 2; ++qd)
        if (qd < p.n_q) {
          const int delta = max(p.q_pos0 + qd - wt * kKeys, 0);
          cp16(sb + 2 * kKeys * kRowBytes + qd * 512 + lane * 16, p.rope_pairs + (long long)delta * 32 + lane, true);
        }
    }
    cp_commit();   // possibly empty: keeps the group count uniform
  };

  float o[16][4];
#pragma unroll
  for (int n = 0; n < 16; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};

  const int my_tiles = wt1 - wt0 > warp ? (wt1 - wt0 - warp + kWarps - 1) / kWarps : 0;
#pragma unroll 1
  for (int i = 0; i < kStages - 1; ++i) issue(i, i);
  for (int it = 0; it < my_tiles; ++it) {
    issue(it + kStages - 1, (it + kStages - 1) % kStages);
    cp_wait<kStages - 1>();
    __syncwarp();
    const int stage = it % kStages;
    const uint32_t kb = wbase + stage * kStageBytes, vb = kb + kKeys * kRowBytes;
    const int n0 = (wt0 + warp + it * kWarps) * kKeys;

    // queries rotated by R(m - n0) into A fragments (rows g8, g8 + 8)
    uint32_t a[8][4];
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      if (h2 == 1 && !two_halves) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) a[kk][1] = a[kk][3] = 0u;
        break;
      }
      const int delta = max(qpos[h2] - n0, 0);
      const float4* tb = p.rope_pairs + (long long)delta * 32;
      const float4* ts = reinterpret_cast<const float4*>(wbuf + stage * kStageBytes + 2 * kKeys * kRowBytes +
                                                         qrow[h2] * 512);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {            // dims 16kk + 2t (+8 for hf = 1)
          const float4 cs = qrow[h2] < 2 ? ts[8 * kk + t4 + 4 * hf] : __ldg(tb + 8 * kk + t4 + 4 * hf);
          const float x0 = qf[h2][kk][2 * hf], x1 = qf[h2][kk][2 * hf + 1];
          const float y0 = qf[h2][kk + 4][2 * hf], y1 = qf[h2][kk + 4][2 * hf + 1];
          a[kk][2 * hf + h2] = pk(x0 * cs.x - y0 * cs.z, x1 * cs.y - y1 * cs.w);
          a[kk + 4][2 * hf + h2] = pk(x0 * cs.z + y0 * cs.x, x1 * cs.w + y1 * cs.y);
        }
      }
    }

    // S = Q K^T over the 16 keys (two n8 tiles).  The K B fragments are rotated by R(j) in
    // registers (j = key within the tile: the lane holds keys g8 and 8 + g8, dims
    // 16kk + 8hf + 2t, +1 in k-step kk and their split-half partners + 64 in k-step kk + 4)
    float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
    {
      const int key = (lane & 7) + 8 * (lane >> 4);
      const int hsel = (lane >> 3) & 1;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        uint32_t lo[4], hi[4];
        ldsm4(kb + swz(key, 2 * kk + hsel), lo[0], lo[1], lo[2], lo[3]);
        ldsm4(kb + swz(key, 2 * (kk + 4) + hsel), hi[0], hi[1], hi[2], hi[3]);
#pragma unroll
        for (int e = 0; e < 4; ++e) {   // e = 2 * n-tile + hf
          const float4 cs = __ldg(p.rope_pairs + (8 * (e >> 1) + g8) * 32 + 8 * kk + 4 * (e & 1) + t4);
          const float2 x = unpk(lo[e]), y = unpk(hi[e]);
          lo[e] = pk(x.x * cs.x - y.x * cs.z, x.y * cs.y - y.y * cs.w);
          hi[e] = pk(x.x * cs.z + y.x * cs.x, x.y * cs.w + y.y * cs.y);
        }
        mma16816(sc[0], a[kk], lo[0], lo[1]);
        mma16816(sc[1], a[kk], lo[2], lo[3]);
        mma16816(sc[0], a[kk + 4], hi[0], hi[1]);
        mma16816(sc[1], a[kk + 4], hi[2], hi[3]);
      }
    }
    // mask (beyond the keys, or after the row's own query id: causal inside the self
    // segment), online softmax in the log2 domain
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = n0 + 8 * nt + 2 * t4 + (e & 1);
        const int h2 = e >> 1;
        const bool vis = key < p.n_keys && key <= qpos[h2];
        const float v = vis ? sc[nt][e] * p.scale_log2 : -INFINITY;
        sc[nt][e] = v;
        mx[h2] = fmaxf(mx[h2], v);
      }
    }
    float corr[2], mu[2];
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      mx[h2] = fmaxf(mx[h2], __shfl_xor_sync(0xffffffffu, mx[h2], 1));
      mx[h2] = fmaxf(mx[h2], __shfl_xor_sync(0xffffffffu, mx[h2], 2));
      const float mn = fmaxf(m_run[h2], mx[h2]);
      mu[h2] = mn == -INFINITY ? 0.f : mn;
      corr[h2] = exp2f(m_run[h2] - mu[h2]);
      m_run[h2] = mn;
    }
    uint32_t pa[4];
    {
      float ps[2][4];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) ps[nt][e] = exp2f(sc[nt][e] - mu[e >> 1]);
      l_run[0] = l_run[0] * corr[0] + ps[0][0] + ps[0][1] + ps[1][0] + ps[1][1];
      l_run[1] = l_run[1] * corr[1] + ps[0][2] + ps[0][3] + ps[1][2] + ps[1][3];
      pa[0] = pk(ps[0][0], ps[0][1]);
      pa[1] = pk(ps[0][2], ps[0][3]);
      pa[2] = pk(ps[1][0], ps[1][1]);
      pa[3] = pk(ps[1][2], ps[1][3]);
    }
    // O = O * corr + P V (the rescale is skipped when no row's max moved: corr == 1 exactly)
    const bool rescale = __any_sync(0xffffffffu, corr[0] != 1.f || corr[1] != 1.f);
    {
      const int key = (lane & 7) + 8 * ((lane >> 3) & 1);
      const int csel = lane >> 4;
#pragma unroll
      for (int nt = 0; nt < 16; nt += 2) {
        uint32_t b0, b1, b2, b3;
        ldsm4t(vb + swz(key, nt + csel), b0, b1, b2, b3);
        if (rescale) {
          o[nt][0] *= corr[0]; o[nt][1] *= corr[0]; o[nt][2] *= corr[1]; o[nt][3] *= corr[1];
          o[nt + 1][0] *= corr[0]; o[nt + 1][1] *= corr[0]; o[nt + 1][2] *= corr[1]; o[nt + 1][3] *= corr[1];
        }
        mma16816(o[nt], pa, b0, b1);
        mma16816(o[nt + 1], pa, b2, b3);
      }
    }
    __syncwarp();
  }
  cp_wait<0>();

  // ---- merge the 8 warps: (m, l) per row, each warp's O slice in smem, summed with weights
  l_run[0] += __shfl_xor_sync(0xffffffffu, l_run[0], 1);
  l_run[0] += __shfl_xor_sync(0xffffffffu, l_run[0], 2);
  l_run[1] += __shfl_xor_sync(0xffffffffu, l_run[1], 1);
  l_run[1] += __shfl_xor_sync(0xffffffffu, l_run[1], 2);
  __syncthreads();                                   // every warp is done with its stage buffers
  float* ml = reinterpret_cast<float*>(smem);        // [kWarps][16] m, then [kWarps][16] l
  float* ow = ml + 2 * kWarps * 16;                  // [kWarps][16][128] fp32 per-warp O
  if (t4 == 0) {
    ml[warp * 16 + g8] = m_run[0];
    ml[warp * 16 + g8 + 8] = m_run[1];
    ml[(kWarps + warp) * 16 + g8] = l_run[0];
    ml[(kWarps + warp) * 16 + g8 + 8] = l_run[1];
  }
  {
    float* mine = ow + warp * 16 * 128;
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) {
      const int c = 8 * nt + 2 * t4;
      *reinterpret_cast<float2*>(mine + g8 * 128 + c) = make_float2(o[nt][0], o[nt][1]);
      if (two_halves) *reinterpret_cast<float2*>(mine + (g8 + 8) * 128 + c) = make_float2(o[nt][2], o[nt][3]);
    }
  }
  __syncthreads();
  const int tid = threadIdx.x;
  const long long rows_total = (long long)p.P * p.n_q * p.Hq;
  __nv_bfloat16* O = reinterpret_cast<__nv_bfloat16*>(p.o);
  for (int i = tid; i < rows * 32; i += blockDim.x) {   // 4 dims per thread
    const int r = i >> 5, c = (i & 31) * 4;
    float mm = -INFINITY;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) mm = fmaxf(mm, ml[w * 16 + r]);
    float L = 0.f;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (mm != -INFINITY) {
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        const float wt = exp2f(ml[w * 16 + r] - mm);
        L += ml[(kWarps + w) * 16 + r] * wt;
        const float4 x = *reinterpret_cast<const float4*>(ow + (w * 16 + r) * 128 + c);
        v.x = fmaf(wt, x.x, v.x); v.y = fmaf(wt, x.y, v.y); v.z = fmaf(wt, x.z, v.z); v.w = fmaf(wt, x.w, v.w);
      }
    }
    const float inv = L > 0.f ? 1.f / L : 0.f;
    const int qi = r / p.grp, h = g * p.grp + r % p.grp;
    const long long orow = ((long long)pp * p.n_q + qi) * p.Hq + h;
    if (p.n_splits == 1) {
      uint2 w;
      w.x = pk(v.x * inv, v.y * inv);
      w.y = pk(v.z * inv, v.w * inv);
      *reinterpret_cast<uint2*>(O + orow * 128 + c) = w;
    } else {
      *reinterpret_cast<float4*>(p.ws_o + ((long long)split * rows_total + orow) * 128 + c) =
          make_float4(v.x * inv, v.y * inv, v.z * inv, v.w * inv);
      if (c == 0) p.ws_lse[(long long)split * rows_total + orow] = L > 0.f ? mm + log2f(L) : -INFINITY;
    }
  }
  if (p.n_splits == 1) return;
  // ---- split-KV: the last CTA of this (problem, kv head) merges every split's partial
  __shared__ int last;
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    const int ticket = atomicAdd(p.counters + hr, 1);
    last = ticket == p.n_splits - 1;
    if (last) p.counters[hr] = 0;                   // ready for the next launch (stream-ordered)
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // split weights per row (a warp per row: lanes over splits), then the weighted sum
  float* wsm = ow;                                   // [16][n_splits] normalised weights
  for (int r = warp; r < rows; r += kWarps) {
    const long long orow = ((long long)pp * p.n_q + r / p.grp) * p.Hq + g * p.grp + r % p.grp;
    float mm = -INFINITY;
    for (int sp = lane; sp < p.n_splits; sp += 32) mm = fmaxf(mm, __ldcg(p.ws_lse + (long long)sp * rows_total + orow));
#pragma unroll
    for (int o2 = 16; o2 > 0; o2 >>= 1) mm = fmaxf(mm, __shfl_xor_sync(0xffffffffu, mm, o2));
    float den = 0.f;
    for (int sp = lane; sp < p.n_splits; sp += 32) {
      const float lse = __ldcg(p.ws_lse + (long long)sp * rows_total + orow);
      const float w = lse == -INFINITY ? 0.f : exp2f(lse - mm);
      wsm[r * p.n_splits + sp] = w;
      den += w;
    }
#pragma unroll
    for (int o2 = 16; o2 > 0; o2 >>= 1) den += __shfl_xor_sync(0xffffffffu, den, o2);
    const float inv = den > 0.f ? 1.f / den : 0.f;
    for (int sp = lane; sp < p.n_splits; sp += 32) wsm[r * p.n_splits + sp] *= inv;
  }
  __syncthreads();
  for (int i = tid; i < rows * 32; i += blockDim.x) {
    const int r = i >> 5, c = (i & 31) * 4;
    const long long orow = ((long long)pp * p.n_q + r / p.grp) * p.Hq + g * p.grp + r % p.grp;
    const float* wr = wsm + r * p.n_splits;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 8
    for (int sp = 0; sp < p.n_splits; ++sp) {
      const float w = wr[sp];
      const float4 v = __ldcg(reinterpret_cast<const float4*>(p.ws_o + ((long long)sp * rows_total + orow) * 128 + c));
      acc.x = fmaf(w, v.x, acc.x); acc.y = fmaf(w, v.y, acc.y);
      acc.z = fmaf(w, v.z, acc.z); acc.w = fmaf(w, v.w, acc.w);
    }
    uint2 w;
    w.x = pk(acc.x, acc.y);
    w.y = pk(acc.z, acc.w);
    *reinterpret_cast<uint2*>(O + orow * 128 + c) = w;
  }
}

}  // namespace

cudaError_t launch_decode(const DecodeParams& p, cudaStream_t st) {
  static int configured_mask = 0;   // bit per device (cudaFuncSetAttribute is per device)
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 31 && !(configured_mask & (1 << dev))) {
    cudaError_t e = cudaFuncSetAttribute(decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (e != cudaSuccess) return e;
    configured_mask |= 1 << dev;
  }
  const long long blocks = (long long)p.P * p.Hkv * p.n_splits;
  if (blocks == 0) return cudaSuccess;
  decode_kernel<<<(unsigned)blocks, kWarps * 32, kSmemBytes, st>>>(p);
  return cudaGetLastError();
}

}  // namespace dsc
