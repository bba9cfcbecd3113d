// Memory-bound decode attention ("autoregressive decoding is
// performed using the KV cache C_{t+1}"), with the optional 0.5-FPS sampling of the
// cumulative cache during decoding (zeta_decode; reading Q24).
//
// One CTA = one (problem, kv head, key split); its n_q * grp <= 16 query rows (every q head
// of the GQA group, every query token) form ONE m16 tile, so each K/V byte is read from HBM
// once per kv head and feeds all grp q heads.  The CTA streams 128-key tiles through a
// 3-stage ring (64 KB of K and V per stage in the TMA 128-byte swizzle, plus the two RoPE
// table rows that rotate the queries for that tile, one mbarrier per stage): a tile that is
// one consecutive run of ring slots (the common case) is four TMA boxes; sink / self /
// sampled-past boundary tiles fall back to per-thread cp.async into the same layout.
// Per tile:
//   * the queries are rotated once by R(m - n0) (n0 = the tile's first id) into a shared
//     bf16 tile that every warp reads with ldmatrix;
//   * warp w owns keys 16w .. 16w+15 of the tile and rotates their K by R(j), j = 16w + ..,
//     in its mma B fragments, with the R(j) table held in registers for the whole kernel:
//     (R(m - n0) q) . (R(j) k) = (R(m) q) . (R(n0 + j) k) -- the use-time RoPE of Def. 4.1
//      without any per-key table traffic;
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
constexpr int kWarpKeys = 16;                    // keys of a tile each warp owns
constexpr int kTileKeys = kWarps * kWarpKeys;    // 128 keys per CTA tile
constexpr int kStages = 3;
constexpr int kRowBytes = 256;                   // d = 128 bf16
constexpr int kTabBytes = 2 * 512;               // RoPE rows R(m - n0) of query tokens 0, 1
// stage = K then V, each as two 64-column halves of [128 rows][128 B] in the TMA 128-byte
// swizzle (16-byte chunk c of row r at r*128 + ((c ^ (r & 7)) << 4)), then the table rows
constexpr int kHalfBytes = kTileKeys * 128;
constexpr int kVOff = 2 * kHalfBytes;
constexpr int kTabOff = 4 * kHalfBytes;
constexpr int kStageBytes = kTabOff + kTabBytes;   // 65 KB (a multiple of 1024: SW128 alignment)
constexpr int kQRawOff = kStages * kStageBytes;  // fp32 raw queries [16][128]
constexpr int kQRotOff = kQRawOff + 16 * 128 * 4;   // bf16 rotated queries [16][256 B], swizzled
constexpr int kBarOff = kQRotOff + 16 * kRowBytes;  // one mbarrier per stage
constexpr int kSmemBytes = kBarOff + 64;            // 211 KB; the merge reuses the stages

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void cp16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0) : "memory");
}

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
// byte offset of 16-byte chunk c of row r inside a [rows][256 B] tile (chunk XOR row swizzle:
// the 8 rows an ldmatrix phase reads land in 8 distinct bank groups)
__device__ __forceinline__ uint32_t swz(int r, int c) { return (uint32_t)(r * kRowBytes + ((c ^ (r & 7)) << 4)); }
// byte offset of 16-byte chunk c (0..15) of key row r inside a K or V stage tile (SW128 halves)
__device__ __forceinline__ uint32_t swz2(int r, int c) {
  return (uint32_t)((c >> 3) * kHalfBytes + r * 128 + (((c & 7) ^ (r & 7)) << 4));
}
__device__ __forceinline__ void bar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void bar_arrive_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_cp_arrive(uint32_t bar) {   // arrives once this thread's cp.asyncs land
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void bar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n}\n" ::"r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

// source row of logical key x of (problem pp, head row hr): [sink | kept past | instant | self]
template <bool EXT>
__device__ __forceinline__ long long key_row(const DecodeParams& p, int pp, long long hr, int g, int x, int& kind,
                                             int& slot) {
  if (x < p.A) { kind = 0; slot = x; return hr * p.A + x; }
  x -= p.A;
  const int past = p.kept_frames * p.tpf;
  if (EXT && x >= past && x < past + p.inst_count) {   // real-model mode: caller's instant K/V
    kind = 3; slot = x - past;
    return ((long long)pp * p.inst_count + (x - past)) * p.Hkv + g;
  }
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
    DSC_ASSERT(off >= 0 && off < p.R && (x < past ? (p.stride == 1 || (x / p.tpf) < p.kept_frames) : true),
               "decode ring slot");
    kind = 1; slot = off;
    return hr * p.Rp + off;
  }
  x -= past + p.inst_count;
  kind = 2; slot = x;
  DSC_ASSERT(x < p.n_self && pp < p.P, "decode self row");
  return ((long long)pp * p.n_self + x) * p.Hkv + g;
}

// EXT: real-model mode (the instant keys come from the caller's k_inst, not the ring)
template <bool EXT>
__global__ void __launch_bounds__(kWarps * 32, 1) decode_kernel(const __grid_constant__ DecodeParams p) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int split = blockIdx.x % p.n_splits;
  const int unit = blockIdx.x / p.n_splits;
  const int g = unit % p.Hkv, pp = unit / p.Hkv;
  const int s = pp / p.layer_count, l = pp % p.layer_count;
  const long long hr = ((long long)s * p.N_total + p.layer_begin + l) * p.Hkv + g;   // head row
  const int rows = p.n_q * p.grp;                 // <= 16
  const int tiles = (p.n_keys + kTileKeys - 1) / kTileKeys;
  const int tb0 = split * p.tiles_per_split;
  const int tb1 = min(tiles, tb0 + p.tiles_per_split);
  const int n_my = max(tb1 - tb0, 0);
  int* const dbgp = (p.dbg_pos && g == 0) ? p.dbg_pos + (hr / p.Hkv) * p.dbg_len : nullptr;
  const uint32_t sbase = smem_u32(smem);

  // ---- cp.async producer (all 256 threads): threads 2r, 2r+1 load key r of the tile, the
  // thread parity picking the even / odd 16-byte chunks (whole 32-byte sectors per copy)
  const __nv_bfloat16* SK = reinterpret_cast<const __nv_bfloat16*>(p.sink_k);
  const __nv_bfloat16* SV = reinterpret_cast<const __nv_bfloat16*>(p.sink_v);
  const __nv_bfloat16* RK = reinterpret_cast<const __nv_bfloat16*>(p.ring_k);
  const __nv_bfloat16* RV = reinterpret_cast<const __nv_bfloat16*>(p.ring_v);
  const __nv_bfloat16* XK = reinterpret_cast<const __nv_bfloat16*>(p.self_k);
  const __nv_bfloat16* XV = reinterpret_cast<const __nv_bfloat16*>(p.self_v);
  const __nv_bfloat16* IK = reinterpret_cast<const __nv_bfloat16*>(p.inst_k);
  const __nv_bfloat16* IV = reinterpret_cast<const __nv_bfloat16*>(p.inst_v);
  const int lr = tid >> 1, lhalf = tid & 1;
  // ring keys [ring0, ring1): kept past then instant, slots consecutive from past_start when
  // every past frame is kept (stride 1); with a stride, runs inside one kept frame or inside
  // the instant window are consecutive
  const int ring0 = p.A, past_end = p.A + p.kept_frames * p.tpf;
  const int ring1 = past_end + (EXT ? 0 : p.inst_count);   // real-model mode: instant not in the ring
  const int n_tab = min(p.n_q, 2);
  if (tid < kStages) bar_init(sbase + kBarOff + 8 * tid, kWarps * 32 + 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  auto issue = [&](int it) {
    if (it >= n_my) return;
    const int tile = tb0 + it;
    const int stage = it % kStages;
    const uint32_t sb = sbase + stage * kStageBytes;
    const uint32_t bar = sbase + kBarOff + 8 * stage;
    const int n0 = tile * kTileKeys, n1 = n0 + kTileKeys - 1;
    bool tma = n0 >= ring0 && n1 < ring1;
    if (tma && p.stride != 1 && n0 < past_end)
      tma = n1 < past_end && (n0 - p.A) / p.tpf == (n1 - p.A) / p.tpf;
    // query tokens 0 and 1's rotation rows R(m - n0): one bulk copy (rows base, base + 1; the
    // rows of a query token before the tile are never used: all its keys here are masked)
    const int base = p.q_pos0 - n0;
    const uint32_t tab_bytes = base >= 0 ? n_tab * 512 : 512;
    if (tma) {
      int kind = 0, slot = 0;
      const long long row0 = key_row<EXT>(p, pp, hr, g, n0, kind, slot);
      DSC_ASSERT(kind == 1 && slot + kTileKeys <= p.Rp, "decode TMA box rows");
      if (tid == 0) {
        bar_arrive_tx(bar, 4 * kHalfBytes + tab_bytes);
        tma2d(sb, &p.tmap_k, 0, (int)row0, bar);
        tma2d(sb + kHalfBytes, &p.tmap_k, 64, (int)row0, bar);
        tma2d(sb + kVOff, &p.tmap_v, 0, (int)row0, bar);
        tma2d(sb + kVOff + kHalfBytes, &p.tmap_v, 64, (int)row0, bar);
        if (base >= 0) bulk_g2s(sb + kTabOff, p.rope_pairs + (long long)base * 32, tab_bytes, bar);
        else bulk_g2s(sb + kTabOff + 512, p.rope_pairs, 512, bar);
      }
      bar_arrive(bar);
      if (dbgp && lhalf == 0) {
        int sl = slot + lr;
        if (sl >= p.R) sl -= p.R;
        dbgp[p.dbg_A + sl] = n0 + lr;
      }
    } else {
      const int x = n0 + lr;
      const bool valid = x < p.n_keys;
      int kind = 0, slot = 0;
      const long long row = valid ? key_row<EXT>(p, pp, hr, g, x, kind, slot) : 0;
      const __nv_bfloat16* ks = (kind == 0 ? SK : kind == 1 ? RK : (!EXT || kind == 2) ? XK : IK) + row * 128;
      const __nv_bfloat16* vs = (kind == 0 ? SV : kind == 1 ? RV : (!EXT || kind == 2) ? XV : IV) + row * 128;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int c = 2 * j + lhalf;
        cp16(sb + swz2(lr, c), ks + 8 * c, valid);
        cp16(sb + kVOff + swz2(lr, c), vs + 8 * c, valid);
      }
      if (tid == 0) {
        bar_arrive_tx(bar, tab_bytes);
        if (base >= 0) bulk_g2s(sb + kTabOff, p.rope_pairs + (long long)base * 32, tab_bytes, bar);
        else bulk_g2s(sb + kTabOff + 512, p.rope_pairs, 512, bar);
      }
      bar_cp_arrive(bar);
      if (dbgp && valid && lhalf == 0 && (!EXT || kind != 3))
        dbgp[kind == 0 ? slot : kind == 1 ? p.dbg_A + slot : p.dbg_A + p.dbg_R + slot] = x;
    }
  };
#pragma unroll 1
  for (int i = 0; i < kStages - 1; ++i) issue(i);

  // ---- raw queries (fp32, smem) and the rotated-query tile (zero rows beyond `rows`)
  float* qraw = reinterpret_cast<float*>(smem + kQRawOff);
  unsigned char* qrot = smem + kQRotOff;
  const __nv_bfloat16* Q = reinterpret_cast<const __nv_bfloat16*>(p.q);
  {   // one 16-byte load per thread: row tid / 16, dims 8 * (tid % 16) ..
    const int r = tid >> 4, c = (tid & 15) * 8;
    uint4 w = make_uint4(0, 0, 0, 0);
    if (r < rows) {
      const int qi = r / p.grp, hh = r % p.grp;
      w = __ldg(reinterpret_cast<const uint4*>(Q + (((long long)pp * p.n_q + qi) * p.Hq + g * p.grp + hh) * 128 + c));
    }
    const float2 a = unpk(w.x), b = unpk(w.y), e = unpk(w.z), f = unpk(w.w);
    *reinterpret_cast<float4*>(qraw + r * 128 + c) = make_float4(a.x, a.y, b.x, b.y);
    *reinterpret_cast<float4*>(qraw + r * 128 + c + 4) = make_float4(e.x, e.y, f.x, f.y);
  }
  for (int i = tid; i < 16 * kRowBytes / 16; i += blockDim.x) reinterpret_cast<uint4*>(qrot)[i] = make_uint4(0, 0, 0, 0);
  if (dbgp && split == 0 && tid < p.n_q) dbgp[p.dbg_A + p.dbg_R + p.dbg_M + tid] = p.q_pos0 + tid;

  // ---- per-lane constants: fragment rows g8, g8 + 8 (their query ids), and the R(j) table
  // of the lane's two keys (j = 16 warp + g8 (+8)) at its 16 frequencies f = 16kk + 8hf + 2t
  const int g8 = lane >> 2, t4 = lane & 3;
  int qpos[2];
#pragma unroll
  for (int h2 = 0; h2 < 2; ++h2) {
    const int r = g8 + 8 * h2;
    qpos[h2] = r < rows ? p.q_pos0 + r / p.grp : -1;
  }
  float4 kt[4][4];
#pragma unroll
  for (int kk = 0; kk < 4; ++kk)
#pragma unroll
    for (int e = 0; e < 4; ++e)
      kt[kk][e] = __ldg(p.rope_pairs + (kWarpKeys * warp + 8 * (e >> 1) + g8) * 32 + 8 * kk + 4 * (e & 1) + t4);

  float o[16][4];
#pragma unroll
  for (int n = 0; n < 16; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};
  // q rotation work of this thread: row qr_r, frequencies qr_f .. qr_f + 3
  const int qr_r = tid >> 4, qr_f = (tid & 15) * 4;

  for (int it = 0; it < n_my; ++it) {
    const int stage = it % kStages;
    bar_wait(sbase + kBarOff + 8 * stage, (it / kStages) & 1);   // tile it landed (TMA or cp.async)
    __syncthreads();                   // every warp is done with tile it-1
    issue(it + kStages - 1);           // into the stage tile it-1 used
    const uint32_t kb = sbase + stage * kStageBytes, vb = kb + kVOff;
    const int n0 = (tb0 + it) * kTileKeys;

    // queries rotated by R(m - n0) (bf16, swizzled), shared by the 8 warps
    if (qr_r < rows) {
      const int qi = qr_r / p.grp;
      const float4* ts;
      if (qi < 2) {
        ts = reinterpret_cast<const float4*>(smem + stage * kStageBytes + kTabOff + qi * 512);
      } else {
        ts = p.rope_pairs + (long long)max(p.q_pos0 + qi - n0, 0) * 32;
      }
      const float4 c0 = ts[qr_f / 2], c1 = ts[qr_f / 2 + 1];
      const float4 x = *reinterpret_cast<const float4*>(qraw + qr_r * 128 + qr_f);
      const float4 y = *reinterpret_cast<const float4*>(qraw + qr_r * 128 + 64 + qr_f);
      uint2 lo, hi;
      lo.x = pk(x.x * c0.x - y.x * c0.z, x.y * c0.y - y.y * c0.w);
      lo.y = pk(x.z * c1.x - y.z * c1.z, x.w * c1.y - y.w * c1.w);
      hi.x = pk(x.x * c0.z + y.x * c0.x, x.y * c0.w + y.y * c0.y);
      hi.y = pk(x.z * c1.z + y.z * c1.x, x.w * c1.w + y.w * c1.y);
      *reinterpret_cast<uint2*>(qrot + swz(qr_r, qr_f >> 3) + (qr_f & 7) * 2) = lo;
      *reinterpret_cast<uint2*>(qrot + swz(qr_r, 8 + (qr_f >> 3)) + (qr_f & 7) * 2) = hi;
    }
    __syncthreads();                   // rotated queries ready

    // S = Q K^T over this warp's 16 keys; K B fragments rotated by R(j) in registers (the lane
    // holds keys g8, 8 + g8 at dims 16kk + 8hf + 2t, +1 and their partners + 64 in kk + 4)
    float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
    {
      const uint32_t qb = sbase + kQRotOff;
      const int arow = (lane & 7) + 8 * ((lane >> 3) & 1), asel = lane >> 4;
      const int key = kWarpKeys * warp + (lane & 7) + 8 * (lane >> 4);
      const int hsel = (lane >> 3) & 1;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        uint32_t a0[4], a1[4], lo[4], hi[4];
        ldsm4(qb + swz(arow, 2 * kk + asel), a0[0], a0[1], a0[2], a0[3]);
        ldsm4(qb + swz(arow, 2 * (kk + 4) + asel), a1[0], a1[1], a1[2], a1[3]);
        ldsm4(kb + swz2(key, 2 * kk + hsel), lo[0], lo[1], lo[2], lo[3]);
        ldsm4(kb + swz2(key, 2 * (kk + 4) + hsel), hi[0], hi[1], hi[2], hi[3]);
#pragma unroll
        for (int e = 0; e < 4; ++e) {   // e = 2 * n-tile + hf
          const float4 cs = kt[kk][e];
          const float2 x = unpk(lo[e]), y = unpk(hi[e]);
          lo[e] = pk(x.x * cs.x - y.x * cs.z, x.y * cs.y - y.y * cs.w);
          hi[e] = pk(x.x * cs.z + y.x * cs.x, x.y * cs.w + y.y * cs.y);
        }
        mma16816(sc[0], a0, lo[0], lo[1]);
        mma16816(sc[1], a0, lo[2], lo[3]);
        mma16816(sc[0], a1, hi[0], hi[1]);
        mma16816(sc[1], a1, hi[2], hi[3]);
      }
    }
    // mask (beyond the keys, or after the row's own query id: causal inside the self
    // segment), online softmax in the log2 domain
    const int kbase = n0 + kWarpKeys * warp + 2 * t4;
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = kbase + 8 * nt + (e & 1);
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
      const int key = kWarpKeys * warp + (lane & 7) + 8 * ((lane >> 3) & 1);
      const int csel = lane >> 4;
#pragma unroll
      for (int nt = 0; nt < 16; nt += 2) {
        uint32_t b0, b1, b2, b3;
        ldsm4t(vb + swz2(key, nt + csel), b0, b1, b2, b3);
        if (rescale) {
          o[nt][0] *= corr[0]; o[nt][1] *= corr[0]; o[nt][2] *= corr[1]; o[nt][3] *= corr[1];
          o[nt + 1][0] *= corr[0]; o[nt + 1][1] *= corr[0]; o[nt + 1][2] *= corr[1]; o[nt + 1][3] *= corr[1];
        }
        mma16816(o[nt], pa, b0, b1);
        mma16816(o[nt + 1], pa, b2, b3);
      }
    }
  }
  const bool two_halves = rows > 8;

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
    DSC_ASSERT(qi < p.n_q && h < p.Hq && orow < rows_total && split < p.n_splits, "decode O / partial row");
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
    const int ticket = atomicAdd(p.counters + unit, 1);   // this call's zeroed ticket of (problem, kv head)
    last = ticket == p.n_splits - 1;
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
    cudaError_t e = cudaFuncSetAttribute(decode_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(decode_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (e != cudaSuccess) return e;
    configured_mask |= 1 << dev;
  }
  const long long blocks = (long long)p.P * p.Hkv * p.n_splits;
  if (blocks == 0) return cudaSuccess;
  if (p.inst_k != nullptr) decode_kernel<true><<<(unsigned)blocks, kWarps * 32, kSmemBytes, st>>>(p);
  else decode_kernel<false><<<(unsigned)blocks, kWarps * 32, kSmemBytes, st>>>(p);
  return cudaGetLastError();
}

}  // namespace dsc
