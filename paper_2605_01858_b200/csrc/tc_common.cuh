// Device helpers of the tcgen05 attention kernel (attn_fa.cu): PTX wrappers (mbarrier, TMA,
// tcgen05, cp.async), the work-item decode (also run on the host to build the item tables),
// the key-tile segment map, and the in-place rotate-on-load RoPE of SW128 bf16 tiles.
#pragma once
#include "dscache_internal.h"

#include <cuda_bf16.h>
#include <cstdint>

namespace dsc {
namespace tcc {

constexpr int kMBlockRows = 256;              // query rows (q token x q head) per work item

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred P1;\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P1;\n}\n"
      : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
  return ok != 0;
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// shared-memory matrix descriptor (tcgen05 "matrix descriptor"): start>>4 [0,14),
// LBO>>4 [16,30), SBO>>4 [32,46), version 1 [46,48), base offset 0, swizzle
// mode 2 = 128B [61,64).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
// instruction descriptor, kind::f16: D f32 [4,6)=1, A bf16 [7,10)=1, B bf16 [10,13)=1,
// A major [15], B major [16] (1 = MN-major), N>>3 [17,23), M>>4 [24,29).
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// Warp-converged variants: the whole (MMA) warp executes the call with warp-uniform
// operands and one elected lane issues, so the descriptors stay in uniform registers.
__device__ __forceinline__ void mma_ts_w(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit_w(uint32_t bar) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(bar)
      : "memory");
}
// 32 lanes x 32 consecutive 32-bit columns (thread = lane = row)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ float fmax3f(float a, float b, float c) {
  float m;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(m) : "f"(a), "f"(b), "f"(c));
  return m;
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

__device__ __forceinline__ void stg256(void* p, const uint32_t (&v)[8]) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]),
               "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
#ifndef DSC_ORDER
#define DSC_ORDER 2
#endif
// A work item: (problem = stream x layer, kv head, 256-row m-block of (query, head) rows, key
// split) with its key-tile range.
struct Item {
  int pp, g, mb, sp;
  long long head_row;
  int m0, rows_total;
  int cnt;            // window keys needed by this m-block (causal cut)
  int n_extra;        // leading tiles holding sink + self rows (0 when A + n_self = 0)
  int t_begin, n_tiles;
  // per-launch geometry copied to registers once per item: the tile map below reads no
  // kernel parameters (parameters of a pa/pb-selected launch are indexed constant loads)
  int A, n_self, ring_count, ring_start, R;
  int Rp, staged;     // ring rows per head (R + mirror, or the staging rows); staged build
};

// work item idx -> split fastest, then (DSC_ORDER 2) longest m-block first inside groups of
// DSC_OGRP (problem, kv head) pairs, so a group's staged windows stay in L2 while all its
// m-blocks read them (LPT-like balance of the persistent CTAs with L2 reuse).  Run on the host
// (sched.cu item tables): the kernel reads the decoded records.
template <int BN = kTileN, class PT>
__host__ __device__ __forceinline__ Item decode_item(const PT& p, int idx) {
  Item w;
  const bool one = p.split_only >= 0;          // context-parallel partial: one split per launch
  w.sp = one ? p.split_only : idx % p.n_splits;
  const int rest = one ? idx : idx / p.n_splits;
#if DSC_ORDER == 1   // longest-first across all (problem, head) pairs
  const int ph = rest % (p.P * p.Hkv);
  w.mb = p.n_mblocks - 1 - rest / (p.P * p.Hkv);
#elif DSC_ORDER == 2   // longest-first inside groups of kOrderGroup (problem, head) pairs (L2 reuse)
#ifndef DSC_OGRP
#define DSC_OGRP 37   // v8 (74 clusters): 37 measured c3 +1.5 % vs 74, c5 / c2 / c4 within noise, 148 -1 to -2 %
                      // (profiles/r2c/ab_ogrp_stage.txt); v7 (148 CTAs) measured 74 best
#endif
  constexpr int kOrderGroup = DSC_OGRP;
  const int nph = p.P * p.Hkv;
  const int grp0 = rest / (kOrderGroup * p.n_mblocks) * kOrderGroup;   // first pair of this group
  const int gsz = min(kOrderGroup, nph - grp0);
  const int r2 = rest - grp0 * p.n_mblocks;
  const int ph = grp0 + r2 % gsz;
  w.mb = p.n_mblocks - 1 - r2 / gsz;
#else
  w.mb = p.n_mblocks - 1 - rest % p.n_mblocks;
  const int ph = rest / p.n_mblocks;
#endif
  w.g = ph % p.Hkv;
  w.pp = ph / p.Hkv;
  const int s = w.pp / p.layer_count, l = w.pp % p.layer_count;
  w.head_row = ((long long)s * p.N_total + p.layer_begin + l) * p.Hkv + w.g;
  w.rows_total = p.n_q * p.grp;
  w.m0 = w.mb * (kMBlockRows);
  const int last_row = min(w.m0 + kMBlockRows, w.rows_total) - 1;
  const int lim_max = p.q_pos0 + last_row / p.grp;
  w.cnt = min(max(lim_max - p.A + 1, 0), p.ring_count);
  w.A = p.A; w.n_self = p.n_self; w.ring_count = p.ring_count; w.ring_start = p.ring_start; w.R = p.R;
  w.Rp = p.Rp; w.staged = p.staged;
  w.n_extra = (p.A + p.n_self + BN - 1) / BN;
  const int total = w.n_extra + (w.cnt + BN - 1) / BN;
  w.t_begin = min(w.sp * p.tiles_per_split, total);
  w.n_tiles = min(total, w.t_begin + p.tiles_per_split) - w.t_begin;
  return w;
}

// Key rows of tile u (BN = kTileN = 128 keys) as (at most) two segments; key row r of
// segment s has id pos0_s + r.  Tiles u < n_extra hold the sink rows (extra index x = BN u + r
// < A, id x) and then the self rows (A <= x < A + n_self, id ring_count + x).  Tile u >= n_extra
// is the LOGICAL window tile b = u - n_extra: window keys [BN b, BN b + BN), i.e. the ring
// slots (ring_start + BN b + r) mod R, read as one BN-row box from slot0 = (ring_start +
// BN b) mod R -- the ring keeps a mirror of slots [0, kMirror) after slot R - 1, so the box
// never wraps.  Row r is valid iff BN b + r < cnt, with id A + BN b + r.
// `width` = valid rows rounded up to 16: the N of the QK^T MMA and the K of the PV MMA.
struct TileSeg {
  int lo0, hi0, pos0_0;
  int lo1, hi1, pos0_1;
  int slot0;          // first ring slot of a window tile, -1 for sink/self tiles
  int width;
};

template <int BN = kTileN, class PT>
__device__ __forceinline__ TileSeg tile_segments(const PT&, const Item& w, int u) {
  TileSeg t;
  int valid;
  if (u < w.n_extra) {
    const int x0 = BN * u;
    t.lo0 = 0; t.hi0 = min(max(w.A - x0, 0), BN); t.pos0_0 = x0;
    t.lo1 = t.hi0; t.hi1 = min(max(w.A + w.n_self - x0, 0), BN); t.pos0_1 = w.ring_count + x0;
    t.slot0 = -1;
    valid = t.hi1;
  } else {
    const int base = BN * (u - w.n_extra);
    valid = min(w.cnt - base, BN);
    t.lo0 = 0; t.hi0 = valid; t.pos0_0 = w.A + base;
    t.lo1 = 0; t.hi1 = 0; t.pos0_1 = 0;
    int s0 = w.ring_start + base;
    if (s0 >= w.R) s0 -= w.R;
    t.slot0 = s0;
  }
  t.width = (valid + 15) & ~15;
  return t;
}
__device__ __forceinline__ int seg_pos(const TileSeg& t, int r) {
  if (r >= t.lo0 && r < t.hi0) return t.pos0_0 + r;
  if (r >= t.lo1 && r < t.hi1) return t.pos0_1 + r;
  return -1;
}

__device__ __forceinline__ uint4 ldg128(const void* ptr) {
  uint4 r;
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(ptr));
  return r;
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(addr) : "memory");
  return r;
}
__device__ __forceinline__ void sts128(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ float2 bf2(uint32_t w) { return make_float2(bf_lo(w), bf_hi(w)); }
__device__ __forceinline__ uint32_t get_w(const uint4& v, int j) { return j == 0 ? v.x : j == 1 ? v.y : j == 2 ? v.z : v.w; }

// In-place RoPE of 8 rows x 8 frequencies (f = 8*c8 .. 8*c8+7: 16-byte chunk c8 of the
// low and of the high 64-column block) of a SW128 bf16 tile in smem.  Row k gets
// id pos[k] (-1 = clear the row).  All 16 chunks are loaded first (ILP); between
// consecutive ids the (cos, sin) advance by R(theta) (id + 1) or stay (same id),
// any other jump reloads the fp64-built pair table rp[id][32].
template <int NH, int HI>   // NH groups of 4 rows; HI = byte offset of the high (cols 64..127) block
__device__ __forceinline__ void rotate_rows(uint32_t tile, int r0, int c8, const float4* __restrict__ rp,
                                            const float2 (&cth)[4], const float2 (&sth)[4], const int (&pos)[4 * NH],
                                            const float4 (&pre)[4], int pre_pos) {
  // (cs, sn) start at the prefetched table entry of id pre_pos (the first valid row)
  float2 cs[4], sn[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) { cs[j] = make_float2(pre[j].x, pre[j].y); sn[j] = make_float2(pre[j].z, pre[j].w); }
  int prev = pre_pos;
#pragma unroll
  for (int half = 0; half < NH; ++half) {
    uint4 lo[4], hi[4];
    uint32_t addr[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int r = r0 + half * 4 + k;
      addr[k] = tile + r * 128 + ((c8 ^ (r & 7)) << 4);
      lo[k] = lds128(addr[k]);
      hi[k] = lds128(addr[k] + HI);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int pk = pos[half * 4 + k];
      uint4 ylo = make_uint4(0, 0, 0, 0), yhi = make_uint4(0, 0, 0, 0);
      if (pk >= 0) {
        if (pk == prev) {
        } else if (pk == prev + 1) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float2 nc = __ffma2_rn(cs[j], cth[j], __fmul2_rn(make_float2(-sn[j].x, -sn[j].y), sth[j]));
            sn[j] = __ffma2_rn(sn[j], cth[j], __fmul2_rn(cs[j], sth[j]));
            cs[j] = nc;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float4 t = rp[(long long)pk * 32 + 4 * c8 + j];
            cs[j] = make_float2(t.x, t.y);
            sn[j] = make_float2(t.z, t.w);
          }
        }
        prev = pk;
        uint32_t ol[4], oh[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 av = bf2(get_w(lo[k], j)), bv = bf2(get_w(hi[k], j));
          const float2 yl = __ffma2_rn(av, cs[j], __fmul2_rn(make_float2(-bv.x, -bv.y), sn[j]));   // a cos - b sin
          const float2 yh = __ffma2_rn(av, sn[j], __fmul2_rn(bv, cs[j]));                        // a sin + b cos
          ol[j] = pack_bf16(yl.x, yl.y);
          oh[j] = pack_bf16(yh.x, yh.y);
        }
        ylo = make_uint4(ol[0], ol[1], ol[2], ol[3]);
        yhi = make_uint4(oh[0], oh[1], oh[2], oh[3]);
      } else {
        prev = -3;
      }
      sts128(addr[k], ylo);
      sts128(addr[k] + HI, yhi);
    }
  }
}

// rotate_rows for 4 rows r0 .. r0+3 with CONSECUTIVE ids p0 .. p0+3 (a window tile: no
// per-row branches): (cs, sn) start at the table entry of p0 and advance by R(theta) per row
template <int HI>
__device__ __forceinline__ void rotate4_consec(uint32_t tile, int r0, int c8, const float2 (&cth)[4],
                                               const float2 (&sth)[4], const float4 (&pre)[4]) {
  float2 cs[4], sn[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) { cs[j] = make_float2(pre[j].x, pre[j].y); sn[j] = make_float2(pre[j].z, pre[j].w); }
  uint4 lo[4], hi[4];
  uint32_t addr[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int r = r0 + k;
    addr[k] = tile + r * 128 + ((c8 ^ (r & 7)) << 4);
    lo[k] = lds128(addr[k]);
    hi[k] = lds128(addr[k] + HI);
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (k > 0) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 nc = __ffma2_rn(cs[j], cth[j], __fmul2_rn(make_float2(-sn[j].x, -sn[j].y), sth[j]));
        sn[j] = __ffma2_rn(sn[j], cth[j], __fmul2_rn(cs[j], sth[j]));
        cs[j] = nc;
      }
    }
    uint32_t ol[4], oh[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 av = bf2(get_w(lo[k], j)), bv = bf2(get_w(hi[k], j));
      const float2 yl = __ffma2_rn(av, cs[j], __fmul2_rn(make_float2(-bv.x, -bv.y), sn[j]));   // a cos - b sin
      const float2 yh = __ffma2_rn(av, sn[j], __fmul2_rn(bv, cs[j]));                        // a sin + b cos
      ol[j] = pack_bf16(yl.x, yl.y);
      oh[j] = pack_bf16(yh.x, yh.y);
    }
    sts128(addr[k], make_uint4(ol[0], ol[1], ol[2], ol[3]));
    sts128(addr[k] + HI, make_uint4(oh[0], oh[1], oh[2], oh[3]));
  }
}

}  // namespace tcc
}  // namespace dsc
