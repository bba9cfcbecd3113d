// K3/K4 v6: fused rotate-on-load RoPE + GQA flash attention on the sm_100a tensor cores
// with the Q tiles resident in TMEM.  Same work items, key tiles, softmax and staged build
// as attn_tc.cu (v5); what changes is where the operands live:
//
//   * Q of both 128-row Q tiles sits in TMEM (bf16x2, 64 columns each) and S = Q K^T is a
//     TS MMA (A from TMEM, B = the K tile in smem).  The SS form re-read the 32 KB Q tile
//     from shared memory for every 64-key tile (4 KB per K16 step, which made the N = 64
//     MMA shared-memory-bound at 48 instead of 32 clk); now only K and V are read from smem.
//   * Shared memory holds only K / V stages: 7 + 7 stages of 16 KB.
//   * TMEM (512 cols): S[qt] = qt*64 (64 cols, P overwrites its first 32), Q[qt] = 128 +
//     qt*64, O[qt] = 256 + qt*128.  S is single-buffered per Q tile: S(g+1) is issued right
//     after PV(g) consumed P(g); the two Q tiles alternate on the tensor core.
//   * The rotation warpgroup writes Q: thread r loads row r of each Q tile (256 B), rotates
//     the split-half pairs at the query id in registers and stores the row to its TMEM lane
//     (tcgen05.st), once the previous item's last QK^T MMA has been committed (B_QE).
//
// Position-agnostic encoding (Def. 4.1): raw K in the ring, rotated at
// its use-time id in shared memory (attend) or once per step in the staging
// buffer (build); softmax(Q K^T / sqrt(d)) V, exp2 domain, lazy rescale.
//
// CTA = 16 warps: 0-3 softmax of Q tile 0, 4-7 softmax of Q tile 1, 8-11 rotation (K tiles
// of attend items, Q rows of every item), 12 K copy, 13 V copy, 14 TMEM alloc + MMA issuer,
// 15 idle.  setmaxnreg: softmax 144, rotation 136, copy/MMA 88.
#include "tc_common.cuh"

namespace dsc {
namespace tc6 {
using namespace tcc;

constexpr int kWarps = 16;
constexpr int kThreads = kWarps * 32;
constexpr int kKT = kTileN;                   // keys per K/V tile (64)
constexpr int kKVHalf = kKT * 128;            // one 64-column SW128 block of a K/V tile
constexpr int kKVBytes = 2 * kKVHalf;         // 16 KB
#ifndef DSC6_KST
#define DSC6_KST 7
#endif
#ifndef DSC6_VST
#define DSC6_VST 7
#endif
constexpr int KST = DSC6_KST, VST = DSC6_VST;
constexpr int OFF_K = 0;
constexpr int OFF_V = OFF_K + KST * kKVBytes;
constexpr int OFF_BAR = OFF_V + VST * kKVBytes;
// barriers: Q ready [qt] | Q free | K landed | K rotated | K free | V landed | V free |
// S ready [qt] | P ready [qt] | PV done [qt] | O read [qt]
constexpr int B_Q = 0, B_QE = 2, B_KR = 3, B_KF = B_KR + KST, B_KE = B_KF + KST, B_VF = B_KE + KST,
              B_VE = B_VF + VST, B_S = B_VE + VST, B_P = B_S + 2, B_O = B_P + 2, B_OF = B_O + 2, B_N = B_OF + 2;
constexpr int kRegSoftmax = 144, kRegRotate = 136, kRegCopy = 88;
static_assert(2 * kRegSoftmax + kRegRotate + kRegCopy <= 512, "setmaxnreg budget");
constexpr int kThreadRegs = 65536 / kThreads;
constexpr int kSmemBytes = OFF_BAR + B_N * 8 + 16 + 1024;
static_assert(kSmemBytes <= 227 * 1024, "shared memory budget");
static_assert(kKT == 64, "64-key tiles");
constexpr float kRescaleThreshold = 8.0f;
constexpr uint32_t TC_S = 0, TC_Q = 128, TC_O = 256;   // TMEM column bases

// Q row `rloc` of Q tile qt of item w, rotated at its query id, stored to TMEM lane rloc
// (columns TC_Q + qt*64 .. +63, bf16x2); zeros for padding rows.  Executed by the thread
// whose warp owns that lane quarter (warp % 4 == rloc / 32).
__device__ __forceinline__ void q_row_to_tmem(const AttnParams& p, const Item& w, int qt, int rloc, uint32_t taddr) {
  const int rglob = w.m0 + qt * 128 + rloc;
  const bool ok = rglob < w.rows_total;
  const int qi = ok ? rglob / p.grp : 0, hh = ok ? rglob % p.grp : 0;
  const int pos = p.q_pos0 + qi;
  const uint4* __restrict__ src = reinterpret_cast<const uint4*>(
      reinterpret_cast<const __nv_bfloat16*>(p.q) + (((long long)w.pp * p.n_q + qi) * p.Hq + w.g * p.grp + hh) * 128);
  const float4* __restrict__ tab = p.rope_pairs + (long long)pos * 32;
  if (ok && p.dbg_pos != nullptr && w.pp == 0 && w.g == 0 && hh == 0) p.dbg_pos[p.A + p.R + p.dbg_M + qi] = pos;
  uint32_t lo_w[32], hi_w[32];   // rotated words: elements 2j, 2j+1 (lo) and 64+2j, 65+2j (hi)
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const uint4 lo = ok ? src[c] : make_uint4(0, 0, 0, 0);
    const uint4 hi = ok ? src[c + 8] : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float4 t = tab[4 * c + j];   // (cos f, cos f+1, sin f, sin f+1), f = 8c + 2j
      const float2 cs = make_float2(t.x, t.y), sn = make_float2(t.z, t.w);
      const float2 av = bf2(get_w(lo, j)), bv = bf2(get_w(hi, j));
      const float2 yl = __ffma2_rn(av, cs, __fmul2_rn(make_float2(-bv.x, -bv.y), sn));
      const float2 yh = __ffma2_rn(av, sn, __fmul2_rn(bv, cs));
      lo_w[4 * c + j] = pack_bf16(yl.x, yl.y);
      hi_w[4 * c + j] = pack_bf16(yh.x, yh.y);
    }
  }
  tmem_st32(taddr, lo_w);
  tmem_st32(taddr + 32, hi_w);
}

__global__ void __launch_bounds__(kThreads, 1)
    attn_tc6_kernel(const __grid_constant__ AttnParams pa, const __grid_constant__ AttnParams pb, int na, int nb,
                    int ka, int kb) {
  const AttnParams& p = pa;   // launch-wide fields (rope table, tensor maps) are shared
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = ((uint32_t)__cvta_generic_to_shared(smem_raw) + 1023u) & ~1023u;
  const uint32_t bar0 = sbase + OFF_BAR;
  auto bar = [&](int i) { return bar0 + 8u * (uint32_t)i; };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + OFF_BAR + B_N * 8);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_items = na + nb;
#define ITEM_B(I) (kb > 0 ? ((I) % (ka + kb)) >= ka : (I) >= na)
#define ITEM_PARAMS(I) (ITEM_B(I) ? pb : pa)
#define ITEM_LOCAL(I)                                                                                  \
  (kb > 0 ? (ITEM_B(I) ? ((I) / (ka + kb)) * kb + ((I) % (ka + kb)) - ka : ((I) / (ka + kb)) * ka + ((I) % (ka + kb))) \
          : (ITEM_B(I) ? (I) - na : (I)))

  if (threadIdx.x == 0) {
    mbar_init(bar(B_Q + 0), 128);
    mbar_init(bar(B_Q + 1), 128);
    mbar_init(bar(B_QE), 1);
    for (int i = 0; i < KST; ++i) {
      mbar_init(bar(B_KR + i), 1);
      mbar_init(bar(B_KF + i), 128);
      mbar_init(bar(B_KE + i), 1);
    }
    for (int i = 0; i < VST; ++i) {
      mbar_init(bar(B_VF + i), 1);
      mbar_init(bar(B_VE + i), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar(B_S + i), 1);
      mbar_init(bar(B_P + i), 128);
      mbar_init(bar(B_O + i), 1);
      mbar_init(bar(B_OF + i), 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_proxy_async();
  }
  if (warp == 14) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (warp == 12 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&pa.tmap_k)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&pa.tmap_v)) : "memory");
    if (nb > 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&pb.tmap_k)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&pb.tmap_v)) : "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_alloc = *tmem_slot;
  if (tmem_alloc != 0u) __trap();   // one CTA per SM owns all 512 columns
  constexpr uint32_t tmem = 0u;

  if (warp < 8) {
    // ================================================================ softmax
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegSoftmax));
    const int qt = warp >> 2, quarter = warp & 3;
    const int rloc = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const uint32_t tS = tmem + lane_off + TC_S + (uint32_t)(qt * 64);
    const uint32_t tO = tmem + lane_off + TC_O + (uint32_t)(qt * 128);
    const float sl2 = p.scale_log2;
    const float2 scale2 = make_float2(sl2, sl2);
    int gt = 0, kk = 0;
    for (int idx = blockIdx.x; idx < n_items; idx += gridDim.x, ++kk) {
      const AttnParams& p = ITEM_PARAMS(idx);
      const Item w = decode_item(p, ITEM_LOCAL(idx));
      const int A = w.A;
      const int n = w.n_tiles;
      const int rglob = w.m0 + qt * 128 + rloc;
      const bool valid_row = rglob < w.rows_total;
      const int qi = valid_row ? rglob / p.grp : 0;
      const int lim = valid_row ? p.q_pos0 + qi : -1;
      const bool warp_dead = __all_sync(0xffffffffu, !valid_row);
      float m = -INFINITY;
      float2 lsum2 = make_float2(0.f, 0.f);
      for (int jj = 0; jj < n; ++jj) {
        const int g = gt + jj;
        const int u = w.t_begin + jj;
        int c_lo, c_hi;
        const TileSeg t = tile_segments(p, w, u);
        const int nu = t.width;
        if (!valid_row) {
          c_lo = 0; c_hi = 0;
        } else if (u < w.n_extra) {                // sink always visible, self row j iff its id <= lim
          c_lo = 0;
          c_hi = min(max(min(A + w.n_self, max(A, lim - w.ring_count + 1)) - kKT * u, 0), kKT);
        } else {
          c_lo = t.lo0;
          c_hi = max(c_lo, min(t.hi0, lim - t.pos0_0 + 1));
        }
        const bool full = (c_lo == 0) && (c_hi == kKT);
        mbar_wait(bar(B_S + qt), g & 1);
        if (warp_dead) {   // all 32 rows are padding: their P / O are never used
          mbar_arrive(bar(B_P + qt));
          continue;
        }
        tc_fence_after();
        const bool two = nu > 32;
        uint32_t r[64];
        tmem_ld32(tS, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
        if (two) tmem_ld32(tS + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
        tmem_wait_ld();
        const bool any_partial = __any_sync(0xffffffffu, !full);
        if (any_partial) {
          const unsigned span = (unsigned)max(c_hi - c_lo, 0);
#pragma unroll
          for (int c = 0; c < 64; ++c) r[c] = ((unsigned)(c - c_lo) < span) ? r[c] : 0xFF800000u;
        }
        float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
#pragma unroll
        for (int c = 0; c < 32; c += 8) {
          mx0 = fmax3f(mx0, __uint_as_float(r[c]), __uint_as_float(r[c + 1]));
          mx1 = fmax3f(mx1, __uint_as_float(r[c + 2]), __uint_as_float(r[c + 3]));
          mx2 = fmax3f(mx2, __uint_as_float(r[c + 4]), __uint_as_float(r[c + 5]));
          mx3 = fmax3f(mx3, __uint_as_float(r[c + 6]), __uint_as_float(r[c + 7]));
        }
        if (two) {
#pragma unroll
          for (int c = 32; c < 64; c += 8) {
            mx0 = fmax3f(mx0, __uint_as_float(r[c]), __uint_as_float(r[c + 1]));
            mx1 = fmax3f(mx1, __uint_as_float(r[c + 2]), __uint_as_float(r[c + 3]));
            mx2 = fmax3f(mx2, __uint_as_float(r[c + 4]), __uint_as_float(r[c + 5]));
            mx3 = fmax3f(mx3, __uint_as_float(r[c + 6]), __uint_as_float(r[c + 7]));
          }
        }
        const float m_tile = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3)) * sl2;
        const bool upd = m_tile > m + kRescaleThreshold;
        const bool need_o = upd && (m != -INFINITY);
        const float f = need_o ? ex2(m - m_tile) : 1.f;
        if (upd) {
          lsum2.x *= f; lsum2.y *= f;
          m = m_tile;
        }
        if (__any_sync(0xffffffffu, need_o)) {
          // O_qt holds P V up to tile g-1 (complete: S(g) was issued after PV(g-1))
          mbar_wait(bar(B_O + qt), (g - 1) & 1);
          tc_fence_after();
#pragma unroll 1
          for (int ch = 0; ch < 4; ++ch) {
            uint32_t o[32];
            tmem_ld32(tO + ch * 32, o);
            tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * f);
            tmem_st32(tO + ch * 32, o);
          }
          tmem_wait_st();
        }
        const float m_use = (m == -INFINITY) ? 0.f : m;
        const float2 negm2 = make_float2(-m_use, -m_use);
        float2 l0 = make_float2(0.f, 0.f), l1 = l0;
        auto exp_chunk = [&](const int cb) {
#pragma unroll
          for (int c = cb; c < cb + 32; c += 4) {
            const float2 x0 = __ffma2_rn(make_float2(__uint_as_float(r[c]), __uint_as_float(r[c + 1])), scale2, negm2);
            const float2 x1 = __ffma2_rn(make_float2(__uint_as_float(r[c + 2]), __uint_as_float(r[c + 3])), scale2, negm2);
            const float2 p0 = make_float2(ex2(x0.x), ex2(x0.y));
            const float2 p1 = make_float2(ex2(x1.x), ex2(x1.y));
            l0 = __fadd2_rn(l0, p0);
            l1 = __fadd2_rn(l1, p1);
            r[c >> 1] = pack_bf16(p0.x, p0.y);
            r[(c >> 1) + 1] = pack_bf16(p1.x, p1.y);
          }
        };
        exp_chunk(0);
        if (two) {
          exp_chunk(32);
          tmem_st32(tS, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
        } else {
          tmem_st16(tS, *reinterpret_cast<uint32_t(*)[16]>(&r[0]));
        }
        lsum2 = __fadd2_rn(lsum2, __fadd2_rn(l0, l1));
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(bar(B_P + qt));
      }
      gt += n;
      // epilogue: O / l once the last PV is done
      const float lsum = lsum2.x + lsum2.y;
      mbar_wait(bar(B_O + qt), (gt - 1) & 1);
      tc_fence_after();
      const float inv = lsum > 0.f ? 1.f / lsum : 0.f;
      const int h = valid_row ? w.g * p.grp + rglob % p.grp : 0;
      const long long orow = ((long long)w.pp * p.n_q + qi) * p.Hq + h;
#pragma unroll 1
      for (int hf = 0; hf < 2; ++hf) {
        uint32_t o[64];
        tmem_ld32(tO + 64 * hf, *reinterpret_cast<uint32_t(*)[32]>(&o[0]));
        tmem_ld32(tO + 64 * hf + 32, *reinterpret_cast<uint32_t(*)[32]>(&o[32]));
        tmem_wait_ld();
        if (hf == 1) {
          tc_fence_before();
          mbar_arrive(bar(B_OF + qt));      // O_qt may be overwritten by the next item
        }
        if (!valid_row) continue;
        if (p.n_splits == 1 && p.split_only < 0) {
          __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(p.o) + orow * 128 + 64 * hf;
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            uint32_t q[8];
#pragma unroll
            for (int j = 0; j < 8; ++j)
              q[j] = pack_bf16(__uint_as_float(o[16 * v + 2 * j]) * inv, __uint_as_float(o[16 * v + 2 * j + 1]) * inv);
            stg256(dst + 16 * v, q);
          }
        } else {
          const long long rows = (long long)p.P * p.n_q * p.Hq;
          const long long slot = p.split_only >= 0 ? 0 : w.sp;
          float4* dst = reinterpret_cast<float4*>(p.ws_o + (slot * rows + orow) * 128 + 64 * hf);
#pragma unroll
          for (int v = 0; v < 16; ++v)
            dst[v] = make_float4(__uint_as_float(o[4 * v]) * inv, __uint_as_float(o[4 * v + 1]) * inv,
                                 __uint_as_float(o[4 * v + 2]) * inv, __uint_as_float(o[4 * v + 3]) * inv);
          if (hf == 0) p.ws_lse[slot * rows + orow] = lsum > 0.f ? m + __log2f(lsum) : -INFINITY;
        }
      }
    }
  } else if (warp < 12) {
    // ================================================================ rotation: K tiles + Q rows
    if constexpr (kRegRotate > kThreadRegs) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegRotate));
    const int lt = threadIdx.x - 256;                 // = TMEM lane of this thread's Q rows
    const uint32_t lane_off = (uint32_t)((lt >> 5) * 32) << 16;
    const int c8 = lt & 7;
    const int rg = lt >> 3;
    const float4* __restrict__ rp = p.rope_pairs;
    float2 cth[4], sth[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float4 t = rp[32 + 4 * c8 + j];
      cth[j] = make_float2(t.x, t.y);
      sth[j] = make_float2(t.z, t.w);
    }
    // Q rows of item k (index qidx) into TMEM; for k >= 1 after item k-1's last QK^T MMA
    auto prep_q = [&](int k, int qidx) {
      if (k >= 1) mbar_wait(bar(B_QE), (k - 1) & 1);
      tc_fence_after();
      const AttnParams& pq = ITEM_PARAMS(qidx);
      const Item wq = decode_item(pq, ITEM_LOCAL(qidx));
#pragma unroll 1
      for (int q = 0; q < 2; ++q) q_row_to_tmem(pq, wq, q, lt, tmem + lane_off + TC_Q + (uint32_t)(q * 64));
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(bar(B_Q + 0));
      mbar_arrive(bar(B_Q + 1));
    };
    if (blockIdx.x < (unsigned)n_items) prep_q(0, blockIdx.x);
    int gt = 0, kk = 0;
    for (int idx = blockIdx.x; idx < n_items; idx += gridDim.x, ++kk) {
      const AttnParams& p = ITEM_PARAMS(idx);
      const Item w = decode_item(p, ITEM_LOCAL(idx));
      const int A = p.A;
      const bool dbg = p.dbg_pos != nullptr && w.pp == 0 && w.g == 0;
      const int nidx = idx + gridDim.x;
      if (!w.staged) {
        int kpos[4];
        float4 kpre[4];
        auto first_pos = [&](int u) {
          const TileSeg t = tile_segments(p, w, u);
          int q = -1;
#pragma unroll
          for (int k = 3; k >= 0; --k) {
            const int pk = seg_pos(t, rg * 4 + k);
            if (pk >= 0) q = pk;
          }
          return q;
        };
        int pre_pos = w.n_tiles > 0 ? first_pos(w.t_begin) : -1;
#pragma unroll
        for (int j = 0; j < 4; ++j) kpre[j] = rp[(long long)max(pre_pos, 0) * 32 + 4 * c8 + j];
        for (int jj = 0; jj < w.n_tiles; ++jj) {
          const int g = gt + jj, u = w.t_begin + jj, ks = g % KST;
          const TileSeg t = tile_segments(p, w, u);
#pragma unroll
          for (int k = 0; k < 4; ++k) kpos[k] = seg_pos(t, rg * 4 + k);
          float4 cur[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) cur[j] = kpre[j];
          const int cur_pos = pre_pos;
          if (jj + 1 < w.n_tiles) {
            pre_pos = first_pos(u + 1);
#pragma unroll
            for (int j = 0; j < 4; ++j) kpre[j] = rp[(long long)max(pre_pos, 0) * 32 + 4 * c8 + j];
          }
          mbar_wait(bar(B_KR + ks), (g / KST) & 1);
          if (rg * 4 < t.width)
            rotate_rows<1, kKVHalf>(sbase + OFF_K + ks * kKVBytes, rg * 4, c8, rp, cth, sth, kpos, cur,
                                    max(cur_pos, 0));
          fence_proxy_async();
          mbar_arrive(bar(B_KF + ks));
          if (dbg && c8 == 0) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int r = rg * 4 + k;
              const int x = kKT * u + r;
              int slot = t.slot0 + r;
              if (slot >= p.R) slot -= p.R;
              if (kpos[k] >= 0) p.dbg_pos[(u < w.n_extra) ? (x < A ? x : A + p.R + (x - A)) : A + slot] = kpos[k];
            }
          }
        }
      }
      if (nidx < n_items) prep_q(kk + 1, nidx);
      gt += w.n_tiles;
    }
  } else {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegCopy));
    if (warp == 12 || warp == 13) {
      // ============================================================== copy warps (12: K, 13: V)
      const bool isk = warp == 12;
      const int nst = isk ? KST : VST;
      const int off = isk ? OFF_K : OFF_V;
      const int b_full = isk ? B_KR : B_VF, b_free = isk ? B_KE : B_VE;
      int gt = 0;
      for (int idx = blockIdx.x; idx < n_items; idx += gridDim.x) {
        const AttnParams& p = ITEM_PARAMS(idx);
        const Item w = decode_item(p, ITEM_LOCAL(idx));
        const int A = p.A;
        const __nv_bfloat16* __restrict__ SX = reinterpret_cast<const __nv_bfloat16*>(isk ? p.sink_k : p.sink_v);
        const __nv_bfloat16* __restrict__ XX = reinterpret_cast<const __nv_bfloat16*>(isk ? p.self_k : p.self_v);
#pragma unroll 1
        for (int jj = 0; jj < w.n_tiles; ++jj) {
          const int g = gt + jj, u = w.t_begin + jj, st = g % nst;
          if (g >= nst) mbar_wait(bar(b_free + st), ((g - nst) / nst) & 1);
          const uint32_t dst = sbase + off + st * kKVBytes;
          const TileSeg t = tile_segments(p, w, u);
          if (u < w.n_extra) {
            const int nit = t.width >> 1;
#pragma unroll 1
            for (int it = 0; it < nit; ++it) {
              const int id = it * 32 + lane;
              const int r = id >> 4, ch = id & 15;
              const int x = kKT * u + r;
              const __nv_bfloat16* src = nullptr;
              if (x < A) src = SX + (w.head_row * A + x) * 128;
              else if (x < A + w.n_self) src = XX + (((long long)w.pp * w.n_self + (x - A)) * p.Hkv + w.g) * 128;
              const uint32_t d = dst + (ch >> 3) * kKVHalf + r * 128 + (((ch & 7) ^ (r & 7)) << 4);
              cp_async16(d, src ? (const void*)(src + 8 * ch) : (const void*)SX, src ? 16u : 0u);
            }
            cp_async_wait_all();
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar(b_full + st));
          } else if (lane == 0) {
            const CUtensorMap* tmap = isk ? &p.tmap_k : &p.tmap_v;
            const int row = (int)(w.head_row * w.Rp) + t.slot0;
            mbar_arrive_tx(bar(b_full + st), kKVBytes);
            tma_load_2d(dst, tmap, 0, row, bar(b_full + st));
            tma_load_2d(dst + kKVHalf, tmap, 64, row, bar(b_full + st));
          }
          __syncwarp();
        }
        gt += w.n_tiles;
      }
    } else if (warp == 14) {
      // ============================================================== MMA issuer (whole warp, elected lane issues)
      constexpr uint32_t IQK0 = idesc_bf16(128, 0, 0, 0);    // S = Q K^T: A (Q) from TMEM, B (K) K-major smem
      constexpr uint32_t IPV = idesc_bf16(128, 128, 0, 1);   // O += P V: A (P) from TMEM, B (V) MN-major smem
      const uint64_t dk0 = sdesc(sbase + OFF_K, 16, 1024);
      const uint64_t dv0 = sdesc(sbase + OFF_V, kKVHalf, 1024);
      auto issue_qk = [&](int qt, int ks, int nu) {
        const uint32_t iqk = IQK0 | ((uint32_t)(nu >> 3) << 17);
        mma_qk8_ts_w(tmem + TC_S + qt * 64, tmem + TC_Q + qt * 64, dk0 + (uint64_t)(ks * (kKVBytes >> 4)), iqk);
      };
      auto issue_pv = [&](int qt, int vs, bool acc, int nu) {
        const uint64_t dv = dv0 + (uint64_t)(vs * (kKVBytes >> 4));
        const uint32_t d = tmem + TC_O + qt * 128, a = tmem + TC_S + qt * 64;
        const int nk = nu >> 4;
        if (nk == 4) {
          mma_pv4_w(d, a, dv, IPV, acc ? 1u : 0u);
        } else {
          mma_ts_w(d, a, dv, IPV, acc ? 1u : 0u);
#pragma unroll
          for (int k8 = 1; k8 < kKT / 16; ++k8)
            if (k8 < nk) mma_ts_w(d, a + k8 * 8, dv + (uint64_t)(k8 * 128), IPV, 1u);
        }
      };
      int gt = 0, kk = 0;
      for (int idx = blockIdx.x; idx < n_items; idx += gridDim.x, ++kk) {
        const ItemGeo p = item_geo(pa, pb, ITEM_B(idx));
        const Item w = decode_item(p, ITEM_LOCAL(idx));
        const int n = w.n_tiles;
        const int kbar = w.staged ? B_KR : B_KF;    // staged K arrives rotated: no rotation barrier
        mbar_wait(bar(B_Q + 0), kk & 1);
        mbar_wait(bar(B_Q + 1), kk & 1);
        if (n == 0) mma_commit_w(bar(B_QE));   // nothing reads this item's Q
        if (n > 0) {
          const int ks = gt % KST, nu = tile_segments(p, w, w.t_begin).width;
          mbar_wait(bar(kbar + ks), (gt / KST) & 1);
          tc_fence_after();
          issue_qk(0, ks, nu);
          mma_commit_w(bar(B_S + 0));
          issue_qk(1, ks, nu);
          mma_commit_w(bar(B_S + 1));
          mma_commit_w(bar(B_KE + ks));
          if (n == 1) mma_commit_w(bar(B_QE));      // the item's last QK^T: Q may be replaced
        }
        for (int jj = 0; jj < n; ++jj) {
          const int g = gt + jj, vs = g % VST;
          const int nu = tile_segments(p, w, w.t_begin + jj).width;
          const bool more = jj + 1 < n;
          const int ks1 = (g + 1) % KST;
          const int nu1 = more ? tile_segments(p, w, w.t_begin + jj + 1).width : 0;
          mbar_wait(bar(B_VF + vs), (g / VST) & 1);
#pragma unroll 1
          for (int qt = 0; qt < 2; ++qt) {
            mbar_wait(bar(B_P + qt), g & 1);
            if (jj == 0 && kk > 0) mbar_wait(bar(B_OF + qt), (kk - 1) & 1);   // previous item's O read
            tc_fence_after();
            issue_pv(qt, vs, jj > 0, nu);
            mma_commit_w(bar(B_O + qt));
            if (more) {      // S(g+1) overwrites S/P of this Q tile: after PV(g), in issue order
              if (qt == 0) {
                mbar_wait(bar(kbar + ks1), ((g + 1) / KST) & 1);
                tc_fence_after();
              }
              issue_qk(qt, ks1, nu1);
              mma_commit_w(bar(B_S + qt));
            }
          }
          mma_commit_w(bar(B_VE + vs));
          if (more) {
            mma_commit_w(bar(B_KE + ks1));
            if (jj + 2 == n) mma_commit_w(bar(B_QE));   // the item's last QK^T was just issued
          }
        }
        gt += n;
      }
      if (gt > 0) mbar_wait(bar(B_VE + (gt - 1) % VST), ((gt - 1) / VST) & 1);
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 14) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_alloc) : "memory");
  }
#undef ITEM_B
#undef ITEM_PARAMS
#undef ITEM_LOCAL
}

}  // namespace tc6

static long long tc6_items(const AttnParams& p) {
  return (long long)p.P * p.Hkv * p.n_mblocks * (p.split_only >= 0 ? 1 : p.n_splits);
}

cudaError_t launch_attn_tc6(const AttnParams& pa, const AttnParams* pb, cudaStream_t st) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(tc6::attn_tc6_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         tc6::kSmemBytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  static int num_sms = 0;
  if (num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const long long na = tc6_items(pa), nb = pb ? tc6_items(*pb) : 0;
  const long long items = na + nb;
  const unsigned grid = (unsigned)(items < num_sms ? items : num_sms);
  tc6::attn_tc6_kernel<<<grid, tc6::kThreads, tc6::kSmemBytes, st>>>(pa, pb ? *pb : pa, (int)na, (int)nb, 0, 0);
  return cudaGetLastError();
}

}  // namespace dsc
