// K3/K4: fused rotate-on-load RoPE + GQA flash attention on the sm_100a tensor
// cores (tcgen05.mma, accumulators in TMEM), used by both dscache_build_instant
// (Eq. 7: instant tokens over [sink | instant], causal) and dscache_attend
// (Eq. 8 + self: the query chunk over [sink | past | instant | self]).
//
// Position-agnostic encoding (Def. 4.1): the ring holds raw
// K; each K tile is rotated in registers by its use-time id (consecutive from 0,
// PAPER.md:236) while it is moved global -> shared, once per CTA for the 256
// query rows (2 x 128-row Q tiles) that share it.  Softmax a_ij =
// softmax(Q_i K_j / sqrt(d)) in the exp2 domain with lazy rescale.
//
// Persistent CTAs (grid <= #SMs) walk a longest-first list of work items
// (problem, kv head, 256-row m-block, key split); every pipeline phase runs on a
// CTA-global tile counter, Q and O are recycled across items by barriers.
//
// CTA = 16 warps:
//   warps 0-3  softmax of Q tile 0 (thread = query row = TMEM lane)
//   warps 4-7  softmax of Q tile 1
//   warps 8-11 rotation: every raw K tile in place in shared memory
//              (LDS -> rotate -> STS), with R(p+1) = R(p) R(1) between consecutive ids
//   (each softmax warpgroup loads + rotates the Q tile of its next item itself, as soon
//    as it has consumed S of its last tile, overlapped with its epilogue)
//   warp 12    K copy: raw K tiles -> SW128 smem; TMA (2 x 64x128 boxes) for ring
//              tiles, cp.async for the sink/self tile
//   warp 13    V copy: same for V (K and V stage recycling is independent)
//   warp 14    TMEM allocator + single-thread tcgen05.mma issuer
//   warp 15    idle
// Softmax reads each S row from TMEM in two 64-column halves (max pass, then
// exp pass); registers (setmaxnreg): softmax 144, rotation 136, copy/MMA 88.
// TMEM (512 cols): S0 [0,128) S1 [128,256) O0 [256,384) O1 [384,512);
// P_qt (bf16x2) overwrites S_qt cols [0,64) and feeds O_qt += P V as the TMEM A operand.
// MMA issue order S0_0 S1_0 | PV0_j S0_{j+1} PV1_j S1_{j+1} | ... so each softmax
// warpgroup overlaps the other Q tile's MMAs.
#include "tc_common.cuh"

namespace dsc {
namespace tc {
using namespace tcc;

constexpr int kNQT = 2;                       // Q tiles per CTA
constexpr int kWarps = 16;
constexpr int kThreads = kWarps * 32;
constexpr int kTileBytes = 128 * 128 * 2;     // one 128 x 128 bf16 tile
constexpr int KST = 3;                        // K stages (raw -> rotated in place)
constexpr int VST = 2;                        // V stages
constexpr int OFF_Q = 0;
constexpr int OFF_K = OFF_Q + kNQT * kTileBytes;
constexpr int OFF_V = OFF_K + KST * kTileBytes;
constexpr int OFF_BAR = OFF_V + VST * kTileBytes;
// barriers (8 B each): Q ready | Q free | K raw landed | K rotated | K free | V landed | V free |
// S ready | P ready | O done | O read (epilogue done)
constexpr int B_Q = 0 /* +qt */, B_KR = 2, B_KF = 5, B_KE = 8, B_VF = 11, B_VE = 13, B_S = 15, B_P = 17, B_O = 19,
              B_OF = 21, B_N = 23;
// setmaxnreg budget per warpgroup: 2*softmax + rotation + copy/MMA <= 512 (x 128 threads)
constexpr int kRegSoftmax = 144, kRegRotate = 136, kRegCopy = 88;
static_assert(2 * kRegSoftmax + kRegRotate + kRegCopy <= 512, "setmaxnreg budget exceeds the 64K register file");
constexpr int kThreadRegs = 65536 / kThreads;   // allocation at launch (128); inc above it, dec below it
static_assert(kRegSoftmax > kThreadRegs && kRegCopy < kThreadRegs, "softmax must grow, copy/MMA must shrink");
constexpr int kSmemBytes = OFF_BAR + B_N * 8 + 16 + 1024;   // + tmem slot + alignment slack
constexpr float kRescaleThreshold = 8.0f;     // log2 units (factor 256)
static_assert(kNQT * 128 == kMBlockRows, "work items are 256-row m-blocks");
#ifndef DSC_POLY
#define DSC_POLY 0
#endif
// ablation knobs (timing experiments only; results are wrong when set):
// DSC_ABL_SOFTMAX skips the softmax body, DSC_ABL_ROT skips the K rotation
#ifndef DSC_ABL_SOFTMAX
#define DSC_ABL_SOFTMAX 0
#endif
#ifndef DSC_ABL_ROT
#define DSC_ABL_ROT 0
#endif
// DSC_ABL_EX2 replaces ex2 by a copy (MUFU-free softmax), DSC_ABL_PST skips the P store to TMEM
#ifndef DSC_ABL_EX2
#define DSC_ABL_EX2 0
#endif
#ifndef DSC_ABL_PST
#define DSC_ABL_PST 0
#endif
constexpr int kPolyPerGroup = DSC_POLY;   // of every 8 columns of a full tile, this many use exp2_poly2
// DSC_PINGPONG: the exp passes of the two softmax warpgroups alternate (a token passed
// through two named barriers), so each runs with the MUFU to itself while the tensor core
// works on the other Q tile; the max passes still overlap
#ifndef DSC_PINGPONG
#define DSC_PINGPONG 1
#endif
constexpr int kBarTok0 = 4, kBarTok1 = 5;     // named barriers: exp-pass token of WG0 / WG1
// DSC_INTERLEAVE: the fused step interleaves attend and build items per (problem, kv head)
#ifndef DSC_INTERLEAVE
#define DSC_INTERLEAVE 0
#endif
#ifndef DSC_QFIRST
#define DSC_QFIRST 0
#endif

// ------------------------------------------------------------------ kernel
// Two attention problems can share one persistent launch (the fused step: attend items
// first, then build_instant items); items [0, na) use pa, [na, na + nb) use pb.
__global__ void __launch_bounds__(kThreads, 1)
    attn_tc_kernel(const __grid_constant__ AttnParams pa, const __grid_constant__ AttnParams pb, int na, int nb, int ka,
                   int kb) {
  const AttnParams& p = pa;   // launch-wide fields (rope table, tensor maps, trace) are shared
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = su32(smem);
  const uint32_t bar0 = sbase + OFF_BAR;
  auto bar = [&](int i) { return bar0 + 8u * (uint32_t)i; };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + OFF_BAR + B_N * 8);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_items = na + nb;
  // kb > 0: the items of pa and pb are interleaved in groups of ka (pa) + kb (pb) items
  // (one group per (problem, kv head) when both use the head-major item order)
#define ITEM_B(I) (kb > 0 ? ((I) % (ka + kb)) >= ka : (I) >= na)
#define ITEM_PARAMS(I) (ITEM_B(I) ? pb : pa)
#define ITEM_LOCAL(I)                                                                                  \
  (kb > 0 ? (ITEM_B(I) ? ((I) / (ka + kb)) * kb + ((I) % (ka + kb)) - ka : ((I) / (ka + kb)) * ka + ((I) % (ka + kb))) \
          : (ITEM_B(I) ? (I) - na : (I)))

  if (threadIdx.x == 0) {
    mbar_init(bar(B_Q + 0), 128);
    mbar_init(bar(B_Q + 1), 128);
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
    TRACE(EV_START, 0);
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tmap_k)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tmap_v)) : "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 8) {
    // ================================================================ softmax
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegSoftmax));
    const int qt = warp >> 2, quarter = warp & 3;
    const int rloc = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const uint32_t tS = tmem + lane_off + (uint32_t)(qt * 128);
    const uint32_t tO = tmem + lane_off + (uint32_t)(256 + qt * 128);
    const float sl2 = p.scale_log2;
    const float2 scale2 = make_float2(sl2, sl2);
    const int lt = threadIdx.x - qt * 128;          // 0..127 within the warpgroup
    const uint32_t qtile = sbase + OFF_Q + qt * kTileBytes;
    if (blockIdx.x < (unsigned)n_items) {            // Q tile of the first item
      const AttnParams& p0 = ITEM_PARAMS((int)blockIdx.x);
      const Item w0 = decode_item(p0, ITEM_LOCAL((int)blockIdx.x));
      issue_q_tile(p0, w0, qt, lt, qtile);
      rotate_q_tile(p0, w0, qt, lt, qtile, 2 + qt);
      mbar_arrive(bar(B_Q + qt));
    }
    const int tok_mine = qt == 0 ? kBarTok0 : kBarTok1, tok_other = qt == 0 ? kBarTok1 : kBarTok0;
    if (DSC_PINGPONG && qt == 1) named_bar_arrive(kBarTok0, 256);   // WG0 takes the first exp pass
    int gt = 0, kk = 0;
    for (int idx = blockIdx.x; idx < n_items; idx += gridDim.x, ++kk) {
      const AttnParams& p = ITEM_PARAMS(idx);
      const Item w = decode_item(p, ITEM_LOCAL(idx));
      const int A = p.A;
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
        const int nu = t.width;                // S columns [0, nu) hold this tile's scores
        if (!valid_row) {
          c_lo = 0; c_hi = 0;
        } else if (u < w.n_extra) {       // sink always visible, self row j iff its id <= lim
          c_lo = 0;
          c_hi = min(max(min(A + p.n_self, max(A, lim - p.ring_count + 1)) - 128 * u, 0), 128);
        } else {
          c_lo = t.lo0;
          c_hi = max(c_lo, min(t.hi0, lim - t.pos0_0 + 1));   // id pos0 + c <= lim
        }
        const bool full = (c_lo == 0) && (c_hi == 128);
        mbar_wait(bar(B_S + qt), g & 1);
        if (rloc == 0) TRACE(EV_S0 + qt, g);
        if (warp_dead || DSC_ABL_SOFTMAX) {   // all 32 rows are padding: their P / O are never used
          if (DSC_PINGPONG) { named_bar_sync(tok_mine, 256); named_bar_arrive(tok_other, 256); }
          mbar_arrive(bar(B_P + qt));
          continue;
        }
        tc_fence_after();
        // pass 1: row max over the visible columns, in 64-column halves.  In a partial
        // tile the invisible columns are set to -inf and written back to TMEM, so the exp
        // pass needs no mask (2^-inf = 0).  A tile narrower than 128 is always partial
        // (columns past its width are stale and get masked).
        const bool any_partial = __any_sync(0xffffffffu, !full);
        const unsigned span = (unsigned)max(c_hi - c_lo, 0);
        const int nh = (nu + 63) >> 6;
        float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
#pragma unroll 1
        for (int hf = 0; hf < nh; ++hf) {
          uint32_t r[64];
          tmem_ld32(tS + 64 * hf, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
          tmem_ld32(tS + 64 * hf + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
          tmem_wait_ld();
          if (warp == 0 && lane == 0) TRACE(EV_L + hf, g);
          if (any_partial) {
#pragma unroll
            for (int c = 0; c < 64; ++c) r[c] = ((unsigned)(64 * hf + c - c_lo) < span) ? r[c] : 0xFF800000u;
            tmem_st32(tS + 64 * hf, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
            tmem_st32(tS + 64 * hf + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
          }
#pragma unroll
          for (int c = 0; c < 64; c += 8) {     // 3-input max (FMNMX3): 2 columns per instruction
            mx0 = fmax3f(mx0, __uint_as_float(r[c]), __uint_as_float(r[c + 1]));
            mx1 = fmax3f(mx1, __uint_as_float(r[c + 2]), __uint_as_float(r[c + 3]));
            mx2 = fmax3f(mx2, __uint_as_float(r[c + 4]), __uint_as_float(r[c + 5]));
            mx3 = fmax3f(mx3, __uint_as_float(r[c + 6]), __uint_as_float(r[c + 7]));
          }
        }
        if (any_partial) tmem_wait_st();
        const float m_tile = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3)) * sl2;
        // lazy rescale: move the running max only when it grew by > 2^8; the TMEM
        // load/store of O is warp-collective, so the decision is made per warp.
        const bool upd = m_tile > m + kRescaleThreshold;
        const bool need_o = upd && (m != -INFINITY);
        const float f = need_o ? ex2(m - m_tile) : 1.f;
        if (upd) {
          lsum2.x *= f; lsum2.y *= f;
          m = m_tile;
        }
        if (__any_sync(0xffffffffu, need_o)) {
          // O_qt holds PV up to the previous tile: wait for it, rescale in TMEM
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
        if (warp == 0 && lane == 0) TRACE(EV_L + 5, g);
        const float m_use = (m == -INFINITY) ? 0.f : m;
        const float2 negm2 = make_float2(-m_use, -m_use);
        // pass 2: P = 2^(s*scale - m) (masked -> 2^-inf = 0), packed bf16x2; half hf of S
        // (cols 64hf..64hf+63) becomes P cols 32hf..32hf+31 (already consumed S columns);
        // a 32-column chunk past the tile width is skipped
        float2 l0 = make_float2(0.f, 0.f), l1 = l0;
        if (DSC_PINGPONG) named_bar_sync(tok_mine, 256);
#pragma unroll 1
        for (int hf = 0; hf < nh; ++hf) {
          const bool two = 64 * hf + 32 < nu;
          uint32_t r[64];
          tmem_ld32(tS + 64 * hf, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
          if (two) tmem_ld32(tS + 64 * hf + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
          tmem_wait_ld();
          if (warp == 0 && lane == 0) TRACE(EV_L + 2 + hf, g);
          auto exp_chunk = [&](const int cb) {   // columns cb .. cb+31 -> P words cb/2 .. cb/2+15
#pragma unroll
            for (int c = cb; c < cb + 32; c += 4) {
              const float2 x0 = __ffma2_rn(make_float2(__uint_as_float(r[c]), __uint_as_float(r[c + 1])), scale2, negm2);
              const float2 x1 = __ffma2_rn(make_float2(__uint_as_float(r[c + 2]), __uint_as_float(r[c + 3])), scale2, negm2);
              float2 p0, p1;
              constexpr bool poly0_any = kPolyPerGroup > 0;
              const bool poly0 = poly0_any && ((c % 8) + 2 > 8 - kPolyPerGroup);
              const bool poly1 = poly0_any && ((c % 8) + 4 > 8 - kPolyPerGroup);
              if (DSC_ABL_EX2) { p0 = x0; p1 = x1; } else {
              if (poly0 && !any_partial) p0 = exp2_poly2(x0); else p0 = make_float2(ex2(x0.x), ex2(x0.y));
              if (poly1 && !any_partial) p1 = exp2_poly2(x1); else p1 = make_float2(ex2(x1.x), ex2(x1.y));
              }
              l0 = __fadd2_rn(l0, p0);
              l1 = __fadd2_rn(l1, p1);
              r[c >> 1] = pack_bf16(p0.x, p0.y);
              r[(c >> 1) + 1] = pack_bf16(p1.x, p1.y);
            }
          };
          exp_chunk(0);
          if (two) exp_chunk(32);
          if (DSC_ABL_PST && r[0] != 0x12345u) continue;
          if (two) tmem_st32(tS + 32 * hf, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
          else tmem_st16(tS + 32 * hf, *reinterpret_cast<uint32_t(*)[16]>(&r[0]));
        }
        if (DSC_PINGPONG) named_bar_arrive(tok_other, 256);
        lsum2 = __fadd2_rn(lsum2, __fadd2_rn(l0, l1));
        if (warp == 0 && lane == 0) TRACE(EV_L + 4, g);
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(bar(B_P + qt));
        if (rloc == 0) TRACE(EV_P0 + qt, g);
        if (lane == 0) TRACE(EV_PW0 + warp, g);
      }
      gt += n;
      // S_qt of the last tile has been read: the MMA is done with Q tile qt, so the next
      // item's Q tile is fetched now (overlapping this item's epilogue)
      const int nidx = idx + gridDim.x;
      Item wn;
      if (nidx < n_items) {
        wn = decode_item(ITEM_PARAMS(nidx), ITEM_LOCAL(nidx));
        issue_q_tile(ITEM_PARAMS(nidx), wn, qt, lt, qtile);
      }
      // publish the next item's Q before this item's epilogue, so the tensor core can start
      // the next item's first S MMAs while O is read out (the MMA waits for B_OF before it
      // overwrites O with the next item's first PV)
#if DSC_QFIRST
      if (nidx < n_items) {
        rotate_q_tile(ITEM_PARAMS(nidx), wn, qt, lt, qtile, 2 + qt);
        mbar_arrive(bar(B_Q + qt));
        if (rloc == 0) TRACE(EV_QDONE, gt);
      }
#endif
      // epilogue of the item
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
        if (p.n_splits == 1) {
          uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.o) + orow * 128 + 64 * hf);
#pragma unroll
          for (int v = 0; v < 8; ++v) {
            uint4 q;
            q.x = pack_bf16(__uint_as_float(o[8 * v + 0]) * inv, __uint_as_float(o[8 * v + 1]) * inv);
            q.y = pack_bf16(__uint_as_float(o[8 * v + 2]) * inv, __uint_as_float(o[8 * v + 3]) * inv);
            q.z = pack_bf16(__uint_as_float(o[8 * v + 4]) * inv, __uint_as_float(o[8 * v + 5]) * inv);
            q.w = pack_bf16(__uint_as_float(o[8 * v + 6]) * inv, __uint_as_float(o[8 * v + 7]) * inv);
            dst[v] = q;
          }
        } else {
          const long long rows = (long long)p.P * p.n_q * p.Hq;
          float4* dst = reinterpret_cast<float4*>(p.ws_o + ((long long)w.sp * rows + orow) * 128 + 64 * hf);
#pragma unroll
          for (int v = 0; v < 16; ++v)
            dst[v] = make_float4(__uint_as_float(o[4 * v]) * inv, __uint_as_float(o[4 * v + 1]) * inv,
                                 __uint_as_float(o[4 * v + 2]) * inv, __uint_as_float(o[4 * v + 3]) * inv);
          if (hf == 0) p.ws_lse[(long long)w.sp * rows + orow] = lsum > 0.f ? m + __log2f(lsum) : -INFINITY;
        }
      }
#if !DSC_QFIRST
      if (nidx < n_items) {
        rotate_q_tile(ITEM_PARAMS(nidx), wn, qt, lt, qtile, 2 + qt);
        mbar_arrive(bar(B_Q + qt));
        if (rloc == 0) TRACE(EV_QDONE, gt);
      }
#endif
    }
    if (DSC_PINGPONG && qt == 0) named_bar_sync(kBarTok0, 256);   // WG1's last token
  } else if (warp < 12) {
    // ================================================================ rotation (Q per item, then K tiles)
    if constexpr (kRegRotate > kThreadRegs) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegRotate));
    else if constexpr (kRegRotate < kThreadRegs) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegRotate));
    const int lt = threadIdx.x - 256;
    const int c8 = lt & 7;             // frequencies 8*c8 .. 8*c8+7
    const int rg8 = lt >> 3;           // rows rg8*8 .. +7 of a 128-row tile
    const float4* __restrict__ rp = p.rope_pairs;
    float2 cth[4], sth[4];             // R(theta_f) = table entry of id 1
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float4 t = rp[32 + 4 * c8 + j];
      cth[j] = make_float2(t.x, t.y);
      sth[j] = make_float2(t.z, t.w);
    }
    int gt = 0, kk = 0;
    for (int idx = blockIdx.x; idx < n_items; idx += gridDim.x, ++kk) {
      const AttnParams& p = ITEM_PARAMS(idx);
      const Item w = decode_item(p, ITEM_LOCAL(idx));
      const int A = p.A;
      const bool dbg = p.dbg_pos != nullptr && w.pp == 0 && w.g == 0;
      // ---- K tiles of this item; the table entry of each tile's first row is fetched
      // one tile ahead so the L2 latency is off the rotation's critical path
      int kpos[8];
      float4 kpre[4];
      auto first_pos = [&](int u) {
        const TileSeg t = tile_segments(p, w, u);
        int q = -1;
#pragma unroll
        for (int k = 7; k >= 0; --k) {
          const int pk = seg_pos(t, rg8 * 8 + k);
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
        for (int k = 0; k < 8; ++k) kpos[k] = seg_pos(t, rg8 * 8 + k);
        float4 cur[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) cur[j] = kpre[j];
        const int cur_pos = pre_pos;
        if (jj + 1 < w.n_tiles) {          // prefetch for the next tile
          pre_pos = first_pos(u + 1);
#pragma unroll
          for (int j = 0; j < 4; ++j) kpre[j] = rp[(long long)max(pre_pos, 0) * 32 + 4 * c8 + j];
        }
        mbar_wait(bar(B_KR + ks), (g / KST) & 1);
        if (lt == 0) TRACE(EV_KR, g);
        if (!DSC_ABL_ROT && rg8 * 8 < t.width)   // rows >= width are never read by the MMA
          rotate8(sbase + OFF_K + ks * kTileBytes, rg8 * 8, c8, rp, cth, sth, kpos, cur, max(cur_pos, 0));
        fence_proxy_async();
        mbar_arrive(bar(B_KF + ks));
        if (lt == 0) TRACE(EV_KDONE, g);
        if (dbg && c8 == 0) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int r = rg8 * 8 + k;
            const int x = 128 * u + r;
            int slot = t.slot0 + r;
            if (slot >= p.R) slot -= p.R;
            if (kpos[k] >= 0) p.dbg_pos[(u < w.n_extra) ? (x < A ? x : A + p.R + (x - A)) : A + slot] = kpos[k];
          }
        }
      }
      gt += w.n_tiles;
    }
  } else {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegCopy));
    if (warp == 12 || warp == 13) {
      // ============================================================== copy warps (12: K, 13: V)
      const bool isk = warp == 12;
      const CUtensorMap* tmap = isk ? &p.tmap_k : &p.tmap_v;
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
          const uint32_t dst = sbase + off + st * kTileBytes;
          const TileSeg t = tile_segments(p, w, u);
          if (u < w.n_extra) {
            // sink rows (x < A) + self rows (A <= x < A + n_self), zeros up to the tile
            // width, with cp.async
            const int nit = t.width >> 1;
#pragma unroll 1
            for (int it = 0; it < nit; ++it) {
              const int id = it * 32 + lane;          // 2048 16-byte chunks
              const int r = id >> 4, ch = id & 15;
              const int x = 128 * u + r;
              const __nv_bfloat16* src = nullptr;
              if (x < A) src = SX + (w.head_row * A + x) * 128;
              else if (x < A + p.n_self) src = XX + (((long long)w.pp * p.n_self + (x - A)) * p.Hkv + w.g) * 128;
              const uint32_t d = dst + (ch >> 3) * 16384 + r * 128 + (((ch & 7) ^ (r & 7)) << 4);
              cp_async16(d, src ? (const void*)(src + 8 * ch) : (const void*)SX, src ? 16u : 0u);
            }
            cp_async_wait_all();
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar(b_full + st));
          } else if (lane == 0) {
            const int row = (int)(w.head_row * p.Rp) + t.slot0;   // logical window tile (mirror: no wrap)
            mbar_arrive_tx(bar(b_full + st), kTileBytes);
            tma_load_2d(dst, tmap, 0, row, bar(b_full + st));
            tma_load_2d(dst + 16384, tmap, 64, row, bar(b_full + st));
          }
          if (lane == 0) TRACE(isk ? EV_K_ISSUE : EV_V_ISSUE, g);
          __syncwarp();
        }
        gt += w.n_tiles;
      }
    } else if (warp == 14) {
      // ============================================================== MMA issuer (whole warp, elected lane issues)
      constexpr uint32_t IQK0 = idesc_bf16(128, 0, 0, 0);    // S = Q K^T, both K-major; N = tile width
      constexpr uint32_t IPV = idesc_bf16(128, 128, 0, 1);   // O += P V, P from TMEM, V MN-major
      // descriptors advance in the 14-bit start-address field: +32 B (2) per 16-element
      // K step inside a 128 B swizzle row, +16 KB (1024) to the second 64-column block
      // fully unrolled: the descriptors are formed once per call and advanced by
      // immediates, so each tcgen05.mma costs a handful of uniform-datapath instructions
      // (a rolled loop re-materialised them per MMA and capped the issue rate well below
      // the tensor pipe's 64 cycles per M128 N128 K16 MMA)
      auto issue_qk = [&](int qt, int ks, int nu) {
        const uint64_t da = sdesc(sbase + OFF_Q + qt * kTileBytes, 16, 1024);
        const uint64_t db = sdesc(sbase + OFF_K + ks * kTileBytes, 16, 1024);
        const uint32_t iqk = IQK0 | ((uint32_t)(nu >> 3) << 17);
        const uint32_t d = tmem + qt * 128;
#pragma unroll
        for (int k8 = 0; k8 < 8; ++k8) {
          const uint64_t off = (uint64_t)((k8 >> 2) * 1024 + (k8 & 3) * 2);
          mma_ss_w(d, da + off, db + off, iqk, k8 > 0);
        }
      };
      // K of the PV product = tile width (keys), 16 per MMA
      auto issue_pv = [&](int qt, int vs, bool acc, int nu) {
        const uint64_t dv = sdesc(sbase + OFF_V + vs * kTileBytes, 16384, 1024);
        const uint32_t d = tmem + 256 + qt * 128, a = tmem + qt * 128;
        const int nk = nu >> 4;
        mma_ts_w(d, a, dv, IPV, acc ? 1u : 0u);
#pragma unroll
        for (int k8 = 1; k8 < 8; ++k8)
          if (k8 < nk) mma_ts_w(d, a + k8 * 8, dv + (uint64_t)(k8 * 128), IPV, 1u);
      };
      int gt = 0, kk = 0;
      for (int idx = blockIdx.x; idx < n_items; idx += gridDim.x, ++kk) {
        const AttnParams& p = ITEM_PARAMS(idx);
        const Item w = decode_item(p, ITEM_LOCAL(idx));
        const int n = w.n_tiles;
        mbar_wait(bar(B_KF + gt % KST), (gt / KST) & 1);
        if (lane == 0) TRACE(EV_KF, gt);
        mbar_wait(bar(B_Q + 0), kk & 1);
        if (kk == 0 && lane == 0) TRACE(EV_Q, 0);
        tc_fence_after();
        int nu = tile_segments(p, w, w.t_begin).width;
        issue_qk(0, gt % KST, nu); mma_commit_w(bar(B_S + 0));
        mbar_wait(bar(B_Q + 1), kk & 1);
        tc_fence_after();
        issue_qk(1, gt % KST, nu); mma_commit_w(bar(B_S + 1));
        mma_commit_w(bar(B_KE + gt % KST));
        for (int jj = 0; jj < n; ++jj) {
          const int g = gt + jj, vs = g % VST;
          const int nu_next = jj + 1 < n ? tile_segments(p, w, w.t_begin + jj + 1).width : 0;
          mbar_wait(bar(B_VF + vs), (g / VST) & 1);
          if (lane == 0) TRACE(EV_VF, g);
          for (int qt = 0; qt < 2; ++qt) {
            mbar_wait(bar(B_P + qt), g & 1);
            if (jj == 0 && kk > 0) mbar_wait(bar(B_OF + qt), (kk - 1) & 1);   // previous item's O read
            if (lane == 0) TRACE(EV_PV0 + qt, g);
            tc_fence_after();
            issue_pv(qt, vs, jj > 0, nu);
            mma_commit_w(bar(B_O + qt));
            if (qt == 1) mma_commit_w(bar(B_VE + vs));
            if (jj + 1 < n) {
              const int ks = (g + 1) % KST;
              if (qt == 0) {
                mbar_wait(bar(B_KF + ks), ((g + 1) / KST) & 1);
                if (lane == 0) TRACE(EV_KF, g + 1);
                tc_fence_after();
              }
              issue_qk(qt, ks, nu_next);
              mma_commit_w(bar(B_S + qt));
              if (qt == 1) mma_commit_w(bar(B_KE + ks));
            }
          }
          nu = nu_next;
        }
        gt += n;
      }
      // drain: the last V-free commit tracks every MMA of this CTA
      if (gt > 0) mbar_wait(bar(B_VE + (gt - 1) % VST), ((gt - 1) / VST) & 1);
      if (lane == 0) TRACE(EV_END, 0);
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 14) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

}  // namespace tc

int attn_tc_smem_bytes() { return tc::kSmemBytes; }

cudaError_t make_ring_tmap(CUtensorMap* map, void* base, unsigned long long rows) {
  using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Encode encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || fn == nullptr) return e != cudaSuccess ? e : cudaErrorNotSupported;
    encode = reinterpret_cast<Encode>(fn);
  }
  const cuuint64_t dims[2] = {128, rows};   // rows = heads * (R + 128): ring + mirror
  const cuuint64_t strides[1] = {128 * 2};
  const cuuint32_t box[2] = {64, 128};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

static long long tc_items(const AttnParams& p) { return (long long)p.P * p.Hkv * p.n_mblocks * p.n_splits; }

cudaError_t launch_attn_tc2(const AttnParams& pa, const AttnParams* pb, cudaStream_t st) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(tc::attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         tc::kSmemBytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  static int num_sms = 0;
  if (num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const long long na = tc_items(pa), nb = pb ? tc_items(*pb) : 0;
  const long long items = na + nb;
  const unsigned grid = (unsigned)(items < num_sms ? items : num_sms);
  int ka = 0, kb = 0;
#if DSC_INTERLEAVE
  const long long G = (long long)pa.P * pa.Hkv;
  if (pb && nb > 0 && G == (long long)pb->P * pb->Hkv && na % G == 0 && nb % G == 0) {
    ka = (int)(na / G);
    kb = (int)(nb / G);
  }
#endif
  tc::attn_tc_kernel<<<grid, tc::kThreads, tc::kSmemBytes, st>>>(pa, pb ? *pb : pa, (int)na, (int)nb, ka, kb);
  return cudaGetLastError();
}

cudaError_t launch_attn_tc(const AttnParams& p, cudaStream_t st) { return launch_attn_tc2(p, nullptr, st); }

}  // namespace dsc
