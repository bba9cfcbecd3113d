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
// CTA = 14 warps:
//   warps 0-3  softmax of Q tile 0 (thread = query row = TMEM lane)
//   warps 4-7  softmax of Q tile 1
//   warps 8-11 rotation: Q (LDG -> rotate -> STS) once; then every raw K tile
//              in place in shared memory (LDS -> rotate -> STS), R(p+1) = R(p)R(1)
//   warp 12    copy: raw K and V tiles -> SW128 smem; TMA (2 x 64x128 boxes) for
//              ring tiles, cp.async for the sink/self tile
//   warp 13    TMEM allocator + single-thread tcgen05.mma issuer
// TMEM (512 cols): S0 [0,128) S1 [128,256) O0 [256,384) O1 [384,512);
// P_qt (bf16x2) overwrites S_qt cols [0,64) and feeds O_qt += P V as the TMEM A operand.
// MMA issue order S0_0 S1_0 | PV0_j S0_{j+1} PV1_j S1_{j+1} | ... so each softmax
// warpgroup overlaps the other Q tile's MMAs.
#include "dscache_internal.h"

#include <cuda_bf16.h>
#include <cstdint>

namespace dsc {
namespace tc {

constexpr int kNQT = 2;                       // Q tiles per CTA
constexpr int kWarps = 14;
constexpr int kThreads = kWarps * 32;
constexpr int kTileBytes = 128 * 128 * 2;     // one 128 x 128 bf16 tile
constexpr int KST = 3;                        // K stages (raw -> rotated in place)
constexpr int VST = 2;                        // V stages
constexpr int OFF_Q = 0;
constexpr int OFF_K = OFF_Q + kNQT * kTileBytes;
constexpr int OFF_V = OFF_K + KST * kTileBytes;
constexpr int OFF_BAR = OFF_V + VST * kTileBytes;
// barriers (8 B each): Q | K raw landed | K rotated | K free | V landed | V free | S | P | O
constexpr int B_Q = 0, B_KR = 1, B_KF = 4, B_KE = 7, B_VF = 10, B_VE = 12, B_S = 14, B_P = 16, B_O = 18, B_N = 20;
constexpr int kSmemBytes = OFF_BAR + B_N * 8 + 16 + 1024;   // + tmem slot + alignment slack
constexpr float kRescaleThreshold = 8.0f;     // log2 units (factor 256)

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
// Watchdog: a pipeline bug must not hang the GPU -- trap after ~2^31 cycles (~1 s).
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  if (mbar_try(bar, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try(bar, parity)) {
    if (clock64() - t0 > (1ll << 31)) __trap();
  }
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

__device__ __forceinline__ void mma_ss(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
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
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

__device__ __forceinline__ uint2 ldg64(const void* p) {
  uint2 r;
  asm volatile("ld.global.nc.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void sts64(uint32_t addr, uint32_t a, uint32_t b) {
  asm volatile("st.shared.v2.u32 [%0], {%1,%2};" ::"r"(addr), "r"(a), "r"(b) : "memory");
}

// byte offset of element (row, col) in a 128 x 128 bf16 tile stored as two
// 64-column SW128 blocks (16 KB each): the canonical K-major SWIZZLE_128B layout
// (8 rows x 128 B atoms, 16-byte chunk index XOR row%8).
__device__ __forceinline__ uint32_t sw128(int row, int col) {
  const int blk = col >> 6;
  const int byte = (col & 63) * 2;
  return (uint32_t)(blk * 16384 + row * 128 + ((((byte >> 4) ^ (row & 7))) << 4) + (byte & 15));
}

// Ring tile k covers slots [k*128, min(k*128+128, R)).  Valid keys of the window
// [start, start+cnt) (mod R) form one column interval [c_a, c_b) with logical ring
// index rel_a at c_a (needs R - cnt >= 128, guaranteed by tpf >= 128).
__device__ __forceinline__ void ring_tile_info(int k, int R, int start, int cnt, int& c_a, int& c_b, int& rel_a) {
  const int base = k * 128;
  const int width = min(128, R - base);
  if (start > base && start < base + width) {
    c_a = start - base;
    rel_a = 0;
  } else {
    c_a = 0;
    rel_a = base - start;
    if (rel_a < 0) rel_a += R;
  }
  const int rem = cnt - rel_a;
  c_b = rem > 0 ? min(width, c_a + rem) : c_a;
}

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
__device__ __forceinline__ uint2 lds64(uint32_t addr) {
  uint2 r;
  asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "r"(addr) : "memory");
  return r;
}
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

struct Work {
  int pp, g, mb, sp;
  long long head_row;
  int m0, rows_total;
  int cnt;            // ring keys needed by this m-block (causal cut)
  int k0, nT;         // first physical ring tile, number of physical tiles
  int t_begin, n_tiles;
};

__device__ __forceinline__ Work decode_work(const AttnParams& p) {
  Work w;
  int x = blockIdx.x;
  w.sp = x % p.n_splits; x /= p.n_splits;
  w.mb = p.n_mblocks - 1 - (x % p.n_mblocks); x /= p.n_mblocks;   // longest (causal) m-blocks first
  w.g = x % p.Hkv;
  w.pp = x / p.Hkv;
  const int s = w.pp / p.layer_count, l = w.pp % p.layer_count;
  w.head_row = ((long long)s * p.N_total + p.layer_begin + l) * p.Hkv + w.g;
  w.rows_total = p.n_q * p.grp;
  w.m0 = w.mb * (kNQT * 128);
  const int last_row = min(w.m0 + kNQT * 128, w.rows_total) - 1;
  const int lim_max = p.q_pos0 + last_row / p.grp;
  w.cnt = min(max(lim_max - p.A + 1, 0), p.ring_count);
  w.nT = (p.R + 127) / 128;
  w.k0 = p.ring_start / 128;
  int rt = 0;
  if (w.cnt > 0) {
    const int end = p.ring_start + w.cnt;
    rt = end <= p.R ? (end + 127) / 128 - w.k0 : (w.nT - w.k0) + (end - p.R + 127) / 128;
    rt = min(rt, w.nT);
  }
  const int total = 1 + rt;
  w.t_begin = min(w.sp * p.tiles_per_split, total);
  w.n_tiles = min(total, w.t_begin + p.tiles_per_split) - w.t_begin;
  return w;
}

// Key rows of tile u as (at most) two segments; key row r of segment s has id
// pos0_s + r.  Tile 0 = sink rows [0, A) + self rows [A, A+n_self); tile u > 0 =
// physical ring tile (k0 + u - 1) mod nT, valid rows [c_a, c_b).
struct TileSeg {
  int lo0, hi0, pos0_0;
  int lo1, hi1, pos0_1;
  int phys;           // physical ring tile (u > 0), -1 for tile 0
};

__device__ __forceinline__ TileSeg tile_segments(const AttnParams& p, const Work& w, int u) {
  TileSeg t;
  if (u == 0) {
    t.lo0 = 0; t.hi0 = p.A; t.pos0_0 = 0;
    t.lo1 = p.A; t.hi1 = p.A + p.n_self; t.pos0_1 = p.ring_count;
    t.phys = -1;
  } else {
    int k = w.k0 + u - 1;
    if (k >= w.nT) k -= w.nT;
    int c_a, c_b, rel_a;
    ring_tile_info(k, p.R, p.ring_start, w.cnt, c_a, c_b, rel_a);
    t.lo0 = c_a; t.hi0 = c_b; t.pos0_0 = p.A + rel_a - c_a;
    t.lo1 = 0; t.hi1 = 0; t.pos0_1 = 0;
    t.phys = k;
  }
  return t;
}
__device__ __forceinline__ int seg_pos(const TileSeg& t, int r) {
  if (r >= t.lo0 && r < t.hi0) return t.pos0_0 + r;
  if (r >= t.lo1 && r < t.hi1) return t.pos0_1 + r;
  return -1;
}

// ------------------------------------------------------------------ kernel
__global__ void __launch_bounds__(kThreads, 1) attn_tc_kernel(const __grid_constant__ AttnParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = su32(smem);
  const uint32_t bar0 = sbase + OFF_BAR;
  auto bar = [&](int i) { return bar0 + 8u * (uint32_t)i; };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + OFF_BAR + B_N * 8);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Work w = decode_work(p);

  if (threadIdx.x == 0) {
    mbar_init(bar(B_Q), 128);
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
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_proxy_async();
  }
  if (warp == 13) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (warp == 12 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tmap_k)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tmap_v)) : "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int n = w.n_tiles;
  const int A = p.A;

  if (warp < 8) {
    // ================================================================ softmax
    const int qt = warp >> 2, quarter = warp & 3;
    const int rloc = quarter * 32 + lane;
    const int rglob = w.m0 + qt * 128 + rloc;
    const bool valid_row = rglob < w.rows_total;
    const int qi = valid_row ? rglob / p.grp : 0;
    const int lim = valid_row ? p.q_pos0 + qi : -1;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const uint32_t tS = tmem + lane_off + (uint32_t)(qt * 128);
    const uint32_t tO = tmem + lane_off + (uint32_t)(256 + qt * 128);
    const float sl2 = p.scale_log2;
    const float2 scale2 = make_float2(sl2, sl2);
    float m = -INFINITY;
    float2 lsum2 = make_float2(0.f, 0.f);
    for (int jj = 0; jj < n; ++jj) {
      const int u = w.t_begin + jj;
      int c_lo, c_hi;
      if (!valid_row) {
        c_lo = 0; c_hi = 0;
      } else if (u == 0) {
        c_lo = 0;
        c_hi = min(A + p.n_self, max(A, lim - p.ring_count + 1));
      } else {
        const TileSeg t = tile_segments(p, w, u);
        c_lo = t.lo0;
        // key at column c has id pos0 + c; visible iff id <= lim
        c_hi = max(c_lo, min(t.hi0, lim - t.pos0_0 + 1));
      }
      const bool full = (c_lo == 0) && (c_hi == 128);
      mbar_wait(bar(B_S + qt), jj & 1);
      tc_fence_after();
      // pass 1: row max over the visible columns
      float mx = -INFINITY;
#pragma unroll 1
      for (int ch = 0; ch < 4; ++ch) {
        uint32_t r[32];
        tmem_ld32(tS + ch * 32, r);
        tmem_wait_ld();
        if (full) {
#pragma unroll
          for (int c = 0; c < 32; c += 2) mx = fmaxf(mx, fmaxf(__uint_as_float(r[c]), __uint_as_float(r[c + 1])));
        } else {
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            const int col = ch * 32 + c;
            if (col >= c_lo && col < c_hi) mx = fmaxf(mx, __uint_as_float(r[c]));
          }
        }
      }
      const float m_tile = mx * sl2;
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
        // O_qt holds PV up to tile jj-1: wait for it, rescale in TMEM
        mbar_wait(bar(B_O + qt), (jj - 1) & 1);
        tc_fence_after();
#pragma unroll 1
        for (int ch = 0; ch < 4; ++ch) {
          uint32_t r[32];
          tmem_ld32(tO + ch * 32, r);
          tmem_wait_ld();
#pragma unroll
          for (int c = 0; c < 32; ++c) r[c] = __float_as_uint(__uint_as_float(r[c]) * f);
          tmem_st32(tO + ch * 32, r);
        }
        tmem_wait_st();
      }
      const float m_use = (m == -INFINITY) ? 0.f : m;
      const float2 negm2 = make_float2(-m_use, -m_use);
      // pass 2: P = 2^(s*scale - m) -> bf16x2 into S cols [0,64)
#pragma unroll 1
      for (int ch = 0; ch < 4; ++ch) {
        uint32_t r[32];
        tmem_ld32(tS + ch * 32, r);
        tmem_wait_ld();
        uint32_t pk[16];
#pragma unroll
        for (int c = 0; c < 32; c += 2) {
          const float2 x = __ffma2_rn(make_float2(__uint_as_float(r[c]), __uint_as_float(r[c + 1])), scale2, negm2);
          float p0 = ex2(x.x), p1 = ex2(x.y);
          if (!full) {
            const int col = ch * 32 + c;
            p0 = (col >= c_lo && col < c_hi) ? p0 : 0.f;
            p1 = (col + 1 >= c_lo && col + 1 < c_hi) ? p1 : 0.f;
          }
          lsum2 = __fadd2_rn(lsum2, make_float2(p0, p1));
          pk[c >> 1] = pack_bf16(p0, p1);
        }
        tmem_st16(tS + ch * 16, pk);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(bar(B_P + qt));
    }
    // epilogue
    const float lsum = lsum2.x + lsum2.y;
    mbar_wait(bar(B_O + qt), (n - 1) & 1);
    tc_fence_after();
    const float inv = lsum > 0.f ? 1.f / lsum : 0.f;
    const int h = valid_row ? w.g * p.grp + rglob % p.grp : 0;
    const long long orow = ((long long)w.pp * p.n_q + qi) * p.Hq + h;
#pragma unroll 1
    for (int ch = 0; ch < 4; ++ch) {
      uint32_t r[32];
      tmem_ld32(tO + ch * 32, r);
      tmem_wait_ld();
      if (!valid_row) continue;
      if (p.n_splits == 1) {
        uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.o) + orow * 128 + ch * 32);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          uint4 o;
          o.x = pack_bf16(__uint_as_float(r[8 * v + 0]) * inv, __uint_as_float(r[8 * v + 1]) * inv);
          o.y = pack_bf16(__uint_as_float(r[8 * v + 2]) * inv, __uint_as_float(r[8 * v + 3]) * inv);
          o.z = pack_bf16(__uint_as_float(r[8 * v + 4]) * inv, __uint_as_float(r[8 * v + 5]) * inv);
          o.w = pack_bf16(__uint_as_float(r[8 * v + 6]) * inv, __uint_as_float(r[8 * v + 7]) * inv);
          dst[v] = o;
        }
      } else {
        const long long rows = (long long)p.P * p.n_q * p.Hq;
        float4* dst = reinterpret_cast<float4*>(p.ws_o + ((long long)w.sp * rows + orow) * 128 + ch * 32);
#pragma unroll
        for (int v = 0; v < 8; ++v)
          dst[v] = make_float4(__uint_as_float(r[4 * v]) * inv, __uint_as_float(r[4 * v + 1]) * inv,
                               __uint_as_float(r[4 * v + 2]) * inv, __uint_as_float(r[4 * v + 3]) * inv);
        if (ch == 0)
          p.ws_lse[(long long)w.sp * rows + orow] = lsum > 0.f ? m + __log2f(lsum) : -INFINITY;
      }
    }
  } else if (warp < 12) {
    // ================================================================ rotation (Q once, then K tiles)
    const int lt = threadIdx.x - 256;
    const int c = lt & 15;             // frequency chunk: freqs 4c..4c+3 (elements 4c.. and 64+4c..)
    const int rgrp = lt >> 4;          // 0..7
    const __nv_bfloat16* __restrict__ Qg = reinterpret_cast<const __nv_bfloat16*>(p.q);
    const bool dbg = p.dbg_pos != nullptr && w.pp == 0 && w.g == 0;
    const float4* __restrict__ rope4 = reinterpret_cast<const float4*>(p.rope);   // [pos][32] float4
    // ---- Q: 256 rows, thread rows rgrp*32 .. +31, rotated at the query id (table values)
#pragma unroll 1
    for (int rb = 0; rb < 32; rb += 8) {
      uint2 lo[8], hi[8];
      int pos[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int r = rgrp * 32 + rb + k;
        const int rg = w.m0 + r;
        pos[k] = -1;
        lo[k] = make_uint2(0, 0); hi[k] = make_uint2(0, 0);
        if (rg < w.rows_total) {
          const int i = rg / p.grp, h = w.g * p.grp + rg % p.grp;
          const __nv_bfloat16* src = Qg + (((long long)w.pp * p.n_q + i) * p.Hq + h) * 128;
          lo[k] = ldg64(src + 4 * c);
          hi[k] = ldg64(src + 64 + 4 * c);
          pos[k] = p.q_pos0 + i;
          if (dbg && c == 0 && (rg % p.grp) == 0) p.dbg_pos[A + p.R + p.dbg_M + i] = pos[k];
        }
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int r = rgrp * 32 + rb + k;
        const int qt = r >> 7, rl = r & 127;
        uint32_t olo0 = 0, olo1 = 0, ohi0 = 0, ohi1 = 0;
        if (pos[k] >= 0) {
          const float4 cs0 = rope4[(long long)pos[k] * 32 + 2 * c];
          const float4 cs1 = rope4[(long long)pos[k] * 32 + 2 * c + 1];
          const float a0 = bf_lo(lo[k].x), a1 = bf_hi(lo[k].x), a2 = bf_lo(lo[k].y), a3 = bf_hi(lo[k].y);
          const float b0 = bf_lo(hi[k].x), b1 = bf_hi(hi[k].x), b2 = bf_lo(hi[k].y), b3 = bf_hi(hi[k].y);
          olo0 = pack_bf16(a0 * cs0.x - b0 * cs0.y, a1 * cs0.z - b1 * cs0.w);
          olo1 = pack_bf16(a2 * cs1.x - b2 * cs1.y, a3 * cs1.z - b3 * cs1.w);
          ohi0 = pack_bf16(a0 * cs0.y + b0 * cs0.x, a1 * cs0.w + b1 * cs0.z);
          ohi1 = pack_bf16(a2 * cs1.y + b2 * cs1.x, a3 * cs1.w + b3 * cs1.z);
        }
        const uint32_t qb = sbase + OFF_Q + qt * kTileBytes;
        sts64(qb + sw128(rl, 4 * c), olo0, olo1);
        sts64(qb + sw128(rl, 64 + 4 * c), ohi0, ohi1);
      }
    }
    fence_proxy_async();
    mbar_arrive(bar(B_Q));

    // per-thread rotation step R(theta_f), f = 4c..4c+3 (table row of id 1), packed by freq pairs
    const float4 st0 = rope4[32 + 2 * c], st1 = rope4[32 + 2 * c + 1];
    const float2 cth01 = make_float2(st0.x, st0.z), sth01 = make_float2(st0.y, st0.w);
    const float2 cth23 = make_float2(st1.x, st1.z), sth23 = make_float2(st1.y, st1.w);
#pragma unroll 1
    for (int jj = 0; jj < n; ++jj) {
      const int u = w.t_begin + jj, ks = jj % KST;
      const TileSeg t = tile_segments(p, w, u);
      const uint32_t kb = sbase + OFF_K + ks * kTileBytes;
      mbar_wait(bar(B_KR + ks), (jj / KST) & 1);
      float2 c01 = make_float2(1.f, 1.f), s01 = make_float2(0.f, 0.f);
      float2 c23 = c01, s23 = s01;
      int prev = -2;
#pragma unroll 4
      for (int k = 0; k < 16; ++k) {
        const int r = rgrp * 16 + k;
        const int pos = seg_pos(t, r);
        const uint32_t alo = kb + sw128(r, 4 * c), ahi = kb + sw128(r, 64 + 4 * c);
        if (pos < 0) {       // no key in this row: clear whatever the copy left there
          sts64(alo, 0, 0);
          sts64(ahi, 0, 0);
          prev = -2;
          continue;
        }
        if (dbg && c == 0) {
          const int di = (u == 0) ? (r < A ? r : A + p.R + (r - A)) : A + t.phys * 128 + r;
          p.dbg_pos[di] = pos;
        }
        if (pos == prev + 1) {   // R((p+1) theta) = R(p theta) R(theta)
          const float2 nc01 = __ffma2_rn(c01, cth01, __fmul2_rn(make_float2(-s01.x, -s01.y), sth01));
          const float2 ns01 = __ffma2_rn(s01, cth01, __fmul2_rn(c01, sth01));
          const float2 nc23 = __ffma2_rn(c23, cth23, __fmul2_rn(make_float2(-s23.x, -s23.y), sth23));
          const float2 ns23 = __ffma2_rn(s23, cth23, __fmul2_rn(c23, sth23));
          c01 = nc01; s01 = ns01; c23 = nc23; s23 = ns23;
        } else {                 // exact table value (fp64-built) at a segment start
          const float4 a = rope4[(long long)pos * 32 + 2 * c];
          const float4 b = rope4[(long long)pos * 32 + 2 * c + 1];
          c01 = make_float2(a.x, a.z); s01 = make_float2(a.y, a.w);
          c23 = make_float2(b.x, b.z); s23 = make_float2(b.y, b.w);
        }
        prev = pos;
        const uint2 lo = lds64(alo), hi = lds64(ahi);
        const float2 a01 = make_float2(bf_lo(lo.x), bf_hi(lo.x)), a23 = make_float2(bf_lo(lo.y), bf_hi(lo.y));
        const float2 b01 = make_float2(bf_lo(hi.x), bf_hi(hi.x)), b23 = make_float2(bf_lo(hi.y), bf_hi(hi.y));
        // y_lo = a cos - b sin ; y_hi = a sin + b cos
        const float2 ylo01 = __ffma2_rn(a01, c01, __fmul2_rn(make_float2(-b01.x, -b01.y), s01));
        const float2 ylo23 = __ffma2_rn(a23, c23, __fmul2_rn(make_float2(-b23.x, -b23.y), s23));
        const float2 yhi01 = __ffma2_rn(a01, s01, __fmul2_rn(b01, c01));
        const float2 yhi23 = __ffma2_rn(a23, s23, __fmul2_rn(b23, c23));
        sts64(alo, pack_bf16(ylo01.x, ylo01.y), pack_bf16(ylo23.x, ylo23.y));
        sts64(ahi, pack_bf16(yhi01.x, yhi01.y), pack_bf16(yhi23.x, yhi23.y));
      }
      fence_proxy_async();
      mbar_arrive(bar(B_KF + ks));
    }
  } else if (warp == 12) {
    // ================================================================ copy warp
    const __nv_bfloat16* __restrict__ SK = reinterpret_cast<const __nv_bfloat16*>(p.sink_k);
    const __nv_bfloat16* __restrict__ SV = reinterpret_cast<const __nv_bfloat16*>(p.sink_v);
    const __nv_bfloat16* __restrict__ XK = reinterpret_cast<const __nv_bfloat16*>(p.self_k);
    const __nv_bfloat16* __restrict__ XV = reinterpret_cast<const __nv_bfloat16*>(p.self_v);
    // tile 0 (sink rows [0,A) + self rows [A, A+n_self), zeros elsewhere) with cp.async
    auto copy_extra = [&](uint32_t dst, const __nv_bfloat16* sink, const __nv_bfloat16* self) {
#pragma unroll 4
      for (int it = 0; it < 64; ++it) {
        const int idx = it * 32 + lane;          // 2048 16-byte chunks
        const int r = idx >> 4, ch = idx & 15;
        const __nv_bfloat16* src = nullptr;
        if (r < A) src = sink + (w.head_row * A + r) * 128;
        else if (r < A + p.n_self) src = self + (((long long)w.pp * p.n_self + (r - A)) * p.Hkv + w.g) * 128;
        const uint32_t d = dst + (ch >> 3) * 16384 + r * 128 + (((ch & 7) ^ (r & 7)) << 4);
        cp_async16(d, src ? (const void*)(src + 8 * ch) : (const void*)sink, src ? 16u : 0u);
      }
      cp_async_wait_all();
      fence_proxy_async();
      __syncwarp();
    };
#pragma unroll 1
    for (int jj = 0; jj < n; ++jj) {
      const int u = w.t_begin + jj;
      int phys = -1;
      if (u > 0) {
        phys = w.k0 + u - 1;
        if (phys >= w.nT) phys -= w.nT;
      }
      const int row = (int)(w.head_row * p.R) + phys * 128;
      const int ks = jj % KST, vs = jj % VST;
      if (jj >= KST) mbar_wait(bar(B_KE + ks), ((jj - KST) / KST) & 1);
      const uint32_t kdst = sbase + OFF_K + ks * kTileBytes;
      if (u == 0) {
        copy_extra(kdst, SK, XK);
        if (lane == 0) mbar_arrive(bar(B_KR + ks));
      } else if (lane == 0) {
        mbar_arrive_tx(bar(B_KR + ks), kTileBytes);
        tma_load_2d(kdst, &p.tmap_k, 0, row, bar(B_KR + ks));
        tma_load_2d(kdst + 16384, &p.tmap_k, 64, row, bar(B_KR + ks));
      }
      if (jj >= VST) mbar_wait(bar(B_VE + vs), ((jj - VST) / VST) & 1);
      const uint32_t vdst = sbase + OFF_V + vs * kTileBytes;
      if (u == 0) {
        copy_extra(vdst, SV, XV);
        if (lane == 0) mbar_arrive(bar(B_VF + vs));
      } else if (lane == 0) {
        mbar_arrive_tx(bar(B_VF + vs), kTileBytes);
        tma_load_2d(vdst, &p.tmap_v, 0, row, bar(B_VF + vs));
        tma_load_2d(vdst + 16384, &p.tmap_v, 64, row, bar(B_VF + vs));
      }
      __syncwarp();
    }
  } else if (lane == 0) {
    // ================================================================ MMA issuer (warp 13)
    constexpr uint32_t IQK = idesc_bf16(128, 128, 0, 0);   // S = Q K^T, both K-major
    constexpr uint32_t IPV = idesc_bf16(128, 128, 0, 1);   // O += P V, P from TMEM, V MN-major
    auto issue_qk = [&](int qt, int ks) {
      const uint32_t qa = sbase + OFF_Q + qt * kTileBytes, kb = sbase + OFF_K + ks * kTileBytes;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
        mma_ss(tmem + qt * 128, sdesc(qa + off, 16, 1024), sdesc(kb + off, 16, 1024), IQK, kk > 0);
      }
    };
    auto issue_pv = [&](int qt, int vs, bool acc) {
      const uint32_t vb = sbase + OFF_V + vs * kTileBytes;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        mma_ts(tmem + 256 + qt * 128, tmem + qt * 128 + kk * 8, sdesc(vb + kk * 2048, 16384, 1024), IPV,
               (acc || kk > 0) ? 1u : 0u);
    };
    mbar_wait(bar(B_Q), 0);
    mbar_wait(bar(B_KF + 0), 0);
    tc_fence_after();
    issue_qk(0, 0); mma_commit(bar(B_S + 0));
    issue_qk(1, 0); mma_commit(bar(B_S + 1));
    mma_commit(bar(B_KE + 0));
    for (int jj = 0; jj < n; ++jj) {
      const int vs = jj % VST;
      mbar_wait(bar(B_VF + vs), (jj / VST) & 1);
      for (int qt = 0; qt < 2; ++qt) {
        mbar_wait(bar(B_P + qt), jj & 1);
        tc_fence_after();
        issue_pv(qt, vs, jj > 0);
        mma_commit(bar(B_O + qt));
        if (qt == 1) mma_commit(bar(B_VE + vs));
        if (jj + 1 < n) {
          const int ks = (jj + 1) % KST;
          if (qt == 0) {
            mbar_wait(bar(B_KF + ks), ((jj + 1) / KST) & 1);
            tc_fence_after();
          }
          issue_qk(qt, ks);
          mma_commit(bar(B_S + qt));
          if (qt == 1) mma_commit(bar(B_KE + ks));
        }
      }
    }
    // drain: the last V-free commit tracks every MMA of this CTA
    mbar_wait(bar(B_VE + (n - 1) % VST), ((n - 1) / VST) & 1);
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 13) {
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
  const cuuint64_t dims[2] = {128, rows};
  const cuuint64_t strides[1] = {128 * 2};
  const cuuint32_t box[2] = {64, 128};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t launch_attn_tc(const AttnParams& p, cudaStream_t st) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(tc::attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         tc::kSmemBytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const long long blocks = (long long)p.P * p.Hkv * p.n_mblocks * p.n_splits;
  tc::attn_tc_kernel<<<(unsigned)blocks, tc::kThreads, tc::kSmemBytes, st>>>(p);
  return cudaGetLastError();
}

}  // namespace dsc
