// K3/K4 v7: fused rotate-on-load RoPE + GQA flash attention on the sm_100a tensor cores
// (tcgen05.mma, accumulators in TMEM) for both dscache_build_instant (Eq. 7: instant
// tokens over [sink | instant], causal) and dscache_attend (Eq. 8 + self: the query chunk
// over [sink | past | instant | self]).
//
// Position-agnostic encoding (Def. 4.1): the ring holds raw K; every K
// tile of an attend item is rotated in shared memory at its use-time ids (consecutive from
// 0) once for the 256 query rows that share it; a staged build reads K that
// the staging kernel already rotated at the build ids.  Softmax a_ij = softmax(Q_i K_j /
// sqrt(d)) in the exp2 domain with lazy rescale.
//
// Structure (one CTA per SM, persistent over work items = (problem, kv head, 256-row
// m-block, key split)):
//   * 128-key tiles: QK^T is one SS MMA of M = 128, N = 128 per K16 step (full tensor rate;
//     N = 64 SS MMAs run at 2/3 rate, scripts/micro/mma_bench), PV a TS MMA (P in TMEM).
//   * Two 128-row Q tiles per item ping-pong on the tensor core: while softmax warpgroup 0
//     works on S0(j), the MMA computes PV1(j-1) and S1(j); while warpgroup 1 works on S1(j),
//     PV0(j) and S0(j+1).  TMEM (512 columns): S0 = cols 0..127, S1 = 128..255, O0 = 256..383,
//     O1 = 384..511; P_qt (bf16x2, 64 columns) overwrites the first half of S_qt and is the
//     TMEM A operand of O_qt += P_qt V.  S_qt(j+1) is issued after PV_qt(j) (tcgen05 MMAs of
//     one CTA execute in issue order), so the commit of S_qt(j) also tells the softmax that
//     O_qt is quiescent (PV_qt(j-1) done): the lazy O rescale needs no extra wait.
//   * Shared memory: 3 Q tile buffers (item k uses buffers (2k) % 3 and (2k+1) % 3, so the
//     next item's first Q tile is loaded and rotated while the current item runs), 2 K and
//     2 V stages of 32 KB (128 keys x 256 B, two 64-column SW128 blocks).
//
// CTA = 16 warps:
//   warps 0-3  softmax of Q tile 0 (thread = query row = TMEM lane) + its O epilogue
//   warps 4-7  softmax of Q tile 1
//   warps 8-11 rotation: raw K tiles of attend items in place in smem, the Q tiles of every
//              item (loaded and rotated in registers at the query ids, then stored) one item
//              ahead, and the O epilogue of plain launches
//   warp 12    K copy (TMA box 64 cols x 128 rows; cp.async for sink/self tiles)
//   warp 13    V copy
//   warp 14    TMEM allocator + MMA issuer of Q tile 0 (S0, PV0; one elected lane issues)
//   warp 15    MMA issuer of Q tile 1 (S1, PV1); both commit to the shared K / V free barriers
#include "tc_common.cuh"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <utility>
#include <vector>

namespace dsc {
namespace fa {
using namespace tcc;

constexpr int BN = kTileN;                    // keys per K/V tile (128)
constexpr int kWarps = 16;
constexpr int kThreads = kWarps * 32;
constexpr int kQBytes = 128 * 128 * 2;        // one 128-row Q tile (2 x 64-column SW128 blocks)
constexpr int kKVHalf = BN * 128;             // one 64-column SW128 block of a K/V tile (16 KB)
constexpr int kKVBytes = 2 * kKVHalf;         // one K or V tile (32 KB)
constexpr int NQB = 3;                        // Q tile buffers
#ifndef FA_KST
#define FA_KST 2
#endif
#ifndef FA_VST
#define FA_VST 2
#endif
constexpr int KST = FA_KST, VST = FA_VST;
constexpr int OFF_Q = 0;
constexpr int OFF_K = OFF_Q + NQB * kQBytes;
constexpr int OFF_V = OFF_K + KST * kKVBytes;
constexpr int OFF_BAR = OFF_V + VST * kKVBytes;
// barriers (8 B each)
constexpr int B_QR = 0;                 // [NQB] Q tile buffer ready (128 arrivals)
constexpr int B_QF = B_QR + NQB;        // [NQB] Q tile buffer free (MMA commit after its item's last QK^T)
constexpr int B_KR = B_QF + NQB;        // [KST] K landed (TMA tx / copy warp arrive)
constexpr int B_KF = B_KR + KST;        // [KST] K rotated (128 arrivals; attend tiles only)
constexpr int B_KE = B_KF + KST;        // [KST] K stage free (commit after S1)
constexpr int B_VR = B_KE + KST;        // [VST] V landed
constexpr int B_VE = B_VR + VST;        // [VST] V stage free (commit after PV1)
constexpr int B_S = B_VE + VST;         // [2] S_qt ready (commit)
constexpr int B_P = B_S + 2;            // [2] P_qt ready (128 arrivals)
constexpr int B_O = B_P + 2;            // [2] O_qt final for the item (commit after its last PV)
constexpr int B_OF = B_O + 2;           // [2] O_qt read out by the epilogue (128 arrivals)
constexpr int B_LR = B_OF + 2;          // 1/l of an item's 256 rows written (256 softmax arrivals)
constexpr int B_LF = B_LR + 1;          // ... and read by the epilogue warpgroup (128 arrivals)
constexpr int B_N = B_LF + 1;
constexpr int OFF_L = OFF_BAR + B_N * 8 + 16;                  // 1/l handoff [256] fp32
constexpr int kSmemBytes = OFF_L + 256 * 4 + 1024;             // + alignment slack
static_assert(kSmemBytes <= 227 * 1024, "shared memory budget");
// setmaxnreg budget: 2 softmax warpgroups + rotation + (copy, MMA) <= 512 per thread x 128
#ifndef FA_REG_SM
#define FA_REG_SM 152
#endif
constexpr int kRegSoftmax = FA_REG_SM, kRegRotate = 136, kRegCopy = 512 - 2 * FA_REG_SM - 136;
static_assert(kRegCopy >= 40, "copy/MMA warps need registers");
static_assert(kRegCopy % 8 == 0 && kRegSoftmax % 8 == 0 && kRegRotate % 8 == 0, "setmaxnreg takes multiples of 8");
static_assert(kRegSoftmax > 128 && kRegCopy < 128, "launch allocation is 128 per thread: softmax grows, copy/MMA shrink");
constexpr float kRescaleThreshold = 8.0f;    // log2 units: move the running max only when it grew by > 2^8

// ablation knobs (timing experiments only; results are wrong when set): FA_ABL_SOFTMAX skips
// the softmax body, FA_ABL_ROT the K rotation, FA_ABL_EPI the O read-out and stores,
// FA_ABL_Q the Q loads + rotation, FA_ABL_PV the PV MMAs
#ifndef FA_ABL_SOFTMAX
#define FA_ABL_SOFTMAX 0
#endif
#ifndef FA_ABL_ROT
#define FA_ABL_ROT 0
#endif
#ifndef FA_ABL_EPI
#define FA_ABL_EPI 0
#endif
#ifndef FA_ABL_Q
#define FA_ABL_Q 0
#endif
#ifndef FA_ABL_PV
#define FA_ABL_PV 0
#endif
// FA_TRACE 1 (profiling variant): clock64 of pipeline events into p.trace, layout
// [ntrace_cta][kFtEvents][kFtIdx] for the first ntrace_cta CTAs; per-tile events are indexed
// by the CTA's tile counter g, per-item events by the CTA's item counter
#ifndef FA_TRACE
#define FA_TRACE 0
#endif
constexpr int kFtEvents = 32, kFtIdx = 1024;
enum {
  FT_MMA_P0 = 0, FT_MMA_P1, FT_MMA_K, FT_MMA_V, FT_SM0_S, FT_SM0_P, FT_SM1_S, FT_SM1_P, FT_ROT_KR, FT_ROT_KF,
  FT_CPK, FT_CPV,                                                                // per tile
  FT_MMA_ITEM = 12, FT_MMA_Q0, FT_MMA_Q1, FT_EPI0_O, FT_EPI0_END, FT_QE_START, FT_QE_END, FT_QO_START, FT_QO_FREE,
  FT_QO_END, FT_MMA_OF, FT_EPI1_O, FT_EPI1_END, FT_END,                           // per item
  FT_SMX_LD0 = 26, FT_SMX_EX0, FT_SMX_LD1, FT_SMX_EX1,                              // per tile, warp 0 steps
  FT_MMA_PV0I = 30, FT_MMA_S0I                                                      // per tile, MMA issue done
};
#if FA_TRACE
#define FT(ev, i)                                                                                      \
  do {                                                                                                 \
    if (ft_cta && (i) < kFtIdx) ft_cta[(ev) * kFtIdx + (i)] = clock64();                                \
  } while (0)
#else
#define FT(ev, i) do { } while (0)
#endif

// S = Q K^T over K = 128 (8 x K16), N = tile width: A (Q tile, 128 rows) and B (K tile,
// 128 rows) SW128 K-major; the second 64-column block of either is +16 KB (1024 x 16 B).
__device__ __forceinline__ void mma_qk(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc) {
  asm volatile(
      "{\n.reg .pred e;\n.reg .b64 a1, a2, a3, a4, a5, a6, a7, b1, b2, b3, b4, b5, b6, b7;\n"
      "add.s64 a1, %1, 2; add.s64 a2, %1, 4; add.s64 a3, %1, 6;\n"
      "add.s64 a4, %1, 1024; add.s64 a5, %1, 1026; add.s64 a6, %1, 1028; add.s64 a7, %1, 1030;\n"
      "add.s64 b1, %2, 2; add.s64 b2, %2, 4; add.s64 b3, %2, 6;\n"
      "add.s64 b4, %2, 1024; add.s64 b5, %2, 1026; add.s64 b6, %2, 1028; add.s64 b7, %2, 1030;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %3, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a4, b4, %3, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a5, b5, %3, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a6, b6, %3, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a7, b7, %3, 1;\n}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc)
      : "memory");
}
// O += P V over a full 128-key tile (8 x K16): A (P) in TMEM, 8 columns per K16 step; B (V)
// MN-major SW128, 16 keys = 2048 B (128 x 16 B) per step.  acc = 0 overwrites O.
__device__ __forceinline__ void mma_pv8(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred e, p;\n.reg .b64 b1, b2, b3, b4, b5, b6, b7;\n.reg .b32 t1, t2, t3, t4, t5, t6, t7;\n"
      "add.s64 b1, %2, 128; add.s64 b2, %2, 256; add.s64 b3, %2, 384;\n"
      "add.s64 b4, %2, 512; add.s64 b5, %2, 640; add.s64 b6, %2, 768; add.s64 b7, %2, 896;\n"
      "add.u32 t1, %1, 8; add.u32 t2, %1, 16; add.u32 t3, %1, 24;\n"
      "add.u32 t4, %1, 32; add.u32 t5, %1, 40; add.u32 t6, %1, 48; add.u32 t7, %1, 56;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t1], b1, %3, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t2], b2, %3, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t3], b3, %3, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t4], b4, %3, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t5], b5, %3, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t6], b6, %3, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t7], b7, %3, 1;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

// Watchdog record (debugging a pipeline deadlock): a wait that spins ~2^31 cycles writes
// (cta, warp, barrier index, parity, clock) into a host-mapped buffer, readable after the
// context has died, then traps.  Null (default) = just trap.
__device__ unsigned long long* g_fa_wd = nullptr;
__device__ long long g_fa_wd_lim = 1ll << 31;   // clk before a stuck wait traps (DSC_WATCHDOG_CLK)
__device__ __noinline__ void fa_wd_fail(uint32_t bar_off, uint32_t parity) {
  unsigned long long* wd = g_fa_wd;
  if (wd) {
    const unsigned long long i = atomicAdd(wd, 1ull);
    if (i < 64) {
      volatile unsigned long long* rec = wd + 1 + 4 * i;
      rec[0] = blockIdx.x;
      rec[1] = threadIdx.x >> 5;
      rec[2] = ((unsigned long long)bar_off << 32) | parity;
      rec[3] = clock64();
      __threadfence_system();
    }
  }
  __trap();
}
// The limit is read once per blocked wait, before the spin (the asm "memory" clobbers would
// otherwise reload it from global memory on every iteration).
__device__ __forceinline__ void fwait(uint32_t bar, uint32_t parity, uint32_t bar0) {
  if (mbar_try(bar, parity)) return;
  const long long lim = g_fa_wd_lim;
  const long long t0 = clock64();
  while (!mbar_try(bar, parity)) {
    if (clock64() - t0 > lim) fa_wd_fail((bar - bar0) / 8, parity);
  }
}

// 2^x on the MUFU (not volatile: the compiler may schedule it like any arithmetic)
__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void tmem_ld32x(uint32_t taddr, uint32_t* r) {
  tmem_ld32(taddr, *reinterpret_cast<uint32_t(*)[32]>(r));
}

// Q tile qt of item w (rows m0 + 128 qt .. +127 = (query, head) pairs) loaded straight from
// global memory into registers and rotated there at the query ids; the caller stores the 16
// chunks into the SW128 tile once its buffer is free (so the HBM latency of the load runs
// before the wait, not after it).  Thread lt holds frequencies 8*c8 .. 8*c8+7 (16-byte chunk
// c8 of the low and the high 64-column block) of rows rg8*8 .. +7.
__device__ __forceinline__ void load_rotate_q_regs(const AttnParams& p, const Item& w, int qt, int lt,
                                                   uint4 (&lo)[8], uint4 (&hi)[8]) {
  const float4* __restrict__ rp = p.rope_pairs;
  const __nv_bfloat16* __restrict__ Qg = reinterpret_cast<const __nv_bfloat16*>(p.q);
  const int c8 = lt & 7, rg8 = lt >> 3;
  const int row0 = w.m0 + qt * 128 + rg8 * 8;
  // debug export (set_debug): every problem, kv head 0, block [head_row / Hkv] of the buffer
  const bool dbg = p.dbg_pos != nullptr && w.g == 0 && c8 == 0;
  int* const dbgp = dbg ? p.dbg_pos + (w.head_row / p.Hkv) * p.dbg_len : nullptr;
  const __nv_bfloat16* qbase = Qg + ((long long)w.pp * p.n_q) * p.Hq * 128 + (long long)w.g * p.grp * 128 + 8 * c8;
  int pos[8];
  {
    int i = row0 / p.grp, hh = row0 % p.grp;
#pragma unroll
    for (int k = 0; k < 8; ++k) {   // all 16 loads in flight before any use
      const bool ok = row0 + k < w.rows_total;
      pos[k] = ok ? p.q_pos0 + i : -1;
      if (dbg && hh == 0 && ok) dbgp[p.dbg_A + p.dbg_R + p.dbg_M + i] = pos[k];
      if (ok) {
        const __nv_bfloat16* src = qbase + ((long long)i * p.Hq + hh) * 128;
        DSC_ASSERT(i < p.n_q && w.pp < p.P, "attn_fa Q row");
        lo[k] = ldg128(src);
        hi[k] = ldg128(src + 64);
      } else {
        lo[k] = hi[k] = make_uint4(0, 0, 0, 0);
      }
      if (++hh == p.grp) { hh = 0; ++i; }
    }
  }
  float2 cth[4], sth[4], cs[4], sn[4];
  const int p0 = max(pos[0], 0);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float4 t = rp[32 + 4 * c8 + j];
    cth[j] = make_float2(t.x, t.y);
    sth[j] = make_float2(t.z, t.w);
    const float4 u = rp[(long long)p0 * 32 + 4 * c8 + j];
    cs[j] = make_float2(u.x, u.y);
    sn[j] = make_float2(u.z, u.w);
  }
  int prev = p0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int pk = pos[k];
    if (pk < 0) continue;   // padding row: zeros
    if (pk == prev + 1) {   // next query id: advance (cos, sin) by R(theta)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 nc = __ffma2_rn(cs[j], cth[j], __fmul2_rn(make_float2(-sn[j].x, -sn[j].y), sth[j]));
        sn[j] = __ffma2_rn(sn[j], cth[j], __fmul2_rn(cs[j], sth[j]));
        cs[j] = nc;
      }
    } else if (pk != prev) {
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
    lo[k] = make_uint4(ol[0], ol[1], ol[2], ol[3]);
    hi[k] = make_uint4(oh[0], oh[1], oh[2], oh[3]);
  }
}

// Item of a host-decoded record (sched.cu item_table): per-item fields from the record,
// per-launch ones from its parameter block
__device__ __forceinline__ Item item_of(const AttnParams& p, const ItemRec& r) {
  Item w;
  w.pp = r.pp; w.g = r.flags >> 8; w.sp = r.sp; w.mb = r.m0 >> 8;
  w.head_row = r.head_row; w.m0 = r.m0; w.rows_total = p.n_q * p.grp; w.cnt = r.cnt;
  w.n_extra = (p.A + p.n_self + BN - 1) / BN; w.t_begin = r.t_begin; w.n_tiles = r.n_tiles;
  w.A = p.A; w.n_self = p.n_self; w.ring_count = p.ring_count; w.ring_start = p.ring_start; w.R = p.R;
  w.Rp = p.Rp; w.staged = p.staged;
  return w;
}
__device__ __forceinline__ ItemRec load_rec(const ItemRec* __restrict__ recs, int i) {
  const int4 a = __ldg(reinterpret_cast<const int4*>(recs + i));
  const int4 b = __ldg(reinterpret_cast<const int4*>(recs + i) + 1);
  ItemRec r;
  r.pp = a.x; r.head_row = a.y; r.m0 = a.z; r.t_begin = a.w; r.n_tiles = b.x; r.cnt = b.y; r.flags = b.z; r.sp = b.w;
  return r;
}

// ------------------------------------------------------------------ kernel
// Items [0, na) use pa, [na, na + nb) use pb (the fused step: attend items first, then the
// build items).
__global__ void __launch_bounds__(kThreads, 1)
    attn_fa_kernel(const __grid_constant__ AttnParams pa, const __grid_constant__ AttnParams pb, int na, int nb) {
  const AttnParams& p = pa;   // launch-wide fields (rope table, trace) are shared
#if FA_TRACE
  long long* const ft_cta = (pa.trace && blockIdx.x < (unsigned)pa.ntrace_cta)
                                ? pa.trace + (long long)blockIdx.x * kFtEvents * kFtIdx : nullptr;
#endif
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = ((uint32_t)__cvta_generic_to_shared(smem_raw) + 1023u) & ~1023u;
  const uint32_t bar0 = sbase + OFF_BAR;
  auto bar = [&](int i) { return bar0 + 8u * (uint32_t)i; };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + OFF_BAR + B_N * 8);
  float* lbuf = reinterpret_cast<float*>(smem + OFF_L);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_items = na + nb;
#define REC_PARAMS(R) (((R).flags & 1) ? pb : pa)

  if (threadIdx.x == 0) {
    for (int i = 0; i < NQB; ++i) {
      mbar_init(bar(B_QR + i), 128);
      mbar_init(bar(B_QF + i), 1);
    }
    for (int i = 0; i < KST; ++i) {
      mbar_init(bar(B_KR + i), 1);
      mbar_init(bar(B_KF + i), 128);
      mbar_init(bar(B_KE + i), 2);   // one commit per MMA issuer
    }
    for (int i = 0; i < VST; ++i) {
      mbar_init(bar(B_VR + i), 1);
      mbar_init(bar(B_VE + i), 2);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar(B_S + i), 1);
      mbar_init(bar(B_P + i), 128);
      mbar_init(bar(B_O + i), 1);
      mbar_init(bar(B_OF + i), 128);
    }
    {
      mbar_init(bar(B_LR), 256);
      mbar_init(bar(B_LF), 128);
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
  // all 512 columns of this SM's TMEM: the allocation starts at lane 0, column 0; the
  // descriptors take the returned base (no assumption about its value)
  const uint32_t tmem = *tmem_slot;

  // this CTA's items, in order: host-decoded records (sched.cu item_table); every role walks
  // the same sequence
  const ItemRec* __restrict__ recs = pa.item_recs + pa.item_off[blockIdx.x];
  const int n_my = pa.item_off[blockIdx.x + 1] - pa.item_off[blockIdx.x];
  // Q tile use u = 2 * item + qt lives in buffer u % 3
  auto qbuf_addr = [&](int u) { return sbase + OFF_Q + (uint32_t)((u % NQB) * kQBytes); };

  if (warp < 8) {
    // ================================================================ softmax + epilogue
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegSoftmax));
    const int qt = warp >> 2, quarter = warp & 3;
    const int rloc = quarter * 32 + lane;
    const int lt = threadIdx.x - qt * 128;           // 0..127 within the warpgroup
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const uint32_t tS = tmem + lane_off + (uint32_t)(qt * 128);
    const uint32_t tO = tmem + lane_off + (uint32_t)(256 + qt * 128);
    const float sl2 = p.scale_log2;
    const float2 scale2 = make_float2(sl2, sl2);
    const uint32_t barS = bar(B_S + qt), barP = bar(B_P + qt);
    // The epilogue of item k (O / l -> global) runs after the FIRST tile of item k+1: the
    // softmax of that tile is not delayed by it, only the next item's first PV waits for
    // the O read-out (B_OF).  O_qt(k) is final by then: PV_qt(last of k) was issued before
    // S_qt(first of k+1).  One call site: kk = n_my is a virtual item without tiles.
    int g = 0;
    int ne = 0;                   // items whose O the rotation warpgroup writes out (B_LR / B_LF phases)
    int idx_e = -1;               // item whose epilogue is pending
    float m_e = 0.f, lsum_e = 0.f;
    for (int kk = 0; kk <= n_my; ++kk) {
      const bool real = kk < n_my;
      const ItemRec rec = load_rec(recs, real ? kk : 0);
      const AttnParams& p = REC_PARAMS(rec);
      const Item w = item_of(p, rec);
      const int A = w.A;
      const int n = real ? w.n_tiles : 0;
      const int rglob = w.m0 + qt * 128 + rloc;
      const bool valid_row = real && rglob < w.rows_total;
      const int qi = valid_row ? rglob / p.grp : 0;
      const int lim = valid_row ? p.q_pos0 + qi : -1;
      const bool warp_dead = __all_sync(0xffffffffu, !valid_row);
      float m = -INFINITY;
      float2 lsum2 = make_float2(0.f, 0.f);
      uint32_t r[64];
      const int n1 = n > 0 ? n : 1;
      for (int jj = 0; jj < n1; ++jj) {
        if (real) {
          const int u = w.t_begin + jj;
          const TileSeg t = tile_segments<BN>(p, w, u);
          const int nu = t.width;                    // S columns [0, nu) hold this tile's scores
          int c_lo, c_hi;
          if (!valid_row) {
            c_lo = 0; c_hi = 0;
          } else if (u < w.n_extra) {                // sink always visible, self row j iff its id <= lim
            c_lo = 0;
            c_hi = min(max(min(A + w.n_self, max(A, lim - w.ring_count + 1)) - BN * u, 0), BN);
          } else {
            c_lo = t.lo0;
            c_hi = max(c_lo, min(t.hi0, lim - t.pos0_0 + 1));   // id pos0 + c <= lim
          }
          fwait(barS, g & 1, bar0);
          if (rloc == 0) FT(qt ? FT_SM1_S : FT_SM0_S, g);
          if (warp_dead || FA_ABL_SOFTMAX) {   // all 32 rows are padding: their P / O are never used
            mbar_arrive(barP);
          } else {
            tc_fence_after();
            // The tile's scores in 64-column halves (64 registers; one copy of the code, not
            // unrolled over the halves).  The running max is updated lazily per half; P of a
            // half goes to TMEM at once (P words 32h..32h+31 alias S columns already read).  If
            // half 1 moves the max, half 0's P words are rescaled in TMEM (rare).
            float2 l0 = make_float2(0.f, 0.f), l1 = l0;
            const int nh = nu > 64 ? 2 : 1;
#pragma unroll 1
            for (int hf = 0; hf < nh; ++hf) {
              const int c0 = 64 * hf;
              tmem_ld32x(tS + c0, &r[0]);
              if (nu > c0 + 32) tmem_ld32x(tS + c0 + 32, &r[32]);
              tmem_wait_ld();
              if (warp == 0 && lane == 0) FT(hf ? FT_SMX_LD1 : FT_SMX_LD0, g);
              // invisible columns (and columns >= nu, which are never loaded) -> -inf
              const bool partial = __any_sync(0xffffffffu, !(c_lo <= c0 && c_hi >= c0 + 64));
              if (partial) {
                const unsigned span = (unsigned)max(c_hi - c_lo, 0);
                const int off = c0 - c_lo;
#pragma unroll
                for (int c = 0; c < 64; ++c) r[c] = ((unsigned)(off + c) < span) ? r[c] : 0xFF800000u;
              }
              float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
#pragma unroll
              for (int c = 0; c < 64; c += 8) {     // 3-input max (FMNMX3): 2 columns per instruction
                mx0 = fmax3f(mx0, __uint_as_float(r[c]), __uint_as_float(r[c + 1]));
                mx1 = fmax3f(mx1, __uint_as_float(r[c + 2]), __uint_as_float(r[c + 3]));
                mx2 = fmax3f(mx2, __uint_as_float(r[c + 4]), __uint_as_float(r[c + 5]));
                mx3 = fmax3f(mx3, __uint_as_float(r[c + 6]), __uint_as_float(r[c + 7]));
              }
              const float m_half = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3)) * sl2;
              // lazy rescale: move the running max only when it grew by > 2^8.  The TMEM load /
              // store of O is warp-collective, so the O decision is taken per warp.  O_qt is
              // quiescent: S_qt(g) was issued after PV_qt(g-1) and its commit covers both.
              const bool upd = m_half > m + kRescaleThreshold;
              const bool need_o = upd && (m != -INFINITY);
              const float f = need_o ? ex2f(m - m_half) : 1.f;
              if (upd) {
                lsum2.x *= f; lsum2.y *= f;
                l0.x *= f; l0.y *= f; l1.x *= f; l1.y *= f;
                m = m_half;
              }
              if (__any_sync(0xffffffffu, need_o)) {
#pragma unroll 1
                for (int ch = 0; ch < 4; ++ch) {
                  uint32_t o[32];
                  tmem_ld32(tO + ch * 32, o);
                  tmem_wait_ld();
#pragma unroll
                  for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * f);
                  tmem_st32(tO + ch * 32, o);
                }
                if (hf == 1) {   // half 0's P was exponentiated against the old max
                  uint32_t o[32];
                  tmem_ld32(tS, o);
                  tmem_wait_ld();
#pragma unroll
                  for (int c = 0; c < 32; ++c) o[c] = pack_bf16(bf_lo(o[c]) * f, bf_hi(o[c]) * f);
                  tmem_st32(tS, o);
                }
                tmem_wait_st();
              }
              // P = 2^(s*scale - m) (masked -> 2^-inf = 0) packed bf16x2 into r[0..31]
              const float m_use = (m == -INFINITY) ? 0.f : m;
              const float2 negm2 = make_float2(-m_use, -m_use);
#pragma unroll
              for (int c = 0; c < 64; c += 4) {
                const float2 x0 = __ffma2_rn(make_float2(__uint_as_float(r[c]), __uint_as_float(r[c + 1])), scale2, negm2);
                const float2 x1 = __ffma2_rn(make_float2(__uint_as_float(r[c + 2]), __uint_as_float(r[c + 3])), scale2, negm2);
                const float2 p0 = make_float2(ex2f(x0.x), ex2f(x0.y));
                const float2 p1 = make_float2(ex2f(x1.x), ex2f(x1.y));
                l0 = __fadd2_rn(l0, p0);
                l1 = __fadd2_rn(l1, p1);
                r[c >> 1] = pack_bf16(p0.x, p0.y);
                r[(c >> 1) + 1] = pack_bf16(p1.x, p1.y);
              }
              tmem_st32(tS + 32 * hf, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
              if (warp == 0 && lane == 0) FT(hf ? FT_SMX_EX1 : FT_SMX_EX0, g);
            }
            lsum2 = __fadd2_rn(lsum2, __fadd2_rn(l0, l1));
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(barP);
            if (rloc == 0) FT(qt ? FT_SM1_P : FT_SM0_P, g);
          }
          ++g;
        }
        if (jj == 0 && idx_e >= 0) {
          // ---- epilogue of the previous item
          const ItemRec rec = load_rec(recs, idx_e);
          const AttnParams& p = REC_PARAMS(rec);
          const Item w = item_of(p, rec);
          const int rglob = w.m0 + qt * 128 + rloc;
          const bool valid_row = rglob < w.rows_total;
          const int qi = valid_row ? rglob / p.grp : 0;
          const float lsum = lsum_e, m = m_e;
          fwait(bar(B_O + qt), (kk - 1) & 1, bar0);
          if (rloc == 0) FT(qt ? FT_EPI1_O : FT_EPI0_O, kk - 1);
          tc_fence_after();
          if (FA_ABL_EPI) {
            tc_fence_before();
            mbar_arrive(bar(B_OF + qt));
          } else {
            const float inv = lsum > 0.f ? 1.f / lsum : 0.f;
            const int h = valid_row ? w.g * p.grp + rglob % p.grp : 0;
            const long long orow = ((long long)w.pp * p.n_q + qi) * p.Hq + h;
#pragma unroll 1
            for (int hf = 0; hf < 2; ++hf) {
              tmem_ld32x(tO + 64 * hf, &r[0]);
              tmem_ld32x(tO + 64 * hf + 32, &r[32]);
              tmem_wait_ld();
              if (hf == 1) {
                tc_fence_before();
                mbar_arrive(bar(B_OF + qt));      // O_qt may be overwritten by the next item's first PV
              }
              if (!valid_row) continue;
              {   // split-KV / context-parallel partial: fp32 O / l and log2-sum-exp per split
                const long long rows = (long long)p.P * p.n_q * p.Hq;
                const long long slot = p.split_only >= 0 ? 0 : w.sp;
                DSC_ASSERT(slot < max(p.n_splits, 1) && orow < rows, "attn_fa split partial row");
                float4* dst = reinterpret_cast<float4*>(p.ws_o + (slot * rows + orow) * 128 + 64 * hf);
#pragma unroll
                for (int v = 0; v < 16; ++v)
                  dst[v] = make_float4(__uint_as_float(r[4 * v]) * inv, __uint_as_float(r[4 * v + 1]) * inv,
                                       __uint_as_float(r[4 * v + 2]) * inv, __uint_as_float(r[4 * v + 3]) * inv);
                if (hf == 0) p.ws_lse[slot * rows + orow] = lsum > 0.f ? m + __log2f(lsum) : -INFINITY;
              }
            }
          }
          if (rloc == 0) FT(qt ? FT_EPI1_END : FT_EPI0_END, kk - 1);
        }
      }
      // plain / peer-store launches: the rotation warpgroup writes O out (rot_epilogue), this
      // warpgroup only hands over 1/l and goes straight to the next item
      const bool roe = real && p.n_splits == 1 && p.split_only < 0;
      if (roe) {
        const float ls = lsum2.x + lsum2.y;
        if (ne > 0) fwait(bar(B_LF), (ne - 1) & 1, bar0);
        lbuf[qt * 128 + rloc] = ls > 0.f ? 1.f / ls : 0.f;
        mbar_arrive(bar(B_LR));
        ++ne;
      }
      idx_e = real && !roe ? kk : -1;
      m_e = m;
      lsum_e = lsum2.x + lsum2.y;
    }
  } else if (warp < 12) {
    // ================================================================ rotation (K tiles) + Q prep
    if constexpr (kRegRotate > 128) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegRotate));
    else if constexpr (kRegRotate < 128) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegRotate));
    const int lt = threadIdx.x - 256;
    const int c8 = lt & 7;             // frequencies 8*c8 .. 8*c8+7
    const int rg = lt >> 3;            // rows rg*8 .. rg*8+7 of a 128-row tile
    const float4* __restrict__ rp = p.rope_pairs;
    float2 cth[4], sth[4];             // R(theta_f) = table entry of id 1
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float4 t = rp[32 + 4 * c8 + j];
      cth[j] = make_float2(t.x, t.y);
      sth[j] = make_float2(t.z, t.w);
    }
    // Q tile use qu (= 2 * item + qt) of item qidx: buffer qu % 3, free once use qu - 3's
    // last QK^T has completed
    auto prep_q = [&](int qu, int qidx) {
      if (lt == 0) FT((qu & 1) ? FT_QO_START : FT_QE_START, qu >> 1);
      const ItemRec rq = load_rec(recs, qidx);
      const AttnParams& pq = REC_PARAMS(rq);
      const Item wq = item_of(pq, rq);
      uint4 lo[8], hi[8];
      if (!FA_ABL_Q) load_rotate_q_regs(pq, wq, qu & 1, lt, lo, hi);
      if (qu >= NQB) fwait(bar(B_QF + qu % NQB), ((qu - NQB) / NQB) & 1, bar0);
      if (lt == 0 && (qu & 1)) FT(FT_QO_FREE, qu >> 1);
      if (!FA_ABL_Q) {
        const uint32_t qtile = qbuf_addr(qu);
        const int c8 = lt & 7, rg8 = lt >> 3;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int r = rg8 * 8 + k;
          const uint32_t a = qtile + r * 128 + ((c8 ^ (r & 7)) << 4);
          sts128(a, lo[k]);
          sts128(a + 16384, hi[k]);
        }
        fence_proxy_async();
      }
      mbar_arrive(bar(B_QR + qu % NQB));
      if (lt == 0) FT((qu & 1) ? FT_QO_END : FT_QE_END, qu >> 1);
    };
    // Epilogue of item kk for plain / peer-store launches: O / l -> bf16 rows.  Runs here, not
    // on the softmax warpgroups, so their next item starts at once; thread lt owns row lt of
    // both Q tiles (warp 8 + lt/32 reads TMEM lane quarter lt/32).
    int ne = 0;
    auto rot_epilogue = [&](int kk) {
      const ItemRec rec = load_rec(recs, kk);
      const AttnParams& p = REC_PARAMS(rec);
      const Item w = item_of(p, rec);
      fwait(bar(B_LR), ne & 1, bar0);
      const float inv0 = lbuf[lt], inv1 = lbuf[128 + lt];
      mbar_arrive(bar(B_LF));
      ++ne;
      const uint32_t lane_off = (uint32_t)((lt >> 5) * 32) << 16;
#pragma unroll 1
      for (int qt = 0; qt < 2; ++qt) {
        fwait(bar(B_O + qt), kk & 1, bar0);
        if (lt == 0) FT(qt ? FT_EPI1_O : FT_EPI0_O, kk);
        tc_fence_after();
        const int rglob = w.m0 + qt * 128 + lt;
        const bool valid_row = rglob < w.rows_total;
        const int qi = valid_row ? rglob / p.grp : 0;
        const int h = valid_row ? w.g * p.grp + rglob % p.grp : 0;
        const float inv = qt ? inv1 : inv0;
        const uint32_t tO = tmem + lane_off + (uint32_t)(256 + qt * 128);
        uint32_t r[64];
#pragma unroll 1
        for (int hf = 0; hf < 2; ++hf) {
          tmem_ld32x(tO + 64 * hf, &r[0]);
          tmem_ld32x(tO + 64 * hf + 32, &r[32]);
          tmem_wait_ld();
          if (hf == 1) {
            tc_fence_before();
            mbar_arrive(bar(B_OF + qt));   // O_qt may be overwritten by the next item's first PV
          }
          if (!valid_row || FA_ABL_EPI) continue;
          uint32_t q[8];
          const bool peers = p.n_peers > 0;
          int oq = qi + p.o_rot;   // o_rot = 0 unless ring-ordered output (o_rows > 0)
          if (p.o_rows > 0 && oq >= p.o_rows) oq -= p.o_rows;
          const long long row = peers ? ((long long)w.pp * p.n_q + qi) * p.o_hq + p.o_head_off + h
                                      : ((long long)w.pp * (p.o_rows > 0 ? p.o_rows : p.n_q) + oq) * p.Hq + h;
          DSC_ASSERT(qi < p.n_q && w.pp < p.P && h < p.Hq && oq < (p.o_rows > 0 ? p.o_rows : p.n_q), "attn_fa O row");
          const int nd = peers ? p.n_peers : 1;
#pragma unroll
          for (int v = 0; v < 4; ++v) {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              q[j] = pack_bf16(__uint_as_float(r[16 * v + 2 * j]) * inv, __uint_as_float(r[16 * v + 2 * j + 1]) * inv);
#pragma unroll 1
            for (int d = 0; d < nd; ++d)
              stg256(reinterpret_cast<__nv_bfloat16*>(peers ? p.peer_o[d] : p.o) + row * 128 + 64 * hf + 16 * v, q);
          }
        }
        if (lt == 0) FT(qt ? FT_EPI1_END : FT_EPI0_END, kk);
      }
    };
    // Job order (one call site each for the Q prep and the K rotation, so each is inlined
    // once): a virtual item -1 prepares item 0's Q tiles; item kk with rotated K tiles runs
    // K(0), Q0(kk+1), K(1) .. K(n-1), Q1(kk+1); an item without (staged build) runs Q0(kk+1),
    // Q1(kk+1).  Q0(kk+1)'s buffer is free early (item kk-1's Q1), Q1(kk+1)'s only after
    // item kk's last S0: every K tile of item kk is rotated before that wait.
    int gt = 0;
    for (int kk = -1; kk < n_my; ++kk) {
      const bool q_next = kk + 1 < n_my;
      const int nidx = q_next ? kk + 1 : 0;
      const ItemRec rec = load_rec(recs, kk >= 0 ? kk : nidx);
      const AttnParams& p = REC_PARAMS(rec);
      const Item w = item_of(p, rec);
      const bool rot = kk >= 0 && !w.staged && w.n_tiles > 0;
      const int nk = rot ? w.n_tiles : 0;
      const int njobs = nk + 2;
      const int A = w.A;
      const bool dbg = p.dbg_pos != nullptr && w.g == 0;   // every problem, kv head 0
      int* const dbgp = dbg ? p.dbg_pos + (w.head_row / p.Hkv) * p.dbg_len : nullptr;
#pragma unroll 1
      for (int t = 0; t < njobs; ++t) {
        const bool is_q = rot ? (t == 1 || t == njobs - 1) : true;
        if (is_q) {
          if (q_next) prep_q(2 * kk + 2 + (rot ? (t == 1 ? 0 : 1) : t), nidx);   // Q tile 0 / 1 of item kk+1
          continue;
        }
        const int jj = t == 0 ? 0 : t - 1;
        const int g = gt + jj, u = w.t_begin + jj, ks = g % KST;
        const TileSeg tg = tile_segments<BN>(p, w, u);
        int kpos[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) kpos[k] = seg_pos(tg, rg * 8 + k);
        int p0 = -1;
#pragma unroll
        for (int k = 7; k >= 0; --k)
          if (kpos[k] >= 0) p0 = kpos[k];
        float4 pre[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) pre[j] = rp[(long long)max(p0, 0) * 32 + 4 * c8 + j];
        fwait(bar(B_KR + ks), (g / KST) & 1, bar0);
        if (lt == 0) FT(FT_ROT_KR, g);
        if (rg * 8 < tg.width && !FA_ABL_ROT)   // rows >= width are never read by the MMA
          rotate_rows<2, kKVHalf>(sbase + OFF_K + ks * kKVBytes, rg * 8, c8, rp, cth, sth, kpos, pre, max(p0, 0));
        fence_proxy_async();
        mbar_arrive(bar(B_KF + ks));
        if (lt == 0) FT(FT_ROT_KF, g);
        if (dbg && c8 == 0) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int rr = rg * 8 + k;
            const int x = BN * u + rr;
            int slot = tg.slot0 + rr;
            if (slot >= p.R) slot -= p.R;
            if (kpos[k] >= 0)
              dbgp[(u < w.n_extra) ? (x < A ? x : p.dbg_A + p.dbg_R + (x - A)) : p.dbg_A + slot] = kpos[k];
          }
        }
      }
      if (kk >= 0 && p.n_splits == 1 && p.split_only < 0) rot_epilogue(kk);
      if (kk >= 0) gt += w.n_tiles;
    }
  } else {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegCopy));
    if (warp == 12 || warp == 13) {
      // ============================================================== copy warps (12: K, 13: V)
      const bool isk = warp == 12;
      const int nst = isk ? KST : VST;
      const int off = isk ? OFF_K : OFF_V;
      const int b_full = isk ? B_KR : B_VR, b_free = isk ? B_KE : B_VE;
      int gt = 0;
      for (int kk = 0; kk < n_my; ++kk) {
        const ItemRec rec = load_rec(recs, kk);
        const AttnParams& p = REC_PARAMS(rec);
        const Item w = item_of(p, rec);
        const int A = p.A;
        const __nv_bfloat16* __restrict__ SX = reinterpret_cast<const __nv_bfloat16*>(isk ? p.sink_k : p.sink_v);
        const __nv_bfloat16* __restrict__ XX = reinterpret_cast<const __nv_bfloat16*>(isk ? p.self_k : p.self_v);
#pragma unroll 1
        for (int jj = 0; jj < w.n_tiles; ++jj) {
          const int g = gt + jj, u = w.t_begin + jj, st = g % nst;
          if (g >= nst) fwait(bar(b_free + st), ((g - nst) / nst) & 1, bar0);
          const uint32_t dst = sbase + off + st * kKVBytes;
          const TileSeg t = tile_segments<BN>(p, w, u);
          if (u < w.n_extra) {
            // sink rows (x < A) + self rows (A <= x < A + n_self), zeros up to the tile width
            const int nit = t.width >> 1;   // 16 chunks of 16 B per row, 32 lanes
#pragma unroll 1
            for (int it = 0; it < nit; ++it) {
              const int id = it * 32 + lane;
              const int rr = id >> 4, ch = id & 15;
              const int x = BN * u + rr;
              const __nv_bfloat16* src = nullptr;
              if (x < A) src = SX + (w.head_row * A + x) * 128;
              else if (x < A + w.n_self) src = XX + (((long long)w.pp * w.n_self + (x - A)) * p.Hkv + w.g) * 128;
              DSC_ASSERT(w.head_row < (long long)p.S * p.N_total * p.Hkv && w.pp < p.P && rr < BN, "attn_fa sink/self row");
              const uint32_t d = dst + (ch >> 3) * kKVHalf + rr * 128 + (((ch & 7) ^ (rr & 7)) << 4);
              cp_async16(d, src ? (const void*)(src + 8 * ch) : (const void*)SX, src ? 16u : 0u);
            }
            cp_async_wait_all();
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar(b_full + st));
          } else if (lane == 0) {
            // logical window tile: one 128-row box per 64-column block (ring mirror or staging rows)
            const CUtensorMap* tmap = isk ? &p.tmap_k : &p.tmap_v;
            const int row = (int)(w.head_row * w.Rp) + t.slot0;
            // the box starts inside this head's rows; a staged window's last box may run past
            // them (rows >= the tile width are masked; past the tensor end TMA fills zeros)
            DSC_ASSERT(t.slot0 >= 0 && t.slot0 < w.Rp && (w.staged || t.slot0 + BN <= w.Rp) &&
                           w.head_row < (long long)p.S * p.N_total * p.Hkv,
                       "attn_fa TMA box rows");
            FT(isk ? FT_CPK : FT_CPV, g);
            mbar_arrive_tx(bar(b_full + st), kKVBytes);
            tma_load_2d(dst, tmap, 0, row, bar(b_full + st));
            tma_load_2d(dst + kKVHalf, tmap, 64, row, bar(b_full + st));
          }
          __syncwarp();
        }
        gt += w.n_tiles;
      }
    } else if (warp == 14 || warp == 15) {
      // ============================================================== MMA issuer(s)
      constexpr uint32_t IQK0 = idesc_bf16(128, 0, 0, 0);    // S = Q K^T, both K-major; N = tile width
      constexpr uint32_t IPV = idesc_bf16(128, 128, 0, 1);   // O += P V, P from TMEM, V MN-major
      auto issue_qk = [&](int qu, int ks, int nu, int qt) {
        const uint64_t da = sdesc(qbuf_addr(qu), 16, 1024);
        const uint64_t db = sdesc(sbase + OFF_K + ks * kKVBytes, 16, 1024);
        mma_qk(tmem + qt * 128, da, db, IQK0 | ((uint32_t)(nu >> 3) << 17));
      };
      auto issue_pv = [&](int qt, int vs, bool acc, int nu) {
        if (FA_ABL_PV) return;
        const uint64_t dv = sdesc(sbase + OFF_V + vs * kKVBytes, kKVHalf, 1024);
        const uint32_t d = tmem + 256 + qt * 128, a = tmem + qt * 128;
        if (nu == BN) {
          mma_pv8(d, a, dv, IPV, acc ? 1u : 0u);
        } else {
          const int nk = nu >> 4;
          mma_ts_w(d, a, dv, IPV, acc ? 1u : 0u);
#pragma unroll 1
          for (int k8 = 1; k8 < nk; ++k8) mma_ts_w(d, a + k8 * 8, dv + (uint64_t)(k8 * 128), IPV, 1u);
        }
      };
      // What the issue loop needs of an item (few registers: this warp runs with kRegCopy).
      struct MI {
        int n, t_begin, staged, n_extra, aps, cnt;
      };
      auto mi_of = [&](int kk) {
        const ItemRec r = load_rec(recs, kk);
        const bool isb = r.flags & 1;
        const int A = isb ? pb.A : pa.A, n_self = isb ? pb.n_self : pa.n_self;
        MI m;
        m.n = r.n_tiles; m.t_begin = r.t_begin; m.staged = isb ? pb.staged : pa.staged;
        m.n_extra = (A + n_self + BN - 1) / BN; m.aps = A + n_self; m.cnt = r.cnt;
        return m;
      };
      // tile width (valid keys rounded up to 16) of tile jj of an item: tile_segments' rule
      auto width_of = [&](const MI& m, int jj) {
        const int u = m.t_begin + jj;
        const int valid = u < m.n_extra ? min(max(m.aps - BN * u, 0), BN) : min(m.cnt - BN * (u - m.n_extra), BN);
        return (valid + 15) & ~15;
      };
      uint32_t kf_ph = 0;   // B_KF phase bit per K stage (only rotated tiles arrive there)
      auto wait_kmi = [&](const MI& m, int g) {
        const int ks = g % KST;
        if (m.staged) {
          fwait(bar(B_KR + ks), (g / KST) & 1, bar0);
        } else {
          fwait(bar(B_KF + ks), (kf_ph >> ks) & 1, bar0);
          kf_ph ^= 1u << ks;
        }
        tc_fence_after();
      };
      // Every item has n >= 1 tiles (the host splits never leave a split empty, a causal
      // m-block always sees a key).  The issue order is one stream across items: the next
      // item's S0(0) follows this item's last PV0, its S1(0) the last PV1, exactly as S(g+1)
      // follows PV(g) inside an item, so an item switch costs the tensor core nothing but the
      // O read-out of the epilogue (B_OF) before the next item's first PV.
      const int mq = warp - 14;   // the Q tile whose MMAs this warp issues
      int gt = 0;
      MI cur = {};
      if (n_my > 0) {
        cur = mi_of(0);
        const int nu = width_of(cur, 0);
        if (lane == 0 && mq == 0) FT(FT_MMA_ITEM, 0);
        wait_kmi(cur, 0);
        fwait(bar(B_QR + mq), 0, bar0);
        tc_fence_after();
        issue_qk(mq, 0, nu, mq);
        mma_commit_w(bar(B_S + mq));
        mma_commit_w(bar(B_KE + 0));
        if (cur.n == 1) mma_commit_w(bar(B_QF + mq));
      }
      for (int kk = 0; kk < n_my; ++kk) {
        const int n = cur.n;
        const bool has_next = kk + 1 < n_my;
        const MI nxt = has_next ? mi_of(kk + 1) : cur;
        int nu = width_of(cur, 0);
        for (int jj = 0; jj < n; ++jj) {
          const int g = gt + jj, vs = g % VST;
          const bool last = jj + 1 == n;
          const bool nx = !last || has_next;
          const MI& wn = last ? nxt : cur;
          const int qn = (last ? 2 * (kk + 1) : 2 * kk) + mq;   // Q tile use of the next S
          const int jn = last ? 0 : jj + 1;
          const int nu2 = nx ? width_of(wn, jn) : 0;
          const bool last_s = jn + 1 == wn.n;
          fwait(bar(B_VR + vs), (g / VST) & 1, bar0);
          fwait(bar(B_P + mq), g & 1, bar0);
          if (lane == 0) FT(mq ? FT_MMA_P1 : FT_MMA_P0, g);
          if (jj == 0 && kk > 0) fwait(bar(B_OF + mq), (kk - 1) & 1, bar0);   // previous item's O read out
          if (lane == 0 && jj == 0 && mq == 0) FT(FT_MMA_OF, kk);
          tc_fence_after();
          issue_pv(mq, vs, jj > 0, nu);
          if (lane == 0 && mq == 0) FT(FT_MMA_PV0I, g);
          mma_commit_w(bar(B_VE + vs));
          if (last) mma_commit_w(bar(B_O + mq));
          if (nx) {
            wait_kmi(wn, g + 1);
            if (lane == 0 && mq == 0) FT(FT_MMA_K, g + 1);
            if (last) {
              if (lane == 0 && mq == 0) FT(FT_MMA_ITEM, kk + 1);
              fwait(bar(B_QR + qn % NQB), (qn / NQB) & 1, bar0);
              if (lane == 0) FT(mq ? FT_MMA_Q1 : FT_MMA_Q0, kk + 1);
              tc_fence_after();
            }
            issue_qk(qn, (g + 1) % KST, nu2, mq);
            if (lane == 0 && mq == 0) FT(FT_MMA_S0I, g + 1);
            mma_commit_w(bar(B_S + mq));
            mma_commit_w(bar(B_KE + (g + 1) % KST));
            if (last_s) mma_commit_w(bar(B_QF + qn % NQB));
          }
          nu = nu2;
        }
        gt += n;
        cur = nxt;
      }
      // drain: the last V-free commit tracks every MMA of this CTA
      if (gt > 0) fwait(bar(B_VE + (gt - 1) % VST), ((gt - 1) / VST) & 1, bar0);
      if (lane == 0) FT(FT_END, 0);
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 14) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
#undef REC_PARAMS
}

}  // namespace fa

// ==========================================================================================
// v8: the CTA-pair kernel (tcgen05.mma.cta_group::2, M = 256).  Same work items, same Eq. 7 /
// Eq. 8 arithmetic as v7; the 256 query rows of an item are split over the two SMs of a
// cluster (CTA r holds Q rows 128 r .. 128 r + 127 of the m-block and owns TMEM lanes = those
// rows), each 128-key tile is split by the B operand's N: CTA r loads and rotates keys
// [r nu/2, (r + 1) nu/2) of the tile for QK^T and the d columns [64 r, 64 r + 64) of all
// its V rows for PV (scripts/micro/pair_mma_test.cu checks these layouts and the full
// 8190 flop/clk/SM rate of the pair MMA).  Per SM that halves the K rotation, the Q prep,
// the O epilogue and the shared-memory operand traffic of a tile, and it frees TMEM:
//   S[3] = cols 0..383: S is issued two tiles ahead of PV (S(g+2), then PV(g)), so the
//          softmax finds S(g+1) done when it finishes S(g);
//   O    = cols 384..511, read out by the epilogue as soon as its item's last PV is done.
// The leader CTA (rank 0) issues every MMA; its waits gather arrivals from both CTAs
// (remote mbarrier arrives), its commits are multicast to both.
//   warps 0-7  softmax: warps w and w + 4 share the 32 rows of TMEM lane quarter w % 4, warp
//              w < 4 owns score columns 0..63, w >= 4 columns 64..127; the row max is
//              exchanged through shared memory once per tile (then P needs no re-scaling)
//   warps 8-11 K rotation of this CTA's key half, the Q tile prep one item ahead, the epilogue
//   warp 12    K copy (TMA 64 x 64 boxes / cp.async sink+self rows), warp 13 V copy
//   warp 14    TMEM allocation; MMA issuer (leader)
//   warp 15    forwarder: locally landed V (and pre-rotated staged K) -> the leader's barriers
namespace pr {
using namespace tcc;
using fa::fwait;
using fa::ex2f;
using fa::tmem_ld32x;
using fa::load_rotate_q_regs;
using fa::item_of;
using fa::load_rec;

constexpr int BN = kTileN;
constexpr int kWarps = 16;
constexpr int kThreads = kWarps * 32;
constexpr int kQBytes = 128 * 128 * 2;    // this CTA's Q tile: two 64-column SW128 blocks of 128 rows
constexpr int kKHalf = 64 * 128;          // one 64-column SW128 block of this CTA's <= 64 keys (8 KB)
constexpr int kKBytes = 2 * kKHalf;
constexpr int kVBytes = 128 * 128;        // 128 keys x this CTA's 64 d columns (16 KB)
constexpr int NQB = 2, KST = 4, VST = 3;
constexpr int OFF_Q = 0;
constexpr int OFF_K = OFF_Q + NQB * kQBytes;
constexpr int OFF_V = OFF_K + KST * kKBytes;
constexpr int OFF_BAR = OFF_V + VST * kVBytes;
// TMEM: NSB S buffers + NOB O buffers of 128 columns (PR_NOB = 1: S[3], O; 2: S[2], O[2])
#ifndef PR_NOB
#define PR_NOB 1
#endif
constexpr int NOB = PR_NOB;
constexpr int NSB = 4 - NOB;
enum {
  B_QR = 0,             // [2] Q buffer ready (leader: 4 warps x 2 CTAs)
  B_QF = B_QR + 2,      // [2] Q buffer free (commit after its item's last QK^T)
  B_KR = B_QF + 2,      // [KST] K half landed in this CTA (TMA tx / cp.async)
  B_KF = B_KR + KST,    // [KST] K tile ready for the MMA (leader: 8 = rotation warps, or forwarders x 4)
  B_KE = B_KF + KST,    // [KST] K stage free (commit)
  B_VL = B_KE + KST,    // [VST] V landed in this CTA
  B_VR = B_VL + VST,    // [VST] V ready (leader: 2 forwarders)
  B_VE = B_VR + VST,    // [VST] V stage free = PV done (commit)
  B_S = B_VE + VST,     // [NSB] S buffer ready (commit)
  B_P = B_S + NSB,      // [NSB] P ready (leader: 8 softmax warps x 2 CTAs)
  B_O = B_P + NSB,      // [NOB] O final for its item (commit)
  B_OF = B_O + NOB,     // [NOB] O read out (leader: 4 warps x 2 CTAs)
  B_LR = B_OF + NOB,      // [2] (l, m) of an item's rows written (256 softmax threads)
  B_LF = B_LR + 2,      // [2] ... read by the epilogue (128)
  B_N = B_LF + 2
};
constexpr int OFF_L = OFF_BAR + B_N * 8 + 8;                  // (l, m) handoff [2 items][2 halves][128] float2
constexpr int OFF_X = OFF_L + 2 * 2 * 128 * 8;                // row max exchange [2 tiles][2 halves][128] float
constexpr int kSmemBytes = OFF_X + 2 * 2 * 128 * 4 + 1024;
static_assert(kSmemBytes <= 227 * 1024, "shared memory budget");
constexpr float kRescaleThreshold = 8.0f;
// ablation knobs (timing experiments only; results are wrong when set)
#ifndef PR_ABL_SM
#define PR_ABL_SM 0
#endif
#ifndef PR_ABL_Q
#define PR_ABL_Q 0
#endif
#ifndef PR_ABL_EPI
#define PR_ABL_EPI 0
#endif
#ifndef PR_ABL_ROT
#define PR_ABL_ROT 0
#endif

// PR_TRACE 1 (profiling variant): clock64 of pipeline events into p.trace for the first
// ntrace_cta CTAs, [cta][kPtEvents][kPtIdx]; per-tile events by the global tile g, per-item by item
#ifndef PR_TRACE
#define PR_TRACE 0
#endif
constexpr int kPtEvents = 32, kPtIdx = 1024;
enum {
  PT_S_ISS = 0, PT_PV_ISS, PT_KF_OK, PT_VR_OK, PT_P_OK, PT_SM_S, PT_SM_P, PT_CPK, PT_CPV, PT_FWV, PT_ROT,   // per tile
  PT_ITEM = 12, PT_Q_START, PT_Q_FREE, PT_Q_END, PT_EPI_O, PT_EPI_END, PT_QR_OK, PT_OF_OK, PT_END,           // per item
  PT_KR_FW = 21, PT_S_MMA = 22, PT_PV_MMA = 23, PT_S_FENCE = 24, PT_ROT_PRE = 25, PT_ROT_KR = 26, PT_ROT_RR = 27,   // per tile
  PT_ROT9 = 28, PT_ROT10 = 29, PT_ROT11 = 30
};
#if PR_TRACE
#define PT(ev, i)                                                                                      \
  do {                                                                                                 \
    if (pt_cta && (i) < kPtIdx) pt_cta[(ev) * kPtIdx + (i)] = clock64();                                \
  } while (0)
#else
#define PT(ev, i) do { } while (0)
#endif

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cluster address of the same offset in the leader CTA (rank 0)
__device__ __forceinline__ uint32_t map_lead(uint32_t a) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(a));
  return r;
}
// remote arrive with the default .release.cta semantics (the producer's writes are ordered for
// the consumer by the proxy / tcgen05 fences before it; .release.cluster compiles to a GPU-scope
// MEMBAR before every arrival)
__device__ __forceinline__ void arrive_cl(uint32_t cbar, uint32_t cnt) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0], %1;" ::"r"(cbar), "r"(cnt) : "memory");
}
__device__ __forceinline__ bool mbar_try_cl(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred P1;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P1;\n}\n"
      : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
  return ok != 0;
}
// non-blocking phase test (try_wait may suspend the thread until the phase completes)
__device__ __forceinline__ bool mbar_test(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred P1;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P1;\n}\n"
      : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
  return ok != 0;
}
// wait on a barrier that collects arrivals from both CTAs (cluster-scope acquire)
__device__ __forceinline__ void cwait(uint32_t bar, uint32_t parity, uint32_t bar0) {
  if (mbar_try_cl(bar, parity)) return;
  const long long lim = fa::g_fa_wd_lim;
  const long long t0 = clock64();
  while (!mbar_try_cl(bar, parity)) {
    if (clock64() - t0 > lim) fa::fa_wd_fail((bar - bar0) / 8, parity);
  }
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// commit of the pair's MMAs, arriving on the barrier at this offset in BOTH CTAs
__device__ __forceinline__ void commit2_w(uint32_t bar) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}\n" ::"r"(
          bar),
      "h"((uint16_t)3)
      : "memory");
}
// S = Q K^T (M = 256 over the pair, K = 128 as 8 x K16): A = Q tile (second 64-column block
// +16 KB = 1024 units), B = this CTA's key half (second block +8 KB = 512 units)
__device__ __forceinline__ void mma2_qk(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc) {
  asm volatile(
      "{\n.reg .pred e;\n.reg .b64 a1, a2, a3, a4, a5, a6, a7, b1, b2, b3, b4, b5, b6, b7;\n"
      "add.s64 a1, %1, 2; add.s64 a2, %1, 4; add.s64 a3, %1, 6;\n"
      "add.s64 a4, %1, 1024; add.s64 a5, %1, 1026; add.s64 a6, %1, 1028; add.s64 a7, %1, 1030;\n"
      "add.s64 b1, %2, 2; add.s64 b2, %2, 4; add.s64 b3, %2, 6;\n"
      "add.s64 b4, %2, 512; add.s64 b5, %2, 514; add.s64 b6, %2, 516; add.s64 b7, %2, 518;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, 0;\n"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a1, b1, %3, 1;\n"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a2, b2, %3, 1;\n"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a3, b3, %3, 1;\n"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a4, b4, %3, 1;\n"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a5, b5, %3, 1;\n"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a6, b6, %3, 1;\n"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a7, b7, %3, 1;\n}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc)
      : "memory");
}
// O += P V over a full 128-key tile: A = P in TMEM (8 columns per K16 step), B = V rows
// (MN-major SW128, 16 keys = 2048 B = 128 units per step)
__device__ __forceinline__ void mma2_pv8(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred e, p;\n.reg .b64 b1, b2, b3, b4, b5, b6, b7;\n.reg .b32 t1, t2, t3, t4, t5, t6, t7;\n"
      "add.s64 b1, %2, 128; add.s64 b2, %2, 256; add.s64 b3, %2, 384;\n"
      "add.s64 b4, %2, 512; add.s64 b5, %2, 640; add.s64 b6, %2, 768; add.s64 b7, %2, 896;\n"
      "add.u32 t1, %1, 8; add.u32 t2, %1, 16; add.u32 t3, %1, 24;\n"
      "add.u32 t4, %1, 32; add.u32 t5, %1, 40; add.u32 t6, %1, 48; add.u32 t7, %1, 56;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [t1], b1, %3, 1;\n"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [t2], b2, %3, 1;\n"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [t3], b3, %3, 1;\n"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [t4], b4, %3, 1;\n"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [t5], b5, %3, 1;\n"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [t6], b6, %3, 1;\n"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [t7], b7, %3, 1;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma2_pv1(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// the pair's tile width: valid keys rounded up to 32, so each CTA's half is a multiple of 16
__device__ __forceinline__ int width2(const TileSeg& t) { return (t.width + 31) & ~31; }

constexpr int kRegSoftmax = 136, kRegAux = 168, kRegMisc = 72;   // setmaxnreg: 2 x 136 + 168 + 72 = 512
static_assert(2 * kRegSoftmax + kRegAux + kRegMisc <= 512, "register budget");

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    attn_pair_kernel(const __grid_constant__ AttnParams pa, const __grid_constant__ AttnParams pb, int na, int nb) {
  const AttnParams& p = pa;   // launch-wide fields (rope table) are shared
#if PR_TRACE
  long long* const pt_cta = (pa.trace && blockIdx.x < (unsigned)pa.ntrace_cta)
                                ? pa.trace + (long long)blockIdx.x * kPtEvents * kPtIdx : nullptr;
#endif
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = ((uint32_t)__cvta_generic_to_shared(smem_raw) + 1023u) & ~1023u;
  const uint32_t bar0 = sbase + OFF_BAR;
  auto bar = [&](int i) { return bar0 + 8u * (uint32_t)i; };
  const uint32_t lbar0 = map_lead(bar0);   // the leader's barriers in the cluster window
  auto lbar = [&](int i) { return lbar0 + 8u * (uint32_t)i; };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + OFF_BAR + B_N * 8);
  float2* lbuf = reinterpret_cast<float2*>(smem + OFF_L);
  float* xbuf = reinterpret_cast<float*>(smem + OFF_X);
  const int rank = (int)cta_rank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#define REC_PARAMS(R) (((R).flags & 1) ? pb : pa)

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar(B_QR + i), 8);
      mbar_init(bar(B_QF + i), 1);
      mbar_init(bar(B_LR + i), 256);
      mbar_init(bar(B_LF + i), 128);
    }
    for (int i = 0; i < NSB; ++i) {
      mbar_init(bar(B_S + i), 1);
      mbar_init(bar(B_P + i), 16);
    }
    for (int i = 0; i < NOB; ++i) {
      mbar_init(bar(B_O + i), 1);
      mbar_init(bar(B_OF + i), 8);
    }
    for (int i = 0; i < KST; ++i) {
      mbar_init(bar(B_KR + i), 1);
      mbar_init(bar(B_KF + i), 8);
      mbar_init(bar(B_KE + i), 1);
    }
    for (int i = 0; i < VST; ++i) {
      mbar_init(bar(B_VL + i), 1);
      mbar_init(bar(B_VR + i), 2);
      mbar_init(bar(B_VE + i), 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_proxy_async();
  }
  if (warp == 14) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  if (warp == 12 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&pa.tmap_k64)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&pa.tmap_v)) : "memory");
    if (nb > 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&pb.tmap_k64)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&pb.tmap_v)) : "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // this cluster's items (both CTAs walk the same list)
  const int cl = blockIdx.x >> 1;
  const ItemRec* __restrict__ recs = pa.item_recs + pa.item_off[cl];
  const int n_my = pa.item_off[cl + 1] - pa.item_off[cl];
  auto qbuf_addr = [&](int k) { return sbase + OFF_Q + (uint32_t)((k & 1) * kQBytes); };
  const uint32_t tO_base = tmem + (uint32_t)(NSB * 128);

  if (warp < 8) {
    // ================================================================ softmax (64 columns per thread)
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegSoftmax));
    const int quarter = warp & 3, hc = warp >> 2;    // lane quarter, column half
    const int rloc = quarter * 32 + lane;
    const int c0 = 64 * hc;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const uint32_t tO0 = tO_base + lane_off + (uint32_t)c0;
    const float sl2 = p.scale_log2;
    const float2 scale2 = make_float2(sl2, sl2);
    int g = 0;
    for (int kk = 0; kk < n_my; ++kk) {
      const ItemRec rec = load_rec(recs, kk);
      const AttnParams& p = REC_PARAMS(rec);
      const Item w = item_of(p, rec);
      const int A = w.A;
      const int n = w.n_tiles;
      const int rglob = w.m0 + rank * 128 + rloc;
      const bool valid_row = rglob < w.rows_total;
      const int qi = valid_row ? rglob / p.grp : 0;
      const int lim = valid_row ? p.q_pos0 + qi : -1;
      const bool warp_dead = __all_sync(0xffffffffu, !valid_row);   // same for both halves of a quarter
      const uint32_t tO = tO0 + (uint32_t)((kk % NOB) * 128);
      float m = -INFINITY;
      float2 lsum2 = make_float2(0.f, 0.f);
      uint32_t r[64];
      for (int jj = 0; jj < n; ++jj, ++g) {
        const int u = w.t_begin + jj;
        const TileSeg t = tile_segments<BN>(p, w, u);
        const int nu = width2(t);
        int c_lo, c_hi;
        if (!valid_row) {
          c_lo = 0; c_hi = 0;
        } else if (u < w.n_extra) {
          c_lo = 0;
          c_hi = min(max(min(A + w.n_self, max(A, lim - w.ring_count + 1)) - BN * u, 0), BN);
        } else {
          c_lo = t.lo0;
          c_hi = max(c_lo, min(t.hi0, lim - t.pos0_0 + 1));
        }
        const int sb = g % NSB;
        const uint32_t tS = tmem + lane_off + (uint32_t)(sb * 128);
        fwait(bar(B_S + sb), (g / NSB) & 1, bar0);
        if (rloc == 0 && hc == 0) PT(PT_SM_S, g);
        if (!warp_dead && !PR_ABL_SM) {
          tc_fence_after();
          // this half's scores (columns >= nu are never loaded: masked below)
          if (nu > c0) tmem_ld32x(tS + c0, &r[0]);
          if (nu > c0 + 32) tmem_ld32x(tS + c0 + 32, &r[32]);
          tmem_wait_ld();
          const bool partial = __any_sync(0xffffffffu, !(c_lo <= c0 && c_hi >= c0 + 64));
          if (partial) {
            const unsigned span = (unsigned)max(c_hi - c_lo, 0);
            const int off = c0 - c_lo;
#pragma unroll
            for (int c = 0; c < 64; ++c) r[c] = ((unsigned)(off + c) < span) ? r[c] : 0xFF800000u;
          }
          float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
#pragma unroll
          for (int c = 0; c < 64; c += 8) {
            mx0 = fmax3f(mx0, __uint_as_float(r[c]), __uint_as_float(r[c + 1]));
            mx1 = fmax3f(mx1, __uint_as_float(r[c + 2]), __uint_as_float(r[c + 3]));
            mx2 = fmax3f(mx2, __uint_as_float(r[c + 4]), __uint_as_float(r[c + 5]));
            mx3 = fmax3f(mx3, __uint_as_float(r[c + 6]), __uint_as_float(r[c + 7]));
          }
          // row max over both halves: exchange with the other warp of this lane quarter (both
          // have loaded their S columns before either writes P over S columns 0..63)
          float* xb = xbuf + (g & 1) * 256;
          xb[hc * 128 + rloc] = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3));
          asm volatile("bar.sync %0, 64;" ::"r"(1 + quarter) : "memory");
          const float m_tile = fmaxf(xb[rloc], xb[128 + rloc]) * sl2;
          // lazy rescale (2^8): O holds this item's sum only from tile 1 on (tile 0's PV
          // overwrites it), and then PV(g-1) must have completed before O is touched
          const bool upd = m_tile > m + kRescaleThreshold;
          const bool need_o = upd && (m != -INFINITY);
          const float f = need_o ? ex2f(m - m_tile) : 1.f;
          if (upd) {
            lsum2.x *= f; lsum2.y *= f;
            m = m_tile;
          }
          if (__any_sync(0xffffffffu, need_o) && jj > 0) {
            fwait(bar(B_VE + (g - 1) % VST), ((g - 1) / VST) & 1, bar0);
            tc_fence_after();
#pragma unroll 1
            for (int ch = 0; ch < 2; ++ch) {   // this half's 64 O columns
              uint32_t o[32];
              tmem_ld32(tO + ch * 32, o);
              tmem_wait_ld();
#pragma unroll
              for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * f);
              tmem_st32(tO + ch * 32, o);
            }
          }
          // P = 2^(s*scale - m) (masked -> 0) packed bf16x2 into r[0..31] -> P words 32 hc ..
          const float m_use = (m == -INFINITY) ? 0.f : m;
          const float2 negm2 = make_float2(-m_use, -m_use);
          float2 l0 = make_float2(0.f, 0.f), l1 = l0;
#pragma unroll
          for (int c = 0; c < 64; c += 4) {
            const float2 x0 = __ffma2_rn(make_float2(__uint_as_float(r[c]), __uint_as_float(r[c + 1])), scale2, negm2);
            const float2 x1 = __ffma2_rn(make_float2(__uint_as_float(r[c + 2]), __uint_as_float(r[c + 3])), scale2, negm2);
            const float2 p0 = make_float2(ex2f(x0.x), ex2f(x0.y));
            const float2 p1 = make_float2(ex2f(x1.x), ex2f(x1.y));
            l0 = __fadd2_rn(l0, p0);
            l1 = __fadd2_rn(l1, p1);
            r[c >> 1] = pack_bf16(p0.x, p0.y);
            r[(c >> 1) + 1] = pack_bf16(p1.x, p1.y);
          }
          tmem_st32(tS + 32 * hc, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
          lsum2 = __fadd2_rn(lsum2, __fadd2_rn(l0, l1));
          tmem_wait_st();
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) arrive_cl(lbar(B_P + sb), 1);
        if (rloc == 0 && hc == 0) PT(PT_SM_P, g);
      }
      // the item's (l, m) of this half for the epilogue warpgroup
      if (kk >= 2) fwait(bar(B_LF + (kk & 1)), ((kk - 2) >> 1) & 1, bar0);
      lbuf[((kk & 1) * 2 + hc) * 128 + rloc] = make_float2(lsum2.x + lsum2.y, m);
      mbar_arrive(bar(B_LR + (kk & 1)));
    }
  } else if (warp < 12) {
    // ================================================================ rotation + Q prep + epilogue
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegAux));
    const int lt = threadIdx.x - 256;
    const int c8 = lt & 7;             // frequencies 8*c8 .. 8*c8+7
    const int rg = lt >> 3;            // key rows rg*4 .. rg*4+3 of this CTA's half
    const float4* __restrict__ rp = p.rope_pairs;
    float2 cth[4], sth[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float4 t = rp[32 + 4 * c8 + j];
      cth[j] = make_float2(t.x, t.y);
      sth[j] = make_float2(t.z, t.w);
    }
    auto prep_q = [&](int kq) {
      const ItemRec rq = load_rec(recs, kq);
      const AttnParams& pq = REC_PARAMS(rq);
      const Item wq = item_of(pq, rq);
      uint4 lo[8], hi[8];
      if (lt == 0) PT(PT_Q_START, kq);
      if (!PR_ABL_Q) load_rotate_q_regs(pq, wq, rank, lt, lo, hi);
      if (kq >= NQB) fwait(bar(B_QF + (kq & 1)), ((kq - NQB) >> 1) & 1, bar0);
      if (lt == 0) PT(PT_Q_FREE, kq);
      const uint32_t qtile = qbuf_addr(kq);
      const int rg8 = lt >> 3;
#pragma unroll
      for (int k = 0; k < 8 * (1 - PR_ABL_Q); ++k) {
        const int r = rg8 * 8 + k;
        const uint32_t a = qtile + r * 128 + ((c8 ^ (r & 7)) << 4);
        sts128(a, lo[k]);
        sts128(a + 16384, hi[k]);
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) arrive_cl(lbar(B_QR + (kq & 1)), 1);
      if (lt == 0) PT(PT_Q_END, kq);
    };
    // item ke's O: read out of TMEM at once (the next item's first PV waits for it), then / l
    auto epilogue = [&](int ke) {
      const ItemRec rec = load_rec(recs, ke);
      const AttnParams& p = REC_PARAMS(rec);
      const Item w = item_of(p, rec);
      fwait(bar(B_LR + (ke & 1)), (ke >> 1) & 1, bar0);
      const float2 lm0 = lbuf[((ke & 1) * 2 + 0) * 128 + lt], lm1 = lbuf[((ke & 1) * 2 + 1) * 128 + lt];
      mbar_arrive(bar(B_LF + (ke & 1)));
      const int rglob = w.m0 + rank * 128 + lt;
      const bool valid_row = rglob < w.rows_total;
      const int qi = valid_row ? rglob / p.grp : 0;
      const int h = valid_row ? w.g * p.grp + rglob % p.grp : 0;
      const float lsum = lm0.x + lm1.x;
      const float inv = lsum > 0.f ? 1.f / lsum : 0.f;
      const bool part = p.n_splits > 1 || p.split_only >= 0;
      fwait(bar(B_O + ke % NOB), (ke / NOB) & 1, bar0);
      if (lt == 0) PT(PT_EPI_O, ke);
      tc_fence_after();
      const uint32_t tO = tO_base + (uint32_t)((ke % NOB) * 128) + ((uint32_t)((lt >> 5) * 32) << 16);
      uint32_t r[64];
      if (!part) {
        uint32_t pk[64];   // O / l as bf16 pairs: the O columns leave TMEM before any store
#pragma unroll 1
        for (int hf = 0; hf < 2; ++hf) {
          if (!PR_ABL_EPI) {
            tmem_ld32x(tO + 64 * hf, &r[0]);
            tmem_ld32x(tO + 64 * hf + 32, &r[32]);
            tmem_wait_ld();
          }
#pragma unroll
          for (int j = 0; j < 32; ++j)
            pk[32 * hf + j] = pack_bf16(__uint_as_float(r[2 * j]) * inv, __uint_as_float(r[2 * j + 1]) * inv);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) arrive_cl(lbar(B_OF + ke % NOB), 1);   // this O buffer may take item ke + NOB
        if (valid_row && !PR_ABL_EPI) {
          const bool peers = p.n_peers > 0;
          int oq = qi + p.o_rot;   // o_rot = 0 unless ring-ordered output (o_rows > 0)
          if (p.o_rows > 0 && oq >= p.o_rows) oq -= p.o_rows;
          const long long row = peers ? ((long long)w.pp * p.n_q + qi) * p.o_hq + p.o_head_off + h
                                      : ((long long)w.pp * (p.o_rows > 0 ? p.o_rows : p.n_q) + oq) * p.Hq + h;
          DSC_ASSERT(qi < p.n_q && w.pp < p.P && h < p.Hq && oq < (p.o_rows > 0 ? p.o_rows : p.n_q), "attn_pair O row");
          const int nd = peers ? p.n_peers : 1;
#pragma unroll 1
          for (int d = 0; d < nd; ++d) {
            __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(peers ? p.peer_o[d] : p.o) + row * 128;
#pragma unroll
            for (int v = 0; v < 8; ++v) stg256(dst + 16 * v, *reinterpret_cast<const uint32_t(*)[8]>(&pk[8 * v]));
          }
        }
      } else {
        // split-KV / context-parallel partial: fp32 O / l and log2-sum-exp per split
        const long long orow = ((long long)w.pp * p.n_q + qi) * p.Hq + h;
        const long long rows = (long long)p.P * p.n_q * p.Hq;
        const long long slot = p.split_only >= 0 ? 0 : w.sp;
        DSC_ASSERT(!valid_row || (slot < max(p.n_splits, 1) && orow < rows), "attn_pair split partial row");
#pragma unroll 1
        for (int hf = 0; hf < 2; ++hf) {
          tmem_ld32x(tO + 64 * hf, &r[0]);
          tmem_ld32x(tO + 64 * hf + 32, &r[32]);
          tmem_wait_ld();
          if (hf == 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) arrive_cl(lbar(B_OF + ke % NOB), 1);
          }
          if (!valid_row) continue;
          float4* dst = reinterpret_cast<float4*>(p.ws_o + (slot * rows + orow) * 128 + 64 * hf);
#pragma unroll
          for (int v = 0; v < 16; ++v)
            dst[v] = make_float4(__uint_as_float(r[4 * v]) * inv, __uint_as_float(r[4 * v + 1]) * inv,
                                 __uint_as_float(r[4 * v + 2]) * inv, __uint_as_float(r[4 * v + 3]) * inv);
          if (hf == 0) p.ws_lse[slot * rows + orow] = lsum > 0.f ? lm0.y + __log2f(lsum) : -INFINITY;
        }
      }
      if (lt == 0) PT(PT_EPI_END, ke);
    };
    // Jobs in global tile order: tile g's K half rotated (raw K only), item k+1's Q after the
    // first tile of item k, and item e's epilogue once the tiles whose QK^T precede e's last
    // PV in the issue order (S runs two tiles ahead) are rotated.
    int gt = 0, ep = 0;   // ep: next item to write out
    int ep_last = n_my > 0 ? load_rec(recs, 0).n_tiles - 1 : 0;   // global index of item ep's last tile
    int qn = 0;           // next item whose Q tile to prepare
    for (int kk = 0; kk <= n_my; ++kk) {
      const bool real = kk < n_my;
      const ItemRec rec = load_rec(recs, real ? kk : 0);
      const AttnParams& p = REC_PARAMS(rec);
      const Item w = item_of(p, rec);
      const bool rot = real && !w.staged;
      const int A = w.A;
      const bool dbg = p.dbg_pos != nullptr && w.g == 0;   // every problem, kv head 0
      int* const dbgp = dbg ? p.dbg_pos + (w.head_row / p.Hkv) * p.dbg_len : nullptr;
      const int n = real ? w.n_tiles : 1;
#pragma unroll 1
      for (int jj = 0; jj < n; ++jj) {
        const int g = gt + jj, u = w.t_begin + jj, ks = g % KST;
        if (rot) {
          // this thread's 4 key rows: lr = rg*4 .. rg*4+3 of the CTA's half (tile rows rank*nh + lr)
          int nh, p0 = -1;
          bool consec;
          int kpos[4];
          const uint32_t tile = sbase + OFF_K + ks * kKBytes;
          if (u >= w.n_extra) {   // window tile: ids A + 128 b + row, rows < valid
            const int base = BN * (u - w.n_extra);
            const int valid = min(w.cnt - base, BN);
            nh = (((valid + 15) & ~15) + 31 & ~31) >> 1;
            const int row0 = rank * nh + rg * 4;
#pragma unroll
            for (int k = 0; k < 4; ++k) kpos[k] = (rg * 4 + k < nh && row0 + k < valid) ? w.A + base + row0 + k : -1;
            consec = row0 + 3 < valid && rg * 4 + 3 < nh;
          } else {
            const TileSeg tg = tile_segments<BN>(p, w, u);
            nh = width2(tg) >> 1;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int lr = rg * 4 + k;
              kpos[k] = lr < nh ? seg_pos(tg, rank * nh + lr) : -1;
            }
            consec = false;
          }
#pragma unroll
          for (int k = 3; k >= 0; --k)
            if (kpos[k] >= 0) p0 = kpos[k];
          float4 pre[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) pre[j] = rp[(long long)max(p0, 0) * 32 + 4 * c8 + j];
          if (lt == 0) PT(PT_ROT_PRE, g);
          fwait(bar(B_KR + ks), (g / KST) & 1, bar0);
          if (lt == 0) PT(PT_ROT_KR, g);
          if (!PR_ABL_ROT) {
            if (__all_sync(0xffffffffu, consec))
              rotate4_consec<kKHalf>(tile, rg * 4, c8, cth, sth, pre);
            else if (rg * 4 < nh)   // rows >= nh are never read by the MMA
              rotate_rows<1, kKHalf>(tile, rg * 4, c8, rp, cth, sth, kpos, pre, max(p0, 0));
          }
          if (lt == 0) PT(PT_ROT_RR, g);
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) arrive_cl(lbar(B_KF + ks), 1);
          if (lt == 0) PT(PT_ROT, g);
          if (lt == 32) PT(PT_ROT9, g);
          if (lt == 64) PT(PT_ROT10, g);
          if (lt == 96) PT(PT_ROT11, g);
          if (dbg && c8 == 0) {
            const TileSeg tg = tile_segments<BN>(p, w, u);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int rr = rank * nh + rg * 4 + k;
              const int x = BN * u + rr;
              int slot = tg.slot0 + rr;
              if (slot >= p.R) slot -= p.R;
              if (kpos[k] >= 0)
                dbgp[(u < w.n_extra) ? (x < A ? x : p.dbg_A + p.dbg_R + (x - A)) : p.dbg_A + slot] = kpos[k];
            }
          }
        }
        // Q tiles of items up to kk + 1 (item 0's and 1's after item 0's first K tile)
        if (jj == 0) {
#pragma unroll 1
          for (; qn <= kk + 1 && qn < n_my; ++qn) prep_q(qn);
        }
        // epilogue of item ep once tile last(ep) + 2 is rotated (its S goes out before the
        // next item's first PV, which waits for this read-out)
#pragma unroll 1
        while (ep < kk && (!real || ep_last + 2 <= g)) {
          epilogue(ep);
          ++ep;
          if (ep < n_my) ep_last += load_rec(recs, ep).n_tiles;
        }
      }
      if (real) gt += w.n_tiles;
    }
  } else {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegMisc));
    if (warp == 12 || warp == 13) {
      // ============================================================== copy warps (12: K half, 13: V columns)
      const bool isk = warp == 12;
      int gt = 0;
      for (int kk = 0; kk < n_my; ++kk) {
        const ItemRec rec = load_rec(recs, kk);
        const AttnParams& p = REC_PARAMS(rec);
        const Item w = item_of(p, rec);
        const int A = p.A;
        const __nv_bfloat16* __restrict__ SX = reinterpret_cast<const __nv_bfloat16*>(isk ? p.sink_k : p.sink_v);
        const __nv_bfloat16* __restrict__ XX = reinterpret_cast<const __nv_bfloat16*>(isk ? p.self_k : p.self_v);
#pragma unroll 1
        for (int jj = 0; jj < w.n_tiles; ++jj) {
          const int g = gt + jj, u = w.t_begin + jj;
          const int nst = isk ? KST : VST, st = g % nst;
          if (g >= nst) fwait(bar((isk ? B_KE : B_VE) + st), ((g - nst) / nst) & 1, bar0);
          const uint32_t full = bar((isk ? B_KR : B_VL) + st);
          const uint32_t dst = sbase + (isk ? OFF_K + st * kKBytes : OFF_V + st * kVBytes);
          const TileSeg t = tile_segments<BN>(p, w, u);
          const int nu = width2(t), nh = nu >> 1;
          if (u < w.n_extra) {
            // sink rows (x < A) + self rows (A <= x < A + n_self), zeros up to the pair width
            const int nrows = isk ? nh : nu;
            const int cpr = isk ? 16 : 8;          // 16-byte chunks per row this CTA loads
            const int key0 = isk ? rank * nh : 0;
            const int col0 = isk ? 0 : 64 * rank;
#pragma unroll 1
            for (int id = lane; id < nrows * cpr; id += 32) {
              const int rr = id / cpr, ch = id % cpr;
              const int x = BN * u + key0 + rr;
              const __nv_bfloat16* src = nullptr;
              if (x < A) src = SX + ((long long)w.head_row * A + x) * 128;
              else if (x < A + w.n_self) src = XX + (((long long)w.pp * w.n_self + (x - A)) * p.Hkv + w.g) * 128;
              DSC_ASSERT(w.head_row < (long long)p.S * p.N_total * p.Hkv && w.pp < p.P, "attn_pair sink/self row");
              const uint32_t d = isk ? dst + (ch >> 3) * kKHalf + rr * 128 + (((ch & 7) ^ (rr & 7)) << 4)
                                     : dst + rr * 128 + ((ch ^ (rr & 7)) << 4);
              cp_async16(d, src ? (const void*)(src + col0 + 8 * ch) : (const void*)SX, src ? 16u : 0u);
            }
            cp_async_wait_all();
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) mbar_arrive(full);
          } else if (lane == 0) {
            const int row = (int)(w.head_row * w.Rp) + t.slot0;
            DSC_ASSERT(t.slot0 >= 0 && t.slot0 < w.Rp && (w.staged || t.slot0 + BN <= w.Rp) &&
                           w.head_row < (long long)p.S * p.N_total * p.Hkv,
                       "attn_pair TMA box rows");
            PT(isk ? PT_CPK : PT_CPV, g);
            if (isk) {
              mbar_arrive_tx(full, kKBytes);
              tma_load_2d(dst, &p.tmap_k64, 0, row + rank * nh, full);
              tma_load_2d(dst + kKHalf, &p.tmap_k64, 64, row + rank * nh, full);
            } else {
              mbar_arrive_tx(full, kVBytes);
              tma_load_2d(dst, &p.tmap_v, 64 * rank, row, full);
            }
          }
          __syncwarp();
        }
        gt += w.n_tiles;
      }
    } else if (warp == 15) {
      // ============================================================== forwarder
      if (lane == 0) {
        int gt = 0;
        for (int kk = 0; kk < n_my; ++kk) {
          const ItemRec rec = load_rec(recs, kk);
          const bool staged = REC_PARAMS(rec).staged;
          const int n = rec.n_tiles;
#pragma unroll 1
          for (int jj = 0; jj < n; ++jj) {
            const int g = gt + jj;
            if (staged) {   // pre-rotated K: landed = ready
              fwait(bar(B_KR + g % KST), (g / KST) & 1, bar0);
              arrive_cl(lbar(B_KF + g % KST), 4);
              PT(PT_KR_FW, g);
            }
            fwait(bar(B_VL + g % VST), (g / VST) & 1, bar0);
            arrive_cl(lbar(B_VR + g % VST), 1);
            PT(PT_FWV, g);
          }
          gt += n;
        }
      }
    } else if (warp == 14 && rank == 0) {
      // ============================================================== MMA issuer (leader)
      constexpr uint32_t IQK0 = idesc_bf16(256, 0, 0, 0);    // S = Q K^T, both K-major; N = pair width
      constexpr uint32_t IPV = idesc_bf16(256, 128, 0, 1);   // O += P V, P from TMEM, V MN-major
      struct MI {
        int n, t_begin, n_extra, aps, cnt;
      };
      auto mi_of = [&](int kk) {
        const ItemRec r = load_rec(recs, kk);
        const bool isb = r.flags & 1;
        const int A = isb ? pb.A : pa.A, n_self = isb ? pb.n_self : pa.n_self;
        MI m;
        m.n = r.n_tiles; m.t_begin = r.t_begin;
        m.n_extra = (A + n_self + BN - 1) / BN; m.aps = A + n_self; m.cnt = r.cnt;
        return m;
      };
      auto width_of = [&](const MI& m, int jj) {   // tile_segments' valid keys, rounded up to 32
        const int u = m.t_begin + jj;
        const int valid = u < m.n_extra ? min(max(m.aps - BN * u, 0), BN) : min(m.cnt - BN * (u - m.n_extra), BN);
        return (valid + 31) & ~31;
      };
      // S(g) of item k, local tile jj: ready once the item's Q tile (jj = 0) and the K tile are
      auto ready_s = [&](int k, int jj, int g) {
        if (jj == 0 && !mbar_test(bar(B_QR + (k & 1)), (k >> 1) & 1)) return false;
        return mbar_test(bar(B_KF + g % KST), (g / KST) & 1);
      };
      auto issue_s = [&](const MI& m, int k, int jj, int g) {
        const int ks = g % KST, qb = k & 1, sb = g % NSB;
        if (lane == 0) PT(PT_KF_OK, g);
        tc_fence_after();
        const int nu = width_of(m, jj);
        const uint64_t da = sdesc(qbuf_addr(k), 16, 1024);
        const uint64_t db = sdesc(sbase + OFF_K + ks * kKBytes, 16, 1024);
        if (lane == 0) PT(PT_S_FENCE, g);
        mma2_qk(tmem + (uint32_t)(sb * 128), da, db, IQK0 | ((uint32_t)(nu >> 3) << 17));
        if (lane == 0) PT(PT_S_MMA, g);
        commit2_w(bar(B_S + sb));
        commit2_w(bar(B_KE + ks));
        if (jj + 1 == m.n) commit2_w(bar(B_QF + qb));
        if (lane == 0) PT(PT_S_ISS, g);
        if (jj == 0 && lane == 0) PT(PT_ITEM, k);
      };
      // PV(g): V tile, P (both CTAs) and, for an item's first PV, the previous item's O read out
      auto ready_pv = [&](int k, int jj, int g) {
        if (!mbar_test(bar(B_VR + g % VST), (g / VST) & 1)) return false;
        if (!mbar_test(bar(B_P + g % NSB), (g / NSB) & 1)) return false;
        return !(jj == 0 && k >= NOB) || mbar_test(bar(B_OF + k % NOB), ((k - NOB) / NOB) & 1);
      };
      auto issue_pv = [&](const MI& m, int k, int jj, int g) {
        const int vs = g % VST, sb = g % NSB;
        if (lane == 0) PT(PT_P_OK, g);
        tc_fence_after();
        const int nu = width_of(m, jj);
        const uint64_t dv = sdesc(sbase + OFF_V + vs * kVBytes, 16, 1024);
        const uint32_t d = tO_base + (uint32_t)((k % NOB) * 128), a = tmem + (uint32_t)(sb * 128);
        const uint32_t acc = jj > 0 ? 1u : 0u;
        if (nu == BN) {
          mma2_pv8(d, a, dv, IPV, acc);
        } else {
          mma2_pv1(d, a, dv, IPV, acc);
#pragma unroll 1
          for (int k8 = 1; k8 < (nu >> 4); ++k8) mma2_pv1(d, a + k8 * 8, dv + (uint64_t)(k8 * 128), IPV, 1u);
        }
        if (lane == 0) PT(PT_PV_MMA, g);
        commit2_w(bar(B_VE + vs));
        if (jj + 1 == m.n) commit2_w(bar(B_O + k % NOB));
        if (lane == 0) PT(PT_PV_ISS, g);
      };
      // Two cursors over the same tile sequence, each issued as soon as its operands are
      // ready: S(s) at most two tiles ahead of the next PV (S buffer s % 3 held P(s - 3),
      // whose PV is then already issued: tcgen05 MMAs of one thread execute in order), and
      // PV(v) after S(v).  A late K tile no longer holds back a PV whose P is ready.
      if (n_my > 0) {
        int s_k = 0, s_jj = 0, s_g = 0, v_k = 0, v_jj = 0, v_g = 0;
        MI s_m = mi_of(0), v_m = s_m;
        long long t_idle = 0;
        while (v_k < n_my) {
          bool did = false;
          if (s_k < n_my && s_g <= v_g + (NSB - 1) && ready_s(s_k, s_jj, s_g)) {
            issue_s(s_m, s_k, s_jj, s_g);
            ++s_g;
            if (++s_jj == s_m.n) {
              s_jj = 0;
              if (++s_k < n_my) s_m = mi_of(s_k);
            }
            did = true;
          }
          if (v_g < s_g && ready_pv(v_k, v_jj, v_g)) {
            issue_pv(v_m, v_k, v_jj, v_g);
            ++v_g;
            if (++v_jj == v_m.n) {
              v_jj = 0;
              if (++v_k < n_my) v_m = mi_of(v_k);
            }
            did = true;
          }
          if (did) {
            t_idle = 0;
          } else {   // both queues blocked: back off instead of spinning on the SMSP (the
                     // sleep plus the watchdog check's global load make a ~0.5K clk backoff;
                     // a tight test_wait poll slows the rotation / softmax warps of this
                     // sub-partition, a suspending in-order issuer measured slower too)
            __nanosleep(32);
            if (t_idle == 0) t_idle = clock64();
            else if (clock64() - t_idle > fa::g_fa_wd_lim) fa::fa_wd_fail(B_P, v_g);
          }
        }
        fwait(bar(B_VE + (v_g - 1) % VST), ((v_g - 1) / VST) & 1, bar0);
        if (lane == 0) PT(PT_END, 0);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  if (warp == 14) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
#undef REC_PARAMS
}

}  // namespace pr

int attn_fa_smem_bytes() { return fa::kSmemBytes; }

namespace {
// per-device one-time kernel attributes (a process may drive handles on several GPUs)
std::mutex g_cfg_mu;
uint64_t g_cfg_done = 0;
int g_num_sms[64] = {0};
cudaError_t configure_device(int* num_sms) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(g_cfg_mu);
  if (dev < 64 && (g_cfg_done >> dev) & 1) { *num_sms = g_num_sms[dev]; return cudaSuccess; }
  e = cudaFuncSetAttribute(fa::attn_fa_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, fa::kSmemBytes);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(pr::attn_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, pr::kSmemBytes);
  if (e != cudaSuccess) return e;
  int sms = 0;
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  if (dev < 64) { g_cfg_done |= 1ull << dev; g_num_sms[dev] = sms; }
  *num_sms = sms;
  return cudaSuccess;
}
}  // namespace

long long attn_fa_items(const AttnParams& p) {
  return (long long)p.P * p.Hkv * p.n_mblocks * (p.split_only >= 0 ? 1 : p.n_splits);
}
// the host decode of one work item (the kernel reads these records instead of decoding)
ItemRec attn_fa_decode(const AttnParams& p, int local, int isb) {
  const tcc::Item w = tcc::decode_item<fa::BN>(p, local);
  ItemRec r;
  r.pp = w.pp; r.head_row = (int)w.head_row; r.m0 = w.m0; r.t_begin = w.t_begin; r.n_tiles = w.n_tiles;
  r.cnt = w.cnt; r.flags = isb | (w.g << 8); r.sp = w.sp;
  return r;
}

// DSC_WATCHDOG=1: pipeline waits that time out leave a record in host-mapped memory
// (dscache_watchdog_read) before trapping
// DSC_WATCHDOG_CLK=N: the timeout in clk (0 = never trap; e.g. under compute-sanitizer,
// which slows every wait by orders of magnitude)
static unsigned long long* g_wd_host = nullptr;
cudaError_t fa_watchdog_setup() {
  static unsigned done_mask = 0;   // per device: the symbols live in each device's module
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 32 && (done_mask & (1u << dev))) return cudaSuccess;
  if (dev < 32) done_mask |= 1u << dev;
  if (const char* c = std::getenv("DSC_WATCHDOG_CLK")) {
    long long lim = std::atoll(c);
    if (lim <= 0) lim = 0x7fffffffffffffffll;
    cudaError_t r = cudaMemcpyToSymbol(fa::g_fa_wd_lim, &lim, sizeof(lim));
    if (r != cudaSuccess) return r;
  }
  const char* e = std::getenv("DSC_WATCHDOG");
  if (!e || e[0] != '1') return cudaSuccess;
  if (!g_wd_host) {
    void* hp = nullptr;
    cudaError_t r = cudaHostAlloc(&hp, 4096, cudaHostAllocMapped | cudaHostAllocPortable);
    if (r != cudaSuccess) return r;
    std::memset(hp, 0, 4096);
    g_wd_host = static_cast<unsigned long long*>(hp);
  }
  void* dp = nullptr;
  cudaError_t r = cudaHostGetDevicePointer(&dp, g_wd_host, 0);
  if (r != cudaSuccess) return r;
  return cudaMemcpyToSymbol(fa::g_fa_wd, &dp, sizeof(dp));
}
int fa_watchdog_read(unsigned long long* out, int n) {
  if (!g_wd_host) return -1;
  for (int i = 0; i < n && i < 512; ++i) out[i] = reinterpret_cast<volatile unsigned long long*>(g_wd_host)[i];
  return 0;
}

// Default: the CTA-pair kernel (v8); DSC_FA=7 selects the single-CTA v7 kernel (A/B runs)
static bool pair_kernel_on() {
  static const bool on = [] {
    const char* e = std::getenv("DSC_FA");
    return !(e && e[0] == '7');
  }();
  return on;
}

cudaError_t launch_attn_fa(const AttnParams& pa, const AttnParams* pb, SchedCache* cache, cudaStream_t st) {
  int num_sms = 0;
  cudaError_t e = configure_device(&num_sms);
  if (e != cudaSuccess) return e;
  e = fa_watchdog_setup();
  if (e != cudaSuccess) return e;
  const long long na = attn_fa_items(pa), nb = pb ? attn_fa_items(*pb) : 0;
  const long long items = na + nb;
  if (items == 0) return cudaSuccess;
  if (pair_kernel_on() && (!pa.trace || PR_TRACE)) {
    // v8: one item per CTA pair, num_sms / 2 clusters
    const long long ncl_max = num_sms / 2;
    const unsigned ncl = (unsigned)(items < ncl_max ? items : ncl_max);
    AttnParams qa = pa;
    const int* off = nullptr;
    qa.item_recs = item_table(cache, pa, pb, na, nb, ncl, &attn_fa_decode, &off, st);
    qa.item_off = off;
    if (!qa.item_recs) return cudaErrorMemoryAllocation;
    pr::attn_pair_kernel<<<2 * ncl, pr::kThreads, pr::kSmemBytes, st>>>(qa, pb ? *pb : qa, (int)na, (int)nb);
    return cudaGetLastError();
  }
  const unsigned grid = (unsigned)(items < num_sms ? items : num_sms);
  AttnParams qa = pa;
  const int* off = nullptr;
  qa.item_recs = item_table(cache, pa, pb, na, nb, grid, &attn_fa_decode, &off, st);
  qa.item_off = off;
  if (!qa.item_recs) return cudaErrorMemoryAllocation;
  fa::attn_fa_kernel<<<grid, fa::kThreads, fa::kSmemBytes, st>>>(qa, pb ? *pb : qa, (int)na, (int)nb);
  return cudaGetLastError();
}

}  // namespace dsc
