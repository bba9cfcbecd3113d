// K3/K4: fused rotate-on-load RoPE + GQA flash attention on the sm_100a tensor
// cores (tcgen05.mma, accumulators in TMEM), used by both dscache_build_instant
// (Eq. 7: instant tokens over [sink | instant], causal) and dscache_attend
// (Eq. 8 + self: the query chunk over [sink | past | instant | self]).
//
// Position-agnostic encoding (Def. 4.1): the ring holds raw
// K; each K tile is rotated in registers by its use-time id (consecutive from 0,
// PAPER.md:236) while it sits in shared memory, once per CTA for the 256 query rows
// (2 x 128-row Q tiles) that share it.  Softmax a_ij = softmax(Q_i K_j / sqrt(d))
// in the exp2 domain with lazy rescale.
//
// Persistent CTAs (grid <= #SMs) walk a list of work items (problem, kv head,
// 256-row m-block, key split); every pipeline phase runs on a CTA-global tile counter
// g, Q and O are recycled across items by barriers.
//
// Key tiles are 64 keys wide, so S of each Q tile is DOUBLE-BUFFERED in TMEM: the MMA
// computes S(g+1) (and issues S(g+2) right after PV(g)) while the softmax works on
// S(g), and a softmax warpgroup moves to its next tile without waiting for the tensor
// core.  TMEM (512 columns):
//   S[qt][b] = cols qt*128 + b*64 (b = g & 1)   O[qt] = cols 256 + qt*128
// P(g) (bf16x2, 32 columns) overwrites the first half of S[qt][g&1] and feeds
// O[qt] += P V as the TMEM A operand.  MMA issue order per tile g (after the item's
// prologue S(g0), S(g0+1)): PV0(g) PV1(g) S0(g+2) S1(g+2) (DSC_SORDER 0).
//
// CTA = 16 warps:
//   warps 0-3  softmax of Q tile 0 (thread = query row = TMEM lane); one TMEM read per
//              tile (64 columns), row max, exps, P store
//   warps 4-7  softmax of Q tile 1
//   warps 8-11 rotation: every raw K tile in place in shared memory
//              (LDS -> rotate -> STS), with R(p+1) = R(p) R(1) between consecutive ids,
//              and the Q tiles of the NEXT item (loaded + rotated into the other Q set,
//              DSC_QROT); the first item's Q tiles are prepared by the softmax warpgroups
//              (DSC_Q0SM), which are idle until the first S arrives
//   warp 12    K copy: raw K tiles -> SW128 smem; TMA (2 x 64x64 boxes) for window
//              tiles, cp.async for sink/self tiles
//   warp 13    V copy: same for V (K and V stage recycling is independent)
//   warp 14    TMEM allocator + MMA issuer (whole warp, elected lane issues)
//   warp 15    idle (second MMA issuer with DSC_MMA2)
// Registers (setmaxnreg): softmax 144, rotation 136, copy/MMA 88.
#include "tc_common.cuh"

#include <algorithm>
#include <mutex>
#include <utility>
#include <vector>

namespace dsc {
namespace tc {
using namespace tcc;

constexpr int kNQT = 2;                       // Q tiles per CTA
constexpr int kWarps = 16;
constexpr int kThreads = kWarps * 32;
constexpr int kQBytes = 128 * 128 * 2;        // one 128-row Q tile (2 x 64-column SW128 blocks)
constexpr int kKT = kTileN;                   // keys per K/V tile
constexpr int kKVHalf = kKT * 128;            // bytes of one 64-column SW128 block of a K/V tile
constexpr int kKVBytes = 2 * kKVHalf;         // one K or V tile (16 KB)
// DSC_QROT: the rotation warpgroup loads + rotates every item's Q tiles (into the second Q
// buffer, a whole item ahead), so item switches cost the softmax warpgroups only their
// epilogue; staged build items need no K rotation, so their K tiles go straight from the
// copy warp to the MMA (the rotation warpgroup is free for Q during builds)
#ifndef DSC_QROT
#define DSC_QROT 1
#endif
// DSC_Q0SM 1: the softmax warpgroups (idle until the first S) load + rotate the FIRST item's
// Q tiles, so the rotation warpgroup starts on the first K tiles at once instead of after
// both Q tiles (launch latency of small launches: c2 / c4 CTAs run only 1-3 items;
// measured c2 +4.5%, c4 +3%, c5 +0.2%)
#ifndef DSC_Q0SM
#define DSC_Q0SM 1
#endif
// DSC_Q2ISSUE 1: the rotation warpgroup issues both Q tiles' cp.async before rotating either
// (measured 1-3% slower on c2 / c4 / c5: off)
#ifndef DSC_Q2ISSUE
#define DSC_Q2ISSUE 0
#endif
// DSC_LASTO 1: O_qt is committed once per item (after its last PV) instead of per tile: a
// rescale waits on the V-stage-free commit of tile g-1 (PV0 and PV1 of g-1 complete)
#ifndef DSC_LASTO
#define DSC_LASTO 1
#endif
// DSC_OFHALF 1: O_qt is released to the next item in two column halves (see issue_pv_half)
#ifndef DSC_OFHALF
#define DSC_OFHALF 0
#endif
// DSC_EXBF 1: softmax exponentials as ex2.approx.bf16x2 (the exponent argument rounded to
// bf16, two columns per MUFU op; P is bf16 for the PV MMA anyway and l sums that same P)
#ifndef DSC_EXBF
#define DSC_EXBF 0
#endif
// DSC_PJOIN 1: one P-ready barrier per S buffer for BOTH softmax warpgroups (256 arrivals):
// the MMA warp waits once per tile before PV0 PV1 instead of once per Q tile
#ifndef DSC_PJOIN
#define DSC_PJOIN 0
#endif
// DSC_PAIR 1: softmax / MMA handshakes per PAIR of 64-key tiles (128 keys): S single-
// buffered per Q tile over both 64-column halves, PV(pair) then S(next pair) per Q tile
#ifndef DSC_PAIR
#define DSC_PAIR 0
#endif
// DSC_QLDG 1: the rotation warpgroup reads Q rows from global into registers, rotates and
// stores them once (else cp.async into the tile, then an in-place rotation pass)
#ifndef DSC_QLDG
#define DSC_QLDG 0
#endif
// DSC_QSINGLE 1: one Q tile set; the rotation warpgroup refills it for the next item as
// soon as the current item's last QK^T has completed (B_QE is committed right after that
// MMA, two tiles before the item ends), and the 64 KB the second set took become K/V
// stages (5 + 5): more TMA loads in flight against the HBM latency
#ifndef DSC_QSINGLE
#define DSC_QSINGLE 0
#endif
#ifndef DSC_QDB   // double-buffered Q tiles (next item's Q loaded + rotated during the current item)
#define DSC_QDB (DSC_QROT && !DSC_QSINGLE)
#endif
static_assert(!DSC_QROT || DSC_QDB || DSC_QSINGLE, "DSC_QROT needs the Q double buffer or DSC_QSINGLE");
static_assert(!DSC_QSINGLE || (DSC_QROT && !DSC_QDB), "DSC_QSINGLE is the single-set variant of DSC_QROT");
#ifndef DSC_KST
#define DSC_KST (DSC_QDB ? 3 : (DSC_QSINGLE ? 5 : 6))
#endif
#ifndef DSC_VST
#define DSC_VST (DSC_QDB ? 3 : (DSC_QSINGLE ? 5 : 4))
#endif
constexpr int KST = DSC_KST;                  // K stages (raw -> rotated in place)
constexpr int VST = DSC_VST;                  // V stages
constexpr int kQBufs = DSC_QDB ? 2 : 1;       // Q tile sets (double-buffered: next item's Q prepared early)
constexpr int OFF_Q = 0;
constexpr int OFF_K = OFF_Q + kQBufs * kNQT * kQBytes;
constexpr int OFF_V = OFF_K + KST * kKVBytes;
constexpr int OFF_BAR = OFF_V + VST * kKVBytes;
// barriers (8 B each): Q ready [qt] | K raw landed | K rotated | K free | V landed | V free |
// S ready [qt][buf] | P ready [qt][buf] | PV done [qt][buf] | O read (epilogue done) [qt].
// Every barrier a waiter may lag is per buffer parity, so no waiter is ever two phases
// behind (the parity test of mbarrier.try_wait cannot tell phase k from phase k+2): with S
// prefetched two tiles ahead, PV(g-1) may still be pending when the softmax finishes tile g.
constexpr int B_Q = 0, B_KR = 2 * kQBufs, B_KF = B_KR + KST, B_KE = B_KF + KST, B_VF = B_KE + KST, B_VE = B_VF + VST,
              B_S = B_VE + VST, B_P = B_S + 4, B_O = B_P + 4, B_OF = B_O + 4, B_QE = B_OF + 2, B_EP = B_QE + 2, B_OFH = B_EP + 2,
              B_N = B_OFH + 2;
// setmaxnreg budget per warpgroup: 2*softmax + rotation + copy/MMA <= 512 (x 128 threads)
constexpr int kRegSoftmax = 144, kRegRotate = 136, kRegCopy = 88;
static_assert(2 * kRegSoftmax + kRegRotate + kRegCopy <= 512, "setmaxnreg budget exceeds the 64K register file");
constexpr int kThreadRegs = 65536 / kThreads;   // allocation at launch (128); inc above it, dec below it
static_assert(kRegSoftmax > kThreadRegs && kRegCopy < kThreadRegs, "softmax must grow, copy/MMA must shrink");
constexpr int kSmemBytes = OFF_BAR + B_N * 8 + 16 + 1024;   // + tmem slot + alignment slack
static_assert(kSmemBytes <= 227 * 1024, "shared memory budget");
static_assert(kKT == 64, "the S double buffer assumes 64-key tiles");
#ifndef DSC_RESCALE_T
#define DSC_RESCALE_T 8.0f
#endif
constexpr float kRescaleThreshold = DSC_RESCALE_T;   // log2 units (8: factor 256)
static_assert(kNQT * 128 == kMBlockRows, "work items are 256-row m-blocks");
#ifndef DSC_POLY
#define DSC_POLY 0
#endif
// ablation knobs (timing experiments only; results are wrong when set):
// DSC_ABL_MMAONLY: only the MMA warp runs, issuing every MMA and commit without waiting
// (measures the issue loop alone),
// DSC_ABL_SOFTMAX skips the softmax body, DSC_ABL_ROT skips the K rotation,
// DSC_ABL_EX2 replaces ex2 by a copy (MUFU-free softmax)
#ifndef DSC_ABL_MMAONLY
#define DSC_ABL_MMAONLY 0
#endif
// DSC_MWSLEEP > 0: the MMA warp backs off with nanosleep(DSC_MWSLEEP) between failed polls,
// leaving its sub-partition's issue slots to the two softmax warps that share it
// (measured: 128 ns c5 +0.7%, c3 +0.8% over plain polling; 32 ns mixed)
#ifndef DSC_MWSLEEP
#define DSC_MWSLEEP 128
#endif
__device__ __forceinline__ void mma_wait(uint32_t b, uint32_t ph) {
  if (DSC_MWSLEEP > 0) {
    if (tcc::mbar_try(b, ph)) return;
    const long long t0 = clock64();
    do {
      __nanosleep(DSC_MWSLEEP);
      if (clock64() - t0 > (1ll << 31)) __trap();   // same watchdog as mbar_wait
    } while (!tcc::mbar_try(b, ph));
  } else {
    tcc::mbar_wait(b, ph);
  }
}
#define MWAIT(b, ph) do { if (!DSC_ABL_MMAONLY) mma_wait((b), (ph)); } while (0)
#ifndef DSC_ABL_SOFTMAX
#define DSC_ABL_SOFTMAX 0
#endif
#ifndef DSC_ABL_ROT
#define DSC_ABL_ROT 0
#endif
#ifndef DSC_ABL_EX2
#define DSC_ABL_EX2 0
#endif
#ifndef DSC_ABL_TMEM
#define DSC_ABL_TMEM 0
#endif
#ifndef DSC_ABL_SWITCH   // ablation: item switches without the Q load/rotation (bit 0) / the O epilogue (bit 1)
#define DSC_ABL_SWITCH 0
#endif
#ifndef DSC_ABL_LOADS   // ablation: window K/V tiles are not loaded
#define DSC_ABL_LOADS 0
#endif
#ifndef DSC_ABL_NOWAIT_V   // ablation: the MMA warp does not wait for V tiles to land (measured: no change on
#define DSC_ABL_NOWAIT_V 0     // c5, so V arrival never gates the MMA; skipping the P or K waits breaks the phases)
#endif
#ifndef DSC_ABL_SMSP2   // ablation: the softmax warps sharing the MMA warp's sub-partition idle
#define DSC_ABL_SMSP2 0
#endif
constexpr int kPolyPerGroup = DSC_POLY;   // of every 8 columns of a full tile, this many use exp2_poly2
// DSC_MMA2 1: two MMA-issuing warps (14: Q tile 0, 15: Q tile 1).  Faster steady tiles,
// but warp 15 then competes for issue slots with the softmax/rotation warps of SMSP 3 and
// the item switches got slower: measured 11.1K vs 13.3K frames/s (c5), so off by default.
#ifndef DSC_MMA2
#define DSC_MMA2 0
#endif
// DSC_QPREF: L2 prefetch of the next item's Q rows at item start (measured slower, off)
#ifndef DSC_QPREF
#define DSC_QPREF 0
#endif
// DSC_SORDER: MMA order per tile -- 0 (default): PV0(g) PV1(g) S0(g+2) S1(g+2), two batches
// (measured +1.2% c5 / +1.3% c3 over 1 in round 1's last session); 1: PV0(g) S0(g+2) PV1(g)
// S1(g+2); 2: every wait first, then one burst
#ifndef DSC_SORDER
#define DSC_SORDER 0
#endif
#if DSC_QSINGLE && DSC_SORDER != 1
#error "DSC_QSINGLE commits the Q-free barrier in the DSC_SORDER 1 MMA loop (build with DSC_SORDER=1)"
#endif
// DSC_QEARLY 1: the next item's Q cp.async are issued at the last tile's S wait (else
// after the last tile)
#ifndef DSC_QEARLY
#define DSC_QEARLY 1
#endif
// DSC_INTERLEAVE: the fused step interleaves attend and build items per (problem, kv head)
#ifndef DSC_INTERLEAVE
#define DSC_INTERLEAVE 0
#endif
// DSC_EPIROT 1 (measured neutral on c5/c4/c2, off): the O epilogue of staged (build) items
// runs on the rotation warpgroup (idle
// there: staged K arrives rotated), so the softmax warpgroups go straight to the next item.
// The softmax hands l over through the item's consumed Q tile (B_EP), the rotation
// warpgroup reads O out of TMEM and releases it (B_OF) as the softmax would.
// (DSC_L2PF, a TMA L2 prefetch of the K/V tiles 2-8 tiles ahead, measured 1-3% slower and
// was removed)
#ifndef DSC_EPIROT
#define DSC_EPIROT 0
#endif
static_assert(!DSC_EPIROT || (DSC_QROT && !DSC_QSINGLE), "DSC_EPIROT hands l over through the other Q set");
static_assert(!DSC_PAIR || (!DSC_EPIROT && !DSC_QSINGLE && DSC_QROT), "DSC_PAIR: QROT path");
static_assert(!DSC_LASTO || (!DSC_PAIR && !DSC_EPIROT && DSC_SORDER != 2), "DSC_LASTO: SORDER 0/1 loops");
static_assert(!DSC_PJOIN || (!DSC_PAIR && !DSC_MMA2 && DSC_SORDER == 0), "DSC_PJOIN: SORDER 0 loop, one MMA warp");
// DSC_QFIRST 1: the next item's Q tile is published before the epilogue, so its first S
// MMAs run while O is read out
#ifndef DSC_QFIRST
#define DSC_QFIRST 1
#endif

// ------------------------------------------------------------------ kernel
// Two attention problems can share one persistent launch (the fused step: attend items
// first, then build_instant items); items [0, na) use pa, [na, na + nb) use pb.
__global__ void __launch_bounds__(kThreads, 1)
    attn_tc_kernel(const __grid_constant__ AttnParams pa, const __grid_constant__ AttnParams pb, int na, int nb, int ka,
                   int kb) {
  const AttnParams& p = pa;   // launch-wide fields (rope table, tensor maps, trace) are shared
#if DSC_TRACE
  long long* const trace_cta =
      (pa.trace && blockIdx.x < (unsigned)pa.ntrace_cta) ? pa.trace + (long long)blockIdx.x * kTraceEvents * kTraceTiles
                                                         : nullptr;
#endif
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // shared-window base computed from the dynamic-smem symbol itself (not via a generic
  // pointer) so the compiler keeps it, and every descriptor derived from it, uniform
  const uint32_t sbase = ((uint32_t)__cvta_generic_to_shared(smem_raw) + 1023u) & ~1023u;
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
    for (int i = 0; i < 2 * kQBufs; ++i) mbar_init(bar(B_Q + i), 128);
    for (int i = 0; i < KST; ++i) {
      mbar_init(bar(B_KR + i), 1);
      mbar_init(bar(B_KF + i), 128);
      mbar_init(bar(B_KE + i), DSC_MMA2 ? 2 : 1);   // one commit per MMA warp
    }
    for (int i = 0; i < VST; ++i) {
      mbar_init(bar(B_VF + i), 1);
      mbar_init(bar(B_VE + i), DSC_MMA2 ? 2 : 1);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(bar(B_S + i), 1);
      mbar_init(bar(B_P + i), DSC_PJOIN ? 256 : 128);   // PJOIN: both softmax WGs on B_P[buf]
      mbar_init(bar(B_O + i), 1);
    }
    for (int i = 0; i < 2; ++i) mbar_init(bar(B_OF + i), 128);
    for (int i = 0; i < 2; ++i) mbar_init(bar(B_OFH + i), 128);   // DSC_OFHALF: O columns 64..127 read
    for (int i = 0; i < 2; ++i) mbar_init(bar(B_QE + i), DSC_MMA2 ? 2 : 1);   // Q buffer i free (MMA commit(s) after an item)
    for (int i = 0; i < 2; ++i) mbar_init(bar(B_EP + i), 128); // l of a staged item handed to the rotation WG
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
    if (nb > 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&pb.tmap_k)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&pb.tmap_v)) : "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 12 && lane == 0) TRACE(EV_START, 1);   // prologue timeline (trace builds): after the CTA sync
  // one CTA per SM allocates all 512 columns, so the allocation is column 0 of lane 0;
  // the MMA descriptors use that constant (uniform registers, no per-MMA moves)
  const uint32_t tmem_alloc = *tmem_slot;
  if (tmem_alloc != 0u) __trap();
  constexpr uint32_t tmem = 0u;

  const int n_role_items = (DSC_ABL_MMAONLY && warp < 14) ? 0 : n_items;   // ablation: only the MMA issuer works
  // this CTA's items, in order: the launcher's list-scheduled work list, else the stride
  // blockIdx.x, + gridDim.x, ...  Every role walks the same sequence.
  const int* __restrict__ sched = pa.sched_items;
  const int sj0 = sched ? pa.sched_off[blockIdx.x] : 0;
  const int n_my = sched ? pa.sched_off[blockIdx.x + 1] - sj0
                         : (n_items > (int)blockIdx.x ? (n_items - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0);
  const int n_my_role = (DSC_ABL_MMAONLY && warp < 14) ? 0 : n_my;
  auto item_at = [&](int t) { return sched ? sched[sj0 + t] : (int)blockIdx.x + t * (int)gridDim.x; };
  if (warp < 8) {
    // ================================================================ softmax
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegSoftmax));
    const int qt = warp >> 2, quarter = warp & 3;
    const int rloc = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const uint32_t tS0 = tmem + lane_off + (uint32_t)(qt * 128);
    const uint32_t tO = tmem + lane_off + (uint32_t)(256 + qt * 128);
    const float sl2 = p.scale_log2;
    const float2 scale2 = make_float2(sl2, sl2);
    const uint32_t barS = bar(B_S + qt * 2), barP = bar(B_P + (DSC_PJOIN ? 0 : qt * 2));   // + 8 * buffer
    const int lt = threadIdx.x - qt * 128;           // 0..127 within the warpgroup
    auto qtile_of = [&](int kk) { return sbase + OFF_Q + (uint32_t)(((DSC_QDB ? (kk & 1) : 0) * 2 + qt) * kQBytes); };
    auto qbar_of = [&](int kk) { return bar(B_Q + (DSC_QDB ? (kk & 1) : 0) * 2 + qt); };
    if ((!DSC_QROT || DSC_Q0SM) && n_my_role > 0) {   // Q tile of the first item
      const int i0 = item_at(0);
      const AttnParams& p0 = ITEM_PARAMS(i0);
      const Item w0 = decode_item(p0, ITEM_LOCAL(i0));
      issue_q_tile(p0, w0, qt, lt, qtile_of(0));
      rotate_q_tile(p0, w0, qt, lt, qtile_of(0), 2 + qt);
      mbar_arrive(qbar_of(0));
    }
    int gt = 0, kk = 0, gp = 0;   // gp: tile pairs (DSC_PAIR)
    for (; kk < n_my_role; ++kk) {
      const int idx = item_at(kk);
      const AttnParams& p = ITEM_PARAMS(idx);
      const Item w = decode_item(p, ITEM_LOCAL(idx));
      const int A = w.A;
      const int n = w.n_tiles;
      const int nidx = kk + 1 < n_my_role ? item_at(kk + 1) : n_items;
      const bool has_next = nidx < n_role_items;
#if !DSC_QROT   // (with DSC_QROT the rotation warpgroup prepares the next item's Q)
      Item wn;
      if (has_next) wn = decode_item(ITEM_PARAMS(nidx), ITEM_LOCAL(nidx));
#endif
#if DSC_QDB && !DSC_QROT
      // the other Q buffer held item kk-1's Q, whose last S we have consumed: the next
      // item's Q rows are fetched now and rotated after this item's first tile
      if (has_next) issue_q_tile(ITEM_PARAMS(nidx), wn, qt, lt, qtile_of(kk + 1));
#endif
      const int rglob = w.m0 + qt * 128 + rloc;
      const bool valid_row = rglob < w.rows_total;
      const int qi = valid_row ? rglob / p.grp : 0;
      const int lim = valid_row ? p.q_pos0 + qi : -1;
      const bool warp_dead = __all_sync(0xffffffffu, !valid_row);
      if (DSC_QPREF) {   // warm L2 with this thread's Q row of the NEXT item (fetched at the item switch)
        const int nidx = kk + 1 < n_my_role ? item_at(kk + 1) : n_items;
        if (nidx < n_items) {
          const AttnParams& pn = ITEM_PARAMS(nidx);
          const Item wn = decode_item(pn, ITEM_LOCAL(nidx));
          const int rn = wn.m0 + qt * 128 + rloc;
          if (rn < wn.rows_total) {
            const char* row = reinterpret_cast<const char*>(pn.q) +
                              ((((long long)wn.pp * pn.n_q + rn / pn.grp) * pn.Hq + wn.g * pn.grp + rn % pn.grp) * 256);
            asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(row));
            asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(row + 128));
          }
        }
      }
      float m = -INFINITY;
      float2 lsum2 = make_float2(0.f, 0.f);
#if DSC_PAIR
      // pairs of 64-key tiles (a, b) per handshake: S_qt(pair) fills both 64-column halves of
      // the Q tile's S region, one max / rescale decision per 128 keys, P(a) -> cols 0..31,
      // P(b) -> cols 64..95.  S is single-buffered per Q tile: S(pair + 1) is issued after
      // PV(pair), so when S(pair) is in every earlier PV of this Q tile has completed and O
      // can be rescaled without a wait.
      for (int jp = 0; jp < n; jp += 2, ++gp) {
        const bool hasb = jp + 1 < n;
        auto vis = [&](int u, int& c_lo, int& c_hi) {
          const TileSeg t = tile_segments(p, w, u);
          if (!valid_row) {
            c_lo = 0; c_hi = 0;
          } else if (u < w.n_extra) {
            c_lo = 0;
            c_hi = min(max(min(A + w.n_self, max(A, lim - w.ring_count + 1)) - kKT * u, 0), kKT);
          } else {
            c_lo = t.lo0;
            c_hi = max(c_lo, min(t.hi0, lim - t.pos0_0 + 1));
          }
          return t.width;
        };
        int alo, ahi, blo = 0, bhi = 0;
        const int anu = vis(w.t_begin + jp, alo, ahi);
        const int bnu = hasb ? vis(w.t_begin + jp + 1, blo, bhi) : 0;
        mbar_wait(barS, gp & 1);
        if (rloc == 0) TRACE(EV_S0 + qt, gt + jp);
        if (warp_dead || DSC_ABL_SOFTMAX) {
          mbar_arrive(barP);
          continue;
        }
        tc_fence_after();
        uint32_t r[64];
        // (re)load one sub-tile's scores into r, invisible columns -> -inf; returns its max
        auto load_sub = [&](uint32_t taddr, int nu, int c_lo, int c_hi) {
          tmem_ld32(taddr, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
          if (nu > 32) tmem_ld32(taddr + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
          tmem_wait_ld();
          const bool partial = __any_sync(0xffffffffu, !(c_lo == 0 && c_hi == kKT));
          if (partial) {
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
          if (nu > 32) {
#pragma unroll
            for (int c = 32; c < 64; c += 8) {
              mx0 = fmax3f(mx0, __uint_as_float(r[c]), __uint_as_float(r[c + 1]));
              mx1 = fmax3f(mx1, __uint_as_float(r[c + 2]), __uint_as_float(r[c + 3]));
              mx2 = fmax3f(mx2, __uint_as_float(r[c + 4]), __uint_as_float(r[c + 5]));
              mx3 = fmax3f(mx3, __uint_as_float(r[c + 6]), __uint_as_float(r[c + 7]));
            }
          }
          return fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3));
        };
        float mt = load_sub(tS0, anu, alo, ahi);
        if (hasb) mt = fmaxf(mt, load_sub(tS0 + 64, bnu, blo, bhi));   // r now holds sub-tile b
        const float m_tile = mt * sl2;
        const bool upd = m_tile > m + kRescaleThreshold;
        const bool need_o = upd && (m != -INFINITY);
        const float f = need_o ? ex2(m - m_tile) : 1.f;
        if (upd) {
          lsum2.x *= f; lsum2.y *= f;
          m = m_tile;
        }
        if (__any_sync(0xffffffffu, need_o)) {   // every earlier PV of this Q tile is complete
#pragma unroll 1
          for (int ch = 0; ch < 4; ++ch) {
            uint32_t o[32];
            tmem_ld32(tO + ch * 32, o);
            tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * f);
            tmem_st32(tO + ch * 32, o);
          }
        }
        const float m_use = (m == -INFINITY) ? 0.f : m;
        const float2 negm2 = make_float2(-m_use, -m_use);
        float2 l0 = make_float2(0.f, 0.f), l1 = l0;
        auto exp_store = [&](uint32_t taddr, int nu) {   // r (one sub-tile) -> P at taddr
#pragma unroll
          for (int cb = 0; cb < 64; cb += 32) {
            if (cb == 32 && nu <= 32) break;
#pragma unroll
            for (int c = cb; c < cb + 32; c += 4) {
              const float2 x0 = __ffma2_rn(make_float2(__uint_as_float(r[c]), __uint_as_float(r[c + 1])), scale2, negm2);
              const float2 x1 = __ffma2_rn(make_float2(__uint_as_float(r[c + 2]), __uint_as_float(r[c + 3])), scale2, negm2);
              float2 p0, p1;
              if (DSC_ABL_EX2) { p0 = x0; p1 = x1; } else {
                p0 = make_float2(ex2(x0.x), ex2(x0.y));
                p1 = make_float2(ex2(x1.x), ex2(x1.y));
              }
              l0 = __fadd2_rn(l0, p0);
              l1 = __fadd2_rn(l1, p1);
              r[c >> 1] = pack_bf16(p0.x, p0.y);
              r[(c >> 1) + 1] = pack_bf16(p1.x, p1.y);
            }
          }
          if (nu > 32) tmem_st32(taddr, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
          else tmem_st16(taddr, *reinterpret_cast<uint32_t(*)[16]>(&r[0]));
        };
        if (hasb) {
          exp_store(tS0 + 64, bnu);
          tmem_wait_st();                         // r is reused for sub-tile a
          (void)load_sub(tS0, anu, alo, ahi);
        }
        exp_store(tS0, anu);
        lsum2 = __fadd2_rn(lsum2, __fadd2_rn(l0, l1));
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(barP);
        if (rloc == 0) TRACE(EV_P0 + qt, gt + jp);
      }
      gt += n;
#else
      for (int jj = 0; jj < n; ++jj) {
        const int g = gt + jj;
        const int u = w.t_begin + jj;
        const uint32_t tS = tS0 + (uint32_t)((g & 1) * 64);
        int c_lo, c_hi;
        const TileSeg t = tile_segments(p, w, u);
        const int nu = t.width;                    // S columns [0, nu) hold this tile's scores
        if (!valid_row) {
          c_lo = 0; c_hi = 0;
        } else if (u < w.n_extra) {                // sink always visible, self row j iff its id <= lim
          c_lo = 0;
          c_hi = min(max(min(A + w.n_self, max(A, lim - w.ring_count + 1)) - kKT * u, 0), kKT);
        } else {
          c_lo = t.lo0;
          c_hi = max(c_lo, min(t.hi0, lim - t.pos0_0 + 1));   // id pos0 + c <= lim
        }
        const bool full = (c_lo == 0) && (c_hi == kKT);
        mbar_wait(barS + 8u * (uint32_t)(g & 1), (g >> 1) & 1);
        if (rloc == 0) TRACE(EV_S0 + qt, g);
#if DSC_QROT
#elif DSC_QDB
        if (jj == 1 && has_next) {   // next item's Q: rotate in place and publish (every warp takes part)
          rotate_q_tile(ITEM_PARAMS(nidx), wn, qt, lt, qtile_of(kk + 1), 2 + qt);
          mbar_arrive(qbar_of(kk + 1));
        }
#elif DSC_QEARLY
        // S(last) is in: the MMA is done reading this Q tile, so the next item's Q rows are
        // fetched now and land while the last tile's softmax runs
        if (jj == n - 1 && has_next && !(DSC_ABL_SWITCH & 1)) issue_q_tile(ITEM_PARAMS(nidx), wn, qt, lt, qtile_of(kk + 1));
#endif
        if (warp_dead || DSC_ABL_SOFTMAX || (DSC_ABL_SMSP2 && (warp & 3) == 2)) {   // all 32 rows are padding: their P / O are never used
          mbar_arrive(barP + 8u * (uint32_t)(g & 1));
          continue;
        }
        tc_fence_after();
        // one TMEM read of the tile's (up to) 64 scores; invisible columns -> -inf
        const bool two = nu > 32;
        uint32_t r[64];
#if DSC_ABL_TMEM   // ablation: no TMEM traffic from the softmax (scores fabricated)
#pragma unroll
        for (int c = 0; c < 64; ++c) r[c] = __float_as_uint((float)((c * 7 + rloc) & 15) * 0.01f);
#else
        tmem_ld32(tS, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
        if (two) tmem_ld32(tS + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
        tmem_wait_ld();
#endif
        if (warp == 0 && lane == 0) TRACE(EV_L + 0, g);
        const bool any_partial = __any_sync(0xffffffffu, !full);
        if (any_partial) {
          const unsigned span = (unsigned)max(c_hi - c_lo, 0);
#pragma unroll
          for (int c = 0; c < 64; ++c) r[c] = ((unsigned)(c - c_lo) < span) ? r[c] : 0xFF800000u;
        }
        float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
#pragma unroll
        for (int c = 0; c < 32; c += 8) {     // 3-input max (FMNMX3): 2 columns per instruction
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
          // O_qt holds P V up to tile g-1: wait for that PV, rescale in TMEM
#if DSC_LASTO
          // V stage of tile g-1 freed = PV0(g-1) and PV1(g-1) complete (no per-tile O commit)
          mbar_wait(bar(B_VE + (g - 1) % VST), ((g - 1) / VST) & 1);
#else
          mbar_wait(bar(B_O + qt * 2 + ((g - 1) & 1)), ((g - 1) >> 1) & 1);
#endif
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
        // P = 2^(s*scale - m) (masked -> 2^-inf = 0) packed bf16x2 into words 0..31
        float2 l0 = make_float2(0.f, 0.f), l1 = l0;
        auto exp_chunk = [&](const int cb) {   // columns cb .. cb+31 -> P words cb/2 .. cb/2+15
#pragma unroll
          for (int c = cb; c < cb + 32; c += 4) {
            const float2 x0 = __ffma2_rn(make_float2(__uint_as_float(r[c]), __uint_as_float(r[c + 1])), scale2, negm2);
            const float2 x1 = __ffma2_rn(make_float2(__uint_as_float(r[c + 2]), __uint_as_float(r[c + 3])), scale2, negm2);
            float2 p0, p1;
            constexpr bool poly_any = kPolyPerGroup > 0;
            const bool poly0 = poly_any && ((c % 8) + 2 > 8 - kPolyPerGroup);
            const bool poly1 = poly_any && ((c % 8) + 4 > 8 - kPolyPerGroup);
            if (DSC_EXBF) {   // exponent rounded to bf16, one MUFU op per two columns; l sums the bf16 P
              const uint32_t e0 = ex2_bf16x2(pack_bf16(x0.x, x0.y)), e1 = ex2_bf16x2(pack_bf16(x1.x, x1.y));
              l0 = __fadd2_rn(l0, make_float2(bf_lo(e0), bf_hi(e0)));
              l1 = __fadd2_rn(l1, make_float2(bf_lo(e1), bf_hi(e1)));
              r[c >> 1] = e0;
              r[(c >> 1) + 1] = e1;
              continue;
            }
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
        if (two) {
          exp_chunk(32);
          if (!DSC_ABL_TMEM) tmem_st32(tS, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
        } else {
          if (!DSC_ABL_TMEM) tmem_st16(tS, *reinterpret_cast<uint32_t(*)[16]>(&r[0]));
        }
        lsum2 = __fadd2_rn(lsum2, __fadd2_rn(l0, l1));
        if (warp == 0 && lane == 0) TRACE(EV_L + 4, g);
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(barP + 8u * (uint32_t)(g & 1));
        if (rloc == 0) TRACE(EV_P0 + qt, g);
        if (lane == 0) TRACE(EV_PW0 + warp, g);
      }
      gt += n;
#endif
#if DSC_QROT
#elif DSC_QDB
      if (has_next && n < 2) {     // a one-tile item never reached the in-loop rotation point
        rotate_q_tile(ITEM_PARAMS(nidx), wn, qt, lt, qtile_of(kk + 1), 2 + qt);
        mbar_arrive(qbar_of(kk + 1));
      }
#elif DSC_QFIRST
      // S_qt of the last tile has been read: the MMA is done with Q tile qt, so the next
      // item's Q tile is fetched (unless already issued) and published before the epilogue
      if (has_next) {
        if (rloc == 0) TRACE(EV_QSTART, gt);
        if (!(DSC_ABL_SWITCH & 1)) {
          if (!DSC_QEARLY || n == 0) issue_q_tile(ITEM_PARAMS(nidx), wn, qt, lt, qtile_of(kk + 1));
          rotate_q_tile(ITEM_PARAMS(nidx), wn, qt, lt, qtile_of(kk + 1), 2 + qt);
        }
        if (rloc == 0) TRACE(EV_QLOADED, gt);
        mbar_arrive(qbar_of(kk + 1));
        if (rloc == 0) TRACE(EV_QDONE, gt);
      }
#endif
#if DSC_EPIROT
      if (w.staged && p.n_splits == 1 && p.split_only < 0 && p.n_peers == 0) {
        // the rotation warpgroup writes O out.  l goes into Q tile qt of this item's buffer
        // (its last QK^T has completed; the buffer is refilled by the rotation warpgroup
        // itself, after this epilogue).  Waiting for the previous item's O release keeps the
        // slot and B_EP at most one phase ahead of the reader.
        if (kk > 0) mbar_wait(bar(B_OF + qt), (kk - 1) & 1);
        reinterpret_cast<float*>(smem + OFF_Q + (uint32_t)(((kk & 1) * 2 + qt) * kQBytes))[rloc] = lsum2.x + lsum2.y;
        mbar_arrive(bar(B_EP + qt));
        continue;
      }
#endif
      // epilogue of the item: O / l once the last PV is done
      const float lsum = lsum2.x + lsum2.y;
#if DSC_PAIR || DSC_LASTO
      mbar_wait(bar(B_O + qt * 2), kk & 1);   // one O commit per item
#else
      mbar_wait(bar(B_O + qt * 2 + ((gt - 1) & 1)), ((gt - 1) >> 1) & 1);
#endif
      if (rloc == 0) TRACE(EV_EPI0, gt);
      tc_fence_after();
      const float inv = lsum > 0.f ? 1.f / lsum : 0.f;
      const int h = valid_row ? w.g * p.grp + rglob % p.grp : 0;
      const long long orow = ((long long)w.pp * p.n_q + qi) * p.Hq + h;
#pragma unroll 1
      for (int hf = 0; hf < 2; ++hf) {
        if (DSC_ABL_SWITCH & 2) {   // ablation: no O read-out / stores
          if (hf == 1) {
            tc_fence_before();
            mbar_arrive(bar(B_OF + qt));
            if (DSC_OFHALF) mbar_arrive(bar(B_OFH + qt));
          }
          continue;
        }
        uint32_t o[64];
        tmem_ld32(tO + 64 * hf, *reinterpret_cast<uint32_t(*)[32]>(&o[0]));
        tmem_ld32(tO + 64 * hf + 32, *reinterpret_cast<uint32_t(*)[32]>(&o[32]));
        tmem_wait_ld();
        if (DSC_OFHALF) {
          // each half of O_qt is released as soon as it is in registers: the next item's
          // first PV writes columns 0..63 (B_OF) and 64..127 (B_OFH) as two N = 64 halves
          tc_fence_before();
          mbar_arrive(bar((hf == 0 ? B_OF : B_OFH) + qt));
        } else if (hf == 1) {
          tc_fence_before();
          mbar_arrive(bar(B_OF + qt));      // O_qt may be overwritten by the next item
        }
        if (!valid_row) continue;
        if (p.n_splits == 1 && p.split_only < 0 && p.n_peers > 0) {
          // fused all-gather: the same row to every peer's gathered O (NVLink stores)
          const long long prow = ((long long)w.pp * p.n_q + qi) * p.o_hq + p.o_head_off + h;
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            uint32_t q[8];
#pragma unroll
            for (int j = 0; j < 8; ++j)
              q[j] = pack_bf16(__uint_as_float(o[16 * v + 2 * j]) * inv, __uint_as_float(o[16 * v + 2 * j + 1]) * inv);
#pragma unroll 1
            for (int r = 0; r < p.n_peers; ++r)
              stg256(reinterpret_cast<__nv_bfloat16*>(p.peer_o[r]) + prow * 128 + 64 * hf + 16 * v, q);
          }
        } else if (p.n_splits == 1 && p.split_only < 0) {
          // 32-byte stores (STG.256): each one fills a whole L2 sector of this thread's row
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
      if (rloc == 0) TRACE(EV_EPI1, gt);
#if !DSC_QDB && !DSC_QFIRST
      if (has_next) {
        issue_q_tile(ITEM_PARAMS(nidx), wn, qt, lt, qtile_of(kk + 1));
        rotate_q_tile(ITEM_PARAMS(nidx), wn, qt, lt, qtile_of(kk + 1), 2 + qt);
        mbar_arrive(qbar_of(kk + 1));
        if (rloc == 0) TRACE(EV_QDONE, gt);
      }
#endif
    }
  } else if (warp < 12) {
    // ================================================================ rotation (K tiles)
    if constexpr (kRegRotate > kThreadRegs) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegRotate));
    else if constexpr (kRegRotate < kThreadRegs) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegRotate));
    const int lt = threadIdx.x - 256;
    const int c8 = lt & 7;             // frequencies 8*c8 .. 8*c8+7
    const int rg = lt >> 3;            // rows rg*4 .. rg*4+3 of a 64-row tile
    const float4* __restrict__ rp = p.rope_pairs;
    float2 cth[4], sth[4];             // R(theta_f) = table entry of id 1
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float4 t = rp[32 + 4 * c8 + j];
      cth[j] = make_float2(t.x, t.y);
      sth[j] = make_float2(t.z, t.w);
    }
#if DSC_QROT
    // Q tiles (both) of item k into Q buffer k & 1; the buffer's previous item (k - 2) must be
    // done with it (its last QK^T MMA committed to B_QE)
    auto prep_q = [&](int k, int qidx) {
      const uint32_t qb = DSC_QDB ? (uint32_t)(k & 1) : 0u;
      if (DSC_QDB && k >= 2) mbar_wait(bar(B_QE + qb), ((k - 2) >> 1) & 1);
      if (!DSC_QDB && k >= 1) mbar_wait(bar(B_QE), (k - 1) & 1);   // item k-1's last QK^T done
      const AttnParams& pq = ITEM_PARAMS(qidx);
      const Item wq = decode_item(pq, ITEM_LOCAL(qidx));
      if (DSC_Q2ISSUE && !DSC_QLDG) {   // both tiles' loads in flight before the first wait
        issue_q_tile(pq, wq, 0, lt, sbase + OFF_Q + (qb * 2) * kQBytes);
        issue_q_tile(pq, wq, 1, lt, sbase + OFF_Q + (qb * 2 + 1) * kQBytes);
      }
#pragma unroll 1
      for (int q = 0; q < 2; ++q) {
        const uint32_t qtile = sbase + OFF_Q + (qb * 2 + q) * kQBytes;
        if (DSC_QLDG) {
          load_rotate_q_tile(pq, wq, q, lt, qtile);
        } else {
          if (!DSC_Q2ISSUE) issue_q_tile(pq, wq, q, lt, qtile);
          rotate_q_tile(pq, wq, q, lt, qtile, 6);
        }
        mbar_arrive(bar(B_Q + qb * 2 + q));
      }
    };
    if (!DSC_Q0SM && n_my_role > 0) prep_q(0, item_at(0));   // (else the softmax WGs do it)
#endif
    int gt = 0, kk = 0, ne = 0;   // ne: staged items whose epilogue this warpgroup ran (B_EP phase)
    for (; kk < n_my_role; ++kk) {
      const int idx = item_at(kk);
      const AttnParams& p = ITEM_PARAMS(idx);
      const Item w = decode_item(p, ITEM_LOCAL(idx));
      const int A = p.A;
      const bool dbg = p.dbg_pos != nullptr && w.pp == 0 && w.g == 0;
#if DSC_QROT
      const bool q_next = kk + 1 < n_my_role;
      const int nidx_q = q_next ? item_at(kk + 1) : n_items;
      if (w.staged) {   // no K to rotate: the MMA waits on the copy barrier; prepare the next Q
        if (q_next) prep_q(kk + 1, nidx_q);
        gt += w.n_tiles;
#if DSC_EPIROT
        if (p.n_splits == 1 && p.split_only < 0 && p.n_peers == 0) {   // O epilogue of both Q tiles (DSC_EPIROT)
          const uint32_t tq = tmem + ((uint32_t)((lt >> 5) * 32) << 16);
#pragma unroll 1
          for (int qt = 0; qt < 2; ++qt) {
            mbar_wait(bar(B_EP + qt), ne & 1);
            const float lsum = reinterpret_cast<const float*>(smem + OFF_Q + (uint32_t)(((kk & 1) * 2 + qt) * kQBytes))[lt];
            mbar_wait(bar(B_O + qt * 2 + ((gt - 1) & 1)), ((gt - 1) >> 1) & 1);
            tc_fence_after();
            const float inv = lsum > 0.f ? 1.f / lsum : 0.f;
            const int rglob = w.m0 + qt * 128 + lt;
            const bool valid_row = rglob < w.rows_total;
            const int qi = valid_row ? rglob / p.grp : 0;
            const int h = valid_row ? w.g * p.grp + rglob % p.grp : 0;
            __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(p.o) + (((long long)w.pp * p.n_q + qi) * p.Hq + h) * 128;
#pragma unroll 1
            for (int hf = 0; hf < 2; ++hf) {
              uint32_t o[64];
              tmem_ld32(tq + 256 + qt * 128 + 64 * hf, *reinterpret_cast<uint32_t(*)[32]>(&o[0]));
              tmem_ld32(tq + 256 + qt * 128 + 64 * hf + 32, *reinterpret_cast<uint32_t(*)[32]>(&o[32]));
              tmem_wait_ld();
              if (hf == 1) {
                tc_fence_before();
                mbar_arrive(bar(B_OF + qt));
              }
              if (!valid_row) continue;
#pragma unroll
              for (int v = 0; v < 4; ++v) {
                uint32_t q[8];
#pragma unroll
                for (int j = 0; j < 8; ++j)
                  q[j] = pack_bf16(__uint_as_float(o[16 * v + 2 * j]) * inv, __uint_as_float(o[16 * v + 2 * j + 1]) * inv);
                stg256(dst + 64 * hf + 16 * v, q);
              }
            }
          }
          ++ne;
        }
#endif
        continue;
      }
#endif
      // ---- K tiles of this item; the table entry of each tile's first row is fetched
      // one tile ahead so the L2 latency is off the rotation's critical path
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
        if (jj + 1 < w.n_tiles) {          // prefetch for the next tile
          pre_pos = first_pos(u + 1);
#pragma unroll
          for (int j = 0; j < 4; ++j) kpre[j] = rp[(long long)max(pre_pos, 0) * 32 + 4 * c8 + j];
        }
        mbar_wait(bar(B_KR + ks), (g / KST) & 1);
        if (lt == 0) TRACE(EV_KR, g);
        if (!DSC_ABL_ROT && !w.staged && rg * 4 < t.width)   // rows >= width are never read by the MMA;
                                                             // staged K arrives rotated
          rotate_rows<1, kKVHalf>(sbase + OFF_K + ks * kKVBytes, rg * 4, c8, rp, cth, sth, kpos, cur,
                                  max(cur_pos, 0));
        fence_proxy_async();
        mbar_arrive(bar(B_KF + ks));
        if (lt == 0) TRACE(EV_KDONE, g);
#if DSC_QROT
        if (!DSC_QSINGLE && jj == min(1, w.n_tiles - 1) && q_next) prep_q(kk + 1, nidx_q);   // after the item's first K tiles
#endif
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
#if DSC_QROT
      if ((DSC_QSINGLE || w.n_tiles == 0) && q_next) prep_q(kk + 1, nidx_q);   // single set: after every K tile
#endif
      gt += w.n_tiles;
    }
  } else {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegCopy));
    if (warp == 12 && lane == 0) TRACE(EV_START, 2);   // after the register hand-off
    if (warp == 12 || warp == 13) {
      // ============================================================== copy warps (12: K, 13: V)
      const bool isk = warp == 12;

      const int nst = isk ? KST : VST;
      const int off = isk ? OFF_K : OFF_V;
      const int b_full = isk ? B_KR : B_VF, b_free = isk ? B_KE : B_VE;
      int gt = 0;
      for (int t = 0; t < n_my_role; ++t) {
        const int idx = item_at(t);
        const AttnParams& p = ITEM_PARAMS(idx);
        const Item w = decode_item(p, ITEM_LOCAL(idx));
        if (isk && lane == 0 && t == 0) TRACE(EV_START, 3);   // first item decoded
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
            // sink rows (x < A) + self rows (A <= x < A + n_self), zeros up to the tile
            // width, with cp.async
            const int nit = t.width >> 1;
#pragma unroll 1
            for (int it = 0; it < nit; ++it) {
              const int id = it * 32 + lane;          // 16-byte chunks
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
            // logical window tile: one box (the ring's mirror rows, or the staging rows)
            const AttnParams& pi = ITEM_PARAMS(idx);
            const CUtensorMap* tmap = isk ? &pi.tmap_k : &pi.tmap_v;
            const int row = (int)(w.head_row * w.Rp) + t.slot0;
            if (DSC_ABL_LOADS) {   // ablation: no K/V bytes move (tiles keep stale data)
              mbar_arrive(bar(b_full + st));
            } else {
              mbar_arrive_tx(bar(b_full + st), kKVBytes);
              tma_load_2d(dst, tmap, 0, row, bar(b_full + st));
              tma_load_2d(dst + kKVHalf, tmap, 64, row, bar(b_full + st));
            }
          }
          if (lane == 0) TRACE(isk ? EV_K_ISSUE : EV_V_ISSUE, g);
          __syncwarp();
        }
        gt += w.n_tiles;
      }
    } else {
      // ============================================================== MMA issuers: warp 14 for Q tile 0,
      // warp 15 for Q tile 1 (whole warp runs the loop, an elected lane issues); two issuers
      // halve the per-warp tcgen05 issue work, which otherwise bounds the tile rate
      // DSC_MMA2 = 0: warp 14 issues for both Q tiles (warp 15 idles)
      const int q_lo = DSC_MMA2 ? warp - 14 : 0, q_hi = DSC_MMA2 ? warp - 13 : 2;
      if (!DSC_MMA2 && warp == 15) goto mma_done;
      {
      int qbuf = 0;                                          // Q tile set of the current item
      constexpr uint32_t IQK0 = idesc_bf16(128, 0, 0, 0);    // S = Q K^T, both K-major; N = tile width
      constexpr uint32_t IPV = idesc_bf16(128, 128, 0, 1);   // O += P V, P from TMEM, V MN-major
      // fully unrolled: the descriptors are formed once per call and advanced by
      // immediates (16-element K steps: +32 B inside a 128 B swizzle row, then the next
      // 64-column block), so each tcgen05.mma costs a few uniform-datapath instructions
      auto issue_qk = [&](int qt, int ks, int nu, int buf) {
        const uint64_t da = sdesc(sbase + OFF_Q + (qbuf * 2 + qt) * kQBytes, 16, 1024);
        const uint64_t db = sdesc(sbase + OFF_K + ks * kKVBytes, 16, 1024);
        const uint32_t iqk = IQK0 | ((uint32_t)(nu >> 3) << 17);
        const uint32_t d = tmem + qt * 128 + buf * 64;
        static_assert(kQBytes / 2 / 16 == 1024 && kKVHalf / 16 == 512, "mma_qk8_w block offsets");
        mma_qk8_w(d, da, db, iqk);
      };
      // K of the PV product = tile width (keys), 16 per MMA; V rows advance 16 x 128 B
      auto issue_pv = [&](int qt, int vs, bool acc, int nu, int buf) {
        const uint64_t dv = sdesc(sbase + OFF_V + vs * kKVBytes, kKVHalf, 1024);
        const uint32_t d = tmem + 256 + qt * 128, a = tmem + qt * 128 + buf * 64;
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
      // first PV of an item as two N = 64 column halves (DSC_OFHALF): V block `half` (columns
      // 64*half .. +63 of the tile) into O_qt columns 64*half .. +63, no accumulate
      auto issue_pv_half = [&](int qt, int vs, int nu, int buf, int half) {
        constexpr uint32_t IPVH = idesc_bf16(128, 64, 0, 1);
        const uint64_t dv = sdesc(sbase + OFF_V + vs * kKVBytes + half * kKVHalf, kKVHalf, 1024);
        const uint32_t d = tmem + 256 + qt * 128 + half * 64, a = tmem + qt * 128 + buf * 64;
        const int nk = nu >> 4;
        mma_ts_w(d, a, dv, IPVH, 0u);
#pragma unroll
        for (int k8 = 1; k8 < kKT / 16; ++k8)
          if (k8 < nk) mma_ts_w(d, a + k8 * 8, dv + (uint64_t)(k8 * 128), IPVH, 1u);
      };
      // S of tile g for Q tile qt into buffer g & 1; K stage g % KST is free when both MMA
      // warps' QK^T of the tile are done (K-free barrier counts 2 commits)
      auto issue_s = [&](const ItemGeo& p, const Item& w, int g, int u) {
        const int ks = g % KST, buf = g & 1;
        const int nu = tile_segments(p, w, u).width;
        MWAIT(bar((DSC_QROT && w.staged ? B_KR : B_KF) + ks), (g / KST) & 1);
        if (lane == 0 && q_lo == 0) TRACE(EV_KF, g);
        tc_fence_after();
#pragma unroll 1
        for (int qt = q_lo; qt < q_hi; ++qt) {
          issue_qk(qt, ks, nu, buf);
          mma_commit_w(bar(B_S + qt * 2 + buf));
        }
        mma_commit_w(bar(B_KE + ks));
        if (lane == 0 && q_lo == 0) TRACE(EV_QKI, g);
      };
      int gt = 0, kk = 0, gp = 0;
      for (; kk < n_my; ++kk) {
        const int idx = item_at(kk);
        const ItemGeo p = item_geo(pa, pb, ITEM_B(idx));
        const Item w = decode_item(p, ITEM_LOCAL(idx));
        const int n = w.n_tiles;
        qbuf = DSC_QDB ? (kk & 1) : 0;
        for (int qt = q_lo; qt < q_hi; ++qt) MWAIT(bar(B_Q + qbuf * 2 + qt), DSC_QDB ? ((kk >> 1) & 1) : (kk & 1));
        if (kk == 0 && lane == 0 && q_lo == 0) TRACE(EV_Q, 0);
#if DSC_PAIR
        {
          // S(pair) for both Q tiles: tile a -> S cols 0..63, tile b -> cols 64..127
          auto kbar = [&](int g) { return bar((DSC_QROT && w.staged ? B_KR : B_KF) + g % KST); };
          auto wait_k = [&](int g, bool hb) {
            MWAIT(kbar(g), (g / KST) & 1);
            if (hb) MWAIT(kbar(g + 1), ((g + 1) / KST) & 1);
            tc_fence_after();
          };
          auto width = [&](int g) { return tile_segments(p, w, w.t_begin + (g - gt)).width; };
          if (n == 0) {
            for (int qt = q_lo; qt < q_hi; ++qt) mma_commit_w(bar(B_O + qt * 2));   // keep the per-item O phase
          } else {
            const bool hb = n > 1;
            wait_k(gt, hb);
            const int na_ = width(gt), nb_ = hb ? width(gt + 1) : 0;
#pragma unroll 1
            for (int qt = q_lo; qt < q_hi; ++qt) {
              issue_qk(qt, gt % KST, na_, 0);
              if (hb) issue_qk(qt, (gt + 1) % KST, nb_, 1);
              mma_commit_w(bar(B_S + qt * 2));
            }
            mma_commit_w(bar(B_KE + gt % KST));
            if (hb) mma_commit_w(bar(B_KE + (gt + 1) % KST));
          }
          for (int jp = 0; jp < n; jp += 2, ++gp) {
            const int a = gt + jp;
            const bool hb = jp + 1 < n, more = jp + 2 < n, hb2 = jp + 3 < n;
            const int na_ = width(a), nb_ = hb ? width(a + 1) : 0;
            const int na2 = more ? width(a + 2) : 0, nb2 = hb2 ? width(a + 3) : 0;
            MWAIT(bar(B_VF + a % VST), (a / VST) & 1);
            if (hb) MWAIT(bar(B_VF + (a + 1) % VST), ((a + 1) / VST) & 1);
#pragma unroll 1
            for (int qt = q_lo; qt < q_hi; ++qt) {
              MWAIT(bar(B_P + qt * 2), gp & 1);
              if (jp == 0 && kk > 0) MWAIT(bar(B_OF + qt), (kk - 1) & 1);   // previous item's O read
              tc_fence_after();
              issue_pv(qt, a % VST, jp > 0, na_, 0);
              if (hb) issue_pv(qt, (a + 1) % VST, true, nb_, 1);
              if (!more) mma_commit_w(bar(B_O + qt * 2));
              if (more) {
                if (qt == q_lo) wait_k(a + 2, hb2);
                issue_qk(qt, (a + 2) % KST, na2, 0);
                if (hb2) issue_qk(qt, (a + 3) % KST, nb2, 1);
                mma_commit_w(bar(B_S + qt * 2));
              }
            }
            mma_commit_w(bar(B_VE + a % VST));
            if (hb) mma_commit_w(bar(B_VE + (a + 1) % VST));
            if (more) {
              mma_commit_w(bar(B_KE + (a + 2) % KST));
              if (hb2) mma_commit_w(bar(B_KE + (a + 3) % KST));
            }
          }
        }
#else
        if (n > 0) issue_s(p, w, gt, w.t_begin);
        if (n > 1) issue_s(p, w, gt + 1, w.t_begin + 1);
        if (DSC_QSINGLE && n <= 2) mma_commit_w(bar(B_QE));   // the item's last QK^T is issued
        if (DSC_LASTO && n == 0)
          for (int qt = q_lo; qt < q_hi; ++qt) mma_commit_w(bar(B_O + qt * 2));   // keep the per-item O phase
        for (int jj = 0; jj < n; ++jj) {
          const int g = gt + jj, vs = g % VST, buf = g & 1;
          const int nu = tile_segments(p, w, w.t_begin + jj).width;
          if (!DSC_ABL_NOWAIT_V) MWAIT(bar(B_VF + vs), (g / VST) & 1);
          if (lane == 0 && q_lo == 0) TRACE(EV_VF, g);
#if DSC_SORDER == 2
          // one burst per tile: every wait first (V(g), P0(g), P1(g), K(g+2) rotated), then
          // PV0 PV1 S0(g+2) S1(g+2) back to back and the commits.  The tensor pipe queues
          // only a couple of MMAs, so every wait/commit between MMA groups left it idle.
          const bool more = jj + 2 < n;
          const int ks2 = (g + 2) % KST;
          const int nu2 = more ? tile_segments(p, w, w.t_begin + jj + 2).width : 0;
          for (int qt = q_lo; qt < q_hi; ++qt) {
            MWAIT(bar(B_P + qt * 2 + buf), (g >> 1) & 1);
            if (jj == 0 && kk > 0) MWAIT(bar(B_OF + qt), (kk - 1) & 1);   // previous item's O read
          }
          if (more) MWAIT(bar((DSC_QROT && w.staged ? B_KR : B_KF) + ks2), ((g + 2) / KST) & 1);
          tc_fence_after();
#pragma unroll 1
          for (int qt = q_lo; qt < q_hi; ++qt) issue_pv(qt, vs, jj > 0, nu, buf);
          if (more) {
#pragma unroll 1
            for (int qt = q_lo; qt < q_hi; ++qt) issue_qk(qt, ks2, nu2, buf);
          }
#pragma unroll 1
          for (int qt = q_lo; qt < q_hi; ++qt) mma_commit_w(bar(B_O + qt * 2 + buf));
          mma_commit_w(bar(B_VE + vs));
          if (more) {
#pragma unroll 1
            for (int qt = q_lo; qt < q_hi; ++qt) mma_commit_w(bar(B_S + qt * 2 + buf));
            mma_commit_w(bar(B_KE + ks2));
          }
#elif DSC_SORDER
          // per Q tile: PV(g) then S(g+2) into the buffer PV(g) just consumed, so Q tile 0's
          // next scores do not wait for Q tile 1's P(g)
          const bool more = jj + 2 < n;
          const int ks2 = (g + 2) % KST;
          const int nu2 = more ? tile_segments(p, w, w.t_begin + jj + 2).width : 0;
#pragma unroll 1
          for (int qt = q_lo; qt < q_hi; ++qt) {
            MWAIT(bar(B_P + qt * 2 + buf), (g >> 1) & 1);
            if (jj == 0 && kk > 0) MWAIT(bar(B_OF + qt), (kk - 1) & 1);   // previous item's O read
            if (lane == 0) TRACE(EV_PV0 + qt, g);
            tc_fence_after();
            issue_pv(qt, vs, jj > 0, nu, buf);
            if (!DSC_LASTO) mma_commit_w(bar(B_O + qt * 2 + buf));
            else if (jj == n - 1) mma_commit_w(bar(B_O + qt * 2));   // one O commit per item (epilogue)
            if (lane == 0) TRACE(EV_PVI + qt, g);
            if (more) {
              if (qt == q_lo) {
                if (lane == 0) TRACE(EV_L + 5, g + 2);   // (trace) K wait entered
                MWAIT(bar((DSC_QROT && w.staged ? B_KR : B_KF) + ks2), ((g + 2) / KST) & 1);
                if (lane == 0) TRACE(EV_KF, g + 2);      // K(g+2) ready at the MMA
                tc_fence_after();
              }
              issue_qk(qt, ks2, nu2, buf);
              mma_commit_w(bar(B_S + qt * 2 + buf));
            }
          }
          if (DSC_QSINGLE && more && jj + 3 == n) mma_commit_w(bar(B_QE));   // S(n-1) issued: Q set free when done
          mma_commit_w(bar(B_VE + vs));
          if (more) mma_commit_w(bar(B_KE + ks2));
#else
          if (DSC_PJOIN) MWAIT(bar(B_P + buf), (g >> 1) & 1);   // P(g) of both Q tiles: one wait
#pragma unroll 1
          for (int qt = q_lo; qt < q_hi; ++qt) {
            if (!DSC_PJOIN) MWAIT(bar(B_P + qt * 2 + buf), (g >> 1) & 1);
            if (DSC_OFHALF && jj == 0 && kk > 0) {
              // first PV of the item in two column halves, each after its half of the
              // previous item's O has been read out
              MWAIT(bar(B_OF + qt), (kk - 1) & 1);
              tc_fence_after();
              issue_pv_half(qt, vs, nu, buf, 0);
              MWAIT(bar(B_OFH + qt), (kk - 1) & 1);
              tc_fence_after();
              issue_pv_half(qt, vs, nu, buf, 1);
            } else {
            if (jj == 0 && kk > 0) MWAIT(bar(B_OF + qt), (kk - 1) & 1);   // previous item's O read
            if (lane == 0) TRACE(EV_PV0 + qt, g);
            tc_fence_after();
            issue_pv(qt, vs, jj > 0, nu, buf);
            }
            if (!DSC_LASTO) mma_commit_w(bar(B_O + qt * 2 + buf));
            else if (jj == n - 1) mma_commit_w(bar(B_O + qt * 2));   // one O commit per item (epilogue)
            if (lane == 0) TRACE(EV_PVI + qt, g);
          }
          mma_commit_w(bar(B_VE + vs));
          // S(g+2) reuses buffer g & 1: issued after PV(g) has consumed P(g)
          if (jj + 2 < n) issue_s(p, w, g + 2, w.t_begin + jj + 2);
#endif
        }
#endif   // DSC_PAIR
        if (DSC_QROT && !DSC_QSINGLE) mma_commit_w(bar(B_QE + qbuf));   // Q buffer of this item free once its MMAs are done
        gt += n;
      }
      // drain: the last V-free commit tracks every MMA of this CTA
      if (gt > 0) mbar_wait(bar(B_VE + (gt - 1) % VST), ((gt - 1) / VST) & 1);   // drain (kept in every variant)
      if (lane == 0) TRACE(EV_END, 0);
      }
    mma_done:;
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 14) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_alloc) : "memory");
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
  const cuuint32_t box[2] = {64, (cuuint32_t)kTileN};   // 64 columns x one key tile
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t make_stage_tmap(CUtensorMap* map, void* base, unsigned long long rows) {
  return make_ring_tmap(map, base, rows);   // same geometry: [rows][128] bf16, box 64 x kTileN, SW128
}

static long long tc_items(const AttnParams& p) {
  return (long long)p.P * p.Hkv * p.n_mblocks * (p.split_only >= 0 ? 1 : p.n_splits);
}

cudaError_t launch_attn_tc6(const AttnParams& pa, const AttnParams* pb, cudaStream_t st);
// DSC_V6 1: kernel v6 (attn_tc6.cu: Q in TMEM, TS QK^T, 7 + 7 K/V stages)
#ifndef DSC_V6
#define DSC_V6 0
#endif

// DSC_SCHED 1: per-CTA work lists by list scheduling -- items in launch order (attend first,
// then build; longest first inside each), each to the CTA with the least work so far
// (cost = its key tiles + kSwitchCost for the item switch).  The static stride gives CTA b
// items b, b + grid, ...: with item lengths that differ a lot (c3: 224 attend items of 223
// tiles on 148 CTAs, then 4.8K build items of 1-25 tiles) half the CTAs ran two attend
// items AND a full share of builds.  Lists are cached per launch shape.
#ifndef DSC_SCHED
#define DSC_SCHED 1
#endif
#ifndef DSC_SCHED_STRIDE
#define DSC_SCHED_STRIDE 0
#endif
namespace {
#ifndef DSC_SWCOST
#define DSC_SWCOST 2
#endif
constexpr int kSwitchCost = DSC_SWCOST;   // item-switch cost in key tiles (epilogue + pipeline refill)
struct SchedEntry {
  std::vector<long long> key;
  int* dev = nullptr;
  size_t cap = 0;     // ints allocated
  int device = -1;
  bool use = false;   // false: the static stride is within 2% of the list schedule's makespan
};
long long item_tiles_host(const AttnParams& p, int local) { return tcc::decode_item(p, local).n_tiles; }

// returns device [grid + 1 offsets | n items] for this launch shape (cached), or nullptr
const int* sched_lists(const AttnParams& pa, const AttnParams* pb, long long na, long long nb, int ka, int kb,
                       unsigned grid, cudaStream_t st) {
  static SchedEntry cache[4];
  static int next = 0;
  static std::mutex mu;                 // handles may launch from several host threads
  std::lock_guard<std::mutex> lock(mu);
  int device = 0;
  cudaGetDevice(&device);
  std::vector<long long> key = {device, na, nb, ka, kb, grid};
  for (const AttnParams* p : {&pa, pb}) {
    if (!p) continue;
    for (long long v : {(long long)p->n_splits, (long long)p->split_only, (long long)p->P, (long long)p->Hkv,
                        (long long)p->n_mblocks, (long long)p->n_q, (long long)p->grp, (long long)p->q_pos0,
                        (long long)p->A, (long long)p->ring_count, (long long)p->n_self,
                        (long long)p->tiles_per_split})
      key.push_back(v);
  }
  for (auto& e : cache)
    if (!e.key.empty() && e.key == key) return e.use ? e.dev : nullptr;
  const long long items = na + nb;
  std::vector<int> off(grid + 1, 0), owner(items);
  std::vector<long long> stride_load(grid, 0);
  // min-heap on (load, cta): each item in launch order goes to the least-loaded CTA
  std::vector<std::pair<long long, int>> heap;
  heap.reserve(grid);
  for (unsigned b = 0; b < grid; ++b) heap.push_back({0, (int)b});
  auto cmp = [](const std::pair<long long, int>& x, const std::pair<long long, int>& y) { return x > y; };
  std::make_heap(heap.begin(), heap.end(), cmp);
  for (long long I = 0; I < items; ++I) {
    const bool isb = kb > 0 ? (I % (ka + kb)) >= ka : I >= na;
    const long long local = kb > 0 ? (isb ? (I / (ka + kb)) * kb + (I % (ka + kb)) - ka : (I / (ka + kb)) * ka + (I % (ka + kb)))
                                   : (isb ? I - na : I);
    const long long cost = item_tiles_host(isb ? *pb : pa, (int)local) + kSwitchCost;
    stride_load[I % grid] += cost;
#if DSC_SCHED_STRIDE   // debug: the lists reproduce the static stride
    (void)cost;
    owner[I] = (int)(I % grid);
    ++off[owner[I] + 1];
#else
    std::pop_heap(heap.begin(), heap.end(), cmp);
    const int b = heap.back().second;
    owner[I] = b;
    heap.back().first += cost;
    std::push_heap(heap.begin(), heap.end(), cmp);   // (moves heap.back(): b saved above)
    ++off[b + 1];
#endif
  }
  for (unsigned b = 0; b < grid; ++b) off[b + 1] += off[b];
  long long list_max = 0;
  for (auto& h : heap) list_max = std::max(list_max, h.first);
  const long long stride_max = *std::max_element(stride_load.begin(), stride_load.end());
  // keep the stride (and its L2 locality: c5) unless the lists shorten the makespan by > 2%
  const bool use = list_max * 50 < stride_max * 49;
  std::vector<int> host(grid + 1 + items);
  std::copy(off.begin(), off.end(), host.begin());
  std::vector<int> fill(off.begin(), off.end() - 1);
  for (long long I = 0; I < items; ++I) host[grid + 1 + fill[owner[I]]++] = (int)I;   // increasing I per CTA
  SchedEntry& e = cache[next];
  next = (next + 1) % 4;
  e.key = key;
  e.use = use;
  if (!use) return nullptr;
  if (e.cap < host.size() || e.device != device) {
    if (e.dev) cudaFree(e.dev);
    e.dev = nullptr; e.cap = 0;
    if (cudaMalloc(&e.dev, host.size() * sizeof(int)) != cudaSuccess) { cudaGetLastError(); e.key.clear(); return nullptr; }
    e.cap = host.size();
    e.device = device;
  }
  // pageable source: staged synchronously, so `host` may go out of scope afterwards
  if (cudaMemcpyAsync(e.dev, host.data(), host.size() * sizeof(int), cudaMemcpyHostToDevice, st) != cudaSuccess) {
    e.key.clear();
    return nullptr;
  }
  return e.dev;
}
}  // namespace

cudaError_t launch_attn_tc2(const AttnParams& pa, const AttnParams* pb, cudaStream_t st) {
  if (DSC_V6) {
    if (pa.n_peers > 0 || (pb && pb->n_peers > 0)) return cudaErrorNotSupported;   // v6 has no peer epilogue
    return launch_attn_tc6(pa, pb, st);
  }
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
  AttnParams qa = pa;
  qa.sched_off = qa.sched_items = nullptr;
  if (DSC_SCHED && grid > 0 && items > grid) {
    const int* lists = sched_lists(pa, pb, na, nb, ka, kb, grid, st);
    if (lists) { qa.sched_off = lists; qa.sched_items = lists + grid + 1; }
  }
  tc::attn_tc_kernel<<<grid, tc::kThreads, tc::kSmemBytes, st>>>(qa, pb ? *pb : qa, (int)na, (int)nb, ka, kb);
  return cudaGetLastError();
}

cudaError_t launch_attn_tc(const AttnParams& p, cudaStream_t st) { return launch_attn_tc2(p, nullptr, st); }

}  // namespace dsc
