// Device helpers shared by the tcgen05 attention kernels (attn_tc.cu: one CTA per
// 256-row m-block; attn_pair.cu: a CTA pair with cta_group::2 MMAs): PTX wrappers
// (mbarrier, TMA, tcgen05, cp.async), the work-item decode, the key-tile segment
// map, and the in-place rotate-on-load RoPE of SW128 bf16 tiles.
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
// Watchdog: a pipeline bug must not hang the GPU -- trap after ~2^31 cycles (~1 s).
// DSC_WSLEEP > 0: failed polls back off with nanosleep(DSC_WSLEEP), leaving the
// sub-partition's issue slots to the warps that have work
#ifndef DSC_WSLEEP
#define DSC_WSLEEP 0
#endif
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  if (mbar_try(bar, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try(bar, parity)) {
    if (DSC_WSLEEP > 0) __nanosleep(DSC_WSLEEP);
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
// Warp-converged variants: the whole (MMA) warp executes the call with warp-uniform
// operands and one elected lane issues, so the descriptors stay in uniform registers.
__device__ __forceinline__ void mma_ss_w(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_ts_w(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// Batched warp-converged issue: ONE elect for a whole K sweep (the per-MMA elect of
// mma_ss_w costs a WARPSYNC/ELECT sequence and operand moves per instruction, which
// capped the issue rate of the single MMA warp below the tensor pipe's).
// S = Q K^T over K = 128 (8 x K16): A (Q, 128 rows) and B (K tile, 64 rows) SW128
// K-major; the second 64-column block of A is +16 KB (1024 in 16-B units), of B +8 KB (512).
__device__ __forceinline__ void mma_qk8_w(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc) {
  asm volatile(
      "{\n.reg .pred e;\n.reg .b64 a1, a2, a3, a4, a5, a6, a7, b1, b2, b3, b4, b5, b6, b7;\n"
      "add.s64 a1, %1, 2; add.s64 a2, %1, 4; add.s64 a3, %1, 6;\n"
      "add.s64 a4, %1, 1024; add.s64 a5, %1, 1026; add.s64 a6, %1, 1028; add.s64 a7, %1, 1030;\n"
      "add.s64 b1, %2, 2; add.s64 b2, %2, 4; add.s64 b3, %2, 6;\n"
      "add.s64 b4, %2, 512; add.s64 b5, %2, 514; add.s64 b6, %2, 516; add.s64 b7, %2, 518;\n"
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
// S = Q K^T over K = 128 with Q in TMEM (TS form): A step k8 = TMEM columns a + 8k8 (16 bf16
// of the head dim per lane), B = the K tile (64 rows, K-major SW128; second 64-column block
// +8 KB = 512 in 16-B units).  Only B is read from shared memory.
__device__ __forceinline__ void mma_qk8_ts_w(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc) {
  asm volatile(
      "{\n.reg .pred e;\n.reg .b64 b1, b2, b3, b4, b5, b6, b7;\n.reg .b32 t1, t2, t3, t4, t5, t6, t7;\n"
      "add.s64 b1, %2, 2; add.s64 b2, %2, 4; add.s64 b3, %2, 6;\n"
      "add.s64 b4, %2, 512; add.s64 b5, %2, 514; add.s64 b6, %2, 516; add.s64 b7, %2, 518;\n"
      "add.u32 t1, %1, 8; add.u32 t2, %1, 16; add.u32 t3, %1, 24; add.u32 t4, %1, 32;\n"
      "add.u32 t5, %1, 40; add.u32 t6, %1, 48; add.u32 t7, %1, 56;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t1], b1, %3, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t2], b2, %3, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t3], b3, %3, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t4], b4, %3, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t5], b5, %3, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t6], b6, %3, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t7], b7, %3, 1;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc)
      : "memory");
}
// O += P V over one 64-key tile (4 x K16): A (P) in TMEM, 8 columns per K16 step; B (V)
// MN-major SW128, 16 keys = 2048 B (128 in 16-B units) per step.  acc = 0 overwrites O.
__device__ __forceinline__ void mma_pv4_w(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred e, p;\n.reg .b64 b1, b2, b3;\n.reg .b32 t1, t2, t3;\n"
      "add.s64 b1, %2, 128; add.s64 b2, %2, 256; add.s64 b3, %2, 384;\n"
      "add.u32 t1, %1, 8; add.u32 t2, %1, 16; add.u32 t3, %1, 24;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t1], b1, %3, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t2], b2, %3, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t3], b3, %3, 1;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit_w(uint32_t bar) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(bar)
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

__device__ __forceinline__ float fmax3f(float a, float b, float c) {
  float m;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(m) : "f"(a), "f"(b), "f"(c));
  return m;
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 2^x on the FMA/ALU pipes (keeps the MUFU free): x = j + f with j = round(x) via the
// 1.5*2^23 trick, 2^f on [-1/2, 1/2] by a degree-3 fit (max rel. error 1.4e-4 incl.
// rounding, far below bf16's 2^-9), 2^j added into the exponent bits.  x >= -126.
constexpr float kP0 = 0.99992829561233520f, kP1 = 0.69326096773147580f, kP2 = 0.24260866641998290f,
                kP3 = 0.05517056211829185f;
__device__ __forceinline__ float2 exp2_poly2(float2 x) {
  x.x = fmaxf(x.x, -126.f);
  x.y = fmaxf(x.y, -126.f);
  const float2 y = __fadd2_rn(x, make_float2(12582912.f, 12582912.f));
  const float2 j = __fadd2_rn(y, make_float2(-12582912.f, -12582912.f));
  const float2 f = __fadd2_rn(x, make_float2(-j.x, -j.y));
  float2 q = __ffma2_rn(make_float2(kP3, kP3), f, make_float2(kP2, kP2));
  q = __ffma2_rn(q, f, make_float2(kP1, kP1));
  q = __ffma2_rn(q, f, make_float2(kP0, kP0));
  return make_float2(__uint_as_float(__float_as_uint(q.x) + (__float_as_uint(y.x) << 23)),
                     __uint_as_float(__float_as_uint(q.y) + (__float_as_uint(y.y) << 23)));
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
// 2^x of two bf16 lanes in one MUFU op (x rounded to bf16 first)
__device__ __forceinline__ uint32_t ex2_bf16x2(uint32_t x) {
  uint32_t y;
  asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

__device__ __forceinline__ uint2 ldg64(const void* p) {
  uint2 r;
  asm volatile("ld.global.nc.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ void stg256(void* p, const uint32_t (&v)[8]) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]),
               "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
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
// L2 prefetch of one 2-D box (no shared memory, no completion): warms L2 for a later TMA load
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ uint2 lds64(uint32_t addr) {
  uint2 r;
  asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "r"(addr) : "memory");
  return r;
}
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void named_bar_sync(int id, int n) { named_bar(id, n); }
__device__ __forceinline__ void named_bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// timeline events (TRACE): clock64 per (event, tile) for the first ntrace_cta CTAs
enum { EV_K_ISSUE = 0, EV_V_ISSUE, EV_KR, EV_KF, EV_S0, EV_S1, EV_P0, EV_P1, EV_PV0, EV_PV1, EV_Q, EV_START, EV_END,
       EV_VF, EV_PW0 /* 14..21: P arrival of softmax warps 0..7 */, EV_L = 22 /* 22..27: warp-0 softmax steps */,
       EV_KDONE = 28, EV_QDONE = 29, EV_QLOADED = 30, EV_QSTART = 31,
       EV_QKI = 32 /* MMA warp: S(g) issued */, EV_PVI = 33 /* PV0(g) issued */, EV_PV1I = 34 /* PV1(g) issued */,
       EV_EPI0 = 35 /* epilogue: last PV done */, EV_EPI1 = 36 /* epilogue stores issued */ };
// `trace_cta` = the launch-wide trace row of this CTA (nullptr = off), hoisted at kernel start.
// Compiled in only with -DDSC_TRACE=1 (the profiling variant built by scripts/trace_attn.py):
// even disabled, the checks cost registers and a reload per event in the softmax loop.
#ifndef DSC_TRACE
#define DSC_TRACE 0
#endif
#if DSC_TRACE
#define TRACE(ev, tile)                                                                                  \
  do {                                                                                                   \
    if (trace_cta && (tile) < kTraceTiles) trace_cta[(ev) * kTraceTiles + (tile)] = clock64();           \
  } while (0)
#else
#define TRACE(ev, tile) do { } while (0)
#endif

#ifndef DSC_ORDER
#define DSC_ORDER 2
#endif
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

// work item idx -> split fastest, then (DSC_ORDER 1, default) problem x kv head, then
// m-block descending: all (problem, head) pairs of the longest causal m-block first
// (LPT-like balance of the persistent CTAs).  DSC_ORDER 0 groups the m-blocks of one
// (problem, head) for L2 reuse of its K/V; measured slower on c5 (9.8K vs 12.4K frames/s).
// The integer fields decode_item needs, selected per item from the two launch parameter
// blocks with constant-offset loads (a reference chosen at run time turns every field read
// into an indexed constant load whose result the compiler cannot keep uniform).
struct ItemGeo {
  int n_splits, P, Hkv, n_mblocks, layer_count, N_total, layer_begin, n_q, grp, q_pos0, A, ring_count, n_self,
      ring_start, R, tiles_per_split, Rp, staged, split_only;
};
__device__ __forceinline__ ItemGeo item_geo(const AttnParams& pa, const AttnParams& pb, bool isb) {
  ItemGeo q;
#define DSC_SEL(f) q.f = isb ? pb.f : pa.f
  DSC_SEL(n_splits); DSC_SEL(P); DSC_SEL(Hkv); DSC_SEL(n_mblocks); DSC_SEL(layer_count); DSC_SEL(N_total);
  DSC_SEL(layer_begin); DSC_SEL(n_q); DSC_SEL(grp); DSC_SEL(q_pos0); DSC_SEL(A); DSC_SEL(ring_count);
  DSC_SEL(n_self); DSC_SEL(ring_start); DSC_SEL(R); DSC_SEL(tiles_per_split); DSC_SEL(Rp); DSC_SEL(staged); DSC_SEL(split_only);
#undef DSC_SEL
  return q;
}
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
#define DSC_OGRP 74   // measured: 74 +0.3-0.8%, 37 +0.3%, 296 -2.8% vs 148 (c5)
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

// Key rows of tile u (kTileN = 64 keys) as (at most) two segments; key row r of segment s
// has id pos0_s + r.  Tiles u < n_extra hold the sink rows (extra index x = 64u + r < A,
// id x) and then the self rows (A <= x < A + n_self, id ring_count + x).  Tile u >= n_extra
// is the LOGICAL window tile b = u - n_extra: window keys [64b, 64b + 64), i.e. the ring
// slots (ring_start + 64b + r) mod R, read as one 64-row box from slot0 = (ring_start +
// 64b) mod R -- the ring keeps a mirror of slots [0, kMirror) after slot R - 1, so the box
// never wraps.  Row r is valid iff 64b + r < cnt, with id A + 64b + r.
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

__device__ __forceinline__ void rotate8(uint32_t tile, int r0, int c8, const float4* __restrict__ rp,
                                        const float2 (&cth)[4], const float2 (&sth)[4], const int (&pos)[8],
                                        const float4 (&pre)[4], int pre_pos) {
  rotate_rows<2, 16384>(tile, r0, c8, rp, cth, sth, pos, pre, pre_pos);
}

// Raw Q rows [m0 + 128*qt, +128) of an item -> SW128 tile in smem by cp.async (16 chunks
// per thread, (query, head) advanced incrementally), then rotated in place at the query
// id (8 rows x 8 frequencies per thread).  Executed by one 128-thread warpgroup.
__device__ __forceinline__ void issue_q_tile(const AttnParams& p, const Item& w, int qt, int lt, uint32_t qtile) {
  const __nv_bfloat16* __restrict__ Qg = reinterpret_cast<const __nv_bfloat16*>(p.q);
  const int ch = lt & 15;
  int rgl = w.m0 + qt * 128 + (lt >> 4);
  int qi = rgl / p.grp, hh = rgl % p.grp;
  const int step_i = 8 / p.grp, step_h = 8 % p.grp;
  const __nv_bfloat16* qbase = Qg + ((long long)w.pp * p.n_q) * p.Hq * 128 + (long long)w.g * p.grp * 128 + 8 * ch;
  const uint32_t dbase = qtile + (ch >> 3) * 16384;
#pragma unroll 4
  for (int it = 0; it < 16; ++it) {
    const int r = it * 8 + (lt >> 4);
    const bool ok = rgl < w.rows_total;
    const __nv_bfloat16* src = qbase + ((long long)qi * p.Hq + hh) * 128;
    cp_async16(dbase + r * 128 + (((ch & 7) ^ (r & 7)) << 4), ok ? (const void*)src : (const void*)Qg, ok ? 16u : 0u);
    rgl += 8;
    qi += step_i;
    hh += step_h;
    if (hh >= p.grp) { hh -= p.grp; ++qi; }
  }
}
__device__ __forceinline__ void rotate_q_tile(const AttnParams& p, const Item& w, int qt, int lt, uint32_t qtile,
                                              int bar_id) {
  const float4* __restrict__ rp = p.rope_pairs;
  const int c8 = lt & 7, rg8 = lt >> 3;
  float2 cth[4], sth[4];
  float4 pre[4];
  int pos[8];
  const int row0 = w.m0 + qt * 128 + rg8 * 8;
  int i = row0 / p.grp, hh = row0 % p.grp;
  const bool dbg = p.dbg_pos != nullptr && w.pp == 0 && w.g == 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    pos[k] = (row0 + k < w.rows_total) ? p.q_pos0 + i : -1;
    if (dbg && c8 == 0 && hh == 0 && pos[k] >= 0) p.dbg_pos[p.dbg_A + p.dbg_R + p.dbg_M + i] = pos[k];
    if (++hh == p.grp) { hh = 0; ++i; }
  }
  const int p0 = max(pos[0], 0);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float4 t = rp[32 + 4 * c8 + j];
    cth[j] = make_float2(t.x, t.y);
    sth[j] = make_float2(t.z, t.w);
    pre[j] = rp[(long long)p0 * 32 + 4 * c8 + j];
  }
  cp_async_wait_all();
  named_bar(bar_id, 128);
  rotate8(qtile, rg8 * 8, c8, rp, cth, sth, pos, pre, p0);
  fence_proxy_async();
}

// Q tile qt of item w straight from global memory into registers, rotated there at the
// query ids and stored once into the SW128 tile (no cp.async staging copy + re-read:
// 64 KB less shared-memory traffic per Q tile pair).  Thread lt rotates frequencies
// 8*c8 .. 8*c8+7 (16-byte chunk c8 of the low and the high 64-column block) of rows
// rg8*8 .. +7; the 8 threads of a row read its 2 x 128 contiguous bytes.
__device__ __forceinline__ uint4 ldg128(const void* ptr) {
  uint4 r;
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(ptr));
  return r;
}
__device__ __forceinline__ void load_rotate_q_tile(const AttnParams& p, const Item& w, int qt, int lt, uint32_t qtile) {
  const float4* __restrict__ rp = p.rope_pairs;
  const __nv_bfloat16* __restrict__ Qg = reinterpret_cast<const __nv_bfloat16*>(p.q);
  const int c8 = lt & 7, rg8 = lt >> 3;
  const int row0 = w.m0 + qt * 128 + rg8 * 8;
  int i = row0 / p.grp, hh = row0 % p.grp;
  const bool dbg = p.dbg_pos != nullptr && w.pp == 0 && w.g == 0;
  const __nv_bfloat16* qbase = Qg + ((long long)w.pp * p.n_q) * p.Hq * 128 + (long long)w.g * p.grp * 128 + 8 * c8;
  float2 cth[4], sth[4], cs[4], sn[4];
  const int p0 = row0 < w.rows_total ? p.q_pos0 + i : 0;
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
#pragma unroll 1
  for (int half = 0; half < 2; ++half) {   // 4 rows per pass: 8 x 16-byte loads in flight
    int pos[4];
    uint4 lo[4], hi[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const bool ok = row0 + half * 4 + k < w.rows_total;
      pos[k] = ok ? p.q_pos0 + i : -1;
      if (dbg && c8 == 0 && hh == 0 && ok) p.dbg_pos[p.dbg_A + p.dbg_R + p.dbg_M + i] = pos[k];
      if (ok) {
        const __nv_bfloat16* src = qbase + ((long long)i * p.Hq + hh) * 128;
        lo[k] = ldg128(src);
        hi[k] = ldg128(src + 64);
      } else {
        lo[k] = hi[k] = make_uint4(0, 0, 0, 0);
      }
      if (++hh == p.grp) { hh = 0; ++i; }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int r = rg8 * 8 + half * 4 + k, pk = pos[k];
      const uint32_t addr = qtile + r * 128 + ((c8 ^ (r & 7)) << 4);
      uint4 ylo = make_uint4(0, 0, 0, 0), yhi = make_uint4(0, 0, 0, 0);
      if (pk >= 0) {
        if (pk == prev) {
        } else if (pk == prev + 1) {   // next id: advance (cos, sin) by R(theta)
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
      sts128(addr, ylo);
      sts128(addr + 16384, yhi);
    }
  }
  fence_proxy_async();
}

}  // namespace tcc
}  // namespace dsc
