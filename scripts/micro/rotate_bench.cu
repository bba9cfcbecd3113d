// Microbenchmark of the in-place RoPE routine of attn_tc.cu (rotate8), isolated:
// 148 CTAs x 128 threads rotate a 128x128 bf16 SW128 tile in smem 200 times.
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
#include <cuda.h>
namespace dsc { namespace tc {
constexpr float kRescaleThreshold = 8.0f;
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
#ifndef DSC_POLY
#define DSC_POLY 0
#endif
constexpr int kPolyPerGroup = DSC_POLY;   // of every 8 columns of a full tile, this many use exp2_poly2

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

// timeline events (TRACE): clock64 per (event, tile) for the first ntrace_cta CTAs
enum { EV_K_ISSUE = 0, EV_V_ISSUE, EV_KR, EV_KF, EV_S0, EV_S1, EV_P0, EV_P1, EV_PV0, EV_PV1, EV_Q, EV_START, EV_END,
       EV_VF, EV_PW0 /* 14..21: P arrival of softmax warps 0..7 */, EV_L = 22 /* 22..27: warp-0 softmax steps */,
       EV_KDONE = 28, EV_QDONE = 29, EV_QLOADED = 30, EV_QSTART = 31 };
#define TRACE(ev, tile)                                                                                  \
  do {                                                                                                   \
    if (p.trace && blockIdx.x < (unsigned)p.ntrace_cta && (tile) < kTraceTiles)                          \
      p.trace[((long long)blockIdx.x * kTraceEvents + (ev)) * kTraceTiles + (tile)] = clock64();          \
  } while (0)

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
__device__ __forceinline__ void rotate8(uint32_t tile, int r0, int c8, const float4* __restrict__ rp,
                                        const float2 (&cth)[4], const float2 (&sth)[4], const int (&pos)[8],
                                        const float4 (&pre)[4], int pre_pos) {
  // (cs, sn) start at the prefetched table entry of id pre_pos (the first valid row)
  float2 cs[4], sn[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) { cs[j] = make_float2(pre[j].x, pre[j].y); sn[j] = make_float2(pre[j].z, pre[j].w); }
  int prev = pre_pos;
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    uint4 lo[4], hi[4];
    uint32_t addr[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int r = r0 + half * 4 + k;
      addr[k] = tile + r * 128 + ((c8 ^ (r & 7)) << 4);
      lo[k] = lds128(addr[k]);
      hi[k] = lds128(addr[k] + 16384);
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
      sts128(addr[k] + 16384, yhi);
    }
  }
}

// straight-line variant: all 8 rows valid with ids pos0 .. pos0+7
__device__ __forceinline__ void rotate8_lin(uint32_t tile, int r0, int c8, const float2 (&cth)[4], const float2 (&sth)[4],
                                            const float4 (&pre)[4]) {
  float2 cs[4], sn[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) { cs[j] = make_float2(pre[j].x, pre[j].y); sn[j] = make_float2(pre[j].z, pre[j].w); }
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    uint4 lo[4], hi[4];
    uint32_t addr[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int r = r0 + half * 4 + k;
      addr[k] = tile + r * 128 + ((c8 ^ (r & 7)) << 4);
      lo[k] = lds128(addr[k]);
      hi[k] = lds128(addr[k] + 16384);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (half + k > 0) {
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
        const float2 yl = __ffma2_rn(av, cs[j], __fmul2_rn(make_float2(-bv.x, -bv.y), sn[j]));
        const float2 yh = __ffma2_rn(av, sn[j], __fmul2_rn(bv, cs[j]));
        ol[j] = pack_bf16(yl.x, yl.y);
        oh[j] = pack_bf16(yh.x, yh.y);
      }
      sts128(addr[k], make_uint4(ol[0], ol[1], ol[2], ol[3]));
      sts128(addr[k] + 16384, make_uint4(oh[0], oh[1], oh[2], oh[3]));
    }
  }
}
}}  // namespace
using namespace dsc::tc;
__global__ void __launch_bounds__(512, 1) bench(const float4* rp, long long* out, int variant, int nwarps_active) {
  __shared__ __align__(1024) uint8_t tile[32768];
  const int t = threadIdx.x;
  for (int i = t; i < 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(tile)[i] = 0x3F803F80u * (i & 1);
  __syncthreads();
  if (t >= 32 * nwarps_active) return;
  const int lt = t & 127, grp = t >> 7;
  const int c8 = lt & 7, rg8 = lt >> 3;
  float2 cth[4], sth[4];
  float4 pre[4];
  for (int j = 0; j < 4; ++j) {
    const float4 q = rp[32 + 4 * c8 + j];
    cth[j] = make_float2(q.x, q.y); sth[j] = make_float2(q.z, q.w);
    pre[j] = rp[1000 * 32 + 4 * c8 + j];
  }
  int pos[8];
  for (int k = 0; k < 8; ++k) pos[k] = 1000 + rg8 * 8 + k;
  const uint32_t base = su32(tile);
  // groups of 128 threads beyond the first share rows (only timing matters)
  const long long t0 = clock64();
  for (int it = 0; it < 200; ++it) {
    if (variant == 0) rotate8(base, rg8 * 8, c8, rp, cth, sth, pos, pre, pos[0]);
    else rotate8_lin(base, rg8 * 8, c8, cth, sth, pre);
  }
  const long long t1 = clock64();
  if (t == 0) out[blockIdx.x] = (t1 - t0) / 200;
  (void)grp;
}
int main() {
  float4* rp; long long* out;
  cudaMalloc(&rp, 2000 * 32 * sizeof(float4));
  cudaMemset(rp, 0, 2000 * 32 * sizeof(float4));
  cudaMalloc(&out, 148 * sizeof(long long));
  for (int variant = 0; variant < 2; ++variant)
    for (int nw = 4; nw <= 16; nw *= 2) {
      bench<<<148, 512>>>(rp, out, variant, nw);
      cudaDeviceSynchronize();
      long long h[148];
      cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
      printf("variant %s warps %2d: %lld cycles per 8-row x 8-freq rotation call (%s)\n",
             variant ? "straight-line" : "rotate8", nw, h[0], cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
