// tcgen05.mma (cta_group::1, kind::f16, bf16 -> f32) issue throughput per SM, 148 CTAs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_bench mma_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
               "l"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
               "r"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void wait(uint32_t bar, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(bar), "r"(ph) : "memory");
}

// MODE 0: SS N=128 into one accumulator; 1: TS N=128 (A from TMEM); 2: SS N=256;
// 3: SS N=128 alternating 4 accumulators (S0 S1 O0 O1 pattern); 4: our QK/PV mix (SS N128 + TS N128)
#define LD32(taddr, r)                                                                                        \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15," \
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                      \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), \
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),      \
                 "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),    \
                 "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),    \
                 "=r"(r[29]), "=r"(r[30]), "=r"(r[31])                                                         \
               : "r"(taddr))
// INTF bit 0: 4 warps of LDS/STS.128 traffic on a separate 32 KB smem region;
// bit 1: 8 warps of tcgen05.ld x32 loops (softmax-like) on TMEM columns 128..255 (lanes of their quarter)
template <int MODE, int INTF = 0>
__global__ void __launch_bounds__(512, 1) k(long long* cyc, int rounds) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t barx[6];
  uint32_t bar_b[6];
  for (int i = 0; i < 6; ++i) bar_b[i] = (uint32_t)__cvta_generic_to_shared(&barx[i]);
  const int warp = threadIdx.x >> 5;
  const uint32_t sbase = ((uint32_t)__cvta_generic_to_shared(sm) + 1023) & ~1023u;
  const uint32_t bar_a = (uint32_t)__cvta_generic_to_shared(&bar);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_a));
  if (threadIdx.x == 0) for (int i = 0; i < 6; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_b[i]));
  __shared__ __align__(8) uint64_t bard;
  const uint32_t bar_done = (uint32_t)__cvta_generic_to_shared(&bard);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_done));
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar_done) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  long long t0 = 0, t1 = 0;
  __shared__ volatile int done;
  if (threadIdx.x == 0) done = 0;
  __syncthreads();
  if ((INTF & 1) && warp >= 4 && warp < 8) {
    const uint32_t region = sbase + 65536 - 32768 + 0;   // overlaps operand B region (bytes only matter for bandwidth)
    uint32_t acc = 0;
    while (!done) {
      for (int i = 0; i < 16; ++i) {
        const uint32_t a = region + ((threadIdx.x * 16 + i * 2048) & 32767);
        uint32_t x, y, z, w;
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "r"(a));
        acc += x ^ y ^ z ^ w;
        asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(a + 16384 * 0), "r"(acc), "r"(x), "r"(y), "r"(z));
      }
    }
    if (acc == 12345) cyc[1000] = acc;
  }
  if ((INTF & 2) && warp >= 8) {
    uint32_t acc = 0;
    const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + 128u;
    while (!done) {
      for (int c = 0; c < 4; ++c) { uint32_t r[32]; LD32(base + c * 32, r); asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); for (int i = 0; i < 32; ++i) acc ^= r[i]; }
    }
    if (acc == 12345) cyc[1000] = acc;
  }
  if (threadIdx.x == 0) {
    const uint64_t da = sdesc(sbase, 16, 1024), db = sdesc(sbase + 32768, 16, 1024);
    t0 = clock64();
    for (int r = 0; r < rounds; ++r) {
      for (int k8 = 0; k8 < 8; ++k8) {
        const uint64_t off = (uint64_t)((k8 >> 2) * 1024 + (k8 & 3) * 2);
        if (MODE == 0) mma_ss(tmem, da + off, db + off, idesc_bf16(128, 128, 0, 0), k8 > 0);
        if (MODE == 1) mma_ts(tmem + 256, tmem + k8 * 8, db + off, idesc_bf16(128, 128, 0, 0), k8 > 0);
        if (MODE == 2) mma_ss(tmem, da + off, db + off, idesc_bf16(128, 256, 0, 0), k8 > 0);
        if (MODE == 3) mma_ss(tmem + (r & 3) * 128, da + off, db + off, idesc_bf16(128, 128, 0, 0), k8 > 0);
        if (MODE == 5) mma_ss(tmem, da + off, db + off, idesc_bf16(128, 64, 0, 0), k8 > 0);
        if (MODE == 6) mma_ss(tmem, da + off, db + off, idesc_bf16(128, 16, 0, 0), k8 > 0);
        if (MODE == 7) mma_ss(tmem, da + off, db + off, idesc_bf16(128, 256, 0, 0), k8 > 0);
        if (MODE == 8) {   // one 64-key tile of the v5 attention: QK0 QK1 (SS N64) + PV0 PV1 (TS K=64 -> 4 MMAs each)
          const uint64_t offb = (uint64_t)((k8 >> 2) * 512 + (k8 & 3) * 2);
          mma_ss(tmem + (r & 1) * 64, da + off, db + offb, idesc_bf16(128, 64, 0, 0), k8 > 0);
          mma_ss(tmem + 128 + (r & 1) * 64, da + off, db + offb, idesc_bf16(128, 64, 0, 0), k8 > 0);
          if (k8 < 4) {
            mma_ts(tmem + 256, tmem + (r & 1) * 64 + k8 * 8, db + (uint64_t)(k8 * 128), idesc_bf16(128, 128, 0, 1), 1);
            mma_ts(tmem + 384, tmem + 128 + (r & 1) * 64 + k8 * 8, db + (uint64_t)(k8 * 128), idesc_bf16(128, 128, 0, 1), 1);
          }
        }
        if (MODE == 9 || MODE == 10 || MODE == 11) {   // v5 tile with the kernel's commits (MODE 10: 1 commit per tile)
          const uint64_t offb = (uint64_t)((k8 >> 2) * 512 + (k8 & 3) * 2);
          mma_ss(tmem + (r & 1) * 64, da + off, db + offb, idesc_bf16(128, 64, 0, 0), k8 > 0);
          if (MODE == 9 && k8 == 7) commit(bar_b[0]);
          mma_ss(tmem + 128 + (r & 1) * 64, da + off, db + offb, idesc_bf16(128, 64, 0, 0), k8 > 0);
          if (MODE == 9 && k8 == 7) { commit(bar_b[1]); commit(bar_b[2]); }
          if (k8 < 4) {
            mma_ts(tmem + 256, tmem + (r & 1) * 64 + k8 * 8, db + (uint64_t)(k8 * 128), idesc_bf16(128, 128, 0, 1), 1);
            if (MODE == 9 && k8 == 3) commit(bar_b[3]);
            mma_ts(tmem + 384, tmem + 128 + (r & 1) * 64 + k8 * 8, db + (uint64_t)(k8 * 128), idesc_bf16(128, 128, 0, 1), 1);
            if (MODE == 9 && k8 == 3) { commit(bar_b[4]); commit(bar_b[5]); }
          }
          if (MODE == 10 && k8 == 7) commit(bar_b[0]);
          if (MODE == 11 && (k8 == 3 || k8 == 7)) {   // satisfied mbarrier waits between MMA groups (4 per tile)
            wait(bar_done, 0); wait(bar_done, 0);
          }
        }
        if (MODE == 4) {
          if (r & 1) mma_ts(tmem + 256 + (r & 2) * 64, tmem + (r & 2) * 64 + k8 * 8, db + (uint64_t)(k8 * 128),
                            idesc_bf16(128, 128, 0, 1), 1);
          else mma_ss(tmem + (r & 2) * 64, da + off, db + off, idesc_bf16(128, 128, 0, 0), k8 > 0);
        }
      }
    }
    commit(bar_a);
    wait(bar_a, 0);
    t1 = clock64();
    cyc[blockIdx.x] = t1 - t0;
    done = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int MODE, int INTF>
void run(const char* name, long long* c, int smem) {
  const int rounds = 4000;
  cudaFuncSetAttribute(k<MODE, INTF>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<MODE, INTF><<<148, 512, smem>>>(c, rounds);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); exit(1); }
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  const double flop_sm = 2.0 * 128 * 128 * 16 * 8 * rounds;
  printf("%-22s intf %d: %7.1f cyc/MMA  %7.0f flop/clk/SM\n", name, INTF, (double)h / (8.0 * rounds), flop_sm / h);
}
int main() {
  long long* c;
  cudaMalloc(&c, 2000 * 8);
  const int smem = 64 * 1024 + 1024;
  run<0, 0>("SS M128 N128 K16", c, smem); run<0, 1>("SS M128 N128 K16", c, smem);
  run<0, 2>("SS M128 N128 K16", c, smem); run<0, 3>("SS M128 N128 K16", c, smem);
  run<1, 0>("TS M128 N128 K16", c, smem); run<1, 1>("TS M128 N128 K16", c, smem);
  run<1, 2>("TS M128 N128 K16", c, smem); run<1, 3>("TS M128 N128 K16", c, smem);
  run<5, 0>("SS M128 N64 K16 (flop as N128)", c, smem);
  run<6, 0>("SS M128 N16 K16 (flop as N128)", c, smem);

  run<8, 0>("v5 tile (per 3 MMAs)", c, smem);
  run<8, 1>("v5 tile (per 3 MMAs)", c, smem);
  run<9, 0>("v5 tile + 6 commits", c, smem);
  run<10, 0>("v5 tile + 1 commit", c, smem);
  run<11, 0>("v5 tile + 4 waits", c, smem);
  run<4, 0>("QK+PV mix", c, smem); run<4, 1>("QK+PV mix", c, smem);
  run<4, 2>("QK+PV mix", c, smem); run<4, 3>("QK+PV mix", c, smem);
  return 0;
}
