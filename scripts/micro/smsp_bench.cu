// Does a warp issuing tcgen05.mma into a saturated tensor queue slow the ALU work of a warp
// on the SAME sub-partition?  One CTA per SM, 8 warps: warp 0 = MMA issuer (SMSP 0), warps
// 4 (SMSP 0) and 5 (SMSP 1) = FFMA loops.  Reports the FFMA loop time of warp 4 and of
// warp 5 with the MMA warp idle (mode 0) and issuing back-to-back SS MMAs M=128 N=64 K=16
// (mode 1: the QK^T shape of attn_tc, smem-operand-bound).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o smsp_bench smsp_bench.cu
#include <cstdio>
#include <cstdint>

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

__global__ void __launch_bounds__(256, 1) k(long long* out, int mode, int n_mma) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t sb = ((uint32_t)__cvta_generic_to_shared(sm) + 1023u) & ~1023u;
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tslot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  if (warp == 0 && mode == 1) {
    const uint64_t da = sdesc(sb, 16, 1024), db = sdesc(sb + 32768, 16, 1024);
    constexpr uint32_t id = idesc_bf16(128, 64, 0, 0);
    long long t0 = clock64();
    for (int i = 0; i < n_mma; ++i) {
      if (lane == 0)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                     ::"r"(tmem + (uint32_t)((i & 3) * 64)), "l"(da + (uint64_t)(2 * (i & 7))), "l"(db + (uint64_t)(2 * (i & 7))),
                     "r"(id), "r"(1u) : "memory");
      __syncwarp();
    }
    if (lane == 0) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b) : "memory");
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(b) : "memory");
    if (lane == 0 && blockIdx.x == 0) out[2] = clock64() - t0;
  }
  if (warp == 4 || warp == 5) {
    float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    long long t0 = clock64();
    for (int i = 0; i < 20000; ++i) {
      a0 = fmaf(a0, 1.0001f, 0.5f); a1 = fmaf(a1, 1.0001f, 0.5f); a2 = fmaf(a2, 1.0001f, 0.5f); a3 = fmaf(a3, 1.0001f, 0.5f);
      a4 = fmaf(a4, 1.0001f, 0.5f); a5 = fmaf(a5, 1.0001f, 0.5f); a6 = fmaf(a6, 1.0001f, 0.5f); a7 = fmaf(a7, 1.0001f, 0.5f);
    }
    long long t = clock64() - t0;
    if (lane == 0 && blockIdx.x == 0) out[warp - 4] = t;
    if (a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 == 12345.f) out[3] = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(d, 0, 64);
      k<<<148, 256, 100 * 1024>>>(d, mode, 4000);
      long long h[4];
      cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
      printf("mode %d (%s): FFMA loop warp4 (same SMSP as the MMA warp) %lld clk, warp5 (other SMSP) %lld clk, MMA loop %lld clk\n",
             mode, mode ? "MMA warp issuing" : "MMA warp idle", h[0], h[1], h[2]);
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
}
