// Layout + throughput check of tcgen05.mma.cta_group::2 (CTA pair, M=256) for the
// attention shapes: S = Q K^T (SS, K-major A and B) and O = P V (TS: P in TMEM, V MN-major).
// Assumed: A is M-split (CTA r holds rows 128r..), B is N-split (CTA r holds N/2 columns),
// D is M-split (CTA r's TMEM lanes = rows 128r..).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pair_mma_test pair_mma_test.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_bf16.h>

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
__device__ __forceinline__ void mma2_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
               "l"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma2_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
               "r"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ void commit2(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
               "h"((uint16_t)3) : "memory");
}
__device__ __forceinline__ void wait(uint32_t bar, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(bar), "r"(ph) : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
#define LD32(taddr, r)                                                                                        \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15," \
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                      \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), \
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),      \
                 "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),    \
                 "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),    \
                 "=r"(r[29]), "=r"(r[30]), "=r"(r[31])                                                         \
               : "r"(taddr))
#define ST32(taddr, r)                                                                                         \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14," \
               "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),      \
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),          \
               "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),   \
               "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), \
               "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])  \
               : "memory")

// sw128 byte offset of element (row r, col c) of a K-major (row = M/N index, col = K) tile
// stored as 64-column boxes of `rows` rows each
__device__ __host__ inline uint32_t sw_off(int r, int c, int rows) {
  return (uint32_t)((c / 64) * rows * 128 + r * 128 + ((((c % 64) / 8) ^ (r % 8)) << 4) + (c % 8) * 2);
}

// Q: [256][128], K: [128 keys][128], P: [256][128 keys], V: [128 keys][128 d] (bf16 in global)
// S out: [256][128] f32, O out: [256][128] f32
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    pair_kernel(const __nv_bfloat16* Q, const __nv_bfloat16* K, const __nv_bfloat16* P, const __nv_bfloat16* V,
                float* S, float* O, long long* cyc, int reps) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar[2];
  const uint32_t rank = cluster_rank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t sbase = ((uint32_t)__cvta_generic_to_shared(sm) + 1023) & ~1023u;
  uint8_t* gs = sm + (sbase - (uint32_t)__cvta_generic_to_shared(sm));
  const uint32_t sQ = sbase, sK = sbase + 32768, sV = sbase + 49152;   // Q 32K, K half 16K, V half 16K
  // fill: Q rows 128*rank.., K keys 64*rank.., V d-cols 64*rank..
  for (int i = threadIdx.x; i < 128 * 128; i += 128) {
    const int r = i / 128, c = i % 128;
    *reinterpret_cast<__nv_bfloat16*>(gs + sw_off(r, c, 128)) = Q[(128 * rank + r) * 128 + c];
  }
  for (int i = threadIdx.x; i < 64 * 128; i += 128) {
    const int r = i / 128, c = i % 128;
    *reinterpret_cast<__nv_bfloat16*>(gs + 32768 + sw_off(r, c, 64)) = K[(64 * rank + r) * 128 + c];
  }
  for (int i = threadIdx.x; i < 128 * 64; i += 128) {
    const int k = i / 64, n = i % 64;     // V MN-major: row = key, 64 d-columns of this CTA
    *reinterpret_cast<__nv_bfloat16*>(gs + 49152 + sw_off(k, n, 128)) = V[k * 128 + 64 * rank + n];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  const uint32_t b0 = (uint32_t)__cvta_generic_to_shared(&bar[0]);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b0));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b0 + 8));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  // P (this CTA's 128 rows) -> TMEM cols 256.. as packed bf16x2 (row = lane)
  {
    const int row = 128 * rank + warp * 32 + lane;
    for (int ch = 0; ch < 2; ++ch) {
      uint32_t r[32];
      for (int j = 0; j < 32; ++j) {
        const __nv_bfloat16 lo = P[row * 128 + ch * 64 + 2 * j], hi = P[row * 128 + ch * 64 + 2 * j + 1];
        r[j] = (uint32_t)__bfloat16_as_ushort(lo) | ((uint32_t)__bfloat16_as_ushort(hi) << 16);
      }
      ST32(tmem + ((uint32_t)(warp * 32) << 16) + 256 + ch * 32, r);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  long long t0 = clock64();
  if (rank == 0 && threadIdx.x == 0) {
    const uint64_t da = sdesc(sQ, 16, 1024), db = sdesc(sK, 16, 1024), dv = sdesc(sV, 16, 1024);
    for (int rep = 0; rep < reps; ++rep) {
      for (int k8 = 0; k8 < 8; ++k8) {
        const uint64_t oa = (uint64_t)((k8 >> 2) * 1024 + (k8 & 3) * 2);     // Q: 64-col boxes of 128 rows (16 KB)
        const uint64_t ob = (uint64_t)((k8 >> 2) * 512 + (k8 & 3) * 2);      // K: 64-col boxes of 64 rows (8 KB)
        mma2_ss(tmem, da + oa, db + ob, idesc_bf16(256, 128, 0, 0), k8 > 0);
      }
      for (int k8 = 0; k8 < 8; ++k8)
        mma2_ts(tmem + 128, tmem + 256 + k8 * 8, dv + (uint64_t)(k8 * 128), idesc_bf16(256, 128, 0, 1), k8 > 0);
    }
    commit2(b0);
  }
  wait(b0, 0);
  long long t1 = clock64();
  asm volatile("tcgen05.fence::after_thread_sync;");
  {
    const int row = 128 * rank + warp * 32 + lane;
    for (int ch = 0; ch < 4; ++ch) {
      uint32_t r[32];
      LD32(tmem + ((uint32_t)(warp * 32) << 16) + ch * 32, r);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int j = 0; j < 32; ++j) S[row * 128 + ch * 32 + j] = __uint_as_float(r[j]);
      LD32(tmem + ((uint32_t)(warp * 32) << 16) + 128 + ch * 32, r);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int j = 0; j < 32; ++j) O[row * 128 + ch * 32 + j] = __uint_as_float(r[j]);
    }
  }
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  const int nQ = 256 * 128, nK = 128 * 128;
  std::vector<__nv_bfloat16> hQ(nQ), hK(nK), hP(nQ), hV(nK);
  std::vector<float> fQ(nQ), fK(nK), fP(nQ), fV(nK);
  srand(1);
  auto rnd = [] { return (float)(rand() % 2001 - 1000) / 1000.f; };
  for (int i = 0; i < nQ; ++i) { hQ[i] = __float2bfloat16(rnd()); fQ[i] = __bfloat162float(hQ[i]); }
  for (int i = 0; i < nQ; ++i) { hP[i] = __float2bfloat16(rnd()); fP[i] = __bfloat162float(hP[i]); }
  for (int i = 0; i < nK; ++i) { hK[i] = __float2bfloat16(rnd()); fK[i] = __bfloat162float(hK[i]); }
  for (int i = 0; i < nK; ++i) { hV[i] = __float2bfloat16(rnd()); fV[i] = __bfloat162float(hV[i]); }
  __nv_bfloat16 *dQ, *dK, *dP, *dV; float *dS, *dO; long long* dc;
  cudaMalloc(&dQ, nQ * 2); cudaMalloc(&dK, nK * 2); cudaMalloc(&dP, nQ * 2); cudaMalloc(&dV, nK * 2);
  cudaMalloc(&dS, nQ * 4); cudaMalloc(&dO, nQ * 4); cudaMalloc(&dc, 8 * 300);
  cudaMemcpy(dQ, hQ.data(), nQ * 2, cudaMemcpyHostToDevice); cudaMemcpy(dK, hK.data(), nK * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dP, hP.data(), nQ * 2, cudaMemcpyHostToDevice); cudaMemcpy(dV, hV.data(), nK * 2, cudaMemcpyHostToDevice);
  const int smem = 65536 + 1024;
  cudaFuncSetAttribute(pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  pair_kernel<<<2, 128, smem>>>(dQ, dK, dP, dV, dS, dO, dc, 1);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<float> S(nQ), O(nQ);
  cudaMemcpy(S.data(), dS, nQ * 4, cudaMemcpyDeviceToHost); cudaMemcpy(O.data(), dO, nQ * 4, cudaMemcpyDeviceToHost);
  double es = 0, eo = 0;
  for (int m = 0; m < 256; ++m)
    for (int n = 0; n < 128; ++n) {
      double s = 0, o = 0;
      for (int k = 0; k < 128; ++k) { s += (double)fQ[m * 128 + k] * fK[n * 128 + k]; o += (double)fP[m * 128 + k] * fV[k * 128 + n]; }
      es = fmax(es, fabs(s - S[m * 128 + n])); eo = fmax(eo, fabs(o - O[m * 128 + n]));
    }
  printf("S = Q K^T  (cta_group::2 SS): max abs err %.3e  (S[0]=%f S[200*128+77]=%f)\n", es, S[0], S[200 * 128 + 77]);
  printf("O = P V    (cta_group::2 TS): max abs err %.3e\n", eo);
  // throughput: 148 CTAs = 74 pairs, reps of (8 QK + 8 PV) MMAs
  const int reps = 2000;
  pair_kernel<<<148, 128, smem>>>(dQ, dK, dP, dV, dS, dO, dc, reps);
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  long long h; cudaMemcpy(&h, dc, 8, cudaMemcpyDeviceToHost);
  const double flop_pair = 2.0 * 256 * 128 * 128 * 2 * reps;
  printf("pair throughput: %.1f cycles per M256 N128 K16 MMA, %.0f flop/clk/SM\n", (double)h / (16.0 * reps),
         flop_pair / h / 2);
  return 0;
}
