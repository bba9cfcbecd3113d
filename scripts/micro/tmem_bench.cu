// TMEM load/store throughput (tcgen05.ld/st 32x32b) and a softmax-shaped loop, per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_bench tmem_bench.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint32_t pk(float a, float b) { uint32_t r; asm("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(r) : "f"(a), "f"(b)); return r; }

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
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// MODE 0: ld x32 + wait per load; 1: 4 loads then wait; 2: st x32; 3: softmax-shaped 2-pass tile
// (ld 2x32 + wait, max; ld again, ffma/ex2/add/pack, st 32), 4: one-pass tile (ld 4x32, wait, max, exp...)
template <int MODE>
__global__ void __launch_bounds__(512, 1) k(uint32_t* out, long long* cyc, int iters) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 128);
  uint32_t acc = 0;
  float accf = 0.f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {
#pragma unroll 1
      for (int c = 0; c < 4; ++c) { uint32_t r[32]; LD32(base + c * 32, r); wait_ld(); for (int i = 0; i < 32; ++i) acc ^= r[i]; }
    } else if (MODE == 1) {
      uint32_t r[32], s[32], u[32], v[32];
      LD32(base, r); LD32(base + 32, s); LD32(base + 64, u); LD32(base + 96, v); wait_ld();
      for (int i = 0; i < 32; ++i) acc ^= r[i] + s[i] + u[i] + v[i];
    } else if (MODE == 2) {
      uint32_t r[32];
      for (int i = 0; i < 32; ++i) r[i] = acc + i;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) ST32(base + c * 32, r);
      wait_st();
      acc += 1;
    } else if (MODE == 3 || MODE == 5) {
      float mx = -1e30f;
#pragma unroll 1
      for (int hf = 0; hf < 2; ++hf) {
        uint32_t r[64];
        LD32(base + 64 * hf, r); LD32(base + 64 * hf + 32, (&r[32])); wait_ld();
        for (int i = 0; i < 64; ++i) mx = fmaxf(mx, __uint_as_float(r[i]));
      }
      float l = 0.f;
#pragma unroll 1
      for (int hf = 0; hf < 2; ++hf) {
        uint32_t r[64];
        LD32(base + 64 * hf, r); LD32(base + 64 * hf + 32, (&r[32])); wait_ld();
#pragma unroll
        for (int i = 0; i < 64; i += 2) {
          float2 x = __ffma2_rn(make_float2(__uint_as_float(r[i]), __uint_as_float(r[i + 1])), make_float2(0.1f, 0.1f),
                                make_float2(-mx, -mx));
          float a = MODE == 5 ? x.x : ex2(x.x), b = ex2(x.y);
          l += a + b;
          r[i >> 1] = pk(a, b);
        }
        ST32(base + 32 * hf, r);
      }
      wait_st();
      accf += l;
    } else if (MODE == 4) {
      uint32_t r[128];
      LD32(base, r); LD32(base + 32, (&r[32])); LD32(base + 64, (&r[64])); LD32(base + 96, (&r[96])); wait_ld();
      float mx = -1e30f;
      for (int i = 0; i < 128; ++i) mx = fmaxf(mx, __uint_as_float(r[i]));
      float l = 0.f;
#pragma unroll
      for (int i = 0; i < 128; i += 2) {
        float2 x = __ffma2_rn(make_float2(__uint_as_float(r[i]), __uint_as_float(r[i + 1])), make_float2(0.1f, 0.1f),
                              make_float2(-mx, -mx));
        float a = ex2(x.x), b = ex2(x.y);
        l += a + b;
        r[i >> 1] = pk(a, b);
      }
      ST32(base, r); ST32(base + 32, (&r[32]));
      wait_st();
      accf += l;
    }
  }
  long long t1 = clock64();
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc + __float_as_uint(accf);
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  uint32_t* o; long long* c;
  cudaMalloc(&o, 148 * 512 * 4); cudaMalloc(&c, 148 * 8);
  const char* names[6] = {"ld x32 +wait each", "ld 4x32 then wait", "st 4x32", "softmax 2-pass tile",
                          "softmax 1-pass tile", "2-pass, half exps"};
  for (int mode = 0; mode < 6; ++mode)
    for (int warps : {4, 8, 16}) {
      const int iters = 400;
      const int th = warps * 32;
      switch (mode) {
        case 0: k<0><<<148, th>>>(o, c, iters); break;
        case 1: k<1><<<148, th>>>(o, c, iters); break;
        case 2: k<2><<<148, th>>>(o, c, iters); break;
        case 3: k<3><<<148, th>>>(o, c, iters); break;
        case 4: k<4><<<148, th>>>(o, c, iters); break;
        case 5: k<5><<<148, th>>>(o, c, iters); break;
      }
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
      // bytes per SM per iteration: each thread touches 128 columns x 4 B (per pass)
      const double bytes = (double)th * 128 * 4 * iters;
      const double tiles = (double)warps / 4 * iters;   // 128-row x 128-col tiles per SM
      printf("%-22s warps %2d: %8.1f B/clk/SM (per pass)  %7.0f cycles per 128x128 tile-row-set  (%lld cyc)\n",
             names[mode], warps, bytes / h, h / tiles, h);
    }
  return 0;
}
