// Throughput of ex2.approx (MUFU) and cvt.rn.bf16x2.f32 (F2FP) per SM on this GPU.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint32_t pk(float a, float b) { uint32_t r; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a), "f"(b)); return r; }
template <int MODE>
__global__ void k(float* out, long long* cyc, int iters) {
  float a[8]; uint32_t acc = 0;
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0 || MODE == 2) a[i] = ex2(a[i] * -0.001f);
      if (MODE == 1 || MODE == 2) acc ^= pk(a[i], a[(i + 1) & 7]);
      if (MODE == 1) a[i] += 1e-7f;
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  float s = acc; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* o; long long* c; cudaMalloc(&o, 148 * 1024 * 4); cudaMalloc(&c, 148 * 8);
  const char* names[3] = {"MUFU.EX2 only", "F2FP(bf16x2) only", "EX2 + F2FP"};
  for (int mode = 0; mode < 3; ++mode) for (int threads : {128, 512, 1024}) {
    int iters = 200;
    if (mode == 0) k<0><<<148, threads>>>(o, c, iters);
    if (mode == 1) k<1><<<148, threads>>>(o, c, iters);
    if (mode == 2) k<2><<<148, threads>>>(o, c, iters);
    cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    double ops = (double)threads * iters * 8;   // per SM, of each kind
    printf("%-20s threads %4d: %.2f ops/clk/SM (%lld cycles)\n", names[mode], threads, ops / h, h);
  }
  return 0;
}
