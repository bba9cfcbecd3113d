#include <cstdio>
#include <cstdint>
__global__ void k(long long* out, int mode) {
  __shared__ __align__(8) uint64_t bar;
  uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(b) : "memory");   // phase 0 complete
  }
  __syncthreads();
  if (threadIdx.x >= 32) return;
  long long t0 = clock64();
  uint32_t acc = 0;
  for (int i = 0; i < 1000; ++i) {
    uint32_t ok;
    if (mode == 0)
      asm volatile("{\n.reg .pred P1;\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n" : "=r"(ok) : "r"(b), "r"(0) : "memory");
    else if (mode == 1)
      asm volatile("{\n.reg .pred P1;\nmbarrier.test_wait.parity.acquire.cta.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n" : "=r"(ok) : "r"(b), "r"(0) : "memory");
    else if (mode == 2)
      asm volatile("{\n.reg .pred P1;\nmbarrier.try_wait.parity.relaxed.cta.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n" : "=r"(ok) : "r"(b), "r"(0) : "memory");
    else
      asm volatile("{\n.reg .pred P1;\nmbarrier.test_wait.parity.relaxed.cta.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n" : "=r"(ok) : "r"(b), "r"(0) : "memory");
    acc += ok;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = acc; }
}
int main() {
  long long* d; cudaMalloc(&d, 16);
  for (int m = 0; m < 4; ++m) {
    k<<<1, 64>>>(d, m); long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("mode %d (%s): %.1f cycles per satisfied wait (ok=%lld)\n", m, m==0?"try_wait acquire":m==1?"test_wait acquire":m==2?"try_wait relaxed":"test_wait relaxed", h[0] / 1000.0, h[1]);
  }
}
