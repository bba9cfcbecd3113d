// Per-SM throughput of the softmax building blocks on this GPU (one CTA per SM, W warps):
// MUFU.EX2, FFMA2, FADD2, F2FP.BF16 pack, and the v7 kernel's exp loop over 64 columns
// (FFMA2 -> EX2 -> FADD2 + F2FP) with and without a polynomial share.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o softmax_bench softmax_bench.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ float ex2f(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  uint32_t r; asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo)); return r;
}
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

template <int MODE, int POLY>
__global__ void k(uint32_t* out, long long* cyc, int iters) {
  uint32_t r[64];
  for (int i = 0; i < 64; ++i) r[i] = __float_as_uint((float)((threadIdx.x * 7 + i * 13) & 63) * -0.05f);
  float2 acc = make_float2(0.f, 0.f), acc2 = acc;
  const float2 sc = make_float2(1.1f, 1.1f), nm = make_float2(-0.3f, -0.3f);
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {   // EX2 only: 64 per thread per iteration
#pragma unroll
      for (int c = 0; c < 64; ++c) r[c] = __float_as_uint(ex2f(__uint_as_float(r[c])));
    } else if (MODE == 1) {   // FFMA2 only: 32 per thread per iteration (64 flops-pairs)
#pragma unroll
      for (int c = 0; c < 64; c += 2) {
        float2 x = __ffma2_rn(make_float2(__uint_as_float(r[c]), __uint_as_float(r[c + 1])), sc, nm);
        r[c] = __float_as_uint(x.x); r[c + 1] = __float_as_uint(x.y);
      }
    } else if (MODE == 2) {   // F2FP pack only: 32 per iteration
#pragma unroll
      for (int c = 0; c < 64; c += 2) r[c >> 1] ^= pack_bf16(__uint_as_float(r[c]), __uint_as_float(r[c + 1]));
    } else if (MODE == 3) {   // the exp loop of one 64-column half
#pragma unroll
      for (int c = 0; c < 64; c += 4) {
        const float2 x0 = __ffma2_rn(make_float2(__uint_as_float(r[c]), __uint_as_float(r[c + 1])), sc, nm);
        const float2 x1 = __ffma2_rn(make_float2(__uint_as_float(r[c + 2]), __uint_as_float(r[c + 3])), sc, nm);
        float2 p0, p1;
        if (POLY > 0 && (c % 16) >= 16 - POLY) {
          p0 = exp2_poly2(x0); p1 = exp2_poly2(x1);
        } else {
          p0 = make_float2(ex2f(x0.x), ex2f(x0.y)); p1 = make_float2(ex2f(x1.x), ex2f(x1.y));
        }
        acc = __fadd2_rn(acc, p0); acc2 = __fadd2_rn(acc2, p1);
        r[c >> 1] ^= pack_bf16(p0.x, p0.y);
        r[(c >> 1) + 1] ^= pack_bf16(p1.x, p1.y);
      }
    }
  }
  const long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  uint32_t s = __float_as_uint(acc.x + acc.y + acc2.x + acc2.y);
  for (int i = 0; i < 64; ++i) s ^= r[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE, int POLY>
void run(const char* name, int threads, double per_iter_per_thread, uint32_t* o, long long* c) {
  const int iters = 100;
  k<MODE, POLY><<<148, threads>>>(o, c, iters);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  const double ops = (double)threads * iters * per_iter_per_thread;
  printf("%-28s warps %2d: %7.2f /clk/SM   (%.1f clk per warp-iteration)\n", name, threads / 32, ops / h,
         (double)h / iters);
}
int main() {
  uint32_t* o; long long* c;
  cudaMalloc(&o, 148 * 1024 * 4); cudaMalloc(&c, 148 * 8);
  for (int t : {128, 256, 512}) {
    run<0, 0>("EX2 (ops)", t, 64, o, c);
    run<1, 0>("FFMA2 (instr)", t, 32, o, c);
    run<2, 0>("F2FP pack (instr)", t, 32, o, c);
    run<3, 0>("exp loop, 64 cols (cols)", t, 64, o, c);
    run<3, 4>("exp loop 25% poly (cols)", t, 64, o, c);
    run<3, 8>("exp loop 50% poly (cols)", t, 64, o, c);
  }
  return 0;
}
