#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long pk(float a, float b) { unsigned long long r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ unsigned long long add2(unsigned long long a, unsigned long long b) {
  unsigned long long d; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
template <int MODE>
__global__ void k(float* out, int iters) {
  float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0+4, a5=a0+5, a6=a0+6, a7=a0+7;
  const float b = 1.0001f, c = 0.5f;
  if (MODE == 0) {
    for (int i = 0; i < iters; ++i) {
      a0 = fmaf(a0, b, c); a1 = fmaf(a1, b, c); a2 = fmaf(a2, b, c); a3 = fmaf(a3, b, c);
      a4 = fmaf(a4, b, c); a5 = fmaf(a5, b, c); a6 = fmaf(a6, b, c); a7 = fmaf(a7, b, c);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  } else {
    unsigned long long p0 = pk(a0, a1), p1 = pk(a2, a3), p2 = pk(a4, a5), p3 = pk(a6, a7), bb = pk(b, b), cc = pk(c, c);
    for (int i = 0; i < iters; ++i) {
      p0 = fma2(p0, bb, cc); p1 = fma2(p1, bb, cc); p2 = fma2(p2, bb, cc); p3 = fma2(p3, bb, cc);
    }
    float x0, x1, x2, x3, x4, x5, x6, x7;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(x0), "=f"(x1) : "l"(p0)); asm("mov.b64 {%0,%1}, %2;" : "=f"(x2), "=f"(x3) : "l"(p1));
    asm("mov.b64 {%0,%1}, %2;" : "=f"(x4), "=f"(x5) : "l"(p2)); asm("mov.b64 {%0,%1}, %2;" : "=f"(x6), "=f"(x7) : "l"(p3));
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  }
}
int main() {
  float* o; cudaMalloc(&o, 148 * 8 * 256 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int it = 100000;
  for (int m = 0; m < 2; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (m == 0) k<0><<<148 * 8, 256>>>(o, it); else k<1><<<148 * 8, 256>>>(o, it);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 8 * it * 148.0 * 8 * 256;
      if (rep) printf("mode %d (%s): %.2f ms, %.1f TFLOP/s fp32\n", m, m ? "fma.rn.f32x2" : "fmaf", ms, flops / ms / 1e9);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
