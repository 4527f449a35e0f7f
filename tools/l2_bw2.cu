// l2_bw2.cu -- L2-resident bandwidth measured inside ONE launch (round 1's tools/l2_bw.cu timed
// one launch per pass, so launch overhead capped the small working sets).  Each kernel loops R
// times over a working set W with 16-byte .cg accesses (L1 bypassed), 4 independent accesses in
// flight per thread; the time of one long launch is divided by R*W.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l2_bw2 tools/l2_bw2.cu && /tmp/l2_bw2
#include <cstdio>
#include <cuda_runtime.h>

__global__ void rd(const float4* __restrict__ a, size_t n, int reps, float* out) {
  float4 acc = make_float4(0, 0, 0, 0);
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n; i += 4 * stride) {
      float4 v0 = __ldcg(a + i), v1 = __ldcg(a + i + stride), v2 = __ldcg(a + i + 2 * stride),
             v3 = __ldcg(a + i + 3 * stride);
      acc.x += v0.x + v1.x + v2.x + v3.x;
      acc.y += v0.y + v1.y + v2.y + v3.y;
    }
    for (; i < n; i += stride) acc.x += __ldcg(a + i).x;
  }
  if (acc.x + acc.y == 1234.5f) out[0] = acc.x;
}
__global__ void wr(float4* __restrict__ a, size_t n, int reps) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride)
      __stcg(a + i, make_float4(1.f, 2.f, (float)r, (float)i));
}
// ring: every pass writes slot (r % 2) and reads slot ((r+1) % 2) -- the producer / consumer
// pattern of an L2-resident V ring (W = both slots)
__global__ void ring(float4* __restrict__ a, size_t n, int reps, float* out) {
  const size_t stride = (size_t)gridDim.x * blockDim.x, half = n / 2;
  float acc = 0.f;
  for (int r = 0; r < reps; ++r) {
    float4* w = a + (r & 1) * half;
    const float4* rr = a + ((r + 1) & 1) * half;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < half; i += stride) {
      float4 v = __ldcg(rr + (half - 1 - i));
      acc += v.x;
      __stcg(w + i, make_float4(v.y, 2.f, (float)r, (float)i));
    }
  }
  if (acc == 1234.5f) out[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int l2 = 0;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  printf("SMs %d, L2 %d bytes\n", sms, l2);
  const size_t big = (size_t)4 << 30;
  float4* A;
  float* out;
  cudaMalloc(&A, big);
  cudaMalloc(&out, 4);
  cudaMemset(A, 0, big);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const size_t mb = (size_t)1 << 20;
  const size_t sizes[] = {8 * mb, 16 * mb, 24 * mb, 32 * mb, 48 * mb, 64 * mb, 80 * mb, 96 * mb, 112 * mb, big};
  for (int blocks_per_sm : {4, 8}) {
    for (size_t bytes : sizes) {
      const size_t n = bytes / 16;
      const int grid = sms * blocks_per_sm, blk = 256;
      const int reps = (int)((size_t)16 << 30) / bytes > 2000 ? 2000 : (int)(((size_t)16 << 30) / bytes);
      float ms;
      double r, w, g;
      rd<<<grid, blk>>>(A, n, 2, out);
      cudaEventRecord(e0);
      rd<<<grid, blk>>>(A, n, reps, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      r = (double)bytes * reps / (ms * 1e-3) / 1e9;
      wr<<<grid, blk>>>(A, n, 2);
      cudaEventRecord(e0);
      wr<<<grid, blk>>>(A, n, reps);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      w = (double)bytes * reps / (ms * 1e-3) / 1e9;
      ring<<<grid, blk>>>(A, n, 2, out);
      cudaEventRecord(e0);
      ring<<<grid, blk>>>(A, n, reps, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      g = (double)bytes * reps / (ms * 1e-3) / 1e9;  // half read + half written per pass
      printf("%d CTA/SM  W %7.1f MB reps %5d: read %8.1f GB/s  write %8.1f GB/s  ring(rd+wr) %8.1f GB/s\n",
             blocks_per_sm, bytes / 1e6, reps, r, w, g);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
