// l2_bw.cu -- microbenchmark: L2-resident read / write / copy bandwidth vs HBM on one GPU,
// and the effect of discard.global.L2 on write-back traffic.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l2_bw tools/l2_bw.cu && /tmp/l2_bw
#include <cstdio>
#include <cuda_runtime.h>

__global__ void rd(const float4* __restrict__ a, size_t n, float* out) {
  float4 acc = make_float4(0, 0, 0, 0);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float4 v = __ldcg(a + i);
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
  }
  if (acc.x + acc.y + acc.z + acc.w == 1234.5f) out[0] = acc.x;
}
__global__ void wr(float4* __restrict__ a, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcg(a + i, make_float4(1.f, 2.f, 3.f, (float)i));
}
__global__ void cp(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcg(b + i, __ldcg(a + i));
}
// read then discard each 128-byte line (one lane per line)
__global__ void rd_discard(const float4* __restrict__ a, size_t n, float* out) {
  float4 acc = make_float4(0, 0, 0, 0);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float4 v = __ldcg(a + i);
    acc.x += v.x;
    if ((i & 7) == 0) asm volatile("discard.global.L2 [%0], 128;" ::"l"(a + i) : "memory");
  }
  if (acc.x == 1234.5f) out[0] = acc.x;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t big = (size_t)4 << 30;  // 4 GiB (HBM)
  float4 *A, *B;
  float* out;
  cudaMalloc(&A, big);
  cudaMalloc(&B, big);
  cudaMalloc(&out, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const size_t sizes[] = {(size_t)16 << 20, (size_t)32 << 20, (size_t)48 << 20, (size_t)64 << 20,
                          (size_t)96 << 20, big};
  for (size_t bytes : sizes) {
    const size_t n = bytes / 16;
    const int grid = sms * 8, blk = 512;
    const int reps = bytes > ((size_t)1 << 30) ? 3 : 50;
    float ms;
    double r, w, c;
    rd<<<grid, blk>>>(A, n, out);
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) rd<<<grid, blk>>>(A, n, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    r = (double)bytes * reps / (ms * 1e-3) / 1e9;
    wr<<<grid, blk>>>(A, n);
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) wr<<<grid, blk>>>(A, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    w = (double)bytes * reps / (ms * 1e-3) / 1e9;
    const size_t half = n / 2;
    cp<<<grid, blk>>>(A, A + half, half);
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) cp<<<grid, blk>>>(A, A + half, half);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    c = (double)bytes * reps / (ms * 1e-3) / 1e9;
    printf("working set %8.1f MB: read %8.1f GB/s  write %8.1f GB/s  copy(rd+wr) %8.1f GB/s\n", bytes / 1e6, r, w, c);
  }
  // producer / consumer through L2: write 32 MB, read it back (+ discard), repeat
  for (int disc = 0; disc < 2; ++disc) {
    const size_t bytes = (size_t)32 << 20, n = bytes / 16;
    float ms;
    cudaEventRecord(e0);
    for (int i = 0; i < 50; ++i) {
      float4* buf = A + (size_t)(i % 64) * n;  // march through 2 GiB so nothing is reused
      wr<<<sms * 8, 512>>>(buf, n);
      if (disc) rd_discard<<<sms * 8, 512>>>(buf, n, out);
      else rd<<<sms * 8, 512>>>(buf, n, out);
    }
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("write+read 32 MB chunks (%s): %8.1f GB/s of write+read traffic\n", disc ? "discard after read" : "plain",
           (double)bytes * 2 * 50 / (ms * 1e-3) / 1e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
