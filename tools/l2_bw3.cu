// l2_bw3.cu -- is the ~7.6 TB/s L2-resident write ceiling (tools/l2_bw2.cu) per SM or per L2?
// Writes / reads from a subset of the SMs, and TMA bulk stores (cp.async.bulk.global.shared::cta)
// against st.global.cg, all in one long launch over an L2-resident working set.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2_bw3.bin tools/l2_bw3.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void wr(float4* __restrict__ a, size_t n, int reps) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride)
      __stcg(a + i, make_float4(1.f, 2.f, (float)r, (float)i));
}
__global__ void rd(const float4* __restrict__ a, size_t n, int reps, float* out) {
  float acc = 0.f;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n; i += 4 * stride) {
      float4 v0 = __ldcg(a + i), v1 = __ldcg(a + i + stride), v2 = __ldcg(a + i + 2 * stride),
             v3 = __ldcg(a + i + 3 * stride);
      acc += v0.x + v1.y + v2.z + v3.w;
    }
  }
  if (acc == 1234.5f) out[0] = acc;
}
// one thread per CTA streams 16 KB chunks from shared memory with bulk stores, up to 8 in flight
__global__ void wr_bulk(char* __restrict__ a, size_t bytes, int reps) {
  extern __shared__ __align__(128) char sm[];
  for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = (float)i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint32_t src = (uint32_t)__cvta_generic_to_shared(sm);
  const size_t chunks = bytes / 16384;
  for (int r = 0; r < reps; ++r) {
    for (size_t c = blockIdx.x; c < chunks; c += gridDim.x) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 16384;" ::"l"(a + c * 16384), "r"(src)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 8;" ::: "memory");
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  char* A;
  float* out;
  const size_t big = (size_t)1 << 30;
  cudaMalloc(&A, big);
  cudaMalloc(&out, 4);
  cudaMemset(A, 0, big);
  cudaFuncSetAttribute(wr_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const size_t W = (size_t)48 << 20;
  const int reps = 300;
  auto time = [&](auto f) {
    f(2);
    cudaEventRecord(e0);
    f(reps);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return (double)W * reps / (ms * 1e-3) / 1e9;
  };
  for (int nsm : {16, 37, 74, 111, 148}) {
    const double w4 = time([&](int r) { wr<<<nsm * 4, 256>>>((float4*)A, W / 16, r); });
    const double r4 = time([&](int r) { rd<<<nsm * 4, 256>>>((const float4*)A, W / 16, r, out); });
    const double b1 = time([&](int r) { wr_bulk<<<nsm, 32, 16384>>>(A, W, r); });
    const double b4 = time([&](int r) { wr_bulk<<<nsm * 4, 32, 16384>>>(A, W, r); });
    printf("SMs %3d: st.global.cg %8.1f GB/s (%5.1f B/clk/SM)  ld.cg %8.1f GB/s  bulk-store 1 CTA/SM %8.1f  4 CTA/SM %8.1f GB/s\n",
           nsm, w4, w4 * 1e9 / nsm / 1.965e9, r4, b1, b4);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
