// Pure-read / pure-write / copy HBM bandwidth probe (development tool): the
// column stages of the operator are read-dominated (forward: reads only), so
// their ceiling is the read bandwidth, not the copy peak of MEASURED_PEAKS.json.
#include <cuda_runtime.h>

#include <cstdio>

__global__ void k_read(const double2* __restrict__ a, size_t n, double* sink) {
  double acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double2 v = __ldcs(a + i);
    acc += v.x + v.y;
  }
  if (acc == 1.2345) *sink = acc;
}
__global__ void k_write(double2* __restrict__ a, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcs(a + i, make_double2(1, 2));
}
__global__ void k_copy(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcs(b + i, __ldcs(a + i));
}

int main() {
  const size_t bytes = (size_t)4 << 30, n = bytes / 16;
  double2 *a, *b;
  double* sink;
  cudaMalloc(&a, bytes);
  cudaMalloc(&b, bytes);
  cudaMalloc(&sink, 8);
  cudaMemset(a, 0, bytes);
  cudaMemset(b, 0, bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  for (int blocks_per_sm : {4, 8, 16}) {
    const int grid = nsm * blocks_per_sm, blk = 256;
    float ms;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      k_read<<<grid, blk>>>(a, n, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("blocks/SM %2d  read  %.0f GB/s\n", blocks_per_sm, bytes / ms / 1e6);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      k_write<<<grid, blk>>>(b, n);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("blocks/SM %2d  write %.0f GB/s\n", blocks_per_sm, bytes / ms / 1e6);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      k_copy<<<grid, blk>>>(a, b, n);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("blocks/SM %2d  copy  %.0f GB/s (read+write)\n", blocks_per_sm, 2 * bytes / ms / 1e6);
  }
  return 0;
}
