// Hardware probe (development tool, not product code): the rates that bound
// the fused FFT operator on this B200.
//  * L2-resident read / write / read+write bandwidth vs working-set size
//    (is an L2-resident intermediate cheaper than an HBM round trip?)
//  * FP64 / FP32 add and FMA instruction throughput (the FFT engine's pipe)
//  * shared-memory 8/16-byte load bandwidth and warp-shuffle throughput
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/hwprobe tools/hwprobe.cu
#include <cuda_runtime.h>

#include <cstdio>

__global__ void k_read(const double2* __restrict__ a, size_t n, int reps, double* sink) {
  double acc = 0;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      double2 v = a[i];
      acc += v.x + v.y;
    }
  if (acc == 1.2345) *sink = acc;
}
__global__ void k_write(double2* __restrict__ a, size_t n, int reps) {
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
      a[i] = make_double2(r, 2);
}
// write then read back a different thread's element (forces the L2 round trip)
__global__ void k_rw(double2* __restrict__ a, size_t n, int reps, double* sink) {
  double acc = 0;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      double2 v = a[(i + 4096) % n];
      acc += v.x;
      a[i] = make_double2(acc, v.y);
    }
  if (acc == 1.2345) *sink = acc;
}

template <class T, int OP>
__global__ void k_alu(T* sink, int iters, T seed) {
  T a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = seed + (T)(threadIdx.x + k);
  const T b = (T)1.0000001, c = (T)1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (OP == 0) a[k] = a[k] + c;
      else a[k] = a[k] * b + c;
    }
  }
  T s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == (T)1.2345) *sink = s;
}

template <class T>
__global__ void k_smem(double* sink, int iters) {
  __shared__ T buf[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = T();
  __syncthreads();
  T acc = T();
  int idx = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      T v = buf[(idx + k * 128) & 2047];
      if constexpr (sizeof(T) == 8) acc += v; else { acc.x += v.x; acc.y += v.y; }
    }
    idx = (idx + 1) & 2047;
  }
  double s;
  if constexpr (sizeof(T) == 8) s = acc; else s = acc.x + acc.y;
  if (s == 1.2345) *sink = s;
}

__global__ void k_shfl(double* sink, int iters) {
  double v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = threadIdx.x + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __shfl_xor_sync(0xffffffffu, v[k], (k + 1) & 31);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += v[k];
  if (s == 1.2345) *sink = s;
}

int main() {
  int nsm = 148, clk = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  int l2 = 0;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  printf("SMs %d, clock %d kHz, L2 %d MB\n", nsm, clk, l2 >> 20);
  double* sink;
  cudaMalloc(&sink, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  const size_t maxb = (size_t)1 << 30;
  double2* a;
  cudaMalloc(&a, maxb);
  cudaMemset(a, 0, maxb);
  const int grid = nsm * 8, blk = 256;
  for (size_t mb : {4, 8, 16, 24, 32, 48, 64, 96, 128, 1024}) {
    const size_t n = (mb << 20) / 16;
    const int reps = mb >= 512 ? 2 : (int)(4096 / mb);
    double best[3] = {1e30, 1e30, 1e30};
    for (int trial = 0; trial < 3; ++trial) {
      k_read<<<grid, blk>>>(a, n, 1, sink);
      cudaEventRecord(e0);
      k_read<<<grid, blk>>>(a, n, reps, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      best[0] = ms < best[0] ? ms : best[0];
      cudaEventRecord(e0);
      k_write<<<grid, blk>>>(a, n, reps);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      best[1] = ms < best[1] ? ms : best[1];
      cudaEventRecord(e0);
      k_rw<<<grid, blk>>>(a, n, reps, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      best[2] = ms < best[2] ? ms : best[2];
    }
    const double bytes = (double)n * 16 * reps;
    printf("ws %5zu MB: read %7.1f GB/s  write %7.1f GB/s  read+write %7.1f GB/s\n", mb, bytes / best[0] / 1e6,
           bytes / best[1] / 1e6, 2 * bytes / best[2] / 1e6);
  }
  // ALU throughput: grid of 148*8 CTAs x 256 threads, 8 independent chains
  const int iters = 20000;
  auto alu = [&](auto kern, const char* name) {
    kern<<<nsm * 8, 256>>>(nullptr, 10, 1);
    cudaEventRecord(e0);
    kern<<<nsm * 8, 256>>>(nullptr, iters, 1);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = (double)nsm * 8 * 256 * iters * 8;
    printf("%-10s %8.2f Tinstr/s  (%.1f thread-instr/clk/SM at %d MHz)\n", name, ops / ms / 1e9,
           ops / (ms * 1e-3) / nsm / (clk * 1e3), clk / 1000);
  };
  alu(k_alu<double, 0>, "DADD");
  alu(k_alu<double, 1>, "DFMA");
  alu(k_alu<float, 0>, "FADD");
  alu(k_alu<float, 1>, "FFMA");
  {
    k_smem<double><<<nsm * 4, 256>>>(sink, 10);
    cudaEventRecord(e0);
    k_smem<double><<<nsm * 4, 256>>>(sink, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double b = (double)nsm * 4 * 256 * iters * 8 * 8;
    printf("LDS.64     %8.1f B/clk/SM\n", b / (ms * 1e-3) / nsm / (clk * 1e3));
    k_smem<double2><<<nsm * 4, 256>>>(sink, 10);
    cudaEventRecord(e0);
    k_smem<double2><<<nsm * 4, 256>>>(sink, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    b = (double)nsm * 4 * 256 * iters * 8 * 16;
    printf("LDS.128    %8.1f B/clk/SM\n", b / (ms * 1e-3) / nsm / (clk * 1e3));
    k_shfl<<<nsm * 4, 256>>>(sink, 10);
    cudaEventRecord(e0);
    k_shfl<<<nsm * 4, 256>>>(sink, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    b = (double)nsm * 4 * 256 * iters * 8;
    printf("SHFL(f64)  %8.1f doubles/clk/SM (2 SHFL.32 each)\n", b / (ms * 1e-3) / nsm / (clk * 1e3));
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
