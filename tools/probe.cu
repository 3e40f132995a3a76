// Device probe: attributes, FP64/FP32 FMA rate, shared-memory and L2 bandwidth.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0000001, c = 1e-9, d = 0.5, e = 0.25, f = 0.125, g = 0.3, h = 0.7;
  for (int i = 0; i < iters; ++i) {
    a = fma(a, b, c); d = fma(d, b, c); e = fma(e, b, c); f = fma(f, b, c);
    g = fma(g, b, c); h = fma(h, b, c);
  }
  if (a + d + e + f + g + h == 12345.0) out[0] = a;
}
__global__ void ffma_loop(float* out, int iters) {
  float a = threadIdx.x * 1e-3f, b = 1.0000001f, c = 1e-9f, d = 0.5f, e = 0.25f, f = 0.125f, g = 0.3f, h = 0.7f;
  for (int i = 0; i < iters; ++i) {
    a = fmaf(a, b, c); d = fmaf(d, b, c); e = fmaf(e, b, c); f = fmaf(f, b, c);
    g = fmaf(g, b, c); h = fmaf(h, b, c);
  }
  if (a + d + e + f + g + h == 12345.0f) out[0] = a;
}
__global__ void smem_loop(double2* out, int iters) {
  extern __shared__ double2 sm[];
  int t = threadIdx.x;
  sm[t] = make_double2(t, t);
  __syncthreads();
  double2 acc = make_double2(0, 0);
  for (int i = 0; i < iters; ++i) {
    double2 v = sm[(t + i) & (blockDim.x - 1)];
    acc.x += v.x; acc.y += v.y;
    sm[(t + 3 * i) & (blockDim.x - 1)] = acc;
  }
  if (acc.x == 1.2345) out[0] = acc;
}
__global__ void copy_k(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) b[i] = a[i];
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int v;
  printf("name %s sms %d cc %d.%d l2 %d smem/sm %zu smem/block optin %zu regs/sm %d\n", p.name,
         p.multiProcessorCount, p.major, p.minor, p.l2CacheSize, p.sharedMemPerMultiprocessor,
         p.sharedMemPerBlockOptin, p.regsPerMultiprocessor);
  cudaDeviceGetAttribute(&v, cudaDevAttrClockRate, 0); printf("clock kHz %d\n", v);
  cudaDeviceGetAttribute(&v, cudaDevAttrMaxPersistingL2CacheSize, 0); printf("max persisting L2 %d\n", v);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  double* dout; cudaMalloc(&dout, 64);
  int iters = 1 << 16; int blocks = p.multiProcessorCount * 8, threads = 256;
  dfma_loop<<<blocks, threads>>>(dout, 1000); cudaDeviceSynchronize();
  cudaEventRecord(e0); dfma_loop<<<blocks, threads>>>(dout, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("FP64 FMA: %.2f TFLOP/s\n", 2.0 * 6 * iters * (double)blocks * threads / ms / 1e9);
  ffma_loop<<<blocks, threads>>>((float*)dout, 1000); cudaDeviceSynchronize();
  cudaEventRecord(e0); ffma_loop<<<blocks, threads>>>((float*)dout, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("FP32 FMA: %.2f TFLOP/s\n", 2.0 * 6 * iters * (double)blocks * threads / ms / 1e9);
  smem_loop<<<blocks, 1024, 1024 * 16>>>((double2*)dout, 1000); cudaDeviceSynchronize();
  cudaEventRecord(e0); smem_loop<<<blocks, 1024, 1024 * 16>>>((double2*)dout, 4096); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("smem 16B ld+st: %.2f TB/s (ld+st bytes)\n", 2.0 * 16 * 4096.0 * blocks * 1024 / ms / 1e9 / 1e3);
  for (size_t mb : {32, 64, 96, 2048}) {
    size_t n = mb * (1 << 20) / 16;
    double2 *a, *b; cudaMalloc(&a, n * 16); cudaMalloc(&b, n * 16);
    cudaMemset(a, 0, n * 16);
    for (int w = 0; w < 3; ++w) copy_k<<<p.multiProcessorCount * 8, 512>>>(a, b, n);
    cudaEventRecord(e0);
    for (int w = 0; w < 20; ++w) copy_k<<<p.multiProcessorCount * 8, 512>>>(a, b, n);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("copy %zu MB: %.1f GB/s (r+w)\n", mb, 2.0 * n * 16 * 20 / ms / 1e6);
    cudaFree(a); cudaFree(b);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
