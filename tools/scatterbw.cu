// DRAM behaviour of the transposed-intermediate access patterns (development probe).
// The row R2C writes, per CTA (row pair p of slab s), 1025 box rows of 32 bytes,
// one per kx, 16 KB apart (Y[s][kx][q], q fastest); the row C2R reads the same
// pattern.  Compare with a q-blocked layout Y[s][q / QB][kx][q % QB] in which a
// group of QB/2 neighbouring CTAs covers one contiguous Hx*QB*16-byte region.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scatterbw tools/scatterbw.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

constexpr int HX = 1025, NY = 1000, NZ = 128;

// mode 0: linear rows (each CTA streams 32.8 KB contiguous); 1: current transposed; 2: blocked QB
// [kx][R rows] tiles: one CTA per group of R rows, R*16-byte box rows
template <bool WRITE>
__global__ void __launch_bounds__(128) kr(double2* y, int R, double* sink) {
  const int p = blockIdx.x, s = blockIdx.y, t = threadIdx.x;
  double2* base = y + (size_t)s * HX * NY;
  double acc = 0;
  for (int e = t; e < R * HX; e += 128) {
    const int kx = e / R, o = e % R;
    const size_t idx = (size_t)kx * NY + R * p + o;
    if (R * p + o < NY) {
      if (WRITE) __stcs(&base[idx], make_double2(e, p));
      else { double2 v = __ldcs(&base[idx]); acc += v.x + v.y; }
    }
  }
  if (!WRITE && acc == 1.2345) *sink = acc;
}

template <bool WRITE>
__global__ void __launch_bounds__(128) k(double2* y, int mode, int QB, double* sink) {
  const int p = blockIdx.x, s = blockIdx.y, t = threadIdx.x;
  const int nqb = (NY + QB - 1) / QB;
  const size_t slab = mode == 2 ? (size_t)nqb * HX * QB : (size_t)HX * NY;
  double2* base = y + (size_t)s * slab;
  double acc = 0;
  for (int i = 0; i < (2 * HX + 127) / 128; ++i) {
    const int e = t + 128 * i;  // element of the [kx][2] tile
    if (e >= 2 * HX) break;
    const int kx = e >> 1, o = e & 1;
    size_t idx;
    if (mode == 0) idx = (size_t)p * 2 * HX + e;
    else if (mode == 1) idx = (size_t)kx * NY + 2 * p + o;
    else idx = (size_t)((2 * p) / QB) * HX * QB + (size_t)kx * QB + (2 * p) % QB + o;
    if (WRITE) __stcs(&base[idx], make_double2(e, p));
    else { double2 v = __ldcs(&base[idx]); acc += v.x + v.y; }
  }
  if (!WRITE && acc == 1.2345) *sink = acc;
}

int main() {
  const size_t n = (size_t)NZ * (HX + 1) * 1024;
  double2* y; double* sink;
  cudaMalloc(&y, n * sizeof(double2)); cudaMalloc(&sink, 8);
  cudaMemset(y, 0, n * sizeof(double2));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const double bytes = (double)NZ * 500 * 2 * HX * 16;
  struct { int mode, qb; const char* name; } cases[] = {{0, 2, "linear"}, {1, 2, "transposed (current)"},
      {2, 8, "blocked QB=8"}, {2, 16, "blocked QB=16"}, {2, 32, "blocked QB=32"}, {2, 64, "blocked QB=64"}, {2, 128, "blocked QB=128"}};
  for (auto c : cases) for (int w = 0; w < 2; ++w) {
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      if (w) k<true><<<dim3(500, NZ), 128>>>(y, c.mode, c.qb, sink);
      else k<false><<<dim3(500, NZ), 128>>>(y, c.mode, c.qb, sink);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("%-22s %s %.3f ms  %.0f GB/s\n", c.name, w ? "write" : "read ", best, bytes / best / 1e6);
  }
  for (int R : {2, 4, 8, 16, 32}) for (int w = 0; w < 2; ++w) {
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      if (w) kr<true><<<dim3((NY + R - 1) / R, NZ), 128>>>(y, R, sink);
      else kr<false><<<dim3((NY + R - 1) / R, NZ), 128>>>(y, R, sink);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("tile [kx][%2d rows]      %s %.3f ms  %.0f GB/s\n", R, w ? "write" : "read ", best, bytes / best / 1e6);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
