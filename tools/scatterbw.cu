// DRAM behaviour of the transposed-intermediate access patterns (development probe).
// The row R2C writes, per CTA (row pair p of slab s), 1025 box rows of 32 bytes,
// one per kx, 16 KB apart (Y[s][kx][q], q fastest); the row C2R reads the same
// pattern; the column stages read / write whole columns (16 KB contiguous).
// Compared here with a q-blocked layout Y[s][q / QB][kx][q % QB] (QB rows of one
// kx contiguous; a group of QB/2 neighbouring row CTAs covers one contiguous
// Hx*QB*16-byte region, a column becomes 1000/QB chunks of QB*16 bytes).
// All index arithmetic is compile-time shifts so that the kernels are memory-bound.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scatterbw tools/scatterbw.cu
#include <cuda_runtime.h>
#include <cstdio>

constexpr int HX = 1025, NY = 1000, NZ = 128;

// row side: CTA (p, s) moves the [kx][2 rows] tile of row pair p.  QB = 0: linear rows
// (reference), QB = 1: the current transposed layout, QB >= 2: blocked.
template <bool WRITE, int QB>
__global__ void __launch_bounds__(128) k_row(double2* y, double* sink) {
  const int p = blockIdx.x, s = blockIdx.y, t = threadIdx.x;
  constexpr int NQB = QB >= 2 ? (NY + QB - 1) / QB : 1;
  constexpr size_t SLAB = QB >= 2 ? (size_t)NQB * HX * QB : (size_t)HX * 1024;
  double2* base = y + (size_t)s * SLAB;
  double acc = 0;
#pragma unroll 4
  for (int e = t; e < 2 * HX; e += 128) {
    const int kx = e >> 1, o = e & 1;
    size_t idx;
    if constexpr (QB == 0) idx = (size_t)p * 2 * HX + e;
    else if constexpr (QB == 1) idx = (size_t)kx * NY + 2 * p + o;
    else idx = (size_t)((2 * p) / QB) * HX * QB + (size_t)kx * QB + (2 * p) % QB + o;
    if (WRITE) __stcs(&base[idx], make_double2(e, p));
    else { double2 v = __ldcs(&base[idx]); acc += v.x + v.y; }
  }
  if (!WRITE && acc == 1.2345) *sink = acc;
}

// column side: CTA (kx, s) moves column kx of slab s (1000 values)
template <bool WRITE, int QB>
__global__ void __launch_bounds__(128) k_col(double2* y, double* sink) {
  const int kx = blockIdx.x, s = blockIdx.y, t = threadIdx.x;
  constexpr int NQB = QB >= 2 ? (NY + QB - 1) / QB : 1;
  constexpr size_t SLAB = QB >= 2 ? (size_t)NQB * HX * QB : (size_t)HX * 1024;
  double2* base = y + (size_t)s * SLAB;
  double acc = 0;
#pragma unroll 4
  for (int q = t; q < NY; q += 128) {
    size_t idx;
    if constexpr (QB <= 1) idx = (size_t)kx * NY + q;
    else idx = (size_t)(q / QB) * HX * QB + (size_t)kx * QB + q % QB;
    if (WRITE) __stcs(&base[idx], make_double2(q, kx));
    else { double2 v = __ldcs(&base[idx]); acc += v.x + v.y; }
  }
  if (!WRITE && acc == 1.2345) *sink = acc;
}

// row side, current transposed layout, R rows per CTA: box rows of R*16 bytes
template <bool WRITE, int R, int NT>
__global__ void __launch_bounds__(NT) k_rowR(double2* y, double* sink) {
  const int p = blockIdx.x, s = blockIdx.y, t = threadIdx.x;
  double2* base = y + (size_t)s * HX * 1024;
  double acc = 0;
#pragma unroll 4
  for (int e = t; e < R * HX; e += NT) {
    const int kx = e / R, o = e % R;  // compile-time power of two
    const size_t idx = (size_t)kx * NY + R * p + o;
    if (WRITE) __stcs(&base[idx], make_double2(e, p));
    else { double2 v = __ldcs(&base[idx]); acc += v.x + v.y; }
  }
  if (!WRITE && acc == 1.2345) *sink = acc;
}

template <class F> float best_of(F f) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  return best;
}

template <int QB> void run(double2* y, double* sink, const char* name) {
  const double rb = (double)NZ * 500 * 2 * HX * 16, cb = (double)NZ * HX * NY * 16;
  float a = best_of([&] { k_row<false, QB><<<dim3(500, NZ), 128>>>(y, sink); });
  float b = best_of([&] { k_row<true, QB><<<dim3(500, NZ), 128>>>(y, sink); });
  float c = best_of([&] { k_col<false, QB><<<dim3(HX, NZ), 128>>>(y, sink); });
  float d = best_of([&] { k_col<true, QB><<<dim3(HX, NZ), 128>>>(y, sink); });
  printf("%-24s row read %5.0f  row write %5.0f  col read %5.0f  col write %5.0f GB/s\n", name, rb / a / 1e6, rb / b / 1e6,
         cb / c / 1e6, cb / d / 1e6);
}

int main() {
  const size_t n = (size_t)NZ * (HX + 8) * 1152;
  double2* y; double* sink;
  cudaMalloc(&y, n * sizeof(double2)); cudaMalloc(&sink, 8);
  cudaMemset(y, 0, n * sizeof(double2));
  run<0>(y, sink, "linear rows (reference)");
  run<1>(y, sink, "transposed (current)");
  run<2>(y, sink, "blocked QB=2");
  run<8>(y, sink, "blocked QB=8");
  run<32>(y, sink, "blocked QB=32");
  run<128>(y, sink, "blocked QB=128");
  {
    const double rb = (double)NZ * 500 * 2 * HX * 16;
#define ROWR(R, NT) { float a = best_of([&] { k_rowR<false, R, NT><<<dim3(NY / R, NZ), NT>>>(y, sink); }); \
    float b = best_of([&] { k_rowR<true, R, NT><<<dim3(NY / R, NZ), NT>>>(y, sink); }); \
    printf("tile [kx][%2d rows] %3d thr  row read %5.0f  row write %5.0f GB/s\n", R, NT, rb / a / 1e6, rb / b / 1e6); }
    ROWR(2, 128) ROWR(4, 128) ROWR(4, 256) ROWR(8, 128) ROWR(8, 256) ROWR(8, 512)
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
