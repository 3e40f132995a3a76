// Fused whole-stack operator kernels for 2048 x 2048 plans (fused2.cu).
#pragma once
#include <cuda_runtime.h>

namespace bttb {

struct F2Args {
  const void* in;   // forward: model (layer-major, nx-fastest rows, n_r values per layer)
  void* out;        // forward: W[kx][j < sy] (ld sy), the station half spectrum
  const void* S;    // the plan's spectra, natural layout S[r][kx][ky]
  long long s_rstride;  // complex values per layer (Hx * lds)
  int lds;              // ky stride (Ly)
  void* ring;       // nb slots of [kx][q < ny] (ld ring_ld) complex
  long long ring_sstride;
  int ring_ld, nb;
  int* sync;        // f2_counter_ints(nz) zeroed ints: rows_done[nz], cols_done[nz], err
  const void* tw;   // exp(-2 pi i m / 2048), m < 2048, in the plan's precision
  int nz, nx, ny, sx, sy, Hx, npairs;
  long long n_r;
  int lookahead;    // layers between a layer's row items and its column items (nb >= lookahead + 1)
  long long* stats; // optional per-warp cycle accounting, F2_NSTAT per warp, or null
};
// stats buckets: [0] loads/waits, [1] row FFT, [2] row store, [3] column items,
// [4] epilogue, [5] total, [6] #rows, [7] #cols
constexpr int F2_NSTAT = 8;

int f2_counter_ints(int nz);
int f2_grid();
int f2_warps(bool fp64);
bool f2_supported(long long Lx, long long Ly, long long nx, long long ny, long long sx, long long sy, bool fp64);
template <class T> cudaError_t launch_f2(int mode, const F2Args& a, cudaStream_t st);

}  // namespace bttb
