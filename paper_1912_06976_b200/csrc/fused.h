// Fused whole-stack operator kernels for 2048 x 2048 FFT lengths (fused.cu).
//
// One persistent cooperative kernel per application runs BOTH the row
// transforms and the column stages of every depth layer; the per-layer
// transposed intermediate [kx][q] lives in an L2-resident ring of a few layer
// slots instead of a 2.1 GB HBM round trip, and the per-column state (the
// forward's spectral accumulator, the transpose's data spectrum) lives in
// tensor memory.  Every 2048-point transform of the path has either half its
// input zero (n < 1024) or only half its output used, so each runs as two
// independent 1024-point transforms -- the even and odd frequency halves --
// on the two warps of a warp pair (warp FFT: 32 elements per lane, one
// shared-memory exchange, warp-level synchronisation only).
//
// Spectrum layout of a fused plan ("ky-split"): S'[r][kx][p][k] = S_r[kx][2k+p],
// p in {0, 1}, k < 1024 -- each warp's half is contiguous and lands in its
// lanes in the order the warp FFT produces it.
#pragma once
#include <cuda_runtime.h>

namespace bttb {

struct FusedArgs {
  const void* in;   // forward: model (layer-major, rows of nx, n_r per layer); transpose: D[kx][j < sy] (ld sy)
  void* out;        // forward: W[kx][j < sy] (ld sy); transpose: model
  const void* S;    // ky-split spectra of the plan's layers
  long long s_rstride;  // complex values per layer (Hx * 2048)
  void* ring;       // nb slots of [kx][q < ny] (ld ring_ld) complex
  long long ring_sstride;
  int ring_ld, nb;
  int* sync;        // fused_counter_ints(nz) zeroed ints: rows_done, cols_done, row_next, err
  const void* tw;   // exp(-2 pi i n / 2048), n < 2048, in the plan's precision
  int nz, nx, ny, sx, sy, Hx, npairs;
  long long n_r;
  int lookahead;    // layers between a layer's row items and its column items (nb = lookahead + 1)
  long long* stats; // optional per-warp cycle accounting (development aid), FZ_NSTAT per warp, or null
};
constexpr int FZ_NSTAT = 8;  // [0] wait, [1] grab, [2] row items, [3] col items, [4] epilogue/prologue, [5] total, [6] #rows, [7] #cols

int fused_counter_ints(int nz);
int fused_grid();  // CTAs (one per SM)
int fused_warps(bool fp64);  // warps per CTA
// true if the fused kernels run this geometry: Lx = Ly = 2048, rows / stations
// <= 1024 along both axes, columns fit the tensor memory of the grid
bool fused_supported(long long Lx, long long Ly, long long nx, long long ny, long long sx, long long sy);
template <class T> cudaError_t launch_fused(int mode, const FusedArgs& a, cudaStream_t st);
// ky-split permutation of nl layers of (Hx, 2048) spectra, in place (dir = +1 split, -1 merge)
template <class T> cudaError_t launch_ky_split(void* S, long long nrows, int dir, cudaStream_t st);

}  // namespace bttb
