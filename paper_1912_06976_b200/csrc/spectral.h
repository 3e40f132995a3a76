// Internal interface of the spectral (FFT-domain) kernels (spectral.cu).
#pragma once
#include <cuda_runtime.h>

#include "fft.cuh"

namespace bttb {

// Real rows -> transposed half spectra.  Slab s, row q, column i of the input
// lives at in + (s/spb)*in_bstride + (s%spb)*in_sstride + q*ld_in + i (i < nvalid,
// zero beyond).  Output (s, kx, q) at out + s*out_sstride + kx*ld_out + q.
struct RowR2CArgs {
  const void* in;
  long long in_bstride, in_sstride;
  int spb, ld_in, nrows, nvalid, nslabs;
  void* out;
  long long out_sstride;
  int ld_out, Hx;
};

// Half spectra -> real rows.  Input (s, kx, j) at in + s*in_sstride +
// kx*ld_in + j (rowmajor = 0, the column stage's natural [kx][j] layout) or
// in + s*in_sstride + j*ld_in + kx (rowmajor = 1, contiguous rows); j < nrows.
// Output row j, column i < nout at
// out + (s/spb)*out_bstride + (s%spb)*out_sstride + j*ld_out + i.
struct RowC2RArgs {
  const void* in;
  long long in_sstride;
  int ld_in, nrows, Hx, nslabs;
  void* out;
  long long out_bstride, out_sstride;
  int spb, ld_out, nout;
  int rowmajor;
  // per-pass twiddle tables of the 8/16/16 radix order at L = 2048 (the
  // mirrored first pass of k_row_c2r_mirror), or null
  const void* tw_816;
};

// Forward operator, column stage for one chunk of K layers:
// W[b][kx][j<nout] (+)= IFFT_y( sum_r S_r[kx] * FFT_y(Y[b][r][kx][0:nvalid]) ).
struct ColFwdArgs {
  const void* Y;
  long long y_bstride, y_rstride;
  int ldy, nvalid;
  const void* S;
  long long s_rstride;
  int lds, K;
  void* W;
  long long w_bstride;
  int ldw, nout, accumulate, Hx, nbatch;
  int ahead;  // > 0: L2-prefetch the Y and S columns of layer r + ahead (TMA kernels)
};

// Transpose operator, column stage for one chunk of K layers:
// Wt[b][r](kx, q<nout) = IFFT_y( conj(S_r[kx]) * FFT_y(D[b][kx][0:nvalid]) ),
// stored at kx*ldw + q (rowmajor = 0) or q*ldw + kx (rowmajor = 1: the C2R
// row pass then reads contiguous rows; the transposition is paid by stores).
struct ColTraArgs {
  const void* D;
  long long d_bstride;
  int ldd, nvalid;
  const void* S;
  long long s_rstride;
  int lds, K;
  void* W;
  long long w_bstride, w_rstride;
  int ldw, nout, Hx, nbatch;
  int rowmajor;
  int ahead;  // > 0: L2-prefetch the S column of layer r + ahead (TMA kernels)
};

// Spectrum build, column stage: S[kx][ky] = scale * FFT_y(Y[kx][0:Ly]) (fp64 FFT,
// stored as T).
struct ColSpecArgs {
  const void* Y;
  int ldy;
  void* S;
  int lds, Hx;
  double scale;
};

template <class T> cudaError_t launch_row_r2c(const RowR2CArgs& a, const FFTDesc<T>& d, int E, cudaStream_t st);
template <class T> cudaError_t launch_row_c2r(const RowC2RArgs& a, const FFTDesc<T>& d, int E, cudaStream_t st);
template <class T> cudaError_t launch_col_fwd(const ColFwdArgs& a, const FFTDesc<T>& d, int E, cudaStream_t st);
template <class T> cudaError_t launch_col_tra(const ColTraArgs& a, const FFTDesc<T>& d, int E, cudaStream_t st);
template <class TS> cudaError_t launch_col_spec(const ColSpecArgs& a, const FFTDesc<double>& d, int E, cudaStream_t st);

// radix sequence of the registered compile-time plan of (L, dtype), 0 if none
int static_radices(int L, bool fp64, int* out);

// Fused layer pipeline (pipeline.cuh): one persistent cooperative kernel per
// application and vector.  Forward: in = model (layer-major, rows of nx, n_r
// per layer), out = W[kx][j < sy] (the column-inverse-transformed station
// half spectrum; a row C2R pass finishes it).  Transpose: in = D[kx][j < sy]
// (row R2C of the data), out = model.  ring: nb >= 2 slots [kx][q < ny] of
// ring_sstride complex; sync: pipe_counter_ints(nz) zeroed ints.
struct PipeArgs {
  const void* in;
  void* out;
  const void* S;
  long long s_rstride;
  int lds;
  void* ring;
  long long ring_sstride;
  int nb;
  int* sync;
  int nz, nx, ny, sy, Hx;
  long long n_r;
  long long* stats;  // optional per-team cycle accounting (6 x teams x grid), or null
};
int pipe_grid();   // CTAs of the pipeline kernels (one per SM)
int pipe_teams();  // teams per CTA
int pipe_counter_ints(int nz);  // ints of PipeArgs::sync (the err flag is the last)
// true if the fused pipeline runs this length (square plans only) and dtype
template <class T> bool pipe_supported(int L, int Hx);
template <class T> cudaError_t launch_pipe(int mode, const PipeArgs& a, const FFTDesc<T>& d, cudaStream_t st);

}  // namespace bttb
