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
// kx*ld_in + j (the column stage's natural [kx][j] layout); j < nrows.
// Output row j, column i < nout at
// out + (s/spb)*out_bstride + (s%spb)*out_sstride + j*ld_out + i.
struct RowC2RArgs {
  const void* in;
  long long in_sstride;
  int ld_in, nrows, Hx, nslabs;
  void* out;
  long long out_bstride, out_sstride;
  int spb, ld_out, nout;
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
};

// Transpose operator, column stage for one chunk of K layers:
// Wt[b][r](kx, q<nout) = IFFT_y( conj(S_r[kx]) * FFT_y(D[b][kx][0:nvalid]) ),
// stored at kx*ldw + q.
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


}  // namespace bttb
