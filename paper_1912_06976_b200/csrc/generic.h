// Generic-length operator path (generic.cu): any 2^a 3^b 5^c FFT length up to
// 65536, in particular the embeddings above the shared-memory engine's 8192.
#pragma once
#include <cuda_runtime.h>

namespace bttb {

bool generic_length_ok(long long L);
long long generic_length(long long n);  // smallest 2^a 3^b 5^c >= n (<= 65536), or -1

// radix-pass plan of one length over the plan's exp(-2 pi i t / L) table (fp64)
struct GenericFFT {
  int L = 0, np = 0;
  int radix[24] = {0};
  const double2* tw = nullptr;
  int init(int len, const double2* table);
  cudaError_t run(double2* buf, double2* tmp, long long total, long long batch, long long bs, long long es,
                  cudaStream_t st) const;
};

// per-plan context: lengths, transforms and three [Ly][Lx] complex work grids
struct GenericCtx {
  int Lx = 0, Ly = 0, Hx = 0;
  GenericFFT fx, fy;
  double2 *A = nullptr, *B = nullptr, *C = nullptr;
};

template <class S>
cudaError_t generic_build_layer(const GenericCtx& g, const double* emb, void* spectrum, cudaStream_t st);
template <class S>
cudaError_t generic_forward(const GenericCtx& g, const void* spectra, long long nl, const S* x, int nx, int ny,
                            S* d, int sx, int sy, cudaStream_t st);
template <class S>
cudaError_t generic_transpose(const GenericCtx& g, const void* spectra, long long nl, const S* d, int sx, int sy,
                              S* x, int nx, int ny, cudaStream_t st);

}  // namespace bttb
