// Internal interface of the CGLS vector kernels (cgls.cu).
#pragma once
#include <cuda_runtime.h>

namespace bttb {

// per-item CGLS scalars (fp64 for both vector dtypes)
struct CglsScalars {
  double gamma, alpha, beta, floor;  // floor = rtol^2 |s_0|^2: below it the loop freezes
};

enum { CGLS_INIT = 0, CGLS_ALPHA = 1, CGLS_BETA = 2 };

// blocks per item of the vector kernels for vectors of `len` elements
int cgls_blocks(long long len, int batch, int nsm);

// part[b*nblk + blk] = partial a_b . b_b
template <class T>
cudaError_t cgls_dot(const T* a, const T* b, long long len, int batch, int nblk, double* part, cudaStream_t st);
// r_b -= alpha_b q_b; part = partial r_b . r_b
template <class T>
cudaError_t cgls_resid(T* r, const T* q, long long len, int batch, int nblk, const CglsScalars* sc, double* part,
                       cudaStream_t st);
// phase 0: (damp2 == 0) part = s.s; (damp2 > 0) m += alpha p, s -= damp2 m, part = s.s
// phase 1: (damp2 == 0) m += alpha p, p = s + beta p; (damp2 > 0) p = s + beta p
template <class T>
cudaError_t cgls_update(T* m, T* p, T* s, long long len, int batch, int nblk, const CglsScalars* sc, double damp2,
                        double* part, int phase, cudaStream_t st);
// scalar step `op` from the partials (pb optional); hist[b*hist_ld + hist_col]
// receives the residual norm at INIT and BETA (hist optional); rtol (INIT)
// sets the freeze floor: once |s_k| <= rtol |s_0|, alpha = beta = 0
cudaError_t cgls_scalars(int op, int batch, const double* pa, int nblk_a, const double* pb, int nblk_b,
                         double damp2, double rtol, CglsScalars* sc, double* hist, int hist_ld, int hist_col,
                         cudaStream_t st);

}  // namespace bttb
