// Spectral kernels of the fast operator: row R2C / C2R passes (x axis, the
// contiguous axis of model and data vectors) and the fused column stages (y
// axis) that multiply by the cached per-layer spectra.
//
// Reference semantics: /root/reference/pkg/src/bttb/multiply.py:37-57 and
// transform.py:97-102.  Differences of formulation (same operator):
//  * FFT length L >= s+n-1 instead of exactly s+n-1 (zero gap);
//  * half spectra along x (real data), transposed [kx][y] intermediates;
//  * forward: spectra of a chunk of layers are summed before ONE inverse
//    column FFT per chunk (multiply.py:42-45 does one per layer);
//  * transpose spectrum = conj(forward spectrum) (transform.py:75-82,102).
#include <cuda_runtime.h>

#include "spectral.h"

namespace bttb {

namespace {

constexpr int kMaxThreads = 1024;

template <class T> struct Prec;
template <> struct Prec<double> { static constexpr int pairs = 4; static constexpr int cols_threads = 256; };
template <> struct Prec<float> { static constexpr int pairs = 8; static constexpr int cols_threads = 256; };

__host__ __device__ inline int team_stride(int L) { return L + 1; }  // +1 element staggers teams across banks

template <class K>
cudaError_t set_smem(K kernel, size_t bytes) {
  if (bytes > 48 * 1024) return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  return cudaSuccess;
}

}  // namespace

// ---------------------------------------------------------------------------
// Row pass, real -> half spectrum, two rows per complex FFT
// ---------------------------------------------------------------------------
template <class T, int E>
__global__ void k_row_r2c(RowR2CArgs a, FFTDesc<T> d, int P) {
  using V = cplx<T>;
  extern __shared__ __align__(16) unsigned char smraw[];
  V* smb = reinterpret_cast<V*>(smraw);
  const int L = d.L, nt = d.nt, Ls = team_stride(L);
  const int tid = threadIdx.x, c = tid / nt, t = tid - c * nt;
  const int s = blockIdx.y;
  const int q0 = blockIdx.x * 2 * P;
  const int qa = q0 + 2 * c, qb = qa + 1;
  const T* in = static_cast<const T*>(a.in) + (long long)(s / a.spb) * a.in_bstride +
                (long long)(s % a.spb) * a.in_sstride;
  const bool va = (c < P) && qa < a.nrows, vb = (c < P) && qb < a.nrows;
  const T* ra = in + (long long)(va ? qa : 0) * a.ld_in;
  const T* rb = in + (long long)(vb ? qb : 0) * a.ld_in;
  V v[E];
#pragma unroll
  for (int k = 0; k < E; ++k) {
    const int i = t + nt * k;
    const bool inb = i < a.nvalid;
    v[k] = mkc<V>(va && inb ? ra[i] : T(0), vb && inb ? rb[i] : T(0));
  }
  V* sm = smb + (long long)c * Ls;
  team_fft<T, E>(v, sm, t, d);
  __syncthreads();
#pragma unroll
  for (int k = 0; k < E; ++k) sm[t + nt * k] = v[k];
  __syncthreads();
  // separate the two real transforms and store transposed: out[s][kx][q]
  V* out = static_cast<V*>(a.out) + (long long)s * a.out_sstride;
  const int nitems = a.Hx * P;
  for (int it = tid; it < nitems; it += blockDim.x) {
    const int kx = it / P, cc = it - kx * P;
    const int q = q0 + 2 * cc;
    const V* z = smb + (long long)cc * Ls;
    const V zk = z[kx];
    const V zm = z[kx == 0 ? 0 : L - kx];
    const T h = T(0.5);
    V* o = out + (long long)kx * a.ld_out + q;
    if (q < a.nrows) o[0] = mkc<V>(h * (zk.x + zm.x), h * (zk.y - zm.y));
    if (q + 1 < a.nrows) o[1] = mkc<V>(h * (zk.y + zm.y), h * (zm.x - zk.x));
  }
}

// ---------------------------------------------------------------------------
// Row pass, half spectrum -> real rows (two rows per complex inverse FFT)
// ---------------------------------------------------------------------------
template <class T, int E>
__global__ void k_row_c2r(RowC2RArgs a, FFTDesc<T> d, int P) {
  using V = cplx<T>;
  extern __shared__ __align__(16) unsigned char smraw[];
  V* smb = reinterpret_cast<V*>(smraw);
  const int L = d.L, nt = d.nt, Ls = team_stride(L);
  const int tid = threadIdx.x, c = tid / nt, t = tid - c * nt;
  const int s = blockIdx.y;
  const int j0 = blockIdx.x * 2 * P;
  const V* in = static_cast<const V*>(a.in) + (long long)s * a.in_sstride;
  const int nitems = a.Hx * P;
  for (int it = tid; it < nitems; it += blockDim.x) {
    const int kx = it / P, cc = it - kx * P;
    const int j = j0 + 2 * cc;
    const V* p = in + (long long)kx * a.ld_in + j;
    V A = j < a.nrows ? p[0] : mkc<V>(T(0), T(0));
    V B = j + 1 < a.nrows ? p[1] : mkc<V>(T(0), T(0));
    if (kx == 0 || 2 * kx == L) {  // Hermitian projection (.real semantics)
      A.y = T(0);
      B.y = T(0);
    }
    V* z = smb + (long long)cc * Ls;
    z[kx] = mkc<V>(A.x - B.y, A.y + B.x);
    if (kx >= 1 && kx <= L - a.Hx) z[L - kx] = mkc<V>(A.x + B.y, B.x - A.y);
  }
  __syncthreads();
  V* sm = smb + (long long)c * Ls;
  V v[E];
#pragma unroll
  for (int k = 0; k < E; ++k) v[k] = conjv(sm[t + nt * k]);
  team_fft<T, E>(v, sm, t, d);
  const int ja = j0 + 2 * c, jb = ja + 1;
  const bool va = (c < P) && ja < a.nrows, vb = (c < P) && jb < a.nrows;
  T* out = static_cast<T*>(a.out) + (long long)(s / a.spb) * a.out_bstride + (long long)(s % a.spb) * a.out_sstride;
  T* oa = out + (long long)(va ? ja : 0) * a.ld_out;
  T* ob = out + (long long)(vb ? jb : 0) * a.ld_out;
#pragma unroll
  for (int k = 0; k < E; ++k) {
    const int i = t + nt * k;
    if (i < a.nout) {
      if (va) oa[i] = v[k].x;
      if (vb) ob[i] = -v[k].y;
    }
  }
}

// ---------------------------------------------------------------------------
// Forward column stage: FFT along y, multiply by cached spectrum, accumulate
// over the chunk's layers in registers, one inverse FFT, extract stations.
// ---------------------------------------------------------------------------
template <class T, int E>
__global__ void k_col_fwd(ColFwdArgs a, FFTDesc<T> d, int C) {
  using V = cplx<T>;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int L = d.L, nt = d.nt, Ls = team_stride(L);
  const int tid = threadIdx.x, c = tid / nt, t = tid - c * nt;
  const int kx = blockIdx.x * C + c;
  const bool kv = (c < C) && kx < a.Hx;
  const int kxc = kv ? kx : 0;
  const int b = blockIdx.y;
  V* sm = reinterpret_cast<V*>(smraw) + (long long)c * Ls;
  V acc[E], v[E];
#pragma unroll
  for (int k = 0; k < E; ++k) acc[k] = mkc<V>(T(0), T(0));
  const V* Yb = static_cast<const V*>(a.Y) + (long long)b * a.y_bstride + (long long)kxc * a.ldy;
  const V* Sb = static_cast<const V*>(a.S) + (long long)kxc * a.lds;
  for (int r = 0; r < a.K; ++r) {
    const V* yc = Yb + (long long)r * a.y_rstride;
#pragma unroll
    for (int k = 0; k < E; ++k) {
      const int q = t + nt * k;
      v[k] = q < a.nvalid ? yc[q] : mkc<V>(T(0), T(0));
    }
    team_fft<T, E>(v, sm, t, d);
    const V* sc = Sb + (long long)r * a.s_rstride;
#pragma unroll
    for (int k = 0; k < E; ++k) {
      const V w = __ldg(&sc[t + nt * k]);
      acc[k].x += w.x * v[k].x - w.y * v[k].y;
      acc[k].y += w.x * v[k].y + w.y * v[k].x;
    }
  }
#pragma unroll
  for (int k = 0; k < E; ++k) acc[k] = conjv(acc[k]);
  team_fft<T, E>(acc, sm, t, d);
  if (kv) {
    V* wc = static_cast<V*>(a.W) + (long long)b * a.w_bstride + (long long)kx * a.ldw;
#pragma unroll
    for (int k = 0; k < E; ++k) {
      const int j = t + nt * k;
      if (j < a.nout) {
        V val = conjv(acc[k]);
        if (a.accumulate) val = val + wc[j];
        wc[j] = val;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Transpose column stage: FFT of the data column once, then per layer
// conj(spectrum) multiply and inverse FFT, extract prism rows.
// ---------------------------------------------------------------------------
template <class T, int E>
__global__ void k_col_tra(ColTraArgs a, FFTDesc<T> d, int C) {
  using V = cplx<T>;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int L = d.L, nt = d.nt, Ls = team_stride(L);
  const int tid = threadIdx.x, c = tid / nt, t = tid - c * nt;
  const int kx = blockIdx.x * C + c;
  const bool kv = (c < C) && kx < a.Hx;
  const int kxc = kv ? kx : 0;
  const int b = blockIdx.y;
  V* sm = reinterpret_cast<V*>(smraw) + (long long)c * Ls;
  V dh[E], v[E];
  const V* dc = static_cast<const V*>(a.D) + (long long)b * a.d_bstride + (long long)kxc * a.ldd;
#pragma unroll
  for (int k = 0; k < E; ++k) {
    const int j = t + nt * k;
    dh[k] = j < a.nvalid ? dc[j] : mkc<V>(T(0), T(0));
  }
  team_fft<T, E>(dh, sm, t, d);
  const V* Sb = static_cast<const V*>(a.S) + (long long)kxc * a.lds;
  V* Wb = static_cast<V*>(a.W) + (long long)b * a.w_bstride + (long long)kxc * a.ldw;
  for (int r = 0; r < a.K; ++r) {
    const V* sc = Sb + (long long)r * a.s_rstride;
#pragma unroll
    for (int k = 0; k < E; ++k) {
      // conj(conj(S) * dh) = S * conj(dh): inverse FFT via the conjugation identity
      const V w = __ldg(&sc[t + nt * k]);
      v[k] = mkc<V>(w.x * dh[k].x + w.y * dh[k].y, w.y * dh[k].x - w.x * dh[k].y);
    }
    team_fft<T, E>(v, sm, t, d);
    if (kv) {
      V* wc = Wb + (long long)r * a.w_rstride;
#pragma unroll
      for (int k = 0; k < E; ++k) {
        const int q = t + nt * k;
        if (q < a.nout) wc[q] = conjv(v[k]);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Spectrum build, column stage (fp64 FFT, stored as TS, scaled)
// ---------------------------------------------------------------------------
template <class TS, int E>
__global__ void k_col_spec(ColSpecArgs a, FFTDesc<double> d, int C) {
  using V = double2;
  using VS = cplx<TS>;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int L = d.L, nt = d.nt, Ls = team_stride(L);
  const int tid = threadIdx.x, c = tid / nt, t = tid - c * nt;
  const int kx = blockIdx.x * C + c;
  const bool kv = (c < C) && kx < a.Hx;
  const int kxc = kv ? kx : 0;
  V* sm = reinterpret_cast<V*>(smraw) + (long long)c * Ls;
  V v[E];
  const V* yc = static_cast<const V*>(a.Y) + (long long)kxc * a.ldy;
#pragma unroll
  for (int k = 0; k < E; ++k) v[k] = yc[t + nt * k];
  team_fft<double, E>(v, sm, t, d);
  if (kv) {
    VS* sc = static_cast<VS*>(a.S) + (long long)kx * a.lds;
#pragma unroll
    for (int k = 0; k < E; ++k) sc[t + nt * k] = mkc<VS>((TS)(v[k].x * a.scale), (TS)(v[k].y * a.scale));
  }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
namespace {

template <class T>
int pairs_per_cta(int nt, int L, int nrows) {
  int P = Prec<T>::pairs;
  while (P > 1 && (P * nt > kMaxThreads || (size_t)P * team_stride(L) * sizeof(cplx<T>) > 200 * 1024)) P /= 2;
  // small transforms: more teams per CTA
  while (P * nt < 128 && 2 * P * team_stride(L) * sizeof(cplx<T>) <= 96 * 1024 && 2 * P <= (nrows + 1) / 2 + 1) P *= 2;
  return P;
}

template <class T>
int cols_per_cta(int nt, int L, int Hx) {
  int C = Prec<T>::cols_threads / nt;
  if (C < 1) C = 1;
  while (C > 1 && (size_t)C * team_stride(L) * sizeof(cplx<T>) > 100 * 1024) --C;
  if (C > Hx) C = Hx;
  return C;
}

}  // namespace

#define BTTB_E_DISPATCH(E, ...)                        \
  switch (E) {                                         \
    case 8: { constexpr int EE = 8; __VA_ARGS__; } break;   \
    case 12: { constexpr int EE = 12; __VA_ARGS__; } break; \
    case 20: { constexpr int EE = 20; __VA_ARGS__; } break; \
    default: return cudaErrorInvalidValue;             \
  }

template <class K>
int team_limit(K kern, int nt) {
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, kern) != cudaSuccess) return 1;
  return fa.maxThreadsPerBlock / nt > 0 ? fa.maxThreadsPerBlock / nt : 1;
}

template <class T>
cudaError_t launch_row_r2c(const RowR2CArgs& a, const FFTDesc<T>& d, int E, cudaStream_t st) {
  if (a.nslabs <= 0 || a.nrows <= 0) return cudaSuccess;
  BTTB_E_DISPATCH(E, {
    auto kern = k_row_r2c<T, EE>;
    int P = pairs_per_cta<T>(d.nt, d.L, a.nrows);
    P = P < team_limit(kern, d.nt) ? P : team_limit(kern, d.nt);
    const size_t smem = (size_t)P * team_stride(d.L) * sizeof(cplx<T>);
    dim3 grd((a.nrows + 2 * P - 1) / (2 * P), a.nslabs), blk(P * d.nt);
    cudaError_t e = set_smem(kern, smem);
    if (e != cudaSuccess) return e;
    kern<<<grd, blk, smem, st>>>(a, d, P);
  });
  return cudaGetLastError();
}

template <class T>
cudaError_t launch_row_c2r(const RowC2RArgs& a, const FFTDesc<T>& d, int E, cudaStream_t st) {
  if (a.nslabs <= 0 || a.nrows <= 0) return cudaSuccess;
  BTTB_E_DISPATCH(E, {
    auto kern = k_row_c2r<T, EE>;
    int P = pairs_per_cta<T>(d.nt, d.L, a.nrows);
    P = P < team_limit(kern, d.nt) ? P : team_limit(kern, d.nt);
    const size_t smem = (size_t)P * team_stride(d.L) * sizeof(cplx<T>);
    dim3 grd((a.nrows + 2 * P - 1) / (2 * P), a.nslabs), blk(P * d.nt);
    cudaError_t e = set_smem(kern, smem);
    if (e != cudaSuccess) return e;
    kern<<<grd, blk, smem, st>>>(a, d, P);
  });
  return cudaGetLastError();
}

template <class T>
cudaError_t launch_col_fwd(const ColFwdArgs& a, const FFTDesc<T>& d, int E, cudaStream_t st) {
  if (a.nbatch <= 0 || a.K <= 0) return cudaSuccess;
  BTTB_E_DISPATCH(E, {
    auto kern = k_col_fwd<T, EE>;
    int C = cols_per_cta<T>(d.nt, d.L, a.Hx);
    C = C < team_limit(kern, d.nt) ? C : team_limit(kern, d.nt);
    const size_t smem = (size_t)C * team_stride(d.L) * sizeof(cplx<T>);
    dim3 grd((a.Hx + C - 1) / C, a.nbatch), blk(C * d.nt);
    cudaError_t e = set_smem(kern, smem);
    if (e != cudaSuccess) return e;
    kern<<<grd, blk, smem, st>>>(a, d, C);
  });
  return cudaGetLastError();
}

template <class T>
cudaError_t launch_col_tra(const ColTraArgs& a, const FFTDesc<T>& d, int E, cudaStream_t st) {
  if (a.nbatch <= 0 || a.K <= 0) return cudaSuccess;
  BTTB_E_DISPATCH(E, {
    auto kern = k_col_tra<T, EE>;
    int C = cols_per_cta<T>(d.nt, d.L, a.Hx);
    C = C < team_limit(kern, d.nt) ? C : team_limit(kern, d.nt);
    const size_t smem = (size_t)C * team_stride(d.L) * sizeof(cplx<T>);
    dim3 grd((a.Hx + C - 1) / C, a.nbatch), blk(C * d.nt);
    cudaError_t e = set_smem(kern, smem);
    if (e != cudaSuccess) return e;
    kern<<<grd, blk, smem, st>>>(a, d, C);
  });
  return cudaGetLastError();
}

template <class TS>
cudaError_t launch_col_spec(const ColSpecArgs& a, const FFTDesc<double>& d, int E, cudaStream_t st) {
  BTTB_E_DISPATCH(E, {
    auto kern = k_col_spec<TS, EE>;
    int C = cols_per_cta<double>(d.nt, d.L, a.Hx);
    C = C < team_limit(kern, d.nt) ? C : team_limit(kern, d.nt);
    const size_t smem = (size_t)C * team_stride(d.L) * sizeof(double2);
    dim3 grd((a.Hx + C - 1) / C), blk(C * d.nt);
    cudaError_t e = set_smem(kern, smem);
    if (e != cudaSuccess) return e;
    kern<<<grd, blk, smem, st>>>(a, d, C);
  });
  return cudaGetLastError();
}

template cudaError_t launch_row_r2c<double>(const RowR2CArgs&, const FFTDesc<double>&, int, cudaStream_t);
template cudaError_t launch_row_r2c<float>(const RowR2CArgs&, const FFTDesc<float>&, int, cudaStream_t);
template cudaError_t launch_row_c2r<double>(const RowC2RArgs&, const FFTDesc<double>&, int, cudaStream_t);
template cudaError_t launch_row_c2r<float>(const RowC2RArgs&, const FFTDesc<float>&, int, cudaStream_t);
template cudaError_t launch_col_fwd<double>(const ColFwdArgs&, const FFTDesc<double>&, int, cudaStream_t);
template cudaError_t launch_col_fwd<float>(const ColFwdArgs&, const FFTDesc<float>&, int, cudaStream_t);
template cudaError_t launch_col_tra<double>(const ColTraArgs&, const FFTDesc<double>&, int, cudaStream_t);
template cudaError_t launch_col_tra<float>(const ColTraArgs&, const FFTDesc<float>&, int, cudaStream_t);
template cudaError_t launch_col_spec<double>(const ColSpecArgs&, const FFTDesc<double>&, int, cudaStream_t);
template cudaError_t launch_col_spec<float>(const ColSpecArgs&, const FFTDesc<double>&, int, cudaStream_t);

}  // namespace bttb
