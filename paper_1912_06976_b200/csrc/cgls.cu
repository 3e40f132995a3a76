// Vector kernels of the device-resident batched CGLS driver (bttb_cgls).
//
// The paper names a GPU inversion loop as future work (the
// reference lists it as a non-goal).  CGLS for
//   min ||G m - d||^2 + damp^2 ||m||^2
// needs, besides one forward and one transpose product per iteration, a few
// dot products and vector updates; these kernels keep them on the device with
// the scalars in device memory (no host round trip inside the loop, so the
// loop is stream-ordered and graph-capturable):
//   * dot products reduce in fp64 into per-block partials that a one-warp
//     scalar kernel sums in a fixed order (deterministic, no atomics);
//   * the n-length updates are fused: m += alpha p and p = s + beta p in one
//     pass (undamped), or m += alpha p; s -= damp^2 m with the s.s partials in
//     one pass and p = s + beta p in a second (damped).
// All vectors are batch-major (item b at base + b*len), fp64 or fp32; the
// scalars are fp64 for both.
#include <cuda_runtime.h>

#include <cstring>
#include <type_traits>

#include "cgls.h"

namespace bttb {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double red[kThreads / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (w == 0) {
    s = l < kThreads / 32 ? red[l] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  }
  return s;  // valid in thread 0
}

// 16-byte packs: the vector kernels stream with 128-bit accesses when an
// item's length allows (every slice then starts on a pack boundary)
template <class T> struct VecOf;
template <> struct VecOf<float> { using type = float4; static constexpr int N = 4; };
template <> struct VecOf<double> { using type = double2; static constexpr int N = 2; };

template <class T, int N> struct Pack {
  T v[N];
};
template <class T, int N> __device__ __forceinline__ Pack<T, N> ld(const T* p) {
  Pack<T, N> r;
  if constexpr (N == 1) {
    r.v[0] = *p;
  } else {
    using W = typename VecOf<T>::type;
    const W w = *reinterpret_cast<const W*>(p);
    static_assert(sizeof(W) == sizeof(Pack<T, N>), "pack size");
    memcpy(&r, &w, sizeof(W));
  }
  return r;
}
template <class T, int N> __device__ __forceinline__ void st(T* p, const Pack<T, N>& r) {
  if constexpr (N == 1) {
    *p = r.v[0];
  } else {
    using W = typename VecOf<T>::type;
    W w;
    memcpy(&w, &r, sizeof(W));
    *reinterpret_cast<W*>(p) = w;
  }
}

// Block blockIdx.x's slice of item blockIdx.y: body(i, N) on elements
// [i, i+N) of the item, N = the pack width when len is a multiple of it (the
// slice bounds then are too), else 1.
template <class T, class F> __device__ __forceinline__ void for_slice(long long len, F&& body) {
  constexpr int VN = VecOf<T>::N;
  const bool vec = len % VN == 0;
  long long chunk = (len + gridDim.x - 1) / gridDim.x;
  chunk = (chunk + VN - 1) / VN * VN;
  const long long lo = chunk * blockIdx.x;
  const long long hi = lo + chunk < len ? lo + chunk : len;
  if (vec) {
#pragma unroll 2
    for (long long i = lo + (long long)VN * threadIdx.x; i < hi; i += (long long)VN * kThreads)
      body(i, std::integral_constant<int, VN>{});
  } else {
    for (long long i = lo + threadIdx.x; i < hi; i += kThreads) body(i, std::integral_constant<int, 1>{});
  }
}

__device__ __forceinline__ void put_partial(double v, double* part) {
  v = block_sum(v);
  if (threadIdx.x == 0) part[(long long)blockIdx.y * gridDim.x + blockIdx.x] = v;
}

// part = a . b per block (a == b: squared norm)
template <class T>
__global__ void __launch_bounds__(kThreads) k_dot(const T* __restrict__ a, const T* __restrict__ b, long long len,
                                                  double* __restrict__ part) {
  const T* ab = a + (long long)blockIdx.y * len;
  const T* bb = b + (long long)blockIdx.y * len;
  double acc = 0.0;
  for_slice<T>(len, [&](long long i, auto nc) {
    constexpr int N = decltype(nc)::value;
    const auto x = ld<T, N>(ab + i), y = ld<T, N>(bb + i);
#pragma unroll
    for (int j = 0; j < N; ++j) acc += (double)x.v[j] * (double)y.v[j];
  });
  put_partial(acc, part);
}

// r -= alpha q, part = r . r (the data residual norm)
template <class T>
__global__ void __launch_bounds__(kThreads) k_resid(T* __restrict__ r, const T* __restrict__ q, long long len,
                                                    const CglsScalars* __restrict__ sc, double* __restrict__ part) {
  const long long base = (long long)blockIdx.y * len;
  const double alpha = sc[blockIdx.y].alpha;
  double acc = 0.0;
  for_slice<T>(len, [&](long long i, auto nc) {
    constexpr int N = decltype(nc)::value;
    auto rv = ld<T, N>(r + base + i);
    const auto qv = ld<T, N>(q + base + i);
#pragma unroll
    for (int j = 0; j < N; ++j) {
      rv.v[j] = (T)((double)rv.v[j] - alpha * (double)qv.v[j]);
      acc += (double)rv.v[j] * (double)rv.v[j];
    }
    st<T, N>(r + base + i, rv);
  });
  put_partial(acc, part);
}

// undamped: m += alpha p; p = s + beta p
template <class T>
__global__ void __launch_bounds__(kThreads) k_update_mp(T* __restrict__ m, T* __restrict__ p, const T* __restrict__ s,
                                                        long long len, const CglsScalars* __restrict__ sc) {
  const long long base = (long long)blockIdx.y * len;
  const double alpha = sc[blockIdx.y].alpha, beta = sc[blockIdx.y].beta;
  for_slice<T>(len, [&](long long i, auto nc) {
    constexpr int N = decltype(nc)::value;
    auto mv = ld<T, N>(m + base + i), pv = ld<T, N>(p + base + i);
    const auto sv = ld<T, N>(s + base + i);
#pragma unroll
    for (int j = 0; j < N; ++j) {
      const double pj = (double)pv.v[j];
      mv.v[j] = (T)((double)mv.v[j] + alpha * pj);
      pv.v[j] = (T)((double)sv.v[j] + beta * pj);
    }
    st<T, N>(m + base + i, mv);
    st<T, N>(p + base + i, pv);
  });
}

// damped, first pass: m += alpha p; s -= damp2 m; part = s . s
template <class T>
__global__ void __launch_bounds__(kThreads) k_damp_s(T* __restrict__ m, const T* __restrict__ p, T* __restrict__ s,
                                                     long long len, const CglsScalars* __restrict__ sc, double damp2,
                                                     double* __restrict__ part) {
  const long long base = (long long)blockIdx.y * len;
  const double alpha = sc[blockIdx.y].alpha;
  double acc = 0.0;
  for_slice<T>(len, [&](long long i, auto nc) {
    constexpr int N = decltype(nc)::value;
    auto mv = ld<T, N>(m + base + i), sv = ld<T, N>(s + base + i);
    const auto pv = ld<T, N>(p + base + i);
#pragma unroll
    for (int j = 0; j < N; ++j) {
      mv.v[j] = (T)((double)mv.v[j] + alpha * (double)pv.v[j]);
      sv.v[j] = (T)((double)sv.v[j] - damp2 * (double)mv.v[j]);
      acc += (double)sv.v[j] * (double)sv.v[j];
    }
    st<T, N>(m + base + i, mv);
    st<T, N>(s + base + i, sv);
  });
  put_partial(acc, part);
}

// damped, second pass: p = s + beta p
template <class T>
__global__ void __launch_bounds__(kThreads) k_update_p(T* __restrict__ p, const T* __restrict__ s, long long len,
                                                       const CglsScalars* __restrict__ sc) {
  const long long base = (long long)blockIdx.y * len;
  const double beta = sc[blockIdx.y].beta;
  for_slice<T>(len, [&](long long i, auto nc) {
    constexpr int N = decltype(nc)::value;
    auto pv = ld<T, N>(p + base + i);
    const auto sv = ld<T, N>(s + base + i);
#pragma unroll
    for (int j = 0; j < N; ++j) pv.v[j] = (T)((double)sv.v[j] + beta * (double)pv.v[j]);
    st<T, N>(p + base + i, pv);
  });
}

// one warp per item: fixed-order sum of nblk partials
__device__ __forceinline__ double warp_total(const double* part, int nblk) {
  double v = 0.0;
  for (int i = threadIdx.x & 31; i < nblk; i += 32) v += part[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void k_scalars(int op, int batch, const double* __restrict__ pa, int nblk_a, const double* __restrict__ pb,
                          int nblk_b, double damp2, double rtol, CglsScalars* __restrict__ sc, double* __restrict__ hist, int hist_ld,
                          int hist_col) {
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (b >= batch) return;
  const double a = warp_total(pa + (long long)b * nblk_a, nblk_a);
  const double c = pb ? warp_total(pb + (long long)b * nblk_b, nblk_b) : 0.0;
  if ((threadIdx.x & 31) != 0) return;
  CglsScalars& s = sc[b];
  switch (op) {
    case CGLS_INIT:  // a = s.s (s = G^T d), c = d.d
      s.gamma = a;
      s.floor = rtol * rtol * a;
      s.alpha = s.beta = 0.0;
      if (hist) hist[(long long)b * hist_ld + hist_col] = sqrt(c);
      break;
    case CGLS_ALPHA: {  // a = q.q, c = p.p
      const double delta = a + damp2 * c;
      s.alpha = (delta > 0.0 && s.gamma > s.floor) ? s.gamma / delta : 0.0;
      break;
    }
    case CGLS_BETA:  // a = s.s (new gradient), c = r.r
      s.beta = s.gamma > s.floor ? a / s.gamma : 0.0;
      s.gamma = a;
      if (hist) hist[(long long)b * hist_ld + hist_col] = sqrt(c);
      break;
    default:
      break;
  }
}

inline dim3 vec_grid(int batch, int nblk) { return dim3((unsigned)nblk, (unsigned)batch); }

}  // namespace

int cgls_blocks(long long len, int batch, int nsm) {
  // about 16 blocks per SM over the whole batch (two waves of 8 resident),
  // at least 2048 elements per block, at most 1024 blocks per item
  long long want = (16LL * nsm + batch - 1) / batch;
  const long long cap = (len + 2047) / 2048;
  if (want > cap) want = cap;
  if (want > 1024) want = 1024;
  return want < 1 ? 1 : (int)want;
}

template <class T>
cudaError_t cgls_dot(const T* a, const T* b, long long len, int batch, int nblk, double* part, cudaStream_t st) {
  k_dot<T><<<vec_grid(batch, nblk), kThreads, 0, st>>>(a, b, len, part);
  return cudaGetLastError();
}

template <class T>
cudaError_t cgls_resid(T* r, const T* q, long long len, int batch, int nblk, const CglsScalars* sc, double* part,
                       cudaStream_t st) {
  k_resid<T><<<vec_grid(batch, nblk), kThreads, 0, st>>>(r, q, len, sc, part);
  return cudaGetLastError();
}

template <class T>
cudaError_t cgls_update(T* m, T* p, T* s, long long len, int batch, int nblk, const CglsScalars* sc, double damp2,
                        double* part, int phase, cudaStream_t st) {
  const dim3 g = vec_grid(batch, nblk);
  if (damp2 == 0.0) {
    if (phase == 0) k_dot<T><<<g, kThreads, 0, st>>>(s, s, len, part);
    else k_update_mp<T><<<g, kThreads, 0, st>>>(m, p, s, len, sc);
  } else {
    if (phase == 0) k_damp_s<T><<<g, kThreads, 0, st>>>(m, p, s, len, sc, damp2, part);
    else k_update_p<T><<<g, kThreads, 0, st>>>(p, s, len, sc);
  }
  return cudaGetLastError();
}

cudaError_t cgls_scalars(int op, int batch, const double* pa, int nblk_a, const double* pb, int nblk_b,
                         double damp2, double rtol, CglsScalars* sc, double* hist, int hist_ld, int hist_col,
                         cudaStream_t st) {
  const int per = 4;  // items (warps) per block
  k_scalars<<<(batch + per - 1) / per, 32 * per, 0, st>>>(op, batch, pa, nblk_a, pb, nblk_b, damp2, rtol, sc, hist,
                                                          hist_ld, hist_col);
  return cudaGetLastError();
}

#define INST(T)                                                                                                  \
  template cudaError_t cgls_dot<T>(const T*, const T*, long long, int, int, double*, cudaStream_t);              \
  template cudaError_t cgls_resid<T>(T*, const T*, long long, int, int, const CglsScalars*, double*,             \
                                     cudaStream_t);                                                              \
  template cudaError_t cgls_update<T>(T*, T*, T*, long long, int, int, const CglsScalars*, double, double*, int, \
                                      cudaStream_t);
INST(double)
INST(float)
#undef INST

}  // namespace bttb
