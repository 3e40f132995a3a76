// Generic-length operator path: embeddings the shared-memory FFT engine does
// not cover (any 2^a 3^b 5^c length, in particular above 8192 -- the
// reference has no size cap: grid.py:101-104 embed_shape, transform.py:101
// np.fft.fft2 of any shape).
//
// Same operator, same spectrum cache layout as the main path (per layer the
// half spectrum S[kx][ky], kx < Lx/2+1, scaled by 1/(Lx*Ly)), but every 2-D
// transform is a complex one done by batched radix passes through global
// memory (Stockham autosort, one kernel per pass, ping-pong buffers):
//
//   build:     embed (entries.cu) -> complex [y][x] -> FFT_x, FFT_y -> S
//   forward:   per layer  C = FFT2(embed(x_r));  A += S_full * C
//              then       d = Re(IFFT2(A))[i < sx, j < sy]
//   transpose: D = FFT2(embed(d)) once; per layer
//              x_r = Re(IFFT2(conj(S_full) * D))[p < nx, q < ny]
//
// (multiply.py:37-57; S_full(kx, ky) = conj(S[Lx-kx][-ky]) for kx >= Lx/2+1,
// the Hermitian symmetry of a real kernel's spectrum.)  The inverse runs as
// conj(FFT(conj z)).  Arithmetic is fp64 throughout; fp32 plans store their
// spectra and vectors in fp32 and promote on load.  This path trades speed
// for generality: each radix pass is one HBM round trip of the buffer.
#include <cuda_runtime.h>

#include <cstdint>

#include "fft.cuh"
#include "generic.h"

namespace bttb {
namespace gx {

using V = double2;

// one radix-R Stockham pass over `batch` sequences of length L:
// element e of sequence s lives at base + s*bs + e*es (in and out alike).
// Thread mapping: when the elements are contiguous (es == 1) the butterfly
// index j runs fastest (coalesced along the sequence), otherwise the
// sequence index does (coalesced across neighbouring sequences).
template <int R>
__global__ void k_pass(const V* __restrict__ in, V* __restrict__ out, int L, int Ns, long long batch, long long bs,
                       long long es, const V* __restrict__ tw) {
  const int Q = L / R;
  const long long total = (long long)Q * batch;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    long long s;
    int j;
    if (es == 1) {
      s = t / Q;
      j = (int)(t - s * Q);
    } else {
      j = (int)(t / batch);
      s = t - (long long)j * batch;
    }
    const V* src = in + s * bs;
    V* dst = out + s * bs;
    V v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = src[(long long)(j + r * Q) * es];
    const int k = j % Ns;
    if (Ns > 1) {
      // w_{Ns R}^{r k} = W_L[r k L / (Ns R)], exact table index
      const long long step = (long long)k * (L / (Ns * R));
#pragma unroll
      for (int r = 1; r < R; ++r) v[r] = cmul(v[r], __ldg(&tw[(r * step) % L]));
    }
    dft<R>(v);
    const long long base = (long long)(j / Ns) * Ns * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) dst[(base + (long long)r * Ns) * es] = v[r];
  }
}

// real [y][x] (Ly x Lx) -> complex
template <class S>
__global__ void k_to_complex(const S* __restrict__ in, V* __restrict__ out, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = make_double2((double)in[i], 0.0);
}

// vector (rows of w values, `rows` rows) placed into a zeroed complex [y][x] grid of row length Lx
template <class S>
__global__ void k_place(const S* __restrict__ v, int w, int rows, V* __restrict__ out, int Lx, int Ly) {
  const long long n = (long long)Lx * Ly;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int y = (int)(i / Lx), x = (int)(i - (long long)y * Lx);
    out[i] = make_double2(x < w && y < rows ? (double)v[(long long)y * w + x] : 0.0, 0.0);
  }
}

// F[ky][kx] (full spectrum, y-major) -> S[kx][ky] = scale * F for kx < Hx
template <class S>
__global__ void k_extract_spectrum(const V* __restrict__ F, S* __restrict__ out, int Lx, int Ly, int Hx,
                                   double scale) {
  const long long n = (long long)Hx * Ly;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int kx = (int)(i / Ly), ky = (int)(i - (long long)kx * Ly);
    const V f = F[(long long)ky * Lx + kx];
    out[2 * i] = (S)(scale * f.x);
    out[2 * i + 1] = (S)(scale * f.y);
  }
}

template <class S>
__device__ __forceinline__ V spec_full(const S* __restrict__ Sp, int Lx, int Ly, int Hx, int kx, int ky) {
  if (kx < Hx) {
    const long long o = 2 * ((long long)kx * Ly + ky);
    return make_double2((double)Sp[o], (double)Sp[o + 1]);
  }
  const long long o = 2 * ((long long)(Lx - kx) * Ly + (ky == 0 ? 0 : Ly - ky));
  return make_double2((double)Sp[o], -(double)Sp[o + 1]);
}

// forward: A (+)= S_full * C; transpose: C <- conj(conj(S_full) * D) (pre-conjugated for the inverse)
template <class S>
__global__ void k_spec_mul(const S* __restrict__ Sp, const V* __restrict__ C, V* __restrict__ A, int Lx, int Ly,
                           int Hx, int mode, int first) {
  const long long n = (long long)Lx * Ly;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int ky = (int)(i / Lx), kx = (int)(i - (long long)ky * Lx);
    const V s = spec_full(Sp, Lx, Ly, Hx, kx, ky);
    const V c = C[i];
    if (mode == 0) {
      const V p = cmul(s, c);
      A[i] = first ? p : A[i] + p;
    } else {
      // conj(conj(s) * d) = s * conj(d)
      A[i] = cmul(s, conjv(c));
    }
  }
}

// out[y][x] = Re(conj(Z[y][x])) = Re(Z) for x < w, y < rows (row length w)
template <class S>
__global__ void k_crop(const V* __restrict__ Z, int Lx, S* __restrict__ out, int w, int rows) {
  const long long n = (long long)w * rows;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int y = (int)(i / w), x = (int)(i - (long long)y * w);
    out[i] = (S)Z[(long long)y * Lx + x].x;
  }
}

__global__ void k_conj(V* z, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    z[i].y = -z[i].y;
}

int grid_for(long long n) {
  long long b = (n + 255) / 256;
  return (int)(b < 148 * 16 ? (b < 1 ? 1 : b) : 148 * 16);
}

cudaError_t launch_pass(int R, const V* in, V* out, int L, int Ns, long long batch, long long bs, long long es,
                        const V* tw, cudaStream_t st) {
  const long long total = (long long)(L / R) * batch;
  const int g = grid_for(total);
  switch (R) {
    case 2: k_pass<2><<<g, 256, 0, st>>>(in, out, L, Ns, batch, bs, es, tw); break;
    case 3: k_pass<3><<<g, 256, 0, st>>>(in, out, L, Ns, batch, bs, es, tw); break;
    case 4: k_pass<4><<<g, 256, 0, st>>>(in, out, L, Ns, batch, bs, es, tw); break;
    case 5: k_pass<5><<<g, 256, 0, st>>>(in, out, L, Ns, batch, bs, es, tw); break;
    case 8: k_pass<8><<<g, 256, 0, st>>>(in, out, L, Ns, batch, bs, es, tw); break;
    case 16: k_pass<16><<<g, 128, 0, st>>>(in, out, L, Ns, batch, bs, es, tw); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace gx

bool generic_length_ok(long long L) {
  if (L < 1 || L > 65536) return false;
  long long t = L;
  for (int f : {2, 3, 5})
    while (t % f == 0) t /= f;
  return t == 1;
}

long long generic_length(long long n) {
  for (long long L = n < 1 ? 1 : n; L <= 65536; ++L)
    if (generic_length_ok(L)) return L;
  return -1;
}

int GenericFFT::init(int len, const double2* table) {
  L = len;
  tw = table;
  np = 0;
  int rem = L;
  for (int f : {16, 8, 4, 2, 5, 3})
    while (rem % f == 0 && np < 24) {
      radix[np++] = f;
      rem /= f;
    }
  return rem == 1 ? 0 : -1;
}

// transform of `batch` sequences in `buf` (tmp: scratch of the same extent,
// `total` complex values); the result lands back in `buf`
cudaError_t GenericFFT::run(double2* buf, double2* tmp, long long total, long long batch, long long bs,
                            long long es, cudaStream_t st) const {
  const double2* src = buf;
  double2* dst = tmp;
  int Ns = 1;
  for (int p = 0; p < np; ++p) {
    cudaError_t e = gx::launch_pass(radix[p], src, dst, L, Ns, batch, bs, es, tw, st);
    if (e != cudaSuccess) return e;
    Ns *= radix[p];
    src = dst;
    dst = (dst == tmp) ? buf : tmp;
  }
  if (src != buf) return cudaMemcpyAsync(buf, src, sizeof(double2) * (size_t)total, cudaMemcpyDeviceToDevice, st);
  return cudaSuccess;
}

// FFT along x then y of a [Ly][Lx] complex grid
static cudaError_t fft2(const GenericCtx& g, double2* z, double2* tmp, cudaStream_t st) {
  const long long n = (long long)g.Lx * g.Ly;
  cudaError_t e = g.fx.run(z, tmp, n, g.Ly, g.Lx, 1, st);
  if (e == cudaSuccess) e = g.fy.run(z, tmp, n, g.Lx, 1, g.Lx, st);
  return e;
}

template <class S>
cudaError_t generic_build_layer(const GenericCtx& g, const double* emb, void* spectrum, cudaStream_t st) {
  const long long n = (long long)g.Lx * g.Ly;
  gx::k_to_complex<double><<<gx::grid_for(n), 256, 0, st>>>(emb, g.C, n);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = fft2(g, g.C, g.B, st);
  if (e != cudaSuccess) return e;
  const double scale = 1.0 / ((double)g.Lx * (double)g.Ly);
  gx::k_extract_spectrum<S><<<gx::grid_for((long long)g.Hx * g.Ly), 256, 0, st>>>(g.C, static_cast<S*>(spectrum),
                                                                                   g.Lx, g.Ly, g.Hx, scale);
  return cudaGetLastError();
}

template <class S>
cudaError_t generic_forward(const GenericCtx& g, const void* spectra, long long nl, const S* x, int nx, int ny,
                            S* d, int sx, int sy, cudaStream_t st) {
  const long long n = (long long)g.Lx * g.Ly, sl = 2LL * g.Hx * g.Ly;
  cudaError_t e = cudaSuccess;
  for (long long r = 0; r < nl && e == cudaSuccess; ++r) {
    gx::k_place<S><<<gx::grid_for(n), 256, 0, st>>>(x + r * (long long)nx * ny, nx, ny, g.C, g.Lx, g.Ly);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = fft2(g, g.C, g.B, st);
    if (e != cudaSuccess) break;
    gx::k_spec_mul<S><<<gx::grid_for(n), 256, 0, st>>>(static_cast<const S*>(spectra) + r * sl, g.C, g.A, g.Lx,
                                                        g.Ly, g.Hx, 0, r == 0);
    e = cudaGetLastError();
  }
  if (e != cudaSuccess) return e;
  if (nl == 0) e = cudaMemsetAsync(g.A, 0, sizeof(double2) * (size_t)n, st);
  if (e != cudaSuccess) return e;
  gx::k_conj<<<gx::grid_for(n), 256, 0, st>>>(g.A, n);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = fft2(g, g.A, g.B, st);
  if (e != cudaSuccess) return e;
  gx::k_crop<S><<<gx::grid_for((long long)sx * sy), 256, 0, st>>>(g.A, g.Lx, d, sx, sy);
  return cudaGetLastError();
}

template <class S>
cudaError_t generic_transpose(const GenericCtx& g, const void* spectra, long long nl, const S* d, int sx, int sy,
                              S* x, int nx, int ny, cudaStream_t st) {
  const long long n = (long long)g.Lx * g.Ly, sl = 2LL * g.Hx * g.Ly;
  gx::k_place<S><<<gx::grid_for(n), 256, 0, st>>>(d, sx, sy, g.A, g.Lx, g.Ly);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = fft2(g, g.A, g.B, st);
  for (long long r = 0; r < nl && e == cudaSuccess; ++r) {
    gx::k_spec_mul<S><<<gx::grid_for(n), 256, 0, st>>>(static_cast<const S*>(spectra) + r * sl, g.A, g.C, g.Lx,
                                                        g.Ly, g.Hx, 1, 0);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = fft2(g, g.C, g.B, st);
    if (e != cudaSuccess) break;
    gx::k_crop<S><<<gx::grid_for((long long)nx * ny), 256, 0, st>>>(g.C, g.Lx, x + r * (long long)nx * ny, nx, ny);
    e = cudaGetLastError();
  }
  return e;
}

template cudaError_t generic_build_layer<double>(const GenericCtx&, const double*, void*, cudaStream_t);
template cudaError_t generic_build_layer<float>(const GenericCtx&, const double*, void*, cudaStream_t);
template cudaError_t generic_forward<double>(const GenericCtx&, const void*, long long, const double*, int, int,
                                             double*, int, int, cudaStream_t);
template cudaError_t generic_forward<float>(const GenericCtx&, const void*, long long, const float*, int, int,
                                            float*, int, int, cudaStream_t);
template cudaError_t generic_transpose<double>(const GenericCtx&, const void*, long long, const double*, int, int,
                                               double*, int, int, cudaStream_t);
template cudaError_t generic_transpose<float>(const GenericCtx&, const void*, long long, const float*, int, int,
                                              float*, int, int, cudaStream_t);

}  // namespace bttb
