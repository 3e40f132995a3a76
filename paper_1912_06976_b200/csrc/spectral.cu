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
//
// Memory hints: the cached spectra and the model vectors are streamed exactly
// once per application, so they are loaded with evict-first (ld.global.cs)
// and the transpose's model output is stored with st.global.cs; the chunk
// intermediates (row-pass output Y, accumulator W) use the default policy so
// they stay L2-resident between the row and column kernels.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "spectral.h"
#include "tma.cuh"

#ifndef ROW_REGS_F32
#define ROW_REGS_F32 64  // register target of the fp32 row passes: four CTAs per SM (C4 fp32 2.42 -> 2.22 ms/step vs 128)
#endif
#ifndef BTTB_R2C_PAIR
#define BTTB_R2C_PAIR 1  // mirrored last pass + in-register separation in the 2048-point row R2C
#endif
#ifndef ROW_REGS_F64
#define ROW_REGS_F64 128  // register target of the fp64 row passes
#endif
#ifndef COL_REGS_F32
#define COL_REGS_F32 168  // register target of the fp32 column stages (96, 128 measured slower)
#endif
#ifndef TRA_REGS_F64
#define TRA_REGS_F64 168  // register target of the fp64 TMA transpose column stage (see Shape::tra_regs)
#endif
#ifndef T2D_TEAMS
#define T2D_TEAMS 1  // row pairs (teams) per CTA of the tensor-TMA row passes
#endif

namespace bttb {

namespace {

template <class K>
cudaError_t set_smem(K kernel, size_t bytes) {
  if (bytes > 48 * 1024) return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  return cudaSuccess;
}

}  // namespace

// ---------------------------------------------------------------------------
// Row pass, real -> half spectrum, two rows per complex FFT
// ---------------------------------------------------------------------------
template <class PL, int MAXT, int MINB>
__global__ void __launch_bounds__(MAXT, MINB) k_row_r2c(RowR2CArgs a, FFTDesc<typename PL::Scalar> d, int P) {
  using T = typename PL::Scalar;
  using V = cplx<T>;
  constexpr int E = PL::E;
  extern __shared__ __align__(16) unsigned char smraw[];
  V* smb = reinterpret_cast<V*>(smraw);
  const int L = d.L, nt = PL::nt(d), Ls = PL::slots(L);
  const int tid = threadIdx.x, c = tid / nt, t = tid - c * nt;
  const int s = blockIdx.y;
  const int q0 = blockIdx.x * 2 * P;
  const int qa = q0 + 2 * c, qb = qa + 1;
  const T* in = static_cast<const T*>(a.in) + (long long)((unsigned)s / (unsigned)a.spb) * a.in_bstride +
                (long long)((unsigned)s % (unsigned)a.spb) * a.in_sstride;
  const bool va = qa < a.nrows, vb = qb < a.nrows;
  const T* ra = in + (long long)(va ? qa : 0) * a.ld_in;
  const T* rb = in + (long long)(vb ? qb : 0) * a.ld_in;
  V v[E];
#pragma unroll
  for (int k = 0; k < E; ++k) {
    const int i = t + nt * k;
    const bool inb = i < a.nvalid;
    v[k] = mkc<V>(va && inb ? __ldcs(ra + i) : T(0), vb && inb ? __ldcs(rb + i) : T(0));
  }
  V* sm = smb + (long long)c * Ls;
  PL::fft(v, sm, t, d);
  __syncthreads();
#pragma unroll
  for (int k = 0; k < E; ++k) sm[PL::slot(t + nt * k)] = v[k];
  __syncthreads();
  // separate the two real transforms and store transposed: out[s][kx][q]
  V* out = static_cast<V*>(a.out) + (long long)s * a.out_sstride;
  const int nitems = a.Hx * P;
  for (int it = tid; it < nitems; it += blockDim.x) {
    const int kx = it / P, cc = it - kx * P;
    const int q = q0 + 2 * cc;
    const V* z = smb + (long long)cc * Ls;
    const V zk = z[PL::slot(kx)];
    const V zm = z[PL::slot(kx == 0 ? 0 : L - kx)];
    const T h = T(0.5);
    V* o = out + (long long)kx * a.ld_out + q;
    if (q < a.nrows) o[0] = mkc<V>(h * (zk.x + zm.x), h * (zk.y - zm.y));
    if (q + 1 < a.nrows) o[1] = mkc<V>(h * (zk.y + zm.y), h * (zm.x - zk.x));
  }
}

// ---------------------------------------------------------------------------
// Row pass, half spectrum -> real rows (two rows per complex inverse FFT)
// ---------------------------------------------------------------------------
template <class PL, int MAXT, int MINB>
__global__ void __launch_bounds__(MAXT, MINB) k_row_c2r(RowC2RArgs a, FFTDesc<typename PL::Scalar> d, int P) {
  using T = typename PL::Scalar;
  using V = cplx<T>;
  constexpr int E = PL::E;
  extern __shared__ __align__(16) unsigned char smraw[];
  V* smb = reinterpret_cast<V*>(smraw);
  const int L = d.L, nt = PL::nt(d), Ls = PL::slots(L);
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
    z[PL::slot(kx)] = mkc<V>(A.x - B.y, A.y + B.x);
    if (kx >= 1 && kx <= L - a.Hx) z[PL::slot(L - kx)] = mkc<V>(A.x + B.y, B.x - A.y);
  }
  __syncthreads();
  V* sm = smb + (long long)c * Ls;
  V v[E];
#pragma unroll
  for (int k = 0; k < E; ++k) v[k] = conjv(sm[PL::slot(t + nt * k)]);
  PL::fft(v, sm, t, d);
  const int ja = j0 + 2 * c, jb = ja + 1;
  const bool va = ja < a.nrows, vb = jb < a.nrows;
  T* out = static_cast<T*>(a.out) + (long long)((unsigned)s / (unsigned)a.spb) * a.out_bstride +
           (long long)((unsigned)s % (unsigned)a.spb) * a.out_sstride;
  T* oa = out + (long long)(va ? ja : 0) * a.ld_out;
  T* ob = out + (long long)(vb ? jb : 0) * a.ld_out;
#pragma unroll
  for (int k = 0; k < E; ++k) {
    const int i = t + nt * k;
    if (i < a.nout) {
      if (va) __stcs(oa + i, v[k].x);
      if (vb) __stcs(ob + i, -v[k].y);
    }
  }
}

// ---------------------------------------------------------------------------
// Forward column stage: FFT along y, multiply by cached spectrum, accumulate
// over the chunk's layers in registers, one inverse FFT, extract stations.
// ---------------------------------------------------------------------------
template <class PL, int MAXT, int MINB, bool ACCS>
__global__ void __launch_bounds__(MAXT, MINB) k_col_fwd(ColFwdArgs a, FFTDesc<typename PL::Scalar> d, int C) {
  using T = typename PL::Scalar;
  using V = cplx<T>;
  constexpr int E = PL::E;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int nt = PL::nt(d), Ls = PL::slots(d.L);
  const int tid = threadIdx.x, c = tid / nt, t = tid - c * nt;
  const int kx = blockIdx.x * C + c;
  const bool kv = kx < a.Hx;
  const int kxc = kv ? kx : 0;
  const int b = blockIdx.y;
  // team buffer: [exchange (Ls padded slots)] [+ accumulator, L slots, if ACCS]
  V* sm = reinterpret_cast<V*>(smraw) + (long long)c * (Ls + (ACCS ? d.L : 0));
  V* accs = sm + Ls;  // thread t owns slots t + nt*k: conflict-free, no barrier needed
  V acc[ACCS ? 1 : E], v[E];
  if constexpr (!ACCS) {
#pragma unroll
    for (int k = 0; k < E; ++k) acc[k] = mkc<V>(T(0), T(0));
  }
  const V* Yb = static_cast<const V*>(a.Y) + (long long)b * a.y_bstride + (long long)kxc * a.ldy;
  const V* Sb = static_cast<const V*>(a.S) + (long long)kxc * a.lds;
  for (int r = 0; r < a.K; ++r) {
    const V* yc = Yb + (long long)r * a.y_rstride;
#pragma unroll
    for (int k = 0; k < E; ++k) {
      const int q = t + nt * k;
      v[k] = q < a.nvalid ? yc[q] : mkc<V>(T(0), T(0));
    }
    PL::fft(v, sm, t, d);
    const V* sc = Sb + (long long)r * a.s_rstride;
#pragma unroll
    for (int k = 0; k < E; ++k) {
      const V w = __ldcs(sc + t + nt * k);
      if constexpr (ACCS) {
        V o = r == 0 ? mkc<V>(T(0), T(0)) : accs[t + nt * k];
        o.x += w.x * v[k].x - w.y * v[k].y;
        o.y += w.x * v[k].y + w.y * v[k].x;
        accs[t + nt * k] = o;
      } else {
        acc[k].x += w.x * v[k].x - w.y * v[k].y;
        acc[k].y += w.x * v[k].y + w.y * v[k].x;
      }
    }
  }
  if constexpr (ACCS) {
#pragma unroll
    for (int k = 0; k < E; ++k) v[k] = conjv(accs[t + nt * k]);
  } else {
#pragma unroll
    for (int k = 0; k < E; ++k) v[k] = conjv(acc[k]);
  }
  PL::fft(v, sm, t, d);
  if (kv) {
    V* wc = static_cast<V*>(a.W) + (long long)b * a.w_bstride + (long long)kx * a.ldw;
#pragma unroll
    for (int k = 0; k < E; ++k) {
      const int j = t + nt * k;
      if (j < a.nout) {
        V val = conjv(v[k]);
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
template <class PL, int MAXT, int MINB, bool ACCS>
__global__ void __launch_bounds__(MAXT, MINB) k_col_tra(ColTraArgs a, FFTDesc<typename PL::Scalar> d, int C) {
  using T = typename PL::Scalar;
  using V = cplx<T>;
  constexpr int E = PL::E;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int nt = PL::nt(d), Ls = PL::slots(d.L);
  const int tid = threadIdx.x, c = tid / nt, t = tid - c * nt;
  const int kx = blockIdx.x * C + c;
  const bool kv = kx < a.Hx;
  const int kxc = kv ? kx : 0;
  const int b = blockIdx.y;
  V* sm = reinterpret_cast<V*>(smraw) + (long long)c * (Ls + (ACCS ? d.L : 0));
  V* dhs = sm + Ls;  // data spectrum, thread-owned slots (ACCS)
  V dh[ACCS ? 1 : E], v[E];
  const V* dc = static_cast<const V*>(a.D) + (long long)b * a.d_bstride + (long long)kxc * a.ldd;
#pragma unroll
  for (int k = 0; k < E; ++k) {
    const int j = t + nt * k;
    v[k] = j < a.nvalid ? dc[j] : mkc<V>(T(0), T(0));
  }
  PL::fft(v, sm, t, d);
#pragma unroll
  for (int k = 0; k < E; ++k) {
    if constexpr (ACCS) dhs[t + nt * k] = v[k]; else dh[k] = v[k];
  }
  const V* Sb = static_cast<const V*>(a.S) + (long long)kxc * a.lds;
  V* Wb = static_cast<V*>(a.W) + (long long)b * a.w_bstride + (long long)kxc * a.ldw;
  const long long qstride = 1;
  for (int r = 0; r < a.K; ++r) {
    const V* sc = Sb + (long long)r * a.s_rstride;
#pragma unroll
    for (int k = 0; k < E; ++k) {
      // conj(conj(S) * dh) = S * conj(dh): inverse FFT via the conjugation identity
      const V w = __ldcs(sc + t + nt * k);
      V h;
      if constexpr (ACCS) h = dhs[t + nt * k]; else h = dh[k];
      v[k] = mkc<V>(w.x * h.x + w.y * h.y, w.y * h.x - w.x * h.y);
    }
    PL::fft(v, sm, t, d);
    if (kv) {
      V* wc = Wb + (long long)r * a.w_rstride;
#pragma unroll
      for (int k = 0; k < E; ++k) {
        const int q = t + nt * k;
        if (q < a.nout) wc[q * qstride] = conjv(v[k]);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// TMA-pipelined column stages (compile-time plans, one column per CTA).
// Thread 0 streams the next layer's Y column and spectrum column into shared
// memory with cp.async.bulk while the team runs the current FFT, so the
// global-memory latency is off the critical path and the in-flight data
// costs no registers.  Spectra are fetched with an L2 evict-first policy.
// Shared layout: [exchange Ls][spectrum L][Y or D column nv][2 mbarriers].
// ---------------------------------------------------------------------------
// TWC: the plan's pass twiddles live in a per-CTA TMEM cache (fft.cuh,
// TmemTwCache), filled once and reused for every layer.
template <class PL, bool TWC> struct TwCache {
  static constexpr int cols = TWC ? PL::kTwCols : 0;
  static constexpr int ncols = cols <= 32 ? 32 : cols <= 64 ? 64 : cols <= 128 ? 128 : cols <= 256 ? 256 : 512;
  __device__ __forceinline__ static TmemTwCache setup(uint32_t* taddr_s, int t, const FFTDesc<typename PL::Scalar>& d) {
    TmemTwCache tc{0u};
    if constexpr (TWC) {
      tmem_fence_before();
      __syncthreads();
      tmem_fence_after();
      tc.ta = *taddr_s + ((uint32_t)(32 * ((t / 32) & 3)) << 16);
      PL::tw_fill(t, d, tc.ta);
      tmem_wait_st();
    }
    return tc;
  }
  __device__ __forceinline__ static void alloc(uint32_t* taddr_s, int t) {
    if constexpr (TWC) {
      if (t < 32) tmem_alloc<ncols>(taddr_s);
    }
  }
  __device__ __forceinline__ static void release(uint32_t* taddr_s, int t) {
    if constexpr (TWC) {
      tmem_fence_before();
      __syncthreads();
      tmem_fence_after();
      if (t < 32) tmem_dealloc<ncols>(*taddr_s);
    }
  }
  template <int E>
  __device__ __forceinline__ static void fft(cplx<typename PL::Scalar> (&v)[E], cplx<typename PL::Scalar>* sm, int t,
                                             const FFTDesc<typename PL::Scalar>& d, TmemTwCache tc) {
    if constexpr (TWC)
      PL::fft_tc(v, sm, t, d, tc);
    else
      PL::fft(v, sm, t, d);
  }
};

template <class PL, int MAXT, int MINB, bool TWC = false>
__global__ void __launch_bounds__(MAXT, MINB) k_col_fwd_tma(ColFwdArgs a, FFTDesc<typename PL::Scalar> d) {
  using TCC = TwCache<PL, TWC>;
  using T = typename PL::Scalar;
  using V = cplx<T>;
  constexpr int E = PL::E, NT = PL::NT, L = PL::L;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int Ls = (PL::slots(L) + 1) & ~1;  // keep the TMA staging buffers 16-byte aligned
  V* sm = reinterpret_cast<V*>(smraw);
  V* sbuf = sm + Ls;
  V* ybuf = sbuf + L;
  const int nv = a.nvalid;
  uint64_t* bars = reinterpret_cast<uint64_t*>(ybuf + ((nv + 1) & ~1));
  uint32_t* taddr_s = reinterpret_cast<uint32_t*>(bars + 2);
  const int t = threadIdx.x;
  TCC::alloc(taddr_s, t);
  const int kx = blockIdx.x, b = blockIdx.y;
  // layer split (gridDim.z > 1): this CTA sums layers [r0, r1) and adds its
  // part of W atomically (two splits onto a zeroed W: exact and order-free)
  const int r0 = (a.K * (int)blockIdx.z) / (int)gridDim.z, K = (a.K * ((int)blockIdx.z + 1)) / (int)gridDim.z - r0;
  const uint32_t ybytes = nv * sizeof(V), sbytes = L * sizeof(V);
  const V* Yb = static_cast<const V*>(a.Y) + (long long)b * a.y_bstride + (long long)kx * a.ldy + (long long)r0 * a.y_rstride;
  const V* Sb = static_cast<const V*>(a.S) + (long long)kx * a.lds + (long long)r0 * a.s_rstride;
  const uint64_t pol = policy_evict_first();
  // a batch (gridDim.y models, e.g. BASELINE C5's 64) re-reads every spectrum
  // column once per model: keep the spectra in L2 then (C5: 33.7 MB; with
  // evict-first they were re-read from DRAM per model, ncu L2 hit rate 2%)
  const uint64_t spol = gridDim.y > 1 ? policy_evict_last() : pol;
  if (t == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(&bars[0], ybytes);
    tma_load(ybuf, Yb, ybytes, &bars[0], pol);
    mbar_arrive_expect_tx(&bars[1], sbytes);
    tma_load(sbuf, Sb, sbytes, &bars[1], spol);
  }
  __syncthreads();
  const TmemTwCache tc = TCC::setup(taddr_s, t, d);
  V acc[E], v[E];
#pragma unroll
  for (int k = 0; k < E; ++k) acc[k] = mkc<V>(T(0), T(0));
  for (int r = 0; r < K; ++r) {
    mbar_wait(&bars[0], r & 1);
#pragma unroll
    for (int k = 0; k < E; ++k) {
      const int q = t + NT * k;
      v[k] = q < nv ? ybuf[q] : mkc<V>(T(0), T(0));
    }
    __syncthreads();
    if (t == 0 && r + 1 < K) {
      fence_proxy_async();
      mbar_arrive_expect_tx(&bars[0], ybytes);
      tma_load(ybuf, Yb + (long long)(r + 1) * a.y_rstride, ybytes, &bars[0], pol);
    }
    TCC::fft(v, sm, t, d, tc);
    mbar_wait(&bars[1], r & 1);
#pragma unroll
    for (int k = 0; k < E; ++k) {
      const V w = sbuf[t + NT * k];
      acc[k].x += w.x * v[k].x - w.y * v[k].y;
      acc[k].y += w.x * v[k].y + w.y * v[k].x;
    }
    __syncthreads();
    if (t == 0 && r + 1 < K) {
      fence_proxy_async();
      mbar_arrive_expect_tx(&bars[1], sbytes);
      tma_load(sbuf, Sb + (long long)(r + 1) * a.s_rstride, sbytes, &bars[1], spol);
    }
  }
#pragma unroll
  for (int k = 0; k < E; ++k) acc[k] = conjv(acc[k]);
  TCC::fft(acc, sm, t, d, tc);
  TCC::release(taddr_s, t);
  V* wc = static_cast<V*>(a.W) + (long long)b * a.w_bstride + (long long)kx * a.ldw;
#pragma unroll
  for (int k = 0; k < E; ++k) {
    const int j = t + NT * k;
    if (j < a.nout) {
      V val = conjv(acc[k]);
      if (gridDim.z > 1) {
        atomicAdd(&wc[j].x, val.x);
        atomicAdd(&wc[j].y, val.y);
      } else {
        if (a.accumulate) val = val + wc[j];
        wc[j] = val;
      }
    }
  }
}

template <class PL, int MAXT, int MINB, bool TWC = false>
__global__ void __launch_bounds__(MAXT, MINB) k_col_tra_tma(ColTraArgs a, FFTDesc<typename PL::Scalar> d) {
  using TCC = TwCache<PL, TWC>;
  using T = typename PL::Scalar;
  using V = cplx<T>;
  constexpr int E = PL::E, NT = PL::NT, L = PL::L;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int Ls = (PL::slots(L) + 1) & ~1;  // keep the TMA staging buffers 16-byte aligned
  V* sm = reinterpret_cast<V*>(smraw);
  V* sbuf = sm + Ls;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sbuf + L);
  uint32_t* taddr_s = reinterpret_cast<uint32_t*>(bars + 1);
  const int t = threadIdx.x;
  TCC::alloc(taddr_s, t);
  const int kx = blockIdx.x, b = blockIdx.y;
  const int r0 = (a.K * (int)blockIdx.z) / (int)gridDim.z, K = (a.K * ((int)blockIdx.z + 1)) / (int)gridDim.z - r0;
  const uint32_t sbytes = L * sizeof(V);
  const V* Sb = static_cast<const V*>(a.S) + (long long)kx * a.lds + (long long)r0 * a.s_rstride;
  const uint64_t pol = policy_evict_first();
  // a batch (gridDim.y models, e.g. BASELINE C5's 64) re-reads every spectrum
  // column once per model: keep the spectra in L2 then (C5: 33.7 MB; with
  // evict-first they were re-read from DRAM per model, ncu L2 hit rate 2%)
  const uint64_t spol = gridDim.y > 1 ? policy_evict_last() : pol;
  if (t == 0) {
    mbar_init(&bars[0], 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(&bars[0], sbytes);
    tma_load(sbuf, Sb, sbytes, &bars[0], spol);
  }
  V dh[E], v[E];
  const V* dc = static_cast<const V*>(a.D) + (long long)b * a.d_bstride + (long long)kx * a.ldd;
#pragma unroll
  for (int k = 0; k < E; ++k) {
    const int j = t + NT * k;
    dh[k] = j < a.nvalid ? dc[j] : mkc<V>(T(0), T(0));
  }
  __syncthreads();
  const TmemTwCache tc = TCC::setup(taddr_s, t, d);
  TCC::fft(dh, sm, t, d, tc);
  V* Wb = static_cast<V*>(a.W) + (long long)b * a.w_bstride + (long long)kx * a.ldw +
          (long long)r0 * a.w_rstride;
  const long long qstride = 1;
  for (int r = 0; r < K; ++r) {
    mbar_wait(&bars[0], r & 1);
#pragma unroll
    for (int k = 0; k < E; ++k) {
      // conj(conj(S) * dh) = S * conj(dh): inverse FFT via the conjugation identity
      const V w = sbuf[t + NT * k];
      v[k] = mkc<V>(w.x * dh[k].x + w.y * dh[k].y, w.y * dh[k].x - w.x * dh[k].y);
    }
    __syncthreads();
    if (t == 0 && r + 1 < K) {
      fence_proxy_async();
      mbar_arrive_expect_tx(&bars[0], sbytes);
      tma_load(sbuf, Sb + (long long)(r + 1) * a.s_rstride, sbytes, &bars[0], spol);
    }
    TCC::fft(v, sm, t, d, tc);
    V* wc = Wb + (long long)r * a.w_rstride;
#pragma unroll
    for (int k = 0; k < E; ++k) {
      const int q = t + NT * k;
      if (q < a.nout) wc[q * qstride] = conjv(v[k]);
    }
  }
  TCC::release(taddr_s, t);
}

// ---------------------------------------------------------------------------
// TMEM variants of the TMA column stages (fp64 plans whose team is not a whole
// number of warps, e.g. L=2000: 100 threads).  The per-thread E-element
// accumulator (forward) or data spectrum (transpose) -- 80 registers in fp64
// -- lives in tensor memory, which this workload otherwise leaves idle; the
// CTA is padded to whole warps (helper lanes follow the control flow and
// barriers, touch no shared memory) as tcgen05 ld/st are warp-collective.
// With registers freed and the Y column loaded straight from global, three
// CTAs fit per SM instead of two.  Shared: [exchange][spectrum L][mbarrier][tmem addr].
// ---------------------------------------------------------------------------
template <class PL> struct TmemCfg {
  static constexpr int NTR = (PL::NT + 31) / 32 * 32;
  static constexpr int COLS = PL::E * 4;  // fp64 complex = 4 x 32-bit columns
  static constexpr int GROUPS = COLS / 16;
  static constexpr int NCOLS = COLS <= 32 ? 32 : COLS <= 64 ? 64 : COLS <= 128 ? 128 : COLS <= 256 ? 256 : 512;
  static_assert(COLS % 16 == 0, "TMEM groups of 16 columns = 4 complex");
};

__device__ __forceinline__ void split4(double2 a, uint32_t* r) {
  r[0] = (uint32_t)__double2loint(a.x);
  r[1] = (uint32_t)__double2hiint(a.x);
  r[2] = (uint32_t)__double2loint(a.y);
  r[3] = (uint32_t)__double2hiint(a.y);
}
__device__ __forceinline__ double2 join4(const uint32_t* r) {
  return make_double2(__hiloint2double((int)r[1], (int)r[0]), __hiloint2double((int)r[3], (int)r[2]));
}

template <class PL, int MINB>
__global__ void __launch_bounds__(TmemCfg<PL>::NTR, MINB) k_col_tra_tmem(ColTraArgs a, FFTDesc<double> d) {
  using V = double2;
  using TC = TmemCfg<PL>;
  constexpr int E = PL::E, NT = PL::NT, L = PL::L;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int Ls = (PL::slots(L) + 1) & ~1;
  V* sm = reinterpret_cast<V*>(smraw);
  V* sbuf = sm + Ls;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sbuf + L);
  uint32_t* taddr_s = reinterpret_cast<uint32_t*>(bar + 1);
  const int t = threadIdx.x, warp = t / 32;
  const bool active = t < NT;
  const int kx = blockIdx.x, b = blockIdx.y;
  const int r0 = (a.K * (int)blockIdx.z) / (int)gridDim.z, K = (a.K * ((int)blockIdx.z + 1)) / (int)gridDim.z - r0;
  const uint32_t sbytes = L * sizeof(V);
  const V* Sb = static_cast<const V*>(a.S) + (long long)kx * a.lds + (long long)r0 * a.s_rstride;
  const uint64_t pol = policy_evict_first();
  // a batch (gridDim.y models, e.g. BASELINE C5's 64) re-reads every spectrum
  // column once per model: keep the spectra in L2 then (C5: 33.7 MB; with
  // evict-first they were re-read from DRAM per model, ncu L2 hit rate 2%)
  const uint64_t spol = gridDim.y > 1 ? policy_evict_last() : pol;
  if (warp == 0) tmem_alloc<TC::NCOLS>(taddr_s);
  if (t == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(bar, sbytes);
    tma_load(sbuf, Sb, sbytes, bar, spol);
  }
  V v[E];
  const V* dc = static_cast<const V*>(a.D) + (long long)b * a.d_bstride + (long long)kx * a.ldd;
#pragma unroll
  for (int k = 0; k < E; ++k) {
    const int j = t + NT * k;
    v[k] = active && j < a.nvalid ? dc[j] : mkc<V>(0.0, 0.0);
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t ta = *taddr_s + ((uint32_t)(32 * (warp & 3)) << 16);
  PL::fft_masked(v, sm, t, d, active);
#pragma unroll
  for (int g = 0; g < TC::GROUPS; ++g) {  // the data spectrum, read once per layer below
    uint32_t u[16];
#pragma unroll
    for (int c = 0; c < 4; ++c) split4(v[4 * g + c], u + 4 * c);
    tmem_st16(ta + 16 * g, u);
  }
  tmem_wait_st();
  V* Wb = static_cast<V*>(a.W) + (long long)b * a.w_bstride + (long long)kx * a.ldw +
          (long long)r0 * a.w_rstride;
  const long long qstride = 1;
  for (int r = 0; r < K; ++r) {
    mbar_wait(bar, r & 1);
#pragma unroll
    for (int g = 0; g < TC::GROUPS; ++g) {
      uint32_t u[16];
      tmem_ld16(ta + 16 * g, u);
      tmem_wait_ld();
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int k = 4 * g + c;
        const V h = join4(u + 4 * c);
        // conj(conj(S) * dh) = S * conj(dh): inverse FFT via the conjugation identity
        const V w = active ? sbuf[t + NT * k] : mkc<V>(0.0, 0.0);
        v[k] = mkc<V>(w.x * h.x + w.y * h.y, w.y * h.x - w.x * h.y);
      }
    }
    __syncthreads();
    if (t == 0 && r + 1 < K) {
      fence_proxy_async();
      mbar_arrive_expect_tx(bar, sbytes);
      tma_load(sbuf, Sb + (long long)(r + 1) * a.s_rstride, sbytes, bar, spol);
    }
    PL::fft_masked(v, sm, t, d, active);
    if (active) {
      V* wc = Wb + (long long)r * a.w_rstride;
#pragma unroll
      for (int k = 0; k < E; ++k) {
        const int q = t + NT * k;
        if (q < a.nout) wc[q * qstride] = conjv(v[k]);
      }
    }
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if (warp == 0) tmem_dealloc<TC::NCOLS>(*taddr_s);
}

// ---------------------------------------------------------------------------
// Row passes with tensor-TMA transposed tiles (compile-time plans, one row
// pair per CTA).  The pair's half spectra form a [kx][2 rows] box of the
// transposed intermediate; it is staged in shared memory and moved by
// cp.async.bulk.tensor (store for R2C, load for C2R) instead of one
// 16-byte access per lane into a different L2 line.
// Shared layout: [exchange Lsa][stage Hx x 2 complex][mbarrier].
// ---------------------------------------------------------------------------
constexpr int kBoxKx = 256;  // TMA box extent along kx (hardware maximum)

template <class V> __host__ __device__ __forceinline__ int stage_offset(int slots) {
  // 128-byte aligned start of the staging tile
  const int per = 128 / (int)sizeof(V);
  return (slots + per - 1) / per * per;
}

// The staging tile lives in the exchange buffer itself: the separated values
// are first gathered into the registers the finished FFT no longer needs,
// then written as the [kx][2 rows] box -> one team buffer per CTA (36 KB for
// fp64 L=2000), four CTAs per SM.
template <class PL> struct RowTile {
  static constexpr int HX = PL::L / 2 + 1;
  static constexpr int NI = (HX + PL::NT - 1) / PL::NT;  // kx items per thread
  static constexpr int BOXK = HX < kBoxKx ? HX : kBoxKx;  // box extent along kx (the tensor map's)
  static constexpr int NBOX = (HX + BOXK - 1) / BOXK;
  static constexpr int PER = 128 / (int)sizeof(cplx<typename PL::Scalar>);
  // kx extent of the staged boxes, rounded to 128 bytes (the [kx][2 rows]
  // tile holds 2 * SPAN complex values)
  static constexpr int SPAN = (NBOX * BOXK + PER - 1) / PER * PER;
  // shared slots (complex) of one team: exchange buffer or staged box, whichever
  // is larger, rounded to 128 bytes (tensor-TMA shared addresses are 128-B aligned)
  static constexpr int slots(int exchange_slots) {
    const int n = exchange_slots > 2 * SPAN ? exchange_slots : 2 * SPAN;
    return (n + PER - 1) / PER * PER;
  }
};

// QUAD (two teams): the CTA's four rows leave as ONE [kx][4 rows] box, so the
// box rows are 32 bytes in fp32 (full L2 sectors) instead of 16.
template <class PL, int MAXT, int MINB, int TEAMS, bool QUAD = false>
__global__ void __launch_bounds__(MAXT, MINB)
    k_row_r2c_t2d(RowR2CArgs a, FFTDesc<typename PL::Scalar> d, const __grid_constant__ CUtensorMap omap) {
  static_assert(!QUAD || TEAMS == 2, "a four-row box takes two teams");
  using T = typename PL::Scalar;
  using V = cplx<T>;
  using RT = RowTile<PL>;
  constexpr int E = PL::E, NT = PL::NT, L = PL::L, HX = RT::HX;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int c = TEAMS > 1 ? threadIdx.x / NT : 0;
  V* sm = reinterpret_cast<V*>(smraw) + (long long)c * RT::slots((PL::slots(L) + 1) & ~1);
  const int t = threadIdx.x - c * NT, s = blockIdx.y, qa = 2 * (blockIdx.x * TEAMS + c), qb = qa + 1;
  const bool active = qa < a.nrows;
  const T* in = static_cast<const T*>(a.in) + (long long)((unsigned)s / (unsigned)a.spb) * a.in_bstride +
                (long long)((unsigned)s % (unsigned)a.spb) * a.in_sstride;
  const bool vb = qb < a.nrows;
  const T* ra = in + (long long)(active ? qa : 0) * a.ld_in;
  const T* rb = in + (long long)(vb ? qb : qa) * a.ld_in;
  V v[E];
  // one compare per load: the row's valid length is 0 for a missing row
  const int na = active ? a.nvalid : 0, nb = vb ? a.nvalid : 0;
#pragma unroll
  for (int k = 0; k < E; ++k) {
    const int i = t + NT * k;
    v[k] = mkc<V>(i < na ? __ldcs(ra + i) : T(0), i < nb ? __ldcs(rb + i) : T(0));
  }
  const T h = T(0.5);
  if constexpr (PL::kR16x16x8 && PL::kPerPass && BTTB_R2C_PAIR) {
    // Mirrored last pass: thread t runs the radix-8 butterflies j0 = t and
    // j1 = 256 - t (t = 0: 128) instead of t and t + 128, so it ends up holding
    // Z[k] AND Z[L - k] (L - (j0 + 256 r) = j1 + 256 (7 - r)) and separates the
    // two real rows in registers -- no exchange-buffer store / reload of the
    // whole spectrum before the tile is staged.
    sfft<T, E, L, PL::kPad, true, 0, 1, 16, 16>(v, sm, t, PL::table(d));
    __syncthreads();
    spass_store<T, E, 16, 16, NT, PL::kPad>(v, sm, t);
    __syncthreads();
    const int j1 = t == 0 ? 128 : 256 - t;
    V u0[8], u1[8];
#pragma unroll
    const int s0 = pad_slot<PL::kPad>(t), s1 = pad_slot<PL::kPad>(j1);
    for (int r = 0; r < 8; ++r) {
      u0[r] = sm[pad_slot_at<PL::kPad, 256>(s0, t, r)];
      u1[r] = sm[pad_slot_at<PL::kPad, 256>(s1, j1, r)];
    }
    V w[8];
    gen_twiddles<V, 8, 256>(w, PL::table(d) + 15 * 16, t);  // w[r] = w_2048^(r t)
    sfor<1, 8>([&](auto rc) {
      constexpr int r = decltype(rc)::value;
      u0[r] = cmul(u0[r], w[r]);
      // w^(r (256 - t)) = w_8^r conj(w^(r t)); t = 0 pairs with j1 = 128: w_16^r
      u1[r] = t == 0 ? twc<16, r>(u1[r]) : twc<8, r>(cmul(u1[r], conjv(w[r])));
    });
    dft<8>(u0);
    dft<8>(u1);  // u0[r] = Z[t + 256 r], u1[r] = Z[j1 + 256 r]
    __syncthreads();  // every thread has read its inputs: the tile may overwrite the buffer
    auto put = [&](int kx, V zk, V zm) {
      const V A = mkc<V>(h * (zk.x + zm.x), h * (zk.y - zm.y));
      const V B = mkc<V>(h * (zk.y + zm.y), h * (zm.x - zk.x));
      if constexpr (QUAD) {
        V* stage = reinterpret_cast<V*>(smraw);
        stage[4 * kx + 2 * c] = A;
        stage[4 * kx + 2 * c + 1] = B;
      } else {
        sm[2 * kx] = A;
        sm[2 * kx + 1] = B;
      }
    };
    if (t == 0) {
#pragma unroll
      for (int r = 0; r <= 4; ++r) put(256 * r, u0[r], u0[(8 - r) & 7]);
#pragma unroll
      for (int r = 0; r < 4; ++r) put(128 + 256 * r, u1[r], u1[7 - r]);
    } else {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        put(t + 256 * r, u0[r], u1[7 - r]);
        put(256 - t + 256 * r, u1[r], u0[7 - r]);
      }
    }
  } else {
  PL::fft(v, sm, t, d);
  __syncthreads();
#pragma unroll
  for (int k = 0; k < E; ++k) sm[PL::slot(t + NT * k)] = v[k];
  __syncthreads();
  // Separation, one stage element per lane: element e of the team's [kx][2]
  // tile is A (e even) or B (e odd) of kx = e/2, so a warp's tile stores are
  // contiguous 16-byte lanes (the [kx] x {A, B} pairs at a 32-byte stride cost
  // twice the shared-memory wavefronts); the two lanes of a kx read the same
  // zk / zm (broadcast).
  constexpr int NE = (2 * HX + NT - 1) / NT;
  V P[NE];
#pragma unroll
  for (int i = 0; i < NE; ++i) {
    const int e = t + NT * i, kx = e >> 1;
    if (kx < HX) {
      const V zk = sm[PL::slot(kx)];
      const V zm = sm[PL::slot(kx == 0 ? 0 : L - kx)];
      const bool odd = e & 1;
      P[i] = mkc<V>(h * (odd ? zk.y + zm.y : zk.x + zm.x), h * (odd ? zm.x - zk.x : zk.y - zm.y));
    }
  }
  __syncthreads();
  if constexpr (QUAD) {
    V* stage = reinterpret_cast<V*>(smraw);
#pragma unroll
    for (int i = 0; i < NE; ++i) {
      const int e = t + NT * i;
      if (e < 2 * HX) stage[4 * (e >> 1) + 2 * c + (e & 1)] = P[i];
    }
  } else {
#pragma unroll
    for (int i = 0; i < NE; ++i) {
      const int e = t + NT * i;
      if (e < 2 * HX) sm[e] = P[i];
    }
  }
  }
  if constexpr (QUAD) {
    V* stage = reinterpret_cast<V*>(smraw);
    fence_proxy_async();
    __syncthreads();
    if (threadIdx.x == 0 && 4 * (int)blockIdx.x < a.nrows) {
      for (int kx0 = 0; kx0 < HX; kx0 += RT::BOXK) tma_store_3d(&omap, stage + 4 * kx0, 8 * blockIdx.x, kx0, s);
      tma_store_commit();
      tma_store_wait_read();
    }
  } else {
    fence_proxy_async();
    __syncthreads();
    if (t == 0 && active) {
      for (int kx0 = 0; kx0 < HX; kx0 += RT::BOXK) tma_store_3d(&omap, sm + 2 * kx0, 2 * qa, kx0, s);
      tma_store_commit();
      tma_store_wait_read();
    }
  }
}

// The FFT input is read straight from the staged tile: element n of the
// packed row pair is z[n] = A[n] + i B[n] (n <= L/2) or conj(A[L-n]) +
// i conj(B[L-n]) (Hermitian half), so no intermediate exchange-buffer pass.
template <class PL, int MAXT, int MINB, int TEAMS, bool QUAD = false>
__global__ void __launch_bounds__(MAXT, MINB)
    k_row_c2r_t2d(RowC2RArgs a, FFTDesc<typename PL::Scalar> d, const __grid_constant__ CUtensorMap imap) {
  static_assert(!QUAD || TEAMS == 2, "a four-row box takes two teams");
  using T = typename PL::Scalar;
  using V = cplx<T>;
  using RT = RowTile<PL>;
  constexpr int E = PL::E, NT = PL::NT, L = PL::L, HX = RT::HX, NBOX = RT::NBOX;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int tslots = RT::slots((PL::slots(L) + 1) & ~1);
  const int c = TEAMS > 1 ? threadIdx.x / NT : 0;
  V* sm = reinterpret_cast<V*>(smraw) + (long long)c * tslots;
  uint64_t* bar = reinterpret_cast<uint64_t*>(reinterpret_cast<V*>(smraw) + (long long)TEAMS * tslots) + c;
  const int t = threadIdx.x - c * NT, s = blockIdx.y, ja = 2 * (blockIdx.x * TEAMS + c), jb = ja + 1;
  const bool active = ja < a.nrows;
  // A[n] at sA[n * st], B[n] at sB[n * st]
  const V* sA;
  const V* sB;
  int st;
  if constexpr (QUAD) {
    V* stage = reinterpret_cast<V*>(smraw);
    uint64_t* bar0 = reinterpret_cast<uint64_t*>(reinterpret_cast<V*>(smraw) + (long long)TEAMS * tslots);
    if (threadIdx.x == 0) {
      mbar_init(bar0, 1);
      fence_mbar_init();
      mbar_arrive_expect_tx(bar0, (uint32_t)(NBOX * RT::BOXK * 4 * sizeof(V)));
      for (int b = 0; b < NBOX; ++b) tma_load_3d(stage + 4 * b * RT::BOXK, &imap, 8 * blockIdx.x, b * RT::BOXK, s, bar0);
    }
    __syncthreads();
    mbar_wait(bar0, 0);
    sA = stage + 2 * c;  // out-of-range rows arrive zero-filled
    sB = stage + 2 * c + 1;
    st = 4;
  } else {
    if (t == 0 && active) {
      mbar_init(bar, 1);
      fence_mbar_init();
      // every box delivers its full extent (out-of-range rows zero-filled)
      mbar_arrive_expect_tx(bar, (uint32_t)(NBOX * RT::BOXK * 2 * sizeof(V)));
      for (int b = 0; b < NBOX; ++b) tma_load_3d(sm + 2 * b * RT::BOXK, &imap, 2 * ja, b * RT::BOXK, s, bar);
    }
    __syncthreads();
    if (active) mbar_wait(bar, 0);
    sA = sm;
    sB = sm + 1;
    st = 2;
  }
  V v[E];
#pragma unroll
  for (int k = 0; k < E; ++k) {
    const int n = t + NT * k;
    const bool lo = n < HX;
    const int m = lo ? n : L - n;
    V a0 = sA[m * st], b0 = sB[m * st];
    if (m == 0 || 2 * m == L) {  // Hermitian projection (.real semantics)
      a0.y = T(0);
      b0.y = T(0);
    }
    // conj of z[n]: the inverse FFT runs as conj(fft(conj(.)))
    v[k] = lo ? mkc<V>(a0.x - b0.y, -(a0.y + b0.x)) : mkc<V>(a0.x + b0.y, a0.y - b0.x);
  }
  PL::fft(v, sm, t, d);
  const bool vb = jb < a.nrows;
  T* out = static_cast<T*>(a.out) + (long long)((unsigned)s / (unsigned)a.spb) * a.out_bstride +
           (long long)((unsigned)s % (unsigned)a.spb) * a.out_sstride;
  T* oa = out + (long long)(active ? ja : 0) * a.ld_out;
  T* ob = out + (long long)(vb ? jb : ja) * a.ld_out;
  const int na = active ? a.nout : 0, nb = vb ? a.nout : 0;  // one compare per store
#pragma unroll
  for (int k = 0; k < E; ++k) {
    const int i = t + NT * k;
    if (i < na) __stcs(oa + i, v[k].x);
    if (i < nb) __stcs(ob + i, -v[k].y);
  }
}

// C2R with a MIRRORED first pass (L = 2048): the inverse runs as the radix
// order 8/16/16 (plan PLC, per-pass twiddles in a.tw_816), whose first radix-8
// pass has two butterflies per thread; thread t takes j = t and j = 256 - t
// (t = 0: 128), whose inputs are mirror images (L - (t + 256 r) = (256 - t) +
// 256 (7 - r)).  So each staged (A[n], B[n]) pair is read ONCE and yields
// both z[n] = A + iB and z[L-n] = conj(A) + i conj(B) in registers (the
// direct-read kernel above reads every tile element twice).
template <class PL, class PLC, int MAXT, int MINB, int TEAMS, bool QUAD>
__global__ void __launch_bounds__(MAXT, MINB)
    k_row_c2r_mirror(RowC2RArgs a, FFTDesc<typename PL::Scalar> d, const __grid_constant__ CUtensorMap imap) {
  static_assert(!QUAD || TEAMS == 2, "a four-row box takes two teams");
  static_assert(PLC::L == 2048 && PLC::E == 16 && PL::L == 2048, "mirrored C2R: 2048-point plans");
  using T = typename PL::Scalar;
  using V = cplx<T>;
  using RT = RowTile<PL>;
  constexpr int E = PLC::E, NT = PLC::NT, L = PLC::L, NBOX = RT::NBOX, PADC = PLC::kPad;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int tslots = RT::slots((PLC::slots(L) + 1) & ~1);
  const int c = TEAMS > 1 ? threadIdx.x / NT : 0;
  V* sm = reinterpret_cast<V*>(smraw) + (long long)c * tslots;
  uint64_t* bar = reinterpret_cast<uint64_t*>(reinterpret_cast<V*>(smraw) + (long long)TEAMS * tslots) + c;
  const int t = threadIdx.x - c * NT, s = blockIdx.y, ja = 2 * (blockIdx.x * TEAMS + c), jb = ja + 1;
  const bool active = ja < a.nrows;
  const V* sA;
  const V* sB;
  int st;
  if constexpr (QUAD) {
    V* stage = reinterpret_cast<V*>(smraw);
    uint64_t* bar0 = reinterpret_cast<uint64_t*>(reinterpret_cast<V*>(smraw) + (long long)TEAMS * tslots);
    if (threadIdx.x == 0) {
      mbar_init(bar0, 1);
      fence_mbar_init();
      mbar_arrive_expect_tx(bar0, (uint32_t)(NBOX * RT::BOXK * 4 * sizeof(V)));
      for (int b = 0; b < NBOX; ++b) tma_load_3d(stage + 4 * b * RT::BOXK, &imap, 8 * blockIdx.x, b * RT::BOXK, s, bar0);
    }
    __syncthreads();
    mbar_wait(bar0, 0);
    sA = stage + 2 * c;
    sB = stage + 2 * c + 1;
    st = 4;
  } else {
    if (t == 0 && active) {
      mbar_init(bar, 1);
      fence_mbar_init();
      mbar_arrive_expect_tx(bar, (uint32_t)(NBOX * RT::BOXK * 2 * sizeof(V)));
      for (int b = 0; b < NBOX; ++b) tma_load_3d(sm + 2 * b * RT::BOXK, &imap, 2 * ja, b * RT::BOXK, s, bar);
    }
    __syncthreads();
    if (active) mbar_wait(bar, 0);
    sA = sm;
    sB = sm + 1;
    st = 2;
  }
  // conj(z[n]) and conj(z[L-n]) from one staged pair (the inverse runs as
  // conj(fft(conj(.)))); n = 0 and n = L/2 are their own mirrors and get the
  // Hermitian projection (.real semantics)
  auto zpair = [&](int n, V& zn, V& zm) {
    V a0 = sA[n * st], b0 = sB[n * st];
    if (n == 0 || 2 * n == L) {
      a0.y = T(0);
      b0.y = T(0);
    }
    zn = mkc<V>(a0.x - b0.y, -(a0.y + b0.x));
    zm = mkc<V>(a0.x + b0.y, a0.y - b0.x);
  };
  const int j1 = t == 0 ? 128 : 256 - t;
  V u0[8], u1[8];
  if (t == 0) {
#pragma unroll
    for (int r = 0; r <= 4; ++r) {
      V zn, zm;
      zpair(256 * r, zn, zm);
      u0[r] = zn;
      if (r != 0 && r != 4) u0[8 - r] = zm;
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) zpair(128 + 256 * r, u1[r], u1[7 - r]);
  } else {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      zpair(t + 256 * r, u0[r], u1[7 - r]);
      zpair(256 - t + 256 * r, u1[r], u0[7 - r]);
    }
  }
  dft<8>(u0);  // pass 1 (NS = 1): no twiddles
  dft<8>(u1);
  __syncthreads();  // every thread has read the tile: the exchange may overwrite it
  // 8 consecutive slots from a multiple of 8 never cross a pad boundary (PADC = 8 or 16)
  static_assert(PADC % 8 == 0, "mirrored C2R: pad of the 8/16/16 exchanges");
  const int q0 = pad_slot<PADC>(8 * t), q1 = pad_slot<PADC>(8 * j1);
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    sm[q0 + r] = u0[r];
    sm[q1 + r] = u1[r];
  }
  __syncthreads();
  V v[E];
  const int t0 = pad_slot<PADC>(t);
#pragma unroll
  for (int k = 0; k < E; ++k) v[k] = sm[pad_slot_at<PADC, NT>(t0, t, k)];
  sfft<T, E, L, PADC, true, 0, 8, 16, 16>(v, sm, t, static_cast<const V*>(a.tw_816));
  const bool vb = jb < a.nrows;
  T* out = static_cast<T*>(a.out) + (long long)((unsigned)s / (unsigned)a.spb) * a.out_bstride +
           (long long)((unsigned)s % (unsigned)a.spb) * a.out_sstride;
  T* oa = out + (long long)(active ? ja : 0) * a.ld_out;
  T* ob = out + (long long)(vb ? jb : ja) * a.ld_out;
  const int na = active ? a.nout : 0, nb = vb ? a.nout : 0;  // one compare per store
#pragma unroll
  for (int k = 0; k < E; ++k) {
    const int i = t + NT * k;
    if (i < na) __stcs(oa + i, v[k].x);
    if (i < nb) __stcs(ob + i, -v[k].y);
  }
}

// ---------------------------------------------------------------------------
// Spectrum build, column stage (fp64 FFT, stored as TS, scaled)
// ---------------------------------------------------------------------------
template <class PL, class TS, int MAXT, int MINB>
__global__ void __launch_bounds__(MAXT, MINB) k_col_spec(ColSpecArgs a, FFTDesc<double> d, int C) {
  using V = double2;
  using VS = cplx<TS>;
  constexpr int E = PL::E;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int nt = PL::nt(d), Ls = PL::slots(d.L);
  const int tid = threadIdx.x, c = tid / nt, t = tid - c * nt;
  const int kx = blockIdx.x * C + c;
  const bool kv = kx < a.Hx;
  const int kxc = kv ? kx : 0;
  V* sm = reinterpret_cast<V*>(smraw) + (long long)c * Ls;
  V v[E];
  const V* yc = static_cast<const V*>(a.Y) + (long long)kxc * a.ldy;
#pragma unroll
  for (int k = 0; k < E; ++k) v[k] = yc[t + nt * k];
  PL::fft(v, sm, t, d);
  if (kv) {
    VS* sc = static_cast<VS*>(a.S) + (long long)kx * a.lds;
#pragma unroll
    for (int k = 0; k < E; ++k) sc[t + nt * k] = mkc<VS>((TS)(v[k].x * a.scale), (TS)(v[k].y * a.scale));
  }
}

// ---------------------------------------------------------------------------
// plan registry: compile-time plans for the BASELINE lengths (PAD from
// tools/bank_search.py), runtime-radix plans for every other supported length
// ---------------------------------------------------------------------------
template <class P> struct Tag { using type = P; };

// COL selects the plan of the accumulating column kernels where it differs
// (fp64 L=2000: 10 elements per thread keeps the E-element accumulator cheap)
template <class T, bool COL = false, bool ROW = false, class F>
cudaError_t with_plan(int L, int E, F&& f) {
  if constexpr (sizeof(T) == 8) {
    switch (L) {
      case 2048: return f(Tag<SPlan<double, 16, 16, 16, 16, 8>>{});
      case 2000: return f(Tag<SPlan<double, 20, 20, 20, 20, 5>>{});
      case 512: return f(Tag<SPlan<double, 8, 8, 8, 8, 8>>{});
      case 432: return f(Tag<SPlan<double, 12, 12, 12, 12, 3>>{});
      case 384: return f(Tag<SPlan<double, 12, 24, 12, 4, 4, 2>>{});
      case 100: return f(Tag<SPlan<double, 20, 12, 20, 5>>{});
      case 80: return f(Tag<SPlan<double, 20, 10, 20, 4>>{});
      default: break;
    }
    const bool big = L / E > 256;
    switch (E) {
      case 8: return big ? f(Tag<DPlan<double, 8, 1024>>{}) : f(Tag<DPlan<double, 8, 256>>{});
      case 12: return big ? f(Tag<DPlan<double, 12, 1024>>{}) : f(Tag<DPlan<double, 12, 256>>{});
      case 10: return big ? f(Tag<DPlan<double, 10, 1024>>{}) : f(Tag<DPlan<double, 10, 256>>{});
      default: return cudaErrorInvalidValue;
    }
  } else {
    switch (L) {
      case 2048: return f(Tag<SPlan<float, 16, 16, 16, 16, 8>>{});
      case 2000: return f(Tag<SPlan<float, 20, 80, 20, 20, 5>>{});
      case 512: return f(Tag<SPlan<float, 8, 16, 8, 8, 8>>{});
      case 432: return f(Tag<SPlan<float, 12, 36, 12, 12, 3>>{});
      case 384: return f(Tag<SPlan<float, 12, 48, 12, 4, 4, 2>>{});
      case 100: return f(Tag<SPlan<float, 20, 10, 20, 5>>{});
      case 80: return f(Tag<SPlan<float, 20, 10, 20, 4>>{});
      default: break;
    }
    const bool big = L / E > 256;
    switch (E) {
      case 8: return big ? f(Tag<DPlan<float, 8, 1024>>{}) : f(Tag<DPlan<float, 8, 256>>{});
      case 12: return big ? f(Tag<DPlan<float, 12, 1024>>{}) : f(Tag<DPlan<float, 12, 256>>{});
      case 20: return big ? f(Tag<DPlan<float, 20, 1024>>{}) : f(Tag<DPlan<float, 20, 256>>{});
      default: return cudaErrorInvalidValue;
    }
  }
}

// Radix sequence of the registered compile-time plan of (L, dtype), for the
// host to build that plan's per-pass twiddle tables; 0 if none.
int static_radices(int L, bool fp64, int* out) {
  int n = 0;
  auto take = [&](auto tag) {
    using PL = typename decltype(tag)::type;
    if constexpr (PL::kStatic) {
      n = radix_list(PL{}, out);
    }
    return cudaSuccess;
  };
  if (fp64) with_plan<double>(L, 0, take); else with_plan<float>(L, 0, take);
  return n;
}

}  // namespace bttb
namespace bttb {

// Fixed launch shapes of the compile-time plans: teams per CTA and the
// register target that sets __launch_bounds__ min-blocks (fp64 column kernels
// keep an E-element accumulator, hence the larger budget).
template <class PL> struct Shape {
  using T = typename PL::Scalar;
  static constexpr int NT = PL::NT;
  static constexpr int row_pairs = PL::kStatic ? (128 / (2 * NT) > (sizeof(T) == 8 ? 1 : 2) ? 128 / (2 * NT) : (sizeof(T) == 8 ? 1 : 2)) : 0;
  static constexpr int col_teams = PL::kStatic ? (128 / NT > 1 ? 128 / NT : 1) : 0;
  static constexpr int row_threads = PL::kStatic ? row_pairs * NT : NT;
  static constexpr int col_threads = PL::kStatic ? col_teams * NT : NT;
  static constexpr int warps(int threads) { return (threads + 31) / 32; }
  static constexpr int minb(int threads, int regs) {
    return 2048 / (warps(threads) * regs) > 1 ? 2048 / (warps(threads) * regs) : 1;
  }
  // register targets: the column kernels keep E-element accumulators beside the data
#ifdef COL_REGS_F64
  static constexpr int col_regs = sizeof(T) == 4 ? COL_REGS_F32 : COL_REGS_F64;
#else
  static constexpr int col_regs = sizeof(T) == 4 ? COL_REGS_F32
                                  : (64 + 4 * PL::E * 2 > 255 ? 255 : 64 + 4 * PL::E * 2);
#endif
  static constexpr int col_regs_rounded =
      col_regs <= 96 ? 96 : col_regs <= 128 ? 128 : (col_regs <= 144 ? 144 : (col_regs <= 168 ? 168 : 255));
  // row passes hold E complex values plus the separated tile: fp32 needs far fewer registers
  static constexpr int row_regs = sizeof(T) == 8 ? ROW_REGS_F64 : ROW_REGS_F32;
  static constexpr int row_minb = PL::kStatic ? minb(row_threads, 128) : 1;
  // fp64 plans with 20 elements per thread keep the column accumulator in
  // shared memory (registers would cap occupancy at two teams per SM)
  static constexpr bool acc_smem = false;  // measured slower on C4 fp64 (10.6 vs 9.8 ms/step)
  static constexpr int col_minb = PL::kStatic ? minb(col_threads, acc_smem ? 168 : col_regs_rounded) : 1;
  static constexpr int spec_minb = PL::kStatic ? minb(col_threads, 128) : 1;
  static constexpr int tma_minb = PL::kStatic ? minb(col_threads, col_regs_rounded) : 1;
  // the TMA transpose column stage stages only the spectrum (exchange + S: 67 KB
  // at fp64 L=2048), so three CTAs fit an SM's shared memory if registers allow:
  // fp64 plans of <= 16 elements run at TRA_REGS_F64 (C4 fp64: 1.95 -> 1.88 ms per
  // transpose at 168; the forward also stages Y, 83 KB, and stays at two CTAs)
  static constexpr int tra_regs =
      (sizeof(T) == 8 && PL::E <= 16 && col_regs_rounded > TRA_REGS_F64) ? TRA_REGS_F64 : col_regs_rounded;
  static constexpr int tra_minb = PL::kStatic ? minb(col_threads, tra_regs) : 1;
  static constexpr int t2d_teams = T2D_TEAMS;
  static constexpr int t2d_minb = PL::kStatic ? minb(T2D_TEAMS * NT, row_regs) : 1;
  static constexpr int quad_minb = PL::kStatic ? minb(2 * NT, row_regs) : 1;
};

bool env_flag(const char* name, bool dflt);

// fp32 row passes move four rows per CTA (32-byte box rows); BTTB_QUAD=0 off
// (fp64 box rows are already full sectors: four-row fp64 boxes measured no gain)
bool quad_rows() {
  static const bool on = !(getenv("BTTB_QUAD") && atoi(getenv("BTTB_QUAD")) == 0);
  return on;
}

// mirrored-first-pass C2R (k_row_c2r_mirror) for the 2048 plans: default on,
// BTTB_C2R_MIRROR=0 falls back to the direct-read kernel
bool c2r_mirror_ok() {
  static const bool on = env_flag("BTTB_C2R_MIRROR", true);
  return on;
}
#define C2R_MIRROR_PAD(T) (sizeof(T) == 8 ? 8 : 16)  // bank-searched pad of the 8/16/16 exchanges

// loop-invariant pass twiddles of the TMA column stages in TMEM (fft.cuh TmemTwCache);
// BTTB_TW_TMEM=0 generates them per transform instead
bool tw_tmem_ok() {
  static const bool on = env_flag("BTTB_TW_TMEM", true);
  return on;
}

bool tma_ok() {
  static const bool ok = getenv("BTTB_NO_TMA") == nullptr;
  return ok;
}

// Dynamic plans: teams per CTA chosen for the most resident threads per SM.
template <class K>
int dyn_teams(K kern, int nt, size_t team_bytes, int max_teams, int min_teams, bool prefer_big) {
  cudaFuncAttributes fa;
  int maxthr = 1024;
  if (cudaFuncGetAttributes(&fa, kern) == cudaSuccess) maxthr = fa.maxThreadsPerBlock;
  int best = 1;
  long best_thr = -1;
  for (int P = 1; P <= 32; ++P) {
    if (P > max_teams && P > min_teams) break;
    if (P * nt > maxthr) break;
    const size_t smem = (size_t)P * team_bytes;
    if (smem > 227 * 1024) break;
    if (set_smem(kern, smem) != cudaSuccess) break;
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, P * nt, smem) != cudaSuccess) break;
    long thr = (long)nb * P * nt;
    if (P < min_teams) thr /= 2;
    if (thr > best_thr || (thr == best_thr && prefer_big)) {
      best = P;
      best_thr = thr;
    }
  }
  return best;
}

template <class PL, class K>
int row_teams(K kern, const FFTDesc<typename PL::Scalar>& d, int nrows) {
  using T = typename PL::Scalar;
  if constexpr (PL::kStatic) return Shape<PL>::row_pairs;
  static std::mutex mu;
  static std::map<std::pair<int, int>, int> cache;
  std::lock_guard<std::mutex> g(mu);
  const auto key = std::make_pair(d.L, (nrows + 1) / 2);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  const int P = dyn_teams(kern, PL::nt(d), (size_t)PL::slots(d.L) * sizeof(cplx<T>), (nrows + 1) / 2,
                          sizeof(T) == 8 ? 1 : 2, true);
  cache[key] = P;
  return P;
}

template <class PL, class K>
int col_teams(K kern, const FFTDesc<typename PL::Scalar>& d, int ncols) {
  using T = typename PL::Scalar;
  if constexpr (PL::kStatic) return Shape<PL>::col_teams;
  static std::mutex mu;
  static std::map<std::pair<int, int>, int> cache;
  std::lock_guard<std::mutex> g(mu);
  const auto key = std::make_pair(d.L, ncols);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  const int C = dyn_teams(kern, PL::nt(d), (size_t)PL::slots(d.L) * sizeof(cplx<T>), ncols, 1, false);
  cache[key] = C;
  return C;
}

inline bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn encode_fn() {
  static EncodeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeFn>(p);
  }();
  return fn;
}

// TMEM-resident column state of the transpose (data spectrum in TMEM) for
// teams that are not whole warps (L = 2000): default on, measured 2.84 vs
// 2.95 ms per C4 fp64 transpose (BTTB_TMEM_TRA=0 off).  The forward variant
// (accumulator in TMEM) measured 2.98 vs 2.60 ms and was removed.
bool env_flag(const char* name, bool dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) != 0 : dflt;
}
bool tmem_tra_ok() {
  static const bool on = env_flag("BTTB_TMEM_TRA", env_flag("BTTB_TMEM", true));
  return on;
}

bool t2d_ok() {
  static const bool ok = tma_ok() && encode_fn() != nullptr && !(getenv("BTTB_T2D") && atoi(getenv("BTTB_T2D")) == 0);
  return ok;
}

// View of a transposed [slab][kx][row] complex array as reals: dims (2*rows, Hx,
// slabs), box (4 reals = 2 rows, 256 kx, 1 slab).
template <class T>
bool encode_rowpair_map(CUtensorMap* m, const void* base, int rows, int Hx, int slabs, long long ld_kx,
                        long long ld_slab, int box_rows = 2) {
  const size_t esz = sizeof(T);
  if (!al16(base) || (ld_kx * 2 * esz) % 16 || (ld_slab * 2 * esz) % 16) return false;
  cuuint64_t dims[3] = {(cuuint64_t)2 * rows, (cuuint64_t)Hx, (cuuint64_t)slabs};
  cuuint64_t strides[2] = {(cuuint64_t)(ld_kx * 2 * esz), (cuuint64_t)(ld_slab * 2 * esz)};
  cuuint32_t box[3] = {(cuuint32_t)(2 * box_rows), (cuuint32_t)(Hx < kBoxKx ? Hx : kBoxKx), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = encode_fn()(m, sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                                 const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// Layer splits of the transpose column stage: each column CTA runs all its
// layers, so Hx CTAs on ~300-450 resident CTAs leave the last wave partly idle;
// splitting a column's layers into s parts (each redoes the cheap data-column
// FFT) multiplies the CTA count.  Output values do not depend on s.  Measured
// on C4 fp64: 2.90 -> 2.79 ms per transpose.  (The forward does not split: its
// halves would have to be summed, and a split measured no faster.)
int layer_splits(long ctas, int layers) {
  static const char* env = getenv("BTTB_LAYER_SPLITS");
  if (env) return atoi(env) > 0 ? atoi(env) : 1;
  int sp = 1;
  while (sp < 4 && ctas * sp < 2000 && layers >= 16 * 2 * sp) sp *= 2;
  return sp;
}

// grid of a persistent kernel: every SM filled to its occupancy, never more CTAs than items
template <class K>
int persistent_grid(K kern, int threads, size_t smem, int items) {
  int nb = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, threads, smem) != cudaSuccess || nb < 1) nb = 1;
  const int g = nb * sm_count();
  return items < g ? items : g;
}

template <class T>
cudaError_t launch_row_r2c(const RowR2CArgs& a, const FFTDesc<T>& d, int E, cudaStream_t st) {
  if (a.nslabs <= 0 || a.nrows <= 0) return cudaSuccess;
  return with_plan<T, false, true>(d.L, E, [&](auto tag) {
    using PL = typename decltype(tag)::type;
    if constexpr (PL::kStatic && PL::NT >= 32) {
      CUtensorMap omap;
      if constexpr (sizeof(T) == 4) {
        if (t2d_ok() && quad_rows() && a.Hx <= 65535 &&
            encode_rowpair_map<T>(&omap, a.out, a.nrows, a.Hx, a.nslabs, a.ld_out, a.out_sstride, 4)) {
          auto kern = k_row_r2c_t2d<PL, 2 * PL::NT, Shape<PL>::quad_minb, 2, true>;
          const size_t smem = (size_t)2 * RowTile<PL>::slots((PL::slots(d.L) + 1) & ~1) * sizeof(cplx<T>);
          cudaError_t e = set_smem(kern, smem);
          if (e != cudaSuccess) return e;
          dim3 grd((a.nrows + 3) / 4, a.nslabs);
          kern<<<grd, 2 * PL::NT, smem, st>>>(a, d, omap);
          return cudaGetLastError();
        }
      }
      if (t2d_ok() && a.Hx <= 65535 &&
          encode_rowpair_map<T>(&omap, a.out, a.nrows, a.Hx, a.nslabs, a.ld_out, a.out_sstride)) {
        constexpr int TM = Shape<PL>::t2d_teams;
        auto kern = k_row_r2c_t2d<PL, TM * PL::NT, Shape<PL>::t2d_minb, TM>;
        const size_t smem = (size_t)TM * RowTile<PL>::slots((PL::slots(d.L) + 1) & ~1) * sizeof(cplx<T>);
        cudaError_t e = set_smem(kern, smem);
        if (e != cudaSuccess) return e;
        dim3 grd(((a.nrows + 1) / 2 + TM - 1) / TM, a.nslabs);
        kern<<<grd, TM * PL::NT, smem, st>>>(a, d, omap);
        return cudaGetLastError();
      }
    }
    auto kern = k_row_r2c<PL, Shape<PL>::row_threads, Shape<PL>::row_minb>;
    const int P = row_teams<PL>(kern, d, a.nrows);
    const size_t smem = (size_t)P * PL::slots(d.L) * sizeof(cplx<T>);
    cudaError_t e = set_smem(kern, smem);
    if (e != cudaSuccess) return e;
    dim3 grd((a.nrows + 2 * P - 1) / (2 * P), a.nslabs), blk(P * PL::nt(d));
    kern<<<grd, blk, smem, st>>>(a, d, P);
    return cudaGetLastError();
  });
}

template <class T>
cudaError_t launch_row_c2r(const RowC2RArgs& a, const FFTDesc<T>& d, int E, cudaStream_t st) {
  if (a.nslabs <= 0 || a.nrows <= 0) return cudaSuccess;
  return with_plan<T, false, true>(d.L, E, [&](auto tag) {
    using PL = typename decltype(tag)::type;
    if constexpr (PL::kStatic && PL::NT >= 32) {
      CUtensorMap imap;
      if constexpr (sizeof(T) == 4) {
        if (t2d_ok() && quad_rows() &&
            encode_rowpair_map<T>(&imap, a.in, a.nrows, a.Hx, a.nslabs, a.ld_in, a.in_sstride, 4)) {
          if constexpr (PL::kR16x16x8 && PL::kPerPass) {
            if (a.tw_816 && c2r_mirror_ok()) {
              using PLC = SPlanT<T, 16, C2R_MIRROR_PAD(T), true, 8, 16, 16>;
              auto kern = k_row_c2r_mirror<PL, PLC, 2 * PL::NT, Shape<PL>::quad_minb, 2, true>;
              const size_t smem =
                  (size_t)2 * RowTile<PL>::slots((PLC::slots(d.L) + 1) & ~1) * sizeof(cplx<T>) + 32;
              cudaError_t e = set_smem(kern, smem);
              if (e != cudaSuccess) return e;
              dim3 grd((a.nrows + 3) / 4, a.nslabs);
              kern<<<grd, 2 * PL::NT, smem, st>>>(a, d, imap);
              return cudaGetLastError();
            }
          }
          auto kern = k_row_c2r_t2d<PL, 2 * PL::NT, Shape<PL>::quad_minb, 2, true>;
          const size_t smem = (size_t)2 * RowTile<PL>::slots((PL::slots(d.L) + 1) & ~1) * sizeof(cplx<T>) + 32;
          cudaError_t e = set_smem(kern, smem);
          if (e != cudaSuccess) return e;
          dim3 grd((a.nrows + 3) / 4, a.nslabs);
          kern<<<grd, 2 * PL::NT, smem, st>>>(a, d, imap);
          return cudaGetLastError();
        }
      }
      if (t2d_ok() &&
          encode_rowpair_map<T>(&imap, a.in, a.nrows, a.Hx, a.nslabs, a.ld_in, a.in_sstride, 2)) {
        constexpr int TM = Shape<PL>::t2d_teams;
        if constexpr (PL::kR16x16x8 && PL::kPerPass) {
          if (a.tw_816 && c2r_mirror_ok()) {
            using PLC = SPlanT<T, 16, C2R_MIRROR_PAD(T), true, 8, 16, 16>;
            auto kern = k_row_c2r_mirror<PL, PLC, TM * PL::NT, Shape<PL>::t2d_minb, TM, false>;
            const size_t smem =
                (size_t)TM * RowTile<PL>::slots((PLC::slots(d.L) + 1) & ~1) * sizeof(cplx<T>) + 16 * TM;
            cudaError_t e = set_smem(kern, smem);
            if (e != cudaSuccess) return e;
            dim3 grd(((a.nrows + 1) / 2 + TM - 1) / TM, a.nslabs);
            kern<<<grd, TM * PL::NT, smem, st>>>(a, d, imap);
            return cudaGetLastError();
          }
        }
        auto kern = k_row_c2r_t2d<PL, TM * PL::NT, Shape<PL>::t2d_minb, TM, false>;
        const size_t smem = (size_t)TM * RowTile<PL>::slots((PL::slots(d.L) + 1) & ~1) * sizeof(cplx<T>) + 16 * TM;
        cudaError_t e = set_smem(kern, smem);
        if (e != cudaSuccess) return e;
        dim3 grd(((a.nrows + 1) / 2 + TM - 1) / TM, a.nslabs);
        kern<<<grd, TM * PL::NT, smem, st>>>(a, d, imap);
        return cudaGetLastError();
      }
    }
    auto kern = k_row_c2r<PL, Shape<PL>::row_threads, Shape<PL>::row_minb>;
    const int P = row_teams<PL>(kern, d, a.nrows);
    const size_t smem = (size_t)P * PL::slots(d.L) * sizeof(cplx<T>);
    cudaError_t e = set_smem(kern, smem);
    if (e != cudaSuccess) return e;
    dim3 grd((a.nrows + 2 * P - 1) / (2 * P), a.nslabs), blk(P * PL::nt(d));
    kern<<<grd, blk, smem, st>>>(a, d, P);
    return cudaGetLastError();
  });
}

template <class T>
cudaError_t launch_col_fwd(const ColFwdArgs& a, const FFTDesc<T>& d, int E, cudaStream_t st) {
  if (a.nbatch <= 0 || a.K <= 0) return cudaSuccess;
  return with_plan<T, true>(d.L, E, [&](auto tag) {
    using PL = typename decltype(tag)::type;
    if constexpr (PL::kStatic && PL::NT >= 32) {
      const size_t esz = sizeof(cplx<T>);
      if (tma_ok() && (a.nvalid * esz) % 16 == 0 && (a.ldy * esz) % 16 == 0 && (a.y_rstride * esz) % 16 == 0 &&
          (a.y_bstride * esz) % 16 == 0 && (a.lds * esz) % 16 == 0 && (a.s_rstride * esz) % 16 == 0) {
        constexpr bool twc_ok = PL::kPerPass && PL::NT % 32 == 0 && PL::NT <= 128 && (PL::E == 8 || PL::E == 16);
        auto kern = (twc_ok && tw_tmem_ok()) ? k_col_fwd_tma<PL, Shape<PL>::col_threads, Shape<PL>::tma_minb, twc_ok>
                                             : k_col_fwd_tma<PL, Shape<PL>::col_threads, Shape<PL>::tma_minb, false>;
        const size_t smem = (size_t)(((PL::slots(d.L) + 1) & ~1) + d.L + ((a.nvalid + 1) & ~1)) * esz + 32;
        cudaError_t e = set_smem(kern, smem);
        if (e != cudaSuccess) return e;
        // two layer halves would add into a zeroed W (exact, order-free); opt-in only
        const char* fs = getenv("BTTB_FWD_SPLITS");
        const int sp = (a.accumulate || !fs) ? 1 : (atoi(fs) == 2 ? 2 : 1);
        if (sp > 1) {
          e = cudaMemsetAsync(a.W, 0, (size_t)a.nbatch * a.w_bstride * esz, st);
          if (e != cudaSuccess) return e;
        }
        dim3 grd(a.Hx, a.nbatch, sp), blk(PL::NT);
        kern<<<grd, blk, smem, st>>>(a, d);
        return cudaGetLastError();
      }
    }
    constexpr bool accs = Shape<PL>::acc_smem;
    auto kern = k_col_fwd<PL, Shape<PL>::col_threads, Shape<PL>::col_minb, accs>;
    const int C = col_teams<PL>(kern, d, a.Hx);
    const size_t smem = (size_t)C * (PL::slots(d.L) + (accs ? d.L : 0)) * sizeof(cplx<T>);
    cudaError_t e = set_smem(kern, smem);
    if (e != cudaSuccess) return e;
    dim3 grd((a.Hx + C - 1) / C, a.nbatch), blk(C * PL::nt(d));
    kern<<<grd, blk, smem, st>>>(a, d, C);
    return cudaGetLastError();
  });
}

template <class T>
cudaError_t launch_col_tra(const ColTraArgs& a, const FFTDesc<T>& d, int E, cudaStream_t st) {
  if (a.nbatch <= 0 || a.K <= 0) return cudaSuccess;
  return with_plan<T, true>(d.L, E, [&](auto tag) {
    using PL = typename decltype(tag)::type;
    // (whole-warp teams, e.g. 2048 with 128 threads, measured no gain: 4.18 vs 4.14 ms/step)
    if constexpr (PL::kStatic && PL::NT >= 32 && PL::NT < 128 && PL::NT % 32 != 0 && sizeof(T) == 8 &&
                  (PL::E * 4) % 16 == 0) {
      if (tma_ok() && tmem_tra_ok()) {
        auto kern = k_col_tra_tmem<PL, 3>;
        const size_t smem = (size_t)(((PL::slots(d.L) + 1) & ~1) + d.L) * 16 + 16;
        cudaError_t e = set_smem(kern, smem);
        if (e != cudaSuccess) return e;
        const int sp = layer_splits((long)a.Hx * a.nbatch, a.K);
        dim3 grd(a.Hx, a.nbatch, sp), blk(TmemCfg<PL>::NTR);
        kern<<<grd, blk, smem, st>>>(a, d);
        return cudaGetLastError();
      }
    }
    if constexpr (PL::kStatic && PL::NT >= 32) {
      const size_t esz = sizeof(cplx<T>);
      if (tma_ok() && (a.lds * esz) % 16 == 0 && (a.s_rstride * esz) % 16 == 0) {
        constexpr bool twc_ok = PL::kPerPass && PL::NT % 32 == 0 && PL::NT <= 128 && (PL::E == 8 || PL::E == 16);
        auto kern = (twc_ok && tw_tmem_ok()) ? k_col_tra_tma<PL, Shape<PL>::col_threads, Shape<PL>::tra_minb, twc_ok>
                                             : k_col_tra_tma<PL, Shape<PL>::col_threads, Shape<PL>::tra_minb, false>;
        const size_t smem = (size_t)(((PL::slots(d.L) + 1) & ~1) + d.L) * esz + 16;
        cudaError_t e = set_smem(kern, smem);
        if (e != cudaSuccess) return e;
        const int sp = layer_splits((long)a.Hx * a.nbatch, a.K);
        dim3 grd(a.Hx, a.nbatch, sp), blk(PL::NT);
        kern<<<grd, blk, smem, st>>>(a, d);
        return cudaGetLastError();
      }
    }
    constexpr bool accs = Shape<PL>::acc_smem;
    auto kern = k_col_tra<PL, Shape<PL>::col_threads, Shape<PL>::col_minb, accs>;
    const int C = col_teams<PL>(kern, d, a.Hx);
    const size_t smem = (size_t)C * (PL::slots(d.L) + (accs ? d.L : 0)) * sizeof(cplx<T>);
    cudaError_t e = set_smem(kern, smem);
    if (e != cudaSuccess) return e;
    dim3 grd((a.Hx + C - 1) / C, a.nbatch), blk(C * PL::nt(d));
    kern<<<grd, blk, smem, st>>>(a, d, C);
    return cudaGetLastError();
  });
}

template <class TS>
cudaError_t launch_col_spec(const ColSpecArgs& a, const FFTDesc<double>& d, int E, cudaStream_t st) {
  return with_plan<double>(d.L, E, [&](auto tag) {
    using PL = typename decltype(tag)::type;
    auto kern = k_col_spec<PL, TS, Shape<PL>::col_threads, Shape<PL>::spec_minb>;
    const int C = col_teams<PL>(kern, d, a.Hx);
    const size_t smem = (size_t)C * PL::slots(d.L) * sizeof(double2);
    cudaError_t e = set_smem(kern, smem);
    if (e != cudaSuccess) return e;
    dim3 grd((a.Hx + C - 1) / C), blk(C * PL::nt(d));
    kern<<<grd, blk, smem, st>>>(a, d, C);
    return cudaGetLastError();
  });
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
