// Fused whole-stack forward / transpose operator for 2048 x 2048 FFT lengths
// (see fused.h for the design summary).
//
// Reference semantics: /root/reference/pkg/src/bttb/multiply.py:37-57 --
// forward d = sum_r real(ifft2(T^_r * fft2(embed(x_r))))[:sx, :sy],
// transpose x_r = real(ifft2(conj(T^_r) * fft2(embed(v))))[:nx, :ny]
// (transpose spectrum = conj of the forward one, transform.py:75-82).
// Same operator as the staged kernels of spectral.cu; what changes is where
// the intermediates live:
//
//  * rows -> columns: the row transforms of layer r write the transposed half
//    spectra Y_r[kx][q] into ring slot r % nb (L2 resident: 16.4 MB per slot at
//    C4 fp64); the column stage of layer r reads them there, `lookahead`
//    layers later.  Release/acquire counters order the two; every wait points
//    to an earlier layer (no cycles, all CTAs co-resident: cooperative launch).
//  * per column state in TMEM: CTA c owns columns kx = c + G*j; the even and
//    odd ky halves of column j live in lane quarters 2*(j%2) + {0, 1} at
//    column offset (j/2)*COLS -- the accumulator sum_r S_r * FFT_y(Y_r) of the
//    forward (one inverse column transform per column at the end: the
//    reference does one inverse 2-D FFT per layer, multiply.py:42-45) and the
//    data spectrum FFT_y(D) of the transpose (computed once, multiply.py:52).
//
// Work items, each run by a warp PAIR (two warps of one CTA, 64-thread named
// barrier): the even warp computes the even output frequencies 2k, the odd
// warp the odd ones 2k+1 of a 2048-point transform whose input is zero past
// 1024 (x[n] * w2048^n splits into a 1024-point transform per half) or whose
// outputs are only needed below 1024 (the same split on the inverse side).
#include <cuda_runtime.h>

#include <cstdint>

#include "fft.cuh"
#include "fused.h"
#include "tma.cuh"

namespace bttb {
namespace fz {

#ifndef FUSED_NW_F64
#define FUSED_NW_F64 12  // 168 registers per thread
#endif
#ifndef FUSED_NW_F32
#define FUSED_NW_F32 16  // 128 registers per thread
#endif

constexpr int XS = 33;  // row stride (complex) of the 32 x 32 exchange: conflict-free both ways

template <class T> struct K {
  using V = cplx<T>;
  static constexpr int WORDS = (int)(sizeof(V) / 4);   // 32-bit TMEM words per complex value
  static constexpr int COLS = 32 * WORDS;              // TMEM columns of one half-column state
  static constexpr int SLOTS = 512 / COLS;             // half-column states per lane quarter
  static constexpr int NW = sizeof(T) == 8 ? FUSED_NW_F64 : FUSED_NW_F32;  // warps per CTA (multiple of 4)
  static constexpr int PAIRS = NW / 2;
  static constexpr int PPC = NW / 4;                   // pairs per column class
};

enum { EVEN = 0, ODD_IN = 1, ODD_OUT = 2 };

// ---------------------------------------------------------------------------
// warp FFT, 1024 points: lane t holds x[t + 32 s] in v[s] on entry and
// X[t + 32 k] in v[k] on exit (radix 32 x 32, one exchange through the warp's
// shared buffer xb of 32 x XS values).
//  EVEN:    X = FFT1024(x)
//  ODD_IN:  X = FFT1024(x[n] * w2048^n)         (odd half of a half-zero 2048 FFT)
//  ODD_OUT: X[n] = FFT1024(x)[n] * w2048^n      (odd half of an inverse, conj form)
// The w2048^n factors are split: w64^s / w64^k are exact constants on the
// inputs / outputs, the lane-dependent part is folded into the pass-1
// twiddles, generated as A * B^k from two table loads (<= 10 roundings).
// ---------------------------------------------------------------------------
template <class T, int MODE>
__device__ __forceinline__ void fft1024(cplx<T> (&v)[32], cplx<T>* xb, const cplx<T>* __restrict__ tw, int t) {
  using V = cplx<T>;
  if constexpr (MODE == ODD_IN) {
    sfor<1, 32>([&](auto sc) {
      constexpr int s = decltype(sc)::value;
      v[s] = twc<64, s>(v[s]);
    });
  }
  dft<32>(v);
  {
    const int ib = MODE == ODD_OUT ? 2 * t + 1 : 2 * t;
    const V B = __ldg(&tw[ib]);
    const V B8 = __ldg(&tw[(8 * ib) & 2047]);
    V c[8];
    if constexpr (MODE == ODD_IN) {
      c[0] = __ldg(&tw[t]);
      c[1] = cmul(c[0], B);
    } else {
      c[0] = mkc<V>(T(1), T(0));
      c[1] = B;
    }
    sfor<2, 8>([&](auto ic) {
      constexpr int i = decltype(ic)::value;
      c[i] = cmul(c[i - 1], B);
    });
    sfor<0, 8>([&](auto ic) {
      constexpr int i = decltype(ic)::value;
      if (MODE == ODD_IN || i > 0) v[i] = cmul(v[i], c[i]);
    });
    V b = B8;
    sfor<1, 4>([&](auto ac) {
      constexpr int A = decltype(ac)::value;
      sfor<0, 8>([&](auto ic) {
        constexpr int i = decltype(ic)::value;
        v[8 * A + i] = cmul(v[8 * A + i], (i == 0 && MODE != ODD_IN) ? b : cmul(c[i], b));
      });
      if constexpr (A < 3) b = cmul(b, B8);
    });
  }
  __syncwarp();
  sfor<0, 32>([&](auto kc) {
    constexpr int k = decltype(kc)::value;
    xb[k * XS + t] = v[k];
  });
  __syncwarp();
  sfor<0, 32>([&](auto kc) {
    constexpr int k = decltype(kc)::value;
    v[k] = xb[t * XS + k];
  });
  dft<32>(v);
  if constexpr (MODE == ODD_OUT) {
    sfor<1, 32>([&](auto kc) {
      constexpr int k = decltype(kc)::value;
      v[k] = twc<64, k>(v[k]);
    });
  }
}

template <class T>
__device__ __forceinline__ void fft_half(cplx<T> (&v)[32], cplx<T>* xb, const cplx<T>* tw, int t, int par,
                                         bool inverse_side) {
  if (par == 0)
    fft1024<T, EVEN>(v, xb, tw, t);
  else if (inverse_side)
    fft1024<T, ODD_OUT>(v, xb, tw, t);
  else
    fft1024<T, ODD_IN>(v, xb, tw, t);
}

// ---------------------------------------------------------------------------
// TMEM: 8 complex values (one chunk) of this lane at column offset taddr
// ---------------------------------------------------------------------------
__device__ __forceinline__ void tm_ld32(uint32_t ta, uint32_t (&q)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%"
      "20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]), "=r"(q[7]), "=r"(q[8]),
        "=r"(q[9]), "=r"(q[10]), "=r"(q[11]), "=r"(q[12]), "=r"(q[13]), "=r"(q[14]), "=r"(q[15]), "=r"(q[16]),
        "=r"(q[17]), "=r"(q[18]), "=r"(q[19]), "=r"(q[20]), "=r"(q[21]), "=r"(q[22]), "=r"(q[23]), "=r"(q[24]),
        "=r"(q[25]), "=r"(q[26]), "=r"(q[27]), "=r"(q[28]), "=r"(q[29]), "=r"(q[30]), "=r"(q[31])
      : "r"(ta)
      : "memory");
}
__device__ __forceinline__ void tm_st32(uint32_t ta, const uint32_t (&q)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%"
      "19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta),
      "r"(q[0]), "r"(q[1]), "r"(q[2]), "r"(q[3]), "r"(q[4]), "r"(q[5]), "r"(q[6]), "r"(q[7]), "r"(q[8]), "r"(q[9]),
      "r"(q[10]), "r"(q[11]), "r"(q[12]), "r"(q[13]), "r"(q[14]), "r"(q[15]), "r"(q[16]), "r"(q[17]), "r"(q[18]),
      "r"(q[19]), "r"(q[20]), "r"(q[21]), "r"(q[22]), "r"(q[23]), "r"(q[24]), "r"(q[25]), "r"(q[26]), "r"(q[27]),
      "r"(q[28]), "r"(q[29]), "r"(q[30]), "r"(q[31])
      : "memory");
}

template <class T>
__device__ __forceinline__ void tm_load8(uint32_t ta, cplx<T>* out) {
  if constexpr (sizeof(T) == 8) {
    uint32_t q[32];
    tm_ld32(ta, q);
    tmem_wait_ld();
#pragma unroll
    for (int i = 0; i < 8; ++i)
      out[i] = make_double2(__hiloint2double((int)q[4 * i + 1], (int)q[4 * i]),
                            __hiloint2double((int)q[4 * i + 3], (int)q[4 * i + 2]));
  } else {
    uint32_t q[16];
    tmem_ld16(ta, q);
    tmem_wait_ld();
#pragma unroll
    for (int i = 0; i < 8; ++i) out[i] = make_float2(__uint_as_float(q[2 * i]), __uint_as_float(q[2 * i + 1]));
  }
}
template <class T>
__device__ __forceinline__ void tm_store8(uint32_t ta, const cplx<T>* in) {
  if constexpr (sizeof(T) == 8) {
    uint32_t q[32];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      q[4 * i] = (uint32_t)__double2loint(in[i].x);
      q[4 * i + 1] = (uint32_t)__double2hiint(in[i].x);
      q[4 * i + 2] = (uint32_t)__double2loint(in[i].y);
      q[4 * i + 3] = (uint32_t)__double2hiint(in[i].y);
    }
    tm_st32(ta, q);
  } else {
    uint32_t q[16];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      q[2 * i] = __float_as_uint(in[i].x);
      q[2 * i + 1] = __float_as_uint(in[i].y);
    }
    tmem_st16(ta, q);
  }
}

// ---------------------------------------------------------------------------
// synchronisation
// ---------------------------------------------------------------------------
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// bounded spin of one lane; on timeout (or an error raised elsewhere) the
// err flag is set and every later wait falls through (the host reports it)
__device__ __noinline__ void wait_geq(const int* p, int target, int* err) {
  unsigned ns = 32;
  for (long long spins = 0; ld_acquire(p) < target; ++spins) {
    if (*(volatile int*)err) return;
    if (spins > (1ll << 24)) {
      atomicExch(err, 1);
      return;
    }
    __nanosleep(ns);
    if (ns < 256) ns *= 2;
  }
}
struct PairBar {
  int id;
  __device__ __forceinline__ void operator()() const { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }
};

template <class V> __device__ __forceinline__ V ldcg(const V* p) { return __ldcg(p); }

// 32-byte (fp64) / 16-byte (fp32) store of the (q0, q0+1) pair of one kx row
__device__ __forceinline__ void st_pair(double2* o, double2 A, double2 B) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(o), "d"(A.x), "d"(A.y), "d"(B.x), "d"(B.y)
               : "memory");
}
__device__ __forceinline__ void st_pair(float2* o, float2 A, float2 B) {
  asm volatile("st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(o), "f"(A.x), "f"(A.y), "f"(B.x), "f"(B.y)
               : "memory");
}
__device__ __forceinline__ void ld_pair(const double2* o, double2& A, double2& B) {
  asm volatile("ld.global.cg.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(A.x), "=d"(A.y), "=d"(B.x), "=d"(B.y)
               : "l"(o));
}
__device__ __forceinline__ void ld_pair(const float2* o, float2& A, float2& B) {
  asm volatile("ld.global.cg.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(A.x), "=f"(A.y), "=f"(B.x), "=f"(B.y)
               : "l"(o));
}

struct Stat {
  long long* out;
  long long acc[FZ_NSTAT];
  long long t0, mark;
  __device__ __forceinline__ void init(long long* o) {
    out = o;
#pragma unroll
    for (int i = 0; i < FZ_NSTAT; ++i) acc[i] = 0;
    t0 = mark = out ? clock64() : 0;
  }
  // charge the cycles since the last mark to bucket i
  __device__ __forceinline__ void lap(int i) {
    if (out) {
      const long long now = clock64();
      acc[i] += now - mark;
      mark = now;
    }
  }
  __device__ __forceinline__ void count(int i) {
    if (out) acc[i] += 1;
  }
  __device__ __forceinline__ void flush() {
    if (out && (threadIdx.x & 31) == 0) {
      acc[5] = clock64() - t0;
      long long* o = out + ((long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * FZ_NSTAT;
#pragma unroll
      for (int i = 0; i < FZ_NSTAT; ++i) o[i] = acc[i];
    }
  }
};

struct Ctx {
  int w, t, pair, par, cls, pidx;
  bool lead;
  uint32_t tq;  // TMEM address of this warp's lane quarter, column 0
  int G, c, nc;
  int *rows_done, *cols_done, *row_next, *err;
};

template <class T>
__device__ __forceinline__ Ctx make_ctx(const FusedArgs& a, uint32_t tbase) {
  Ctx x;
  x.w = threadIdx.x >> 5;
  x.t = threadIdx.x & 31;
  x.pair = x.w >> 1;
  x.par = x.w & 1;
  x.cls = x.pair & 1;
  x.pidx = x.pair >> 1;
  x.lead = x.par == 0 && x.t == 0;
  x.tq = tbase + ((uint32_t)(32 * (x.w & 3)) << 16);
  x.G = gridDim.x;
  x.c = blockIdx.x;
  x.nc = x.c < a.Hx ? (a.Hx - 1 - x.c) / x.G + 1 : 0;
  x.rows_done = a.sync;
  x.cols_done = a.sync + a.nz;
  x.row_next = a.sync + 2 * a.nz;
  x.err = a.sync + 3 * a.nz;
  return x;
}

// next row item of layer r for this pair (leader's atomic, broadcast)
__device__ __forceinline__ int grab(const Ctx& x, int* slot, int* counter, PairBar pb) {
  if (x.lead) *slot = atomicAdd(counter, 1);
  pb();
  const int item = *slot;
  pb();
  return item;
}

// ---------------------------------------------------------------------------
// forward work items
// ---------------------------------------------------------------------------
// row pair pr of layer r: two real rows as one complex transform, separated
// into their half spectra, written transposed into the ring slot
template <class T>
__device__ __forceinline__ void row_fwd(const FusedArgs& a, const Ctx& x, int r, int pr, cplx<T>* xb,
                                        cplx<T>* Y, const cplx<T>* tw) {
  using V = cplx<T>;
  const int t = x.t, par = x.par;
  const int q0 = 2 * pr;
  const bool has1 = q0 + 1 < a.ny;
  const T* x0 = static_cast<const T*>(a.in) + (long long)r * a.n_r + (long long)q0 * a.nx;
  const T* x1 = has1 ? x0 + a.nx : x0;
  V v[32];
  sfor<0, 32>([&](auto sc) {
    constexpr int s = decltype(sc)::value;
    const int i = t + 32 * s;
    const bool ok = i < a.nx;
    v[s] = mkc<V>(ok ? __ldcs(x0 + i) : T(0), ok && has1 ? __ldcs(x1 + i) : T(0));
  });
  fft_half<T>(v, xb, tw, t, par, false);
  // Z[k] = A[k] + i B[k] with A, B the rows' spectra: A = (Z[k] + conj Z[L-k]) / 2,
  // B = (Z[k] - conj Z[L-k]) / 2i.  Partner of k = 2k'+p: even k' <-> 1024-k'
  // (lane 32-t, register 31-k1; lane 0: register 32-k1), odd k' <-> 1023-k'
  // (lane 31-t, register 31-k1).
  const int plane = par ? 31 - t : (32 - t) & 31;
  const T h = T(0.5);
  sfor<0, 17>([&](auto kc) {
    constexpr int k1 = decltype(kc)::value;
    const V z = v[k1];
    V m;
    m.x = __shfl_sync(0xffffffffu, v[31 - k1].x, plane);
    m.y = __shfl_sync(0xffffffffu, v[31 - k1].y, plane);
    if (par == 0 && t == 0) m = v[(32 - k1) & 31];
    const int kx = 2 * (t + 32 * k1) + par;
    if (kx < a.Hx) {
      const V A = mkc<V>(h * (z.x + m.x), h * (z.y - m.y));
      const V B = has1 ? mkc<V>(h * (z.y + m.y), h * (m.x - z.x)) : mkc<V>(T(0), T(0));
      st_pair(Y + (long long)kx * a.ring_ld + q0, A, B);
    }
  });
}

// column kx of layer r: FFT_y of the ring column, times the cached spectrum
// half, accumulated in TMEM
template <class T>
__device__ __forceinline__ void col_fwd(const FusedArgs& a, const Ctx& x, int r, int kx, cplx<T>* xb,
                                        const cplx<T>* Y, const cplx<T>* tw, uint32_t tacc) {
  using V = cplx<T>;
  const int t = x.t;
  const V* yc = Y + (long long)kx * a.ring_ld;
  V v[32];
  sfor<0, 32>([&](auto sc) {
    constexpr int s = decltype(sc)::value;
    const int q = t + 32 * s;
    v[s] = q < a.ny ? ldcg(yc + q) : mkc<V>(T(0), T(0));
  });
  fft_half<T>(v, xb, tw, t, x.par, false);
  const V* sc = static_cast<const V*>(a.S) + (long long)r * a.s_rstride + (long long)kx * 2048 + x.par * 1024 + t;
  sfor<0, 32>([&](auto kc) {
    constexpr int k = decltype(kc)::value;
    v[k] = cmul(__ldcs(sc + 32 * k), v[k]);
  });
  sfor<0, 4>([&](auto cc) {
    constexpr int ch = decltype(cc)::value;
    const uint32_t ta = tacc + (uint32_t)(ch * 8 * K<T>::WORDS);
    if (r > 0) {
      V acc[8];
      tm_load8<T>(ta, acc);
#pragma unroll
      for (int i = 0; i < 8; ++i) v[8 * ch + i] = v[8 * ch + i] + acc[i];
    }
    tm_store8<T>(ta, v + 8 * ch);
  });
  tmem_wait_st();
}

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------
template <class T>
__global__ void __launch_bounds__(K<T>::NW * 32, 1) k_fused_fwd(FusedArgs a) {
  using V = cplx<T>;
  constexpr int PPC = K<T>::PPC, COLS = K<T>::COLS;
  extern __shared__ __align__(16) unsigned char smraw[];
  __shared__ uint32_t tbase_s;
  __shared__ int bcast[K<T>::PAIRS];
  if ((threadIdx.x >> 5) == 0) tmem_alloc<512>(&tbase_s);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const Ctx x = make_ctx<T>(a, tbase_s);
  V* xb = reinterpret_cast<V*>(smraw) + x.w * (32 * XS);
  V* xb_odd = reinterpret_cast<V*>(smraw) + (x.w | 1) * (32 * XS);
  const V* tw = static_cast<const V*>(a.tw);
  const PairBar pb{1 + x.pair};
  const int D = a.lookahead, NB = a.nb;
  V* ring = static_cast<V*>(a.ring);
  Stat st;
  st.init(a.stats);
  for (int it = 0; it < a.nz + D; ++it) {
    if (it < a.nz) {  // row items of layer it -> slot it % NB
      V* Y = ring + (long long)(it % NB) * a.ring_sstride;
      bool ready = it < NB;
      for (;;) {
        const int item = grab(x, &bcast[x.pair], &x.row_next[it], pb);
        st.lap(1);
        if (item >= a.npairs) break;
        if (!ready) {  // the slot's previous layer has been read by every column
          if (x.lead) wait_geq(&x.cols_done[it - NB], a.Hx, x.err);
          pb();
          ready = true;
          st.lap(0);
        }
        row_fwd<T>(a, x, it, item, xb, Y, tw);
        pb();
        if (x.lead) red_release(&x.rows_done[it], 1);
        st.lap(2);
        st.count(6);
      }
    }
    const int cc = it - D;
    if (cc >= 0) {  // column items of layer cc
      const V* Y = ring + (long long)(cc % NB) * a.ring_sstride;
      if (x.t == 0)
        for (int j = x.cls + 2 * x.pidx; j < x.nc; j += 2 * PPC)
          l2_prefetch(static_cast<const V*>(a.S) + (long long)cc * a.s_rstride + (long long)(x.c + x.G * j) * 2048 +
                          x.par * 1024,
                      1024 * sizeof(V));
      if (x.lead) wait_geq(&x.rows_done[cc], a.npairs, x.err);
      pb();
      st.lap(0);
      for (int j = x.cls + 2 * x.pidx; j < x.nc; j += 2 * PPC) {
        col_fwd<T>(a, x, cc, x.c + x.G * j, xb, Y, tw, x.tq + (uint32_t)((j >> 1) * COLS));
        pb();
        if (x.lead) atomicAdd(&x.cols_done[cc], 1);
        st.lap(3);
        st.count(7);
      }
    }
  }
  // one inverse column transform per owned column: W[kx][n < sy]
  for (int j = x.cls + 2 * x.pidx; j < x.nc; j += 2 * PPC) {
    const int kx = x.c + x.G * j;
    const uint32_t tacc = x.tq + (uint32_t)((j >> 1) * COLS);
    V v[32];
    sfor<0, 4>([&](auto cc) {
      constexpr int ch = decltype(cc)::value;
      tm_load8<T>(tacc + (uint32_t)(ch * 8 * K<T>::WORDS), v + 8 * ch);
    });
#pragma unroll
    for (int k = 0; k < 32; ++k) v[k] = conjv(v[k]);
    fft_half<T>(v, xb, tw, x.t, x.par, true);
    if (x.par) {
#pragma unroll
      for (int k = 0; k < 32; ++k) xb[32 * k + x.t] = conjv(v[k]);
    }
    pb();
    if (!x.par) {
      V* o = static_cast<V*>(a.out) + (long long)kx * a.sy;
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const int n = x.t + 32 * k;
        if (n < a.sy) o[n] = conjv(v[k]) + xb_odd[32 * k + x.t];
      }
    }
    pb();
  }
  st.lap(4);
  st.flush();
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if (x.w == 0) tmem_dealloc<512>(tbase_s);
}

template <class T>
__global__ void __launch_bounds__(K<T>::NW * 32, 1) k_fused_tra(FusedArgs a) {
  using V = cplx<T>;
  constexpr int PPC = K<T>::PPC, COLS = K<T>::COLS;
  extern __shared__ __align__(16) unsigned char smraw[];
  __shared__ uint32_t tbase_s;
  __shared__ int bcast[K<T>::PAIRS];
  if ((threadIdx.x >> 5) == 0) tmem_alloc<512>(&tbase_s);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const Ctx x = make_ctx<T>(a, tbase_s);
  V* xb = reinterpret_cast<V*>(smraw) + x.w * (32 * XS);
  V* xb_odd = reinterpret_cast<V*>(smraw) + (x.w | 1) * (32 * XS);
  const V* tw = static_cast<const V*>(a.tw);
  const PairBar pb{1 + x.pair};
  const int D = a.lookahead, NB = a.nb;
  V* ring = static_cast<V*>(a.ring);
  const int t = x.t;
  Stat st;
  st.init(a.stats);
  // prologue: data spectrum FFT_y(D[kx]) of every owned column -> TMEM
  for (int j = x.cls + 2 * x.pidx; j < x.nc; j += 2 * PPC) {
    const int kx = x.c + x.G * j;
    const V* dc = static_cast<const V*>(a.in) + (long long)kx * a.sy;
    V v[32];
    sfor<0, 32>([&](auto sc) {
      constexpr int s = decltype(sc)::value;
      const int q = t + 32 * s;
      v[s] = q < a.sy ? __ldg(dc + q) : mkc<V>(T(0), T(0));
    });
    fft_half<T>(v, xb, tw, t, x.par, false);
    const uint32_t ta = x.tq + (uint32_t)((j >> 1) * COLS);
    sfor<0, 4>([&](auto cc) {
      constexpr int ch = decltype(cc)::value;
      tm_store8<T>(ta + (uint32_t)(ch * 8 * K<T>::WORDS), v + 8 * ch);
    });
    tmem_wait_st();
  }
  st.lap(4);
  for (int it = 0; it < a.nz + D; ++it) {
    if (it < a.nz) {  // column items of layer it -> slot it % NB
      V* Y = ring + (long long)(it % NB) * a.ring_sstride;
      if (t == 0)
        for (int j = x.cls + 2 * x.pidx; j < x.nc; j += 2 * PPC)
          l2_prefetch(static_cast<const V*>(a.S) + (long long)it * a.s_rstride + (long long)(x.c + x.G * j) * 2048 +
                          x.par * 1024,
                      1024 * sizeof(V));
      if (it >= NB) {  // the slot's previous layer has been read by every row item
        if (x.lead) wait_geq(&x.rows_done[it - NB], a.npairs, x.err);
        pb();
      }
      st.lap(0);
      for (int j = x.cls + 2 * x.pidx; j < x.nc; j += 2 * PPC) {
        const int kx = x.c + x.G * j;
        const uint32_t ta = x.tq + (uint32_t)((j >> 1) * COLS);
        V v[32];
        sfor<0, 4>([&](auto cc) {
          constexpr int ch = decltype(cc)::value;
          tm_load8<T>(ta + (uint32_t)(ch * 8 * K<T>::WORDS), v + 8 * ch);
        });
        // IFFT(conj(S) * Dh) = conj(FFT(S * conj(Dh)))
        const V* sc = static_cast<const V*>(a.S) + (long long)it * a.s_rstride + (long long)kx * 2048 + x.par * 1024 + t;
        sfor<0, 32>([&](auto kc) {
          constexpr int k = decltype(kc)::value;
          v[k] = cmul(__ldcs(sc + 32 * k), conjv(v[k]));
        });
        fft_half<T>(v, xb, tw, t, x.par, true);
        if (x.par) {
#pragma unroll
          for (int k = 0; k < 32; ++k) xb[32 * k + t] = conjv(v[k]);
        }
        pb();
        if (!x.par) {
          V* o = Y + (long long)kx * a.ring_ld;
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            const int n = t + 32 * k;
            if (n < a.ny) o[n] = conjv(v[k]) + xb_odd[32 * k + t];
          }
        }
        pb();
        if (x.lead) red_release(&x.cols_done[it], 1);
        st.lap(3);
        st.count(7);
      }
    }
    const int rr = it - D;
    if (rr >= 0) {  // row items of layer rr: C2R of row pairs -> model
      const V* Y = ring + (long long)(rr % NB) * a.ring_sstride;
      bool ready = false;
      for (;;) {
        const int item = grab(x, &bcast[x.pair], &x.row_next[rr], pb);
        st.lap(1);
        if (item >= a.npairs) break;
        if (!ready) {
          if (x.lead) wait_geq(&x.cols_done[rr], a.Hx, x.err);
          pb();
          ready = true;
          st.lap(0);
        }
        const int q0 = 2 * item;
        const bool has1 = q0 + 1 < a.ny;
        V v[32];
        sfor<0, 32>([&](auto sc) {
          constexpr int s = decltype(sc)::value;
          const int kp = t + 32 * s;
          const int kx = 2 * kp + x.par;
          const bool mir = kx > 1024;
          const int kk = mir ? 2048 - kx : kx;
          V A, B;
          ld_pair(Y + (long long)kk * a.ring_ld + q0, A, B);
          if (!has1) B = mkc<V>(T(0), T(0));
          if (kk == 0 || kk == 1024) {  // Hermitian projection (.real semantics)
            A.y = T(0);
            B.y = T(0);
          }
          // Z = A + iB (or its mirror conj(A) + i conj(B)); the inverse runs as conj(FFT(conj Z))
          v[s] = mir ? mkc<V>(A.x + B.y, A.y - B.x) : mkc<V>(A.x - B.y, -(A.y + B.x));
        });
        fft_half<T>(v, xb, tw, t, x.par, true);
        if (x.par) {
#pragma unroll
          for (int k = 0; k < 32; ++k) xb[32 * k + t] = conjv(v[k]);
        }
        pb();
        if (!x.par) {
          T* o0 = static_cast<T*>(a.out) + (long long)rr * a.n_r + (long long)q0 * a.nx;
          T* o1 = o0 + a.nx;
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            const int n = t + 32 * k;
            if (n < a.nx) {
              const V z = conjv(v[k]) + xb_odd[32 * k + t];
              __stcs(o0 + n, z.x);
              if (has1) __stcs(o1 + n, z.y);
            }
          }
        }
        pb();
        if (x.lead) atomicAdd(&x.rows_done[rr], 1);
        st.lap(2);
        st.count(6);
      }
    }
  }
  st.flush();
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if (x.w == 0) tmem_dealloc<512>(tbase_s);
}

template <class T>
__global__ void k_ky_split(cplx<T>* S, int dir) {
  __shared__ cplx<T> buf[2048];
  cplx<T>* row = S + (long long)blockIdx.x * 2048;
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = row[i];
  __syncthreads();
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) {
    const int j = (i & 1) * 1024 + (i >> 1);  // natural ky = i  <->  split position j
    if (dir > 0)
      row[j] = buf[i];
    else
      row[i] = buf[j];
  }
}

int sm_count_cached() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace fz

int fused_counter_ints(int nz) { return 3 * nz + 1; }
int fused_grid() { return fz::sm_count_cached(); }
int fused_warps(bool fp64) { return fp64 ? fz::K<double>::NW : fz::K<float>::NW; }

bool fused_supported(long long Lx, long long Ly, long long nx, long long ny, long long sx, long long sy) {
  if (Lx != 2048 || Ly != 2048) return false;
  if (nx > 1024 || ny > 1024 || sx > 1024 || sy > 1024) return false;
  const long long Hx = Lx / 2 + 1;
  // column states: fp64 holds 8 columns per CTA (4 per class), fp32 16
  return Hx <= 8LL * fused_grid();
}

template <class T>
cudaError_t launch_fused(int mode, const FusedArgs& a, cudaStream_t st) {
  using namespace fz;
  const size_t smem = (size_t)K<T>::NW * 32 * XS * sizeof(cplx<T>);
  auto kern = mode == 0 ? k_fused_fwd<T> : k_fused_tra<T>;
  static bool attr[2] = {false, false};
  if (!attr[mode]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr[mode] = true;
  }
  FusedArgs args = a;
  void* params[] = {&args};
  return cudaLaunchCooperativeKernel((const void*)kern, dim3(fused_grid()), dim3(K<T>::NW * 32), params, smem, st);
}

template <class T>
cudaError_t launch_ky_split(void* S, long long nrows, int dir, cudaStream_t st) {
  if (nrows <= 0) return cudaSuccess;
  fz::k_ky_split<T><<<(unsigned)nrows, 256, 0, st>>>(static_cast<cplx<T>*>(S), dir);
  return cudaGetLastError();
}

template cudaError_t launch_fused<double>(int, const FusedArgs&, cudaStream_t);
template cudaError_t launch_fused<float>(int, const FusedArgs&, cudaStream_t);
template cudaError_t launch_ky_split<double>(void*, long long, int, cudaStream_t);
template cudaError_t launch_ky_split<float>(void*, long long, int, cudaStream_t);

}  // namespace bttb
