// EXPERIMENT, NOT BUILT (kept as the source of a measurement in DESIGN.md
// section 4).  Built into the library as an opt-in forward path it was
// correct (tests/test_gpu_parity.py C4 blocks green) and measured C4 forward
// 3.90 ms fp64 / 2.78 ms fp32 against 1.74 / 1.00 ms for the staged kernels:
// the column items ran the FP64 pipe at ~30% (synchronous L2 / HBM loads and
// TMEM round trips exposed), which is why the fused design was dropped.
// Fused whole-stack forward operator for 2048 x 2048 plans (experimental).
//
// Reference semantics: /root/reference/pkg/src/bttb/multiply.py:37-46 --
// d = sum_r real(ifft2(T^_r * fft2(embed(x_r))))[:sx, :sy].  Same operator as
// the staged kernels (spectral.cu); the transposed intermediate of each layer
// (its row half spectra, [kx][q]) lives in an L2-resident ring of nb layer
// slots instead of a 2.1 GB HBM round trip, and the cross-layer spectral
// accumulator of every column lives in tensor memory.
//
// One persistent cooperative CTA per SM, NP warp pairs.  Every 2048-point
// transform of the path has half its input zero (rows and columns both hold
// <= 1024 values), so each runs as two 1024-point transforms -- the even and
// odd output frequencies -- on the two warps of a pair (warp FFT: 32 values
// per lane, one shared-memory exchange, warp-level synchronisation only).
//
// Static schedule (no work-stealing atomics): CTA c owns columns kx = c + G*j;
// within the CTA, column j goes to a pair of TMEM class j % 2 (a warp reaches
// only its lane quarter w % 4, so a column's two half-states sit in the
// quarters of the pair that owns it).  Row pairs of layer r are dealt to CTAs
// with a per-layer rotation and, inside a CTA, to the pairs with the fewest
// columns first.  Iteration it: the pair's row items of layer it, then its
// column items of layer it - D.  Cross-CTA order: per-layer counters with
// release/acquire (rows_done[r]: the ring slot holds layer r; cols_done[r]:
// every column has read it, so the slot may take layer r + nb).  Every wait
// points to work of an earlier iteration, and the cooperative launch keeps
// all CTAs resident, so the schedule cannot deadlock; a bounded spin raises
// an error flag instead of hanging.
#include <cuda_runtime.h>

#include <cstdint>

#include "fft.cuh"
#include "fused2.h"
#include "tma.cuh"

namespace bttb {
namespace f2 {

#ifndef F2_NP_F64
#define F2_NP_F64 4
#endif
#ifndef F2_NP_F32
#define F2_NP_F32 8
#endif

constexpr int XS = 33;  // row stride (complex) of the 32 x 32 warp exchange: conflict-free both ways

template <class T> struct Cfg {
  using V = cplx<T>;
  static constexpr int NP = sizeof(T) == 8 ? F2_NP_F64 : F2_NP_F32;  // warp pairs per CTA
  static constexpr int NW = 2 * NP;
  static constexpr int PPC = NP / 2;                     // pairs per TMEM class
  static constexpr int WORDS = (int)(sizeof(V) / 4);     // 32-bit TMEM columns per complex value
  static constexpr int COLS = 32 * WORDS;                // TMEM columns of one half-column state
  static constexpr int SLOTS = 512 / COLS;               // half-column states per lane quarter
  static constexpr size_t SMEM = (size_t)NW * 32 * XS * sizeof(V);
};

enum { EVEN = 0, ODD_IN = 1, ODD_OUT = 2 };

// ---------------------------------------------------------------------------
// warp FFT, 1024 points: lane t holds x[t + 32 s] in v[s] on entry and
// X[t + 32 k] in v[k] on exit (radix 32 x 32, one exchange through xb).
//  EVEN:    X = FFT1024(x)
//  ODD_IN:  X = FFT1024(x[n] * w2048^n)   (odd half of a half-zero 2048 FFT)
//  ODD_OUT: X[n] = FFT1024(x)[n] * w2048^n (odd half of a half-output inverse, conj form)
// tw: exp(-2 pi i m / 2048), m < 2048.  The lane-dependent twiddles are
// generated as powers of two table values; the w64 factors are exact constants.
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
  __syncwarp();
  dft<32>(v);
  if constexpr (MODE == ODD_OUT) {
    sfor<1, 32>([&](auto kc) {
      constexpr int k = decltype(kc)::value;
      v[k] = twc<64, k>(v[k]);
    });
  }
}

// ---------------------------------------------------------------------------
// TMEM: 8 complex values of this lane at column offset ta
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
// cross-CTA order
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
  unsigned ns = 16;
  for (long long spins = 0; ld_acquire(p) < target; ++spins) {
    if (*(volatile int*)err) return;
    if (spins > (1ll << 25)) {
      atomicExch(err, 1);
      return;
    }
    __nanosleep(ns);
    if (ns < 128) ns *= 2;
  }
}
struct PairBar {
  int id;
  __device__ __forceinline__ void operator()() const { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }
};

__device__ __forceinline__ void st_pair(double2* o, double2 A, double2 B) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(o), "d"(A.x), "d"(A.y), "d"(B.x), "d"(B.y)
               : "memory");
}
__device__ __forceinline__ void st_pair(float2* o, float2 A, float2 B) {
  asm volatile("st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(o), "f"(A.x), "f"(A.y), "f"(B.x), "f"(B.y)
               : "memory");
}

struct Stat {
  long long* out;
  long long acc[F2_NSTAT];
  long long mark, t0;
  __device__ __forceinline__ void init(long long* o) {
    out = o;
#pragma unroll
    for (int i = 0; i < F2_NSTAT; ++i) acc[i] = 0;
    t0 = mark = out ? clock64() : 0;
  }
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
      long long* o = out + ((long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * F2_NSTAT;
#pragma unroll
      for (int i = 0; i < F2_NSTAT; ++i) o[i] = acc[i];
    }
  }
};

// row pairs of layer r dealt to CTAs with a rotation; inside the CTA the e-th
// item goes to pair NP-1-(e % NP) (the pairs with the fewest columns)
__device__ __forceinline__ int row_first(int c, int r, int G) {
  const int rot = (int)(((long long)r * 37) % G);
  return (c - rot + G) % G;
}

// ---------------------------------------------------------------------------
// forward
// ---------------------------------------------------------------------------
template <class T>
__global__ void __launch_bounds__(Cfg<T>::NW * 32, 1) k_f2_fwd(F2Args a) {
  using V = cplx<T>;
  using C = Cfg<T>;
  extern __shared__ __align__(16) unsigned char smraw[];
  __shared__ uint32_t tbase_s;
  const int w = threadIdx.x >> 5, t = threadIdx.x & 31;
  if (w == 0) tmem_alloc<512>(&tbase_s);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const int pair = w >> 1, par = w & 1, cls = pair & 1, u = pair >> 1;
  const bool lead = par == 0 && t == 0;
  const uint32_t tq = tbase_s + ((uint32_t)(32 * (w & 3)) << 16);
  const int G = gridDim.x, c = blockIdx.x;
  const int nc = c < a.Hx ? (a.Hx - 1 - c) / G + 1 : 0;
  V* xb = reinterpret_cast<V*>(smraw) + w * (32 * XS);
  V* xb_odd = reinterpret_cast<V*>(smraw) + (w | 1) * (32 * XS);
  const V* tw = static_cast<const V*>(a.tw);
  const V* S = static_cast<const V*>(a.S);
  V* ring = static_cast<V*>(a.ring);
  int* rows_done = a.sync;
  int* cols_done = a.sync + a.nz;
  int* err = a.sync + 2 * a.nz;
  const PairBar pb{1 + pair};
  const int D = a.lookahead, NB = a.nb;
  const T h = T(0.5);
  Stat st;
  st.init(a.stats);
  for (int it = 0; it < a.nz + D; ++it) {
    if (it < a.nz) {  // row items of layer it -> ring slot it % NB
      const int r = it;
      V* Y = ring + (long long)(r % NB) * a.ring_sstride;
      bool ready = r < NB;
      int e = 0;
      for (int i = row_first(c, r, G); i < a.npairs; i += G, ++e) {
        if (C::NP - 1 - (e % C::NP) != pair) continue;
        const int q0 = 2 * i;
        const bool has1 = q0 + 1 < a.ny;
        const T* x0 = static_cast<const T*>(a.in) + (long long)r * a.n_r + (long long)q0 * a.nx;
        const T* x1 = has1 ? x0 + a.nx : x0;
        V v[32];
        sfor<0, 32>([&](auto sc) {
          constexpr int s = decltype(sc)::value;
          const int n = t + 32 * s;
          const bool ok = n < a.nx;
          v[s] = mkc<V>(ok ? __ldcs(x0 + n) : T(0), ok && has1 ? __ldcs(x1 + n) : T(0));
        });
        st.lap(0);
        if (par == 0)
          fft1024<T, EVEN>(v, xb, tw, t);
        else
          fft1024<T, ODD_IN>(v, xb, tw, t);
        if (!ready) {  // every column has read the slot's previous layer
          if (t == 0) wait_geq(&cols_done[r - NB], a.Hx, err);
          __syncwarp();
          ready = true;
        }
        st.lap(1);
        // Z = A + iB with A, B the two rows' spectra: A = (Z[k] + conj Z[L-k]) / 2,
        // B = (Z[k] - conj Z[L-k]) / 2i; the partner of k = 2k'+p is lane
        // (32-t)&31 register 31-k1 (even; lane 0: register 32-k1) or lane 31-t (odd)
        const int plane = par ? 31 - t : (32 - t) & 31;
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
        pb();
        if (lead) red_release(&rows_done[r], 1);
        st.lap(2);
        st.count(6);
      }
    }
    const int r = it - D;
    if (r >= 0) {  // column items of layer r
      const V* Y = ring + (long long)(r % NB) * a.ring_sstride;
      bool ready = false;
      for (int m = 0;; ++m) {
        const int j = cls + 2 * (u + C::PPC * m);
        if (j >= nc) break;
        const int kx = c + G * j;
        const V* sc = S + (long long)r * a.s_rstride + (long long)kx * a.lds;
        if (lead) {  // the next column's spectrum into L2 while this one runs
          const int jn = cls + 2 * (u + C::PPC * (m + 1));
          if (jn < nc)
            l2_prefetch(S + (long long)r * a.s_rstride + (long long)(c + G * jn) * a.lds, 2048 * sizeof(V));
          else if (r + 1 < a.nz)
            l2_prefetch(S + (long long)(r + 1) * a.s_rstride + (long long)(c + G * (cls + 2 * u)) * a.lds,
                        2048 * sizeof(V));
        }
        if (!ready) {
          if (t == 0) wait_geq(&rows_done[r], a.npairs, err);
          __syncwarp();
          ready = true;
        }
        st.lap(0);
        const V* yc = Y + (long long)kx * a.ring_ld;
        V v[32];
        sfor<0, 32>([&](auto s) {
          constexpr int q = decltype(s)::value;
          const int n = t + 32 * q;
          v[q] = n < a.ny ? __ldcg(yc + n) : mkc<V>(T(0), T(0));
        });
        if (par == 0)
          fft1024<T, EVEN>(v, xb, tw, t);
        else
          fft1024<T, ODD_IN>(v, xb, tw, t);
        // natural spectrum layout: this warp's value k' = t + 32k is ky = 2k' + par
        sfor<0, 32>([&](auto kc) {
          constexpr int k = decltype(kc)::value;
          v[k] = cmul(__ldcs(sc + 2 * (t + 32 * k) + par), v[k]);
        });
        const uint32_t tacc = tq + (uint32_t)((j >> 1) * C::COLS);
        sfor<0, 4>([&](auto cc) {
          constexpr int ch = decltype(cc)::value;
          const uint32_t ta = tacc + (uint32_t)(ch * 8 * C::WORDS);
          if (r > 0) {
            V acc[8];
            tm_load8<T>(ta, acc);
#pragma unroll
            for (int i = 0; i < 8; ++i) v[8 * ch + i] = v[8 * ch + i] + acc[i];
          }
          tm_store8<T>(ta, v + 8 * ch);
        });
        tmem_wait_st();
        pb();
        if (lead) red_release(&cols_done[r], 1);
        st.lap(3);
        st.count(7);
      }
    }
  }
  // one inverse column transform per owned column: W[kx][n < sy]
  for (int m = 0;; ++m) {
    const int j = cls + 2 * (u + C::PPC * m);
    if (j >= nc) break;
    const int kx = c + G * j;
    const uint32_t tacc = tq + (uint32_t)((j >> 1) * C::COLS);
    V v[32];
    sfor<0, 4>([&](auto cc) {
      constexpr int ch = decltype(cc)::value;
      tm_load8<T>(tacc + (uint32_t)(ch * 8 * C::WORDS), v + 8 * ch);
    });
#pragma unroll
    for (int k = 0; k < 32; ++k) v[k] = conjv(v[k]);
    if (par == 0)
      fft1024<T, EVEN>(v, xb, tw, t);
    else
      fft1024<T, ODD_OUT>(v, xb, tw, t);
    if (par) {
#pragma unroll
      for (int k = 0; k < 32; ++k) xb[32 * k + t] = conjv(v[k]);
    }
    pb();
    if (!par) {
      V* o = static_cast<V*>(a.out) + (long long)kx * a.sy;
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const int n = t + 32 * k;
        if (n < a.sy) o[n] = conjv(v[k]) + xb_odd[32 * k + t];
      }
    }
    pb();
  }
  st.lap(4);
  st.flush();
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if (w == 0) tmem_dealloc<512>(tbase_s);
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

}  // namespace f2

int f2_counter_ints(int nz) { return 2 * nz + 1; }
int f2_grid() { return f2::sm_count_cached(); }
int f2_warps(bool fp64) { return fp64 ? f2::Cfg<double>::NW : f2::Cfg<float>::NW; }

bool f2_supported(long long Lx, long long Ly, long long nx, long long ny, long long sx, long long sy, bool fp64) {
  if (Lx != 2048 || Ly != 2048) return false;
  if (nx > 1024 || ny > 1024 || sx > 1024 || sy > 1024) return false;
  const long long Hx = Lx / 2 + 1, G = f2_grid();
  const long long per_cta = (Hx + G - 1) / G;  // columns of the busiest CTA
  const int slots = fp64 ? f2::Cfg<double>::SLOTS : f2::Cfg<float>::SLOTS;
  return (per_cta + 1) / 2 <= slots;  // each TMEM class holds ceil(per_cta / 2) columns
}

template <class T>
cudaError_t launch_f2(int mode, const F2Args& a, cudaStream_t st) {
  using namespace f2;
  if (mode != 0) return cudaErrorNotSupported;
  const size_t smem = Cfg<T>::SMEM;
  auto kern = k_f2_fwd<T>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  F2Args args = a;
  void* params[] = {&args};
  return cudaLaunchCooperativeKernel((const void*)kern, dim3(f2_grid()), dim3(Cfg<T>::NW * 32), params, smem, st);
}

template cudaError_t launch_f2<double>(int, const F2Args&, cudaStream_t);
template cudaError_t launch_f2<float>(int, const F2Args&, cudaStream_t);

}  // namespace bttb
