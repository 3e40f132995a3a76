// Shared-memory Stockham FFT engine for sm_100a (fp64 and fp32).
//
// One "team" of nt = L/E threads transforms one length-L complex sequence.
// Thread t of a team always owns the E elements {t + nt*s : s < E} of the
// sequence: it loads them straight from global memory before the first
// radix pass and, because the last Stockham pass of a length-L transform
// writes element (j + r*L/R) from butterfly j's r-th output, it also ends up
// holding exactly those elements of the RESULT in registers.  Only the
// exchanges between passes go through shared memory.  That property is what
// lets the fused operator kernels multiply by the cached spectrum and
// accumulate across depth layers in registers (see spectral.cu).
//
// Radix passes are compile-time DFTs of size R | E (2,3,4,5 and composites
// 6,8,10,12,16,20); the pass sequence for a length is chosen at plan time.
// Transform sign is numpy's forward convention exp(-2*pi*i*n*k/L); the
// inverse is conj(fft(conj(x))) and is never normalised here (the 1/(Lx*Ly)
// factor is folded into the cached spectra).
#pragma once
#include <cuda_runtime.h>
#include <type_traits>

#include "tma.cuh"

namespace bttb {

template <class T> struct CT;
template <> struct CT<double> { using type = double2; };
template <> struct CT<float> { using type = float2; };
template <class T> using cplx = typename CT<T>::type;

template <class V> struct ScalarOf;
template <> struct ScalarOf<double2> { using type = double; };
template <> struct ScalarOf<float2> { using type = float; };

template <class V, class S>
__device__ __forceinline__ V mkc(S a, S b) { V r; r.x = a; r.y = b; return r; }

__device__ __forceinline__ double2 operator+(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 operator-(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 operator+(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 operator-(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }

template <class V> __device__ __forceinline__ V cmul(V a, V b) {
  return mkc<V>(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
template <class V> __device__ __forceinline__ V conjv(V a) { return mkc<V>(a.x, -a.y); }
template <class V, class S> __device__ __forceinline__ V scalev(V a, S s) { return mkc<V>(a.x * s, a.y * s); }
// multiply by -i and +i
template <class V> __device__ __forceinline__ V mul_mi(V a) { return mkc<V>(a.y, -a.x); }
template <class V> __device__ __forceinline__ V mul_pi(V a) { return mkc<V>(-a.y, a.x); }

// compile-time loop
template <int I, int N, class F>
__device__ __forceinline__ void sfor(F&& f) {
  if constexpr (I < N) {
    f(std::integral_constant<int, I>{});
    sfor<I + 1, N>(f);
  }
}

template <int R> struct TwR;
#include "twiddle_consts.h"

// a * w_R^M, w_R = exp(-2*pi*i/R), with the quarter-turn cases exact
template <int R, int M, class V>
__device__ __forceinline__ V twc(V a) {
  constexpr int m = M % R;
  using S = typename ScalarOf<V>::type;
  if constexpr (m == 0) {
    return a;
  } else if constexpr (4 * m == R) {
    return mul_mi(a);
  } else if constexpr (2 * m == R) {
    return mkc<V>(-a.x, -a.y);
  } else if constexpr (4 * m == 3 * R) {
    return mul_pi(a);
  } else {
    const S c = (S)TwR<R>::re[m];
    const S s = (S)TwR<R>::im[m];
    return mkc<V>(a.x * c - a.y * s, a.x * s + a.y * c);
  }
}

template <int R> struct Split {
  static constexpr int A = (R % 4 == 0 && R != 4) ? 4 : (R % 2 == 0 && R != 2) ? 2 : (R % 3 == 0 && R != 3) ? 3 : 5;
  static constexpr int B = R / A;
};

// In-place forward DFT of size R on x[0..R) (natural order in and out).
template <int R, class V>
__device__ __forceinline__ void dft(V* x) {
  using S = typename ScalarOf<V>::type;
  if constexpr (R == 1) {
  } else if constexpr (R == 2) {
    V a = x[0], b = x[1];
    x[0] = a + b;
    x[1] = a - b;
  } else if constexpr (R == 3) {
    const S s3 = (S)0.8660254037844386;
    V t1 = x[1] + x[2];
    V t2 = mkc<V>(x[0].x - (S)0.5 * t1.x, x[0].y - (S)0.5 * t1.y);
    V d = x[1] - x[2];
    V m = mkc<V>(s3 * d.y, -s3 * d.x);  // -i*s3*d
    x[0] = x[0] + t1;
    x[1] = t2 + m;
    x[2] = t2 - m;
  } else if constexpr (R == 4) {
    V t0 = x[0] + x[2], t1 = x[0] - x[2];
    V t2 = x[1] + x[3], t3 = mul_mi(x[1] - x[3]);
    x[0] = t0 + t2;
    x[2] = t0 - t2;
    x[1] = t1 + t3;
    x[3] = t1 - t3;
  } else if constexpr (R == 5) {
    const S c1 = (S)0.30901699437494745, c2 = (S)-0.8090169943749475;
    const S s1 = (S)0.9510565162951535, s2 = (S)0.5877852522924731;
    V t1 = x[1] + x[4], t2 = x[2] + x[3];
    V t3 = x[1] - x[4], t4 = x[2] - x[3];
    V a1 = mkc<V>(x[0].x + c1 * t1.x + c2 * t2.x, x[0].y + c1 * t1.y + c2 * t2.y);
    V a2 = mkc<V>(x[0].x + c2 * t1.x + c1 * t2.x, x[0].y + c2 * t1.y + c1 * t2.y);
    V b1 = mkc<V>(s1 * t3.x + s2 * t4.x, s1 * t3.y + s2 * t4.y);
    V b2 = mkc<V>(s2 * t3.x - s1 * t4.x, s2 * t3.y - s1 * t4.y);
    b1 = mul_mi(b1);
    b2 = mul_mi(b2);
    x[0] = x[0] + t1 + t2;
    x[1] = a1 + b1;
    x[4] = a1 - b1;
    x[2] = a2 + b2;
    x[3] = a2 - b2;
  } else {
    // Cooley-Tukey split R = A*B: n = B*n1 + n2, k = k1 + A*k2
    constexpr int A = Split<R>::A, B = Split<R>::B;
    V u[R];
    sfor<0, B>([&](auto n2c) {
      constexpr int n2 = decltype(n2c)::value;
      V t[A];
      sfor<0, A>([&](auto n1c) { constexpr int n1 = decltype(n1c)::value; t[n1] = x[B * n1 + n2]; });
      dft<A>(t);
      sfor<0, A>([&](auto k1c) {
        constexpr int k1 = decltype(k1c)::value;
        u[n2 * A + k1] = twc<R, n2 * k1>(t[k1]);
      });
    });
    sfor<0, A>([&](auto k1c) {
      constexpr int k1 = decltype(k1c)::value;
      V t[B];
      sfor<0, B>([&](auto n2c) { constexpr int n2 = decltype(n2c)::value; t[n2] = u[n2 * A + k1]; });
      dft<B>(t);
      sfor<0, B>([&](auto k2c) { constexpr int k2 = decltype(k2c)::value; x[k1 + A * k2] = t[k2]; });
    });
  }
}

// Shared-memory slot of element i of a team buffer: one pad slot after every
// 8 (fp64) / 16 (fp32) elements, so the strided Stockham scatters spread over
// the 32 banks.  team_slots(L) is the padded size of one team buffer (+1 slot
// staggers consecutive teams).
template <class T> __host__ __device__ __forceinline__ int pslot(int i) {
  return i + (i >> (sizeof(T) == 8 ? 3 : 4));
}
template <class T> __host__ __device__ __forceinline__ int team_slots(int L) { return pslot<T>(L) + 1; }
// plan-specific padding e + e / PAD (PAD chosen per plan by a bank-conflict search
// over all of the plan's exchange patterns, tools/bank_search.py)
// (indices are non-negative: the unsigned division is one shift for the
// power-of-two pads, where the signed one costs a sign fix-up per access --
// 12% of the fp32 row kernels' instructions, which are issue-bound)
template <int PAD> __host__ __device__ __forceinline__ int pad_slot(int i) {
  return i + (int)((unsigned)i / (unsigned)PAD);
}
// pad_slot(base + c * STEP) for a compile-time c, given b0 = pad_slot(base):
// when STEP is a multiple of PAD the slot is affine in c (the quotient moves by
// exactly c * STEP / PAD), so the access takes an immediate offset instead of
// its own address arithmetic (the integer pipe runs at half the FP32 rate and
// binds the fp32 row kernels together with it).
template <int PAD, int STEP> __host__ __device__ __forceinline__ int pad_slot_at(int b0, int base, int c) {
  if constexpr (STEP % PAD == 0)
    return b0 + c * (STEP + STEP / PAD);
  else
    return pad_slot<PAD>(base + c * STEP);
}

// Plan for one transform length, passed by value to kernels.
template <class T>
struct FFTDesc {
  const cplx<T>* tw;   // tw[m] = exp(-2*pi*i*m/L), m < L
  const cplx<T>* twp;  // per-pass tables of this length's compile-time plan (see sfft), or null
  int L;              // transform length
  int nt;             // threads per team = L / E
  int npass;
  unsigned code;      // radix of pass p = radix_of((code >> 4p) & 15)
};

__host__ __device__ inline int radix_of(unsigned c) {
  switch (c) {
    case 1: return 2; case 2: return 3; case 3: return 4; case 4: return 5; case 5: return 6;
    case 6: return 8; case 7: return 10; case 8: return 12; case 9: return 16; case 10: return 20;
    default: return 0;
  }
}
__host__ __device__ inline unsigned radix_code(int r) {
  switch (r) {
    case 2: return 1; case 3: return 2; case 4: return 3; case 5: return 4; case 6: return 5;
    case 8: return 6; case 10: return 7; case 12: return 8; case 16: return 9; case 20: return 10;
    default: return 0;
  }
}

// One Stockham radix-R pass on the thread's registers (butterflies j = t + nt*b).
template <class T, int E, int R>
__device__ __forceinline__ void pass_compute(cplx<T> (&v)[E], int t, int nt, int Ns, int L,
                                             const cplx<T>* __restrict__ tw) {
  using V = cplx<T>;
  constexpr int NB = E / R;
  const int stride = L / (Ns * R);
  sfor<0, NB>([&](auto bc) {
    constexpr int b = decltype(bc)::value;
    V u[R];
    sfor<0, R>([&](auto rc) { constexpr int r = decltype(rc)::value; u[r] = v[b + r * NB]; });
    if (Ns > 1) {
      const int j = t + nt * b;
      const int k = j % Ns;
      const int step = k * stride;
      sfor<1, R>([&](auto rc) {
        constexpr int r = decltype(rc)::value;
        u[r] = cmul(u[r], __ldg(&tw[r * step]));
      });
    }
    dft<R>(u);
    sfor<0, R>([&](auto rc) { constexpr int r = decltype(rc)::value; v[b + r * NB] = u[r]; });
  });
}

// Scatter the pass outputs to their Stockham positions in shared memory.
template <class T, int E, int R>
__device__ __forceinline__ void pass_store(const cplx<T> (&v)[E], cplx<T>* sm, int t, int nt, int Ns) {
  constexpr int NB = E / R;
  sfor<0, NB>([&](auto bc) {
    constexpr int b = decltype(bc)::value;
    const int j = t + nt * b;
    const int k = j % Ns;
    const int base = (j - k) * R + k;
    sfor<0, R>([&](auto rc) { constexpr int r = decltype(rc)::value; sm[pslot<T>(base + r * Ns)] = v[b + r * NB]; });
  });
}

template <class T, int E>
__device__ __forceinline__ void run_compute(int R, cplx<T> (&v)[E], int t, int nt, int Ns, int L,
                                            const cplx<T>* __restrict__ tw) {
  switch (R) {
    case 2: if constexpr (E % 2 == 0) pass_compute<T, E, 2>(v, t, nt, Ns, L, tw); break;
    case 3: if constexpr (E % 3 == 0) pass_compute<T, E, 3>(v, t, nt, Ns, L, tw); break;
    case 4: if constexpr (E % 4 == 0) pass_compute<T, E, 4>(v, t, nt, Ns, L, tw); break;
    case 5: if constexpr (E % 5 == 0) pass_compute<T, E, 5>(v, t, nt, Ns, L, tw); break;
    case 6: if constexpr (E % 6 == 0) pass_compute<T, E, 6>(v, t, nt, Ns, L, tw); break;
    case 8: if constexpr (E % 8 == 0) pass_compute<T, E, 8>(v, t, nt, Ns, L, tw); break;
    case 10: if constexpr (E % 10 == 0) pass_compute<T, E, 10>(v, t, nt, Ns, L, tw); break;
    case 12: if constexpr (E % 12 == 0) pass_compute<T, E, 12>(v, t, nt, Ns, L, tw); break;
    case 16: if constexpr (E % 16 == 0) pass_compute<T, E, 16>(v, t, nt, Ns, L, tw); break;
    case 20: if constexpr (E % 20 == 0) pass_compute<T, E, 20>(v, t, nt, Ns, L, tw); break;
    default: break;
  }
}

template <class T, int E>
__device__ __forceinline__ void run_store(int R, const cplx<T> (&v)[E], cplx<T>* sm, int t, int nt, int Ns) {
  switch (R) {
    case 2: if constexpr (E % 2 == 0) pass_store<T, E, 2>(v, sm, t, nt, Ns); break;
    case 3: if constexpr (E % 3 == 0) pass_store<T, E, 3>(v, sm, t, nt, Ns); break;
    case 4: if constexpr (E % 4 == 0) pass_store<T, E, 4>(v, sm, t, nt, Ns); break;
    case 5: if constexpr (E % 5 == 0) pass_store<T, E, 5>(v, sm, t, nt, Ns); break;
    case 6: if constexpr (E % 6 == 0) pass_store<T, E, 6>(v, sm, t, nt, Ns); break;
    case 8: if constexpr (E % 8 == 0) pass_store<T, E, 8>(v, sm, t, nt, Ns); break;
    case 10: if constexpr (E % 10 == 0) pass_store<T, E, 10>(v, sm, t, nt, Ns); break;
    case 12: if constexpr (E % 12 == 0) pass_store<T, E, 12>(v, sm, t, nt, Ns); break;
    case 16: if constexpr (E % 16 == 0) pass_store<T, E, 16>(v, sm, t, nt, Ns); break;
    case 20: if constexpr (E % 20 == 0) pass_store<T, E, 20>(v, sm, t, nt, Ns); break;
    default: break;
  }
}

// Forward FFT of the team's sequence.  v holds elements {t + nt*s} on entry and
// the same elements of the transform on exit.  sm is the team's L-element
// shared buffer.  Contains __syncthreads(): every thread of the CTA must call
// it the same number of times (teams never diverge on the plan).
template <class T, int E>
__device__ __forceinline__ void team_fft(cplx<T> (&v)[E], cplx<T>* sm, int t, const FFTDesc<T>& d) {
  int Ns = 1;
  for (int p = 0; p < d.npass; ++p) {
    const int R = radix_of((d.code >> (4 * p)) & 15u);
    run_compute<T, E>(R, v, t, d.nt, Ns, d.L, d.tw);
    if (p + 1 < d.npass) {
      __syncthreads();
      run_store<T, E>(R, v, sm, t, d.nt, Ns);
      __syncthreads();
#pragma unroll
      for (int s = 0; s < E; ++s) v[s] = sm[pslot<T>(t + d.nt * s)];
    }
    Ns *= R;
  }
}

// ---------------------------------------------------------------------------
// Compile-time radix plans for the hot lengths: the pass sequence, Ns, the
// twiddle stride and the team size are constants, so the index arithmetic
// folds (no runtime integer division) and every pass is fully unrolled.
// ---------------------------------------------------------------------------
// PP (per-pass twiddles): tw points at this pass's table, entry (r-1)*NS + k =
// exp(-2*pi*i*r*k/(NS*R)) -- a warp's loads for one r are then contiguous in k
// instead of striding r*k*L/(NS*R) through the length-L table.
// exactly-rounded constant tables exist for these roots (twiddle_consts.h;
// 1, 2, 4: quarter turns are exact)
constexpr bool has_twr(int q) {
  return q == 1 || q == 2 || q == 4 || q == 3 || q == 5 || q == 6 || q == 8 || q == 10 || q == 12 || q == 16 ||
         q == 20 || q == 25;
}

// Generated pass twiddles (BTTB_TWGEN, default on): of the R-1 twiddles
// w^(r*k) of a butterfly only w^k and w^(Q*k) (Q ~ sqrt(R)) are loaded from
// the per-pass table; the rest are products w^(a*Q*k) * w^(c*k) of powers of
// the two (at most ~5 roundings: relative error < 1e-15 in fp64).  A table
// load is a 512-byte warp access of the L1 data pipe that binds the FFT
// passes (4 wavefronts), a complex multiply is 4 FP64 (or FP32) instructions
// on a pipe with headroom.
#ifndef BTTB_TWGEN
#define BTTB_TWGEN 1
#endif
#ifndef BTTB_TWGEN_F32
#define BTTB_TWGEN_F32 BTTB_TWGEN  // fp32 kernels are issue-bound rather than L1-bound
#endif
template <int R> struct TwQ {
  static constexpr int Q = R >= 16 ? 4 : R >= 8 ? 4 : R >= 4 ? 2 : 1;
};
template <class V, int R, int NS>
__device__ __forceinline__ void gen_twiddles(V (&w)[R], const V* __restrict__ tw, int k) {
  constexpr int Q = TwQ<R>::Q;
  w[1] = __ldg(&tw[k]);
  if constexpr (Q > 1 && Q < R) w[Q] = __ldg(&tw[(Q - 1) * NS + k]);
  sfor<2, (Q < R ? Q : R)>([&](auto cc) {
    constexpr int c = decltype(cc)::value;
    w[c] = cmul(w[c - 1], w[1]);
  });
  sfor<2, (R + Q - 1) / Q>([&](auto ac) {
    constexpr int a = decltype(ac)::value;
    w[a * Q] = cmul(w[(a - 1) * Q], w[Q]);
  });
  sfor<1, (R + Q - 1) / Q>([&](auto ac) {
    constexpr int a = decltype(ac)::value;
    sfor<1, Q>([&](auto cc) {
      constexpr int c = decltype(cc)::value;
      if constexpr (a * Q + c < R) w[a * Q + c] = cmul(w[a * Q], w[c]);
    });
  });
}

// ---------------------------------------------------------------------------
// Loop-invariant pass twiddles in tensor memory.  A column-stage CTA runs the
// SAME compile-time plan with the same thread index for every depth layer, so
// the R-1 twiddles of each of its butterfly blocks never change: they are
// computed once per CTA (exactly as the passes below would compute them, so
// the products are bit-identical) and parked in the thread's TMEM lane.  Each
// pass then fetches them with tcgen05.ld -- no L1 wavefronts (the table
// loads), no FP64 twiddle products (the generation) -- at the cost of 64-128
// TMEM columns per CTA, which this workload otherwise leaves idle.
// Layout: pass p (NS > 1) block b at column TOFF_p + b * tw_cols<V, R_p>,
// complex w^r at (r-1)*sizeof(V)/4; chunks of 16 columns (tcgen05 x16).
// ---------------------------------------------------------------------------
template <class V, int R> __host__ __device__ constexpr int tw_cols() {
  return ((int)(sizeof(V) / 4) * (R - 1) + 15) / 16 * 16;
}
struct NoTwCache {
  static constexpr bool on = false;
  uint32_t ta = 0;
};
struct TmemTwCache {  // ta = TMEM address of this thread's lane, column 0 of the cache
  static constexpr bool on = true;
  uint32_t ta;
};
__device__ __forceinline__ void tw_pack(double2 a, uint32_t* r) {
  r[0] = (uint32_t)__double2loint(a.x);
  r[1] = (uint32_t)__double2hiint(a.x);
  r[2] = (uint32_t)__double2loint(a.y);
  r[3] = (uint32_t)__double2hiint(a.y);
}
__device__ __forceinline__ void tw_pack(float2 a, uint32_t* r) {
  r[0] = __float_as_uint(a.x);
  r[1] = __float_as_uint(a.y);
}
__device__ __forceinline__ void tw_unpack(const uint32_t* r, double2& a) {
  a = make_double2(__hiloint2double((int)r[1], (int)r[0]), __hiloint2double((int)r[3], (int)r[2]));
}
__device__ __forceinline__ void tw_unpack(const uint32_t* r, float2& a) {
  a = make_float2(__uint_as_float(r[0]), __uint_as_float(r[1]));
}
template <class V, int R, int COL>
__device__ __forceinline__ void tw_store(uint32_t ta, const V (&w)[R]) {
  constexpr int N = tw_cols<V, R>(), CPC = sizeof(V) / 4;
  uint32_t u[N];
#pragma unroll
  for (int i = 0; i < N; ++i) u[i] = 0u;
  sfor<1, R>([&](auto rc) { constexpr int r = decltype(rc)::value; tw_pack(w[r], u + (r - 1) * CPC); });
  sfor<0, N / 16>([&](auto gc) {
    constexpr int g = decltype(gc)::value;
    uint32_t c[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) c[i] = u[16 * g + i];
    tmem_st16(ta + COL + 16 * g, c);
  });
}
template <class V, int R, int COL>
__device__ __forceinline__ void tw_load(uint32_t ta, V (&w)[R]) {
  constexpr int N = tw_cols<V, R>(), CPC = sizeof(V) / 4;
  uint32_t u[N];
  sfor<0, N / 16>([&](auto gc) {
    constexpr int g = decltype(gc)::value;
    uint32_t c[16];
    tmem_ld16(ta + COL + 16 * g, c);
#pragma unroll
    for (int i = 0; i < 16; ++i) u[16 * g + i] = c[i];
  });
  tmem_wait_ld();
  sfor<1, R>([&](auto rc) { constexpr int r = decltype(rc)::value; tw_unpack(u + (r - 1) * CPC, w[r]); });
}

template <class T, int E, int R, int NS, int NT, int L, bool PP = false, int TOFF = 0, class TwC = NoTwCache>
__device__ __forceinline__ void spass_compute(cplx<T> (&v)[E], int t, const cplx<T>* __restrict__ tw,
                                              const TwC& tc = TwC{}) {
  using V = cplx<T>;
  constexpr int NB = E / R;
  constexpr int STRIDE = L / (NS * R);
  if constexpr (TwC::on && PP && NS > 1) {
    sfor<0, NB>([&](auto bc) {
      constexpr int b = decltype(bc)::value;
      V u[R], w[R];
      sfor<0, R>([&](auto rc) { constexpr int r = decltype(rc)::value; u[r] = v[b + r * NB]; });
      tw_load<V, R, TOFF + b * tw_cols<V, R>()>(tc.ta, w);
      sfor<1, R>([&](auto rc) {
        constexpr int r = decltype(rc)::value;
        u[r] = cmul(u[r], w[r]);
      });
      dft<R>(u);
      sfor<0, R>([&](auto rc) { constexpr int r = decltype(rc)::value; v[b + r * NB] = u[r]; });
    });
    return;
  }
  constexpr bool GEN = (sizeof(T) == 8 ? BTTB_TWGEN : BTTB_TWGEN_F32) && PP && NS > 1 && R >= 4;
  // When a thread's blocks b sit at k = t + NT*b (NT*NB <= NS), the twiddle
  // w^(r*k) of block b is block 0's times the constant w_Q^(r*b), Q = NS*R/NT:
  // one table load per r instead of NB (the table loads are L1 wavefronts,
  // the binding resource of the exchanges; the constant multiply is FP64 work).
  constexpr bool DERIVE = PP && NS > 1 && NB > 1 && NT * NB <= NS && (NS * R) % NT == 0 && has_twr((NS * R) / NT);
  if constexpr (DERIVE) {
    constexpr int Q = (NS * R) / NT;
    V w0[R];
    if constexpr (GEN) {
      gen_twiddles<V, R, NS>(w0, tw, t);
    } else {
      sfor<1, R>([&](auto rc) {
        constexpr int r = decltype(rc)::value;
        w0[r] = __ldg(&tw[(r - 1) * NS + t]);
      });
    }
    sfor<0, NB>([&](auto bc) {
      constexpr int b = decltype(bc)::value;
      V u[R];
      sfor<0, R>([&](auto rc) { constexpr int r = decltype(rc)::value; u[r] = v[b + r * NB]; });
      sfor<1, R>([&](auto rc) {
        constexpr int r = decltype(rc)::value;
        u[r] = cmul(u[r], b == 0 ? w0[r] : twc<Q, (r * b) % Q>(w0[r]));
      });
      dft<R>(u);
      sfor<0, R>([&](auto rc) { constexpr int r = decltype(rc)::value; v[b + r * NB] = u[r]; });
    });
    return;
  }
  sfor<0, NB>([&](auto bc) {
    constexpr int b = decltype(bc)::value;
    V u[R];
    sfor<0, R>([&](auto rc) { constexpr int r = decltype(rc)::value; u[r] = v[b + r * NB]; });
    if constexpr (GEN) {
      const int k = (t + NT * b) % NS;
      V w[R];
      gen_twiddles<V, R, NS>(w, tw, k);
      sfor<1, R>([&](auto rc) {
        constexpr int r = decltype(rc)::value;
        u[r] = cmul(u[r], w[r]);
      });
    } else if constexpr (NS > 1) {
      const int k = (t + NT * b) % NS;
      sfor<1, R>([&](auto rc) {
        constexpr int r = decltype(rc)::value;
        if constexpr (PP)
          u[r] = cmul(u[r], __ldg(&tw[(r - 1) * NS + k]));
        else
          u[r] = cmul(u[r], __ldg(&tw[r * STRIDE * k]));
      });
    }
    dft<R>(u);
    sfor<0, R>([&](auto rc) { constexpr int r = decltype(rc)::value; v[b + r * NB] = u[r]; });
  });
}

// The twiddles spass_compute (no cache) multiplies block b of pass (NS, R)
// by, computed the same way; stored to the TMEM cache.
template <class T, int E, int R, int NS, int NT, int L, int TOFF>
__device__ __forceinline__ void spass_tw_fill(int t, const cplx<T>* __restrict__ tw, uint32_t ta) {
  using V = cplx<T>;
  constexpr int NB = E / R;
  constexpr bool GEN = (sizeof(T) == 8 ? BTTB_TWGEN : BTTB_TWGEN_F32) && NS > 1 && R >= 4;
  constexpr bool DERIVE = NS > 1 && NB > 1 && NT * NB <= NS && (NS * R) % NT == 0 && has_twr((NS * R) / NT);
  if constexpr (NS > 1) {
    if constexpr (DERIVE) {
      constexpr int Q = (NS * R) / NT;
      V w0[R];
      if constexpr (GEN) {
        gen_twiddles<V, R, NS>(w0, tw, t);
      } else {
        sfor<1, R>([&](auto rc) {
          constexpr int r = decltype(rc)::value;
          w0[r] = __ldg(&tw[(r - 1) * NS + t]);
        });
      }
      sfor<0, NB>([&](auto bc) {
        constexpr int b = decltype(bc)::value;
        V w[R];
        sfor<1, R>([&](auto rc) {
          constexpr int r = decltype(rc)::value;
          w[r] = b == 0 ? w0[r] : twc<Q, (r * b) % Q>(w0[r]);
        });
        tw_store<V, R, TOFF + b * tw_cols<V, R>()>(ta, w);
      });
    } else {
      sfor<0, NB>([&](auto bc) {
        constexpr int b = decltype(bc)::value;
        const int k = (t + NT * b) % NS;
        V w[R];
        if constexpr (GEN) {
          gen_twiddles<V, R, NS>(w, tw, k);
        } else {
          sfor<1, R>([&](auto rc) {
            constexpr int r = decltype(rc)::value;
            w[r] = __ldg(&tw[(r - 1) * NS + k]);
          });
        }
        tw_store<V, R, TOFF + b * tw_cols<V, R>()>(ta, w);
      });
    }
  }
}

template <class T, int E, int L, int OFF, int NS, int TOFF, int R, int... Rest>
__device__ __forceinline__ void sfft_tw_fill(int t, const cplx<T>* __restrict__ tw, uint32_t ta) {
  constexpr int NT = L / E;
  spass_tw_fill<T, E, R, NS, NT, L, TOFF>(t, tw + OFF, ta);
  if constexpr (sizeof...(Rest) > 0)
    sfft_tw_fill<T, E, L, (NS > 1 ? OFF + (R - 1) * NS : OFF), NS * R,
                 (NS > 1 ? TOFF + (E / R) * tw_cols<cplx<T>, R>() : TOFF), Rest...>(t, tw, ta);
}
// TMEM columns of a plan's twiddle cache
template <class V, int E, int NS, int R, int... Rest> __host__ __device__ constexpr int sfft_tw_cols() {
  constexpr int here = NS > 1 ? (E / R) * tw_cols<V, R>() : 0;
  if constexpr (sizeof...(Rest) > 0)
    return here + sfft_tw_cols<V, E, NS * R, Rest...>();
  else
    return here;
}

template <class T, int E, int R, int NS, int NT, int PAD>
__device__ __forceinline__ void spass_store(const cplx<T> (&v)[E], cplx<T>* sm, int t, bool active = true) {
  constexpr int NB = E / R;
  sfor<0, NB>([&](auto bc) {
    constexpr int b = decltype(bc)::value;
    const int j = t + NT * b;
    const int k = j % NS;
    const int base = (j - k) * R + k;
    const int b0 = pad_slot<PAD>(base);
    sfor<0, R>([&](auto rc) {
      constexpr int r = decltype(rc)::value;
      int slot;
      if constexpr (NS == 1 && PAD % R == 0) {
        // first pass: base = j * R is a multiple of R, so with R | PAD the
        // butterfly's R consecutive slots never cross a pad boundary
        slot = b0 + r;
      } else if constexpr (NS % PAD != 0 && PAD % NS == 0 && (NS * R) % PAD == 0) {
        // base = (multiple of NS * R, hence of PAD) + k with k < NS <= PAD and NS | PAD:
        // (k + r * NS) / PAD = (r * NS) / PAD, so the slot is b0 plus a constant
        slot = b0 + r * NS + (r * NS) / PAD;
      } else {
        slot = pad_slot_at<PAD, NS>(b0, base, r);
      }
      if (active) sm[slot] = v[b + r * NB];
    });
  });
}

// `active` = false: the thread follows the same control flow and barriers but
// touches no shared memory (helper lanes that pad a team to whole warps).
struct NoHook {
  __device__ __forceinline__ void operator()() const {}
};

// Barrier of the exchanges: the whole CTA (default) or one team of a CTA that
// runs several independent teams (named barrier `id`, `n` threads).
struct CtaSync {
  __device__ __forceinline__ void operator()() const { __syncthreads(); }
};
struct TeamSync {
  int id, n;
  __device__ __forceinline__ void operator()() const {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
  }
};

// hook() runs once, before the first exchange's barrier (e.g. to wait for an
// asynchronous copy that still reads the exchange buffer)
// PP: tw is the per-pass table block (OFF = this pass's offset in it);
// otherwise tw is the length-L table.
template <class T, int E, int L, int PAD, bool PP, int OFF, int NS, int TOFF, class TwC, int R, int... Rest,
          class Hook = NoHook, class Sync = CtaSync>
__device__ __forceinline__ void sfft_c(cplx<T> (&v)[E], cplx<T>* sm, int t, const cplx<T>* __restrict__ tw,
                                       const TwC& tc, bool active = true, Hook hook = Hook{}, Sync sync = Sync{}) {
  constexpr int NT = L / E;
  static_assert(E % R == 0, "radix must divide elements per thread");
  spass_compute<T, E, R, NS, NT, L, PP, TOFF, TwC>(v, active ? t : 0, PP ? tw + OFF : tw, tc);
  if constexpr (sizeof...(Rest) > 0) {
    if constexpr (NS == 1) hook();
    sync();
    spass_store<T, E, R, NS, NT, PAD>(v, sm, t, active);
    sync();
    const int t0 = pad_slot<PAD>(t);
#pragma unroll
    for (int s = 0; s < E; ++s)
      if (active) v[s] = sm[pad_slot_at<PAD, NT>(t0, t, s)];
    sfft_c<T, E, L, PAD, PP, (NS > 1 ? OFF + (R - 1) * NS : OFF), NS * R,
           (NS > 1 ? TOFF + (E / R) * tw_cols<cplx<T>, R>() : TOFF), TwC, Rest...>(v, sm, t, tw, tc, active,
                                                                                  NoHook{}, sync);
  }
}

template <class T, int E, int L, int PAD, bool PP, int OFF, int NS, int R, int... Rest, class Hook = NoHook,
          class Sync = CtaSync>
__device__ __forceinline__ void sfft(cplx<T> (&v)[E], cplx<T>* sm, int t, const cplx<T>* __restrict__ tw,
                                     bool active = true, Hook hook = Hook{}, Sync sync = Sync{}) {
  sfft_c<T, E, L, PAD, PP, OFF, NS, 0, NoTwCache, R, Rest...>(v, sm, t, tw, NoTwCache{}, active, hook, sync);
}

// Plan concepts used by the kernels: Scalar, E, nt(d), slot(e), slots(L),
// fft(v, sm, t, d); kStatic / NT for launch bounds.
// Total entries of the per-pass twiddle tables of a radix sequence.
template <int NS, int... Rs> struct PassTw;
template <int NS> struct PassTw<NS> { static constexpr int size = 0; };
template <int NS, int R, int... Rest> struct PassTw<NS, R, Rest...> {
  static constexpr int size = (NS > 1 ? (R - 1) * NS : 0) + PassTw<NS * R, Rest...>::size;
};

// PP = true: twiddles from d.twp, the per-pass tables the host builds for the
// registered plan of this length (spectral.cu static_radices); PP = false:
// the generic length-L table (plans that are not the registered one).
template <class T, int E_, int PAD, bool PP, int... Rs>
struct SPlanT {
  using Scalar = T;
  static constexpr bool kPerPass = PP;
  static constexpr int kPad = PAD;
  // radices 16/16/8 (L = 2048, 128 threads): the row R2C pass runs its last
  // radix-8 pass on mirrored butterfly pairs (k_row_r2c_t2d)
  static constexpr bool kR16x16x8 = sizeof...(Rs) == 3 && E_ == 16 && ((Rs == 16 || Rs == 8) && ...) &&
                                    (Rs * ...) == 2048;
  static constexpr bool kStatic = true;
  static constexpr int E = E_;
  static constexpr int L = (Rs * ...);
  static constexpr int NT = L / E_;
  static_assert(L % E_ == 0, "E must divide L");
  __host__ __device__ __forceinline__ static int nt(const FFTDesc<T>&) { return NT; }
  __host__ __device__ __forceinline__ static int slot(int e) { return pad_slot<PAD>(e); }
  __host__ __device__ __forceinline__ static int slots(int len) { return pad_slot<PAD>(len) + 1; }
  __device__ __forceinline__ static const cplx<T>* table(const FFTDesc<T>& d) { return PP ? d.twp : d.tw; }
  __device__ __forceinline__ static void fft(cplx<T> (&v)[E_], cplx<T>* sm, int t, const FFTDesc<T>& d) {
    sfft<T, E_, L, PAD, PP, 0, 1, Rs...>(v, sm, t, table(d));
  }
  __device__ __forceinline__ static void fft_masked(cplx<T> (&v)[E_], cplx<T>* sm, int t, const FFTDesc<T>& d,
                                                    bool active) {
    sfft<T, E_, L, PAD, PP, 0, 1, Rs...>(v, sm, t, table(d), active);
  }
  template <class Hook>
  __device__ __forceinline__ static void fft_hook(cplx<T> (&v)[E_], cplx<T>* sm, int t, const FFTDesc<T>& d,
                                                  Hook hook) {
    sfft<T, E_, L, PAD, PP, 0, 1, Rs...>(v, sm, t, table(d), true, hook);
  }
  // twiddle cache in TMEM (PP plans): columns, fill once per CTA, transforms that use it
  static constexpr int kTwCols = sfft_tw_cols<cplx<T>, E_, 1, Rs...>();
  __device__ __forceinline__ static void tw_fill(int t, const FFTDesc<T>& d, uint32_t ta) {
    sfft_tw_fill<T, E_, L, 0, 1, 0, Rs...>(t, table(d), ta);
  }
  __device__ __forceinline__ static void fft_tc(cplx<T> (&v)[E_], cplx<T>* sm, int t, const FFTDesc<T>& d,
                                                TmemTwCache tc) {
    sfft_c<T, E_, L, PAD, PP, 0, 1, 0, TmemTwCache, Rs...>(v, sm, t, table(d), tc);
  }
  // one team of a multi-team CTA: exchanges synchronise on the team's barrier
  __device__ __forceinline__ static void fft_team(cplx<T> (&v)[E_], cplx<T>* sm, int t, const FFTDesc<T>& d,
                                                  bool active, TeamSync sync) {
    sfft<T, E_, L, PAD, PP, 0, 1, Rs...>(v, sm, t, table(d), active, NoHook{}, sync);
  }
};

template <class T, int E_, int PAD, bool PP, int... Rs>
__host__ __device__ inline int radix_list(SPlanT<T, E_, PAD, PP, Rs...>, int* out) {
  int n = 0;
  ((out[n++] = Rs), ...);
  return n;
}

template <class T, int E_, int PAD, int... Rs> using SPlan = SPlanT<T, E_, PAD, true, Rs...>;
template <class T, int E_, int PAD, int... Rs> using SPlanG = SPlanT<T, E_, PAD, false, Rs...>;

// Runtime-radix plan; MAXT bounds the CTA size (256 keeps registers free for
// the common small lengths, 1024 is for teams of more than 256 threads).
template <class T, int E_, int MAXT = 256>
struct DPlan {
  using Scalar = T;
  static constexpr bool kStatic = false;
  static constexpr int E = E_;
  static constexpr int NT = MAXT;
  __host__ __device__ __forceinline__ static int nt(const FFTDesc<T>& d) { return d.nt; }
  __host__ __device__ __forceinline__ static int slot(int e) { return pslot<T>(e); }
  __host__ __device__ __forceinline__ static int slots(int len) { return team_slots<T>(len); }
  __device__ __forceinline__ static void fft(cplx<T> (&v)[E_], cplx<T>* sm, int t, const FFTDesc<T>& d) {
    team_fft<T, E_>(v, sm, t, d);
  }
};

}  // namespace bttb
