// Fused layer pipeline: ONE persistent kernel per application runs the row
// passes and the column stages of every layer, so the per-layer row-pass
// intermediate never leaves the chip's L2 and the spectral accumulator (forward)
// or the data spectrum (transpose) never leaves the SMs' tensor memory.
// Included by spectral.cu (uses its plan registry).
//
// Reference semantics: multiply.py:37-57 (same operator as the staged path).
//
// Layout and roles (one CTA per SM, TEAMS teams of 128 threads, each team runs
// its own FFTs on its own shared-memory exchange buffer and named barrier):
//  * column ownership: CTA c owns columns kx = c + G*i (G = grid size); column
//    slot i always runs on team i % TEAMS (so one column's layers are processed
//    in order by one team) and keeps its E-element state in TMEM columns
//    [i*COLS, (i+1)*COLS) -- lane = thread of the team;
//  * row pairs are taken dynamically from a per-layer global counter by any team;
//  * ring: NB slots of one layer's transposed intermediate [kx][q < ny] (L2 resident);
//  * counters: rows_done[l], cols_done[l] (release/acquire), row_next[l], err.
// Forward, team loop l = 0..nz: rows(l) -> slot l%NB (waits cols_done[l-NB] ==
// Hx), then cols(l-1) (waits rows_done[l-1] == npairs): Y column FFT, times
// S_l, accumulated in TMEM; epilogue: one inverse column FFT per column -> W.
// Transpose, after a prologue that puts FFT_y of the data half spectrum in
// TMEM: cols(l) -> slot l%NB (waits rows_done[l-NB] == npairs), then rows(l-1)
// (waits cols_done[l-1] == Hx): C2R -> model layer l-1.
// Every dependency points to a lower layer or to the same layer's other phase,
// which each team runs earlier in its loop, so with NB >= 2 the pipeline cannot
// deadlock; all CTAs are co-resident (cooperative launch).  Every spin is
// bounded: on timeout the err flag is raised and all waits fall through.

namespace bttb {

namespace pipe {

constexpr int TT = 128;  // threads per team (four warps: the four TMEM lane quarters)

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// leader-only bounded spin; returns false (and raises err) on timeout
__device__ __noinline__ bool wait_geq(const int* p, int target, int* err) {
  unsigned ns = 32;
  for (long long spins = 0; ld_acquire(p) < target; ++spins) {
    if (*(volatile int*)err) return false;
    if (spins > (1ll << 23)) {
      atomicExch(err, 1);
      return false;
    }
    __nanosleep(ns);
    if (ns < 512) ns *= 2;
  }
  return true;
}

// complex <-> 32-bit TMEM words
template <class V> struct Words;
template <> struct Words<double2> {
  static constexpr int W = 4;
  __device__ __forceinline__ static void put(double2 a, uint32_t* r) {
    r[0] = (uint32_t)__double2loint(a.x);
    r[1] = (uint32_t)__double2hiint(a.x);
    r[2] = (uint32_t)__double2loint(a.y);
    r[3] = (uint32_t)__double2hiint(a.y);
  }
  __device__ __forceinline__ static double2 get(const uint32_t* r) {
    return make_double2(__hiloint2double((int)r[1], (int)r[0]), __hiloint2double((int)r[3], (int)r[2]));
  }
};
template <> struct Words<float2> {
  static constexpr int W = 2;
  __device__ __forceinline__ static void put(float2 a, uint32_t* r) {
    r[0] = __float_as_uint(a.x);
    r[1] = __float_as_uint(a.y);
  }
  __device__ __forceinline__ static float2 get(const uint32_t* r) {
    return make_float2(__uint_as_float(r[0]), __uint_as_float(r[1]));
  }
};

template <class PL> struct Cfg {
  using T = typename PL::Scalar;
  using V = cplx<T>;
  static constexpr int E = PL::E, NT = PL::NT, L = PL::L, HX = L / 2 + 1;
  static constexpr int W = Words<V>::W;
  static constexpr int COLS = E * W;         // TMEM columns of one column's state
  static constexpr int PER = 16 / W;         // complex values per 16-column access
  static constexpr int GROUPS = COLS / 16;
  static constexpr int NI = (HX + TT - 1) / TT;  // kx items per thread in the row passes
  static_assert(COLS % 16 == 0, "TMEM state in groups of 16 columns");
  static_assert(NT <= TT, "one team of at most 128 threads");
  // shared slots of one team (exchange buffer), rounded to 128 bytes
  static constexpr int team_slots() {
    constexpr int per = 128 / (int)sizeof(V);
    return (PL::slots(L) + per - 1) / per * per;
  }
};

struct Team {
  int id, t, leader;
  TeamSync sync;
  __device__ __forceinline__ void bar() const { sync(); }
};

// optional per-team cycle accounting (PipeArgs::stats, development aid):
// [0] waiting on counters, [1] row items, [2] column items, [3] rows, [4] cols, [5] total
__device__ __forceinline__ long long gtimer() {
  long long v;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
  return v;
}

// [6] globaltimer at start, [7] globaltimer at end (ns)
struct Stats {
  long long* out;
  long long acc[8];
  long long t0;
  __device__ __forceinline__ void init(long long* o) {
    out = o;
    for (int i = 0; i < 8; ++i) acc[i] = 0;
    t0 = clock64();
    if (out) acc[6] = gtimer();
  }
  __device__ __forceinline__ long long now() const { return out ? clock64() : 0; }
  __device__ __forceinline__ void add(int i, long long since) {
    if (out) acc[i] += clock64() - since;
  }
  __device__ __forceinline__ void count(int i) {
    if (out) acc[i] += 1;
  }
  __device__ __forceinline__ void flush(int t) {
    if (out && t == 0) {
      acc[5] = clock64() - t0;
      acc[7] = gtimer();
      for (int i = 0; i < 8; ++i) out[i] = acc[i];
    }
  }
};

// take the next item of a shared counter (leader) and broadcast it to the team
__device__ __forceinline__ int take(const Team& tm, int* counter, int* slot) {
  if (tm.t == 0) *slot = atomicAdd(counter, 1);
  tm.bar();
  const int v = *slot;
  tm.bar();
  return v;
}

__device__ __forceinline__ void team_wait(const Team& tm, const int* p, int target, int* err) {
  if (tm.t == 0) wait_geq(p, target, err);
  tm.bar();
}

// publish the team's global writes: the barrier orders them before the
// leader's release (cumulative), the consumer acquires the counter
__device__ __forceinline__ void team_signal(const Team& tm, int* p, int v) {
  tm.bar();
  if (tm.t == 0) red_release(p, v);
}

// "reads done" (a ring slot may be overwritten): the team's loads have all
// returned (their values were consumed before the barrier), so a relaxed
// increment suffices and does not wait for the team's outstanding stores
__device__ __forceinline__ void team_reads_done(const Team& tm, int* p, int v) {
  tm.bar();
  if (tm.t == 0) atomicAdd(p, v);
}

// next item of a shared-memory pool (leader) broadcast to the team
__device__ __forceinline__ int take_smem(const Team& tm, int* counter, int* slot) {
  if (tm.t == 0) *slot = atomicAdd(counter, 1);
  tm.bar();
  const int v = *slot;
  tm.bar();
  return v;
}

// Global row-item counter with one item in flight: the leader requests the
// next index while the team works on the current one.
struct RowTaker {
  int* counter;
  int nxt;
  __device__ __forceinline__ void start(const Team& tm, int* c) {
    counter = c;
    if (tm.t == 0) nxt = atomicAdd(counter, 1);
  }
  __device__ __forceinline__ int next(const Team& tm, int* slot, int limit) {
    if (tm.t == 0) *slot = nxt;
    tm.bar();
    const int v = *slot;
    tm.bar();
    if (tm.t == 0 && v < limit) nxt = atomicAdd(counter, 1);
    return v;
  }
};

}  // namespace pipe

// Counters (ints, zeroed per vector): [0,nz) rows_done, [nz,2nz) cols_done,
// [2nz,3nz) row_next, then the err flag.  The per-CTA column pools (one per
// layer, index nz = prologue / epilogue) live in shared memory after the team
// buffers.
__host__ __device__ inline int pipe_err_index(int nz, int) { return 3 * nz; }

namespace pipe {

// Per-CTA column bookkeeping in shared memory: coldone[ci] = layers finished
// on column slot ci (forward: layer l of a column starts when coldone == l, so
// any team may run it while one column's accumulations stay ordered).
__device__ __forceinline__ void col_wait(const Team& tm, volatile int* flag, int target, int* err) {
  if (tm.t == 0) {
    for (long long spins = 0; *flag < target; ++spins) {
      if (spins > (1ll << 26)) {
        atomicExch(err, 1);
        break;
      }
      __nanosleep(20);
    }
  }
  tm.bar();
  tmem_fence_after();
}

__device__ __forceinline__ void col_release(const Team& tm, volatile int* flag, int value) {
  tmem_fence_before();
  tm.bar();
  if (tm.t == 0) {
    __threadfence_block();
    *flag = value;
  }
}

}  // namespace pipe

template <class PL, int TEAMS>
__global__ void __launch_bounds__(TEAMS * pipe::TT, 1) k_pipe_fwd(PipeArgs a, FFTDesc<typename PL::Scalar> d) {
  using namespace pipe;
  using C = Cfg<PL>;
  using T = typename C::T;
  using V = typename C::V;
  using WD = Words<V>;
  constexpr int E = C::E, NT = C::NT, L = C::L, HX = C::HX, NI = C::NI;
  constexpr int MAXC = 512 / C::COLS;
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ uint32_t taddr_s;
  __shared__ int item_s[TEAMS];
  __shared__ int coldone_s[MAXC];
  const int warp = threadIdx.x / 32, team = threadIdx.x / TT;
  const Team tm{team, (int)threadIdx.x % TT, 0, TeamSync{1 + team, TT}};
  const int t = tm.t;
  const bool active = t < NT;
  V* sm = reinterpret_cast<V*>(smraw) + (long long)team * C::team_slots();
  const int G = gridDim.x, cta = blockIdx.x;
  const int ncol = a.Hx > cta ? (a.Hx - cta + G - 1) / G : 0;  // columns owned by this CTA
  int* rows_done = a.sync;
  int* cols_done = a.sync + a.nz;
  int* row_next = a.sync + 2 * a.nz;
  int* cpool = reinterpret_cast<int*>(smraw + (size_t)TEAMS * C::team_slots() * sizeof(V));
  int* err = a.sync + pipe_err_index(a.nz, G);
  const int npairs = (a.ny + 1) / 2;
  Stats st;
  st.init(a.stats ? a.stats + 8 * (cta * TEAMS + team) : nullptr);
  if (warp == 0) tmem_alloc<512>(&taddr_s);
  if (threadIdx.x < MAXC) coldone_s[threadIdx.x] = 0;
  for (int i = threadIdx.x; i <= a.nz; i += blockDim.x) cpool[i] = 0;
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tbase = taddr_s + ((uint32_t)(32 * (warp & 3)) << 16);
  for (int ci = team; ci < ncol; ci += TEAMS) {  // zero the accumulators
    uint32_t z[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) z[i] = 0u;
#pragma unroll
    for (int g = 0; g < C::GROUPS; ++g) tmem_st16(tbase + ci * C::COLS + 16 * g, z);
  }
  tmem_wait_st();
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const T h = T(0.5);
  const V* S = static_cast<const V*>(a.S);
  V* ring = static_cast<V*>(a.ring);
  const T* X = static_cast<const T*>(a.in);
  const uint32_t rowbytes = (uint32_t)(a.nx * sizeof(T));
  const bool rows_pf = (rowbytes % 16) == 0 && (a.n_r * sizeof(T)) % 16 == 0;
  for (int l = 0; l <= a.nz; ++l) {
    if (l < a.nz) {  // ---- row pairs of layer l -> ring slot l % NB
      V* Y = ring + (long long)(l % a.nb) * a.ring_sstride;
      const T* xl = X + (long long)l * a.n_r;
      bool waited = l < a.nb;
      RowTaker rt;
      rt.start(tm, row_next + l);
      for (;;) {
        const int item = rt.next(tm, item_s + team, npairs);
        if (item >= npairs) break;
        if (t == 0 && rows_pf && item + TEAMS < npairs) {  // rows a few items ahead -> L2
          const T* nxt = xl + (long long)2 * (item + TEAMS) * a.nx;
          prefetch_l2(nxt, rowbytes);
          if (2 * (item + TEAMS) + 1 < a.ny) prefetch_l2(nxt + a.nx, rowbytes);
        }
        if (!waited) {
          const long long w0 = st.now();
          team_wait(tm, cols_done + (l - a.nb), a.Hx, err);
          st.add(0, w0);
          waited = true;
        }
        const long long r0 = st.now();
        const int qa = 2 * item, qb = qa + 1;
        const bool vb = qb < a.ny;
        const T* ra = xl + (long long)qa * a.nx;
        const T* rb = xl + (long long)(vb ? qb : qa) * a.nx;
        V v[E];
#pragma unroll
        for (int k = 0; k < E; ++k) {
          const int i = t + NT * k;
          const bool inb = active && i < a.nx;
          v[k] = mkc<V>(inb ? __ldcs(ra + i) : T(0), inb && vb ? __ldcs(rb + i) : T(0));
        }
        PL::fft_team(v, sm, t, d, active, tm.sync);
        tm.bar();
#pragma unroll
        for (int k = 0; k < E; ++k)
          if (active) sm[PL::slot(t + NT * k)] = v[k];
        tm.bar();
#pragma unroll
        for (int i = 0; i < NI; ++i) {
          const int kx = t + TT * i;
          if (kx < HX) {
            const V zk = sm[PL::slot(kx)];
            const V zm = sm[PL::slot(kx == 0 ? 0 : L - kx)];
            V* o = Y + (long long)kx * a.ny + qa;
            o[0] = mkc<V>(h * (zk.x + zm.x), h * (zk.y - zm.y));
            if (vb) o[1] = mkc<V>(h * (zk.y + zm.y), h * (zm.x - zk.x));
          }
        }
        team_signal(tm, rows_done + l, 1);
        st.add(1, r0);
        st.count(3);
      }
    }
    if (l > 0) {  // ---- this CTA's columns of layer l-1: FFT_y, times S, accumulate in TMEM
      const int lc = l - 1;
      const V* Y = ring + (long long)(lc % a.nb) * a.ring_sstride;
      {
        const long long w0 = st.now();
        team_wait(tm, rows_done + lc, npairs, err);
        st.add(0, w0);
      }
      for (;;) {
        const int ci = take_smem(tm, cpool + lc, item_s + team);
        if (ci >= ncol) break;
        {
          const long long w0 = st.now();
          col_wait(tm, coldone_s + ci, lc, err);
          st.add(0, w0);
        }
        const long long c0 = st.now();
        const int kx = cta + G * ci;
        const V* sc = S + (long long)lc * a.s_rstride + (long long)kx * a.lds;
        const V* yc = Y + (long long)kx * a.ny;
        // fp32: the spectrum column is loaded into registers before the FFT
        // (latency hidden by it); fp64 has no registers to spare for that, so
        // the column is bulk-prefetched into L2 and read per TMEM group after.
        constexpr bool SREG = sizeof(T) == 4;
        V w[SREG ? E : 1], v[E];
        if constexpr (SREG) {
#pragma unroll
          for (int k = 0; k < E; ++k) w[k] = active ? __ldcs(sc + t + NT * k) : mkc<V>(T(0), T(0));
        } else {
          if (t == 0) prefetch_l2(sc, (uint32_t)(L * sizeof(V)));
        }
        if (t == 0 && lc + 1 < a.nz) prefetch_l2(sc + a.s_rstride, (uint32_t)(L * sizeof(V)));
#pragma unroll
        for (int k = 0; k < E; ++k) {
          const int q = t + NT * k;
          v[k] = active && q < a.ny ? __ldcg(yc + q) : mkc<V>(T(0), T(0));
        }
        PL::fft_team(v, sm, t, d, active, tm.sync);
        team_reads_done(tm, cols_done + lc, 1);  // this column of the ring slot is consumed
#pragma unroll
        for (int g = 0; g < C::GROUPS; ++g) {
          uint32_t u[16];
          V wg[C::PER];
#pragma unroll
          for (int c = 0; c < C::PER; ++c) {
            const int k = C::PER * g + c;
            if constexpr (SREG)
              wg[c] = w[k];
            else
              wg[c] = active ? __ldcs(sc + t + NT * k) : mkc<V>(T(0), T(0));
          }
          tmem_ld16(tbase + ci * C::COLS + 16 * g, u);
          tmem_wait_ld();
#pragma unroll
          for (int c = 0; c < C::PER; ++c) {
            const int k = C::PER * g + c;
            V o = WD::get(u + WD::W * c);
            o.x += wg[c].x * v[k].x - wg[c].y * v[k].y;
            o.y += wg[c].x * v[k].y + wg[c].y * v[k].x;
            WD::put(o, u + WD::W * c);
          }
          tmem_st16(tbase + ci * C::COLS + 16 * g, u);
        }
        tmem_wait_st();
        col_release(tm, coldone_s + ci, lc + 1);
        st.add(2, c0);
        st.count(4);
      }
    }
  }
  // ---- epilogue: one inverse column FFT per owned column -> W[kx][j < sy]
  V* Wout = static_cast<V*>(a.out);
  for (;;) {
    const int ci = take_smem(tm, cpool + a.nz, item_s + team);
    if (ci >= ncol) break;
    col_wait(tm, coldone_s + ci, a.nz, err);
    const int kx = cta + G * ci;
    V v[E];
#pragma unroll
    for (int g = 0; g < C::GROUPS; ++g) {
      uint32_t u[16];
      tmem_ld16(tbase + ci * C::COLS + 16 * g, u);
      tmem_wait_ld();
#pragma unroll
      for (int c = 0; c < C::PER; ++c) v[C::PER * g + c] = conjv(WD::get(u + WD::W * c));
    }
    PL::fft_team(v, sm, t, d, active, tm.sync);
    V* wc = Wout + (long long)kx * a.sy;
#pragma unroll
    for (int k = 0; k < E; ++k) {
      const int j = t + NT * k;
      if (active && j < a.sy) wc[j] = conjv(v[k]);
    }
    tm.bar();
  }
  st.flush(t);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if (warp == 0) tmem_dealloc<512>(taddr_s);
}

template <class PL, int TEAMS>
__global__ void __launch_bounds__(TEAMS * pipe::TT, 1) k_pipe_tra(PipeArgs a, FFTDesc<typename PL::Scalar> d) {
  using namespace pipe;
  using C = Cfg<PL>;
  using T = typename C::T;
  using V = typename C::V;
  using WD = Words<V>;
  constexpr int E = C::E, NT = C::NT, L = C::L, HX = C::HX, NI = C::NI;
  constexpr int MAXC = 512 / C::COLS;
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ uint32_t taddr_s;
  __shared__ int item_s[TEAMS];
  __shared__ int coldone_s[MAXC];
  const int warp = threadIdx.x / 32, team = threadIdx.x / TT;
  const Team tm{team, (int)threadIdx.x % TT, 0, TeamSync{1 + team, TT}};
  const int t = tm.t;
  const bool active = t < NT;
  V* sm = reinterpret_cast<V*>(smraw) + (long long)team * C::team_slots();
  const int G = gridDim.x, cta = blockIdx.x;
  const int ncol = a.Hx > cta ? (a.Hx - cta + G - 1) / G : 0;
  int* rows_done = a.sync;
  int* cols_done = a.sync + a.nz;
  int* row_next = a.sync + 2 * a.nz;
  int* cpool = reinterpret_cast<int*>(smraw + (size_t)TEAMS * C::team_slots() * sizeof(V));
  int* err = a.sync + pipe_err_index(a.nz, G);
  const int npairs = (a.ny + 1) / 2;
  Stats st;
  st.init(a.stats ? a.stats + 8 * (cta * TEAMS + team) : nullptr);
  if (warp == 0) tmem_alloc<512>(&taddr_s);
  if (threadIdx.x < MAXC) coldone_s[threadIdx.x] = 0;
  for (int i = threadIdx.x; i <= a.nz; i += blockDim.x) cpool[i] = 0;
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tbase = taddr_s + ((uint32_t)(32 * (warp & 3)) << 16);
  const V* D = static_cast<const V*>(a.in);
  // ---- prologue: the data spectrum of every owned column into TMEM (read-only after)
  for (;;) {
    const int ci = take_smem(tm, cpool + a.nz, item_s + team);
    if (ci >= ncol) break;
    const int kx = cta + G * ci;
    const V* dc = D + (long long)kx * a.sy;
    V v[E];
#pragma unroll
    for (int k = 0; k < E; ++k) {
      const int j = t + NT * k;
      v[k] = active && j < a.sy ? dc[j] : mkc<V>(T(0), T(0));
    }
    PL::fft_team(v, sm, t, d, active, tm.sync);
#pragma unroll
    for (int g = 0; g < C::GROUPS; ++g) {
      uint32_t u[16];
#pragma unroll
      for (int c = 0; c < C::PER; ++c) WD::put(v[C::PER * g + c], u + WD::W * c);
      tmem_st16(tbase + ci * C::COLS + 16 * g, u);
    }
    tmem_wait_st();
    col_release(tm, coldone_s + ci, 1);
  }
  const V* S = static_cast<const V*>(a.S);
  V* ring = static_cast<V*>(a.ring);
  T* Xo = static_cast<T*>(a.out);
  for (int l = 0; l <= a.nz; ++l) {
    if (l < a.nz) {  // ---- owned columns of layer l: S * conj(D^), inverse FFT_y -> ring
      V* Y = ring + (long long)(l % a.nb) * a.ring_sstride;
      if (l >= a.nb) {
        const long long w0 = st.now();
        team_wait(tm, rows_done + (l - a.nb), npairs, err);
        st.add(0, w0);
      }
      int done = 0;
      for (;;) {
        const int ci = take_smem(tm, cpool + l, item_s + team);
        if (ci >= ncol) break;
        {
          const long long w0 = st.now();
          col_wait(tm, coldone_s + ci, 1, err);
          st.add(0, w0);
        }
        const long long c0 = st.now();
        const int kx = cta + G * ci;
        const V* sc = S + (long long)l * a.s_rstride + (long long)kx * a.lds;
        if (t == 0 && l + 1 < a.nz) prefetch_l2(sc + a.s_rstride, (uint32_t)(L * sizeof(V)));
        V v[E];
#pragma unroll
        for (int k = 0; k < E; ++k) v[k] = active ? __ldcs(sc + t + NT * k) : mkc<V>(T(0), T(0));
#pragma unroll
        for (int g = 0; g < C::GROUPS; ++g) {
          uint32_t u[16];
          tmem_ld16(tbase + ci * C::COLS + 16 * g, u);
          tmem_wait_ld();
#pragma unroll
          for (int c = 0; c < C::PER; ++c) {
            const int k = C::PER * g + c;
            const V hh = WD::get(u + WD::W * c);
            const V w = v[k];
            // conj(conj(S) * dh) = S * conj(dh): inverse FFT via the conjugation identity
            v[k] = mkc<V>(w.x * hh.x + w.y * hh.y, w.y * hh.x - w.x * hh.y);
          }
        }
        PL::fft_team(v, sm, t, d, active, tm.sync);
        V* yc = Y + (long long)kx * a.ny;
#pragma unroll
        for (int k = 0; k < E; ++k) {
          const int q = t + NT * k;
          if (active && q < a.ny) yc[q] = conjv(v[k]);
        }
        ++done;
        st.add(2, c0);
        st.count(4);
      }
      team_signal(tm, cols_done + l, done);
    }
    if (l > 0) {  // ---- row pairs of layer l-1: C2R -> model rows
      const int lr = l - 1;
      const V* Y = ring + (long long)(lr % a.nb) * a.ring_sstride;
      T* xl = Xo + (long long)lr * a.n_r;
      bool waited = false;
      RowTaker rt;
      rt.start(tm, row_next + lr);
      for (;;) {
        const int item = rt.next(tm, item_s + team, npairs);
        if (item >= npairs) break;
        if (!waited) {
          const long long w0 = st.now();
          team_wait(tm, cols_done + lr, a.Hx, err);
          st.add(0, w0);
          waited = true;
        }
        const long long r0 = st.now();
        const int ja = 2 * item, jb = ja + 1;
        const bool vb = jb < a.ny;
#pragma unroll
        for (int i = 0; i < NI; ++i) {
          const int kx = t + TT * i;
          if (kx < HX) {
            const V* p = Y + (long long)kx * a.ny + ja;
            V A = __ldcg(p);
            V B = vb ? __ldcg(p + 1) : mkc<V>(T(0), T(0));
            if (kx == 0 || 2 * kx == L) {  // Hermitian projection (.real semantics)
              A.y = T(0);
              B.y = T(0);
            }
            sm[PL::slot(kx)] = mkc<V>(A.x - B.y, A.y + B.x);
            if (kx >= 1 && kx <= L - HX) sm[PL::slot(L - kx)] = mkc<V>(A.x + B.y, B.x - A.y);
          }
        }
        team_reads_done(tm, rows_done + lr, 1);  // includes the barrier before the smem reads
        V v[E];
#pragma unroll
        for (int k = 0; k < E; ++k) v[k] = active ? conjv(sm[PL::slot(t + NT * k)]) : mkc<V>(T(0), T(0));
        PL::fft_team(v, sm, t, d, active, tm.sync);
        T* oa = xl + (long long)ja * a.nx;
        T* ob = xl + (long long)(vb ? jb : ja) * a.nx;
#pragma unroll
        for (int k = 0; k < E; ++k) {
          const int i = t + NT * k;
          if (active && i < a.nx) {
            __stcs(oa + i, v[k].x);
            if (vb) __stcs(ob + i, -v[k].y);
          }
        }
        tm.bar();  // the exchange buffer is rewritten by the next item
        st.add(1, r0);
        st.count(3);
      }
    }
  }
  st.flush(t);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if (warp == 0) tmem_dealloc<512>(taddr_s);
}

}  // namespace bttb
