// C ABI (include/bttb_sm100.h): plan = the device-resident spectrum cache plus
// the launch schedule of the fused forward / transpose operator.
//
// Reference counterparts: build_transform_stack (transform.py:91-104),
// apply (multiply.py:22-58), layer_response_window (kernels.py:158-184),
// gravity_layer_response / magnetic_response (kernels.py:81-155).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "bttb_sm100.h"
#include "cgls.h"
#include "entries.h"
#include "generic.h"
#include "hoststage.h"
#include "spectral.h"

using namespace bttb;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CU(expr)                                                                                   \
  do {                                                                                             \
    cudaError_t e_ = (expr);                                                                       \
    if (e_ != cudaSuccess) return fail(BTTB_ECUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                                       __FILE__, __LINE__);                                       \
  } while (0)

// --- FFT length family and radix plans ------------------------------------
int length_family(int64_t L) {  // returns E (elements per thread) or 0
  if (L < 8 || L > 8192) return 0;
  int64_t t = L;
  int a = 0, b = 0, c = 0;
  while (t % 2 == 0) { t /= 2; ++a; }
  while (t % 3 == 0) { t /= 3; ++b; }
  while (t % 5 == 0) { t /= 5; ++c; }
  if (t != 1) return 0;
  if (b == 0 && c == 0 && a >= 3) return 8;
  if (c == 0 && a >= 2 && b >= 1) return 12;
  if (b == 0 && a >= 2 && c >= 1) return 20;
  return 0;
}

// FFT length for an embedding of n: the smallest supported length >= n,
// except that a power of two within 5% of it is preferred when it has a
// compile-time plan (fp64 2048 with 16 elements per thread runs the team FFT
// at 338 vs 246 Gpt/s for 2000; the C4 step measured 4.14 vs 5.00 ms).
// BTTB_FFT_POW2=0 turns the preference off.
int64_t pick_length(int64_t n) {
  int64_t best = -1;
  for (int64_t L = std::max<int64_t>(n, 8); L <= 8192; ++L)
    if (length_family(L)) { best = L; break; }
  if (best < 0) return generic_length(n);  // above 8192: the generic path (generic.cu)
  static const bool pow2 = !(getenv("BTTB_FFT_POW2") && atoi(getenv("BTTB_FFT_POW2")) == 0);
  int64_t p2 = 8;
  while (p2 < n) p2 *= 2;
  if (pow2 && p2 != best && p2 <= 8192 && p2 * 100 <= best * 105) {
    int rad[16];
    if (static_radices((int)p2, true, rad) > 0 && static_radices((int)p2, false, rad) > 0) return p2;
  }
  return best;
}

// Radix plan of one length at one precision: E elements per thread
// (fp64 keeps E small for register pressure: 8 / 12 / 10; fp32: 8 / 12 / 20).
struct RadixPlan {
  int E = 0, nt = 0, npass = 0;
  int radix[8] = {0};
  int init(int L, int fam, bool fp64) {
    E = fam == 20 && fp64 ? 10 : fam;
    nt = L / E;
    static const int c8[] = {8, 4, 2, 0}, c12[] = {12, 6, 4, 3, 2, 0}, c20[] = {20, 10, 5, 4, 2, 0},
                     c10[] = {10, 5, 2, 0};
    const int* cand = E == 8 ? c8 : E == 12 ? c12 : E == 20 ? c20 : c10;
    int rem = L;
    npass = 0;
    while (rem > 1) {
      int r = 0;
      for (const int* p = cand; *p; ++p)
        if (rem % *p == 0) { r = *p; break; }
      if (!r || npass == 8) return fail(BTTB_EINVAL, "no radix plan for length %d", L);
      radix[npass++] = r;
      rem /= r;
    }
    return BTTB_OK;
  }
  unsigned code() const {
    unsigned c = 0;
    for (int i = 0; i < npass; ++i) c |= radix_code(radix[i]) << (4 * i);
    return c;
  }
};

// Per-pass twiddle tables of a radix sequence: for each pass p with NS > 1,
// entry (r-1)*NS + k = exp(-2*pi*i*r*k/(NS*R)), r < R, k < NS (fft.cuh sfft).
template <class C>
std::vector<C> per_pass_table(const int* radix, int npass) {
  std::vector<C> out;
  long ns = 1;
  for (int p = 0; p < npass; ++p) {
    const int R = radix[p];
    if (ns > 1)
      for (int r = 1; r < R; ++r)
        for (long k = 0; k < ns; ++k) {
          const long double ang = 2.0L * 3.141592653589793238462643383279502884L * (long double)(r * k) /
                                  (long double)(ns * R);
          C c;
          c.x = (decltype(c.x))cosl(ang);
          c.y = (decltype(c.y))(-sinl(ang));
          out.push_back(c);
        }
    ns *= R;
  }
  return out;
}

struct FFTPlanHost;
template <class T> const void* tw816(const FFTPlanHost& h);
struct FFTPlanHost {
  int L = 0;
  RadixPlan p64, p32;
  double2* tw64 = nullptr;
  float2* tw32 = nullptr;
  double2* twp64 = nullptr;  // per-pass tables of the registered compile-time plans (or null)
  float2* twp32 = nullptr;
  double2* tw816_64 = nullptr;  // L = 2048: per-pass tables of the 8/16/16 order (mirrored C2R)
  float2* tw816_32 = nullptr;

  int init(int64_t len) {
    L = (int)len;
    const int fam = length_family(len);
    if (!fam) return fail(BTTB_EINVAL, "unsupported FFT length %lld", (long long)len);
    int rc;
    if ((rc = p64.init(L, fam, true)) || (rc = p32.init(L, fam, false))) return rc;
    std::vector<double2> h64(L);
    std::vector<float2> h32(L);
    for (int m = 0; m < L; ++m) {
      // exp(-2 pi i m / L), evaluated in extended precision then rounded
      const long double ang = 2.0L * 3.141592653589793238462643383279502884L * (long double)m / (long double)L;
      const long double c = cosl(ang), s = -sinl(ang);
      h64[m] = make_double2((double)c, (double)s);
      h32[m] = make_float2((float)c, (float)s);
    }
    CU(cudaMalloc(&tw64, sizeof(double2) * L));
    CU(cudaMalloc(&tw32, sizeof(float2) * L));
    CU(cudaMemcpy(tw64, h64.data(), sizeof(double2) * L, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(tw32, h32.data(), sizeof(float2) * L, cudaMemcpyHostToDevice));
    int rad[16];
    int np = static_radices(L, true, rad);
    if (np > 0) {
      std::vector<double2> t = per_pass_table<double2>(rad, np);
      CU(cudaMalloc(&twp64, sizeof(double2) * std::max<size_t>(t.size(), 1)));
      if (!t.empty()) CU(cudaMemcpy(twp64, t.data(), sizeof(double2) * t.size(), cudaMemcpyHostToDevice));
    }
    np = static_radices(L, false, rad);
    if (np > 0) {
      std::vector<float2> t = per_pass_table<float2>(rad, np);
      CU(cudaMalloc(&twp32, sizeof(float2) * std::max<size_t>(t.size(), 1)));
      if (!t.empty()) CU(cudaMemcpy(twp32, t.data(), sizeof(float2) * t.size(), cudaMemcpyHostToDevice));
    }
    if (L == 2048) {
      const int r816[3] = {8, 16, 16};
      std::vector<double2> t64 = per_pass_table<double2>(r816, 3);
      std::vector<float2> t32 = per_pass_table<float2>(r816, 3);
      CU(cudaMalloc(&tw816_64, sizeof(double2) * t64.size()));
      CU(cudaMalloc(&tw816_32, sizeof(float2) * t32.size()));
      CU(cudaMemcpy(tw816_64, t64.data(), sizeof(double2) * t64.size(), cudaMemcpyHostToDevice));
      CU(cudaMemcpy(tw816_32, t32.data(), sizeof(float2) * t32.size(), cudaMemcpyHostToDevice));
    }
    return BTTB_OK;
  }
  void release() {
    if (tw64) cudaFree(tw64);
    if (tw32) cudaFree(tw32);
    if (twp64) cudaFree(twp64);
    if (twp32) cudaFree(twp32);
    if (tw816_64) cudaFree(tw816_64);
    if (tw816_32) cudaFree(tw816_32);
    tw816_64 = nullptr;
    tw816_32 = nullptr;
    tw64 = nullptr;
    tw32 = nullptr;
    twp64 = nullptr;
    twp32 = nullptr;
  }
  template <class T> const RadixPlan& plan() const {
    if constexpr (std::is_same<T, double>::value) return p64; else return p32;
  }
  template <class T> int E() const { return plan<T>().E; }
  template <class T> FFTDesc<T> desc() const {
    FFTDesc<T> d;
    if constexpr (std::is_same<T, double>::value) {
      d.tw = tw64;
      d.twp = twp64;
    } else {
      d.tw = tw32;
      d.twp = twp32;
    }
    const RadixPlan& rp = plan<T>();
    d.L = L;
    d.nt = rp.nt;
    d.npass = rp.npass;
    d.code = rp.code();
    return d;
  }
};
template <> const void* tw816<double>(const FFTPlanHost& h) { return h.tw816_64; }
template <> const void* tw816<float>(const FFTPlanHost& h) { return h.tw816_32; }

// Development guard zones (BTTB_GUARD=1, read once per process): every plan
// buffer and the spectrum cache get kGuard bytes of a fixed byte pattern on
// both sides; bttb_debug_check_guards reports buffers whose guards changed --
// out-of-bounds writes of any kernel into neighbouring memory.  (The pool's
// compute-sanitizer is unavailable; this plus the boundary / determinism
// tests in tests/test_gpu_guards.py stands in for memcheck.)
constexpr size_t kGuard = 1 << 16;
constexpr unsigned char kGuardByte = 0xA5;
bool guards_on() {
  static const bool on = getenv("BTTB_GUARD") && atoi(getenv("BTTB_GUARD")) != 0;
  return on;
}
int guard_alloc(void** p, size_t n) {
  if (!guards_on()) return cudaMalloc(p, n) == cudaSuccess ? 0 : 1;
  char* base = nullptr;
  if (cudaMalloc(reinterpret_cast<void**>(&base), n + 2 * kGuard) != cudaSuccess) return 1;
  if (cudaMemset(base, kGuardByte, kGuard) != cudaSuccess ||
      cudaMemset(base + kGuard + n, kGuardByte, kGuard) != cudaSuccess) {
    cudaFree(base);
    return 1;
  }
  *p = base + kGuard;
  return 0;
}
void guard_free(void* p) {
  if (p) cudaFree(guards_on() ? static_cast<char*>(p) - kGuard : p);
}
// 0: both guards intact (or guards off), 1: a guard byte changed, -1: copy failed
int guard_intact(const void* p, size_t n) {
  if (!guards_on() || !p) return 0;
  std::vector<unsigned char> h(kGuard);
  const char* base = static_cast<const char*>(p) - kGuard;
  for (const char* g : {base, base + kGuard + n}) {
    if (cudaMemcpy(h.data(), g, kGuard, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
    for (unsigned char c : h)
      if (c != kGuardByte) return 1;
  }
  return 0;
}

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  int ensure(size_t n) {
    if (n <= bytes) return BTTB_OK;
    guard_free(p);
    p = nullptr;
    bytes = 0;
    if (guard_alloc(&p, n)) {
      p = nullptr;
      cudaError_t e = cudaGetLastError();
      return fail(BTTB_ENOMEM, "cudaMalloc(%zu bytes) failed: %s", n, cudaGetErrorString(e));
    }
    bytes = n;
    return BTTB_OK;
  }
  void release() {
    guard_free(p);
    p = nullptr;
    bytes = 0;
  }
  int intact() const { return guard_intact(p, bytes); }
};

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// Bytes of chunk intermediate per apply.  Measured on C4 fp64: one chunk for
// all 128 layers (2 GB; 5.56 ms/step) beats L2-sized chunks (96 MB: 7.16 ms):
// the kernels are compute/latency-bound, and one chunk means no accumulator
// round trips, one inverse column FFT per column and 6 launches per step.
size_t chunk_budget() {
  const char* env = getenv("BTTB_CHUNK_BYTES");
  if (env) return (size_t)atoll(env);
  return (size_t)4 << 30;
}

size_t round_up(size_t n, size_t a) { return (n + a - 1) / a * a; }

}  // namespace

struct bttb_plan_s {
  int device = 0, dtype = BTTB_F64, kind = BTTB_GRAVITY;
  int64_t sx = 0, sy = 0, nz = 0, pxl = 0, pxr = 0, pyl = 0, pyr = 0, nx = 0, ny = 0, mx = 0, my = 0;
  double dx = 0, dy = 0;
  std::vector<double> z;
  int64_t l0 = 0, l1 = 0, nzl = 0;
  double gs = 0, gc[5] = {0, 0, 0, 0, 0};
  int64_t Lx = 0, Ly = 0, Hx = 0;
  FFTPlanHost fx, fy;
  size_t elem = 16;
  void* spectra = nullptr;
  // generic-length path (generic.cu): lengths outside the shared-memory
  // engine's family (above 8192), or every plan under BTTB_GENERIC=1
  bool generic = false;
  GenericCtx gen;
  double2* gen_tw[2] = {nullptr, nullptr};
  DevBuf work, hin, hout;
  HostStage hstage;  // pinned chunk ring for pageable host buffers (BTTB_HOST_PTR)
  DevBuf cg, cg_hist;  // CGLS driver workspace and residual history (bttb_cgls)
  cudaStream_t stream = nullptr;   // internal stream the products run on
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  // BTTB_HOST_ASYNC: copy streams and a ring of device staging slots, so one
  // call's device-to-host copy overlaps the next calls' host-to-device copies
  // (full-duplex PCIe) and both overlap compute; four slots let alternating
  // forward / transpose calls each double-buffer their input
  static constexpr int kRing = 4;
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  DevBuf ain[kRing], aout[kRing];
  cudaEvent_t ev_h2d[kRing] = {}, ev_in_free[kRing] = {}, ev_out_ready[kRing] = {}, ev_out_free[kRing] = {};
  cudaEvent_t ev_call = nullptr;
  static constexpr int kHostChunks = 4;  // layer ranges of the chunked BTTB_HOST_PTR path
  cudaEvent_t ev_chunk[kHostChunks] = {};
  int ring = 0;
  int64_t last_K = 0, last_G = 0, last_launches = 0;
  std::mutex mu;

  int64_t n_r() const { return nx * ny; }
  int64_t m() const { return sx * sy; }
  int64_t nloc() const { return n_r() * nzl; }
};

namespace {

// corner vectors exactly as the reference forms its distance tables
void corner_vectors(const bttb_plan_s* p, std::vector<double>& cx, std::vector<double>& cy) {
  if (p->kind == BTTB_GRAVITY) {  // sym_distances, grid.py:177-187
    const int64_t lx = p->sx + std::max(p->pxl, p->pxr) + 1, ly = p->sy + std::max(p->pyl, p->pyr) + 1;
    cx.resize(lx);
    cy.resize(ly);
    for (int64_t l = 0; l < lx; ++l) cx[l] = ((double)l - 0.5) * p->dx;
    for (int64_t l = 0; l < ly; ++l) cy[l] = ((double)l - 0.5) * p->dy;
  } else {  // full_distances sliced to the window, grid.py:190-199 + kernels.py:178-183
    cx.resize(p->mx + 1);
    cy.resize(p->my + 1);
    for (int64_t c = 0; c <= p->mx; ++c) cx[c] = ((double)(c - p->sx - p->pxl) + 0.5) * p->dx;
    for (int64_t c = 0; c <= p->my; ++c) cy[c] = ((double)(c - p->sy - p->pyl) + 0.5) * p->dy;
  }
}

struct EntryScratch {
  DevBuf cx, cy, cm, mag, flag;
  int ncx = 0, ncy = 0;
  MagCorners mc{};
  int init(const std::vector<double>& hx, const std::vector<double>& hy, int kind) {
    ncx = (int)hx.size();
    ncy = (int)hy.size();
    const size_t nc = (size_t)ncx * ncy;
    int rc;
    if ((rc = cx.ensure(sizeof(double) * ncx)) || (rc = cy.ensure(sizeof(double) * ncy)) ||
        (rc = flag.ensure(sizeof(int))))
      return rc;
    CU(cudaMemcpy(cx.p, hx.data(), sizeof(double) * ncx, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(cy.p, hy.data(), sizeof(double) * ncy, cudaMemcpyHostToDevice));
    CU(cudaMemset(flag.p, 0, sizeof(int)));
    if (kind == BTTB_GRAVITY) {
      if ((rc = cm.ensure(sizeof(double) * nc))) return rc;
    } else {
      if ((rc = mag.ensure(sizeof(double) * nc * 6))) return rc;
      double* b = static_cast<double*>(mag.p);
      mc = MagCorners{b, b + nc, b + 2 * nc, b + 3 * nc, b + 4 * nc, b + 5 * nc};
    }
    return BTTB_OK;
  }
  void release() {
    cx.release();
    cy.release();
    cm.release();
    mag.release();
    flag.release();
  }
};

const char* kind_name(int kind) { return kind == BTTB_GRAVITY ? "gravity" : "magnetic"; }

int check_flag(EntryScratch& s, int kind) {
  int h = 0;
  CU(cudaMemcpy(&h, s.flag.p, sizeof(int), cudaMemcpyDeviceToHost));
  if (h)
    return fail(BTTB_ENONFINITE,
                "non-finite value in %s response; staggered distances should make this impossible",
                kind_name(kind));
  return BTTB_OK;
}

EmbedArgs embed_args(const bttb_plan_s* p) {
  EmbedArgs a;
  a.kind = p->kind;
  a.sx = (int)p->sx;
  a.sy = (int)p->sy;
  a.nx = (int)p->nx;
  a.ny = (int)p->ny;
  a.pxl = (int)p->pxl;
  a.pyl = (int)p->pyl;
  a.Lx = (int)p->Lx;
  a.Ly = (int)p->Ly;
  return a;
}

GC5 gc5(const bttb_plan_s* p) {
  GC5 g;
  for (int i = 0; i < 5; ++i) g.v[i] = p->gc[i];
  return g;
}

int layer_corners(bttb_plan_s* p, EntryScratch& s, int64_t layer, cudaStream_t st) {
  const double z1 = p->z[layer], z2 = p->z[layer + 1];
  CU(launch_corners(p->kind, (const double*)s.cx.p, s.ncx, (const double*)s.cy.p, s.ncy, nullptr, nullptr, z1, z2,
                    p->gs, (double*)s.cm.p, s.mc, st));
  return BTTB_OK;
}

// host_windows (optional): local layers x mx x my caller-supplied response
// windows (the reference-format stack loader); otherwise entries are generated.
int build_spectra(bttb_plan_s* p, const double* host_windows = nullptr) {
  std::vector<double> hx, hy;
  EntryScratch s;
  DevBuf emb, yb, win;
  int rc = BTTB_OK;
  if (host_windows) {
    rc = s.flag.ensure(sizeof(int));
    if (!rc) rc = win.ensure(sizeof(double) * p->mx * p->my);
    if (!rc && cudaMemset(s.flag.p, 0, sizeof(int)) != cudaSuccess) rc = fail(BTTB_ECUDA, "flag reset failed");
  } else {
    corner_vectors(p, hx, hy);
    rc = s.init(hx, hy, p->kind);
  }
  if (!rc) rc = emb.ensure(sizeof(double) * p->Lx * p->Ly);
  if (!rc) rc = yb.ensure(sizeof(double2) * p->Hx * p->Ly);
  if (rc) {
    s.release();
    return rc;
  }
  cudaStream_t st = 0;
  const EmbedArgs ea = embed_args(p);
  const FFTDesc<double> dx = p->generic ? FFTDesc<double>{} : p->fx.desc<double>();
  const FFTDesc<double> dy = p->generic ? FFTDesc<double>{} : p->fy.desc<double>();
  const double scale = 1.0 / ((double)p->Lx * (double)p->Ly);
  for (int64_t r = 0; r < p->nzl && !rc; ++r) {
    const int64_t g = p->l0 + r;
    cudaError_t e;
    if (host_windows) {
      const size_t wn = (size_t)p->mx * p->my;
      e = cudaMemcpyAsync(win.p, host_windows + (size_t)r * wn, sizeof(double) * wn, cudaMemcpyHostToDevice, st);
      if (e == cudaSuccess) e = launch_embed_window(ea, (int)p->my, (const double*)win.p, (int*)s.flag.p,
                                                    (double*)emb.p, st);
    } else {
      rc = layer_corners(p, s, g, st);
      if (rc) break;
      e = launch_embed(ea, (const double*)s.cm.p, s.mc, (const double*)s.cx.p, (const double*)s.cy.p, s.ncy,
                       p->z[g], p->z[g + 1], gc5(p), (int*)s.flag.p, (double*)emb.p, st);
    }
    if (e != cudaSuccess) { rc = fail(BTTB_ECUDA, "embed: %s", cudaGetErrorString(e)); break; }
    if (p->generic) {
      void* sr = static_cast<char*>(p->spectra) + (size_t)r * p->Hx * p->Ly * p->elem;
      e = p->dtype == BTTB_F64 ? generic_build_layer<double>(p->gen, (const double*)emb.p, sr, st)
                               : generic_build_layer<float>(p->gen, (const double*)emb.p, sr, st);
      if (e != cudaSuccess) { rc = fail(BTTB_ECUDA, "generic spectrum build: %s", cudaGetErrorString(e)); break; }
      continue;
    }
    RowR2CArgs ra{};
    ra.in = emb.p;
    ra.in_bstride = 0;
    ra.in_sstride = 0;
    ra.spb = 1;
    ra.ld_in = (int)p->Lx;
    ra.nrows = (int)p->Ly;
    ra.nvalid = (int)p->Lx;
    ra.nslabs = 1;
    ra.out = yb.p;
    ra.out_sstride = 0;
    ra.ld_out = (int)p->Ly;
    ra.Hx = (int)p->Hx;
    e = launch_row_r2c<double>(ra, dx, p->fx.E<double>(), st);
    if (e != cudaSuccess) { rc = fail(BTTB_ECUDA, "build row pass: %s", cudaGetErrorString(e)); break; }
    ColSpecArgs ca{};
    ca.Y = yb.p;
    ca.ldy = (int)p->Ly;
    ca.S = static_cast<char*>(p->spectra) + (size_t)r * p->Hx * p->Ly * p->elem;
    ca.lds = (int)p->Ly;
    ca.Hx = (int)p->Hx;
    ca.scale = scale;
    e = p->dtype == BTTB_F64 ? launch_col_spec<double>(ca, dy, p->fy.E<double>(), st)
                             : launch_col_spec<float>(ca, dy, p->fy.E<double>(), st);
    if (e != cudaSuccess) { rc = fail(BTTB_ECUDA, "build column pass: %s", cudaGetErrorString(e)); break; }
  }
  if (!rc) {
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = fail(BTTB_ECUDA, "spectrum build: %s", cudaGetErrorString(e));
  }
  if (!rc) rc = check_flag(s, p->kind);
  s.release();
  emb.release();
  yb.release();
  win.release();
  return rc;
}

// stage: BTTB_STAGE_ALL runs the whole product; the split stages meet at the
// station half spectrum W[b][kx][j < sy] (x frequency, y space: Hx x sy complex
// per item) -- forward: TO_SPECTRUM = row R2C + column stage (the plan's layers'
// partial W, column-inverse-transformed), FROM_SPECTRUM = row C2R of a (summed)
// W; transpose: TO_SPECTRUM = row R2C of the data, FROM_SPECTRUM = column stage +
// row C2R into the plan's layers.  x / y are then W where the stage says so.
// generic-length path (generic.cu): whole products only, one vector at a time
template <class T>
int run_generic(bttb_plan_s* p, int mode, const void* x, void* y, int64_t batch, cudaStream_t st, int stage) {
  if (stage != BTTB_STAGE_ALL)
    return fail(BTTB_EINVAL, "split products are not available for the generic-length plan (FFT lengths %lld x %lld)",
                (long long)p->Lx, (long long)p->Ly);
  const int64_t nloc = p->nloc(), m = p->m();
  for (int64_t b = 0; b < batch; ++b) {
    if (mode == BTTB_FORWARD)
      CU((generic_forward<T>(p->gen, p->spectra, p->nzl, static_cast<const T*>(x) + b * nloc, (int)p->nx, (int)p->ny,
                             static_cast<T*>(y) + b * m, (int)p->sx, (int)p->sy, st)));
    else
      CU((generic_transpose<T>(p->gen, p->spectra, p->nzl, static_cast<const T*>(x) + b * m, (int)p->sx,
                               (int)p->sy, static_cast<T*>(y) + b * nloc, (int)p->nx, (int)p->ny, st)));
  }
  p->last_K = p->nzl;
  p->last_G = 1;
  p->last_launches = -1;  // many small pass kernels; not counted
  return BTTB_OK;
}

// [L0, L1): the plan's layers this call covers (default all).  A partial range
// (the chunked host path below: batch 1, whole product) adds its layers to the
// station half spectrum W of the earlier ranges (forward; the row inverse runs
// with the last range) or fills its layers of the output (transpose; the data
// half spectrum is built with the first range and kept in the workspace).
template <class T>
int run_apply(bttb_plan_s* p, int mode, const void* x, void* y, int64_t batch, cudaStream_t st,
              int stage = BTTB_STAGE_ALL, int64_t L0 = 0, int64_t L1 = -1) {
  if (p->generic) return run_generic<T>(p, mode, x, y, batch, st, stage);
  if (L1 < 0) L1 = p->nzl;
  const bool rows_in = stage != BTTB_STAGE_FROM_SPECTRUM, rows_out = stage != BTTB_STAGE_TO_SPECTRUM;
  using V = cplx<T>;
  const FFTDesc<T> dx = p->fx.desc<T>(), dy = p->fy.desc<T>();
  const int64_t Hx = p->Hx, nx = p->nx, ny = p->ny, sx = p->sx, sy = p->sy, n_r = p->n_r(), m = p->m(),
                nloc = p->nloc();
  const size_t slab = (size_t)Hx * ny * sizeof(V);
  const size_t budget = chunk_budget();
  int64_t K = std::max<int64_t>(1, std::min<int64_t>(p->nzl, (int64_t)(budget / slab)));
  int64_t G = 1;
  if (K == p->nzl) G = std::max<int64_t>(1, std::min<int64_t>(batch, (int64_t)(budget / (slab * p->nzl))));
  int rc;
  // workspace: the chunk intermediate Y (row-pass output / transposed column
  // output) then the accumulator / data half-spectrum W
  const size_t ybytes = round_up(slab * K * G, 4096), wbytes = round_up((size_t)Hx * sy * sizeof(V) * G, 4096);
  if ((rc = p->work.ensure(ybytes + wbytes))) return rc;
  p->last_K = K;
  p->last_G = G;
  int64_t launches = L0 > 0 ? p->last_launches : 0;
  V* Yb = static_cast<V*>(p->work.p);
  V* Wb = reinterpret_cast<V*>(static_cast<char*>(p->work.p) + ybytes);
  const V* S = static_cast<const V*>(p->spectra);
  const long long s_rstride = (long long)Hx * p->Ly;
  for (int64_t b0 = 0; b0 < batch; b0 += G) {
    const int gb = (int)std::min<int64_t>(G, batch - b0);
    if (mode == BTTB_FORWARD) {
      const T* xin = static_cast<const T*>(x) + b0 * nloc;
      // split stages: W lives in the caller's buffer (y for TO_, x for FROM_)
      V* Wg = stage == BTTB_STAGE_TO_SPECTRUM     ? static_cast<V*>(y) + b0 * Hx * sy
              : stage == BTTB_STAGE_FROM_SPECTRUM ? const_cast<V*>(static_cast<const V*>(x)) + b0 * Hx * sy
                                                  : Wb;
      for (int64_t r0 = L0; rows_in && r0 < L1; r0 += K) {
        const int k = (int)std::min<int64_t>(K, L1 - r0);
        RowR2CArgs ra{};
        ra.in = xin + r0 * n_r;
        ra.in_bstride = nloc;
        ra.in_sstride = n_r;
        ra.spb = k;
        ra.ld_in = (int)nx;
        ra.nrows = (int)ny;
        ra.nvalid = (int)nx;
        ra.nslabs = gb * k;
        ra.out = Yb;
        ra.out_sstride = (long long)Hx * ny;
        ra.ld_out = (int)ny;
        ra.Hx = (int)Hx;
        CU(launch_row_r2c<T>(ra, dx, p->fx.template E<T>(), st));
        ColFwdArgs ca{};
        ca.Y = Yb;
        ca.y_bstride = (long long)k * Hx * ny;
        ca.y_rstride = (long long)Hx * ny;
        ca.ldy = (int)ny;
        ca.nvalid = (int)ny;
        ca.S = S + r0 * s_rstride;
        ca.s_rstride = s_rstride;
        ca.lds = (int)p->Ly;
        ca.K = k;
        ca.W = Wg;
        ca.w_bstride = (long long)Hx * sy;
        ca.ldw = (int)sy;
        ca.nout = (int)sy;
        ca.accumulate = r0 > 0;
        ca.Hx = (int)Hx;
        ca.nbatch = gb;
        CU(launch_col_fwd<T>(ca, dy, p->fy.template E<T>(), st));
        launches += 2;
      }
      if (!rows_out || L1 != p->nzl) continue;
      RowC2RArgs oa{};
      oa.in = Wg;
      oa.in_sstride = (long long)Hx * sy;
      oa.ld_in = (int)sy;
      oa.nrows = (int)sy;
      oa.Hx = (int)Hx;
      oa.nslabs = gb;
      oa.out = static_cast<T*>(y) + b0 * m;
      oa.out_bstride = m;
      oa.out_sstride = 0;
      oa.spb = 1;
      oa.ld_out = (int)sx;
      oa.nout = (int)sx;
      oa.tw_816 = tw816<T>(p->fx);
      CU(launch_row_c2r<T>(oa, dx, p->fx.template E<T>(), st));
      launches += 1;
    } else {
      V* Dg = stage == BTTB_STAGE_TO_SPECTRUM     ? static_cast<V*>(y) + b0 * Hx * sy
              : stage == BTTB_STAGE_FROM_SPECTRUM ? const_cast<V*>(static_cast<const V*>(x)) + b0 * Hx * sy
                                                  : Wb;
      if (rows_in && L0 == 0) {
        RowR2CArgs ra{};
        ra.in = static_cast<const T*>(x) + b0 * m;
        ra.in_bstride = m;
        ra.in_sstride = 0;
        ra.spb = 1;
        ra.ld_in = (int)sx;
        ra.nrows = (int)sy;
        ra.nvalid = (int)sx;
        ra.nslabs = gb;
        ra.out = Dg;
        ra.out_sstride = (long long)Hx * sy;
        ra.ld_out = (int)sy;
        ra.Hx = (int)Hx;
        CU(launch_row_r2c<T>(ra, dx, p->fx.template E<T>(), st));
        launches += 1;
      }
      T* yout = static_cast<T*>(y) + b0 * nloc;
      for (int64_t r0 = L0; rows_out && r0 < L1; r0 += K) {
        const int k = (int)std::min<int64_t>(K, L1 - r0);
        ColTraArgs ca{};
        ca.D = Dg;
        ca.d_bstride = (long long)Hx * sy;
        ca.ldd = (int)sy;
        ca.nvalid = (int)sy;
        ca.S = S + r0 * s_rstride;
        ca.s_rstride = s_rstride;
        ca.lds = (int)p->Ly;
        ca.K = k;
        ca.W = Yb;
        ca.w_bstride = (long long)k * Hx * ny;
        ca.w_rstride = (long long)Hx * ny;
        ca.ldw = (int)ny;
        ca.nout = (int)ny;
        ca.Hx = (int)Hx;
        ca.nbatch = gb;
        CU(launch_col_tra<T>(ca, dy, p->fy.template E<T>(), st));
        RowC2RArgs oa{};
        oa.in = Yb;
        oa.in_sstride = (long long)Hx * ny;
        oa.ld_in = (int)ny;
        oa.nrows = (int)ny;
        oa.Hx = (int)Hx;
        oa.nslabs = gb * k;
        oa.out = yout + r0 * n_r;
        oa.out_bstride = nloc;
        oa.out_sstride = n_r;
        oa.spb = k;
        oa.ld_out = (int)nx;
        oa.nout = (int)nx;
        oa.tw_816 = tw816<T>(p->fx);
        CU(launch_row_c2r<T>(oa, dx, p->fx.template E<T>(), st));
        launches += 2;
      }
    }
  }
  p->last_launches = launches;
  return BTTB_OK;
}

void generic_release(bttb_plan_s* p) {
  for (double2*& t : p->gen_tw) {
    if (t) cudaFree(t);
    t = nullptr;
  }
  for (double2** b : {&p->gen.A, &p->gen.B, &p->gen.C}) {
    guard_free(*b);
    *b = nullptr;
  }
}

void destroy_plan(bttb_plan_s* p) {
  if (!p) return;
  DeviceGuard g(p->device);
  if (p->spectra) guard_free(p->spectra);
  generic_release(p);
  p->hstage.release();
  p->fx.release();
  p->fy.release();
  p->work.release();
  p->cg.release();
  p->cg_hist.release();
  if (p->stream) cudaStreamDestroy(p->stream);
  if (p->s_h2d) cudaStreamDestroy(p->s_h2d);
  if (p->s_d2h) cudaStreamDestroy(p->s_d2h);
  for (int i = 0; i < bttb_plan_s::kRing; ++i) {
    p->ain[i].release();
    p->aout[i].release();
    for (cudaEvent_t ev : {p->ev_h2d[i], p->ev_in_free[i], p->ev_out_ready[i], p->ev_out_free[i]})
      if (ev) cudaEventDestroy(ev);
  }
  if (p->ev_call) cudaEventDestroy(p->ev_call);
  for (cudaEvent_t& ev : p->ev_chunk) {
    if (ev) cudaEventDestroy(ev);
    ev = nullptr;
  }
  if (p->ev_in) cudaEventDestroy(p->ev_in);
  if (p->ev_out) cudaEventDestroy(p->ev_out);
  p->hin.release();
  p->hout.release();
  delete p;
}

}  // namespace

namespace {

// Device-resident batched CGLS (PAPER.md:640 future work).
// Textbook CGLS (Hestenes-Stiefel form on the normal equations) from m0 = 0:
//   r = d, s = G^T r, p = s, gamma = |s|^2
//   per iteration: q = G p; alpha = gamma / (|q|^2 + damp^2 |p|^2);
//                  m += alpha p; r -= alpha q; s = G^T r - damp^2 m;
//                  beta = |s|^2 / gamma; gamma = |s|^2; p = s + beta p.
// Everything stays on the plan's stream: products through run_apply, vector
// updates and fp64 reductions through cgls.cu, scalars in device memory.
// Converged items freeze (alpha = beta = 0) once |s_k| <= rtol |s_0|, rtol =
// 1e-13 (fp64) / 1e-6 (fp32): past convergence CG only amplifies rounding.
template <class T>
int run_cgls(bttb_plan_s* p, const T* d, T* mo, int64_t batch, int iters, double damp, double* hist_dev,
                    cudaStream_t st) {
  const int64_t m = p->m(), n = p->nloc();
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, p->device);
  const int bm = cgls_blocks(m, (int)batch, nsm), bn = cgls_blocks(n, (int)batch, nsm);
  const double damp2 = damp * damp;
  const size_t vm = round_up(sizeof(T) * m * batch, 256), vn = round_up(sizeof(T) * n * batch, 256);
  const size_t pa = round_up(sizeof(double) * batch * (bm > bn ? bm : bn), 256);
  const size_t scb = round_up(sizeof(CglsScalars) * batch, 256);
  int rc;
  if ((rc = p->cg.ensure(2 * vm + 2 * vn + 2 * pa + scb))) return rc;
  char* w = static_cast<char*>(p->cg.p);
  T* r = reinterpret_cast<T*>(w);
  T* q = reinterpret_cast<T*>(w + vm);
  T* s = reinterpret_cast<T*>(w + 2 * vm);
  T* pv = reinterpret_cast<T*>(w + 2 * vm + vn);
  double* pa0 = reinterpret_cast<double*>(w + 2 * vm + 2 * vn);
  double* pa1 = reinterpret_cast<double*>(w + 2 * vm + 2 * vn + pa);
  CglsScalars* sc = reinterpret_cast<CglsScalars*>(w + 2 * vm + 2 * vn + 2 * pa);
  const int hld = iters + 1;
  int64_t nl = 0;  // kernels launched (operator products + vector kernels)
  CU(cudaMemcpyAsync(r, d, sizeof(T) * m * batch, cudaMemcpyDeviceToDevice, st));
  CU(cudaMemsetAsync(mo, 0, sizeof(T) * n * batch, st));
  if ((rc = run_apply<T>(p, BTTB_TRANSPOSE, r, s, batch, st))) return rc;
  nl += p->last_launches + 3;
  CU(cgls_dot<T>(s, s, n, (int)batch, bn, pa0, st));
  CU(cgls_dot<T>(r, r, m, (int)batch, bm, pa1, st));
  CU(cgls_scalars(CGLS_INIT, (int)batch, pa0, bn, pa1, bm, damp2, sizeof(T) == 8 ? 1e-13 : 1e-6, sc, hist_dev, hld, 0,
                    st));
  CU(cudaMemcpyAsync(pv, s, sizeof(T) * n * batch, cudaMemcpyDeviceToDevice, st));
  for (int it = 0; it < iters; ++it) {
    if ((rc = run_apply<T>(p, BTTB_FORWARD, pv, q, batch, st))) return rc;
    nl += p->last_launches + (damp2 != 0.0 ? 7 : 6);
    CU(cgls_dot<T>(q, q, m, (int)batch, bm, pa0, st));
    if (damp2 != 0.0) CU(cgls_dot<T>(pv, pv, n, (int)batch, bn, pa1, st));
    CU(cgls_scalars(CGLS_ALPHA, (int)batch, pa0, bm, damp2 != 0.0 ? pa1 : nullptr, bn, damp2, 0.0, sc, nullptr, hld,
                    0, st));
    CU(cgls_resid<T>(r, q, m, (int)batch, bm, sc, pa1, st));
    if ((rc = run_apply<T>(p, BTTB_TRANSPOSE, r, s, batch, st))) return rc;
    nl += p->last_launches;
    // |s|^2 partials; damped: first m += alpha p and s -= damp^2 m
    CU(cgls_update<T>(mo, pv, s, n, (int)batch, bn, sc, damp2, pa0, 0, st));
    CU(cgls_scalars(CGLS_BETA, (int)batch, pa0, bn, pa1, bm, damp2, 0.0, sc, hist_dev, hld, it + 1, st));
    CU(cgls_update<T>(mo, pv, s, n, (int)batch, bn, sc, damp2, nullptr, 1, st));
  }
  p->last_launches = nl;
  return BTTB_OK;
}

}  // namespace

extern "C" {

const char* bttb_last_error(void) { return g_err.c_str(); }

const char* bttb_version(void) { return "bttb_sm100 0.1.0 (sm_100a)"; }

int64_t bttb_fft_length(int64_t n) { return pick_length(n); }

// generic path setup: exact twiddle tables exp(-2 pi i t / L) (extended
// precision, rounded once) and the three work grids
static int generic_init(bttb_plan_s* p) {
  const int64_t Ls[2] = {p->Lx, p->Ly};
  for (int a = 0; a < 2; ++a) {
    std::vector<double2> h(Ls[a]);
    for (int64_t m = 0; m < Ls[a]; ++m) {
      const long double ang = 2.0L * 3.141592653589793238462643383279502884L * (long double)m / (long double)Ls[a];
      h[m] = make_double2((double)cosl(ang), (double)(-sinl(ang)));
    }
    CU(cudaMalloc(&p->gen_tw[a], sizeof(double2) * Ls[a]));
    CU(cudaMemcpy(p->gen_tw[a], h.data(), sizeof(double2) * Ls[a], cudaMemcpyHostToDevice));
  }
  GenericCtx& g = p->gen;
  g.Lx = (int)p->Lx;
  g.Ly = (int)p->Ly;
  g.Hx = (int)p->Hx;
  if (g.fx.init(g.Lx, p->gen_tw[0]) || g.fy.init(g.Ly, p->gen_tw[1]))
    return fail(BTTB_EINVAL, "no radix plan for lengths (%d, %d)", g.Lx, g.Ly);
  const size_t n = (size_t)p->Lx * p->Ly * sizeof(double2);
  double2** bufs[3] = {&g.A, &g.B, &g.C};
  for (double2** b : bufs)
    if (guard_alloc(reinterpret_cast<void**>(b), n)) {
      *b = nullptr;
      return fail(BTTB_ENOMEM, "cannot allocate %zu bytes of generic-path work grid", n);
    }
  return BTTB_OK;
}

static int plan_create_impl(bttb_plan** out, const bttb_grid* grid, const bttb_kernel* kernel, int dtype,
                            int device, int64_t layer_begin, int64_t layer_end, int64_t Lx, int64_t Ly,
                            const void* host_spectra, const double* host_windows = nullptr) {
  g_err.clear();
  if (!out || !grid || !kernel) return fail(BTTB_EINVAL, "null argument");
  *out = nullptr;
  if (grid->sx < 1 || grid->sy < 1 || grid->nz < 1) return fail(BTTB_EINVAL, "sx, sy, nz must be positive");
  if (grid->pxl < 0 || grid->pxr < 0 || grid->pyl < 0 || grid->pyr < 0)
    return fail(BTTB_EINVAL, "padding must be non-negative");
  if (!(grid->dx > 0) || !(grid->dy > 0)) return fail(BTTB_EINVAL, "dx, dy must be positive");
  if (!grid->z_blocks) return fail(BTTB_EINVAL, "z_blocks is null");
  if (kernel->kind != BTTB_GRAVITY && kernel->kind != BTTB_MAGNETIC) return fail(BTTB_EINVAL, "unknown kernel kind");
  if (dtype != BTTB_F64 && dtype != BTTB_F32) return fail(BTTB_EINVAL, "unknown dtype");
  if (layer_begin < 0 || layer_end > grid->nz || layer_begin >= layer_end)
    return fail(BTTB_EINVAL, "layer range [%lld, %lld) outside [0, %lld)", (long long)layer_begin,
                (long long)layer_end, (long long)grid->nz);
  for (int64_t r = 0; r < grid->nz; ++r) {
    const double z1 = grid->z_blocks[r], z2 = grid->z_blocks[r + 1];
    if (z2 < z1) return fail(BTTB_EINVAL, "layer depths must satisfy z2 >= z1, got (%g, %g)", z1, z2);
    if (z1 < 0) return fail(BTTB_EINVAL, "layer top must satisfy z1 >= 0, got %g", z1);
  }
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return fail(BTTB_ECUDA, "no CUDA device available (%s)", cudaGetErrorString(e));
  if (device < 0 || device >= ndev) return fail(BTTB_EINVAL, "device %d out of range (%d devices)", device, ndev);
  DeviceGuard dg(device);
  bttb_plan_s* p = new bttb_plan_s();
  p->device = device;
  p->dtype = dtype;
  p->kind = kernel->kind;
  p->sx = grid->sx; p->sy = grid->sy; p->nz = grid->nz;
  p->pxl = grid->pxl; p->pxr = grid->pxr; p->pyl = grid->pyl; p->pyr = grid->pyr;
  p->nx = p->sx + p->pxl + p->pxr;
  p->ny = p->sy + p->pyl + p->pyr;
  p->mx = p->sx + p->nx - 1;
  p->my = p->sy + p->ny - 1;
  p->dx = grid->dx;
  p->dy = grid->dy;
  p->z.assign(grid->z_blocks, grid->z_blocks + grid->nz + 1);
  p->l0 = layer_begin;
  p->l1 = layer_end;
  p->nzl = layer_end - layer_begin;
  p->gs = kernel->gamma_scaled;
  for (int i = 0; i < 5; ++i) p->gc[i] = kernel->gc[i];
  p->Lx = Lx > 0 ? Lx : pick_length(p->mx);
  p->Ly = Ly > 0 ? Ly : pick_length(p->my);
  int rc = BTTB_OK;
  // the shared-memory engine covers its length family up to 8192; anything
  // else 2^a 3^b 5^c runs the generic path (BTTB_GENERIC=1 forces it, tests)
  const char* genv = getenv("BTTB_GENERIC");
  p->generic = (genv && atoi(genv) != 0) || !length_family(p->Lx) || !length_family(p->Ly);
  if (p->Lx < p->mx || p->Ly < p->my || !generic_length_ok(p->Lx) || !generic_length_ok(p->Ly) ||
      (double)p->Lx * (double)p->Ly >= 2147483648.0) {
    rc = fail(BTTB_EINVAL,
              "FFT lengths (%lld, %lld) unsupported for embedding (%lld, %lld): each must be >= the embedding, "
              "of the form 2^a 3^b 5^c and at most 65536, with Lx*Ly < 2^31",
              (long long)p->Lx, (long long)p->Ly, (long long)p->mx, (long long)p->my);
  }
  if (!rc) {
    p->Hx = p->Lx / 2 + 1;
    p->elem = dtype == BTTB_F64 ? sizeof(double2) : sizeof(float2);
    rc = p->generic ? generic_init(p) : p->fx.init(p->Lx);
  }
  if (!rc && !p->generic) rc = p->fy.init(p->Ly);
  if (!rc) {
    const size_t bytes = (size_t)p->nzl * p->Hx * p->Ly * p->elem;
    e = guard_alloc(&p->spectra, bytes) ? cudaErrorMemoryAllocation : cudaSuccess;
    if (e != cudaSuccess) {
      p->spectra = nullptr;
      rc = fail(BTTB_ENOMEM, "cannot allocate %zu bytes of spectrum cache: %s", bytes, cudaGetErrorString(e));
    }
  }
  if (!rc) {
    bool ok = cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking) == cudaSuccess &&
              cudaEventCreateWithFlags(&p->ev_in, cudaEventDisableTiming) == cudaSuccess &&
              cudaEventCreateWithFlags(&p->ev_out, cudaEventDisableTiming) == cudaSuccess;
    for (int i = 0; i < bttb_plan_s::kRing && ok; ++i)
      ok = cudaEventCreateWithFlags(&p->ev_h2d[i], cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&p->ev_in_free[i], cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&p->ev_out_ready[i], cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&p->ev_out_free[i], cudaEventDisableTiming) == cudaSuccess;
    ok = ok && cudaStreamCreateWithFlags(&p->s_h2d, cudaStreamNonBlocking) == cudaSuccess &&
         cudaStreamCreateWithFlags(&p->s_d2h, cudaStreamNonBlocking) == cudaSuccess &&
         cudaEventCreateWithFlags(&p->ev_call, cudaEventDisableTiming) == cudaSuccess;
    if (!ok) rc = fail(BTTB_ECUDA, "cannot create the plan streams/events");
  }
  if (!rc) {
    if (host_spectra) {
      const size_t bytes = (size_t)p->nzl * p->Hx * p->Ly * p->elem;
      cudaError_t ce = cudaMemcpy(p->spectra, host_spectra, bytes, cudaMemcpyHostToDevice);
      if (ce != cudaSuccess) rc = fail(BTTB_ECUDA, "spectrum upload: %s", cudaGetErrorString(ce));
    } else {
      rc = build_spectra(p, host_windows);
    }
  }
  if (rc) {
    std::string msg = g_err;
    destroy_plan(p);
    g_err = msg;
    return rc;
  }
  *out = p;
  return BTTB_OK;
}

int bttb_plan_create(bttb_plan** out, const bttb_grid* grid, const bttb_kernel* kernel, int dtype, int device,
                     int64_t layer_begin, int64_t layer_end, int64_t Lx, int64_t Ly) {
  return plan_create_impl(out, grid, kernel, dtype, device, layer_begin, layer_end, Lx, Ly, nullptr);
}

int bttb_plan_create_from_spectra(bttb_plan** out, const bttb_grid* grid, const bttb_kernel* kernel, int dtype,
                                  int device, int64_t layer_begin, int64_t layer_end, int64_t Lx, int64_t Ly,
                                  const void* host_spectra) {
  if (!host_spectra) return fail(BTTB_EINVAL, "null spectra");
  if (Lx <= 0 || Ly <= 0) return fail(BTTB_EINVAL, "FFT lengths must be given for cached spectra");
  return plan_create_impl(out, grid, kernel, dtype, device, layer_begin, layer_end, Lx, Ly, host_spectra);
}

int bttb_plan_create_from_windows(bttb_plan** out, const bttb_grid* grid, const bttb_kernel* kernel, int dtype,
                                  int device, int64_t layer_begin, int64_t layer_end, int64_t Lx, int64_t Ly,
                                  const double* host_windows) {
  if (!host_windows) return fail(BTTB_EINVAL, "null windows");
  return plan_create_impl(out, grid, kernel, dtype, device, layer_begin, layer_end, Lx, Ly, nullptr, host_windows);
}

int bttb_debug_check_guards(bttb_plan* p) {
  g_err.clear();
  if (!p) return fail(BTTB_EINVAL, "null plan");
  if (!guards_on()) return 0;
  std::lock_guard<std::mutex> lock(p->mu);
  DeviceGuard dg(p->device);
  if (cudaDeviceSynchronize() != cudaSuccess) return fail(BTTB_ECUDA, "device error before the guard check");
  int bad = 0;
  const size_t sbytes = (size_t)p->nzl * p->Hx * p->Ly * p->elem;
  bad += guard_intact(p->spectra, sbytes) != 0;
  const DevBuf* bufs[] = {&p->work, &p->hin, &p->hout, &p->cg, &p->cg_hist};
  for (const DevBuf* b : bufs) bad += b->intact() != 0;
  for (int i = 0; i < bttb_plan_s::kRing; ++i) bad += (p->ain[i].intact() != 0) + (p->aout[i].intact() != 0);
  return bad;
}

int bttb_plan_destroy(bttb_plan* plan) {
  destroy_plan(plan);
  return BTTB_OK;
}

// layer-chunked overlap of copies and compute in the synchronous host path; BTTB_HOST_CHUNKS=0 off
static bool host_chunks_ok() {
  static const bool on = !(getenv("BTTB_HOST_CHUNKS") && atoi(getenv("BTTB_HOST_CHUNKS")) == 0);
  return on;
}

int bttb_apply(bttb_plan* p, int mode, const void* x, void* y, int64_t batch, int where, void* stream) {
  g_err.clear();
  if (!p || !x || !y) return fail(BTTB_EINVAL, "null argument");
  if (mode != BTTB_FORWARD && mode != BTTB_TRANSPOSE)
    return fail(BTTB_EINVAL, "mode must be 'forward' or 'transpose', got %d", mode);
  if (batch < 0) return fail(BTTB_EINVAL, "batch must be >= 0");
  if (batch == 0) return BTTB_OK;
  std::lock_guard<std::mutex> lock(p->mu);
  DeviceGuard dg(p->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t in_elems = (size_t)batch * (mode == BTTB_FORWARD ? p->nloc() : p->m());
  const size_t out_elems = (size_t)batch * (mode == BTTB_FORWARD ? p->m() : p->nloc());
  const size_t esz = p->elem / 2;
  if (where == BTTB_HOST_ASYNC || where == BTTB_HOST_ASYNC_UNORDERED) {
    // ring slot i: H2D (s_h2d) -> compute (plan stream) -> D2H (s_d2h); a slot
    // is reused only after its previous compute read ain[i] / its previous D2H
    // read aout[i].  The caller's stream waits for this call's D2H.
    const int i = p->ring;
    p->ring = (p->ring + 1) % bttb_plan_s::kRing;
    int rc;
    if ((rc = p->ain[i].ensure(in_elems * esz)) || (rc = p->aout[i].ensure(out_elems * esz))) return rc;
    // BTTB_HOST_ASYNC: the input copy follows the work queued on the caller's
    // stream (x may be produced there); BTTB_HOST_ASYNC_UNORDERED drops that
    // edge (it would chain the copy behind the previous call's output copy):
    // x must be final at call time
    if (where == BTTB_HOST_ASYNC) {
      CU(cudaEventRecord(p->ev_in, st));
      CU(cudaStreamWaitEvent(p->s_h2d, p->ev_in, 0));
    }
    CU(cudaStreamWaitEvent(p->s_h2d, p->ev_in_free[i], 0));
    CU(cudaMemcpyAsync(p->ain[i].p, x, in_elems * esz, cudaMemcpyHostToDevice, p->s_h2d));
    CU(cudaEventRecord(p->ev_h2d[i], p->s_h2d));
    CU(cudaStreamWaitEvent(p->stream, p->ev_h2d[i], 0));
    CU(cudaStreamWaitEvent(p->stream, p->ev_out_free[i], 0));
    rc = p->dtype == BTTB_F64 ? run_apply<double>(p, mode, p->ain[i].p, p->aout[i].p, batch, p->stream)
                              : run_apply<float>(p, mode, p->ain[i].p, p->aout[i].p, batch, p->stream);
    if (rc) return rc;
    CU(cudaEventRecord(p->ev_in_free[i], p->stream));
    CU(cudaEventRecord(p->ev_out_ready[i], p->stream));
    CU(cudaStreamWaitEvent(p->s_d2h, p->ev_out_ready[i], 0));
    CU(cudaMemcpyAsync(y, p->aout[i].p, out_elems * esz, cudaMemcpyDeviceToHost, p->s_d2h));
    CU(cudaEventRecord(p->ev_out_free[i], p->s_d2h));
    CU(cudaStreamWaitEvent(st, p->ev_out_free[i], 0));
    return BTTB_OK;
  }
  const void* xd = x;
  void* yd = y;
  // BTTB_HOST_PTR with one large model: the copy of one layer range crosses
  // PCIe while the previous range is computed (forward) / the next range is
  // computed while this one's result leaves (transpose) -- the synchronous
  // call hides its ~1.7 ms of C4 compute behind its 1.03 GB copy.
  constexpr int NC = bttb_plan_s::kHostChunks;
  if (where == BTTB_HOST_PTR && batch == 1 && !p->generic && p->nzl >= 2 * NC &&
      (size_t)p->nloc() * esz >= ((size_t)64 << 20) && host_chunks_ok()) {
    int rc;
    if ((rc = p->hin.ensure(in_elems * esz)) || (rc = p->hout.ensure(out_elems * esz))) return rc;
    for (cudaEvent_t& ev : p->ev_chunk)
      if (!ev) CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    const size_t lbytes = (size_t)p->n_r() * esz;  // one layer of the model
    auto run = [&](int64_t lo, int64_t hi) {
      return p->dtype == BTTB_F64 ? run_apply<double>(p, mode, p->hin.p, p->hout.p, 1, p->stream, BTTB_STAGE_ALL, lo, hi)
                                  : run_apply<float>(p, mode, p->hin.p, p->hout.p, 1, p->stream, BTTB_STAGE_ALL, lo, hi);
    };
    if (mode == BTTB_FORWARD) {
      for (int c = 0; c < NC; ++c) {
        const int64_t lo = p->nzl * c / NC, hi = p->nzl * (c + 1) / NC;
        CU(stage_h2d(p->hstage, static_cast<char*>(p->hin.p) + lo * lbytes, static_cast<const char*>(x) + lo * lbytes,
                     (size_t)(hi - lo) * lbytes, st));
        CU(cudaEventRecord(p->ev_chunk[c], st));
        CU(cudaStreamWaitEvent(p->stream, p->ev_chunk[c], 0));
        if ((rc = run(lo, hi))) return rc;
      }
      CU(cudaEventRecord(p->ev_out, p->stream));
      CU(cudaStreamWaitEvent(st, p->ev_out, 0));
      CU(stage_d2h(p->hstage, y, p->hout.p, out_elems * esz, st));
    } else {
      CU(stage_h2d(p->hstage, p->hin.p, x, in_elems * esz, st));
      CU(cudaEventRecord(p->ev_in, st));
      CU(cudaStreamWaitEvent(p->stream, p->ev_in, 0));
      for (int c = 0; c < NC; ++c) {
        if ((rc = run(p->nzl * c / NC, p->nzl * (c + 1) / NC))) return rc;
        CU(cudaEventRecord(p->ev_chunk[c], p->stream));
      }
      for (int c = 0; c < NC; ++c) {
        const int64_t lo = p->nzl * c / NC, hi = p->nzl * (c + 1) / NC;
        CU(cudaStreamWaitEvent(st, p->ev_chunk[c], 0));
        CU(stage_d2h(p->hstage, static_cast<char*>(y) + lo * lbytes, static_cast<char*>(p->hout.p) + lo * lbytes,
                     (size_t)(hi - lo) * lbytes, st));
      }
    }
    return BTTB_OK;
  }
  if (where == BTTB_HOST_PTR) {
    int rc;
    if ((rc = p->hin.ensure(in_elems * esz)) || (rc = p->hout.ensure(out_elems * esz))) return rc;
    CU(stage_h2d(p->hstage, p->hin.p, x, in_elems * esz, st));
    xd = p->hin.p;
    yd = p->hout.p;
  } else if (where != BTTB_DEVICE_PTR) {
    return fail(BTTB_EINVAL, "where must be BTTB_DEVICE_PTR, BTTB_HOST_PTR, BTTB_HOST_ASYNC or BTTB_HOST_ASYNC_UNORDERED");
  }
  // the work runs on the plan's stream, ordered
  // after everything already queued on the caller's stream and before
  // anything the caller queues next
  CU(cudaEventRecord(p->ev_in, st));
  CU(cudaStreamWaitEvent(p->stream, p->ev_in, 0));
  int rc = p->dtype == BTTB_F64 ? run_apply<double>(p, mode, xd, yd, batch, p->stream)
                                : run_apply<float>(p, mode, xd, yd, batch, p->stream);
  if (rc) return rc;
  CU(cudaEventRecord(p->ev_out, p->stream));
  CU(cudaStreamWaitEvent(st, p->ev_out, 0));
  if (where == BTTB_HOST_PTR) CU(stage_d2h(p->hstage, y, yd, out_elems * esz, st));
  return BTTB_OK;
}

int bttb_cgls(bttb_plan* p, const void* d, void* m_out, int64_t batch, int iters, double damp, int where,
              void* stream, double* resid_norms) {
  g_err.clear();
  if (!p || !d || !m_out) return fail(BTTB_EINVAL, "null argument");
  if (batch < 0 || iters < 0) return fail(BTTB_EINVAL, "batch and iters must be >= 0");
  if (!(damp >= 0.0) || !std::isfinite(damp)) return fail(BTTB_EINVAL, "damp must be finite and >= 0");
  if (p->l0 != 0 || p->l1 != p->nz)
    return fail(BTTB_EINVAL, "cgls needs a plan holding every layer (this plan holds [%lld, %lld) of %lld)",
                (long long)p->l0, (long long)p->l1, (long long)p->nz);
  if (where != BTTB_DEVICE_PTR && where != BTTB_HOST_PTR)
    return fail(BTTB_EINVAL, "where must be BTTB_DEVICE_PTR or BTTB_HOST_PTR");
  if (batch == 0) return BTTB_OK;
  std::lock_guard<std::mutex> lock(p->mu);
  DeviceGuard dg(p->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t esz = p->elem / 2;
  const size_t dbytes = (size_t)batch * p->m() * esz, mbytes = (size_t)batch * p->nloc() * esz;
  const void* dd = d;
  void* md = m_out;
  int rc;
  if (where == BTTB_HOST_PTR) {
    if ((rc = p->hin.ensure(dbytes)) || (rc = p->hout.ensure(mbytes))) return rc;
    CU(stage_h2d(p->hstage, p->hin.p, d, dbytes, st));
    dd = p->hin.p;
    md = p->hout.p;
  }
  // residual history: device scratch owned by the plan (freed with it)
  double* hist = nullptr;
  if (resid_norms) {
    if ((rc = p->cg_hist.ensure(sizeof(double) * batch * (iters + 1)))) return rc;
    hist = static_cast<double*>(p->cg_hist.p);
  }
  CU(cudaEventRecord(p->ev_in, st));
  CU(cudaStreamWaitEvent(p->stream, p->ev_in, 0));
  rc = p->dtype == BTTB_F64
           ? run_cgls<double>(p, static_cast<const double*>(dd), static_cast<double*>(md), batch, iters, damp, hist,
                              p->stream)
           : run_cgls<float>(p, static_cast<const float*>(dd), static_cast<float*>(md), batch, iters, damp, hist,
                             p->stream);
  if (rc) return rc;
  CU(cudaEventRecord(p->ev_out, p->stream));
  CU(cudaStreamWaitEvent(st, p->ev_out, 0));
  if (resid_norms) {
    CU(cudaMemcpyAsync(resid_norms, hist, sizeof(double) * batch * (iters + 1), cudaMemcpyDeviceToHost, st));
  }
  if (where == BTTB_HOST_PTR) CU(stage_d2h(p->hstage, m_out, md, mbytes, st));
  if (resid_norms) CU(cudaStreamSynchronize(st));
  return BTTB_OK;
}

int bttb_apply_staged(bttb_plan* p, int mode, int stage, const void* x, void* y, int64_t batch, void* stream) {
  g_err.clear();
  if (!p || !x || !y) return fail(BTTB_EINVAL, "null argument");
  if (mode != BTTB_FORWARD && mode != BTTB_TRANSPOSE)
    return fail(BTTB_EINVAL, "mode must be 'forward' or 'transpose', got %d", mode);
  if (stage != BTTB_STAGE_ALL && stage != BTTB_STAGE_TO_SPECTRUM && stage != BTTB_STAGE_FROM_SPECTRUM)
    return fail(BTTB_EINVAL, "stage must be BTTB_STAGE_ALL, _TO_SPECTRUM or _FROM_SPECTRUM, got %d", stage);
  if (batch < 0) return fail(BTTB_EINVAL, "batch must be >= 0");
  if (batch == 0) return BTTB_OK;
  std::lock_guard<std::mutex> lock(p->mu);
  DeviceGuard dg(p->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CU(cudaEventRecord(p->ev_in, st));
  CU(cudaStreamWaitEvent(p->stream, p->ev_in, 0));
  int rc = p->dtype == BTTB_F64 ? run_apply<double>(p, mode, x, y, batch, p->stream, stage)
                                : run_apply<float>(p, mode, x, y, batch, p->stream, stage);
  if (rc) return rc;
  CU(cudaEventRecord(p->ev_out, p->stream));
  CU(cudaStreamWaitEvent(st, p->ev_out, 0));
  return BTTB_OK;
}

int bttb_layer_window(bttb_plan* p, int64_t layer, double* host_out) {
  g_err.clear();
  if (!p || !host_out) return fail(BTTB_EINVAL, "null argument");
  if (layer < 0 || layer >= p->nz) return fail(BTTB_EINVAL, "layer %lld out of range", (long long)layer);
  std::lock_guard<std::mutex> lock(p->mu);
  DeviceGuard dg(p->device);
  std::vector<double> hx, hy;
  corner_vectors(p, hx, hy);
  EntryScratch s;
  DevBuf w;
  int rc = s.init(hx, hy, p->kind);
  if (!rc) rc = w.ensure(sizeof(double) * p->mx * p->my);
  if (!rc) rc = layer_corners(p, s, layer, 0);
  if (!rc) {
    cudaError_t e = launch_window(embed_args(p), (int)p->mx, (int)p->my, (const double*)s.cm.p, s.mc,
                                  (const double*)s.cx.p, (const double*)s.cy.p, s.ncy, p->z[layer],
                                  p->z[layer + 1], gc5(p), (int*)s.flag.p, (double*)w.p, 0);
    if (e != cudaSuccess) rc = fail(BTTB_ECUDA, "window: %s", cudaGetErrorString(e));
  }
  if (!rc) {
    cudaError_t e = cudaMemcpy(host_out, w.p, sizeof(double) * p->mx * p->my, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) rc = fail(BTTB_ECUDA, "window copy: %s", cudaGetErrorString(e));
  }
  if (!rc) rc = check_flag(s, p->kind);
  s.release();
  w.release();
  return rc;
}

int bttb_layer_spectrum(bttb_plan* p, int64_t local_layer, void* host_out) {
  g_err.clear();
  if (!p || !host_out) return fail(BTTB_EINVAL, "null argument");
  if (local_layer < 0 || local_layer >= p->nzl) return fail(BTTB_EINVAL, "local layer out of range");
  DeviceGuard dg(p->device);
  const size_t bytes = (size_t)p->Hx * p->Ly * p->elem;
  CU(cudaMemcpy(host_out, static_cast<char*>(p->spectra) + bytes * local_layer, bytes, cudaMemcpyDeviceToHost));
  return BTTB_OK;
}

int bttb_plan_info(const bttb_plan* p, int64_t* info) {
  if (!p || !info) return fail(BTTB_EINVAL, "null argument");
  info[0] = p->Lx;
  info[1] = p->Ly;
  info[2] = p->Hx;
  info[3] = p->l0;
  info[4] = p->l1;
  info[5] = p->dtype;
  info[6] = p->kind;
  info[7] = p->last_K;
  info[8] = p->last_G;
  info[9] = p->last_launches;
  return BTTB_OK;
}

static int raw_response(int kind, const double* x, int64_t ncx, const double* y, int64_t ncy, const double* xy,
                        const double* r2, double z1, double z2, double gs, const double* gc, double* out,
                        int device) {
  g_err.clear();
  if (!x || !y || !out) return fail(BTTB_EINVAL, "null argument");
  if (z2 < z1) return fail(BTTB_EINVAL, "layer depths must satisfy z2 >= z1, got (%g, %g)", z1, z2);
  if (z1 < 0) return fail(BTTB_EINVAL, "layer top must satisfy z1 >= 0, got %g", z1);
  if (ncx < 2 || ncy < 2) return fail(BTTB_EINVAL, "need at least two corners per axis");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(BTTB_ECUDA, "no CUDA device available");
  DeviceGuard dg(device);
  std::vector<double> hx(x, x + ncx), hy(y, y + ncy);
  EntryScratch s;
  DevBuf dxy, dr2, dout;
  int rc = s.init(hx, hy, kind);
  const size_t nc = (size_t)ncx * ncy;
  if (!rc && xy) {
    rc = dxy.ensure(sizeof(double) * nc);
    if (!rc && cudaMemcpy(dxy.p, xy, sizeof(double) * nc, cudaMemcpyHostToDevice) != cudaSuccess)
      rc = fail(BTTB_ECUDA, "copy xy");
  }
  if (!rc && r2) {
    rc = dr2.ensure(sizeof(double) * nc);
    if (!rc && cudaMemcpy(dr2.p, r2, sizeof(double) * nc, cudaMemcpyHostToDevice) != cudaSuccess)
      rc = fail(BTTB_ECUDA, "copy r2");
  }
  const size_t no = (size_t)(ncx - 1) * (ncy - 1);
  if (!rc) rc = dout.ensure(sizeof(double) * no);
  GC5 g{};
  if (gc)
    for (int i = 0; i < 5; ++i) g.v[i] = gc[i];
  if (!rc) {
    cudaError_t e = launch_corners(kind, (const double*)s.cx.p, s.ncx, (const double*)s.cy.p, s.ncy,
                                   (const double*)dxy.p, (const double*)dr2.p, z1, z2, gs, (double*)s.cm.p, s.mc, 0);
    if (e == cudaSuccess)
      e = launch_entries_raw(kind, (const double*)s.cm.p, s.mc, (const double*)s.cx.p, (const double*)s.cy.p, s.ncx,
                             s.ncy, z1, z2, g, (int*)s.flag.p, (double*)dout.p, 0);
    if (e == cudaSuccess) e = cudaMemcpy(out, dout.p, sizeof(double) * no, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) rc = fail(BTTB_ECUDA, "response: %s", cudaGetErrorString(e));
  }
  if (!rc) rc = check_flag(s, kind);
  s.release();
  dxy.release();
  dr2.release();
  dout.release();
  return rc;
}

int bttb_gravity_response(const double* x, int64_t ncx, const double* y, int64_t ncy, const double* xy,
                          const double* r2, double z1, double z2, double gamma_scaled, double* out, int device) {
  return raw_response(BTTB_GRAVITY, x, ncx, y, ncy, xy, r2, z1, z2, gamma_scaled, nullptr, out, device);
}

int bttb_magnetic_response(const double* x, int64_t ncx, const double* y, int64_t ncy, const double* r2,
                           double z1, double z2, const double* gc, double* out, int device) {
  if (!gc) return fail(BTTB_EINVAL, "null gc");
  return raw_response(BTTB_MAGNETIC, x, ncx, y, ncy, nullptr, r2, z1, z2, 0.0, gc, out, device);
}

}  // extern "C"
