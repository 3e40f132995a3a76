// Kernel-entry generators (K1 gravity, K2 magnetic), fp64 always.
//
// COMPILED WITH -fmad=false: every expression below keeps the reference's
// operation order and rounding (no FMA contraction), because the far-field
// entries of the reference are cancellation-prone and the fp64 parity gate
// (rel-L2 <= 1e-10) is only met by reproducing them (risk 1).
// No fast-math, no flush-to-zero: the z1 = 0 top layer relies on signed zeros
// in atan2 (risk 2).
//
// Reference: /root/reference/pkg/src/bttb/kernels.py:81-155 (closed forms),
// kernels.py:158-184 (window), transform.py:85-88 (circulant embedding).
#include <cuda_runtime.h>
#include <cstdint>

#include "entries.h"

namespace bttb {

// ---------------------------------------------------------------------------
// gravity: corner term CM (kernels.py:92-98), one thread per corner
// ---------------------------------------------------------------------------
__global__ void k_grav_corners(const double* __restrict__ cx, int ncx, const double* __restrict__ cy, int ncy,
                               const double* __restrict__ xy_in, const double* __restrict__ r2_in, double z1,
                               double z2, double gs, double* __restrict__ cm) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;  // y corner (contiguous)
  const int i = blockIdx.y;                             // x corner
  if (j >= ncy || i >= ncx) return;
  const double x = cx[i], y = cy[j];
  const long long o = (long long)i * ncy + j;
  const double xy = xy_in ? xy_in[o] : x * y;
  const double r2 = r2_in ? r2_in[o] : x * x + y * y;
  const double R1 = sqrt(r2 + z1 * z1);
  const double R2 = sqrt(r2 + z2 * z2);
  const double cmx = log((x + R1) / (x + R2)) * y;
  const double cmy = log((y + R1) / (y + R2)) * x;
  const double cm56 = atan2(xy, R1 * z1) * z1 - atan2(xy, R2 * z2) * z2;
  cm[o] = (cm56 - cmy - cmx) * gs;
}

// 4-corner difference of entry (p, q) (kernels.py:99)
__device__ __forceinline__ double grav_entry(const double* __restrict__ cm, int ncy, int p, int q) {
  const double* c0 = cm + (long long)p * ncy + q;
  const double* c1 = c0 + ncy;
  return -(c0[0] - c0[1] - c1[0] + c1[1]);
}

// ---------------------------------------------------------------------------
// magnetic: per-corner rho and atan2 terms (kernels.py:116-117, 137-150).
// Sharing a corner term between the four entries that use it is bit-exact:
// each is the same deterministic function of the same inputs.
// ---------------------------------------------------------------------------
__global__ void k_mag_corners(const double* __restrict__ cx, int ncx, const double* __restrict__ cy, int ncy,
                              const double* __restrict__ r2_in, double z1, double z2, MagCorners c) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (j >= ncy || i >= ncx) return;
  const double x = cx[i], y = cy[j];
  const long long o = (long long)i * ncy + j;
  const double r2 = r2_in ? r2_in[o] : x * x + y * y;
  const double p1 = sqrt(r2 + z1 * z1);
  const double p2 = sqrt(r2 + z2 * z2);
  c.p1[o] = p1;
  c.p2[o] = p2;
  c.axz1[o] = atan2(x * z1, p1 * y);
  c.axz2[o] = atan2(x * z2, p2 * y);
  c.ayz1[o] = atan2(y * z1, p1 * x);
  c.ayz2[o] = atan2(y * z2, p2 * x);
}

// Entry (a, b) from corners (a..a+1) x (b..b+1) (kernels.py:119-155)
__device__ __forceinline__ double mag_entry(const MagCorners& c, const double* __restrict__ cx,
                                            const double* __restrict__ cy, int ncy, int a, int b, double z1,
                                            double z2, const double* gc) {
  const long long o00 = (long long)a * ncy + b, o01 = o00 + 1, o10 = o00 + ncy, o11 = o10 + 1;
  const double x1 = cx[a], x2 = cx[a + 1], y1 = cy[b], y2 = cy[b + 1];
  const double P100 = c.p1[o00], P101 = c.p1[o01], P110 = c.p1[o10], P111 = c.p1[o11];
  const double P200 = c.p2[o00], P201 = c.p2[o01], P210 = c.p2[o10], P211 = c.p2[o11];
  // log_factors(rk, t11, t22, t21, t12): even=(rk00+t11)*(rk11+t22), odd=(rk10+t21)*(rk01+t12)
  double e1 = (P100 + x1) * (P111 + x2), o1 = (P110 + x2) * (P101 + x1);
  double e2 = (P200 + x1) * (P211 + x2), o2 = (P210 + x2) * (P201 + x1);
  const double f1 = (e2 * o1) / (e1 * o2);
  e1 = (P100 + y1) * (P111 + y2); o1 = (P110 + y1) * (P101 + y2);
  e2 = (P200 + y1) * (P211 + y2); o2 = (P210 + y1) * (P201 + y2);
  const double f2 = (e2 * o1) / (e1 * o2);
  e1 = (P100 + z1) * (P111 + z1); o1 = (P110 + z1) * (P101 + z1);
  e2 = (P200 + z2) * (P211 + z2); o2 = (P210 + z2) * (P201 + z2);
  const double f3 = (e2 * o1) / (e1 * o2);
  const double ax2 = c.axz2[o11] - c.axz2[o01] - c.axz2[o10] + c.axz2[o00];
  const double ax1 = c.axz1[o11] - c.axz1[o01] - c.axz1[o10] + c.axz1[o00];
  const double f4 = ax2 - ax1;
  const double ay2 = c.ayz2[o11] - c.ayz2[o01] - c.ayz2[o10] + c.ayz2[o00];
  const double ay1 = c.ayz1[o11] - c.ayz1[o01] - c.ayz1[o10] + c.ayz1[o00];
  const double f5 = ay2 - ay1;
  return gc[0] * log(f1) + gc[1] * log(f2) + gc[2] * log(f3) + gc[3] * f4 + gc[4] * f5;
}

__device__ __forceinline__ void flag_nonfinite(double g, int* flag) {
  if (!isfinite(g)) atomicOr(flag, 1);
}

// window index -> embedding position (transform.py:85-88 at FFT length L):
// E[t] = window[s-1-t] for t < s; E[t] = window[L-t+s-1] for t >= L-n+1; 0 in the gap.
__device__ __forceinline__ int emb_to_win(int t, int s, int n, int L) {
  if (t < s) return s - 1 - t;
  if (t >= L - n + 1) return L - t + s - 1;
  return -1;
}

// Embedding E[ty][tx] (tx contiguous, Ly rows of Lx) for one layer, in 32 x 32
// tiles: the corner tables are [a][b] with b (y) contiguous, so lanes run along
// y while the entries are evaluated (coalesced corner gathers: lanes along x
// would touch one cache line per lane and per corner load, 24 per magnetic
// entry), and the tile is written back through shared memory with lanes along
// x.  Entry values are unchanged (same function of the same inputs).
constexpr int kEmbTile = 32, kEmbRows = 8;
__global__ void __launch_bounds__(kEmbTile* kEmbRows)
    k_embed(EmbedArgs a, const double* __restrict__ cm, MagCorners mc, const double* __restrict__ cx,
            const double* __restrict__ cy, int ncy, double z1, double z2, GC5 gc, int* flag,
            double* __restrict__ out) {
  __shared__ double tile[kEmbTile][kEmbTile + 1];  // [x][y]
  const int y0 = blockIdx.x * kEmbTile, x0 = blockIdx.y * kEmbTile;
  const int ty = y0 + threadIdx.x;
  const int wb = ty < a.Ly ? emb_to_win(ty, a.sy, a.ny, a.Ly) : -1;
#pragma unroll
  for (int i = 0; i < kEmbTile / kEmbRows; ++i) {
    const int xl = threadIdx.y + kEmbRows * i, tx = x0 + xl;
    const int wa = tx < a.Lx ? emb_to_win(tx, a.sx, a.nx, a.Lx) : -1;
    double v = 0.0;
    if (wa >= 0 && wb >= 0) {
      if (a.kind == 0) {
        int p = wa - (a.sx + a.pxl - 1);
        int q = wb - (a.sy + a.pyl - 1);
        p = p < 0 ? -p : p;
        q = q < 0 ? -q : q;
        v = grav_entry(cm, ncy, p, q);
      } else {
        v = mag_entry(mc, cx, cy, ncy, wa, wb, z1, z2, gc.v);
      }
      flag_nonfinite(v, flag);
    }
    tile[xl][threadIdx.x] = v;
  }
  __syncthreads();
  const int tx = x0 + threadIdx.x;
#pragma unroll
  for (int i = 0; i < kEmbTile / kEmbRows; ++i) {
    const int yl = threadIdx.y + kEmbRows * i, y = y0 + yl;
    if (tx < a.Lx && y < a.Ly) out[(long long)y * a.Lx + tx] = tile[threadIdx.x][yl];
  }
}

// Window (mx x my, [a][b] with b contiguous; kernels.py:158-184) for one layer.
__global__ void k_window(EmbedArgs a, int mx, int my, const double* __restrict__ cm, MagCorners mc,
                         const double* __restrict__ cx, const double* __restrict__ cy, int ncy, double z1,
                         double z2, GC5 gc, int* flag, double* __restrict__ out) {
  const int wb = blockIdx.x * blockDim.x + threadIdx.x;
  const int wa = blockIdx.y;
  if (wb >= my) return;
  double v;
  if (a.kind == 0) {
    int p = wa - (a.sx + a.pxl - 1);
    int q = wb - (a.sy + a.pyl - 1);
    p = p < 0 ? -p : p;
    q = q < 0 ? -q : q;
    v = grav_entry(cm, ncy, p, q);
  } else {
    v = mag_entry(mc, cx, cy, ncy, wa, wb, z1, z2, gc.v);
  }
  flag_nonfinite(v, flag);
  out[(long long)wa * my + wb] = v;
}

// Entries over arbitrary corner vectors (the drop-in gravity_layer_response /
// magnetic_response): out is (ncx-1) x (ncy-1).
__global__ void k_entries_raw(int kind, const double* __restrict__ cm, MagCorners mc, const double* __restrict__ cx,
                              const double* __restrict__ cy, int ncx, int ncy, double z1, double z2, GC5 gc,
                              int* flag, double* __restrict__ out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  const int a = blockIdx.y;
  if (b >= ncy - 1 || a >= ncx - 1) return;
  const double v = kind == 0 ? grav_entry(cm, ncy, a, b) : mag_entry(mc, cx, cy, ncy, a, b, z1, z2, gc.v);
  flag_nonfinite(v, flag);
  out[(long long)a * (ncy - 1) + b] = v;
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
cudaError_t launch_corners(int kind, const double* cx, int ncx, const double* cy, int ncy, const double* xy,
                           const double* r2, double z1, double z2, double gs, double* cm, MagCorners mc,
                           cudaStream_t st) {
  dim3 blk(128), grd((ncy + 127) / 128, ncx);
  if (kind == 0)
    k_grav_corners<<<grd, blk, 0, st>>>(cx, ncx, cy, ncy, xy, r2, z1, z2, gs, cm);
  else
    k_mag_corners<<<grd, blk, 0, st>>>(cx, ncx, cy, ncy, r2, z1, z2, mc);
  return cudaGetLastError();
}

cudaError_t launch_embed(const EmbedArgs& a, const double* cm, MagCorners mc, const double* cx, const double* cy,
                         int ncy, double z1, double z2, GC5 gc, int* flag, double* out, cudaStream_t st) {
  dim3 blk(kEmbTile, kEmbRows), grd((a.Ly + kEmbTile - 1) / kEmbTile, (a.Lx + kEmbTile - 1) / kEmbTile);
  k_embed<<<grd, blk, 0, st>>>(a, cm, mc, cx, cy, ncy, z1, z2, gc, flag, out);
  return cudaGetLastError();
}

// circulant embedding of a caller-supplied window (mx x my, row-major) at
// (Lx, Ly): the persisted-stack path (transform.py:85-88 applied to a window
// recovered from a reference stack file)
__global__ void k_embed_window(EmbedArgs a, int my, const double* __restrict__ win, int* flag,
                               double* __restrict__ out) {
  const int tx = blockIdx.x * blockDim.x + threadIdx.x;
  const int ty = blockIdx.y;
  if (tx >= a.Lx) return;
  const int wa = emb_to_win(tx, a.sx, a.nx, a.Lx);
  const int wb = emb_to_win(ty, a.sy, a.ny, a.Ly);
  double v = 0.0;
  if (wa >= 0 && wb >= 0) {
    v = win[(long long)wa * my + wb];
    flag_nonfinite(v, flag);
  }
  out[(long long)ty * a.Lx + tx] = v;
}

cudaError_t launch_embed_window(const EmbedArgs& a, int my, const double* win, int* flag, double* out,
                                cudaStream_t st) {
  dim3 blk(128), grd((a.Lx + 127) / 128, a.Ly);
  k_embed_window<<<grd, blk, 0, st>>>(a, my, win, flag, out);
  return cudaGetLastError();
}

cudaError_t launch_window(const EmbedArgs& a, int mx, int my, const double* cm, MagCorners mc, const double* cx,
                          const double* cy, int ncy, double z1, double z2, GC5 gc, int* flag, double* out,
                          cudaStream_t st) {
  dim3 blk(128), grd((my + 127) / 128, mx);
  k_window<<<grd, blk, 0, st>>>(a, mx, my, cm, mc, cx, cy, ncy, z1, z2, gc, flag, out);
  return cudaGetLastError();
}

cudaError_t launch_entries_raw(int kind, const double* cm, MagCorners mc, const double* cx, const double* cy,
                               int ncx, int ncy, double z1, double z2, GC5 gc, int* flag, double* out,
                               cudaStream_t st) {
  dim3 blk(128), grd((ncy - 1 + 127) / 128, ncx - 1);
  k_entries_raw<<<grd, blk, 0, st>>>(kind, cm, mc, cx, cy, ncx, ncy, z1, z2, gc, flag, out);
  return cudaGetLastError();
}

}  // namespace bttb
