// Internal interface of the kernel-entry generators (entries.cu).
#pragma once
#include <cuda_runtime.h>

namespace bttb {

struct MagCorners {  // per-corner magnetic terms, each ncx*ncy doubles
  double* p1;
  double* p2;
  double* axz1;
  double* axz2;
  double* ayz1;
  double* ayz2;
};

struct GC5 {
  double v[5];
};

struct EmbedArgs {
  int kind;  // 0 gravity, 1 magnetic
  int sx, sy, nx, ny, pxl, pyl;
  int Lx, Ly;
};

cudaError_t launch_corners(int kind, const double* cx, int ncx, const double* cy, int ncy, const double* xy,
                           const double* r2, double z1, double z2, double gs, double* cm, MagCorners mc,
                           cudaStream_t st);
cudaError_t launch_embed(const EmbedArgs& a, const double* cm, MagCorners mc, const double* cx, const double* cy,
                         int ncy, double z1, double z2, GC5 gc, int* flag, double* out, cudaStream_t st);
cudaError_t launch_embed_window(const EmbedArgs& a, int my, const double* win, int* flag, double* out,
                                cudaStream_t st);
cudaError_t launch_window(const EmbedArgs& a, int mx, int my, const double* cm, MagCorners mc, const double* cx,
                          const double* cy, int ncy, double z1, double z2, GC5 gc, int* flag, double* out,
                          cudaStream_t st);
cudaError_t launch_entries_raw(int kind, const double* cm, MagCorners mc, const double* cx, const double* cy,
                               int ncx, int ncy, double z1, double z2, GC5 gc, int* flag, double* out,
                               cudaStream_t st);

}  // namespace bttb
