/*
 * bttb_sm100.h -- C ABI of the B200-native (sm_100a) fast BTTB forward operator.
 *
 * Drop-in boundary for the hot path of the reference package `bttb`
 * (arXiv 1912.06976; /root/reference/pkg/src/bttb).  The reference has no FFI
 * of its own: its boundary is a pure-Python function API.  Each entry point
 * below replaces one reference function; the Python mirror in
 * paper_1912_06976_b200/ binds them with ctypes.
 *
 * Conventions
 *  - Every call returns BTTB_OK (0) or a negative status; the message of the
 *    last failure on the calling thread is in bttb_last_error().
 *  - Vectors are C-contiguous float64 (plan dtype F64) or float32 (F32) in the
 *    reference ordering (multiply.py:25-26): model = layer-major, x-fastest
 *    (prism (p,q) of layer r at r*n_r + q*nx + p); data = x-fastest (j*sx + i).
 *  - The plan owns all device memory it allocates; callers own x and y.
 *  - Plans are safe to share across threads: bttb_apply serialises on a
 *    per-plan mutex (the reference's apply is reentrant, README.md:120-122).
 */
#ifndef BTTB_SM100_H
#define BTTB_SM100_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { BTTB_OK = 0, BTTB_EINVAL = -1, BTTB_ECUDA = -2, BTTB_ENONFINITE = -3, BTTB_ENOMEM = -4 };
enum { BTTB_GRAVITY = 0, BTTB_MAGNETIC = 1 };
enum { BTTB_F64 = 0, BTTB_F32 = 1 };
enum { BTTB_FORWARD = 0, BTTB_TRANSPOSE = 1 };
enum { BTTB_DEVICE_PTR = 0, BTTB_HOST_PTR = 1, BTTB_HOST_ASYNC = 2, BTTB_HOST_ASYNC_UNORDERED = 3 };
enum { BTTB_STAGE_ALL = 0, BTTB_STAGE_TO_SPECTRUM = 1, BTTB_STAGE_FROM_SPECTRUM = 2 };

/* Geometry; mirrors GridSpec (grid.py:26-104).  z_blocks has nz+1 entries. */
typedef struct {
  int64_t sx, sy, nz, pxl, pxr, pyl, pyr;
  double dx, dy;
  const double* z_blocks;
} bttb_grid;

/* Kernel constants; mirrors KernelParams (kernels.py:19-45):
 * gravity -> gamma_scaled = gamma*scale (kernels.py:98);
 * magnetic -> gc = magnetic_constants(D, I, F) (kernels.py:48-64). */
typedef struct {
  int kind;
  double gamma_scaled;
  double gc[5];
} bttb_kernel;

typedef struct bttb_plan_s bttb_plan;

/* Replaces build_transform_stack (transform.py:91-104): generates every
 * layer's kernel entries on the GPU (kernels.py:158-184), embeds them
 * (transform.py:85-88) at FFT lengths Lx >= sx+nx-1, Ly >= sy+ny-1 (0 = pick
 * automatically) and caches one half spectrum per layer in HBM.  The plan
 * holds layers [layer_begin, layer_end) of the grid (layer sharding across
 * GPUs; pass 0, nz for all).  Returns BTTB_ENONFINITE with the reference's
 * FloatingPointError text (kernels.py:74-78) if an entry is not finite. */
int bttb_plan_create(bttb_plan** out, const bttb_grid* grid, const bttb_kernel* kernel, int dtype, int device,
                     int64_t layer_begin, int64_t layer_end, int64_t Lx, int64_t Ly);

/* Replaces load_stack (transform.py:135-159): a plan whose spectrum cache is
 * uploaded from host memory (local layers x Hx x Ly complex of the plan dtype,
 * as bttb_layer_spectrum returns them) instead of being rebuilt.  Lx, Ly must
 * be the lengths the spectra were built at. */
int bttb_plan_create_from_spectra(bttb_plan** out, const bttb_grid* grid, const bttb_kernel* kernel, int dtype,
                                  int device, int64_t layer_begin, int64_t layer_end, int64_t Lx, int64_t Ly,
                                  const void* host_spectra);

/* Replaces load_stack of a REFERENCE-format file (transform.py:130-159): a
 * plan whose spectra are built on the GPU (embedding at (Lx, Ly), FFTs) from
 * caller-supplied response windows -- local layers x mx x my float64,
 * row-major, in the layer_response_window layout (kernels.py:158-184) -- as
 * recovered from the file's fft2(T^circ) arrays.  Lx, Ly = 0 picks them.
 * Returns BTTB_ENONFINITE if a window holds a non-finite value. */
int bttb_plan_create_from_windows(bttb_plan** out, const bttb_grid* grid, const bttb_kernel* kernel, int dtype,
                                  int device, int64_t layer_begin, int64_t layer_end, int64_t Lx, int64_t Ly,
                                  const double* host_windows);

int bttb_plan_destroy(bttb_plan* plan);

/* Replaces apply(stack, x, mode) (multiply.py:22-58) for `batch` vectors.
 * FORWARD: x = batch x (n_r * local layers), y = batch x m (the partial
 *          sum over the plan's layers; overwritten).
 * TRANSPOSE: x = batch x m, y = batch x (n_r * local layers).
 * where = BTTB_DEVICE_PTR (x, y in device memory of the plan's GPU; runs
 * asynchronously on `stream`, a cudaStream_t or NULL), BTTB_HOST_PTR
 * (host memory; copies in and out, synchronous), BTTB_HOST_ASYNC (host
 * memory, pinned for overlap; returns at once: the input copy is ordered
 * after the work queued on `stream` at call time, x must stay unchanged and y
 * be left unread until the caller synchronises `stream`, which is ordered
 * after y's copy) or BTTB_HOST_ASYNC_UNORDERED (the same, except that the
 * input copy is NOT ordered after `stream`: x must hold its final values at
 * call time.  Dropping that edge is what lets consecutive calls pipeline --
 * one call's device-to-host copy overlaps the next call's host-to-device copy
 * through plan-owned staging slots; with the ordered mode `stream` already
 * waits for the previous call's output copy, so the next input copy queues
 * behind it). */
int bttb_apply(bttb_plan* plan, int mode, const void* x, void* y, int64_t batch, int where, void* stream);

/* Split product for layer-sharded multi-GPU plans (BASELINE north_star: the
 * per-GPU partial spectra are summed by an NCCL reduce before ONE inverse
 * transform; the transpose broadcasts the data spectrum).  The split point is
 * the station half spectrum W: batch x Hx x sy complex (plan dtype), x
 * frequency by station row, = sum over layers of S_r * FFT(model_r) already
 * inverse-transformed along y.  Device pointers, asynchronous on `stream`.
 *   FORWARD   TO_SPECTRUM:   x = model (local layers) -> y = partial W
 *   FORWARD   FROM_SPECTRUM: x = W (summed over shards) -> y = data
 *   TRANSPOSE TO_SPECTRUM:   x = data -> y = W (the data's half spectrum)
 *   TRANSPOSE FROM_SPECTRUM: x = W -> y = model (local layers)
 * STAGE_ALL is bttb_apply's device path.  Replaces the layer loop of apply
 * (multiply.py:37-57) split at its cross-layer sum. */
int bttb_apply_staged(bttb_plan* plan, int mode, int stage, const void* x, void* y, int64_t batch, void* stream);

/* Device-resident batched CGLS -- the inversion loop the paper names as future
 * work (no reference function: the reference stops at apply,
 * multiply.py:22-58, and lists inversion as a non-goal).
 * Minimises |G m - d|^2 + damp^2 |m|^2 from m = 0 for `batch` independent
 * data vectors with `iters` CGLS iterations (one forward and one transpose
 * product each, fused vector updates, fp64 reductions, no host round trip
 * inside the loop).  d = batch x m, m_out = batch x n (the plan must hold every
 * layer).  where / stream as in bttb_apply.  resid_norms (optional host
 * array, batch x (iters+1)) receives |d - G m_k| for k = 0..iters; the call
 * then synchronises. */
int bttb_cgls(bttb_plan* plan, const void* d, void* m_out, int64_t batch, int iters, double damp, int where,
              void* stream, double* resid_norms);

/* Entry-generator parity hook: the layer's response window, shape
 * (sx+nx-1) x (sy+ny-1), row-major, as layer_response_window returns it
 * (kernels.py:158-184).  `layer` is a global layer index. */
int bttb_layer_window(bttb_plan* plan, int64_t layer, double* host_out);

/* Copy the cached half spectrum of a local layer (Hx x Ly complex, as stored:
 * scaled by 1/(Lx*Ly), dtype of the plan) to host memory. */
int bttb_layer_spectrum(bttb_plan* plan, int64_t local_layer, void* host_out);

/* Plan facts: info[0..9] = Lx, Ly, Hx, layer_begin, layer_end, dtype, kind,
 * layers per chunk, batch per group, kernels launched by the last apply. */
int bttb_plan_info(const bttb_plan* plan, int64_t* info);

/* Replace gravity_layer_response (kernels.py:81-102) and magnetic_response
 * (kernels.py:105-155) over arbitrary corner vectors x (ncx) and y (ncy):
 * out is (ncx-1) x (ncy-1), row-major, host memory.  xy / r2 are the
 * DistanceTables arrays (ncx x ncy) or NULL to form them as x*y, x*x+y*y. */
int bttb_gravity_response(const double* x, int64_t ncx, const double* y, int64_t ncy, const double* xy,
                          const double* r2, double z1, double z2, double gamma_scaled, double* out, int device);
int bttb_magnetic_response(const double* x, int64_t ncx, const double* y, int64_t ncy, const double* r2,
                           double z1, double z2, const double* gc, double* out, int device);

/* FFT length the plan picks for an embedding of n: the smallest length of
 * the shared-memory engine's family >= n up to 8192 (2^a, a>=3; 2^a*3^b or
 * 2^a*5^b with a>=2, b>=1), except that a power of two within 5% of it is
 * preferred when the library has a compile-time FFT plan for it (e.g.
 * 1999 -> 2048); above 8192 the smallest 2^a 3^b 5^c >= n (at most 65536),
 * which plans run on the generic-length path (global-memory radix passes;
 * no split products).  -1 if n > 65536. */
int64_t bttb_fft_length(int64_t n);

/* Development check (no reference counterpart): with BTTB_GUARD=1 in the
 * environment every plan buffer and the spectrum cache carry 64 KB guard
 * zones of a fixed pattern on both sides; this synchronises the device and
 * returns how many buffers had a guard byte overwritten (0 = clean; always 0
 * when guards are off), or a negative error code. */
int bttb_debug_check_guards(bttb_plan* plan);

/* Last error message on the calling thread ("" if none). */
const char* bttb_last_error(void);

/* Library version string. */
const char* bttb_version(void);

#ifdef __cplusplus
}
#endif

#endif /* BTTB_SM100_H */
