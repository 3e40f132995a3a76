// Microbenchmark of the team FFT engine (development tool, not product code).
// Batched column FFTs of length L from global to global, fp64 or fp32; reports
// ns per transform, points/s and max error against a direct O(L^2) DFT on a few
// columns.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//   --expt-relaxed-constexpr -I paper_1912_06976_b200/csrc tools/fftbench.cu
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "fft.cuh"

using namespace bttb;

template <class Plan, int MAXT = 1024, int MINB = 1>
__global__ void __launch_bounds__(MAXT, MINB) k_bench(const cplx<typename Plan::Scalar>* __restrict__ in, cplx<typename Plan::Scalar>* __restrict__ out,
                        int ncols, FFTDesc<typename Plan::Scalar> d, int C, int reps) {
  using T = typename Plan::Scalar;
  using V = cplx<T>;
  constexpr int E = Plan::E;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int nt = Plan::nt(d), Ls = team_slots<T>(d.L);
  const int tid = threadIdx.x, c = tid / nt, t = tid - c * nt;
  const int col = blockIdx.x * C + c;
  const int cc = col < ncols ? col : 0;
  V* sm = reinterpret_cast<V*>(smraw) + (long long)c * Ls;
  V v[E];
  const V* src = in + (long long)cc * d.L;
#pragma unroll
  for (int k = 0; k < E; ++k) v[k] = src[t + nt * k];
  for (int r = 0; r < reps; ++r) Plan::fft(v, sm, t, d);
  if (col < ncols) {
    V* dst = out + (long long)col * d.L;
#pragma unroll
    for (int k = 0; k < E; ++k) dst[t + nt * k] = v[k];
  }
}

template <class Plan, int MAXT = 1024, int MINB = 1>
void run(int L, const int* radices, int npass, int ncols, int C, int reps) {
  using T = typename Plan::Scalar;
  constexpr int E = Plan::E;
  using V = cplx<T>;
  std::vector<V> h((size_t)ncols * L);
  srand(1);
  for (auto& x : h) { x.x = (T)(rand() / (double)RAND_MAX - 0.5); x.y = (T)(rand() / (double)RAND_MAX - 0.5); }
  V *din, *dout, *tw;
  cudaMalloc(&din, sizeof(V) * h.size());
  cudaMalloc(&dout, sizeof(V) * h.size());
  cudaMalloc(&tw, sizeof(V) * L);
  std::vector<V> htw(L);
  for (int m = 0; m < L; ++m) {
    long double a = 2.0L * 3.141592653589793238462643383279502884L * m / L;
    htw[m].x = (T)cosl(a);
    htw[m].y = (T)-sinl(a);
  }
  cudaMemcpy(tw, htw.data(), sizeof(V) * L, cudaMemcpyHostToDevice);
  cudaMemcpy(din, h.data(), sizeof(V) * h.size(), cudaMemcpyHostToDevice);
  // per-pass twiddle tables (as capi.cu per_pass_table builds them)
  std::vector<V> hp;
  {
    long ns = 1;
    const int np = npass < 0 ? -npass : npass;
    for (int p = 0; p < np; ++p) {
      const int R = radices[p];
      if (ns > 1)
        for (int r = 1; r < R; ++r)
          for (long k = 0; k < ns; ++k) {
            long double a = 2.0L * 3.141592653589793238462643383279502884L * (long double)(r * k) / (ns * R);
            V c;
            c.x = (T)cosl(a);
            c.y = (T)-sinl(a);
            hp.push_back(c);
          }
      ns *= R;
    }
  }
  V* twp;
  cudaMalloc(&twp, sizeof(V) * (hp.size() + 1));
  cudaMemcpy(twp, hp.data(), sizeof(V) * hp.size(), cudaMemcpyHostToDevice);
  FFTDesc<T> d;
  d.tw = tw;
  d.twp = twp;
  d.L = L;
  d.nt = L / E;
  d.npass = npass < 0 ? -npass : npass;
  d.code = 0;
  for (int i = 0; i < (npass < 0 ? -npass : npass); ++i) d.code |= radix_code(radices[i]) << (4 * i);
  const size_t smem = (size_t)C * team_slots<T>(L) * sizeof(V);
  cudaFuncSetAttribute(k_bench<Plan, MAXT, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_bench<Plan, MAXT, MINB>, C * d.nt, smem);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, k_bench<Plan, MAXT, MINB>);
  dim3 grd((ncols + C - 1) / C), blk(C * d.nt);
  k_bench<Plan, MAXT, MINB><<<grd, blk, smem>>>(din, dout, ncols, d, C, 1);
  cudaDeviceSynchronize();
  // accuracy (reps=1)
  std::vector<V> o(h.size());
  cudaMemcpy(o.data(), dout, sizeof(V) * h.size(), cudaMemcpyDeviceToHost);
  double maxerr = 0, maxref = 0;
  for (int col = 0; col < 3; ++col)
    for (int k = 0; k < L; k += 7) {
      long double re = 0, im = 0;
      for (int n = 0; n < L; ++n) {
        long double a = -2.0L * 3.141592653589793238462643383279502884L * (long double)((long long)n * k % L) / L;
        re += h[(size_t)col * L + n].x * cosl(a) - h[(size_t)col * L + n].y * sinl(a);
        im += h[(size_t)col * L + n].x * sinl(a) + h[(size_t)col * L + n].y * cosl(a);
      }
      V g = o[(size_t)col * L + k];
      maxerr = fmax(maxerr, (double)hypotl(g.x - re, g.y - im));
      maxref = fmax(maxref, (double)hypotl(re, im));
    }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_bench<Plan, MAXT, MINB><<<grd, blk, smem>>>(din, dout, ncols, d, C, reps);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double nfft = (double)ncols * reps;
  printf("MINB=%d %s %s L=%d E=%d C=%d regs=%d blocks/SM=%d: %.2f ns/FFT (%.3f ns/pt/SM... %.2f Gpt/s)  relerr %.2e  %s\n",
         MINB, sizeof(T) == 8 ? "f64" : "f32", npass < 0 ? "static" : "dyn   ", L, E, C, fa.numRegs, nb, ms * 1e6 / nfft, ms * 1e6 / nfft / L * 148,
         nfft * L / ms / 1e6, maxerr / maxref, cudaGetErrorString(cudaGetLastError()));
  cudaFree(din);
  cudaFree(dout);
  cudaFree(tw);
  cudaFree(twp);
}

int main(int argc, char** argv) {
  // E=32 / E=64 fp32 plans (fewer passes) measured no faster than E=16:
  // 586-634 / 581-645 vs 661 Gpt/s at L=2048 (round 1)
  const int reps = argc > 1 ? atoi(argv[1]) : 20;
  const int r20[] = {20, 20, 5};
  const int r16[] = {16, 16, 8};
  run<SPlan<double, 20, 20, 20, 20, 5>, 100, 4>(2000, r20, -3, 1001 * 32, 1, reps);
  run<SPlan<double, 16, 16, 16, 16, 8>, 128, 4>(2048, r16, -3, 1025 * 32, 1, reps);
  run<SPlan<float, 20, 80, 20, 20, 5>, 100, 4>(2000, r20, -3, 1001 * 32, 1, reps);
  run<SPlan<float, 16, 16, 16, 16, 8>, 128, 4>(2048, r16, -3, 1025 * 32, 1, reps);
  // half-length transforms (a zero-padded 2048 = two 1024s): one warp, one
  // exchange; measured round 1: fp32 832-892 Gpt/s vs 690 for 2048/E=16, fp64
  // 419-441 vs 357 (1.2-1.3x per point before the split's twiddle pass)
  const int r1024[] = {32, 32};
  run<SPlan<float, 32, 16, 32, 32>, 32, 16>(1024, r1024, -2, 2050 * 32, 1, reps);
  run<SPlan<float, 32, 32, 32, 32>, 32, 16>(1024, r1024, -2, 2050 * 32, 1, reps);
  run<SPlan<float, 32, 16, 32, 32>, 32, 24>(1024, r1024, -2, 2050 * 32, 1, reps);
  run<SPlan<double, 32, 16, 32, 32>, 32, 8>(1024, r1024, -2, 2050 * 32, 1, reps);
  run<SPlan<double, 32, 8, 32, 32>, 32, 8>(1024, r1024, -2, 2050 * 32, 1, reps);
  run<SPlan<double, 32, 16, 32, 32>, 32, 12>(1024, r1024, -2, 2050 * 32, 1, reps);
  return 0;
}
