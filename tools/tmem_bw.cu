// TMEM load/store throughput probe (development tool): bytes per clock per SM
// of tcgen05.ld / tcgen05.st (32x32b.x16 and x32) with 4, 8 and 16 warps.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmem_bw tools/tmem_bw.cu
#include <cstdint>
#include <cstdio>

template <int X>
__device__ __forceinline__ void ldx(uint32_t ta, uint32_t (&q)[32]);
template <>
__device__ __forceinline__ void ldx<16>(uint32_t ta, uint32_t (&q)[32]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]), "=r"(q[7]),
                 "=r"(q[8]), "=r"(q[9]), "=r"(q[10]), "=r"(q[11]), "=r"(q[12]), "=r"(q[13]), "=r"(q[14]), "=r"(q[15])
               : "r"(ta)
               : "memory");
}
template <>
__device__ __forceinline__ void ldx<32>(uint32_t ta, uint32_t (&q)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,"
      "%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]), "=r"(q[7]), "=r"(q[8]),
        "=r"(q[9]), "=r"(q[10]), "=r"(q[11]), "=r"(q[12]), "=r"(q[13]), "=r"(q[14]), "=r"(q[15]), "=r"(q[16]),
        "=r"(q[17]), "=r"(q[18]), "=r"(q[19]), "=r"(q[20]), "=r"(q[21]), "=r"(q[22]), "=r"(q[23]), "=r"(q[24]),
        "=r"(q[25]), "=r"(q[26]), "=r"(q[27]), "=r"(q[28]), "=r"(q[29]), "=r"(q[30]), "=r"(q[31])
      : "r"(ta)
      : "memory");
}
__device__ __forceinline__ void st16(uint32_t ta, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(ta),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

template <int X, int MODE>
__global__ void k(double* out, int iters) {
  __shared__ uint32_t taddr_s;
  const int w = threadIdx.x / 32;
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = taddr_s;
  const int nwq = blockDim.x / 128;  // warps per lane quarter
  const uint32_t col0 = (uint32_t)((w / 4) * (512 / nwq));
  const uint32_t ta = tbase + ((uint32_t)(32 * (w & 3)) << 16) + col0;
  uint32_t q[32];
  for (int i = 0; i < 32; ++i) q[i] = threadIdx.x + i;
  double s = 0;
  for (int it = 0; it < iters; ++it) {
    const uint32_t c = (uint32_t)((it * X) % (512 / nwq - X + 1));
    if (MODE == 0) {
      ldx<X>(ta + c, q);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      s += q[0] + q[X - 1];
    } else {
      q[0] += it;
      st16(ta + c, q);
      if (X == 32) st16(ta + c + 16, q);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + q[3];
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

int main() {
  int nsm = 148, clk = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* d;
  cudaMalloc(&d, (size_t)nsm * 512 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  auto run = [&](auto kern, const char* name, int X) {
    for (int nw : {4, 8, 16}) {
      kern<<<nsm, nw * 32>>>(d, 10);
      cudaEventRecord(e0);
      kern<<<nsm, nw * 32>>>(d, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double bytes = (double)nsm * nw * 32 * X * 4 * iters;
      printf("%s x%d warps=%2d: %7.1f B/clk/SM  (%s)\n", name, X, nw, bytes / (ms * 1e-3) / nsm / (clk * 1e3),
             cudaGetErrorString(cudaGetLastError()));
    }
  };
  run(k<16, 0>, "LDTM", 16);
  run(k<32, 0>, "LDTM", 32);
  run(k<16, 1>, "STTM", 16);
  run(k<32, 1>, "STTM", 32);
  return 0;
}
