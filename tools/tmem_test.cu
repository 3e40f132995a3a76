#include <cstdint>
#include <cstdio>
__global__ void k(double* out) {
  __shared__ uint32_t taddr_s;
  const int w = threadIdx.x / 32;
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" :: "r"((uint32_t)__cvta_generic_to_shared(&taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = taddr_s;
  const uint32_t ta = tbase + ((uint32_t)(32 * (w & 3)) << 16);
  uint32_t r[16];
  for (int i = 0; i < 16; ++i) r[i] = threadIdx.x * 100 + i;
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
               :: "r"(ta), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
                  "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]) : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  uint32_t q[16];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]), "=r"(q[7]),
                 "=r"(q[8]), "=r"(q[9]), "=r"(q[10]), "=r"(q[11]), "=r"(q[12]), "=r"(q[13]), "=r"(q[14]), "=r"(q[15])
               : "r"(ta) : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  double s = 0;
  for (int i = 0; i < 16; ++i) s += q[i];
  out[threadIdx.x] = s;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" :: "r"(tbase));
}
int main() {
  double* d; cudaMalloc(&d, 100 * 8);
  k<<<3, 100>>>(d);
  double h[100]; cudaMemcpy(h, d, 800, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int t = 0; t < 100; ++t) { double e = 0; for (int i = 0; i < 16; ++i) e += t * 100 + i; if (h[t] != e) ++bad; }
  printf("tmem test: %s, bad=%d (%s)\n", bad ? "FAIL" : "ok", bad, cudaGetErrorString(cudaGetLastError()));
}
