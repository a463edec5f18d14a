// Resolution of %globaltimer on this GPU: one thread reads it back to back and records the
// distinct non-zero steps it sees (and how many SM cycles a read takes).
// nvcc -arch=sm_100a -o globaltimer_res globaltimer_res.cu && ./globaltimer_res
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(unsigned long long* steps, unsigned long long* cyc, int n) {
  unsigned long long prev, now;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(prev));
  long long c0 = clock64();
  int k = 0;
  for (int i = 0; i < 2000000 && k < n; ++i) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if (now != prev) { steps[k++] = now - prev; prev = now; }
  }
  cyc[0] = clock64() - c0;
  cyc[1] = k;
}
int main() {
  const int n = 64;
  unsigned long long *d, *c, h[n], hc[2];
  cudaMalloc(&d, n * 8); cudaMalloc(&c, 16);
  cudaMemset(d, 0, n * 8);
  probe<<<1, 1>>>(d, c, n);
  cudaMemcpy(h, d, n * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(hc, c, 16, cudaMemcpyDeviceToHost);
  printf("globaltimer steps (ns):");
  for (int i = 0; i < 24; ++i) printf(" %llu", h[i]);
  printf("\nsteps seen %llu in %llu cycles\n", hc[1], hc[0]);
  return 0;
}
