// Semantics check of mbarrier.arrive_drop (sm_100a).
#include <cstdio>
#include <cstdint>
__device__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ int done(uint64_t *b, uint32_t par) {
  uint32_t d;
  asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
               : "=r"(d) : "r"(sa(b)), "r"(par) : "memory");
  return (int)d;
}
__device__ void init(uint64_t *b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(n));
  asm volatile("fence.mbarrier_init.release.cluster;");
}
__device__ void arr(uint64_t *b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory"); }
__device__ void drp(uint64_t *b) { asm volatile("mbarrier.arrive_drop.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory"); }
// script: string of 'a' (arrive) / 'd' (drop) / '|' (record phase-0 completion, then phase-1) issued by thread 0
__global__ void k(int *out) {
  __shared__ uint64_t bar;
  const char *scripts[6] = {"dd", "ad", "dda", "ddddddaa", "ddddddaa|aa", "ddd|a"};
  const int counts[6] = {2, 2, 3, 8, 8, 4};
  for (int t = 0; t < 6; t++) {
    if (threadIdx.x == 0) {
      init(&bar, counts[t]);
      int r = 0;
      for (const char *c = scripts[t]; *c; c++) {
        if (*c == 'a') arr(&bar);
        else if (*c == 'd') drp(&bar);
        else { out[t * 2] = done(&bar, 0); r = 1; }
      }
      out[t * 2 + r] = done(&bar, r);
      if (!r) out[t * 2 + 1] = -1;
    }
    __syncthreads();
  }
}
int main() {
  int *d, h[12];
  cudaMalloc(&d, sizeof(h));
  k<<<1, 32>>>(d);
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const char *names[6] = {"E2 dd", "E2 ad", "E3 dda", "E8 d*6 a*2", "E8 d*6 a*2 | a*2 (phase1)", "E4 ddd | a (phase1)"};
  for (int t = 0; t < 6; t++) printf("%-28s phase0 done %d  second %d\n", names[t], h[2 * t], h[2 * t + 1]);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
