#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ bool test(uint64_t* b, uint32_t ph) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
  return ok != 0;
}
__global__ void k(long long* out, int mode) {
  __shared__ uint64_t bar[2];
  if (threadIdx.x == 0) { init(&bar[0], mode == 1 ? 4 : 128); init(&bar[1], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < 1000; ++i) {
    if (mode == 0) { arrive(&bar[0]); wait(&bar[0], i & 1); }
    else if (mode == 1) { __syncwarp(); if ((threadIdx.x & 31) == 0) arrive(&bar[0]); wait(&bar[0], i & 1); }
    else if (mode == 2) { wait(&bar[1], 1); }  // phase 1 parity: "previous phase" complete -> immediate
    else if (mode == 3) { arrive(&bar[0]); }
    else if (mode == 4) { while (!test(&bar[1], 1)) {} }  // test_wait on a completed phase
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[mode] = (t1 - t0) / 1000;
}
int main() {
  long long* d; cudaMalloc(&d, 64); long long h[5];
  for (int m = 0; m < 5; ++m) k<<<1, 128>>>(d, m);
  cudaMemcpy(h, d, 40, cudaMemcpyDeviceToHost);
  printf("arrive(128)+wait: %lld clk/iter\narrive(lane0,4)+wait: %lld\nwait on completed phase: %lld\narrive only: %lld\n", h[0], h[1], h[2], h[3]);
  printf("test_wait on completed phase: %lld\n", h[4]);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
