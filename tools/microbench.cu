// tools/microbench.cu — measured rates of the sm_100a primitives the fused NA
// kernels are built from (one CTA per SM, clock64 per CTA, all SMs busy):
//   ldtm   tcgen05.ld 32x32b.x32 + wait, W warps            -> bytes/clk/SM
//   sttm   tcgen05.st 32x32b.x32 + wait                      -> bytes/clk/SM
//   mufu   ex2.approx.f32, W warps, 8 independent chains     -> ex2/clk/SM
//   ffma2  packed fp32 FMA, W warps                          -> flop/clk/SM
//   mma    tcgen05.mma kind::f16 M128 N64 K16 back to back   -> clk/MMA (issue+exec)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench tools/microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "../paper_2403_04690_b200/csrc/tc_ptx.cuh"

using namespace na;

__global__ void k_ldtm(unsigned long long* out, int iters, int nwarps) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) ptx::tmem_alloc<256>(&slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tm = slot + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 32;
  uint32_t acc = 0;
  __syncthreads();
  const unsigned long long t0 = clock64();
  if (warp < nwarps) {
    for (int i = 0; i < iters; ++i) {
      uint32_t r[32];
      NA_TMEM_LD32(tm, r);
      ptx::tmem_ld_wait();
#pragma unroll
      for (int c = 0; c < 32; ++c) acc ^= r[c];
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 0x12345678u) out[gridDim.x] = acc;
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<256>(slot);
  }
}

__global__ void k_sttm(unsigned long long* out, int iters, int nwarps) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) ptx::tmem_alloc<256>(&slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tm = slot + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 32;
  uint32_t r[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) r[c] = threadIdx.x * c;
  __syncthreads();
  const unsigned long long t0 = clock64();
  if (warp < nwarps) {
    for (int i = 0; i < iters; ++i) {
      NA_TMEM_ST32(tm, r);
      ptx::tmem_st_wait();
      r[i & 31] += 1;
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<256>(slot);
  }
}

__global__ void k_mufu(unsigned long long* out, int iters, int nwarps, float* sink) {
  const int warp = threadIdx.x >> 5;
  float x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = -0.001f * (threadIdx.x + c);
  __syncthreads();
  const unsigned long long t0 = clock64();
  if (warp < nwarps) {
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int c = 0; c < 8; ++c) x[c] = ptx::ex2(x[c]) - 1.0f;
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += x[c];
  if (s == 12345.f) sink[0] = s;
}

__global__ void k_mufu16(unsigned long long* out, int iters, int nwarps, float* sink) {
  const int warp = threadIdx.x >> 5;
  uint32_t x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = 0xBC00BC00u ^ (threadIdx.x + c);  // ~ -1.0 halves
  __syncthreads();
  const unsigned long long t0 = clock64();
  if (warp < nwarps) {
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        uint32_t y;
        asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x[c]));
        x[c] = y ^ 0x80008000u;  // keep values negative, dependent chain
      }
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s ^= x[c];
  if (s == 12345u) sink[0] = (float)s;
}

__global__ void k_ffma2(unsigned long long* out, int iters, int nwarps, float* sink) {
  const int warp = threadIdx.x >> 5;
  float2 x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = make_float2(0.001f * c, 0.002f * threadIdx.x);
  const float2 a = make_float2(0.999f, 0.998f), b = make_float2(0.001f, 0.002f);
  __syncthreads();
  const unsigned long long t0 = clock64();
  if (warp < nwarps) {
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int c = 0; c < 8; ++c) x[c] = __ffma2_rn(x[c], a, b);
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += x[c].x + x[c].y;
  if (s == 12345.f) sink[0] = s;
}

// Back-to-back MMAs (M=128, N=64, K=16, SS, fp16) from one warp; smem operands
// are whatever smem holds (values irrelevant).  Measures issue + execution.
// mode 0: SS, B K-major; mode 1: SS, B MN-major; mode 2: TS (A in TMEM cols
// 128..), B MN-major; mode 3: TS, B K-major.
template <int MODE, int N>
__global__ void k_mma(unsigned long long* out, int iters) {
  constexpr int mode = MODE, n = N;
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) ptx::tmem_alloc<256>(&slot);
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_barrier_init();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t a = ptx::smem_u32(sm), b = a + 16384;
  constexpr bool bmn = mode == 1 || mode == 2;
  constexpr uint32_t idesc = ptx::make_idesc(128, n, false, bmn);
  unsigned long long t0 = 0, t1 = 0;
  if (warp == 0) {
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t bd = bmn ? ptx::make_sdesc(b + kk * 16 * 128, 128 * 128, 1024, 2)
                                : ptx::make_sdesc(b + kk * 32, 16, 1024, 2);
        if constexpr (mode >= 2)
          ptx::mma_ts_w(slot, slot + 128 + kk * 8, bd, idesc, 1u);
        else
          ptx::mma_ss_w(slot, ptx::make_sdesc(a + kk * 32, 16, 1024, 2), bd, idesc, 1u);
      }
    }
    ptx::mma_commit_w(&bar);
    ptx::mbar_wait(&bar, 0);
    t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<256>(slot);
  }
}

static double avg(unsigned long long* h, int n) {
  double s = 0;
  for (int i = 0; i < n; ++i) s += (double)h[i];
  return s / n;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long *d, h[1024];
  float* sink;
  cudaMalloc(&d, sizeof(h));
  cudaMalloc(&sink, 64);
  const int iters = 2000;
  for (int nw : {4, 8}) {
    k_ldtm<<<sms, 32 * 8>>>(d, iters, nw);
    cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
    const double cyc = avg(h, sms);
    printf("ldtm  warps=%d: %.1f clk/iter  -> %.1f B/clk/SM (32x32b.x32 = 4 KB/warp)\n", nw, cyc / iters,
           nw * 4096.0 * iters / cyc);
    k_sttm<<<sms, 32 * 8>>>(d, iters, nw);
    cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
    const double cs = avg(h, sms);
    printf("sttm  warps=%d: %.1f clk/iter  -> %.1f B/clk/SM\n", nw, cs / iters, nw * 4096.0 * iters / cs);
  }
  for (int nw : {1, 2, 4, 8, 16}) {
    k_mufu<<<sms, 32 * 16>>>(d, iters, nw, sink);
    cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
    const double cyc = avg(h, sms);
    printf("mufu  warps=%2d: %.2f ex2/clk/SM\n", nw, nw * 32.0 * 8 * iters / cyc);
    k_mufu16<<<sms, 32 * 16>>>(d, iters, nw, sink);
    cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
    const double ch = avg(h, sms);
    printf("mufu16x2 warps=%2d: %.2f ex2 results/clk/SM (f16x2: 2 per op)\n", nw, nw * 32.0 * 16 * iters / ch);
    k_ffma2<<<sms, 32 * 16>>>(d, iters, nw, sink);
    cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
    const double cf = avg(h, sms);
    printf("ffma2 warps=%2d: %.1f fp32 FMA/clk/SM\n", nw, nw * 32.0 * 16 * iters / cf);
  }
  auto run = [&](auto kern, const char* name, int n) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    kern<<<sms, 128, 65536>>>(d, 200);
    cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
    const double cyc = avg(h, sms);
    printf("mma %s M128 N%-3d K16: %.1f clk/MMA  -> %.0f flop/clk/SM\n", name, n, cyc / (200 * 4),
           2.0 * 128 * n * 16 * 200 * 4 / cyc);
  };
  run(k_mma<0, 64>, "SS Bk ", 64);
  run(k_mma<0, 128>, "SS Bk ", 128);
  run(k_mma<0, 256>, "SS Bk ", 256);
  run(k_mma<1, 64>, "SS Bmn", 64);
  run(k_mma<1, 128>, "SS Bmn", 128);
  run(k_mma<2, 64>, "TS Bmn", 64);
  run(k_mma<2, 128>, "TS Bmn", 128);
  run(k_mma<3, 64>, "TS Bk ", 64);
  run(k_mma<3, 128>, "TS Bk ", 128);
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
