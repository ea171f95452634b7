// Softmax-round microbenchmark: the forward kernel's per-round register/TMEM
// work (4 x tcgen05.ld of 32 logits, partial-group mask, row max, lazy
// rescale test, exponentials (MUFU + FMA-pipe polynomial), in-place 16-bit
// pack, 2 x tcgen05.st) in a loop, without MMAs or barriers.  2 CTAs x 128
// threads per SM, like the forward's softmax warpgroups.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2403_04690_b200/csrc \
//        tools/softmax_bench.cu -o tools/softmax_bench
#include <cstdio>
#include <cuda_fp16.h>
#include "tc_ptx.cuh"
#include "tc_common.cuh"

using namespace na;

template <int MASKED, int MODE, int NG = 4>
__global__ void __launch_bounds__(128, 1) rounds(unsigned long long* out, int iters, uint32_t wbits) {
  // MODE 0 full round; 1 loads + stores only; 2 + mask/max; 3 + exponentials without the max
  __shared__ uint32_t slot;
  const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
  if (warp == 0) ptx::tmem_alloc<(NG == 4 ? 256 : 128)>(&slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t trow = tmem + ((warp * 32u) << 16);
  float m_ref = -INFINITY, l = 0.f;
  const float sl2 = 0.18f;
  uint32_t mw[4] = {0xffffffffu, 0xffffffffu, MASKED ? (wbits << (lane & 7)) : 0xffffffffu, 0x0000ffffu};
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    bool live[4];
#pragma unroll
    for (int gq = 0; gq < NG; ++gq) live[gq] = __any_sync(0xffffffffu, mw[gq] != 0u);
    uint32_t sv[128];
#pragma unroll
    for (int gq = 0; gq < NG; ++gq)
      if (live[gq]) NA_TMEM_LD32(trow + 32 * gq, (sv + 32 * gq));
    ptx::tmem_ld_wait();
#ifndef MAXCH
#define MAXCH 4
#endif
    float m4[MAXCH];
#pragma unroll
    for (int i = 0; i < MAXCH; ++i) m4[i] = -INFINITY;
#pragma unroll
    for (int gq = 0; gq < NG; ++gq) {
      if (!live[gq] || MODE == 1 || MODE == 3) continue;
      const uint32_t w = mw[gq];
      if (!__all_sync(0xffffffffu, w == 0xffffffffu)) {
#pragma unroll
        for (int c = 0; c < 32; ++c) sv[32 * gq + c] = (w >> c) & 1u ? sv[32 * gq + c] : __float_as_uint(-INFINITY);
      }
#pragma unroll
      for (int c = 0; c < 32; c += 2 * MAXCH)
#pragma unroll
        for (int i = 0; i < MAXCH; ++i)
          m4[i] = fmaxf(m4[i], fmaxf(__uint_as_float(sv[32 * gq + c + i]), __uint_as_float(sv[32 * gq + c + MAXCH + i])));
    }
    float mx = m4[0];
#pragma unroll
    for (int i = 1; i < MAXCH; ++i) mx = fmaxf(mx, m4[i]);
    const float mx2 = mx * sl2;
    const bool need = mx2 > m_ref + 8.f;
    if (need) m_ref = mx2;
    const float nmu = m_ref == -INFINITY ? 0.f : -m_ref;
    float2 acc0 = make_float2(0.f, 0.f), acc1 = make_float2(0.f, 0.f);
#pragma unroll
    for (int gq = 0; gq < NG; ++gq) {
      if (MODE == 1 || MODE == 2) {
#pragma unroll
        for (int c = 0; c < 16; ++c) sv[16 * gq + c] ^= sv[32 * gq + c + 16] + __float_as_uint(nmu);
        continue;
      }
      if (!live[gq]) {
#pragma unroll
        for (int c = 0; c < 16; ++c) sv[16 * gq + c] = 0u;
        continue;
      }
#pragma unroll
      for (int c = 0; c < 32; c += 4) {
        const uint32_t* s4 = sv + 32 * gq + c;
        const float2 x0 = __ffma2_rn(make_float2(__uint_as_float(s4[0]), __uint_as_float(s4[1])),
                                     make_float2(sl2, sl2), make_float2(nmu, nmu));
        const float2 x1 = __ffma2_rn(make_float2(__uint_as_float(s4[2]), __uint_as_float(s4[3])),
                                     make_float2(sl2, sl2), make_float2(nmu, nmu));
        const float2 p0 = make_float2(ptx::ex2(x0.x), ptx::ex2(x0.y));
        const float2 p1 = use_poly(c) ? exp2_poly2(x1) : make_float2(ptx::ex2(x1.x), ptx::ex2(x1.y));
        acc0 = __fadd2_rn(acc0, p0);
        acc1 = __fadd2_rn(acc1, p1);
        sv[16 * gq + (c >> 1)] = pack2<false>(p0.x, p0.y);
        sv[16 * gq + (c >> 1) + 1] = pack2<false>(p1.x, p1.y);
      }
    }
    l += (acc0.x + acc0.y) + (acc1.x + acc1.y);
    if (NG == 4) {
      NA_TMEM_ST32(trow + 128, sv);
      NA_TMEM_ST32(trow + 160, (sv + 32));
    } else {
      NA_TMEM_ST32(trow + 64, sv);
    }
    ptx::tmem_st_wait();
  }
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / iters;
  if (l == 123.f) out[0] = 0;  // keep l alive
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<(NG == 4 ? 256 : 128)>(tmem);
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8 * 600);
  unsigned long long h[600];
  auto run = [&](void (*k)(unsigned long long*, int, uint32_t), const char* name, int ctas, uint32_t wb) {
    k<<<ctas, 128>>>(d, 2000, wb);
    cudaMemcpy(h, d, 8 * ctas, cudaMemcpyDeviceToHost);
    double s = 0;
    for (int i = 0; i < ctas; ++i) s += h[i];
    printf("%-28s ctas %d: %.0f clk per round per CTA (%s)\n", name, ctas, s / ctas,
           cudaGetErrorString(cudaGetLastError()));
  };
  for (int per : {2, 3, 4}) run(rounds<0, 0, 2>, "64-col round", 148 * per, 0);
  for (int ctas : {148, 296}) {
    run(rounds<0, 0>, "full", ctas, 0);
    run(rounds<1, 0>, "full, partial mask", ctas, 0x00ffff00u);
    run(rounds<0, 1>, "ld + st only", ctas, 0);
    run(rounds<0, 2>, "ld + max + st", ctas, 0);
    run(rounds<0, 3>, "ld + exps + st (no max)", ctas, 0);
  }
}
