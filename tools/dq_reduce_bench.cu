// dq_reduce_bench.cu -- measures the memory traffic a single-pass backward
// (dK/dV key-stationary kernel that also reduces fp32
// dQ partials into a global accumulator, instead of a separate query-
// stationary dQ kernel) would ADD, on config B_d1 (1-D, B*H = 128, N = 16384,
// D = 64, k = 255), in the dK/dV kernel's own persistent tile order.
//
// Per key tile of 128 keys the inverse halo is 382 queries = 3 chunks of 128
// = 6 sub-chunks of 64 queries; per sub-chunk the kernel would reduce a
// 64 x 64 fp32 dQ partial (16 KB, contiguous rows of dQacc[BH, N, D]) into
// global memory.  Measured here, with the reduction as:
//   (a) TMA bulk reduce  cp.reduce.async.bulk.global.shared::cta.add.f32
//   (b) red.global.add.v4.f32 from registers (thread = query row)
// plus the two passes the mode needs around it: zeroing dQacc (fp32) and
// converting it to the fp16 dQ (x scale).  If the sum is not well below the
// two-pass dQ kernel's time (0.47-0.57 ms on B_d1, bench per-kernel), the
// mode cannot win regardless of the MMA and exp work it saves.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dq_reduce_bench dq_reduce_bench.cu
#include <cuda_fp16.h>
#include <cstdint>
#include <cstdio>

constexpr int BH = 128, N = 16384, D = 64, TILE = 128, SUB = 64, K = 255;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Sub-chunk origin (first query) of sub-chunk j of key tile t of head bh.
__device__ __forceinline__ int sub_origin(int t, int j) {
  const int y0 = t * TILE, y1 = y0 + TILE - 1;
  const int lo = y0 <= K - 1 ? 0 : y0 - K / 2;
  return lo + j * SUB;
}
__device__ __forceinline__ int sub_count(int t) {
  const int y0 = t * TILE, y1 = y0 + TILE - 1;
  const int lo = y0 <= K - 1 ? 0 : y0 - K / 2;
  const int hi = y1 >= N - K ? N - 1 : y1 + K / 2;
  return (hi - lo + SUB) / SUB;
}

__global__ void __launch_bounds__(128) reduce_tma(float* acc, int tiles) {
  __shared__ __align__(128) float stage[2][SUB * D];
  for (int i = threadIdx.x; i < 2 * SUB * D; i += blockDim.x) (&stage[0][0])[i] = 1e-3f * (i & 7);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x != 0) return;
  int it = 0;
  for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int bh = tile / (N / TILE), t = tile % (N / TILE);
    const int ns = sub_count(t);
    for (int j = 0; j < ns; ++j, ++it) {
      int q0 = sub_origin(t, j);
      int rows = q0 + SUB <= N ? SUB : N - q0;
      float* dst = acc + ((size_t)bh * N + q0) * D;
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");  // staging buffer it&1 free
      asm volatile(
          "cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(dst),
          "r"(smem_u32(stage[it & 1])), "r"(rows * D * 4)
          : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void __launch_bounds__(128) reduce_red(float* acc, int tiles) {
  // thread = query row of the sub-chunk (64 rows x 64 floats: 2 threads per row)
  const int row = threadIdx.x >> 1, half = threadIdx.x & 1;
  for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int bh = tile / (N / TILE), t = tile % (N / TILE);
    const int ns = sub_count(t);
    for (int j = 0; j < ns; ++j) {
      const int q = sub_origin(t, j) + row;
      if (q >= N) continue;
      float* dst = acc + ((size_t)bh * N + q) * D + half * 32;
#pragma unroll
      for (int c = 0; c < 32; c += 4)
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst + c), "f"(1e-3f), "f"(2e-3f),
                     "f"(3e-3f), "f"(4e-3f)
                     : "memory");
    }
  }
}

__global__ void convert(const float4* __restrict__ acc, uint2* __restrict__ out, size_t n4, float scale) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    const float4 a = acc[i];
    __half2 lo = __floats2half2_rn(a.x * scale, a.y * scale), hi = __floats2half2_rn(a.z * scale, a.w * scale);
    out[i] = make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
  }
}

int main() {
  const size_t elems = (size_t)BH * N * D;
  float* acc;
  uint2* out;
  cudaMalloc(&acc, elems * 4);
  cudaMalloc(&out, elems * 2);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int tiles = BH * (N / TILE);
  cudaEvent_t e[8];
  for (auto& x : e) cudaEventCreate(&x);
  float best[4] = {1e9f, 1e9f, 1e9f, 1e9f};
  for (int rep = 0; rep < 6; ++rep) {
    cudaEventRecord(e[0]);
    cudaMemsetAsync(acc, 0, elems * 4);
    cudaEventRecord(e[1]);
    reduce_tma<<<sms, 128>>>(acc, tiles);
    cudaEventRecord(e[2]);
    cudaMemsetAsync(acc, 0, elems * 4);
    cudaEventRecord(e[3]);
    reduce_red<<<sms * 4, 128>>>(acc, tiles);
    cudaEventRecord(e[4]);
    convert<<<sms * 8, 256>>>(reinterpret_cast<const float4*>(acc), out, elems / 4, 0.125f);
    cudaEventRecord(e[5]);
    cudaEventSynchronize(e[5]);
    float t[5];
    for (int i = 0; i < 5; ++i) cudaEventElapsedTime(&t[i], e[i], e[i + 1]);
    if (rep > 0) {
      best[0] = fminf(best[0], t[0]);
      best[1] = fminf(best[1], t[1]);
      best[2] = fminf(best[2], t[3]);
      best[3] = fminf(best[3], t[4]);
    }
  }
  cudaError_t err = cudaGetLastError();
  long long subs = 0;
  for (int t = 0; t < N / TILE; ++t) {
    const int y0 = t * TILE, y1 = y0 + TILE - 1;
    const int lo = y0 <= K - 1 ? 0 : y0 - K / 2;
    const int hi = y1 >= N - K ? N - 1 : y1 + K / 2;
    subs += (hi - lo + SUB) / SUB;
  }
  subs *= BH;
  printf("B_d1 single-pass dQ reduction emulation (%s)\n", cudaGetErrorString(err));
  printf("sub-chunks %lld, reduced bytes %.3f GB (fp32 partials)\n", subs, subs * SUB * D * 4.0 / 1e9);
  printf("memset dQacc fp32 (%.0f MB):       %.4f ms\n", elems * 4 / 1e6, best[0]);
  printf("reduce (TMA bulk reduce-add):        %.4f ms  (%.0f GB/s of partials)\n", best[1],
         subs * SUB * D * 4.0 / (best[1] * 1e-3) / 1e9);
  printf("reduce (red.global.add.v4.f32):      %.4f ms\n", best[2]);
  printf("convert fp32 -> fp16 dQ:             %.4f ms\n", best[3]);
  printf("added by the mode (memset + TMA reduce + convert): %.4f ms\n", best[0] + best[1] + best[3]);
  return 0;
}
