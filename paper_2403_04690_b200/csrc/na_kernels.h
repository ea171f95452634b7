// na_kernels.h — internal launcher declarations (not part of the ABI).
#pragma once
#include <cuda_runtime.h>

#include "na_geom.cuh"
#include "tc_plan.h"

namespace na {

// Kernel ids for the profiling hook (na_profile_*; names in na_abi.cpp).
enum KernelId {
  KID_FWD_TC = 0,
  KID_FWD_SIMT = 1,
  KID_BWD_PRE = 2,
  KID_DKDV_TC = 3,
  KID_DQ_TC = 4,
  KID_DKDV_SIMT = 5,
  KID_DQ_SIMT = 6,
  KID_COUNT = 7
};
// Bracket one launch with events when profiling is enabled on this thread.
void prof_begin(int kernel_id, cudaStream_t st);
void prof_end(cudaStream_t st);

// dtype: 0 = fp32, 1 = fp16, 2 = bf16 (matches na_dtype)
cudaError_t simt_fwd(int dtype, const Geom& g, const Layout& ly, const void* q, const void* k, const void* v,
                     void* o, float* lse, cudaStream_t st);
cudaError_t simt_bwd(int dtype, const Geom& g, const Layout& ly, const void* q, const void* k, const void* v,
                     const void* o, const void* d_o, const float* lse, void* dq, void* dk,
                     void* dv, float* Dvec, cudaStream_t st);

// D_x = <dO_x, O_x> (fp32).  lse == nullptr: D_x at the token index of Dvec
// [BH*N].  lse != nullptr (16-bit only): the tensor-core row-vector layout
// (-LSE_x*log2(e), D_x) of Geom::rv_* in Dvec.
// Zero the row-vector layout's padding slots (ragged residue classes) before
// the tensor-core backward writes the rest.
cudaError_t rv_clear_padding(const Geom& g, float* Dvec, cudaStream_t st);
cudaError_t bwd_preprocess(int dtype, const Geom& g, const Layout& ly, const void* o, const void* d_o, const float* lse,
                           float* Dvec, cudaStream_t st);

// tcgen05 path.  tc_supported() is a pure host check; the launchers return
// cudaErrorNotSupported for problems outside it.
bool tc_supported(int dtype, const Geom& g, const char** why);
// bf16 only: whether the kernels take the error-compensated variant (DESIGN.md
// R13): the forward normalises O by the sum of the bf16-rounded P, the
// backward splits its bf16 P / dS MMA operands hi + lo and corrects D_x in
// the dQ kernel.  It is needed where outputs can reach magnitudes >= 2,
// whose bf16 half-ulp (2^-8 .. 2^-7) leaves < 0.0022 of the 1e-2 bound for
// the 2^-9-relative rounding of P / dS: with few keys per window single
// probabilities approach 1 and gradients concentrate.  Every window holds
// at least prod over NON-causal axes of k keys (a causal axis leaves its
// first query one key); below kBf16PlainMinKeys the precise variant runs.
// Measured on unit-normal data (profiles/r02_bf16_variants.md): the plain
// variant exceeds the bound at 35-75 keys (dK/dV up to 0.013) and stays
// within it with >= 0.0033 to spare at 169-255 keys (config D: backward
// 0.94 vs 1.64 ms).
constexpr int kBf16PlainMinKeys = 128;
bool bf16_precise(const Geom& g);
// Opt a kernel into `bytes` of dynamic shared memory on the current device
// (once per kernel and device; thread-safe).
cudaError_t ensure_smem_attr(const void* func, int bytes);
// Candidate plans of the tile planner for g (1 for rank 1), and the measured
// choice per kernel (tc_host.cpp; na_tune sets it).
int tc_plan_candidates(const Geom& g);
PlanChoice plan_choice(const Geom& g, int dtype);
void set_plan_choice(const Geom& g, int dtype, PlanChoice c);
// Calling thread only: every plan_choice() returns *c (nullptr: off).  na_tune
// times candidates with it, so the process-wide table never holds a
// transient pick.
void set_plan_override(const PlanChoice* c);
cudaError_t tc_fwd(int dtype, const Geom& g, const Layout& ly, const void* q, const void* k, const void* v,
                   void* o, float* lse, cudaStream_t st, int* launches);
cudaError_t tc_bwd(int dtype, const Geom& g, const Layout& ly, const void* q, const void* k, const void* v,
                   const void* o, const void* d_o, const float* lse, void* dq, void* dk,
                   void* dv, float* Dvec, cudaStream_t st, int* launches);

}  // namespace na
