// na_kernels.h — internal launcher declarations (not part of the ABI).
#pragma once
#include <cuda_runtime.h>

#include "na_geom.cuh"

namespace na {

// dtype: 0 = fp32, 1 = fp16, 2 = bf16 (matches na_dtype)
cudaError_t simt_fwd(int dtype, const Geom& g, const void* q, const void* k, const void* v,
                     void* o, float* lse, cudaStream_t st);
cudaError_t simt_bwd(int dtype, const Geom& g, const void* q, const void* k, const void* v,
                     const void* o, const void* d_o, const float* lse, void* dq, void* dk,
                     void* dv, float* Dvec, cudaStream_t st);

// D_x = <dO_x, O_x> (fp32), one warp per row.
cudaError_t bwd_preprocess(int dtype, const Geom& g, const void* o, const void* d_o, float* Dvec,
                           cudaStream_t st);

// tcgen05 path.  tc_supported() is a pure host check; the launchers return
// cudaErrorNotSupported for problems outside it.
bool tc_supported(int dtype, const Geom& g, const char** why);
cudaError_t tc_fwd(int dtype, const Geom& g, const void* q, const void* k, const void* v,
                   void* o, float* lse, cudaStream_t st, int* launches);
cudaError_t tc_bwd(int dtype, const Geom& g, const void* q, const void* k, const void* v,
                   const void* o, const void* d_o, const float* lse, void* dq, void* dk,
                   void* dv, float* Dvec, cudaStream_t st, int* launches);

}  // namespace na
