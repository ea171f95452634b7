/*
 * include/na.h — C ABI of the B200 fused neighborhood attention library
 * (libna.so, built from paper_2403_04690_b200/csrc for sm_100a).
 *
 * The operation (PAPER.md = /root/reference/PAPER.md, cited as P:line):
 *   Eq. 1, scaled dot-product attention, restricted per query x
 *   to its neighborhood N(x) (Fig. 2 caption):
 *     O_x   = sum_{y in N(x)} softmax_y(scale <q_x, k_y>) v_y
 *     LSE_x = log sum_{y in N(x)} exp(scale <q_x, k_y>)      (natural log)
 *   N(x) is the Cartesian product over axes a of a per-axis window: the
 *   query's residue class r = x_a mod dilation_a is treated as a
 *   non-dilated axis of ceil((L_a - r)/dilation_a) tokens (§3.4);
 *   on it the window holds kernel_size_a consecutive members, centred on the
 *   query and shifted inward at the borders, or, on a
 *   causal axis, the kernel_size_a members ending at the query (P:117-118,
 *   P:332-334).  See DESIGN.md "Readings" for every choice the paper leaves
 *   open (window placement rule, even kernels, LSE base, tolerances ...).
 *   The forward is fused (§3.3): attention weights never reach
 *   global memory.  The backward (§3.1 operators PN/NN/IN)
 *   recomputes the weights from LSE and writes dQ, dK, dV with exactly one
 *   writer per element (no atomics).
 *
 * Conventions (all entry points):
 *   - Tensors Q, K, V, O, dO, dQ, dK, dV are DEVICE pointers to
 *     [batch, heads, X0 (, X1 (, X2)), head_dim] arrays of `dtype`
 *     (X0 outermost; e.g. T, H, W for video): contiguous when
 *     na_problem.strides is NULL, else all eight share those element strides
 *     (see na_problem).  LSE is a device pointer to a contiguous fp32
 *     [batch, heads, X0 (, X1 (, X2))] array.  All base pointers must be
 *     16-byte aligned.
 *   - The caller owns every buffer; the library never allocates device
 *     memory.  The backward workspace is caller-supplied.
 *   - Calls are asynchronous and stream-ordered on `stream` (a cudaStream_t;
 *     0 = legacy default stream).  Buffers must stay live until the stream
 *     reaches the call.
 *   - The problem is validated before anything is launched.  On any error
 *     nothing is launched and nothing is written; the status is returned
 *     (never thrown, never abort()).  na_last_error() gives a thread-local
 *     detail string for the last failing call on this thread.
 *   - Results are deterministic: identical inputs on the same device give
 *     bitwise identical outputs.
 *   - Thread safety: entry points may be called concurrently from several
 *     host threads.
 *   - Multi-GPU is not part of the ABI: callers shard batch x heads and call
 *     the library once per device.
 */
#ifndef NA_H_
#define NA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum { NA_F32 = 0, NA_F16 = 1, NA_BF16 = 2 } na_dtype;

typedef enum {
  NA_OK = 0,
  NA_ERR_NULL = 1,            /* null problem or required tensor pointer                  */
  NA_ERR_RANK = 2,            /* rank not in {1,2,3}         */
  NA_ERR_SHAPE = 3,           /* batch, heads, head_dim or an extent < 1                   */
  NA_ERR_BAD_KERNEL = 4,      /* kernel_size < 1                                           */
  NA_ERR_EVEN_WINDOW = 5,     /* even kernel_size on a non-causal axis  */
  NA_ERR_BAD_DILATION = 6,    /* dilation < 1         */
  NA_ERR_WINDOW_EXCEEDS = 7,  /* kernel_size * dilation > extent: the window would not fit
                                 in the smallest residue class  */
  NA_ERR_DTYPE = 8,           /* dtype not one of na_dtype                                 */
  NA_ERR_HEAD_DIM = 9,        /* head_dim > 256 or not a multiple of 8 (16-bit) / 4 (fp32) */
  NA_ERR_ALIGNMENT = 10,      /* a base pointer or a stride is not a 16-byte multiple      */
  NA_ERR_LAYOUT = 11,         /* strides: head_dim stride != 1 or a stride < 1             */
  NA_ERR_WORKSPACE = 12,      /* backward workspace missing or smaller than required       */
  NA_ERR_CUDA = 13,           /* CUDA launch/driver error (see na_last_error)              */
  NA_ERR_IMPL = 14            /* the requested `impl` cannot run this problem              */
} na_status;

/* Kernel family selection (tests and benchmarks use it to pin a path). */
/* Kernel family selection.  There is no silent fallback: with NA_IMPL_AUTO a
 * 16-bit problem runs on the tensor cores, and a 16-bit problem outside that
 * path (tc_supported: head_dim not in {16, 32, 64, 128}, or a dilation
 * above 8) fails with NA_ERR_IMPL
 * unless the caller selects NA_IMPL_SIMT explicitly.  fp32 inputs always run
 * on the CUDA-core kernels (TF32 off, north_star's 1e-4 bound). */
typedef enum {
  NA_IMPL_AUTO = 0,  /* fp16/bf16: tensor cores (or NA_ERR_IMPL); fp32: SIMT */
  NA_IMPL_SIMT = 1,  /* fp32 CUDA-core kernels (any dtype; fp32 inputs always) */
  NA_IMPL_TC = 2     /* tcgen05 + TMEM + TMA kernels (fp16 / bf16 only)        */
} na_impl;

typedef struct {
  int32_t rank;            /* 1..3 spatial axes                                   */
  int32_t batch, heads;    /* >= 1                                                */
  int32_t head_dim;        /* d in Eq. 1                                          */
  int32_t extent[3];       /* L_a, outermost axis first; entries >= rank ignored  */
  int32_t kernel_size[3];  /* k_a: window size per axis        */
  int32_t dilation[3];     /* dilation_a >= 1                  */
  int32_t is_causal[3];    /* 0/1 per axis                 */
  float scale;             /* softmax scale; <= 0 means 1/sqrt(head_dim)  */
  na_dtype dtype;          /* of Q,K,V,O,dO,dQ,dK,dV; LSE/workspace always fp32   */
  na_impl impl;            /* NA_IMPL_AUTO unless pinning a kernel family         */
  /* NULL: contiguous [B, H, X0 (, X1 (, X2)), D].  Else 6 element strides
   * {B, H, X0, X1, X2, D} shared by Q, K, V, O, dO, dQ, dK, dV (X_a with
   * a >= rank ignored): D's must be 1, the others >= 1 and multiples of 16
   * bytes (the tensor-core path addresses rows through TMA tensor maps).
   * E.g. heads-last [B, X..., H, D] storage viewed as [B, H, X..., D], or
   * one slice of a packed [B, X..., 3, H, D] QKV buffer.  When the batch
   * stride is not heads x the head stride, each batch entry runs as its own
   * launch set on the same stream (na_last_launch_count counts them all).
   * The caller guarantees that output rows do not overlap. */
  const int64_t* strides;
} na_problem;

/* Validates `p` alone (no pointers).  Pure host function; never touches a GPU. */
na_status na_validate(const na_problem* p);

/* Forward.  Reads q, k, v; writes o and, if lse != NULL, lse (fp32 natural-log
 * LSE_x, needed by na_bwd).  One kernel launch on `stream`. */
na_status na_fwd(const na_problem* p, const void* q, const void* k, const void* v, void* o,
                 float* lse, void* stream);

/* Bytes of device workspace na_bwd needs for the fp32 row vectors
 * D_x = <dO_x, O_x> and, on the tensor-core path, -LSE_x*log2(e):
 * max(B*H*N*4, B*H*nres*2*plane*4) with nres = prod(dilation) residue
 * classes and plane = prod_a ceil(extent_a / dilation_a), the innermost factor
 * rounded up to a multiple of 4 (class-compacted layout, 16-byte TMA strides). */
size_t na_bwd_workspace_size(const na_problem* p);

/* Backward.  Reads q, k, v, o, d_o (dL/dO) and lse from na_fwd on the same
 * inputs; writes dq, dk, dv (each element by exactly one thread; no
 * atomics).  The softmax-Jacobian term D_x = sum_y P_xy dP_xy = <dO_x, O_x>
 * (reading R12): fp16 forms it from the `o` passed in (the stored
 * forward output); bf16 in its precise variant (na_bf16_precise), whose
 * stored O is 8x coarser, uses <dO_x, o_x> only as an estimate and corrects
 * it inside the dQ kernel to sum_y P_xy dP_xy in fp32, so its gradient is
 * that of the exact forward.  `workspace` (device,
 * >= na_bwd_workspace_size bytes) is scratch owned by the caller.  Launches
 * on `stream`, in order:
 *   rank 1:   [a memset of the workspace's padding slots when a residue
 *             class is ragged], dQ (query-stationary, forward map; it also
 *             forms the row values -LSE_x*log2(e), D_x from the O and dO
 *             tiles it loads), then dK/dV (key-stationary, inverse map);
 *   rank 2-3: the row-value pass (-LSE_x*log2(e), <dO_x, O_x>), dQ, dK/dV.
 * na_last_launch_count() reports the number of kernels (2 or 3). */
na_status na_bwd(const na_problem* p, const void* q, const void* k, const void* v,
                 const void* o, const void* d_o, const float* lse, void* dq, void* dk,
                 void* dv, void* workspace, size_t workspace_bytes, void* stream);

/* Tile-plan tuning (tensor-core path).  The planner ranks tile / KV-chunk
 * shapes with a cost model; na_tune runs the
 * forward and backward with each of the na_plan_candidates(p) cheapest
 * plans on the caller's buffers (all outputs are overwritten; inputs as for
 * na_fwd / na_bwd), keeps the fastest plan per kernel (forward, dK/dV, dQ)
 * in a process-wide table keyed by the problem's geometry, head_dim and
 * dtype, and returns the picks in choice_out (may be NULL).  Synchronizes
 * `stream`.  Later na_fwd / na_bwd calls with that geometry use the picks.
 * Every plan computes the same result up to floating-point summation order.
 * na_get/set_plan_choice read and set the picks directly (e.g. to broadcast
 * rank 0's choice to the other ranks of a job); picks are in
 * [0, na_plan_candidates(p)).  na_plan_candidates returns 1 for rank 1 and
 * for the SIMT path, -1 for an invalid problem. */
int na_plan_candidates(const na_problem* p);
na_status na_tune(const na_problem* p, const void* q, const void* k, const void* v, void* o,
                  float* lse, const void* d_o, void* dq, void* dk, void* dv, void* workspace,
                  size_t workspace_bytes, void* stream, int32_t choice_out[3]);
na_status na_get_plan_choice(const na_problem* p, int32_t choice[3]);
na_status na_set_plan_choice(const na_problem* p, const int32_t choice[3]);

/* Which kernel family na_fwd/na_bwd would run for `p` (NA_IMPL_SIMT or
 * NA_IMPL_TC), or -1 if `p` is invalid or its `impl` cannot run it (the calls
 * would return NA_ERR_IMPL).  Host only. */
int na_selected_impl(const na_problem* p);

/* bf16 on the tensor cores (R13): 1 if na_fwd / na_bwd run the
 * error-compensated variant for `p` (O normalised by the sum of the
 * bf16-rounded P; the backward's bf16 P / dS MMA operands split hi + lo and
 * D_x corrected in the dQ kernel), 0 if the plain one (also for every
 * non-bf16 or non-tensor-core problem), -1 if `p` is invalid.  The precise
 * variant runs when some window holds fewer than 128 keys -- the product of
 * k over the NON-causal axes (a causal axis leaves its first query a single
 * key) -- where single probabilities approach 1 and outputs reach magnitudes
 * whose bf16 half-ulp leaves too little of the 1e-2 bound.  Host only. */
int na_bf16_precise(const na_problem* p);

/* Static description of a status code. */
const char* na_status_string(na_status s);

/* Detail message of the last failing call on this host thread ("" if none). */
const char* na_last_error(void);

/* Number of kernel launches the last successful na_fwd / na_bwd issued on
 * this host thread (for the benchmark's gpu_launches count). */
int na_last_launch_count(void);

/* Benchmark instrumentation (per host thread, off by default).  While
 * enabled, every kernel launch made by na_fwd / na_bwd on this thread is
 * bracketed by two CUDA events recorded on the launch stream (the stream the
 * kernel runs on).  na_profile_collect() waits for those events, writes up to
 * `max_entries` (kernel id, device milliseconds) pairs in launch order,
 * returns how many launches were recorded, and clears the list.  Kernel ids
 * are named by na_kernel_name(). */
void na_profile_enable(int on);
int na_profile_collect(int* kernel_ids, float* ms, int max_entries);
const char* na_kernel_name(int kernel_id);

#ifdef __cplusplus
}
#endif
#endif /* NA_H_ */
