/*
 * oracle/na_oracle.h — plain fp64 CPU oracle for neighborhood attention.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load, call or link
 * anything under oracle/.  The product path (include/na.h, libna.so) never
 * does, and shares no header, helper or table with this file.
 *
 * What it computes (PAPER.md = P, SPEC.md = S):
 *   Eq. 1 restricted to each query's neighborhood N(x):
 *     s_xy = scale * <q_x, k_y>,  y in N(x);  scale defaults to 1/sqrt(d)
 *     LSE_x = log sum_y exp(s_xy);  P_xy = exp(s_xy - LSE_x)
 *     O_x   = sum_y P_xy v_y
 *   N(x) per axis (Fig. 2 caption P:110-120; dilation P:329-331; causal
 *   P:117-118): x = r + dil*x', window in compacted coordinates of
 *   the residue class r, size L_r = ceil((L-r)/dil):
 *     non-causal: start = clamp(x' - k/2, 0, L_r - k), window [start, start+k-1]
 *     causal    : window [max(0, x'-k+1), x']
 *   N(x) is the Cartesian product over axes.
 *   Backward (composition of PN/NN/IN; softmax Jacobian, reading
 *   R12 in DESIGN.md):
 *     D_x = <dO_x, O_x>;  dS_xy = P_xy (<dO_x, v_y> - D_x)
 *     dQ_x = scale sum_{y in N(x)} dS_xy k_y
 *     dK_y = scale sum_{x : y in N(x)} dS_xy q_x
 *     dV_y = sum_{x : y in N(x)} P_xy dO_x
 *
 * Layout of every tensor: contiguous [B, H, X0 (, X1 (, X2)), D]; LSE is
 * [B, H, X0 (, X1 (, X2))].  Inputs are read through a dtype code and upcast
 * exactly to double; all outputs are double.
 */
#ifndef NA_ORACLE_H
#define NA_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { NAR_F64 = 0, NAR_F32 = 1, NAR_F16 = 2, NAR_BF16 = 3 };

typedef struct {
  int32_t rank;               /* 1..3 */
  int32_t batch, heads, head_dim;
  int32_t extent[3];          /* L per axis, outermost first */
  int32_t kernel_size[3];     /* k per axis */
  int32_t dilation[3];        /* dil per axis */
  int32_t is_causal[3];       /* 0/1 per axis */
  double scale;               /* <= 0 -> 1/sqrt(head_dim) */
} nar_problem;

/* 0 if the problem is one the oracle defines, else a nonzero code
 * (1 rank, 2 shape, 3 kernel<1, 4 even k on non-causal axis, 5 dilation<1,
 *  6 k*dil > L).  Same constraint list as S:62-70 / S:132-137. */
int nar_check(const nar_problem* p);

/* Per-axis window of query coordinate x (original coordinates, 0 <= x < L).
 * Writes the first and last key coordinate (original coordinates; keys are
 * first, first+dil, ..., last).  Returns the number of keys. */
int nar_axis_window(int L, int k, int dil, int causal, int x, int* first, int* last);

/* 1 iff key token y is in N(x); x, y are flat spatial indices. */
int nar_contains(const nar_problem* p, int64_t x, int64_t y);

/* Full forward over every (b, h, x).  o: [B,H,N,D] double, lse: [B,H,N]. */
int nar_fwd(const nar_problem* p, int dtype, const void* q, const void* k,
            const void* v, double* o, double* lse);

/* Forward for n selected flat token indices t = (b*H + h)*N + x. */
int nar_fwd_tokens(const nar_problem* p, int dtype, const void* q, const void* k,
                   const void* v, int64_t n, const int64_t* tokens,
                   double* o /* [n, D] */, double* lse /* [n] */);

/* Full backward (scatter form).  Recomputes O and LSE internally in fp64.
 * o_dtype: NAR_F64 -> the exact gradient (D_x from the fp64 O); a 16-bit
 * code -> D_x = <dO_x, O_x> with O as the method stores it, the fp64 O
 * rounded to fp32 then to that dtype (reading R12).  The rounding
 * is the oracle's own; no value from the GPU enters. */
int nar_bwd(const nar_problem* p, int dtype, int o_dtype, const void* q, const void* k,
            const void* v, const void* d_o, double* dq, double* dk, double* dv);

/* Backward at n selected flat token indices (gather form): dq of query t,
 * dk and dv of key t.  Each output is [n, D]. */
int nar_bwd_tokens(const nar_problem* p, int dtype, int o_dtype, const void* q, const void* k,
                   const void* v, const void* d_o, int64_t n, const int64_t* tokens,
                   double* dq, double* dk, double* dv);

/* Full backward in gather form, every token of every slice, parallel over
 * tokens (for whole-slice checks of large problems, where nar_bwd's
 * per-slice parallelism leaves cores idle).  Per slice: one pass over the
 * queries x computes LSE_x, D_x = <dO_x, O_x> (o_dtype as in nar_bwd) and
 * dQ_x; a second pass over the keys t gathers dK_t, dV_t from the queries
 * {x : t in N(x)} with P_xt = exp(s_xt - LSE_x) (the same expression
 * forward_row uses), so the result is nar_bwd's up to fp64 summation order.
 * Outputs [B,H,N,D]. */
int nar_bwd_gather(const nar_problem* p, int dtype, int o_dtype, const void* q, const void* k,
                   const void* v, const void* d_o, double* dq, double* dk, double* dv);

/* Threads the OpenMP runtime will use (for reporting `cores`). */
int nar_num_threads(void);

#ifdef __cplusplus
}
#endif
#endif
