// na_abi.cpp — the C ABI of libna.so (include/na.h): validation, kernel-family
// selection and launch.  Everything here is host code; the arithmetic runs in
// the CUDA kernels (fna_simt.cu, fna_tc_fwd.cu, fna_tc_bwd.cu).
#include "../../include/na.h"

#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "na_kernels.h"

namespace {

thread_local std::string g_last_error;
thread_local int g_last_launches = 0;

struct ProfEntry {
  int id;
  cudaEvent_t a, b;
};
thread_local bool g_prof = false;
thread_local std::vector<ProfEntry> g_prof_list;

na_status fail(na_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return s;
}

// Constraint list of S:62-70 / S:132-137 plus the ABI's own limits.
na_status validate(const na_problem* p) {
  if (!p) return fail(NA_ERR_NULL, "problem is NULL");
  if (p->rank < 1 || p->rank > 3) return fail(NA_ERR_RANK, "rank %d not in {1,2,3}", p->rank);
  if (p->batch < 1 || p->heads < 1 || p->head_dim < 1)
    return fail(NA_ERR_SHAPE, "batch/heads/head_dim must be >= 1");
  int64_t n = 1;
  for (int a = 0; a < p->rank; ++a) {
    if (p->extent[a] < 1) return fail(NA_ERR_SHAPE, "extent[%d] = %d < 1", a, p->extent[a]);
    if (p->kernel_size[a] < 1)
      return fail(NA_ERR_BAD_KERNEL, "kernel_size[%d] = %d < 1", a, p->kernel_size[a]);
    if (!p->is_causal[a] && p->kernel_size[a] % 2 == 0)
      return fail(NA_ERR_EVEN_WINDOW, "even kernel_size[%d] = %d on a non-causal axis", a,
                  p->kernel_size[a]);
    if (p->dilation[a] < 1)
      return fail(NA_ERR_BAD_DILATION, "dilation[%d] = %d < 1", a, p->dilation[a]);
    if ((int64_t)p->kernel_size[a] * p->dilation[a] > p->extent[a])
      return fail(NA_ERR_WINDOW_EXCEEDS,
                  "kernel_size[%d]*dilation[%d] = %lld > extent %d (window exceeds the "
                  "smallest residue class)",
                  a, a, (long long)p->kernel_size[a] * p->dilation[a], p->extent[a]);
    n *= p->extent[a];
  }
  if (p->dtype != NA_F32 && p->dtype != NA_F16 && p->dtype != NA_BF16)
    return fail(NA_ERR_DTYPE, "dtype %d unknown", (int)p->dtype);
  const int align = p->dtype == NA_F32 ? 4 : 8;   // rows must be 16-byte multiples
  if (p->head_dim > 256 || p->head_dim % align)
    return fail(NA_ERR_HEAD_DIM, "head_dim %d: need <= 256 and a multiple of %d", p->head_dim,
                align);
  if (p->strides) {
    // [B, H, X0, X1, X2, D] element strides; entries X_a for a >= rank ignored.
    const int64_t* st = p->strides;
    if (st[5] != 1) return fail(NA_ERR_LAYOUT, "head_dim stride must be 1 (got %lld)", (long long)st[5]);
    const int esz = p->dtype == NA_F32 ? 4 : 2;
    for (int i = 0; i < 5; ++i) {
      if (i >= 2 && i - 2 >= p->rank) continue;
      if (st[i] < 1) return fail(NA_ERR_LAYOUT, "stride[%d] = %lld < 1", i, (long long)st[i]);
      if ((st[i] * esz) % 16)
        return fail(NA_ERR_ALIGNMENT, "stride[%d] = %lld elements is not a multiple of 16 bytes", i,
                    (long long)st[i]);
    }
  }
  if ((int64_t)p->batch * p->heads * n * p->head_dim > (int64_t(1) << 40))
    return fail(NA_ERR_SHAPE, "problem too large");
  if ((int64_t)p->batch * p->heads > 0x7fffffff || n > 0x7fffffff)
    return fail(NA_ERR_SHAPE, "B*H or tokens exceed int32");
  // Row indices are 32-bit in the kernels; Q, K, V, O of 2^32 rows cannot fit
  // in device memory at any head_dim.
  if ((int64_t)p->batch * p->heads * n > (int64_t)0xffffffff)
    return fail(NA_ERR_SHAPE, "B*H*tokens exceeds 2^32");
  if (p->impl != NA_IMPL_AUTO && p->impl != NA_IMPL_SIMT && p->impl != NA_IMPL_TC)
    return fail(NA_ERR_IMPL, "impl %d unknown", (int)p->impl);
  return NA_OK;
}

na::Geom make_geom(const na_problem* p) {
  na::Geom g{};
  g.rank = p->rank;
  g.BH = p->batch * p->heads;
  g.D = p->head_dim;
  int n = 1;
  for (int a = 0; a < 3; ++a) {
    bool on = a < p->rank;
    g.L[a] = on ? p->extent[a] : 1;
    g.k[a] = on ? p->kernel_size[a] : 1;
    g.dil[a] = on ? p->dilation[a] : 1;
    g.causal[a] = on ? (p->is_causal[a] ? 1 : 0) : 0;
    n *= g.L[a];
  }
  g.N = n;
  int s = 1;
  for (int a = p->rank - 1; a >= 0; --a) {
    g.tstride[a] = s;
    s *= g.L[a];
  }
  for (int a = p->rank; a < 3; ++a) g.tstride[a] = 1;
  g.scale = p->scale > 0.f ? p->scale : 1.f / std::sqrt((float)p->head_dim);
  g.scale_log2 = g.scale * 1.4426950408889634f;
  g.nres = 1;
  for (int a = 0; a < 3; ++a) {
    g.nres *= g.dil[a];
    g.rv_lc[a] = (g.L[a] + g.dil[a] - 1) / g.dil[a];
  }
  g.rv_lc[p->rank - 1] = (g.rv_lc[p->rank - 1] + 3) / 4 * 4;
  long long cs = 1;
  for (int a = 2; a >= 0; --a) {
    g.rv_cs[a] = (int)cs;
    cs *= g.rv_lc[a];
  }
  g.rv_plane = cs;
  return g;
}

// Element strides of the Q/K/V/O-type tensors (na_geom.cuh, Layout).
na::Layout make_layout(const na_problem* p, const na::Geom& g) {
  na::Layout ly{};
  for (int a = 0; a < 3; ++a) ly.sX[a] = a < p->rank ? (long long)g.tstride[a] * g.D : 0;
  ly.sBH = (long long)g.N * g.D;
  ly.contig = 1;
  if (p->strides) {
    ly.contig = 0;
    for (int a = 0; a < p->rank; ++a) ly.sX[a] = p->strides[2 + a];
    // B and H merge into one slice index when stride_B = H * stride_H; the
    // ABI calls split other layouts into one launch set per batch entry
    // (split_batches), each with B = 1, where sBH = stride_H.
    ly.sBH = p->heads > 1 ? p->strides[1] : p->strides[0];
  }
  return ly;
}

// Backward workspace: the SIMT path's D_x vector [BH*N] or the tensor-core
// path's row-vector layout [BH*nres][2][plane], whichever is larger.
size_t bwd_workspace_bytes(const na::Geom& g) {
  const size_t simt = (size_t)g.BH * (size_t)g.N * sizeof(float);
  const size_t tc = (size_t)g.BH * (size_t)g.nres * 2 * (size_t)g.rv_plane * sizeof(float);
  return simt > tc ? simt : tc;
}

// Which family runs problem p (assumes p validated), or -1: no silent
// fallback -- a 16-bit problem runs on the tensor cores unless the caller
// asks for the CUDA-core kernels explicitly (NA_IMPL_SIMT).
int select_impl(const na_problem* p, const na::Geom& g, const char** why) {
  *why = "";
  if (p->dtype == NA_F32) {
    if (p->impl == NA_IMPL_TC) {
      *why = "fp32 inputs run on the CUDA-core kernels (TF32 off)";
      return -1;
    }
    return NA_IMPL_SIMT;
  }
  if (p->impl == NA_IMPL_SIMT) return NA_IMPL_SIMT;
  if (na::tc_supported((int)p->dtype, g, why)) return NA_IMPL_TC;
  return -1;
}

bool aligned16(const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15u) == 0; }

// Strided layouts whose batch and head strides do not merge into one slice
// index (stride_B != H * stride_H, e.g. heads-last [B, X..., H, D] views):
// every batch entry is run as its own B = 1 problem on the same stream
// (base pointers advanced by stride_B; LSE by H*N; the backward workspace
// is reused, each sub-call consuming its row vectors before the next
// writes them).
bool split_batches(const na_problem* p) {
  return p->strides && p->batch > 1 && p->heads > 1 && p->strides[0] != (int64_t)p->heads * p->strides[1];
}
const void* adv(const void* ptr, long long elems, int esz) {
  return static_cast<const char*>(ptr) + elems * esz;
}
void* adv(void* ptr, long long elems, int esz) { return static_cast<char*>(ptr) + elems * esz; }

na_status cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return NA_OK;
  return fail(NA_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

}  // namespace

namespace na {

void prof_begin(int kernel_id, cudaStream_t st) {
  if (!g_prof) return;
  ProfEntry e{kernel_id, nullptr, nullptr};
  cudaEventCreate(&e.a);
  cudaEventCreate(&e.b);
  cudaEventRecord(e.a, st);
  g_prof_list.push_back(e);
}

void prof_end(cudaStream_t st) {
  if (!g_prof || g_prof_list.empty()) return;
  cudaEventRecord(g_prof_list.back().b, st);
}

}  // namespace na

extern "C" {

void na_profile_enable(int on) { g_prof = on != 0; }

int na_profile_collect(int* kernel_ids, float* ms, int max_entries) {
  const int n = (int)g_prof_list.size();
  for (int i = 0; i < n; ++i) {
    ProfEntry& e = g_prof_list[i];
    float t = -1.f;
    if (cudaEventSynchronize(e.b) == cudaSuccess) cudaEventElapsedTime(&t, e.a, e.b);
    if (i < max_entries) {
      if (kernel_ids) kernel_ids[i] = e.id;
      if (ms) ms[i] = t;
    }
    cudaEventDestroy(e.a);
    cudaEventDestroy(e.b);
  }
  g_prof_list.clear();
  return n;
}

const char* na_kernel_name(int kernel_id) {
  static const char* names[na::KID_COUNT] = {"fna_fwd_tc",  "fna_fwd_simt", "fna_bwd_pre",
                                             "fna_dkdv_tc", "fna_dq_tc",    "fna_dkdv_simt",
                                             "fna_dq_simt"};
  return kernel_id >= 0 && kernel_id < na::KID_COUNT ? names[kernel_id] : "unknown";
}


na_status na_validate(const na_problem* p) {
  na_status s = validate(p);
  if (s == NA_OK) g_last_error.clear();
  return s;
}

int na_selected_impl(const na_problem* p) {
  if (validate(p) != NA_OK) return -1;
  na::Geom g = make_geom(p);
  const char* why;
  return select_impl(p, g, &why);
}

int na_bf16_precise(const na_problem* p) {
  if (validate(p) != NA_OK) return -1;
  na::Geom g = make_geom(p);
  const char* why;
  if (p->dtype != NA_BF16 || select_impl(p, g, &why) != NA_IMPL_TC) return 0;
  return na::bf16_precise(g) ? 1 : 0;
}

na_status na_fwd(const na_problem* p, const void* q, const void* k, const void* v, void* o,
                 float* lse, void* stream) {
  na_status s = validate(p);
  if (s != NA_OK) return s;
  if (!q || !k || !v || !o) return fail(NA_ERR_NULL, "q, k, v and o are required");
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o) || (lse && !aligned16(lse)))
    return fail(NA_ERR_ALIGNMENT, "tensor base pointers must be 16-byte aligned");
  na::Geom g = make_geom(p);
  const char* why;
  int impl = select_impl(p, g, &why);
  if (impl < 0)
    return fail(NA_ERR_IMPL, "tensor-core path cannot run this problem: %s (impl=NA_IMPL_SIMT selects the "
                "CUDA-core kernels explicitly)", why);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int launches = 1, total = 0;
  const na::Layout ly = make_layout(p, g);
  const int nb = split_batches(p) ? p->batch : 1;
  if (nb > 1) g.BH = p->heads;
  const int esz = p->dtype == NA_F32 ? 4 : 2;
  cudaError_t e = cudaSuccess;
  for (int b = 0; b < nb && e == cudaSuccess; ++b) {
    const long long eo = (long long)b * (nb > 1 ? p->strides[0] : 0);
    const void *qb = adv(q, eo, esz), *kb = adv(k, eo, esz), *vb = adv(v, eo, esz);
    void* ob = adv(o, eo, esz);
    float* lb = lse ? lse + (long long)b * (nb > 1 ? (long long)g.BH * g.N : 0) : nullptr;
    e = impl == NA_IMPL_TC ? na::tc_fwd((int)p->dtype, g, ly, qb, kb, vb, ob, lb, st, &launches)
                           : na::simt_fwd((int)p->dtype, g, ly, qb, kb, vb, ob, lb, st);
    total += launches;
  }
  launches = total;
  s = cuda_status(e, "na_fwd launch");
  if (s == NA_OK) {
    g_last_error.clear();
    g_last_launches = launches;
  }
  return s;
}

size_t na_bwd_workspace_size(const na_problem* p) {
  if (validate(p) != NA_OK) return 0;
  return bwd_workspace_bytes(make_geom(p));
}

na_status na_bwd(const na_problem* p, const void* q, const void* k, const void* v, const void* o,
                 const void* d_o, const float* lse, void* dq, void* dk, void* dv, void* workspace,
                 size_t workspace_bytes, void* stream) {
  na_status s = validate(p);
  if (s != NA_OK) return s;
  if (!q || !k || !v || !o || !d_o || !lse || !dq || !dk || !dv)
    return fail(NA_ERR_NULL, "q, k, v, o, d_o, lse, dq, dk, dv are required");
  const void* ptrs[] = {q, k, v, o, d_o, lse, dq, dk, dv};
  for (const void* ptr : ptrs)
    if (!aligned16(ptr)) return fail(NA_ERR_ALIGNMENT, "tensor base pointers must be 16-byte aligned");
  na::Geom g = make_geom(p);
  const size_t need = bwd_workspace_bytes(g);
  if (!workspace || workspace_bytes < need || !aligned16(workspace))
    return fail(NA_ERR_WORKSPACE, "workspace needs %zu bytes (16-byte aligned), got %zu", need,
                workspace_bytes);
  const char* why;
  int impl = select_impl(p, g, &why);
  if (impl < 0)
    return fail(NA_ERR_IMPL, "tensor-core path cannot run this problem: %s (impl=NA_IMPL_SIMT selects the "
                "CUDA-core kernels explicitly)", why);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int launches = 3, total = 0;
  const na::Layout ly = make_layout(p, g);
  const int nb = split_batches(p) ? p->batch : 1;
  if (nb > 1) g.BH = p->heads;
  const int esz = p->dtype == NA_F32 ? 4 : 2;
  cudaError_t e = cudaSuccess;
  for (int b = 0; b < nb && e == cudaSuccess; ++b) {
    const long long eo = (long long)b * (nb > 1 ? p->strides[0] : 0);
    const float* lb = lse + (long long)b * (nb > 1 ? (long long)g.BH * g.N : 0);
    e = impl == NA_IMPL_TC
            ? na::tc_bwd((int)p->dtype, g, ly, adv(q, eo, esz), adv(k, eo, esz), adv(v, eo, esz), adv(o, eo, esz),
                         adv(d_o, eo, esz), lb, adv(dq, eo, esz), adv(dk, eo, esz), adv(dv, eo, esz),
                         (float*)workspace, st, &launches)
            : na::simt_bwd((int)p->dtype, g, ly, adv(q, eo, esz), adv(k, eo, esz), adv(v, eo, esz),
                           adv(o, eo, esz), adv(d_o, eo, esz), lb, adv(dq, eo, esz), adv(dk, eo, esz),
                           adv(dv, eo, esz), (float*)workspace, st);
    total += launches;
  }
  launches = total;
  s = cuda_status(e, "na_bwd launch");
  if (s == NA_OK) {
    g_last_error.clear();
    g_last_launches = launches;
  }
  return s;
}

int na_plan_candidates(const na_problem* p) {
  if (validate(p) != NA_OK) return -1;
  na::Geom g = make_geom(p);
  const char* why;
  if (select_impl(p, g, &why) != NA_IMPL_TC) return 1;
  return na::tc_plan_candidates(g);
}

na_status na_get_plan_choice(const na_problem* p, int32_t choice[3]) {
  na_status s = validate(p);
  if (s != NA_OK) return s;
  if (!choice) return fail(NA_ERR_NULL, "choice is NULL");
  const na::PlanChoice c = na::plan_choice(make_geom(p), (int)p->dtype);
  choice[0] = c.fwd;
  choice[1] = c.dkdv;
  choice[2] = c.dq;
  g_last_error.clear();
  return NA_OK;
}

na_status na_set_plan_choice(const na_problem* p, const int32_t choice[3]) {
  na_status s = validate(p);
  if (s != NA_OK) return s;
  if (!choice) return fail(NA_ERR_NULL, "choice is NULL");
  const int n = na_plan_candidates(p);
  for (int i = 0; i < 3; ++i)
    if (choice[i] < 0 || choice[i] >= n)
      return fail(NA_ERR_SHAPE, "plan choice %d out of range [0, %d)", choice[i], n);
  na::set_plan_choice(make_geom(p), (int)p->dtype, na::PlanChoice{choice[0], choice[1], choice[2]});
  g_last_error.clear();
  return NA_OK;
}

na_status na_tune(const na_problem* p, const void* q, const void* k, const void* v, void* o, float* lse,
                  const void* d_o, void* dq, void* dk, void* dv, void* workspace, size_t workspace_bytes,
                  void* stream, int32_t choice_out[3]) {
  na_status s = validate(p);
  if (s != NA_OK) return s;
  const int n = na_plan_candidates(p);
  int32_t best[3] = {0, 0, 0};
  if (n > 1) {
    // Time every candidate plan for each kernel (forward, dK/dV, dQ) with
    // the launch-event hook, keep the fastest per kernel.  Candidates run
    // under a plan override local to this thread, so the process-wide table
    // (and other threads) never see a transient pick; it changes only once,
    // at the end, to the winners.  The caller's own profiling state is set
    // aside meanwhile.  A candidate whose timing fails counts as +inf.
    const bool prof_saved = g_prof;
    std::vector<ProfEntry> list_saved;
    list_saved.swap(g_prof_list);
    float best_ms[3] = {INFINITY, INFINITY, INFINITY};
    for (int c = 0; c < n && s == NA_OK; ++c) {
      const na::PlanChoice pick{c, c, c};
      na::set_plan_override(&pick);
      for (int it = 0; it < 3 && s == NA_OK; ++it) {
        g_prof = it > 0;  // first pass warms up
        s = na_fwd(p, q, k, v, o, lse, stream);
        if (s == NA_OK)
          s = na_bwd(p, q, k, v, o, d_o, lse, dq, dk, dv, workspace, workspace_bytes, stream);
      }
      na::set_plan_override(nullptr);
      g_prof = false;
      float sum[3] = {0.f, 0.f, 0.f};
      bool ok[3] = {true, true, true};
      for (ProfEntry& e : g_prof_list) {
        float t = 0.f;
        const bool good = cudaEventSynchronize(e.b) == cudaSuccess && cudaEventElapsedTime(&t, e.a, e.b) == cudaSuccess;
        const int slot = e.id == na::KID_FWD_TC ? 0 : e.id == na::KID_DKDV_TC ? 1 : e.id == na::KID_DQ_TC ? 2 : -1;
        if (slot >= 0) {
          sum[slot] += t;
          ok[slot] = ok[slot] && good;
        }
        cudaEventDestroy(e.a);
        cudaEventDestroy(e.b);
      }
      g_prof_list.clear();
      for (int i = 0; i < 3; ++i)
        if (ok[i] && sum[i] > 0.f && sum[i] < best_ms[i]) {
          best_ms[i] = sum[i];
          best[i] = c;
        }
    }
    g_prof = prof_saved;
    g_prof_list.swap(list_saved);
    if (s != NA_OK) return s;  // the table still holds the previous picks
    s = na_set_plan_choice(p, best);
    if (s != NA_OK) return s;
  }
  if (choice_out) {
    for (int i = 0; i < 3; ++i) choice_out[i] = best[i];
  }
  g_last_error.clear();
  return NA_OK;
}

const char* na_status_string(na_status s) {
  switch (s) {
    case NA_OK: return "ok";
    case NA_ERR_NULL: return "null pointer";
    case NA_ERR_RANK: return "rank not in {1,2,3}";
    case NA_ERR_SHAPE: return "bad shape";
    case NA_ERR_BAD_KERNEL: return "kernel_size < 1";
    case NA_ERR_EVEN_WINDOW: return "even kernel_size on a non-causal axis";
    case NA_ERR_BAD_DILATION: return "dilation < 1";
    case NA_ERR_WINDOW_EXCEEDS: return "kernel_size * dilation exceeds extent";
    case NA_ERR_DTYPE: return "unsupported dtype";
    case NA_ERR_HEAD_DIM: return "unsupported head_dim";
    case NA_ERR_ALIGNMENT: return "misaligned pointer";
    case NA_ERR_LAYOUT: return "unsupported layout";
    case NA_ERR_WORKSPACE: return "workspace too small";
    case NA_ERR_CUDA: return "CUDA error";
    case NA_ERR_IMPL: return "requested kernel family cannot run this problem";
  }
  return "unknown status";
}

const char* na_last_error(void) { return g_last_error.c_str(); }

int na_last_launch_count(void) { return g_last_launches; }

}  // extern "C"
