// fw1d.cu -- host entry points of the batched 1-D OT oracle and Frank-Wolfe
// kernels (kernels in fw1d_kernel.cuh; the pairwise instantiation is built in
// fw1d_pfw.cu) and the dense feasibility check.
#include <algorithm>

#include "fw1d_kernel.cuh"

namespace uot {
namespace {
using namespace fwk;

// Dense feasibility max(0, max_ij f_i + g_j - C_ij): duality.py:117-121.
__global__ void feasibility_kernel(int n, int m, const double* x, const double* y, double p,
                                   const double* C, const double* f, const double* g,
                                   double* out) {
  __shared__ double scr[32];
  const int b = blockIdx.y;
  double worst = -CUDART_INF;
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < (long)n * m;
       t += (long)gridDim.x * blockDim.x) {
    const int i = (int)(t / m), j = (int)(t % m);
    const double c = C != nullptr ? C[(long)b * n * m + t]
                                  : pcost(x[(long)b * n + i], y[(long)b * m + j], p);
    const double v = f[(long)b * n + i] + g[(long)b * m + j] - c;
    worst = fmax(worst, v);
  }
  worst = block_reduce(worst, scr, MaxOp(), -CUDART_INF);
  if (threadIdx.x == 0) {
    // max over blocks via the integer ordering of non-negative doubles
    const double v = fmax(worst, 0.0);
    atomicMax(reinterpret_cast<unsigned long long*>(out + b), __double_as_longlong(v));
  }
}


// Plan-extraction scratch (vals [batch][n+m] doubles, codes [batch][n+m][2]
// ints), then -- for problems on the large path (fwk::fw_big) -- the
// per-problem arrays the resident path keeps in shared memory.
size_t fw_scratch_core(int batch, int n, int m) {
  return ((sizeof(double) + 2 * sizeof(int)) * (size_t)batch * (n + m) + 255) / 256 * 256;
}
size_t fw_scratch_bytes(int batch, int n, int m) {
  size_t b = fw_scratch_core(batch, n, m) + 256;
  if (fwk::fw_big(n, m)) b += (size_t)batch * fwk::fw_big_stride(n, m);
  return b;
}
char* fw_big_region(void* scratch, int batch, int n, int m) {
  return fwk::fw_big(n, m) ? (char*)scratch + fw_scratch_core(batch, n, m) : nullptr;
}

int launch_fw(const FwArgs& a0, int batch, cudaStream_t st) {
  FwArgs a = a0;
  if (a.big == nullptr) a.big = fw_big_region(a.scratch, batch, a.n, a.m);
  if (a.mode == 0 && a.step == UOT_STEP_PAIRWISE) return launch_fw_pairwise(a, batch, st);
  return launch_fw_impl<false>(a, batch, st);
}

// pairwise atom store: atoms [batch][cap][n+m] doubles; beyond PFW_CAP_S slots
// also the slot weights [batch][cap] (doubles) and the active list [batch][cap]
// (ints), which otherwise live in shared memory; cap = max_iters + 1
size_t pfw_store_bytes(int batch, int n, int m, int max_iters) {
  const size_t cap = (size_t)max_iters + 1;
  return sizeof(double) * (size_t)batch * cap * (n + m) +
         (3 * sizeof(double) + sizeof(int)) * (size_t)batch * cap + 1024;
}

bool generic_entropies(const uot_fw_desc* d) {
  return d->ent1 != UOT_ENT_KL || d->ent2 != UOT_ENT_KL;
}

size_t fw_ws_bytes(const uot_fw_desc* d) {
  if (generic_entropies(d)) return fwk::generic_ws_bytes(d->batch, d->n, d->m);
  size_t b = fw_scratch_bytes(d->batch, d->n, d->m);
  if (d->step == UOT_STEP_PAIRWISE) b += pfw_store_bytes(d->batch, d->n, d->m, d->max_iters);
  return b;
}

}  // namespace

namespace fwk {
int launch_fw_ot(const FwArgs& a, int batch, cudaStream_t st) { return launch_fw(a, batch, st); }
size_t ot_scratch_bytes(int batch, int n, int m) { return fw_scratch_bytes(batch, n, m); }
}  // namespace fwk
}  // namespace uot

using namespace uot;

extern "C" int uot_fw1d_workspace_size(const uot_fw_desc* d, size_t* bytes) {
  if (d == nullptr || d->batch < 1 || d->n < 1 || d->m < 1) {
    set_error("uot_fw1d_workspace_size: invalid descriptor");
    return UOT_INVALID;
  }
  *bytes = fw_ws_bytes(d);
  return UOT_OK;
}

extern "C" int uot_fw1d_run(const uot_fw_desc* d, void* ws, size_t ws_bytes, void* stream) {
  if (d == nullptr || d->batch < 1 || d->n < 1 || d->m < 1 || d->max_iters < 1) {
    set_error("uot_fw1d_run: invalid descriptor");
    return UOT_INVALID;
  }
  if (!(d->rho1 > 0) || !(d->rho2 > 0) || (d->c == nullptr && !(d->p >= 1.0))) {
    set_error("uot_fw1d_run: need rho > 0 and p >= 1 (or an explicit cost c)");
    return UOT_INVALID;
  }
  if (d->step != UOT_STEP_HARMONIC && d->step != UOT_STEP_LINESEARCH &&
      d->step != UOT_STEP_PAIRWISE) {
    set_error("uot_fw1d_run: step must be harmonic, linesearch or pairwise");
    return UOT_INVALID;
  }
  const bool gen = generic_entropies(d);
  if (gen) {  // fw.py:98-103: KL or Berg on each side
    if ((d->ent1 != UOT_ENT_KL && d->ent1 != UOT_ENT_BERG) ||
        (d->ent2 != UOT_ENT_KL && d->ent2 != UOT_ENT_BERG)) {
      set_error("frank-wolfe needs strictly convex conjugates (KL or Berg)");
      return UOT_UNSUPPORTED_ENTROPY;
    }
    if (d->step == UOT_STEP_PAIRWISE) {
      set_error("uot_fw1d_run: pairwise FW runs KL/KL penalties on the B200 path");
      return UOT_UNSUPPORTED_ENTROPY;
    }
  }
  if (ws_bytes < fw_ws_bytes(d)) {
    set_error("uot_fw1d_run: workspace too small");
    return UOT_INVALID;
  }
  FwArgs a{};
  a.n = d->n;
  a.m = d->m;
  a.p = d->p;
  a.r1 = d->rho1;
  a.r2 = d->rho2;
  a.step = d->step;
  a.max_iters = d->max_iters;
  a.gap_tol = d->gap_tol;
  a.early_exit = d->early_exit;
  a.mode = 0;
  a.x = d->x;
  a.y = d->y;
  a.a = d->a;
  a.b = d->b;
  a.f = d->f;
  a.g = d->g;
  a.h0 = d->h0;
  a.fw_gap = d->fw_gap;
  a.pd_gap = d->pd_gap;
  a.iterations = d->iterations;
  a.ei = d->ei;
  a.ej = d->ej;
  a.em = d->em;
  a.count = d->count;
  a.summary = d->summary;
  a.status = d->status;
  a.step_size = d->step_size;
  a.scratch = (double*)ws;
  a.scratch_i = (int*)((char*)ws + sizeof(double) * (size_t)d->batch * (d->n + d->m));
  a.natoms = d->natoms;
  a.ref_f = d->ref_f;
  a.err_f = d->err_f;
  a.C = d->c;
  a.step_in = d->step_in;
  a.away_in = d->away_in;
  a.supp_hash = reinterpret_cast<unsigned long long*>(d->supp_hash);
  a.supp_nnz = d->supp_nnz;
  if ((a.supp_hash == nullptr) != (a.supp_nnz == nullptr)) {
    set_error("uot_fw1d_run: supp_hash and supp_nnz go together");
    return UOT_INVALID;
  }
  if (gen && (a.step_in != nullptr || a.supp_hash != nullptr)) {
    set_error("uot_fw1d_run: the replay / support-trace mode runs KL/KL penalties");
    return UOT_INVALID;
  }
  if (a.away_in != nullptr && (d->step != UOT_STEP_PAIRWISE || a.step_in == nullptr)) {
    set_error("uot_fw1d_run: away_in replays pairwise steps together with step_in");
    return UOT_INVALID;
  }
  if (gen) return fwk::run_fw_generic(a, d->batch, d->ent1, d->ent2, ws, ws_bytes,
                                     (cudaStream_t)stream);
  if (d->step == UOT_STEP_PAIRWISE) {
    const size_t cap = (size_t)d->max_iters + 1;
    const size_t bc = (size_t)d->batch * cap;
    char* p = (char*)ws + (fw_scratch_bytes(d->batch, d->n, d->m) + 255) / 256 * 256;
    a.cap = (int)cap;
    a.atoms = (double*)p;
    p += sizeof(double) * bc * (d->n + d->m);
    a.wts = (double*)p;
    a.act = (int*)(a.wts + bc);
  }
  return launch_fw(a, d->batch, (cudaStream_t)stream);
}

extern "C" int uot_ot1d_workspace_size(int32_t batch, int32_t n, int32_t m, size_t* bytes) {
  if (batch < 1 || n < 1 || m < 1) {
    set_error("uot_ot1d_workspace_size: invalid sizes");
    return UOT_INVALID;
  }
  *bytes = fw_scratch_bytes(batch, n, m);
  return UOT_OK;
}

extern "C" int uot_ot1d_batched(int32_t batch, int32_t n, int32_t m, const double* x,
                                const double* y, const double* a, const double* b, int32_t cost,
                                double p, const double* c, double* f, double* g, int32_t* ei,
                                int32_t* ej, double* em, int32_t* count, int32_t* status,
                                void* workspace, size_t workspace_bytes, void* stream) {
  if (batch < 1 || n < 1 || m < 1 || (cost == UOT_COST_POWER && !(p >= 1.0))) {
    set_error("uot_ot1d_batched: invalid arguments");
    return UOT_INVALID;
  }
  if (cost != UOT_COST_POWER && !(cost == UOT_COST_EXPLICIT && c != nullptr)) {
    set_error("uot_ot1d_batched: cost must be UOT_COST_POWER or UOT_COST_EXPLICIT with c");
    return UOT_INVALID;
  }
  if (workspace_bytes < fw_scratch_bytes(batch, n, m)) {
    set_error("uot_ot1d_batched: workspace too small");
    return UOT_INVALID;
  }
  FwArgs A{};
  A.n = n;
  A.m = m;
  A.p = p;
  A.mode = 1;
  A.x = x;
  A.y = y;
  A.a = a;
  A.b = b;
  A.f = f;
  A.g = g;
  A.ei = ei;
  A.ej = ej;
  A.em = em;
  A.count = count;
  A.status = status;
  A.C = cost == UOT_COST_EXPLICIT ? c : nullptr;
  A.scratch = (double*)workspace;
  A.scratch_i = (int*)((char*)workspace + sizeof(double) * (size_t)batch * (n + m));
  return launch_fw(A, batch, (cudaStream_t)stream);
}

extern "C" int uot_feasibility_1d(int32_t batch, int32_t n, int32_t m, const double* x,
                                  const double* y, double p, const double* f, const double* g,
                                  double* out, void* stream) {
  if (batch < 1 || n < 1 || m < 1) {
    set_error("uot_feasibility_1d: invalid sizes");
    return UOT_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  UOT_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(double) * batch, st));
  const long nm = (long)n * m;
  const int blocks = (int)std::min<long>(1024, (nm + 255) / 256);
  feasibility_kernel<<<dim3(blocks, batch), 256, 0, st>>>(n, m, x, y, p, nullptr, f, g, out);
  UOT_CHECK_LAUNCH();
  return UOT_OK;
}

extern "C" int uot_feasibility_explicit(int32_t batch, int32_t n, int32_t m, const double* C,
                                        const double* f, const double* g, double* out,
                                        void* stream) {
  if (batch < 1 || n < 1 || m < 1 || C == nullptr) {
    set_error("uot_feasibility_explicit: invalid arguments");
    return UOT_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  UOT_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(double) * batch, st));
  const long nm = (long)n * m;
  const int blocks = (int)std::min<long>(1024, (nm + 255) / 256);
  feasibility_kernel<<<dim3(blocks, batch), 256, 0, st>>>(n, m, nullptr, nullptr, 0.0, C, f, g,
                                                          out);
  UOT_CHECK_LAUNCH();
  return UOT_OK;
}

#ifdef UOT_NEWTON_STATS
// scripts/newton_stats.py (stats build only): Newton passes / line searches
extern "C" int uot_debug_fw_stats(unsigned long long* out, int reset) {
  unsigned long long h[2];
  cudaMemcpyFromSymbol(h, uot::fwk::g_newton_stats, sizeof(h));
  out[0] = h[0];
  out[1] = h[1];
  if (reset) {
    h[0] = h[1] = 0;
    cudaMemcpyToSymbol(uot::fwk::g_newton_stats, h, sizeof(h));
  }
  return 0;
}
#endif
