// abi.cu -- C-ABI plumbing: error strings, version, small batched scalar
// reductions used by the API mirror, NCCL communicator setup.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include "../../include/uot_b200.h"
#include "common.cuh"

#if defined(UOT_WITH_NCCL)
#include <nccl.h>
#endif

namespace uot {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

const char* get_error() { return g_err; }

// One block per problem: natural-domain log-sum-exps of -f/rho1 (weights a)
// and -g/rho2 (weights b), zero weights masked (src/entropies.py:77-83).
__global__ void kl_scalars_kernel(int n, int m, const double* a, const double* b, const double* f,
                                  const double* g, double r1, double r2, double* out) {
  __shared__ double sm[32], ss[32], sx[32];
  const int p = blockIdx.x;
  LsePair la{-CUDART_INF, 0.0}, lb{-CUDART_INF, 0.0};
  double ma = 0.0, mb = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double w = a[(long)p * n + i];
    ma += w;
    if (w > 0.0) la = lse_merge(la, LsePair{-f[(long)p * n + i] / r1, w});
  }
  for (int j = threadIdx.x; j < m; j += blockDim.x) {
    const double w = b[(long)p * m + j];
    mb += w;
    if (w > 0.0) lb = lse_merge(lb, LsePair{-g[(long)p * m + j] / r2, w});
  }
  la = block_lse(la, sm, ss);
  lb = block_lse(lb, sm, ss);
  ma = block_reduce(ma, sx, SumOp(), 0.0);
  mb = block_reduce(mb, sx, SumOp(), 0.0);
  if (threadIdx.x == 0) {
    const double qa = la.s > 0.0 ? la.m + log(la.s) : -CUDART_INF;
    const double qb = lb.s > 0.0 ? lb.m + log(lb.s) : -CUDART_INF;
    const double t1 = r1 / (r1 + r2), t2 = r2 / (r1 + r2);
    out[p * 3 + 0] = (r1 * r2 / (r1 + r2)) * (qa - qb);                        // duality.py:175-178
    out[p * 3 + 1] = r1 * ma + r2 * mb - (r1 + r2) * exp(t1 * qa + t2 * qb);  // duality.py:279-290
    out[p * 3 + 2] = -r1 * qa;                                                // entropies.py:187-200
  }
}

}  // namespace uot

extern "C" {

const char* uot_version(void) { return "paper_2201_00730_b200 0.1.0 (sm_100a)"; }

const char* uot_last_error(void) { return uot::get_error(); }

int uot_device_arch(int device, int* sm_major, int* sm_minor) {
  UOT_CUDA_TRY(cudaDeviceGetAttribute(sm_major, cudaDevAttrComputeCapabilityMajor, device));
  UOT_CUDA_TRY(cudaDeviceGetAttribute(sm_minor, cudaDevAttrComputeCapabilityMinor, device));
  return UOT_OK;
}

int uot_kl_scalars(int32_t batch, int32_t n, int32_t m, const double* a, const double* b,
                   const double* f, const double* g, double rho1, double rho2, double* out,
                   void* stream) {
  if (batch < 1 || n < 1 || m < 1 || !(rho1 > 0) || !(rho2 > 0)) {
    uot::set_error("uot_kl_scalars: invalid arguments");
    return uot::UOT_INVALID;
  }
  uot::kl_scalars_kernel<<<batch, 256, 0, (cudaStream_t)stream>>>(n, m, a, b, f, g, rho1, rho2,
                                                                  out);
  UOT_CHECK_LAUNCH();
  return UOT_OK;
}

int uot_nccl_unique_id(char out[128]) {
#if defined(UOT_WITH_NCCL)
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) {
    uot::set_error("ncclGetUniqueId failed");
    return uot::UOT_NCCL;
  }
  memcpy(out, id.internal, 128);
  return UOT_OK;
#else
  (void)out;
  uot::set_error("built without NCCL");
  return uot::UOT_NCCL;
#endif
}

int uot_nccl_comm_init(const char id[128], int32_t nranks, int32_t rank, void** comm) {
#if defined(UOT_WITH_NCCL)
  ncclUniqueId uid;
  memcpy(uid.internal, id, 128);
  ncclComm_t c;
  ncclResult_t r = ncclCommInitRank(&c, nranks, uid, rank);
  if (r != ncclSuccess) {
    uot::set_error("ncclCommInitRank failed: %s", ncclGetErrorString(r));
    return uot::UOT_NCCL;
  }
  *comm = (void*)c;
  return UOT_OK;
#else
  (void)id;
  (void)nranks;
  (void)rank;
  (void)comm;
  uot::set_error("built without NCCL");
  return uot::UOT_NCCL;
#endif
}

int uot_nccl_comm_destroy(void* comm) {
#if defined(UOT_WITH_NCCL)
  if (comm != nullptr) ncclCommDestroy((ncclComm_t)comm);
  return UOT_OK;
#else
  (void)comm;
  return UOT_OK;
#endif
}

}  // extern "C"
