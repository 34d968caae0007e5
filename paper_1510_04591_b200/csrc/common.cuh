// Shared device helpers for the sm_100a merge-step kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/hsseig_b200.h"

#include <atomic>

// Every kernel launch is followed by HSS_CHECK_LAUNCH(), which also counts it
// (hsseig_launch_count() reports the total; bench.py reports it as gpu_launches).
namespace hsseig {
extern std::atomic<long long> g_launches;
}
namespace hsseig {
void set_arg_error(const char* file, int line);
// Small host->device uploads that return without waiting: the parts are staged in a
// pinned ring slot (reused only after its copies have completed, tracked by an event).
bool upload_async(int nparts, void* const* dst, const void* const* src, const size_t* bytes,
                  cudaStream_t s);
}
// argument / configuration failure: remember where (hsseig_last_error) and return code 1
#define HSS_ARG_FAIL()                               \
  do {                                               \
    hsseig::set_arg_error(__FILE__, __LINE__);       \
    return HSSEIG_ERR_ARG;                           \
  } while (0)

#define HSS_CHECK_LAUNCH()                                       \
  do {                                                           \
    hsseig::g_launches.fetch_add(1, std::memory_order_relaxed);  \
    cudaError_t _e = cudaGetLastError();                         \
    if (_e != cudaSuccess) return HSSEIG_ERR_CUDA;               \
  } while (0)

namespace hsseig {

__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t imax64(int64_t a, int64_t b) { return a > b ? a : b; }

constexpr double kEps = 2.220446049250313e-16;

// rows of a leaf's D slot: a zero row, the m data rows, zero rows to a whole 16-deep chunk
__host__ __device__ __forceinline__ int hsseig_drows(int mmax) { return (mmax + 1 + 15) / 16 * 16 + 2; }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_prod(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v *= __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Reciprocal to ~1 ulp: MUFU seed + two Newton steps (no IEEE division sequence).
__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// Reciprocal from the MUFU seed with one cubic correction r (1 + e + e^2), e = 1 - x r:
// three FP64 operations instead of rcp_nr's four; the residual error is O(e^3), below
// double rounding for the MUFU seed (the secular / Loewner parity tests hold at 64 eps).
__device__ __forceinline__ double rcp_c3(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);
}

// Stable d_i - lam_j from the gap pair of root j (pkg/src/hsseig/secular.py:183-203):
//   i <= j : (d_i - d_j) - gamma_j        i > j : (d_i - d_{j+1}) + mu_j
// dnext_j is d_{j+1} (the virtual pole d_{k-1}+gamma_{k-1}+mu_{k-1} for j = k-1).
__device__ __forceinline__ double stable_gap(int64_t i, int64_t j, double di, double dj,
                                             double dnext_j, double gam_j, double mu_j) {
  return (i <= j) ? ((di - dj) - gam_j) : ((di - dnext_j) + mu_j);
}

// Generators of the Cauchy-like eigenvector matrix C_ij = zhat_i v_j / (d_i - lam_j)
// (pkg/src/hsseig/cauchy.py:15-56).  dnext has the virtual pole appended at k-1.
struct CauchyGen {
  const double* d;
  const double* dnext;
  const double* gam;
  const double* mu;
  const double* zhat;
  const double* v;
  int64_t k;
  // leaf id of every index (tree partition) for the off-diagonal sample, or nullptr: the
  // sampling kernels then skip the diagonal leaf blocks (C(t, t) = 0 in the product)
  const int32_t* lid = nullptr;

  __device__ __forceinline__ double entry(int64_t i, int64_t j) const {
    double g = stable_gap(i, j, __ldg(d + i), __ldg(d + j), __ldg(dnext + j), __ldg(gam + j),
                          __ldg(mu + j));
    return (__ldg(zhat + i) * __ldg(v + j)) / g;
  }
};

// ---- FP64 warp MMA (DMMA) --------------------------------------------------
// m8n8k4, A row-major fragment a = A[lane/4][lane%4], B col fragment b = B[lane%4][lane/4],
// C fragment c0,c1 = C[lane/4][2*(lane%4) + {0,1}].
__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int n = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N));
}

}  // namespace hsseig
