// Divide-and-conquer glue around the merge path:
//   * batched base-case QL on the leaves of the recursion     (_kernels.pyx:352-411, dc.py:118-129)
//   * host deflation of the merged rank-one system            (secular.py:91-156)
//   * device assembly of blockdiag(Q1, Q2) permuted to [kept | deflated], the deflation
//     Givens rotations, and the final eigenvalue-order column gather (dc.py:215-257)
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <numeric>
#include <thread>
#include <vector>

#include <unistd.h>

#include "common.cuh"

namespace hsseig {

namespace {
struct UploadSlot {
  char* host = nullptr;
  size_t cap = 0;
  cudaEvent_t done = nullptr;
};
std::mutex g_upload_mu;
UploadSlot g_upload_ring[32];
int g_upload_next = 0;
}  // namespace

bool upload_async(int nparts, void* const* dst, const void* const* src, const size_t* bytes,
                  cudaStream_t s) {
  size_t total = 0;
  for (int i = 0; i < nparts; ++i) total += (bytes[i] + 15) & ~size_t(15);
  std::lock_guard<std::mutex> g(g_upload_mu);
  UploadSlot& sl = g_upload_ring[g_upload_next];
  g_upload_next = (g_upload_next + 1) % 32;
  if (sl.done) {
    if (cudaEventSynchronize(sl.done) != cudaSuccess) return false;   // normally long done
  } else if (cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming) != cudaSuccess) {
    return false;
  }
  if (sl.cap < total) {
    if (sl.host) cudaFreeHost(sl.host);
    sl.cap = std::max<size_t>(total, 1 << 16);
    if (cudaHostAlloc(reinterpret_cast<void**>(&sl.host), sl.cap, cudaHostAllocDefault) != cudaSuccess) {
      sl.host = nullptr;
      sl.cap = 0;
      return false;
    }
  }
  size_t off = 0;
  for (int i = 0; i < nparts; ++i) {
    if (bytes[i]) {
      std::memcpy(sl.host + off, src[i], bytes[i]);
      if (cudaMemcpyAsync(dst[i], sl.host + off, bytes[i], cudaMemcpyHostToDevice, s) != cudaSuccess)
        return false;
    }
    off += (bytes[i] + 15) & ~size_t(15);
  }
  return cudaEventRecord(sl.done, s) == cudaSuccess;
}

// ---------------------------------------------------------------------------
// batched implicit QL with Wilkinson shift (tql2, _kernels.pyx:352-411).  A group of GROUP
// threads owns one tridiagonal of order <= NMAX: a warp per matrix (4 per block) for the
// usual base cases (n <= 32), a whole 128-thread block for base sizes up to kQLBig.  Thread
// t owns rows t, t + GROUP, ... of the rotation accumulator.  Scalar recurrences run
// redundantly in every thread on shared d/e (identical values, so every branch is uniform
// across the group), rounding kept IEEE (no FMA contraction) like the reference's C loop.
// flags: kQLInit = Q holds the initial accumulator (the kernel contract's in/out Z),
//        kQLUnsorted = leave d / Z in QL order (the contract); default = ascending stable
//        sort of dc.py:127 with the identity as the initial accumulator.
// ---------------------------------------------------------------------------
constexpr int kQLMax = 32;
constexpr int kQLBig = 160;
constexpr int kQLInit = 1, kQLUnsorted = 2;

template <int NMAX, int GROUP>
__device__ __forceinline__ void ql_sync() {
  if (GROUP == 32) __syncwarp(); else __syncthreads();
}

template <int NMAX, int GROUP>
__global__ void tql2_batched_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                    const int64_t* __restrict__ off, int64_t nmat, int max_iter,
                                    double* __restrict__ lam, double* __restrict__ Q,
                                    const int64_t* __restrict__ qoff, int32_t* __restrict__ status,
                                    int flags) {
  constexpr int PER = 128 / GROUP;            // matrices per block
  extern __shared__ double ql_smem[];
  const int wl = threadIdx.x / GROUP, lane = threadIdx.x % GROUP;
  const int64_t m = (int64_t)blockIdx.x * PER + wl;
  if (m >= nmat) return;                      // uniform over the group
  double* d = ql_smem + (size_t)wl * (NMAX + NMAX + 1 + NMAX * (NMAX + 1));
  double* e = d + NMAX;
  double* Z = e + NMAX + 1;                   // Z[row * (NMAX + 1) + col]
  constexpr int LDZ = NMAX + 1;
  const int64_t o = off[m];
  const int n = (int)(off[m + 1] - o);
  double* q = Q + qoff[m];
  for (int r = lane; r < n; r += GROUP) {
    d[r] = a[o + r];
    e[r] = (r + 1 < n) ? b[o - m + r] : 0.0;   // b has n-1 entries per matrix
    for (int c = 0; c < n; ++c)
      Z[r * LDZ + c] = (flags & kQLInit) ? q[(int64_t)r * n + c] : ((r == c) ? 1.0 : 0.0);
  }
  ql_sync<NMAX, GROUP>();
  int fail = 0;
  if (n > 1) {
    for (int l = 0; l < n && !fail; ++l) {
      int it = 0;
      for (;;) {
        int mm = l;
        for (; mm < n - 1; ++mm) {
          const double dd = __dadd_rn(fabs(d[mm]), fabs(d[mm + 1]));
          if (fabs(e[mm]) <= __dmul_rn(kEps, dd)) break;
        }
        if (mm == l) break;
        if (++it > max_iter) { fail = 1 + l; break; }
        double g = __ddiv_rn(__dsub_rn(d[l + 1], d[l]), __dmul_rn(2.0, e[l]));
        double r = hypot(g, 1.0);
        g = __dadd_rn(__dsub_rn(d[mm], d[l]), __ddiv_rn(e[l], __dadd_rn(g, copysign(r, g))));
        double s = 1.0, c = 1.0, p = 0.0;
        bool clean = true;
        for (int i = mm - 1; i >= l; --i) {
          const double f = __dmul_rn(s, e[i]);
          const double bb = __dmul_rn(c, e[i]);
          r = hypot(f, g);
          ql_sync<NMAX, GROUP>();
          if (lane == 0) e[i + 1] = r;
          ql_sync<NMAX, GROUP>();
          if (r == 0.0) {
            if (lane == 0) {
              d[i + 1] = __dsub_rn(d[i + 1], p);
              e[mm] = 0.0;
            }
            ql_sync<NMAX, GROUP>();
            clean = false;
            break;
          }
          s = __ddiv_rn(f, r);
          c = __ddiv_rn(g, r);
          g = __dsub_rn(d[i + 1], p);
          r = __dadd_rn(__dmul_rn(__dsub_rn(d[i], g), s), __dmul_rn(__dmul_rn(2.0, c), bb));
          p = __dmul_rn(s, r);
          ql_sync<NMAX, GROUP>();
          if (lane == 0) d[i + 1] = __dadd_rn(g, p);
          g = __dsub_rn(__dmul_rn(c, r), bb);
          for (int row = lane; row < n; row += GROUP) {
            double* zr = Z + row * LDZ;
            const double zi = zr[i], zi1 = zr[i + 1];
            zr[i + 1] = __dadd_rn(__dmul_rn(s, zi), __dmul_rn(c, zi1));
            zr[i] = __dsub_rn(__dmul_rn(c, zi), __dmul_rn(s, zi1));
          }
          ql_sync<NMAX, GROUP>();
        }
        if (clean) {
          ql_sync<NMAX, GROUP>();
          if (lane == 0) {
            d[l] = __dsub_rn(d[l], p);
            e[l] = g;
            e[mm] = 0.0;
          }
          ql_sync<NMAX, GROUP>();
        }
      }
    }
  }
  ql_sync<NMAX, GROUP>();
  // ascending order, stable (np.argsort kind="stable", dc.py:127), unless the caller sorts
  for (int col = lane; col < n; col += GROUP) {
    const double v = d[col];
    int pos = col;
    if (!(flags & kQLUnsorted)) {
      pos = 0;
      for (int j = 0; j < n; ++j) pos += (d[j] < v) || (d[j] == v && j < col);
    }
    lam[o + pos] = v;
    for (int row = 0; row < n; ++row) q[(int64_t)row * n + pos] = Z[row * LDZ + col];
  }
  if (lane == 0 && fail) status[m] = fail;
}

template <int NMAX, int GROUP>
static int launch_tql2(const double* a, const double* b, const int64_t* off, int64_t nmat,
                       int max_iter, double* lam, double* Q, const int64_t* qoff, int32_t* status,
                       int flags, cudaStream_t s) {
  constexpr int PER = 128 / GROUP;
  const size_t smem = sizeof(double) * PER * (size_t)(2 * NMAX + 1 + NMAX * (NMAX + 1));
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute(tql2_batched_kernel<NMAX, GROUP>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return HSSEIG_ERR_CUDA;
  tql2_batched_kernel<NMAX, GROUP><<<(unsigned)((nmat + PER - 1) / PER), 128, smem, s>>>(
      a, b, off, nmat, max_iter, lam, Q, qoff, status, flags);
  HSS_CHECK_LAUNCH();
  return HSSEIG_OK;
}

// W[:, c] = blockdiag(Q1, Q2)[:, src[c]] for c < n, W row-major (ldw)
__global__ void assemble_kernel(const double* __restrict__ Q1, int64_t n1, const double* __restrict__ Q2,
                                int64_t n2, const int64_t* __restrict__ src, double* __restrict__ W,
                                int64_t ldw) {
  const int64_t n = n1 + n2;
  for (int64_t row = blockIdx.y; row < n; row += gridDim.y)   // gridDim.y <= 65535
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n;
         c += (int64_t)gridDim.x * blockDim.x) {
      const int64_t sc = src[c];
      double v = 0.0;
      if (row < n1) { if (sc < n1) v = Q1[row * n1 + sc]; }
      else if (sc >= n1) v = Q2[(row - n1) * n2 + (sc - n1)];
      W[row * ldw + c] = v;
    }
}

// deflation Givens rotations on column pairs, in order, every row independently
// (dc.py:225-230: col_a = c*a + s*b, col_b = -s*a + c*b, no FMA contraction)
__global__ void rotate_kernel(double* __restrict__ W, int64_t ldw, int64_t rows,
                              const int64_t* __restrict__ ca, const int64_t* __restrict__ cb,
                              const double* __restrict__ cs, const double* __restrict__ sn,
                              int64_t nrot) {
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= rows) return;
  double* w = W + row * ldw;
  for (int64_t t = 0; t < nrot; ++t) {
    const int64_t ia = ca[t], ib = cb[t];
    const double c = cs[t], s = sn[t];
    const double x = w[ia], y = w[ib];
    w[ia] = __dadd_rn(__dmul_rn(c, x), __dmul_rn(s, y));
    w[ib] = __dadd_rn(__dmul_rn(-s, x), __dmul_rn(c, y));
  }
}

// out[:, c] = (src[c] < k ? A[:, src[c]] : B[:, src[c]])  (final eigenvalue order)
__global__ void gather2_kernel(const double* __restrict__ A, int64_t lda, const double* __restrict__ B,
                               int64_t ldb, int64_t k, const int64_t* __restrict__ src, int64_t ncol,
                               int64_t nrow, double* __restrict__ out, int64_t ldo) {
  for (int64_t row = blockIdx.y; row < nrow; row += gridDim.y)   // gridDim.y <= 65535
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < ncol;
         c += (int64_t)gridDim.x * blockDim.x) {
      const int64_t sc = src[c];
      out[row * ldo + c] = sc < k ? A[row * lda + sc] : B[row * ldb + sc];
    }
}

// ---------------------------------------------------------------------------
// Level-batched ("wave") glue: every merge of one recursion depth per launch.  Merge m
// has children blocks Q1 (n1 x n1) and Q2 (n2 x n2) at arbitrary device addresses, its
// rows occupy [roff[m], roff[m+1]) of the concatenated row space and its n x n merge
// block sits at W + woff[m] with rows padded to an even leading dimension n + (n & 1) (16-byte
// aligned rows for the TMA update engine); row_merge maps a concatenated row to its merge.
// ---------------------------------------------------------------------------
__global__ void wave_zrows_kernel(const unsigned long long* __restrict__ q1,
                                  const unsigned long long* __restrict__ q2,
                                  const int64_t* __restrict__ n1, const int64_t* __restrict__ n2,
                                  const int64_t* __restrict__ roff, double* __restrict__ zrow) {
  const int m = blockIdx.x;
  const int64_t a = n1[m], b = n2[m];
  const double* Q1 = reinterpret_cast<const double*>(q1[m]);
  const double* Q2 = reinterpret_cast<const double*>(q2[m]);
  double* z = zrow + roff[m];
  for (int64_t c = threadIdx.x; c < a + b; c += blockDim.x)
    z[c] = c < a ? Q1[(a - 1) * a + c] : Q2[c - a];   // last row of Q1, first row of Q2
}

// W_m holds only the columns the update and the rotations need (the kept ones first, then
// the deflated columns a rotation touches): n x wd[m], leading dimension wd + (wd & 1);
// csrc[coff[m] + j] is the blockdiag column of compact column j.
__global__ void wave_assemble_kernel(const unsigned long long* __restrict__ q1,
                                     const unsigned long long* __restrict__ q2,
                                     const int64_t* __restrict__ n1, const int64_t* __restrict__ n2,
                                     const int64_t* __restrict__ roff,
                                     const int32_t* __restrict__ row_merge,
                                     const int64_t* __restrict__ csrc, const int64_t* __restrict__ coff,
                                     const int64_t* __restrict__ wd, double* __restrict__ W,
                                     const int64_t* __restrict__ woff, int64_t nrows) {
  for (int64_t gr = blockIdx.x; gr < nrows; gr += gridDim.x) {
    const int m = row_merge[gr];
    const int64_t a = n1[m], b = n2[m], row = gr - roff[m], nc = wd[m];
    const double* Q1 = reinterpret_cast<const double*>(q1[m]);
    const double* Q2 = reinterpret_cast<const double*>(q2[m]);
    const int64_t* sm = csrc + coff[m];
    double* w = W + woff[m] + row * (nc + (nc & 1));
    for (int64_t c = threadIdx.x; c < nc; c += blockDim.x) {
      const int64_t sc = sm[c];
      double v = 0.0;
      if (row < a) { if (sc < a) v = Q1[row * a + sc]; }
      else if (sc >= a) v = Q2[(row - a) * b + (sc - a)];
      w[c] = v;
    }
  }
}

// Deflation rotations (dc.py:225-230: col_a = c*a + s*b, col_b = -s*a + c*b, no FMA
// contraction), split into runs: deflation's pair t is (survivor, deflated) (secular.py:
// 96-156); a survivor holds for a contiguous run of rotations and is never deflated later,
// and each deflated column appears once, so different runs touch disjoint columns.  Every
// (row, run) pair is an independent task -- consecutive threads take consecutive runs of
// one row (neighbouring columns) -- and a run carries its survivor in a register.
__global__ void wave_rotate_kernel(double* __restrict__ W, const int64_t* __restrict__ woff,
                                   const int64_t* __restrict__ nn, const int64_t* __restrict__ wd,
                                   const int64_t* __restrict__ run_t,
                                   const int64_t* __restrict__ run_off,
                                   const int64_t* __restrict__ ca, const int64_t* __restrict__ cb,
                                   const double* __restrict__ cs, const double* __restrict__ sn) {
  const int m = blockIdx.y;
  const int64_t q0 = run_off[m], nr = run_off[m + 1] - q0;
  if (nr <= 0) return;
  const int64_t n = nn[m], ld = wd[m] + (wd[m] & 1), ntask = n * nr;
  for (int64_t task = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; task < ntask;
       task += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = task / nr, r = task - row * nr;
    const int64_t t0 = __ldg(run_t + q0 + r), t1 = __ldg(run_t + q0 + r + 1);
    double* w = W + woff[m] + row * ld;
    const int64_t ia = __ldg(ca + t0);
    double xa = w[ia];
    for (int64_t t = t0; t < t1; ++t) {
      const int64_t ib = __ldg(cb + t);
      const double c = __ldg(cs + t), s = __ldg(sn + t);
      const double y = w[ib];
      const double na = __dadd_rn(__dmul_rn(c, xa), __dmul_rn(s, y));
      w[ib] = __dadd_rn(__dmul_rn(-s, xa), __dmul_rn(c, y));
      xa = na;
    }
    w[ia] = xa;
  }
}

// out_m[:, c] from the column descriptor desc[c] = (source << 40) | index: source 0 = Qk_m
// column (an updated eigenvector), 1 = compact W_m column (a rotated deflated column), 2 =
// blockdiag(Q1, Q2) column read straight from the children (an untouched deflated column).
struct GatherSrc {
  const double* Qk;
  const int64_t *qoff, *kept;
  const double* W;
  const int64_t *woff, *wd, *desc;
  const unsigned long long *q1, *q2;
  const int64_t *n1, *n2, *roff;
};

// Row `row` of merge m's output in eigenvalue order, written to o (n doubles).
__device__ __forceinline__ void gather_row(const GatherSrc& g, int m, int64_t row, double* o) {
  constexpr int64_t kMask = (1ll << 40) - 1;
  const int64_t a = g.n1[m], b = g.n2[m], n = a + b, k = g.kept[m];
  const int64_t* dm = g.desc + g.roff[m];
  const double* q = g.Qk + g.qoff[m] + row * k;
  const double* w = g.W + g.woff[m] + row * (g.wd[m] + (g.wd[m] & 1));
  // this row's half of blockdiag(Q1, Q2): child columns [c0, c0 + nc)
  const bool top = row < a;
  const double* qc = top ? reinterpret_cast<const double*>(g.q1[m]) + row * a
                         : reinterpret_cast<const double*>(g.q2[m]) + (row - a) * b;
  const int64_t c0 = top ? 0 : a, nc = top ? a : b;
  for (int64_t c = threadIdx.x; c < n; c += blockDim.x) {
    const int64_t dsc = dm[c];
    const int64_t src = dsc >> 40, idx = dsc & kMask;
    double v;
    if (src == 0) v = q[idx];
    else if (src == 1) v = w[idx];
    else v = (idx >= c0 && idx < c0 + nc) ? qc[idx - c0] : 0.0;
    o[c] = v;
  }
}

// resident blocks per SM the gather is compiled for: 4 (64 registers, no spills) measured
// against 5 / 6 / 8 (48 / 40 / 32 registers with 8 / 48 / 80 bytes of spills): config-5
// gathers 20.2 ms against 21.1 / 25.2 / 30.0 ms
#ifndef HSSEIG_GATHER_MINB
#define HSSEIG_GATHER_MINB 4
#endif
// ROWS rows per block and CPT columns per thread and iteration: rows of one merge share the
// column descriptors, so the descriptor array (8 B per output entry) is read once per ROWS
// rows, and a thread keeps ROWS * CPT independent source loads in flight and stores
// 16 bytes at a time when the output rows are 16-byte aligned (n even).  Groups that
// straddle a merge boundary fall back to row by row.
template <int ROWS, int CPT>
__global__ void __launch_bounds__(256, HSSEIG_GATHER_MINB)
    wave_gather_kernel(GatherSrc g, const int32_t* __restrict__ row_merge,
                       double* __restrict__ out, const int64_t* __restrict__ ooff, int64_t nrows) {
  static_assert(CPT % 2 == 0, "columns per thread come in 16-byte pairs");
  constexpr int64_t kMask = (1ll << 40) - 1;
  const int64_t ngroups = (nrows + ROWS - 1) / ROWS;
  for (int64_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
    const int64_t gr0 = grp * ROWS;
    const int m = row_merge[gr0];
    const bool whole = gr0 + ROWS <= nrows && row_merge[gr0 + ROWS - 1] == m;
    if (!whole) {
      for (int64_t gr = gr0; gr < min(gr0 + (int64_t)ROWS, nrows); ++gr) {
        const int mm = row_merge[gr];
        const int64_t row = gr - g.roff[mm], n = g.n1[mm] + g.n2[mm];
        gather_row(g, mm, row, out + ooff[mm] + row * n);
      }
      continue;
    }
    const int64_t a = g.n1[m], b = g.n2[m], n = a + b, k = g.kept[m];
    const int64_t row0 = gr0 - g.roff[m], ldw = g.wd[m] + (g.wd[m] & 1);
    const int64_t* dm = g.desc + g.roff[m];
    const double* q[ROWS];
    const double* w[ROWS];
    const double* qc[ROWS];
    int64_t c0[ROWS], nc[ROWS];
    double* o[ROWS];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
      const int64_t row = row0 + r;
      q[r] = g.Qk + g.qoff[m] + row * k;
      w[r] = g.W + g.woff[m] + row * ldw;
      const bool top = row < a;
      qc[r] = top ? reinterpret_cast<const double*>(g.q1[m]) + row * a
                  : reinterpret_cast<const double*>(g.q2[m]) + (row - a) * b;
      c0[r] = top ? 0 : a;
      nc[r] = top ? a : b;
      o[r] = out + ooff[m] + row * n;
    }
    const bool vec = (n & 1) == 0 && (reinterpret_cast<uintptr_t>(o[0]) & 15) == 0;
    for (int64_t c = CPT * (int64_t)threadIdx.x; c < n; c += CPT * (int64_t)blockDim.x) {
      int64_t src[CPT], idx[CPT];
#pragma unroll
      for (int u = 0; u < CPT; ++u) {
        const int64_t dsc = dm[c + u < n ? c + u : n - 1];
        src[u] = dsc >> 40;
        idx[u] = dsc & kMask;
      }
      double v[ROWS][CPT];
#pragma unroll
      for (int r = 0; r < ROWS; ++r)
#pragma unroll
        for (int u = 0; u < CPT; ++u) {
          if (src[u] == 0) v[r][u] = q[r][idx[u]];
          else if (src[u] == 1) v[r][u] = w[r][idx[u]];
          else v[r][u] = (idx[u] >= c0[r] && idx[u] < c0[r] + nc[r]) ? qc[r][idx[u] - c0[r]] : 0.0;
        }
      if (vec) {   // n even: column pairs never straddle the end of a row
#pragma unroll
        for (int r = 0; r < ROWS; ++r)
#pragma unroll
          for (int u = 0; u < CPT; u += 2)
            if (c + u < n) *reinterpret_cast<double2*>(o[r] + c + u) = make_double2(v[r][u], v[r][u + 1]);
      } else {
#pragma unroll
        for (int r = 0; r < ROWS; ++r)
#pragma unroll
          for (int u = 0; u < CPT; ++u)
            if (c + u < n) o[r][c + u] = v[r][u];
      }
    }
  }
}

// Selected rows only (the boundary rows the next depth's z needs, before the full gather).
__global__ void wave_gather_rows_kernel(GatherSrc g, const int32_t* __restrict__ sel_merge,
                                        const int64_t* __restrict__ sel_row,
                                        const int64_t* __restrict__ sel_off, int64_t nsel,
                                        double* __restrict__ out) {
  for (int64_t i = blockIdx.x; i < nsel; i += gridDim.x)
    gather_row(g, sel_merge[i], sel_row[i], out + sel_off[i]);
}

// One rank's row block of W = blockdiag(Q1, Q2)[:, src] when its rows all come from one
// child: W[i][c] = Qc[i][src[c] - coff] if that column belongs to the child, else 0.
__global__ void assemble_rows_kernel(const double* __restrict__ Qc, int64_t ldq, int64_t nrow,
                                     int64_t coff, int64_t nc, const int64_t* __restrict__ src,
                                     int64_t n, double* __restrict__ W, int64_t ldw) {
  for (int64_t row = blockIdx.y; row < nrow; row += gridDim.y)
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n;
         c += (int64_t)gridDim.x * blockDim.x) {
      const int64_t sc = src[c] - coff;
      W[row * ldw + c] = (sc >= 0 && sc < nc) ? Qc[row * ldq + sc] : 0.0;
    }
}


}  // namespace hsseig

using namespace hsseig;

extern "C" int hsseig_tql2_batched(const double* a, const double* b, const int64_t* off,
                                   int64_t nmat, int nmax, int max_iter, double* lam, double* Q,
                                   const int64_t* qoff, int32_t* status, int flags, void* stream) {
  if (nmat < 0 || !a || !off || !lam || !Q || !qoff || !status || nmax < 0 || nmax > kQLBig ||
      (flags & ~(kQLInit | kQLUnsorted)))
    HSS_ARG_FAIL();
  if (nmat == 0) return HSSEIG_OK;
  if (nmax <= kQLMax)
    return launch_tql2<kQLMax, 32>(a, b, off, nmat, max_iter, lam, Q, qoff, status, flags,
                                   (cudaStream_t)stream);
  return launch_tql2<kQLBig, 128>(a, b, off, nmat, max_iter, lam, Q, qoff, status, flags,
                                  (cudaStream_t)stream);
}

extern "C" int hsseig_assemble_merge(const double* Q1, int64_t n1, const double* Q2, int64_t n2,
                                     const int64_t* src, double* W, int64_t ldw, void* stream) {
  const int64_t n = n1 + n2;
  if (n <= 0 || ldw < n || n > 0x7fffffff) HSS_ARG_FAIL();
  dim3 grid((unsigned)std::min<int64_t>((n + 255) / 256, 64), (unsigned)std::min<int64_t>(n, 65535));
  assemble_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(Q1, n1, Q2, n2, src, W, ldw);
  HSS_CHECK_LAUNCH();
  return HSSEIG_OK;
}

extern "C" int hsseig_apply_rotations(double* W, int64_t ldw, int64_t rows, const int64_t* ca,
                                      const int64_t* cb, const double* c, const double* s,
                                      int64_t nrot, void* stream) {
  if (rows < 0 || nrot < 0) HSS_ARG_FAIL();
  if (nrot == 0 || rows == 0) return HSSEIG_OK;
  rotate_kernel<<<(unsigned)((rows + 127) / 128), 128, 0, (cudaStream_t)stream>>>(W, ldw, rows, ca,
                                                                                  cb, c, s, nrot);
  HSS_CHECK_LAUNCH();
  return HSSEIG_OK;
}

extern "C" int hsseig_gather_columns(const double* A, int64_t lda, const double* B, int64_t ldb,
                                     int64_t k, const int64_t* src, int64_t ncol, int64_t rows,
                                     double* out, int64_t ldo, void* stream) {
  if (rows < 0 || ncol < 0 || rows > 0x7fffffff) HSS_ARG_FAIL();
  if (rows == 0 || ncol == 0) return HSSEIG_OK;
  dim3 grid((unsigned)std::min<int64_t>((ncol + 255) / 256, 64), (unsigned)std::min<int64_t>(rows, 65535));
  gather2_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(A, lda, B, ldb, k, src, ncol, rows, out,
                                                         ldo);
  HSS_CHECK_LAUNCH();
  return HSSEIG_OK;
}

/*
 * Host deflation (secular.py:91-156), restated: negligible weights deflate at their pole,
 * pole pairs closer than tol are merged by a Givens rotation that zeroes one weight.
 * Inputs d, z (n), rho.  Outputs: d_out/z_out with the kept system first (k entries,
 * sorted poles) followed by the deflated poles (ascending); perm[n] = sorted-input index
 * of each output slot; rotations (ri, rj, rc, rs; n_rot <= n) in sorted-input indices.
 * Returns k.
 */
extern "C" int64_t hsseig_deflate_tol(const double* d, const double* z, int64_t n, double rho,
                                      double tol, double* d_out, double* z_out, int64_t* perm,
                                      int64_t* ri, int64_t* rj, double* rc, double* rs,
                                      int64_t* n_rot);

// sum of z[t]^2 in NumPy's order: np.sum(z * z) (secular.py:92) reduces a contiguous float64
// array with pairwise_sum (blocks of <= 128 in 8 accumulators, halves split at multiples of 8),
// so a merge sitting exactly on a deflation threshold keeps the reference's decision
static double numpy_sum_sq(const double* z, int64_t n) {
  if (n < 8) {
    double r = -0.0;
    for (int64_t i = 0; i < n; ++i) r += z[i] * z[i];
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = z[j] * z[j];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += z[i + j] * z[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += z[i] * z[i];
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return numpy_sum_sq(z, n2) + numpy_sum_sq(z + n2, n - n2);
}

extern "C" int64_t hsseig_deflate(const double* d, const double* z, int64_t n, double rho,
                                  double* d_out, double* z_out, int64_t* perm, int64_t* ri,
                                  int64_t* rj, double* rc, double* rs, int64_t* n_rot,
                                  double* tol_out) {
  if (n < 1) return -1;
  double dmax = 0.0;
  for (int64_t t = 0; t < n; ++t) dmax = std::max(dmax, std::fabs(d[t]));
  const double zz = numpy_sum_sq(z, n);
  const double tol = 8.0 * kEps * std::max(dmax, rho * zz);   // secular.py:91-93
  if (tol_out) *tol_out = tol;
  return hsseig_deflate_tol(d, z, n, rho, tol, d_out, z_out, perm, ri, rj, rc, rs, n_rot);
}

extern "C" int64_t hsseig_deflate_tol(const double* d, const double* z, int64_t n, double rho,
                                      double tol, double* d_out, double* z_out, int64_t* perm,
                                      int64_t* ri, int64_t* rj, double* rc, double* rs,
                                      int64_t* n_rot) {
  if (n < 1) return -1;
  std::vector<int64_t> order(n);
  std::iota(order.begin(), order.end(), 0);
  if (!std::is_sorted(d, d + n))   // callers usually pass sorted poles: stable order is identity
    std::stable_sort(order.begin(), order.end(), [&](int64_t x, int64_t y) { return d[x] < d[y]; });
  std::vector<double> ds(n), zs(n);
  for (int64_t t = 0; t < n; ++t) { ds[t] = d[order[t]]; zs[t] = z[order[t]]; }
  std::vector<char> keep(n, 1);
  int64_t surv = -1, nr = 0;
  for (int64_t t = 0; t < n; ++t) {
    if (rho * std::fabs(zs[t]) <= tol) { keep[t] = 0; continue; }
    if (surv >= 0 && ds[t] - ds[surv] <= tol) {
      const double h = std::hypot(zs[surv], zs[t]);
      const double c = zs[surv] / h, s = zs[t] / h;
      zs[surv] = h;
      zs[t] = 0.0;
      const double dp = ds[surv], dt = ds[t];
      ds[surv] = c * c * dp + s * s * dt;
      ds[t] = s * s * dp + c * c * dt;
      ri[nr] = order[surv]; rj[nr] = order[t]; rc[nr] = c; rs[nr] = s; ++nr;
      keep[t] = 0;
    } else {
      surv = t;
    }
  }
  std::vector<int64_t> kept, defl;
  for (int64_t t = 0; t < n; ++t) (keep[t] ? kept : defl).push_back(t);
  if (!std::is_sorted(defl.begin(), defl.end(), [&](int64_t x, int64_t y) { return ds[x] < ds[y]; }))
    std::stable_sort(defl.begin(), defl.end(), [&](int64_t x, int64_t y) { return ds[x] < ds[y]; });
  int64_t q = 0;
  for (int64_t t : kept) { d_out[q] = ds[t]; z_out[q] = zs[t]; perm[q] = order[t]; ++q; }
  for (int64_t t : defl) { d_out[q] = ds[t]; z_out[q] = zs[t]; perm[q] = order[t]; ++q; }
  *n_rot = nr;
  return (int64_t)kept.size();
}

// ---------------------------------------------------------------------------- wave ABI
static unsigned rows_grid(int64_t nrows) { return (unsigned)std::min<int64_t>(nrows, 1 << 20); }

extern "C" int hsseig_wave_zrows(const uint64_t* q1, const uint64_t* q2, const int64_t* n1,
                                 const int64_t* n2, const int64_t* roff, int64_t nm, double* zrow,
                                 void* stream) {
  if (nm < 0 || !q1 || !q2 || !n1 || !n2 || !roff || !zrow) HSS_ARG_FAIL();
  if (nm == 0) return HSSEIG_OK;
  wave_zrows_kernel<<<(unsigned)nm, 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const unsigned long long*>(q1), reinterpret_cast<const unsigned long long*>(q2),
      n1, n2, roff, zrow);
  HSS_CHECK_LAUNCH();
  return HSSEIG_OK;
}

extern "C" int hsseig_wave_assemble(const uint64_t* q1, const uint64_t* q2, const int64_t* n1,
                                    const int64_t* n2, const int64_t* roff, const int32_t* row_merge,
                                    const int64_t* csrc, const int64_t* coff, const int64_t* wd,
                                    double* W, const int64_t* woff, int64_t nrows, void* stream) {
  if (nrows < 0 || !q1 || !q2 || !n1 || !n2 || !roff || !row_merge || !csrc || !coff || !wd || !W ||
      !woff)
    HSS_ARG_FAIL();
  if (nrows == 0) return HSSEIG_OK;
  wave_assemble_kernel<<<rows_grid(nrows), 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const unsigned long long*>(q1), reinterpret_cast<const unsigned long long*>(q2),
      n1, n2, roff, row_merge, csrc, coff, wd, W, woff, nrows);
  HSS_CHECK_LAUNCH();
  return HSSEIG_OK;
}

extern "C" int hsseig_wave_rotate(double* W, const int64_t* woff, const int64_t* n,
                                  const int64_t* wd, const int64_t* run_t, const int64_t* run_off,
                                  const int64_t* ca, const int64_t* cb, const double* c,
                                  const double* s, int64_t nm, int64_t max_tasks, void* stream) {
  if (nm < 0 || max_tasks < 0 || nm > 65535 || !W || !run_t || !run_off) HSS_ARG_FAIL();
  if (nm == 0 || max_tasks == 0) return HSSEIG_OK;
  dim3 grid((unsigned)std::min<int64_t>((max_tasks + 255) / 256, 8192), (unsigned)nm);
  wave_rotate_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(W, woff, n, wd, run_t, run_off, ca, cb,
                                                             c, s);
  HSS_CHECK_LAUNCH();
  return HSSEIG_OK;
}

extern "C" int hsseig_wave_gather(const double* Qk, const int64_t* qoff, const int64_t* kept,
                                  const double* W, const int64_t* woff, const int64_t* wd,
                                  const int64_t* desc, const uint64_t* q1, const uint64_t* q2,
                                  const int64_t* n1, const int64_t* n2, const int64_t* roff,
                                  const int32_t* row_merge, double* out, const int64_t* ooff,
                                  int64_t nrows, void* stream) {
  if (nrows < 0 || !W || !woff || !wd || !desc || !q1 || !q2 || !n1 || !n2 || !roff ||
      !row_merge || !out || !ooff || !kept || !qoff)
    HSS_ARG_FAIL();
  if (nrows == 0) return HSSEIG_OK;
  GatherSrc g{Qk ? Qk : W, qoff, kept, W, woff, wd, desc,
              reinterpret_cast<const unsigned long long*>(q1),
              reinterpret_cast<const unsigned long long*>(q2), n1, n2, roff};
  // shape swept at config 5 (rows x columns per thread: 4x2, 4x4, 8x2, 2x4, 1x4, 1x8, 3x4):
  // 2 x 4 -- a full 32-byte sector per thread and row -- moves the top-level gather's 51.9 GB
  // at 5.66 TB/s (87% of the measured copy bandwidth)
  wave_gather_kernel<2, 4><<<rows_grid((nrows + 1) / 2), 256, 0, (cudaStream_t)stream>>>(
      g, row_merge, out, ooff, nrows);
  HSS_CHECK_LAUNCH();
  return HSSEIG_OK;
}

extern "C" int hsseig_wave_gather_rows(const double* Qk, const int64_t* qoff, const int64_t* kept,
                                       const double* W, const int64_t* woff, const int64_t* wd,
                                       const int64_t* desc, const uint64_t* q1, const uint64_t* q2,
                                       const int64_t* n1, const int64_t* n2, const int64_t* roff,
                                       const int32_t* sel_merge, const int64_t* sel_row,
                                       const int64_t* sel_off, int64_t nsel, double* out,
                                       void* stream) {
  if (nsel < 0 || !W || !woff || !wd || !desc || !q1 || !q2 || !n1 || !n2 || !roff || !kept ||
      !qoff || !sel_merge || !sel_row || !sel_off || !out)
    HSS_ARG_FAIL();
  if (nsel == 0) return HSSEIG_OK;
  GatherSrc g{Qk ? Qk : W, qoff, kept, W, woff, wd, desc,
              reinterpret_cast<const unsigned long long*>(q1),
              reinterpret_cast<const unsigned long long*>(q2), n1, n2, roff};
  wave_gather_rows_kernel<<<rows_grid(nsel), 256, 0, (cudaStream_t)stream>>>(
      g, sel_merge, sel_row, sel_off, nsel, out);
  HSS_CHECK_LAUNCH();
  return HSSEIG_OK;
}

/*
 * Host side of one depth of merges (dc.py:205-235 for every merge m of the depth):
 * z from the boundary rows (theta = sign(b), 1/sqrt(2)), joint stable sort of [L1 L2],
 * deflation (hsseig_deflate), the blockdiag column of every W slot (src, local) and the
 * Givens rotations as W-column pairs.  rho == 0 merges (exactly decoupled) keep nothing
 * and only sort.  Arrays over merges: n1, n2, bk, kept, rho_eff, rot_off (nm + 1);
 * concatenated over rows (roff): L, zrow, d_out, z_out, src; rotations: ca, cb, rc, rs
 * (capacity roff[nm]).  Returns the total number of kept roots.
 */
// Stable argsort of key[0..n) made of two ascending runs [0, split) and [split, n) (children's
// eigenvalues, or roots followed by deflated poles): a stable merge, O(n); a full stable
// sort when a run is not sorted.  Equal keys keep their original order, as np.argsort(kind=
// "stable") does.
static void stable_argsort_runs(const double* key, int64_t split, int64_t n, int64_t* out) {
  std::vector<int64_t> idx(n);
  std::iota(idx.begin(), idx.end(), 0);
  auto lt = [&](int64_t x, int64_t y) { return key[x] < key[y]; };
  if (std::is_sorted(key, key + split) && std::is_sorted(key + split, key + n)) {
    std::merge(idx.begin(), idx.begin() + split, idx.begin() + split, idx.end(), out, lt);
  } else {
    std::stable_sort(idx.begin(), idx.end(), lt);
    std::copy(idx.begin(), idx.end(), out);
  }
}

// The merges of one level are independent: the host-side passes over them (deflation,
// final order, descriptors) run on a persistent worker pool once a level carries enough rows
// to pay for it.  (Spawning std::threads per call cost 0.3-0.5 ms of each of the three passes
// of every recursion depth -- a quarter of the host time of the deep, small-merge depths.)
namespace {
class MergePool {
 public:
  // f runs on the caller and on nt - 1 workers
  void run(int nt, const std::function<void()>& f) {
    std::lock_guard<std::mutex> one(run_mu_);
    if (pid_ != getpid()) {   // a forked child starts without the parent's workers
      workers_ = 0;
      pid_ = getpid();
    }
    for (; workers_ < nt - 1; ++workers_) std::thread(&MergePool::worker, this, workers_).detach();
    {
      std::lock_guard<std::mutex> g(mu_);
      job_ = &f;
      want_ = nt - 1;
      running_ = nt - 1;
      ++gen_;
    }
    start_.notify_all();
    f();
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [&] { return running_ == 0; });
    job_ = nullptr;
  }

 private:
  void worker(int id) {
    uint64_t seen = 0;
    for (;;) {
      std::unique_lock<std::mutex> lk(mu_);
      start_.wait(lk, [&] { return gen_ != seen; });
      seen = gen_;
      if (id >= want_) continue;
      const std::function<void()>* j = job_;
      lk.unlock();
      (*j)();
      lk.lock();
      if (--running_ == 0) done_.notify_one();
    }
  }
  std::mutex run_mu_, mu_;
  std::condition_variable start_, done_;
  const std::function<void()>* job_ = nullptr;
  uint64_t gen_ = 0;
  int want_ = 0, running_ = 0, workers_ = 0;
  pid_t pid_ = 0;
};
MergePool& merge_pool() {
  static MergePool* p = new MergePool;   // never destroyed: its workers outlive static teardown
  return *p;
}
}  // namespace

template <class F>
static void for_each_merge(int64_t nm, const int64_t* roff, F&& f) {
  const int64_t rows = roff[nm] - roff[0];
  const int64_t hw = std::max<int64_t>(1, std::min<unsigned>(std::thread::hardware_concurrency(), 32u));
  const int64_t nt = std::min<int64_t>({hw, nm, rows / 4096 + 1});
  if (nt <= 1) {
    for (int64_t m = 0; m < nm; ++m) f(m);
    return;
  }
  const int64_t chunk = std::max<int64_t>(1, nm / (nt * 8));
  std::atomic<int64_t> next{0};
  const std::function<void()> work = [&] {
    for (int64_t m0; (m0 = next.fetch_add(chunk)) < nm;)
      for (int64_t m = m0; m < std::min(nm, m0 + chunk); ++m) f(m);
  };
  merge_pool().run((int)nt, work);
}

extern "C" int64_t hsseig_wave_deflate(int64_t nm, const int64_t* n1, const int64_t* n2,
                                       const int64_t* roff, const double* L, const double* zrow,
                                       const double* bk, int64_t* kept, double* rho_eff,
                                       double* d_out, double* z_out, int64_t* src, int64_t* rot_off,
                                       int64_t* ca, int64_t* cb, double* rc, double* rs) {
  // pass 1 (parallel): merge m leaves its rotations at its own row offset of ca/cb/rc/rs
  std::vector<int64_t> nrot(nm, 0);
  for_each_merge(nm, roff, [&](int64_t m) {
    thread_local std::vector<int64_t> perm, dperm, ri, rj, posW;
    thread_local std::vector<double> ds, zs, z;
    const int64_t a = n1[m], n = a + n2[m], o = roff[m], r0 = o - roff[0];
    const double* Lm = L + o;
    perm.resize(n);
    stable_argsort_runs(Lm, a, n, perm.data());
    const double b = bk[m];
    const double rho = std::fabs(b);
    if (rho == 0.0) {   // dc.py:206-213: decoupled halves, merge by sorting only
      kept[m] = 0;
      rho_eff[m] = 0.0;
      for (int64_t t = 0; t < n; ++t) { d_out[o + t] = Lm[perm[t]]; z_out[o + t] = 0.0; src[o + t] = perm[t]; }
      return;
    }
    const double theta = b >= 0.0 ? 1.0 : -1.0;
    z.resize(n);
    for (int64_t t = 0; t < n; ++t) {
      double zr = zrow[o + t];
      if (t >= a) zr *= theta;
      z[t] = zr / std::sqrt(2.0);
    }
    ds.resize(n); zs.resize(n);
    for (int64_t t = 0; t < n; ++t) { ds[t] = Lm[perm[t]]; zs[t] = z[perm[t]]; }
    dperm.resize(n); ri.resize(n); rj.resize(n);
    int64_t nr = 0;
    const int64_t k = hsseig_deflate(ds.data(), zs.data(), n, 2.0 * rho, d_out + o, z_out + o,
                                     dperm.data(), ri.data(), rj.data(), rc + r0, rs + r0, &nr,
                                     nullptr);
    kept[m] = k;
    rho_eff[m] = 2.0 * rho;
    posW.resize(n);
    for (int64_t t = 0; t < n; ++t) {
      src[o + t] = perm[dperm[t]];
      posW[perm[dperm[t]]] = t;
    }
    for (int64_t t = 0; t < nr; ++t) {
      ca[r0 + t] = posW[perm[ri[t]]];
      cb[r0 + t] = posW[perm[rj[t]]];
    }
    nrot[m] = nr;
  });
  // pass 2: pack the rotations (a merge's packed offset never passes its row offset, so
  // forward moves in merge order are safe)
  int64_t ktot = 0, nrot_tot = 0;
  rot_off[0] = 0;
  for (int64_t m = 0; m < nm; ++m) {
    const int64_t r0 = roff[m] - roff[0], nr = nrot[m];
    if (nr && r0 != nrot_tot) {
      std::memmove(ca + nrot_tot, ca + r0, nr * sizeof(int64_t));
      std::memmove(cb + nrot_tot, cb + r0, nr * sizeof(int64_t));
      std::memmove(rc + nrot_tot, rc + r0, nr * sizeof(double));
      std::memmove(rs + nrot_tot, rs + r0, nr * sizeof(double));
    }
    nrot_tot += nr;
    rot_off[m + 1] = nrot_tot;
    ktot += kept[m];
  }
  return ktot;
}

/*
 * Final order of every merge (dc.py:253-257): lam_cat = [roots, deflated poles], stable
 * argsort.  lam (concatenated kept roots, koff) and d_out (rows) in; order / lam_out
 * (rows) out.
 */
extern "C" int hsseig_wave_order(int64_t nm, const int64_t* roff, const int64_t* kept,
                                 const int64_t* koff, const double* lam, const double* d_out,
                                 int64_t* order, double* lam_out) {
  for_each_merge(nm, roff, [&](int64_t m) {
    thread_local std::vector<double> cat;
    const int64_t o = roff[m], n = roff[m + 1] - o, k = kept[m];
    cat.resize(n);
    for (int64_t t = 0; t < n; ++t) cat[t] = t < k ? lam[koff[m] + t] : d_out[o + t];
    int64_t* ord = order + o;
    stable_argsort_runs(cat.data(), k, n, ord);
    for (int64_t t = 0; t < n; ++t) lam_out[o + t] = cat[ord[t]];
  });
  return HSSEIG_OK;
}

extern "C" int hsseig_wave_desc(int64_t nm, const int64_t* roff, const int64_t* kept,
                                const int64_t* order, const int64_t* cmap, const int64_t* src,
                                int64_t* desc) {
  for_each_merge(nm, roff, [&](int64_t m) {
    const int64_t o = roff[m], n = roff[m + 1] - o, k = kept[m];
    for (int64_t t = 0; t < n; ++t) {
      const int64_t p = order[o + t];
      const int64_t cm = cmap[o + p];
      desc[o + t] = p < k ? p : (cm >= 0 ? ((1ll << 40) | cm) : ((2ll << 40) | src[o + p]));
    }
  });
  return HSSEIG_OK;
}

extern "C" int hsseig_assemble_rows(const double* Qc, int64_t ldq, int64_t nrow, int64_t coff,
                                    int64_t nc, const int64_t* src, int64_t n, double* W,
                                    int64_t ldw, void* stream) {
  if (nrow < 0 || n < 0 || nc < 0 || ldw < n || (nrow > 0 && (!Qc || !src || !W))) HSS_ARG_FAIL();
  if (nrow == 0 || n == 0) return HSSEIG_OK;
  dim3 grid((unsigned)std::min<int64_t>((n + 255) / 256, 64), (unsigned)std::min<int64_t>(nrow, 65535));
  assemble_rows_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(Qc, ldq, nrow, coff, nc, src, n, W, ldw);
  HSS_CHECK_LAUNCH();
  return HSSEIG_OK;
}

/*
 * Compact W layout of one depth of merges: merge m materialises only its kept positions
 * [0, k_m) and the deflated positions some rotation touches (ascending), wd[m] columns.
 * csrc (at coff[m]) = blockdiag column of each compact column; cmap (rows layout, roff) =
 * compact column of each W position or -1; the rotation column pairs ca / cb are rewritten
 * in place to compact indices.  Returns the total compact width.
 */
extern "C" int64_t hsseig_wave_compact(int64_t nm, const int64_t* roff, const int64_t* kept,
                                       const int64_t* src, const int64_t* rot_off, int64_t* ca,
                                       int64_t* cb, int64_t* wd, int64_t* coff, int64_t* csrc,
                                       int64_t* cmap) {
  int64_t tot = 0;
  coff[0] = 0;
  for (int64_t m = 0; m < nm; ++m) {
    const int64_t o = roff[m], n = roff[m + 1] - o, k = kept[m];
    int64_t* cm = cmap + o;
    for (int64_t p = 0; p < n; ++p) cm[p] = p < k ? p : -1;
    for (int64_t t = rot_off[m]; t < rot_off[m + 1]; ++t) {
      if (ca[t] >= k) cm[ca[t]] = -2;
      if (cb[t] >= k) cm[cb[t]] = -2;
    }
    int64_t nc = k;
    for (int64_t p = k; p < n; ++p)
      if (cm[p] == -2) cm[p] = nc++;
    for (int64_t p = 0; p < n; ++p)
      if (cm[p] >= 0) csrc[tot + cm[p]] = src[o + p];
    for (int64_t t = rot_off[m]; t < rot_off[m + 1]; ++t) {
      ca[t] = cm[ca[t]];
      cb[t] = cm[cb[t]];
    }
    wd[m] = nc;
    tot += nc;
    coff[m + 1] = tot;
  }
  return tot;
}
