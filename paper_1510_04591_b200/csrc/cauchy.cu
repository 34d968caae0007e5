// Cauchy-like eigenvector matrix C_ij = zhat_i v_j / (d_i - lam_j), generated on the fly.
//
// Reference path (pkg/src/hsseig/cauchy.py):
//   block / entry           cauchy.py:44-56   -> cauchy_block_kernel
//   multiply                cauchy.py:70-84   -> sample_kernel<TRANS=false> (Y = C Omega)
//   transpose_multiply      cauchy.py:86-100  -> sample_kernel<TRANS=true>  (Z = C^T Omega)
//   update_vectors_dense    dc.py:132-138     -> dense_update_kernel (Q C, C never stored)
//
// The sampling kernels generate a BM x BK tile of C (or C^T) into shared memory and
// contract it with the staged Omega chunk on FP64 DMMA.  K is split across
// blockIdx.y; partial tiles go to a workspace and are summed in a fixed order so
// the result is deterministic run to run (the reference's determinism-in-seed
// contract, pkg/tests/test_hss.py:192-200).
#include "dmma_gemm.cuh"

namespace hsseig {

__global__ void cauchy_block_kernel(CauchyGen g, const int64_t* __restrict__ rows, int64_t nr,
                                    const int64_t* __restrict__ cols, int64_t nc,
                                    double* __restrict__ out, int64_t ldo) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nr * nc) return;
  int64_t a = e / nc, b = e % nc;
  out[a * ldo + b] = g.entry(rows[a], cols[b]);
}

template <class T, bool TRANS>
__global__ void __launch_bounds__(T::THREADS) sample_kernel(CauchyGen g,
                                                            const double* __restrict__ om,
                                                            int64_t ldom, int w,
                                                            double* __restrict__ part,
                                                            int64_t ldp, int64_t kchunk) {
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / T::WN, wn = warp % T::WN;
  const int64_t k = g.k;
  const int64_t m0 = (int64_t)blockIdx.x * T::BM;
  const int64_t kbeg = (int64_t)blockIdx.y * kchunk;
  const int64_t kend = min(k, kbeg + kchunk);
  const int nch = (int)((kend - kbeg + T::BK - 1) / T::BK);
  Acc<T> acc;
  acc.zero();

  auto stage_a = [&](int s) { return smem + s * T::STAGE_ELEMS; };
  auto stage_b = [&](int s) { return smem + s * T::STAGE_ELEMS + T::A_ELEMS; };
  auto produce = [&](int c, int s) {
    const int64_t k0 = kbeg + (int64_t)c * T::BK;
    // Omega rows [k0, k0+BK) (async)
    load_b_async<T>(stage_b(s), om + k0 * ldom, ldom, 1, (int)imin64(T::BK, kend - k0), 0, w,
                    0, tid);
    cp_async_commit();
    // C tile (computed): A[r][c] = C[m0+r][k0+c]  or  C[k0+c][m0+r] for C^T
    double* sA = stage_a(s);
    for (int e = tid; e < T::BM * T::BK; e += T::THREADS) {
      int r = e / T::BK, cc = e % T::BK;
      int64_t row = m0 + r, col = k0 + cc;
      double val = 0.0;
      if (row < k && col < kend) val = TRANS ? g.entry(col, row) : g.entry(row, col);
      sA[r * T::SA + cc] = val;
    }
  };

  produce(0, 0);
  for (int c = 0; c < nch; ++c) {
    const int s = c & 1;
    if (c + 1 < nch) {
      produce(c + 1, s ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    mma_chunk<T>(stage_a(s), stage_b(s), acc, wm, wn, lane);
    __syncthreads();
  }
  store_acc<T>(acc, part + (int64_t)blockIdx.y * k * ldp, ldp, k, m0, w, 0, wm, wn, lane);
}

// out[row][col] = sum_s part[s][row][col], s ascending (fixed order)
__global__ void splitk_reduce_kernel(const double* __restrict__ part, int nsplit, int64_t k, int w,
                                     int64_t ldp, double* __restrict__ out, int64_t ldo) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= k * w) return;
  int64_t row = e / w;
  int col = (int)(e % w);
  double s = 0.0;
  for (int t = 0; t < nsplit; ++t) s += part[(int64_t)t * k * ldp + row * ldp + col];
  out[row * ldo + col] = s;
}

// out = Qb @ C with B-operand tiles of C generated in shared memory.
template <class T>
__global__ void __launch_bounds__(T::THREADS) dense_update_kernel(const double* __restrict__ Q,
                                                                  int64_t ldq, int64_t P,
                                                                  CauchyGen g,
                                                                  double* __restrict__ out,
                                                                  int64_t ldo) {
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / T::WN, wn = warp % T::WN;
  const int64_t k = g.k;
  const int64_t m0 = (int64_t)blockIdx.x * T::BM;
  const int64_t n0 = (int64_t)blockIdx.y * T::BN;
  const int nch = (int)((k + T::BK - 1) / T::BK);
  Acc<T> acc;
  acc.zero();
  auto stage_a = [&](int s) { return smem + s * T::STAGE_ELEMS; };
  auto stage_b = [&](int s) { return smem + s * T::STAGE_ELEMS + T::A_ELEMS; };
  auto produce = [&](int c, int s) {
    const int64_t k0 = (int64_t)c * T::BK;
    load_a_async<T>(stage_a(s), Q + k0, ldq, P, m0, (int)imin64(T::BK, k - k0), 0, tid);
    cp_async_commit();
    double* sB = stage_b(s);
    for (int e = tid; e < T::BK * T::BN; e += T::THREADS) {
      int r = e / T::BN, cc = e % T::BN;
      int64_t row = k0 + r, col = n0 + cc;
      sB[r * T::SB + cc] = (row < k && col < k) ? g.entry(row, col) : 0.0;
    }
  };
  produce(0, 0);
  for (int c = 0; c < nch; ++c) {
    const int s = c & 1;
    if (c + 1 < nch) {
      produce(c + 1, s ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    mma_chunk<T>(stage_a(s), stage_b(s), acc, wm, wn, lane);
    __syncthreads();
  }
  store_acc<T>(acc, out + n0, ldo, P, m0, (int)imin64(T::BN, k - n0), 0, wm, wn, lane);
}

template <class T>
static int launch_sample(const CauchyGen& g, const double* om, int64_t ldom, int w, double* Y,
                         double* Z, int64_t ldy, double* work, cudaStream_t s) {
  const int64_t k = g.k;
  const int64_t tiles = (k + T::BM - 1) / T::BM;
  const int64_t ldp = ((w + 1) / 2) * 2;
  // split K so that each of the two passes fills ~8 CTAs per SM
  int64_t nsplit = (148 * 8 + tiles - 1) / tiles;
  nsplit = imax64(1, imin64(nsplit, (k + 255) / 256));
  int64_t kchunk = (k + nsplit - 1) / nsplit;
  kchunk = ((kchunk + T::BK - 1) / T::BK) * T::BK;
  nsplit = (k + kchunk - 1) / kchunk;
  const size_t smem = sizeof(double) * T::STAGE_ELEMS * 2;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(sample_kernel<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(sample_kernel<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  dim3 grid((unsigned)tiles, (unsigned)nsplit);
  double* pY = work;
  double* pZ = work + nsplit * k * ldp;
  sample_kernel<T, false><<<grid, T::THREADS, smem, s>>>(g, om, ldom, w, pY, ldp, kchunk);
  HSS_CHECK_LAUNCH();
  sample_kernel<T, true><<<grid, T::THREADS, smem, s>>>(g, om, ldom, w, pZ, ldp, kchunk);
  HSS_CHECK_LAUNCH();
  unsigned rb = (unsigned)((k * w + 255) / 256);
  splitk_reduce_kernel<<<rb, 256, 0, s>>>(pY, (int)nsplit, k, w, ldp, Y, ldy);
  HSS_CHECK_LAUNCH();
  splitk_reduce_kernel<<<rb, 256, 0, s>>>(pZ, (int)nsplit, k, w, ldp, Z, ldy);
  HSS_CHECK_LAUNCH();
  return HSSEIG_OK;
}

}  // namespace hsseig

using namespace hsseig;

static CauchyGen to_gen(const hsseig_gen* g) {
  CauchyGen c;
  c.d = g->d;
  c.dnext = g->dnext;
  c.gam = g->gamma;
  c.mu = g->mu;
  c.zhat = g->zhat;
  c.v = g->v;
  c.k = g->k;
  return c;
}

extern "C" int hsseig_cauchy_block(const hsseig_gen* gen, const int64_t* rows, int64_t nr,
                                   const int64_t* cols, int64_t nc, double* out, int64_t ldo,
                                   void* stream) {
  if (!gen || nr < 0 || nc < 0 || ldo < nc) return HSSEIG_ERR_ARG;
  if (nr == 0 || nc == 0) return HSSEIG_OK;
  int64_t n = nr * nc;
  cauchy_block_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      to_gen(gen), rows, nr, cols, nc, out, ldo);
  HSS_CHECK_LAUNCH();
  return HSSEIG_OK;
}

extern "C" int64_t hsseig_sample_work_doubles(int64_t k, int64_t w) {
  // upper bound: nsplit <= 148*8 / tiles + 1 with tiles = ceil(k/128); two passes
  int64_t tiles = (k + 127) / 128;
  int64_t nsplit = (148 * 8 + tiles - 1) / tiles;
  nsplit = nsplit < 1 ? 1 : nsplit;
  int64_t cap = (k + 255) / 256;
  if (nsplit > cap) nsplit = cap;
  if (nsplit < 1) nsplit = 1;
  int64_t ldp = ((w + 1) / 2) * 2;
  return 2 * (nsplit + 1) * k * ldp;
}

extern "C" int hsseig_cauchy_sample(const hsseig_gen* gen, const double* omega, int64_t ldom,
                                    int64_t w, double* Y, double* Z, int64_t ldy, double* work,
                                    void* stream) {
  if (!gen || w < 1 || w > 112 || ldom < w || ldy < w) return HSSEIG_ERR_ARG;
  CauchyGen g = to_gen(gen);
  cudaStream_t s = (cudaStream_t)stream;
  switch ((w + 15) / 16) {
    case 1: return launch_sample<Tile<4, 1, 4, 2, 2>>(g, omega, ldom, (int)w, Y, Z, ldy, work, s);
    case 2: return launch_sample<Tile<4, 2, 4, 2, 2>>(g, omega, ldom, (int)w, Y, Z, ldy, work, s);
    case 3: return launch_sample<Tile<4, 3, 4, 2, 2>>(g, omega, ldom, (int)w, Y, Z, ldy, work, s);
    case 4: return launch_sample<Tile<4, 4, 4, 2, 2>>(g, omega, ldom, (int)w, Y, Z, ldy, work, s);
    case 5: return launch_sample<Tile<4, 5, 4, 2, 2>>(g, omega, ldom, (int)w, Y, Z, ldy, work, s);
    case 6: return launch_sample<Tile<4, 6, 4, 2, 2>>(g, omega, ldom, (int)w, Y, Z, ldy, work, s);
    default: return launch_sample<Tile<4, 7, 4, 2, 2>>(g, omega, ldom, (int)w, Y, Z, ldy, work, s);
  }
}

extern "C" int hsseig_dense_update(const double* Qb, int64_t ldq, int64_t P, const hsseig_gen* gen,
                                   double* out, int64_t ldo, void* stream) {
  if (!gen || P < 0 || ldq < gen->k || ldo < gen->k) return HSSEIG_ERR_ARG;
  if (P == 0) return HSSEIG_OK;
  using T = Tile<4, 8, 4, 2, 2>;
  const size_t smem = sizeof(double) * T::STAGE_ELEMS * 2;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(dense_update_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  dim3 grid((unsigned)((P + T::BM - 1) / T::BM), (unsigned)((gen->k + T::BN - 1) / T::BN));
  dense_update_kernel<T><<<grid, T::THREADS, smem, (cudaStream_t)stream>>>(Qb, ldq, P, to_gen(gen),
                                                                           out, ldo);
  HSS_CHECK_LAUNCH();
  return HSSEIG_OK;
}
