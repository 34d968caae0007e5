// HSS x dense product from the right, out = X H (Algorithm 3), on sm_100a.
//
// Reference: hss_matmul_right (pkg/src/hsseig/hss.py:309-361).
// Every step of the algorithm is a tall-skinny contraction over the P rows of X
// with a node-local factor, so each tree level is ONE launch of a batched
// two-segment DMMA GEMM (one job per node):
//   up, leaf  : G_i = X[:, t_i] U_i
//   up, inner : G_i = [G_l | G_r] U_i
//   down      : F_i = [G_sib | F_par] [B_sib ; V_par(rows of i)^T]     (the "inherit" term)
//   final     : out[:, t_i] = [X[:, t_i] | F_i] [D_i ; V_i^T]
// Job descriptors are built on the device from the ranks the construction wrote,
// so no host synchronisation is needed between construction and multiply.
#include <cstdlib>

#include "dmma_gemm.cuh"

namespace hsseig {

struct GemmJob {
  const double* A1;
  const double* A2;
  const double* B1;
  const double* B2;
  double* C;
  int64_t lda1, lda2, b1r, b1c, b2r, b2c, ldc;
  int32_t K1, K2, N, pad;
};

// Persistent batched two-segment GEMM.  CTA c walks the (job, row-tile) list
// c, c + gridDim.x, ...; the (tile, k-chunk) sequence is one continuous cp.async
// pipeline, so the next tile's operands stream in while this tile's last chunks
// are multiplied and its accumulators are stored.
template <class T>
struct Seg {
  const double* A;
  const double* B;
  int64_t lda, ldb;
  int K;
  bool a16, b16;
};

template <class T>
__device__ __forceinline__ void job_seg(const GemmJob& jb, int c, int nc1, Seg<T>& sg, int& k0) {
  if (c < nc1) {
    sg.A = jb.A1; sg.B = jb.B1; sg.lda = jb.lda1; sg.ldb = jb.b1r; sg.K = jb.K1;
    k0 = c * T::BK;
  } else {
    sg.A = jb.A2; sg.B = jb.B2; sg.lda = jb.lda2; sg.ldb = jb.b2r; sg.K = jb.K2;
    k0 = (c - nc1) * T::BK;
  }
  sg.a16 = ((reinterpret_cast<uintptr_t>(sg.A) & 15) == 0) && ((sg.lda & 1) == 0);
  sg.b16 = ((reinterpret_cast<uintptr_t>(sg.B) & 15) == 0) && ((sg.ldb & 1) == 0);
}

template <class T>
__global__ void __launch_bounds__(T::THREADS) batched_gemm2_kernel(const GemmJob* __restrict__ jobs,
                                                                   int njobs, int64_t M,
                                                                   int tiles_m) {
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / T::WN, wn = warp % T::WN;
  const int total = njobs * tiles_m;
  auto sa = [&](int s) { return smem + s * T::STAGE_ELEMS; };
  auto sb = [&](int s) { return smem + s * T::STAGE_ELEMS + T::A_ELEMS; };

  // producer cursor
  int pt = blockIdx.x, pc = 0, pslot = 0;
  GemmJob pj;
  int pnc1 = 0, pnch = 0;
  auto load_pjob = [&]() {
    if (pt < total) {
      pj = jobs[pt / tiles_m];
      pnc1 = (pj.K1 + T::BK - 1) / T::BK;
      pnch = pj.N > 0 ? pnc1 + (pj.K2 + T::BK - 1) / T::BK : 0;
    }
  };
  load_pjob();
  auto produce = [&]() {
    while (pt < total && pc >= pnch) {  // skip empty tiles
      pt += gridDim.x;
      pc = 0;
      load_pjob();
    }
    if (pt < total) {
      Seg<T> sg;
      int k0;
      job_seg<T>(pj, pc, pnc1, sg, k0);
      const int64_t m0 = (int64_t)(pt % tiles_m) * T::BM;
      if (sg.a16) load_a_async16<T>(sa(pslot), sg.A, sg.lda, M, m0, sg.K, k0, tid);
      else load_a_async<T>(sa(pslot), sg.A, sg.lda, M, m0, sg.K, k0, tid);
      if (sg.b16) load_b_async16<T>(sb(pslot), sg.B, sg.ldb, sg.K, k0, pj.N, tid);
      else load_b_async<T>(sb(pslot), sg.B, sg.ldb, 1, sg.K, k0, pj.N, 0, tid);
      if (++pc >= pnch) {
        pt += gridDim.x;
        pc = 0;
        load_pjob();
      }
    }
    cp_async_commit();
    pslot = (pslot + 1) % T::STAGES;
  };

#pragma unroll 1
  for (int s = 0; s < T::STAGES - 1; ++s) produce();

  // consumer cursor
  int ct = blockIdx.x, cslot = 0;
  Acc<T> acc;
  while (ct < total) {
    const GemmJob cj = jobs[ct / tiles_m];
    const int nc1 = (cj.K1 + T::BK - 1) / T::BK;
    const int nch = cj.N > 0 ? nc1 + (cj.K2 + T::BK - 1) / T::BK : 0;
    if (nch == 0) { ct += gridDim.x; continue; }
    const int64_t m0 = (int64_t)(ct % tiles_m) * T::BM;
    const int jmax = max(0, min(T::NF, (cj.N - wn * T::NF * 8 + 7) / 8));
    acc.zero();
    for (int c = 0; c < nch; ++c) {
      cp_async_wait<T::STAGES - 2>();
      __syncthreads();
      produce();
      const int kseg = c < nc1 ? cj.K1 - c * T::BK : cj.K2 - (c - nc1) * T::BK;
      const int kv = min(T::BK, (kseg + 3) & ~3);
      if (kv == T::BK && jmax == T::NF)
        mma_chunk<T>(sa(cslot), sb(cslot), acc, wm, wn, lane);
      else
        mma_chunk_part<T>(sa(cslot), sb(cslot), acc, wm, wn, lane, kv, jmax);
      cslot = (cslot + 1) % T::STAGES;
    }
    store_acc<T>(acc, cj.C, cj.ldc, M, m0, cj.N, 0, wm, wn, lane);
    ct += gridDim.x;
  }
  cp_async_wait<0>();
}

struct MultPlan {
  int32_t depth, n_leaves, ws, pmax, mmax, dld;
  const int32_t *lo, *hi, *left, *right, *lnodes, *rU, *rV;
  const double *U, *V, *Vt, *B, *D;
  const double* X;
  int64_t ldx;
  double* out;
  int64_t ldo;
  double* Gb;  // levels 1..depth, level l at Gb + P*ws*(2^l - 2), ld = 2^l * ws
  double* Fb;
  int64_t P;
};

__device__ __forceinline__ double* lvl_buf(double* base, int64_t P, int ws, int l) {
  return base + P * (int64_t)ws * ((1ll << l) - 2);
}

// Job table: up-sweep level l at [2^l - 2, 2^{l+1} - 2) for l = 1..depth (2n-2 jobs),
// down-sweep the same offsets shifted by 2n-2, the leaf finish last (n jobs).
__global__ void setup_jobs_kernel(MultPlan p, GemmJob* __restrict__ jobs) {
  const int n = p.n_leaves;
  const int nup = 2 * n - 2;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= 2 * nup + n) return;
  const int ws = p.ws;
  const size_t pw = (size_t)p.pmax * ws, ww = (size_t)ws * ws;
  GemmJob jb;
  jb.A2 = nullptr; jb.B2 = nullptr;
  jb.lda2 = 0; jb.b2r = 0; jb.b2c = 0; jb.K2 = 0; jb.pad = 0;
  if (e < 2 * nup) {
    const bool up = e < nup;
    const int q = up ? e : e - nup;
    int l = 1;
    while (q >= (1 << (l + 1)) - 2) ++l;
    const int j = q - ((1 << l) - 2);
    const int node = p.lnodes[(1 << l) - 1 + j];
    const int64_t ldl = (int64_t)(1 << l) * ws;
    if (up) {
      // G_node = A U_node,  A = X[:, t] (leaf) or [G_left | G_right]
      jb.C = lvl_buf(p.Gb, p.P, ws, l) + (int64_t)j * ws;
      jb.ldc = ldl;
      jb.N = p.rU[node];
      jb.B1 = p.U + (size_t)node * pw;
      jb.b1r = ws; jb.b1c = 1;
      if (l == p.depth) {
        const int lo = p.lo[node];
        jb.A1 = p.X + lo;
        jb.lda1 = p.ldx;
        jb.K1 = p.hi[node] - lo;
      } else {
        const int a = p.left[node], b = p.right[node];
        const int64_t ldc1 = (int64_t)(1 << (l + 1)) * ws;
        jb.A1 = lvl_buf(p.Gb, p.P, ws, l + 1) + (int64_t)(2 * j) * ws;
        jb.lda1 = ldc1;
        jb.K1 = p.rU[a];
        jb.A2 = jb.A1 + ws;
        jb.lda2 = ldc1;
        jb.K2 = p.rU[b];
        jb.B2 = jb.B1 + (size_t)p.rU[a] * ws;
        jb.b2r = ws; jb.b2c = 1;
      }
    } else {
      // F_node = G_sib B_sib (+ F_parent V_parent[rows of node]^T)
      const int sib = p.lnodes[(1 << l) - 1 + (j ^ 1)];
      jb.A1 = lvl_buf(p.Gb, p.P, ws, l) + (int64_t)(j ^ 1) * ws;
      jb.lda1 = ldl;
      jb.K1 = p.rU[sib];
      jb.B1 = p.B + (size_t)sib * ww;
      jb.b1r = ws; jb.b1c = 1;
      jb.C = lvl_buf(p.Fb, p.P, ws, l) + (int64_t)j * ws;
      jb.ldc = ldl;
      jb.N = p.rV[node];
      if (l > 1) {
        const int par = p.lnodes[(1 << (l - 1)) - 1 + (j >> 1)];
        const int off = (j & 1) ? p.rV[p.left[par]] : 0;
        jb.A2 = lvl_buf(p.Fb, p.P, ws, l - 1) + (int64_t)(j >> 1) * ws;
        jb.lda2 = (int64_t)(1 << (l - 1)) * ws;
        jb.K2 = p.rV[par];
        jb.B2 = p.Vt + (size_t)par * ws * p.pmax + off;   // V_par[off:off+rV, :]^T
        jb.b2r = p.pmax; jb.b2c = 1;
      }
    }
  } else {
    // out[:, t] = X[:, t] D + F_leaf V_leaf^T
    const int j = e - 2 * nup;
    const int node = p.lnodes[(1 << p.depth) - 1 + j];
    const int lo = p.lo[node];
    jb.A1 = p.X + lo;
    jb.lda1 = p.ldx;
    jb.K1 = p.hi[node] - lo;
    jb.B1 = p.D + (size_t)j * p.dld * p.dld;
    jb.b1r = p.dld; jb.b1c = 1;
    jb.A2 = lvl_buf(p.Fb, p.P, ws, p.depth) + (int64_t)j * ws;
    jb.lda2 = (int64_t)(1 << p.depth) * ws;
    jb.K2 = p.rV[node];
    jb.B2 = p.Vt + (size_t)node * ws * p.pmax;
    jb.b2r = p.pmax; jb.b2c = 1;
    jb.C = p.out + lo;
    jb.ldc = p.ldo;
    jb.N = p.hi[node] - lo;
  }
  jobs[e] = jb;
}

static int g_sms = 0;

template <class T>
static int launch_batched(const GemmJob* jobs, int njobs, int64_t M, cudaStream_t s) {
  if (njobs <= 0 || M <= 0) return HSSEIG_OK;
  static int per_sm = 0;
  if (!per_sm) {
    cudaFuncSetAttribute(batched_gemm2_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)T::SMEM_BYTES);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, batched_gemm2_kernel<T>, T::THREADS,
                                                  T::SMEM_BYTES);
    if (per_sm < 1) per_sm = 1;
    if (!g_sms) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    }
  }
  const int tiles_m = (int)((M + T::BM - 1) / T::BM);
  const int64_t total = (int64_t)tiles_m * njobs;
  const int grid = (int)imin64(total, (int64_t)g_sms * per_sm);
  batched_gemm2_kernel<T><<<grid, T::THREADS, T::SMEM_BYTES, s>>>(jobs, njobs, M, tiles_m);
  HSS_CHECK_LAUNCH();
  return HSSEIG_OK;
}

// Tile variants (HSSEIG_TILE_NARROW / HSSEIG_TILE_WIDE select one for tuning runs).
static int tile_choice(const char* var, int dflt) {
  const char* v = getenv(var);
  return v ? atoi(v) : dflt;
}

// narrow outputs (ranks, N <= 112)
static int launch_narrow(int n, const GemmJob* jobs, int njobs, int64_t M, cudaStream_t s) {
  static const int variant = tile_choice("HSSEIG_TILE_NARROW", 1);
  if (variant == 0) {   // BM 128, 8 warps of 32 x 8NF, NF = ceil(n/16)
    switch ((n + 15) / 16) {
      case 1: return launch_batched<Tile<4, 1, 4, 2, 4>>(jobs, njobs, M, s);
      case 2: return launch_batched<Tile<4, 2, 4, 2, 4>>(jobs, njobs, M, s);
      case 3: return launch_batched<Tile<4, 3, 4, 2, 4>>(jobs, njobs, M, s);
      case 4: return launch_batched<Tile<4, 4, 4, 2, 4>>(jobs, njobs, M, s);
      case 5: return launch_batched<Tile<4, 5, 4, 2, 4>>(jobs, njobs, M, s);
      case 6: return launch_batched<Tile<4, 6, 4, 2, 4>>(jobs, njobs, M, s);
      case 7: return launch_batched<Tile<4, 7, 4, 2, 4>>(jobs, njobs, M, s);
      default: return HSSEIG_ERR_ARG;
    }
  }
  if (variant == 2) {   // BM 64, 4 warps of 32 x 8NF, NF = ceil(n/16)
    switch ((n + 15) / 16) {
      case 1: return launch_batched<Tile<4, 1, 2, 2, 4>>(jobs, njobs, M, s);
      case 2: return launch_batched<Tile<4, 2, 2, 2, 4>>(jobs, njobs, M, s);
      case 3: return launch_batched<Tile<4, 3, 2, 2, 4>>(jobs, njobs, M, s);
      case 4: return launch_batched<Tile<4, 4, 2, 2, 4>>(jobs, njobs, M, s);
      case 5: return launch_batched<Tile<4, 5, 2, 2, 4>>(jobs, njobs, M, s);
      case 6: return launch_batched<Tile<4, 6, 2, 2, 4>>(jobs, njobs, M, s);
      case 7: return launch_batched<Tile<4, 7, 2, 2, 4>>(jobs, njobs, M, s);
      default: return HSSEIG_ERR_ARG;
    }
  }
  // default: BM 64, 8 warps of 32 x 8NF, NF = ceil(n/32)
  switch ((n + 31) / 32) {
    case 1: return launch_batched<Tile<4, 1, 2, 4, 4>>(jobs, njobs, M, s);
    case 2: return launch_batched<Tile<4, 2, 2, 4, 4>>(jobs, njobs, M, s);
    case 3: return launch_batched<Tile<4, 3, 2, 4, 4>>(jobs, njobs, M, s);
    case 4: return launch_batched<Tile<4, 4, 2, 4, 4>>(jobs, njobs, M, s);
    default: return HSSEIG_ERR_ARG;
  }
}

// wide outputs (leaf finish N = leaf size; plain GEMM tiles)
static int launch_wide(int n, const GemmJob* jobs, int njobs, int64_t M, cudaStream_t s) {
  static const int variant = tile_choice("HSSEIG_TILE_WIDE", 1);
  if (variant == 0) {   // BM 64, 8 warps of 16 x 8NF, NF = ceil(n/16)
    switch ((n + 15) / 16) {
      case 1: case 2: case 3: case 4: return launch_batched<Tile<2, 4, 4, 2, 4>>(jobs, njobs, M, s);
      case 5: return launch_batched<Tile<2, 5, 4, 2, 4>>(jobs, njobs, M, s);
      case 6: return launch_batched<Tile<2, 6, 4, 2, 4>>(jobs, njobs, M, s);
      case 7: return launch_batched<Tile<2, 7, 4, 2, 4>>(jobs, njobs, M, s);
      case 8: return launch_batched<Tile<2, 8, 4, 2, 4>>(jobs, njobs, M, s);
      case 9: return launch_batched<Tile<2, 9, 4, 2, 4>>(jobs, njobs, M, s);
      case 10: return launch_batched<Tile<2, 10, 4, 2, 3>>(jobs, njobs, M, s);
      case 11: return launch_batched<Tile<2, 11, 4, 2, 3>>(jobs, njobs, M, s);
      case 12: return launch_batched<Tile<2, 12, 4, 2, 3>>(jobs, njobs, M, s);
      case 13: return launch_batched<Tile<2, 13, 4, 2, 3>>(jobs, njobs, M, s);
      default: return HSSEIG_ERR_ARG;
    }
  }
  // default: BM 64, 8 warps of 32 x 8NF, NF = ceil(n/32)
  switch ((n + 31) / 32) {
    case 1: case 2: return launch_batched<Tile<4, 2, 2, 4, 4>>(jobs, njobs, M, s);
    case 3: return launch_batched<Tile<4, 3, 2, 4, 4>>(jobs, njobs, M, s);
    case 4: return launch_batched<Tile<4, 4, 2, 4, 4>>(jobs, njobs, M, s);
    case 5: return launch_batched<Tile<4, 5, 2, 4, 3>>(jobs, njobs, M, s);
    case 6: return launch_batched<Tile<4, 6, 2, 4, 3>>(jobs, njobs, M, s);
    case 7: return launch_batched<Tile<4, 7, 2, 4, 3>>(jobs, njobs, M, s);
    default: return HSSEIG_ERR_ARG;
  }
}

__global__ void single_job_kernel(GemmJob* jobs, const double* A, int64_t lda, const double* B,
                                  int64_t ldb, double* C, int64_t ldc, int N, int K, int n0) {
  GemmJob jb;
  jb.A1 = A; jb.lda1 = lda; jb.K1 = K;
  jb.B1 = B + n0; jb.b1r = ldb; jb.b1c = 1;
  jb.A2 = nullptr; jb.B2 = nullptr; jb.lda2 = 0; jb.b2r = 0; jb.b2c = 0; jb.K2 = 0;
  jb.C = C + n0; jb.ldc = ldc; jb.N = N; jb.pad = 0;
  jobs[blockIdx.x] = jb;
}

}  // namespace hsseig

using namespace hsseig;

static int64_t jobs_doubles(int64_t n_leaves) {
  int64_t njobs = 2 * (2 * n_leaves - 2) + n_leaves;
  return (njobs * (int64_t)sizeof(GemmJob) + 7) / 8 + 32;
}

extern "C" int64_t hsseig_matmul_work_doubles(int64_t P, const hsseig_tree* t) {
  if (!t) return -1;
  return 2 * P * (int64_t)t->ws * (2 * (int64_t)t->n_leaves - 2) + jobs_doubles(t->n_leaves);
}

extern "C" int hsseig_hss_matmul_right(const double* X, int64_t ldx, int64_t P,
                                       const hsseig_tree* t, double* out, int64_t ldo,
                                       double* work, void* stream) {
  if (!t || !X || !out || !work || P < 0 || ldx < t->k || ldo < t->k) return HSSEIG_ERR_ARG;
  if (P == 0) return HSSEIG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t lvl_total = P * (int64_t)t->ws * (2 * (int64_t)t->n_leaves - 2);
  MultPlan p;
  p.depth = t->depth; p.n_leaves = t->n_leaves; p.ws = t->ws; p.pmax = t->pmax; p.mmax = t->mmax;
  p.dld = t->dld; p.Vt = t->Vt;
  p.lo = t->lo; p.hi = t->hi; p.left = t->left; p.right = t->right; p.lnodes = t->level_nodes;
  p.rU = t->rU; p.rV = t->rV; p.U = t->U; p.V = t->V; p.B = t->B; p.D = t->D;
  p.X = X; p.ldx = ldx; p.out = out; p.ldo = ldo; p.P = P;
  p.Gb = work;
  p.Fb = work + lvl_total;
  GemmJob* jobs = reinterpret_cast<GemmJob*>(work + 2 * lvl_total);
  const int n = t->n_leaves, nup = 2 * n - 2;
  const int total = 2 * nup + n;
  setup_jobs_kernel<<<(total + 127) / 128, 128, 0, s>>>(p, jobs);
  HSS_CHECK_LAUNCH();
  int rc;
  for (int l = t->depth; l >= 1; --l)
    if ((rc = launch_narrow(t->w, jobs + ((1 << l) - 2), 1 << l, P, s))) return rc;
  for (int l = 1; l <= t->depth; ++l)
    if ((rc = launch_narrow(t->w, jobs + nup + ((1 << l) - 2), 1 << l, P, s))) return rc;
  return launch_wide(t->mmax, jobs + 2 * nup, n, P, s);
}

extern "C" int hsseig_gemm(const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                           int64_t ldc, int64_t M, int64_t N, int64_t K, void* stream) {
  // Test/bench helper: plain C = A B on the same DMMA engine, N split in 128-wide jobs.
  // The caller passes C's job scratch implicitly: jobs live in a small static device buffer.
  static GemmJob* jobs = nullptr;
  static int cap = 0;
  if (M < 0 || N < 0 || K < 0 || lda < K || ldb < N || ldc < N) return HSSEIG_ERR_ARG;
  if (M == 0 || N == 0) return HSSEIG_OK;
  const int nj = (int)((N + 127) / 128);
  cudaStream_t s = (cudaStream_t)stream;
  if (nj > cap) {
    if (jobs) cudaFree(jobs);
    if (cudaMalloc(&jobs, sizeof(GemmJob) * nj) != cudaSuccess) return HSSEIG_ERR_CUDA;
    cap = nj;
  }
  for (int q = 0; q < nj; ++q) {
    int n0 = q * 128;
    int nn = (int)std::min<int64_t>(128, N - n0);
    single_job_kernel<<<1, 1, 0, s>>>(jobs + q, A, lda, B, ldb, C, ldc, nn, (int)K, n0);
    HSS_CHECK_LAUNCH();
  }
  return launch_wide(128, jobs, nj, M, s);
}

extern "C" const char* hsseig_version(void) { return "hsseig_b200 0.1 sm_100a"; }

namespace hsseig {
std::atomic<long long> g_launches{0};
}
extern "C" int64_t hsseig_launch_count(void) { return hsseig::g_launches.load(); }
