// HSS x dense product from the right, out = X H (Algorithm 3), on sm_100a.
//
// Reference: hss_matmul_right (pkg/src/hsseig/hss.py:309-361).
// Every step of the algorithm is a tall-skinny contraction over the P rows of X
// with a node-local factor, so each tree level is ONE launch of a batched
// two-segment FP64 GEMM (one job per node):
//   up, leaf  : G_i = X[:, t_i] U_i
//   up, inner : G_i = [G_l | G_r] U_i
//   down      : F_i = [G_sib | F_par] [B_sib ; V_par(rows of i)^T]     (the "inherit" term)
//   final     : out[:, t_i] = [X[:, t_i] | F_i] [D_i ; V_i^T]
//
// Kernel shape (Blackwell): persistent CTAs, one TMA producer warp and WM x WN DMMA
// consumer warps.  Operand tiles move by cp.async.bulk.tensor (TMA) into a STAGES-deep
// shared-memory ring guarded by full/empty mbarriers, so no block-wide barrier sits in
// the main loop; FP64 has no tcgen05 kind on sm_100a, so the contraction runs on the
// warp-level DMMA.8x8x4 tensor sub-pipe.  Boxes are 4 columns wider than the tile
// so the dense TMA rows land with a stride of 4 (mod 16) doubles, which keeps every
// fragment load bank-conflict free without a swizzle.
//
// Exactness of K tails: factor slots are stored zero-padded to the 16-aligned slot
// width and G/F slots get zeros from their rank up to the next multiple of 4 (store width
// SW), so a k-step that runs past a segment's K multiplies finite values by zeros.
//
// Job descriptors are built on the device from the ranks the construction wrote, so
// no host synchronisation is needed between construction and multiply.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "tma.cuh"

namespace hsseig {

// tensor-map roles: 0 X, 1 G_l, 2 G_{l+1}, 3 F_{l-1} (or F_depth), 4 U, 5 B, 6 Vt, 7 D


// One job tile for a warp whose first JM n-fragments are live (compile-time): accumulators,
// k-chunks (both segments) and the epilogue are all sized by JM, so a tile sized for the
// widest job of a launch spends neither DMMA work nor zeroing / store instructions on the
// padding fragments of narrower jobs (inner HSS levels: ranks 34..82 under one tile shape).
template <class T, int JM>
__device__ __forceinline__ void run_job(const TJob& jb, unsigned char* sm, uint64_t* full,
                                        uint64_t* empty, uint32_t& q, int64_t m0, int64_t M,
                                        int wm, int wn, int lane) {
  constexpr int JA = JM > 0 ? JM : 1;
  double acc[T::MF][JA][2];
#pragma unroll
  for (int i = 0; i < T::MF; ++i)
#pragma unroll
    for (int j = 0; j < JA; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int sg = 0; sg < 2; ++sg) {
    const int K = jb.K[sg];
    const int nc = (K + T::BK - 1) / T::BK;
    for (int c = 0; c < nc; ++c, ++q) {
      const int slot = q % T::STAGES;
      mbar_wait(&full[slot], (q / T::STAGES) & 1);
      const double* sA = reinterpret_cast<const double*>(sm + (size_t)slot * T::STAGE_BYTES);
      const double* sB =
          reinterpret_cast<const double*>(sm + (size_t)slot * T::STAGE_BYTES + T::A_BYTES);
      if (K - c * T::BK >= T::BK)
        tmma_chunk_j<T, JM, true>(sA, sB, acc, wm, wn, lane, T::BK);
      else
        tmma_chunk_j<T, JM, false>(sA, sB, acc, wm, wn, lane, (K - c * T::BK + 3) & ~3);
      stage_release(&empty[slot], lane);
    }
  }
  if (JM == 0) return;
  // epilogue: accumulators for columns < N, zeros in [N, SW); a thread owns column pairs
  // (2 gc, 2 gc + 1), stored as one 16-byte store when the job's rows are 16-byte aligned
  const int gr = lane >> 2, gc = lane & 3;
  const bool vec = ((reinterpret_cast<uintptr_t>(jb.C) | (uintptr_t)(jb.ldc * 8)) & 15) == 0;
#pragma unroll
  for (int i = 0; i < T::MF; ++i) {
    const int64_t row = m0 + wm * T::MF * 8 + i * 8 + gr;
    if (row >= M) continue;
    double* crow = jb.C + row * jb.ldc;
#pragma unroll
    for (int j = 0; j < JA; ++j) {
      const int col = wn * T::NF * 8 + j * 8 + 2 * gc;
      const double v0 = col < jb.N ? acc[i][j][0] : 0.0;
      const double v1 = col + 1 < jb.N ? acc[i][j][1] : 0.0;
      if (vec && col + 1 < jb.SW) {
        *reinterpret_cast<double2*>(crow + col) = make_double2(v0, v1);
      } else {
        if (col < jb.SW) crow[col] = v0;
        if (col + 1 < jb.SW) crow[col + 1] = v1;
      }
    }
  }
}

template <class T>
__global__ void __launch_bounds__(T::THREADS, T::MINB)
    tma_gemm_kernel(const __grid_constant__ MapSet maps, const TJob* __restrict__ jobs, int njobs,
                    int64_t M, int tiles_m) {
  extern __shared__ __align__(128) unsigned char smraw[];
  // 128-byte aligned ring; pointer arithmetic on the __shared__ array keeps the shared
  // address space (fragment loads compile to LDS, not generic LD)
  unsigned char* sm = smraw + ((128u - (smem_u32(smraw) & 127u)) & 127u);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)T::STAGE_BYTES * T::STAGES);
  uint64_t* empty = full + T::STAGES;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int total = njobs * tiles_m;
  if (tid == 0) {
    for (int s = 0; s < T::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], T::CONSUMERS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == T::CONSUMERS) {
    // ---------------- TMA producer (one lane) ----------------
    if (lane == 0) {
      uint32_t q = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const TJob jb = jobs[t / tiles_m];
        if (jb.N <= 0) continue;
        const int m0 = (t % tiles_m) * T::BM;
        for (int sg = 0; sg < 2; ++sg) {
          const int nc = (jb.K[sg] + T::BK - 1) / T::BK;
          for (int c = 0; c < nc; ++c, ++q) {
            const int slot = q % T::STAGES;
            mbar_wait(&empty[slot], ((q / T::STAGES) & 1) ^ 1);
            mbar_expect_tx(&full[slot], T::A_BYTES + T::B_BYTES);
            unsigned char* st = sm + (size_t)slot * T::STAGE_BYTES;
            tma_load_2d(st, &maps.m[jb.am[sg]], jb.acol[sg] + c * T::BK, m0, &full[slot]);
            tma_load_2d(st + T::A_BYTES, &maps.m[jb.bm[sg]], jb.bcol[sg], jb.brow[sg] + c * T::BK,
                        &full[slot]);
          }
        }
      }
    }
    return;
  }

  // ---------------- DMMA consumers ----------------
  const int wm = warp / T::WN, wn = warp % T::WN;
  uint32_t q = 0;
  for (int t = blockIdx.x; t < total; t += gridDim.x) {
    const TJob jb = jobs[t / tiles_m];
    if (jb.N <= 0) continue;
    const int64_t m0 = (int64_t)(t % tiles_m) * T::BM;
    // n-fragments of this warp that carry output columns of this job (warp-uniform)
    const int jmax = min(T::NF, max(0, (jb.N - wn * T::NF * 8 + 7) >> 3));
    switch (jmax) {
#define HSS_JM_CASE(J)                                                                   \
  case J:                                                                                \
    if constexpr (J <= T::NF) run_job<T, J>(jb, sm, full, empty, q, m0, M, wm, wn, lane); \
    break;
      HSS_JM_CASE(0) HSS_JM_CASE(1) HSS_JM_CASE(2) HSS_JM_CASE(3) HSS_JM_CASE(4)
      HSS_JM_CASE(5) HSS_JM_CASE(6) HSS_JM_CASE(7) HSS_JM_CASE(8) HSS_JM_CASE(9)
      HSS_JM_CASE(10) HSS_JM_CASE(11) HSS_JM_CASE(12) HSS_JM_CASE(13) HSS_JM_CASE(14)
#undef HSS_JM_CASE
      default: break;
    }
  }
}

struct MultPlan {
  int32_t depth, n_leaves, ws, pmax, dld, mmax;
  const int32_t *lo, *hi, *left, *right, *lnodes, *rU, *rV;
  double* out;
  int64_t ldo;
  double* Gb;  // levels 1..depth, level l at Gb + P*ws*(2^l - 2), ld = 2^l * ws
  double* Fb;
  int64_t P;
};

__host__ __device__ __forceinline__ int64_t lvl_off(int64_t P, int ws, int l) {
  return P * (int64_t)ws * ((1ll << l) - 2);
}

// Job table: up-sweep level l at [2^l - 2, 2^{l+1} - 2) for l = 1..depth (2n-2 jobs),
// down-sweep the same offsets shifted by 2n-2, the leaf finish last (n jobs).
// Entries [e_lo, e_hi) only (a split multiply builds the leaf up-level's jobs first, the
// rest once the upper ranks exist).
__global__ void setup_jobs_kernel(MultPlan p, TJob* __restrict__ jobs, int e_lo, int e_hi) {
  const int n = p.n_leaves;
  const int nup = 2 * n - 2;
  const int e = e_lo + blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= e_hi || e >= 2 * nup + n) return;
  const int ws = p.ws;
  TJob jb;
  jb.am[0] = jb.am[1] = 0;
  jb.bm[0] = jb.bm[1] = 4;
  jb.acol[0] = jb.acol[1] = jb.brow[0] = jb.brow[1] = jb.bcol[0] = jb.bcol[1] = 0;
  jb.K[0] = jb.K[1] = 0;
  if (e < 2 * nup) {
    const bool up = e < nup;
    const int q = up ? e : e - nup;
    int l = 1;
    while (q >= (1 << (l + 1)) - 2) ++l;
    const int j = q - ((1 << l) - 2);
    const int node = p.lnodes[(1 << l) - 1 + j];
    jb.ldc = (int64_t)(1 << l) * ws;
    if (up) {
      jb.C = p.Gb + lvl_off(p.P, ws, l) + (int64_t)j * ws;
      jb.N = p.rU[node];
      if (l == p.depth) {
        // TMA boxes must start on a 16-byte column: an odd leaf start begins one column
        // early against the zero row that precedes every U slot
        const int lo = p.lo[node], sh = lo & 1;
        jb.am[0] = 0; jb.acol[0] = lo - sh; jb.K[0] = p.hi[node] - lo + sh;
        jb.bm[0] = 4; jb.brow[0] = node * p.pmax + 1 - sh;
      } else {
        const int a = p.left[node], b = p.right[node];
        jb.am[0] = 2; jb.acol[0] = 2 * j * ws; jb.K[0] = p.rU[a];
        jb.bm[0] = 4; jb.brow[0] = node * p.pmax + 1;
        jb.am[1] = 2; jb.acol[1] = (2 * j + 1) * ws; jb.K[1] = p.rU[b];
        jb.bm[1] = 4; jb.brow[1] = node * p.pmax + 1 + p.rU[a];
      }
    } else {
      const int sib = p.lnodes[(1 << l) - 1 + (j ^ 1)];
      jb.C = p.Fb + lvl_off(p.P, ws, l) + (int64_t)j * ws;
      jb.N = p.rV[node];
      jb.am[0] = 1; jb.acol[0] = (j ^ 1) * ws; jb.K[0] = p.rU[sib];
      jb.bm[0] = 5; jb.brow[0] = sib * ws;
      if (l > 1) {
        const int par = p.lnodes[(1 << (l - 1)) - 1 + (j >> 1)];
        jb.am[1] = 3; jb.acol[1] = (j >> 1) * ws; jb.K[1] = p.rV[par];
        const int nl = p.rV[p.left[par]];
        jb.bm[1] = 6; jb.brow[1] = par * ws; jb.bcol[1] = (j & 1) ? nl + (nl & 1) : 0;
      }
    }
    // a consumer reads this slot's columns up to its K rounded to 4 (tmma_chunk's k-steps),
    // so zeros are stored only up to there, not across the whole slot width
    jb.SW = (jb.N + 3) & ~3;
  } else {
    const int j = e - 2 * nup;
    const int node = p.lnodes[(1 << p.depth) - 1 + j];
    const int lo = p.lo[node], sh = lo & 1;
    jb.C = p.out + lo;
    jb.ldc = p.ldo;
    jb.N = jb.SW = p.hi[node] - lo;
    jb.am[0] = 0; jb.acol[0] = lo - sh; jb.K[0] = p.hi[node] - lo + sh;
    jb.bm[0] = 7; jb.brow[0] = j * hsseig_drows(p.mmax) + 1 - sh;
    jb.am[1] = 3; jb.acol[1] = j * ws; jb.K[1] = p.rV[node];
    jb.bm[1] = 6; jb.brow[1] = node * ws;
  }
  jobs[e] = jb;
}

// ---------------------------------------------------------------------------- host side

static int g_sms = 0;

// The launch's tensor maps travel as one __grid_constant__ MapSet kernel parameter (no
// device copy, no extra launch); the producer picks a map by role at run time through its
// parameter-space address.
// max_ctas > 0 caps the persistent grid (a split multiply leaves SMs to the construction
// kernels running beside it).
template <class T>
static int launch_tma(const Operand (&ops)[kMaps], MapSet* dmaps, const TJob* jobs, int njobs,
                      int64_t M, cudaStream_t s, int max_ctas = 0) {
  if (njobs <= 0 || M <= 0) return HSSEIG_OK;
  static int per_sm = 0;
  if (!per_sm) {
    cudaFuncSetAttribute(tma_gemm_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)T::SMEM_BYTES);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tma_gemm_kernel<T>, T::THREADS,
                                                  T::SMEM_BYTES);
    if (per_sm < 1) per_sm = 1;
    if (!g_sms) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    }
  }
  MapSet maps;
  for (int r = 0; r < kMaps; ++r) {
    const bool is_a = r < 4;
    const uint32_t bc = is_a ? T::SA : T::SB;
    const uint32_t br = is_a ? T::BM : T::BK;
    if (!make_map(&maps.m[r], ops[r].base, ops[r].rows, ops[r].cols, ops[r].ld, bc, br))
      HSS_ARG_FAIL();
  }
  (void)dmaps;   // the maps travel as a __grid_constant__ kernel parameter
  const int tiles_m = (int)((M + T::BM - 1) / T::BM);
  const int64_t total = (int64_t)tiles_m * njobs;
  int64_t cap = (int64_t)g_sms * per_sm;
  if (max_ctas > 0 && max_ctas < cap) cap = max_ctas;
  const int grid = (int)imin64(total, cap);
  tma_gemm_kernel<T><<<grid, T::THREADS, T::SMEM_BYTES, s>>>(maps, jobs, njobs, M, tiles_m);
  HSS_CHECK_LAUNCH();
  return HSSEIG_OK;
}


// Rank-width tiles: 8 consumer warps stacked along M (BM = 128), one warp spans the whole
// output width in NF 8-column fragments, so N is padded to a multiple of 8 only.
constexpr int narrow_stages(int nf) {
  return (200 * 1024) / (128 * 20 * 8 + 16 * (((nf * 8 + 15) / 16) * 16 + 4) * 8) < 8
             ? (200 * 1024) / (128 * 20 * 8 + 16 * (((nf * 8 + 15) / 16) * 16 + 4) * 8)
             : 8;
}
template <int NF>
using RankTile = TTile<2, NF, 8, 1, narrow_stages(NF)>;

// narrow outputs (ranks, N <= 112).  Measured alternatives (BM 64 with 8 warps of 32 x 8NF,
// BM 128 with NF = N/16, two CTAs per SM) were 5-10% slower at config 4.
static int launch_narrow(int n, const Operand (&ops)[kMaps], MapSet* dm, const TJob* jobs, int njobs,
                         int64_t M, cudaStream_t s, int max_ctas = 0) {
  switch ((n + 7) / 8) {
    case 1: case 2: case 3: case 4: return launch_tma<RankTile<4>>(ops, dm, jobs, njobs, M, s, max_ctas);
    case 5: return launch_tma<RankTile<5>>(ops, dm, jobs, njobs, M, s, max_ctas);
    case 6: return launch_tma<RankTile<6>>(ops, dm, jobs, njobs, M, s, max_ctas);
    case 7: return launch_tma<RankTile<7>>(ops, dm, jobs, njobs, M, s, max_ctas);
    case 8: return launch_tma<RankTile<8>>(ops, dm, jobs, njobs, M, s, max_ctas);
    case 9: return launch_tma<RankTile<9>>(ops, dm, jobs, njobs, M, s, max_ctas);
    case 10: return launch_tma<RankTile<10>>(ops, dm, jobs, njobs, M, s, max_ctas);
    case 11: return launch_tma<RankTile<11>>(ops, dm, jobs, njobs, M, s, max_ctas);
    case 12: return launch_tma<RankTile<12>>(ops, dm, jobs, njobs, M, s, max_ctas);
    case 13: return launch_tma<RankTile<13>>(ops, dm, jobs, njobs, M, s, max_ctas);
    case 14: return launch_tma<RankTile<14>>(ops, dm, jobs, njobs, M, s, max_ctas);
    default: HSS_ARG_FAIL();
  }
}

// wide outputs (leaf finish N = leaf size; plain GEMM tiles), N <= 224: BM 64, 8 consumer
// warps of 32 x 8NF, NF = ceil(n/32) (94% of the DMMA pipe at config 4)
static int launch_wide(int n, const Operand (&ops)[kMaps], MapSet* dm, const TJob* jobs, int njobs,
                       int64_t M, cudaStream_t s) {
  switch ((n + 31) / 32) {
    case 1: case 2: case 3: case 4: return launch_tma<TTile<4, 4, 2, 4, 6>>(ops, dm, jobs, njobs, M, s);
    case 5: return launch_tma<TTile<4, 5, 2, 4, 6>>(ops, dm, jobs, njobs, M, s);
    case 6: return launch_tma<TTile<4, 6, 2, 4, 5>>(ops, dm, jobs, njobs, M, s);
    case 7: return launch_tma<TTile<4, 7, 2, 4, 5>>(ops, dm, jobs, njobs, M, s);
    default: HSS_ARG_FAIL();
  }
}

// short-M outputs (M = the sample width m <= 112, N = k: Z^T = Omega^T C): one warp row
// spans all M rows in ceil(m/8) fragments (M padded to 8 only), 8 warps of 16 columns
template <int MF>
using ShortTile = TTile<MF, 2, 1, 8, 6>;
static int launch_short(int m, const Operand (&ops)[kMaps], MapSet* dm, const TJob* jobs, int njobs,
                        cudaStream_t s) {
  switch ((m + 7) / 8) {
    case 1: case 2: case 3: case 4: return launch_tma<ShortTile<4>>(ops, dm, jobs, njobs, m, s);
    case 5: return launch_tma<ShortTile<5>>(ops, dm, jobs, njobs, m, s);
    case 6: return launch_tma<ShortTile<6>>(ops, dm, jobs, njobs, m, s);
    case 7: return launch_tma<ShortTile<7>>(ops, dm, jobs, njobs, m, s);
    case 8: return launch_tma<ShortTile<8>>(ops, dm, jobs, njobs, m, s);
    case 9: return launch_tma<ShortTile<9>>(ops, dm, jobs, njobs, m, s);
    case 10: return launch_tma<ShortTile<10>>(ops, dm, jobs, njobs, m, s);
    case 11: return launch_tma<ShortTile<11>>(ops, dm, jobs, njobs, m, s);
    case 12: return launch_tma<ShortTile<12>>(ops, dm, jobs, njobs, m, s);
    case 13: return launch_tma<ShortTile<13>>(ops, dm, jobs, njobs, m, s);
    case 14: return launch_tma<ShortTile<14>>(ops, dm, jobs, njobs, m, s);
    default: HSS_ARG_FAIL();
  }
}

// job-table GEMMs for other paths (sampling): shape 0 rank-width (N = n), 1 wide, 2 short-M
// (M = n = the sample width, N = 128-column jobs)
int tma_jobs_gemm(int shape, int n, const Operand (&ops)[kMaps], MapSet* dmaps, const TJob* jobs,
                  int njobs, int64_t M, cudaStream_t s) {
  if (shape == 0) return launch_narrow(n, ops, dmaps, jobs, njobs, M, s);
  if (shape == 1) return launch_wide(n, ops, dmaps, jobs, njobs, M, s);
  if (M != n) HSS_ARG_FAIL();
  return launch_short(n, ops, dmaps, jobs, njobs, s);
}

__global__ void plain_jobs_kernel(TJob* jobs, int nj, double* C, int64_t ldc, int N, int K) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nj) return;
  TJob jb;
  jb.am[0] = 0; jb.am[1] = 0; jb.acol[0] = 0; jb.acol[1] = 0;
  jb.bm[0] = 4; jb.bm[1] = 4; jb.brow[0] = 0; jb.brow[1] = 0; jb.bcol[0] = q * 128; jb.bcol[1] = 0;
  jb.K[0] = K; jb.K[1] = 0;
  jb.N = min(128, N - q * 128);
  jb.SW = jb.N;
  jb.C = C + q * 128;
  jb.ldc = ldc;
  jobs[q] = jb;
}

}  // namespace hsseig

using namespace hsseig;

static int64_t jobs_doubles(int64_t n_leaves) {
  const int64_t njobs = 2 * (2 * n_leaves - 2) + n_leaves;
  return (njobs * (int64_t)sizeof(TJob) + 7) / 8 + 32 + 66 * (int64_t)sizeof(MapSet) / 8 + 32;
}

extern "C" int64_t hsseig_matmul_work_doubles(int64_t P, const hsseig_tree* t) {
  if (!t) return -1;
  return 2 * P * (int64_t)t->ws * (2 * (int64_t)t->n_leaves - 2) + jobs_doubles(t->n_leaves);
}

// part -1: the whole product; part 0: only the leaf up-level G_depth = X U_leaf (it needs
// nothing above the leaf level of the tree, so it can run beside the construction of the
// upper levels, on at most max_ctas SMs); part 1: the rest, after part 0 and the full build.
static int matmul_right(const double* X, int64_t ldx, int64_t P, const hsseig_tree* t, double* out,
                        int64_t ldo, double* work, int part, int max_ctas, cudaStream_t s) {
  if (!t || !X || !out || !work || P < 0 || ldx < t->k || ldo < t->k) HSS_ARG_FAIL();
  if (part < -1 || part > 1) HSS_ARG_FAIL();
  if (P == 0) return HSSEIG_OK;
  if ((reinterpret_cast<uintptr_t>(X) & 15) || (ldx & 1) || (reinterpret_cast<uintptr_t>(work) & 15))
    HSS_ARG_FAIL();   // TMA needs 16-byte aligned rows
  if (P > 0x7fffffff) HSS_ARG_FAIL();
  const int ws = t->ws, n = t->n_leaves, nn = t->n_nodes, nup = 2 * n - 2;
  const int64_t lvl_total = P * (int64_t)ws * (2 * (int64_t)n - 2);
  MultPlan p;
  p.depth = t->depth; p.n_leaves = n; p.ws = ws; p.pmax = t->pmax; p.dld = t->dld;
  p.mmax = t->mmax;
  p.lo = t->lo; p.hi = t->hi; p.left = t->left; p.right = t->right; p.lnodes = t->level_nodes;
  p.rU = t->rU; p.rV = t->rV;
  p.out = out; p.ldo = ldo; p.P = P;
  p.Gb = work;
  p.Fb = work + lvl_total;
  TJob* jobs = reinterpret_cast<TJob*>(work + 2 * lvl_total);
  const int njob_total = 2 * nup + n;
  MapSet* dmaps = reinterpret_cast<MapSet*>(
      (reinterpret_cast<uintptr_t>(jobs + njob_total) + 255) & ~(uintptr_t)255);
  if (t->depth > 31) HSS_ARG_FAIL();
  const int D = t->depth;
  const int leaf_lo = (1 << D) - 2, leaf_hi = (1 << (D + 1)) - 2;   // the leaf up-level's jobs
  auto setup = [&](int e_lo, int e_hi) -> int {
    if (e_hi <= e_lo) return HSSEIG_OK;
    setup_jobs_kernel<<<(e_hi - e_lo + 127) / 128, 128, 0, s>>>(p, jobs, e_lo, e_hi);
    HSS_CHECK_LAUNCH();
    return HSSEIG_OK;
  };
  if (part == -1) setup(0, njob_total);
  else if (part == 0) setup(leaf_lo, leaf_hi);
  else { setup(0, leaf_lo); setup(leaf_hi, njob_total); }
  auto lvl = [&](double* base, int l) -> Operand {
    if (l < 1 || l > t->depth) return Operand{nullptr, 0, 0, 0};
    const uint64_t cols = (uint64_t)(1u << l) * ws;
    return Operand{base + lvl_off(P, ws, l), (uint64_t)P, cols, cols};
  };
  const Operand none{nullptr, 0, 0, 0};
  const Operand Xop{X, (uint64_t)P, (uint64_t)t->k, (uint64_t)ldx};
  const Operand Uop{t->U, (uint64_t)nn * t->pmax, (uint64_t)ws, (uint64_t)ws};
  const Operand Bop{t->B, (uint64_t)nn * ws, (uint64_t)ws, (uint64_t)ws};
  const Operand Vtop{t->Vt, (uint64_t)nn * ws, (uint64_t)t->pmax, (uint64_t)t->pmax};
  const Operand Dop{t->D, (uint64_t)n * hsseig_drows(t->mmax), (uint64_t)t->dld, (uint64_t)t->dld};
  int rc;
  // output tiles cover the ranks (host bound rmax when the caller supplied it)
  const int nr = (t->rmax > 0 && t->rmax < t->w) ? t->rmax : t->w;
  for (int l = D; l >= 1; --l) {
    if ((part == 0 && l != D) || (part == 1 && l == D)) continue;
    const Operand ops[kMaps] = {Xop, lvl(p.Gb, l), lvl(p.Gb, l + 1), none, Uop, Bop, Vtop, Dop};
    if ((rc = launch_narrow(nr, ops, dmaps + (D - l), jobs + ((1 << l) - 2), 1 << l, P, s,
                            part == 0 ? max_ctas : 0)))
      return rc;
  }
  if (part == 0) return HSSEIG_OK;
  for (int l = 1; l <= D; ++l) {
    const Operand ops[kMaps] = {Xop, lvl(p.Gb, l), none, lvl(p.Fb, l - 1), Uop, Bop, Vtop, Dop};
    if ((rc = launch_narrow(nr, ops, dmaps + D + l - 1, jobs + nup + ((1 << l) - 2), 1 << l, P, s)))
      return rc;
  }
  const Operand ops[kMaps] = {Xop, none, none, lvl(p.Fb, D), Uop, Bop, Vtop, Dop};
  return launch_wide(t->mmax, ops, dmaps + 2 * D, jobs + 2 * nup, n, P, s);
}

extern "C" int hsseig_hss_matmul_right(const double* X, int64_t ldx, int64_t P,
                                       const hsseig_tree* t, double* out, int64_t ldo,
                                       double* work, void* stream) {
  return matmul_right(X, ldx, P, t, out, ldo, work, -1, 0, (cudaStream_t)stream);
}

extern "C" int hsseig_hss_matmul_right_part(const double* X, int64_t ldx, int64_t P,
                                            const hsseig_tree* t, double* out, int64_t ldo,
                                            double* work, int32_t part, int32_t max_ctas,
                                            void* stream) {
  if (part != 0 && part != 1) HSS_ARG_FAIL();
  return matmul_right(X, ldx, P, t, out, ldo, work, part, max_ctas, (cudaStream_t)stream);
}

namespace hsseig {
int tma_plain_gemm(const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                   int64_t ldc, int64_t M, int64_t N, int64_t K, TJob* jobs, MapSet* dmaps,
                   cudaStream_t s) {
  if (M < 0 || N < 0 || K < 0 || lda < K || ldb < N || ldc < N) HSS_ARG_FAIL();
  if (M == 0 || N == 0) return HSSEIG_OK;
  if ((reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(B) & 15) || (lda & 1) ||
      (ldb & 1) || K == 0)
    HSS_ARG_FAIL();
  const int nj = (int)((N + 127) / 128);
  plain_jobs_kernel<<<(nj + 127) / 128, 128, 0, s>>>(jobs, nj, C, ldc, (int)N, (int)K);
  HSS_CHECK_LAUNCH();
  // the maps carry the exact extents, so TMA zero-fills the K / N tails
  const Operand none{nullptr, 0, 0, 0};
  const Operand ops[kMaps] = {Operand{A, (uint64_t)M, (uint64_t)K, (uint64_t)lda}, none, none, none,
                              Operand{B, (uint64_t)K, (uint64_t)N, (uint64_t)ldb}, none, none, none};
  return launch_wide(128, ops, dmaps, jobs, nj, M, s);
}
}  // namespace hsseig

extern "C" int hsseig_gemm(const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                           int64_t ldc, int64_t M, int64_t N, int64_t K, void* stream) {
  // Test/bench helper: plain C = A B on the same TMA/DMMA engine, N split in 128-wide jobs.
  static TJob* jobs = nullptr;
  static MapSet* dmaps = nullptr;
  static int cap = 0;
  const int nj = (int)((N + 127) / 128);
  if (nj > cap) {
    if (jobs) cudaFree(jobs);
    if (cudaMalloc(&jobs, sizeof(TJob) * nj) != cudaSuccess) return HSSEIG_ERR_CUDA;
    cap = nj;
  }
  if (!dmaps) {
    if (cudaMalloc(&dmaps, sizeof(MapSet)) != cudaSuccess) return HSSEIG_ERR_CUDA;
  }
  return tma_plain_gemm(A, lda, B, ldb, C, ldc, M, N, K, jobs, dmaps, (cudaStream_t)stream);
}

extern "C" const char* hsseig_version(void) { return "hsseig_b200 0.2 sm_100a"; }

namespace hsseig {
std::atomic<long long> g_launches{0};
static thread_local char g_err[256] = "";
void set_arg_error(const char* file, int line) {
  const char* base = strrchr(file, '/');
  snprintf(g_err, sizeof(g_err), "invalid argument (%s:%d)", base ? base + 1 : file, line);
}
}
extern "C" const char* hsseig_last_error(void) { return hsseig::g_err; }
extern "C" int64_t hsseig_launch_count(void) { return hsseig::g_launches.load(); }
