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
#include <cstdlib>
#include <vector>

#include "tma.cuh"

namespace hsseig {

__global__ void cauchy_block_kernel(CauchyGen g, const int64_t* __restrict__ rows, int64_t nr,
                                    const int64_t* __restrict__ cols, int64_t nc,
                                    double* __restrict__ out, int64_t ldo) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nr * nc) return;
  int64_t a = e / nc, b = e % nc;
  out[a * ldo + b] = g.entry(rows[a], cols[b]);
}

// Sampling, warp-specialised: GEN generator warps evaluate the BM x BK tile of C (or C^T)
// on the FP64 pipe straight into a shared-memory ring and one of them arms the TMA copy
// of the matching Omega rows; WM x WN consumer warps contract on the DMMA tensor
// sub-pipe.  The two pipes overlap, and full/empty mbarriers replace block barriers.
// Work items are (row tile, K split) pairs walked persistently; partial tiles go to
// part[split] and are reduced in a fixed order (deterministic).
constexpr int kGenWarps = 8;

template <class T, bool TRANS>
__global__ void __launch_bounds__((T::CONSUMERS + kGenWarps) * 32, 1)
    sample_ws_kernel(CauchyGen g, const MapSet* __restrict__ omap, int w, double* __restrict__ part,
                     int64_t ldp, int kchunk, int nsplit, int tiles, int64_t row0, int64_t row1) {
  // output rows [row0, row1) of Y (or Z); part rows are indexed from row0
  extern __shared__ __align__(128) unsigned char smraw[];
  // 128-byte aligned ring; pointer arithmetic on the __shared__ array keeps the shared
  // address space (fragment loads compile to LDS, not generic LD)
  unsigned char* sm = smraw + ((128u - (smem_u32(smraw) & 127u)) & 127u);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)T::STAGE_BYTES * T::STAGES);
  uint64_t* empty = full + T::STAGES;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t k = g.k;
  const int items = tiles * nsplit;
  if (tid == 0) {
    for (int s = 0; s < T::STAGES; ++s) {
      mbar_init(&full[s], kGenWarps * 32 + 1);   // every generator thread + the TMA arm
      mbar_init(&empty[s], T::CONSUMERS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp >= T::CONSUMERS) {
    // ---------------- generators ----------------
    // thread -> one K position vk of the chunk and FR tile rows (a, a + RS, ...);
    // the tile-row ("fixed") generator data stays in registers for the whole item
    constexpr int GT = kGenWarps * 32;
    constexpr int RS = GT / T::BK;               // row groups
    constexpr int FR = T::BM / RS;               // tile rows per thread
    const int gt = tid - T::CONSUMERS * 32;
    const int vk = gt % T::BK, a0 = gt / T::BK;
    if (warp == T::CONSUMERS && lane == 0) tmap_acquire(&omap->m[0]);
    uint32_t q = 0;
    for (int it = blockIdx.x; it < items; it += gridDim.x) {
      const int tile = it % tiles, split = it / tiles;
      const int64_t m0 = row0 + (int64_t)tile * T::BM;
      const int64_t kbeg = (int64_t)split * kchunk;
      const int64_t kend = imin64(k, kbeg + kchunk);
      const int nch = (int)((kend - kbeg + T::BK - 1) / T::BK);
      double fd[FR], f1[FR], f2[FR], f3[FR], f4[FR];
      int fl[FR];
      bool fok[FR];
#pragma unroll
      for (int u = 0; u < FR; ++u) {
        const int64_t fix = m0 + a0 + u * RS;
        fok[u] = fix < row1;
        const int64_t fi = fok[u] ? fix : 0;
        fl[u] = g.lid ? __ldg(g.lid + fi) : -1;
        fd[u] = __ldg(g.d + fi);
        if (TRANS) {   // column j = fix of C
          f1[u] = __ldg(g.dnext + fi); f2[u] = __ldg(g.gam + fi); f3[u] = __ldg(g.mu + fi);
          f4[u] = __ldg(g.v + fi);
        } else {       // row i = fix of C
          f4[u] = __ldg(g.zhat + fi);
          f1[u] = f2[u] = f3[u] = 0.0;
        }
      }
      // K-running generator data of the next chunk is loaded one chunk ahead
      auto load_var = [&](int cc, double& od, double& o1, double& o2, double& o3, double& o4,
                          int& ol) {
        const int64_t vv = kbeg + (int64_t)cc * T::BK + vk;
        const int64_t vi = vv < kend ? vv : 0;
        ol = g.lid ? __ldg(g.lid + vi) : -2;
        od = __ldg(g.d + vi);
        if (TRANS) {
          o4 = __ldg(g.zhat + vi);
          o1 = o2 = o3 = 0.0;
        } else {
          o1 = __ldg(g.dnext + vi); o2 = __ldg(g.gam + vi); o3 = __ldg(g.mu + vi);
          o4 = __ldg(g.v + vi);
        }
      };
      double nd = 0.0, n1 = 0.0, n2 = 0.0, n3 = 0.0, n4 = 0.0;
      int nl = -2;
      if (nch > 0) load_var(0, nd, n1, n2, n3, n4, nl);
      for (int c = 0; c < nch; ++c, ++q) {
        const int slot = q % T::STAGES;
        const int64_t var = kbeg + (int64_t)c * T::BK + vk;   // index running along K
        const bool vok = var < kend;
        const double vd = nd, v1 = n1, v2 = n2, v3 = n3, v4 = n4;
        const int vl = nl;
        if (c + 1 < nch) load_var(c + 1, nd, n1, n2, n3, n4, nl);
        mbar_wait(&empty[slot], ((q / T::STAGES) & 1) ^ 1);
        double* sA = reinterpret_cast<double*>(sm + (size_t)slot * T::STAGE_BYTES);
#pragma unroll
        for (int u = 0; u < FR; ++u) {
          const int64_t fix = m0 + a0 + u * RS;
          double val = 0.0;
          if (fok[u] && vok && vl != fl[u]) {   // off-diagonal sample: own leaf block zero
            double gap;
            if (TRANS)   // C[var][fix]: row var, column fix
              gap = stable_gap(var, fix, vd, fd[u], f1[u], f2[u], f3[u]);
            else         // C[fix][var]
              gap = stable_gap(fix, var, fd[u], vd, v1, v2, v3);
            val = (v4 * f4[u]) * rcp_nr(gap);
          }
          sA[(a0 + u * RS) * T::SA + vk] = val;
        }
        if (warp == T::CONSUMERS && lane == 0) {
          mbar_expect_tx(&full[slot], T::B_BYTES);
          tma_load_2d(sm + (size_t)slot * T::STAGE_BYTES + T::A_BYTES, &omap->m[0], 0,
                      (int)(kbeg + (int64_t)c * T::BK), &full[slot]);
        }
        // each generator thread releases its own tile writes (mbarrier.arrive is .release)
        mbar_arrive(&full[slot]);
      }
    }
    return;
  }

  // ---------------- DMMA consumers ----------------
  const int wm = warp / T::WN, wn = warp % T::WN;
  const int gr = lane >> 2, gc = lane & 3;
  uint32_t q = 0;
  double acc[T::MF][T::NF][2];
  for (int it = blockIdx.x; it < items; it += gridDim.x) {
    const int tile = it % tiles, split = it / tiles;
    const int64_t m0 = (int64_t)tile * T::BM;   // relative to row0
    const int64_t kbeg = (int64_t)split * kchunk;
    const int64_t kend = imin64(k, kbeg + kchunk);
    const int nch = (int)((kend - kbeg + T::BK - 1) / T::BK);
#pragma unroll
    for (int i = 0; i < T::MF; ++i)
#pragma unroll
      for (int j = 0; j < T::NF; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int c = 0; c < nch; ++c, ++q) {
      const int slot = q % T::STAGES;
      mbar_wait(&full[slot], (q / T::STAGES) & 1);
      const double* sA = reinterpret_cast<const double*>(sm + (size_t)slot * T::STAGE_BYTES);
      const double* sB =
          reinterpret_cast<const double*>(sm + (size_t)slot * T::STAGE_BYTES + T::A_BYTES);
      tmma_chunk<T>(sA, sB, acc, wm, wn, lane);
      stage_release(&empty[slot], lane);
    }
    const int64_t nrows = row1 - row0;
    double* P = part + (int64_t)split * nrows * ldp;
#pragma unroll
    for (int i = 0; i < T::MF; ++i) {
      const int64_t row = m0 + wm * T::MF * 8 + i * 8 + gr;
      if (row >= nrows) continue;
#pragma unroll
      for (int j = 0; j < T::NF; ++j) {
        const int col = wn * T::NF * 8 + j * 8 + 2 * gc;
        if (col < w) P[row * ldp + col] = acc[i][j][0];
        if (col + 1 < w) P[row * ldp + col + 1] = acc[i][j][1];
      }
    }
  }
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

// The same reduction for rows [r0, r0 + nr) of the partials only (same order of the splits, so
// the sums are bit-identical): the rows of one panel chunk, reduced as soon as its product is done.
__global__ void splitk_reduce_rows_kernel(const double* __restrict__ part, int nsplit,
                                          int64_t split_stride, int64_t r0, int64_t nr, int w,
                                          int64_t ldp, double* __restrict__ out, int64_t ldo) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nr * w) return;
  int64_t row = r0 + e / w;
  int col = (int)(e % w);
  double s = 0.0;
  for (int t = 0; t < nsplit; ++t) s += part[(int64_t)t * split_stride + row * ldp + col];
  out[row * ldo + col] = s;
}

// out = Qb @ C with B-operand tiles of C generated in shared memory; one BM x BN tile.
template <class T>
__device__ __forceinline__ void dense_update_tile(const double* __restrict__ Q, int64_t ldq,
                                                  int64_t P, const CauchyGen& g,
                                                  double* __restrict__ out, int64_t ldo,
                                                  int64_t m0, int64_t n0, double* smem) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / T::WN, wn = warp % T::WN;
  const int64_t k = g.k;
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
__global__ void __launch_bounds__(T::THREADS) dense_update_kernel(const double* __restrict__ Q,
                                                                  int64_t ldq, int64_t P,
                                                                  CauchyGen g,
                                                                  double* __restrict__ out,
                                                                  int64_t ldo) {
  extern __shared__ __align__(16) double smem[];
  dense_update_tile<T>(Q, ldq, P, g, out, ldo, (int64_t)blockIdx.x * T::BM,
                       (int64_t)blockIdx.y * T::BN, smem);
}

// Level-batched dense updates: task t = (system s, row tile, column tile) of
// out_s = W_s[:, :k_s] @ C_s, with W_s the n_s x n_s merge block (ld n_s) and out_s n_s x k_s.
template <class T>
__global__ void __launch_bounds__(T::THREADS) wave_dense_kernel(
    const double* __restrict__ W, const int64_t* __restrict__ woff, const int64_t* __restrict__ nrow,
    const int64_t* __restrict__ ldw, CauchyGen g, const int64_t* __restrict__ koff,
    double* __restrict__ out, const int64_t* __restrict__ ooff, const int32_t* __restrict__ tasks) {
  extern __shared__ __align__(16) double smem[];
  const int s = tasks[3 * blockIdx.x], mt = tasks[3 * blockIdx.x + 1], nt = tasks[3 * blockIdx.x + 2];
  const int64_t a = koff[s], k = koff[s + 1] - a, n = nrow[s];
  CauchyGen gs = g;
  gs.d += a; gs.dnext += a; gs.gam += a; gs.mu += a; gs.zhat += a; gs.v += a;
  gs.k = k;
  dense_update_tile<T>(W + woff[s], ldw[s], n, gs, out + ooff[s], k, (int64_t)mt * T::BM,
                       (int64_t)nt * T::BN, smem);
}

static void sample_split(int64_t k, int64_t nrows, int64_t bm, int64_t* nsplit, int64_t* kchunk) {
  const int64_t tiles = (nrows + bm - 1) / bm;
  int64_t ns = (148 * 6 + tiles - 1) / tiles;     // enough items to keep every SM busy
  ns = imax64(1, imin64(ns, (k + 511) / 512));
  int64_t kc = (k + ns - 1) / ns;
  kc = (kc + 15) / 16 * 16;
  *nsplit = (k + kc - 1) / kc;
  *kchunk = kc;
}

template <class T>
static int launch_sample(const CauchyGen& g, const double* om, int64_t ldom, int w, int64_t row0,
                         int64_t row1, double* Y, double* Z, int64_t ldy, double* work,
                         cudaStream_t s) {
  const int64_t k = g.k;
  const int64_t nrows = row1 - row0;
  const int64_t tiles = (nrows + T::BM - 1) / T::BM;
  const int64_t ldp = ((w + 1) / 2) * 2;
  int64_t nsplit, kchunk;
  sample_split(k, nrows, T::BM, &nsplit, &kchunk);
  constexpr int threads = (T::CONSUMERS + kGenWarps) * 32;
  static int per_sm = 0, sms = 0;
  if (!per_sm) {
    cudaFuncSetAttribute(sample_ws_kernel<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)T::SMEM_BYTES);
    cudaFuncSetAttribute(sample_ws_kernel<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)T::SMEM_BYTES);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sample_ws_kernel<T, false>, threads, T::SMEM_BYTES);
    if (per_sm < 1) per_sm = 1;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  double* pY = work;
  double* pZ = work + nsplit * nrows * ldp;
  MapSet* dmap = reinterpret_cast<MapSet*>(
      (reinterpret_cast<uintptr_t>(work + 2 * nsplit * nrows * ldp) + 255) & ~(uintptr_t)255);
  MapSet maps;
  for (int r = 1; r < kMaps; ++r) make_map(&maps.m[r], nullptr, 0, 0, 0, 0, 0);
  if (!make_map(&maps.m[0], om, (uint64_t)k, (uint64_t)w, (uint64_t)ldom, T::SB, T::BK))
    HSS_ARG_FAIL();
  if (!upload_maps(maps, dmap, s)) return HSSEIG_ERR_CUDA;
  const int64_t items = tiles * nsplit;
  const int grid = (int)imin64(items, (int64_t)sms * per_sm);
  sample_ws_kernel<T, false><<<grid, threads, T::SMEM_BYTES, s>>>(g, dmap, w, pY, ldp, (int)kchunk,
                                                                (int)nsplit, (int)tiles, row0, row1);
  HSS_CHECK_LAUNCH();
  sample_ws_kernel<T, true><<<grid, threads, T::SMEM_BYTES, s>>>(g, dmap, w, pZ, ldp, (int)kchunk,
                                                               (int)nsplit, (int)tiles, row0, row1);
  HSS_CHECK_LAUNCH();
  unsigned rb = (unsigned)((nrows * w + 255) / 256);
  splitk_reduce_kernel<<<rb, 256, 0, s>>>(pY, (int)nsplit, nrows, w, ldp, Y, ldy);
  HSS_CHECK_LAUNCH();
  splitk_reduce_kernel<<<rb, 256, 0, s>>>(pZ, (int)nsplit, nrows, w, ldp, Z, ldy);
  HSS_CHECK_LAUNCH();
  return HSSEIG_OK;
}

// ---------------------------------------------------------------------------
// Materialised sampling: the Cauchy panel is generated once into HBM (FP64 pipe,
// HBM-write bound) and both products run on the TMA/DMMA engine without generator work
// competing for the FP64 issue slots:  Y_R = C[R, :] Omega   and   Z_R^T = Omega^T C[:, R].
// ---------------------------------------------------------------------------
constexpr double kMatCapBytes = 12.0 * (1 << 30);   // largest panel pair materialised
constexpr int64_t kPanelChunks = 4;

// out[i][j] = C[i0 + i][j0 + j] for i < ni, j < nj.  DIV (the dense update's panels): the
// reference's entry bit for bit, (zhat_i v_j) / gap with IEEE division; otherwise (the
// sample) the MUFU reciprocal + 2 Newton steps, within 2 ulp.  With g.lid set the entries of
// the diagonal leaf blocks (lid[i] == lid[j]) are zero: the off-diagonal sample.
template <bool DIV>
__global__ void gen_panel_kernel(CauchyGen g, int64_t i0, int64_t ni, int64_t j0, int64_t nj,
                                 double* __restrict__ out, int64_t ld) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nj) return;
  const int64_t gj = j0 + j;
  const double dj = __ldg(g.d + gj), dnj = __ldg(g.dnext + gj), gmj = __ldg(g.gam + gj);
  const double mj = __ldg(g.mu + gj), vj = __ldg(g.v + gj);
  const int lj = g.lid ? __ldg(g.lid + gj) : -1;
  for (int64_t i = blockIdx.y; i < ni; i += gridDim.y) {
    const int64_t gi = i0 + i;
    const double gap = stable_gap(gi, gj, __ldg(g.d + gi), dj, dnj, gmj, mj);
    double val = DIV ? (__ldg(g.zhat + gi) * vj) / gap : (__ldg(g.zhat + gi) * vj) * rcp_nr(gap);
    if (g.lid && __ldg(g.lid + gi) == lj) val = 0.0;
    out[i * ld + j] = val;
  }
}

// The sample's panel generator, rows [i0, i0 + ni) x columns [0, nj): each thread carries R
// independent rows of its column, so the dependent gap -> reciprocal -> scale chain of one
// entry (about nine FP64 operations) overlaps the other rows' and the stores of a row group
// leave together: 5.8 TB/s of HBM writes against 4.1 TB/s for one row per iteration
// (config 4: 0.52 -> 0.37 ms per 2.1 GB chunk).  Same arithmetic, entry for entry, as
// gen_panel_kernel<false>.  Work items are (128-column block, kPanelRowGroup-row group) pairs.
// (Measured and dropped: a grid small enough to stay co-resident with the persistent DMMA
// CTAs of the previous chunk's products -- the generator's FP64 chain then slows the products
// by as much as the overlap saves, tools/round2_an.sh.)
constexpr int kPanelRowGroup = 64;
template <int R>
__global__ void __launch_bounds__(128, 7)
    gen_panel_rows_kernel(CauchyGen g, int64_t i0, int64_t ni, int64_t nj,
                          double* __restrict__ out, int64_t ld) {
  const int64_t gx = (nj + 127) / 128, gyn = (ni + kPanelRowGroup - 1) / kPanelRowGroup;
  for (int64_t t = blockIdx.x; t < gx * gyn; t += gridDim.x) {
    const int64_t gj = (t % gx) * 128 + threadIdx.x;
    if (gj >= nj) continue;
    const int64_t ib = (t / gx) * kPanelRowGroup;
    const int64_t ie = ib + kPanelRowGroup < ni ? ib + kPanelRowGroup : ni;
    const double dj = __ldg(g.d + gj), dnj = __ldg(g.dnext + gj), gmj = __ldg(g.gam + gj);
    const double mj = __ldg(g.mu + gj), vj = __ldg(g.v + gj);
    const int lj = g.lid ? __ldg(g.lid + gj) : -1;
    int64_t i = ib;
    for (; i + R <= ie; i += R) {
      double di[R], zi[R], val[R];
      int li[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        di[r] = __ldg(g.d + i0 + i + r);
        zi[r] = __ldg(g.zhat + i0 + i + r);
        li[r] = g.lid ? __ldg(g.lid + i0 + i + r) : -2;
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double gap = stable_gap(i0 + i + r, gj, di[r], dj, dnj, gmj, mj);
        val[r] = (zi[r] * vj) * rcp_nr(gap);
        if (li[r] == lj) val[r] = 0.0;
      }
#pragma unroll
      for (int r = 0; r < R; ++r) out[(i + r) * ld + gj] = val[r];
    }
    for (; i < ie; ++i) {
      const int64_t gi = i0 + i;
      const double gap = stable_gap(gi, gj, __ldg(g.d + gi), dj, dnj, gmj, mj);
      double val = (__ldg(g.zhat + gi) * vj) * rcp_nr(gap);
      if (g.lid && __ldg(g.lid + gi) == lj) val = 0.0;
      out[i * ld + gj] = val;
    }
  }
}

static void gen_panel_rows(const CauchyGen& g, int64_t i0, int64_t ni, int64_t nj, double* out,
                           int64_t ld, cudaStream_t s) {
  const int64_t items = ((nj + 127) / 128) * ((ni + kPanelRowGroup - 1) / kPanelRowGroup);
  if (items <= 0) return;
  gen_panel_rows_kernel<8><<<(unsigned)imin64(items, 1 << 20), 128, 0, s>>>(g, i0, ni, nj, out, ld);
}

// out[c][i] = in[i][c]  (Omega^T, w x k)
__global__ void transpose_kernel(const double* __restrict__ in, int64_t ldi, int64_t rows, int w,
                                 double* __restrict__ out, int64_t ldo) {
  __shared__ double t[32][33];
  const int64_t i0 = (int64_t)blockIdx.x * 32;
  const int c0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t i = i0 + r;
    const int c = c0 + threadIdx.x;
    t[r][threadIdx.x] = (i < rows && c < w) ? in[i * ldi + c] : 0.0;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int c = c0 + r;
    const int64_t i = i0 + threadIdx.x;
    if (c < w && i < rows) out[(int64_t)c * ldo + i] = t[threadIdx.x][r];
  }
}

// Peer destinations of a fused gather: the reduced value of a row of this rank's block goes
// straight to row (row0 + row) of every rank's full buffer (IPC-mapped over NVLink), so the
// split-K reduction and the all-gather are one kernel; a system-scope fence publishes the
// stores before the kernel retires (then the group fences: distributed.peer_fence).
struct PeerOut {
  const uint64_t* base;   // npeers device pointers (this rank's own buffer included)
  int npeers;
  int64_t row0, ld;
};

__device__ __forceinline__ void peer_store(const PeerOut& po, int64_t row, int col, double v) {
  for (int q = 0; q < po.npeers; ++q)
    reinterpret_cast<double*>(po.base[q])[(po.row0 + row) * po.ld + col] = v;
}

__global__ void splitk_reduce_peers_kernel(const double* __restrict__ part, int nsplit, int64_t k,
                                           int w, int64_t ldp, PeerOut po) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < k * w) {
    int64_t row = e / w;
    int col = (int)(e % w);
    double s = 0.0;
    for (int t = 0; t < nsplit; ++t) s += part[(int64_t)t * k * ldp + row * ldp + col];
    peer_store(po, row, col, s);
  }
  __threadfence_system();
}

__global__ void splitk_reduce_t_peers_kernel(const double* __restrict__ part, int nsplit,
                                             int64_t nrows, int w, int64_t ldp, int64_t pstride,
                                             PeerOut po) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < nrows * w) {
    const int c = (int)(e / nrows);
    const int64_t row = e % nrows;
    double acc = 0.0;
    for (int p = 0; p < nsplit; ++p) acc += part[(int64_t)p * pstride + (int64_t)c * ldp + row];
    peer_store(po, row, c, acc);
  }
  __threadfence_system();
}

// Z[row][c] = sum_p part[p][c][row], p ascending (fixed order)
__global__ void splitk_reduce_t_kernel(const double* __restrict__ part, int nsplit, int64_t nrows,
                                       int w, int64_t ldp, int64_t pstride, double* __restrict__ Z,
                                       int64_t ldz) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nrows * w) return;
  const int c = (int)(e / nrows);
  const int64_t row = e % nrows;
  double acc = 0.0;
  for (int p = 0; p < nsplit; ++p) acc += part[(int64_t)p * pstride + (int64_t)c * ldp + row];
  Z[row * ldz + c] = acc;
}

struct MatPlan {
  int64_t nrows, kld, nld, ldp, sy, sz, kcy, kcz, tiles_n, nch;
  int64_t off_py, off_pz, off_omt, off_c1, off_c2, off_jobs, off_maps, total;
  bool shared;   // C[R, :] and C[:, R] are the same panel (R = all rows)
  // panel row chunk c (shared panel): rows [row_of(c), row_of(c + 1)), Z splits
  // [zsplit_of(c), zsplit_of(c + 1)) -- chunk bounds are Z split-K bounds
  __host__ __device__ int64_t zsplit_of(int64_t c) const { return c * sz / nch; }
  __host__ __device__ int64_t row_of(int64_t c) const {
    const int64_t r = zsplit_of(c) * kcz;
    return r < nrows ? r : nrows;
  }
};

// Split-K factor for a persistent launch of tiles x ns work items on one CTA per SM.
// Accuracy first: every split sums at most ~512 terms of K in its DMMA accumulators before
// the fixed-order reduction adds the partials, so the sample's rounding noise stays low --
// the interpolative decompositions truncate at 1e-15 relative, near that noise, and a
// cleaner sample gives measurably lower tree ranks (config 4: leaf / level-6 ranks
// 40 / 66 with 4 splits, 34 / 48 with 64; the multiply does 19% fewer flops).  Among the
// split counts with at least ~512 columns of K each (at most 64), the largest whose items
// fill at least three whole-ish waves (>= 97% of the last wave busy) is taken.
static void split_k(int64_t k, int64_t tiles, int64_t* ns, int64_t* kc) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms < 1) sms = 148;
  }
  const int64_t nmax = imax64(1, imin64(64, k / 512));
  int64_t best = 1;
  double best_eff = -1.0;
  for (int64_t n = nmax; n >= 1; --n) {
    const int64_t items = tiles * n;
    const int64_t waves = (items + sms - 1) / sms;
    const double eff = (double)items / (double)(waves * sms) - (waves < 3 ? 0.5 : 0.0);
    if (eff >= 0.97) { best = n; break; }
    if (eff > best_eff) { best_eff = eff; best = n; }
  }
  int64_t c = (k + best - 1) / best;
  c = (c + 15) / 16 * 16;
  *ns = (k + c - 1) / c;
  *kc = c;
}

static MatPlan mat_plan(int64_t k, int64_t w, int64_t nrows) {
  MatPlan p;
  p.nrows = nrows;
  p.shared = nrows == k;
  p.kld = k + (k & 1);
  p.nld = nrows + (nrows & 1);
  p.ldp = ((w + 1) / 2) * 2;
  // the shared panel is generated in row chunks on a side stream, each chunk's products
  // starting as soon as it is written (the HBM-bound generation hides under the DMMA-bound
  // products of the previous chunk); the split-K factors are sized for one chunk's tiles
  p.tiles_n = (nrows + 127) / 128;
  const int64_t chunks = p.shared ? kPanelChunks : 1;
  const int64_t ctiles = (p.tiles_n + chunks - 1) / chunks;
  split_k(k, ctiles, &p.sy, &p.kcy);
  // Z^T: a chunk's launch holds (its q splits) x tiles_n items; q is picked for one chunk's
  // K range, and every chunk gets q splits
  int64_t q, kcq;
  split_k((k + chunks - 1) / chunks, p.tiles_n, &q, &kcq);
  p.kcz = (((k + q * chunks - 1) / (q * chunks)) + 15) / 16 * 16;
  p.sz = (k + p.kcz - 1) / p.kcz;
  p.nch = imin64(chunks, p.sz);
  int64_t o = 0;
  auto take = [&](int64_t n) { int64_t at = o; o += (n + 31) / 32 * 32; return at; };
  p.off_py = take(p.sy * nrows * p.ldp);
  p.off_pz = take(p.sz * w * p.nld);
  p.off_omt = take(w * p.kld);
  p.off_c1 = take(nrows * p.kld);
  p.off_c2 = p.shared ? p.off_c1 : take(k * p.nld);
  p.off_jobs = take(((p.nch * p.sy + p.sz * p.tiles_n) * (int64_t)sizeof(TJob) + 7) / 8);
  p.off_maps = take((p.nch + 1) * (int64_t)sizeof(MapSet) / 8 + 32);
  p.total = o;
  return p;
}

static bool mat_fits(int64_t k, int64_t nrows) {
  const double bytes = 8.0 * (double)nrows * (double)k * (nrows == k ? 1.0 : 2.0);
  return bytes <= kMatCapBytes;
}

// Y jobs: chunk-major (chunk c, K split q) with the chunk's rows; then Z^T jobs
// (split qq, column tile t), split-major so a chunk's Z jobs are contiguous.
__global__ void mat_jobs_kernel(TJob* __restrict__ jobs, MatPlan p, int64_t k, int w, double* pY,
                                double* pZ) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nr = p.nrows;
  if (q >= p.nch * p.sy + p.sz * p.tiles_n) return;
  TJob jb;
  jb.am[0] = jb.am[1] = 0;
  jb.acol[1] = 0; jb.K[1] = 0;
  jb.bm[0] = jb.bm[1] = 4;
  jb.brow[1] = jb.bcol[1] = 0;
  if (q < p.nch * p.sy) {
    const int64_t c = q / p.sy, sp = q % p.sy;
    jb.acol[0] = (int32_t)(sp * p.kcy); jb.K[0] = (int32_t)imin64(p.kcy, k - sp * p.kcy);
    jb.brow[0] = (int32_t)(sp * p.kcy); jb.bcol[0] = 0;
    jb.N = jb.SW = w;
    jb.C = pY + sp * nr * p.ldp + p.row_of(c) * p.ldp;
    jb.ldc = p.ldp;
  } else {
    const int64_t e = q - p.nch * p.sy;
    const int64_t qq = e / p.tiles_n, t = e % p.tiles_n;
    jb.acol[0] = (int32_t)(qq * p.kcz); jb.K[0] = (int32_t)imin64(p.kcz, k - qq * p.kcz);
    jb.brow[0] = (int32_t)(qq * p.kcz); jb.bcol[0] = (int32_t)(t * 128);
    jb.N = jb.SW = (int32_t)imin64(128, nr - t * 128);
    jb.C = pZ + qq * w * p.nld + t * 128;
    jb.ldc = p.nld;
  }
  jobs[q] = jb;
}

// side stream + events of the chunked panel generation (one set per process: the library
// drives one device per process)
struct PanelSide {
  cudaStream_t s = nullptr;
  cudaEvent_t in = nullptr, gen[kPanelChunks] = {}, ygemm[kPanelChunks] = {}, yred = nullptr;
  bool ok = false;
  PanelSide() {
    ok = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) == cudaSuccess &&
         cudaEventCreateWithFlags(&in, cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&yred, cudaEventDisableTiming) == cudaSuccess;
    for (int c = 0; ok && c < kPanelChunks; ++c)
      ok = cudaEventCreateWithFlags(&gen[c], cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&ygemm[c], cudaEventDisableTiming) == cudaSuccess;
  }
};

static int launch_sample_mat(const CauchyGen& g, const double* om, int64_t ldom, int w, int64_t row0,
                             int64_t row1, double* Y, double* Z, int64_t ldy, double* work,
                             cudaStream_t s, const PeerOut* peY = nullptr,
                             const PeerOut* peZ = nullptr) {
  const int64_t k = g.k;
  const MatPlan p = mat_plan(k, w, row1 - row0);
  const int64_t nr = p.nrows;
  double* pY = work + p.off_py;
  double* pZ = work + p.off_pz;
  double* omt = work + p.off_omt;
  double* C1 = work + p.off_c1;
  double* C2 = work + p.off_c2;
  TJob* djobs = reinterpret_cast<TJob*>(work + p.off_jobs);
  MapSet* dmaps = reinterpret_cast<MapSet*>(
      (reinterpret_cast<uintptr_t>(work + p.off_maps) + 255) & ~(uintptr_t)255);
  const Operand none{nullptr, 0, 0, 0};
  const int njobs = (int)(p.nch * p.sy + p.sz * p.tiles_n);
  int rc;
  bool y_early = false;
  // Omega^T and the job tables (built on the device)
  dim3 gt((unsigned)((k + 31) / 32), (unsigned)((w + 31) / 32));
  transpose_kernel<<<gt, dim3(32, 8), 0, s>>>(om, ldom, k, w, omt, p.kld);
  HSS_CHECK_LAUNCH();
  mat_jobs_kernel<<<(njobs + 127) / 128, 128, 0, s>>>(djobs, p, k, w, pY, pZ);
  HSS_CHECK_LAUNCH();
  auto z_gemm = [&](int64_t c) -> int {
    const int64_t q0 = p.zsplit_of(c), q1 = p.zsplit_of(c + 1);
    if (q1 <= q0) return HSSEIG_OK;
    const Operand ops[kMaps] = {Operand{omt, (uint64_t)w, (uint64_t)k, (uint64_t)p.kld}, none, none,
                                none, Operand{C2, (uint64_t)k, (uint64_t)nr, (uint64_t)p.nld}, none,
                                none, none};
    return tma_jobs_gemm(2, w, ops, dmaps + p.nch, djobs + p.nch * p.sy + q0 * p.tiles_n,
                         (int)((q1 - q0) * p.tiles_n), w, s);
  };
  if (p.shared) {
    static PanelSide side;
    if (!side.ok) return HSSEIG_ERR_CUDA;
    // generators and the panel's previous readers are ordered before the first chunk
    if (cudaEventRecord(side.in, s) != cudaSuccess || cudaStreamWaitEvent(side.s, side.in, 0) != cudaSuccess)
      return HSSEIG_ERR_CUDA;
    for (int64_t c = 0; c < p.nch; ++c) {
      const int64_t r0 = p.row_of(c), r1 = p.row_of(c + 1);
      if (r1 > r0) {
        gen_panel_rows(g, row0 + r0, r1 - r0, k, C1 + r0 * p.kld, p.kld, side.s);
        HSS_CHECK_LAUNCH();
      }
      if (cudaEventRecord(side.gen[c], side.s) != cudaSuccess) return HSSEIG_ERR_CUDA;
    }
    for (int64_t c = 0; c < p.nch; ++c) {
      const int64_t r0 = p.row_of(c), r1 = p.row_of(c + 1);
      if (cudaStreamWaitEvent(s, side.gen[c], 0) != cudaSuccess) return HSSEIG_ERR_CUDA;
      if (r1 <= r0) continue;
      const Operand ops[kMaps] = {Operand{C1 + r0 * p.kld, (uint64_t)(r1 - r0), (uint64_t)k,
                                          (uint64_t)p.kld},
                                  none, none, none, Operand{om, (uint64_t)k, (uint64_t)w, (uint64_t)ldom},
                                  none, none, none};
      if ((rc = tma_jobs_gemm(0, w, ops, dmaps + c, djobs + c * p.sy, (int)p.sy, r1 - r0, s)))
        return rc;
      if (!peY) {
        // this chunk's rows of Y are reduced on the side stream (idle once the panel is
        // written) under the DMMA-bound Z^T products instead of after them
        if (cudaEventRecord(side.ygemm[c], s) != cudaSuccess ||
            cudaStreamWaitEvent(side.s, side.ygemm[c], 0) != cudaSuccess)
          return HSSEIG_ERR_CUDA;
        splitk_reduce_rows_kernel<<<(unsigned)(((r1 - r0) * w + 255) / 256), 256, 0, side.s>>>(
            pY, (int)p.sy, nr * p.ldp, r0, r1 - r0, w, p.ldp, Y, ldy);
        HSS_CHECK_LAUNCH();
        y_early = true;
      }
      if ((rc = z_gemm(c))) return rc;
    }
    if (y_early && (cudaEventRecord(side.yred, side.s) != cudaSuccess ||
                    cudaStreamWaitEvent(s, side.yred, 0) != cudaSuccess))
      return HSSEIG_ERR_CUDA;
  } else {
    gen_panel_rows(g, row0, nr, k, C1, p.kld, s);
    HSS_CHECK_LAUNCH();
    dim3 g2((unsigned)((nr + 255) / 256), (unsigned)imin64(k, 128));
    gen_panel_kernel<false><<<g2, 256, 0, s>>>(g, 0, k, row0, nr, C2, p.nld);
    HSS_CHECK_LAUNCH();
    const Operand ops[kMaps] = {Operand{C1, (uint64_t)nr, (uint64_t)k, (uint64_t)p.kld}, none, none,
                                none, Operand{om, (uint64_t)k, (uint64_t)w, (uint64_t)ldom}, none,
                                none, none};
    if ((rc = tma_jobs_gemm(0, w, ops, dmaps, djobs, (int)p.sy, nr, s))) return rc;
    if ((rc = z_gemm(0))) return rc;
  }
  const unsigned rb = (unsigned)((nr * w + 255) / 256);
  if (peY) {   // fused with the all-gather: rows land in every rank's full Y / Z
    splitk_reduce_peers_kernel<<<rb, 256, 0, s>>>(pY, (int)p.sy, nr, w, p.ldp, *peY);
    HSS_CHECK_LAUNCH();
    splitk_reduce_t_peers_kernel<<<rb, 256, 0, s>>>(pZ, (int)p.sz, nr, w, p.nld, w * p.nld, *peZ);
    HSS_CHECK_LAUNCH();
    return HSSEIG_OK;
  }
  if (!y_early) {
    splitk_reduce_kernel<<<rb, 256, 0, s>>>(pY, (int)p.sy, nr, w, p.ldp, Y, ldy);
    HSS_CHECK_LAUNCH();
  }
  splitk_reduce_t_kernel<<<rb, 256, 0, s>>>(pZ, (int)p.sz, nr, w, p.nld, w * p.nld, Z, ldy);
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
  if (!gen || nr < 0 || nc < 0 || ldo < nc) HSS_ARG_FAIL();
  if (nr == 0 || nc == 0) return HSSEIG_OK;
  int64_t n = nr * nc;
  cauchy_block_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      to_gen(gen), rows, nr, cols, nc, out, ldo);
  HSS_CHECK_LAUNCH();
  return HSSEIG_OK;
}

extern "C" int64_t hsseig_sample_work_doubles(int64_t k, int64_t w) {
  // covers every row range: nsplit * nrows is maximal for the full range
  int64_t worst = 0;
  for (int64_t nrows = k; nrows >= 1; nrows = nrows / 2) {
    int64_t nsplit, kchunk;
    sample_split(k, nrows, 64, &nsplit, &kchunk);
    worst = imax64(worst, nsplit * nrows);
    if (nrows == 1) break;
  }
  const int64_t ldp = ((w + 1) / 2) * 2;
  int64_t need = 2 * (worst + 64) * ldp + (int64_t)(sizeof(MapSet) + 512) / 8;
  if (w <= 112) {   // materialised path: the full range, and the largest partial range that fits
    if (mat_fits(k, k)) need = imax64(need, mat_plan(k, w, k).total + 64);
    const int64_t np = imin64(k - 1, (int64_t)(kMatCapBytes / (16.0 * (double)k)));
    if (np >= 1) need = imax64(need, mat_plan(k, w, np).total + 64);
  }
  return need;
}

extern "C" int hsseig_cauchy_sample_part(const hsseig_gen* gen, const int32_t* leaf_of,
                                         const double* omega, int64_t ldom, int64_t w, int64_t row0,
                                         int64_t row1, double* Y, double* Z, int64_t ldy,
                                         double* work, void* stream) {
  if (!gen || w < 1 || w > 128 || ldom < w || ldy < w || row0 < 0 || row1 > gen->k || row0 > row1)
    HSS_ARG_FAIL();
  if ((reinterpret_cast<uintptr_t>(omega) & 15) || (ldom & 1)) HSS_ARG_FAIL();  // TMA rows
  if (row0 == row1) return HSSEIG_OK;
  CauchyGen g = to_gen(gen);
  g.lid = leaf_of;
  cudaStream_t s = (cudaStream_t)stream;
  static const bool fused_only = getenv("HSSEIG_SAMPLE_FUSED") != nullptr;
  if (!fused_only && w <= 112 && mat_fits(gen->k, row1 - row0) &&
      (reinterpret_cast<uintptr_t>(work) & 15) == 0)
    return launch_sample_mat(g, omega, ldom, (int)w, row0, row1, Y, Z, ldy, work, s);
  switch ((w + 31) / 32) {   // BM 64: 8 DMMA warps of 32 x 8NF + 8 generator warps
    case 1: return launch_sample<TTile<4, 1, 2, 4, 8>>(g, omega, ldom, (int)w, row0, row1, Y, Z, ldy, work, s);
    case 2: return launch_sample<TTile<4, 2, 2, 4, 8>>(g, omega, ldom, (int)w, row0, row1, Y, Z, ldy, work, s);
    case 3: return launch_sample<TTile<4, 3, 2, 4, 8>>(g, omega, ldom, (int)w, row0, row1, Y, Z, ldy, work, s);
    default: return launch_sample<TTile<4, 4, 2, 4, 6>>(g, omega, ldom, (int)w, row0, row1, Y, Z, ldy, work, s);
  }
}

// Rows [row0, row1) of Y and Z written straight into every rank's full Y / Z (row-major,
// leading dimension ldy): the split-K reductions store to the peers' IPC-mapped buffers.
extern "C" int hsseig_cauchy_sample_part_peers(const hsseig_gen* gen, const int32_t* leaf_of,
                                               const double* omega, int64_t ldom, int64_t w,
                                               int64_t row0, int64_t row1, const uint64_t* Yp,
                                               const uint64_t* Zp, int32_t npeers, int64_t ldy,
                                               double* work, void* stream) {
  if (!gen || w < 1 || w > 112 || ldom < w || ldy < w || row0 < 0 || row1 > gen->k ||
      row0 > row1 || !Yp || !Zp || npeers < 1 || !work)
    HSS_ARG_FAIL();
  if ((reinterpret_cast<uintptr_t>(omega) & 15) || (ldom & 1) ||
      (reinterpret_cast<uintptr_t>(work) & 15))
    HSS_ARG_FAIL();
  if (!mat_fits(gen->k, row1 - row0)) HSS_ARG_FAIL();   // the materialised path only
  if (row0 == row1) return HSSEIG_OK;
  const PeerOut py{Yp, npeers, row0, ldy}, pz{Zp, npeers, row0, ldy};
  CauchyGen g = to_gen(gen);
  g.lid = leaf_of;
  return launch_sample_mat(g, omega, ldom, (int)w, row0, row1, nullptr, nullptr, ldy, work,
                           (cudaStream_t)stream, &py, &pz);
}

// Whether hsseig_cauchy_sample_part_peers takes a row range of `nrows` rows of an order-k
// system at sample width w.  Monotone in nrows, so ranks that test the padded shard size they
// all share reach the same decision before anything is launched.
extern "C" int hsseig_sample_peers_fits(int64_t k, int64_t nrows, int64_t w) {
  return (k >= 1 && nrows >= 0 && nrows <= k && w >= 1 && w <= 112 && mat_fits(k, nrows)) ? 1 : 0;
}

extern "C" int hsseig_cauchy_sample(const hsseig_gen* gen, const int32_t* leaf_of,
                                    const double* omega, int64_t ldom, int64_t w, double* Y,
                                    double* Z, int64_t ldy, double* work, void* stream) {
  if (!gen) HSS_ARG_FAIL();
  return hsseig_cauchy_sample_part(gen, leaf_of, omega, ldom, w, 0, gen->k, Y, Z, ldy, work,
                                   stream);
}

extern "C" int hsseig_dense_update(const double* Qb, int64_t ldq, int64_t P, const hsseig_gen* gen,
                                   double* out, int64_t ldo, void* stream) {
  if (!gen || P < 0 || ldq < gen->k || ldo < gen->k) HSS_ARG_FAIL();
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

extern "C" int hsseig_wave_dense_update(const double* W, const int64_t* woff, const int64_t* nrow,
                                        const int64_t* ldw,
                                        const double* d, const double* dnext, const double* gamma,
                                        const double* mu, const double* zhat, const double* v,
                                        const int64_t* koff, double* out, const int64_t* ooff,
                                        const int32_t* tasks, int64_t ntasks, void* stream) {
  if (ntasks < 0 || !W || !woff || !nrow || !ldw || !koff || !out || !ooff || !tasks) HSS_ARG_FAIL();
  if (ntasks == 0) return HSSEIG_OK;
  using T = Tile<4, 8, 4, 2, 2>;
  const size_t smem = sizeof(double) * T::STAGE_ELEMS * 2;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(wave_dense_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  CauchyGen g;
  g.d = d; g.dnext = dnext; g.gam = gamma; g.mu = mu; g.zhat = zhat; g.v = v; g.k = 0;
  wave_dense_kernel<T><<<(unsigned)ntasks, T::THREADS, smem, (cudaStream_t)stream>>>(
      W, woff, nrow, ldw, g, koff, out, ooff, tasks);
  HSS_CHECK_LAUNCH();
  return HSSEIG_OK;
}

extern "C" int hsseig_wave_tile_shape(int32_t* bm, int32_t* bn) {
  using T = Tile<4, 8, 4, 2, 2>;
  *bm = T::BM;
  *bn = T::BN;
  return HSSEIG_OK;
}

// Dense update out = Qb C through materialised column panels of C (the reference's
// to_dense entries) and the TMA/DMMA engine; falls back to the fused kernel when the
// workspace is too small.  work: hsseig_dense_update_work_doubles(k, panel_cols).
static int64_t dense_ws_overhead(int64_t k) {
  return ((k + 127) / 128 * (int64_t)sizeof(TJob) + 7) / 8 + (int64_t)(sizeof(MapSet) + 512) / 8 + 64;
}

extern "C" int64_t hsseig_dense_update_work_doubles(int64_t k, int64_t panel_cols) {
  if (k < 1 || panel_cols < 1) return -1;
  const int64_t kc = imin64(k, (panel_cols + 127) / 128 * 128);
  return k * (kc + (kc & 1)) + dense_ws_overhead(k);
}

extern "C" int hsseig_dense_update_ws(const double* Qb, int64_t ldq, int64_t P,
                                      const hsseig_gen* gen, double* out, int64_t ldo,
                                      double* work, int64_t work_doubles, void* stream) {
  if (!gen || P < 0 || ldq < gen->k || ldo < gen->k) HSS_ARG_FAIL();
  if (P == 0) return HSSEIG_OK;
  const int64_t k = gen->k;
  const bool aligned = !(reinterpret_cast<uintptr_t>(Qb) & 15) && !(ldq & 1) &&
                       !(reinterpret_cast<uintptr_t>(work) & 15);
  int64_t kc = work ? (work_doubles - dense_ws_overhead(k)) / (k + 1) : 0;
  kc = imin64(k, kc / 128 * 128);
  if (k < 512 || !aligned || kc < 128)
    return hsseig_dense_update(Qb, ldq, P, gen, out, ldo, stream);
  const int64_t ldp = kc + (kc & 1);
  double* panel = work;
  TJob* jobs = reinterpret_cast<TJob*>(work + k * ldp);
  MapSet* dmaps = reinterpret_cast<MapSet*>(
      (reinterpret_cast<uintptr_t>(jobs + (k + 127) / 128) + 255) & ~(uintptr_t)255);
  CauchyGen g = to_gen(gen);
  cudaStream_t s = (cudaStream_t)stream;
  for (int64_t c0 = 0; c0 < k; c0 += kc) {
    const int64_t nc = imin64(kc, k - c0);
    dim3 gr((unsigned)((nc + 255) / 256), (unsigned)imin64(k, 128));
    gen_panel_kernel<true><<<gr, 256, 0, s>>>(g, 0, k, c0, nc, panel, ldp);
    HSS_CHECK_LAUNCH();
    const int rc = tma_plain_gemm(Qb, ldq, panel, ldp, out + c0, ldo, P, nc, k, jobs, dmaps, s);
    if (rc) return rc;
  }
  return HSSEIG_OK;
}

// ---------------------------------------------------------------------------
// Dense update of a DC merge without the structural zeros (the dlaed3 observation): the
// merge's eigenvector block is blockdiag(Q1, Q2) with permuted columns, so a kept column
// that comes from child 1 and that no deflation rotation touched is zero below row n1, and
// a child-2 column is zero above it.  perm orders the k kept columns as
// [child 1 only | rotated (dense) | child 2 only]; the top n1 rows then contract over
// perm[0, ka) only and the bottom rows over perm[kb, k):
//   out[0:n1, :]  = W[0:n1, perm[0:ka]]  C[perm[0:ka], :]
//   out[n1:P, :]  = W[n1:P, perm[kb:k]]  C[perm[kb:k], :]
// -- about half the flops of out = W C, with exactly the terms that are not products with a
// structural zero.  The two row blocks of W are compacted once, C's panels are generated
// with their rows in perm order (entries as gen_panel_kernel<true>, the reference's
// to_dense values) and both products run on the TMA/DMMA engine.
// ---------------------------------------------------------------------------
__global__ void compact_halves_kernel(const double* __restrict__ W, int64_t ldw, int64_t P,
                                      int64_t n1, const int64_t* __restrict__ perm, int64_t ka,
                                      int64_t kb, int64_t k, double* __restrict__ top,
                                      int64_t ldt, double* __restrict__ bot, int64_t ldb) {
  for (int64_t r = blockIdx.x; r < P; r += gridDim.x) {
    const double* w = W + r * ldw;
    if (r < n1) {
      double* o = top + r * ldt;
      for (int64_t c = threadIdx.x; c < ka; c += blockDim.x) o[c] = w[__ldg(perm + c)];
    } else {
      double* o = bot + (r - n1) * ldb;
      for (int64_t c = threadIdx.x; c < k - kb; c += blockDim.x) o[c] = w[__ldg(perm + kb + c)];
    }
  }
}

// panel[i][j] = C[perm[i]][j0 + j], i < k, j < nj: the reference's entry, IEEE division
__global__ void gen_panel_perm_kernel(CauchyGen g, const int64_t* __restrict__ perm, int64_t k,
                                      int64_t j0, int64_t nj, double* __restrict__ out,
                                      int64_t ld) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nj) return;
  const int64_t gj = j0 + j;
  const double dj = __ldg(g.d + gj), dnj = __ldg(g.dnext + gj), gmj = __ldg(g.gam + gj);
  const double mj = __ldg(g.mu + gj), vj = __ldg(g.v + gj);
  for (int64_t i = blockIdx.y; i < k; i += gridDim.y) {
    const int64_t gi = __ldg(perm + i);
    const double gap = stable_gap(gi, gj, __ldg(g.d + gi), dj, dnj, gmj, mj);
    out[i * ld + j] = (__ldg(g.zhat + gi) * vj) / gap;
  }
}

static int64_t even64(int64_t x) { return x + (x & 1); }

extern "C" int64_t hsseig_dense_update_halves_work_doubles(int64_t P, int64_t k,
                                                           int64_t panel_cols) {
  if (P < 1 || k < 1 || panel_cols < 1) return -1;
  return P * even64(k) + 64 + hsseig_dense_update_work_doubles(k, panel_cols);
}

extern "C" int hsseig_dense_update_halves(const double* Qb, int64_t ldq, int64_t P, int64_t n1,
                                          const hsseig_gen* gen, const int64_t* perm, int64_t ka,
                                          int64_t kb, double* out, int64_t ldo, double* work,
                                          int64_t work_doubles, void* stream) {
  if (!gen || !perm || P < 0 || n1 < 0 || n1 > P || ldq < gen->k || ldo < gen->k || ka < 0 ||
      kb < 0 || kb > ka || ka > gen->k || !work)
    HSS_ARG_FAIL();
  if (P == 0) return HSSEIG_OK;
  const int64_t k = gen->k, n2 = P - n1, kt = ka, kbn = k - kb;
  const int64_t ldt = even64(imax64(kt, 1)), ldb = even64(imax64(kbn, 1));
  const int64_t halves = ((n1 * ldt + n2 * ldb + 31) / 32) * 32;
  double* top = work;
  double* bot = work + n1 * ldt;
  double* rest = work + halves;
  int64_t kc = (work_doubles - halves - dense_ws_overhead(k)) / (k + 1);
  kc = imin64(k, kc / 128 * 128);
  if ((reinterpret_cast<uintptr_t>(work) & 15) || kc < 128) HSS_ARG_FAIL();
  const int64_t ldp = kc + (kc & 1);
  double* panel = rest;
  TJob* jobs = reinterpret_cast<TJob*>(rest + k * ldp);
  MapSet* dmaps = reinterpret_cast<MapSet*>(
      (reinterpret_cast<uintptr_t>(jobs + (k + 127) / 128) + 255) & ~(uintptr_t)255);
  CauchyGen g = to_gen(gen);
  cudaStream_t s = (cudaStream_t)stream;
  compact_halves_kernel<<<(unsigned)imin64(P, 1 << 20), 256, 0, s>>>(Qb, ldq, P, n1, perm, ka, kb, k,
                                                                   top, ldt, bot, ldb);
  HSS_CHECK_LAUNCH();
  for (int64_t c0 = 0; c0 < k; c0 += kc) {
    const int64_t nc = imin64(kc, k - c0);
    dim3 gr((unsigned)((nc + 255) / 256), (unsigned)imin64(k, 128));
    gen_panel_perm_kernel<<<gr, 256, 0, s>>>(g, perm, k, c0, nc, panel, ldp);
    HSS_CHECK_LAUNCH();
    int rc;
    if (n1 > 0) {
      if (kt > 0) {
        if ((rc = tma_plain_gemm(top, ldt, panel, ldp, out + c0, ldo, n1, nc, kt, jobs, dmaps, s)))
          return rc;
      } else if (cudaMemset2DAsync(out + c0, ldo * 8, 0, nc * 8, n1, s) != cudaSuccess) {
        return HSSEIG_ERR_CUDA;
      }
    }
    if (n2 > 0) {
      if (kbn > 0) {
        if ((rc = tma_plain_gemm(bot, ldb, panel + kb * ldp, ldp, out + n1 * ldo + c0, ldo, n2, nc,
                                 kbn, jobs, dmaps, s)))
          return rc;
      } else if (cudaMemset2DAsync(out + n1 * ldo + c0, ldo * 8, 0, nc * 8, n2, s) != cudaSuccess) {
        return HSSEIG_ERR_CUDA;
      }
    }
  }
  return HSSEIG_OK;
}

// Every panel update of one recursion depth in one call (the host loop in C: ~25 us of
// ctypes overhead per merge otherwise).  rec (host, 9 int64 per merge): W offset, ldw, rows,
// n1, generator offset, k, ka, kb, out offset; perm holds the merges' K orders back to back.
// The updates of a depth are independent and, below the top depths, each too small to fill
// the GPU (a 1024 x 600 update has 40 output tiles for 148 SMs): they are dealt round-robin
// to nstreams side streams (forked from / joined into `stream` by events), each with its own
// slice of the workspace (work_doubles / nstreams doubles).
namespace {
constexpr int kHalvesStreams = 8;
struct HalvesSide {
  cudaStream_t s[kHalvesStreams] = {};
  cudaEvent_t in = nullptr, done[kHalvesStreams] = {};
  bool ok = false;
  HalvesSide() {
    ok = cudaEventCreateWithFlags(&in, cudaEventDisableTiming) == cudaSuccess;
    for (int i = 0; ok && i < kHalvesStreams; ++i)
      ok = cudaStreamCreateWithFlags(&s[i], cudaStreamNonBlocking) == cudaSuccess &&
           cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming) == cudaSuccess;
  }
};
}  // namespace

extern "C" int hsseig_wave_dense_halves(int64_t nbig, const int64_t* rec, const double* W,
                                        const double* d, const double* dnext, const double* gamma,
                                        const double* mu, const double* zhat, const double* v,
                                        const int64_t* perm, double* out, double* work,
                                        int64_t work_doubles, int32_t nstreams, void* stream) {
  if (nbig < 0 || nstreams < 1 || (nbig > 0 && (!rec || !W || !perm || !out || !work)))
    HSS_ARG_FAIL();
  if (nbig == 0) return HSSEIG_OK;
  static HalvesSide side;
  const int ns = (int)imin64(imin64(nstreams, kHalvesStreams), nbig);
  const int64_t per = (work_doubles / ns) & ~int64_t(31);
  cudaStream_t main_s = (cudaStream_t)stream;
  if (ns > 1) {
    if (!side.ok) return HSSEIG_ERR_CUDA;
    if (cudaEventRecord(side.in, main_s) != cudaSuccess) return HSSEIG_ERR_CUDA;
    for (int i = 0; i < ns; ++i)
      if (cudaStreamWaitEvent(side.s[i], side.in, 0) != cudaSuccess) return HSSEIG_ERR_CUDA;
  }
  int64_t po = 0;
  int rc = HSSEIG_OK;
  for (int64_t q = 0; q < nbig && rc == HSSEIG_OK; ++q) {
    const int64_t* r = rec + 9 * q;
    const int64_t go = r[4], k = r[5];
    hsseig_gen g{d + go, dnext + go, gamma + go, mu + go, zhat + go, v + go, k};
    const int lane = (int)(q % ns);
    rc = hsseig_dense_update_halves(W + r[0], r[1], r[2], r[3], &g, perm + po, r[6], r[7],
                                    out + r[8], k, work + lane * per, per,
                                    ns > 1 ? (void*)side.s[lane] : stream);
    po += k;
  }
  if (ns > 1) {   // join even after a failure so the caller's stream stays ordered
    for (int i = 0; i < ns; ++i)
      if (cudaEventRecord(side.done[i], side.s[i]) != cudaSuccess ||
          cudaStreamWaitEvent(main_s, side.done[i], 0) != cudaSuccess)
        return HSSEIG_ERR_CUDA;
  }
  return rc;
}
