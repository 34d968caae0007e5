// Randomized HSS construction (ADC2) on sm_100a, level by level.
//
// Reference path (pkg/src/hsseig/hss.py):
//   _build_skeleton           hss.py:188-214   -> hsseig_tree_layout (host topology)
//   rand_hss_construct        hss.py:217-306   -> leaf_form / genB / inner_form / id kernels
//   _interp_rows              hss.py:120-148   -> id_kernel: column-pivoted Householder QR of
//                                                 M^T following LAPACK dgeqp3/dlaqp2 (pivot on
//                                                 downdated norms, sqrt(eps) recompute rule),
//                                                 trailing-mass truncation, saturation flag,
//                                                 in-place dtrsm back substitution
// One CTA per (node, side): side 0 compresses the block row (Phi -> U, rows_sel),
// side 1 the block column (Theta -> V, cols_sel).  Every matrix an ID sees is at
// most (2w) x w, so it lives in shared memory for the whole factorization.
#include <cstdlib>
#include <vector>

#include "tree_dev.cuh"

namespace hsseig {

// ---------------------------------------------------------------------------
// leaf level: D = C(t,t);  Phi = Y_t - D Omega_t (side 0);  Theta = Z_t - D^T Omega_t (side 1)
// (hss.py:261-268)
// ---------------------------------------------------------------------------
// shared-memory strides that keep the DMMA fragment loads conflict-free: A (D chunk) rows
// at a stride of 4 (mod 8) doubles, B (Omega_t) rows at 8 or 24 (mod 32)
__host__ __device__ __forceinline__ int leaf_kp(int mmax) { return (mmax + 3) / 4 * 4; }
__host__ __device__ __forceinline__ int leaf_sd(int mmax) {
  const int kp = leaf_kp(mmax);
  return kp % 8 == 0 ? kp + 4 : kp;
}
__host__ __device__ __forceinline__ int leaf_so(int w) {
  int s = (w + 7) / 8 * 8;
  while (s % 32 != 8 && s % 32 != 24) s += 8;
  return s;
}
__global__ void __launch_bounds__(256) leaf_form_kernel(CauchyGen g, TreeDev T,
                                                        const double* __restrict__ om,
                                                        int64_t ldom,
                                                        const double* __restrict__ Y,
                                                        const double* __restrict__ Z,
                                                        int64_t ldy, int j0, int offdiag) {
  // D Omega_t on the DMMA pipe: 16-row chunks of D generated in shared memory (A operand,
  // row stride SD = 4 mod 8), Omega_t resident (B operand, row stride SO = 8|24 mod 32),
  // 2 x ceil(w/8) output fragments of 8 x 8 spread over the 8 warps, K padded to 4 with zeros
  extern __shared__ __align__(16) double sm[];
  const int j = j0 + blockIdx.x, side = blockIdx.y, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int node = T.lnodes[(1 << T.depth) - 1 + j];
  const int lo = T.lo[node], m = T.hi[node] - lo, w = T.w;
  constexpr int RA = 16;
  const int KP = leaf_kp(T.mmax), SO = leaf_so(w), SD = leaf_sd(T.mmax);
  const int kp = (m + 3) / 4 * 4, nf = (w + 7) / 8;
  double* sOm = sm;                       // KP x SO (rows >= m and columns >= w zero)
  double* sD = sm + (size_t)KP * SO;      // RA x SD chunk (columns >= m zero)
  for (int e = tid; e < kp * SO; e += blockDim.x) {
    const int b = e / SO, c = e % SO;
    sOm[e] = (b < m && c < w) ? om[(int64_t)(lo + b) * ldom + c] : 0.0;
  }
  const double* src = side == 0 ? Y : Z;
  double* Mo = T.M + (size_t)(2 * j + side) * T.pmax * T.ws;
  // D slot: drows x dld, row 0 and rows/cols past m are zero, D[a][b] at row a + 1
  const int drows = hsseig_drows(T.mmax);
  double* Dslot = T.D + (size_t)j * drows * T.dld;
  if (side == 0) {
    for (int e = tid; e < drows * T.dld; e += blockDim.x) {
      const int a = e / T.dld - 1, b = e % T.dld;
      if (a < 0 || a >= m || b >= m) Dslot[e] = 0.0;
    }
  }
  if (offdiag) {
    // off-diagonal sample: Y_t, Z_t already are Phi, Theta (no D Omega_t to subtract);
    // side 0 still generates D for the tree
    for (int e = tid; e < m * w; e += blockDim.x) {
      const int a = e / w, c = e % w;
      Mo[(size_t)a * T.ws + c] = src[(int64_t)(lo + a) * ldy + c];
    }
    if (side == 0) {
      for (int e = tid; e < m * m; e += blockDim.x) {
        const int a = e / m, b = e % m;
        Dslot[(size_t)(a + 1) * T.dld + b] = g.entry(lo + a, lo + b);
      }
    }
    return;
  }
  const int gr = lane >> 2, gc = lane & 3;
  for (int a0 = 0; a0 < m; a0 += RA) {
    const int na = min(RA, m - a0);
    __syncthreads();
    for (int e = tid; e < RA * kp; e += blockDim.x) {
      const int aa = e / kp, b = e % kp;
      double val = 0.0;
      if (aa < na && b < m) {
        val = side == 0 ? g.entry(lo + a0 + aa, lo + b) : g.entry(lo + b, lo + a0 + aa);
        if (side == 0) Dslot[(size_t)(a0 + aa + 1) * T.dld + b] = val;
      }
      sD[aa * SD + b] = val;
    }
    __syncthreads();
    for (int f = warp; f < 2 * nf; f += 8) {     // fragment (mi, ni) = (f / nf, f % nf)
      const int mi = f / nf, ni = f % nf;
      double c0 = 0.0, c1 = 0.0;
      const double* arow = sD + (mi * 8 + gr) * SD + gc;
      const double* bcol = sOm + gc * SO + ni * 8 + gr;
      for (int k0 = 0; k0 < kp; k0 += 4) dmma_8x8x4(c0, c1, arow[k0], bcol[k0 * SO]);
      const int r = mi * 8 + gr, c = ni * 8 + 2 * gc;
      if (r < na) {
        const int64_t yr = (int64_t)(lo + a0 + r) * ldy;
        double* mo = Mo + (size_t)(a0 + r) * T.ws;
        if (c < w) mo[c] = src[yr + c] - c0;
        if (c + 1 < w) mo[c + 1] = src[yr + c + 1] - c1;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// skeleton blocks of the children of every node at one level (hss.py:270-271, 299-301):
//   B_left = C(rows_sel(left), cols_sel(right)),  B_right = C(rows_sel(right), cols_sel(left))
// ---------------------------------------------------------------------------
__global__ void genB_kernel(CauchyGen g, TreeDev T, int level, int j0) {
  const int j = j0 + blockIdx.x, which = blockIdx.y, tid = threadIdx.x;
  const int node = T.lnodes[(1 << level) - 1 + j];
  const int a = T.left[node], b = T.right[node];
  const int me = which == 0 ? a : b, sib = which == 0 ? b : a;
  const int nr = T.rU[me], nc = T.rV[sib];
  const int32_t* rs = T.rsel + (size_t)me * T.ws;
  const int32_t* cs = T.csel + (size_t)sib * T.ws;
  double* Bo = T.B + slot_ww(T, me);
  // the whole ws x ws slot is written: zero padding makes K-tail chunks of the multiply exact
  for (int e = tid; e < T.ws * T.ws; e += blockDim.x) {
    int r = e / T.ws, c = e % T.ws;
    Bo[e] = (r < nr && c < nc) ? g.entry(rs[r], cs[c]) : 0.0;
  }
}

int launch_genB(const CauchyGen& g, const TreeDev& T, int level, int j0, int cnt, cudaStream_t s) {
  genB_kernel<<<dim3(cnt, 2), 256, 0, s>>>(g, T, level, j0);
  HSS_CHECK_LAUNCH();
  return HSSEIG_OK;
}

// ---------------------------------------------------------------------------
// inner level (hss.py:272-277):
//   Phi   = [ psel_a - B_a ycomp_b ; psel_b - B_b ycomp_a ]
//   Theta = [ tsel_a - B_b^T zcomp_b ; tsel_b - B_a^T zcomp_a ]
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) inner_form_kernel(TreeDev T, int level, int j0) {
  // one CTA per (node, side, half): rows [off, off + nrow) of Phi (side 0) or Theta (side 1).
  // B block and sibling compression are staged in shared memory.
  // blockIdx.z = half + 2 * (row chunk): upper levels have few nodes, so each half's rows
  // are split over gridDim.z / 2 CTAs (latency-bound otherwise)
  extern __shared__ __align__(16) double fs[];
  const int j = j0 + blockIdx.x, side = blockIdx.y, half = blockIdx.z & 1, tid = threadIdx.x;
  const int rc = blockIdx.z >> 1, nrc = gridDim.z >> 1;
  const int node = T.lnodes[(1 << level) - 1 + j];
  const int a = T.left[node], b = T.right[node], w = T.w, ws = T.ws;
  const int me = half == 0 ? a : b, sib = half == 0 ? b : a;
  const int na = side == 0 ? T.rU[a] : T.rV[a];
  const int nall = side == 0 ? T.rU[me] : T.rV[me];
  const int rchunk = (nall + nrc - 1) / nrc;
  const int r0 = min(nall, rc * rchunk);
  const int nrow = min(nall, r0 + rchunk) - r0;
  const int off = (half == 0 ? 0 : na) + r0;
  const int nk = side == 0 ? T.rV[sib] : T.rU[sib];
  double* Mo = T.M + (size_t)(2 * j + side) * T.pmax * ws;
  const double* comp = (side == 0 ? T.ycomp : T.zcomp) + slot_ww(T, sib);
  const double* sel = (side == 0 ? T.psel : T.tsel) + slot_ww(T, me);
  const double* Bb = T.B + slot_ww(T, side == 0 ? me : sib);
  // B_me rows (A operand, stride SA = 4 mod 8) times the sibling compression (B operand,
  // stride SO = 8|24 mod 32) on the DMMA pipe, K padded to 4 and rows to 8 with zeros
  const int kpm = (w + 3) / 4 * 4, SA = kpm % 8 == 0 ? kpm + 4 : kpm, SO = leaf_so(w);
  const int kp = (nk + 3) / 4 * 4, mr = (nrow + 7) / 8 * 8, nf = (w + 7) / 8;
  double* sBt = fs;                          // mr x SA  (B_me, or B_sib^T)
  double* sCm = fs + (size_t)((w + 7) / 8 * 8) * SA;   // kpm x SO
  for (int e = tid; e < mr * kp; e += blockDim.x) {
    const int r = e / kp, t = e % kp;
    sBt[r * SA + t] = (r < nrow && t < nk)
                          ? (side == 0 ? Bb[(size_t)(r0 + r) * ws + t] : Bb[(size_t)t * ws + r0 + r])
                          : 0.0;
  }
  for (int e = tid; e < kp * SO; e += blockDim.x) {
    const int t = e / SO, c = e % SO;
    sCm[e] = (t < nk && c < w) ? comp[(size_t)t * ws + c] : 0.0;
  }
  __syncthreads();
  const int lane = tid & 31, warp = tid >> 5, gr = lane >> 2, gc = lane & 3;
  for (int f = warp; f < (mr / 8) * nf; f += blockDim.x >> 5) {
    const int mi = f / nf, ni = f % nf;
    double c0 = 0.0, c1 = 0.0;
    const double* arow = sBt + (mi * 8 + gr) * SA + gc;
    const double* bcol = sCm + gc * SO + ni * 8 + gr;
    for (int k0 = 0; k0 < kp; k0 += 4) dmma_8x8x4(c0, c1, arow[k0], bcol[k0 * SO]);
    const int r = mi * 8 + gr, c = ni * 8 + 2 * gc;
    if (r < nrow) {
      const double* sr = sel + (size_t)(r0 + r) * ws;
      double* mo = Mo + (size_t)(off + r) * ws;
      if (c < w) mo[c] = sr[c] - c0;
      if (c + 1 < w) mo[c + 1] = sr[c + 1] - c1;
    }
  }
}

// LAPACK dlapy2: sqrt(x^2 + y^2) without destructive under/overflow
__device__ __forceinline__ double lapy2(double x, double y) {
  double xa = fabs(x), ya = fabs(y);
  double wv = fmax(xa, ya), zv = fmin(xa, ya);
  if (zv == 0.0) return wv;
  double q = zv / wv;
  return wv * sqrt(1.0 + q * q);
}

// Truncation of the factored A = M^T (hss.py:128-148): trailing Frobenius mass of R's
// rows, rank r = min(first t with tail(t) <= (tol ||M||_F)^2, max_rank, nonzero diagonal),
// saturation flag, relative residual, then T = R11^{-1} R12 in place (dtrsm L/U/N/N).
// `steps` reflectors were applied (id_eliminate); rows >= steps of R are not formed, their
// mass is the trailing block's Frobenius mass `trail` (orthogonal invariance: the rows the
// remaining reflectors would produce carry exactly that mass).
__device__ __forceinline__ void id_truncate(double* sA, double* tail, int p, int w, int SW,
                                            double nf, double tol, int max_rank, int steps,
                                            double trail, int& r, int& sat, double& resid) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int nthr = blockDim.x;
  __shared__ double s_resid;
  __shared__ int s_r, s_sat;
  r = 0;
  sat = 0;
  resid = 0.0;
  const int mn = min(steps, min(w, p));
  if (!(nf == 0.0 || p == 0 || w == 0)) {
    // trailing Frobenius mass of R's rows, cumulated from the bottom (hss.py:134-136)
    for (int t = warp; t < mn; t += nwarps) {
      double s = 0.0;
      for (int c = t + lane; c < p; c += 32) s = fma(sA[c * SW + t], sA[c * SW + t], s);
      s = warp_sum(s);
      if (lane == 0) tail[t] = s;
    }
    __syncthreads();
    if (tid == 0) {
      double acc = trail;
      tail[mn] = trail;
      for (int t = mn - 1; t >= 0; --t) {
        acc += tail[t];
        tail[t] = acc;
      }
      const double cut = (tol * nf) * (tol * nf);
      int wanted = mn;
      for (int t = 0; t <= mn; ++t)
        if (tail[t] <= cut) { wanted = t; break; }
      int nz = 0;
      for (int t = 0; t < mn; ++t) nz += (fabs(sA[t * SW + t]) > 0.0) ? 1 : 0;
      const int rr = min(min(wanted, max_rank), nz);
      s_r = rr;
      s_sat = (wanted >= max_rank && max_rank >= 1)
                  ? (sqrt(fmax(tail[max_rank - 1], 0.0)) > kFlagTol * nf ? 1 : 0)
                  : 0;
      s_resid = sqrt(fmax(tail[rr], 0.0)) / nf;
    }
    __syncthreads();
    r = s_r;
    sat = s_sat;
    resid = s_resid;
    // T = R[:r,:r]^{-1} R[:r, r:] in place, column-oriented back substitution (dtrsm L/U/N/N)
    for (int c = r + tid; c < p; c += nthr) {
      double* x = sA + c * SW;
      for (int t = r - 1; t >= 0; --t) {
        const double xt = x[t] / sA[t * SW + t];
        x[t] = xt;
        if (xt != 0.0) {
          const double* rc = sA + t * SW;
          int s2 = 0;
          for (; s2 + 7 < t; s2 += 8) {   // loads ahead of the stores (x, rc in one array)
            double rr[8], xx[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) { rr[u] = rc[s2 + u]; xx[u] = x[s2 + u]; }
#pragma unroll
            for (int u = 0; u < 8; ++u) x[s2 + u] = fma(-xt, rr[u], xx[u]);
          }
          for (; s2 < t; ++s2) x[s2] = fma(-xt, rc[s2], x[s2]);
        }
      }
    }
    __syncthreads();
  }

}

// Truncation, saturation flag, T = R11^{-1} R12 and the ID outputs for the factored M^T held
// in shared memory in pivot order (sA[j*SW + t], piv[j] = candidate at position j).
__device__ __forceinline__ void id_finish(const TreeDev& T, int side, int node, bool leaf, int p,
                                          double nf, int steps, double trail, double tol, const double* __restrict__ om,
                                          int64_t ldom, hsseig_status* st, const double* Mg,
                                          double* sA, double* tail, double* red, int* piv) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int nthr = blockDim.x;
  const int w = T.w, ws = T.ws, SW = w | 1;
  (void)red;
  int r = 0, sat = 0;
  double resid = 0.0;
  id_truncate(sA, tail, p, w, SW, nf, tol, w, steps, trail, r, sat, resid);

  // ---- outputs: basis X (p x r) (+ X^T for V), skeleton indices, selected rows, compressions
  int32_t* rank_arr = side == 0 ? T.rU : T.rV;
  double* X = (side == 0 ? T.U : T.V) + slot_pw(T, node);
  double* Xt = T.Vt + (size_t)node * T.ws * T.pmax;
  int32_t* loc = (side == 0 ? T.rloc : T.cloc) + (size_t)node * ws;
  int32_t* sel = (side == 0 ? T.rsel : T.csel) + (size_t)node * ws;
  double* selrows = (side == 0 ? T.psel : T.tsel) + slot_ww(T, node);
  double* comp = (side == 0 ? T.zcomp : T.ycomp) + slot_ww(T, node);
  if (tid == 0) {
    rank_arr[node] = r;
    T.flags[2 * node + side] = sat;
    (side == 0 ? T.rres : T.cres)[node] = resid;
    if (sat) atomicAdd(reinterpret_cast<unsigned long long*>(&st->v[4]), 1ull);
    atomicMax(reinterpret_cast<long long*>(&st->v[5]), (long long)r);
  }
  // Full slots: zero padding beyond p rows / r columns keeps the multiply's K tails exact.
  // U/V: candidate row q at slot row q + 1 (row 0 stays zero, so a TMA box may start one
  // row early when its A operand starts at an odd column).  V^T: candidate q at column q,
  // except that an inner node's right-child candidates start at an even column (TMA box
  // starts must be 16-byte aligned).
  // The slots were zeroed by hsseig_hss_build_rand; only the data region is written.
  int na_v = p;
  if (!leaf) na_v = side == 0 ? T.rU[T.left[node]] : T.rV[T.left[node]];
  const int rshift = (!leaf && (na_v & 1)) ? 1 : 0;
  int* ipiv = piv + T.pmax;            // candidate -> pivoted position
  for (int e = tid; e < p; e += nthr) ipiv[piv[e]] = e;
  __syncthreads();
  for (int e = tid; e < p * r; e += nthr) {   // X[q][t], t fastest (coalesced rows)
    const int q = e / r, t = e % r;
    const int jj = ipiv[q];
    const double val = jj < r ? (jj == t ? 1.0 : 0.0) : sA[jj * SW + t];
    X[(size_t)(q + 1) * ws + t] = val;
  }
  if (side == 1) {
    for (int e = tid; e < r * p; e += nthr) {   // X^T[t][col(q)], q fastest (coalesced rows)
      const int t = e / p, q = e % p;
      const int jj = ipiv[q];
      const double val = jj < r ? (jj == t ? 1.0 : 0.0) : sA[jj * SW + t];
      Xt[(size_t)t * T.pmax + (q < na_v ? q : q + rshift)] = val;
    }
  }
  for (int t = tid; t < r; t += nthr) {
    const int pj = piv[t];
    loc[t] = pj;
    int gsel;
    if (leaf) gsel = T.lo[node] + pj;
    else {
      const int a = T.left[node], b = T.right[node];
      const int32_t* sa = (side == 0 ? T.rsel : T.csel) + (size_t)a * ws;
      const int32_t* sb = (side == 0 ? T.rsel : T.csel) + (size_t)b * ws;
      const int na = side == 0 ? T.rU[a] : T.rV[a];
      gsel = pj < na ? sa[pj] : sb[pj - na];
    }
    sel[t] = gsel;
  }
  for (int e = tid; e < r * w; e += nthr) {
    const int t = e / w, c = e % w;
    selrows[(size_t)t * ws + c] = Mg[(size_t)piv[t] * ws + c];
  }
  // comp = X^T S with S = Omega_t (leaf) or [comp_a; comp_b] (inner)   (hss.py:281-282, 295-296)
  const double* Sa;
  const double* Sb;
  int64_t lds;
  int na = p;
  if (leaf) {
    Sa = om + (int64_t)T.lo[node] * ldom;
    Sb = Sa;
    lds = ldom;
  } else {
    const int a = T.left[node], b = T.right[node];
    na = side == 0 ? T.rU[a] : T.rV[a];
    Sa = (side == 0 ? T.zcomp : T.ycomp) + slot_ww(T, a);
    Sb = (side == 0 ? T.zcomp : T.ycomp) + slot_ww(T, b);
    lds = ws;
  }
  // S rows are staged through shared memory in chunks of kSChunk (coalesced loads, one
  // latency per chunk); warp -> groups of 4 output rows t, lane -> up to 4 columns c
  auto srow_ptr = [&](int q) -> const double* {
    return q < na ? Sa + (int64_t)q * lds : Sb + (int64_t)(q - na) * lds;
  };
  // staging reuses the pivot columns of sA (positions < r), dead once X is written
  double* sS = sA;
  const int kSChunk = max(1, min(16, (r * SW) / max(w, 1)));
  const int ngroups = (r + 3) / 4;
  const int myg = (ngroups + nwarps - 1) / nwarps;   // groups per warp (<= 4 for w <= 128)
  for (int gb = 0; gb < myg; gb += 2) {              // two groups per pass (register budget)
    double acc[2][4][4];
#pragma unroll
    for (int gi = 0; gi < 2; ++gi) {
      const int t0 = (warp + (gb + gi) * nwarps) * 4;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int t = t0 + u;
        const double* sr = (gb + gi < myg && t < r) ? srow_ptr(piv[t]) : nullptr;
#pragma unroll
        for (int cq = 0; cq < 4; ++cq) {
          const int c = lane + 32 * cq;
          acc[gi][u][cq] = (sr && c < w) ? sr[c] : 0.0;
        }
      }
    }
    for (int j0 = r; j0 < p; j0 += kSChunk) {
      const int nj = min(kSChunk, p - j0);
      __syncthreads();
      for (int e = tid; e < nj * w; e += nthr) {
        const int q = e / w, c = e % w;
        sS[q * w + c] = srow_ptr(piv[j0 + q])[c];
      }
      __syncthreads();
      for (int q = 0; q < nj; ++q) {
        double sv[4];
#pragma unroll
        for (int cq = 0; cq < 4; ++cq) {
          const int c = lane + 32 * cq;
          sv[cq] = c < w ? sS[q * w + c] : 0.0;
        }
        const double* arow = sA + (j0 + q) * SW;
#pragma unroll
        for (int gi = 0; gi < 2; ++gi) {
          const int t0 = (warp + (gb + gi) * nwarps) * 4;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const double coef = (gb + gi < myg && t0 + u < r) ? arow[t0 + u] : 0.0;
#pragma unroll
            for (int cq = 0; cq < 4; ++cq) acc[gi][u][cq] = fma(coef, sv[cq], acc[gi][u][cq]);
          }
        }
      }
    }
#pragma unroll
    for (int gi = 0; gi < 2; ++gi) {
      const int t0 = (warp + (gb + gi) * nwarps) * 4;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int t = t0 + u;
        if (gb + gi >= myg || t >= r) continue;
#pragma unroll
        for (int cq = 0; cq < 4; ++cq) {
          const int c = lane + 32 * cq;
          if (c < w) comp[(size_t)t * ws + c] = acc[gi][u][cq];
        }
      }
    }
  }
}

#ifdef HSSEIG_ID_TIMING
// per-phase clock64 totals of block 0 / thread 0 (tools/id_timing.cu):
// [0] warp-0 pivot + reflector, [1] wait at the reflector barrier, [2] own update,
// [3] wait at the end-of-step barrier, [4] steps, [5] elimination total, [6] finish total
__device__ unsigned long long g_id_t[8];
#define ID_T0(v) long long v = 0; if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0) v = clock64()
#define ID_ACC(k, from, to) if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0) { to = clock64(); g_id_t[k] += to - from; }
#else
#define ID_T0(v)
#define ID_ACC(k, from, to)
#endif

// Norms and column-pivoted Householder elimination of A = M^T held in sA (candidate j at
// sA[j*SW + t]; piv[j] = j on entry).  dgeqp3/dlaqp2 semantics: pivot = first maximum of
// the downdated norms (idamax), dlarfg reflector, dlaqp2 norm downdate with the sqrt(eps)
// recompute rule.  Returns ||M||_F.
//
// Early stop: the truncation only reads R's rows above the rank and the trailing masses,
// and the mass of R's rows >= t equals the Frobenius mass of the trailing block after t
// reflectors.  After each step the sum of the downdated norms (accurate to ~1e-11 relative
// under the sqrt(eps) recompute rule) is compared with the cut; when it is within 4x the
// exact trailing mass is summed and the elimination stops at the first step whose mass is
// at or under (tol ||M||_F)^2, or at max_rank.  Rank, skeleton, T and the saturation flag
// are those of the full factorisation (its columns beyond the rank only permute among
// themselves); steps / trail return the reflector count and the trailing mass.
__device__ __forceinline__ double id_eliminate(double* sA, double* vn1, double* vn2, double* red,
                                               int* piv, int p, int w, int SW, double tol,
                                               int max_rank, int& steps, double& trail) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int nthr = blockDim.x;
  __shared__ double s_tau, s_nf;
  // Frobenius norm (hss.py:128) and the initial column norms (dgeqp3: dnrm2 per column)
  {
    double s = 0.0;
    for (int c = tid; c < p; c += nthr) {
      const double* a = sA + c * SW;
      double q0 = 0.0, q1 = 0.0;
      int t = 0;
      for (; t + 1 < w; t += 2) { q0 = fma(a[t], a[t], q0); q1 = fma(a[t + 1], a[t + 1], q1); }
      if (t < w) q0 = fma(a[t], a[t], q0);
      double q = q0 + q1;
      vn1[c] = vn2[c] = sqrt(q);
      s += q;
    }
    s = warp_sum(s);
    if (lane == 0) red[warp] = s;
  }
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int t = 0; t < nwarps; ++t) s += red[t];
    s_nf = sqrt(s);
  }
  __syncthreads();
  const double nf = s_nf;
  const int mn = min(w, p);
  steps = mn;
  trail = 0.0;
  const double cut = (tol * nf) * (tol * nf);
  const int stop_at = min(mn, max(max_rank, 1));
  if (!(nf == 0.0 || p == 0 || w == 0)) {
    for (int i = 0; i < mn; ++i) {
      ID_T0(ta);
#ifdef HSSEIG_ID_TIMING
      long long tb = 0, tc = 0, td = 0, te = 0;
      if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0) g_id_t[4] += 1;
#endif
      if (warp == 0) {
        double best = -1.0;
        int bi = i;
        for (int c = i + lane; c < p; c += 32) {
          double v = vn1[c];
          if (v > best) { best = v; bi = c; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          double ob = __shfl_xor_sync(0xffffffffu, best, o);
          int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
        }
        // swap and reflector in one pass: the pivot column and column i come into
        // registers (w <= 128: four rows per lane), dlarfg runs on the pivot's values, and
        // position i receives the reflected column while position pvt receives old column i
        const int pvt = bi;
        double* ci = sA + i * SW;
        double* cp = sA + pvt * SW;
        double pv[4], cv[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int t = lane + 32 * j;
          pv[j] = t < w ? cp[t] : 0.0;
          cv[j] = (t < w && pvt != i) ? ci[t] : 0.0;
        }
        // the sum of squares with the lane association of the sequential version (lane l
        // takes rows i + 1 + l + 32 j): the reflector, and the merge records pinned to it,
        // stay bit-identical
        double xs = 0.0;
        for (int t = i + 1 + lane; t < w; t += 32) xs = fma(cp[t], cp[t], xs);
        xs = warp_sum(xs);
        const double alpha = cp[i];
        double tau = 0.0, beta = alpha, scal = 1.0;
        const double xnorm = sqrt(xs);
        if (xnorm != 0.0) {
          // dlarfg with dlapy2: the rounding the merge records are pinned to (a flagged-tree
          // decision at the noise level flips with a cheaper beta)
          beta = -copysign(lapy2(alpha, xnorm), alpha);
          tau = (beta - alpha) / beta;
          scal = 1.0 / (alpha - beta);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int t = lane + 32 * j;
          if (t < w) {
            ci[t] = t < i ? pv[j] : (t == i ? beta : pv[j] * scal);
            if (pvt != i) cp[t] = cv[j];
          }
        }
        if (pvt != i) {
          if (lane == 0) { const int tp = piv[pvt]; piv[pvt] = piv[i]; piv[i] = tp; }
          if (lane == 1) vn1[pvt] = vn1[i];
          if (lane == 2) vn2[pvt] = vn2[i];
        }
        if (lane == 0) s_tau = tau;
      }
      ID_ACC(0, ta, tb);
      __syncthreads();
      ID_ACC(1, tb, tc);
      const double tau = s_tau;
      const double* v = sA + i * SW;
      double mine = 0.0;   // downdated norms^2 of this thread's trailing candidates
      for (int c = i + 1 + tid; c < p; c += nthr) {
        double* a = sA + c * SW;
        if (tau != 0.0) {
          double d0 = a[i], d1 = 0.0, d2 = 0.0, d3 = 0.0;
          int t = i + 1;
          for (; t + 3 < w; t += 4) {
            d0 = fma(v[t], a[t], d0);
            d1 = fma(v[t + 1], a[t + 1], d1);
            d2 = fma(v[t + 2], a[t + 2], d2);
            d3 = fma(v[t + 3], a[t + 3], d3);
          }
          for (; t < w; ++t) d0 = fma(v[t], a[t], d0);
          const double f = tau * ((d0 + d1) + (d2 + d3));
          a[i] -= f;
          // eight loads in flight before the stores (a and v never overlap, but the
          // compiler cannot prove it, so a plain loop serialises load -> fma -> store)
          for (t = i + 1; t + 7 < w; t += 8) {
            double vv[8], aa[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) { vv[u] = v[t + u]; aa[u] = a[t + u]; }
#pragma unroll
            for (int u = 0; u < 8; ++u) a[t + u] = fma(-f, vv[u], aa[u]);
          }
          for (; t < w; ++t) a[t] = fma(-f, v[t], a[t]);
        }
        const double n1 = vn1[c];
        if (n1 != 0.0) {
          const double q = fabs(a[i]) / n1;
          const double temp = fmax(1.0 - q * q, 0.0);
          const double ratio = n1 / vn2[c];
          if (temp * ratio * ratio <= kTol3z) {
            double s0 = 0.0, s1 = 0.0;
            int t = i + 1;
            for (; t + 1 < w; t += 2) { s0 = fma(a[t], a[t], s0); s1 = fma(a[t + 1], a[t + 1], s1); }
            if (t < w) s0 = fma(a[t], a[t], s0);
            const double nv = (i + 1 < w) ? sqrt(s0 + s1) : 0.0;
            vn1[c] = nv;
            vn2[c] = nv;
          } else {
            vn1[c] = n1 * sqrt(temp);
          }
        }
        mine = fma(vn1[c], vn1[c], mine);
      }
      ID_ACC(2, tc, td);
      if (i + 1 >= mn) break;   // full factorisation: trailing mass 0
      mine = warp_sum(mine);
      if (lane == 0) red[8 + warp] = mine;
      __syncthreads();
      ID_ACC(3, td, te);
      double proxy = 0.0;
      for (int t = 0; t < nwarps; ++t) proxy += red[8 + t];   // same order in every thread
      if (proxy <= 4.0 * cut || i + 1 == stop_at) {
        double ex = 0.0;
        for (int c = i + 1 + tid; c < p; c += nthr) {
          const double* a = sA + c * SW;
          for (int t = i + 1; t < w; ++t) ex = fma(a[t], a[t], ex);
        }
        ex = warp_sum(ex);
        if (lane == 0) red[16 + warp] = ex;
        __syncthreads();
        ex = 0.0;
        for (int t = 0; t < nwarps; ++t) ex += red[16 + t];
        if (ex <= cut || i + 1 == stop_at) {   // uniform: every thread summed the same values
          steps = i + 1;
          trail = ex;
          break;
        }
      }
    }
  }
  __syncthreads();
  return nf;
}

// ---------------------------------------------------------------------------
// Interpolative decomposition of one p x w matrix M (rows = candidates), hss.py:120-148.
// Column-pivoted QR of A = M^T (w x p): candidate j of M is column j of A, stored
// contiguously in shared memory (sA[j*SW + t] = A[t][j], SW odd => conflict-free when
// consecutive threads own consecutive candidates).
// Per elimination step: warp 0 picks the pivot (first max of the downdated norms,
// idamax) and forms the Householder reflector (dlarfg); then every thread owns one
// trailing candidate and applies the reflector and the dlaqp2 norm downdate to it.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256, 2) id_kernel(TreeDev T, int level, double tol,
                                                 const double* __restrict__ om, int64_t ldom,
                                                 hsseig_status* st, int j0) {
  extern __shared__ __align__(16) double sm[];
  const int j = j0 + blockIdx.x, side = blockIdx.y, tid = threadIdx.x;
  const int nthr = blockDim.x;
  const int node = T.lnodes[(1 << level) - 1 + j];
  const bool leaf = T.left[node] < 0;
  const int w = T.w, ws = T.ws, SW = w | 1;
  int p;
  if (leaf) p = T.hi[node] - T.lo[node];
  else {
    int a = T.left[node], b = T.right[node];
    p = side == 0 ? T.rU[a] + T.rU[b] : T.rV[a] + T.rV[b];
  }
  double* Mg = T.M + (size_t)(2 * j + side) * T.pmax * ws;
  double* sA = sm;                              // p x SW
  double* vn1 = sA + (size_t)T.pmax * SW;       // p
  double* vn2 = vn1 + T.pmax;                   // p
  double* tail = vn2 + T.pmax;                  // w + 1
  double* red = tail + (w + 1);                 // 32 scratch
  int* piv = reinterpret_cast<int*>(red + 32);  // p

  {
    for (int e = tid; e < p * w; e += nthr) {
      int row = e / w, c = e % w;
      sA[row * SW + c] = Mg[(size_t)row * ws + c];
    }
  }
  for (int e = tid; e < p; e += nthr) piv[e] = e;
  __syncthreads();
  int steps;
  double trail;
  ID_T0(t0);
#ifdef HSSEIG_ID_TIMING
  long long t1 = 0, t2 = 0;
#endif
  const double nf = id_eliminate(sA, vn1, vn2, red, piv, p, w, SW, tol, w, steps, trail);
  ID_ACC(5, t0, t1);
  id_finish(T, side, node, leaf, p, nf, steps, trail, tol, om, ldom, st, Mg, sA, tail, red, piv);
  ID_ACC(6, t1, t2);
}


// Standalone interpolative decomposition of a batch of p x w matrices (hss.py:104-148):
// one CTA per matrix, the same elimination and truncation as the tree construction.
__global__ void __launch_bounds__(256) interp_kernel(const double* __restrict__ M, int64_t ldm,
                                                     int64_t sm, int p, int w, double tol,
                                                     int max_rank, double* __restrict__ X,
                                                     int64_t ldx, int64_t sx, int32_t* J,
                                                     int32_t* rank, double* resid_out,
                                                     int32_t* sat_out) {
  extern __shared__ __align__(16) double smi[];
  const int b = blockIdx.x, tid = threadIdx.x, nthr = blockDim.x;
  const int SW = w | 1;
  const double* Mb = M + (size_t)b * sm;
  double* Xb = X + (size_t)b * sx;
  double* sA = smi;
  double* vn1 = sA + (size_t)p * SW;
  double* vn2 = vn1 + p;
  double* tail = vn2 + p;
  double* red = tail + (w + 1);
  int* piv = reinterpret_cast<int*>(red + 32);
  int* ipiv = piv + p;
  for (int e = tid; e < p * w; e += nthr) {
    const int row = e / w, c = e % w;
    sA[row * SW + c] = Mb[(size_t)row * ldm + c];
  }
  for (int e = tid; e < p; e += nthr) piv[e] = e;
  __syncthreads();
  int steps;
  double trail;
  const double nf = id_eliminate(sA, vn1, vn2, red, piv, p, w, SW, tol, max_rank, steps, trail);
  int r, sat;
  double resid;
  id_truncate(sA, tail, p, w, SW, nf, tol, max_rank, steps, trail, r, sat, resid);
  for (int e = tid; e < p; e += nthr) ipiv[piv[e]] = e;
  __syncthreads();
  for (int e = tid; e < p * r; e += nthr) {   // X[q][t]: identity on J, T^T elsewhere
    const int q = e / r, t = e % r;
    const int jj = ipiv[q];
    Xb[(size_t)q * ldx + t] = jj < r ? (jj == t ? 1.0 : 0.0) : sA[jj * SW + t];
  }
  for (int t = tid; t < r; t += nthr) J[(size_t)b * max_rank + t] = piv[t];
  if (tid == 0) {
    rank[b] = r;
    resid_out[b] = resid;
    sat_out[b] = sat;
  }
}

}  // namespace hsseig

using namespace hsseig;

static int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

// leaf_of[i] = position of the leaf holding index i (binary search over the leaf starts)
__global__ void leaf_of_kernel(const int32_t* __restrict__ lo, const int32_t* __restrict__ left,
                               const int32_t* __restrict__ lnodes, int depth, int n_leaves,
                               int32_t k, int32_t* __restrict__ leaf_of) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= k) return;
  const int32_t* leaves = lnodes + (1 << depth) - 1;   // leaf node ids by position
  int a = 0, b = n_leaves - 1;
  while (a < b) {
    const int mid = (a + b + 1) >> 1;
    if (lo[leaves[mid]] <= i) a = mid; else b = mid - 1;
  }
  (void)left;
  leaf_of[i] = a;
}

struct TreeCarve {
  int64_t off_lo, off_hi, off_left, off_right, off_lnodes, off_rU, off_rV, off_rsel, off_csel,
      off_rloc, off_cloc, off_flags, off_U, off_V, off_Vt, off_B, off_D, off_rres, off_cres, off_M,
      off_psel, off_tsel, off_ycomp, off_zcomp, off_lid, total;
};

static TreeCarve carve(int32_t k, int32_t n_leaves, int32_t w, int32_t mmax) {
  TreeCarve c;
  const int64_t nn = 2 * (int64_t)n_leaves - 1;
  const int64_t ws = (w + 15) / 16 * 16;
  // slots hold zero rows past their data far enough for whole 16-deep K chunks
  int64_t pmax = std::max<int64_t>((mmax + 1 + 15) / 16 * 16, 2 * (int64_t)w);
  pmax += (pmax & 1) + 2;
  const int64_t dld = mmax + (mmax & 1);
  int64_t o = 0;
  auto take = [&](int64_t bytes) { int64_t at = o; o = align_up(o + bytes, 256); return at; };
  c.off_lo = take(4 * nn); c.off_hi = take(4 * nn); c.off_left = take(4 * nn);
  c.off_right = take(4 * nn); c.off_lnodes = take(4 * nn);
  c.off_rU = take(4 * nn); c.off_rV = take(4 * nn);
  c.off_rsel = take(4 * nn * ws); c.off_csel = take(4 * nn * ws);
  c.off_rloc = take(4 * nn * ws); c.off_cloc = take(4 * nn * ws);
  c.off_flags = take(4 * 2 * nn);
  c.off_U = take(8 * nn * pmax * ws); c.off_V = take(8 * nn * pmax * ws);
  c.off_Vt = take(8 * nn * ws * pmax);
  c.off_B = take(8 * nn * ws * ws); c.off_D = take(8 * (int64_t)n_leaves * hsseig_drows(mmax) * dld);
  c.off_rres = take(8 * nn); c.off_cres = take(8 * nn);
  c.off_M = take(8 * 2 * (int64_t)n_leaves * pmax * ws);
  c.off_psel = take(8 * nn * ws * ws); c.off_tsel = take(8 * nn * ws * ws);
  c.off_ycomp = take(8 * nn * ws * ws); c.off_zcomp = take(8 * nn * ws * ws);
  c.off_lid = take(4 * (int64_t)k);
  c.total = o;
  return c;
}

extern "C" int64_t hsseig_tree_bytes(int32_t k, int32_t n_leaves, int32_t w, int32_t mmax) {
  return carve(k, n_leaves, w, mmax).total;
}

extern "C" int hsseig_tree_layout(hsseig_tree* t, const int32_t* bounds, int32_t n_leaves, int32_t w,
                                  void* dev_mem, void* stream) {
  if (!t || !bounds || n_leaves < 2 || (n_leaves & (n_leaves - 1)) || w < 1 || !dev_mem)
    HSS_ARG_FAIL();
  int depth = 0;
  while ((1 << depth) < n_leaves) ++depth;
  if (depth > 31) HSS_ARG_FAIL();
  int32_t mmax = 0;
  for (int i = 0; i < n_leaves; ++i) {
    if (bounds[i + 1] <= bounds[i]) HSS_ARG_FAIL();
    mmax = std::max(mmax, bounds[i + 1] - bounds[i]);
  }
  const int32_t k = bounds[n_leaves];
  const int nn = 2 * n_leaves - 1;
  // postorder numbering (hss.py:188-214) and (level, position) -> node map
  std::vector<int32_t> lo(nn), hi(nn), left(nn, -1), right(nn, -1), lnodes(nn);
  int counter = 0;
  struct Rec {
    static int go(int a, int b, int lev, int pos, const int32_t* bd, std::vector<int32_t>& lo,
                  std::vector<int32_t>& hi, std::vector<int32_t>& L, std::vector<int32_t>& R,
                  std::vector<int32_t>& ln, int& cnt) {
      if (b - a == 1) {
        int id = cnt++;
        lo[id] = bd[a]; hi[id] = bd[a + 1];
        ln[(1 << lev) - 1 + pos] = id;
        return id;
      }
      int h = (a + b) / 2;
      int l = go(a, h, lev + 1, 2 * pos, bd, lo, hi, L, R, ln, cnt);
      int r = go(h, b, lev + 1, 2 * pos + 1, bd, lo, hi, L, R, ln, cnt);
      int id = cnt++;
      lo[id] = lo[l]; hi[id] = hi[r]; L[id] = l; R[id] = r;
      ln[(1 << lev) - 1 + pos] = id;
      return id;
    }
  };
  int root = Rec::go(0, n_leaves, 0, 0, bounds, lo, hi, left, right, lnodes, counter);
  TreeCarve c = carve(k, n_leaves, w, mmax);
  char* base = static_cast<char*>(dev_mem);
  t->k = k; t->n_leaves = n_leaves; t->depth = depth; t->n_nodes = nn; t->w = w;
  t->ws = (w + 15) / 16 * 16;
  t->pmax = std::max<int32_t>((mmax + 1 + 15) / 16 * 16, 2 * w);
  t->pmax += (t->pmax & 1) + 2;
  t->mmax = mmax;
  t->dld = mmax + (mmax & 1);
  t->root = root;
  t->rmax = 0;
  for (int l = 0; l <= depth && l < 31; ++l) t->level_off_h[l] = (1 << l) - 1;
  t->lo = reinterpret_cast<int32_t*>(base + c.off_lo);
  t->hi = reinterpret_cast<int32_t*>(base + c.off_hi);
  t->left = reinterpret_cast<int32_t*>(base + c.off_left);
  t->right = reinterpret_cast<int32_t*>(base + c.off_right);
  t->level_nodes = reinterpret_cast<int32_t*>(base + c.off_lnodes);
  t->level_off = nullptr;
  t->rU = reinterpret_cast<int32_t*>(base + c.off_rU);
  t->rV = reinterpret_cast<int32_t*>(base + c.off_rV);
  t->rsel = reinterpret_cast<int32_t*>(base + c.off_rsel);
  t->csel = reinterpret_cast<int32_t*>(base + c.off_csel);
  t->rloc = reinterpret_cast<int32_t*>(base + c.off_rloc);
  t->cloc = reinterpret_cast<int32_t*>(base + c.off_cloc);
  t->flags = reinterpret_cast<int32_t*>(base + c.off_flags);
  t->U = reinterpret_cast<double*>(base + c.off_U);
  t->V = reinterpret_cast<double*>(base + c.off_V);
  t->Vt = reinterpret_cast<double*>(base + c.off_Vt);
  t->B = reinterpret_cast<double*>(base + c.off_B);
  t->D = reinterpret_cast<double*>(base + c.off_D);
  t->rres = reinterpret_cast<double*>(base + c.off_rres);
  t->cres = reinterpret_cast<double*>(base + c.off_cres);
  t->M = reinterpret_cast<double*>(base + c.off_M);
  t->psel = reinterpret_cast<double*>(base + c.off_psel);
  t->tsel = reinterpret_cast<double*>(base + c.off_tsel);
  t->ycomp = reinterpret_cast<double*>(base + c.off_ycomp);
  t->zcomp = reinterpret_cast<double*>(base + c.off_zcomp);
  t->leaf_of = reinterpret_cast<int32_t*>(base + c.off_lid);
  cudaStream_t s = (cudaStream_t)stream;
  void* dst[5] = {(void*)t->lo, (void*)t->hi, (void*)t->left, (void*)t->right, (void*)t->level_nodes};
  const void* src[5] = {lo.data(), hi.data(), left.data(), right.data(), lnodes.data()};
  const size_t nb[5] = {4u * nn, 4u * nn, 4u * nn, 4u * nn, 4u * nn};
  bool ok = upload_async(5, dst, src, nb, s) &&
            cudaMemsetAsync(t->rU, 0, 4 * nn, s) == cudaSuccess &&
            cudaMemsetAsync(t->rV, 0, 4 * nn, s) == cudaSuccess &&
            cudaMemsetAsync(t->flags, 0, 8 * nn, s) == cudaSuccess &&
            cudaMemsetAsync(t->U, 0, (size_t)8 * nn * t->pmax * t->ws, s) == cudaSuccess &&
            cudaMemsetAsync(t->V, 0, (size_t)8 * nn * t->pmax * t->ws, s) == cudaSuccess &&
            cudaMemsetAsync(t->B, 0, (size_t)8 * nn * t->ws * t->ws, s) == cudaSuccess;
  if (!ok) return HSSEIG_ERR_CUDA;
  // leaf id of every index (the off-diagonal sample masks the diagonal leaf blocks)
  leaf_of_kernel<<<(unsigned)((k + 255) / 256), 256, 0, s>>>(t->lo, t->left, t->level_nodes, depth,
                                                             n_leaves, k, t->leaf_of);
  HSS_CHECK_LAUNCH();
  return HSSEIG_OK;
}

// Levels lev_from (deepest) .. lev_to of the construction, restricted at every level to
// the node positions of part `part` of `nparts` (positions are split evenly, so a part is
// the subtree set under level log2(nparts)); the root's skeleton blocks when lev_to == 0.
static int build_levels(const hsseig_gen* gen, const double* omega, int64_t ldom, const double* Y,
                        const double* Z, int64_t ldy, double id_tol, int offdiag,
                        hsseig_tree* tree, hsseig_status* st, int lev_from, int lev_to, int part,
                        int nparts, cudaStream_t s) {
  if (!gen || !tree || !omega || !Y || !Z || !st || gen->k != tree->k) HSS_ARG_FAIL();
  if (tree->w > tree->mmax || tree->w > 128) HSS_ARG_FAIL();
  if (nparts < 1 || (nparts & (nparts - 1)) || part < 0 || part >= nparts) HSS_ARG_FAIL();
  if (lev_from > tree->depth || lev_to < 0 || lev_to > lev_from + 1) HSS_ARG_FAIL();
  CauchyGen g;
  g.d = gen->d; g.dnext = gen->dnext; g.gam = gen->gamma; g.mu = gen->mu; g.zhat = gen->zhat;
  g.v = gen->v; g.k = gen->k;
  TreeDev T = to_dev(tree);
  const size_t smem_leaf = sizeof(double) * ((size_t)leaf_kp(T.mmax) * leaf_so(T.w) +
                                             16 * (size_t)leaf_sd(T.mmax));
  if (T.pmax > 4096) HSS_ARG_FAIL();
  const size_t smem_id = sizeof(double) * ((size_t)T.pmax * (T.w | 1) + 2 * T.pmax + T.w + 1 + 32) +
                         sizeof(int) * 2 * T.pmax + 64;
  const int kpm = (T.w + 3) / 4 * 4;
  const size_t smem_form = sizeof(double) * ((size_t)((T.w + 7) / 8 * 8) * (kpm % 8 == 0 ? kpm + 4 : kpm) +
                                             (size_t)kpm * leaf_so(T.w) + 8);
  if (smem_leaf > 227 * 1024 || smem_id > 227 * 1024 || smem_form > 227 * 1024) HSS_ARG_FAIL();
  cudaFuncSetAttribute(inner_form_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_form);
  cudaFuncSetAttribute(leaf_form_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_leaf);
  cudaFuncSetAttribute(id_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_id);
  for (int lev = lev_from; lev >= lev_to && lev >= 1; --lev) {
    const int npos = 1 << lev;
    if (npos % nparts) HSS_ARG_FAIL();
    const int cnt = npos / nparts, j0 = part * cnt;
    dim3 grid(cnt, 2);
    if (lev == T.depth) {
      leaf_form_kernel<<<grid, 256, smem_leaf, s>>>(g, T, omega, ldom, Y, Z, ldy, j0, offdiag);
    } else {
      genB_kernel<<<grid, 256, 0, s>>>(g, T, lev, j0);
      HSS_CHECK_LAUNCH();
      const int nrc = cnt >= 64 ? 1 : (cnt >= 16 ? 2 : 4);   // row chunks per half
      inner_form_kernel<<<dim3(cnt, 2, 2 * nrc), 256, smem_form, s>>>(T, lev, j0);
    }
    HSS_CHECK_LAUNCH();
    id_kernel<<<grid, 256, smem_id, s>>>(T, lev, id_tol, omega, ldom, st, j0);
    HSS_CHECK_LAUNCH();
  }
  if (lev_to == 0) {
    genB_kernel<<<dim3(1, 2), 256, 0, s>>>(g, T, 0, 0);
    HSS_CHECK_LAUNCH();
  }
  return HSSEIG_OK;
}

extern "C" int hsseig_tree_clear(hsseig_tree* tree, void* stream) {
  // zero the factor slots; the ID kernels then write only their data regions
  if (!tree) HSS_ARG_FAIL();
  cudaStream_t s = (cudaStream_t)stream;
  const size_t nn = (size_t)tree->n_nodes;
  if (cudaMemsetAsync(tree->U, 0, 8 * nn * tree->pmax * tree->ws, s) != cudaSuccess ||
      cudaMemsetAsync(tree->V, 0, 8 * nn * tree->pmax * tree->ws, s) != cudaSuccess ||
      cudaMemsetAsync(tree->Vt, 0, 8 * nn * tree->pmax * tree->ws, s) != cudaSuccess)
    return HSSEIG_ERR_CUDA;
  return HSSEIG_OK;
}

extern "C" int hsseig_hss_build_rand(const hsseig_gen* gen, const double* omega, int64_t ldom,
                                     const double* Y, const double* Z, int64_t ldy, double id_tol,
                                     int32_t offdiag, hsseig_tree* tree, hsseig_status* st,
                                     void* stream) {
  if (!tree) HSS_ARG_FAIL();
  const int rc = hsseig_tree_clear(tree, stream);
  if (rc) return rc;
  return build_levels(gen, omega, ldom, Y, Z, ldy, id_tol, offdiag, tree, st, tree->depth, 0, 0,
                      1, (cudaStream_t)stream);
}

extern "C" int hsseig_hss_build_rand_levels(const hsseig_gen* gen, const double* omega,
                                            int64_t ldom, const double* Y, const double* Z,
                                            int64_t ldy, double id_tol, int32_t offdiag,
                                            hsseig_tree* tree, hsseig_status* st, int lev_from,
                                            int lev_to, int part, int nparts, void* stream) {
  return build_levels(gen, omega, ldom, Y, Z, ldy, id_tol, offdiag, tree, st, lev_from, lev_to,
                      part, nparts, (cudaStream_t)stream);
}

extern "C" int64_t hsseig_interp_smem_bytes(int32_t p, int32_t w) {
  return (int64_t)sizeof(double) * ((int64_t)p * (w | 1) + 2 * (int64_t)p + w + 1 + 32) +
         (int64_t)sizeof(int) * 2 * p + 64;
}

extern "C" int hsseig_interp_decomp(const double* M, int64_t ldm, int64_t stride_m, int32_t p,
                                    int32_t w, int64_t batch, double tol, int32_t max_rank,
                                    double* X, int64_t ldx, int64_t stride_x, int32_t* J,
                                    int32_t* rank, double* resid, int32_t* saturated, void* stream) {
  if (p < 0 || w < 0 || w > 128 || batch < 0 || max_rank < 0 || ldm < w || ldx < max_rank)
    HSS_ARG_FAIL();
  if (batch == 0) return HSSEIG_OK;
  const int64_t smem = hsseig_interp_smem_bytes(p, w);
  if (smem > 227 * 1024 || !M || !X || !J || !rank || !resid || !saturated) HSS_ARG_FAIL();
  cudaFuncSetAttribute(interp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  interp_kernel<<<(unsigned)batch, 256, smem, (cudaStream_t)stream>>>(
      M, ldm, stride_m, p, w, tol, max_rank, X, ldx, stride_x, J, rank, resid, saturated);
  HSS_CHECK_LAUNCH();
  return HSSEIG_OK;
}

#ifdef HSSEIG_ID_TIMING
extern "C" int hsseig_debug_id_timing(unsigned long long* out, int reset) {
  if (cudaMemcpyFromSymbol(out, hsseig::g_id_t, sizeof(unsigned long long) * 8) != cudaSuccess)
    return HSSEIG_ERR_CUDA;
  if (reset) {
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(hsseig::g_id_t, z, sizeof(z));
  }
  return HSSEIG_OK;
}
#endif

