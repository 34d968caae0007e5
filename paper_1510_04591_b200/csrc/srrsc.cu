// ADC1: HSS construction of the Cauchy-like eigenvector matrix by structured rank-revealing
// Schur complements (SRRSC) on its generators, level by level, on sm_100a.
//
// PARITY UNPINNED.  BASELINE.json names ADC1 but the reference package has no implementation
// (pkg/src/hsseig/dc.py:23 knows only "dense-dc" and "adc-rand").  The
// algorithm is defined by oracle/srrsc_oracle.py, which this kernel follows operation for
// operation so that pivots, ranks and skeletons are bit-identical to it.
//
// Node t, side 0 (block row C[R, t^c]) or side 1 (block column C[t^c, R]^T), candidates R
// (leaf: its indices; inner: the children's skeletons).  The block is M_ab = s_a t_b / g_ab
// with g the stable gaps (secular.py:183-203).  Gaussian elimination with complete pivoting
// keeps the Schur complement Cauchy-like: pivot (p, q) rescales the generators
//   side 0:  s_i *= (d_i - d_p) / g(i, q)          t_j *= (lam_q - lam_j) / g(p, j)
//   side 1:  s_j *= (lam_p - lam_j) / g(q, j)      t_i *= (d_i - d_q) / g(i, p)
// and the multipliers L[a][s] = M^(s)[a][q] / M^(s)[p][q] give the interpolation matrix
// X = L L_J^{-1} (identity on the skeleton J).  Stop when max|M^(s)| <= tol * max|M^(0)|
// or at the rank cap (saturation flag when the residual is still above 1e-12).
//
// One CTA per (node, side); the candidate rows and their generators live in shared memory,
// the column generators (k - |t| of them) in a per-(node, side) HBM/L2 vector that each
// elimination step sweeps once: the sweep applies the previous pivot's column rescaling and
// searches the new maximum.  The search is division-free: an entry only reaches the exact
// IEEE value |s t / g| (and the argmax compare) when |s| |t| / best >= |g|, so per entry the
// sweep costs two DADD (the stable gap), one DMUL and one compare.
// Cost: sum over nodes of |R| (k - |t|) rank entries, O(k^2 r) per merge, the complexity the
// paper quotes for ADC1.
#include <climits>

#include "tree_dev.cuh"

namespace hsseig {

constexpr int kSrThreads = 256;
constexpr int kSrCols = 4;  // columns a thread holds in registers during a sweep

// lam_a - lam_b for eigen indices a != b through the pole between them (both terms carry the
// sign of the result):  a < b: ((d_{a+1} - d_b) - gam_b) - mu_a;  a > b: mu_b - ((d_{b+1} - d_a) - gam_a)
__device__ __forceinline__ double lamdiff(int a, int b, double da, double ga, double na, double ma,
                                          double db, double gb, double nb, double mb) {
  return a < b ? (((na - db) - gb) - ma) : (mb - ((nb - da) - ga));
}

__device__ __forceinline__ bool better(double v, long long key, double bv, long long bk) {
  return v > bv || (v == bv && key < bk);
}

__global__ void __launch_bounds__(kSrThreads) srrsc_kernel(CauchyGen g, TreeDev T, int level,
                                                           int j0, double tol, int cap,
                                                           double* __restrict__ work, int64_t ldw,
                                                           hsseig_status* st) {
  extern __shared__ __align__(16) double sm[];
  const int j = j0 + blockIdx.x, side = blockIdx.y, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int node = T.lnodes[(1 << level) - 1 + j];
  const bool leaf = T.left[node] < 0;
  const int lo = T.lo[node], hi = T.hi[node], width = hi - lo;
  const int ncomp = T.k - width;
  const int P = T.pmax, ws = T.ws;
  int p, na = 0;
  if (leaf) {
    p = width;
  } else {
    const int a = T.left[node], b = T.right[node];
    na = side == 0 ? T.rU[a] : T.rV[a];
    p = na + (side == 0 ? T.rU[b] : T.rV[b]);
  }
  // row state: s (signed generator, 0 once pivoted) and the row's points:
  //   side 0 (poles i):     X = d_i
  //   side 1 (eigen j):     X = d_j, Y = gam_j, Z = d_{j+1}, W = -mu_j
  double* sS = sm;
  double* sX = sS + P;
  double* sY = sX + P;
  double* sZ = sY + P;
  double* sW = sZ + P;
  int* sG = reinterpret_cast<int*>(sW + P);  // global index of the candidate
  int* sPos = sG + P;                         // elimination step that pivoted it, or -1
  int* sPiv = sPos + P;                       // candidate pivoted at each step
  __shared__ double sRedV[kSrThreads / 32];
  __shared__ long long sRedK[kSrThreads / 32];
  __shared__ double sMax0, sMx, sPv, sTq, sPd, sPg, sPn, sPm;
  __shared__ int sStop, sAst, sGb, sStep;

  double* tstate = work + (size_t)(2 * j + side) * ldw;
  double* Lm = T.M + (size_t)(2 * j + side) * P * ws;   // multipliers L[a][s] at a * ws + s

  for (int a = tid; a < p; a += kSrThreads) {
    int ga;
    if (leaf) {
      ga = lo + a;
    } else {
      const int32_t* sa = (side == 0 ? T.rsel : T.csel) + (size_t)T.left[node] * ws;
      const int32_t* sb = (side == 0 ? T.rsel : T.csel) + (size_t)T.right[node] * ws;
      ga = a < na ? sa[a] : sb[a - na];
    }
    sG[a] = ga;
    sPos[a] = -1;
    if (side == 0) {
      sS[a] = __ldg(g.zhat + ga);
      sX[a] = __ldg(g.d + ga);
    } else {
      sS[a] = __ldg(g.v + ga);
      sX[a] = __ldg(g.d + ga);
      sY[a] = __ldg(g.gam + ga);
      sZ[a] = __ldg(g.dnext + ga);
      sW[a] = -__ldg(g.mu + ga);
    }
  }
  // leaf D = C(t, t) (hss.py:263), written once by the row side
  if (leaf && side == 0) {
    const int drows = hsseig_drows(T.mmax);
    double* Dslot = T.D + (size_t)j * drows * T.dld;
    for (int e = tid; e < drows * T.dld; e += kSrThreads) {
      const int a = e / T.dld - 1, b = e % T.dld;
      Dslot[e] = (a < 0 || a >= width || b >= width) ? 0.0 : g.entry(lo + a, lo + b);
    }
  }
  if (tid == 0) {
    sGb = -1;
    sStep = 0;
  }
  __syncthreads();

  int step = 0;
  for (;; ++step) {
    // ---- sweep: apply the previous pivot's column rescaling, search max |M^(step)| ----
    const int pgb = sGb, past = sStep > 0 ? sPiv[step - 1] : 0;
    double bv = 0.0;
    long long bk = LLONG_MAX;
    for (int c0 = 0; c0 < ncomp; c0 += kSrThreads * kSrCols) {
      double tv[kSrCols], cy[kSrCols], cz[kSrCols], tb[kSrCols];
      bool right[kSrCols];
      int cc[kSrCols];
#pragma unroll
      for (int u = 0; u < kSrCols; ++u) {
        const int c = c0 + u * kSrThreads + tid;
        cc[u] = c;
        double t = 0.0;
        cy[u] = 0.0;
        cz[u] = 0.0;
        right[u] = false;
        if (c < ncomp) {
          const int b = c < lo ? c : c + width;
          right[u] = b >= hi;
          if (side == 0) {   // columns are eigen indices
            const double db = __ldg(g.d + b), gb = __ldg(g.gam + b);
            const double nb = __ldg(g.dnext + b), mb = __ldg(g.mu + b);
            cy[u] = right[u] ? db : nb;
            cz[u] = right[u] ? gb : -mb;   // g = (x - cy) - cz  ==  (x - dnext) + mu on the left
            if (step == 0) {
              t = __ldg(g.v + b);
            } else if (b == pgb) {
              t = 0.0;
            } else {
              const double gp = (sX[past] - cy[u]) - cz[u];
              const double cf = lamdiff(pgb, b, sPd, sPg, sPn, sPm, db, gb, nb, mb) / gp;
              t = tstate[c] * cf;
            }
          } else {           // columns are poles
            const double db = __ldg(g.d + b);
            cy[u] = db;
            if (step == 0) {
              t = __ldg(g.zhat + b);
            } else if (b == pgb) {
              t = 0.0;
            } else {
              const double gp = right[u] ? ((db - sZ[past]) - sW[past]) : ((db - sX[past]) - sY[past]);
              const double cf = (db - sPd) / gp;
              t = tstate[c] * cf;
            }
          }
          tstate[c] = t;
        }
        tv[u] = t;
      }
      double rthr = bv > 0.0 ? 1.0 / (bv * (1.0 - 1e-9)) : __longlong_as_double(0x7ff0000000000000LL);
#pragma unroll
      for (int u = 0; u < kSrCols; ++u) tb[u] = fabs(tv[u]) * rthr;
      for (int a = 0; a < p; ++a) {
        const double sa = sS[a];
        if (sa == 0.0) continue;
        const double asa = fabs(sa);
        double gv[kSrCols];
        if (side == 0) {
          const double x = sX[a];
#pragma unroll
          for (int u = 0; u < kSrCols; ++u) gv[u] = (x - cy[u]) - cz[u];
        } else {
          const double xl = sX[a], yl = sY[a], xr = sZ[a], yr = sW[a];
#pragma unroll
          for (int u = 0; u < kSrCols; ++u)
            gv[u] = right[u] ? ((cy[u] - xr) - yr) : ((cy[u] - xl) - yl);
        }
        bool hit = false;
#pragma unroll
        for (int u = 0; u < kSrCols; ++u) hit |= (asa * tb[u] >= fabs(gv[u])) && cc[u] < ncomp;
        if (hit) {   // rare: exact values and the argmax compare
#pragma unroll
          for (int u = 0; u < kSrCols; ++u) {
            if (cc[u] >= ncomp) continue;
            const double val = fabs((sa * tv[u]) / gv[u]);
            const long long key = (long long)a * ncomp + cc[u];
            if (better(val, key, bv, bk)) { bv = val; bk = key; }
          }
          rthr = bv > 0.0 ? 1.0 / (bv * (1.0 - 1e-9)) : rthr;
#pragma unroll
          for (int u = 0; u < kSrCols; ++u) tb[u] = fabs(tv[u]) * rthr;
        }
      }
    }
    // ---- CTA argmax (first maximum in row-major order) ----
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const long long ok = __shfl_xor_sync(0xffffffffu, bk, o);
      if (better(ov, ok, bv, bk)) { bv = ov; bk = ok; }
    }
    if (lane == 0) { sRedV[warp] = bv; sRedK[warp] = bk; }
    __syncthreads();
    if (tid == 0) {
      double mv = sRedV[0];
      long long mk = sRedK[0];
      for (int w2 = 1; w2 < kSrThreads / 32; ++w2)
        if (better(sRedV[w2], sRedK[w2], mv, mk)) { mv = sRedV[w2]; mk = sRedK[w2]; }
      if (step == 0) sMax0 = mv;
      sMx = mv;
      const bool stop = mv == 0.0 || mv <= tol * sMax0 || step == cap;
      sStop = stop;
      if (!stop) {
        const int ast = (int)(mk / ncomp), cst = (int)(mk % ncomp);
        const int gb = cst < lo ? cst : cst + width;
        const double tq = tstate[cst];
        double gpv;
        if (side == 0) {
          const double db = __ldg(g.d + gb), gg = __ldg(g.gam + gb);
          const double nb = __ldg(g.dnext + gb), mb = __ldg(g.mu + gb);
          sPd = db; sPg = gg; sPn = nb; sPm = mb;
          gpv = gb >= hi ? ((sX[ast] - db) - gg) : ((sX[ast] - nb) - (-mb));
        } else {
          const double db = __ldg(g.d + gb);
          sPd = db;
          gpv = gb >= hi ? ((db - sZ[ast]) - sW[ast]) : ((db - sX[ast]) - sY[ast]);
        }
        sAst = ast;
        sGb = gb;
        sTq = tq;
        sPv = (sS[ast] * tq) / gpv;
        sPiv[step] = ast;
        sStep = step + 1;
      }
    }
    __syncthreads();
    if (sStop) break;
    // ---- eliminate the pivot on the row generators; multipliers of this step ----
    {
      const int ast = sAst, gb = sGb;
      const double tq = sTq, pv = sPv;
      const bool qright = gb >= hi;
      for (int a = tid; a < p; a += kSrThreads) {
        double L;
        if (sPos[a] >= 0) {
          L = 0.0;
        } else if (a == ast) {
          L = 1.0;
          sS[a] = 0.0;
          sPos[a] = step;
        } else {
          double ga, rf_num;
          if (side == 0) {
            ga = qright ? ((sX[a] - sPd) - sPg) : ((sX[a] - sPn) - (-sPm));
            rf_num = sX[a] - sX[ast];
          } else {
            ga = qright ? ((sPd - sZ[a]) - sW[a]) : ((sPd - sX[a]) - sY[a]);
            rf_num = lamdiff(sG[ast], sG[a], sX[ast], sY[ast], sZ[ast], -sW[ast], sX[a], sY[a],
                             sZ[a], -sW[a]);
          }
          L = ((sS[a] * tq) / ga) / pv;
          const double rf = rf_num / ga;
          sS[a] = sS[a] * rf;
        }
        Lm[(size_t)a * ws + step] = L;
      }
    }
    __syncthreads();
  }
  const int r = step;
  const double max0 = sMax0;
  const double resid = max0 > 0.0 ? sMx / max0 : 0.0;
  const int sat = (r == cap && cap > 0 && resid > kFlagTol) ? 1 : 0;

  // ---- X = L L_J^{-1}: x L11 = l for every non-skeleton candidate, in place in L ----
  for (int a = tid; a < p; a += kSrThreads) {
    if (sPos[a] >= 0) continue;
    double* La = Lm + (size_t)a * ws;
    for (int t = r - 1; t >= 0; --t) {
      double x = La[t];
      for (int s2 = t + 1; s2 < r; ++s2) x -= La[s2] * Lm[(size_t)sPiv[s2] * ws + t];
      La[t] = x;
    }
  }
  __syncthreads();

  // ---- outputs, in the layout of the randomized construction (id_finish in hss_build.cu) ----
  int32_t* rank_arr = side == 0 ? T.rU : T.rV;
  double* X = (side == 0 ? T.U : T.V) + slot_pw(T, node);
  double* Xt = T.Vt + (size_t)node * ws * P;
  int32_t* loc = (side == 0 ? T.rloc : T.cloc) + (size_t)node * ws;
  int32_t* sel = (side == 0 ? T.rsel : T.csel) + (size_t)node * ws;
  if (tid == 0) {
    rank_arr[node] = r;
    T.flags[2 * node + side] = sat;
    (side == 0 ? T.rres : T.cres)[node] = resid;
    if (sat) atomicAdd(reinterpret_cast<unsigned long long*>(&st->v[4]), 1ull);
    atomicMax(reinterpret_cast<long long*>(&st->v[5]), (long long)r);
  }
  const int na_v = leaf ? p : na;
  const int rshift = (!leaf && (na_v & 1)) ? 1 : 0;
  for (int e = tid; e < p * r; e += kSrThreads) {   // X[q][t], candidate q at slot row q + 1
    const int q = e / r, t = e % r;
    const int pos = sPos[q];
    const double val = pos >= 0 ? (pos == t ? 1.0 : 0.0) : Lm[(size_t)q * ws + t];
    X[(size_t)(q + 1) * ws + t] = val;
    if (side == 1) Xt[(size_t)t * P + (q < na_v ? q : q + rshift)] = val;
  }
  for (int t = tid; t < r; t += kSrThreads) {
    loc[t] = sPiv[t];
    sel[t] = sG[sPiv[t]];
  }
}

}  // namespace hsseig

using namespace hsseig;

static int64_t srrsc_ldw(const hsseig_tree* t) { return ((int64_t)t->k + 31) / 32 * 32; }

extern "C" int64_t hsseig_srrsc_work_doubles(const hsseig_tree* tree) {
  if (!tree) return -1;
  return 2 * (int64_t)tree->n_leaves * srrsc_ldw(tree);
}

static int build_srrsc_levels(const hsseig_gen* gen, double tol, int32_t max_rank,
                              hsseig_tree* tree, double* work, hsseig_status* st, int lev_from,
                              int lev_to, int part, int nparts, cudaStream_t s) {
  if (!gen || !tree || !work || !st || gen->k != tree->k) HSS_ARG_FAIL();
  if (!(tol >= 0.0) || max_rank < 1 || max_rank > tree->w || tree->w > 128) HSS_ARG_FAIL();
  if (nparts < 1 || (nparts & (nparts - 1)) || part < 0 || part >= nparts) HSS_ARG_FAIL();
  if (lev_from > tree->depth || lev_to < 0 || lev_to > lev_from + 1) HSS_ARG_FAIL();
  CauchyGen g;
  g.d = gen->d; g.dnext = gen->dnext; g.gam = gen->gamma; g.mu = gen->mu; g.zhat = gen->zhat;
  g.v = gen->v; g.k = gen->k;
  TreeDev T = to_dev(tree);
  const size_t smem = sizeof(double) * 5 * (size_t)T.pmax + sizeof(int) * (2 * (size_t)T.pmax + T.ws + 1);
  if (smem > 227 * 1024) HSS_ARG_FAIL();
  cudaFuncSetAttribute(srrsc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t ldw = srrsc_ldw(tree);
  for (int lev = lev_from; lev >= lev_to && lev >= 1; --lev) {
    const int npos = 1 << lev;
    if (npos % nparts) HSS_ARG_FAIL();
    const int cnt = npos / nparts, j0 = part * cnt;
    if (lev < T.depth) {
      const int rc = launch_genB(g, T, lev, j0, cnt, s);
      if (rc) return rc;
    }
    srrsc_kernel<<<dim3(cnt, 2), kSrThreads, smem, s>>>(g, T, lev, j0, tol, max_rank, work, ldw, st);
    HSS_CHECK_LAUNCH();
  }
  if (lev_to == 0) return launch_genB(g, T, 0, 0, 1, s);
  return HSSEIG_OK;
}

extern "C" int hsseig_hss_build_srrsc(const hsseig_gen* gen, double tol, int32_t max_rank,
                                      hsseig_tree* tree, double* work, hsseig_status* st,
                                      void* stream) {
  if (!tree) HSS_ARG_FAIL();
  const int rc = hsseig_tree_clear(tree, stream);
  if (rc) return rc;
  return build_srrsc_levels(gen, tol, max_rank, tree, work, st, tree->depth, 0, 0, 1,
                            (cudaStream_t)stream);
}

extern "C" int hsseig_hss_build_srrsc_levels(const hsseig_gen* gen, double tol, int32_t max_rank,
                                             hsseig_tree* tree, double* work, hsseig_status* st,
                                             int lev_from, int lev_to, int part, int nparts,
                                             void* stream) {
  return build_srrsc_levels(gen, tol, max_rank, tree, work, st, lev_from, lev_to, part, nparts,
                            (cudaStream_t)stream);
}
