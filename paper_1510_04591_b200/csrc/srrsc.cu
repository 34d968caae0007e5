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
// One thread-block cluster (1-16 CTAs) per (node, side); the candidate rows and their
// generators live in every CTA's shared memory, the column generators (k - |t| of them) in a
// per-(node, side) HBM/L2 vector whose columns are split over the cluster and swept once per
// elimination step: the sweep applies the previous pivot's column rescaling and searches the
// new maximum, and the CTAs' records meet through DSMEM after one cluster barrier.  The
// search is division-free: an entry only reaches the exact IEEE value |s t / g| (and the
// argmax compare) when |s| |t| / best + slack >= |e - c| (the gap with the rounding of its
// folded form covered by the slack).  The column points c are sorted, so that filter is
// first applied to blocks of 32 columns (largest |t| and slack of the block, distance from
// the row's point to the block's span): each row walks outwards from the block holding its
// point and evaluates only the blocks that can pass -- the argmax, and so every pivot, is
// the full sweep's (sr_sweep_blocks, used from kSrPruneMin columns off the node).
// Cost: the column rescaling is O(k - |t|) per elimination step and the search O(|R| (log +
// passing blocks)), against the sum over nodes of |R| (k - |t|) entries per step of a full
// sweep (the O(k^2 r) per merge the paper quotes for ADC1).
#include <algorithm>
#include <climits>
#include <cstdlib>

#include <cooperative_groups.h>

#include "tree_dev.cuh"

namespace hsseig {

namespace cg = cooperative_groups;

constexpr int kSrThreads = 256;
constexpr int kSrMaxCluster = 16;
constexpr int kSrCols = 4;          // columns a thread holds in registers in the full sweep
constexpr int kSrPruneMin = 12288;  // columns off the node from which the pruned search pays

// lam_a - lam_b for eigen indices a != b through the pole between them (both terms carry the
// sign of the result):  a < b: ((d_{a+1} - d_b) - gam_b) - mu_a;  a > b: mu_b - ((d_{b+1} - d_a) - gam_a)
__device__ __forceinline__ double lamdiff(int a, int b, double da, double ga, double na, double ma,
                                          double db, double gb, double nb, double mb) {
  return a < b ? (((na - db) - gb) - ma) : (mb - ((nb - da) - ga));
}

__device__ __forceinline__ bool better(double v, long long key, double bv, long long bk) {
  return v > bv || (v == bv && key < bk);
}

// Row data the sweep reads per candidate (fixed during the elimination except s):
//   e  = the folded row point of the gap (side 0: d_i; side 1: d_j + gam_j for columns left
//        of the node, d_{j+1} - mu_j for columns right of it),
//   sl = the rounding slack of that fold (side 1) — see the filter below.
struct SweepPivot {          // previous pivot, for the deferred column rescaling
  int gb, past;              // its global column index (-1: none yet) and candidate row
  double d, g, n, m;         // column point data (side 0: d, gam, dnext, mu; side 1: d)
  double rx, ry, rz, rw;     // its row's points (sX, sY, sZ, sW)
};

// One sweep over columns [c_lo, c_hi) (all left (RIGHT = false) or all right of the node):
// apply the previous pivot's rescaling to the column generators, then search the largest
// |s t / g| with the division-free filter
//     |s| |t| / best + slack >= |e - c|     (e - c the gap up to the folded rounding)
// and the exact IEEE value and row-major argmax only for entries that pass it.
template <int SIDE, bool RIGHT>
__device__ __forceinline__ void sr_sweep(const CauchyGen& g, int c_lo, int c_hi, int lo, int width,
                                         int ncomp, int p, int step, const SweepPivot& pv,
                                         double* __restrict__ tstate, const double* sS,
                                         const double* sX, const double* sY, const double* sZ,
                                         const double* sW, const double2* sE, double& bv,
                                         long long& bk, double& bt) {
  const int tid = threadIdx.x;
  const double kNaN = __longlong_as_double(0x7ff8000000000000LL);
  const double kInf = __longlong_as_double(0x7ff0000000000000LL);
  for (int c0 = c_lo; c0 < c_hi; c0 += kSrThreads * kSrCols) {
    double tv[kSrCols], ce[kSrCols], cs[kSrCols], tb[kSrCols];
#pragma unroll
    for (int u = 0; u < kSrCols; ++u) {
      const int c = c0 + u * kSrThreads + tid;
      double t = 0.0;
      double cy = kNaN, cz = kNaN;   // invalid column: NaN gaps never pass a compare
      if (c < c_hi) {
        const int b = c < lo ? c : c + width;
        if (SIDE == 0) {     // columns are eigen indices
          const double db = __ldg(g.d + b), gb = __ldg(g.gam + b);
          const double nb = __ldg(g.dnext + b), mb = __ldg(g.mu + b);
          cy = RIGHT ? db : nb;
          cz = RIGHT ? gb : -mb;       // g = (x - cy) - cz  ==  (x - dnext) + mu on the left
          if (step == 0) {
            t = __ldg(g.v + b);
          } else if (b == pv.gb) {
            t = 0.0;
          } else {
            const double gp = (pv.rx - cy) - cz;
            const double cf = lamdiff(pv.gb, b, pv.d, pv.g, pv.n, pv.m, db, gb, nb, mb) / gp;
            t = tstate[c] * cf;
          }
        } else {             // columns are poles
          const double db = __ldg(g.d + b);
          cy = db;
          if (step == 0) {
            t = __ldg(g.zhat + b);
          } else if (b == pv.gb) {
            t = 0.0;
          } else {
            const double gp = RIGHT ? ((db - pv.rz) - pv.rw) : ((db - pv.rx) - pv.ry);
            const double cf = (db - pv.d) / gp;
            t = tstate[c] * cf;
          }
        }
        tstate[c] = t;
      }
      tv[u] = t;
      if (SIDE == 0) {
        ce[u] = cy + cz;
        cs[u] = 0x1p-50 * (fabs(cy) + fabs(cz));
      } else {
        ce[u] = cy;
        cs[u] = 0.0;
      }
    }
    double rthr = bv > 0.0 ? 1.0 / (bv * (1.0 - 1e-9)) : kInf;
#pragma unroll
    for (int u = 0; u < kSrCols; ++u) tb[u] = fabs(tv[u]) * rthr;
    // two rows per iteration (independent filter chains); p is padded by a zero row
    // (s = 0 never passes) when odd, see the row setup
    for (int a0 = 0; a0 < p; a0 += 2) {
      const double as0 = fabs(sS[a0]), as1 = fabs(sS[a0 + 1]);
      const double2 e0 = sE[a0], e1 = sE[a0 + 1];  // (folded point, slack) for this branch
      unsigned hm = 0;   // bit u: (row a0, column u) passes; bit kSrCols + u: row a0 + 1
#pragma unroll
      for (int u = 0; u < kSrCols; ++u) {
        hm |= (fma(as0, tb[u], SIDE == 0 ? cs[u] : e0.y) >= fabs(ce[u] - e0.x)) ? 1u << u : 0u;
        hm |= (fma(as1, tb[u], SIDE == 0 ? cs[u] : e1.y) >= fabs(ce[u] - e1.x))
                  ? 1u << (kSrCols + u) : 0u;
      }
      if (!hm) continue;
      for (int a = a0; a < a0 + 2; ++a, hm >>= kSrCols) {   // rare: exact values, argmax
        const double sa = sS[a];
        if (sa == 0.0) continue;
#pragma unroll
        for (int u = 0; u < kSrCols; ++u) {
          const int c = c0 + u * kSrThreads + tid;
          if (!((hm >> u) & 1u) || c >= c_hi) continue;
          const int b = c < lo ? c : c + width;   // exact gap from the column's points again
          double gv;
          if (SIDE == 0) {
            gv = RIGHT ? ((sX[a] - __ldg(g.d + b)) - __ldg(g.gam + b))
                       : ((sX[a] - __ldg(g.dnext + b)) - (-__ldg(g.mu + b)));
          } else {
            const double db = __ldg(g.d + b);
            gv = RIGHT ? ((db - sZ[a]) - sW[a]) : ((db - sX[a]) - sY[a]);
          }
          const double val = fabs((sa * tv[u]) / gv);
          const long long key = (long long)a * ncomp + c;
          if (better(val, key, bv, bk)) { bv = val; bk = key; bt = tv[u]; }
        }
      }
      rthr = bv > 0.0 ? 1.0 / (bv * (1.0 - 1e-9)) : rthr;
#pragma unroll
      for (int u = 0; u < kSrCols; ++u) tb[u] = fabs(tv[u]) * rthr;
    }
  }
}

// Block-pruned sweep with lazily rescaled column generators: the same search as sr_sweep,
// with the filter applied to whole blocks of 32 columns first.  The column points c are
// ascending in the column index (eigenvalues on side 0, poles on side 1), so a block spans
// [cLo, cHi]; with T_B >= max |t| and S_B = max slack over the block, every column of it fails
// the per-entry filter for row a whenever
//     fl(dist(e_a, [cLo, cHi])) > fma(|s_a|, fl(T_B * rthr), S_B)
// (rounded products and fma are monotone, so the block bound dominates every column's left
// side and the distance is a lower bound of every column's |e - c|).  Every row's point lies
// beyond the node's side of the range (rows are candidates inside the node, columns outside
// it), so rows walk outwards from the block next to the node, stopping once even the largest
// T of all blocks further out cannot pass (prefix / suffix maxima).
//
// Lazy rescaling.  A block's generators are only brought up to date ("materialised": the
// pending pivots' rescalings applied in step order, so every t is bit-identical to the eager
// update) when the block can pass the filter for some row; otherwise only its bound T_B is
// advanced by an upper bound of the step's factor over the block.  The factor of a column is
// a Moebius function of its point (side 0: (lam_q - lam_b) / (d_p - lam_b); side 1:
// (d_b - d_q) / (d_b - lam_p)), monotone on each side of its pole, so away from the pole its
// largest modulus over the block sits at an end column (sr_block_factor, with margins for
// rounding and for the two representations of an eigenvalue).  The argmax is the maximum over
// all entries with the row-major tie-break, whatever the order in which entries are
// evaluated: the result is the full sweep's.
constexpr int kSrBlk = 32;

// blocks of one CTA's two column ranges together (at most k / 32 + 2), rounded up
__host__ __device__ __forceinline__ int sr_nblocks(int k) { return k / kSrBlk + 4; }

// One CTA's share of a column range [c_lo, c_hi): the range's blocks of 32 columns are dealt
// to the cluster's CTAs cyclically (block i of this CTA is the range's block i * cl + rank), so
// every CTA holds blocks near the node, where the search does its work.
struct SrRange {
  int c_lo, c_hi, cl, rank;
  __device__ __forceinline__ int col0(int i) const { return c_lo + (i * cl + rank) * kSrBlk; }
  __device__ __forceinline__ int nblocks() const {
    const int nt = (c_hi - c_lo + kSrBlk - 1) / kSrBlk;
    return nt > rank ? (nt - rank + cl - 1) / cl : 0;
  }
};

struct SrBlocks {       // one column range's blocks, kept over the elimination
  double* lo;           // first / last column point of the block
  double* hi;
  double* T;            // >= max |t| over the block (exact when materialised)
  double* S;            // largest rounding slack of the block's column points (side 0)
  int* st;              // step the block's generators are materialised at
};

template <int SIDE, bool RIGHT>
__device__ __forceinline__ void sr_col_point(const CauchyGen& g, int b, double& cy, double& cz) {
  if (SIDE == 0) {
    cy = RIGHT ? __ldg(g.d + b) : __ldg(g.dnext + b);
    cz = RIGHT ? __ldg(g.gam + b) : -__ldg(g.mu + b);
  } else {
    cy = __ldg(g.d + b);
    cz = 0.0;
  }
}

template <int SIDE>
__device__ __forceinline__ void sr_load_col(const CauchyGen& g, int b, double& db, double& gb,
                                            double& nb, double& mb) {
  db = __ldg(g.d + b);
  if (SIDE == 0) {
    gb = __ldg(g.gam + b); nb = __ldg(g.dnext + b); mb = __ldg(g.mu + b);
  } else {
    gb = nb = mb = 0.0;
  }
}

// rescaling factor of column b for pivot pv (b != pv.gb) and the gap it divides by; the
// operations of the eager update (sr_sweep), so the lazily applied chain is bit-identical
template <int SIDE, bool RIGHT>
__device__ __forceinline__ double sr_col_factor(int b, const SweepPivot& pv, double db, double gb,
                                                double nb, double mb, double& gp) {
  if (SIDE == 0) {
    const double cy = RIGHT ? db : nb, cz = RIGHT ? gb : -mb;
    gp = (pv.rx - cy) - cz;
    return lamdiff(pv.gb, b, pv.d, pv.g, pv.n, pv.m, db, gb, nb, mb) / gp;
  } else {
    gp = RIGHT ? ((db - pv.rz) - pv.rw) : ((db - pv.rx) - pv.ry);
    return (db - pv.d) / gp;
  }
}

// Upper bound of |factor| over the columns of block blk for pivot pv, or +inf when the
// factor's pole may lie in (or within a 2^-20 relative margin of) the block's span.  Both end
// gaps of one sign and above the margin put the pole outside the span; the exact factor is
// then monotone over the block and its modulus peaks at an end.  Computed factors carry a
// relative error of a few ulps plus, on side 0, an absolute error of the numerator from the
// other representation of an eigenvalue (d_b + gam_b vs dnext_b - mu_b, a few ulps of the
// points): 2^-33 of the point scale over the smallest gap covers both with a wide margin.
template <int SIDE, bool RIGHT>
__device__ __forceinline__ double sr_block_factor(const CauchyGen& g, const SrRange& rg, int lo,
                                                  int width, int blk, const SweepPivot& pv,
                                                  double eLo, double eHi) {
  const double kInf = __longlong_as_double(0x7ff0000000000000LL);
  const int c0 = rg.col0(blk), c1 = min(rg.c_hi, c0 + kSrBlk) - 1;
  const int b0 = c0 < lo ? c0 : c0 + width, b1 = c1 < lo ? c1 : c1 + width;
  double db, gb, nb, mb, g0, g1;
  sr_load_col<SIDE>(g, b0, db, gb, nb, mb);
  const double f0 = sr_col_factor<SIDE, RIGHT>(b0, pv, db, gb, nb, mb, g0);
  sr_load_col<SIDE>(g, b1, db, gb, nb, mb);
  const double f1 = sr_col_factor<SIDE, RIGHT>(b1, pv, db, gb, nb, mb, g1);
  const double scale = fabs(eLo) + fabs(eHi) + fabs(pv.rx) + fabs(pv.ry) + fabs(pv.rz) +
                       fabs(pv.rw) + fabs(pv.d);
  const double gmin = fmin(fabs(g0), fabs(g1));
  if (!(g0 * g1 > 0.0) || !(gmin > 0x1p-20 * scale)) return kInf;
  return (fmax(fabs(f0), fabs(f1)) + 0x1p-32 * scale / gmin) * (1.0 + 0x1p-40);
}

// Bring block blk's generators to `step` (a warp, lane = column): the pending pivots'
// rescalings in step order, then the exact max |t| of the block.
template <int SIDE, bool RIGHT>
__device__ __forceinline__ void sr_materialise(const CauchyGen& g, const SrRange& rg, int lo,
                                               int width, int blk, int step,
                                               const SweepPivot* recs,
                                               double* __restrict__ tstate, SrBlocks bs) {
  const int lane = threadIdx.x & 31;
  const int c = rg.col0(blk) + lane;
  const int from = bs.st[blk];
  double t = 0.0;
  if (c < rg.c_hi) {
    const int b = c < lo ? c : c + width;
    double db, gb, nb, mb;
    sr_load_col<SIDE>(g, b, db, gb, nb, mb);
    t = tstate[c];
    for (int s = from + 1; s <= step; ++s) {
      const SweepPivot& pv = recs[s];
      if (b == pv.gb) {
        t = 0.0;
      } else {
        double gp;
        const double cf = sr_col_factor<SIDE, RIGHT>(b, pv, db, gb, nb, mb, gp);
        t = t * cf;
      }
    }
    tstate[c] = t;
  }
  double tm = fabs(t);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) tm = fmax(tm, __shfl_xor_sync(0xffffffffu, tm, o));
  if (lane == 0) {
    bs.T[blk] = tm;
    bs.st[blk] = step;
  }
}

template <int SIDE, bool RIGHT>
__device__ __forceinline__ void sr_sweep_lazy(const CauchyGen& g, const SrRange rg, int lo,
                                              int width, int ncomp, int p, int step,
                                              const SweepPivot* recs, double* __restrict__ tstate,
                                              const double* sS, const double* sX,
                                              const double* sY, const double* sZ,
                                              const double* sW, const double2* sE, SrBlocks bs,
                                              int* mlist,
                                              hsseig_status* st, double& bv, long long& bk,
                                              double& bt) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int kWarps = kSrThreads / 32;
  const double kInf = __longlong_as_double(0x7ff0000000000000LL);
  const int c_hi = rg.c_hi;
  const int nb = rg.nblocks();
  if (nb <= 0) return;   // uniform: every thread has the same range
  double* bLo = bs.lo;
  double* bHi = bs.hi;
  double* bT = bs.T;
  double* bS = bs.S;
  const int near = RIGHT ? 0 : nb - 1;   // the block next to the node
  __shared__ int s_nm;
  __shared__ double s_wbest[kWarps];
  if (step == 0) {
    // ---- every block materialised with the initial generators; points, slack, T ----
    for (int blk = warp; blk < nb; blk += kWarps) {
      const int c0 = rg.col0(blk), c = c0 + lane;
      double t = 0.0, ce = 0.0, cs = 0.0;
      const bool valid = c < c_hi;
      if (valid) {
        const int b = c < lo ? c : c + width;
        double db, gb, nb2, mb;
        sr_load_col<SIDE>(g, b, db, gb, nb2, mb);
        if (SIDE == 0) {
          const double cy = RIGHT ? db : nb2, cz = RIGHT ? gb : -mb;
          t = __ldg(g.v + b);
          ce = cy + cz;
          cs = 0x1p-50 * (fabs(cy) + fabs(cz));
        } else {
          t = __ldg(g.zhat + b);
          ce = db;
        }
        tstate[c] = t;
      }
      double tm = valid ? fabs(t) : 0.0, sm2 = valid ? cs : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        tm = fmax(tm, __shfl_xor_sync(0xffffffffu, tm, o));
        sm2 = fmax(sm2, __shfl_xor_sync(0xffffffffu, sm2, o));
      }
      const int last = min(31, c_hi - 1 - c0);
      const double chi = __shfl_sync(0xffffffffu, ce, last);
      if (lane == 0) {
        bLo[blk] = ce;
        bHi[blk] = chi;
        bT[blk] = tm;
        bS[blk] = sm2;
        bs.st[blk] = 0;
      }
    }
  } else {
    // ---- bounds advanced by the previous pivot's factor; the block next to the node
    // (every row's nearest, always searched) materialised ----
    const SweepPivot& pv = recs[step];
    for (int blk = tid; blk < nb; blk += kSrThreads) {
      if (blk == near) continue;
      const double f = sr_block_factor<SIDE, RIGHT>(g, rg, lo, width, blk, pv, bLo[blk],
                                                    bHi[blk]);
      bT[blk] = f == kInf ? kInf : (bT[blk] * f) * (1.0 + 0x1p-50);
    }
    if (warp == kWarps - 1)
      sr_materialise<SIDE, RIGHT>(g, rg, lo, width, near, step, recs, tstate, bs);
  }
  if (tid == 0) s_nm = 0;
  __syncthreads();
  // A block's columns in a warp's registers (lane = column): generator t, point (cy, cz), the
  // folded point ce and its slack; entry() is the per-entry filter and exact value of one row.
  double tc = 0.0, cy = 0.0, cz = 0.0, ce = 0.0, csl = 0.0;
  int cc = c_hi;
  auto load_block = [&](int blk) {
    if (lane == 0 && bs.st[blk] != step)   // never: only materialised blocks are searched
      atomicAdd(reinterpret_cast<unsigned long long*>(&st->v[7]), 1ull);
    cc = rg.col0(blk) + lane;
    if (cc < c_hi) {
      tc = tstate[cc];
      sr_col_point<SIDE, RIGHT>(g, cc < lo ? cc : cc + width, cy, cz);
      ce = SIDE == 0 ? cy + cz : cy;
      csl = SIDE == 0 ? 0x1p-50 * (fabs(cy) + fabs(cz)) : 0.0;
    }
  };
  auto entry = [&](int a, double rthr) {
    const double sa = sS[a];
    const double2 e = sE[a];
    if (cc < c_hi && fma(fabs(sa), fabs(tc) * rthr, SIDE == 0 ? csl : e.y) >= fabs(ce - e.x)) {
      double gv;
      if (SIDE == 0) gv = (sX[a] - cy) - cz;   // (x - d_b) - gam_b | (x - dnext_b) + mu_b
      else gv = RIGHT ? ((cy - sZ[a]) - sW[a]) : ((cy - sX[a]) - sY[a]);
      const double val = fabs((sa * tc) / gv);
      const long long key = (long long)a * ncomp + cc;
      if (better(val, key, bv, bk)) { bv = val; bk = key; bt = tc; }
    }
  };
  auto warp_max = [&](double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
  };
  // ---- round A: the block next to the node against every row (rows dealt to the warps),
  // every entry exact; the CTA agrees on the best value found, a lower bound of the final
  // maximum ----
  load_block(near);
  for (int a = warp; a < p; a += kWarps)
    if (sS[a] != 0.0) entry(a, kInf);
  {
    const double m = warp_max(bv);
    if (lane == 0) s_wbest[warp] = m;
  }
  __syncthreads();
  double bv0 = 0.0;
  for (int w2 = 0; w2 < kWarps; ++w2) bv0 = fmax(bv0, s_wbest[w2]);
  // ---- candidate blocks: those that can pass for some row -- the distance to the rows'
  // nearest point, the largest |s| and slack of all rows and round A's threshold dominate
  // every row's block test (monotone rounding); candidates behind the step are materialised ----
  {
    double rlo = kInf, rhi = -kInf, mas = 0.0, msl = 0.0;
    for (int a = lane; a < p; a += 32) {
      const double sa = sS[a];
      if (sa == 0.0) continue;
      const double2 e = sE[a];
      rlo = fmin(rlo, e.x);
      rhi = fmax(rhi, e.x);
      mas = fmax(mas, fabs(sa));
      msl = fmax(msl, e.y);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      rlo = fmin(rlo, __shfl_xor_sync(0xffffffffu, rlo, o));
      rhi = fmax(rhi, __shfl_xor_sync(0xffffffffu, rhi, o));
      mas = fmax(mas, __shfl_xor_sync(0xffffffffu, mas, o));
      msl = fmax(msl, __shfl_xor_sync(0xffffffffu, msl, o));
    }
    const double rthr0 = bv0 > 0.0 ? 1.0 / (bv0 * (1.0 - 1e-9)) : kInf;
    for (int blk = tid; blk < nb; blk += kSrThreads) {
      if (blk == near) continue;
      const double dist = RIGHT ? bLo[blk] - rhi : rlo - bHi[blk];
      const double bsl = SIDE == 0 ? bS[blk] : msl;
      if (!(dist > fma(mas, bT[blk] * rthr0, bsl))) mlist[atomicAdd(&s_nm, 1)] = blk;
    }
  }
  __syncthreads();
  const int nm = s_nm;
  if (step > 0) {
    for (int i = warp; i < nm; i += kWarps)
      if (bs.st[mlist[i]] != step)
        sr_materialise<SIDE, RIGHT>(g, rg, lo, width, mlist[i], step, recs, tstate, bs);
    __syncthreads();
  }
  // ---- round B: a warp per candidate block (its columns in registers); lanes over rows for
  // the block test against the warp's best so far, lanes over columns for the entries of the
  // rows that pass ----
  double wbv = fmax(bv0, warp_max(bv));
  for (int i = warp; i < nm; i += kWarps) {
    const int blk = mlist[i];
    load_block(blk);
    const double bTb = bT[blk], bLb = bLo[blk], bHb = bHi[blk], bSb = SIDE == 0 ? bS[blk] : 0.0;
    for (int a0 = 0; a0 < p; a0 += 32) {
      const double rthr = wbv > 0.0 ? 1.0 / (wbv * (1.0 - 1e-9)) : kInf;
      const int a = a0 + lane;
      bool pass = false;
      if (a < p) {
        const double sa = sS[a];
        if (sa != 0.0) {
          const double2 e = sE[a];
          const double dist = RIGHT ? bLb - e.x : e.x - bHb;
          pass = !(dist > fma(fabs(sa), bTb * rthr, SIDE == 0 ? bSb : e.y));
        }
      }
      unsigned pm = __ballot_sync(0xffffffffu, pass);
      while (pm) {
        const int r = a0 + __ffs(pm) - 1;
        pm &= pm - 1;
        entry(r, rthr);
      }
      wbv = fmax(wbv, warp_max(bv));
    }
  }
  __syncthreads();   // the block statistics are read by the next range / step
}

// One thread-block cluster of CL CTAs per (node, side): every CTA keeps the candidate rows
// (replicated, updated identically), CTA `rank` owns the column slice [cbeg, cend).  Per
// elimination step each CTA publishes its slice's (max, key, t at the max) in shared memory
// (double-buffered by step parity), one cluster barrier, and every CTA reads the CL records
// through DSMEM and takes the same decision.
template <bool PRUNED>
__global__ void __launch_bounds__(kSrThreads, PRUNED ? 2 : 0) srrsc_kernel(CauchyGen g, TreeDev T, int level,
                                                           int j0, double tol, int cap,
                                                           double* __restrict__ work, int64_t ldw,
                                                           hsseig_status* st) {
  extern __shared__ __align__(16) double sm[];
  cg::cluster_group cluster = cg::this_cluster();
  const int CL = (int)cluster.num_blocks(), rank = (int)cluster.block_rank();
  const int j = j0 + blockIdx.x / CL, side = blockIdx.y, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int node = T.lnodes[(1 << level) - 1 + j];
  const bool leaf = T.left[node] < 0;
  const int lo = T.lo[node], hi = T.hi[node], width = hi - lo;
  const int ncomp = T.k - width;
  const int slice = (ncomp + CL - 1) / CL;
  const int cbeg = min(ncomp, rank * slice), cend = min(ncomp, cbeg + slice);
  const int P = T.pmax, ws = T.ws;
  const bool lead = rank == 0;
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
  double2* sEL = reinterpret_cast<double2*>(sW + P);  // (folded point, slack), left columns
  double2* sER = sEL + P;                               // the same for right columns
  int* sG = reinterpret_cast<int*>(sER + P);  // global index of the candidate
  int* sPos = sG + P;                         // elimination step that pivoted it, or -1
  int* sPiv = sPos + P;                       // candidate pivoted at each step
  // pruned sweep: the pivots of every step (lazy rescaling) and the block state of the two
  // column ranges (left blocks from 0, right blocks after them), 8-byte aligned
  SweepPivot* recs = reinterpret_cast<SweepPivot*>(
      (reinterpret_cast<uintptr_t>(sPiv + T.ws + 1) + 7) & ~(uintptr_t)7);
  const int NB = sr_nblocks(T.k);
  double* bD = reinterpret_cast<double*>(recs + T.ws + 2);
  int* bI = reinterpret_cast<int*>(bD + 4 * NB);
  const SrRange rgL{0, lo, CL, rank}, rgR{lo, ncomp, CL, rank};
  const int nbL = rgL.nblocks();
  const SrBlocks bsL{bD, bD + NB, bD + 2 * NB, bD + 3 * NB, bI};
  const SrBlocks bsR{bD + nbL, bD + NB + nbL, bD + 2 * NB + nbL, bD + 3 * NB + nbL, bI + nbL};
  int* mlist = bI + NB;
  __shared__ double sRedV[kSrThreads / 32], sRedT[kSrThreads / 32];
  __shared__ long long sRedK[kSrThreads / 32];
  __shared__ double sPartV[2], sPartT[2];     // this CTA's slice record, by step parity
  __shared__ long long sPartK[2];
  __shared__ double sMax0, sMx, sPv, sTq, sPd, sPg, sPn, sPm;
  __shared__ int sStop, sAst, sGb;

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
      sY[a] = 0.0; sZ[a] = 0.0; sW[a] = 0.0;
      sEL[a] = make_double2(sX[a], 0.0);
      sER[a] = make_double2(sX[a], 0.0);
    } else {
      const double x = __ldg(g.d + ga), y = __ldg(g.gam + ga);
      const double z = __ldg(g.dnext + ga), w = -__ldg(g.mu + ga);
      sS[a] = __ldg(g.v + ga);
      sX[a] = x; sY[a] = y; sZ[a] = z; sW[a] = w;
      // gap (c - x) - y  ~  c - (x + y), rounding of the fold and of the subtraction covered
      const double el = x + y, er = z + w;
      sEL[a] = make_double2(el, 0x1p-50 * (fabs(x) + fabs(y) + fabs(el)));
      sER[a] = make_double2(er, 0x1p-50 * (fabs(z) + fabs(w) + fabs(er)));
    }
  }
  if (tid == 0 && (p & 1)) {   // pad row for the two-row sweep: s = 0 never passes the filter
    sS[p] = 0.0;
    sX[p] = sY[p] = sZ[p] = sW[p] = 0.0;
    sEL[p] = make_double2(0.0, 0.0);
    sER[p] = make_double2(0.0, 0.0);
  }
  // leaf D = C(t, t) (hss.py:263), written once by the row side
  if (leaf && side == 0 && lead) {
    const int drows = hsseig_drows(T.mmax);
    double* Dslot = T.D + (size_t)j * drows * T.dld;
    for (int e = tid; e < drows * T.dld; e += kSrThreads) {
      const int a = e / T.dld - 1, b = e % T.dld;
      Dslot[e] = (a < 0 || a >= width || b >= width) ? 0.0 : g.entry(lo + a, lo + b);
    }
  }
  if (tid == 0) {
    sGb = -1;
    sPd = sPg = sPn = sPm = 0.0;
  }
  __syncthreads();

  int step = 0;
  for (;; ++step) {
    // ---- sweep of this CTA's slice: apply the previous pivot's column rescaling, search max ----
    SweepPivot pv;
    pv.gb = sGb;
    pv.past = step > 0 ? sPiv[step - 1] : 0;
    pv.d = sPd; pv.g = sPg; pv.n = sPn; pv.m = sPm;
    pv.rx = sX[pv.past]; pv.ry = sY[pv.past]; pv.rz = sZ[pv.past]; pv.rw = sW[pv.past];
    double bv = 0.0, bt = 0.0;
    long long bk = LLONG_MAX;
    {
      const int l0 = cbeg, l1 = min(cend, lo), r0 = max(cbeg, lo), r1 = cend;
      // the pruned search pays where the rows' point scans are long (config 4: k - |t| ~ 32k
      // columns); below that the full sweep's streaming filter is faster (config 2).  Two
      // instantiations, so each keeps its own register budget.
      if constexpr (PRUNED) {
        if (side == 0) {
          sr_sweep_lazy<0, false>(g, rgL, lo, width, ncomp, p, step, recs, tstate, sS, sX, sY, sZ, sW, sEL, bsL, mlist, st, bv, bk, bt);
          sr_sweep_lazy<0, true>(g, rgR, lo, width, ncomp, p, step, recs, tstate, sS, sX, sY, sZ, sW, sER, bsR, mlist, st, bv, bk, bt);
        } else {
          sr_sweep_lazy<1, false>(g, rgL, lo, width, ncomp, p, step, recs, tstate, sS, sX, sY, sZ, sW, sEL, bsL, mlist, st, bv, bk, bt);
          sr_sweep_lazy<1, true>(g, rgR, lo, width, ncomp, p, step, recs, tstate, sS, sX, sY, sZ, sW, sER, bsR, mlist, st, bv, bk, bt);
        }
      } else if (side == 0) {
        sr_sweep<0, false>(g, l0, l1, lo, width, ncomp, p, step, pv, tstate, sS, sX, sY, sZ, sW, sEL, bv, bk, bt);
        sr_sweep<0, true>(g, r0, r1, lo, width, ncomp, p, step, pv, tstate, sS, sX, sY, sZ, sW, sER, bv, bk, bt);
      } else {
        sr_sweep<1, false>(g, l0, l1, lo, width, ncomp, p, step, pv, tstate, sS, sX, sY, sZ, sW, sEL, bv, bk, bt);
        sr_sweep<1, true>(g, r0, r1, lo, width, ncomp, p, step, pv, tstate, sS, sX, sY, sZ, sW, sER, bv, bk, bt);
      }
    }
    // ---- slice argmax (first maximum in row-major order), then across the cluster ----
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const long long ok = __shfl_xor_sync(0xffffffffu, bk, o);
      const double ot = __shfl_xor_sync(0xffffffffu, bt, o);
      if (better(ov, ok, bv, bk)) { bv = ov; bk = ok; bt = ot; }
    }
    if (lane == 0) { sRedV[warp] = bv; sRedK[warp] = bk; sRedT[warp] = bt; }
    __syncthreads();
    const int par = step & 1;
    if (tid == 0) {
      double mv = sRedV[0], mt = sRedT[0];
      long long mk = sRedK[0];
      for (int w2 = 1; w2 < kSrThreads / 32; ++w2)
        if (better(sRedV[w2], sRedK[w2], mv, mk)) { mv = sRedV[w2]; mk = sRedK[w2]; mt = sRedT[w2]; }
      sPartV[par] = mv;
      sPartK[par] = mk;
      sPartT[par] = mt;
    }
    cluster.sync();
    if (warp == 0) {   // lane r reads CTA r's record (one DSMEM round trip), then a shuffle argmax
      double mv = 0.0, tq = 0.0;
      long long mk = LLONG_MAX;
      if (lane < CL) {
        mv = *cluster.map_shared_rank(&sPartV[par], lane);
        mk = *cluster.map_shared_rank(&sPartK[par], lane);
        tq = *cluster.map_shared_rank(&sPartT[par], lane);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, mv, o);
        const long long ok = __shfl_xor_sync(0xffffffffu, mk, o);
        const double ot = __shfl_xor_sync(0xffffffffu, tq, o);
        if (better(ov, ok, mv, mk)) { mv = ov; mk = ok; tq = ot; }
      }
      if (lane == 0) {
      if (step == 0) sMax0 = mv;
      sMx = mv;
      const bool stop = mv == 0.0 || mv <= tol * sMax0 || step == cap;
      sStop = stop;
      if (!stop) {
        const int ast = (int)(mk / ncomp), cst = (int)(mk % ncomp);
        const int gb = cst < lo ? cst : cst + width;
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
        if (PRUNED) {   // the pivot the next step's rescaling applies (lazy replay)
          SweepPivot& rc = recs[step + 1];
          rc.gb = gb; rc.past = ast;
          rc.d = sPd; rc.g = sPg; rc.n = sPn; rc.m = sPm;
          rc.rx = sX[ast]; rc.ry = sY[ast]; rc.rz = sZ[ast]; rc.rw = sW[ast];
        }
      }
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
        if (lead) Lm[(size_t)a * ws + step] = L;
      }
    }
    __syncthreads();
  }
  // no CTA may leave while another can still read its slice records
  cluster.sync();
  if (!lead) return;
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

static int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

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
  // pruned search when every node of the tree leaves at least kSrPruneMin columns off it;
  // HSSEIG_SRRSC_PRUNE=0/1 forces either search (tests compare the two bit for bit)
  const char* pe = getenv("HSSEIG_SRRSC_PRUNE");
  const bool pruned = pe && pe[0] ? pe[0] == '1' : (int64_t)T.k - (T.k >> 1) - 8 >= kSrPruneMin;
  const auto kern = pruned ? srrsc_kernel<true> : srrsc_kernel<false>;
  const size_t smem_k = sizeof(double) * 9 * (size_t)T.pmax +
                        sizeof(int) * (2 * (size_t)T.pmax + T.ws + 1) + 8 +
                        (pruned ? sizeof(SweepPivot) * (T.ws + 2) + 8 +
                                      (4 * sizeof(double) + 2 * sizeof(int)) * sr_nblocks(T.k)
                                : 0);
  if (smem_k > 227 * 1024) HSS_ARG_FAIL();
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_k);
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const int64_t ldw = srrsc_ldw(tree);
  // resident CTAs of the whole GPU: a level is sized to fill them in one wave
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSrThreads, smem_k);
  const int slots = std::max(1, per_sm) * sm_count();
  for (int lev = lev_from; lev >= lev_to && lev >= 1; --lev) {
    const int npos = 1 << lev;
    if (npos % nparts) HSS_ARG_FAIL();
    const int cnt = npos / nparts, j0 = part * cnt;
    if (lev < T.depth) {
      const int rc = launch_genB(g, T, lev, j0, cnt, s);
      if (rc) return rc;
    }
    // columns of a node split over a cluster so that a level fills about four CTAs per SM,
    // but never thinner than ~cols_per_cta columns a CTA: a small system (the mid-depth
    // merges of a full solve: k of a few hundred to a few thousand) gains nothing from 16
    // CTAs of a few dozen columns each and pays their cluster barrier every elimination step,
    // and its whole-GPU grids kept the independent merges of a depth (one stream each) from
    // running side by side
    static const int cols_per_cta = getenv("HSSEIG_SRRSC_COLS_PER_CTA")
                                        ? std::max(1, atoi(getenv("HSSEIG_SRRSC_COLS_PER_CTA")))
                                        : 1024;
    int cl = 1;
    while (cl < kSrMaxCluster && 2 * cnt * cl * 2 <= slots && (int64_t)cl * cols_per_cta < T.k)
      cl *= 2;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(cnt * cl, 2);
    lc.blockDim = dim3(kSrThreads);
    lc.dynamicSmemBytes = smem_k;
    lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (cudaLaunchKernelEx(&lc, kern, g, T, lev, j0, tol, (int)max_rank, work, ldw, st) !=
        cudaSuccess)
      return HSSEIG_ERR_CUDA;
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
