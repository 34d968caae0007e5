// Secular roots, Loewner weight recomputation and column normalizers on sm_100a.
//
// Reference path (pkg/src/hsseig):
//   secular_all / _solve_one_root   _kernels.pyx:19-234   -> secular_queue_kernel
//   stable_gap / gap_table          secular.py:183-203    -> hsseig::stable_gap
//   recompute_weights (Loewner)     secular.py:206-236    -> loewner_kernel
//   column_normalizers              secular.py:239-250    -> normalizer_kernel
//
// Work decomposition: one warp owns R roots (rows / columns); its lanes stride
// the k poles so every pole read (d_j, z_j^2, gamma_j, ...) feeds R roots.  All
// cross-lane reductions are xor butterflies, which leave bit-identical totals in
// every lane, so the per-root control flow below is warp-uniform.
#include <cstdlib>

#include "common.cuh"

namespace hsseig {

constexpr int kMaxRational = 60;   // _kernels.pyx:11
constexpr int kMaxBisect = 200;    // _kernels.pyx:12
constexpr double kNoStep = -1e308;


__device__ __forceinline__ double quad_inner(double a, double b, double c) {
  double disc = a * a - 4.0 * b * c;
  double s = sqrt(disc < 0.0 ? 0.0 : disc);
  if (c == 0.0) return a != 0.0 ? b / a : kNoStep;
  if (a <= 0.0) return (a - s) / (2.0 * c);
  return (a + s) != 0.0 ? 2.0 * b / (a + s) : kNoStep;
}

__device__ __forceinline__ double quad_outer(double a, double b, double c) {
  double disc = a * a - 4.0 * b * c;
  double s = sqrt(disc < 0.0 ? 0.0 : disc);
  if (a >= 0.0) return c != 0.0 ? (a + s) / (2.0 * c) : kNoStep;
  return (a - s) != 0.0 ? 2.0 * b / (a - s) : kNoStep;
}

// z2 = z*z and sum(z2) in a fixed order (one block).
__global__ void square_sum_kernel(const double* __restrict__ z, int64_t k, double* __restrict__ z2,
                                  double* __restrict__ sum_out) {
  __shared__ double part[32];
  // sum_out[1] is the root counter of secular_queue_kernel (zeroed here, stream-ordered)
  if (threadIdx.x == 0) reinterpret_cast<unsigned long long*>(sum_out)[1] = 0ull;
  double s = 0.0;
  for (int64_t j = threadIdx.x; j < k; j += blockDim.x) {
    double q = z[j] * z[j];
    z2[j] = q;
    s += q;
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = (threadIdx.x < (blockDim.x >> 5)) ? part[threadIdx.x] : 0.0;
    t = warp_sum(t);
    if (threadIdx.x == 0) *sum_out = t;
  }
}

// Packed poles for the sweeps: dz[j] = (d_j, z_j^2) (one 16-byte load per pole and lane),
// and sum(z^2) in a fixed order (one block).
__global__ void pack_square_sum_kernel(const double* __restrict__ d, const double* __restrict__ z,
                                       int64_t k, double2* __restrict__ dz,
                                       double* __restrict__ sum_out) {
  __shared__ double part[32];
  // sum_out[1] is the root counter of secular_queue_kernel (zeroed here, stream-ordered)
  if (threadIdx.x == 0) reinterpret_cast<unsigned long long*>(sum_out)[1] = 0ull;
  double s = 0.0;
  for (int64_t j = threadIdx.x; j < k; j += blockDim.x) {
    const double q = z[j] * z[j];
    dz[j] = make_double2(d[j], q);
    s += q;
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = (threadIdx.x < (blockDim.x >> 5)) ? part[threadIdx.x] : 0.0;
    t = warp_sum(t);
    if (threadIdx.x == 0) *sum_out = t;
  }
}

// Roots i0 .. i0+R-1 (those < iend) of one system, one warp; outputs at index i - ibeg.
template <int R>
__device__ __forceinline__ void secular_roots(
    const double* __restrict__ d, const double* __restrict__ z2, double sumz2, int64_t k,
    double rho, int64_t i0, int64_t ibeg, int64_t iend, double* __restrict__ lam,
    double* __restrict__ gam, double* __restrict__ mu, int32_t* __restrict__ iters,
    hsseig_status* __restrict__ st, int lane) {

  if (k == 1) {  // _kernels.pyx:204-209
    if (lane == 0) {
      double g = rho * sumz2;
      lam[0] = d[0] + g;
      gam[0] = g;
      mu[0] = 0.0;
      iters[0] = 1;
      atomicAdd(reinterpret_cast<unsigned long long*>(&st->v[0]), 1ull);
      if (!(g > 0.0)) atomicMin(reinterpret_cast<long long*>(&st->v[1]), 0ll);
    }
    return;
  }

  double lo[R], hi[R], x[R], dori[R], half[R];
  int64_t split[R], ori[R];
  bool live[R], outer[R], first[R];
  int it[R];

  // --- set-up (_kernels.pyx:66-91).  The reference spends one pole sweep on f at the
  // interval midpoint d_i + delta/2 to pick the origin pole, then starts iterating at the
  // quarter point.  Here that sweep is the first iteration: it evaluates psi, phi and their
  // derivatives at the midpoint (frame d_i), picks the origin / bracket from the sign of f
  // exactly as the reference does, and takes the first rational step from the midpoint
  // (the quarter point is the safeguard when the step leaves the bracket).  One pole
  // sweep per root less; the converged roots are the reference's to 64 eps.
#pragma unroll
  for (int r = 0; r < R; ++r) {
    int64_t i = i0 + r;
    live[r] = i < iend;
    outer[r] = (i == k - 1);
    first[r] = live[r] && !outer[r];
    half[r] = first[r] ? 0.5 * (__ldg(d + i + 1) - __ldg(d + i)) : 0.0;
    it[r] = 0;
    if (!live[r]) {          // placeholders for lanes past k (never read back)
      x[r] = 0.5; lo[r] = 0.0; hi[r] = 1.0; split[r] = k - 1; ori[r] = 0; dori[r] = 0.0;
    } else if (outer[r]) {
      ori[r] = k - 1; lo[r] = 0.0; hi[r] = rho * sumz2; split[r] = k - 2;
      dori[r] = __ldg(d + k - 1);
      x[r] = 0.5 * (lo[r] + hi[r]);
    } else {
      ori[r] = i; lo[r] = 0.0; hi[r] = half[r]; split[r] = i;
      dori[r] = __ldg(d + i);
      x[r] = half[r];
    }
  }

  // --- rational-interpolant iteration (_kernels.pyx:93-156), all R roots per pole sweep.
  // The split j <= split[r] between the psi (left) and phi (right) sums is a prefix of the
  // pole range, so the sweep runs in three ranges: all-left, a mixed band of < R poles,
  // all-right.  Terms on one side share a sign, so sum|t| is |psi| + |phi| (no per-term
  // fabs).  Converged roots keep being evaluated (warp-uniform, branch-free inner loop).
  bool fallback[R];
  int64_t smin = k, smax = -1;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    fallback[r] = live[r];
    if (live[r]) { smin = min(smin, split[r]); smax = max(smax, split[r]); }
  }
  for (int step = 0; step < kMaxRational; ++step) {
    bool any = false;
#pragma unroll
    for (int r = 0; r < R; ++r) any |= fallback[r];
    if (!any) break;
    double sl[R], sr[R], dl[R], dr[R];
#pragma unroll
    for (int r = 0; r < R; ++r) sl[r] = sr[r] = dl[r] = dr[r] = 0.0;
    // all-left range j <= smin
    for (int64_t j = lane; j <= smin; j += 32) {
      const double dj = __ldg(d + j), qj = __ldg(z2 + j);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double g = (dj - dori[r]) - x[r];
        const double inv = rcp_c3(g);
        const double t = qj * inv;
        sl[r] += t;
        dl[r] = fma(t, inv, dl[r]);
      }
    }
    // mixed band smin < j <= smax
    for (int64_t j = smin + 1 + lane; j <= smax; j += 32) {
      const double dj = __ldg(d + j), qj = __ldg(z2 + j);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double g = (dj - dori[r]) - x[r];
        const double inv = rcp_c3(g);
        const double t = qj * inv;
        const double td = t * inv;
        if (j <= split[r]) { sl[r] += t; dl[r] += td; }
        else { sr[r] += t; dr[r] += td; }
      }
    }
    // all-right range j > smax
    for (int64_t j = smax + 1 + lane; j < k; j += 32) {
      const double dj = __ldg(d + j), qj = __ldg(z2 + j);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double g = (dj - dori[r]) - x[r];
        const double inv = rcp_c3(g);
        const double t = qj * inv;
        sr[r] += t;
        dr[r] = fma(t, inv, dr[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double psi = rho * warp_sum(sl[r]), phi = rho * warp_sum(sr[r]);
      const double psip = rho * warp_sum(dl[r]), phip = rho * warp_sum(dr[r]);
      if (!fallback[r]) continue;
      const double mag = fabs(psi) + fabs(phi);
      it[r] += 1;
      const double f = 1.0 + psi + phi;
      if (first[r]) {
        // the midpoint sweep: origin and bracket by the sign of f (_kernels.pyx:75-85)
        first[r] = false;
        if (!(f > 0.0)) {
          ori[r] = i0 + r + 1;
          dori[r] = __ldg(d + ori[r]);
          lo[r] = -half[r];
          hi[r] = 0.0;
          x[r] = -half[r];
        }
      } else if (f > 0.0) {
        hi[r] = x[r];
      } else {
        lo[r] = x[r];
      }
      if (fabs(f) <= kEps * (1.0 + 8.0 * mag)) { fallback[r] = false; continue; }
      const int64_t pa = outer[r] ? k - 2 : i0 + r, pb = pa + 1;
      const double ga = ((__ldg(d + pa) - dori[r]) - x[r]);
      const double gb = ((__ldg(d + pb) - dori[r]) - x[r]);
      const double qa = (ga + gb) * f - ga * gb * (psip + phip);
      const double qb = ga * gb * f;
      const double qc = f - ga * psip - gb * phip;
      const double eta = outer[r] ? quad_outer(qa, qb, qc) : quad_inner(qa, qb, qc);
      double xn = (eta == kNoStep) ? 0.5 * (lo[r] + hi[r]) : x[r] + eta;
      if (!(lo[r] < xn && xn < hi[r])) xn = 0.5 * (lo[r] + hi[r]);
      if (xn == x[r]) { fallback[r] = false; continue; }
      x[r] = xn;
    }
  }

  // --- bisection fallback (_kernels.pyx:158-171); rare, one root at a time
#pragma unroll
  for (int r = 0; r < R; ++r) {
    if (!fallback[r]) continue;
    for (int step = 0; step < kMaxBisect; ++step) {
      it[r] += 1;
      double xm = 0.5 * (lo[r] + hi[r]);
      if (xm <= lo[r] || xm >= hi[r]) break;
      double s = 0.0;
      for (int64_t j = lane; j < k; j += 32)
        s += rho * __ldg(z2 + j) / ((__ldg(d + j) - dori[r]) - xm);
      double f = 1.0 + warp_sum(s);
      if (f > 0.0) hi[r] = xm; else lo[r] = xm;
    }
    x[r] = 0.5 * (lo[r] + hi[r]);
  }

  // --- gap pairs (_kernels.pyx:213-233) and bracket checks (secular.py:172-179)
  if (lane == 0) {
    unsigned long long tot = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (!live[r]) continue;
      int64_t i = i0 + r;
      const int64_t o = i - ibeg;
      double g, m;
      if (outer[r]) {
        g = x[r];
        m = rho * sumz2 - x[r];
        lam[o] = d[i] + x[r];
      } else {
        double width = d[i + 1] - d[i];
        if (ori[r] == i) { g = x[r]; m = width - x[r]; }
        else { g = width + x[r]; m = -x[r]; }
        lam[o] = dori[r] + x[r];
      }
      gam[o] = g;
      mu[o] = m;
      iters[o] = it[r];
      tot += (unsigned long long)it[r];
      if (!(g > 0.0)) atomicMin(reinterpret_cast<long long*>(&st->v[1]), (long long)i);
      if (!(m > 0.0)) atomicMin(reinterpret_cast<long long*>(&st->v[2]), (long long)i);
    }
    atomicAdd(reinterpret_cast<unsigned long long*>(&st->v[0]), tot);
  }
}

// ---------------------------------------------------------------------------------------
// Dynamically scheduled roots (the single-system path, hsseig_secular_part).
//
// A warp keeps R root slots; a slot whose root has converged writes it out and takes the
// next unsolved root from a global counter, so no pole sweep is spent on a converged root
// (the static R-per-warp kernel above sweeps until the slowest of its R roots converges)
// and the tail is one root long.  Slots hold arbitrary roots, so their psi / phi splits are
// arbitrary: the slots are kept sorted by split, and a sweep runs R + 1 pole ranges; in
// range q (split[q-1] < j <= split[q]) slots r < q take the term on the phi side and slots
// r >= q on the psi side -- a compile-time role, so the inner loops stay branch-free.
struct RootSlot {
  double x, lo, hi, dori, half;
  int64_t i, split, ori;
  int it;
  bool first, outer;
};

__device__ __forceinline__ void slot_swap(RootSlot& a, RootSlot& b) {
  RootSlot t = a;
  a = b;
  b = t;
}

// i < 0: idle (split k - 1, never written out)
__device__ __forceinline__ void slot_init(RootSlot& s, int64_t i, const double* __restrict__ d,
                                          int64_t k, double rho, double sumz2) {
  s.i = i;
  s.it = 0;
  s.outer = (i == k - 1);
  s.first = (i >= 0) && !s.outer;
  if (i < 0) {
    s.x = 0.5; s.lo = 0.0; s.hi = 1.0; s.half = 0.0; s.split = k - 1; s.ori = 0; s.dori = d[0];
  } else if (s.outer) {
    s.half = 0.0; s.ori = k - 1; s.lo = 0.0; s.hi = rho * sumz2; s.split = k - 2;
    s.dori = __ldg(d + k - 1);
    s.x = 0.5 * (s.lo + s.hi);
  } else {
    s.half = 0.5 * (__ldg(d + i + 1) - __ldg(d + i));
    s.ori = i; s.lo = 0.0; s.hi = s.half; s.split = i;
    s.dori = __ldg(d + i);
    s.x = s.half;
  }
}

template <int R>
__device__ __forceinline__ void slots_sort(RootSlot (&s)[R]) {
  if constexpr (R == 2) {
    if (s[0].split > s[1].split) slot_swap(s[0], s[1]);
  } else if constexpr (R == 4) {
    if (s[0].split > s[1].split) slot_swap(s[0], s[1]);
    if (s[2].split > s[3].split) slot_swap(s[2], s[3]);
    if (s[0].split > s[2].split) slot_swap(s[0], s[2]);
    if (s[1].split > s[3].split) slot_swap(s[1], s[3]);
    if (s[1].split > s[2].split) slot_swap(s[1], s[2]);
  } else {
#pragma unroll
    for (int a = 0; a < R; ++a)
#pragma unroll
      for (int b = 0; b + 1 < R - a; ++b)
        if (s[b].split > s[b + 1].split) slot_swap(s[b], s[b + 1]);
  }
}

// pole range [jb, je) with slots r < Q on the phi (right) side, r >= Q on the psi side
template <int R, int Q>
__device__ __forceinline__ void sweep_range(const double2* __restrict__ dz,
                                            int64_t jb, int64_t je, const double (&x)[R],
                                            const double (&dori)[R], double (&sl)[R],
                                            double (&sr)[R], double (&dl)[R], double (&dr)[R],
                                            int lane) {
  // pole j always lands on lane j mod 32 (whatever the range bounds, which depend on the
  // other slots' roots), so every root's lane sums -- and its result -- are independent of
  // the schedule: bit-identical across runs and across sharded / single-GPU solves
  for (int64_t j = jb + ((lane - jb) & 31); j < je; j += 32) {
    const double2 p = __ldg(dz + j);
    const double dj = p.x, qj = p.y;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double g = (dj - dori[r]) - x[r];
      const double inv = rcp_c3(g);
      const double t = qj * inv;
      if (r < Q) { sr[r] += t; dr[r] = fma(t, inv, dr[r]); }
      else { sl[r] += t; dl[r] = fma(t, inv, dl[r]); }
    }
  }
}

template <int R, int Q>
__device__ __forceinline__ void sweep_all(const double2* __restrict__ dz,
                                          int64_t k, const int64_t (&split)[R], const double (&x)[R],
                                          const double (&dori)[R], double (&sl)[R], double (&sr)[R],
                                          double (&dl)[R], double (&dr)[R], int lane) {
  const int64_t jb = Q == 0 ? 0 : split[Q - 1] + 1;
  const int64_t je = Q == R ? k : split[Q] + 1;
  sweep_range<R, Q>(dz, jb, je, x, dori, sl, sr, dl, dr, lane);
  if constexpr (Q < R) sweep_all<R, Q + 1>(dz, k, split, x, dori, sl, sr, dl, dr, lane);
}

template <int R, int MINB>
__global__ void __launch_bounds__(256, MINB) secular_queue_kernel(
    const double* __restrict__ d, const double2* __restrict__ dz, const double* __restrict__ sumz2p,
    int64_t k, double rho, int64_t ibeg, int64_t iend, double* __restrict__ lam,
    double* __restrict__ gam, double* __restrict__ mu, int32_t* __restrict__ iters,
    hsseig_status* __restrict__ st, unsigned long long* __restrict__ counter) {
  const int lane = threadIdx.x & 31;
  const double sumz2 = *sumz2p;
  if (k == 1) {  // _kernels.pyx:204-209 (no pole pair to step between)
    if (blockIdx.x == 0 && threadIdx.x == 0 && ibeg == 0 && iend == 1) {
      const double g = rho * sumz2;
      lam[0] = d[0] + g;
      gam[0] = g;
      mu[0] = 0.0;
      iters[0] = 1;
      atomicAdd(reinterpret_cast<unsigned long long*>(&st->v[0]), 1ull);
      if (!(g > 0.0)) atomicMin(reinterpret_cast<long long*>(&st->v[1]), 0ll);
    }
    return;
  }
  auto grab = [&]() -> int64_t {
    unsigned long long v = 0;
    if (lane == 0) v = atomicAdd(counter, 1ull);
    v = __shfl_sync(0xffffffffu, v, 0);
    const int64_t i = ibeg + (int64_t)v;
    return i < iend ? i : -1;
  };
  RootSlot s[R];
#pragma unroll
  for (int r = 0; r < R; ++r) slot_init(s[r], grab(), d, k, rho, sumz2);
  slots_sort<R>(s);
  unsigned long long tot = 0;
  while (true) {
    bool any = false;
#pragma unroll
    for (int r = 0; r < R; ++r) any |= (s[r].i >= 0);
    if (!any) break;
    double x[R], dori[R], sl[R], sr[R], dl[R], dr[R];
    int64_t split[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      x[r] = s[r].x; dori[r] = s[r].dori; split[r] = s[r].split;
      sl[r] = sr[r] = dl[r] = dr[r] = 0.0;
    }
    sweep_all<R, 0>(dz, k, split, x, dori, sl, sr, dl, dr, lane);
    bool refilled = false;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double psi = rho * warp_sum(sl[r]), phi = rho * warp_sum(sr[r]);
      const double psip = rho * warp_sum(dl[r]), phip = rho * warp_sum(dr[r]);
      RootSlot& q = s[r];
      if (q.i < 0) continue;
      const double mag = fabs(psi) + fabs(phi);
      q.it += 1;
      const double f = 1.0 + psi + phi;
      if (q.first) {      // midpoint sweep: origin and bracket by the sign of f
        q.first = false;
        if (!(f > 0.0)) {
          q.ori = q.i + 1;
          q.dori = __ldg(d + q.ori);
          q.lo = -q.half;
          q.hi = 0.0;
          q.x = -q.half;
        }
      } else if (f > 0.0) {
        q.hi = q.x;
      } else {
        q.lo = q.x;
      }
      bool done = fabs(f) <= kEps * (1.0 + 8.0 * mag);
      if (!done) {
        const int64_t pa = q.outer ? k - 2 : q.i, pb = pa + 1;
        const double ga = ((__ldg(d + pa) - q.dori) - q.x);
        const double gb = ((__ldg(d + pb) - q.dori) - q.x);
        const double qa = (ga + gb) * f - ga * gb * (psip + phip);
        const double qb = ga * gb * f;
        const double qc = f - ga * psip - gb * phip;
        const double eta = q.outer ? quad_outer(qa, qb, qc) : quad_inner(qa, qb, qc);
        double xn = (eta == kNoStep) ? 0.5 * (q.lo + q.hi) : q.x + eta;
        if (!(q.lo < xn && xn < q.hi)) xn = 0.5 * (q.lo + q.hi);
        if (xn == q.x) done = true;
        else q.x = xn;
      }
      if (!done && q.it >= kMaxRational) {
        // bisection fallback (_kernels.pyx:158-171), this root alone
        for (int step = 0; step < kMaxBisect; ++step) {
          q.it += 1;
          const double xm = 0.5 * (q.lo + q.hi);
          if (xm <= q.lo || xm >= q.hi) break;
          double acc = 0.0;
          for (int64_t j = lane; j < k; j += 32) {
            const double2 p = __ldg(dz + j);
            acc += rho * p.y / ((p.x - q.dori) - xm);
          }
          const double fm = 1.0 + warp_sum(acc);
          if (fm > 0.0) q.hi = xm; else q.lo = xm;
        }
        q.x = 0.5 * (q.lo + q.hi);
        done = true;
      }
      if (!done) continue;
      // gap pair (_kernels.pyx:213-233) and bracket checks (secular.py:172-179)
      if (lane == 0) {
        const int64_t i = q.i, o = i - ibeg;
        double g, m;
        if (q.outer) {
          g = q.x;
          m = rho * sumz2 - q.x;
          lam[o] = d[i] + q.x;
        } else {
          const double width = d[i + 1] - d[i];
          if (q.ori == i) { g = q.x; m = width - q.x; }
          else { g = width + q.x; m = -q.x; }
          lam[o] = q.dori + q.x;
        }
        gam[o] = g;
        mu[o] = m;
        iters[o] = q.it;
        if (!(g > 0.0)) atomicMin(reinterpret_cast<long long*>(&st->v[1]), (long long)i);
        if (!(m > 0.0)) atomicMin(reinterpret_cast<long long*>(&st->v[2]), (long long)i);
      }
      tot += (unsigned long long)q.it;
      slot_init(q, grab(), d, k, rho, sumz2);
      refilled = true;
    }
    if (refilled) slots_sort<R>(s);
  }
  if (lane == 0 && tot) atomicAdd(reinterpret_cast<unsigned long long*>(&st->v[0]), tot);
}

// dnext[j] = d[j+1]; dnext[k-1] = d[k-1] + gamma[k-1] + mu[k-1]  (secular.py:199)
__global__ void dnext_kernel(const double* __restrict__ d, const double* __restrict__ gam,
                             const double* __restrict__ mu, int64_t k, double* __restrict__ dn) {
  int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= k) return;
  dn[j] = (j + 1 < k) ? d[j + 1] : (d[k - 1] + gam[k - 1]) + mu[k - 1];
}

// zhat_i = sign(z_i) sqrt( prod_{j!=i} (lam_j - d_i)/(d_j - d_i) * gamma_i / rho )
template <int R>
__device__ __forceinline__ void loewner_rows(
    const double* __restrict__ d, const double* __restrict__ dn, const double* __restrict__ gam,
    const double* __restrict__ mu, const double* __restrict__ z, int64_t k, double rho,
    int64_t i0, int64_t ibeg, int64_t iend, double* __restrict__ zhat,
    hsseig_status* __restrict__ st, int lane) {
  double di[R], pr[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    di[r] = (i0 + r < iend) ? __ldg(d + i0 + r) : 0.0;
    pr[r] = 1.0;
  }
  // three ranges so the stable-gap branch is uniform: j < i0 (every row i > j: the
  // (d_i - d_{j+1}) + mu_j form), the band [i0, i0 + R) and j >= i0 + R (i <= j)
  const int64_t jb = min(i0, k), je = min(i0 + R, k);
  for (int64_t j = lane; j < jb; j += 32) {
    const double dj = __ldg(d + j), dnj = __ldg(dn + j), mj = __ldg(mu + j);
#pragma unroll
    for (int r = 0; r < R; ++r) pr[r] *= -((di[r] - dnj) + mj) * rcp_c3(dj - di[r]);
  }
  for (int64_t j = jb + lane; j < je; j += 32) {
    const double dj = __ldg(d + j), dnj = __ldg(dn + j), gj = __ldg(gam + j), mj = __ldg(mu + j);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      int64_t i = i0 + r;
      if (j == i) continue;
      const double num = -stable_gap(i, j, di[r], dj, dnj, gj, mj);
      const double den = dj - di[r];
      pr[r] *= num * rcp_c3(den);
    }
  }
  for (int64_t j = je + lane; j < k; j += 32) {
    const double dj = __ldg(d + j), gj = __ldg(gam + j);
#pragma unroll
    for (int r = 0; r < R; ++r) pr[r] *= -((di[r] - dj) - gj) * rcp_c3(dj - di[r]);
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    double p = warp_prod(pr[r]);
    int64_t i = i0 + r;
    if (lane == 0 && i < iend) {
      double rad = (p * gam[i]) / rho;
      if (!(rad > 0.0) || !isfinite(rad)) {
        atomicMin(reinterpret_cast<long long*>(&st->v[3]), (long long)i);
        zhat[i - ibeg] = 0.0;
      } else {
        zhat[i - ibeg] = copysign(sqrt(rad), z[i]);
      }
    }
  }
}

template <int R>
__global__ void __launch_bounds__(256) loewner_kernel(
    const double* __restrict__ d, const double* __restrict__ dn, const double* __restrict__ gam,
    const double* __restrict__ mu, const double* __restrict__ z, int64_t k, double rho,
    int64_t ibeg, int64_t iend, double* __restrict__ zhat, hsseig_status* __restrict__ st) {
  const int lane = threadIdx.x & 31;
  const int64_t i0 = ibeg + ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * R;
  if (i0 >= iend) return;
  loewner_rows<R>(d, dn, gam, mu, z, k, rho, i0, ibeg, iend, zhat, st, lane);
}

// v_j = 1 / sqrt( sum_i (zhat_i / (d_i - lam_j))^2 )
template <int R>
__device__ __forceinline__ void normalizer_cols(
    const double* __restrict__ d, const double* __restrict__ dn, const double* __restrict__ gam,
    const double* __restrict__ mu, const double* __restrict__ zh, int64_t k, int64_t j0,
    int64_t jbeg, int64_t jend, double* __restrict__ v, int lane) {
  double dj[R], dnj[R], gj[R], mj[R], s[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    int64_t j = j0 + r < jend ? j0 + r : jend - 1;
    dj[r] = __ldg(d + j);
    dnj[r] = __ldg(dn + j);
    gj[r] = __ldg(gam + j);
    mj[r] = __ldg(mu + j);
    s[r] = 0.0;
  }
  // rows i <= j0 use (d_i - d_j) - gam_j for every column of the warp, rows i > j0 + R - 1
  // the (d_i - d_{j+1}) + mu_j form; only the band between needs the branch
  const int64_t ib = min(j0 + 1, k), ie = min(j0 + R, k);
  for (int64_t i = lane; i < ib; i += 32) {
    const double di = __ldg(d + i), zi = __ldg(zh + i);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      double q = zi * rcp_c3((di - dj[r]) - gj[r]);
      s[r] = fma(q, q, s[r]);
    }
  }
  for (int64_t i = ib + lane; i < ie; i += 32) {
    const double di = __ldg(d + i), zi = __ldg(zh + i);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      double g = stable_gap(i, j0 + r, di, dj[r], dnj[r], gj[r], mj[r]);
      double q = zi * rcp_c3(g);
      s[r] = fma(q, q, s[r]);
    }
  }
  for (int64_t i = ie + lane; i < k; i += 32) {
    const double di = __ldg(d + i), zi = __ldg(zh + i);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      double q = zi * rcp_c3((di - dnj[r]) + mj[r]);
      s[r] = fma(q, q, s[r]);
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    double t = warp_sum(s[r]);
    if (lane == 0 && j0 + r < jend) v[j0 + r - jbeg] = 1.0 / sqrt(t);
  }
}

template <int R>
__global__ void __launch_bounds__(256) normalizer_kernel(
    const double* __restrict__ d, const double* __restrict__ dn, const double* __restrict__ gam,
    const double* __restrict__ mu, const double* __restrict__ zh, int64_t k, int64_t jbeg,
    int64_t jend, double* __restrict__ v) {
  const int lane = threadIdx.x & 31;
  const int64_t j0 = jbeg + ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * R;
  if (j0 >= jend) return;
  normalizer_cols<R>(d, dn, gam, mu, zh, k, j0, jbeg, jend, v, lane);
}

// ---------------------------------------------------------------------------
// Level-batched ("wave") variants: every rank-one system of one recursion depth in one
// launch.  System s owns roots [koff[s], koff[s+1]) of the concatenated arrays; seg_of
// maps a root to its system.  One warp per root / row / column (R = 1), so a warp never
// straddles two systems.
// ---------------------------------------------------------------------------
__global__ void wave_square_sum_kernel(const double* __restrict__ z, const int64_t* __restrict__ koff,
                                       double* __restrict__ z2, double* __restrict__ sums) {
  const int s = blockIdx.x;
  const int64_t a = koff[s], k = koff[s + 1] - a;
  __shared__ double part[32];
  double acc = 0.0;
  for (int64_t j = threadIdx.x; j < k; j += blockDim.x) {
    const double q = z[a + j] * z[a + j];
    z2[a + j] = q;
    acc += q;
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = (threadIdx.x < (blockDim.x >> 5)) ? part[threadIdx.x] : 0.0;
    t = warp_sum(t);
    if (threadIdx.x == 0) sums[s] = t;
  }
}

__global__ void __launch_bounds__(256) wave_secular_kernel(
    const double* __restrict__ d, const double* __restrict__ z2, const double* __restrict__ sums,
    const int64_t* __restrict__ koff, const int32_t* __restrict__ seg_of,
    const double* __restrict__ rho, int64_t ntot, double* __restrict__ lam, double* __restrict__ gam,
    double* __restrict__ mu, int32_t* __restrict__ iters, hsseig_status* __restrict__ st) {
  const int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (g >= ntot) return;
  const int s = seg_of[g];
  const int64_t a = koff[s], k = koff[s + 1] - a;
  secular_roots<1>(d + a, z2 + a, sums[s], k, rho[s], g - a, 0, k, lam + a, gam + a, mu + a,
                   iters + a, st + s, threadIdx.x & 31);
}

__global__ void wave_dnext_kernel(const double* __restrict__ d, const double* __restrict__ gam,
                                  const double* __restrict__ mu, const int64_t* __restrict__ koff,
                                  const int32_t* __restrict__ seg_of, int64_t ntot,
                                  double* __restrict__ dn) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= ntot) return;
  const int64_t last = koff[seg_of[g] + 1] - 1;
  dn[g] = (g < last) ? d[g + 1] : (d[last] + gam[last]) + mu[last];
}

__global__ void __launch_bounds__(256) wave_loewner_kernel(
    const double* __restrict__ d, const double* __restrict__ dn, const double* __restrict__ gam,
    const double* __restrict__ mu, const double* __restrict__ z, const int64_t* __restrict__ koff,
    const int32_t* __restrict__ seg_of, const double* __restrict__ rho, int64_t ntot,
    double* __restrict__ zhat, hsseig_status* __restrict__ st) {
  const int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (g >= ntot) return;
  const int s = seg_of[g];
  const int64_t a = koff[s], k = koff[s + 1] - a;
  loewner_rows<1>(d + a, dn + a, gam + a, mu + a, z + a, k, rho[s], g - a, 0, k, zhat + a, st + s,
                  threadIdx.x & 31);
}

__global__ void __launch_bounds__(256) wave_normalizer_kernel(
    const double* __restrict__ d, const double* __restrict__ dn, const double* __restrict__ gam,
    const double* __restrict__ mu, const double* __restrict__ zh, const int64_t* __restrict__ koff,
    const int32_t* __restrict__ seg_of, int64_t ntot, double* __restrict__ v) {
  const int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (g >= ntot) return;
  const int s = seg_of[g];
  const int64_t a = koff[s], k = koff[s + 1] - a;
  normalizer_cols<1>(d + a, dn + a, gam + a, mu + a, zh + a, k, g - a, 0, k, v + a,
                     threadIdx.x & 31);
}

}  // namespace hsseig

using namespace hsseig;

extern "C" int hsseig_status_init(hsseig_status* st, int64_t k, void* stream) {
  hsseig_status h;
  for (int t = 0; t < 8; ++t) h.v[t] = 0;
  h.v[1] = h.v[2] = h.v[3] = k;
  void* dst[1] = {st};
  const void* src[1] = {&h};
  const size_t nb[1] = {sizeof(h)};
  if (!upload_async(1, dst, src, nb, (cudaStream_t)stream)) return HSSEIG_ERR_CUDA;
  return HSSEIG_OK;
}

extern "C" int hsseig_secular_part(const double* d, const double* z, int64_t k, double rho,
                                   int64_t ibeg, int64_t iend, double* lam, double* gamma,
                                   double* mu, int32_t* iters, double* work, hsseig_status* st,
                                   void* stream) {
  if (k < 1 || !(rho > 0.0) || !d || !z || !lam || !gamma || !mu || !iters || !work || !st ||
      ibeg < 0 || iend > k || ibeg > iend)
    HSS_ARG_FAIL();
  if (ibeg == iend) return HSSEIG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (reinterpret_cast<uintptr_t>(work) & 15) HSS_ARG_FAIL();   // packed 16-byte poles
  double2* dz = reinterpret_cast<double2*>(work);
  double* sum = work + 2 * k;
  pack_square_sum_kernel<<<1, 1024, 0, s>>>(d, z, k, dz, sum);
  HSS_CHECK_LAUNCH();
  // dynamically scheduled slots: one wave of resident warps pulls roots from a counter
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int64_t n = iend - ibeg;
  unsigned long long* ctr = reinterpret_cast<unsigned long long*>(sum + 1);
  // two slots per warp, two CTAs per SM (122 registers, no spills): 3.6 ms at k = 32768,
  // against 3.9-4.4 ms for 1-4 slots at 2-4 CTAs per SM and 4.2 ms for the static kernel
  constexpr int R = 2, MINB = 2;
  const int64_t warps = imin64((n + R - 1) / R, (int64_t)sms * MINB * 8);   // one resident wave
  secular_queue_kernel<R, MINB><<<(int)((warps + 7) / 8), 256, 0, s>>>(
      d, dz, sum, k, rho, ibeg, iend, lam, gamma, mu, iters, st, ctr);
  HSS_CHECK_LAUNCH();
  return HSSEIG_OK;
}

extern "C" int hsseig_secular(const double* d, const double* z, int64_t k, double rho,
                              double* lam, double* gamma, double* mu, int32_t* iters, double* work,
                              hsseig_status* st, void* stream) {
  return hsseig_secular_part(d, z, k, rho, 0, k, lam, gamma, mu, iters, work, st, stream);
}

extern "C" int hsseig_dnext(const double* d, const double* gamma, const double* mu, int64_t k,
                            double* dnext, void* stream) {
  if (k < 1) HSS_ARG_FAIL();
  dnext_kernel<<<(unsigned)((k + 255) / 256), 256, 0, (cudaStream_t)stream>>>(d, gamma, mu, k, dnext);
  HSS_CHECK_LAUNCH();
  return HSSEIG_OK;
}

extern "C" int hsseig_loewner_part(const double* d, const double* dnext, const double* gamma,
                                   const double* mu, const double* z, int64_t k, double rho,
                                   int64_t ibeg, int64_t iend, double* zhat, hsseig_status* st,
                                   void* stream) {
  if (k < 1 || !(rho > 0.0) || ibeg < 0 || iend > k || ibeg > iend) HSS_ARG_FAIL();
  if (ibeg == iend) return HSSEIG_OK;
  constexpr int R = 4;   // rows per warp: 2 / 6 / 8 measured 4-17% slower at k = 32768
  const int64_t warps = (iend - ibeg + R - 1) / R;
  loewner_kernel<R><<<(unsigned)((warps + 7) / 8), 256, 0, (cudaStream_t)stream>>>(
      d, dnext, gamma, mu, z, k, rho, ibeg, iend, zhat, st);
  HSS_CHECK_LAUNCH();
  return HSSEIG_OK;
}

extern "C" int hsseig_loewner(const double* d, const double* dnext, const double* gamma,
                              const double* mu, const double* z, int64_t k, double rho,
                              double* zhat, hsseig_status* st, void* stream) {
  return hsseig_loewner_part(d, dnext, gamma, mu, z, k, rho, 0, k, zhat, st, stream);
}

extern "C" int hsseig_normalizers_part(const double* d, const double* dnext, const double* gamma,
                                       const double* mu, const double* zhat, int64_t k,
                                       int64_t jbeg, int64_t jend, double* v, void* stream) {
  if (k < 1 || jbeg < 0 || jend > k || jbeg > jend) HSS_ARG_FAIL();
  if (jbeg == jend) return HSSEIG_OK;
  constexpr int R = 4;
  const int64_t warps = (jend - jbeg + R - 1) / R;
  normalizer_kernel<R><<<(unsigned)((warps + 7) / 8), 256, 0, (cudaStream_t)stream>>>(
      d, dnext, gamma, mu, zhat, k, jbeg, jend, v);
  HSS_CHECK_LAUNCH();
  return HSSEIG_OK;
}

extern "C" int hsseig_normalizers(const double* d, const double* dnext, const double* gamma,
                                  const double* mu, const double* zhat, int64_t k, double* v,
                                  void* stream) {
  return hsseig_normalizers_part(d, dnext, gamma, mu, zhat, k, 0, k, v, stream);
}

// ---------------------------------------------------------------------------- wave ABI
extern "C" int hsseig_wave_secular(const double* d, const double* z, const int64_t* koff,
                                   const int32_t* seg_of, const double* rho, int64_t nseg,
                                   int64_t ntot, double* lam, double* gamma, double* mu,
                                   int32_t* iters, double* work, hsseig_status* st, void* stream) {
  if (nseg < 0 || ntot < 0 || !d || !z || !koff || !seg_of || !rho || !lam || !gamma || !mu ||
      !iters || !work || !st)
    HSS_ARG_FAIL();
  if (nseg == 0 || ntot == 0) return HSSEIG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  double* z2 = work;
  double* sums = work + ntot;
  wave_square_sum_kernel<<<(unsigned)nseg, 256, 0, s>>>(z, koff, z2, sums);
  HSS_CHECK_LAUNCH();
  wave_secular_kernel<<<(unsigned)((ntot + 7) / 8), 256, 0, s>>>(d, z2, sums, koff, seg_of, rho, ntot,
                                                                 lam, gamma, mu, iters, st);
  HSS_CHECK_LAUNCH();
  return HSSEIG_OK;
}

extern "C" int hsseig_wave_dnext(const double* d, const double* gamma, const double* mu,
                                 const int64_t* koff, const int32_t* seg_of, int64_t ntot,
                                 double* dnext, void* stream) {
  if (ntot < 0) HSS_ARG_FAIL();
  if (ntot == 0) return HSSEIG_OK;
  wave_dnext_kernel<<<(unsigned)((ntot + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      d, gamma, mu, koff, seg_of, ntot, dnext);
  HSS_CHECK_LAUNCH();
  return HSSEIG_OK;
}

extern "C" int hsseig_wave_loewner(const double* d, const double* dnext, const double* gamma,
                                   const double* mu, const double* z, const int64_t* koff,
                                   const int32_t* seg_of, const double* rho, int64_t ntot,
                                   double* zhat, hsseig_status* st, void* stream) {
  if (ntot < 0) HSS_ARG_FAIL();
  if (ntot == 0) return HSSEIG_OK;
  wave_loewner_kernel<<<(unsigned)((ntot + 7) / 8), 256, 0, (cudaStream_t)stream>>>(
      d, dnext, gamma, mu, z, koff, seg_of, rho, ntot, zhat, st);
  HSS_CHECK_LAUNCH();
  return HSSEIG_OK;
}

extern "C" int hsseig_wave_normalizers(const double* d, const double* dnext, const double* gamma,
                                       const double* mu, const double* zhat, const int64_t* koff,
                                       const int32_t* seg_of, int64_t ntot, double* v,
                                       void* stream) {
  if (ntot < 0) HSS_ARG_FAIL();
  if (ntot == 0) return HSSEIG_OK;
  wave_normalizer_kernel<<<(unsigned)((ntot + 7) / 8), 256, 0, (cudaStream_t)stream>>>(
      d, dnext, gamma, mu, zhat, koff, seg_of, ntot, v);
  HSS_CHECK_LAUNCH();
  return HSSEIG_OK;
}
