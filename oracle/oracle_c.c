/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle for the merge-step hot path.
 *
 * Plain-C restatement of the reference's two compiled kernels that the
 * merge path touches:
 *   - the secular-equation root solver  (pkg/src/hsseig/_kernels.pyx:19-234)
 *   - the small implicit-QL base case   (pkg/src/hsseig/_kernels.pyx:352-411)
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library (as the checker / CPU baseline); the product path never does.
 *
 * Build: see oracle/Makefile (gcc -O3 -shared -fPIC).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#define ORC_EPS 2.220446049250313e-16
#define ORC_MAX_RATIONAL 60   /* _kernels.pyx:11 */
#define ORC_MAX_BISECT 200    /* _kernels.pyx:12 */
#define ORC_NO_STEP (-1e308)  /* "no usable quadratic root" sentinel */

/* Quadratic c*eta^2 - a*eta + b = 0, interior-root branch (_kernels.pyx:19-34). */
static double quad_root_inner(double a, double b, double c) {
    double disc = a * a - 4.0 * b * c;
    double s = sqrt(disc < 0.0 ? 0.0 : disc);
    if (c == 0.0) return a != 0.0 ? b / a : ORC_NO_STEP;
    if (a <= 0.0) return (a - s) / (2.0 * c);
    return (a + s) != 0.0 ? 2.0 * b / (a + s) : ORC_NO_STEP;
}

/* Same quadratic, branch for the root right of the last pole (_kernels.pyx:37-50). */
static double quad_root_outer(double a, double b, double c) {
    double disc = a * a - 4.0 * b * c;
    double s = sqrt(disc < 0.0 ? 0.0 : disc);
    if (a >= 0.0) return c != 0.0 ? (a + s) / (2.0 * c) : ORC_NO_STEP;
    return (a - s) != 0.0 ? 2.0 * b / (a - s) : ORC_NO_STEP;
}

/*
 * One root (_kernels.pyx:53-175).  The root lives in (d[i], d[i+1]) (or to the
 * right of d[k-1] when i == k-1); it is tracked as x = lam - d[origin] where the
 * origin is the nearer pole, decided from the sign of f at the interval midpoint.
 * Returns the number of iterations; writes origin and x.
 */
static int64_t one_root(const double *d, const double *z2, int64_t k, double rho,
                        int64_t i, double sumz2, double *shift,
                        int64_t *origin_out, double *x_out) {
    int outer = (i == k - 1);
    int64_t origin, pa, pb;
    double lo, hi;
    if (outer) {
        origin = k - 1;
        lo = 0.0;
        hi = rho * sumz2;
        pa = k - 2;
        pb = k - 1;
    } else {
        double half = 0.5 * (d[i + 1] - d[i]);
        double f_half = 1.0;
        for (int64_t j = 0; j < k; ++j) f_half += rho * z2[j] / ((d[j] - d[i]) - half);
        if (f_half > 0.0) { origin = i;     lo = 0.0;   hi = half; }
        else              { origin = i + 1; lo = -half; hi = 0.0;  }
        pa = i;
        pb = i + 1;
    }
    for (int64_t j = 0; j < k; ++j) shift[j] = d[j] - d[origin];

    /* left sum runs over poles j <= split, right sum over the rest */
    int64_t split = outer ? k - 2 : i;
    double x = 0.5 * (lo + hi);
    int64_t iters = 0;
    int done = 0;
    for (int step = 0; step < ORC_MAX_RATIONAL; ++step) {
        ++iters;
        double sl = 0.0, sr = 0.0, dl = 0.0, dr = 0.0, mag = 0.0;
        for (int64_t j = 0; j < k; ++j) {
            double gap = shift[j] - x;
            double term = z2[j] / gap;
            if (j <= split) { sl += term; dl += term / gap; }
            else            { sr += term; dr += term / gap; }
            mag += fabs(term);
        }
        sl *= rho; sr *= rho; dl *= rho; dr *= rho; mag *= rho;
        double f = 1.0 + sl + sr;
        if (f > 0.0) hi = x; else lo = x;
        if (fabs(f) <= ORC_EPS * (1.0 + 8.0 * mag)) { done = 1; break; }
        /* two-pole rational model through the neighbouring poles */
        double ga = shift[pa] - x, gb = shift[pb] - x;
        double qa = (ga + gb) * f - ga * gb * (dl + dr);
        double qb = ga * gb * f;
        double qc = f - ga * dl - gb * dr;
        double eta = outer ? quad_root_outer(qa, qb, qc) : quad_root_inner(qa, qb, qc);
        double xn = (eta == ORC_NO_STEP) ? 0.5 * (lo + hi) : x + eta;
        if (!(lo < xn && xn < hi)) xn = 0.5 * (lo + hi);
        if (xn == x) { done = 1; break; }
        x = xn;
    }
    if (!done) {
        /* bisection fallback on the maintained bracket (_kernels.pyx:158-171) */
        for (int step = 0; step < ORC_MAX_BISECT; ++step) {
            ++iters;
            x = 0.5 * (lo + hi);
            if (x <= lo || x >= hi) break;
            double f = 1.0;
            for (int64_t j = 0; j < k; ++j) f += rho * z2[j] / (shift[j] - x);
            if (f > 0.0) hi = x; else lo = x;
        }
        x = 0.5 * (lo + hi);
    }
    *origin_out = origin;
    *x_out = x;
    return iters;
}

/*
 * All k roots plus gap pairs (_kernels.pyx:178-234):
 *   lam[i] = d[origin] + x, gamma[i] = lam[i] - d[i], mu[i] = d[i+1] - lam[i]
 * (mu[k-1] measured against the virtual pole d[k-1] + rho*sum z^2).
 * Returns total iterations.  per_root (optional) receives per-root counts.
 */
int64_t oracle_secular_all(const double *d, const double *z, int64_t k, double rho,
                           double *lam, double *gamma, double *mu, int64_t *per_root) {
    double *z2 = (double *)malloc(sizeof(double) * (size_t)k);
    double *shift = (double *)malloc(sizeof(double) * (size_t)k);
    double sumz2 = 0.0;
    for (int64_t j = 0; j < k; ++j) { z2[j] = z[j] * z[j]; sumz2 += z2[j]; }
    int64_t total = 0;
    if (k == 1) {
        double g = rho * sumz2;
        lam[0] = d[0] + g; gamma[0] = g; mu[0] = 0.0;
        if (per_root) per_root[0] = 1;
        free(z2); free(shift);
        return 1;
    }
    for (int64_t i = 0; i < k; ++i) {
        int64_t origin; double x;
        int64_t it = one_root(d, z2, k, rho, i, sumz2, shift, &origin, &x);
        total += it;
        if (per_root) per_root[i] = it;
        if (i == k - 1) {
            gamma[i] = x;
            mu[i] = rho * sumz2 - x;
            lam[i] = d[i] + x;
        } else {
            double width = d[i + 1] - d[i];
            if (origin == i) { gamma[i] = x; mu[i] = width - x; }
            else             { gamma[i] = width + x; mu[i] = -x; }
            lam[i] = d[origin] + x;
        }
    }
    free(z2); free(shift);
    return total;
}

/*
 * Implicit QL with Wilkinson shift on a small tridiagonal (_kernels.pyx:352-411).
 * d (n) and e (n-1) are overwritten; Z (n x n, row-major) accumulates rotations.
 * Returns 0, or 1 + l when eigenvalue l stalls after max_iter sweeps.
 */
int oracle_tql2(double *d, const double *e, double *Z, int64_t n, int max_iter) {
    if (n == 1) return 0;
    double *f = (double *)calloc((size_t)n, sizeof(double));
    for (int64_t t = 0; t + 1 < n; ++t) f[t] = e[t];
    for (int64_t l = 0; l < n; ++l) {
        int sweeps = 0;
        for (;;) {
            int64_t m = l;
            for (; m < n - 1; ++m) {
                double scale = fabs(d[m]) + fabs(d[m + 1]);
                if (fabs(f[m]) <= ORC_EPS * scale) break;
            }
            if (m == l) break;
            if (++sweeps > max_iter) { free(f); return (int)(1 + l); }
            double g = (d[l + 1] - d[l]) / (2.0 * f[l]);
            double r = hypot(g, 1.0);
            g = d[m] - d[l] + f[l] / (g + copysign(r, g));
            double s = 1.0, c = 1.0, p = 0.0;
            int underflow = 0;
            for (int64_t t = m - 1; t >= l; --t) {
                double ff = s * f[t], bb = c * f[t];
                r = hypot(ff, g);
                f[t + 1] = r;
                if (r == 0.0) { d[t + 1] -= p; f[m] = 0.0; underflow = 1; break; }
                s = ff / r;
                c = g / r;
                g = d[t + 1] - p;
                r = (d[t] - g) * s + 2.0 * c * bb;
                p = s * r;
                d[t + 1] = g + p;
                g = c * r - bb;
                for (int64_t row = 0; row < n; ++row) {
                    double zl = Z[row * n + t], zr = Z[row * n + t + 1];
                    Z[row * n + t + 1] = s * zl + c * zr;
                    Z[row * n + t] = c * zl - s * zr;
                }
            }
            if (!underflow) { d[l] -= p; f[l] = g; f[m] = 0.0; }
        }
    }
    free(f);
    return 0;
}
