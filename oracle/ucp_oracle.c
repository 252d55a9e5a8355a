/* ORACLE -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference's hot path (`ucpsolve`, arXiv 1908.04489)
 * in plain C, used as the parity checker by tests/, by
 * __graft_entry__.smoke() and as the CPU baseline leg of bench.py.  The
 * product (paper_1908_04489_b200/) never links, loads or calls this file.
 *
 * Every function follows the numba kernel it cites operation by operation
 * (left-to-right evaluation, no FMA contraction: build with
 * -ffp-contract=off) and calls the host glibc `exp`/`erf`, exactly as the
 * numba kernels do (numba lowers np.exp/math.erf to those libm symbols), so
 * on the same host its results are bitwise the reference's.  Pinned against
 * golden vectors produced by the reference itself (tests/golden/, made by
 * tools/gen_golden.py) in tests/test_oracle_golden.py.
 *
 * Parallelism mirrors numba's `prange` over independent outputs (OpenMP),
 * which does not change any result bit.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define GAUSS_CUT 12.0
static const double INV_SQRT_2PI = 0.3989422804014327;  /* 1/np.sqrt(2*pi), kernels.py:47 */
static const double INV_SQRT_2 = 0.7071067811865475;    /* 1/np.sqrt(2),    kernels.py:48 */

int orc_num_threads(void);

/* kernels.py:398-404 (_phi_cdf_nb) */
static double phi_cdf(double z) {
  if (z <= -GAUSS_CUT) return 0.0;
  if (z >= GAUSS_CUT) return 1.0;
  return 0.5 * (1.0 + erf(z * INV_SQRT_2));
}

double orc_phi_cdf(double z) { return phi_cdf(z); }

/* kernels.py:136-144 (_trapezoid_impl) */
double orc_trapezoid(const double* samples, int64_t n, double spacing) {
  if (n == 1) return 0.0;
  double acc = 0.5 * samples[0];
  for (int64_t i = 1; i < n - 1; ++i) acc += samples[i];
  acc += 0.5 * samples[n - 1];
  return acc * spacing;
}

/* kernels.py:147-160 (_segmented_argmin_impl) */
void orc_segmented_argmin(const double* costs, const int64_t* offsets, int64_t nseg,
                          int64_t* out) {
#pragma omp parallel for schedule(static)
  for (int64_t s = 0; s < nseg; ++s) {
    int64_t lo = offsets[s], hi = offsets[s + 1];
    int64_t best = lo;
    double best_val = costs[lo];
    for (int64_t t = lo + 1; t < hi; ++t) {
      if (costs[t] < best_val) {
        best_val = costs[t];
        best = t;
      }
    }
    out[s] = best;
  }
}

/* kernels.py:163-187 (_flatten_windows_impl, with first-occurrence dedup).
 * Pass flat=NULL to get only the total (returned); offsets always written. */
int64_t orc_flatten_windows(const double* values, const int64_t* lo, const int64_t* hi,
                            int64_t d, double* flat, int64_t* offsets) {
  int64_t pos = 0;
  offsets[0] = 0;
  for (int64_t i = 0; i < d; ++i) {
    int64_t start = pos;
    for (int64_t j = lo[i]; j <= hi[i]; ++j) {
      double v = values[j];
      int dup = 0;
      if (flat) {
        for (int64_t t = start; t < pos; ++t) {
          if (flat[t] == v) {
            dup = 1;
            break;
          }
        }
      } else {
        /* counting pass: same rule, read back from `values` */
        for (int64_t t = lo[i]; t < j; ++t) {
          if (values[t] == v) {
            dup = 1;
            break;
          }
        }
      }
      if (!dup) {
        if (flat) flat[pos] = v;
        ++pos;
      }
    }
    offsets[i + 1] = pos;
  }
  return pos;
}

/* One centre of kernels.py:406-445 (_gauss_moments_grid_numba loop body). */
static void gauss_grid_one(double st, const double* v, double a, double h, int64_t d, double b,
                           double q, double* o0, double* o1, double* o2) {
  int64_t jlo = (int64_t)ceil(((st - GAUSS_CUT) - a) / h);
  int64_t jhi = (int64_t)floor(((st + GAUSS_CUT) - a) / h);
  if (jlo < 0) jlo = 0;
  if (jhi > d - 1) jhi = d - 1;
  double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
  if (jlo <= jhi) {
    double tt = (a + (double)jlo * h) - st;
    double pdf = exp((-0.5 * tt) * tt) * INV_SQRT_2PI;
    double ratio = exp((-h) * (tt + 0.5 * h));
    for (int64_t j = jlo; j <= jhi; ++j) {
      double w = h;
      if (j == 0 || j == d - 1) w = 0.5 * h;
      double wp = w * pdf;
      double vj = v[j];
      acc0 += wp;
      acc1 += wp * vj;
      acc2 += (wp * vj) * vj;
      pdf *= ratio;
      ratio *= q;
    }
  }
  double lo = phi_cdf(a - st);
  double hi = phi_cdf(st - b);
  *o0 = (acc0 + lo) + hi;
  *o1 = (acc1 + lo * v[0]) + hi * v[d - 1];
  *o2 = (acc2 + (lo * v[0]) * v[0]) + (hi * v[d - 1]) * v[d - 1];
}

/* kernels.py:406-445 (_gauss_moments_grid_numba) */
void orc_gauss_moments_grid(const double* s, int64_t n, const double* v, double a, double h,
                            int64_t d, double* t0, double* t1, double* t2) {
  double b = a + h * (double)(d - 1);
  double q = exp((-h) * h);
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t t = 0; t < n; ++t) gauss_grid_one(s[t], v, a, h, d, b, q, &t0[t], &t1[t], &t2[t]);
}

/* One query of kernels.py:447-486 (_gauss_moments_points_numba loop body). */
static void gauss_points_one(double yt, const double* x, const double* w, int64_t m, double a,
                             double h, int64_t d, double b, double* o0, double* o1, double* o2) {
  int64_t j = (int64_t)ceil((yt - a) / h - 0.5);
  if (j < 0) j = 0;
  if (j > d - 1) j = d - 1;
  int at_left = j == 0;
  int at_right = j == d - 1;
  double factor = (at_left || at_right) ? 0.5 : 1.0;
  double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
  for (int64_t i = 0; i < m; ++i) {
    double xi = x[i];
    double diff = yt - xi;
    double wp = 0.0;
    if (diff <= GAUSS_CUT && diff >= -GAUSS_CUT)
      wp = (factor * exp((-0.5 * diff) * diff)) * INV_SQRT_2PI;
    if (at_left) wp += phi_cdf(a - xi) / h;
    if (at_right) wp += phi_cdf(xi - b) / h;
    if (wp != 0.0) {
      wp *= w[i];
      acc0 += wp;
      acc1 += wp * xi;
      acc2 += (wp * xi) * xi;
    }
  }
  *o0 = acc0;
  *o1 = acc1;
  *o2 = acc2;
}

/* kernels.py:447-486 (_gauss_moments_points_numba) */
void orc_gauss_moments_points(const double* y, int64_t n, const double* x, const double* w,
                              int64_t m, double a, double h, int64_t d, double* o0, double* o1,
                              double* o2) {
  double b = a + h * (double)(d - 1);
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t t = 0; t < n; ++t) gauss_points_one(y[t], x, w, m, a, h, d, b, &o0[t], &o1[t], &o2[t]);
}

/* witsenhausen.py:31-33 (_quad_in_u): a*u*u - 2.0*b*u + c */
static inline double quad_in_u(double a, double b, double c, double u) {
  return (((a * u) * u) - ((2.0 * b) * u)) + c;
}

/* witsenhausen.py:62-70 (marginal_cost_segmented, m == 0).  `f0` holds
 * numerics.pdf(N(0, sigma), y) per SEGMENT (the reference repeats it per
 * candidate; every repeat is the same value). */
void orc_wc_stage0_cost(const double* u_flat, const int64_t* offsets, int64_t nseg,
                        const double* y, const double* f0, const double* v1, double a1,
                        double h1, int64_t d1, double k, double* out) {
  double b = a1 + h1 * (double)(d1 - 1);
  double q = exp((-h1) * h1);
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t sgi = 0; sgi < nseg; ++sgi) {
    for (int64_t c = offsets[sgi]; c < offsets[sgi + 1]; ++c) {
      double u = u_flat[c];
      double s = y[sgi] + u;
      double t0, t1, t2;
      gauss_grid_one(s, v1, a1, h1, d1, b, q, &t0, &t1, &t2);
      double inner = quad_in_u(t0, t1, t2, s);
      out[c] = f0[sgi] * ((((k * k) * u) * u) + inner);
    }
  }
}

/* witsenhausen.py:71-78 (marginal_cost_segmented, m == 1).  `x1` is the
 * numpy sum grids[0].points + U.values(0); `fw0` the trapezoid-weighted
 * stage-0 density (witsenhausen.py:47-53). */
void orc_wc_stage1_cost(const double* u_flat, const int64_t* offsets, int64_t nseg,
                        const double* y, const double* x1, const double* fw0, int64_t d0,
                        double a1, double h1, int64_t d1, double* out) {
  double* mom = (double*)malloc(sizeof(double) * 3 * (size_t)(nseg > 0 ? nseg : 1));
  orc_gauss_moments_points(y, nseg, x1, fw0, d0, a1, h1, d1, mom, mom + nseg, mom + 2 * nseg);
#pragma omp parallel for schedule(static)
  for (int64_t sgi = 0; sgi < nseg; ++sgi)
    for (int64_t c = offsets[sgi]; c < offsets[sgi + 1]; ++c)
      out[c] = quad_in_u(mom[sgi], mom[nseg + sgi], mom[2 * nseg + sgi], u_flat[c]);
  free(mom);
}

/* ---------------------------------------------------------------------------
 * Uniform-noise kernels (config 5: ZeroDelay, Inventory).  Cell j of a grid
 * spans [a + h(j - 1/2), a + h(j + 1/2)], the end cells extend to -/+HUGE
 * (kernels.py:302-309 _cell_edges; numba bodies kernels.py:488-615).
 * ------------------------------------------------------------------------- */
#define HUGE_EDGE 1.0e300

static inline int64_t cell_index(double x, double a, double h, int64_t d) {
  int64_t j = (int64_t)ceil((x - a) / h - 0.5);
  if (j < 0) j = 0;
  if (j > d - 1) j = d - 1;
  return j;
}

static inline double cell_left(int64_t j, double a, double h) { return j > 0 ? a + h * ((double)j - 0.5) : -HUGE_EDGE; }
static inline double cell_right(int64_t j, double a, double h, int64_t d) {
  return j < d - 1 ? a + h * ((double)j + 0.5) : HUGE_EDGE;
}

/* kernels.py:488-525 (_unif_moments_grid_numba) */
void orc_unif_moments_grid(const double* x, int64_t n, const double* v, double a, double h, int64_t d,
                           double rad, double* s0, double* s1, double* s2) {
  double inv = 1.0 / (2.0 * rad);
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < n; ++t) {
    double xlo = x[t] - rad, xhi = x[t] + rad;
    int64_t jlo = cell_index(xlo, a, h, d), jhi = cell_index(xhi, a, h, d);
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
    for (int64_t j = jlo; j <= jhi; ++j) {
      double lj = cell_left(j, a, h), rj = cell_right(j, a, h, d);
      double lo = xlo > lj ? xlo : lj;
      double hi = xhi < rj ? xhi : rj;
      double ov = hi - lo;
      if (ov > 0.0) {
        double vj = v[j];
        acc0 += ov;
        acc1 += ov * vj;
        acc2 += (ov * vj) * vj;
      }
    }
    s0[t] = acc0 * inv;
    s1[t] = acc1 * inv;
    s2[t] = acc2 * inv;
  }
}

/* kernels.py:528-555 (_unif_ball_sum_numba) */
void orc_unif_ball_sum(const double* x, int64_t n, const double* g, double a, double h, int64_t d, double rad,
                       double* out) {
  double inv = 1.0 / (2.0 * rad);
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < n; ++t) {
    double xlo = x[t] - rad, xhi = x[t] + rad;
    int64_t jlo = cell_index(xlo, a, h, d), jhi = cell_index(xhi, a, h, d);
    double acc = 0.0;
    for (int64_t j = jlo; j <= jhi; ++j) {
      double lj = cell_left(j, a, h), rj = cell_right(j, a, h, d);
      double lo = xlo > lj ? xlo : lj;
      double hi = xhi < rj ? xhi : rj;
      double ov = hi - lo;
      if (ov > 0.0) acc += ov * g[j];
    }
    out[t] = acc * inv;
  }
}

/* kernels.py:558-577 (_unif_propagate_numba): out has d entries */
void orc_unif_propagate(const double* masses, const double* centers, int64_t n, double a, double h, int64_t d,
                        double rad, double* out) {
  double inv = 1.0 / ((2.0 * rad) * h);
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < d; ++j) {
    double lj = cell_left(j, a, h), rj = cell_right(j, a, h, d);
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      double lo = centers[i] - rad, hi = centers[i] + rad;
      if (lo < lj) lo = lj;
      if (hi > rj) hi = rj;
      double ov = hi - lo;
      if (ov > 0.0) acc += masses[i] * ov;
    }
    out[j] = acc * inv;
  }
}

/* kernels.py:580-615 (_unif_moments_points_numba) */
void orc_unif_moments_points(const double* y, int64_t n, const double* centers, const double* w,
                             const double* vals, int64_t m, double a, double h, int64_t d, double rad,
                             double* m0, double* m1, double* m2) {
  double inv = 1.0 / ((2.0 * rad) * h);
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < n; ++t) {
    int64_t j = cell_index(y[t], a, h, d);
    double lj = cell_left(j, a, h), rj = cell_right(j, a, h, d);
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
    for (int64_t i = 0; i < m; ++i) {
      double lo = centers[i] - rad, hi = centers[i] + rad;
      if (lo < lj) lo = lj;
      if (hi > rj) hi = rj;
      double ov = hi - lo;
      if (ov > 0.0) {
        double wov = w[i] * ov, vi = vals[i];
        acc0 += wov;
        acc1 += wov * vi;
        acc2 += (wov * vi) * vi;
      }
    }
    m0[t] = acc0 * inv;
    m1[t] = acc1 * inv;
    m2[t] = acc2 * inv;
  }
}

#ifdef _OPENMP
#include <omp.h>
int orc_num_threads(void) { return omp_get_max_threads(); }
void orc_set_threads(int n) { omp_set_num_threads(n); }
#else
int orc_num_threads(void) { return 1; }
void orc_set_threads(int n) { (void)n; }
#endif
