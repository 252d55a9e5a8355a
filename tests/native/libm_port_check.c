/* Test-only: host build of the product's libm port (csrc/ucp_libm.h) next to
 * the host's own libm, so CPU tests can prove the port bit-exact without a
 * GPU.  Built with -ffp-contract=off -mfma (the port spells its FMAs). */
#include <math.h>
#include <stdint.h>
#include "../../paper_1908_04489_b200/csrc/ucp_libm.h"

static const uint64_t TAB[256] = UCP_EXP_TAB_INIT;

double port_exp(double x) { return ucp_exp_tab(x, TAB); }
double port_exp_core(double x) { return ucp_exp_core(x, (const ucp_exp_entry*)TAB); }

/* exp_core == glibc exp on uniform [lo, hi] (caller keeps |x| < 512). */
int64_t compare_core(int64_t n, uint64_t seed, double lo, double hi, double* first_bad);
double port_erf(double x) { return ucp_erf_tab(x, TAB); }
double host_exp(double x) { return exp(x); }
double host_erf(double x) { return erf(x); }

static uint64_t splitmix(uint64_t* s) {
  uint64_t z = (*s += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

/* Uniform samples on [lo, hi]; returns number of bitwise mismatches and the
 * first offending argument in *first_bad. which: 0 = exp, 1 = erf. */
int64_t compare_uniform(int which, int64_t n, uint64_t seed, double lo, double hi,
                        double* first_bad) {
  int64_t bad = 0;
  uint64_t s = seed;
  for (int64_t i = 0; i < n; ++i) {
    double u = (double)(splitmix(&s) >> 11) * 0x1.0p-53;
    double x = lo + (hi - lo) * u;
    double a = which ? ucp_erf_tab(x, TAB) : ucp_exp_tab(x, TAB);
    double b = which ? erf(x) : exp(x);
    uint64_t ua = ucp_asu64(a), ub = ucp_asu64(b);
    if (ua != ub && !(a != a && b != b)) {
      if (bad == 0) *first_bad = x;
      ++bad;
    }
  }
  return bad;
}

/* Random bit patterns (all exponents), same contract. */
int64_t compare_bits(int which, int64_t n, uint64_t seed, double* first_bad) {
  int64_t bad = 0;
  uint64_t s = seed;
  for (int64_t i = 0; i < n; ++i) {
    double x = ucp_asf64(splitmix(&s));
    double a = which ? ucp_erf_tab(x, TAB) : ucp_exp_tab(x, TAB);
    double b = which ? erf(x) : exp(x);
    uint64_t ua = ucp_asu64(a), ub = ucp_asu64(b);
    if (ua != ub && !(a != a && b != b)) {
      if (bad == 0) *first_bad = x;
      ++bad;
    }
  }
  return bad;
}

int64_t compare_core(int64_t n, uint64_t seed, double lo, double hi, double* first_bad) {
  int64_t bad = 0;
  uint64_t s = seed;
  for (int64_t i = 0; i < n; ++i) {
    double u = (double)(splitmix(&s) >> 11) * 0x1.0p-53;
    double x = lo + (hi - lo) * u;
    if (i % 7 == 0) x = x * 0x1.0p-60; /* tiny arguments: glibc's 1.0 + x branch */
    if (i % 1000 == 1) x = (i & 2) ? 0.0 : -0.0;
    double a = ucp_exp_core(x, (const ucp_exp_entry*)TAB);
    double b = exp(x);
    if (ucp_asu64(a) != ucp_asu64(b)) {
      if (bad == 0) *first_bad = x;
      ++bad;
    }
  }
  return bad;
}
