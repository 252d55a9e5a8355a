// Config 5 (PAPER.md's additional examples): the uniform-noise kernels and
// the ZeroDelay / Inventory (M >= 1 stages) marginal costs, plus generic
// device sweeps templated on a per-problem cost functor.  Included at the
// end of ucp_kernels.cu (shares its workspace, error and launch plumbing).
//
// Same ref-order contract as the Witsenhausen path: every output is one
// thread's serial loop in the reference's order with the reference's
// association; parallelism spans independent outputs only.

namespace {

constexpr double kHugeEdge = 1.0e300;  // kernels.py:61 _HUGE

// cell j spans [a + h(j - 1/2), a + h(j + 1/2)], end cells open (kernels.py:302-309)
__device__ __forceinline__ long long cell_index(double x, double a, double h, int64_t d) {
  long long j = (long long)ceil((x - a) / h - 0.5);
  if (j < 0) j = 0;
  if (j > d - 1) j = d - 1;
  return j;
}
__device__ __forceinline__ double cell_left(long long j, double a, double h) {
  return j > 0 ? a + h * ((double)j - 0.5) : -kHugeEdge;
}
__device__ __forceinline__ double cell_right(long long j, double a, double h, int64_t d) {
  return j < d - 1 ? a + h * ((double)j + 0.5) : kHugeEdge;
}

// numpy.maximum(a, b) as this NumPy evaluates it (NaN in a wins, ties -> b)
__device__ __forceinline__ double np_maximum(double a, double b) { return (a > b || a != a) ? a : b; }

struct Mom3U {
  double s0, s1, s2;
};

// kernels.py:495-525: overlap moments of v under U(x - rad, x + rad)
__device__ __forceinline__ Mom3U unif_moments_at(double x, const double* __restrict__ v, double a, double h,
                                                 int64_t d, double rad) {
  const double xlo = x - rad, xhi = x + rad;
  const long long jlo = cell_index(xlo, a, h, d), jhi = cell_index(xhi, a, h, d);
  double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
  for (long long j = jlo; j <= jhi; ++j) {
    const double lj = cell_left(j, a, h), rj = cell_right(j, a, h, d);
    const double lo = xlo > lj ? xlo : lj;
    const double hi = xhi < rj ? xhi : rj;
    const double ov = hi - lo;
    if (ov > 0.0) {
      const double vj = __ldg(v + j);
      acc0 += ov;
      const double ovv = ov * vj;
      acc1 += ovv;
      acc2 += ovv * vj;
    }
  }
  const double inv = 1.0 / (2.0 * rad);
  Mom3U r;
  r.s0 = acc0 * inv;
  r.s1 = acc1 * inv;
  r.s2 = acc2 * inv;
  return r;
}

// Interior-cell run of one table (unif_ball_at_tab): the additions stay in
// ascending order, while an L1 prefetch runs kPfCells ahead of the loads (a
// lone warp per scheduler otherwise waits one L2 round trip per unrolled
// batch: long-scoreboard stalls on the first add of each batch).  The
// three-table moments loop is left to the compiler: the same prefetching
// made the ZeroDelay probes slower.
constexpr int kPfCells = 128;
__device__ __forceinline__ void prefetch_l1(const double* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }

__device__ __forceinline__ double sum_run(double acc, const double* __restrict__ t, long long j0, long long j1) {
  long long j = j0;
  for (; j + 15 <= j1; j += 16) {
    prefetch_l1(t + (j + kPfCells <= j1 ? j + kPfCells : j1));
    double v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = __ldg(t + j + k);
#pragma unroll
    for (int k = 0; k < 16; ++k) acc += v[k];
  }
  for (; j <= j1; ++j) acc += __ldg(t + j);
  return acc;
}

// The same moments with the interior cells' terms read from tables: a cell
// at least two cells inside the window [cell(x - rad), cell(x + rad)]
// overlaps it completely (its bounds are the neighbours' shared edges,
// computed from the same exact half-integers), so its overlap is rj - lj
// whatever x is and its three terms ov, ov*v, (ov*v)*v are per-grid constants
// for a given v (k_unif_cell_terms).  Same additions in the same order:
// bitwise equal.
__device__ __forceinline__ Mom3U unif_moments_at_tab(double x, const double* __restrict__ v, double a, double h,
                                                     int64_t d, double rad, const double* __restrict__ c0,
                                                     const double* __restrict__ c1, const double* __restrict__ c2) {
  const double xlo = x - rad, xhi = x + rad;
  const long long jlo = cell_index(xlo, a, h, d), jhi = cell_index(xhi, a, h, d);
  double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
  auto edge = [&](long long j) {
    const double lj = cell_left(j, a, h), rj = cell_right(j, a, h, d);
    const double lo = xlo > lj ? xlo : lj;
    const double hi = xhi < rj ? xhi : rj;
    const double ov = hi - lo;
    if (ov > 0.0) {
      const double vj = __ldg(v + j);
      acc0 += ov;
      const double ovv = ov * vj;
      acc1 += ovv;
      acc2 += ovv * vj;
    }
  };
  if (jlo <= jhi) {
    // two cells at each end exactly (the cell next to an end cell may be
    // clipped by the rounding of (x -/+ rad - a)/h), the rest from the tables
    const long long e0 = jlo + 1 < jhi ? jlo + 1 : jhi;
    for (long long j = jlo; j <= e0; ++j) edge(j);
    for (long long j = jlo + 2; j <= jhi - 2; ++j) {
      acc0 += __ldg(c0 + j);
      acc1 += __ldg(c1 + j);
      acc2 += __ldg(c2 + j);
    }
    for (long long j = (jhi - 1 > jlo + 2 ? jhi - 1 : jlo + 2); j <= jhi; ++j) edge(j);
  }
  const double inv = 1.0 / (2.0 * rad);
  Mom3U r;
  r.s0 = acc0 * inv;
  r.s1 = acc1 * inv;
  r.s2 = acc2 * inv;
  return r;
}

// per-cell interior terms for unif_moments_at_tab (end cells are never interior)
__global__ void k_unif_cell_terms(const double* __restrict__ v, double a, double h, int64_t d, double* c0, double* c1,
                                  double* c2) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= d) return;
  const double ov = cell_right(j, a, h, d) - cell_left(j, a, h);
  const double ovv = ov * v[j];
  c0[j] = ov;
  c1[j] = ovv;
  c2[j] = ovv * v[j];
}

// kernels.py:532-555: E[g] under U(x - rad, x + rad)
__device__ __forceinline__ double unif_ball_at(double x, const double* __restrict__ g, double a, double h, int64_t d,
                                               double rad) {
  const double xlo = x - rad, xhi = x + rad;
  const long long jlo = cell_index(xlo, a, h, d), jhi = cell_index(xhi, a, h, d);
  double acc = 0.0;
  for (long long j = jlo; j <= jhi; ++j) {
    const double lj = cell_left(j, a, h), rj = cell_right(j, a, h, d);
    const double lo = xlo > lj ? xlo : lj;
    const double hi = xhi < rj ? xhi : rj;
    const double ov = hi - lo;
    if (ov > 0.0) acc += ov * __ldg(g + j);
  }
  return acc * (1.0 / (2.0 * rad));
}

// unif_ball_at with the interior cells' terms (rj - lj) * g_j from a table
// (k_unif_ball_terms); two cells at each end computed exactly, as in
// unif_moments_at_tab.  Same additions in the same order: bitwise equal.
__device__ __forceinline__ double unif_ball_at_tab(double x, const double* __restrict__ g, double a, double h,
                                                   int64_t d, double rad, const double* __restrict__ tg) {
  const double xlo = x - rad, xhi = x + rad;
  const long long jlo = cell_index(xlo, a, h, d), jhi = cell_index(xhi, a, h, d);
  double acc = 0.0;
  auto edge = [&](long long j) {
    const double lj = cell_left(j, a, h), rj = cell_right(j, a, h, d);
    const double lo = xlo > lj ? xlo : lj;
    const double hi = xhi < rj ? xhi : rj;
    const double ov = hi - lo;
    if (ov > 0.0) acc += ov * __ldg(g + j);
  };
  if (jlo <= jhi) {
    const long long e0 = jlo + 1 < jhi ? jlo + 1 : jhi;
    for (long long j = jlo; j <= e0; ++j) edge(j);
    acc = sum_run(acc, tg, jlo + 2, jhi - 2);
    for (long long j = (jhi - 1 > jlo + 2 ? jhi - 1 : jlo + 2); j <= jhi; ++j) edge(j);
  }
  return acc * (1.0 / (2.0 * rad));
}

__global__ void k_unif_ball_terms(const double* __restrict__ g, double a, double h, int64_t d, double* tg) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= d) return;
  tg[j] = (cell_right(j, a, h, d) - cell_left(j, a, h)) * g[j];
}

__global__ void k_unif_moments_grid(const double* __restrict__ x, int64_t n, const double* __restrict__ v, double a,
                                    double h, int64_t d, double rad, double* s0, double* s1, double* s2) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  Mom3U r = unif_moments_at(x[t], v, a, h, d, rad);
  s0[t] = r.s0;
  s1[t] = r.s1;
  s2[t] = r.s2;
}

__global__ void k_unif_ball_sum(const double* __restrict__ x, const double* __restrict__ xadd, int64_t n,
                                const double* __restrict__ g, double a, double h, int64_t d, double rad,
                                double* out) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const double xt = xadd ? x[t] + xadd[t] : x[t];
  out[t] = unif_ball_at(xt, g, a, h, d, rad);
}

// kernels.py:558-577, one thread per output node j, centres in ascending i.
// masses = mscale * f (the reference forms g.spacing * f as an array first:
// the same single rounding per element), centres = cpts + cu (points + u).
// Sources whose ball [c - rad, c + rad] misses a warp's whole cell span
// [Lw, Rw] add nothing to any of its cells (hi <= Lw <= lj gives ov <= 0, and
// so does lo >= Rw >= rj; NaN centres stay in), so each warp compacts the
// sources that can touch it, in ascending order, into its own shared buffer
// and runs the reference's serial loop over those only: the same additions in
// the same order, bitwise equal, with the loop shortened to the sources in
// reach.  kUnifWarps warps per CTA (few cells: spread them over the SMs).
constexpr int kUnifWarps = 2;
constexpr int kUnifBuf = 512;

__device__ __forceinline__ void warp_span(bool active, double lj, double rj, double& lw, double& rw) {
  lw = active ? lj : INFINITY;
  rw = active ? rj : -INFINITY;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double l2 = __shfl_xor_sync(0xffffffffu, lw, o), r2 = __shfl_xor_sync(0xffffffffu, rw, o);
    lw = l2 < lw ? l2 : lw;
    rw = r2 > rw ? r2 : rw;
  }
}

__global__ void __launch_bounds__(32 * kUnifWarps) k_unif_propagate(const double* __restrict__ f, double mscale,
                                                                   const double* __restrict__ cpts,
                                                                   const double* __restrict__ cu, int64_t n,
                                                                   double a, double h, int64_t d, double rad,
                                                                   double* out) {
  __shared__ double sm_all[kUnifWarps][kUnifBuf], sl_all[kUnifWarps][kUnifBuf], sh_all[kUnifWarps][kUnifBuf];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* sm = sm_all[warp];
  double* sl = sl_all[warp];  // c - rad
  double* sh = sh_all[warp];  // c + rad
  const int64_t j0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31);
  if (j0 >= d) return;  // warp-uniform: no cell of this warp exists
  const int64_t j = j0 + lane;
  const bool active = j < d;
  const double lj = active ? cell_left(j, a, h) : 0.0, rj = active ? cell_right(j, a, h, d) : 0.0;
  double lw, rw;
  warp_span(active, lj, rj, lw, rw);
  const unsigned below = (1u << lane) - 1u;
  // kUnifBuf sources per pass: each lane holds kUnifBuf / 32 of them in
  // registers (independent loads in flight together; the next pass's loads
  // issue before this pass's serial loop)
  constexpr int K = kUnifBuf / 32;
  double rf[K], rc[K];
  auto load = [&](int64_t base) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int64_t r = base + k * 32 + lane;
      rf[k] = 0.0;
      rc[k] = 0.0;
      if (r < n) {
        rf[k] = mscale == 1.0 ? f[r] : mscale * f[r];
        rc[k] = cu ? cpts[r] + cu[r] : cpts[r];
      }
    }
  };
  double acc = 0.0;
  if (n > 0) load(0);
  for (int64_t base = 0; base < n; base += kUnifBuf) {
    int fill = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const bool rel = base + k * 32 + lane < n && !((rc[k] + rad) <= lw || (rc[k] - rad) >= rw);
      const unsigned mask = __ballot_sync(0xffffffffu, rel);
      if (rel) {
        const int pos = fill + __popc(mask & below);
        sm[pos] = rf[k];
        sl[pos] = rc[k] - rad;
        sh[pos] = rc[k] + rad;
      }
      fill += __popc(mask);
    }
    if (base + kUnifBuf < n) load(base + kUnifBuf);
    __syncwarp();
    if (active) {
#pragma unroll 4
      for (int q = 0; q < fill; ++q) {
        double lo = sl[q], hi = sh[q];
        if (lo < lj) lo = lj;
        if (hi > rj) hi = rj;
        const double ov = hi - lo;
        if (ov > 0.0) acc += sm[q] * ov;
      }
    }
    __syncwarp();
  }
  if (active) out[j] = acc * (1.0 / ((2.0 * rad) * h));
}

// kernels.py:580-615, one thread per query, support points in ascending i
// (sources out of the warp's reach skipped as in k_unif_propagate: bitwise)
__global__ void __launch_bounds__(32 * kUnifWarps) k_unif_moments_points(
    const double* __restrict__ y, int64_t n, const double* __restrict__ centers, const double* __restrict__ w,
    const double* __restrict__ vals, int64_t m, double a, double h, int64_t d, double rad, double* m0, double* m1,
    double* m2) {
  __shared__ double sl_all[kUnifWarps][kUnifBuf], sh_all[kUnifWarps][kUnifBuf], sw_all[kUnifWarps][kUnifBuf],
      sv_all[kUnifWarps][kUnifBuf];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* sl = sl_all[warp];  // centre - rad
  double* sh = sh_all[warp];  // centre + rad
  double* sw = sw_all[warp];
  double* sv = sv_all[warp];
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31);
  if (t0 >= n) return;  // warp-uniform
  const int64_t t = t0 + lane;
  const bool active = t < n;
  const long long j = cell_index(active ? y[t] : 0.0, a, h, d);
  const double lj = cell_left(j, a, h), rj = cell_right(j, a, h, d);
  double lw, rw;
  warp_span(active, lj, rj, lw, rw);
  const unsigned below = (1u << lane) - 1u;
  constexpr int K = kUnifBuf / 32;  // register-batched loads as in k_unif_propagate
  double rc[K], rw_[K], rv[K];
  auto load = [&](int64_t base) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int64_t r = base + k * 32 + lane;
      rc[k] = 0.0;
      rw_[k] = 0.0;
      rv[k] = 0.0;
      if (r < m) {
        rc[k] = centers[r];
        rw_[k] = w[r];
        rv[k] = vals[r];
      }
    }
  };
  double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
  if (m > 0) load(0);
  for (int64_t base = 0; base < m; base += kUnifBuf) {
    int fill = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const bool rel = base + k * 32 + lane < m && !((rc[k] + rad) <= lw || (rc[k] - rad) >= rw);
      const unsigned mask = __ballot_sync(0xffffffffu, rel);
      if (rel) {
        const int pos = fill + __popc(mask & below);
        sl[pos] = rc[k] - rad;
        sh[pos] = rc[k] + rad;
        sw[pos] = rw_[k];
        sv[pos] = rv[k];
      }
      fill += __popc(mask);
    }
    if (base + kUnifBuf < m) load(base + kUnifBuf);
    __syncwarp();
    if (active) {
#pragma unroll 4
      for (int q = 0; q < fill; ++q) {
        double lo = sl[q], hi = sh[q];
        if (lo < lj) lo = lj;
        if (hi > rj) hi = rj;
        const double ov = hi - lo;
        if (ov > 0.0) {
          const double wov = sw[q] * ov, vi = sv[q];
          acc0 += wov;
          const double wv = wov * vi;
          acc1 += wv;
          acc2 += wv * vi;
        }
      }
    }
    __syncwarp();
  }
  if (active) {
    const double inv = 1.0 / ((2.0 * rad) * h);
    m0[t] = acc0 * inv;
    m1[t] = acc1 * inv;
    m2[t] = acc2 * inv;
  }
}

// Producer/consumer form of k_unif_propagate (kPlanes = 1) and
// k_unif_moments_points (kPlanes = 3): the reference's per-output loops are
// serial add chains (kernels.py:562-576, 593-613), and one thread per output
// leaves them latency-bound (one warp per scheduler at d = 4096 / 16384,
// every source costing the whole clamp/overlap/product dependency chain).
// Here a CTA owns 32 outputs ("queries": cells j for propagate, points y_t
// for moments).  8 producer warps scan the sources in ascending order,
// compact the ones that can touch the CTA's cell span (ballot + per-warp
// counts: order kept) into a shared-memory ring, and evaluate 32-source
// stages of per-(source, query) terms -- mass*ov, or wov, wov*v, (wov*v)*v
// for ov > 0, +0.0 otherwise -- while one consumer warp per accumulator adds
// the previous stage's terms serially, lane = query.  Every query's
// accumulator receives exactly the reference's addends in the reference's
// order plus +0.0 for sources that do not overlap its own cell; an
// accumulator that starts at +0.0 is never -0.0 (round-to-nearest gives +0.0
// for exact cancellation), so those additions leave its bits unchanged:
// bitwise equal.  Sources out of the CTA's span have ov <= 0 for all its
// cells (as in k_unif_propagate's warp compaction; NaN centres stay in).
// Two stages, named barriers (FULL: producers arrive, consumers wait; EMPTY:
// the reverse; PROD among producers), a stage with nrows = -1 ends the run.
constexpr int kPcQ = 32;            // queries (outputs) per CTA
constexpr int kPcRows = 32;         // sources per stage
constexpr int kPcProdWarps = 8;
constexpr int kPcProd = 32 * kPcProdWarps;
constexpr int kPcRing = 512;        // pending relevant sources (>= kPcRows - 1 + kPcProd)
template <int kPlanes>
__host__ __device__ constexpr int pc_threads() { return 32 * (kPlanes + kPcProdWarps); }
template <int kPlanes>
constexpr size_t pc_smem() {
  return sizeof(double) * ((size_t)2 * kPlanes * kPcRows * kPcQ + (size_t)(kPlanes == 3 ? 4 : 3) * kPcRing);
}

template <int kPlanes>
__global__ void __launch_bounds__(pc_threads<kPlanes>()) k_unif_pc(
    const double* __restrict__ yq, int64_t n, const double* __restrict__ cpts, const double* __restrict__ cu,
    const double* __restrict__ w, double wscale, const double* __restrict__ vals, int64_t m, double a, double h,
    int64_t d, double rad, double* o0, double* o1, double* o2) {
  static_assert(kPlanes == 1 || kPlanes == 3, "planes");
  constexpr int kThreads = pc_threads<kPlanes>();
  constexpr int kFull = 1, kEmpty = 3, kProdBar = 5;
  extern __shared__ __align__(16) double pc_smem_[];
  double* st = pc_smem_;                                   // [2][kPlanes][kPcRows][kPcQ]
  double* rl = st + 2 * kPlanes * kPcRows * kPcQ;          // ring: centre - rad
  double* rh = rl + kPcRing;                               //       centre + rad
  double* rw = rh + kPcRing;                               //       weight / mass
  double* rv = rw + kPcRing;                               //       value (kPlanes == 3)
  __shared__ int s_wc[kPcProdWarps];
  __shared__ int s_nrows[2];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t t0 = (int64_t)blockIdx.x * kPcQ;
  if (warp >= kPlanes) {
    // ------------------------------------------------------------ producers
    const int pt = tid - 32 * kPlanes, pw = pt >> 5;
    const int64_t tq = t0 + lane < n ? t0 + lane : n - 1;  // this thread's query (clamped)
    const long long j = yq ? cell_index(yq[tq], a, h, d) : (long long)tq;
    const double lj = cell_left(j, a, h), rj = cell_right(j, a, h, d);
    double lc = lj, rc = rj;  // the CTA's span (every producer warp covers all 32 queries)
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double l2 = __shfl_xor_sync(0xffffffffu, lc, o), r2 = __shfl_xor_sync(0xffffffffu, rc, o);
      lc = l2 < lc ? l2 : lc;
      rc = r2 > rc ? r2 : rc;
    }
    const unsigned below = (1u << lane) - 1u;
    int head = 0, pend = 0, k = 0;
    auto stage = [&](int nrows) {
      const int buf = k & 1;
      if (k >= 2) named_sync(kEmpty + buf, kThreads);  // consumers are done with stage k - 2
      double* s = st + (size_t)buf * kPlanes * kPcRows * kPcQ;
      for (int r = pw; r < nrows; r += kPcProdWarps) {  // row r, query lane
        const int pos = (head + r) & (kPcRing - 1);
        double lo = rl[pos], hi = rh[pos];
        if (lo < lj) lo = lj;
        if (hi > rj) hi = rj;
        const double ov = hi - lo;
        double e0 = 0.0, e1 = 0.0, e2 = 0.0;
        if (ov > 0.0) {
          e0 = rw[pos] * ov;
          if (kPlanes == 3) {
            const double v = rv[pos];
            e1 = e0 * v;
            e2 = e1 * v;
          }
        }
        s[r * kPcQ + lane] = e0;
        if (kPlanes == 3) {
          s[(kPcRows + r) * kPcQ + lane] = e1;
          s[(2 * kPcRows + r) * kPcQ + lane] = e2;
        }
      }
      if (pt == 0) s_nrows[buf] = nrows;
      named_arrive(kFull + buf, kThreads);
      ++k;
    };
    for (int64_t base = 0; base < m; base += kPcProd) {
      const int64_t r = base + pt;
      bool rel = false;
      double cl = 0.0, ch = 0.0;
      if (r < m) {
        const double c = cu ? cpts[r] + cu[r] : cpts[r];
        cl = c - rad;
        ch = c + rad;
        rel = !(ch <= lc || cl >= rc);
      }
      const unsigned mask = __ballot_sync(0xffffffffu, rel);
      if (lane == 0) s_wc[pw] = __popc(mask);
      named_sync(kProdBar, kPcProd);
      int before = 0, total = 0;
#pragma unroll
      for (int q = 0; q < kPcProdWarps; ++q) {
        const int c = s_wc[q];
        before += q < pw ? c : 0;
        total += c;
      }
      if (rel) {
        const int pos = (head + pend + before + __popc(mask & below)) & (kPcRing - 1);
        rl[pos] = cl;
        rh[pos] = ch;
        rw[pos] = wscale == 1.0 ? w[r] : wscale * w[r];
        if (kPlanes == 3) rv[pos] = vals[r];
      }
      named_sync(kProdBar, kPcProd);  // ring entries visible; s_wc free again
      pend += total;
      UCP_DCHECK(pend < kPcRing);
      while (pend >= kPcRows) {
        stage(kPcRows);
        head = (head + kPcRows) & (kPcRing - 1);
        pend -= kPcRows;
      }
    }
    if (pend > 0) stage(pend);
    stage(-1);  // end marker
    if (k >= 2) named_sync(kEmpty + ((k - 2) & 1), kThreads);  // the consumers' last EMPTY arrival
  } else {
    // ------------------------------------------------------------ consumers
    const int plane = warp;
    double acc = 0.0;
    for (int k = 0;; ++k) {
      const int buf = k & 1;
      named_sync(kFull + buf, kThreads);
      const int nrows = s_nrows[buf];
      if (nrows < 0) break;
      const double* s = st + ((size_t)buf * kPlanes + plane) * kPcRows * kPcQ + lane;
#pragma unroll 8
      for (int r = 0; r < nrows; ++r) acc += s[r * kPcQ];
      named_arrive(kEmpty + buf, kThreads);
    }
    const int64_t t = t0 + lane;
    if (t < n) {
      const double inv = 1.0 / ((2.0 * rad) * h);
      (plane == 0 ? o0 : plane == 1 ? o1 : o2)[t] = acc * inv;
    }
  }
}

// launch helpers (dynamic shared memory opt-in once per kernel and device);
// -DUCP_UNIF_PC=0 builds the one-thread-per-output kernels instead (A/B)
#ifndef UCP_UNIF_PC
#define UCP_UNIF_PC 1
#endif
int launch_unif_propagate(const double* f, double mscale, const double* cpts, const double* cu, int64_t n, double a,
                          double h, int64_t d, double rad, double* out, cudaStream_t st) {
  if (!UCP_UNIF_PC) {
    k_unif_propagate<<<nblocks(d, 32 * kUnifWarps), 32 * kUnifWarps, 0, st>>>(f, mscale, cpts, cu, n, a, h, d, rad, out);
    UCP_LAUNCHED("k_unif_propagate");
    return UCP_OK;
  }
  smem_opt_in(reinterpret_cast<const void*>(k_unif_pc<1>), pc_smem<1>());
  k_unif_pc<1><<<nblocks(d, kPcQ), pc_threads<1>(), pc_smem<1>(), st>>>(nullptr, d, cpts, cu, f, mscale, nullptr, n,
                                                                        a, h, d, rad, out, nullptr, nullptr);
  UCP_LAUNCHED("k_unif_pc<1>");
  return UCP_OK;
}
int launch_unif_moments_points(const double* y, int64_t n, const double* centers, const double* w,
                               const double* vals, int64_t m, double a, double h, int64_t d, double rad, double* m0,
                               double* m1, double* m2, cudaStream_t st) {
  if (!UCP_UNIF_PC) {
    k_unif_moments_points<<<nblocks(n, 32 * kUnifWarps), 32 * kUnifWarps, 0, st>>>(y, n, centers, w, vals, m, a, h, d,
                                                                                   rad, m0, m1, m2);
    UCP_LAUNCHED("k_unif_moments_points");
    return UCP_OK;
  }
  smem_opt_in(reinterpret_cast<const void*>(k_unif_pc<3>), pc_smem<3>());
  k_unif_pc<3><<<nblocks(n, kPcQ), pc_threads<3>(), pc_smem<3>(), st>>>(y, n, centers, nullptr, w, 1.0, vals, m, a, h,
                                                                        d, rad, m0, m1, m2);
  UCP_LAUNCHED("k_unif_pc<3>");
  return UCP_OK;
}

// ------------------------------------------------------- cost functors
// zero_delay.py:69-76: C0(u, y_i) = f0_i (pw u^2 + E[(y - u1(x1))^2]), x1 = u + w
struct ZdCost0 {
  const double* y0;
  const double* f0;
  const double* v1;
  double a1, h1, pw;
  int64_t d1;
  const double* tab = nullptr;  // [3][d1] interior-cell terms of v1 (nullptr: direct loop)
  __device__ __forceinline__ double operator()(double u, int64_t i) const {
    const Mom3U s = tab ? unif_moments_at_tab(u, v1, a1, h1, d1, 1.0, tab, tab + d1, tab + 2 * d1)
                        : unif_moments_at(u, v1, a1, h1, d1, 1.0);
    const double y = y0[i];
    const double distortion = (((s.s0 * y) * y) - ((2.0 * s.s1) * y)) + s.s2;
    return f0[i] * (((pw * u) * u) + distortion);
  }
};

// ZeroDelay stage 0 in partial exhaustion: every candidate is a controller
// value u0[j], and ZdCost0's moments depend on u alone, so they are computed
// once per j (k_zd_mom_table, the same unif_moments_at_tab call) and every
// (point, candidate) pair reads them: the same expression on the same
// operands, bitwise equal to ZdCost0, at O(1) per candidate.
struct ZdCost0Memo {
  const double* y0;
  const double* f0;
  const double* S;  // [3][d0]: s0, s1, s2 of u0[j]
  int64_t d0;
  double pw;
  __device__ __forceinline__ double at(double u, int64_t j, int64_t i) const {
    const double s0 = S[j], s1 = S[d0 + j], s2 = S[2 * d0 + j];
    const double y = y0[i];
    const double distortion = (((s0 * y) * y) - ((2.0 * s1) * y)) + s2;
    return f0[i] * (((pw * u) * u) + distortion);
  }
};

__global__ void k_zd_mom_table(ZdCost0 c, const double* __restrict__ u0, int64_t d0, double* S) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= d0) return;
  const Mom3U s = unif_moments_at_tab(u0[j], c.v1, c.a1, c.h1, c.d1, 1.0, c.tab, c.tab + c.d1, c.tab + 2 * c.d1);
  S[j] = s.s0;
  S[d0 + j] = s.s1;
  S[2 * d0 + j] = s.s2;
}

// candidate j of point i (the memoised functor reads its per-j table)
template <class Cost>
__device__ __forceinline__ double exh_cost(const Cost& c, const double* __restrict__ u, int64_t j, int64_t i) {
  return c(u[j], i);
}
__device__ __forceinline__ double exh_cost(const ZdCost0Memo& c, const double* __restrict__ u, int64_t j, int64_t i) {
  return c.at(u[j], j, i);
}

// any stage whose cost is quadratic in u with per-point moments (ZeroDelay m=1)
struct QuadCost {
  const double* A;
  const double* B;
  const double* C;
  int64_t begin;
  __device__ __forceinline__ double operator()(double u, int64_t i) const {
    const int64_t k = i - begin;
    return quad_in_u(A[k], B[k], C[k], u);
  }
};

// inventory.py:138-150: f_m(nearest(y)) * (c u + E[g_{m+1}(y + u - w)])
struct InvCost {
  const double* ym;
  const double* fm;
  const double* gnext;
  double am, hm, an, hn, oc;
  int64_t dm, dn;
  const double* tg = nullptr;  // interior-cell terms of gnext (nullptr: direct loop)
  __device__ __forceinline__ double operator()(double u, int64_t i) const {
    const double y = ym[i];
    const double expect = tg ? unif_ball_at_tab(y + u, gnext, an, hn, dn, 1.0, tg)
                             : unif_ball_at(y + u, gnext, an, hn, dn, 1.0);
    const double weight = fm[cell_index(y, am, hm, dm)];
    return weight * ((oc * u) + expect);
  }
};

__device__ __forceinline__ double project_value(int kind, double v) { return kind == 1 ? np_maximum(v, 0.0) : v; }

// solver.py:179-203 for any cost functor, in two launches so small grids
// still fill the GPU: (1) the three FD probes u+h, u, u-h of every point in
// parallel (probe-major), (2) per point: derivatives, safeguarded step,
// projection, cost_new and the monotone guard.  The h floor is the
// problem's widened probe (zero_delay.py:56-65, inventory.py:131-136).
template <class Cost>
__global__ void k_gen_probe(Cost cost, const double* __restrict__ u, double fd_step, double h_floor, int64_t begin,
                            int64_t n, double* cost3) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 3 * n) return;
  const int p = (int)(t / n);
  const int64_t i = begin + (t - (int64_t)p * n);
  const double ui = u[i];
  double hh = fd_step * (1.0 + fabs(ui));
  if (h_floor > 0.0) hh = np_maximum(hh, h_floor);
  const double uu = p == 0 ? ui + hh : (p == 1 ? ui : ui - hh);
  cost3[t] = cost(uu, i);
}

template <class Cost>
__global__ void k_gen_finish(Cost cost, const double* __restrict__ u, ucp_local_params lp, double h_floor,
                             int project_kind, int64_t begin, int64_t n, const double* __restrict__ cost3,
                             double* out, int64_t* err) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int64_t i = begin + t;
  const double ui = u[i];
  double hh = lp.fd_step * (1.0 + fabs(ui));
  if (h_floor > 0.0) hh = np_maximum(hh, h_floor);
  const double up = cost3[t], mid = cost3[n + t], dn = cost3[2 * n + t];
  const double c1 = (up - dn) / (2.0 * hh);
  const double c2 = ((up - 2.0 * mid) + dn) / (hh * hh);
  if (!(finite(c1) && finite(c2))) {
    flag_min(err, i);
    out[i] = ui;
    return;
  }
  const double stepped = project_value(project_kind, newton_step(ui, c1, c2, lp));
  const double cost_new = cost(stepped, i);
  if (!(finite(mid) && finite(cost_new))) flag_min(err + 1, i);
  const double r = cost_new <= mid ? stepped : ui;
  if (!finite(r)) flag_min(err + 2, i);
  out[i] = r;
}

// solver.py:206-223 in two launches: (1) every (point, window slot) candidate
// cost in parallel, slot-major per point (wmax = widest window); (2) per
// point, the first strict minimum in window order (kernels.py:147-160), any
// non-finite candidate flagging the point, then the projection.
template <class Cost>
__global__ void k_gen_exh_eval(Cost cost, const double* __restrict__ u, const int64_t* __restrict__ lo,
                               const int64_t* __restrict__ hi, int64_t begin, int64_t n, int64_t wmax,
                               double* costs) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * wmax) return;
  const int64_t k = t / n, p = t - k * n;
  const int64_t i = begin + p;
  const int64_t j = lo[i] + k;
  // a value equal to its window predecessor has the same cost and never wins
  // the first-minimum: not evaluated (the reference's flatten_windows dedups
  // the same adjacent repeats, kernels.py:163-187)
  if (j <= hi[i] && !(k > 0 && u[j] == u[j - 1])) costs[p * wmax + k] = exh_cost(cost, u, j, i);
}

__global__ void k_gen_exh_pick(const double* __restrict__ u, const int64_t* __restrict__ lo,
                               const int64_t* __restrict__ hi, int project_kind, int64_t begin, int64_t n,
                               int64_t wmax, const double* __restrict__ costs, double* out, int64_t* err) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int64_t i = begin + t;
  const double* c = costs + t * wmax;
  const int64_t j0 = lo[i];
  const int64_t w = hi[i] - j0 + 1;
  int64_t best = 0;
  double bv = c[0];
  bool ok = finite(bv);
  for (int64_t k = 1; k < w; ++k) {
    if (u[j0 + k] == u[j0 + k - 1]) continue;  // adjacent repeat: same cost, not evaluated
    const double x = c[k];
    ok = ok && finite(x);
    if (x < bv) {
      bv = x;
      best = k;
    }
  }
  if (!ok) flag_min(err, i);
  out[i] = project_value(project_kind, u[lo[i] + best]);
}

template <class Cost>
__global__ void k_gen_terms(Cost cost, const double* __restrict__ u0, int64_t begin, int64_t end, double* terms,
                            int64_t* err) {
  const int64_t i = begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= end) return;
  const double c = cost(u0[i], i);
  if (!finite(c)) flag_min(err, i);
  terms[i] = c;
}

// marginal_cost_segmented over a flat candidate list; the cost functor is
// built on per-SEGMENT arrays (observation y, density) and indexed by segment
template <class Cost>
__global__ void k_gen_segmented(Cost cost, const double* __restrict__ u_flat, const int64_t* __restrict__ offsets,
                                int64_t nseg, double* out) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = offsets[nseg];
  if (c >= n) return;
  int64_t lo = 0, hi = nseg;
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (offsets[mid] <= c) lo = mid; else hi = mid;
  }
  out[c] = cost(u_flat[c], lo);
}

// Inventory: gs[mm] = gamma(pts) + (c u + E[gs[mm+1](pts + u - w)]) (inventory.py:84-94);
// gs[M] = gamma(terminal points) when gnext == nullptr.
__global__ void k_inv_downstream(const double* __restrict__ pts, const double* __restrict__ u, int64_t n,
                                 const double* __restrict__ gnext, double an, double hn, int64_t dn, double oc,
                                 int quadratic, double hr, double br, double* out,
                                 const double* __restrict__ tg = nullptr) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double x = pts[i];
  const double gam = quadratic ? x * x : hr * np_maximum(x, 0.0) + br * np_maximum(-x, 0.0);
  if (!gnext) {
    out[i] = gam;
    return;
  }
  const double ui = u[i];
  const double expect =
      tg ? unif_ball_at_tab(x + ui, gnext, an, hn, dn, 1.0, tg) : unif_ball_at(x + ui, gnext, an, hn, dn, 1.0);
  out[i] = gam + ((oc * ui) + expect);
}

template <class Cost>
int launch_gen_local(const Cost& c, const double* u, const ucp_local_params* lp, double h_floor, int project_kind,
                     int64_t begin, int64_t n, double* out, int64_t* err, ucp_workspace* ws, cudaStream_t st) {
  void* pc;
  int rc;
  if ((rc = ws_get(ws, WS_COST, sizeof(double) * 3 * (size_t)n, &pc))) return rc;
  k_gen_probe<Cost><<<nblocks(3 * n, 128), 128, 0, st>>>(c, u, lp->fd_step, h_floor, begin, n, (double*)pc);
  UCP_LAUNCHED("k_gen_probe");
  k_gen_finish<Cost><<<nblocks(n, 128), 128, 0, st>>>(c, u, *lp, h_floor, project_kind, begin, n,
                                                      (const double*)pc, out, err);
  UCP_LAUNCHED("k_gen_finish");
  return UCP_OK;
}

template <class Cost>
int launch_gen_exhaust(const Cost& c, const double* u, const int64_t* lo, const int64_t* hi, int64_t wmax,
                       int project_kind, int64_t begin, int64_t n, double* out, int64_t* err, ucp_workspace* ws,
                       cudaStream_t st) {
  if (wmax < 1) return arg_fail("exhaustion: window width must be >= 1");
  void* pc;
  int rc;
  if ((rc = ws_get(ws, WS_COST, sizeof(double) * (size_t)(n * wmax), &pc))) return rc;
  k_gen_exh_eval<Cost><<<nblocks(n * wmax, 128), 128, 0, st>>>(c, u, lo, hi, begin, n, wmax, (double*)pc);
  UCP_LAUNCHED("k_gen_exh_eval");
  k_gen_exh_pick<<<nblocks(n, 128), 128, 0, st>>>(u, lo, hi, project_kind, begin, n, wmax, (const double*)pc, out,
                                                  err);
  UCP_LAUNCHED("k_gen_exh_pick");
  return UCP_OK;
}

int check_zd(const ucp_zd_problem* P) {
  if (!P || !P->y0 || !P->y1 || !P->f0 || !P->fw0) return arg_fail("null zero-delay problem pointer");
  if (P->d0 < 2 || P->d1 < 2) return arg_fail("grid.d must be at least 2");
  return UCP_OK;
}

ZdCost0 zd_cost0(const ucp_zd_problem* P, const double* u1) {
  ZdCost0 c;
  c.y0 = P->y0;
  c.f0 = P->f0;
  c.v1 = u1;
  c.a1 = P->a1;
  c.h1 = P->h1;
  c.d1 = P->d1;
  c.pw = P->power_weight;
  return c;
}

// the functor with its interior-cell tables, built once per call in the workspace
int zd_cost0_tab(const ucp_zd_problem* P, const double* u1, ucp_workspace* ws, cudaStream_t st, ZdCost0* out) {
  ZdCost0 c = zd_cost0(P, u1);
  void* pt;
  int rc;
  if ((rc = ws_get(ws, WS_C5_TAB, sizeof(double) * 3 * (size_t)P->d1, &pt))) return rc;
  double* t = (double*)pt;
  k_unif_cell_terms<<<nblocks(P->d1, 256), 256, 0, st>>>(u1, P->a1, P->h1, P->d1, t, t + P->d1, t + 2 * P->d1);
  UCP_LAUNCHED("k_unif_cell_terms");
  c.tab = t;
  *out = c;
  return UCP_OK;
}

// zero_delay.py:77-83: decoder moments at queries y (centres u0, weights fw0, values y0)
int zd_moments(const ucp_zd_problem* P, const double* u0, const double* yq, int64_t nq, ucp_workspace* ws,
               cudaStream_t st, QuadCost* q) {
  void* pm;
  int rc;
  if ((rc = ws_get(ws, WS_MOM, sizeof(double) * 3 * (size_t)nq, &pm))) return rc;
  double* m0 = (double*)pm;
  if ((rc = launch_unif_moments_points(yq, nq, u0, P->fw0, P->y0, P->d0, P->a1, P->h1, P->d1, 1.0, m0, m0 + nq,
                                       m0 + 2 * nq, st)))
    return rc;
  q->A = m0;
  q->B = m0 + nq;
  q->C = m0 + 2 * nq;
  return UCP_OK;
}

// ----------------------------------------------------------- inventory
int check_inv(const ucp_inv_problem* P, const double* const* u) {
  if (!P || P->stages < 1 || P->stages > UCP_INV_MAX_STAGES) return arg_fail("inventory: bad stage count");
  for (int m = 0; m < P->stages; ++m) {
    if (!P->pts[m] || P->d[m] < 2) return arg_fail("inventory: bad grid");
    if (u && !u[m]) return arg_fail("inventory: null controller");
  }
  return UCP_OK;
}

inline int inv_state(const ucp_inv_problem* P, int mm) { return mm < P->stages - 1 ? mm : P->stages - 1; }

// Reuse across calls when the caller keys its controllers (ucp_inv_problem.ukey):
// *use = false without keys, during graph capture (host decisions would be
// baked into the graph), or on a key of 0.  The slots are reset whenever the
// problem or the cache buffers change.
int inv_cache_prepare(const ucp_inv_problem* P, ucp_workspace* ws, cudaStream_t st, int64_t dmax, double** fb,
                      double** gb, bool* use) {
  *use = false;
  if (!P->ukey) return UCP_OK;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return UCP_OK;
  }
  const int M = P->stages;
  for (int k = 0; k < M; ++k)
    if (P->ukey[k] == 0) return UCP_OK;
  void *pf, *pg;
  int rc;
  if ((rc = ws_get(ws, WS_C5_FC, sizeof(double) * (size_t)(M + 1) * (size_t)dmax, &pf))) return rc;
  if ((rc = ws_get(ws, WS_C5_GC, sizeof(double) * (size_t)(M + 1) * (size_t)dmax, &pg))) return rc;
  ucp_inv_cache& c = ws->inv;
  ucp_inv_problem key = *P;
  key.ukey = nullptr;
  if (!c.valid || c.fbuf != pf || c.gbuf != pg || memcmp(&c.prob, &key, sizeof key) != 0) {
    c = ucp_inv_cache{};
    c.prob = key;
    c.fbuf = pf;
    c.gbuf = pg;
    c.valid = true;
  }
  *fb = (double*)pf;
  *gb = (double*)pg;
  *use = true;
  return UCP_OK;
}

int64_t inv_dmax(const ucp_inv_problem* P) {
  int64_t dmax = 0;
  for (int k = 0; k < P->stages; ++k) dmax = P->d[k] > dmax ? P->d[k] : dmax;
  return dmax;
}

// f_0 = unif_propagate([1.0], [0.0], grid 0)
int inv_density0(const ucp_inv_problem* P, ucp_workspace* ws, cudaStream_t st, double* out) {
  void* pone;
  int rc;
  if ((rc = ws_get(ws, WS_C5_ONE, sizeof(double) * 2, &pone))) return rc;
  static const double one_zero[2] = {1.0, 0.0};
  UCP_CHECK(cudaMemcpyAsync(pone, one_zero, sizeof one_zero, cudaMemcpyHostToDevice, st));
  const double* one = (const double*)pone;
  return launch_unif_propagate(one, 1.0, one + 1, nullptr, 1, P->a[0], P->h[0], P->d[0], 1.0, out, st);
}

// f_{mm+1} = unif_propagate(h_mm * f_mm, pts_mm + u_mm, grid mm+1)
int inv_density_step(const ucp_inv_problem* P, int mm, const double* const* u, const double* f, double* out,
                      cudaStream_t st) {
  return launch_unif_propagate(f, P->h[mm], P->pts[mm], u[mm], P->d[mm], P->a[mm + 1], P->h[mm + 1], P->d[mm + 1], 1.0,
                               out, st);
}

// g_M = gamma(terminal state points), on grid inv_state(M)
int inv_terminal(const ucp_inv_problem* P, double* out, cudaStream_t st) {
  const int term = inv_state(P, P->stages);
  k_inv_downstream<<<nblocks(P->d[term], 128), 128, 0, st>>>(P->pts[term], nullptr, P->d[term], nullptr, 0.0, 0.0, 0,
                                                             0.0, P->quadratic, P->holding_rate, P->backlog_rate, out);
  UCP_LAUNCHED("k_inv_downstream");
  return UCP_OK;
}

// g_mm from g_{mm+1} (tg: scratch for g_{mm+1}'s interior-cell terms)
int inv_downstream_step(const ucp_inv_problem* P, int mm, const double* const* u, const double* gnext, double* tg,
                         double* out, cudaStream_t st) {
  const int nx = inv_state(P, mm + 1);
  k_unif_ball_terms<<<nblocks(P->d[nx], 256), 256, 0, st>>>(gnext, P->a[nx], P->h[nx], P->d[nx], tg);
  UCP_LAUNCHED("k_unif_ball_terms");
  k_inv_downstream<<<nblocks(P->d[mm], 128), 128, 0, st>>>(P->pts[mm], u[mm], P->d[mm], gnext, P->a[nx], P->h[nx],
                                                           P->d[nx], P->order_cost, P->quadratic, P->holding_rate,
                                                           P->backlog_rate, out, tg);
  UCP_LAUNCHED("k_inv_downstream");
  return UCP_OK;
}

// Stock density at stage m (inventory.py:96-110) into *out (device, d[m]).
int inv_forward_density(const ucp_inv_problem* P, int m, const double* const* u, ucp_workspace* ws,
                        cudaStream_t st, const double** out) {
  int rc;
  const int64_t dmax = inv_dmax(P);
  double *F, *G;
  bool use;
  if ((rc = inv_cache_prepare(P, ws, st, dmax, &F, &G, &use))) return rc;
  if (use) {
    ucp_inv_cache& c = ws->inv;
    int start = -1;
    for (int k = m; k >= 0 && start < 0; --k)
      if (c.fok[k] && std::equal(P->ukey, P->ukey + k, c.fkey[k])) start = k;
    if (start < 0) {
      if ((rc = inv_density0(P, ws, st, F))) return rc;
      c.fok[0] = true;
      start = 0;
    }
    for (int mm = start; mm < m; ++mm) {
      if ((rc = inv_density_step(P, mm, u, F + (size_t)mm * dmax, F + (size_t)(mm + 1) * dmax, st))) return rc;
      c.fok[mm + 1] = true;
      std::copy(P->ukey, P->ukey + mm + 1, c.fkey[mm + 1]);
    }
    *out = F + (size_t)m * dmax;
    return UCP_OK;
  }
  void *pa, *pb;
  if ((rc = ws_get(ws, WS_C5_F0, sizeof(double) * (size_t)dmax, &pa))) return rc;
  if ((rc = ws_get(ws, WS_C5_F1, sizeof(double) * (size_t)dmax, &pb))) return rc;
  double* bufs[2] = {(double*)pa, (double*)pb};
  if ((rc = inv_density0(P, ws, st, bufs[0]))) return rc;
  int cur = 0;
  for (int mm = 0; mm < m; ++mm) {
    if ((rc = inv_density_step(P, mm, u, bufs[cur], bufs[cur ^ 1], st))) return rc;
    cur ^= 1;
  }
  *out = bufs[cur];
  return UCP_OK;
}

// g_{m+1} on the stage-(m+1) state grid (inventory.py:78-94), backwards from M.
int inv_downstream(const ucp_inv_problem* P, int m, const double* const* u, ucp_workspace* ws, cudaStream_t st,
                   const double** out) {
  int rc;
  const int64_t dmax = inv_dmax(P);
  const int M = P->stages;
  void* ptg;
  if ((rc = ws_get(ws, WS_C5_GT0, sizeof(double) * (size_t)dmax, &ptg))) return rc;
  double* tg = (double*)ptg;
  double *F, *G;
  bool use;
  if ((rc = inv_cache_prepare(P, ws, st, dmax, &F, &G, &use))) return rc;
  if (use) {
    ucp_inv_cache& c = ws->inv;
    int start = -1;
    for (int k = m + 1; k <= M && start < 0; ++k)
      if (c.gok[k] && std::equal(P->ukey + k, P->ukey + M, c.gkey[k] + k)) start = k;
    if (start < 0) {
      if ((rc = inv_terminal(P, G + (size_t)M * dmax, st))) return rc;
      c.gok[M] = true;
      start = M;
    }
    for (int mm = start - 1; mm >= m + 1; --mm) {
      if ((rc = inv_downstream_step(P, mm, u, G + (size_t)(mm + 1) * dmax, tg, G + (size_t)mm * dmax, st)))
        return rc;
      c.gok[mm] = true;
      std::copy(P->ukey + mm, P->ukey + M, c.gkey[mm] + mm);
    }
    *out = G + (size_t)(m + 1) * dmax;
    return UCP_OK;
  }
  void *pa, *pb;
  if ((rc = ws_get(ws, WS_C5_G0, sizeof(double) * (size_t)dmax, &pa))) return rc;
  if ((rc = ws_get(ws, WS_C5_G1, sizeof(double) * (size_t)dmax, &pb))) return rc;
  double* bufs[2] = {(double*)pa, (double*)pb};
  int cur = 0;
  if ((rc = inv_terminal(P, bufs[cur], st))) return rc;
  for (int mm = M - 1; mm >= m + 1; --mm) {
    if ((rc = inv_downstream_step(P, mm, u, bufs[cur], tg, bufs[cur ^ 1], st))) return rc;
    cur ^= 1;
  }
  *out = bufs[cur];
  return UCP_OK;
}

int inv_cost(const ucp_inv_problem* P, int m, const double* const* u, ucp_workspace* ws, cudaStream_t st,
             InvCost* c) {
  int rc;
  const double *fm, *gn;
  if ((rc = inv_forward_density(P, m, u, ws, st, &fm))) return rc;
  if ((rc = inv_downstream(P, m, u, ws, st, &gn))) return rc;
  const int nx = inv_state(P, m + 1);
  c->ym = P->pts[m];
  c->fm = fm;
  c->gnext = gn;
  c->am = P->a[m];
  c->hm = P->h[m];
  c->dm = P->d[m];
  c->an = P->a[nx];
  c->hn = P->h[nx];
  c->dn = P->d[nx];
  c->oc = P->order_cost;
  void* ptg;
  if ((rc = ws_get(ws, WS_C5_GT1, sizeof(double) * (size_t)P->d[nx], &ptg))) return rc;
  k_unif_ball_terms<<<nblocks(P->d[nx], 256), 256, 0, st>>>(gn, P->a[nx], P->h[nx], P->d[nx], (double*)ptg);
  UCP_LAUNCHED("k_unif_ball_terms");
  c->tg = (const double*)ptg;
  return UCP_OK;
}

}  // namespace

extern "C" {

int ucp_unif_moments_grid(const double* x, int64_t n, const double* v, double a, double h, int64_t d, double rad,
                          double* s0, double* s1, double* s2, void* stream) {
  if (n < 0 || d < 2) return arg_fail("unif_moments_grid: bad sizes");
  if (n == 0) return UCP_OK;
  k_unif_moments_grid<<<nblocks(n, 128), 128, 0, as_stream(stream)>>>(x, n, v, a, h, d, rad, s0, s1, s2);
  UCP_LAUNCHED("k_unif_moments_grid");
  return UCP_OK;
}

int ucp_unif_ball_sum(const double* x, int64_t n, const double* g, double a, double h, int64_t d, double rad,
                      double* out, void* stream) {
  if (n < 0 || d < 2) return arg_fail("unif_ball_sum: bad sizes");
  if (n == 0) return UCP_OK;
  k_unif_ball_sum<<<nblocks(n, 128), 128, 0, as_stream(stream)>>>(x, nullptr, n, g, a, h, d, rad, out);
  UCP_LAUNCHED("k_unif_ball_sum");
  return UCP_OK;
}

int ucp_unif_propagate(const double* masses, const double* centers, int64_t n, double a, double h, int64_t d,
                       double rad, double* out, void* stream) {
  if (n < 0 || d < 2) return arg_fail("unif_propagate: bad sizes");
  return launch_unif_propagate(masses, 1.0, centers, nullptr, n, a, h, d, rad, out, as_stream(stream));
}

int ucp_unif_moments_points(const double* y, int64_t n, const double* centers, const double* w, const double* vals,
                            int64_t m, double a, double h, int64_t d, double rad, double* m0, double* m1,
                            double* m2, void* stream) {
  if (n < 0 || m < 0 || d < 2) return arg_fail("unif_moments_points: bad sizes");
  if (n == 0) return UCP_OK;
  return launch_unif_moments_points(y, n, centers, w, vals, m, a, h, d, rad, m0, m1, m2, as_stream(stream));
}

// ---------------------------------------------------------------- ZeroDelay
int ucp_zd_cost(const ucp_zd_problem* P, int stage, const double* u0, const double* u1, const double* u_flat,
                int64_t n_cand, const int64_t* offsets, const double* y_seg, const double* f0_seg, int64_t nseg,
                double* out, ucp_workspace* ws, void* stream) {
  int rc = check_zd(P);
  if (rc) return rc;
  if (stage < 0 || stage > 1) return arg_fail("stage index out of range for zero_delay");
  if (nseg <= 0 || n_cand <= 0) return UCP_OK;
  cudaStream_t st = as_stream(stream);
  if (stage == 0) {
    ZdCost0 c;
    if ((rc = zd_cost0_tab(P, u1, ws, st, &c))) return rc;
    c.y0 = y_seg;  // per-segment observation and density
    c.f0 = f0_seg;
    k_gen_segmented<ZdCost0><<<nblocks(n_cand, 128), 128, 0, st>>>(c, u_flat, offsets, nseg, out);
    UCP_LAUNCHED("k_gen_segmented");
    return UCP_OK;
  }
  QuadCost q;
  if ((rc = zd_moments(P, u0, y_seg, nseg, ws, st, &q))) return rc;
  q.begin = 0;
  k_gen_segmented<QuadCost><<<nblocks(n_cand, 128), 128, 0, st>>>(q, u_flat, offsets, nseg, out);
  UCP_LAUNCHED("k_gen_segmented");
  return UCP_OK;
}

int ucp_zd_local_update(const ucp_zd_problem* P, int stage, const double* u0, const double* u1,
                        const ucp_local_params* lp, int64_t begin, int64_t end, double* out, int64_t* err,
                        ucp_workspace* ws, void* stream) {
  int rc = check_zd(P);
  if (rc) return rc;
  if (stage < 0 || stage > 1) return arg_fail("stage index out of range for zero_delay");
  const int64_t d = stage == 0 ? P->d0 : P->d1;
  if (!lp || !err || begin < 0 || end > d || begin > end) return arg_fail("zd_local_update: bad arguments");
  const int64_t n = end - begin;
  if (n == 0) return UCP_OK;
  cudaStream_t st = as_stream(stream);
  const double floor = P->h1;  // zero_delay.py:56-65: probe >= one decoder cell, both stages
  if (stage == 0) {
    ZdCost0 c;
    if ((rc = zd_cost0_tab(P, u1, ws, st, &c))) return rc;
    return launch_gen_local(c, u0, lp, floor, 0, begin, n, out, err, ws, st);
  }
  QuadCost q;
  if ((rc = zd_moments(P, u0, P->y1 + begin, n, ws, st, &q))) return rc;
  q.begin = begin;
  return launch_gen_local(q, u1, lp, floor, 0, begin, n, out, err, ws, st);
}

int ucp_zd_exhaustion(const ucp_zd_problem* P, int stage, const double* u0, const double* u1, const int64_t* win_lo,
                      const int64_t* win_hi, int64_t wmax, int64_t begin, int64_t end, double* out, int64_t* err,
                      ucp_workspace* ws, void* stream) {
  int rc = check_zd(P);
  if (rc) return rc;
  if (stage < 0 || stage > 1) return arg_fail("stage index out of range for zero_delay");
  const int64_t d = stage == 0 ? P->d0 : P->d1;
  if (!err || !win_lo || !win_hi || begin < 0 || end > d || begin > end) return arg_fail("zd_exhaustion: bad arguments");
  const int64_t n = end - begin;
  if (n == 0) return UCP_OK;
  cudaStream_t st = as_stream(stream);
  if (stage == 0) {
    ZdCost0 c;
    if ((rc = zd_cost0_tab(P, u1, ws, st, &c))) return rc;
    void* ps;
    if ((rc = ws_get(ws, WS_C5_MEMO, sizeof(double) * 3 * (size_t)P->d0, &ps))) return rc;
    k_zd_mom_table<<<nblocks(P->d0, 128), 128, 0, st>>>(c, u0, P->d0, (double*)ps);
    UCP_LAUNCHED("k_zd_mom_table");
    ZdCost0Memo mc;
    mc.y0 = P->y0;
    mc.f0 = P->f0;
    mc.S = (const double*)ps;
    mc.d0 = P->d0;
    mc.pw = P->power_weight;
    return launch_gen_exhaust(mc, u0, win_lo, win_hi, wmax, 0, begin, n, out, err, ws, st);
  }
  QuadCost q;
  if ((rc = zd_moments(P, u0, P->y1 + begin, n, ws, st, &q))) return rc;
  q.begin = begin;
  return launch_gen_exhaust(q, u1, win_lo, win_hi, wmax, 0, begin, n, out, err, ws, st);
}

int ucp_zd_objective_terms(const ucp_zd_problem* P, const double* u0, const double* u1, int64_t begin, int64_t end,
                           double* terms, int64_t* err, void* stream) {
  int rc = check_zd(P);
  if (rc) return rc;
  if (begin < 0 || end > P->d0 || begin > end) return arg_fail("zd_objective_terms: bad shard");
  if (end == begin) return UCP_OK;
  k_gen_terms<ZdCost0><<<nblocks(end - begin, 128), 128, 0, as_stream(stream)>>>(zd_cost0(P, u1), u0, begin, end,
                                                                                 terms, err);
  UCP_LAUNCHED("k_gen_terms");
  return UCP_OK;
}

// ---------------------------------------------------------------- Inventory
int ucp_inv_cost(const ucp_inv_problem* P, int stage, const double* const* u, const double* u_flat, int64_t n_cand,
                 const int64_t* offsets, const double* y_seg, int64_t nseg, double* out, ucp_workspace* ws,
                 void* stream) {
  int rc = check_inv(P, u);
  if (rc) return rc;
  if (stage < 0 || stage >= P->stages) return arg_fail("stage index out of range for inventory");
  if (nseg <= 0 || n_cand <= 0) return UCP_OK;
  cudaStream_t st = as_stream(stream);
  InvCost c;
  if ((rc = inv_cost(P, stage, u, ws, st, &c))) return rc;
  c.ym = y_seg;  // per-segment observation; weight via its nearest grid cell
  k_gen_segmented<InvCost><<<nblocks(n_cand, 128), 128, 0, st>>>(c, u_flat, offsets, nseg, out);
  UCP_LAUNCHED("k_gen_segmented");
  return UCP_OK;
}

int ucp_inv_local_update(const ucp_inv_problem* P, int stage, const double* const* u, const ucp_local_params* lp,
                         int64_t begin, int64_t end, double* out, int64_t* err, ucp_workspace* ws, void* stream) {
  int rc = check_inv(P, u);
  if (rc) return rc;
  if (stage < 0 || stage >= P->stages) return arg_fail("stage index out of range for inventory");
  if (!lp || !err || begin < 0 || end > P->d[stage] || begin > end) return arg_fail("inv_local_update: bad arguments");
  const int64_t n = end - begin;
  if (n == 0) return UCP_OK;
  cudaStream_t st = as_stream(stream);
  InvCost c;
  if ((rc = inv_cost(P, stage, u, ws, st, &c))) return rc;
  const double floor = P->h[inv_state(P, stage + 1)];  // inventory.py:131-136
  return launch_gen_local(c, u[stage], lp, floor, 1, begin, n, out, err, ws, st);
}

int ucp_inv_exhaustion(const ucp_inv_problem* P, int stage, const double* const* u, const int64_t* win_lo,
                       const int64_t* win_hi, int64_t wmax, int64_t begin, int64_t end, double* out, int64_t* err,
                       ucp_workspace* ws, void* stream) {
  int rc = check_inv(P, u);
  if (rc) return rc;
  if (stage < 0 || stage >= P->stages) return arg_fail("stage index out of range for inventory");
  if (!err || !win_lo || !win_hi || begin < 0 || end > P->d[stage] || begin > end)
    return arg_fail("inv_exhaustion: bad arguments");
  const int64_t n = end - begin;
  if (n == 0) return UCP_OK;
  cudaStream_t st = as_stream(stream);
  InvCost c;
  if ((rc = inv_cost(P, stage, u, ws, st, &c))) return rc;
  return launch_gen_exhaust(c, u[stage], win_lo, win_hi, wmax, 1, begin, n, out, err, ws, st);
}

int ucp_inv_objective_terms(const ucp_inv_problem* P, const double* const* u, int64_t begin, int64_t end,
                            double* terms, int64_t* err, ucp_workspace* ws, void* stream) {
  int rc = check_inv(P, u);
  if (rc) return rc;
  if (begin < 0 || end > P->d[0] || begin > end) return arg_fail("inv_objective_terms: bad shard");
  if (end == begin) return UCP_OK;
  cudaStream_t st = as_stream(stream);
  InvCost c;
  if ((rc = inv_cost(P, 0, u, ws, st, &c))) return rc;
  k_gen_terms<InvCost><<<nblocks(end - begin, 128), 128, 0, st>>>(c, u[0], begin, end, terms, err);
  UCP_LAUNCHED("k_gen_terms");
  return UCP_OK;
}

int ucp_inv_forward_density(const ucp_inv_problem* P, int stage, const double* const* u, double* out,
                            ucp_workspace* ws, void* stream) {
  int rc = check_inv(P, u);
  if (rc) return rc;
  if (stage < 0 || stage >= P->stages) return arg_fail("stage index out of range for inventory");
  const double* f;
  cudaStream_t st = as_stream(stream);
  if ((rc = inv_forward_density(P, stage, u, ws, st, &f))) return rc;
  UCP_CHECK(cudaMemcpyAsync(out, f, sizeof(double) * (size_t)P->d[stage], cudaMemcpyDeviceToDevice, st));
  return UCP_OK;
}

}  // extern "C"
