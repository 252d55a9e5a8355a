// Monte-Carlo objective on the device.
//
// Reference: oracle.monte_carlo_objective (oracle.py:98-105) over the
// problems' simulate_cost (witsenhausen.py:81-89, zero_delay.py:88-94,
// inventory.py:152-166), with controllers evaluated by nearest-point lookup
// (grids.py:141-145, 153-155).
//
// Two draw sources feed one per-sample cost function:
//  * BufferDraws -- draws made on the host by the reference's own NumPy
//    generator (PCG64), in the order simulate_cost consumes them.  Costs are
//    then bitwise the reference's (same expressions, left to right, no FMA).
//  * PhiloxDraws -- counter-based Philox4x32-10 on the device: the draws of
//    sample i depend only on (seed, i), so any sharding of
//    the samples over ranks/CTAs yields the same costs, and the fixed-shape
//    reduction below makes the estimate bitwise independent of the rank count.
//
// Deterministic reduction: samples are cut into chunks of UCP_MC_CHUNK; one
// CTA of kMcThreads sums a chunk in a fixed order (each thread a strided
// serial sum, then a shuffle tree, then the warps in order), and
// k_mc_reduce folds the chunk partials in another fixed order.  Nothing
// depends on grid size, scheduling or atomics.

namespace {

constexpr int kMcThreads = 256;
constexpr int kMcPerThread = UCP_MC_CHUNK / kMcThreads;
static_assert(UCP_MC_CHUNK % kMcThreads == 0, "chunk must be a multiple of the CTA size");
constexpr int kMcReduceThreads = 1024;

// grids.py:141-145: clip(ceil((y - a)/h - 0.5).astype(int64), 0, d - 1).  The
// float->int64 cast of NaN/inf/out-of-range values yields INT64_MIN on x86,
// which the clip maps to 0.
__device__ __forceinline__ int64_t mc_nearest(double y, double a, double h, int64_t d) {
  const double c = ceil(__dsub_rn(__ddiv_rn(__dsub_rn(y, a), h), 0.5));
  if (!(c >= 0.0) || !(c < 9.2233720368547758e18)) return 0;
  const int64_t i = (int64_t)c;
  return i > d - 1 ? d - 1 : i;
}

// Draw interface: uniform2 returns the uniforms of logical streams 2c and
// 2c+1 (the second only if 2c+1 < S); normal2 a pair of normals for streams
// (s0, s1); normal1 one normal.
struct BufferDraws {
  const double* p;  // [streams][n]
  int64_t n;
  __device__ __forceinline__ double at(int64_t i, int s) const { return p[(int64_t)s * n + i]; }
  __device__ __forceinline__ void normal2(int64_t i, double, double, double, double, double& a, double& b) const {
    a = at(i, 0);
    b = at(i, 1);
  }
  __device__ __forceinline__ double normal1(int64_t i, int s, double, double) const { return at(i, s); }
  __device__ __forceinline__ double uniform1(int64_t i, int s, double, double) const { return at(i, s); }
  __device__ __forceinline__ void uniform2(int64_t i, int c, int S, double, double, double out[2]) const {
    out[0] = at(i, 2 * c);
    out[1] = 2 * c + 1 < S ? at(i, 2 * c + 1) : 0.0;
  }
};

__device__ __forceinline__ void philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                                              uint32_t k1, uint32_t out[4]) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
    const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
    c0 = hi1 ^ c1 ^ k0;
    c1 = lo1;
    c2 = hi0 ^ c3 ^ k1;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

// 53 random bits -> the open interval (0, 1): (x + 0.5) * 2^-53.
__device__ __forceinline__ double mc_u01(uint32_t hi, uint32_t lo) {
  const uint64_t x = (((uint64_t)hi << 32) | lo) >> 11;
  return __dmul_rn(__dadd_rn((double)x, 0.5), 1.1102230246251565e-16);
}

// Device generator: counter (i, c) of Philox4x32-10 (key = seed) yields the
// unit uniforms U[i][2c], U[i][2c+1].  Normals come from Box-Muller on the
// pair (U[i][0], U[i][1]): r = sqrt(-2 ln u1), z_cos = r cos(2 pi u2),
// z_sin = r sin(2 pi u2).
struct PhiloxDraws {
  uint32_t k0, k1;
  int ubase;  // logical uniform stream s reads U[i][s + ubase] (zero_delay: 1, past the Box-Muller pair)
  __device__ __forceinline__ void pair(int64_t i, int c, double& u1, double& u2) const {
    uint32_t w[4];
    philox4x32_10((uint32_t)i, (uint32_t)((uint64_t)i >> 32), (uint32_t)c, 0u, k0, k1, w);
    u1 = mc_u01(w[0], w[1]);
    u2 = mc_u01(w[2], w[3]);
  }
  __device__ __forceinline__ void normal2(int64_t i, double loc0, double sc0, double loc1, double sc1, double& a,
                                          double& b) const {
    double u1, u2, sn, cs;
    pair(i, 0, u1, u2);
    const double r = sqrt(__dmul_rn(-2.0, log(u1)));
    sincospi(__dmul_rn(2.0, u2), &sn, &cs);
    a = __dadd_rn(loc0, __dmul_rn(sc0, __dmul_rn(r, cs)));
    b = __dadd_rn(loc1, __dmul_rn(sc1, __dmul_rn(r, sn)));
  }
  // stream 0 only (the cosine normal of pair 0)
  __device__ __forceinline__ double normal1(int64_t i, int, double loc, double scale) const {
    double u1, u2;
    pair(i, 0, u1, u2);
    const double z = __dmul_rn(sqrt(__dmul_rn(-2.0, log(u1))), cospi(__dmul_rn(2.0, u2)));
    return __dadd_rn(loc, __dmul_rn(scale, z));
  }
  // numpy's uniform(lo, hi) = lo + (hi - lo) * u of logical stream s
  __device__ __forceinline__ double uniform1(int64_t i, int s, double lo, double hi) const {
    double u1, u2;
    const int k = s + ubase;
    pair(i, k >> 1, u1, u2);
    return __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), (k & 1) ? u2 : u1));
  }
  __device__ __forceinline__ void uniform2(int64_t i, int c, int, double lo, double hi, double out[2]) const {
    double u1, u2;
    pair(i, c, u1, u2);
    out[0] = __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), u1));
    out[1] = __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), u2));
  }
};

__device__ __forceinline__ double mc_gamma(const ucp_mc_problem& P, double x) {  // inventory.py:61-69
  if (P.quadratic) return __dmul_rn(x, x);
  return __dadd_rn(__dmul_rn(P.holding_rate, np_maximum(x, 0.0)), __dmul_rn(P.backlog_rate, np_maximum(-x, 0.0)));
}

// One simulated run's cost, the reference's expressions left to right.
template <class Draws>
__device__ __forceinline__ double mc_cost(const ucp_mc_problem& P, const Draws& D, int64_t i) {
  if (P.kind == UCP_MC_WITSENHAUSEN) {  // witsenhausen.py:81-89
    double x0, w;
    D.normal2(i, 0.0, P.sigma, 0.0, 1.0, x0, w);
    const double u0 = P.u[0][mc_nearest(x0, P.a[0], P.h[0], P.d[0])];
    const double x1 = __dadd_rn(x0, u0);
    const double u1 = P.u[1][mc_nearest(__dadd_rn(x1, w), P.a[1], P.h[1], P.d[1])];
    const double x2 = __dsub_rn(x1, u1);
    return __dadd_rn(__dmul_rn(__dmul_rn(__dmul_rn(P.k, P.k), u0), u0), __dmul_rn(x2, x2));
  }
  if (P.kind == UCP_MC_ZERO_DELAY) {  // zero_delay.py:88-94
    const double x0 = D.normal1(i, 0, 0.0, 1.0);
    const double u0 = P.u[0][mc_nearest(x0, P.a[0], P.h[0], P.d[0])];
    const double w = D.uniform1(i, 1, -1.0, 1.0);
    const double u1 = P.u[1][mc_nearest(__dadd_rn(u0, w), P.a[1], P.h[1], P.d[1])];
    const double err = __dsub_rn(u1, x0);
    return __dadd_rn(__dmul_rn(__dmul_rn(P.power_weight, u0), u0), __dmul_rn(err, err));
  }
  // inventory.py:152-166: stock snaps to the state grid at every boundary;
  // uniforms U[0] (initial stock) and U[1 + mm] (demand of stage mm), two per draw
  const int M = P.stages, S = M + 1;
  double u2[2];
  D.uniform2(i, 0, S, -1.0, 1.0, u2);
  double x = P.pts[0][mc_nearest(u2[0], P.a[0], P.h[0], P.d[0])];
  double total = 0.0;
  for (int mm = 0; mm < M; ++mm) {
    const double u = P.u[mm][mc_nearest(x, P.a[mm], P.h[mm], P.d[mm])];
    const int s = 1 + mm;
    if (s > 1 && !(s & 1)) D.uniform2(i, s >> 1, S, -1.0, 1.0, u2);
    const double w = u2[s & 1];
    const int nx = mm + 1 < M ? mm + 1 : M - 1;
    x = P.pts[nx][mc_nearest(__dsub_rn(__dadd_rn(x, u), w), P.a[nx], P.h[nx], P.d[nx])];
    total = __dadd_rn(total, __dadd_rn(__dmul_rn(P.order_cost, u), mc_gamma(P, x)));
  }
  return total;
}

__global__ void k_mc_costs(const ucp_mc_problem P, BufferDraws D, int64_t n, double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = mc_cost(P, D, i);
}

// The device generator's draws in the reference's stream layout [S][n]
// (BufferDraws order): what mc_cost consumes for each sample.
__global__ void k_mc_draws(const ucp_mc_problem P, PhiloxDraws D, int64_t begin, int64_t end, double* __restrict__ out) {
  const int64_t n = end - begin;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = begin + t;
    if (P.kind == UCP_MC_WITSENHAUSEN) {
      D.normal2(i, 0.0, P.sigma, 0.0, 1.0, out[t], out[n + t]);
    } else if (P.kind == UCP_MC_ZERO_DELAY) {
      out[t] = D.normal1(i, 0, 0.0, 1.0);
      out[n + t] = D.uniform1(i, 1, -1.0, 1.0);
    } else {
      for (int s = 0; s <= P.stages; ++s) out[(int64_t)s * n + t] = D.uniform1(i, s, -1.0, 1.0);
    }
  }
}

// Fixed-order block sum of v over the CTA; result valid in thread 0.
__device__ __forceinline__ double mc_block_sum(double v, double* warp_sums) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, off));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) warp_sums[warp] = v;
  UCP_SYNC();
  double s = 0.0;
  if (threadIdx.x == 0) {
    s = warp_sums[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) s = __dadd_rn(s, warp_sums[w]);
  }
  UCP_SYNC();
  return s;
}

// Chunk partials over chunks [cb, ce): pass 0 (total == nullptr) sums the
// costs, pass 1 sums (c - mean)^2 with mean = *total / n.
__global__ void __launch_bounds__(kMcThreads) k_mc_partials(const ucp_mc_problem P, PhiloxDraws D, int64_t n,
                                                            int64_t cb, int64_t ce, const double* __restrict__ total,
                                                            double* __restrict__ out) {
  __shared__ double warp_sums[kMcThreads / 32];
  const double mean = total ? __ddiv_rn(*total, (double)n) : 0.0;
  for (int64_t c = cb + blockIdx.x; c < ce; c += gridDim.x) {
    double acc = 0.0;
#pragma unroll 4
    for (int j = 0; j < kMcPerThread; ++j) {
      const int64_t i = c * UCP_MC_CHUNK + threadIdx.x + (int64_t)kMcThreads * j;
      if (i < n) {
        double v = mc_cost(P, D, i);
        if (total) {
          v = __dsub_rn(v, mean);
          v = __dmul_rn(v, v);
        }
        acc = __dadd_rn(acc, v);
      }
    }
    const double s = mc_block_sum(acc, warp_sums);
    if (threadIdx.x == 0) out[c - cb] = s;
  }
}

__global__ void __launch_bounds__(kMcReduceThreads) k_mc_reduce(const double* __restrict__ x, int64_t n,
                                                                double* __restrict__ out) {
  __shared__ double warp_sums[kMcReduceThreads / 32];
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += kMcReduceThreads) acc = __dadd_rn(acc, x[i]);
  const double s = mc_block_sum(acc, warp_sums);
  if (threadIdx.x == 0) *out = s;
}

int check_mc(const ucp_mc_problem* P) {
  if (!P) return arg_fail("mc: null problem");
  if (P->kind < UCP_MC_WITSENHAUSEN || P->kind > UCP_MC_INVENTORY) return arg_fail("mc: unknown problem kind");
  const int M = P->kind == UCP_MC_INVENTORY ? P->stages : 2;
  if (M < 1 || M > UCP_INV_MAX_STAGES) return arg_fail("mc: bad stage count");
  for (int m = 0; m < M; ++m) {
    if (!P->u[m] || P->d[m] < 2) return arg_fail("mc: bad controller / grid");
    if (P->kind == UCP_MC_INVENTORY && !P->pts[m]) return arg_fail("mc: inventory needs grid points");
  }
  return UCP_OK;
}

unsigned mc_grid(int64_t work, int threads) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (work + threads - 1) / threads;
  const int64_t cap = (int64_t)sms * (2048 / threads);
  return (unsigned)(want < cap ? (want > 0 ? want : 1) : cap);
}

PhiloxDraws philox(const ucp_mc_problem* P, uint64_t seed) {
  return PhiloxDraws{(uint32_t)seed, (uint32_t)(seed >> 32), P->kind == UCP_MC_ZERO_DELAY ? 1 : 0};
}

}  // namespace

extern "C" {

int ucp_mc_streams(const ucp_mc_problem* P) {
  if (check_mc(P)) return -1;
  return P->kind == UCP_MC_INVENTORY ? P->stages + 1 : 2;
}

int ucp_mc_costs(const ucp_mc_problem* P, const double* draws, int64_t n, double* costs, void* stream) {
  int rc;
  if ((rc = check_mc(P))) return rc;
  if (n < 0 || (n > 0 && (!draws || !costs))) return arg_fail("mc_costs: bad buffers");
  if (n == 0) return UCP_OK;
  k_mc_costs<<<mc_grid(n, 256), 256, 0, as_stream(stream)>>>(*P, BufferDraws{draws, n}, n, costs);
  UCP_LAUNCHED("k_mc_costs");
  return UCP_OK;
}

int ucp_mc_philox_draws(const ucp_mc_problem* P, uint64_t seed, int64_t begin, int64_t end, double* draws,
                        void* stream) {
  int rc;
  if ((rc = check_mc(P))) return rc;
  if (begin < 0 || end < begin || (end > begin && !draws)) return arg_fail("mc_philox_draws: bad range");
  if (end == begin) return UCP_OK;
  k_mc_draws<<<mc_grid(end - begin, 256), 256, 0, as_stream(stream)>>>(*P, philox(P, seed), begin, end, draws);
  UCP_LAUNCHED("k_mc_draws");
  return UCP_OK;
}

int ucp_mc_partials(const ucp_mc_problem* P, uint64_t seed, int64_t n, int64_t chunk_begin, int64_t chunk_end,
                    const double* total, double* partials, void* stream) {
  int rc;
  if ((rc = check_mc(P))) return rc;
  const int64_t chunks = (n + UCP_MC_CHUNK - 1) / UCP_MC_CHUNK;
  if (n < 1 || chunk_begin < 0 || chunk_end < chunk_begin || chunk_end > chunks)
    return arg_fail("mc_partials: bad sample / chunk range");
  if (chunk_end == chunk_begin) return UCP_OK;
  if (!partials) return arg_fail("mc_partials: null output");
  const unsigned grid = mc_grid((chunk_end - chunk_begin) * kMcThreads, kMcThreads);
  k_mc_partials<<<grid, kMcThreads, 0, as_stream(stream)>>>(*P, philox(P, seed), n, chunk_begin, chunk_end, total,
                                                            partials);
  UCP_LAUNCHED("k_mc_partials");
  return UCP_OK;
}

int ucp_mc_reduce(const double* partials, int64_t n, double* out, void* stream) {
  if (n < 0 || !out || (n > 0 && !partials)) return arg_fail("mc_reduce: bad buffers");
  k_mc_reduce<<<1, kMcReduceThreads, 0, as_stream(stream)>>>(partials, n, out);
  UCP_LAUNCHED("k_mc_reduce");
  return UCP_OK;
}

}  // extern "C"
