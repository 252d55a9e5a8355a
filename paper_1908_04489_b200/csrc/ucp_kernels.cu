// B200 (sm_100a) kernels + C ABI for the Witsenhausen marginal-cost hot path
// of arXiv 1908.04489's UCP solver.  See DESIGN.md for the data layout, the
// roofline of each kernel and the exactness argument; include/ucp_b200.h for
// the boundary.  Build: nvcc -gencode arch=compute_100a,code=sm_100a
// -fmad=false (no FMA contraction: the reference has none).
//
// "ref-order": every kernel evaluates the reference's expressions with the
// same association, the same per-output summation order and glibc-exact
// exp/erf, so outputs are bitwise the reference's.  Parallelism only spans
// independent outputs (candidates, points, queries), as numba's prange does.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <vector>
#include <mutex>
#include <shared_mutex>
#include <map>
#include <set>
#include <unordered_set>
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_scan.cuh>

#include "../../include/ucp_b200.h"
#include "ucp_libm.h"

#ifndef __CUDACC__
#error "compile with nvcc"
#endif

namespace {

// Stress build (-DUCP_STRESS; tools/stress_build.py, tests/test_gpu_stress.py):
// compute-sanitizer is closed on this pool, so races are shaken out by
// delaying a pseudo-random eighth of the threads (up to ~2 us, seeded by the
// clock) around every barrier, mbarrier wait, bulk-copy issue and work-queue
// fetch, and index invariants are checked with device traps.  Results must
// stay bitwise equal to the oracle under any schedule.  Both macros compile
// to nothing in the production build.
#ifdef UCP_STRESS
__device__ __forceinline__ void ucp_jitter(unsigned site) {
  unsigned x = (unsigned)clock64() ^ (threadIdx.x * 0x9E3779B9u) ^ (blockIdx.x * 0x85EBCA6Bu) ^
               (blockIdx.y * 0x27D4EB2Fu) ^ (site * 0xC2B2AE35u);
  x ^= x >> 15;
  x *= 0x2C1B3C6Du;
  x ^= x >> 12;
  x *= 0x297A2D39u;
  x ^= x >> 15;
  if ((x & 7u) == 0u) __nanosleep((x >> 16) & 2047u);
}
#define UCP_JITTER() ucp_jitter(__LINE__)
#define UCP_DCHECK(cond)                                                                        \
  do {                                                                                          \
    if (!(cond)) {                                                                              \
      printf("UCP_DCHECK failed: %s at %s:%d (block %d,%d thread %d)\n", #cond, __FILE__, __LINE__, \
             (int)blockIdx.x, (int)blockIdx.y, (int)threadIdx.x);                               \
      __trap();                                                                                 \
    }                                                                                           \
  } while (0)
#else
#define UCP_JITTER() ((void)0)
#define UCP_DCHECK(cond) ((void)0)
#endif
// __syncthreads with the stress build's jitter on both sides
#define UCP_SYNC()      \
  do {                  \
    UCP_JITTER();       \
    __syncthreads();    \
    UCP_JITTER();       \
  } while (0)

constexpr double kGaussCut = 12.0;  // kernels.py:55 GAUSS_CUT
// Walk kernels (one serial Gaussian walk per thread): 128-thread CTAs, at
// least 12 resident per SM (<= 42 registers) so 12 warps per scheduler hide
// the L1 latency of the v1 stream behind the FP64 pipe.
constexpr int kWalkThreads = 128;
#ifndef UCP_WALK_MIN_BLOCKS
#define UCP_WALK_MIN_BLOCKS 12
#endif
constexpr int kWalkMinBlocks = UCP_WALK_MIN_BLOCKS;
// throughput walk: 4-node groups per tail-check chunk, and the unroll of that loop
#ifndef UCP_WALK_CHUNK4
#define UCP_WALK_CHUNK4 64
#endif
#ifndef UCP_WALK_UNROLL
#define UCP_WALK_UNROLL 8
#endif
constexpr int kWalkChunk4 = UCP_WALK_CHUNK4, kWalkUnroll = UCP_WALK_UNROLL;

__device__ const uint64_t g_exp_tab[256] = UCP_EXP_TAB_INIT;
const uint64_t h_exp_tab[256] = UCP_EXP_TAB_INIT;

std::atomic<int64_t> g_launches{0};
thread_local char g_errbuf[256] = "";

__host__ __device__ __forceinline__ double inv_sqrt_2pi() { return ucp_asf64(UCP_INV_SQRT_2PI_BITS); }

int cuda_fail(cudaError_t e, const char* where) {
  snprintf(g_errbuf, sizeof g_errbuf, "%s: %s", where, cudaGetErrorString(e));
  return UCP_ERR_CUDA;
}

#define UCP_CHECK(call)                                  \
  do {                                                   \
    cudaError_t e_ = (call);                             \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call);  \
  } while (0)

#define UCP_LAUNCHED(name)                                          \
  do {                                                              \
    g_launches.fetch_add(1, std::memory_order_relaxed);             \
    cudaError_t e_ = cudaGetLastError();                            \
    if (e_ != cudaSuccess) return cuda_fail(e_, "launch " name);    \
  } while (0)

int arg_fail(const char* msg) {
  snprintf(g_errbuf, sizeof g_errbuf, "%s", msg);
  return UCP_ERR_ARG;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Opt a kernel in to more than 48 KiB of dynamic shared memory, once per
// (kernel, device): the attribute lives in each device's context.
std::mutex g_smem_mu;
std::set<std::pair<const void*, int>> g_smem_ok;
void smem_opt_in(const void* fn, size_t bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(g_smem_mu);
  if (g_smem_ok.insert({fn, dev}).second) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}
inline unsigned nblocks(int64_t n, int threads) { return (unsigned)((n + threads - 1) / threads); }

// Programmatic dependent launch: kernels of a block iteration are launched
// with programmatic stream serialisation, wait for their predecessor with
// griddepcontrol.wait before touching its outputs, and let their successor
// launch early (griddepcontrol.launch_dependents) -- the launch gap between
// dependent kernels overlaps the predecessor's tail.  Both instructions are
// no-ops for kernels launched without the attribute.  UCP_PDL=0 disables it.
const bool g_pdl = [] {
  const char* e = getenv("UCP_PDL");
  return !(e && e[0] == '0');
}();
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }
template <class... KArgs, class... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// --------------------------------------------------------------------------
// Stage-0 inner moments: the windowed Gaussian walk of kernels.py:406-445.
// --------------------------------------------------------------------------
struct WalkGrid {
  double a, h, b, q;  // b = a + h*(d-1); q = exp(-h*h)   (kernels.py:411-412)
  int64_t d;
  // Range-max bounds for the walk's no-op tail (nullptr: walk every node): a
  // sparse table over 256-node blocks, level k at vsuf + k*nb holding
  // max |v| over blocks [b, b + 2^k), +inf when any v there is not finite
  // (see walk_tail_noop / k_vsuf).
  const double* vsuf;
  int nb;
  int64_t vstride;  // batched engine: slot s's table at vsuf + s * vstride
  // instrumentation (ucp_walk_node_counter): visited walk nodes are added here
  unsigned long long* visits;
  // UCP_WC_FAST (ucp_wc_problem.flags): the tolerance-stated FMA walk
  // (gauss_walk_impl<kMode, true>); 0 = the reference's arithmetic
  int fast;
  // UCP_WC_TABLE: window-sum expansions per cell (nullptr = walk every
  // centre): cell c, centred at ex_s0 + c * ex_dlt, holds kExK x 3
  // coefficients (k_ex_cells), read by ex_moments
  const double* table;
  double ex_s0, ex_dlt, ex_inv;
  double ex_ih, ex_dq2;  // 1/h and dq/2 (the reference walk's bias, ex_moments)
  int64_t ex_n;
};
constexpr int kVsufShift = 8;  // 256 nodes per block

struct Mom3 {
  double t0, t1, t2;
};

// Instance dimension of the batched engine (config 4, ucp_wc_batch_*): a
// launch covers slots blockIdx.y (k_moments: its work items), slot s running
// instance ids[s].  Stage-0 arrays (u0, f0, fw0) of instance b start at
// b*su0, u1 at b*su1; per-slot scratch at s*sslot; error slots at b*serr.
// kNoBatch (ids == nullptr) is the single-instance case: every offset 0.
struct BatchArgs {
  const int32_t* ids;
  int64_t su0, su1, sslot, serr;
  const double* kvec;  // per-instance k (nullptr: the scalar argument)
  __device__ __forceinline__ int inst(int slot) const { return ids ? ids[slot] : 0; }
};
constexpr BatchArgs kNoBatch = {nullptr, 0, 0, 0, 0, nullptr};

// ucp_walk_node_counter (instrumentation only); read once per walk grid
std::atomic<unsigned long long*> g_visits{nullptr};

WalkGrid make_walk_grid(double a, double h, int64_t d, int fast = 0) {
  WalkGrid g;
  g.fast = fast;
  g.table = nullptr;
  g.ex_s0 = g.ex_dlt = g.ex_inv = g.ex_ih = g.ex_dq2 = 0.0;
  g.ex_n = 0;
  g.a = a;
  g.h = h;
  g.d = d;
  g.b = a + h * (double)(d - 1);
  g.q = ucp_exp_tab((-h) * h, h_exp_tab);  // same port as the device: bitwise glibc
  g.vsuf = nullptr;
  g.vstride = 0;
  g.nb = (int)((d + (1 << 8) - 1) >> 8);
  g.visits = g_visits.load(std::memory_order_acquire);
  return g;
}

__device__ __forceinline__ double phi_cdf(double z) { return ucp_phi_cdf_tab(z, g_exp_tab); }

// One centre s: T_k(s) = sum_j W_j pdf(y_j - s) v_j^k + cdf tails.  The
// window walk is inherently serial (multiplicative pdf recurrence,
// kernels.py:438-439); one thread owns one centre.  Nodes 0 and d-1 (half
// trapezoid weight) are peeled so the interior loop is branch-free.
//
// kLat (latency mode, used when a launch has too few walks to fill the GPU,
// e.g. d = 2000): the thread prefetches its whole v1 window into L1 first and
// issues each group's loads one group ahead, so a lone warp per scheduler is
// bound by its DMUL chain instead of L2 latency.  Throughput mode (large d)
// keeps the register footprint at 40 so 12 CTAs/SM hide the latency instead.
// kMode: 0 = throughput (global __ldg, 12 CTAs/SM), 1 = latency (L1
// prefetch + loads one group ahead), 2 = latency with v1 staged whole in
// shared memory (small grids, d <= kSmemWalkMax).
template <int kMode>
__device__ __forceinline__ double walk_ld(const double* v, int j) {
  if (kMode == 2) return v[j];
  return __ldg(v + j);
}
template <int kMode>
__device__ __forceinline__ double2 walk_ld2(const double* v, int j) {
  if (kMode == 2) return *reinterpret_cast<const double2*>(v + j);
  return __ldg(reinterpret_cast<const double2*>(v + j));
}

// Result-invariant early end of a walk (throughput mode only).  Past the
// Gaussian's peak (ratio <= 1; q < 1 keeps every later ratio <= 1) the
// computed pdf never grows (fl is monotone and pdf*ratio <= pdf), so with
// wpc = fl(h*pdf) and vm >= |v_j'| for every remaining node, monotonicity of
// rounding bounds every remaining addend exactly:
//   acc0 += wp' <= wpc,  |acc1 += wv'| <= fl(wpc*vm),  acc2 += fl(wv'*v') <= fl(fl(wpc*vm)*vm).
// An addend t with |t| < |acc| * 2^-55 (< 2^(E-54) for acc in [2^E, 2^(E+1)):
// half the smaller ulp around acc, acc normal) leaves acc unchanged under round-to-nearest, so once all three
// bounds are below their thresholds no remaining node changes a bit and the
// walk may stop.  vm = +inf (a non-finite v ahead) or NaN never passes.
__device__ __forceinline__ bool walk_tail_noop(double pdf, double ratio, double h, double vm, double acc0,
                                               double acc1, double acc2) {
  const double e = 0x1p-55, tiny = 0x1p-960;
  const double wpc = h * pdf;
  const double b1 = wpc * vm;
  const double b2 = b1 * vm;
  const double a1 = fabs(acc1);
  return ratio <= 1.0 && acc0 > tiny && a1 > tiny && acc2 > tiny && wpc < acc0 * e && b1 < a1 * e &&
         b2 < acc2 * e;
}

// max |v| over 256-node blocks [bl, br] (bl <= br) from the sparse table
__device__ __forceinline__ double range_max(const double* __restrict__ t, int nb, int bl, int br) {
  const int k = 31 - __clz(br - bl + 1);
  const double* lv = t + (size_t)k * nb;
  return fmax(__ldg(lv + bl), __ldg(lv + br - (1 << k) + 1));
}

// kFast (UCP_WC_FAST, opt-in, NOT the reference's arithmetic): h is folded
// into the pdf recurrence (p = h*pdf) and the v-weighted sums use FMA --
// acc1 = fma(p, v, acc1), acc2 = fma(p*v, v, acc2) -- 6 FP64 instructions
// per interior node instead of 8.  Same nodes, same order, same exp/erf,
// same no-op tail exit; every sum differs from the reference by rounding
// only (tests/test_gpu_fast_mode.py states and checks the tolerance).
template <int kMode, bool kFast>
__device__ __forceinline__ Mom3 gauss_walk_impl(double st, const double* __restrict__ v, const WalkGrid g) {
  constexpr bool kLat = kMode != 0;
  long long jlo = (long long)ceil(((st - kGaussCut) - g.a) / g.h);
  long long jhi = (long long)floor(((st + kGaussCut) - g.a) / g.h);
  if (jlo < 0) jlo = 0;
  if (jhi > g.d - 1) jhi = g.d - 1;
  double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
  if (jlo <= jhi) {
    const double h = g.h;
    const double q = g.q;
    double tt = (g.a + (double)jlo * h) - st;
    double pdf = ucp_exp_tab((-0.5 * tt) * tt, g_exp_tab) * inv_sqrt_2pi();
    double ratio = ucp_exp_tab((-h) * (tt + 0.5 * h), g_exp_tab);
    if (kFast) pdf = h * pdf;  // p = h * pdf: interior weight 1, end weight 1/2
    const int last = (int)(g.d - 1);
    const int je = (int)jhi;
    int j = (int)jlo;
#define UCP_WALK_STEP_V(W, VJ)                   \
  {                                              \
    double wp = (W) * pdf;                       \
    acc0 += wp;                                  \
    if (kFast) {                                 \
      acc1 = __fma_rn(wp, (VJ), acc1);           \
      acc2 = __fma_rn(wp * (VJ), (VJ), acc2);    \
    } else {                                     \
      double wv = wp * (VJ);                     \
      acc1 += wv;                                \
      acc2 += wv * (VJ);                         \
    }                                            \
    pdf *= ratio;                                \
    ratio *= q;                                  \
  }
#define UCP_WALK_STEP(W)                      \
  {                                           \
    const double vj_ = walk_ld<kMode>(v, j);  \
    UCP_WALK_STEP_V(W, vj_);                  \
  }
    if (kMode == 1) {
      for (int p = j & ~15; p <= je; p += 16) asm volatile("prefetch.global.L1 [%0];" ::"l"(v + p));
    }
    const double hw = kFast ? 1.0 : h;         // interior node weight (folded into p in fast mode)
    const double hh = kFast ? 0.5 : 0.5 * h;   // end node weight
    if (j == 0) {
      UCP_WALK_STEP(hh);
      ++j;
    }
    const int jint = je < last ? je : last - 1;
    // interior nodes, two per 16-byte load (v1 is 16-byte aligned: checked
    // by the host); an odd first node is peeled so the order is unchanged
    if ((j & 1) && j <= jint) {
      UCP_WALK_STEP(hw);
      ++j;
    }
    if (kLat) {
      if (j + 3 <= jint) {
        double2 p0 = walk_ld2<kMode>(v, j);
        double2 p1 = walk_ld2<kMode>(v, j + 2);
        for (; j + 7 <= jint; j += 4) {
          const double2 n0 = walk_ld2<kMode>(v, j + 4);
          const double2 n1 = walk_ld2<kMode>(v, j + 6);
          UCP_WALK_STEP_V(hw, p0.x);
          UCP_WALK_STEP_V(hw, p0.y);
          UCP_WALK_STEP_V(hw, p1.x);
          UCP_WALK_STEP_V(hw, p1.y);
          p0 = n0;
          p1 = n1;
        }
        UCP_WALK_STEP_V(hw, p0.x);
        UCP_WALK_STEP_V(hw, p0.y);
        UCP_WALK_STEP_V(hw, p1.x);
        UCP_WALK_STEP_V(hw, p1.y);
        j += 4;
      }
    } else {
      const double* __restrict__ vsuf = g.vsuf;
      // 256-node chunks (4 x UCP_WALK_CHUNK4; A/B at 2^18: 64-node chunks unrolled x2
      // 455 ms, 256 unrolled x8 425 ms) with a counter-free inner loop;
      // the tail check runs between chunks (any check point is result-invariant)
      while (j + (4 * kWalkChunk4 - 1) <= jint) {
#pragma unroll kWalkUnroll
        for (int c = 0; c < kWalkChunk4; ++c, j += 4) {
          const double2 p0 = __ldg(reinterpret_cast<const double2*>(v + j));
          const double2 p1 = __ldg(reinterpret_cast<const double2*>(v + j + 2));
          UCP_WALK_STEP_V(hw, p0.x);
          UCP_WALK_STEP_V(hw, p0.y);
          UCP_WALK_STEP_V(hw, p1.x);
          UCP_WALK_STEP_V(hw, p1.y);
        }
        if (vsuf && ratio <= 1.0 && j <= jint &&
            walk_tail_noop(pdf, ratio, hw, range_max(vsuf, g.nb, j >> kVsufShift, je >> kVsufShift), acc0, acc1,
                           acc2)) {
          // every remaining node (incl. a half-weight last one) is a no-op; j > je
          // skips them and encodes the first unvisited node for the node counter
          j = 2 * (je + 1) - j;
          break;
        }
      }
      // the rest in 64-node chunks, still checked: a short window (e.g. 960
      // nodes at d = 2000, the batched engine's sizes) reaches its tail here
      while (j + 63 <= jint) {
#pragma unroll 2
        for (int c = 0; c < 16; ++c, j += 4) {
          const double2 p0 = __ldg(reinterpret_cast<const double2*>(v + j));
          const double2 p1 = __ldg(reinterpret_cast<const double2*>(v + j + 2));
          UCP_WALK_STEP_V(hw, p0.x);
          UCP_WALK_STEP_V(hw, p0.y);
          UCP_WALK_STEP_V(hw, p1.x);
          UCP_WALK_STEP_V(hw, p1.y);
        }
        if (vsuf && ratio <= 1.0 && j <= jint &&
            walk_tail_noop(pdf, ratio, hw, range_max(vsuf, g.nb, j >> kVsufShift, je >> kVsufShift), acc0, acc1,
                           acc2)) {
          j = 2 * (je + 1) - j;
          break;
        }
      }
      for (; j + 3 <= jint; j += 4) {
        const double2 p0 = __ldg(reinterpret_cast<const double2*>(v + j));
        const double2 p1 = __ldg(reinterpret_cast<const double2*>(v + j + 2));
        UCP_WALK_STEP_V(hw, p0.x);
        UCP_WALK_STEP_V(hw, p0.y);
        UCP_WALK_STEP_V(hw, p1.x);
        UCP_WALK_STEP_V(hw, p1.y);
      }
    }
    for (; j <= jint; ++j) UCP_WALK_STEP(hw);
    if (je == last && j == last) UCP_WALK_STEP(hh);
    UCP_DCHECK(jlo >= 0 && je <= last && j >= jint + 1 && j <= je + 1 + (int)(je - jlo + 1));
    if (!kLat && g.visits) {  // instrumentation: nodes this walk visited
      const int jstop = (je == last && j == last) ? je + 1 : 2 * (je + 1) - j;  // first unvisited node
      const unsigned n = (unsigned)(jstop - (int)jlo);
      const unsigned mask = __activemask();
      const unsigned tot = __reduce_add_sync(mask, n);
      if ((threadIdx.x & 31) == __ffs(mask) - 1) atomicAdd(g.visits, (unsigned long long)tot);
    }
#undef UCP_WALK_STEP
#undef UCP_WALK_STEP_V
  }
  Mom3 r;
  double lo = phi_cdf(g.a - st);
  double hi = phi_cdf(st - g.b);
  const double v0 = walk_ld<kMode>(v, 0), vl = walk_ld<kMode>(v, (int)(g.d - 1));
  r.t0 = (acc0 + lo) + hi;
  r.t1 = (acc1 + lo * v0) + hi * vl;
  r.t2 = (acc2 + (lo * v0) * v0) + (hi * vl) * vl;
  return r;
}

// UCP_WC_TABLE, expansion form: the window sums about a cell centre sc.  With
// t_j = y_j - sc and d = s - sc, pdf(y_j - s) = pdf(t_j) exp(-d^2/2) exp(t_j d),
// so S_pk(s) = sum_j W_j pdf(y_j - s) t_j^p v_j^k = exp(-d^2/2) sum_n d^n / n! A_(n+p)k,
// A_nk = sum_j W_j pdf(t_j) t_j^n v_j^k (nodes within 12 + dlt/2 of sc).
// |d| <= dlt/2 = 0.008 and |t| <= 12.008: the first omitted term is below
// (12.008 * 0.008)^12 / 12! ~ 1e-21 of the sums; coefficients are summed per
// thread then tree-reduced (~1e-16).
//
// S_0k are the TRUE window sums.  The reference's walk is not: its pdf
// recurrence multiplies by ratio_i = ratio_0 q^i with q = fl(exp(-h^2)), so
// node m = j - jlo of the window carries the factor (1 + dq)^(m(m-1)/2),
// dq = fl(q)/q - 1 -- a bias up to 1.4e-7 relative at h = 4.8e-5 (checked
// against the oracle's walk).  ex_moments reproduces it to first order,
//   T_k = S_0k + dq/2 sum_j W_j pdf v_j^k m_j (m_j - 1),  m_j = t_j / h + c,
// c = (sc - a)/h - jlo(s), i.e. from S_0k, S_1k, S_2k; what remains is the
// walk's per-step rounding (~3e-10 relative at 2^20, 1e-10 at 2^18).
// The sums are smooth in s, so the local update's second differences see only
// the evaluation's own rounding within a cell (unlike an interpolated table
// of independently rounded walks).
constexpr int kExK = 12, kExRows = kExK + 2;
constexpr double kExCell = 0.016;
// UCP_WC_TABLE's expansions are used on grids at least this fine (the
// k_ex_cells pass, ~ncell * 24/h nodes, pays off once windows are long; a
// stage-1 tile then holds >= 8 queries); coarser grids keep the FMA walk and
// the direct moments.
constexpr double kTableMaxH = 2e-3;
template <int kMode>
__device__ __forceinline__ Mom3 ex_moments(double st, const double* __restrict__ v, const WalkGrid& g) {
  double acc[3] = {0.0, 0.0, 0.0};
  const double f = (st - g.ex_s0) * g.ex_inv;
  if (f > -0.5 && f < (double)g.ex_n - 0.5) {
    const double fc = floor(f + 0.5);
    const double sc = g.ex_s0 + fc * g.ex_dlt;
    const double dl = st - sc;
    const double* A = g.table + (int64_t)fc * (3 * kExRows);
    double S[3][3];  // [p][k]
#pragma unroll
    for (int p = 0; p < 3; ++p)
#pragma unroll
      for (int k = 0; k < 3; ++k) S[p][k] = __ldg(A + 3 * (kExK - 1 + p) + k);
#pragma unroll
    for (int n = kExK - 2; n >= 0; --n) {
      const double fn = dl * (1.0 / (double)(n + 1));
#pragma unroll
      for (int p = 0; p < 3; ++p)
#pragma unroll
        for (int k = 0; k < 3; ++k) S[p][k] = __fma_rn(S[p][k], fn, __ldg(A + 3 * (n + p) + k));
    }
    long long jlo = (long long)ceil(((st - kGaussCut) - g.a) / g.h);  // the walk's first node
    if (jlo < 0) jlo = 0;
    const double c = (sc - g.a) * g.ex_ih - (double)jlo;
    const double b0 = c * (c - 1.0), b1 = (2.0 * c - 1.0) * g.ex_ih, b2 = g.ex_ih * g.ex_ih;
    const double gd = ucp_exp_tab((-0.5 * dl) * dl, g_exp_tab);
#pragma unroll
    for (int k = 0; k < 3; ++k)
      acc[k] = gd * (S[0][k] + g.ex_dq2 * ((S[2][k] * b2 + S[1][k] * b1) + S[0][k] * b0));
  }
  const double lo = phi_cdf(g.a - st), hi = phi_cdf(st - g.b);
  const double v0 = walk_ld<kMode>(v, 0), vl = walk_ld<kMode>(v, (int)(g.d - 1));
  Mom3 r;
  r.t0 = (acc[0] + lo) + hi;
  r.t1 = (acc[1] + lo * v0) + hi * vl;
  r.t2 = (acc[2] + (lo * v0) * v0) + (hi * vl) * vl;
  return r;
}

template <int kMode>
__device__ __forceinline__ Mom3 gauss_walk(double st, const double* __restrict__ v, const WalkGrid g) {
#ifdef UCP_NO_FAST_WALK  // (PTX audit of the reference-arithmetic walk: tests/test_abi_and_host.py)
  return gauss_walk_impl<kMode, false>(st, v, g);
#else
  if (g.table) return ex_moments<kMode>(st, v, g);
  return g.fast ? gauss_walk_impl<kMode, true>(st, v, g) : gauss_walk_impl<kMode, false>(st, v, g);
#endif
}

// witsenhausen.py:31-33 (_quad_in_u): a*u*u - 2.0*b*u + c
__device__ __forceinline__ double quad_in_u(double a, double b, double c, double u) {
  return (((a * u) * u) - ((2.0 * b) * u)) + c;
}

// witsenhausen.py:64-70: C0(u, y) = f0(y) * (k^2 u^2 + E[(s - u1(y1))^2]), s = y+u
template <int kMode>
__device__ __forceinline__ double stage0_cost(double u, double y, double f0, double k,
                                              const double* __restrict__ v1, const WalkGrid g) {
  double s = y + u;
  Mom3 t = gauss_walk<kMode>(s, v1, g);
  double inner = quad_in_u(t.t0, t.t1, t.t2, s);
  return f0 * ((((k * k) * u) * u) + inner);
}

__device__ __forceinline__ bool finite(double x) { return isfinite(x); }

__device__ __forceinline__ void flag_min(int64_t* slot, int64_t i) {
  if (slot) atomicMin(reinterpret_cast<unsigned long long*>(slot), (unsigned long long)i);
}

// ---------------------------------------------------------------- kernels
// Mode-2 walk kernels stage the whole v1 (d <= kSmemWalkMax) in shared memory
// before any thread returns; V becomes the shared copy.
#define UCP_WALK_STAGE(V, D)                                        \
  if (kMode == 2) {                                                 \
    extern __shared__ __align__(16) double ucp_sv_[];               \
    for (int r_ = threadIdx.x; r_ < (int)(D); r_ += blockDim.x)    \
      ucp_sv_[r_] = V[r_];                                          \
    UCP_SYNC();                                                \
    V = ucp_sv_;                                                    \
  }

template <int kMode>
__global__ void __launch_bounds__(kWalkThreads, kMode ? 1 : kWalkMinBlocks) k_gauss_grid(const double* __restrict__ s, int64_t n, const double* __restrict__ v,
                             WalkGrid g, double* t0, double* t1, double* t2) {
  pdl_wait();
  pdl_trigger();
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  UCP_WALK_STAGE(v, g.d);
  if (t >= n) return;
  Mom3 r = gauss_walk<kMode>(s[t], v, g);
  t0[t] = r.t0;
  t1[t] = r.t1;
  t2[t] = r.t2;
}

// UCP_WC_TABLE, expansion form: one CTA per cell, the kExRows x 3
// coefficients A_nk of ex_moments (each thread a strided share of the cell's
// nodes, then a fixed-order tree: deterministic).  Out: 3 * kExRows doubles
// per cell, [n][k].
constexpr int kExThreads = 256;
__global__ void __launch_bounds__(kExThreads) k_ex_cells(const double* __restrict__ v, WalkGrid g,
                                                         double* __restrict__ out) {
  __shared__ double red[kExThreads / 32][3 * kExRows];
  __shared__ __align__(16) uint64_t stab[256];
  for (int r = threadIdx.x; r < 256; r += blockDim.x) stab[r] = g_exp_tab[r];
  UCP_SYNC();
  const ucp_exp_entry* stab2 = reinterpret_cast<const ucp_exp_entry*>(stab);
  const double sc = g.ex_s0 + (double)blockIdx.x * g.ex_dlt;
  const double reach = kGaussCut + 0.5 * g.ex_dlt;
  long long jlo = (long long)ceil(((sc - reach) - g.a) / g.h);
  long long jhi = (long long)floor(((sc + reach) - g.a) / g.h);
  if (jlo < 0) jlo = 0;
  if (jhi > g.d - 1) jhi = g.d - 1;
  double A[kExRows][3];
#pragma unroll
  for (int n = 0; n < kExRows; ++n) A[n][0] = A[n][1] = A[n][2] = 0.0;
  const double INV = inv_sqrt_2pi();
  // a thread's nodes are kExThreads apart (D = kExThreads h): pdf(t + D) =
  // pdf(t) r, r(t + D) = r(t) exp(-D^2), re-anchored with fresh exps every
  // kExAnchor nodes (the recurrence's rounding then stays ~kExAnchor^2 ulp)
  constexpr int kExAnchor = 16;
  const double D = (double)kExThreads * g.h;
  const double qD = ucp_exp_core(-(D * D), stab2);
  double pdf = 0.0, ratio = 0.0;
  int it = 0;
  for (long long j = jlo + threadIdx.x; j <= jhi; j += kExThreads, ++it) {
    const double t = (g.a + (double)j * g.h) - sc;
    if ((it & (kExAnchor - 1)) == 0) {
      pdf = ucp_exp_core((-0.5 * t) * t, stab2) * INV;
      ratio = ucp_exp_core(-t * D - 0.5 * D * D, stab2);
    }
    const double W = (j == 0 || j == g.d - 1) ? 0.5 * g.h : g.h;
    const double vj = __ldg(v + j), v2 = vj * vj;
    double c = pdf * W;
    pdf *= ratio;
    ratio *= qD;
#pragma unroll
    for (int n = 0; n < kExRows; ++n) {
      A[n][0] += c;
      A[n][1] = __fma_rn(c, vj, A[n][1]);
      A[n][2] = __fma_rn(c, v2, A[n][2]);
      c *= t;
    }
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int n = 0; n < kExRows; ++n)
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      double x = A[n][k];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
      if (lane == 0) red[wid][3 * n + k] = x;
    }
  UCP_SYNC();
  if (threadIdx.x < 3 * kExRows) {
    double x = 0.0;
    for (int w = 0; w < kExThreads / 32; ++w) x += red[w][threadIdx.x];
    out[(int64_t)blockIdx.x * (3 * kExRows) + threadIdx.x] = x;
  }
}

// marginal_cost_segmented m=0 over a flat candidate list; the segment of
// candidate c is found by binary search in `offsets` (segments are short).
template <int kMode>
__global__ void __launch_bounds__(kWalkThreads, kMode ? 1 : kWalkMinBlocks) k_stage0_segmented(const double* __restrict__ u_flat, const int64_t* __restrict__ offsets,
                                   int64_t nseg, const double* __restrict__ y_seg,
                                   const double* __restrict__ f0_seg, double k,
                                   const double* __restrict__ v1, WalkGrid g, double* out) {
  pdl_wait();
  pdl_trigger();
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t n = offsets[nseg];
  UCP_WALK_STAGE(v1, g.d);
  if (c >= n) return;
  int64_t lo = 0, hi = nseg;  // find s with offsets[s] <= c < offsets[s+1]
  while (hi - lo > 1) {
    int64_t mid = (lo + hi) >> 1;
    if (offsets[mid] <= c) lo = mid; else hi = mid;
  }
  out[c] = stage0_cost<kMode>(u_flat[c], y_seg[lo], f0_seg[lo], k, v1, g);
}

// Local update, stage 0, part 1 (problem.py:95-97): the three FD probes
// u+h, u, u-h of every point.  probe-major layout so a warp walks adjacent
// centres (coalesced v1 reads).
template <int kMode, bool kBatch = false>
__global__ void __launch_bounds__(kWalkThreads, kMode ? 1 : kWalkMinBlocks) k_lu0_probe(const double* __restrict__ y0, const double* __restrict__ f0,
                            const double* __restrict__ u0, double k, const double* __restrict__ v1,
                            WalkGrid g, double fd_step, int64_t begin, int64_t n, double* cost3, const BatchArgs B) {
  pdl_wait();
  pdl_trigger();
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (kBatch) {
    const int b = B.inst(blockIdx.y);
    f0 += b * B.su0;
    u0 += b * B.su0;
    v1 += b * B.su1;
    k = B.kvec[b];
    cost3 += blockIdx.y * B.sslot;    if (g.vsuf) g.vsuf += (int64_t)blockIdx.y * g.vstride;  // this slot's tail-exit table
  }
  UCP_WALK_STAGE(v1, g.d);
  if (t >= 3 * n) return;
  int p = (int)(t / n);
  int64_t i = begin + (t - (int64_t)p * n);
  double u = u0[i];
  double hh = fd_step * (1.0 + fabs(u));  // solver.py:192
  double uu = p == 0 ? u + hh : (p == 1 ? u : u - hh);
  cost3[t] = stage0_cost<kMode>(uu, y0[i], f0[i], k, v1, g);
}

// Newton-or-gradient step shared by both stages (solver.py:130-149).
__device__ __forceinline__ double newton_step(double u, double c1, double c2,
                                              const ucp_local_params lp) {
  if (c2 > lp.curvature_min) {
    double quot = c1 / c2;
    quot = quot < -lp.newton_cap ? -lp.newton_cap : quot;  // np.clip
    quot = quot > lp.newton_cap ? lp.newton_cap : quot;
    return u - quot;
  }
  return u - lp.grad_step * c1;
}

// Local update, stage 0, part 2: derivatives (problem.py:99-101), step,
// cost_new and the monotone guard (solver.py:193-203).  cost_old is the
// bitwise-identical `mid` probe.
template <int kMode, bool kBatch = false>
__global__ void __launch_bounds__(kWalkThreads, kMode ? 1 : kWalkMinBlocks) k_lu0_finish(const double* __restrict__ y0, const double* __restrict__ f0,
                             const double* __restrict__ u0, double k, const double* __restrict__ v1,
                             WalkGrid g, ucp_local_params lp, int64_t begin, int64_t n,
                             const double* __restrict__ cost3, double* out, int64_t* err, const BatchArgs B) {
  pdl_wait();
  pdl_trigger();
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (kBatch) {
    const int b = B.inst(blockIdx.y);
    f0 += b * B.su0;
    u0 += b * B.su0;
    v1 += b * B.su1;
    k = B.kvec[b];
    cost3 += blockIdx.y * B.sslot;
    out += blockIdx.y * n;
    err += b * B.serr;    if (g.vsuf) g.vsuf += (int64_t)blockIdx.y * g.vstride;  // this slot's tail-exit table
  }
  UCP_WALK_STAGE(v1, g.d);
  if (t >= n) return;
  int64_t i = begin + t;
  double u = u0[i];
  double hh = lp.fd_step * (1.0 + fabs(u));
  double up = cost3[t], mid = cost3[n + t], dn = cost3[2 * n + t];
  double c1 = (up - dn) / (2.0 * hh);
  double c2 = ((up - 2.0 * mid) + dn) / (hh * hh);
  if (!(finite(c1) && finite(c2))) {
    flag_min(err, i);
    out[i] = u;
    return;
  }
  double stepped = newton_step(u, c1, c2, lp);  // project() is the identity
  double cost_new = stage0_cost<kMode>(stepped, y0[i], f0[i], k, v1, g);
  if (!(finite(mid) && finite(cost_new))) flag_min(err + 1, i);
  double r = cost_new <= mid ? stepped : u;
  if (!finite(r)) flag_min(err + 2, i);
  out[i] = r;
}

// Objective integrand (problem.py:116-127): c_i = C0(u0_i, y0_i).
template <int kMode, bool kBatch = false>
__global__ void __launch_bounds__(kWalkThreads, kMode ? 1 : kWalkMinBlocks) k_obj_terms(const double* __restrict__ y0, const double* __restrict__ f0,
                            const double* __restrict__ u0, double k, const double* __restrict__ v1,
                            WalkGrid g, int64_t begin, int64_t end, double* terms, int64_t* err,
                            const BatchArgs B) {
  pdl_wait();
  pdl_trigger();
  int64_t i = begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (kBatch) {
    const int b = B.inst(blockIdx.y);
    f0 += b * B.su0;
    u0 += b * B.su0;
    v1 += b * B.su1;
    k = B.kvec[b];
    terms += blockIdx.y * B.sslot;
    err += b * B.serr;    if (g.vsuf) g.vsuf += (int64_t)blockIdx.y * g.vstride;  // this slot's tail-exit table
  }
  UCP_WALK_STAGE(v1, g.d);
  if (i >= end) return;
  double c = stage0_cost<kMode>(u0[i], y0[i], f0[i], k, v1, g);
  if (!finite(c)) flag_min(err, i);
  terms[i] = c;
}

// kernels.py:136-144: serial ascending trapezoid.  The sum is one dependent
// add chain by definition, so the kernel's job is to keep that chain fed: a
// loader warp streams 2048-value chunks into a shared-memory double buffer
// (and finds the first non-finite value) while lane 0 of the adder warp adds
// in index order with the next 8 values already in registers.  Named
// barriers FULL (loader arrives, adder waits) / EMPTY (the reverse).  64
// threads per instance (batched engine: one CTA per slot).
__device__ __forceinline__ void named_sync(int id, int count);
__device__ __forceinline__ void named_arrive(int id, int count);
constexpr int kTrapThreads = 64;
__global__ void __launch_bounds__(kTrapThreads) k_trapezoid(const double* __restrict__ x, int64_t n, double spacing,
                                                           double* out, int64_t* err, const BatchArgs B) {
  constexpr int kChunk = 2048;
  constexpr int kFull = 1, kEmpty = 3;
  if (B.ids) {  // one CTA per slot; J and the error slot per instance
    const int b = B.inst(blockIdx.x);
    x += blockIdx.x * B.sslot;
    out += b;
    if (err) err += b * B.serr;
  }
  __shared__ __align__(16) double buf[2][kChunk];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nchunks = (n + kChunk - 1) / kChunk;
  if (warp == 1) {
    // ---- loader
    int64_t bad = UCP_NO_ERROR;
    for (int64_t c = 0; c < nchunks; ++c) {
      const int sb = (int)(c & 1);
      if (c >= 2) named_sync(kEmpty + sb, kTrapThreads);  // the adder is done with chunk c - 2
      const int64_t base = c * kChunk;
      const int cnt = (int)(n - base < kChunk ? n - base : kChunk);
      for (int r = lane; r < cnt; r += 32) {
        const double xv = x[base + r];
        buf[sb][r] = xv;
        if (!isfinite(xv) && base + r < bad) bad = base + r;
      }
      named_arrive(kFull + sb, kTrapThreads);
    }
    for (int64_t c = nchunks - 2 > 0 ? nchunks - 2 : 0; c < nchunks; ++c)  // the adder's last EMPTY arrivals
      named_sync(kEmpty + (int)(c & 1), kTrapThreads);
    for (int off = 16; off > 0; off >>= 1) {
      long long o = __shfl_down_sync(0xffffffffu, (long long)bad, off);
      bad = o < bad ? o : bad;
    }
    if (lane == 0 && err && bad != UCP_NO_ERROR) flag_min(err, bad);
    return;
  }
  // ---- adder (lane 0; the warp keeps the barrier protocol)
  double acc = 0.0;
  for (int64_t c = 0; c < nchunks; ++c) {
    const int sb = (int)(c & 1);
    named_sync(kFull + sb, kTrapThreads);
    if (lane == 0) {
      const double* bs = buf[sb];
      const int64_t base = c * kChunk;
      const int cnt = (int)(n - base < kChunk ? n - base : kChunk);
      int r = 0;
      if (base == 0) {
        acc = 0.5 * bs[0];
        r = 1;
      }
      const int stop = base + cnt == n ? cnt - 1 : cnt;  // index n-1 gets the half weight
      if (r + 8 <= stop) {
        double p0 = bs[r], p1 = bs[r + 1], p2 = bs[r + 2], p3 = bs[r + 3];
        double p4 = bs[r + 4], p5 = bs[r + 5], p6 = bs[r + 6], p7 = bs[r + 7];
        for (; r + 16 <= stop; r += 8) {
          const double q0 = bs[r + 8], q1 = bs[r + 9], q2 = bs[r + 10], q3 = bs[r + 11];
          const double q4 = bs[r + 12], q5 = bs[r + 13], q6 = bs[r + 14], q7 = bs[r + 15];
          acc += p0; acc += p1; acc += p2; acc += p3;
          acc += p4; acc += p5; acc += p6; acc += p7;
          p0 = q0; p1 = q1; p2 = q2; p3 = q3; p4 = q4; p5 = q5; p6 = q6; p7 = q7;
        }
        acc += p0; acc += p1; acc += p2; acc += p3;
        acc += p4; acc += p5; acc += p6; acc += p7;
        r += 8;
      }
      for (; r < stop; ++r) acc += bs[r];
      if (base + cnt == n && n > 1) acc += 0.5 * bs[cnt - 1];
    }
    named_arrive(kEmpty + sb, kTrapThreads);
  }
  if (lane == 0) *out = n == 1 ? 0.0 : acc * spacing;
}

// ---- The same serial sum, bitwise, in parallel (large n; problem.py:110-127
// via kernels.py:136-144: acc = x0/2; acc += x_i, i = 1..n-2; acc += x_(n-1)/2).
// While the running sum S stays inside one binade [2^(E+52), 2^(E+53)) (or its
// negative), every S is a multiple of u = 2^E and fl(S + a) = S + u * rnd(a/u)
// exactly: with a/u = k + f (k = floor, 0 <= f < 1) the increment is k, k + 1
// for f > 1/2, and for the tie f = 1/2 the even one of N + k, N + k + 1
// (N = S/u) -- only ties depend on the state, through N's parity.  So a chunk
// of kTzL addends reduces, for each parity of N at its start, to an exact
// integer increment, the output parity and the min/max running increment
// (k_tz_decompose, one thread per chunk, E proposed by an approximate prefix:
// k_tz_chunks + k_tz_plan).  One warp then walks the chunks in order
// (k_tz_final): a chunk whose exact start has exponent E and whose running N
// stays inside [2^52 + 1, 2^53 - 1] in magnitude (so every exact intermediate
// sum is inside the binade and rounds on u's grid) is applied as N += inc;
// any other chunk (binade crossings, zero or non-finite sums, huge addends,
// E guessed wrong) is added serially in order.  Either way every addition is
// the reference's, so the result is bitwise the serial kernel's.
constexpr int kTzL = 1024;           // addends per chunk
constexpr int64_t kTzMinN = 32768;   // below: the serial kernel
// per-(device, stream) grow-only scratch of the chunked trapezoid (calls on
// one stream are ordered; cudaFree of an outgrown buffer synchronises)
int tz_scratch(cudaStream_t st, size_t bytes, void** out) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, std::pair<void*, size_t>> bufs;
  int dev = 0;
  UCP_CHECK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  auto& b = bufs[{dev, st}];
  if (b.second < bytes) {
    if (b.first) UCP_CHECK(cudaFree(b.first));
    b.first = nullptr;
    b.second = 0;
    UCP_CHECK(cudaMalloc(&b.first, bytes));
    b.second = bytes;
  }
  *out = b.first;
  return UCP_OK;
}
int tz_parallel() {  // UCP_TZ_PARALLEL=0: always the serial kernel (A/B)
  static const int k = [] {
    const char* e = getenv("UCP_TZ_PARALLEL");
    return e ? atoi(e) : 1;
  }();
  return k;
}
struct TzRec {
  long long inc[2], mn[2], mx[2];  // per start parity: increment, min / max running increment
  int e, flags;                    // flags: bit 0 usable, bit 1 / 2 output parity for start parity 0 / 1
};
__device__ __forceinline__ int64_t tz_lo(int64_t c) { return 1 + c * kTzL; }  // first addend of chunk c
__device__ __forceinline__ double tz_addend(const double* x, int64_t n, int64_t i) {
  return i == n - 1 ? 0.5 * x[n - 1] : x[i];
}
// K1: one warp per chunk: approximate chunk sum; first non-finite sample -> err
__global__ void k_tz_chunks(const double* __restrict__ x, int64_t n, int64_t nch, double* csum, int64_t* err) {
  const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (c >= nch) return;
  const int64_t lo = tz_lo(c), hi = lo + kTzL < n ? lo + kTzL : n;  // addends [lo, hi), hi <= n
  double acc = 0.0;
  long long bad = UCP_NO_ERROR;
  if (c == 0 && lane == 0 && !isfinite(x[0])) bad = 0;
  for (int64_t i = lo + lane; i < hi; i += 32) {
    const double xv = x[i];
    if (!isfinite(xv) && i < bad) bad = i;
    acc += i == n - 1 ? 0.5 * xv : xv;
  }
  for (int o = 16; o > 0; o >>= 1) {
    acc += __shfl_down_sync(0xffffffffu, acc, o);
    const long long ob = __shfl_down_sync(0xffffffffu, bad, o);
    bad = ob < bad ? ob : bad;
  }
  if (lane == 0) {
    csum[c] = acc;
    if (err && bad != UCP_NO_ERROR) flag_min(err, bad);
  }
}
// K2: one CTA: approximate running sum at each chunk start -> proposed exponent
__global__ void __launch_bounds__(1024) k_tz_plan(const double* __restrict__ x, const double* __restrict__ csum,
                                                  int64_t nch, TzRec* rec) {
  __shared__ double sc[1024];
  __shared__ double carry;
  if (threadIdx.x == 0) carry = 0.5 * x[0];
  UCP_SYNC();
  for (int64_t b = 0; b < nch; b += 1024) {
    const int64_t c = b + threadIdx.x;
    const double v = c < nch ? csum[c] : 0.0;
    sc[threadIdx.x] = v;
    UCP_SYNC();
    for (int o = 1; o < 1024; o <<= 1) {  // inclusive Hillis-Steele scan (approximate: E is only a proposal)
      const double add = threadIdx.x >= o ? sc[threadIdx.x - o] : 0.0;
      UCP_SYNC();
      sc[threadIdx.x] += add;
      UCP_SYNC();
    }
    const double start = carry + (sc[threadIdx.x] - v);
    if (c < nch) {
      int e = INT_MIN;
      if (isfinite(start) && start != 0.0) {
        const int lg = ilogb(start);
        if (lg >= -960 && lg <= 1000) e = lg - 52;
      }
      rec[c].e = e;
    }
    UCP_SYNC();
    if (threadIdx.x == 1023) carry = carry + sc[1023];
    UCP_SYNC();
  }
}
// K3: one thread per chunk: the exact integer form for both start parities
__global__ void k_tz_decompose(const double* __restrict__ x, int64_t n, int64_t nch, TzRec* rec) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nch) return;
  const int e = rec[c].e;
  int flags = 0;
  long long inc[2] = {0, 0}, mn[2] = {0, 0}, mx[2] = {0, 0};
  int par[2] = {0, 1};
  if (e != INT_MIN) {
    flags = 1;
    const int64_t lo = tz_lo(c), hi = lo + kTzL < n ? lo + kTzL : n;
    for (int64_t i = lo; i < hi; ++i) {
      const double q = ldexp(tz_addend(x, n, i), -e);  // exact: |a| >= 2^-1074 and e >= -1012
      // a non-finite addend, or one (or a running increment) that leaves the
      // binade by itself: serial (also keeps the int64 sums far from overflow)
      if (!(fabs(q) < 0x1p54) || inc[0] > (1LL << 55) || inc[0] < -(1LL << 55)) {
        flags = 0;
        break;
      }
      // q = k + f, k = floor(q), classified from |q| = K + F (F = |q| - K is
      // exact for |q| >= 0; 1 - F for q < 0 need not be): up = f > 1/2, tie = f == 1/2
      const double r = fabs(q), K = floor(r), F = r - K;
      long long k;
      bool up, tie;
      if (q >= 0.0) {
        k = (long long)K;
        up = F > 0.5;
        tie = F == 0.5;
      } else if (F == 0.0) {
        k = -(long long)K;
        up = tie = false;
      } else {
        k = -(long long)K - 1;
        up = F < 0.5;
        tie = F == 0.5;
      }
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const long long d = k + (up ? 1 : (tie ? (long long)((par[p] + (int)(k & 1)) & 1) : 0));
        inc[p] += d;
        par[p] = (int)((par[p] + (int)(d & 1)) & 1);
        mn[p] = inc[p] < mn[p] ? inc[p] : mn[p];
        mx[p] = inc[p] > mx[p] ? inc[p] : mx[p];
      }
    }
  }
  TzRec r;
  r.e = e;
  r.flags = flags | (par[0] << 1) | (par[1] << 2);
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    r.inc[p] = inc[p];
    r.mn[p] = mn[p];
    r.mx[p] = mx[p];
  }
  rec[c] = r;
}
// K4: one warp walks the chunks in order (lane 0 holds the exact sum)
constexpr int kTzBatch = 128;  // records staged per smem batch
__global__ void __launch_bounds__(32) k_tz_final(const double* __restrict__ x, int64_t n, int64_t nch,
                                                 const TzRec* __restrict__ rec, double spacing, double* out) {
  __shared__ TzRec srec[kTzBatch];
  __shared__ double sx[kTzL];
  const int lane = threadIdx.x;
  double S = 0.5 * x[0];
  const long long lo52 = (1LL << 52) + 1, hi53 = (1LL << 53) - 1;
  for (int64_t b = 0; b < nch; b += kTzBatch) {
    const int nb = (int)(nch - b < kTzBatch ? nch - b : kTzBatch);
    __syncwarp();
    for (int r = lane; r < nb; r += 32) srec[r] = rec[b + r];
    __syncwarp();
    for (int r = 0; r < nb; ++r) {
      const int64_t c = b + r;
      int fast = 0;
      if (lane == 0) {
        const TzRec& R = srec[r];
        if ((R.flags & 1) && isfinite(S) && S != 0.0 && ilogb(S) - 52 == R.e) {
          const long long N = (long long)ldexp(S, -R.e);  // |N| in [2^52, 2^53): exact
          const int p = (int)(N & 1);
          const long long lo = N + R.mn[p], hi = N + R.mx[p];
          const bool ok = N > 0 ? (lo >= lo52 && hi <= hi53) : (hi <= -lo52 && lo >= -hi53);
          if (ok) {
            S = ldexp((double)(N + R.inc[p]), R.e);
            fast = 1;
          }
        }
      }
      fast = __shfl_sync(0xffffffffu, fast, 0);
      if (fast) continue;
      // serial chunk: the warp stages the addends, lane 0 adds them in order
      const int64_t lo = tz_lo(c), hi = lo + kTzL < n ? lo + kTzL : n;
      for (int64_t i = lo + lane; i < hi; i += 32) sx[i - lo] = x[i];
      __syncwarp();
      if (lane == 0) {
        const int cnt = (int)(hi - lo);
        const int stop = hi == n ? cnt - 1 : cnt;
        for (int t = 0; t < stop; ++t) S += sx[t];
        if (hi == n) S += 0.5 * sx[cnt - 1];
      }
      __syncwarp();
    }
  }
  if (lane == 0) *out = S * spacing;
}

__global__ void k_segmented_argmin(const double* __restrict__ costs, const int64_t* __restrict__ offsets,
                                   int64_t nseg, int64_t* out) {
  int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nseg) return;
  int64_t lo = offsets[s], hi = offsets[s + 1];
  int64_t best = lo;
  double bv = costs[lo];
  for (int64_t t = lo + 1; t < hi; ++t) {
    double c = costs[t];
    if (c < bv) {
      bv = c;
      best = t;
    }
  }
  out[s] = best;
}

// kernels.flatten_windows, numba variant (kernels.py:163-187): the window
// values[lo[i]..hi[i]] of point i in order, a value dropped when an earlier
// value of the same window equals it (NaN never equals: always kept).  One
// thread per point; counts (kFill = false) then a scan, then the fill.
template <bool kFill>
__global__ void k_flatten_windows(const double* __restrict__ values, const int64_t* __restrict__ lo,
                                  const int64_t* __restrict__ hi, int64_t n, int64_t* counts,
                                  const int64_t* __restrict__ offsets, double* flat) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t l = lo[i], r = hi[i];
  int64_t pos = kFill ? offsets[i] : 0;
  for (int64_t j = l; j <= r; ++j) {
    const double v = values[j];
    bool dup = false;
    for (int64_t t = l; t < j && !dup; ++t) dup = values[t] == v;
    if (!dup) {
      if (kFill) flat[pos] = v;
      ++pos;
    }
  }
  if (!kFill) counts[i] = pos;
  UCP_DCHECK(!kFill || pos == offsets[i + 1]);
}

// ---- exhaustion, stage 0 (solver.py:206-223) -------------------------------
// Candidates of point i: the snapshot values in its window with adjacent
// repeats collapsed (identical values give identical costs, and the
// first-occurrence argmin returns the same value -- the reference's own
// flatten_windows dedups, kernels.py:163-187).
// Range-max table of |v| over 256-node blocks for walk_tail_noop: one CTA
// (~8 B/node read once plus log2(nb) passes over nb blocks; negligible beside
// the walks that use it).  Level 0: block maxima; level k: max over 2^k blocks.
// A non-finite v makes every entry covering it +inf (the walk never exits there).
__global__ void __launch_bounds__(1024) k_vsuf(const double* __restrict__ v, int64_t d, int nb, double* t,
                                                const int32_t* __restrict__ ids, int64_t su1, int64_t tstride) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (ids) {  // batched engine: CTA s builds slot s's table from instance ids[s]'s v
    v += (int64_t)ids[blockIdx.x] * su1;
    t += (int64_t)blockIdx.x * tstride;
  }
  for (int b = warp; b < nb; b += 32) {
    double m = 0.0;
    for (int64_t j = ((int64_t)b << kVsufShift) + lane; j < d && j < ((int64_t)(b + 1) << kVsufShift); j += 32) {
      double a = fabs(v[j]);
      m = (a <= 1.7976931348623157e308) ? fmax(m, a) : INFINITY;  // NaN / inf -> inf
    }
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) t[b] = m;
  }
  for (int k = 1; (1 << k) <= nb; ++k) {
    UCP_SYNC();
    const double* p = t + (size_t)(k - 1) * nb;
    double* q = t + (size_t)k * nb;
    const int half = 1 << (k - 1);
    for (int b = threadIdx.x; b + 2 * half <= nb; b += blockDim.x) q[b] = fmax(p[b], p[b + half]);
  }
}

int vsuf_levels(int nb) {
  int k = 0;
  while ((2 << k) <= nb) ++k;
  return k + 1;
}

__global__ void k_ex_count(const double* __restrict__ u, const int64_t* __restrict__ lo,
                           const int64_t* __restrict__ hi, int64_t begin, int64_t n, int64_t* counts) {
  pdl_wait();
  pdl_trigger();
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  int64_t i = begin + t;
  int64_t c = 1;
  double prev = u[lo[i]];
  for (int64_t j = lo[i] + 1; j <= hi[i]; ++j) {
    double x = u[j];
    c += (x != prev);
    prev = x;
  }
  counts[t] = c;
}

__global__ void k_ex_fill(const double* __restrict__ u, const int64_t* __restrict__ lo,
                          const int64_t* __restrict__ hi, int64_t begin, int64_t n,
                          const int64_t* __restrict__ offs, int32_t* cand_pt, int32_t* cand_j) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  int64_t i = begin + t;
  int64_t pos = offs[t];
  int64_t j0 = lo[i];
  UCP_DCHECK(j0 >= 0 && j0 <= hi[i] && offs[t + 1] - pos >= 1);
  double prev = u[j0];
  cand_pt[pos] = (int32_t)i;
  cand_j[pos] = (int32_t)j0;
  ++pos;
  for (int64_t j = j0 + 1; j <= hi[i]; ++j) {
    double x = u[j];
    if (x != prev) {
      cand_pt[pos] = (int32_t)i;
      cand_j[pos] = (int32_t)j;
      ++pos;
    }
    prev = x;
  }
  UCP_DCHECK(pos == offs[t + 1]);
}

// Warp-per-point form of k_ex_fill (same candidates, same order): lane l of
// a 32-node chunk keeps node j when j == lo or u[j] != u[j-1]; ballot +
// popc ranks the kept nodes.  Used when the windows are short enough that a
// lone thread's serial fill is latency-bound (small grids).
__global__ void k_ex_fill_warp(const double* __restrict__ u, const int64_t* __restrict__ lo,
                               const int64_t* __restrict__ hi, int64_t begin, int64_t n,
                               const int64_t* __restrict__ offs, int32_t* cand_pt, int32_t* cand_j) {
  pdl_wait();
  pdl_trigger();
  const int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= n) return;  // warp-uniform
  const int64_t i = begin + t;
  const int64_t j0 = lo[i], j1 = hi[i];
  int64_t pos = offs[t];
  for (int64_t c = j0; c <= j1; c += 32) {
    const int64_t j = c + lane;
    const bool valid = j <= j1;
    const bool keep = valid && (j == j0 || u[j] != u[j - 1]);
    const unsigned mask = __ballot_sync(0xffffffffu, keep);
    if (keep) {
      const int64_t at = pos + __popc(mask & ((1u << lane) - 1u));
      cand_pt[at] = (int32_t)i;
      cand_j[at] = (int32_t)j;
    }
    pos += __popc(mask);
  }
  UCP_DCHECK(pos == offs[t + 1]);
}

template <int kMode, bool kBatch = false>
__global__ void __launch_bounds__(kWalkThreads, kMode ? 1 : kWalkMinBlocks) k_ex0_eval(const double* __restrict__ y0, const double* __restrict__ f0,
                           const double* __restrict__ u0, double k, const double* __restrict__ v1,
                           WalkGrid g, const int64_t* __restrict__ total,
                           const int32_t* __restrict__ cand_pt, const int32_t* __restrict__ cand_j,
                           double* costs, const BatchArgs B) {
  pdl_wait();
  pdl_trigger();
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (kBatch) {  // per-slot candidate lists of capacity sslot; totals[slot]
    const int b = B.inst(blockIdx.y);
    total += blockIdx.y;
    if ((int64_t)blockIdx.x * blockDim.x >= *total) return;  // whole CTA idle: skip the staging
    f0 += b * B.su0;
    u0 += b * B.su0;
    v1 += b * B.su1;
    k = B.kvec[b];
    cand_pt += blockIdx.y * B.sslot;
    cand_j += blockIdx.y * B.sslot;
    costs += blockIdx.y * B.sslot;    if (g.vsuf) g.vsuf += (int64_t)blockIdx.y * g.vstride;  // this slot's tail-exit table
  }
  UCP_WALK_STAGE(v1, g.d);
  if (c >= *total) return;
  int32_t i = cand_pt[c];
  costs[c] = stage0_cost<kMode>(u0[cand_j[c]], y0[i], f0[i], k, v1, g);
}

// First strict minimum per point (kernels.py:147-160), kept in registers;
// any non-finite candidate cost flags the point (solver.py:216-221).
__global__ void k_ex_argmin(const double* __restrict__ u, const double* __restrict__ costs,
                            const int64_t* __restrict__ offs, const int32_t* __restrict__ cand_j,
                            int64_t begin, int64_t n, double* out, int64_t* err, const BatchArgs B,
                            int64_t soffs) {
  pdl_wait();
  pdl_trigger();
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  if (B.ids) {
    const int b = B.inst(blockIdx.y);
    u += b * B.su0;
    costs += blockIdx.y * B.sslot;
    cand_j += blockIdx.y * B.sslot;
    offs += blockIdx.y * soffs;
    out += blockIdx.y * n;
    err += b * B.serr;
  }
  int64_t lo = offs[t], hi = offs[t + 1];
  UCP_DCHECK(hi > lo);
  int64_t best = lo;
  double bv = costs[lo];
  bool ok = finite(bv);
  for (int64_t c = lo + 1; c < hi; ++c) {
    double x = costs[c];
    ok = ok && finite(x);
    if (x < bv) {
      bv = x;
      best = c;
    }
  }
  if (!ok) flag_min(err, begin + t);
  out[begin + t] = u[cand_j[best]];
}

// ---- stage 1: the u1 estimator moments (kernels.py:447-486) ----------------
constexpr int kTile = 256;  // support points per shared-memory tile

// Per support point: x1 = y0 + u0 (witsenhausen.py:72), the two edge-tail
// weights the first/last query need (kernels.py:477-480, hoisted out of the
// serial loop: same operands, same bits), and per-tile min/max of x1 for
// tile skipping (a tile holding a NaN is never skipped: NaN contributes to
// the tail-weighted edge queries).
__global__ void k_x1_prepare(const double* __restrict__ y0, const double* __restrict__ u0,
                             const double* __restrict__ w, int64_t d0, double a, double h, double b, double* x1,
                             double2* xw, double2* tails, double2* tile_mm, const BatchArgs B) {
  __shared__ double smin[kTile], smax[kTile];
  pdl_wait();
  pdl_trigger();
  if (B.ids) {
    const int inst = B.inst(blockIdx.y);
    const int64_t ntiles = (d0 + kTile - 1) / kTile;
    u0 += inst * B.su0;
    w += inst * B.su0;
    x1 += blockIdx.y * d0;
    tails += blockIdx.y * d0;
    xw += blockIdx.y * ntiles * kTile;
    tile_mm += blockIdx.y * ntiles;
  }
  __shared__ int snan;
  if (threadIdx.x == 0) snan = 0;
  UCP_SYNC();
  int64_t i = (int64_t)blockIdx.x * kTile + threadIdx.x;
  double x = 0.0, mn = INFINITY, mx = -INFINITY;
  if (i < d0) {
    x = y0 ? y0[i] + u0[i] : u0[i];
    x1[i] = x;
    tails[i] = make_double2(phi_cdf(a - x) / h, phi_cdf(x - b) / h);
    xw[i] = make_double2(x, w[i]);
    if (isnan(x)) snan = 1;
    else mn = mx = x;
  } else {
    xw[i] = make_double2(INFINITY, 0.0);  // tile padding: out of range for every query
  }
  smin[threadIdx.x] = mn;
  smax[threadIdx.x] = mx;
  UCP_SYNC();
  for (int s = kTile / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      smin[threadIdx.x] = fmin(smin[threadIdx.x], smin[threadIdx.x + s]);
      smax[threadIdx.x] = fmax(smax[threadIdx.x], smax[threadIdx.x + s]);
    }
    UCP_SYNC();
  }
  if (threadIdx.x == 0)
    tile_mm[blockIdx.x] = snan ? make_double2(-INFINITY, INFINITY) : make_double2(smin[0], smax[0]);
}

// ---- bulk async copy (TMA engine, cp.async.bulk) + mbarrier helpers ------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "UCP_MBAR_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra UCP_MBAR_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
  UCP_JITTER();  // a late reader: the refill of the other buffer must not overtake it
}
// global -> shared bulk copy completing on `bar` (bytes % 16 == 0, 16-B aligned)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  UCP_JITTER();
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// One thread per query y; the CTA streams (x_i, w_i) tiles through shared
// memory in ascending i (the reference's summation order) and skips whole
// tiles that contribute exactly nothing to any query of the CTA:
//  - Gaussian term: every |y - x| > GAUSS_CUT (fl(y - x) is monotone in both
//    arguments, so the tile min/max decide it);
//  - edge tails (only CTAs holding the first/last grid node): phi_cdf(a - x)
//    and phi_cdf(x - b) are exactly 0 once a - x <= -12 / x - b <= -12.
//
// Interior CTAs take the fast path: four pairs per iteration, their exp()
// evaluated back to back (independent, ILP) with the branch-free main-path
// exp (bitwise glibc for |arg| < 512; out-of-range pairs compute garbage that
// is never accumulated), then accumulated strictly in order.  For interior
// queries `wp != 0` <=> |y - x| <= 12 (exp(-72) * INV > 0) and factor*e == e
// bitwise.  CTAs with an edge query run the general loop, a line-by-line
// restatement of kernels.py:466-482 with the tail weights precomputed.
//
// Persistent CTAs pull 128-query blocks from an atomic counter, the two edge
// blocks first (they visit the most tiles).
#ifndef UCP_MOM_QT
#define UCP_MOM_QT 128
#endif
constexpr int kMomThreads = UCP_MOM_QT;  // queries (threads) per work item
// kUnroll pairs' exp() in flight per thread; the batched engine (few CTAs per
// SM) instantiates a deeper unroll with a looser register bound.
#ifndef UCP_MOM_UNROLL
#define UCP_MOM_UNROLL 16
#endif
#ifndef UCP_MOM_MINB
#define UCP_MOM_MINB 2
#endif
template <int kMomUnroll = UCP_MOM_UNROLL, int kMinBlocks = UCP_MOM_MINB, int kQT = kMomThreads>
__global__ void __launch_bounds__(kQT, kMinBlocks)
k_moments(const double* __restrict__ yq, int64_t n, const double2* __restrict__ xw,
          const double2* __restrict__ tails, int64_t m, const double2* __restrict__ tile_mm, double a, double h,
          int64_t d, double* o0, double* o1, double* o2, int* work_counter, int64_t nslots, int64_t sout) {
  // interior CTAs: (x, w) tiles arrive by bulk async copy (TMA engine) into a
  // double buffer, the next non-skipped tile in flight while this one is used
  __shared__ __align__(128) double2 sbuf[2][kTile];
  __shared__ __align__(8) uint64_t sbar[2];
  __shared__ double2 slr[kTile];
  __shared__ __align__(16) uint64_t stab[256];
  __shared__ double s_ymin[kQT / 32], s_ymax[kQT / 32];
  __shared__ int s_left, s_right;
  __shared__ long long s_work;
  for (int r = threadIdx.x; r < 256; r += blockDim.x) stab[r] = g_exp_tab[r];
  const ucp_exp_entry* stab2 = reinterpret_cast<const ucp_exp_entry*>(stab);
  const int64_t nqb = (n + kQT - 1) / kQT;
  // work items: the edge query blocks of every slot first (they visit the most
  // tiles), then the interior blocks; one slot == the single-instance order
  const int64_t nedge = nqb == 1 ? 1 : 2;
  const int64_t nitems = nslots * nqb;
  const double b = a + h * (double)(d - 1);
  const double INV = inv_sqrt_2pi();
  const int64_t ntiles = (m + kTile - 1) / kTile;
  if (threadIdx.x == 0) {
    s_work = blockIdx.x;
    mbar_init(&sbar[0], 1);
    mbar_init(&sbar[1], 1);
    mbar_init_fence();
  }
  UCP_SYNC();
  uint32_t phase0 = 0, phase1 = 0;  // completions seen per barrier (parity), CTA-uniform
  const double2* xw0 = xw;
  const double2* tails0 = tails;
  const double2* tile_mm0 = tile_mm;
  double *o00 = o0, *o10 = o1, *o20 = o2;
  for (;;) {
    const int64_t k = s_work;
    if (k >= nitems) break;
    int64_t slot, qb;
    if (k < nslots * nedge) {
      slot = k / nedge;
      qb = (k % nedge) ? nqb - 1 : 0;
    } else {
      const int64_t r = k - nslots * nedge, per = nqb - nedge;
      slot = r / per;
      qb = 1 + r % per;
    }
    UCP_DCHECK(slot >= 0 && slot < nslots && qb >= 0 && qb < nqb);
    xw = xw0 + slot * ntiles * kTile;
    tails = tails0 + slot * m;
    tile_mm = tile_mm0 + slot * ntiles;
    o0 = o00 + slot * sout;
    o1 = o10 + slot * sout;
    o2 = o20 + slot * sout;
    if (threadIdx.x == 0) s_left = s_right = 0;
    const int64_t t = qb * kQT + threadIdx.x;
    const bool active = t < n;
    const double yt = active ? yq[t] : yq[n - 1];
    long long j = (long long)ceil((yt - a) / h - 0.5);
    if (j < 0) j = 0;
    if (j > d - 1) j = d - 1;
    const bool at_left = j == 0, at_right = j == d - 1;
    const double factor = (at_left || at_right) ? 0.5 : 1.0;
    double ymin = yt, ymax = yt;
    for (int off = 16; off > 0; off >>= 1) {
      ymin = fmin(ymin, __shfl_xor_sync(0xffffffffu, ymin, off));
      ymax = fmax(ymax, __shfl_xor_sync(0xffffffffu, ymax, off));
    }
    UCP_SYNC();
    if ((threadIdx.x & 31) == 0) {
      s_ymin[threadIdx.x >> 5] = ymin;
      s_ymax[threadIdx.x >> 5] = ymax;
    }
    if (at_left) atomicOr(&s_left, 1);
    if (at_right) atomicOr(&s_right, 1);
    UCP_SYNC();
    ymin = s_ymin[0];
    ymax = s_ymax[0];
    for (int r = 1; r < kQT / 32; ++r) {
      ymin = fmin(ymin, s_ymin[r]);
      ymax = fmax(ymax, s_ymax[r]);
    }
    const bool has_left = s_left != 0, has_right = s_right != 0;
    const bool general = has_left || has_right;
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
    // first tile >= t0 with a nonzero contribution to some query of the CTA
    auto next_tile = [&](int64_t t0) -> int64_t {
      for (int64_t tile = t0; tile < ntiles; ++tile) {
        const double2 mm = tile_mm[tile];
        const bool gauss_out = ymin - mm.y > kGaussCut || ymax - mm.x < -kGaussCut;
        const bool left_out = !has_left || a - mm.x <= -kGaussCut;
        const bool right_out = !has_right || mm.y - b <= -kGaussCut;
        if (!(gauss_out && left_out && right_out)) return tile;
      }
      return ntiles;
    };
    constexpr uint32_t kTileBytes = kTile * sizeof(double2);
    if (!general) {
      int64_t tile = next_tile(0);
      int cur = 0;
      if (threadIdx.x == 0 && tile < ntiles) {
        fence_proxy_async_smem();  // earlier generic reads of sbuf before the async refill
        mbar_arrive_expect_tx(&sbar[0], kTileBytes);
        bulk_g2s(sbuf[0], xw + tile * kTile, kTileBytes, &sbar[0]);
      }
      while (tile < ntiles) {
        const int64_t nxt = next_tile(tile + 1);
        UCP_DCHECK(nxt > tile && nxt <= ntiles);
        if (cur == 0) {
          mbar_wait(&sbar[0], phase0);
          phase0 ^= 1u;
        } else {
          mbar_wait(&sbar[1], phase1);
          phase1 ^= 1u;
        }
        if (threadIdx.x == 0 && nxt < ntiles) {
          // every thread finished reading sbuf[cur ^ 1] (barrier at the end of
          // the previous iteration); order those generic reads before the
          // async-proxy writes of the refill
          fence_proxy_async_smem();
          mbar_arrive_expect_tx(&sbar[cur ^ 1], kTileBytes);
          bulk_g2s(sbuf[cur ^ 1], xw + nxt * kTile, kTileBytes, &sbar[cur ^ 1]);
        }
        const double2* sxw = sbuf[cur];
        for (int r = 0; r < kTile; r += kMomUnroll) {  // padding is (+inf, 0): never accumulated
          double e[kMomUnroll];
          bool in[kMomUnroll];
#pragma unroll
          for (int q = 0; q < kMomUnroll; ++q) {
            const double diff = yt - sxw[r + q].x;
            in[q] = fabs(diff) <= kGaussCut;
            e[q] = ucp_exp_core((-0.5 * diff) * diff, stab2);
          }
#pragma unroll
          for (int q = 0; q < kMomUnroll; ++q) {
            if (in[q]) {
              const double2 xwq = sxw[r + q];
              const double wp = (e[q] * INV) * xwq.y;
              acc0 += wp;
              const double wx = wp * xwq.x;
              acc1 += wx;
              acc2 += wx * xwq.x;
            }
          }
        }
        UCP_SYNC();
        cur ^= 1;
        tile = nxt;
      }
    } else {
      double2* sxw = sbuf[0];
      for (int64_t tile = next_tile(0); tile < ntiles; tile = next_tile(tile + 1)) {
        const int64_t base = tile * kTile;
        const int cnt = (int)(m - base < kTile ? m - base : kTile);
        UCP_SYNC();
        for (int r = threadIdx.x; r < kTile; r += kQT) {
          sxw[r] = xw[base + r];
          slr[r] = r < cnt ? tails[base + r] : make_double2(0.0, 0.0);
        }
        UCP_SYNC();
        // kernels.py:466-482 in order; the exp() of kMomUnroll pairs is
        // evaluated ahead (independent) and used only where the reference
        // evaluates it.  Padding slots (x = +inf, tails 0) give wp == 0.
        for (int r0 = 0; r0 < kTile; r0 += kMomUnroll) {
          double e[kMomUnroll];
#pragma unroll
          for (int q = 0; q < kMomUnroll; ++q) {
            const double diff = yt - sxw[r0 + q].x;
            e[q] = ucp_exp_core((-0.5 * diff) * diff, stab2);
          }
#pragma unroll
          for (int q = 0; q < kMomUnroll; ++q) {
            const int r = r0 + q;
            const double xi = sxw[r].x;
            const double diff = yt - xi;
            double wp = 0.0;
            if (diff <= kGaussCut && diff >= -kGaussCut) wp = (factor * e[q]) * INV;
            if (at_left) wp += slr[r].x;   // phi_cdf(a - xi) / h
            if (at_right) wp += slr[r].y;  // phi_cdf(xi - b) / h
            if (wp != 0.0) {
              wp *= sxw[r].y;
              acc0 += wp;
              const double wx = wp * xi;
              acc1 += wx;
              acc2 += wx * xi;
            }
          }
        }
      }
      UCP_SYNC();
      fence_proxy_async_smem();  // generic writes to sbuf[0] before later bulk copies into it
    }
    if (active) {
      o0[t] = acc0;
      o1[t] = acc1;
      o2[t] = acc2;
    }
    UCP_SYNC();
    if (threadIdx.x == 0) {
      UCP_JITTER();
      s_work = gridDim.x + atomicAdd(work_counter, 1);
    }
    UCP_SYNC();
  }
}

// Small query sets (d ~ 2000 .. 16k): the direct kernel above would run too
// few CTAs, each query's serial pair loop pure latency.  Fused form: one CTA
// owns kFQ queries.  Producer warps compute the per-pair terms of one x1
// tile -- wp*w, (wp*w)*x, ((wp*w)*x)*x for live pairs (wp != 0), +0.0 for
// skipped ones (kernels.py:474-485; adding +0.0 to an accumulator that
// started at +0.0 never changes its bits) -- into a shared-memory stage while
// 3*kFQ consumer threads (one per query and accumulator) add the previous
// stage's terms serially in ascending support order.  Two stages, named
// barriers (FULL: producers arrive / consumers wait; EMPTY: the reverse).
// Tiles without a nonzero term for any query of the CTA are skipped by both
// roles (same test as k_moments).  Bitwise equal to the serial reference.
#ifndef UCP_FQ
#define UCP_FQ 8
#endif
#ifndef UCP_FPROD_WARPS
#define UCP_FPROD_WARPS 10
#endif
constexpr int kFQ = UCP_FQ;                  // queries per CTA
constexpr int kFConsWarps = (3 * kFQ + 31) / 32;  // one consumer thread per (query, accumulator)
constexpr int kFProdWarps = UCP_FPROD_WARPS;
constexpr int kFThreads = 32 * (kFConsWarps + kFProdWarps);
constexpr int kFProd = 32 * kFProdWarps;
static_assert(kFProd % kFQ == 0, "producer threads keep one query each");
constexpr size_t kFSmem = 2 * 3 * kTile * kFQ * sizeof(double);  // 96 KiB at kFQ = 8: two CTAs per SM

__device__ __forceinline__ void named_sync(int id, int count) {
  UCP_JITTER();
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int count) {
  UCP_JITTER();
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

__global__ void __launch_bounds__(kFThreads, kFQ <= 8 ? 2 : 1)
k_mom_fused(const double* __restrict__ yq, int64_t n, const double* __restrict__ x, const double* __restrict__ w,
            const double2* __restrict__ tails, const double2* __restrict__ tile_mm, int64_t m, double a, double h,
            int64_t d, double* o0, double* o1, double* o2, const int32_t* __restrict__ ids, int64_t su0,
            int64_t sout) {
  extern __shared__ __align__(16) double fbuf[];  // [2][3][kTile][kFQ]
  pdl_wait();
  pdl_trigger();
  if (ids) {  // batched engine: slot blockIdx.y runs instance ids[slot]
    const int64_t slot = blockIdx.y, nt = (m + kTile - 1) / kTile;
    x += slot * m;
    tails += slot * m;
    tile_mm += slot * nt;
    w += (int64_t)ids[slot] * su0;
    o0 += slot * sout;
    o1 += slot * sout;
    o2 += slot * sout;
  }
  __shared__ __align__(16) uint64_t stab[256];
  __shared__ double sx[kTile], sw[kTile];
  __shared__ double2 stl[kTile];
  __shared__ int s_left, s_right;
  __shared__ double s_ymin, s_ymax;
  const int tid = threadIdx.x;
  for (int r = tid; r < 256; r += blockDim.x) stab[r] = g_exp_tab[r];
  const ucp_exp_entry* stab2 = reinterpret_cast<const ucp_exp_entry*>(stab);
  const int64_t q0 = (int64_t)blockIdx.x * kFQ;
  const double b = a + h * (double)(d - 1);
  if (tid < 32) {  // the CTA's query range and edge flags (warp 0, one query per lane)
    const int64_t q = q0 + (tid % kFQ) < n ? q0 + (tid % kFQ) : n - 1;
    const double yt = yq[q];
    long long j = (long long)ceil((yt - a) / h - 0.5);
    if (j < 0) j = 0;
    if (j > d - 1) j = d - 1;
    const unsigned l = __ballot_sync(0xffffffffu, j == 0), rr = __ballot_sync(0xffffffffu, j == d - 1);
    double lo = yt, hi = yt;
    for (int off = 16; off > 0; off >>= 1) {
      lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, off));
      hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, off));
    }
    if (tid == 0) {
      s_left = l != 0;
      s_right = rr != 0;
      s_ymin = lo;
      s_ymax = hi;
    }
  }
  UCP_SYNC();
  const bool has_left = s_left != 0, has_right = s_right != 0;
  const double ymin = s_ymin, ymax = s_ymax;
  const int64_t ntiles = (m + kTile - 1) / kTile;
  auto live_tile = [&](int64_t tile) -> bool {
    const double2 mm = tile_mm[tile];
    const bool gauss_out = ymin - mm.y > kGaussCut || ymax - mm.x < -kGaussCut;
    const bool left_out = !has_left || a - mm.x <= -kGaussCut;
    const bool right_out = !has_right || mm.y - b <= -kGaussCut;
    return !(gauss_out && left_out && right_out);
  };
  constexpr int kFull = 1, kEmpty = 3, kProd = 5;  // named barrier ids (0 is __syncthreads)
  const int warp = tid >> 5;
  if (warp >= kFConsWarps) {
    // ---------------- producers
    const int t = tid - 32 * kFConsWarps;
    const int qq = t % kFQ;
    const int64_t q = q0 + qq < n ? q0 + qq : n - 1;
    const double yt = yq[q];
    long long j = (long long)ceil((yt - a) / h - 0.5);
    if (j < 0) j = 0;
    if (j > d - 1) j = d - 1;
    const bool at_left = j == 0, at_right = j == d - 1;
    const double factor = (at_left || at_right) ? 0.5 : 1.0;
    const double INV = inv_sqrt_2pi();
    int k = 0;
    for (int64_t tile = 0; tile < ntiles; ++tile) {
      if (!live_tile(tile)) continue;
      const int buf = k & 1;
      if (k >= 2) named_sync(kEmpty + buf, kFThreads);
      double* st = fbuf + (size_t)buf * 3 * kTile * kFQ;
      const int64_t base = tile * kTile;
      // the tile's support data, staged once per stage by the producers
      named_sync(kProd, kFProd);  // every producer is done with the previous tile's copy
      for (int r = t; r < kTile; r += kFProd) {
        const int64_t i = base + r;
        sx[r] = i < m ? x[i] : 0.0;
        sw[r] = i < m ? w[i] : 0.0;
        stl[r] = i < m ? tails[i] : make_double2(0.0, 0.0);
      }
      named_sync(kProd, kFProd);
      constexpr int kRowStep = kFProd / kFQ;
      constexpr int kRows = (kTile + kRowStep - 1) / kRowStep;
#pragma unroll 4
      for (int rr = 0; rr < kRows; ++rr) {
        const int r = t / kFQ + rr * kRowStep;
        if (r >= kTile) break;
        const int64_t i = base + r;
        double t0 = 0.0, t1 = 0.0, t2 = 0.0;
        if (i < m) {
          const double xi = sx[r];
          const double diff = yt - xi;
          double wp = 0.0;
          if (diff <= kGaussCut && diff >= -kGaussCut)
            wp = (factor * ucp_exp_core((-0.5 * diff) * diff, stab2)) * INV;
          if (at_left) wp += stl[r].x;
          if (at_right) wp += stl[r].y;
          if (wp != 0.0) {
            t0 = wp * sw[r];
            t1 = t0 * xi;
            t2 = t1 * xi;
          }
        }
        st[(0 * kTile + r) * kFQ + qq] = t0;
        st[(1 * kTile + r) * kFQ + qq] = t1;
        st[(2 * kTile + r) * kFQ + qq] = t2;
      }
      named_arrive(kFull + buf, kFThreads);
      ++k;
    }
    // absorb the consumers' last EMPTY arrivals so every barrier completes
    for (int kk = k - 2 > 0 ? k - 2 : 0; kk < k; ++kk) named_sync(kEmpty + (kk & 1), kFThreads);
  } else {
    // ---------------- consumers: thread (plane, query)
    const bool cons = tid < 3 * kFQ;
    const int plane = tid / kFQ, qq = tid % kFQ;
    double acc = 0.0;
    int k = 0;
    for (int64_t tile = 0; tile < ntiles; ++tile) {
      if (!live_tile(tile)) continue;
      const int buf = k & 1;
      named_sync(kFull + buf, kFThreads);
      if (cons) {
        const double* st = fbuf + (size_t)buf * 3 * kTile * kFQ + (size_t)plane * kTile * kFQ + qq;
#pragma unroll 16
        for (int r = 0; r < kTile; ++r) acc += st[r * kFQ];
      }
      named_arrive(kEmpty + buf, kFThreads);
      ++k;
    }
    const int64_t q = q0 + qq;
    if (cons && q < n) (plane == 0 ? o0 : plane == 1 ? o1 : o2)[q] = acc;
  }
}

// Opt-in (UCP_WC_TABLE), tolerance-stated stage-1 moments of a tile of qper
// consecutive grid queries by a Taylor expansion about the tile centre yc:
// with t = x - yc and d = y - yc, phi(y - x) = phi(t) exp(-d^2/2) exp(t d), so
//   M_m(y) = exp(-d^2/2) sum_n d^n / n! A_nm,  A_nm = sum_i w_i x_i^m phi(t_i) t_i^n:
// one exp and kFgtK (1 mul + 1 add + 2 FMA) per (tile, source) pair instead
// of one exp per (query, source) pair.  The tile spans at most kExCell
// (qper = floor(kExCell / h) queries), so |d| <= 0.008 and |t| <= 12.008:
// the first omitted term is ~(0.096)^12 / 12! < 1e-21.  Sources within
// 12 + span/2 of yc are included (the reference cuts at 12 per query: the
// extra terms weigh phi(12) ~ 6e-32).  Partial sums are reduced over the CTA
// in a fixed order: deterministic.  The two grid-end queries (factor 1/2 and
// the cdf tails) are completed by k_edge_tails / k_edge_finish.
constexpr int kFgtK = 12, kFgtThreads = 128;
__global__ void __launch_bounds__(kFgtThreads) k_mom_fgt(const double* __restrict__ yq, int64_t nq, int qper,
                                                         const double2* __restrict__ xw, int64_t m,
                                                         const double2* __restrict__ tile_mm, double* o0,
                                                         double* o1, double* o2) {
  __shared__ __align__(16) uint64_t stab[256];
  __shared__ double red[kFgtThreads / 32][3 * kFgtK];
  __shared__ double sA[3 * kFgtK];
  for (int r = threadIdx.x; r < 256; r += blockDim.x) stab[r] = g_exp_tab[r];
  UCP_SYNC();
  const ucp_exp_entry* stab2 = reinterpret_cast<const ucp_exp_entry*>(stab);
  const int64_t q0 = (int64_t)blockIdx.x * qper;
  const int64_t qn = nq - q0 < qper ? nq - q0 : qper;
  const double ylo = yq[q0], yhi = yq[q0 + qn - 1];
  const double yc = 0.5 * (ylo + yhi), cut = kGaussCut + 0.5 * (yhi - ylo);
  const double INV = inv_sqrt_2pi();
  double A[kFgtK][3];
#pragma unroll
  for (int k = 0; k < kFgtK; ++k) A[k][0] = A[k][1] = A[k][2] = 0.0;
  const int64_t ntiles = (m + kTile - 1) / kTile;
  // live tiles only (a NaN tile is (-inf, inf): visited); each thread owns
  // kTile / kFgtThreads sources of a tile, the next live tile's sources are
  // loaded while this one's are expanded (L2 latency behind the FP64 work)
  auto next_live = [&](int64_t tile) {
    for (; tile < ntiles; ++tile) {
      const double2 mm = tile_mm[tile];
      if (!(yc - mm.y > cut || yc - mm.x < -cut)) break;
    }
    return tile;
  };
  constexpr int kPer = kTile / kFgtThreads;
  double2 cur[kPer], nxt[kPer];
  int64_t tile = next_live(0);
  if (tile < ntiles)
#pragma unroll
    for (int r = 0; r < kPer; ++r) cur[r] = xw[tile * kTile + r * kFgtThreads + threadIdx.x];
  while (tile < ntiles) {
    const int64_t nt = next_live(tile + 1);
    if (nt < ntiles)
#pragma unroll
      for (int r = 0; r < kPer; ++r) nxt[r] = xw[nt * kTile + r * kFgtThreads + threadIdx.x];
#pragma unroll
    for (int r = 0; r < kPer; ++r) {
      const double2 s = cur[r];  // padding is (+inf, 0): out of reach
      const double t = s.x - yc;
      if (!(fabs(t) <= cut)) continue;
      const double x = s.x, x2 = x * x;
      double c = ucp_exp_core((-0.5 * t) * t, stab2) * INV * s.y;
#pragma unroll
      for (int k = 0; k < kFgtK; ++k) {
        A[k][0] += c;
        A[k][1] = __fma_rn(c, x, A[k][1]);
        A[k][2] = __fma_rn(c, x2, A[k][2]);
        c *= t;
      }
    }
#pragma unroll
    for (int r = 0; r < kPer; ++r) cur[r] = nxt[r];
    tile = nt;
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < kFgtK; ++k)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      double x = A[k][j];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
      if (lane == 0) red[wid][3 * k + j] = x;
    }
  UCP_SYNC();
  if (threadIdx.x < 3 * kFgtK) {  // fixed-order sums over the CTA's warps
    double acc = 0.0;
    for (int w = 0; w < kFgtThreads / 32; ++w) acc += red[w][threadIdx.x];
    sA[threadIdx.x] = acc;
  }
  UCP_SYNC();
  for (int64_t i = threadIdx.x; i < qn; i += kFgtThreads) {
    const int64_t q = q0 + i;
    const double dq = yq[q] - yc;
    double r0 = sA[3 * (kFgtK - 1)], r1 = sA[3 * (kFgtK - 1) + 1], r2 = sA[3 * (kFgtK - 1) + 2];
#pragma unroll
    for (int k = kFgtK - 2; k >= 0; --k) {  // sum_n A_n d^n / n!, Horner with 1/(n+1) folded in
      const double f = dq * (1.0 / (double)(k + 1));
      r0 = __fma_rn(r0, f, sA[3 * k]);
      r1 = __fma_rn(r1, f, sA[3 * k + 1]);
      r2 = __fma_rn(r2, f, sA[3 * k + 2]);
    }
    const double gd = ucp_exp_core((-0.5 * dq) * dq, stab2);
    o0[q] = gd * r0;
    o1[q] = gd * r1;
    o2[q] = gd * r2;
  }
}

// Grid-end queries of the expansion path (kernels.py:466-482): the reference
// gives them factor 1/2 on the Gaussian part plus the cdf tails
// phi_cdf(a - x)/h (first node) and phi_cdf(x - b)/h (last node) over EVERY
// support point.  k_edge_tails: per-CTA partial sums of w x^m tail (left and
// right, 6 values); k_edge_finish (one warp): fixed-order total, then
// o[edge] = 0.5 * o[edge] + tails.  Deterministic; 2 launches instead of two
// single-query exact passes over the whole support.
constexpr int kEdgeThreads = 256, kEdgeBlocks = 296;
__global__ void __launch_bounds__(kEdgeThreads) k_edge_tails(const double2* __restrict__ xw,
                                                             const double2* __restrict__ tails, int64_t m,
                                                             double* __restrict__ part) {
  __shared__ double red[kEdgeThreads / 32][6];
  double acc[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * kEdgeThreads + threadIdx.x; i < m; i += (int64_t)gridDim.x * kEdgeThreads) {
    const double2 s = xw[i], tl = tails[i];
    const double wl = tl.x * s.y, wr = tl.y * s.y;
    acc[0] += wl;
    acc[1] = __fma_rn(wl, s.x, acc[1]);
    acc[2] = __fma_rn(wl * s.x, s.x, acc[2]);
    acc[3] += wr;
    acc[4] = __fma_rn(wr, s.x, acc[4]);
    acc[5] = __fma_rn(wr * s.x, s.x, acc[5]);
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    double x = acc[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if (lane == 0) red[wid][k] = x;
  }
  UCP_SYNC();
  if (threadIdx.x < 6) {
    double x = 0.0;
    for (int w = 0; w < kEdgeThreads / 32; ++w) x += red[w][threadIdx.x];
    part[(int64_t)blockIdx.x * 6 + threadIdx.x] = x;
  }
}
__global__ void k_edge_finish(const double* __restrict__ part, int nblk, int64_t lq_left, int64_t lq_right,
                              double* o0, double* o1, double* o2) {
  const int k = threadIdx.x;
  if (k >= 6) return;
  double x = 0.0;
  for (int b = 0; b < nblk; ++b) x += part[(int64_t)b * 6 + k];
  const int64_t lq = k < 3 ? lq_left : lq_right;
  if (lq < 0) return;
  double* o = (k % 3 == 0) ? o0 : (k % 3 == 1 ? o1 : o2);
  o[lq] = 0.5 * o[lq] + x;
}

// Stage-1 candidates: C1(u, y) = A u^2 - 2 B u + C (witsenhausen.py:73-78).
__global__ void k_stage1_segmented(const double* __restrict__ u_flat, const int64_t* __restrict__ offsets,
                                   int64_t nseg, const double* __restrict__ m0,
                                   const double* __restrict__ m1, const double* __restrict__ m2,
                                   double* out) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t n = offsets[nseg];
  if (c >= n) return;
  int64_t lo = 0, hi = nseg;
  while (hi - lo > 1) {
    int64_t mid = (lo + hi) >> 1;
    if (offsets[mid] <= c) lo = mid; else hi = mid;
  }
  out[c] = quad_in_u(m0[lo], m1[lo], m2[lo], u_flat[c]);
}

__global__ void k_lu1(const double* __restrict__ u1, const double* __restrict__ m0,
                      const double* __restrict__ m1, const double* __restrict__ m2,
                      ucp_local_params lp, int64_t begin, int64_t n, double* out, int64_t* err, const BatchArgs BA) {
  pdl_wait();
  pdl_trigger();
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  if (BA.ids) {  // moments per slot (stride sslot), output per slot (stride n)
    const int b = BA.inst(blockIdx.y);
    u1 += b * BA.su1;
    m0 += blockIdx.y * BA.sslot;
    m1 += blockIdx.y * BA.sslot;
    m2 += blockIdx.y * BA.sslot;
    out += blockIdx.y * n;
    err += b * BA.serr;
  }
  int64_t i = begin + t;
  const double A = m0[t], B = m1[t], C = m2[t];
  double u = u1[i];
  double hh = lp.fd_step * (1.0 + fabs(u));
  double up = quad_in_u(A, B, C, u + hh);
  double mid = quad_in_u(A, B, C, u);
  double dn = quad_in_u(A, B, C, u - hh);
  double c1 = (up - dn) / (2.0 * hh);
  double c2 = ((up - 2.0 * mid) + dn) / (hh * hh);
  if (!(finite(c1) && finite(c2))) {
    flag_min(err, i);
    out[i] = u;
    return;
  }
  double stepped = newton_step(u, c1, c2, lp);
  double cost_new = quad_in_u(A, B, C, stepped);
  if (!(finite(mid) && finite(cost_new))) flag_min(err + 1, i);
  double r = cost_new <= mid ? stepped : u;
  if (!finite(r)) flag_min(err + 2, i);
  out[i] = r;
}

__global__ void k_ex1(const double* __restrict__ u1, const double* __restrict__ m0,
                      const double* __restrict__ m1, const double* __restrict__ m2,
                      const int64_t* __restrict__ lo, const int64_t* __restrict__ hi, int64_t begin,
                      int64_t n, double* out, int64_t* err, const BatchArgs BA) {
  pdl_wait();
  pdl_trigger();
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  if (BA.ids) {
    const int b = BA.inst(blockIdx.y);
    u1 += b * BA.su1;
    m0 += blockIdx.y * BA.sslot;
    m1 += blockIdx.y * BA.sslot;
    m2 += blockIdx.y * BA.sslot;
    out += blockIdx.y * n;
    err += b * BA.serr;
  }
  int64_t i = begin + t;
  const double A = m0[t], B = m1[t], C = m2[t];
  int64_t j0 = lo[i], j1 = hi[i];
  double bu = u1[j0];
  double bv = quad_in_u(A, B, C, bu);
  bool ok = finite(bv);
  for (int64_t j = j0 + 1; j <= j1; ++j) {
    double uj = u1[j];
    double c = quad_in_u(A, B, C, uj);
    ok = ok && finite(c);
    if (c < bv) {
      bv = c;
      bu = uj;
    }
  }
  if (!ok) flag_min(err, i);
  out[i] = bu;
}

__global__ void k_copy(const double* __restrict__ src, double* __restrict__ dst, int64_t n) {
  pdl_wait();
  pdl_trigger();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[i];
}

__global__ void k_device_libm(int which, const double* __restrict__ x, int64_t n, double* out) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  double v = x[t];
  out[t] = which == 0 ? ucp_exp_tab(v, g_exp_tab) : (which == 1 ? ucp_erf_tab(v, g_exp_tab) : phi_cdf(v));
}

__global__ void k_fp64_probe(int iters, double* sink) {
  double a0 = threadIdx.x * 1e-9 + 1.0, a1 = a0 + 1e-3, a2 = a0 + 2e-3, a3 = a0 + 3e-3;
  double a4 = a0 + 4e-3, a5 = a0 + 5e-3, a6 = a0 + 6e-3, a7 = a0 + 7e-3;
  const double m = 0.999999999, c = 1e-12;
  for (int i = 0; i < iters; ++i) {
    a0 = a0 * m; a1 = a1 * m; a2 = a2 * m; a3 = a3 * m;
    a4 = a4 * m; a5 = a5 * m; a6 = a6 * m; a7 = a7 * m;
    a0 = a0 + c; a1 = a1 + c; a2 = a2 + c; a3 = a3 + c;
    a4 = a4 + c; a5 = a5 + c; a6 = a6 + c; a7 = a7 + c;
  }
  sink[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

}  // namespace

// ============================================================ workspace
constexpr int kGraphKeyWords = 21;
struct ucp_graph_entry {
  std::array<uint64_t, kGraphKeyWords> key;
  cudaGraphExec_t exec;
  int64_t kernels;  // kernel nodes per replay (the launch counter)
  bool stale;       // recycled workspace: reusable only through cudaGraphExecUpdate
};

// CUDA-graph captures (ThreadLocal mode) run concurrently in the host threads
// of solve_many; a device-synchronising call from ANY thread (cudaFree,
// cudaFreeHost, cudaDeviceSynchronize) while a capture is open would
// invalidate it.  Captures hold this lock shared; the library's
// synchronising calls (workspace growth / destruction) hold it exclusively.
std::shared_mutex g_capture_mu;

// Inventory density / cost-to-go reuse across calls (ucp_inv_problem.ukey):
// slot k of the forward buffer holds f_k computed from controllers with keys
// fkey[k][0..k-1]; slot k of the backward buffer g_k from gkey[k][k..M-1].
struct ucp_inv_cache {
  bool valid = false;
  ucp_inv_problem prob{};  // the problem the slots belong to (ukey cleared)
  const void* fbuf = nullptr;
  const void* gbuf = nullptr;
  bool fok[UCP_INV_MAX_STAGES + 1] = {false};
  bool gok[UCP_INV_MAX_STAGES + 1] = {false};
  uint64_t fkey[UCP_INV_MAX_STAGES + 1][UCP_INV_MAX_STAGES] = {};
  uint64_t gkey[UCP_INV_MAX_STAGES + 1][UCP_INV_MAX_STAGES] = {};
};

struct ucp_workspace {
  void* buf[24] = {nullptr};
  size_t cap[24] = {0};
  void* scan_tmp = nullptr;
  size_t scan_cap = 0;
  int64_t* h_total = nullptr;           // pinned
  cudaStream_t cap_stream = nullptr;    // private stream for CUDA-graph capture
  std::vector<ucp_graph_entry> graphs;  // one instantiated graph per block signature
  ucp_inv_cache inv;
};

namespace {
enum {
  WS_X1 = 0, WS_TILE, WS_MOM, WS_COST, WS_COUNT, WS_CAND_PT, WS_CAND_J, WS_TOTAL, WS_TAILS,
  WS_C5_F0, WS_C5_F1, WS_C5_G0, WS_C5_G1, WS_C5_ONE, WS_XW, WS_C5_TAB, WS_C5_GT0, WS_C5_GT1, WS_C5_MEMO, WS_C5_FC, WS_C5_GC, WS_VSUF, WS_TABLE, WS_EDGE, WS_NSLOTS
};
static_assert(WS_NSLOTS <= 24, "workspace slots");
// fused moments below this many queries (above, k_moments' persistent CTAs
// have enough query blocks to fill the GPU); env UCP_FUSED_MAX_QUERIES
const int64_t kFusedMaxQueries = [] {
  const char* e = getenv("UCP_FUSED_MAX_QUERIES");
  // crossover measured with tools/moments_sweep.py: ~8.7k queries since the
  // persistent kernel keeps 16 exps in flight (it was 16k at 4)
  return e ? (int64_t)atoll(e) : (int64_t)8704;
}();
// warp-per-point candidate fill below this many points (one thread per point above)
constexpr int64_t kWarpFillMaxPoints = 1 << 16;
// sync-free exhaustion when the candidate upper bound fits (16 B per candidate)
// (an eighth of the device memory, read once; at least 2^27 candidates, and
// under 2^31 so candidate positions fit the kernels' int32 point indices):
// C3's 2^22-point, 39-node sweep (1.6e8 candidates, 2.6 GB) stays sync-free.
int64_t sync_free_max_cand() {
  static const int64_t cap = [] {
    size_t free_b = 0, total_b = 0;
    int64_t c = (int64_t)1 << 27;
    if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) c = std::max(c, (int64_t)(total_b / 8 / 16));
    return std::min(c, ((int64_t)1 << 31) - 1);
  }();
  return cap;
}

int ws_get(ucp_workspace* ws, int slot, size_t bytes, void** out) {
  if (ws->cap[slot] < bytes) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (ws->cap_stream && cudaStreamIsCapturing(ws->cap_stream, &cs) == cudaSuccess &&
        cs != cudaStreamCaptureStatusNone)
      return arg_fail("workspace growth during graph capture");
    std::unique_lock<std::shared_mutex> lk(g_capture_mu);
    // captured graphs hold workspace addresses: growing a buffer retires them
    // (an in-flight graph exec is freed asynchronously on completion)
    for (auto& g : ws->graphs) cudaGraphExecDestroy(g.exec);
    ws->graphs.clear();
    if (ws->buf[slot]) UCP_CHECK(cudaFree(ws->buf[slot]));
    ws->buf[slot] = nullptr;
    ws->cap[slot] = 0;
    size_t want = bytes + bytes / 4 + 256;
    UCP_CHECK(cudaMalloc(&ws->buf[slot], want));
    ws->cap[slot] = want;
  }
  *out = ws->buf[slot];
  return UCP_OK;
}

// x1 = y0 + u0 and per-tile min/max, then the moments of `nq` queries.
int run_moments(const double* yq, int64_t nq, const double* y0, const double* u0, const double* w,
                int64_t m, double a, double h, int64_t d, double* o0, double* o1, double* o2,
                ucp_workspace* ws, cudaStream_t st, int64_t grid_begin = -1) {
  if (nq <= 0) return UCP_OK;
  void *px1, *ptile, *pctr, *ptails;
  int rc;
  int64_t ntiles = (m + kTile - 1) / kTile;
  void* pxw;
  if ((rc = ws_get(ws, WS_X1, sizeof(double) * (size_t)m, &px1))) return rc;
  if ((rc = ws_get(ws, WS_TAILS, sizeof(double2) * (size_t)m, &ptails))) return rc;
  if ((rc = ws_get(ws, WS_XW, sizeof(double2) * (size_t)(ntiles * kTile), &pxw))) return rc;
  if ((rc = ws_get(ws, WS_TILE, sizeof(double2) * (size_t)ntiles, &ptile))) return rc;
  if ((rc = ws_get(ws, WS_TOTAL, sizeof(int64_t) * 2, &pctr))) return rc;
  const double b = a + h * (double)(d - 1);
  UCP_CHECK(launch_pdl(k_x1_prepare, dim3((unsigned)ntiles), dim3(kTile), 0, st, y0, u0, w, m, a, h, b, (double*)px1,
                       (double2*)pxw, (double2*)ptails, (double2*)ptile, kNoBatch));
  UCP_LAUNCHED("k_x1_prepare");
  if (grid_begin >= 0 && h <= kTableMaxH && nq >= 2) {
    // UCP_WC_TABLE: the queries are grid points grid_begin.. : expansion moments,
    // then the (at most two) grid-end queries exactly
    const int qper = (int)fmin(floor(kExCell / h), 65536.0);
    k_mom_fgt<<<(unsigned)((nq + qper - 1) / qper), kFgtThreads, 0, st>>>(yq, nq, qper, (const double2*)pxw, m,
                                                                          (const double2*)ptile, o0, o1, o2);
    UCP_LAUNCHED("k_mom_fgt");
    const int64_t ll = grid_begin == 0 ? 0 : -1;                          // first grid node here?
    const int64_t lr = grid_begin + nq == d && d > 1 ? nq - 1 : -1;      // last grid node here?
    if (ll >= 0 || lr >= 0) {
      void* pe;
      if ((rc = ws_get(ws, WS_EDGE, sizeof(double) * 6 * kEdgeBlocks, &pe))) return rc;
      k_edge_tails<<<kEdgeBlocks, kEdgeThreads, 0, st>>>((const double2*)pxw, (const double2*)ptails, m, (double*)pe);
      UCP_LAUNCHED("k_edge_tails");
      k_edge_finish<<<1, 32, 0, st>>>((const double*)pe, kEdgeBlocks, ll, lr, o0, o1, o2);
      UCP_LAUNCHED("k_edge_finish");
    }
    return UCP_OK;
  }
  if (nq <= kFusedMaxQueries) {
    smem_opt_in(reinterpret_cast<const void*>(k_mom_fused), kFSmem);
    UCP_CHECK(launch_pdl(k_mom_fused, dim3(nblocks(nq, kFQ)), dim3(kFThreads), kFSmem, st, yq, nq, (const double*)px1,
                         w, (const double2*)ptails, (const double2*)ptile, m, a, h, d, o0, o1, o2,
                         (const int32_t*)nullptr, (int64_t)0, (int64_t)0));
    UCP_LAUNCHED("k_mom_fused");
    return UCP_OK;
  }
  int* counter = (int*)((int64_t*)pctr + 1);
  UCP_CHECK(cudaMemsetAsync(counter, 0, sizeof(int), st));
  int dev = 0, sms = 0, per_sm = 0;
  UCP_CHECK(cudaGetDevice(&dev));
  UCP_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  UCP_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_moments<>, kMomThreads, 0));
  int64_t nqb = (nq + kMomThreads - 1) / kMomThreads;
  int64_t grid = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
  if (grid > nqb) grid = nqb;
  k_moments<><<<(unsigned)grid, kMomThreads, 0, st>>>(yq, nq, (const double2*)pxw, (const double2*)ptails, m,
                                                      (const double2*)ptile, a, h, d, o0, o1, o2, counter, 1, 0);
  UCP_LAUNCHED("k_moments");
  return UCP_OK;
}

// Walk launches below kWalkLatencyCtasPerSm CTAs per SM run the latency-mode
// walk (one prefetching warp per walk group is faster when warps are scarce);
// from 6 CTAs/SM on the throughput walk (with the no-op tail exit) wins: A/B
// of 12 / 6 / 4 / 2 -- an 8-rank shard of the 2^20 step's local update 127 ->
// 107 ms at 6, C1 35.3 -> 35.1 ms, d=14000 1.296 -> 1.281 s (profiles/r2_walk_latency_threshold.log).
#ifndef UCP_WALK_LAT_CTAS
#define UCP_WALK_LAT_CTAS 6
#endif
constexpr int kWalkLatencyCtasPerSm = UCP_WALK_LAT_CTAS;
bool walk_latency_mode(int64_t n_walks) {
  static const int sms = [] {  // initialised once, thread-safe (function-local static)
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      n = 148;
    return n;
  }();
  return n_walks < (int64_t)sms * kWalkLatencyCtasPerSm * kWalkThreads;
}

// kSmemWalkMax doubles of v1 fit the opt-in shared memory of one CTA
constexpr int64_t kSmemWalkMax = 27648;  // 216 KiB of the 227 KiB opt-in per CTA

template <class K>
void allow_smem(K* kernel) {  // opt in to >48 KiB dynamic shared memory (walk kernels)
  smem_opt_in(reinterpret_cast<const void*>(kernel), kSmemWalkMax * sizeof(double));
}

#define UCP_WALK_LAUNCH(kernel, n_walks, grid, stream, d_v1, ...)                                   \
  do {                                                                                            \
    if (!walk_latency_mode(n_walks)) {                                                            \
      kernel<0><<<(grid), kWalkThreads, 0, (stream)>>>(__VA_ARGS__);                              \
    } else if ((d_v1) <= kSmemWalkMax) {                                                          \
      allow_smem(kernel<2>);                                                                      \
      kernel<2><<<(grid), kWalkThreads, (size_t)(d_v1) * sizeof(double), (stream)>>>(__VA_ARGS__); \
    } else {                                                                                      \
      kernel<1><<<(grid), kWalkThreads, 0, (stream)>>>(__VA_ARGS__);                              \
    }                                                                                             \
  } while (0)

// Same, with programmatic dependent launch in the latency regime (the
// local-update chain, where it measurably shortens the iteration).
#define UCP_WALK_LAUNCH_PDL(kernel, n_walks, grid, stream, d_v1, ...)                               \
  do {                                                                                            \
    if (!walk_latency_mode(n_walks)) {                                                            \
      kernel<0><<<(grid), kWalkThreads, 0, (stream)>>>(__VA_ARGS__);                              \
    } else if ((d_v1) <= kSmemWalkMax) {                                                          \
      allow_smem(kernel<2>);                                                                      \
      UCP_CHECK(launch_pdl(kernel<2>, dim3(grid), dim3(kWalkThreads), (size_t)(d_v1) * sizeof(double), \
                           (stream), __VA_ARGS__));                                               \
    } else {                                                                                      \
      kernel<1><<<(grid), kWalkThreads, 0, (stream)>>>(__VA_ARGS__);                              \
    }                                                                                             \
  } while (0)

// Throughput-mode stage-0 walks over v1 end at their no-op tail
// (walk_tail_noop, result-invariant): build the suffix bounds of v1 on the
// stream first.  UCP_TAIL_EXIT=0 walks every node.
const bool g_tail_exit = [] {
  const char* e = getenv("UCP_TAIL_EXIT");
  return !(e && e[0] == '0');
}();
int attach_vsuf(WalkGrid* g, const double* v1, int64_t n_walks, ucp_workspace* ws, cudaStream_t st) {
  if (!g_tail_exit || walk_latency_mode(n_walks)) return UCP_OK;
  void* p;
  if (int rc = ws_get(ws, WS_VSUF, sizeof(double) * (size_t)g->nb * vsuf_levels(g->nb), &p)) return rc;
  k_vsuf<<<1, 1024, 0, st>>>(v1, g->d, g->nb, (double*)p, nullptr, 0, 0);
  UCP_LAUNCHED("k_vsuf");
  g->vsuf = (const double*)p;
  return UCP_OK;
}


int table_local() {  // UCP_TABLE_LOCAL=0: the stage-0 local update keeps the FMA walk (A/B)
  static const int k = [] {
    const char* e = getenv("UCP_TABLE_LOCAL");
    return e ? atoi(e) : 1;
  }();
  return k;
}

int attach_table(WalkGrid* g, const ucp_wc_problem* P, const double* v1, ucp_workspace* ws, cudaStream_t st) {
  if (!(P->flags & UCP_WC_TABLE) || !(P->h1 <= kTableMaxH)) return UCP_OK;
  // cells cover every centre whose window reaches the grid: [a - 12, b + 12]
  const double s0 = P->a1 - kGaussCut, span = (P->a1 + P->h1 * (double)(P->d1 - 1) + kGaussCut) - s0;
  const int64_t nc = (int64_t)ceil(span / kExCell) + 1;
  void* pt;
  if (int rc = ws_get(ws, WS_TABLE, sizeof(double) * 3 * kExRows * (size_t)nc, &pt)) return rc;
  // dq = fl(q)/q - 1 for the walk's q = fl(exp(-h^2)) (g->q, the same bits):
  // fl(q) - 1 is exact (Sterbenz), expm1 resolves q - 1 to ~1 ulp of h^2
  g->ex_dq2 = 0.5 * (((g->q - 1.0) - expm1(-P->h1 * P->h1)) / g->q);
  g->ex_ih = 1.0 / P->h1;
  g->ex_s0 = s0;
  g->ex_dlt = kExCell;
  g->ex_inv = 1.0 / kExCell;
  g->ex_n = nc;
  k_ex_cells<<<(unsigned)nc, kExThreads, 0, st>>>(v1, *g, (double*)pt);
  UCP_LAUNCHED("k_ex_cells");
  g->table = (const double*)pt;
  return UCP_OK;
}

int check_aligned(const void* v) {
  if (reinterpret_cast<uintptr_t>(v) & 15u) return arg_fail("controller arrays must be 16-byte aligned");
  return UCP_OK;
}

int check_problem(const ucp_wc_problem* P) {
  if (!P || !P->y0 || !P->y1 || !P->f0 || !P->fw0) return arg_fail("null problem pointer");
  if (P->d0 < 2 || P->d1 < 2) return arg_fail("grid.d must be at least 2");
  if (P->d0 > INT32_MAX || P->d1 > INT32_MAX) return arg_fail("grid too large for int32 indices");
  return UCP_OK;
}
}  // namespace

// ============================================================ C ABI
extern "C" {

int ucp_abi_version(void) { return UCP_ABI_VERSION; }

const char* ucp_status_string(int status) {
  switch (status) {
    case UCP_OK: return "ok";
    case UCP_ERR_ARG: return "bad argument";
    case UCP_ERR_CUDA: return "CUDA error";
    default: return "unknown status";
  }
}

const char* ucp_last_error(void) { return g_errbuf; }

int64_t ucp_launch_count(void) { return g_launches.load(); }

int ucp_workspace_create(ucp_workspace** ws) {
  if (!ws) return arg_fail("null workspace handle");
  *ws = new ucp_workspace();
  UCP_CHECK(cudaMallocHost(&(*ws)->h_total, sizeof(int64_t)));
  return UCP_OK;
}

int ucp_workspace_destroy(ucp_workspace* ws) {
  if (!ws) return UCP_OK;
  std::unique_lock<std::shared_mutex> lk(g_capture_mu);
  cudaDeviceSynchronize();  // in-flight work may still read the buffers
  for (int i = 0; i < 24; ++i)
    if (ws->buf[i]) cudaFree(ws->buf[i]);
  if (ws->scan_tmp) cudaFree(ws->scan_tmp);
  if (ws->h_total) cudaFreeHost(ws->h_total);
  for (auto& g : ws->graphs) cudaGraphExecDestroy(g.exec);
  if (ws->cap_stream) cudaStreamDestroy(ws->cap_stream);
  delete ws;
  return UCP_OK;
}

int ucp_workspace_recycle(ucp_workspace* ws) {
  if (!ws) return arg_fail("null workspace");
  std::unique_lock<std::shared_mutex> lk(g_capture_mu);
  // the next owner may queue on another stream: nothing in flight may still use the buffers
  UCP_CHECK(cudaDeviceSynchronize());
  for (auto& g : ws->graphs) g.stale = true;
  ws->inv = ucp_inv_cache{};
  return UCP_OK;
}

int ucp_workspace_reserve(ucp_workspace* ws, int64_t d0, int64_t d1, int64_t max_cand) {
  if (!ws) return arg_fail("null workspace");
  void* p;
  int rc;
  int64_t dm = d0 > d1 ? d0 : d1;
  if ((rc = ws_get(ws, WS_X1, sizeof(double) * (size_t)dm, &p))) return rc;
  if ((rc = ws_get(ws, WS_TAILS, sizeof(double2) * (size_t)dm, &p))) return rc;
  if ((rc = ws_get(ws, WS_TOTAL, sizeof(int64_t) * 2, &p))) return rc;
  if ((rc = ws_get(ws, WS_TILE, sizeof(double2) * (size_t)((dm + kTile - 1) / kTile), &p))) return rc;
  if ((rc = ws_get(ws, WS_MOM, sizeof(double) * 3 * (size_t)dm, &p))) return rc;
  if ((rc = ws_get(ws, WS_COST, sizeof(double) * (size_t)(max_cand > 3 * dm ? max_cand : 3 * dm), &p))) return rc;
  if ((rc = ws_get(ws, WS_COUNT, sizeof(int64_t) * (size_t)(dm + 1), &p))) return rc;
  if ((rc = ws_get(ws, WS_CAND_PT, sizeof(int32_t) * (size_t)max_cand, &p))) return rc;
  if ((rc = ws_get(ws, WS_CAND_J, sizeof(int32_t) * (size_t)max_cand, &p))) return rc;
  {
    const int nb1 = (int)((d1 + (1 << kVsufShift) - 1) >> kVsufShift);
    if ((rc = ws_get(ws, WS_VSUF, sizeof(double) * (size_t)nb1 * vsuf_levels(nb1), &p))) return rc;
  }
  return UCP_OK;
}

int ucp_gauss_moments_grid(const double* s, int64_t n, const double* v, double a, double h, int64_t d,
                           double* t0, double* t1, double* t2, void* stream) {
  if (n < 0 || d < 2 || d > INT32_MAX) return arg_fail("gauss_moments_grid: bad sizes");
  if (n == 0) return UCP_OK;
  if (int rc_ = check_aligned(v)) return rc_;
  WalkGrid g = make_walk_grid(a, h, d);
  UCP_WALK_LAUNCH(k_gauss_grid, n, nblocks(n, kWalkThreads), as_stream(stream), d, s, n, v, g, t0, t1, t2);
  UCP_LAUNCHED("k_gauss_grid");
  return UCP_OK;
}

int ucp_gauss_moments_points(const double* y, int64_t n, const double* x, const double* w, int64_t m,
                             double a, double h, int64_t d, double* o0, double* o1, double* o2,
                             ucp_workspace* ws, void* stream) {
  if (n < 0 || m < 0 || d < 2 || !ws) return arg_fail("gauss_moments_points: bad sizes");
  if (n == 0) return UCP_OK;
  if (m == 0) {
    UCP_CHECK(cudaMemsetAsync(o0, 0, sizeof(double) * n, as_stream(stream)));
    UCP_CHECK(cudaMemsetAsync(o1, 0, sizeof(double) * n, as_stream(stream)));
    UCP_CHECK(cudaMemsetAsync(o2, 0, sizeof(double) * n, as_stream(stream)));
    return UCP_OK;
  }
  return run_moments(y, n, nullptr, x, w, m, a, h, d, o0, o1, o2, ws, as_stream(stream));
}

int ucp_trapezoid_sum(const double* samples, int64_t n, double spacing, double* out, int64_t* err,
                      void* stream) {
  if (n < 1) return arg_fail("trapezoid needs at least one sample");
  cudaStream_t st = as_stream(stream);
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (n >= kTzMinN && tz_parallel() && cudaStreamIsCapturing(st, &cs) == cudaSuccess &&
      cs == cudaStreamCaptureStatusNone) {
    // the chunked exact form (k_tz_*): bitwise the serial sum
    const int64_t nch = (n - 1 + kTzL - 1) / kTzL;
    void* scratch = nullptr;
    if (int rc = tz_scratch(st, nch * (sizeof(double) + sizeof(TzRec)), &scratch)) return rc;
    double* csum = (double*)scratch;
    TzRec* rec = (TzRec*)(csum + nch);
    k_tz_chunks<<<(unsigned)((nch * 32 + 255) / 256), 256, 0, st>>>(samples, n, nch, csum, err);
    UCP_LAUNCHED("k_tz_chunks");
    k_tz_plan<<<1, 1024, 0, st>>>(samples, csum, nch, rec);
    UCP_LAUNCHED("k_tz_plan");
    k_tz_decompose<<<nblocks(nch, 128), 128, 0, st>>>(samples, n, nch, rec);
    UCP_LAUNCHED("k_tz_decompose");
    k_tz_final<<<1, 32, 0, st>>>(samples, n, nch, rec, spacing, out);
    UCP_LAUNCHED("k_tz_final");
    return UCP_OK;
  }
  k_trapezoid<<<1, kTrapThreads, 0, st>>>(samples, n, spacing, out, err, kNoBatch);
  UCP_LAUNCHED("k_trapezoid");
  return UCP_OK;
}

int ucp_segmented_argmin(const double* costs, const int64_t* offsets, int64_t nseg, int64_t* out,
                         void* stream) {
  if (nseg < 0) return arg_fail("segmented_argmin: bad sizes");
  if (nseg == 0) return UCP_OK;
  k_segmented_argmin<<<nblocks(nseg, 128), 128, 0, as_stream(stream)>>>(costs, offsets, nseg, out);
  UCP_LAUNCHED("k_segmented_argmin");
  return UCP_OK;
}

int ucp_flatten_windows(const double* values, int64_t d, const int64_t* lo, const int64_t* hi, int64_t n,
                        double* flat, int64_t* offsets, ucp_workspace* ws, void* stream) {
  if (n < 0 || d < 1 || !values || !lo || !hi || !offsets || !ws) return arg_fail("flatten_windows: bad arguments");
  cudaStream_t st = as_stream(stream);
  UCP_CHECK(cudaMemsetAsync(offsets, 0, sizeof(int64_t) * (size_t)(n + 1), st));
  if (n == 0) return UCP_OK;
  // counts land in offsets[1..n]; an inclusive scan in place makes them offsets
  k_flatten_windows<false><<<nblocks(n, 128), 128, 0, st>>>(values, lo, hi, n, offsets + 1, nullptr, nullptr);
  UCP_LAUNCHED("k_flatten_windows<count>");
  size_t tmp_bytes = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, offsets + 1, offsets + 1, n, st);
  if (ws->scan_cap < tmp_bytes) {
    std::unique_lock<std::shared_mutex> lk(g_capture_mu);
    if (ws->scan_tmp) UCP_CHECK(cudaFree(ws->scan_tmp));
    UCP_CHECK(cudaMalloc(&ws->scan_tmp, tmp_bytes));
    ws->scan_cap = tmp_bytes;
  }
  UCP_CHECK(cub::DeviceScan::InclusiveSum(ws->scan_tmp, tmp_bytes, offsets + 1, offsets + 1, n, st));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (flat) {
    k_flatten_windows<true><<<nblocks(n, 128), 128, 0, st>>>(values, lo, hi, n, nullptr, offsets, flat);
    UCP_LAUNCHED("k_flatten_windows<fill>");
  }
  return UCP_OK;
}

int ucp_device_libm(int which, const double* x, int64_t n, double* out, void* stream) {
  if (which < 0 || which > 2 || n < 0) return arg_fail("device_libm: bad argument");
  if (n == 0) return UCP_OK;
  k_device_libm<<<nblocks(n, 256), 256, 0, as_stream(stream)>>>(which, x, n, out);
  UCP_LAUNCHED("k_device_libm");
  return UCP_OK;
}

int ucp_wc_stage0_cost(const ucp_wc_problem* P, const double* v1, const double* u_flat, int64_t n_cand,
                       const int64_t* offsets, const double* y_seg, const double* f0_seg, int64_t nseg,
                       double* out, void* stream) {
  return ucp_wc_stage0_cost_ws(P, v1, u_flat, n_cand, offsets, y_seg, f0_seg, nseg, out, nullptr, stream);
}

int ucp_wc_stage0_cost_ws(const ucp_wc_problem* P, const double* v1, const double* u_flat, int64_t n_cand,
                          const int64_t* offsets, const double* y_seg, const double* f0_seg, int64_t nseg,
                          double* out, ucp_workspace* ws, void* stream) {
  int rc = check_problem(P);
  if (rc) return rc;
  if (nseg < 0 || n_cand < 0) return arg_fail("stage0_cost: bad sizes");
  if (nseg == 0 || n_cand == 0) return UCP_OK;
  const int64_t n_host = n_cand;
  if (int rc_ = check_aligned(v1)) return rc_;
  WalkGrid g = make_walk_grid(P->a1, P->h1, P->d1, (int)(P->flags & UCP_WC_FAST));
  // with a workspace: the no-op tail exit (same bits) and, under UCP_WC_TABLE,
  // the expansion cells -- as in the phases
  if (ws && (rc = attach_vsuf(&g, v1, n_host, ws, as_stream(stream)))) return rc;
  if (ws && (rc = attach_table(&g, P, v1, ws, as_stream(stream)))) return rc;
  UCP_WALK_LAUNCH(k_stage0_segmented, n_host, nblocks(n_host, kWalkThreads), as_stream(stream), P->d1, u_flat, offsets, nseg, y_seg,
                                                                           f0_seg, P->k, v1, g, out);
  UCP_LAUNCHED("k_stage0_segmented");
  return UCP_OK;
}

int ucp_wc_stage1_cost(const ucp_wc_problem* P, const double* u0, const double* u_flat, int64_t n_cand,
                       const int64_t* offsets, const double* y_seg, int64_t nseg, double* out,
                       ucp_workspace* ws, void* stream) {
  int rc = check_problem(P);
  if (rc) return rc;
  if (nseg < 0 || n_cand < 0 || !ws) return arg_fail("stage1_cost: bad sizes");
  if (nseg == 0 || n_cand == 0) return UCP_OK;
  cudaStream_t st = as_stream(stream);
  void* pm;
  if ((rc = ws_get(ws, WS_MOM, sizeof(double) * 3 * (size_t)nseg, &pm))) return rc;
  double* m0 = (double*)pm;
  if ((rc = run_moments(y_seg, nseg, P->y0, u0, P->fw0, P->d0, P->a1, P->h1, P->d1, m0, m0 + nseg,
                        m0 + 2 * nseg, ws, st)))
    return rc;
  const int64_t n_host = n_cand;
  k_stage1_segmented<<<nblocks(n_host, 256), 256, 0, st>>>(u_flat, offsets, nseg, m0, m0 + nseg,
                                                             m0 + 2 * nseg, out);
  UCP_LAUNCHED("k_stage1_segmented");
  return UCP_OK;
}

int ucp_wc_local_update(const ucp_wc_problem* P, int stage, const double* u0, const double* u1,
                        const ucp_local_params* lp, int64_t begin, int64_t end, double* out, int64_t* err,
                        ucp_workspace* ws, void* stream) {
  int rc = check_problem(P);
  if (rc) return rc;
  if (!lp || !ws || !err) return arg_fail("local_update: null argument");
  int64_t d = stage == 0 ? P->d0 : P->d1;
  if (stage < 0 || stage > 1) return arg_fail("stage index out of range for witsenhausen");
  if (begin < 0 || end > d || begin > end) return arg_fail("local_update: bad shard");
  int64_t n = end - begin;
  if (n == 0) return UCP_OK;
  cudaStream_t st = as_stream(stream);
  if (stage == 0) {
    void* pc;
    if ((rc = ws_get(ws, WS_COST, sizeof(double) * 3 * (size_t)n, &pc))) return rc;
    if (int rc_ = check_aligned(u1)) return rc_;
    WalkGrid g = make_walk_grid(P->a1, P->h1, P->d1, (int)(P->flags & UCP_WC_FAST));
    if ((rc = attach_vsuf(&g, u1, 3 * n, ws, st))) return rc;
    // UCP_WC_TABLE: the expansion is smooth in s, so the local update's second
    // differences over h = 1e-4 (1 + |u|) see only the evaluation's rounding
    // (an interpolated lattice of independently rounded walks was tried: its
    // 1e-14 per-node noise became 1e-5 in c2)
    if (table_local() && (rc = attach_table(&g, P, u1, ws, st))) return rc;
    UCP_WALK_LAUNCH_PDL(k_lu0_probe, 3 * n, nblocks(3 * n, kWalkThreads), st, P->d1, P->y0, P->f0, u0, P->k, u1, g, lp->fd_step, begin, n,
                                                     (double*)pc, kNoBatch);
    UCP_LAUNCHED("k_lu0_probe");
    UCP_WALK_LAUNCH_PDL(k_lu0_finish, n, nblocks(n, kWalkThreads), st, P->d1, P->y0, P->f0, u0, P->k, u1, g, *lp, begin, n,
                                                  (const double*)pc, out, err, kNoBatch);
    UCP_LAUNCHED("k_lu0_finish");
    return UCP_OK;
  }
  void* pm;
  if ((rc = ws_get(ws, WS_MOM, sizeof(double) * 3 * (size_t)n, &pm))) return rc;
  double* m0 = (double*)pm;
  if ((rc = run_moments(P->y1 + begin, n, P->y0, u0, P->fw0, P->d0, P->a1, P->h1, P->d1, m0, m0 + n,
                        m0 + 2 * n, ws, st, (P->flags & UCP_WC_TABLE) ? begin : -1)))
    return rc;
  UCP_CHECK(launch_pdl(k_lu1, dim3(nblocks(n, 256)), dim3(256), 0, st, (const double*)u1, (const double*)m0,
                       (const double*)(m0 + n), (const double*)(m0 + 2 * n), *lp, begin, n, out, err, kNoBatch));
  UCP_LAUNCHED("k_lu1");
  return UCP_OK;
}

int ucp_wc_exhaustion(const ucp_wc_problem* P, int stage, const double* u0, const double* u1,
                      const int64_t* win_lo, const int64_t* win_hi, int64_t cand_bound, int64_t begin,
                      int64_t end, double* out, int64_t* err, ucp_workspace* ws, void* stream) {
  int rc = check_problem(P);
  if (rc) return rc;
  if (!ws || !err || !win_lo || !win_hi) return arg_fail("exhaustion: null argument");
  if (stage < 0 || stage > 1) return arg_fail("stage index out of range for witsenhausen");
  int64_t d = stage == 0 ? P->d0 : P->d1;
  if (begin < 0 || end > d || begin > end) return arg_fail("exhaustion: bad shard");
  int64_t n = end - begin;
  if (n == 0) return UCP_OK;
  cudaStream_t st = as_stream(stream);
  if (stage == 1) {
    void* pm;
    if ((rc = ws_get(ws, WS_MOM, sizeof(double) * 3 * (size_t)n, &pm))) return rc;
    double* m0 = (double*)pm;
    if ((rc = run_moments(P->y1 + begin, n, P->y0, u0, P->fw0, P->d0, P->a1, P->h1, P->d1, m0, m0 + n,
                          m0 + 2 * n, ws, st, (P->flags & UCP_WC_TABLE) ? begin : -1)))
      return rc;
    k_ex1<<<nblocks(n, 256), 256, 0, st>>>(u1, m0, m0 + n, m0 + 2 * n, win_lo, win_hi, begin, n, out, err,
                                           kNoBatch);
    UCP_LAUNCHED("k_ex1");
    return UCP_OK;
  }
  void *pcount, *ptotal;
  if ((rc = ws_get(ws, WS_COUNT, sizeof(int64_t) * (size_t)(n + 1), &pcount))) return rc;
  if ((rc = ws_get(ws, WS_TOTAL, sizeof(int64_t) * 2, &ptotal))) return rc;
  int64_t* counts = (int64_t*)pcount;  // counts[0..n) -> exclusive offsets[0..n]
  k_ex_count<<<nblocks(n, 256), 256, 0, st>>>(u0, win_lo, win_hi, begin, n, counts);
  UCP_LAUNCHED("k_ex_count");
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, counts, counts, n + 1, st);
  if (ws->scan_cap < tmp_bytes) {
    std::unique_lock<std::shared_mutex> lk(g_capture_mu);
    if (ws->scan_tmp) UCP_CHECK(cudaFree(ws->scan_tmp));
    UCP_CHECK(cudaMalloc(&ws->scan_tmp, tmp_bytes));
    ws->scan_cap = tmp_bytes;
  }
  // counts[n] is scratch: the scan over n+1 items leaves the total in it
  UCP_CHECK(cudaMemsetAsync(counts + n, 0, sizeof(int64_t), st));
  UCP_CHECK(cub::DeviceScan::ExclusiveSum(ws->scan_tmp, tmp_bytes, counts, counts, n + 1, st));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  // The candidate count lives on the device.  With a host-known upper bound
  // (sum of window widths) that fits the budget, size everything for the
  // bound and let the kernels read the true count: no host round trip, so a
  // whole block of phases stays queued on the stream.  Otherwise read it back.
  int64_t total;
  if (cand_bound > 0 && cand_bound <= sync_free_max_cand()) {
    total = cand_bound;
  } else {
    UCP_CHECK(cudaMemcpyAsync(ws->h_total, counts + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    UCP_CHECK(cudaStreamSynchronize(st));
    total = *ws->h_total;
  }
  if (total <= 0) total = 1;
  void *ppt, *pj, *pc;
  if ((rc = ws_get(ws, WS_CAND_PT, sizeof(int32_t) * (size_t)total, &ppt))) return rc;
  if ((rc = ws_get(ws, WS_CAND_J, sizeof(int32_t) * (size_t)total, &pj))) return rc;
  if ((rc = ws_get(ws, WS_COST, sizeof(double) * (size_t)total, &pc))) return rc;
  if (n <= kWarpFillMaxPoints)
    k_ex_fill_warp<<<nblocks(32 * n, 256), 256, 0, st>>>(u0, win_lo, win_hi, begin, n, counts, (int32_t*)ppt,
                                                        (int32_t*)pj);
  else
    k_ex_fill<<<nblocks(n, 256), 256, 0, st>>>(u0, win_lo, win_hi, begin, n, counts, (int32_t*)ppt,
                                               (int32_t*)pj);
  UCP_LAUNCHED("k_ex_fill");
  if (int rc_ = check_aligned(u1)) return rc_;
  WalkGrid g = make_walk_grid(P->a1, P->h1, P->d1, (int)(P->flags & UCP_WC_FAST));
  if ((rc = attach_vsuf(&g, u1, total, ws, st))) return rc;
  if ((rc = attach_table(&g, P, u1, ws, st))) return rc;
  UCP_WALK_LAUNCH(k_ex0_eval, total, nblocks(total, kWalkThreads), st, P->d1, P->y0, P->f0, u0, P->k, u1, g, counts + n,
                                                  (const int32_t*)ppt, (const int32_t*)pj, (double*)pc, kNoBatch);
  UCP_LAUNCHED("k_ex0_eval");
  k_ex_argmin<<<nblocks(n, 256), 256, 0, st>>>(u0, (const double*)pc, counts, (const int32_t*)pj, begin, n,
                                               out, err, kNoBatch, 0);
  UCP_LAUNCHED("k_ex_argmin");
  return UCP_OK;
}

int ucp_wc_run_block(const ucp_wc_problem* P, int kind, int iters, double* u0, double* u1,
                     const ucp_local_params* lp, const int64_t* win_lo0, const int64_t* win_hi0,
                     const int64_t* win_lo1, const int64_t* win_hi1, int64_t cand_bound0, double* scratch0,
                     double* scratch1, int64_t* err, ucp_workspace* ws, void* stream) {
  int rc = check_problem(P);
  if (rc) return rc;
  if (kind < 0 || kind > 1 || iters < 0) return arg_fail("run_block: bad kind/iters");
  if (!u0 || !u1 || !scratch0 || !scratch1 || !err || !ws) return arg_fail("run_block: null argument");
  if (kind == 0 && !lp) return arg_fail("run_block: local params missing");
  if (kind == 1 && (!win_lo0 || !win_hi0 || !win_lo1 || !win_hi1)) return arg_fail("run_block: windows missing");
  cudaStream_t st = as_stream(stream);
  double* u[2] = {u0, u1};
  double* scratch[2] = {scratch0, scratch1};
  const int64_t d[2] = {P->d0, P->d1};
  const int64_t* lo[2] = {win_lo0, win_lo1};
  const int64_t* hi[2] = {win_hi0, win_hi1};
  // solver.py:226-231: every phase reads the latest controllers; the new
  // vector is written to scratch (the sweep reads the old one) and copied back
  for (int it = 0; it < iters; ++it) {
    for (int m = 0; m < 2; ++m) {
      int64_t* e = err + 3 * (2 * (int64_t)it + m);
      if (kind == 0)
        rc = ucp_wc_local_update(P, m, u0, u1, lp + m, 0, d[m], scratch[m], e, ws, stream);
      else
        rc = ucp_wc_exhaustion(P, m, u0, u1, lo[m], hi[m], m == 0 ? cand_bound0 : 0, 0, d[m], scratch[m], e, ws,
                               stream);
      if (rc) return rc;
      UCP_CHECK(cudaMemcpyAsync(u[m], scratch[m], sizeof(double) * (size_t)d[m], cudaMemcpyDeviceToDevice, st));
    }
  }
  return UCP_OK;
}

// One block iteration (both stages) on stream st; err6 = 3 slots per stage,
// shared by every iteration (minimum over the block).
static int block_iteration(const ucp_wc_problem* P, int kind, double* u0, double* u1, const ucp_local_params* lp,
                           const int64_t* const lo[2], const int64_t* const hi[2], int64_t cand_bound0,
                           double* const scratch[2], int64_t* err6, ucp_workspace* ws, cudaStream_t st) {
  double* u[2] = {u0, u1};
  const int64_t d[2] = {P->d0, P->d1};
  for (int m = 0; m < 2; ++m) {
    int rc;
    if (kind == 0)
      rc = ucp_wc_local_update(P, m, u0, u1, lp + m, 0, d[m], scratch[m], err6 + 3 * m, ws, st);
    else
      rc = ucp_wc_exhaustion(P, m, u0, u1, lo[m], hi[m], m == 0 ? cand_bound0 : 0, 0, d[m], scratch[m], err6 + 3 * m,
                             ws, st);
    if (rc) return rc;
    UCP_CHECK(launch_pdl(k_copy, dim3(nblocks(d[m], 256)), dim3(256), 0, st, (const double*)scratch[m], u[m], d[m]));
  }
  return UCP_OK;
}

int ucp_wc_run_block_graph(const ucp_wc_problem* P, int kind, int iters, double* u0, double* u1,
                           const ucp_local_params* lp, const int64_t* win_lo0, const int64_t* win_hi0,
                           const int64_t* win_lo1, const int64_t* win_hi1, int64_t cand_bound0, double* scratch0,
                           double* scratch1, int64_t* err6, ucp_workspace* ws, void* stream) {
  int rc = check_problem(P);
  if (rc) return rc;
  if (kind < 0 || kind > 1 || iters < 0) return arg_fail("run_block_graph: bad kind/iters");
  if (!u0 || !u1 || !scratch0 || !scratch1 || !err6 || !ws) return arg_fail("run_block_graph: null argument");
  if (kind == 0 && !lp) return arg_fail("run_block_graph: local params missing");
  if (kind == 1 && (!win_lo0 || !win_hi0 || !win_lo1 || !win_hi1))
    return arg_fail("run_block_graph: windows missing");
  if (iters == 0) return UCP_OK;
  cudaStream_t st = as_stream(stream);
  const int64_t* lo[2] = {win_lo0, win_lo1};
  const int64_t* hi[2] = {win_hi0, win_hi1};
  double* scratch[2] = {scratch0, scratch1};
  // the first iteration runs eagerly: it sizes every workspace buffer, so the
  // captured iteration never allocates (and proves the launch sequence)
  if ((rc = block_iteration(P, kind, u0, u1, lp, lo, hi, cand_bound0, scratch, err6, ws, st))) return rc;
  if (iters == 1) return UCP_OK;
  const bool graphable = kind == 0 || (cand_bound0 > 0 && cand_bound0 <= sync_free_max_cand());
  if (!graphable) {  // exhaustion that must read its candidate count back: stay eager
    for (int it = 1; it < iters; ++it)
      if ((rc = block_iteration(P, kind, u0, u1, lp, lo, hi, cand_bound0, scratch, err6, ws, st))) return rc;
    return UCP_OK;
  }
  std::array<uint64_t, kGraphKeyWords> key{};
  key[0] = (uint64_t)kind;
  key[1] = (uint64_t)(uintptr_t)P;
  key[2] = (uint64_t)(uintptr_t)u0;
  key[3] = (uint64_t)(uintptr_t)u1;
  key[4] = (uint64_t)(uintptr_t)scratch0;
  key[5] = (uint64_t)(uintptr_t)scratch1;
  key[6] = (uint64_t)(uintptr_t)err6;
  key[7] = (uint64_t)(uintptr_t)win_lo0;
  key[8] = (uint64_t)(uintptr_t)win_hi0;
  key[9] = (uint64_t)(uintptr_t)win_lo1;
  key[10] = (uint64_t)(uintptr_t)win_hi1;
  key[11] = (uint64_t)cand_bound0;
  if (lp) {
    const double* lv = reinterpret_cast<const double*>(lp);
    for (int k = 0; k < 8; ++k) key[12 + k] = ucp_asu64(lv[k]);
  }
  // captured walk grids bake in the node-counter pointer
  key[20] = (uint64_t)(uintptr_t)g_visits.load(std::memory_order_acquire);
  cudaGraphExec_t exec = nullptr;
  int64_t kernels = 0;
  for (auto& g : ws->graphs)
    if (!g.stale && g.key == key) {
      exec = g.exec;
      kernels = g.kernels;
    }
  if (!exec) {
    if (!ws->cap_stream) UCP_CHECK(cudaStreamCreateWithFlags(&ws->cap_stream, cudaStreamNonBlocking));
    std::shared_lock<std::shared_mutex> lk(g_capture_mu);
    UCP_CHECK(cudaStreamBeginCapture(ws->cap_stream, cudaStreamCaptureModeThreadLocal));
    rc = block_iteration(P, kind, u0, u1, lp, lo, hi, cand_bound0, scratch, err6, ws, ws->cap_stream);
    cudaGraph_t graph = nullptr;
    cudaError_t ec = cudaStreamEndCapture(ws->cap_stream, &graph);
    if (rc) {
      if (graph) cudaGraphDestroy(graph);
      return rc;
    }
    if (ec != cudaSuccess) return cuda_fail(ec, "cudaStreamEndCapture");
    // kernel nodes of one iteration (the launch counter adds them per replay)
    size_t nn = 0;
    cudaGraphGetNodes(graph, nullptr, &nn);
    std::vector<cudaGraphNode_t> nodes(nn);
    if (nn) cudaGraphGetNodes(graph, nodes.data(), &nn);
    for (size_t q = 0; q < nn; ++q) {
      cudaGraphNodeType t;
      if (cudaGraphNodeGetType(nodes[q], &t) == cudaSuccess && t == cudaGraphNodeTypeKernel) ++kernels;
    }
    // a recycled workspace's graph of the same shape (a previous problem's)
    // takes the new parameters by an in-place update, far cheaper than a new
    // instantiation; otherwise instantiate
    for (size_t q = 0; q < ws->graphs.size() && !exec;) {
      auto& g = ws->graphs[q];
      if (!g.stale || g.key[0] != key[0] || g.kernels != kernels) {
        ++q;
        continue;
      }
      cudaGraphExecUpdateResultInfo info;
      if (cudaGraphExecUpdate(g.exec, graph, &info) == cudaSuccess) {
        g.key = key;
        g.stale = false;
        exec = g.exec;
      } else {  // not updatable (another shape): drop it (recycling synchronised: not in flight)
        cudaGetLastError();
        cudaGraphExecDestroy(g.exec);
        ws->graphs.erase(ws->graphs.begin() + (std::ptrdiff_t)q);
      }
    }
    if (!exec) {
      ec = cudaGraphInstantiate(&exec, graph, 0);
      if (ec != cudaSuccess) {
        cudaGraphDestroy(graph);
        return cuda_fail(ec, "cudaGraphInstantiate");
      }
      ws->graphs.push_back({key, exec, kernels, false});
    }
    cudaGraphDestroy(graph);
  }
  for (int it = 1; it < iters; ++it) {
    UCP_CHECK(cudaGraphLaunch(exec, st));
    g_launches.fetch_add(kernels, std::memory_order_relaxed);
  }
  return UCP_OK;
}

int ucp_wc_objective_terms(const ucp_wc_problem* P, const double* u0, const double* u1, int64_t begin,
                           int64_t end, double* terms, int64_t* err, void* stream) {
  return ucp_wc_objective_terms_ws(P, u0, u1, begin, end, terms, err, nullptr, stream);
}

int ucp_wc_objective_terms_ws(const ucp_wc_problem* P, const double* u0, const double* u1, int64_t begin,
                              int64_t end, double* terms, int64_t* err, ucp_workspace* ws, void* stream) {
  int rc = check_problem(P);
  if (rc) return rc;
  if (begin < 0 || end > P->d0 || begin > end) return arg_fail("objective_terms: bad shard");
  if (end == begin) return UCP_OK;
  if (int rc_ = check_aligned(u1)) return rc_;
  WalkGrid g = make_walk_grid(P->a1, P->h1, P->d1, (int)(P->flags & UCP_WC_FAST));
  // with a workspace: the walks' no-op tail exit (result-invariant, as in the
  // phases) and, under UCP_WC_TABLE, the integrand from the expansion cells
  // (with the reference walk's bias, ex_moments)
  if (ws && (rc = attach_vsuf(&g, u1, end - begin, ws, as_stream(stream)))) return rc;
  if (ws && (rc = attach_table(&g, P, u1, ws, as_stream(stream)))) return rc;
  UCP_WALK_LAUNCH(k_obj_terms, end - begin, nblocks(end - begin, kWalkThreads), as_stream(stream), P->d1, P->y0, P->f0, u0, P->k, u1, g,
                                                                          begin, end, terms, err, kNoBatch);
  UCP_LAUNCHED("k_obj_terms");
  return UCP_OK;
}

int ucp_walk_node_counter(unsigned long long* counter) {
  g_visits.store(counter, std::memory_order_release);
  return UCP_OK;
}

int ucp_fp64_probe(int blocks, int threads, int iters, double* sink, void* stream) {
  if (blocks <= 0 || threads <= 0 || iters <= 0) return arg_fail("fp64_probe: bad sizes");
  k_fp64_probe<<<blocks, threads, 0, as_stream(stream)>>>(iters, sink);
  UCP_LAUNCHED("k_fp64_probe");
  return UCP_OK;
}

}  // extern "C"

#include "ucp_config5.cuh"
#include "ucp_mc.cuh"
#include "ucp_batch.cuh"
#include "ucp_comm.cuh"
