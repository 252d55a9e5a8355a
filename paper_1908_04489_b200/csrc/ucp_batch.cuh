// Batched multi-instance engine (config 4).
//
// B Witsenhausen instances on the same grids (k and sigma free) live in HBM
// as rows: u0[B][ld0], u1[B][ld1], f0/fw0[B][ld0], k[B].  One call advances a
// set of instances ("slots") by whole block iterations -- every kernel of the
// single-instance path runs ONCE for all slots, over (slot, point) grids
// (blockIdx.y = slot), so d = 2000 instances that leave the GPU idle alone
// fill it together.  Per-instance arithmetic is the single-instance path's
// (same device functions, same order): every instance's result is bitwise
// what solve() gives it alone.  The host driver (batch.py) runs each
// instance's own round schedule (reference solver.py:234-290); a "lane" is a
// scratch set, so the local-update group and the exhaustion group of one
// tick run concurrently on two streams.

struct ucp_wc_batch {
  ucp_wc_batch_desc D;
  int64_t cbpad = 0;  // per-slot candidate capacity (cand_bound0, CTA multiple)
  struct Lane {
    int32_t* ids = nullptr;
    double *scratch0 = nullptr, *scratch1 = nullptr, *cost3 = nullptr, *mom = nullptr, *terms = nullptr;
    double *x1 = nullptr, *costs = nullptr;
    double2 *tails = nullptr, *xw = nullptr, *tile_mm = nullptr;
    int64_t *offs = nullptr, *totals = nullptr, *counts = nullptr, *chunk_tot = nullptr;
    int32_t *cand_pt = nullptr, *cand_j = nullptr;
    int* counter = nullptr;
    double* vsuf = nullptr;  // per-slot tail-exit tables of u1 (walk_tail_noop)
  } lane[2];
  int64_t vstride = 0;  // doubles per slot table
  std::vector<void*> allocs;
};

namespace {

constexpr int kMaxBatchIds = 1024;
#ifndef UCP_BATCH_MOM_UNROLL
#define UCP_BATCH_MOM_UNROLL 8
#endif
constexpr int kBatchMomUnroll = UCP_BATCH_MOM_UNROLL;
#ifndef UCP_BATCH_MOM_QT
#define UCP_BATCH_MOM_QT 128
#endif
#ifndef UCP_BATCH_MOM_MINB
#define UCP_BATCH_MOM_MINB 3
#endif
constexpr int kBatchMomQT = UCP_BATCH_MOM_QT;  // queries per CTA work item
#ifndef UCP_BATCH_FUSED_MAX
#define UCP_BATCH_FUSED_MAX 6000
#endif
constexpr int64_t kBatchFusedMaxQueries = UCP_BATCH_FUSED_MAX;  // slots x queries for the fused moments
constexpr int kBatchMomMinB = UCP_BATCH_MOM_MINB;
struct IdList {
  int32_t v[kMaxBatchIds];
};

__global__ void k_set_ids(const IdList ids, int n, int32_t* out) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = ids.v[i];
}

// row copy scratch[slot][0..n) -> dst[ids[slot] * ld ...]
__global__ void k_bcopy(const double* __restrict__ src, int64_t n, double* __restrict__ dst, int64_t ld,
                        const int32_t* __restrict__ ids) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  dst[(int64_t)ids[blockIdx.y] * ld + i] = src[(int64_t)blockIdx.y * n + i];
}

// Exhaustion candidates, (chunk of kCandThreads points, slot) per CTA:
// k_bex_count counts each point's candidates (adjacent repeats collapsed, as
// k_ex_count) and the chunk total; k_bex_fill takes its chunk's base from
// the preceding chunk totals, block-scans the counts and fills (as k_ex_fill).
constexpr int kCandThreads = 256;
__device__ __forceinline__ int64_t window_count(const double* __restrict__ u, int64_t j0, int64_t j1) {
  int64_t c = 1;
  double prev = u[j0];
  for (int64_t j = j0 + 1; j <= j1; ++j) {
    const double x = u[j];
    c += (x != prev);
    prev = x;
  }
  return c;
}

__global__ void __launch_bounds__(kCandThreads) k_bex_count(const double* __restrict__ u0, const int64_t* __restrict__ lo,
                                                            const int64_t* __restrict__ hi, int64_t d0,
                                                            const BatchArgs B, int64_t* counts, int64_t* chunk_tot) {
  using Reduce = cub::BlockReduce<int64_t, kCandThreads>;
  __shared__ typename Reduce::TempStorage tmp;
  const int slot = blockIdx.y;
  const double* u = u0 + (int64_t)B.inst(slot) * B.su0;
  const int64_t i = (int64_t)blockIdx.x * kCandThreads + threadIdx.x;
  const int64_t c = i < d0 ? window_count(u, lo[i], hi[i]) : 0;
  if (i < d0) counts[(int64_t)slot * d0 + i] = c;
  const int64_t tot = Reduce(tmp).Sum(c);
  if (threadIdx.x == 0) chunk_tot[(int64_t)slot * gridDim.x + blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kCandThreads) k_bex_fill(const double* __restrict__ u0, const int64_t* __restrict__ lo,
                                                           const int64_t* __restrict__ hi, int64_t d0,
                                                           const BatchArgs B, const int64_t* __restrict__ counts,
                                                           const int64_t* __restrict__ chunk_tot, int64_t* offs,
                                                           int64_t* totals, int32_t* cand_pt, int32_t* cand_j) {
  using Scan = cub::BlockScan<int64_t, kCandThreads>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int64_t s_base;
  const int slot = blockIdx.y;
  const double* u = u0 + (int64_t)B.inst(slot) * B.su0;
  offs += (int64_t)slot * (d0 + 1);
  cand_pt += (int64_t)slot * B.sslot;
  cand_j += (int64_t)slot * B.sslot;
  if (threadIdx.x == 0) {
    int64_t base = 0;
    for (unsigned c = 0; c < blockIdx.x; ++c) base += chunk_tot[(int64_t)slot * gridDim.x + c];
    s_base = base;
  }
  UCP_SYNC();
  const int64_t i = (int64_t)blockIdx.x * kCandThreads + threadIdx.x;
  const int64_t c = i < d0 ? counts[(int64_t)slot * d0 + i] : 0;
  int64_t pos, agg;
  Scan(tmp).ExclusiveSum(c, pos, agg);
  pos += s_base;
  UCP_DCHECK(pos + c <= B.sslot);
  if (i < d0) {
    offs[i] = pos;
    const int64_t j0 = lo[i];
    double prev = u[j0];
    cand_pt[pos] = (int32_t)i;
    cand_j[pos] = (int32_t)j0;
    ++pos;
    for (int64_t j = j0 + 1; j <= hi[i]; ++j) {
      const double x = u[j];
      if (x != prev) {
        cand_pt[pos] = (int32_t)i;
        cand_j[pos] = (int32_t)j;
        ++pos;
      }
      prev = x;
    }
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
    offs[d0] = s_base + agg;
    totals[slot] = s_base + agg;
  }
}

#define UCP_WALK_LAUNCH_B(kernel, n_walks, grid, stream, d_v1, ...)                                       \
  do {                                                                                                  \
    if (!walk_latency_mode(n_walks)) {                                                                  \
      kernel<0, true><<<(grid), kWalkThreads, 0, (stream)>>>(__VA_ARGS__);                              \
    } else if ((d_v1) <= kSmemWalkMax) {                                                                \
      allow_smem(kernel<2, true>);                                                                      \
      kernel<2, true><<<(grid), kWalkThreads, (size_t)(d_v1) * sizeof(double), (stream)>>>(__VA_ARGS__); \
    } else {                                                                                            \
      kernel<1, true><<<(grid), kWalkThreads, 0, (stream)>>>(__VA_ARGS__);                              \
    }                                                                                                   \
  } while (0)

template <class T>
int balloc(ucp_wc_batch* b, T** p, size_t count) {
  void* q = nullptr;
  UCP_CHECK(cudaMalloc(&q, sizeof(T) * (count > 0 ? count : 1)));
  b->allocs.push_back(q);
  *p = (T*)q;
  return UCP_OK;
}

BatchArgs batch_args(const ucp_wc_batch* b, const int32_t* ids, int64_t sslot) {
  return BatchArgs{ids, b->D.ld0, b->D.ld1, sslot, 6, b->D.k};
}

// stage-1 moments of every slot's x1 = y0 + u0 at the shared queries y1
int batch_moments(ucp_wc_batch* b, ucp_wc_batch::Lane& L, int S, cudaStream_t st) {
  const ucp_wc_batch_desc& D = b->D;
  const int64_t m = D.d0, ntiles = (m + kTile - 1) / kTile;
  const BatchArgs B = batch_args(b, L.ids, 0);
  k_x1_prepare<<<dim3((unsigned)ntiles, S), kTile, 0, st>>>(D.y0, D.u0, D.fw0, m, D.a1, D.h1,
                                                            D.a1 + D.h1 * (double)(D.d1 - 1), L.x1, L.xw, L.tails,
                                                            L.tile_mm, B);
  UCP_LAUNCHED("k_x1_prepare");
  if ((int64_t)S * D.d1 <= kBatchFusedMaxQueries) {
    // few slots (the tail of a sweep): the latency-oriented fused kernel
    smem_opt_in(reinterpret_cast<const void*>(k_mom_fused), kFSmem);
    k_mom_fused<<<dim3(nblocks(D.d1, kFQ), S), kFThreads, kFSmem, st>>>(D.y1, D.d1, L.x1, D.fw0, L.tails, L.tile_mm, m,
                                                                      D.a1, D.h1, D.d1, L.mom, L.mom + D.d1,
                                                                      L.mom + 2 * D.d1, L.ids, D.ld0, 3 * D.d1);
    UCP_LAUNCHED("k_mom_fused");
    return UCP_OK;
  }
  UCP_CHECK(cudaMemsetAsync(L.counter, 0, sizeof(int), st));
  int dev = 0, sms = 0, per_sm = 0;
  UCP_CHECK(cudaGetDevice(&dev));
  UCP_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  UCP_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &per_sm, k_moments<kBatchMomUnroll, kBatchMomMinB, kBatchMomQT>, kBatchMomQT, 0));
  const int64_t nitems = (int64_t)S * ((D.d1 + kBatchMomQT - 1) / kBatchMomQT);
  int64_t grid = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
  if (grid > nitems) grid = nitems;
  k_moments<kBatchMomUnroll, kBatchMomMinB, kBatchMomQT><<<(unsigned)grid, kBatchMomQT, 0, st>>>(D.y1, D.d1, L.xw, L.tails, m, L.tile_mm, D.a1, D.h1, D.d1, L.mom,
                                                    L.mom + D.d1, L.mom + 2 * D.d1, L.counter, S, 3 * D.d1);
  UCP_LAUNCHED("k_moments");
  return UCP_OK;
}

// Throughput-mode walks of every slot stop at their no-op tail as in the
// single-instance path (attach_vsuf): one table per slot, built from that
// slot's instance u1 (the walks' v1) before the stage-0 kernels read it.
void batch_attach_vsuf(ucp_wc_batch* b, ucp_wc_batch::Lane& L, WalkGrid* g, int S, int64_t n_walks, cudaStream_t st) {
  if (!g_tail_exit || walk_latency_mode(n_walks)) return;
  k_vsuf<<<S, 1024, 0, st>>>(b->D.u1, g->d, g->nb, L.vsuf, L.ids, b->D.ld1, b->vstride);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  g->vsuf = L.vsuf;
  g->vstride = b->vstride;
}

int batch_iteration(ucp_wc_batch* b, ucp_wc_batch::Lane& L, int kind, int S, int64_t* err, cudaStream_t st) {
  const ucp_wc_batch_desc& D = b->D;
  const int64_t d0 = D.d0, d1 = D.d1;
  WalkGrid g = make_walk_grid(D.a1, D.h1, D.d1);
  batch_attach_vsuf(b, L, &g, S, kind == 0 ? S * 3 * d0 : S * b->cbpad, st);  // the widest walk launch
  int rc;
  // ---- stage 0
  if (kind == 0) {
    const BatchArgs B = batch_args(b, L.ids, 3 * d0);
    UCP_WALK_LAUNCH_B(k_lu0_probe, S * 3 * d0, dim3(nblocks(3 * d0, kWalkThreads), S), st, d1, D.y0, D.f0, D.u0, 0.0,
                      D.u1, g, D.lp0.fd_step, 0, d0, L.cost3, B);
    UCP_LAUNCHED("k_lu0_probe");
    UCP_WALK_LAUNCH_B(k_lu0_finish, S * d0, dim3(nblocks(d0, kWalkThreads), S), st, d1, D.y0, D.f0, D.u0, 0.0, D.u1,
                      g, D.lp0, 0, d0, L.cost3, L.scratch0, err, B);
    UCP_LAUNCHED("k_lu0_finish");
  } else {
    const BatchArgs B = batch_args(b, L.ids, b->cbpad);
    const dim3 cgrid(nblocks(d0, kCandThreads), S);
    k_bex_count<<<cgrid, kCandThreads, 0, st>>>(D.u0, D.win_lo0, D.win_hi0, d0, B, L.counts, L.chunk_tot);
    UCP_LAUNCHED("k_bex_count");
    k_bex_fill<<<cgrid, kCandThreads, 0, st>>>(D.u0, D.win_lo0, D.win_hi0, d0, B, L.counts, L.chunk_tot, L.offs,
                                               L.totals, L.cand_pt, L.cand_j);
    UCP_LAUNCHED("k_bex_fill");
    UCP_WALK_LAUNCH_B(k_ex0_eval, S * b->cbpad, dim3(nblocks(b->cbpad, kWalkThreads), S), st, d1, D.y0, D.f0, D.u0,
                      0.0, D.u1, g, L.totals, L.cand_pt, L.cand_j, L.costs, B);
    UCP_LAUNCHED("k_ex0_eval");
    k_ex_argmin<<<dim3(nblocks(d0, 256), S), 256, 0, st>>>(D.u0, L.costs, L.offs, L.cand_j, 0, d0, L.scratch0, err,
                                                           B, d0 + 1);
    UCP_LAUNCHED("k_ex_argmin");
  }
  k_bcopy<<<dim3(nblocks(d0, 256), S), 256, 0, st>>>(L.scratch0, d0, D.u0, D.ld0, L.ids);
  UCP_LAUNCHED("k_bcopy");
  // ---- stage 1 (reads the new u0)
  if ((rc = batch_moments(b, L, S, st))) return rc;
  const BatchArgs B1 = batch_args(b, L.ids, 3 * d1);
  if (kind == 0)
    k_lu1<<<dim3(nblocks(d1, 256), S), 256, 0, st>>>(D.u1, L.mom, L.mom + d1, L.mom + 2 * d1, D.lp1, 0, d1, L.scratch1,
                                                     err + 3, B1);
  else
    k_ex1<<<dim3(nblocks(d1, 256), S), 256, 0, st>>>(D.u1, L.mom, L.mom + d1, L.mom + 2 * d1, D.win_lo1, D.win_hi1, 0,
                                                     d1, L.scratch1, err + 3, B1);
  UCP_LAUNCHED("k_lu1/k_ex1");
  k_bcopy<<<dim3(nblocks(d1, 256), S), 256, 0, st>>>(L.scratch1, d1, D.u1, D.ld1, L.ids);
  UCP_LAUNCHED("k_bcopy");
  return UCP_OK;
}

int batch_set_ids(ucp_wc_batch::Lane& L, const int32_t* ids, int32_t n, int64_t B, cudaStream_t st) {
  if (!ids || n < 1 || n > kMaxBatchIds || n > B) return arg_fail("batch: bad instance list");
  IdList p;
  for (int i = 0; i < n; ++i) {
    if (ids[i] < 0 || ids[i] >= B) return arg_fail("batch: instance index out of range");
    p.v[i] = ids[i];
  }
  k_set_ids<<<1, 256, 0, st>>>(p, n, L.ids);
  UCP_LAUNCHED("k_set_ids");
  return UCP_OK;
}

}  // namespace

extern "C" {

int ucp_wc_batch_create(const ucp_wc_batch_desc* desc, ucp_wc_batch** out) {
  if (!desc || !out) return arg_fail("batch_create: null argument");
  const ucp_wc_batch_desc& D = *desc;
  if (D.instances < 1 || D.instances > kMaxBatchIds) return arg_fail("batch_create: 1..1024 instances");
  if (D.d0 < 2 || D.d1 < 2 || D.ld0 < D.d0 || D.ld1 < D.d1 || (D.ld1 & 1) || (D.ld0 & 1))
    return arg_fail("batch_create: bad grid sizes / strides (strides must be even)");
  if (!D.y0 || !D.y1 || !D.u0 || !D.u1 || !D.f0 || !D.fw0 || !D.k || !D.win_lo0 || !D.win_hi0 || !D.win_lo1 ||
      !D.win_hi1)
    return arg_fail("batch_create: null device array");
  if (int rc_ = check_aligned(D.u1)) return rc_;
  if (D.cand_bound0 < D.d0 || D.d0 > INT32_MAX) return arg_fail("batch_create: bad candidate bound");
  ucp_wc_batch* b = new ucp_wc_batch();
  b->D = D;
  b->cbpad = (D.cand_bound0 + kWalkThreads - 1) / kWalkThreads * kWalkThreads;
  const int64_t B = D.instances, d0 = D.d0, d1 = D.d1, ntiles = (d0 + kTile - 1) / kTile;
  int rc = UCP_OK;
  for (int l = 0; l < 2 && rc == UCP_OK; ++l) {
    auto& L = b->lane[l];
    if ((rc = balloc(b, &L.ids, B)) || (rc = balloc(b, &L.scratch0, B * d0)) || (rc = balloc(b, &L.scratch1, B * d1)) ||
        (rc = balloc(b, &L.cost3, B * 3 * d0)) || (rc = balloc(b, &L.mom, B * 3 * d1)) ||
        (rc = balloc(b, &L.terms, B * d0)) || (rc = balloc(b, &L.x1, B * d0)) || (rc = balloc(b, &L.tails, B * d0)) ||
        (rc = balloc(b, &L.xw, B * ntiles * kTile)) || (rc = balloc(b, &L.tile_mm, B * ntiles)) ||
        (rc = balloc(b, &L.counter, 1)))
      break;
    const int nb1 = (int)((d1 + (1 << kVsufShift) - 1) >> kVsufShift);
    b->vstride = (int64_t)nb1 * vsuf_levels(nb1);
    if ((rc = balloc(b, &L.vsuf, B * b->vstride))) break;
    if (l == 1 && ((rc = balloc(b, &L.costs, B * b->cbpad)) || (rc = balloc(b, &L.offs, B * (d0 + 1))) ||
                   (rc = balloc(b, &L.totals, B)) || (rc = balloc(b, &L.counts, B * d0)) ||
                   (rc = balloc(b, &L.chunk_tot, B * ((d0 + kCandThreads - 1) / kCandThreads))) || (rc = balloc(b, &L.cand_pt, B * b->cbpad)) ||
                   (rc = balloc(b, &L.cand_j, B * b->cbpad))))
      break;
  }
  if (rc) {
    for (void* p : b->allocs) cudaFree(p);
    delete b;
    return rc;
  }
  *out = b;
  return UCP_OK;
}

int ucp_wc_batch_destroy(ucp_wc_batch* b) {
  if (!b) return UCP_OK;
  std::unique_lock<std::shared_mutex> lk(g_capture_mu);
  cudaDeviceSynchronize();
  for (void* p : b->allocs) cudaFree(p);
  delete b;
  return UCP_OK;
}

int ucp_wc_batch_iterate(ucp_wc_batch* b, int lane, int kind, const int32_t* ids, int32_t nslots, int iters,
                         int64_t* err, void* stream) {
  if (!b || !err) return arg_fail("batch_iterate: null argument");
  if (lane < 0 || lane > 1 || kind < 0 || kind > 1 || iters < 0) return arg_fail("batch_iterate: bad lane/kind/iters");
  if (kind == 1 && lane != 1) return arg_fail("batch_iterate: exhaustion runs on lane 1");
  if (iters == 0 || nslots == 0) return UCP_OK;
  cudaStream_t st = as_stream(stream);
  auto& L = b->lane[lane];
  int rc;
  if ((rc = batch_set_ids(L, ids, nslots, b->D.instances, st))) return rc;
  for (int it = 0; it < iters; ++it)
    if ((rc = batch_iteration(b, L, kind, nslots, err, st))) return rc;
  return UCP_OK;
}

int ucp_wc_batch_objective(ucp_wc_batch* b, int lane, const int32_t* ids, int32_t nslots, double* J,
                           int64_t* err_obj, void* stream) {
  if (!b || !J || !err_obj) return arg_fail("batch_objective: null argument");
  if (lane < 0 || lane > 1) return arg_fail("batch_objective: bad lane");
  if (nslots == 0) return UCP_OK;
  cudaStream_t st = as_stream(stream);
  auto& L = b->lane[lane];
  int rc;
  if ((rc = batch_set_ids(L, ids, nslots, b->D.instances, st))) return rc;
  const ucp_wc_batch_desc& D = b->D;
  const int64_t d0 = D.d0;
  WalkGrid g = make_walk_grid(D.a1, D.h1, D.d1);
  batch_attach_vsuf(b, L, &g, nslots, nslots * d0, st);
  BatchArgs B = batch_args(b, L.ids, d0);
  B.serr = 1;
  UCP_WALK_LAUNCH_B(k_obj_terms, nslots * d0, dim3(nblocks(d0, kWalkThreads), nslots), st, D.d1, D.y0, D.f0, D.u0,
                    0.0, D.u1, g, 0, d0, L.terms, err_obj, B);
  UCP_LAUNCHED("k_obj_terms");
  k_trapezoid<<<nslots, kTrapThreads, 0, st>>>(L.terms, d0, D.h0, J, err_obj, B);
  UCP_LAUNCHED("k_trapezoid");
  return UCP_OK;
}

}  // extern "C"
