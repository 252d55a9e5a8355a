// NCCL plumbing for hosts that are not Python (ucp_comm_init,
// ucp_allgather_f64).  The Python host uses torch.distributed for the same two
// exchanges (distributed.py); a C/C++ integrator drives them through these
// entry points: one communicator per rank (one process per GPU), the
// in-place all-gather of each phase's controller shard and the MIN all-reduce
// of the error slots.
//
// NCCL is resolved at run time with dlopen/dlsym instead of being linked: the
// process may already hold PyTorch's bundled libnccl.so.2 (a different
// version than the system one), and a second copy under the same soname must
// not be pulled in.  RTLD_NOLOAD first reuses whatever is loaded.
#include <dlfcn.h>
#include <nccl.h>

struct ucp_comm {
  ncclComm_t comm = nullptr;
  int nranks = 0, rank = 0;
};

namespace {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  bool ok = false;
};

const NcclApi& nccl_api() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    a.init_rank = reinterpret_cast<decltype(a.init_rank)>(dlsym(h, "ncclCommInitRank"));
    a.destroy = reinterpret_cast<decltype(a.destroy)>(dlsym(h, "ncclCommDestroy"));
    a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(h, "ncclAllGather"));
    a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
    a.broadcast = reinterpret_cast<decltype(a.broadcast)>(dlsym(h, "ncclBroadcast"));
    a.group_start = reinterpret_cast<decltype(a.group_start)>(dlsym(h, "ncclGroupStart"));
    a.group_end = reinterpret_cast<decltype(a.group_end)>(dlsym(h, "ncclGroupEnd"));
    a.ok = a.get_unique_id && a.init_rank && a.destroy && a.all_gather && a.all_reduce && a.error_string &&
           a.broadcast && a.group_start && a.group_end;
    return a;
  }();
  return api;
}

int nccl_fail(ncclResult_t r, const char* where) {
  const NcclApi& a = nccl_api();
  snprintf(g_errbuf, sizeof g_errbuf, "%s: %s", where, a.error_string ? a.error_string(r) : "NCCL error");
  return UCP_ERR_CUDA;
}

int nccl_ready() {
  if (!nccl_api().ok) return arg_fail("NCCL (libnccl.so.2) not available in this process");
  return UCP_OK;
}

}  // namespace

extern "C" {

int ucp_comm_unique_id(unsigned char* id) {
  int rc;
  if (!id) return arg_fail("comm_unique_id: null buffer");
  if ((rc = nccl_ready())) return rc;
  ncclUniqueId u;
  ncclResult_t r = nccl_api().get_unique_id(&u);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  memcpy(id, u.internal, UCP_COMM_ID_BYTES);
  return UCP_OK;
}

int ucp_comm_init(int nranks, int rank, const unsigned char* id, ucp_comm** comm) {
  int rc;
  if (!id || !comm || nranks < 1 || rank < 0 || rank >= nranks) return arg_fail("comm_init: bad arguments");
  if ((rc = nccl_ready())) return rc;
  ncclUniqueId u;
  memcpy(u.internal, id, UCP_COMM_ID_BYTES);
  ucp_comm* c = new ucp_comm();
  ncclResult_t r = nccl_api().init_rank(&c->comm, nranks, u, rank);
  if (r != ncclSuccess) {
    delete c;
    return nccl_fail(r, "ncclCommInitRank");
  }
  c->nranks = nranks;
  c->rank = rank;
  *comm = c;
  return UCP_OK;
}

int ucp_comm_destroy(ucp_comm* comm) {
  if (!comm) return UCP_OK;
  if (comm->comm && nccl_api().ok) nccl_api().destroy(comm->comm);
  delete comm;
  return UCP_OK;
}

int ucp_allgather_f64(ucp_comm* comm, const double* send, double* recv, int64_t count, void* stream) {
  if (!comm || !recv || count < 0 || (count > 0 && !send)) return arg_fail("allgather_f64: bad arguments");
  if (count == 0) return UCP_OK;
  ncclResult_t r = nccl_api().all_gather(send, recv, (size_t)count, ncclFloat64, comm->comm, as_stream(stream));
  if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather");
  return UCP_OK;
}

int ucp_allgatherv_f64(ucp_comm* comm, double* buf, const int64_t* bounds, void* stream) {
  if (!comm || !buf || !bounds) return arg_fail("allgatherv_f64: bad arguments");
  for (int r = 0; r < comm->nranks; ++r)
    if (bounds[r] < 0 || bounds[r + 1] < bounds[r]) return arg_fail("allgatherv_f64: bounds must ascend from 0");
  if (comm->nranks == 1) return UCP_OK;  // the whole vector is this rank's shard
  // one in-place broadcast per rank (root r sends its shard), grouped so NCCL
  // runs them as one collective: the uneven form of ncclAllGather
  const NcclApi& a = nccl_api();
  ncclResult_t r = a.group_start();
  if (r != ncclSuccess) return nccl_fail(r, "ncclGroupStart");
  for (int q = 0; q < comm->nranks; ++q) {
    const size_t n = (size_t)(bounds[q + 1] - bounds[q]);
    if (n == 0) continue;
    double* p = buf + bounds[q];
    r = a.broadcast(p, p, n, ncclFloat64, q, comm->comm, as_stream(stream));
    if (r != ncclSuccess) {
      a.group_end();
      return nccl_fail(r, "ncclBroadcast");
    }
  }
  r = a.group_end();
  if (r != ncclSuccess) return nccl_fail(r, "ncclGroupEnd");
  return UCP_OK;
}

int ucp_allreduce_min_i64(ucp_comm* comm, int64_t* buf, int64_t count, void* stream) {
  if (!comm || count < 0 || (count > 0 && !buf)) return arg_fail("allreduce_min_i64: bad arguments");
  if (count == 0) return UCP_OK;
  ncclResult_t r = nccl_api().all_reduce(buf, buf, (size_t)count, ncclInt64, ncclMin, comm->comm, as_stream(stream));
  if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce");
  return UCP_OK;
}

}  // extern "C"
