// NCCL data plane of the row-partitioned exchange (replaces the reference's gather /
// send / broadcast of dsvd.py:176-202 and its CommStats byte counters, comm.py:74-88).
//
// With a communicator set (psvd_nccl_init + psvd_nccl_enable) every exchange point of the library —
// the streaming Gram and U^T U of the pipelined deterministic stream, the sketch Grams and projections
// of the randomized update, the Gram-deflation sums of the accurate route and of psvd_qr_robust, the
// per-rank argmax pairs of the tall sign rule — is an in-stream ncclAllGather on the library's own
// stream followed by the fixed-order sum (sum_ordered_kernel: bitwise identical on every rank), with
// no host round trip and no Python callback.  libnccl is loaded at run time (dlopen "libnccl.so.2":
// the copy torch already mapped when it is loaded), so the library has no link-time NCCL dependency.
#include <dlfcn.h>

#include <algorithm>
#include <cstring>

#include "psvd_ctx.cuh"

using namespace psvd_internal;

namespace {

typedef struct { char internal[128]; } NcclUniqueId;  // nccl.h: ncclUniqueId (NCCL_UNIQUE_ID_BYTES = 128)
typedef int NcclResult;                                 // ncclResult_t, ncclSuccess = 0
constexpr int kNcclFloat64 = 8;                         // ncclFloat64

struct NcclApi {
  void* handle = nullptr;
  NcclResult (*get_unique_id)(NcclUniqueId*) = nullptr;
  NcclResult (*comm_init_rank)(void**, int, NcclUniqueId, int) = nullptr;
  NcclResult (*all_gather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
  NcclResult (*comm_destroy)(void*) = nullptr;
  const char* (*error_string)(NcclResult) = nullptr;
  bool ok = false;
};

NcclApi& api() {
  static NcclApi a;
  static bool tried = false;
  if (!tried) {
    tried = true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      a.handle = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (a.handle) break;
    }
    if (a.handle) {
      a.get_unique_id = (NcclResult(*)(NcclUniqueId*))dlsym(a.handle, "ncclGetUniqueId");
      a.comm_init_rank = (NcclResult(*)(void**, int, NcclUniqueId, int))dlsym(a.handle, "ncclCommInitRank");
      a.all_gather = (NcclResult(*)(const void*, void*, size_t, int, void*, cudaStream_t))dlsym(a.handle, "ncclAllGather");
      a.comm_destroy = (NcclResult(*)(void*))dlsym(a.handle, "ncclCommDestroy");
      a.error_string = (const char* (*)(NcclResult))dlsym(a.handle, "ncclGetErrorString");
      a.ok = a.get_unique_id && a.comm_init_rank && a.all_gather && a.comm_destroy && a.error_string;
    }
  }
  return a;
}

__global__ void sum_parts_kernel(const double* __restrict__ parts, int P, int64_t count, double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    double s = parts[i];
    for (int r = 1; r < P; ++r) s += parts[(size_t)r * count + i];  // rank order: bitwise identical everywhere
    out[i] = s;
  }
}

}  // namespace

namespace psvd_internal {

bool ex_active(const psvd_ctx* c) { return c->ex_allreduce != nullptr || c->nccl_on; }

int nccl_allgather(psvd_ctx* c, const double* send, int64_t count, double* recv, cudaStream_t st) {
  NcclApi& a = api();
  const NcclResult r = a.all_gather(send, recv, (size_t)count, kNcclFloat64, c->nccl_comm, st);
  c->ex_calls++;
  c->ex_bytes += 8 * count * (c->ex_nranks - 1);
  if (r != 0) return fail(c, PSVD_ECUDA, "ncclAllGather: %s", a.error_string(r));
  return PSVD_OK;
}

int nccl_allreduce_ordered(psvd_ctx* c, double* buf, int64_t count, cudaStream_t st) {
  int rc = ensure(c, c->nccl_parts, sizeof(double) * (size_t)c->ex_nranks * count);
  if (rc) return rc;
  double* parts = (double*)c->nccl_parts.ptr;
  if ((rc = nccl_allgather(c, buf, count, parts, st))) return rc;
  const int64_t blocks = std::min<int64_t>(1024, (count + 255) / 256);
  sum_parts_kernel<<<(unsigned)std::max<int64_t>(1, blocks), 256, 0, st>>>(parts, c->ex_nranks, count, buf);
  c->launches++;
  return cuda_check(c, "ordered sum");
}

}  // namespace psvd_internal

extern "C" {

int psvd_nccl_available(int* ok) {
  if (!ok) return PSVD_EINVAL;
  *ok = api().ok ? 1 : 0;
  return PSVD_OK;
}

int psvd_nccl_unique_id(psvd_ctx* c, unsigned char* id128) {
  if (!c || !id128) return PSVD_EINVAL;
  NcclApi& a = api();
  if (!a.ok) return fail(c, PSVD_ECUDA, "libnccl.so.2 could not be loaded");
  NcclUniqueId id;
  const NcclResult r = a.get_unique_id(&id);
  if (r != 0) return fail(c, PSVD_ECUDA, "ncclGetUniqueId: %s", a.error_string(r));
  std::memcpy(id128, id.internal, sizeof(id.internal));
  return PSVD_OK;
}

int psvd_nccl_init(psvd_ctx* c, int nranks, int rank, const unsigned char* id128) {
  if (!c || !id128 || nranks < 1 || rank < 0 || rank >= nranks) return PSVD_EINVAL;
  NcclApi& a = api();
  if (!a.ok) return fail(c, PSVD_ECUDA, "libnccl.so.2 could not be loaded");
  if (c->nccl_comm) {
    a.comm_destroy(c->nccl_comm);
    c->nccl_comm = nullptr;
  }
  NcclUniqueId id;
  std::memcpy(id.internal, id128, sizeof(id.internal));
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(c->device);
  const NcclResult r = a.comm_init_rank(&c->nccl_comm, nranks, id, rank);
  cudaSetDevice(prev);
  if (r != 0) {
    c->nccl_comm = nullptr;
    return fail(c, PSVD_ECUDA, "ncclCommInitRank: %s", a.error_string(r));
  }
  c->nccl_nranks = nranks;
  c->nccl_rank = rank;
  return PSVD_OK;
}

int psvd_nccl_enable(psvd_ctx* c, int on, int64_t row_offset) {
  if (!c) return PSVD_EINVAL;
  if (on && !c->nccl_comm) return fail(c, PSVD_EINVAL, "no NCCL communicator (psvd_nccl_init)");
  if (on && c->ex_allreduce) return fail(c, PSVD_EINVAL, "exchange hooks are set (psvd_set_exchange)");
  c->nccl_on = on != 0;
  c->ex_nranks = on ? c->nccl_nranks : 1;
  c->ex_row_offset = on ? row_offset : 0;
  return PSVD_OK;
}

int psvd_nccl_destroy(psvd_ctx* c) {
  if (!c) return PSVD_EINVAL;
  if (c->nccl_comm) api().comm_destroy(c->nccl_comm);
  c->nccl_comm = nullptr;
  c->nccl_on = false;
  c->ex_nranks = 1;
  c->ex_row_offset = 0;
  return PSVD_OK;
}

int psvd_exchange_stats(psvd_ctx* c, long long* out2) {
  if (!c || !out2) return PSVD_EINVAL;
  out2[0] = c->ex_calls;
  out2[1] = c->ex_bytes;
  return PSVD_OK;
}

}  // extern "C"
