// comm.cu — host side of the exchange layer (see comm.h). NCCL is loaded with dlopen when the first
// NCCL communicator is created, so the library itself has no link-time NCCL dependency (and picks up
// the libnccl.so.2 torch has already loaded, if any).
#include "comm.h"

#include <dlfcn.h>

#include <cstring>

#include <nccl.h>

namespace ozr {

// ---------------------------------------------------------------- host group
bool HostExchange::allgather(void* base, size_t bytes, cudaStream_t s) {
  auto& st = g->stage[rank];
  st.resize(bytes);
  char* b = static_cast<char*>(base);
  if (cudaMemcpyAsync(st.data(), b + rank * bytes, bytes, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess) {
    err = "host exchange: D2H";
    return false;
  }
  g->barrier();
  bool ok = true;
  for (int r = 0; r < P; ++r)
    if (r != rank && cudaMemcpyAsync(b + r * bytes, g->stage[r].data(), bytes, cudaMemcpyHostToDevice, s) != cudaSuccess)
      ok = false;
  if (cudaStreamSynchronize(s) != cudaSuccess) ok = false;
  g->barrier();  // nobody refills a stage before every rank has read it
  if (!ok) err = "host exchange: H2D";
  return ok;
}

bool HostExchange::allreduce_sum(double* buf, size_t count, cudaStream_t s) {
  auto& st = g->stage[rank];
  st.resize(count * sizeof(double));
  if (cudaMemcpyAsync(st.data(), buf, count * sizeof(double), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess) {
    err = "host exchange: D2H";
    return false;
  }
  g->barrier();
  std::vector<double> sum(count, 0.0);
  for (int r = 0; r < P; ++r) {  // fixed rank order
    const double* x = reinterpret_cast<const double*>(g->stage[r].data());
    for (size_t i = 0; i < count; ++i) sum[i] += x[i];
  }
  bool ok = cudaMemcpyAsync(buf, sum.data(), count * sizeof(double), cudaMemcpyHostToDevice, s) == cudaSuccess &&
            cudaStreamSynchronize(s) == cudaSuccess;
  g->barrier();
  if (!ok) err = "host exchange: H2D";
  return ok;
}

// ---------------------------------------------------------------- NCCL (dlopen)
namespace {

struct NcclApi {
  bool loaded = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    api.why = std::string("dlopen libnccl.so.2 failed: ") + dlerror();
    return api;
  }
#define OZR_SYM(field, name)                                              \
  api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name));     \
  if (!api.field) {                                                       \
    api.why = std::string("missing NCCL symbol ") + name;                 \
    return api;                                                           \
  }
  OZR_SYM(GetUniqueId, "ncclGetUniqueId");
  OZR_SYM(CommInitRank, "ncclCommInitRank");
  OZR_SYM(CommDestroy, "ncclCommDestroy");
  OZR_SYM(AllGather, "ncclAllGather");
  OZR_SYM(AllReduce, "ncclAllReduce");
  OZR_SYM(GroupStart, "ncclGroupStart");
  OZR_SYM(GroupEnd, "ncclGroupEnd");
  OZR_SYM(GetErrorString, "ncclGetErrorString");
#undef OZR_SYM
  api.loaded = true;
  return api;
}

bool nccl_ok(ncclResult_t r, std::string& err, const char* what) {
  if (r == ncclSuccess) return true;
  err = std::string(what) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "nccl error");
  return false;
}

}  // namespace

static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");

bool nccl_unique_id(void* id128, std::string& err) {
  NcclApi& api = nccl();
  if (!api.loaded) {
    err = api.why;
    return false;
  }
  ncclUniqueId id;
  if (!nccl_ok(api.GetUniqueId(&id), err, "ncclGetUniqueId")) return false;
  memcpy(id128, &id, sizeof id);
  return true;
}

NcclExchange* nccl_create(const void* id128, int nranks, int rank, std::string& err) {
  NcclApi& api = nccl();
  if (!api.loaded) {
    err = api.why;
    return nullptr;
  }
  ncclUniqueId id;
  memcpy(&id, id128, sizeof id);
  ncclComm_t c = nullptr;
  if (!nccl_ok(api.CommInitRank(&c, nranks, id, rank), err, "ncclCommInitRank")) return nullptr;
  NcclExchange* ex = new NcclExchange();
  ex->comm = c;
  ex->P = nranks;
  ex->rank = rank;
  return ex;
}

NcclExchange::~NcclExchange() {
  if (comm && nccl().loaded) nccl().CommDestroy(static_cast<ncclComm_t>(comm));
}

bool NcclExchange::group_begin() {
  in_group = true;
  return nccl_ok(nccl().GroupStart(), err, "ncclGroupStart");
}
bool NcclExchange::group_end(cudaStream_t) {
  in_group = false;
  return nccl_ok(nccl().GroupEnd(), err, "ncclGroupEnd");
}

bool NcclExchange::allgather(void* base, size_t bytes, cudaStream_t s) {
  char* b = static_cast<char*>(base);
  return nccl_ok(nccl().AllGather(b + rank * bytes, b, bytes, ncclUint8, static_cast<ncclComm_t>(comm), s), err,
                 "ncclAllGather");
}

bool NcclExchange::allreduce_sum(double* buf, size_t count, cudaStream_t s) {
  return nccl_ok(nccl().AllReduce(buf, buf, count, ncclDouble, ncclSum, static_cast<ncclComm_t>(comm), s), err,
                 "ncclAllReduce");
}

}  // namespace ozr
