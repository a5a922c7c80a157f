// comm.h — the collective transport of the block-column partition.
// Internal, not ABI. Every collective is IN PLACE on a device buffer laid out as P equal rank chunks
// (rank r's chunk at base + r·bytes) and is issued on the caller's stream.
//   NcclExchange   NCCL over NVLink/NVSwitch (libnccl.so.2 is dlopen'ed when a communicator is created)
//   HostExchange   P ranks that are threads of ONE process (device → host → device through a shared
//                  staging area with a barrier): the test harness that runs the multi-rank protocol on a
//                  single GPU without any kernel waiting on another rank's kernel
#pragma once
#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>

namespace ozr {

struct Exchange {
  int P = 1, rank = 0;
  std::string err;
  virtual ~Exchange() {}
  virtual bool group_begin() { return true; }
  virtual bool group_end(cudaStream_t) { return true; }
  // in-place all-gather: rank r contributes `bytes` at base + r·bytes; every rank receives all chunks
  virtual bool allgather(void* base, size_t bytes, cudaStream_t s) = 0;
  // in-place element-wise sum of `count` doubles over the ranks
  virtual bool allreduce_sum(double* buf, size_t count, cudaStream_t s) = 0;
};

// ---------------------------------------------------------------- host group (test harness)
struct HostGroup {
  int P;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long generation = 0;
  std::vector<std::vector<unsigned char>> stage;  // one staging buffer per rank
  explicit HostGroup(int p) : P(p), stage(p) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long long gen = generation;
    if (++arrived == P) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
};

struct HostExchange : Exchange {
  std::shared_ptr<HostGroup> g;
  bool allgather(void* base, size_t bytes, cudaStream_t s) override;
  bool allreduce_sum(double* buf, size_t count, cudaStream_t s) override;
};

// ---------------------------------------------------------------- NCCL
struct NcclExchange : Exchange {
  void* comm = nullptr;  // ncclComm_t
  bool in_group = false;
  ~NcclExchange() override;
  bool group_begin() override;
  bool group_end(cudaStream_t s) override;
  bool allgather(void* base, size_t bytes, cudaStream_t s) override;
  bool allreduce_sum(double* buf, size_t count, cudaStream_t s) override;
};

bool nccl_unique_id(void* id128, std::string& err);
NcclExchange* nccl_create(const void* id128, int nranks, int rank, std::string& err);

}  // namespace ozr
