// comm.h -- communication layer of the row-slab distributed solve.
//
// Three implementations behind one interface:
//  * NcclComm  -- one process per GPU, NCCL over NVLink/NVSwitch (the product path);
//  * HostComm  -- separate processes over a caller's transport (callbacks on host copies:
//    torch.distributed gloo in the multi-process tests);
//  * LocalComm -- P ranks as P host threads of one process on one device, exchanging
//    through device-to-device copies with host barriers.  It exists so that the
//    distributed setup/solve can be tested on a single GPU: no kernel ever waits on
//    another rank's kernel (all waiting happens on the host), and reductions are summed
//    in rank order, exactly like a deterministic allreduce.
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <cstdint>
#include <mutex>
#include <vector>

namespace amgb {

class CommBase {
 public:
  int nranks = 1, rank = 0;
  virtual ~CommBase() = default;
  // in-place sum over ranks of n fp64 device values, ordered on stream s
  virtual void allreduce_sum(double* d, int n, cudaStream_t s) = 0;
  // host int64 allgather: all[r * n_each + i] = rank r's mine[i]; synchronous
  virtual void allgather_host(const int64_t* mine, int n_each, int64_t* all) = 0;
  // grouped point-to-point on device buffers, executed between begin and end
  virtual void group_begin() = 0;
  virtual void send(const void* buf, size_t bytes, int peer, cudaStream_t s) = 0;
  virtual void recv(void* buf, size_t bytes, int peer, cudaStream_t s) = 0;
  virtual void group_end(cudaStream_t s) = 0;
  virtual void barrier() = 0;
  // may the exchanges be recorded into a CUDA graph (stream-ordered device work only)?
  virtual bool capturable() const { return false; }
};

// shared state of a LocalComm group (one per emulated job)
struct LocalGroup {
  int P = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  int64_t generation = 0;
  struct Msg {
    int src, dst;
    const void* ptr;
    size_t bytes;
  };
  std::vector<std::vector<Msg>> mail;   // per source rank
  std::vector<std::vector<double>> red;  // per rank reduction slots
  std::vector<std::vector<int64_t>> gat;  // per rank allgather slots
  explicit LocalGroup(int p) : P(p), mail(p), red(p), gat(p) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const int64_t gen = generation;
    if (++arrived == P) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
};

struct HostOps {  // mirror of amg_host_comm_ops (amg.h)
  void* ctx;
  int (*allreduce_sum)(void*, double*, int32_t);
  int (*allgather_i64)(void*, const int64_t*, int32_t, int64_t*);
  int (*exchange)(void*, int32_t, const int32_t*, const void* const*, const int64_t*, int32_t, const int32_t*,
                  void* const*, const int64_t*);
  int (*barrier)(void*);
};

CommBase* make_nccl_comm(const void* id128, int nranks, int rank);
CommBase* make_host_comm(const HostOps& ops, int nranks, int rank, bool ordered);
CommBase* make_local_comm(LocalGroup* g, int rank);

}  // namespace amgb
