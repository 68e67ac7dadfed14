// comm.cu -- NcclComm and LocalComm (see comm.h).
#include <nccl.h>

#include <cstring>
#include <string>
#include <vector>
#include <map>
#include <algorithm>

#include "amg.h"
#include "comm.h"
#include "common.cuh"

namespace amgb {

#define AMG_NCCL(expr)                                                                      \
  do {                                                                                      \
    ncclResult_t r_ = (expr);                                                               \
    if (r_ != ncclSuccess) ::amgb::fail(AMG_ENCCL, std::string(#expr) + ": " + ncclGetErrorString(r_)); \
  } while (0)

class NcclComm : public CommBase {
 public:
  ncclComm_t comm = nullptr;
  NcclComm(const void* id128, int n, int r) {
    nranks = n;
    rank = r;
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    AMG_NCCL(ncclCommInitRank(&comm, n, id, r));
  }
  ~NcclComm() override {
    if (comm) ncclCommDestroy(comm);
  }
  void allreduce_sum(double* d, int n, cudaStream_t s) override {
    if (nranks == 1 || n == 0) return;
    AMG_NCCL(ncclAllReduce(d, d, n, ncclDouble, ncclSum, comm, s));
  }
  void allgather_host(const int64_t* mine, int n_each, int64_t* all) override {
    int64_t* d = nullptr;
    AMG_CK(cudaMalloc(&d, sizeof(int64_t) * n_each * (nranks + 1)));
    AMG_CK(cudaMemcpy(d, mine, sizeof(int64_t) * n_each, cudaMemcpyHostToDevice));
    AMG_NCCL(ncclAllGather(d, d + n_each, n_each, ncclInt64, comm, nullptr));
    AMG_CK(cudaStreamSynchronize(nullptr));
    AMG_CK(cudaMemcpy(all, d + n_each, sizeof(int64_t) * n_each * nranks, cudaMemcpyDeviceToHost));
    cudaFree(d);
  }
  void group_begin() override { AMG_NCCL(ncclGroupStart()); }
  void send(const void* buf, size_t bytes, int peer, cudaStream_t s) override {
    AMG_NCCL(ncclSend(buf, bytes, ncclChar, peer, comm, s));
  }
  void recv(void* buf, size_t bytes, int peer, cudaStream_t s) override {
    AMG_NCCL(ncclRecv(buf, bytes, ncclChar, peer, comm, s));
  }
  void group_end(cudaStream_t) override { AMG_NCCL(ncclGroupEnd()); }
  // ncclSend / ncclRecv / ncclAllReduce are stream-ordered and graph-capturable
  bool capturable() const override { return true; }
  void barrier() override {
    double* d = nullptr;
    AMG_CK(cudaMalloc(&d, sizeof(double)));
    AMG_CK(cudaMemset(d, 0, sizeof(double)));
    AMG_NCCL(ncclAllReduce(d, d, 1, ncclDouble, ncclSum, comm, nullptr));
    AMG_CK(cudaStreamSynchronize(nullptr));
    cudaFree(d);
  }
};

class LocalComm : public CommBase {
 public:
  LocalGroup* g;
  struct Pending {
    void* buf;
    const void* sbuf;
    size_t bytes;
    int peer;
  };
  std::vector<Pending> sends, recvs;
  LocalComm(LocalGroup* grp, int r) : g(grp) {
    nranks = grp->P;
    rank = r;
  }
  void allreduce_sum(double* d, int n, cudaStream_t s) override {
    if (nranks == 1 || n == 0) return;
    std::vector<double> mine(n);
    AMG_CK(cudaMemcpyAsync(mine.data(), d, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    AMG_CK(cudaStreamSynchronize(s));
    g->red[rank] = mine;
    g->barrier();
    std::vector<double> tot(n, 0.0);
    for (int r = 0; r < nranks; ++r)  // rank order: deterministic
      for (int i = 0; i < n; ++i) tot[i] += g->red[r][i];
    g->barrier();
    AMG_CK(cudaMemcpyAsync(d, tot.data(), sizeof(double) * n, cudaMemcpyHostToDevice, s));
    AMG_CK(cudaStreamSynchronize(s));
  }
  void allgather_host(const int64_t* mine, int n_each, int64_t* all) override {
    g->gat[rank].assign(mine, mine + n_each);
    g->barrier();
    for (int r = 0; r < nranks; ++r) std::memcpy(all + (size_t)r * n_each, g->gat[r].data(), sizeof(int64_t) * n_each);
    g->barrier();
  }
  void group_begin() override {
    sends.clear();
    recvs.clear();
  }
  void send(const void* buf, size_t bytes, int peer, cudaStream_t) override { sends.push_back({nullptr, buf, bytes, peer}); }
  void recv(void* buf, size_t bytes, int peer, cudaStream_t) override { recvs.push_back({buf, nullptr, bytes, peer}); }
  void group_end(cudaStream_t s) override {
    AMG_CK(cudaStreamSynchronize(s));  // send buffers complete
    g->mail[rank].clear();
    for (auto& p : sends) g->mail[rank].push_back({rank, p.peer, p.sbuf, p.bytes});
    g->barrier();
    // the k-th recv from peer p matches the k-th send of p to this rank
    std::vector<int> seen(nranks, 0);
    for (auto& rv : recvs) {
      int k = seen[rv.peer]++;
      int found = -1;
      for (size_t m = 0, c = 0; m < g->mail[rv.peer].size(); ++m)
        if (g->mail[rv.peer][m].dst == rank && (int)c++ == k) {
          found = (int)m;
          break;
        }
      if (found < 0) fail(AMG_ENCCL, "LocalComm: unmatched recv");
      const auto& msg = g->mail[rv.peer][found];
      if (msg.bytes != rv.bytes) fail(AMG_ENCCL, "LocalComm: size mismatch");
      if (rv.bytes) AMG_CK(cudaMemcpyAsync(rv.buf, msg.ptr, rv.bytes, cudaMemcpyDeviceToDevice, s));
    }
    AMG_CK(cudaStreamSynchronize(s));
    g->barrier();  // senders may reuse their buffers after this
  }
  void barrier() override { g->barrier(); }
};

class HostComm : public CommBase {
 public:
  HostOps ops;
  bool ordered;  // stream-ordered (capturable) mode: copies + cudaLaunchHostFunc, no host sync
  struct Pending {
    void* dbuf;
    const void* sbuf;
    size_t bytes;
    int peer;
  };
  std::vector<Pending> sends, recvs;
  // stream-ordered mode: one pinned staging call record per distinct exchange / reduction
  // (keyed by its device buffers, sizes and peers), kept for the communicator's life so that
  // a captured graph replays with the same host buffers
  struct Call {
    HostOps ops;
    std::vector<int32_t> sp, rp;
    std::vector<const void*> sb;
    std::vector<void*> rb;
    std::vector<int64_t> sz, rz;
    double* red = nullptr;
    int n = 0;
    volatile int rc = 0;
  };
  std::map<std::vector<int64_t>, Call*> calls;
  char* pool = nullptr;
  size_t pool_size = 0, pool_used = 0;
  HostComm(const HostOps& o, int n, int r, bool ord) : ops(o), ordered(ord) {
    nranks = n;
    rank = r;
    if (ordered) {  // allocated up front: no allocation may happen inside a stream capture
      pool_size = (size_t)env_int("AMG_HOSTCOMM_POOL_MB", 256) << 20;
      AMG_CK(cudaMallocHost((void**)&pool, pool_size));
    }
  }
  ~HostComm() override {
    for (auto& kv : calls) delete kv.second;
    if (pool) cudaFreeHost(pool);
  }
  static void ck(int rc, const char* what) {
    if (rc != 0) fail(AMG_ENCCL, std::string("host communicator: ") + what + " callback failed");
  }
  void check_async() {
    for (auto& kv : calls)
      if (kv.second->rc) ck(kv.second->rc, "stream-ordered");
  }
  char* host_buf(size_t bytes) {
    bytes = (std::max<size_t>(bytes, 1) + 255) & ~size_t(255);
    if (pool_used + bytes > pool_size) fail(AMG_ENOMEM, "host communicator: staging pool exhausted (AMG_HOSTCOMM_POOL_MB)");
    char* p = pool + pool_used;
    pool_used += bytes;
    return p;
  }
  static void CUDART_CB run_exchange(void* p) {
    Call* c = static_cast<Call*>(p);
    const int rc = c->ops.exchange(c->ops.ctx, (int32_t)c->sp.size(), c->sp.data(), c->sb.data(), c->sz.data(),
                                   (int32_t)c->rp.size(), c->rp.data(), c->rb.data(), c->rz.data());
    if (rc) c->rc = rc;
  }
  static void CUDART_CB run_allreduce(void* p) {
    Call* c = static_cast<Call*>(p);
    const int rc = c->ops.allreduce_sum(c->ops.ctx, c->red, c->n);
    if (rc) c->rc = rc;
  }
  void allreduce_sum(double* d, int n, cudaStream_t s) override {
    if (nranks == 1 || n == 0) return;
    if (ordered) {
      check_async();
      std::vector<int64_t> key{1, (int64_t)(uintptr_t)d, n};
      Call*& c = calls[key];
      if (!c) {
        c = new Call;
        c->ops = ops;
        c->n = n;
        c->red = reinterpret_cast<double*>(host_buf(sizeof(double) * n));
      }
      AMG_CK(cudaMemcpyAsync(c->red, d, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
      AMG_CK(cudaLaunchHostFunc(s, run_allreduce, c));
      AMG_CK(cudaMemcpyAsync(d, c->red, sizeof(double) * n, cudaMemcpyHostToDevice, s));
      return;
    }
    std::vector<double> h(n);
    AMG_CK(cudaMemcpyAsync(h.data(), d, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    AMG_CK(cudaStreamSynchronize(s));
    ck(ops.allreduce_sum(ops.ctx, h.data(), n), "allreduce_sum");
    AMG_CK(cudaMemcpyAsync(d, h.data(), sizeof(double) * n, cudaMemcpyHostToDevice, s));
    AMG_CK(cudaStreamSynchronize(s));
  }
  void allgather_host(const int64_t* mine, int n_each, int64_t* all) override {
    ck(ops.allgather_i64(ops.ctx, mine, n_each, all), "allgather_i64");
  }
  void group_begin() override {
    sends.clear();
    recvs.clear();
  }
  void send(const void* buf, size_t bytes, int peer, cudaStream_t) override { sends.push_back({nullptr, buf, bytes, peer}); }
  void recv(void* buf, size_t bytes, int peer, cudaStream_t) override { recvs.push_back({buf, nullptr, bytes, peer}); }
  void group_end(cudaStream_t s) override {
    if (ordered) {
      check_async();
      std::vector<int64_t> key{2};
      for (auto& m : sends) key.insert(key.end(), {0, (int64_t)(uintptr_t)m.sbuf, (int64_t)m.bytes, m.peer});
      for (auto& m : recvs) key.insert(key.end(), {1, (int64_t)(uintptr_t)m.dbuf, (int64_t)m.bytes, m.peer});
      Call*& c = calls[key];
      if (!c) {
        c = new Call;
        c->ops = ops;
        for (auto& m : sends) c->sp.push_back(m.peer), c->sb.push_back(host_buf(m.bytes)), c->sz.push_back((int64_t)m.bytes);
        for (auto& m : recvs) c->rp.push_back(m.peer), c->rb.push_back(host_buf(m.bytes)), c->rz.push_back((int64_t)m.bytes);
      }
      for (size_t i = 0; i < sends.size(); ++i)
        if (sends[i].bytes)
          AMG_CK(cudaMemcpyAsync(const_cast<void*>(c->sb[i]), sends[i].sbuf, sends[i].bytes, cudaMemcpyDeviceToHost, s));
      AMG_CK(cudaLaunchHostFunc(s, run_exchange, c));
      for (size_t i = 0; i < recvs.size(); ++i)
        if (recvs[i].bytes) AMG_CK(cudaMemcpyAsync(recvs[i].dbuf, c->rb[i], recvs[i].bytes, cudaMemcpyHostToDevice, s));
      return;
    }
    AMG_CK(cudaStreamSynchronize(s));  // the send buffers are complete
    std::vector<std::vector<char>> sh(sends.size()), rh(recvs.size());
    std::vector<int32_t> sp, rp;
    std::vector<const void*> sb;
    std::vector<void*> rb;
    std::vector<int64_t> sz, rz;
    for (size_t i = 0; i < sends.size(); ++i) {
      sh[i].resize(std::max<size_t>(sends[i].bytes, 1));
      if (sends[i].bytes) AMG_CK(cudaMemcpy(sh[i].data(), sends[i].sbuf, sends[i].bytes, cudaMemcpyDeviceToHost));
      sp.push_back(sends[i].peer), sb.push_back(sh[i].data()), sz.push_back((int64_t)sends[i].bytes);
    }
    for (size_t i = 0; i < recvs.size(); ++i) {
      rh[i].resize(std::max<size_t>(recvs[i].bytes, 1));
      rp.push_back(recvs[i].peer), rb.push_back(rh[i].data()), rz.push_back((int64_t)recvs[i].bytes);
    }
    ck(ops.exchange(ops.ctx, (int32_t)sp.size(), sp.data(), sb.data(), sz.data(), (int32_t)rp.size(), rp.data(),
                    rb.data(), rz.data()),
       "exchange");
    for (size_t i = 0; i < recvs.size(); ++i)
      if (recvs[i].bytes) AMG_CK(cudaMemcpyAsync(recvs[i].dbuf, rh[i].data(), recvs[i].bytes, cudaMemcpyHostToDevice, s));
    AMG_CK(cudaStreamSynchronize(s));
  }
  void barrier() override {
    check_async();
    ck(ops.barrier(ops.ctx), "barrier");
  }
  bool capturable() const override { return ordered; }
};

CommBase* make_nccl_comm(const void* id128, int nranks, int rank) { return new NcclComm(id128, nranks, rank); }
CommBase* make_host_comm(const HostOps& ops, int nranks, int rank, bool ordered) {
  return new HostComm(ops, nranks, rank, ordered);
}
CommBase* make_local_comm(LocalGroup* g, int rank) { return new LocalComm(g, rank); }

}  // namespace amgb
