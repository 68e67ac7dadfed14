// dist.cu -- multi-GPU plumbing: NCCL communicator (one process per GPU, the unique id
// broadcast by torch.distributed) and the row-slab distributed setup.
#include <nccl.h>

#include <cstring>

#include "amg.h"
#include "solver.h"

namespace amgb {
void set_last_error(const std::string& s);
}

struct amg_comm {
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
};

using namespace amgb;

extern "C" {

int amg_comm_unique_id(void* id128) {
  if (!id128) return AMG_EINVAL;
  static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id is 128 bytes");
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return AMG_ENCCL;
  std::memcpy(id128, &id, sizeof(id));
  return AMG_OK;
}

int amg_comm_init(const void* id128, int32_t nranks, int32_t rank, struct amg_comm** out) {
  if (!id128 || !out || nranks < 1 || rank < 0 || rank >= nranks) return AMG_EINVAL;
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  amg_comm* c = new amg_comm;
  c->nranks = nranks;
  c->rank = rank;
  if (ncclCommInitRank(&c->comm, nranks, id, rank) != ncclSuccess) {
    delete c;
    return AMG_ENCCL;
  }
  *out = c;
  return AMG_OK;
}

void amg_comm_destroy(struct amg_comm* c) {
  if (!c) return;
  if (c->comm) ncclCommDestroy(c->comm);
  delete c;
}

int amg_setup_dist(const amg_bsr* A_local, int64_t row_begin, int64_t n_global_block_rows, struct amg_comm* c,
                   const amg_params* p, void* stream, struct amg_handle** out) {
  (void)A_local, (void)row_begin, (void)n_global_block_rows, (void)c, (void)p, (void)stream, (void)out;
  set_last_error("amg_setup_dist: distributed setup not built yet");
  return AMG_EINVAL;
}

}  // extern "C"
