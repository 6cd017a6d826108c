// mg.cu -- multi-GPU entry (pbit_sort_list_mg) and NCCL communicator helpers.
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>
#include <string.h>

#include "../../include/pbit.h"
#include "pbit_internal.h"

static_assert(sizeof(ncclUniqueId) == PBIT_MG_UNIQUE_ID_BYTES, "NCCL unique id size");

using namespace pbit;

extern "C" {

int pbit_mg_get_unique_id(void* id_out) {
  if (!id_out) return PBIT_ERR_INVALID_ARG;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return PBIT_ERR_NCCL;
  memcpy(id_out, &id, sizeof id);
  return PBIT_OK;
}

int pbit_mg_comm_init(void** comm_out, int nranks, const void* id, int rank) {
  if (!comm_out || !id || nranks < 1 || rank < 0 || rank >= nranks) return PBIT_ERR_INVALID_ARG;
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof uid);
  ncclComm_t c;
  if (ncclCommInitRank(&c, nranks, uid, rank) != ncclSuccess) return PBIT_ERR_NCCL;
  *comm_out = (void*)c;
  return PBIT_OK;
}

int pbit_mg_comm_destroy(void* comm) {
  if (!comm) return PBIT_ERR_INVALID_ARG;
  return ncclCommDestroy((ncclComm_t)comm) == ncclSuccess ? PBIT_OK : PBIT_ERR_NCCL;
}

int pbit_sort_list_mg(const void* keys_local, const uint32_t* next_local, uint32_t head, uint64_t n_global,
                      uint64_t node_lo, uint64_t n_local, int key_bits, uint32_t* out_head,
                      uint32_t* out_next_local, void* nccl_comm, const pbit_opts* opts) {
  if (!nccl_comm || !out_head) return PBIT_ERR_INVALID_ARG;
  int G = 0, r = 0;
  if (ncclCommCount((ncclComm_t)nccl_comm, &G) != ncclSuccess) return PBIT_ERR_NCCL;
  if (ncclCommUserRank((ncclComm_t)nccl_comm, &r) != ncclSuccess) return PBIT_ERR_NCCL;
  if (G == 1) {
    if (node_lo != 0 || n_local != n_global) return PBIT_ERR_UNSUPPORTED;
    return pbit_sort_list(keys_local, next_local, head, n_global, key_bits, out_head, out_next_local, opts);
  }
  return PBIT_ERR_UNSUPPORTED;
}

}  // extern "C"
