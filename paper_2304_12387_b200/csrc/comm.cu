// comm.cu — multi-GPU plumbing (element slabs along the last axis, NCCL over NVLink).
// Round-1 placeholder: the slab path is implemented in the next step; single-GPU never
// reaches these functions.
#include <cuda_runtime.h>
#include <nccl.h>

#include "internal.h"

namespace hdiv {

struct Comm {
  ncclComm_t comm = nullptr;
};

hdiv_status comm_init(hdiv_ctx* h, const void* id, cudaStream_t s) {
  (void)h; (void)id; (void)s;
  set_error("multi-GPU slabs not built yet");
  return HDIV_ERR_UNSUPPORTED;
}

void comm_free(hdiv_ctx* h) {
  if (!h->comm) return;
  if (h->comm->comm) ncclCommDestroy(h->comm->comm);
  delete h->comm;
  h->comm = nullptr;
}

hdiv_status comm_reverse_add(hdiv_ctx* h, double* y, cudaStream_t s) {
  (void)h; (void)y; (void)s;
  return HDIV_ERR_UNSUPPORTED;
}

hdiv_status comm_setup_schur_ghosts(hdiv_ctx* h, cudaStream_t s) {
  (void)h; (void)s;
  return HDIV_ERR_UNSUPPORTED;
}

}  // namespace hdiv
