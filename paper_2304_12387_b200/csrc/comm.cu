// comm.cu — multi-GPU plumbing: element slabs along the last axis (z in 3D, y in 2D), one
// rank per GPU, NCCL over NVLink/NVSwitch.
//
//  * Interface face plane (the last-axis faces at the slab boundary) is replicated on both
//    ranks.  After a local apply each rank holds its own partial sum there; comm_reverse_add
//    exchanges the two partials (ncclSend/ncclRecv in one group) and adds them: a+b = b+a, so
//    both replicas stay bitwise identical.
//  * S~ couples L2 cells across the interface (face-neighbour stencil): the SpMV
//    reads a ghost layer of n_x n_y cells per interface, refreshed by comm_l2_ghosts.
//  * Dot products: the interface plane is owned by the lower rank (the upper rank masks its
//    bottom plane); each rank reduces locally in a fixed order, the P scalars are all-gathered
//    and summed in rank order on every rank -> identical on all ranks, independent of the NCCL
//    algorithm.
// NCCL is resolved with dlopen at first use, so libhdiv has no link-time NCCL dependency and
// shares the copy already loaded by the process (torch's).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <thread>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

#include "internal.h"

namespace hdiv {

namespace {
struct NcclApi {
  void* lib = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
};
NcclApi g_nccl;

bool load_nccl(std::string* err) {
  if (g_nccl.lib) return true;
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  void* lib = nullptr;
  for (const char* n : names) {
    lib = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
    if (lib) break;
  }
  if (!lib) { *err = std::string("dlopen libnccl failed: ") + dlerror(); return false; }
#define LOADSYM(field, name)                                                   \
  g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(lib, name));   \
  if (!g_nccl.field) { *err = std::string("missing NCCL symbol ") + name; return false; }
  LOADSYM(GetUniqueId, "ncclGetUniqueId");
  LOADSYM(CommInitRank, "ncclCommInitRank");
  LOADSYM(CommDestroy, "ncclCommDestroy");
  LOADSYM(Send, "ncclSend");
  LOADSYM(Recv, "ncclRecv");
  LOADSYM(GroupStart, "ncclGroupStart");
  LOADSYM(GroupEnd, "ncclGroupEnd");
  LOADSYM(AllGather, "ncclAllGather");
  LOADSYM(GetErrorString, "ncclGetErrorString");
  LOADSYM(CommGetAsyncError, "ncclCommGetAsyncError");
#undef LOADSYM
  g_nccl.lib = lib;
  return true;
}

__global__ void add_planes_kernel(double* lo, const double* rlo, double* hi, const double* rhi,
                                  long long m) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= m) return;
  if (lo) lo[i] += rlo[i];
  if (hi) hi[i] += rhi[i];
}

// cells of the bottom (c = 0 of element layer 0) / top (c = p-1 of the last layer) subcell
// layer, ordered by subcell (X [, Y]) -> send buffers
__global__ void pack_l2_layers_kernel(const double* __restrict__ x, double* lo, double* hi,
                                      long long NLx, long long NLy, long long NLz, int p, int dim,
                                      long long m) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= m) return;
  if (dim == 3) {
    long long nx = NLx * p;
    long long X = i % nx, Y = i / nx;
    long long ex = X / p, ey = Y / p, a = X % p, b = Y % p;
    long long pd = (long long)p * p * p;
    if (lo) lo[i] = x[(ex + NLx * ey) * pd + a + p * b];
    if (hi) hi[i] = x[(ex + NLx * (ey + NLy * (NLz - 1))) * pd + a + p * (b + p * (p - 1))];
  } else {
    long long X = i;
    long long ex = X / p, a = X % p;
    long long pd = (long long)p * p;
    if (lo) lo[i] = x[ex * pd + a];
    if (hi) hi[i] = x[(ex + NLx * (NLy - 1)) * pd + a + p * (p - 1)];
  }
}

// Loopback communicator for single-GPU tests of the slab path: the P ranks live in ONE process,
// each driven by its own host thread on its own stream; the id passed to hdiv_setup is
// "HDIVLOOP" + a 64-bit group key.  Every exchange posts the rank's send pointers, records an
// event, meets the others at a host barrier, then copies device-to-device from the peers'
// buffers after their events (and a second barrier + event wait keeps the senders' buffers
// untouched until the peers' copies are done).  Same data movement as the NCCL path.
struct LoopGroup {
  int P = 0, members = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  std::vector<cudaEvent_t> ev_ready, ev_done;
  std::vector<const double*> send_lo, send_hi;
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const long long g = gen;
    if (++arrived == P) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};
std::mutex g_loop_m;
std::map<unsigned long long, std::shared_ptr<LoopGroup>> g_loops;
const char kLoopMagic[8] = {'H', 'D', 'I', 'V', 'L', 'O', 'O', 'P'};
}  // namespace

struct Comm {
  ncclComm_t comm = nullptr;
  std::shared_ptr<LoopGroup> loop;   // loopback group (tests), else NCCL
  unsigned long long loop_key = 0;
  int rank = 0, P = 1;
  long long plane = 0;      // RT interface plane size (faces)
  long long lplane = 0;     // L2 ghost layer size (cells)
  double* buf = nullptr;    // recv_lo, recv_hi (RT) ; send_lo, send_hi (L2)
  double *rlo, *rhi, *slo, *shi;
  cudaStream_t cs = nullptr;               // exchange stream of the overlapped slab apply
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
};

static hdiv_status nccl_fail(ncclResult_t r, const char* what) {
  set_error(std::string(what) + ": " + (g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?"));
  return HDIV_ERR_NCCL;
}

// exchange with the two slab neighbours over NCCL (one group): send_lo -> rank-1, which
// receives it in its recv_hi, and send_hi -> rank+1 (recv_lo there); every call checked
static hdiv_status nccl_exchange(Comm* c, const double* send_lo, double* recv_lo,
                                 const double* send_hi, double* recv_hi, long long n,
                                 cudaStream_t s, const char* what) {
  ncclResult_t r = g_nccl.GroupStart();
  if (r != ncclSuccess) return nccl_fail(r, what);
  ncclResult_t e = ncclSuccess;
  if (send_lo) {
    if (e == ncclSuccess) e = g_nccl.Send(send_lo, n, ncclDouble, c->rank - 1, c->comm, s);
    if (e == ncclSuccess) e = g_nccl.Recv(recv_lo, n, ncclDouble, c->rank - 1, c->comm, s);
  }
  if (send_hi) {
    if (e == ncclSuccess) e = g_nccl.Send(send_hi, n, ncclDouble, c->rank + 1, c->comm, s);
    if (e == ncclSuccess) e = g_nccl.Recv(recv_hi, n, ncclDouble, c->rank + 1, c->comm, s);
  }
  r = g_nccl.GroupEnd();   // always close the group, even after a failed enqueue
  if (e != ncclSuccess) return nccl_fail(e, what);
  if (r != ncclSuccess) return nccl_fail(r, what);
  return HDIV_OK;
}

// asynchronous NCCL errors (a failed peer): polled by the MINRES / GMRES host loops so a dead
// peer surfaces as HDIV_ERR_NCCL instead of a silent hang
hdiv_status comm_check_async(const hdiv_ctx* h) {
  const Comm* c = h->comm;
  if (!c || c->loop || !c->comm || !g_nccl.CommGetAsyncError) return HDIV_OK;
  ncclResult_t ae = ncclSuccess;
  ncclResult_t r = g_nccl.CommGetAsyncError(c->comm, &ae);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommGetAsyncError");
  if (ae != ncclSuccess && ae != ncclInProgress) return nccl_fail(ae, "NCCL asynchronous error");
  return HDIV_OK;
}

// stream synchronisation that keeps polling NCCL for asynchronous errors while it waits (a
// plain cudaStreamSynchronize would block forever behind a collective whose peer died)
hdiv_status comm_sync(const hdiv_ctx* h, cudaStream_t s) {
  const Comm* c = h->comm;
  if (!c || c->loop || !c->comm) {
    HDIV_CUDA_TRY(cudaStreamSynchronize(s));
    return HDIV_OK;
  }
  for (int k = 0;; ++k) {
    cudaError_t q = cudaStreamQuery(s);
    if (q == cudaSuccess) return HDIV_OK;
    if (q != cudaErrorNotReady) HDIV_CUDA_TRY(q);
    hdiv_status st = comm_check_async(h);
    if (st != HDIV_OK) return st;
    if (k > 64) std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}

// exchange with the two slab neighbours through the loopback group: send_lo -> rank-1 (its
// recv_hi), send_hi -> rank+1 (its recv_lo); n doubles each
static hdiv_status loop_exchange(hdiv_ctx* h, const double* send_lo, const double* send_hi,
                                 double* recv_lo, double* recv_hi, long long n, cudaStream_t s) {
  Comm* c = h->comm;
  LoopGroup& g = *c->loop;
  const int r = c->rank;
  g.send_lo[r] = send_lo;
  g.send_hi[r] = send_hi;
  HDIV_CUDA_TRY(cudaEventRecord(g.ev_ready[r], s));
  g.barrier();
  if (recv_lo && r > 0) {
    HDIV_CUDA_TRY(cudaStreamWaitEvent(s, g.ev_ready[r - 1], 0));
    HDIV_CUDA_TRY(cudaMemcpyAsync(recv_lo, g.send_hi[r - 1], sizeof(double) * n,
                                  cudaMemcpyDeviceToDevice, s));
  }
  if (recv_hi && r < c->P - 1) {
    HDIV_CUDA_TRY(cudaStreamWaitEvent(s, g.ev_ready[r + 1], 0));
    HDIV_CUDA_TRY(cudaMemcpyAsync(recv_hi, g.send_lo[r + 1], sizeof(double) * n,
                                  cudaMemcpyDeviceToDevice, s));
  }
  HDIV_CUDA_TRY(cudaEventRecord(g.ev_done[r], s));
  g.barrier();
  if (r > 0) HDIV_CUDA_TRY(cudaStreamWaitEvent(s, g.ev_done[r - 1], 0));
  if (r < c->P - 1) HDIV_CUDA_TRY(cudaStreamWaitEvent(s, g.ev_done[r + 1], 0));
  g.barrier();   // the event slots may be re-recorded by the next exchange only after this
  return HDIV_OK;
}

bool comm_is_loopback(const hdiv_ctx* h) { return h->comm && h->comm->loop; }

// exchange stream + fork/join events of the overlapped slab apply (created with the comm)
void comm_overlap_handles(const hdiv_ctx* h, cudaStream_t* cs, cudaEvent_t* fork, cudaEvent_t* join) {
  *cs = h->comm->cs;
  *fork = h->comm->ev_fork;
  *join = h->comm->ev_join;
}

hdiv_status comm_init(hdiv_ctx* h, const void* id, cudaStream_t s) {
  (void)s;
  auto* c = new Comm();
  h->comm = c;
  c->rank = h->rank;
  c->P = h->nranks;
  c->plane = (h->dim == 3) ? h->n[0] * h->n[1] : h->n[0];
  c->lplane = c->plane;
  if (std::memcmp(id, kLoopMagic, 8) == 0) {   // loopback group (single-GPU tests)
    std::memcpy(&c->loop_key, (const char*)id + 8, sizeof(c->loop_key));
    {
      std::lock_guard<std::mutex> lk(g_loop_m);
      auto& gp = g_loops[c->loop_key];
      if (!gp) {
        gp = std::make_shared<LoopGroup>();
        gp->P = c->P;
        gp->ev_ready.assign(c->P, nullptr);
        gp->ev_done.assign(c->P, nullptr);
        gp->send_lo.assign(c->P, nullptr);
        gp->send_hi.assign(c->P, nullptr);
      }
      if (gp->P != c->P) { set_error("loopback group size mismatch"); return HDIV_ERR_SHAPE; }
      c->loop = gp;
      ++gp->members;
    }
    HDIV_CUDA_TRY(cudaEventCreateWithFlags(&c->loop->ev_ready[c->rank], cudaEventDisableTiming));
    HDIV_CUDA_TRY(cudaEventCreateWithFlags(&c->loop->ev_done[c->rank], cudaEventDisableTiming));
    c->loop->barrier();   // every rank registered
  } else {
  std::string err;
  if (!load_nccl(&err)) { set_error(err); return HDIV_ERR_NCCL; }
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclResult_t r = g_nccl.CommInitRank(&c->comm, c->P, uid, c->rank);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
  }
  HDIV_CUDA_TRY(cudaMalloc(&c->buf, sizeof(double) * 4 * c->plane));
  HDIV_CUDA_TRY(cudaStreamCreateWithFlags(&c->cs, cudaStreamNonBlocking));
  HDIV_CUDA_TRY(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
  HDIV_CUDA_TRY(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  c->rlo = c->buf;
  c->rhi = c->buf + c->plane;
  c->slo = c->buf + 2 * c->plane;
  c->shi = c->buf + 3 * c->plane;
  return HDIV_OK;
}

void comm_free(hdiv_ctx* h) {
  if (!h->comm) return;
  if (h->comm->loop) {
    std::lock_guard<std::mutex> lk(g_loop_m);
    auto& gp = h->comm->loop;
    if (--gp->members == 0) {
      for (auto e : gp->ev_ready) if (e) cudaEventDestroy(e);
      for (auto e : gp->ev_done) if (e) cudaEventDestroy(e);
      g_loops.erase(h->comm->loop_key);
    }
    h->comm->loop.reset();
  }
  if (h->comm->comm && g_nccl.CommDestroy) g_nccl.CommDestroy(h->comm->comm);
  cudaFree(h->comm->buf);
  if (h->comm->cs) cudaStreamDestroy(h->comm->cs);
  if (h->comm->ev_fork) cudaEventDestroy(h->comm->ev_fork);
  if (h->comm->ev_join) cudaEventDestroy(h->comm->ev_join);
  delete h->comm;
  h->comm = nullptr;
}

// interface plane pointers of an RT vector (last-axis faces at K = 0 and K = n_last)
static void planes(const hdiv_ctx* h, double* y, double** lo, double** hi) {
  const int last = h->dim - 1;
  const long long plane = h->comm->plane;
  *lo = (h->rank > 0) ? y + h->off[last] : nullptr;
  *hi = (h->rank < h->nranks - 1) ? y + h->off[last] + plane * h->n[last] : nullptr;
}

hdiv_status comm_reverse_add(hdiv_ctx* h, double* y, cudaStream_t s) {
  Comm* c = h->comm;
  if (!c) return HDIV_OK;
  double *lo, *hi;
  planes(h, y, &lo, &hi);
  if (c->loop) {
    hdiv_status st = loop_exchange(h, lo, hi, lo ? c->rlo : nullptr, hi ? c->rhi : nullptr,
                                   c->plane, s);
    if (st != HDIV_OK) return st;
    count_op();
    add_planes_kernel<<<(unsigned)((c->plane + 255) / 256), 256, 0, s>>>(lo, c->rlo, hi, c->rhi,
                                                                         c->plane);
    HDIV_CUDA_TRY(cudaGetLastError());
    return HDIV_OK;
  }
  hdiv_status st = nccl_exchange(c, lo, c->rlo, hi, c->rhi, c->plane, s, "reverse-add exchange");
  if (st != HDIV_OK) return st;
  count_op();
  add_planes_kernel<<<(unsigned)((c->plane + 255) / 256), 256, 0, s>>>(lo, c->rlo, hi, c->rhi,
                                                                       c->plane);
  HDIV_CUDA_TRY(cudaGetLastError());
  return HDIV_OK;
}

// refresh the ghost layers stored after the local entries of an L2 vector x[nl2 + 2 lplane]
hdiv_status comm_l2_ghosts(hdiv_ctx* h, double* x, cudaStream_t s) {
  Comm* c = h->comm;
  if (!c) return HDIV_OK;
  const bool down = h->rank > 0, up = h->rank < h->nranks - 1;
  pack_l2_layers_kernel<<<(unsigned)((c->lplane + 255) / 256), 256, 0, s>>>(
      x, down ? c->slo : nullptr, up ? c->shi : nullptr, h->NL[0], h->NL[1], h->NL[2], h->p,
      h->dim, c->lplane);
  HDIV_CUDA_TRY(cudaGetLastError());
  double* glo = x + h->nl2;
  double* ghi = x + h->nl2 + c->lplane;
  if (c->loop)
    return loop_exchange(h, down ? c->slo : nullptr, up ? c->shi : nullptr,
                         down ? glo : nullptr, up ? ghi : nullptr, c->lplane, s);
  return nccl_exchange(c, down ? c->slo : nullptr, down ? glo : nullptr, up ? c->shi : nullptr,
                       up ? ghi : nullptr, c->lplane, s, "L2 ghost exchange");
}

// all-gather of k local scalars into glob[P][k] (rank-ordered)
hdiv_status comm_allgather(hdiv_ctx* h, const double* loc, double* glob, int k, cudaStream_t s) {
  Comm* c = h->comm;
  if (c->loop) {
    LoopGroup& g = *c->loop;
    const int rk = c->rank;
    g.send_lo[rk] = loc;
    HDIV_CUDA_TRY(cudaEventRecord(g.ev_ready[rk], s));
    g.barrier();
    for (int q = 0; q < c->P; ++q) {
      if (q != rk) HDIV_CUDA_TRY(cudaStreamWaitEvent(s, g.ev_ready[q], 0));
      HDIV_CUDA_TRY(cudaMemcpyAsync(glob + (size_t)q * k, g.send_lo[q], sizeof(double) * k,
                                    cudaMemcpyDeviceToDevice, s));
    }
    HDIV_CUDA_TRY(cudaEventRecord(g.ev_done[rk], s));
    g.barrier();
    for (int q = 0; q < c->P; ++q)
      if (q != rk) HDIV_CUDA_TRY(cudaStreamWaitEvent(s, g.ev_done[q], 0));
    g.barrier();
    return HDIV_OK;
  }
  ncclResult_t r = g_nccl.AllGather(loc, glob, k, ncclDouble, c->comm, s);
  if (r != ncclSuccess) return nccl_fail(r, "allgather");
  return HDIV_OK;
}

// S~ ghost columns are built into the CSR by build_schur (columns nl2 + ...); nothing else.
hdiv_status comm_setup_schur_ghosts(hdiv_ctx* h, cudaStream_t s) {
  (void)h; (void)s;
  return HDIV_OK;
}

}  // namespace hdiv

extern "C" hdiv_status hdiv_nccl_unique_id(void* out, int64_t len) {
  using namespace hdiv;
  if (!out) { set_error("NULL out"); return HDIV_ERR_NULL; }
  if (len < (int64_t)sizeof(ncclUniqueId)) { set_error("buffer < 128 bytes"); return HDIV_ERR_SHAPE; }
  std::string err;
  if (!load_nccl(&err)) { set_error(err); return HDIV_ERR_NCCL; }
  ncclUniqueId id;
  ncclResult_t r = g_nccl.GetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  std::memcpy(out, &id, sizeof(id));
  return HDIV_OK;
}
