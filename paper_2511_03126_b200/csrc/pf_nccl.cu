// The per-object reductions of the sharded path over NCCL, callable from C/C++ hosts (SURVEY §8b:
// `pf_allreduce_partials(..., ncclComm_t)`). dist.py drives the same collectives through
// torch.distributed; a C/C++ caller with its own communicator uses this entry instead of
// re-implementing the protocol.
//
// NCCL is resolved at run time (dlopen): the library already loaded in the process (torch's, whose
// communicators a caller may pass in) is preferred, else the system libnccl.so.2. The shared library
// therefore keeps its only link dependency on the CUDA runtime.
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>

#include "pf_common.cuh"

namespace pf {
namespace {

struct Nccl {
  std::once_flag once;
  void* lib = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) =
      nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

Nccl& nccl() {
  static Nccl n;
  std::call_once(n.once, [] {
    n.lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!n.lib) n.lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!n.lib) return;
    n.all_reduce = reinterpret_cast<decltype(n.all_reduce)>(dlsym(n.lib, "ncclAllReduce"));
    n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(dlsym(n.lib, "ncclGetUniqueId"));
    n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(dlsym(n.lib, "ncclCommInitRank"));
    n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(dlsym(n.lib, "ncclCommDestroy"));
    n.error_string = reinterpret_cast<decltype(n.error_string)>(dlsym(n.lib, "ncclGetErrorString"));
  });
  return n;
}

int nccl_status(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return PF_OK;
  return set_error(PF_ERR_CUDA, "%s: %s", what, nccl().error_string ? nccl().error_string(r) : "NCCL error");
}

}  // namespace
}  // namespace pf

using namespace pf;

extern "C" {

int pf_allreduce_partials(float* grid_partials, int64_t n_grid, double* partials, int64_t n_partials, void* comm,
                          void* stream) {
  Nccl& n = nccl();
  if (!n.all_reduce) return set_error(PF_ERR_LOAD, "libnccl.so.2 not found (dlopen)");
  if (!comm) return set_error(PF_ERR_VALUE, "allreduce_partials: null communicator");
  if (n_grid < 0 || n_partials < 0) return set_error(PF_ERR_VALUE, "allreduce_partials: negative length");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  ncclComm_t c = reinterpret_cast<ncclComm_t>(comm);
  if (n_grid > 0) {
    if (!grid_partials) return set_error(PF_ERR_VALUE, "allreduce_partials: null grid");
    if (int rc = nccl_status(n.all_reduce(grid_partials, grid_partials, (size_t)n_grid, ncclFloat32, ncclSum, c, st),
                             "ncclAllReduce(grid)"))
      return rc;
  }
  if (n_partials > 0) {
    if (!partials) return set_error(PF_ERR_VALUE, "allreduce_partials: null partials");
    if (int rc = nccl_status(n.all_reduce(partials, partials, (size_t)n_partials, ncclFloat64, ncclSum, c, st),
                             "ncclAllReduce(partials)"))
      return rc;
  }
  return PF_OK;
}

int pf_nccl_comm_init_single(void** comm) {
  Nccl& n = nccl();
  if (!n.comm_init_rank || !n.get_unique_id) return set_error(PF_ERR_LOAD, "libnccl.so.2 not found (dlopen)");
  if (!comm) return set_error(PF_ERR_VALUE, "nccl_comm_init_single: null output");
  ncclUniqueId id;
  if (int rc = nccl_status(n.get_unique_id(&id), "ncclGetUniqueId")) return rc;
  ncclComm_t c = nullptr;
  if (int rc = nccl_status(n.comm_init_rank(&c, 1, id, 0), "ncclCommInitRank")) return rc;
  *comm = c;
  return PF_OK;
}

int pf_nccl_comm_destroy(void* comm) {
  Nccl& n = nccl();
  if (!n.comm_destroy) return set_error(PF_ERR_LOAD, "libnccl.so.2 not found (dlopen)");
  return nccl_status(n.comm_destroy(reinterpret_cast<ncclComm_t>(comm)), "ncclCommDestroy");
}

}  // extern "C"
