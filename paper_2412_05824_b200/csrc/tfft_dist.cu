// Multi-GPU plumbing of libtfft.so: the one collective of the sharded path
// (north_star item 4) — the per-GPU fault counters reduced over
// NVLink. Everything else in a sharded run is rank-local.
//
// NCCL is resolved at run time (dlsym) from the libnccl.so.2 already loaded
// into the process — the one that created the caller's communicator (for a
// PyTorch caller: ProcessGroupNCCL._comm_ptr()) — so the library never links
// a second NCCL and never mixes communicator and function versions.
#include <dlfcn.h>
#include <nccl.h>

#include <string>

#include "../../include/tfft.h"

namespace {

using AllReduceFn = ncclResult_t (*)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                     cudaStream_t);
using GroupFn = ncclResult_t (*)();
using ErrFn = const char* (*)(ncclResult_t);

struct Nccl {
  AllReduceFn all_reduce = nullptr;
  GroupFn group_start = nullptr, group_end = nullptr;
  ErrFn err = nullptr;
  bool ok() const { return all_reduce && group_start && group_end; }
};

Nccl resolve() {
  Nccl n;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = RTLD_DEFAULT;
  n.all_reduce = (AllReduceFn)dlsym(h, "ncclAllReduce");
  n.group_start = (GroupFn)dlsym(h, "ncclGroupStart");
  n.group_end = (GroupFn)dlsym(h, "ncclGroupEnd");
  n.err = (ErrFn)dlsym(h, "ncclGetErrorString");
  return n;
}

}  // namespace

namespace tfft {
int set_error(int code, const char* msg);
}

extern "C" int tfft_allreduce_stats(int64_t* sums_dev, int nsums, double* max_dev, void* nccl_comm, void* stream) {
  if (!sums_dev || nsums < 0 || !max_dev || !nccl_comm)
    return tfft::set_error(TFFT_EINVAL, "invalid allreduce_stats arguments");
  static Nccl n = resolve();
  if (!n.ok()) return tfft::set_error(TFFT_EUNSUPPORTED, "libnccl.so.2 is not loaded in this process");
  const auto comm = (ncclComm_t)nccl_comm;
  const auto st = (cudaStream_t)stream;
  ncclResult_t r = n.group_start();
  if (r == ncclSuccess && nsums > 0) r = n.all_reduce(sums_dev, sums_dev, (size_t)nsums, ncclInt64, ncclSum, comm, st);
  ncclResult_t r2 = r == ncclSuccess ? n.all_reduce(max_dev, max_dev, 1, ncclFloat64, ncclMax, comm, st) : r;
  ncclResult_t r3 = n.group_end();
  if (r != ncclSuccess || r2 != ncclSuccess || r3 != ncclSuccess) {
    const ncclResult_t bad = r != ncclSuccess ? r : (r2 != ncclSuccess ? r2 : r3);
    std::string m = std::string("ncclAllReduce: ") + (n.err ? n.err(bad) : "error");
    return tfft::set_error(TFFT_ECUDA, m.c_str());
  }
  return TFFT_OK;
}
