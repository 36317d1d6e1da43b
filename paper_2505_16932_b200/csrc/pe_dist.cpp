// Data-parallel Muon sharding inside the C ABI:
// pe_nccl_unique_id, pe_attach_comm, pe_polar_sharded.
//
// In Muon every rank holds every momentum matrix and needs every polar factor
// for its weight update W <- W - lr * polar(M).  The matrices are
// independent (the iteration runs per parameter), so rank r
// orthogonalises the subset pe_shard_plan gives it (LPT, identical on every
// rank, no communication) and the results are exchanged: each matrix is
// broadcast from its owner straight into every rank's output buffer (no
// packing copy; shapes may differ).  The set is cut into buckets of
// consecutive matrices of about equal cost; bucket b's broadcasts run on a
// side stream while bucket b+1 is computed, and the caller's stream waits for
// the last broadcast before the call's work is complete.
//
// NCCL is loaded at run time (dlopen): the copy torch already loaded if there
// is one (same process, same library), else PE_NCCL_LIB, else libnccl.so.2 on
// the loader path.  The library therefore still loads and runs single-GPU
// calls on machines without NCCL.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "pe.h"
#include "pe_internal.h"

namespace {

struct NcclApi {
  void* handle = nullptr;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclCommGetAsyncError) commGetAsyncError = nullptr;
  decltype(&ncclBroadcast) broadcast = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclGetErrorString) getErrorString = nullptr;
  decltype(&ncclGetVersion) getVersion = nullptr;
  std::string error;
};

NcclApi* nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api.handle ? &api : nullptr;
  tried = true;
  const char* env = getenv("PE_NCCL_LIB");
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);            // already loaded (e.g. by torch)
  if (!h && env) h = dlopen(env, RTLD_NOW | RTLD_LOCAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
  if (!h) {
    api.error = std::string("cannot load libnccl.so.2: ") + dlerror();
    return nullptr;
  }
  bool ok = true;
  auto sym = [&](const char* name) {
    void* p = dlsym(h, name);
    if (!p) ok = false;
    return p;
  };
  api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(sym("ncclGetUniqueId"));
  api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(sym("ncclCommInitRank"));
  api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(sym("ncclCommDestroy"));
  api.commGetAsyncError = reinterpret_cast<decltype(api.commGetAsyncError)>(sym("ncclCommGetAsyncError"));
  api.broadcast = reinterpret_cast<decltype(api.broadcast)>(sym("ncclBroadcast"));
  api.allReduce = reinterpret_cast<decltype(api.allReduce)>(sym("ncclAllReduce"));
  api.groupStart = reinterpret_cast<decltype(api.groupStart)>(sym("ncclGroupStart"));
  api.groupEnd = reinterpret_cast<decltype(api.groupEnd)>(sym("ncclGroupEnd"));
  api.getErrorString = reinterpret_cast<decltype(api.getErrorString)>(sym("ncclGetErrorString"));
  api.getVersion = reinterpret_cast<decltype(api.getVersion)>(sym("ncclGetVersion"));
  if (!ok) {
    api.error = "libnccl.so.2 lacks a required symbol";
    return nullptr;
  }
  api.handle = h;
  return &api;
}

pe_status nccl_fail(NcclApi* api, ncclResult_t r, const char* where) {
  std::string m = std::string(where) + ": " + (api ? api->getErrorString(r) : "NCCL unavailable");
  pe_set_error(m.c_str());
  return PE_ERR_NCCL;
}

}  // namespace

struct PeDist {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  cudaStream_t side = nullptr;               // broadcasts of finished buckets
  std::vector<cudaEvent_t> ev;               // per bucket: computed (main) / last one: sent (side)
};

void pe_dist_free(PeDist* d) {
  if (!d) return;
  if (d->comm) {
    if (NcclApi* api = nccl()) api->commDestroy(d->comm);
  }
  for (auto e : d->ev) cudaEventDestroy(e);
  if (d->side) cudaStreamDestroy(d->side);
  delete d;
}

#define PE_CUDA_D(call)                                         \
  do {                                                          \
    cudaError_t e_ = (call);                                    \
    if (e_ != cudaSuccess) {                                    \
      pe_set_error(cudaGetErrorString(e_));                     \
      return PE_ERR_CUDA;                                       \
    }                                                           \
  } while (0)

extern "C" pe_status pe_nccl_unique_id(char id[128]) {
  if (!id) return PE_ERR_INVALID_ARG;
  NcclApi* api = nccl();
  if (!api) {
    pe_set_error("NCCL unavailable");
    return PE_ERR_NCCL;
  }
  ncclUniqueId uid;
  const ncclResult_t r = api->getUniqueId(&uid);
  if (r != ncclSuccess) return nccl_fail(api, r, "ncclGetUniqueId");
  static_assert(sizeof(uid.internal) == 128, "ncclUniqueId is 128 bytes");
  memcpy(id, uid.internal, 128);
  return PE_OK;
}

extern "C" pe_status pe_attach_comm(pe_ctx c, const char id[128], int rank, int world) {
  if (!c || !id || world < 1 || rank < 0 || rank >= world) return PE_ERR_INVALID_ARG;
  NcclApi* api = nccl();
  if (!api) {
    pe_set_error("NCCL unavailable");
    return PE_ERR_NCCL;
  }
  PE_CUDA_D(cudaSetDevice(pe_ctx_device(c)));
  PeDist*& slot = pe_ctx_dist(c);
  if (slot) {                                  // re-attach: drop the old communicator first
    PE_CUDA_D(cudaDeviceSynchronize());
    pe_dist_free(slot);
    slot = nullptr;
  }
  PeDist* d = new PeDist();
  ncclUniqueId uid;
  memcpy(uid.internal, id, 128);
  ncclResult_t r = api->commInitRank(&d->comm, world, uid, rank);   // collective over the `world` ranks
  if (r != ncclSuccess) {
    d->comm = nullptr;
    pe_dist_free(d);
    return nccl_fail(api, r, "ncclCommInitRank");
  }
  d->rank = rank;
  d->world = world;
  if (cudaStreamCreateWithFlags(&d->side, cudaStreamNonBlocking) != cudaSuccess) {
    pe_dist_free(d);
    pe_set_error("cannot create the broadcast stream");
    return PE_ERR_CUDA;
  }
  slot = d;
  return PE_OK;
}

extern "C" pe_status pe_comm_info(pe_ctx c, int* rank, int* world) {
  if (!c || !rank || !world) return PE_ERR_INVALID_ARG;
  PeDist* d = pe_ctx_dist(c);
  *rank = d ? d->rank : 0;
  *world = d ? d->world : 0;
  return PE_OK;
}

// Buckets: consecutive index ranges of about equal cost 3 m^2 n + m^3 (the
// pe_shard_plan cost), identical on every rank.  At most `nb` buckets.
static std::vector<int> cost_buckets(const int64_t* shapes, int count, int nb) {
  std::vector<double> cost(count);
  double total = 0.0;
  for (int i = 0; i < count; ++i) {
    const double r = (double)shapes[2 * i], cc = (double)shapes[2 * i + 1];
    const double m = std::min(r, cc), n = std::max(r, cc);
    cost[i] = 3.0 * m * m * n + m * m * m;
    total += cost[i];
  }
  nb = std::max(1, std::min(nb, count));
  std::vector<int> beg{0};
  double acc = 0.0;
  for (int i = 0; i < count && (int)beg.size() < nb; ++i) {
    acc += cost[i];
    if (acc * nb >= total * (double)beg.size() && i + 1 < count) beg.push_back(i + 1);
  }
  beg.push_back(count);
  return beg;
}

extern "C" pe_status pe_shard_buckets(const int64_t* shapes, int count, int nbuckets, int* begin) {
  if (count < 0 || nbuckets < 1 || (count > 0 && !shapes) || !begin) return PE_ERR_INVALID_ARG;
  for (int i = 0; i < count; ++i)
    if (shapes[2 * i] < 1 || shapes[2 * i + 1] < 1) return PE_ERR_INVALID_ARG;
  const std::vector<int> b = cost_buckets(shapes, count, nbuckets);
  for (int i = 0; i <= nbuckets; ++i) begin[i] = b[std::min<size_t>(i, b.size() - 1)];
  return PE_OK;
}

extern "C" pe_status pe_polar_sharded(pe_ctx c, const void* const* in, void* const* out, const int64_t* shapes,
                                      int count, int iters, pe_dtype dtype, void* stream_) {
  if (!c || count < 0 || iters < 1 || (dtype != PE_BF16 && dtype != PE_FP32)) return PE_ERR_INVALID_ARG;
  if (count > 0 && (!in || !out || !shapes)) return PE_ERR_INVALID_ARG;
  PeDist* d = pe_ctx_dist(c);
  if (!d) {
    pe_set_error("pe_polar_sharded: no communicator (call pe_attach_comm first)");
    return PE_ERR_INVALID_ARG;
  }
  if (count == 0) {
    pe_ctx_set_launches(c, 0);
    return PE_OK;
  }
  std::vector<int> owner(count);
  pe_status s = pe_shard_plan(shapes, count, d->world, owner.data());
  if (s != PE_OK) return s;
  for (int i = 0; i < count; ++i)
    if (!out[i] || (owner[i] == d->rank && !in[i])) return PE_ERR_INVALID_ARG;
  NcclApi* api = nccl();
  if (!api) return PE_ERR_NCCL;
  {
    ncclResult_t ae = ncclSuccess;
    if (api->commGetAsyncError(d->comm, &ae) == ncclSuccess && ae != ncclSuccess && ae != ncclInProgress)
      return nccl_fail(api, ae, "pe_polar_sharded (earlier asynchronous error)");
  }
  int nbk = d->world > 1 ? 4 : 1;              // one rank: nothing to overlap
  if (const char* e = getenv("PE_SHARD_BUCKETS")) nbk = std::max(1, atoi(e));
  const std::vector<int> beg = cost_buckets(shapes, count, nbk);
  const int B = (int)beg.size() - 1;
  PE_CUDA_D(cudaSetDevice(pe_ctx_device(c)));
  while ((int)d->ev.size() < B + 1) {
    cudaEvent_t e;
    PE_CUDA_D(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    d->ev.push_back(e);
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream_);
  const size_t es = (dtype == PE_BF16) ? 2 : 4;
  int launches = 0;
  std::vector<const void*> ins;
  std::vector<void*> outs;
  std::vector<int64_t> shp;
  for (int b = 0; b < B; ++b) {
    ins.clear();
    outs.clear();
    shp.clear();
    for (int i = beg[b]; i < beg[b + 1]; ++i)
      if (owner[i] == d->rank) {
        ins.push_back(in[i]);
        outs.push_back(out[i]);
        shp.push_back(shapes[2 * i]);
        shp.push_back(shapes[2 * i + 1]);
      }
    if (!outs.empty()) {
      s = pe_polar(c, ins.data(), outs.data(), shp.data(), (int)outs.size(), iters, dtype, stream_);
      if (s != PE_OK) return s;
      int l = 0;
      pe_last_launch_count(c, &l);
      launches += l;
    }
    if (d->world == 1) continue;
    // bucket b is computed on this rank: its owners' results go to every rank
    PE_CUDA_D(cudaEventRecord(d->ev[b], st));
    PE_CUDA_D(cudaStreamWaitEvent(d->side, d->ev[b], 0));
    ncclResult_t r = api->groupStart();
    if (r != ncclSuccess) return nccl_fail(api, r, "ncclGroupStart");
    for (int i = beg[b]; i < beg[b + 1]; ++i) {
      const size_t nbytes = (size_t)shapes[2 * i] * (size_t)shapes[2 * i + 1] * es;
      r = api->broadcast(out[i], out[i], nbytes, ncclUint8, owner[i], d->comm, d->side);
      if (r != ncclSuccess) {
        api->groupEnd();
        return nccl_fail(api, r, "ncclBroadcast");
      }
    }
    r = api->groupEnd();
    if (r != ncclSuccess) return nccl_fail(api, r, "ncclGroupEnd");
  }
  if (d->world > 1) {
    PE_CUDA_D(cudaEventRecord(d->ev[B], d->side));
    PE_CUDA_D(cudaStreamWaitEvent(st, d->ev[B], 0));
  }
  pe_ctx_set_launches(c, launches);
  return PE_OK;
}

// pe_polar_split's all-reduce when the caller passes none: an in-place
// ncclAllReduce (SUM) over the context's communicator, on the call's stream.
extern "C" __attribute__((visibility("hidden"))) pe_status pe_comm_allreduce(void* buf, int64_t count, int dtype,
                                                                              void* user, void* stream) {
  pe_ctx c = reinterpret_cast<pe_ctx>(user);
  PeDist* d = c ? pe_ctx_dist(c) : nullptr;
  NcclApi* api = nccl();
  if (!d || !api) {
    pe_set_error("pe_polar_split: no allreduce callback and no communicator (pe_attach_comm)");
    return PE_ERR_INVALID_ARG;
  }
  const ncclResult_t r = api->allReduce(buf, buf, (size_t)count, dtype == 0 ? ncclFloat32 : ncclFloat64, ncclSum,
                                        d->comm, reinterpret_cast<cudaStream_t>(stream));
  return r == ncclSuccess ? PE_OK : nccl_fail(api, r, "ncclAllReduce");
}
