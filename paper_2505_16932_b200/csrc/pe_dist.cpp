// Data-parallel Muon sharding inside the C ABI:
// pe_nccl_unique_id, pe_attach_comm, pe_polar_sharded.
//
// In Muon every rank holds every momentum matrix and needs every polar factor
// for its weight update W <- W - lr * polar(M).  The matrices are
// independent (the iteration runs per parameter), so rank r
// orthogonalises the subset pe_shard_plan gives it (LPT, identical on every
// rank, no communication) and the results are exchanged.  The set is cut
// into buckets of consecutive matrices of about equal cost (their number
// chosen from the per-rank work, pe_shard_nbuckets); bucket b's exchange runs
// on a side stream while bucket b+1 is computed, and the caller's stream
// waits for the last exchange before the call's work is complete.
//
// Exchange.  When the caller's outputs sit in one flat buffer laid out by
// pe_shard_layout -- per bucket, one equal-sized chunk per rank holding that
// rank's matrices -- the last update epilogue of every owned matrix already
// stores into this rank's chunk, and one in-place all-gather per bucket fills
// the other ranks' chunks: no packing copy, one collective per bucket (the
// north-star all-gather).  Otherwise each matrix is broadcast from its owner
// into every rank's out[i] (one NCCL group per bucket).  Both go through
// NCCL (pe_attach_comm) or through a caller-supplied exchange function
// (pe_attach_exchange), which is how one GPU tests several virtual ranks.
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
  decltype(&ncclAllGather) allGather = nullptr;
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
  api.allGather = reinterpret_cast<decltype(api.allGather)>(sym("ncclAllGather"));
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
  ncclComm_t comm = nullptr;                 // NCCL communicator, or
  pe_exchange_fn hook = nullptr;             // the caller's exchange function (pe_attach_exchange)
  void* hook_user = nullptr;
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

extern "C" pe_status pe_attach_exchange(pe_ctx c, int rank, int world, pe_exchange_fn fn, void* user) {
  if (!c || !fn || world < 1 || rank < 0 || rank >= world) return PE_ERR_INVALID_ARG;
  PE_CUDA_D(cudaSetDevice(pe_ctx_device(c)));
  PeDist*& slot = pe_ctx_dist(c);
  if (slot) {
    PE_CUDA_D(cudaDeviceSynchronize());
    pe_dist_free(slot);
    slot = nullptr;
  }
  PeDist* d = new PeDist();
  d->hook = fn;
  d->hook_user = user;
  d->rank = rank;
  d->world = world;
  if (cudaStreamCreateWithFlags(&d->side, cudaStreamNonBlocking) != cudaSuccess) {
    pe_dist_free(d);
    pe_set_error("cannot create the exchange stream");
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

// Default bucket count of pe_polar_sharded / pe_shard_layout: one bucket per
// ~2.4 TFLOP of per-rank work (about 2 ms at the measured GEMM rate), so each
// bucket's compute is long next to its fixed cost (a norm pass and 3T GEMM
// fills and drains) and the exposed tail -- the last bucket's exchange -- is
// 1/nb of the total; at most 8, 1 for one rank (nothing to overlap).
// $PE_SHARD_BUCKETS overrides.
static int default_nbuckets(const int64_t* shapes, int count, int world) {
  if (const char* e = getenv("PE_SHARD_BUCKETS")) return std::max(1, atoi(e));
  if (world <= 1) return 1;
  double f = 0.0;
  for (int i = 0; i < count; ++i) {
    const double r = (double)shapes[2 * i], cc = (double)shapes[2 * i + 1];
    const double m = std::min(r, cc), n = std::max(r, cc);
    f += 3.0 * m * m * n + m * m * m;          // x T (= 5) x 2 flop/MAC ~ 10 x this per call
  }
  const double per_rank = 10.0 * f / world;
  return std::max(1, std::min(8, (int)(per_rank / 2.4e12)));
}

extern "C" pe_status pe_shard_nbuckets(const int64_t* shapes, int count, int world, int* nbuckets) {
  if (count < 0 || world < 1 || (count > 0 && !shapes) || !nbuckets) return PE_ERR_INVALID_ARG;
  // the buckets cost_buckets actually forms (skewed costs can leave fewer)
  *nbuckets = count == 0 ? 1 : (int)cost_buckets(shapes, count, default_nbuckets(shapes, count, world)).size() - 1;
  return PE_OK;
}

// Matrix -> rank plan: longest-processing-time greedy on the
// cost 3 m^2 n + m^3, run bucket by bucket over pe_polar_sharded's buckets
// (largest first inside a bucket, to the rank with the least work in this
// bucket, ties to the least total work, then the lowest rank): every bucket
// is balanced across ranks, so the ranks finish a bucket together and its
// per-rank chunks of the all-gather layout are about equally long (global
// LPT ignoring the buckets left 27 % padding on the Llama-3-8B set at
// 8 ranks, this 7.7 %), and the whole set stays balanced (exactly, on the
// BASELINE layer sets at 1/2/4/8 ranks).  Deterministic: every rank
// computes the same plan with no communication.
extern "C" pe_status pe_shard_plan(const int64_t* shapes, int count, int world, int* owner) {
  if (world < 1 || count < 0 || (count > 0 && (!shapes || !owner))) return PE_ERR_INVALID_ARG;
  std::vector<double> cost(count);
  for (int i = 0; i < count; ++i) {
    const double r = (double)shapes[2 * i], cc = (double)shapes[2 * i + 1];
    if (r < 1 || cc < 1) return PE_ERR_INVALID_ARG;
    const double m = std::min(r, cc), n = std::max(r, cc);
    cost[i] = 3.0 * m * m * n + m * m * m;
  }
  if (count == 0) return PE_OK;
  const std::vector<int> beg = cost_buckets(shapes, count, default_nbuckets(shapes, count, world));
  std::vector<double> load(world, 0.0);
  for (size_t b = 0; b + 1 < beg.size(); ++b) {
    std::vector<int> idx;
    for (int i = beg[b]; i < beg[b + 1]; ++i) idx.push_back(i);
    std::stable_sort(idx.begin(), idx.end(), [&](int x, int y) { return cost[x] > cost[y]; });
    std::vector<double> bl(world, 0.0);
    for (int i : idx) {
      int best = 0;
      for (int w = 1; w < world; ++w)
        if (bl[w] < bl[best] || (bl[w] == bl[best] && load[w] < load[best])) best = w;
      owner[i] = best;
      bl[best] += cost[i];
      load[best] += cost[i];
    }
  }
  return PE_OK;
}

// Flat output layout of the all-gather exchange: bucket after bucket, each
// bucket world equal chunks (the largest rank's share, 256-byte granules),
// rank r's matrices of the bucket packed in index order in chunk r.
struct Layout {
  std::vector<int> beg, owner;
  std::vector<int64_t> off, chunk, base;     // per matrix byte offset; per bucket chunk bytes / start
  int64_t total = 0;
};

static pe_status make_layout(const int64_t* shapes, int count, int world, int nb, size_t es, Layout* L) {
  L->owner.assign(count, 0);
  pe_status s = pe_shard_plan(shapes, count, world, L->owner.data());
  if (s != PE_OK) return s;
  L->beg = cost_buckets(shapes, count, nb);
  const int B = (int)L->beg.size() - 1;
  L->off.assign(count, 0);
  L->chunk.assign(B, 0);
  L->base.assign(B, 0);
  int64_t base = 0;
  for (int b = 0; b < B; ++b) {
    std::vector<int64_t> fill(world, 0);
    for (int i = L->beg[b]; i < L->beg[b + 1]; ++i) {
      const int64_t bytes = shapes[2 * i] * shapes[2 * i + 1] * (int64_t)es;
      L->off[i] = fill[L->owner[i]];
      fill[L->owner[i]] += (bytes + 255) / 256 * 256;
    }
    const int64_t ch = std::max<int64_t>(256, *std::max_element(fill.begin(), fill.end()));
    for (int i = L->beg[b]; i < L->beg[b + 1]; ++i) L->off[i] += base + (int64_t)L->owner[i] * ch;
    L->chunk[b] = ch;
    L->base[b] = base;
    base += (int64_t)world * ch;
  }
  L->total = base;
  return PE_OK;
}

extern "C" pe_status pe_shard_layout(const int64_t* shapes, int count, int world, pe_dtype dtype, int64_t* offsets,
                                     int64_t* chunk_bytes, int64_t* total_bytes) {
  if (count < 1 || world < 1 || !shapes || !offsets || !total_bytes) return PE_ERR_INVALID_ARG;
  if (dtype != PE_BF16 && dtype != PE_FP32) return PE_ERR_INVALID_ARG;
  for (int i = 0; i < count; ++i)
    if (shapes[2 * i] < 1 || shapes[2 * i + 1] < 1) return PE_ERR_INVALID_ARG;
  Layout L;
  pe_status s = make_layout(shapes, count, world, default_nbuckets(shapes, count, world),
                            dtype == PE_BF16 ? 2 : 4, &L);
  if (s != PE_OK) return s;
  std::copy(L.off.begin(), L.off.end(), offsets);
  if (chunk_bytes) std::copy(L.chunk.begin(), L.chunk.end(), chunk_bytes);
  *total_bytes = L.total;
  return PE_OK;
}

extern "C" pe_status pe_shard_buckets(const int64_t* shapes, int count, int nbuckets, int* begin) {
  if (count < 0 || nbuckets < 1 || (count > 0 && !shapes) || !begin) return PE_ERR_INVALID_ARG;
  for (int i = 0; i < count; ++i)
    if (shapes[2 * i] < 1 || shapes[2 * i + 1] < 1) return PE_ERR_INVALID_ARG;
  const std::vector<int> b = cost_buckets(shapes, count, nbuckets);
  for (int i = 0; i <= nbuckets; ++i) begin[i] = b[std::min<size_t>(i, b.size() - 1)];
  return PE_OK;
}

static pe_status sharded_impl(pe_ctx c, const void* const* in, void* const* out, const int64_t* shapes, int count,
                              int iters, pe_dtype dtype, void* stream_, bool compute) {
  if (!c || count < 0 || iters < 1 || (dtype != PE_BF16 && dtype != PE_FP32)) return PE_ERR_INVALID_ARG;
  if (count > 0 && ((compute && !in) || !out || !shapes)) return PE_ERR_INVALID_ARG;
  PeDist* d = pe_ctx_dist(c);
  if (!d) {
    pe_set_error("pe_polar_sharded: no communicator (call pe_attach_comm or pe_attach_exchange first)");
    return PE_ERR_INVALID_ARG;
  }
  if (count == 0) {
    pe_ctx_set_launches(c, 0);
    return PE_OK;
  }
  for (int i = 0; i < count; ++i)
    if (shapes[2 * i] < 1 || shapes[2 * i + 1] < 1) return PE_ERR_INVALID_ARG;
  const size_t es = (dtype == PE_BF16) ? 2 : 4;
  Layout L;
  pe_status s = make_layout(shapes, count, d->world, default_nbuckets(shapes, count, d->world), es, &L);
  if (s != PE_OK) return s;
  const std::vector<int>& owner = L.owner;
  for (int i = 0; i < count; ++i)
    if (!out[i] || (compute && owner[i] == d->rank && !in[i])) return PE_ERR_INVALID_ARG;
  // zero-copy all-gather when out[] is the pe_shard_layout of one buffer
  uint8_t* flat = reinterpret_cast<uint8_t*>(out[0]) - L.off[0];
  bool gather = d->world > 1 && !getenv("PE_SHARD_BROADCAST");
  for (int i = 0; i < count && gather; ++i)
    if (reinterpret_cast<uint8_t*>(out[i]) != flat + L.off[i]) gather = false;
  NcclApi* api = nullptr;
  if (!d->hook) {
    api = nccl();
    if (!api) return PE_ERR_NCCL;
    ncclResult_t ae = ncclSuccess;
    if (api->commGetAsyncError(d->comm, &ae) == ncclSuccess && ae != ncclSuccess && ae != ncclInProgress)
      return nccl_fail(api, ae, "pe_polar_sharded (earlier asynchronous error)");
  }
  const int B = (int)L.beg.size() - 1;
  PE_CUDA_D(cudaSetDevice(pe_ctx_device(c)));
  while ((int)d->ev.size() < B + 1) {
    cudaEvent_t e;
    PE_CUDA_D(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    d->ev.push_back(e);
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream_);
  bool side_used = false;
  // join the side stream back into the caller's stream (also on errors, so
  // the caller's stream never runs ahead of an exchange already enqueued)
  auto join = [&]() -> pe_status {
    if (!side_used) return PE_OK;
    PE_CUDA_D(cudaEventRecord(d->ev[B], d->side));
    PE_CUDA_D(cudaStreamWaitEvent(st, d->ev[B], 0));
    return PE_OK;
  };
  auto fail = [&](pe_status e) {
    join();
    return e;
  };
  int launches = 0;
  std::vector<const void*> ins;
  std::vector<void*> outs;
  std::vector<int64_t> shp;
  for (int b = 0; b < B; ++b) {
    ins.clear();
    outs.clear();
    shp.clear();
    for (int i = L.beg[b]; i < L.beg[b + 1] && compute; ++i)
      if (owner[i] == d->rank) {
        ins.push_back(in[i]);
        outs.push_back(out[i]);
        shp.push_back(shapes[2 * i]);
        shp.push_back(shapes[2 * i + 1]);
      }
    if (!outs.empty() && compute) {
      s = pe_polar(c, ins.data(), outs.data(), shp.data(), (int)outs.size(), iters, dtype, stream_);
      if (s != PE_OK) return fail(s);
      int l = 0;
      pe_last_launch_count(c, &l);
      launches += l;
    }
    if (d->world == 1) continue;
    // bucket b is computed on this rank: exchange it on the side stream
    if (cudaEventRecord(d->ev[b], st) != cudaSuccess || cudaStreamWaitEvent(d->side, d->ev[b], 0) != cudaSuccess) {
      pe_set_error("pe_polar_sharded: cannot order the exchange stream");
      return fail(PE_ERR_CUDA);
    }
    side_used = true;
    if (gather) {
      uint8_t* rb = flat + L.base[b];
      const int64_t ch = L.chunk[b];
      if (d->hook) {
        s = d->hook(PE_EXCHANGE_ALLGATHER, rb, ch, d->rank, d->hook_user, d->side);
        if (s != PE_OK) return fail(s);
      } else {
        const ncclResult_t r = api->allGather(rb + (int64_t)d->rank * ch, rb, (size_t)ch, ncclUint8, d->comm, d->side);
        if (r != ncclSuccess) return fail(nccl_fail(api, r, "ncclAllGather"));
      }
      continue;
    }
    if (d->hook) {
      for (int i = L.beg[b]; i < L.beg[b + 1]; ++i) {
        s = d->hook(PE_EXCHANGE_BROADCAST, out[i], shapes[2 * i] * shapes[2 * i + 1] * (int64_t)es, owner[i],
                    d->hook_user, d->side);
        if (s != PE_OK) return fail(s);
      }
      continue;
    }
    ncclResult_t r = api->groupStart();
    if (r != ncclSuccess) return fail(nccl_fail(api, r, "ncclGroupStart"));
    for (int i = L.beg[b]; i < L.beg[b + 1]; ++i) {
      const size_t nbytes = (size_t)shapes[2 * i] * (size_t)shapes[2 * i + 1] * es;
      r = api->broadcast(out[i], out[i], nbytes, ncclUint8, owner[i], d->comm, d->side);
      if (r != ncclSuccess) {
        api->groupEnd();
        return fail(nccl_fail(api, r, "ncclBroadcast"));
      }
    }
    r = api->groupEnd();
    if (r != ncclSuccess) return fail(nccl_fail(api, r, "ncclGroupEnd"));
  }
  if ((s = join()) != PE_OK) return s;
  pe_ctx_set_launches(c, launches);
  return PE_OK;
}

extern "C" pe_status pe_polar_sharded(pe_ctx c, const void* const* in, void* const* out, const int64_t* shapes,
                                      int count, int iters, pe_dtype dtype, void* stream) {
  return sharded_impl(c, in, out, shapes, count, iters, dtype, stream, true);
}

// The exchange of pe_polar_sharded alone (each rank's owned out[i] already
// hold its results): the same buckets, collectives and stream ordering, no
// compute.  The benchmark times it to report the exchange span in isolation.
extern "C" pe_status pe_sharded_exchange(pe_ctx c, void* const* out, const int64_t* shapes, int count,
                                         pe_dtype dtype, void* stream) {
  return sharded_impl(c, nullptr, out, shapes, count, 1, dtype, stream, false);
}

// pe_polar_split's all-reduce when the caller passes none: an in-place
// ncclAllReduce (SUM) over the context's communicator, on the call's stream.
extern "C" __attribute__((visibility("hidden"))) pe_status pe_comm_allreduce(void* buf, int64_t count, int dtype,
                                                                              void* user, void* stream) {
  pe_ctx c = reinterpret_cast<pe_ctx>(user);
  PeDist* d = c ? pe_ctx_dist(c) : nullptr;
  NcclApi* api = nccl();
  if (!d || !d->comm || !api) {
    pe_set_error("pe_polar_split: no allreduce callback and no NCCL communicator (pe_attach_comm)");
    return PE_ERR_INVALID_ARG;
  }
  const ncclResult_t r = api->allReduce(buf, buf, (size_t)count, dtype == 0 ? ncclFloat32 : ncclFloat64, ncclSum,
                                        d->comm, reinterpret_cast<cudaStream_t>(stream));
  return r == ncclSuccess ? PE_OK : nccl_fail(api, r, "ncclAllReduce");
}
