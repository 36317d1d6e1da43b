// Host side of the C ABI (include/pe.h): context, workspace, planner and the
// launch sequence of one Polar Express call (Listing 2):
//
//   pe_norm_kernel                       s = ||M||_F*1.01 + 1e-7
//   copy pass (unfolded inputs only)     X_0 = M 2^e, wide orientation; the
//                                        rest of 1/s is applied by iteration 1 (fp32 input: X_0 = M/s)
//   T x { pe_gemm_sm100 Gram            A = X X^T
//         pe_gemm_sm100 Poly            B = b A + c A^2
//         pe_gemm_sm100 Update          X = a X + B X }
//   copy pass (unfolded outputs only)    transpose back
//
// bf16 matrices whose rows are 16-byte multiples are folded (no copy passes,
// gemm_sm100.cuh).  fp32 matrices run the same tensor-core GEMM on three
// bf16 planes per buffer (kP = 3) between a split pass and a join pass.
//
// Every launch covers the whole batch (grouped scheduling).  A plan (tile
// lists, tensor maps, workspace carve-up) depends only on the shape list; the
// context caches the last few plans, all carving the same workspace (their
// kernels are stream-ordered).  Per-call data (caller pointers and tensor
// maps) goes through a small ring of pinned upload buffers, each guarded by
// an event, so back-to-back asynchronous calls never overwrite an upload the
// GPU has not consumed yet.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <utility>
#include <vector>

#include "elementwise.cuh"
#include "gemm_sm100.cuh"
#include "small_sm100.cuh"
#include "pe.h"
#include "pe_internal.h"
#include "pe_types.h"

using namespace pe;

// smem ring depths of the GEMM instantiations (gemm_smem_bytes must stay
// below the 227 KB per-CTA limit): poly/update 6 x 32 KB ring + 32 KB
// epilogue slots (one per warp)
#ifndef PE_LONG_STAGES
#define PE_LONG_STAGES 6
#endif
constexpr int kLongStages = PE_LONG_STAGES;
// the Gram (no epilogue operand, one 4 KB staging slot per warp) takes 6
#ifndef PE_GRAM_STAGES
#define PE_GRAM_STAGES 6
#endif
constexpr int kGramStages = PE_GRAM_STAGES;
// 4 KB epilogue slots per warp of poly/update: 1 = one slot (operand chunk 1
// is loaded after chunk 0's result left it), which pays for the sixth ring
// stage; 2 = the whole tile's operand prefetched during its main loop (with a
// 5-stage ring).  GPT-2 S update 119.1 -> 114.8 us per launch with 6 / 1,
// poly unchanged (profiles/r1_variants.md)
#ifndef PE_OP_SLOTS
#define PE_OP_SLOTS 1
#endif
constexpr int kOpSlots = PE_OP_SLOTS;
// fp32 (three bf16 planes): 4 x 32 KB ring + 8 warps x 3 plane slots x 4 KB
constexpr int kP3Stages = 4;

namespace {

thread_local std::string g_last_error;

#define PE_CUDA(call)                                                                    \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess) {                                                             \
      g_last_error = std::string(#call) + ": " + cudaGetErrorString(e_);                \
      return PE_ERR_CUDA;                                                                \
    }                                                                                    \
  } while (0)

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

inline int64_t rup(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

// Every launch is programmatic (PDL): the kernel's prologue overlaps the tail
// of the previous kernel in the stream; each kernel calls griddepcontrol.wait
// before touching memory (see ptx.cuh pdl_wait).  PE_NO_PDL=1 disables it.
template <typename... KArgs, typename... Args>
cudaError_t launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  static const bool pdl = getenv("PE_NO_PDL") == nullptr;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
inline int cdiv(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

// Append host arrays into one device blob.
struct Blob {
  std::vector<uint8_t> host;
  size_t add(const void* p, size_t bytes, size_t align = 128) {
    size_t off = rup(host.size(), align);
    host.resize(off + bytes);
    if (bytes) std::memcpy(host.data() + off, p, bytes);
    return off;
  }
  template <typename T> size_t add(const std::vector<T>& v, size_t align = 128) {
    return add(v.data(), v.size() * sizeof(T), align);
  }
};

}  // namespace

// One cached plan: the device-side description of a shape list.
struct Plan {
  std::vector<int64_t> key;     // shapes
  pe_dtype dtype = PE_BF16;
  int count = 0;
  std::vector<MatDev> mats;
  std::vector<int> flags;       // per matrix kFlag* (folded input, tall, direct output)
  void* meta = nullptr;         // device blob
  size_t meta_bytes = 0;
  // offsets into meta
  size_t o_mats = 0, o_tmaps = 0, o_emaps = 0, o_sym = 0, o_upd = 0, o_sym_r = 0, o_upd_r = 0;
  size_t o_elems = 0, o_cmat = 0, o_cidx = 0, o_nch = 0, o_part = 0, o_cnt = 0, o_inv = 0;
  // copy passes: scale/orient (rows: wide inputs, tr: tall inputs) and
  // finalize (tr: tall outputs, rows: wide outputs whose rows are not 16-byte multiples)
  size_t o_smats = 0, o_fmats = 0, o_x0 = 0, o_flags = 0, o_it[4] = {0, 0, 0, 0};
  int n_it[4] = {0, 0, 0, 0};
  int n_sym = 0, n_upd = 0, n_chunks = 0;
  size_t o_need = 0;            // per (matrix, mode) completion target of the fused schedule
  // spectrum-aware first step (App. G, pe_set_spectrum_init): power-method
  // work items (matrix, 32 rows), vectors (two ping-pong sets of sum m floats),
  // per-item partials, per-matrix counters / lambda / ||w||^2 (x2) / sum of squares / (a, b)
  size_t o_sitem_mat = 0, o_sitem_r0 = 0, o_sitem0 = 0, o_snitem = 0, o_svoff = 0, o_sv = 0, o_sv0 = 0, o_spart = 0;
  size_t o_scnt = 0, o_slam = 0, o_snrm = 0, o_sssq = 0, o_smcoef = 0, o_str = 0;
  size_t o_a32 = 0;             // per matrix fp32 Gram (App. G plans, `init`), device pointers
  bool init = false;
  int n_sitems = 0;
  int64_t sv_len = 0;
  // fused schedule (one launch for all 3T phases), built for one T at a time
  int fused_T = 0, n_fused = 0;
  Tile* fused = nullptr;
  size_t fused_cap = 0;
  // fast rectangular iteration (App. H, Alg. 4): map strides, full m x m
  // tile lists (both directions) and the Q_1 expansion items
  bool rect = false;
  int tstride = 6, estride = 4;
  size_t o_sq = 0, o_sq_r = 0, o_exp = 0;
  int n_sq = 0, n_exp = 0;
  size_t ws_needed = 0;
  uint64_t last_use = 0;
  bool pinned = false;          // used by a captured CUDA graph: kept (with its workspace) until pe_destroy
};

// One pinned upload buffer of the per-call ring.
struct CallSlot {
  void* h = nullptr;            // pinned host (mapped)
  const void* hd = nullptr;     // the same buffer as seen from the device (UVA), or nullptr
  void* d = nullptr;            // device
  size_t bytes = 0;
  cudaEvent_t done = nullptr;   // recorded after the upload on the call's stream
  bool armed = false;
};

constexpr int kMaxPlans = 8;
constexpr int kCallSlots = 4;

struct pe_ctx_s {
  int device = 0;
  int num_sms = 148;
  int norm_blocks = 148;         // resident blocks of the persistent norm kernel (one wave)
  std::vector<double> table;   // ntab * nq
  int degree = 5;
  int ntab = 0;

  // workspace shared by every cached plan
  void* ws = nullptr;
  size_t ws_bytes = 0;
  std::vector<Plan*> plans;
  // plans a captured graph points into, and workspaces they carve, retired
  // from the cache (workspace growth, LRU) but alive until pe_destroy
  std::vector<Plan*> retired_plans;
  std::vector<void*> retired_ws;
  uint64_t use_clock = 0;

  CallSlot calls[kCallSlots];
  int next_call = 0;
  // CUDA-graph capture: every captured call consumes one of these for good
  // (the graph's memcpy node re-reads its pinned host buffer at each replay);
  // pe_reserve keeps kCaptureSpare unused ones of the reserved batch's size
  std::vector<CallSlot> cap_slots;
  size_t cap_used = 0;

  // pe_polar_host: staging + copy streams
  void* staging = nullptr;
  size_t staging_bytes = 0;
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  std::vector<cudaEvent_t> host_ev;

  int last_launches = 0;
  int uploads = 0;              // upload-kernel launches of the current call (counted in last_launches)
  int* done = nullptr;          // fused schedule completion counters (cleared by the norm kernel)
  float* scratch = nullptr;     // fp32 path: per-CTA running sums of the K passes (gemm_sm100.cuh)
  // pe_polar_split: fp32 partial Gram (and a device pointer to it), local sum of squares
  float* sh_a32 = nullptr;
  size_t sh_cap = 0;
  float** sh_ptr = nullptr;
  double* sh_sum = nullptr;
  // pe_polar_split_peers: device copies of the slot pointers, and of this
  // rank's two partial-Gram destinations (by iteration parity)
  uint8_t** peer_slots = nullptr;
  int peer_cap = 0;
  float** peer_out = nullptr;
  size_t done_cap = 0;
  int dbg = 0;   // PE_DEBUG_GEMM (timing experiments only; results are wrong when bits 0/1/3 are set)
  long long* stats = nullptr;   // PE_DEBUG_GEMM bit 2: per-CTA wait counters of the last launch per mode

  // profiling
  bool profiling = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  struct Pending { int kind; cudaEvent_t a, b; };
  std::vector<Pending> pending;

  PeDist* dist = nullptr;       // pe_attach_comm (pe_dist.cpp)
  int init_iters = 0;           // pe_set_spectrum_init: power iterations of App. G's first step (0 = off)
  double init_margin = 0.0;     // pe_set_spectrum_init_ex: 1 / (1 + |b| margin) (0 = eq. (init_poly) exactly, R17)
  // pe_set_rect_iteration (App. H, Alg. 4): iterations per application (0 = off)
  int rect_restart = 0;
  double rect_min_aspect = 0.0;  // <= 0: the paper's rule alpha > 1.5 T / (T - 1)
  double rect_shift = 1e-3;      // added to Y's diagonal in the first application
  int rect_mode = 0;             // internal: 0 = split the batch by aspect, 1 = Listing 2 only, 2 = Alg. 4 only
  int debug = 0;                 // pe_set_debug flags (PE_DEBUG_CHECK_FINITE)
  int small_planes = 1;          // pe_set_small_planes: A / B planes of the bf16 small path (1 = R8, 2 = R8p)
  unsigned long long* nf = nullptr;   // device counter of pe_count_nonfinite
};

PeDist*& pe_ctx_dist(pe_ctx c) { return c->dist; }
int pe_ctx_device(pe_ctx c) { return c->device; }
void pe_ctx_set_launches(pe_ctx c, int n) { c->last_launches = n; }
void pe_set_error(const char* msg) { g_last_error = msg; }

static void free_plan(Plan* p) {
  if (p->meta) cudaFree(p->meta);
  if (p->fused) cudaFree(p->fused);
  delete p;
}

namespace {
cudaEvent_t take_event(pe_ctx c) {
  if (c->ev_used == c->ev_pool.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    c->ev_pool.push_back(e);
  }
  return c->ev_pool[c->ev_used++];
}
// Bracket one launch with events when profiling (kind = PE profile kind).
struct ProfScope {
  pe_ctx c; int kind; cudaStream_t st; cudaEvent_t a = nullptr;
  ProfScope(pe_ctx c_, int k, cudaStream_t s) : c(c_), kind(k), st(s) {
    if (c->profiling && (a = take_event(c))) cudaEventRecord(a, st);
  }
  ~ProfScope() {
    if (!a) return;
    cudaEvent_t b = take_event(c);
    if (!b) return;
    cudaEventRecord(b, st);
    c->pending.push_back({kind, a, b});
  }
};
}  // namespace

// debug-only: copy the per-CTA wait counters of the last GEMM launch of each
// mode (3 x 2048 int64) to host memory `out` (not part of the public header).
extern "C" pe_status pe_debug_stats(pe_ctx c, long long* out) {
  if (!c || !out || !c->stats) return PE_ERR_INVALID_ARG;
  PE_CUDA(cudaDeviceSynchronize());
  PE_CUDA(cudaMemcpy(out, c->stats, 8 * 1024 * sizeof(long long), cudaMemcpyDeviceToHost));
  return PE_OK;
}

extern "C" pe_status pe_profile_enable(pe_ctx c, int on) {
  if (!c) return PE_ERR_INVALID_ARG;
  c->profiling = on != 0;
  return PE_OK;
}

extern "C" pe_status pe_profile_read(pe_ctx c, double* ms, int* counts, int nkinds) {
  if (!c || nkinds < 0 || (nkinds > 0 && (!ms || !counts))) return PE_ERR_INVALID_ARG;
  PE_CUDA(cudaSetDevice(c->device));
  for (const auto& p : c->pending) {
    PE_CUDA(cudaEventSynchronize(p.b));
    float t = 0.f;
    PE_CUDA(cudaEventElapsedTime(&t, p.a, p.b));
    if (p.kind < nkinds) { ms[p.kind] += t; counts[p.kind] += 1; }
  }
  c->pending.clear();
  c->ev_used = 0;
  return PE_OK;
}

// ---------------------------------------------------------------- basics
extern "C" const char* pe_status_string(pe_status s) {
  switch (s) {
    case PE_OK: return "PE_OK";
    case PE_ERR_INVALID_ARG: return "PE_ERR_INVALID_ARG";
    case PE_ERR_UNSUPPORTED: return "PE_ERR_UNSUPPORTED";
    case PE_ERR_NO_CONVERGENCE: return "PE_ERR_NO_CONVERGENCE";
    case PE_ERR_CUDA: return "PE_ERR_CUDA";
    case PE_ERR_NCCL: return "PE_ERR_NCCL";
    case PE_ERR_WORKSPACE: return "PE_ERR_WORKSPACE";
    case PE_ERR_NONFINITE: return "PE_ERR_NONFINITE";
  }
  return "PE_ERR_UNKNOWN";
}

extern "C" const char* pe_version(void) { return "pe-b200 0.1 sm_100a"; }

extern "C" const char* pe_last_error_message(void) { return g_last_error.c_str(); }

extern "C" pe_status pe_create(pe_ctx* out, int device) {
  if (!out) return PE_ERR_INVALID_ARG;
  *out = nullptr;
  int ndev = 0;
  PE_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return PE_ERR_INVALID_ARG;
  cudaDeviceProp prop;
  PE_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10 || prop.minor != 0) {
    g_last_error = "device is not sm_100 (B200)";
    return PE_ERR_UNSUPPORTED;
  }
  PE_CUDA(cudaSetDevice(device));
  PE_CUDA(cudaFuncSetAttribute(pe_gemm_sm100<kGramStages, 1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)gemm_smem_bytes<kGramStages, 1>()));
  PE_CUDA(cudaFuncSetAttribute(pe_gemm_sm100<kGramStages, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)gemm_smem_bytes<kGramStages, 1>()));
  PE_CUDA(cudaFuncSetAttribute(pe_gemm_sm100<kLongStages, kOpSlots, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)gemm_smem_bytes<kLongStages, kOpSlots>()));
  PE_CUDA(cudaFuncSetAttribute(pe_gemm_sm100<kLongStages, kOpSlots, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)gemm_smem_bytes<kLongStages, kOpSlots>()));
  PE_CUDA(cudaFuncSetAttribute(pe_gemm_sm100<kP3Stages, 3, false, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)gemm_smem_bytes<kP3Stages, 3>()));
  PE_CUDA(cudaFuncSetAttribute(pe_small_sm100<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)small_smem_bytes<1>(kSmallMaxNpadBf16)));
  PE_CUDA(cudaFuncSetAttribute(pe_small_sm100<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)small_smem_bytes<3>(128)));
  PE_CUDA(cudaFuncSetAttribute(pe_small_sm100<1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)small_smem_bytes<1, 2>(kSmallMaxNpadPrecise)));
  if (!get_encode_fn()) {
    g_last_error = "cuTensorMapEncodeTiled unavailable";
    return PE_ERR_CUDA;
  }
  pe_ctx c = new pe_ctx_s();
  c->device = device;
  c->num_sms = prop.multiProcessorCount;
  {
    int per_sm = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pe_norm_kernel, kNormThreads, 0) != cudaSuccess)
      per_sm = 1;
    c->norm_blocks = c->num_sms * std::max(1, per_sm);
  }
  if (const char* d = getenv("PE_DEBUG_GEMM")) c->dbg = atoi(d);
  c->table.resize(8 * 3);
  pe_status s = pe_coeffs(1e-3, 5, 8, 1.01, c->table.data());   // Listing 2 table
  if (s != PE_OK) { delete c; return s; }
  c->degree = 5;
  c->ntab = 8;
  *out = c;
  return PE_OK;
}

extern "C" pe_status pe_destroy(pe_ctx c) {
  if (!c) return PE_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  if (c->ws) cudaFree(c->ws);
  if (c->nf) cudaFree(c->nf);
  for (Plan* p : c->plans) free_plan(p);
  for (Plan* p : c->retired_plans) free_plan(p);
  for (void* w : c->retired_ws) cudaFree(w);
  for (CallSlot& cs : c->calls) {
    if (cs.d) cudaFree(cs.d);
    if (cs.h) cudaFreeHost(cs.h);
    if (cs.done) cudaEventDestroy(cs.done);
  }
  for (CallSlot& cs : c->cap_slots) {
    if (cs.d) cudaFree(cs.d);
    if (cs.h) cudaFreeHost(cs.h);
  }
  if (c->staging) cudaFree(c->staging);
  if (c->s_h2d) cudaStreamDestroy(c->s_h2d);
  if (c->s_d2h) cudaStreamDestroy(c->s_d2h);
  for (auto e : c->host_ev) cudaEventDestroy(e);
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  if (c->stats) cudaFree(c->stats);
  if (c->done) cudaFree(c->done);
  if (c->scratch) cudaFree(c->scratch);
  if (c->sh_a32) cudaFree(c->sh_a32);
  if (c->sh_ptr) cudaFree(c->sh_ptr);
  if (c->sh_sum) cudaFree(c->sh_sum);
  if (c->peer_slots) cudaFree(c->peer_slots);
  if (c->peer_out) cudaFree(c->peer_out);
  if (c->dist) pe_dist_free(c->dist);
  delete c;
  return PE_OK;
}

extern "C" pe_status pe_set_coeffs(pe_ctx c, const double* coeffs, int ntuples, int degree) {
  if (!c || !coeffs || ntuples < 1) return PE_ERR_INVALID_ARG;
  if (degree != 3 && degree != 5) return PE_ERR_UNSUPPORTED;
  const int nq = (degree + 1) / 2;
  for (int i = 0; i < ntuples * nq; ++i)
    if (!std::isfinite(coeffs[i])) return PE_ERR_INVALID_ARG;
  c->table.assign(coeffs, coeffs + ntuples * nq);
  c->degree = degree;
  c->ntab = ntuples;
  return PE_OK;
}

extern "C" pe_status pe_set_spectrum_init(pe_ctx c, int power_iters) {
  if (!c || power_iters < 0 || power_iters > 1000) return PE_ERR_INVALID_ARG;
  c->init_iters = power_iters;
  c->init_margin = 0.0;
  return PE_OK;
}

extern "C" pe_status pe_set_spectrum_init_ex(pe_ctx c, int power_iters, double margin) {
  if (!c || power_iters < 0 || power_iters > 1000 || !(margin >= 0.0) || !(margin <= 1.0))
    return PE_ERR_INVALID_ARG;
  c->init_iters = power_iters;
  c->init_margin = margin;
  return PE_OK;
}

extern "C" pe_status pe_set_rect_iteration(pe_ctx c, int restart, double min_aspect, double shift) {
  if (!c || restart < 0 || !(shift >= 0.0) || !(shift < 1.0) || std::isnan(min_aspect)) return PE_ERR_INVALID_ARG;
  c->rect_restart = restart;
  c->rect_min_aspect = min_aspect;
  c->rect_shift = shift;
  return PE_OK;
}

extern "C" pe_status pe_last_launch_count(pe_ctx c, int* n) {
  if (!c || !n) return PE_ERR_INVALID_ARG;
  *n = c->last_launches;
  return PE_OK;
}

// ---------------------------------------------------------------- planning
static pe_status validate_shapes(const int64_t* shapes, int count) {
  if (count < 0 || (count > 0 && !shapes)) return PE_ERR_INVALID_ARG;
  for (int i = 0; i < count; ++i) {
    const int64_t r = shapes[2 * i], cc = shapes[2 * i + 1];
    if (r < 1 || cc < 1 || r > (1 << 20) || cc > (1 << 20)) return PE_ERR_INVALID_ARG;
  }
  return PE_OK;
}

// bf16 2-D tensor map over a rows x cols row-major buffer with leading dim ld
// and a box of (box_cols x box_rows) elements.  Main-loop operands use 64x64
// boxes with the 128B swizzle; epilogue chunks 16x32 (or 32x16 for the
// transposed chunks of tall caller matrices) without swizzle.
static pe_status make_tmap(CUtensorMap* map, void* base, int rows, int cols, int ld, int box_cols = 64,
                           int box_rows = 64, bool sw128 = true) {
  EncodeTiledFn enc = get_encode_fn();
  cuuint64_t gdim[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t gstride[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, gdim, gstride, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    g_last_error = "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")";
    return PE_ERR_CUDA;
  }
  return PE_OK;
}
// Epilogue chunk maps: 64 columns x 32 rows with the 128B swizzle, or the
// transposed 32 x 64 chunk (tall caller matrices) without swizzle.
static pe_status make_emap(CUtensorMap* map, void* base, int rows, int cols, int ld, bool transposed = false) {
  return transposed ? make_tmap(map, base, rows, cols, ld, 32, kEpiCols, false)
                    : make_tmap(map, base, rows, cols, ld, kEpiCols, 32, true);
}

// Grow the shared workspace; every cached plan points into it, so growth
// drops the cache (after the device has finished with it).  Plans a captured
// CUDA graph uses (pinned) and the workspace they carve are retired instead of
// freed: the graph may be replayed until pe_destroy.
static pe_status ensure_workspace(pe_ctx c, size_t bytes) {
  if (bytes <= c->ws_bytes) return PE_OK;
  PE_CUDA(cudaDeviceSynchronize());
  bool keep_ws = false;
  for (Plan* p : c->plans) {
    if (p->pinned) { c->retired_plans.push_back(p); keep_ws = true; }
    else free_plan(p);
  }
  c->plans.clear();
  if (c->ws) {
    if (keep_ws) c->retired_ws.push_back(c->ws);
    else cudaFree(c->ws);
    c->ws = nullptr;
    c->ws_bytes = 0;
  }
  if (cudaMalloc(&c->ws, bytes) != cudaSuccess) {
    cudaGetLastError();
    g_last_error = "workspace allocation of " + std::to_string(bytes) + " bytes failed";
    return PE_ERR_WORKSPACE;
  }
  c->ws_bytes = bytes;
  return PE_OK;
}

// per-call upload: 4*count pointers, then 3 tensor maps per matrix (caller
// input main loop, caller input epilogue chunk, caller output epilogue chunk)
static size_t call_ptr_bytes(int count) { return rup((size_t)5 * count * sizeof(void*), 128); }
static size_t call_coef_off(int count) { return call_ptr_bytes(count) + (size_t)3 * count * sizeof(CUtensorMap); }
static size_t call_bytes(int count, int T) { return call_coef_off(count) + (size_t)3 * T * sizeof(float); }

// no_orient: keep rows as the Gram side even when rows > cols (a column
// shard of a wide matrix, pe_polar_split).
// io (bf16 compute only, pe_polar_ex): bit 0 = the caller's input is fp32,
// bit 1 = the caller's output is fp32; such matrices go through the copy
// passes (conversion) instead of being folded into the first / last GEMM.
// no_direct: the last update never writes the caller's buffer (it writes the
// workspace and the finalize pass copies out) -- a one-step call whose output
// overlaps an input: that update reads the caller's M across whole column
// panels while other tiles store, so a direct store would race (in == out).
static std::vector<int64_t> plan_key(const int64_t* shapes, int count, bool no_orient, int io, bool no_direct,
                                     bool rect = false, bool init = false) {
  std::vector<int64_t> key(shapes, shapes + 2 * count);
  if (no_orient) key.push_back(-1);
  if (io) key.push_back(-2 - io);
  if (no_direct) key.push_back(-100);
  if (rect) key.push_back(-200);
  if (init) key.push_back(-300);
  return key;
}

static pe_status build_plan(pe_ctx c, const int64_t* shapes, int count, pe_dtype dtype, Plan** out,
                            bool no_orient = false, int io = 0, bool no_direct = false, bool rect = false,
                            bool init = false) {
  const std::vector<int64_t> key = plan_key(shapes, count, no_orient, io, no_direct, rect, init);
  for (Plan* p : c->plans)
    if (p->dtype == dtype && p->key == key) {
      p->last_use = ++c->use_clock;
      *out = p;
      return PE_OK;
    }
  // workspace element: bf16; fp32 buffers are three stacked bf16 planes
  const size_t np = (dtype == PE_BF16) ? 1 : 3;
  Plan* P = nullptr;

  // workspace carve-up
  std::vector<MatDev> mats(count);
  std::vector<size_t> offs(count * 9, 0);
  size_t total = 0;
  for (int i = 0; i < count; ++i) {
    MatDev& md = mats[i];
    md.rows = (int)shapes[2 * i];
    md.cols = (int)shapes[2 * i + 1];
    md.tall = !no_orient && md.rows > md.cols;   // P:493, strict (R10)
    md.m = md.tall ? md.cols : md.rows;
    md.n = md.tall ? md.rows : md.cols;
    md.ldx = (int)rup(md.n, 8);
    md.ldm = (int)rup(md.m, 8);
    const size_t xb = rup(np * md.m * md.ldx * 2, 256);
    const size_t mb = rup(np * md.m * md.ldm * 2, 256);
    offs[9 * i + 0] = total; total += xb;
    offs[9 * i + 1] = total; total += xb;
    offs[9 * i + 2] = total; total += mb;
    offs[9 * i + 3] = total; total += mb;
    for (int e = 0; e < 4 && rect; ++e) { offs[9 * i + 4 + e] = total; total += mb; }   // Q_0, Q_1, T, R
    if (init) { offs[9 * i + 8] = total; total += rup((size_t)md.m * md.ldm * 4, 256); }  // fp32 Gram
  }
  pe_status s = ensure_workspace(c, std::max<size_t>(total, 256));
  if (s != PE_OK) return s;
  P = new Plan();
  P->key = key;
  P->dtype = dtype;
  P->ws_needed = total;
  uint8_t* ws = reinterpret_cast<uint8_t*>(c->ws);
  P->rect = rect;
  P->tstride = rect ? 11 : 6;
  P->estride = rect ? 8 : 4;
  for (int i = 0; i < count; ++i) {
    mats[i].X[0] = ws + offs[9 * i + 0];
    mats[i].X[1] = ws + offs[9 * i + 1];
    mats[i].A = ws + offs[9 * i + 2];
    mats[i].B = ws + offs[9 * i + 3];
    for (int e = 0; e < 4; ++e) mats[i].E[e] = rect ? ws + offs[9 * i + 4 + e] : nullptr;
  }
  P->init = init;

  // GEMM tile lists: 256x256 pair tiles, symmetric phases only I <= J.
  // Update tiles are generated row-block fastest so concurrently running
  // tiles share a column panel of X (L2 reuse); lists are then stably sorted
  // longest K first.
  // Matrices with more than 16 row blocks (m > 4096) are walked in bands of
  // kBand = 8 row blocks (grouped rasterisation): a wave of ~74 concurrent
  // tiles then touches about 8 + 74 / 8 operand panels instead of 1 + 74, so
  // the panels it streams are shared through L2 (16384^2: 8 MB per panel;
  // call 77.6 -> 70.7 ms, 8192^2 7.63 -> 7.48 ms).  At m = 4096 the plain
  // orders measured 2-4 % faster (the whole iterate is about L2-sized), so
  // smaller matrices keep them.
  std::vector<Tile> sym, upd;
  const int tile = kBN;
  static const int kBand = getenv("PE_BAND") ? std::max(1, atoi(getenv("PE_BAND"))) : 8;   // A/B knob
  for (int i = 0; i < count; ++i) {
    const MatDev& md = mats[i];
    const int nm = cdiv(md.m, tile), nn = cdiv(md.n, tile);
    const int band = (nm > 16) ? kBand : nm;
    if (band == nm) {
      for (int tm = 0; tm < nm; ++tm)
        for (int tn = tm; tn < nm; ++tn) sym.push_back({i, tm, tn, 0});
    } else {
      for (int b0 = 0; b0 < nm; b0 += band)
        for (int tn = b0; tn < nm; ++tn)
          for (int tm = b0; tm < std::min(b0 + band, nm) && tm <= tn; ++tm) sym.push_back({i, tm, tn, 0});
    }
    for (int b0 = 0; b0 < nm; b0 += band)
      for (int tn = 0; tn < nn; ++tn)
        for (int tm = b0; tm < std::min(b0 + band, nm); ++tm) upd.push_back({i, tm, tn, 0});
  }
  auto by_k = [&](bool gram) {
    return [&, gram](const Tile& x, const Tile& y) {
      const int64_t kx = gram ? mats[x.mat].n : mats[x.mat].m;
      const int64_t ky = gram ? mats[y.mat].n : mats[y.mat].m;
      return kx > ky;
    };
  };
  std::stable_sort(sym.begin(), sym.end(), by_k(true));
  std::stable_sort(upd.begin(), upd.end(), by_k(false));
  // Alg. 4 plans: every 256 x 256 tile of the m x m products (T = Y Q,
  // Q' = a Q + H Q), and the 64 x 64 tiles of the Q_1 expansion
  std::vector<Tile> sq;
  std::vector<CopyItem> exp_items;
  for (int i = 0; i < count && rect; ++i) {
    const int nm = cdiv(mats[i].m, tile);
    for (int tm = 0; tm < nm; ++tm)
      for (int tn = 0; tn < nm; ++tn) sq.push_back({i, tm, tn, 0});
    for (int a = 0; a < cdiv(mats[i].m, 64); ++a)
      for (int b = 0; b < cdiv(mats[i].m, 64); ++b) exp_items.push_back({i, a, b, 0});
  }
  std::stable_sort(sq.begin(), sq.end(), by_k(false));

  // tensor maps: main loop over all planes of a buffer stacked (plane p =
  // rows [p m, (p+1) m)), epilogue one map per plane (stores clip at row m)
  // (A and B: 128-row boxes for the stored blocks, 64x64 boxes for the
  // transposed reads of the blocks below the diagonal, gemm_sm100.cuh)
  // Alg. 4 plans add main-loop maps 6 Q_0, 7 Q_1, 8 T (64 x 64 boxes: read
  // K-major as a left operand or MN-major as a right one), 9 / 10 R (as A),
  // and epilogue maps 4 Q_0, 5 Q_1, 6 T, 7 R
  const int ts = P->tstride, es = P->estride;
  std::vector<CUtensorMap> tmaps(ts * (size_t)count), emaps(es * np * (size_t)count);
  for (int i = 0; i < count; ++i) {
    const MatDev& md = mats[i];
    const int pr = (int)np * md.m;
    CUtensorMap* tm = &tmaps[(size_t)ts * i];
    if ((s = make_tmap(&tm[0], md.X[0], pr, md.n, md.ldx)) != PE_OK ||
        (s = make_tmap(&tm[1], md.X[1], pr, md.n, md.ldx)) != PE_OK ||
        (s = make_tmap(&tm[2], md.A, pr, md.m, md.ldm, 64, 128)) != PE_OK ||
        (s = make_tmap(&tm[3], md.B, pr, md.m, md.ldm, 64, 128)) != PE_OK ||
        (s = make_tmap(&tm[4], md.A, pr, md.m, md.ldm)) != PE_OK ||
        (s = make_tmap(&tm[5], md.B, pr, md.m, md.ldm)) != PE_OK ||
        (rect && ((s = make_tmap(&tm[6], md.E[0], md.m, md.m, md.ldm)) != PE_OK ||
                  (s = make_tmap(&tm[7], md.E[1], md.m, md.m, md.ldm)) != PE_OK ||
                  (s = make_tmap(&tm[8], md.E[2], md.m, md.m, md.ldm)) != PE_OK ||
                  (s = make_tmap(&tm[9], md.E[3], md.m, md.m, md.ldm, 64, 128)) != PE_OK ||
                  (s = make_tmap(&tm[10], md.E[3], md.m, md.m, md.ldm)) != PE_OK))) {
      delete P;
      return s;
    }
    void* bufs[8] = {md.X[0], md.X[1], md.A, md.B, md.E[0], md.E[1], md.E[2], md.E[3]};
    for (int b = 0; b < es; ++b) {
      const int cols = (b < 2) ? md.n : md.m, ld = (b < 2) ? md.ldx : md.ldm;
      for (size_t p = 0; p < np; ++p) {
        void* base = reinterpret_cast<uint8_t*>(bufs[b]) + p * md.m * ld * 2;
        if ((s = make_emap(&emaps[((size_t)es * i + b) * np + p], base, md.m, cols, ld)) != PE_OK) {
          delete P;
          return s;
        }
      }
    }
  }

  // norm chunks
  std::vector<int64_t> elems(count);
  std::vector<int> cmat, cidx, nch(count);
  for (int i = 0; i < count; ++i) {
    elems[i] = (int64_t)mats[i].rows * mats[i].cols;
    nch[i] = cdiv(elems[i], kNormChunk);
    for (int k = 0; k < nch[i]; ++k) { cmat.push_back(i); cidx.push_back(k); }
  }
  // Folding (gemm_sm100.cuh): bf16 matrices whose rows are 16-byte multiples
  // are read by the first iteration straight from the caller's buffer and the
  // last iteration writes the caller's buffer; the others go through the copy
  // passes (see elementwise.cuh): item lists 0 scale-rows, 1 scale-transpose,
  // 2 finalize-transpose, 3 finalize-rows.  fp32: every matrix goes through
  // the split (0/1) and join (2/3) passes, items are 64x64 source tiles.
  std::vector<int> mflags(count, 0);
  std::vector<CopyItem> it[4];
  std::vector<CopyMat> smats(count), fmats(count);
  std::vector<void*> x0(count);
  for (int i = 0; i < count; ++i) {
    const MatDev& md = mats[i];
    const bool foldable = (dtype == PE_BF16) && (md.cols % 8 == 0) && !getenv("PE_NO_FOLD");
    const bool folded = foldable && !(io & 1);
    const bool direct = foldable && !(io & 2) && !no_direct;
    // bf16 input: X_0 is never rounded -- the copy pass (if any) stores
    // M * 2^e exactly (pow2_part of 1/s) and iteration 1 applies the residual
    // 1/s * 2^-e, bit-identical to the folded path (R8, R18); rounding
    // bf16(M/s) would add a second input-sized rounding noise that the
    // iteration lifts as if it were spectrum
    const bool scaled = (dtype == PE_BF16) && !(io & 1);
    mflags[i] = (folded ? kFlagFolded : 0) | (md.tall ? kFlagTall : 0) | (direct ? kFlagDirect : 0) |
                (scaled ? kFlagScaled : 0);
    x0[i] = md.X[0];
    const int64_t pst = (int64_t)md.m * md.ldx;
    smats[i] = {md.rows, md.cols, md.cols, md.ldx, pst};
    fmats[i] = {md.m, md.n, md.ldx, md.tall ? md.m : md.n, pst};
    const int band = std::max(1, 16384 / md.cols);
    if (dtype == PE_FP32) {
      for (int a = 0; a < cdiv(md.rows, 64); ++a)
        for (int b = 0; b < cdiv(md.cols, 64); ++b) it[md.tall ? 1 : 0].push_back({i, a, b, 0});
      for (int a = 0; a < cdiv(md.m, 64); ++a)
        for (int b = 0; b < cdiv(md.n, 64); ++b) it[md.tall ? 2 : 3].push_back({i, a, b, 0});
      continue;
    }
    if (!folded) {
      if (md.tall) {
        for (int a = 0; a < cdiv(md.rows, 64); ++a)
          for (int b = 0; b < cdiv(md.cols, 64); ++b) it[1].push_back({i, a, b, 0});
      } else {
        for (int r = 0; r < md.rows; r += band) it[0].push_back({i, r, std::min(band, md.rows - r), 0});
      }
    }
    if (!direct) {
      if (md.tall) {
        for (int a = 0; a < cdiv(md.m, 64); ++a)
          for (int b = 0; b < cdiv(md.n, 64); ++b) it[2].push_back({i, a, b, 0});
      } else {
        for (int r = 0; r < md.m; r += band) it[3].push_back({i, r, std::min(band, md.m - r), 0});
      }
    }
  }

  Blob bl;
  P->o_mats = bl.add(mats);
  P->o_tmaps = bl.add(tmaps, 128);
  P->o_emaps = bl.add(emaps, 128);
  P->o_sym = bl.add(sym);
  P->o_upd = bl.add(upd);
  // the same lists reversed: consecutive phases walk the batch in opposite
  // directions, so each phase starts on the buffers the previous one wrote
  // last (still in L2)
  std::vector<Tile> sym_r(sym.rbegin(), sym.rend()), upd_r(upd.rbegin(), upd.rend());
  P->o_sym_r = bl.add(sym_r);
  P->o_upd_r = bl.add(upd_r);
  if (rect) {
    std::vector<Tile> sq_r(sq.rbegin(), sq.rend());
    P->o_sq = bl.add(sq);
    P->o_sq_r = bl.add(sq_r);
    P->o_exp = bl.add(exp_items);
    P->n_sq = (int)sq.size();
    P->n_exp = (int)exp_items.size();
  }
  for (int k = 0; k < 4; ++k) P->o_it[k] = bl.add(it[k]);
  P->o_smats = bl.add(smats);
  P->o_fmats = bl.add(fmats);
  P->o_x0 = bl.add(x0);
  P->o_flags = bl.add(mflags);
  P->o_elems = bl.add(elems);
  P->o_cmat = bl.add(cmat);
  P->o_cidx = bl.add(cidx);
  P->o_nch = bl.add(nch);
  std::vector<double> part(cmat.size(), 0.0);
  P->o_part = bl.add(part);
  std::vector<unsigned> cnt(count, 0u);
  P->o_cnt = bl.add(cnt);
  std::vector<float> inv(count, 0.f);
  P->o_inv = bl.add(inv);
  std::vector<int> need(3 * (size_t)count);
  for (int i = 0; i < count; ++i) {
    const int nm = cdiv(mats[i].m, kBN), nn = cdiv(mats[i].n, kBN);
    need[3 * i + kModeGram] = need[3 * i + kModePoly] = 2 * kEpiWarps * nm * (nm + 1) / 2;
    need[3 * i + kModeUpdate] = 2 * kEpiWarps * nm * nn;
  }
  P->o_need = bl.add(need);
  {
    std::vector<int> imat, ir0, i0(count), ni(count);
    std::vector<int64_t> voff(count);
    int64_t vlen = 0;
    for (int i = 0; i < count; ++i) {
      i0[i] = (int)imat.size();
      for (int r = 0; r < mats[i].m; r += kSymvRows) { imat.push_back(i); ir0.push_back(r); }
      ni[i] = (int)imat.size() - i0[i];
      voff[i] = vlen;
      vlen += rup(mats[i].m, 32);
    }
    P->o_sitem_mat = bl.add(imat);
    P->o_sitem_r0 = bl.add(ir0);
    P->o_sitem0 = bl.add(i0);
    P->o_snitem = bl.add(ni);
    P->o_svoff = bl.add(voff);
    P->o_sv = bl.add(std::vector<float>(2 * (size_t)vlen, 0.f));
    // the power method's start vector, v0_i = frac((i + 1) / phi) + 0.5 per
    // matrix (the oracle's power_start, same counter; reading R17)
    std::vector<float> v0((size_t)vlen, 0.f);
    for (int i = 0; i < count; ++i)
      for (int r = 0; r < mats[i].m; ++r) {
        const double x = (double)(r + 1) * 0.6180339887498949;
        v0[(size_t)voff[i] + r] = (float)(x - std::floor(x) + 0.5);
      }
    P->o_sv0 = bl.add(v0);
    P->o_spart = bl.add(std::vector<double>(3 * imat.size() + 3, 0.0));
    P->o_scnt = bl.add(std::vector<unsigned>(count, 0u));
    P->o_slam = bl.add(std::vector<double>(count, 0.0));
    P->o_snrm = bl.add(std::vector<double>(2 * (size_t)count, 0.0));
    P->o_sssq = bl.add(std::vector<double>(count, 0.0));
    P->o_str = bl.add(std::vector<double>(count, 0.0));
    P->o_smcoef = bl.add(std::vector<float>(2 * (size_t)count, 0.f));
    std::vector<float*> a32(count, nullptr);
    for (int i = 0; i < count && init; ++i) a32[i] = reinterpret_cast<float*>(ws + offs[9 * i + 8]);
    P->o_a32 = bl.add(a32);
    P->n_sitems = (int)imat.size();
    P->sv_len = vlen;
  }

  if (cudaMalloc(&P->meta, bl.host.size()) != cudaSuccess) {
    cudaGetLastError();
    delete P;
    return PE_ERR_WORKSPACE;
  }
  P->meta_bytes = bl.host.size();
  if (cudaMemcpy(P->meta, bl.host.data(), bl.host.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
    g_last_error = "plan upload failed";
    free_plan(P);
    return PE_ERR_CUDA;
  }
  P->flags = mflags;
  P->mats = mats;
  P->count = count;
  P->n_sym = (int)sym.size();
  P->n_upd = (int)upd.size();
  for (int k = 0; k < 4; ++k) P->n_it[k] = (int)it[k].size();
  P->n_chunks = (int)cmat.size();
  // LRU eviction (the evicted plan's kernels may still be queued: sync
  // first); a pinned plan leaves the cache but stays alive (retired)
  if ((int)c->plans.size() >= kMaxPlans) {
    auto lru = std::min_element(c->plans.begin(), c->plans.end(),
                                [](const Plan* a, const Plan* b) { return a->last_use < b->last_use; });
    PE_CUDA(cudaDeviceSynchronize());
    if ((*lru)->pinned) c->retired_plans.push_back(*lru);
    else free_plan(*lru);
    c->plans.erase(lru);
  }
  P->last_use = ++c->use_clock;
  c->plans.push_back(P);
  *out = P;
  return PE_OK;
}

// Tile order of the fused schedule (GemmArgs::nphase): a window of matrices
// advances one phase per round, every matrix of the window emitting all tiles
// of its next phase; matrices join (largest cost first) while a round has
// fewer than ~3 tiles per cluster or fewer than two matrices.  Phase p of a
// matrix is emitted one round after phase p - 1, so the list is in dependency
// order (no deadlock under static round-robin assignment) and the tiles a
// cluster waits for were issued about a round earlier; the window's buffers
// stay L2-resident across its phases.
static void build_fused_order(const std::vector<MatDev>& mats, int T, int nclusters, std::vector<Tile>& out) {
  const int count = (int)mats.size();
  auto ntiles = [&](int i, int mode) {
    const int nm = cdiv(mats[i].m, kBN), nn = cdiv(mats[i].n, kBN);
    return mode == kModeUpdate ? nm * nn : nm * (nm + 1) / 2;
  };
  auto emit = [&](int i, int p) {
    const int nm = cdiv(mats[i].m, kBN), nn = cdiv(mats[i].n, kBN);
    if (p % 3 == kModeUpdate) {
      for (int tn = 0; tn < nn; ++tn)
        for (int tm = 0; tm < nm; ++tm) out.push_back({i, tm, tn, p});
    } else {
      for (int tm = 0; tm < nm; ++tm)
        for (int tn = tm; tn < nm; ++tn) out.push_back({i, tm, tn, p});
    }
  };
  std::vector<double> cost(count);
  for (int i = 0; i < count; ++i) cost[i] = 3.0 * mats[i].m * (double)mats[i].m * mats[i].n + (double)mats[i].m * mats[i].m * mats[i].m;
  std::vector<int> order(count);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost[a] > cost[b]; });
  const int nph = 3 * T;
  static const int round_mult = getenv("PE_FUSED_ROUND") ? atoi(getenv("PE_FUSED_ROUND")) : 3;   // experiments
  const int round_min = round_mult * nclusters;
  std::vector<int> ph(count, 0), window, keep;
  size_t next = 0;
  out.clear();
  while (next < order.size() || !window.empty()) {
    int est = 0;
    for (int i : window) est += ntiles(i, ph[i] % 3);
    while (next < order.size() && (est < round_min || window.size() < 2)) {
      const int i = order[next++];
      window.push_back(i);
      est += ntiles(i, 0);
    }
    keep.clear();
    for (int i : window) {
      emit(i, ph[i]);
      if (++ph[i] < nph) keep.push_back(i);
    }
    window.swap(keep);
  }
}

static pe_status ensure_fused(pe_ctx c, Plan* P, int T) {
  if (P->fused_T == T) return PE_OK;
  std::vector<Tile> order;
  build_fused_order(P->mats, T, c->num_sms / 2, order);
  const size_t bytes = order.size() * sizeof(Tile);
  PE_CUDA(cudaDeviceSynchronize());          // the previous list may still be in use
  if (bytes > P->fused_cap) {
    if (P->fused) cudaFree(P->fused);
    P->fused = nullptr;
    P->fused_cap = 0;
    if (cudaMalloc(&P->fused, bytes) != cudaSuccess) { cudaGetLastError(); return PE_ERR_WORKSPACE; }
    P->fused_cap = bytes;
  }
  PE_CUDA(cudaMemcpy(P->fused, order.data(), bytes, cudaMemcpyHostToDevice));
  P->n_fused = (int)order.size();
  P->fused_T = T;
  return PE_OK;
}

// Device buffer + mapped pinned host buffer of one upload slot.
static bool alloc_slot(CallSlot& cs, size_t nb) {
  void* hd = nullptr;
  if (cudaMalloc(&cs.d, nb) != cudaSuccess || cudaHostAlloc(&cs.h, nb, cudaHostAllocMapped) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  cs.hd = (cudaHostGetDevicePointer(&hd, cs.h, 0) == cudaSuccess) ? hd : nullptr;
  cudaGetLastError();
  return true;
}

constexpr int kCaptureSpare = 4;
constexpr int kCaptureMaxIters = 64;

extern "C" pe_status pe_reserve(pe_ctx c, const int64_t* shapes, int count, pe_dtype dtype) {
  if (!c || (dtype != PE_BF16 && dtype != PE_FP32)) return PE_ERR_INVALID_ARG;
  pe_status s = validate_shapes(shapes, count);
  if (s != PE_OK) return s;
  PE_CUDA(cudaSetDevice(c->device));
  Plan* P = nullptr;
  // the plan a later call will look up (App. G plans carry the fp32 Gram)
  const bool init = c->init_iters > 0 && dtype == PE_BF16;
  if ((s = build_plan(c, shapes, count, dtype, &P, false, 0, false, false, init)) != PE_OK) return s;
  if (dtype == PE_FP32 && !c->scratch) {
    const size_t sb = (size_t)c->num_sms * (kBM / 2) * kBN * sizeof(float);
    if (cudaMalloc(&c->scratch, sb) != cudaSuccess) { cudaGetLastError(); return PE_ERR_WORKSPACE; }
  }
  // spare upload slots for calls captured into CUDA graphs
  const size_t need = call_bytes(count, kCaptureMaxIters);
  size_t spare = 0;
  for (size_t i = c->cap_used; i < c->cap_slots.size(); ++i) {
    CallSlot& cs = c->cap_slots[i];
    if (cs.bytes < need) {
      if (cs.d) cudaFree(cs.d);
      if (cs.h) cudaFreeHost(cs.h);
      cs = CallSlot();
      if (!alloc_slot(cs, need)) return PE_ERR_WORKSPACE;
      cs.bytes = need;
    }
    ++spare;
  }
  while (spare < (size_t)kCaptureSpare) {
    CallSlot cs;
    if (!alloc_slot(cs, need)) return PE_ERR_WORKSPACE;
    cs.bytes = need;
    c->cap_slots.push_back(cs);
    ++spare;
  }
  return PE_OK;
}

// ---------------------------------------------------------------- online
template <typename T> static T* at(const Plan* p, size_t off) {
  return reinterpret_cast<T*>(reinterpret_cast<uint8_t*>(p->meta) + off);
}

// Next upload buffer of the ring, large enough for `bytes`; waits only if the
// GPU has not yet consumed this slot's previous upload.
static pe_status take_call_slot(pe_ctx c, size_t bytes, CallSlot** out) {
  CallSlot& cs = c->calls[c->next_call];
  c->next_call = (c->next_call + 1) % kCallSlots;
  if (cs.armed) PE_CUDA(cudaEventSynchronize(cs.done));
  cs.armed = false;
  if (!cs.done) PE_CUDA(cudaEventCreateWithFlags(&cs.done, cudaEventDisableTiming));
  if (cs.bytes < bytes) {
    if (cs.d) { cudaFree(cs.d); cs.d = nullptr; }
    if (cs.h) { cudaFreeHost(cs.h); cs.h = nullptr; }
    cs.bytes = 0;
    const size_t nb = std::max<size_t>(bytes, 64 * 1024);
    if (!alloc_slot(cs, nb)) return PE_ERR_WORKSPACE;
    cs.bytes = nb;
  }
  *out = &cs;
  return PE_OK;
}

// Upload buffer of one call: the next ring slot, or -- while the stream is
// being captured into a CUDA graph -- a reserved slot the graph keeps.
static pe_status upload_slot(pe_ctx c, size_t bytes, bool capturing, int T, CallSlot** out) {
  if (!capturing) return take_call_slot(c, bytes, out);
  while (c->cap_used < c->cap_slots.size() && c->cap_slots[c->cap_used].bytes < bytes) ++c->cap_used;
  if (c->cap_used == c->cap_slots.size() || T > kCaptureMaxIters) {
    g_last_error = "pe_polar under CUDA-graph capture: call pe_reserve for this batch before capturing "
                   "(it keeps 4 upload slots per reservation; iters <= 64)";
    return PE_ERR_WORKSPACE;
  }
  *out = &c->cap_slots[c->cap_used++];
  return PE_OK;
}

// Small-matrix fused path (small_sm100.cuh): every matrix of the call has
// min side <= 128 and max side <= 768 (bf16) / 128 (fp32): one CTA per
// matrix runs the whole call.
static bool small_eligible(const int64_t* shapes, int count, pe_dtype dtype, int* max_npad) {
  static const bool on = !(getenv("PE_SMALL") && !strcmp(getenv("PE_SMALL"), "0"));   // A/B knob
  if (!on || count < 1) return false;
  int mx = 64;
  for (int i = 0; i < count; ++i) {
    const int64_t r = shapes[2 * i], cc = shapes[2 * i + 1];
    const int64_t m = std::min(r, cc), npad = rup(std::max(r, cc), 64);
    if (m > kSmallMaxM || npad > (dtype == PE_BF16 ? kSmallMaxNpadBf16 : kSmallMaxNpadF32)) return false;
    mx = std::max<int>(mx, (int)npad);
  }
  *max_npad = mx;
  return true;
}

// Per-call upload of `bytes` from the slot's pinned buffer.  `up` (pe_polar_host)
// is the H2D copy stream: queued there, the small upload is not stuck behind
// the next group's bulk copies in the copy engine; the kernels on `st` wait
// for it through the slot's event.
static pe_status upload_call(pe_ctx c, CallSlot* cs, size_t bytes, cudaStream_t st, cudaStream_t up,
                             bool capturing) {
  if (cs->hd && !getenv("PE_UPLOAD_MEMCPY")) {
    // the SMs read the mapped host buffer: no copy-engine queue on the way
    const int n = (int)((bytes + 15) / 16);
    launch(pe_upload_kernel, std::min(cdiv(n, 256), 16), 256, 0, st, reinterpret_cast<const uint4*>(cs->hd),
           reinterpret_cast<uint4*>(cs->d), n);
    ++c->uploads;
    if (!capturing) {
      PE_CUDA(cudaEventRecord(cs->done, st));
      cs->armed = true;
    }
    return PE_OK;
  }
  cudaStream_t us = up ? up : st;
  PE_CUDA(cudaMemcpyAsync(cs->d, cs->h, bytes, cudaMemcpyHostToDevice, us));
  if (!capturing) {
    PE_CUDA(cudaEventRecord(cs->done, us));
    cs->armed = true;
    if (us != st) PE_CUDA(cudaStreamWaitEvent(st, cs->done, 0));
  }
  return PE_OK;
}

static pe_status small_call(pe_ctx c, const void* const* in, void* const* out, const int64_t* shapes, int count,
                            int T, pe_dtype dtype, cudaStream_t st, bool capturing, int max_npad, cudaStream_t up) {
  SmallArgs a;                                      // ~3 KB of kernel parameters
  c->uploads = 0;
  // CTA table: one matrix per CTA while that fits in one wave (one CTA per
  // SM); beyond, just enough pairs of matrices with min side <= 64 share a
  // CTA (packed rows 0-63 / 64-127; neighbours in padded width) to get back
  // to one wave if possible (a pair takes longer than one matrix, but two
  // waves take longer than a pair: 148 tall 768x64 slices 154 us unpacked /
  // 220 us packed, 296 of them 316 / 222 us)
  std::vector<SmallCta> ctas;
  {
    std::vector<int> half, whole;
    for (int i = 0; i < count; ++i) {
      const int64_t m = std::min(shapes[2 * i], shapes[2 * i + 1]);
      (m <= 64 && !getenv("PE_SMALL_NOPACK") ? half : whole).push_back(i);
    }
    std::stable_sort(half.begin(), half.end(), [&](int x, int y) {
      return std::max(shapes[2 * x], shapes[2 * x + 1]) < std::max(shapes[2 * y], shapes[2 * y + 1]);
    });
    const int npairs = (int)std::min<int64_t>(std::max(0, count - c->num_sms), (int64_t)half.size() / 2);
    for (int k = 0; k < npairs; ++k) ctas.push_back({half[2 * k], half[2 * k + 1]});
    for (size_t k = 2 * (size_t)npairs; k < half.size(); ++k) ctas.push_back({half[k], -1});
    for (int i : whole) ctas.push_back({i, -1});
  }
  const int nctas = (int)ctas.size();
  const bool inl = count <= kSmallInlineMats && T <= kSmallInlineIters;
  CallSlot* cs = nullptr;
  const size_t mats_bytes = rup((size_t)count * sizeof(SmallMat), 128);
  const size_t cta_bytes = rup((size_t)nctas * sizeof(SmallCta), 128);
  const size_t up_bytes = mats_bytes + cta_bytes + (size_t)3 * T * sizeof(float);
  if (!inl) {
    pe_status s = upload_slot(c, std::max(call_bytes(count, T), up_bytes), capturing, T, &cs);
    if (s != PE_OK) return s;
  }
  SmallMat* hm = inl ? a.inl : reinterpret_cast<SmallMat*>(cs->h);
  for (int i = 0; i < count; ++i) {
    SmallMat& sm = hm[i];
    sm.in = in[i];
    sm.out = out[i];
    sm.rows = (int)shapes[2 * i];
    sm.cols = (int)shapes[2 * i + 1];
    sm.tall = sm.rows > sm.cols;                    // P:493, strict (R10)
    sm.m = sm.tall ? sm.cols : sm.rows;
    sm.n = sm.tall ? sm.rows : sm.cols;
    sm.n_pad = (int)rup(sm.n, 64);
    sm.fold = (dtype == PE_BF16);   // X_0 = M exactly, 1/s in iteration 1 (kFlagScaled in build_plan)
    sm.pad = 0;
  }
  SmallCta* hct = inl ? a.inl_cta : reinterpret_cast<SmallCta*>(reinterpret_cast<uint8_t*>(cs->h) + mats_bytes);
  std::copy(ctas.begin(), ctas.end(), hct);
  float* hc = inl ? a.inl_coef
                  : reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(cs->h) + mats_bytes + cta_bytes);
  const int nq = (c->degree + 1) / 2;
  for (int t = 0; t < T; ++t) {
    const double* tup = &c->table[(size_t)std::min(t, c->ntab - 1) * nq];
    hc[3 * t] = (float)tup[0];
    hc[3 * t + 1] = (float)tup[1];
    hc[3 * t + 2] = (nq == 3) ? (float)tup[2] : 0.0f;
  }
  a.T = T;
  a.lin = (nq == 2) ? 1 : 0;
  if (inl) {
    a.mats = nullptr;
    a.ctas = nullptr;
    a.coef = nullptr;
  } else {
    pe_status s = upload_call(c, cs, up_bytes, st, up, capturing);
    if (s != PE_OK) return s;
    const uint8_t* d = reinterpret_cast<const uint8_t*>(cs->d);
    a.mats = reinterpret_cast<const SmallMat*>(d);
    a.ctas = reinterpret_cast<const SmallCta*>(d + mats_bytes);
    a.coef = reinterpret_cast<const float*>(d + mats_bytes + cta_bytes);
  }
  { ProfScope ps(c, 7, st);
    if (dtype == PE_BF16 && c->small_planes == 2 && max_npad <= kSmallMaxNpadPrecise)
      launch(pe_small_sm100<1, 2>, nctas, kSmallThreads, small_smem_bytes<1, 2>(max_npad), st, a);
    else if (dtype == PE_BF16)
      launch(pe_small_sm100<1>, nctas, kSmallThreads, small_smem_bytes<1>(max_npad), st, a);
    else launch(pe_small_sm100<3>, nctas, kSmallThreads, small_smem_bytes<3>(max_npad), st, a); }
  PE_CUDA(cudaGetLastError());
  c->last_launches = 1 + c->uploads;
  return PE_OK;
}

// Does any output range overlap any input range (byte intervals)?
static bool outputs_overlap_inputs(const void* const* in, void* const* out, const int64_t* shapes, int count,
                                   pe_dtype dtype, int io) {
  const size_t ies = (dtype == PE_FP32 || (io & 1)) ? 4 : 2, oes = (dtype == PE_FP32 || (io & 2)) ? 4 : 2;
  std::vector<std::pair<uintptr_t, uintptr_t>> ri(count), ro(count);
  for (int i = 0; i < count; ++i) {
    const size_t e = (size_t)shapes[2 * i] * (size_t)shapes[2 * i + 1];
    ri[i] = {reinterpret_cast<uintptr_t>(in[i]), reinterpret_cast<uintptr_t>(in[i]) + e * ies};
    ro[i] = {reinterpret_cast<uintptr_t>(out[i]), reinterpret_cast<uintptr_t>(out[i]) + e * oes};
  }
  std::sort(ri.begin(), ri.end());
  std::vector<uintptr_t> end_max(count);            // max end over the first k + 1 sorted inputs
  for (int i = 0; i < count; ++i) end_max[i] = std::max(ri[i].second, i ? end_max[i - 1] : 0);
  for (const auto& o : ro) {
    // inputs starting before o's end overlap o iff one of them ends after o's start
    const size_t k = std::lower_bound(ri.begin(), ri.end(), std::make_pair(o.second, (uintptr_t)0)) - ri.begin();
    if (k > 0 && end_max[k - 1] > o.first) return true;
  }
  return false;
}

// pe_polar_split: the all-reduce hook of one call
struct SplitCtx {
  pe_allreduce_fn fn;            // all-reduce hook (pe_polar_split), or
  void* user;
  // pe_polar_split_peers: every rank's partials in peer-visible slots, a
  // barrier between writing and summing them (fn == nullptr)
  void* const* slots = nullptr;
  int rank = 0, world = 1;
  pe_barrier_fn barrier = nullptr;
};

// pe_polar and pe_muon_step.  Muon (grads != nullptr, bf16): `in` are the
// momentum buffers M, updated in place by the norm kernel to
// bf16(beta M + (1 - beta) G); `out` are the weights W, updated to
// bf16(W - lr bf16(polar(M))) by the last update's epilogue (folded
// matrices) or the finalize pass (the others).
static pe_status polar_impl(pe_ctx c, const void* const* in, void* const* out, const void* const* grads,
                            const int64_t* shapes, int count, int iters, pe_dtype dtype, void* stream_,
                            double beta, double lr, cudaStream_t up = nullptr, const SplitCtx* sh = nullptr,
                            int io = 0) {
  if (!c || iters < 1 || (dtype != PE_BF16 && dtype != PE_FP32)) return PE_ERR_INVALID_ARG;
  if (count == 0) { c->last_launches = 0; return PE_OK; }
  if (!in || !out) return PE_ERR_INVALID_ARG;
  const bool muon = grads != nullptr;
  if (muon && dtype != PE_BF16) return PE_ERR_UNSUPPORTED;
  pe_status s = validate_shapes(shapes, count);
  if (s != PE_OK) return s;
  for (int i = 0; i < count; ++i) {
    if (!in[i] || !out[i] || (muon && !grads[i])) return PE_ERR_INVALID_ARG;
    if ((reinterpret_cast<uintptr_t>(in[i]) & 15) || (reinterpret_cast<uintptr_t>(out[i]) & 15) ||
        (muon && (reinterpret_cast<uintptr_t>(grads[i]) & 15))) {
      g_last_error = "buffers must be 16-byte aligned";
      return PE_ERR_INVALID_ARG;
    }
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream_);
  PE_CUDA(cudaSetDevice(c->device));
  PE_CUDA(cudaGetLastError());
  cudaStreamCaptureStatus cap_status = cudaStreamCaptureStatusNone;
  PE_CUDA(cudaStreamIsCapturing(st, &cap_status));
  const bool capturing = cap_status == cudaStreamCaptureStatusActive;
  int max_npad = 0;
  if (sh && (count != 1 || dtype != PE_BF16 || muon || capturing || shapes[1] % 8 != 0)) {
    g_last_error = "pe_polar_split: one bf16 shard with cols % 8 == 0, not under graph capture";
    return PE_ERR_UNSUPPORTED;
  }
  if (io && (dtype != PE_BF16 || muon || sh)) return PE_ERR_UNSUPPORTED;
  // App. G first step (pe_set_spectrum_init): bf16 pe_polar / pe_polar_ex, large path
  const bool init = c->init_iters > 0 && dtype == PE_BF16 && !muon && !sh;
  // App. H fast rectangular iteration (pe_set_rect_iteration): the matrices
  // whose aspect ratio passes the threshold run Alg. 4, the
  // others Listing 2; a mixed batch becomes two grouped calls on the stream
  const bool rect_ok = c->rect_restart > 0 && dtype == PE_BF16 && !muon && !sh && !init && c->degree == 5;
  if (rect_ok && c->rect_mode == 0) {
    const double thr = c->rect_min_aspect > 0.0 ? c->rect_min_aspect
                       : (iters > 1 ? 1.5 * iters / (iters - 1) : 1e300);
    std::vector<int> ri, bi;
    for (int i = 0; i < count; ++i) {
      const double m = (double)std::min(shapes[2 * i], shapes[2 * i + 1]);
      const double n = (double)std::max(shapes[2 * i], shapes[2 * i + 1]);
      ((m > kSmallMaxM && n > thr * m) ? ri : bi).push_back(i);
    }
    if (!ri.empty()) {
      if (capturing) {
        g_last_error = "pe_set_rect_iteration: Alg. 4 calls are not capturable";
        return PE_ERR_UNSUPPORTED;
      }
      int launches = 0;
      for (int part = 0; part < 2; ++part) {
        const std::vector<int>& idx = part == 0 ? bi : ri;
        if (idx.empty()) continue;
        std::vector<const void*> pin;
        std::vector<void*> pout;
        std::vector<int64_t> psh;
        for (int i : idx) {
          pin.push_back(in[i]);
          pout.push_back(out[i]);
          psh.push_back(shapes[2 * i]);
          psh.push_back(shapes[2 * i + 1]);
        }
        c->rect_mode = part == 0 ? 1 : 2;
        s = polar_impl(c, pin.data(), pout.data(), nullptr, psh.data(), (int)idx.size(), iters, dtype, stream_,
                       beta, lr, up, nullptr, io);
        c->rect_mode = 0;
        if (s != PE_OK) return s;
        launches += c->last_launches;
      }
      c->last_launches = launches;
      return PE_OK;
    }
  }
  const bool rect = rect_ok && c->rect_mode == 2;
  const int T_ = iters;
  const int rk = rect ? std::min(c->rect_restart, T_) : 1;    // iterations per application
  const int nblocks = rect ? (T_ + rk - 1) / rk : 0;
  if (!muon && !sh && !io && !init && !rect && small_eligible(shapes, count, dtype, &max_npad))
    return small_call(c, in, out, shapes, count, iters, dtype, st, capturing, max_npad, up);
  // one-step call (T = 1 without the App. G step): its only update reads the
  // caller's inputs while storing results, so an output overlapping any input
  // goes through the workspace and the finalize pass
  const bool no_direct = (rect ? nblocks == 1 : iters + (init ? 1 : 0) == 1) &&
                         outputs_overlap_inputs(in, out, shapes, count, dtype, io);
  Plan* P = nullptr;
  if (capturing) {
    // no allocation or synchronisation is allowed: the plan must be cached
    const std::vector<int64_t> key = plan_key(shapes, count, false, io, no_direct, rect, init);
    for (Plan* q : c->plans)
      if (q->dtype == dtype && q->key == key) P = q;
    if (!P || (dtype == PE_FP32 && !c->scratch)) {
      g_last_error = "pe_polar under CUDA-graph capture: call pe_reserve for this batch before capturing";
      return PE_ERR_WORKSPACE;
    }
    P->last_use = ++c->use_clock;
    P->pinned = true;       // the graph keeps pointers into it: never evicted or freed before pe_destroy
  } else if ((s = build_plan(c, shapes, count, dtype, &P, sh != nullptr, io, no_direct, rect, init)) != PE_OK) {
    return s;
  }

  // per-call pointers: [in | outs_direct | fin_src | out] + caller tensor maps
  const int T = iters;
  const int S = T + (init ? 1 : 0);     // GEMM steps: [App. G step] + T iterations
  const int xfinal = (rect ? nblocks : S) & 1;   // Alg. 4: one X-producing step per application
  // fused schedule: every GEMM phase in one launch (bf16, opt-in with
  // PE_FUSED=1; measured equal to one launch per phase on the GPT-2 sets and
  // within noise on Llama, profiles/r1_variants.md)
  static const bool fused_on = getenv("PE_FUSED") && strcmp(getenv("PE_FUSED"), "0") != 0;
  const int nq = (c->degree + 1) / 2;
  const bool fused = fused_on && dtype == PE_BF16 && !capturing && !sh && !init && !rect && nq == 3;   // (its setup may synchronise)
  if (fused) {
    if ((s = ensure_fused(c, P, T)) != PE_OK) return s;
    const size_t need_done = (size_t)count * 3 * T;
    if (need_done > c->done_cap) {
      PE_CUDA(cudaDeviceSynchronize());
      if (c->done) cudaFree(c->done);
      c->done = nullptr;
      c->done_cap = 0;
      if (cudaMalloc(&c->done, need_done * sizeof(int)) != cudaSuccess) { cudaGetLastError(); return PE_ERR_WORKSPACE; }
      PE_CUDA(cudaMemset(c->done, 0, need_done * sizeof(int)));
      c->done_cap = need_done;
    }
  }
  if (dtype == PE_FP32 && !c->scratch) {
    const size_t sb = (size_t)c->num_sms * (kBM / 2) * kBN * sizeof(float);
    if (cudaMalloc(&c->scratch, sb) != cudaSuccess) { cudaGetLastError(); return PE_ERR_WORKSPACE; }
  }
  CallSlot* cs = nullptr;
  if ((s = upload_slot(c, call_bytes(count, T), capturing, T, &cs)) != PE_OK) return s;
  void** h = reinterpret_cast<void**>(cs->h);
  const size_t omap_off = call_ptr_bytes(count);
  CUtensorMap* h_maps = reinterpret_cast<CUtensorMap*>(reinterpret_cast<uint8_t*>(h) + omap_off);
  for (int i = 0; i < count; ++i) {
    const MatDev& md = P->mats[i];
    h[i] = const_cast<void*>(in[i]);
    const int fl = P->flags[i];
    h[count + i] = (fl & kFlagDirect) ? out[i] : nullptr;
    h[2 * count + i] = md.X[xfinal];
    h[3 * count + i] = out[i];
    h[4 * count + i] = muon ? const_cast<void*>(grads[i]) : nullptr;
    if (fl & kFlagFolded) {
      void* src = const_cast<void*>(in[i]);
      if ((s = make_tmap(&h_maps[2 * i], src, md.rows, md.cols, md.cols)) != PE_OK) return s;
      if ((s = make_emap(&h_maps[2 * i + 1], src, md.rows, md.cols, md.cols, md.tall)) != PE_OK) return s;
    }
    if (dtype == PE_BF16 && (fl & kFlagDirect))
      if ((s = make_emap(&h_maps[2 * count + i], out[i], md.rows, md.cols, md.cols, md.tall)) != PE_OK) return s;
  }
  float* h_coef = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(h) + call_coef_off(count));
  for (int t = 0; t < T; ++t) {
    const double* tup = &c->table[(size_t)std::min(t, c->ntab - 1) * nq];
    h_coef[3 * t] = (float)tup[0];
    h_coef[3 * t + 1] = (float)tup[1];
    h_coef[3 * t + 2] = (nq == 3) ? (float)tup[2] : 0.0f;
  }
  c->uploads = 0;
  if ((s = upload_call(c, cs, call_bytes(count, T), st, up, capturing)) != PE_OK) return s;
  void** d_ptrs = reinterpret_cast<void**>(cs->d);
  const CUtensorMap* d_imaps =
      reinterpret_cast<const CUtensorMap*>(reinterpret_cast<const uint8_t*>(cs->d) + omap_off);
  const CUtensorMap* d_omaps = d_imaps + 2 * count;
  void** d_in = d_ptrs;
  const float* d_coef = reinterpret_cast<const float*>(reinterpret_cast<const uint8_t*>(cs->d) + call_coef_off(count));
  void** d_fin_src = d_ptrs + 2 * count;
  void** d_out = d_ptrs + 3 * count;
  const int src_f32 = (dtype == PE_FP32) || (io & 1);
  int launches = 0;

  // 1) norm
  NormArgs na;
  na.srcs = d_in;
  na.elems = at<int64_t>(P, P->o_elems);
  na.chunk_mat = at<int>(P, P->o_cmat);
  na.chunk_idx = at<int>(P, P->o_cidx);
  na.nchunks = at<int>(P, P->o_nch);
  na.partials = at<double>(P, P->o_part);
  na.counters = at<unsigned>(P, P->o_cnt);
  na.inv = at<float>(P, P->o_inv);
  na.src_f32 = src_f32;
  na.zero = fused ? c->done : nullptr;
  na.nzero = fused ? count * 3 * T : 0;
  na.grads = muon ? d_ptrs + 4 * count : nullptr;
  na.beta = (float)beta;
  na.omb = (float)(1.0 - beta);
  na.sums = nullptr;
  na.nblk = P->n_chunks;
  na.ssq = init ? at<double>(P, P->o_sssq) : nullptr;
  if (sh) {
    // buffers of the sharded call: local sum of squares, fp32 partial Gram
    const MatDev& md = P->mats[0];
    const size_t need = (size_t)md.m * md.ldm;
    if (need > c->sh_cap) {
      PE_CUDA(cudaDeviceSynchronize());
      if (c->sh_a32) cudaFree(c->sh_a32);
      c->sh_a32 = nullptr;
      c->sh_cap = 0;
      if (cudaMalloc(&c->sh_a32, need * sizeof(float)) != cudaSuccess) { cudaGetLastError(); return PE_ERR_WORKSPACE; }
      c->sh_cap = need;
      if (!c->sh_sum && cudaMalloc(&c->sh_sum, 64) != cudaSuccess) { cudaGetLastError(); return PE_ERR_WORKSPACE; }
      if (!c->sh_ptr && cudaMalloc(&c->sh_ptr, sizeof(float*)) != cudaSuccess) { cudaGetLastError(); return PE_ERR_WORKSPACE; }
      PE_CUDA(cudaMemcpy(c->sh_ptr, &c->sh_a32, sizeof(float*), cudaMemcpyHostToDevice));
    }
    na.sums = c->sh_sum;
    if (sh->slots) {
      // the local ||M_r||^2 goes straight into this rank's slot; the slot
      // pointers (and this rank's two Gram destinations) to the device
      if (sh->world > c->peer_cap) {
        PE_CUDA(cudaDeviceSynchronize());
        if (c->peer_slots) cudaFree(c->peer_slots);
        c->peer_slots = nullptr;
        c->peer_cap = 0;
        if (cudaMalloc(&c->peer_slots, sizeof(uint8_t*) * sh->world) != cudaSuccess) {
          cudaGetLastError();
          return PE_ERR_WORKSPACE;
        }
        c->peer_cap = sh->world;
      }
      if (!c->peer_out && cudaMalloc(&c->peer_out, 2 * sizeof(float*)) != cudaSuccess) {
        cudaGetLastError();
        return PE_ERR_WORKSPACE;
      }
      const int64_t gbytes = (int64_t)rup(need * sizeof(float), 256);
      uint8_t* mine = reinterpret_cast<uint8_t*>(sh->slots[sh->rank]);
      float* outs2[2] = {reinterpret_cast<float*>(mine + 256), reinterpret_cast<float*>(mine + 256 + gbytes)};
      PE_CUDA(cudaMemcpy(c->peer_slots, sh->slots, sizeof(uint8_t*) * sh->world, cudaMemcpyHostToDevice));
      PE_CUDA(cudaMemcpy(c->peer_out, outs2, sizeof(outs2), cudaMemcpyHostToDevice));
      na.sums = reinterpret_cast<double*>(mine);
    }
  }
  { ProfScope ps(c, 0, st);
    launch(pe_norm_kernel, PE_NORM_PERSIST ? std::min(P->n_chunks, c->norm_blocks) : P->n_chunks, kNormThreads, 0,
           st, na); }
  ++launches;
  PeerSlots peers{};
  if (sh && sh->slots) {
    const MatDev& md0 = P->mats[0];
    peers.slots = c->peer_slots;
    peers.world = sh->world;
    peers.gbytes = (int64_t)rup((size_t)md0.m * md0.ldm * sizeof(float), 256);
  }
  if (sh) {
    // ||M||_F^2 over every rank's columns, then inv on the device
    if (sh->slots) {
      if ((s = sh->barrier(sh->user, stream_)) != PE_OK) {
        g_last_error = "pe_polar_split_peers: the barrier failed";
        return s;
      }
      launch(pe_inv_peers_kernel, 1, 32, 0, st, peers, at<float>(P, P->o_inv));
    } else {
      if ((s = sh->fn(c->sh_sum, 1, 1, sh->user, stream_)) != PE_OK) {
        g_last_error = "pe_polar_split: the all-reduce callback failed";
        return s;
      }
      launch(pe_inv_kernel, 1, 32, 0, st, (const double*)c->sh_sum, at<float>(P, P->o_inv));
    }
    ++launches;
  }

  // 2) X_0 = M 2^e (bf16, exact) or M / s (fp32 input), oriented
  auto copy_pass = [&](int k, bool scale, bool fin) {
    if (P->n_it[k] == 0) return;
    CopyArgs ca;
    ca.items = at<CopyItem>(P, P->o_it[k]);
    ca.nitems = P->n_it[k];
    ca.mats = at<CopyMat>(P, fin ? P->o_fmats : P->o_smats);
    ca.srcs = fin ? d_fin_src : d_in;
    ca.dsts = fin ? d_out : at<void*>(P, P->o_x0);
    ca.scale = scale ? at<float>(P, P->o_inv) : nullptr;
    ca.pow2 = (!fin && dtype == PE_BF16 && !(io & 1)) ? 1 : 0;    // kFlagScaled copies: X_0 = M * 2^e
    ca.muon = (muon && fin) ? 1 : 0;
    ca.lr = (float)lr;
    const int grid = std::min(P->n_it[k], c->num_sms * 8);
    ProfScope ps(c, fin ? 5 : 1, st);
    const bool tr = (k == 1 || k == 2);
    using bf = __nv_bfloat16;
    if (dtype == PE_BF16 && ((!fin && (io & 1)) || (fin && (io & 2)))) {
      // pe_polar_ex: fp32 caller input -> bf16 X_0, or bf16 result -> fp32 caller output
      if (!fin) {
        if (tr) launch(pe_transpose_kernel<float, bf>, grid, 256, 0, st, ca);
        else launch(pe_rows_kernel<float, bf>, grid, 256, 0, st, ca);
      } else {
        if (tr) launch(pe_transpose_kernel<bf, float>, grid, 256, 0, st, ca);
        else launch(pe_rows_kernel<bf, float>, grid, 256, 0, st, ca);
      }
    } else if (dtype == PE_BF16) {
      if (tr) launch(pe_transpose_kernel<bf>, grid, 256, 0, st, ca);
      else launch(pe_rows_kernel<bf>, grid, 256, 0, st, ca);
    } else if (scale) {
      if (tr) launch(pe_planes_kernel<true, true>, grid, 256, 0, st, ca);
      else launch(pe_planes_kernel<true, false>, grid, 256, 0, st, ca);
    } else {
      if (tr) launch(pe_planes_kernel<false, true>, grid, 256, 0, st, ca);
      else launch(pe_planes_kernel<false, false>, grid, 256, 0, st, ca);
    }
    ++launches;
  };
  copy_pass(0, true, false);
  copy_pass(1, true, false);

  // 3) T iterations
  auto base_args = [&](GemmArgs& g) {
    g.mats = at<MatDev>(P, P->o_mats);
    g.tmaps = at<CUtensorMap>(P, P->o_tmaps);
    g.emaps = at<CUtensorMap>(P, P->o_emaps);
    g.imaps = d_imaps;
    g.omaps = d_omaps;
    g.mflags = at<int>(P, P->o_flags);
    g.inv = at<float>(P, P->o_inv);
    g.scratch = c->scratch;
    g.muon = muon ? 1 : 0;
    g.out32 = nullptr;
    g.lr = (float)lr;
    g.nphase = 0;
    g.coef = d_coef;
    g.done = c->done;
    g.need = at<int>(P, P->o_need);
    g.dbg = c->dbg;
    g.stats = nullptr;
    g.mcoef = nullptr;
    g.lin = 0;
    g.tstride = P->tstride;
    g.estride = P->estride;
    g.shift = 0.f;
    g.psrc = 0;
    g.gen = 0;
    g.g_l = g.g_lmn = g.g_lsym = g.g_rx = g.g_r = g.g_wide = 0;
    g.g_ein = g.g_eout = -1;
  };
  if (fused) {
    // one persistent launch: all 3T phases of all matrices, dataflow-ordered
    GemmArgs g;
    base_args(g);
    g.tiles = P->fused;
    g.ntiles = P->n_fused;
    g.nphase = 3 * T;
    g.mode = 0; g.xin = 0; g.first_iter = 0; g.final_iter = 0;
    g.a = g.b = g.c = 0.f;
    const int grid = 2 * std::min(g.ntiles, c->num_sms / 2);
    ProfScope ps(c, 6, st);
    launch(pe_gemm_sm100<kLongStages, kOpSlots, true>, grid, kGemmThreads, gemm_smem_bytes<kLongStages, kOpSlots>(), st, g);
    ++launches;
  }
  if (rect) {
    // Alg. 4 in applications of rk iterations (restarts,
    // P:1337-1341).  Workspace per matrix (wide orientation, m <= n):
    // A = Y, B = H, E[0] / E[1] = Q (ping-pong), E[2] = T = Y Q, E[3] = R.
    // Main-loop maps: 2 / 4 A, 3 / 5 B, 6 / 7 Q, 8 T, 9 / 10 R; epilogue
    // maps: 2 A, 3 B, 4 / 5 Q, 6 T, 7 R (gemm_sm100.cuh GemmArgs).
    auto coef_t = [&](int t, float* f) {
      const double* tup = &c->table[(size_t)std::min(t, c->ntab - 1) * nq];
      f[0] = (float)tup[0]; f[1] = (float)tup[1]; f[2] = (float)tup[2];
    };
    auto run = [&](GemmArgs& g, const Tile* tiles, int ntiles, bool edge, int kind) {
      g.tiles = tiles;
      g.ntiles = ntiles;
      const int grid = 2 * std::min(ntiles, c->num_sms / 2);
      ProfScope ps(c, kind, st);
      if (g.mode == kModeGram) {
        const size_t sm = gemm_smem_bytes<kGramStages, 1>();
        if (edge) launch(pe_gemm_sm100<kGramStages, 1, true>, grid, kGemmThreads, sm, st, g);
        else launch(pe_gemm_sm100<kGramStages, 1, false>, grid, kGemmThreads, sm, st, g);
      } else {
        const size_t sm = gemm_smem_bytes<kLongStages, kOpSlots>();
        if (edge) launch(pe_gemm_sm100<kLongStages, kOpSlots, true>, grid, kGemmThreads, sm, st, g);
        else launch(pe_gemm_sm100<kLongStages, kOpSlots, false>, grid, kGemmThreads, sm, st, g);
      }
      ++launches;
    };
    const Tile* sym_f = at<Tile>(P, P->o_sym);
    const Tile* sym_r = at<Tile>(P, P->o_sym_r);
    const Tile* sq_f = at<Tile>(P, P->o_sq);
    const Tile* sq_r = at<Tile>(P, P->o_sq_r);
    int ph = 0;                                    // phase counter: alternate the tile-list direction
    for (int b = 0, t0 = 0; b < nblocks; ++b, t0 += rk) {
      const int kb = std::min(rk, T - t0);
      const bool firstb = (b == 0), lastb = (b == nblocks - 1);
      const int xin = b & 1;
      float f[3];
      coef_t(t0, f);
      {  // Y = X X^T (+ shift I in the first application)
        GemmArgs g;
        base_args(g);
        g.mode = kModeGram; g.xin = xin; g.first_iter = firstb; g.final_iter = 0;
        g.a = f[0]; g.b = f[1]; g.c = f[2];
        g.shift = firstb ? (float)c->rect_shift : 0.f;
        run(g, (ph++ & 1) ? sym_r : sym_f, P->n_sym, firstb, 2);
      }
      {  // H_1 = b_1 Y + c_1 Y^2 (R_1 = Y since Q_0 = I)
        GemmArgs g;
        base_args(g);
        g.mode = kModePoly; g.xin = xin; g.first_iter = 0; g.final_iter = 0;
        g.a = f[0]; g.b = f[1]; g.c = f[2];
        run(g, (ph++ & 1) ? sym_r : sym_f, P->n_sym, false, 3);
      }
      if (kb == 1) {
        // a one-iteration application is Listing 2's step: X' = a X + H X
        GemmArgs g;
        base_args(g);
        g.mode = kModeUpdate; g.xin = xin; g.first_iter = firstb; g.final_iter = lastb;
        g.a = f[0]; g.b = f[1]; g.c = f[2];
        run(g, at<Tile>(P, (ph++ & 1) ? P->o_upd_r : P->o_upd), P->n_upd, firstb || lastb, 4);
        continue;
      }
      {  // Q_1 = a_1 I + H_1, full storage
        ExpandArgs ea;
        ea.items = at<CopyItem>(P, P->o_exp);
        ea.nitems = P->n_exp;
        ea.mats = at<MatDev>(P, P->o_mats);
        ea.a = f[0];
        ProfScope ps(c, 1, st);
        launch(pe_expand_kernel, std::min(P->n_exp, c->num_sms * 8), 256, 0, st, ea);
        ++launches;
      }
      int q = 0;                                   // Q_{t-1} lives in E[q]
      for (int j = 1; j < kb; ++j) {
        coef_t(t0 + j, f);
        GemmArgs g;
        // T = Y Q (first half of R_t = Q^T Y Q)
        base_args(g);
        g.mode = kModeUpdate; g.xin = xin; g.first_iter = 0; g.final_iter = 0; g.a = 0.f;
        g.gen = 1; g.g_l = 2; g.g_lmn = 4; g.g_lsym = 1; g.g_rx = 0; g.g_r = 6 + q; g.g_ein = -1; g.g_eout = 6;
        g.g_wide = 0;
        run(g, (ph++ & 1) ? sq_r : sq_f, P->n_sq, false, 4);
        // R = Q T (symmetric: upper block triangle only)
        base_args(g);
        g.mode = kModeUpdate; g.xin = xin; g.first_iter = 0; g.final_iter = 0; g.a = 0.f;
        g.gen = 1; g.g_l = 6 + q; g.g_lsym = 0; g.g_rx = 0; g.g_r = 8; g.g_ein = -1; g.g_eout = 7; g.g_wide = 0;
        run(g, (ph++ & 1) ? sym_r : sym_f, P->n_sym, false, 4);
        // H = b R + c R^2 (Horner's inner part)
        base_args(g);
        g.mode = kModePoly; g.xin = xin; g.first_iter = 0; g.final_iter = 0;
        g.a = f[0]; g.b = f[1]; g.c = f[2]; g.psrc = 1;
        run(g, (ph++ & 1) ? sym_r : sym_f, P->n_sym, false, 3);
        // Q_t = Q_{t-1} h_t(R_t) = a Q + H Q (H and Q commute in exact arithmetic)
        base_args(g);
        g.mode = kModeUpdate; g.xin = xin; g.first_iter = 0; g.final_iter = 0; g.a = f[0];
        g.gen = 1; g.g_l = 3; g.g_lmn = 5; g.g_lsym = 1; g.g_rx = 0; g.g_r = 6 + q; g.g_ein = 4 + q;
        g.g_eout = 4 + (q ^ 1); g.g_wide = 0;
        run(g, (ph++ & 1) ? sq_r : sq_f, P->n_sq, false, 4);
        q ^= 1;
      }
      {  // X' = Q X (P:1312 in the wide orientation: the result is Q_T^T X^T's transpose)
        GemmArgs g;
        base_args(g);
        g.mode = kModeUpdate; g.xin = xin; g.first_iter = firstb; g.final_iter = lastb; g.a = 0.f;
        g.gen = 1; g.g_l = 6 + q; g.g_lsym = 0; g.g_rx = 1; g.g_ein = -1; g.g_eout = -1; g.g_wide = 1;
        run(g, at<Tile>(P, (ph++ & 1) ? P->o_upd_r : P->o_upd), P->n_upd, firstb || lastb, 4);
      }
    }
  }
  for (int sidx = 0; sidx < S && !fused && !rect; ++sidx) {
    // step sidx: the App. G first step (init, sidx == 0) or iteration t
    const bool istep = init && sidx == 0;
    const int t = sidx - (init ? 1 : 0);
    const double* tup = &c->table[(size_t)std::min(std::max(t, 0), c->ntab - 1) * nq];
    const float fa = (float)tup[0], fb = (float)tup[1], fc = (nq == 3) ? (float)tup[2] : 0.0f;
    const int xin = sidx & 1;
    const int fin = (sidx == S - 1);
    // odd cubic step (degree-3 table, or App. G's p(x) = a x + b x^3): no
    // poly launch; the update reads A and computes a X + b (A X)
    const bool cubic = istep || nq == 2;
    for (int mode = kModeGram; mode <= kModeUpdate; ++mode) {
      if (cubic && mode == kModePoly) continue;
      GemmArgs g;
      base_args(g);
      g.lin = cubic ? 1 : 0;
      static const bool alt = !(getenv("PE_ORDER") && !strcmp(getenv("PE_ORDER"), "fwd"));   // A/B knob
      const bool rev = alt && ((3 * sidx + mode) & 1);
      g.tiles = at<Tile>(P, mode == kModeUpdate ? (rev ? P->o_upd_r : P->o_upd) : (rev ? P->o_sym_r : P->o_sym));
      g.ntiles = mode == kModeUpdate ? P->n_upd : P->n_sym;
      g.first_iter = (sidx == 0);
      g.mode = mode; g.xin = xin; g.final_iter = fin;
      g.a = fa; g.b = fb; g.c = fc;
      if (istep && mode != kModeGram) g.mcoef = at<float>(P, P->o_smcoef);
      if (c->dbg & (4 | 128)) {
        if (!c->stats && cudaMalloc(&c->stats, 8 * 1024 * sizeof(long long)) != cudaSuccess) {
          cudaGetLastError();          // debug counters only: run without them
          c->stats = nullptr;
        }
        if (c->stats) g.stats = c->stats + (size_t)mode * 2048;
      }
      const int grid = 2 * std::min(g.ntiles, c->num_sms / 2);   // CTA pairs
      if (sh && mode == kModeGram)                               // partial Gram in fp32: own buffer, or
        g.out32 = sh->slots ? c->peer_out + (t & 1) : c->sh_ptr;  // this rank's peer-visible slot
      if (istep && mode == kModeGram) {
        // App. G: the same Gram launch also stores its raw fp32 accumulator,
        // for the power method (the Rayleigh quotient of bf16(A_0) can exceed
        // sigma_1^2 by ~2^-9 relative, which breaks z <= sigma_1
        // and with it the tail bound sqrt(1 - z^2): R17)
        g.out32 = at<float*>(P, P->o_a32);
        g.out32_both = 1;
      }
      {
      ProfScope ps(c, 2 + mode, st);
      const bool edge = (sidx == 0) || (sidx == S - 1);
      if (dtype == PE_FP32) {
        launch(pe_gemm_sm100<kP3Stages, 3, false, 3>, grid, kGemmThreads, gemm_smem_bytes<kP3Stages, 3>(), st, g);
      } else if (mode == kModeGram) {
        const size_t sm = gemm_smem_bytes<kGramStages, 1>();
        if (edge) launch(pe_gemm_sm100<kGramStages, 1, true>, grid, kGemmThreads, sm, st, g);
        else launch(pe_gemm_sm100<kGramStages, 1, false>, grid, kGemmThreads, sm, st, g);
      } else {
        const size_t sm = gemm_smem_bytes<kLongStages, kOpSlots>();
        if (edge) launch(pe_gemm_sm100<kLongStages, kOpSlots, true>, grid, kGemmThreads, sm, st, g);
        else launch(pe_gemm_sm100<kLongStages, kOpSlots, false>, grid, kGemmThreads, sm, st, g);
      }
      ++launches;
      }
      if (istep && mode == kModeGram) {
        // App. G: power method on A_0, then the per-matrix (a/F, b/F^3)
        SymvArgs sa;
        sa.mats = at<MatDev>(P, P->o_mats);
        sa.item_mat = at<int>(P, P->o_sitem_mat);
        sa.item_r0 = at<int>(P, P->o_sitem_r0);
        sa.nitems = P->n_sitems;
        sa.item0 = at<int>(P, P->o_sitem0);
        sa.nitem = at<int>(P, P->o_snitem);
        sa.voff = at<int64_t>(P, P->o_svoff);
        sa.part = at<double>(P, P->o_spart);
        sa.counters = at<unsigned>(P, P->o_scnt);
        sa.lam = at<double>(P, P->o_slam);
        sa.a32 = at<float*>(P, P->o_a32);
        float* vb = at<float>(P, P->o_sv);
        double* nb = at<double>(P, P->o_snrm);
        const int sgrid = std::min(P->n_sitems, c->num_sms * 8);
        for (int k = 0; k < c->init_iters; ++k) {
          sa.vin = (k == 0) ? at<float>(P, P->o_sv0) : vb + (size_t)((k - 1) & 1) * P->sv_len;
          sa.nrm2_in = (k == 0) ? nullptr : nb + (size_t)((k - 1) & 1) * count;
          sa.wout = vb + (size_t)(k & 1) * P->sv_len;
          sa.nrm2_out = nb + (size_t)(k & 1) * count;
          launch(pe_symv_kernel<float>, sgrid, kSymvThreads, 0, st, sa);
          ++launches;
        }
        const double* tr = nullptr;
        if (io & 1) {                         // fp32 input: ||X_0||^2 of the rounded X_0
          launch(pe_trace_kernel, count, 256, 0, st, (float* const*)sa.a32, (const MatDev*)sa.mats,
                 at<double>(P, P->o_str), count);
          ++launches;
          tr = at<double>(P, P->o_str);
        }
        launch(pe_init_coef_kernel, cdiv(count, 128), 128, 0, st, (const double*)sa.lam,
               (const double*)at<double>(P, P->o_sssq), (const float*)at<float>(P, P->o_inv),
               at<float>(P, P->o_smcoef), count, c->init_margin, (const int*)at<int>(P, P->o_flags), tr);
        ++launches;
      }
      if (sh && mode == kModeGram) {
        // A = sum over ranks of the partial Grams (P:498 on the whole
        // matrix), then rounded once to bf16 (R8; iteration 1 also scales)
        const MatDev& md = P->mats[0];
        const int64_t na32 = (int64_t)md.m * md.ldm;
        const int grid = (int)std::min<int64_t>(cdiv(na32, 256), c->num_sms * 4);
        if (sh->slots) {
          // every rank's partial is in its slot once all ranks pass the
          // barrier; the sum over the slots (rank order) and the rounding
          // are one kernel reading peer memory -- no collective call
          if ((s = sh->barrier(sh->user, stream_)) != PE_OK) {
            g_last_error = "pe_polar_split_peers: the barrier failed";
            return s;
          }
          launch(pe_round_peers_kernel, grid, 256, 0, st, peers, t & 1, reinterpret_cast<__nv_bfloat16*>(md.A),
                 na32, (const float*)at<float>(P, P->o_inv), t == 0 ? 1 : 0);
        } else {
          if ((s = sh->fn(c->sh_a32, na32, 0, sh->user, stream_)) != PE_OK) {
            g_last_error = "pe_polar_split: the all-reduce callback failed";
            return s;
          }
          launch(pe_round_gram_kernel, grid, 256, 0, st, (const float*)c->sh_a32,
                 reinterpret_cast<__nv_bfloat16*>(md.A), na32, (const float*)at<float>(P, P->o_inv), t == 0 ? 1 : 0);
        }
        ++launches;
      }
    }
  }

  // 4) transpose back (tall inputs) / copy out (rows not 16-byte multiples)
  copy_pass(2, false, true);
  copy_pass(3, false, true);
  PE_CUDA(cudaGetLastError());
  c->last_launches = launches + c->uploads;
  return PE_OK;
}

extern "C" pe_status pe_count_nonfinite(pe_ctx c, const void* const* bufs, const int64_t* shapes, int count,
                                        pe_dtype dtype, int64_t* nonfinite, void* stream) {
  if (!c || !nonfinite || (dtype != PE_BF16 && dtype != PE_FP32)) return PE_ERR_INVALID_ARG;
  pe_status s = validate_shapes(shapes, count);
  if (s != PE_OK) return s;
  for (int i = 0; i < count; ++i)
    if (!bufs || !bufs[i]) return PE_ERR_INVALID_ARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  PE_CUDA(cudaSetDevice(c->device));
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  PE_CUDA(cudaStreamIsCapturing(st, &cap));
  if (cap != cudaStreamCaptureStatusNone) {
    g_last_error = "pe_count_nonfinite synchronises: not under graph capture";
    return PE_ERR_UNSUPPORTED;
  }
  if (!c->nf && cudaMalloc(&c->nf, sizeof(unsigned long long)) != cudaSuccess) {
    cudaGetLastError();
    return PE_ERR_WORKSPACE;
  }
  PE_CUDA(cudaMemsetAsync(c->nf, 0, sizeof(unsigned long long), st));
  for (int i = 0; i < count; ++i) {
    const int64_t n = shapes[2 * i] * shapes[2 * i + 1];
    const int grid = (int)std::min<int64_t>(cdiv(n, 256 * 8), c->num_sms * 8);
    if (dtype == PE_BF16)
      launch(pe_nonfinite_kernel<__nv_bfloat16>, grid, 256, 0, st, (const __nv_bfloat16*)bufs[i], n, c->nf);
    else
      launch(pe_nonfinite_kernel<float>, grid, 256, 0, st, (const float*)bufs[i], n, c->nf);
  }
  unsigned long long h = 0;
  PE_CUDA(cudaMemcpyAsync(&h, c->nf, sizeof(h), cudaMemcpyDeviceToHost, st));
  PE_CUDA(cudaStreamSynchronize(st));
  *nonfinite = (int64_t)h;
  return PE_OK;
}

extern "C" pe_status pe_set_small_planes(pe_ctx c, int planes) {
  if (!c || (planes != 1 && planes != 2)) return PE_ERR_INVALID_ARG;
  c->small_planes = planes;
  return PE_OK;
}

extern "C" pe_status pe_set_debug(pe_ctx c, int flags) {
  if (!c || (flags & ~PE_DEBUG_CHECK_FINITE)) return PE_ERR_INVALID_ARG;
  c->debug = flags;
  return PE_OK;
}

// PE_DEBUG_CHECK_FINITE around a pe_polar / pe_polar_ex call: non-finite
// inputs are refused before anything is launched, non-finite outputs of
// finite inputs are reported after the call (both synchronise the stream).
template <typename F>
static pe_status checked_call(pe_ctx c, const void* const* in, void* const* out, const int64_t* shapes, int count,
                              pe_dtype in_t, pe_dtype out_t, void* stream, F&& call) {
  if (!c || !(c->debug & PE_DEBUG_CHECK_FINITE) || count <= 0 || !in || !out) return call();
  int64_t k = 0;
  pe_status s = pe_count_nonfinite(c, in, shapes, count, in_t, &k, stream);
  if (s != PE_OK) return s;
  if (k > 0) {
    g_last_error = "PE_DEBUG_CHECK_FINITE: " + std::to_string(k) + " non-finite input values";
    return PE_ERR_NONFINITE;
  }
  if ((s = call()) != PE_OK) return s;
  if ((s = pe_count_nonfinite(c, const_cast<const void* const*>(out), shapes, count, out_t, &k, stream)) != PE_OK)
    return s;
  if (k > 0) {
    g_last_error = "PE_DEBUG_CHECK_FINITE: " + std::to_string(k) + " non-finite outputs from finite inputs";
    return PE_ERR_NONFINITE;
  }
  return PE_OK;
}

extern "C" pe_status pe_polar(pe_ctx c, const void* const* in, void* const* out, const int64_t* shapes,
                              int count, int iters, pe_dtype dtype, void* stream) {
  return checked_call(c, in, out, shapes, count, dtype, dtype, stream, [&] {
    return polar_impl(c, in, out, nullptr, shapes, count, iters, dtype, stream, 0.0, 0.0);
  });
}

extern "C" pe_status pe_polar_ex(pe_ctx c, const void* const* in, void* const* out, const int64_t* shapes,
                                 int count, int iters, pe_dtype in_dtype, pe_dtype out_dtype, pe_dtype compute,
                                 void* stream) {
  auto ok = [](pe_dtype d) { return d == PE_BF16 || d == PE_FP32; };
  if (!ok(in_dtype) || !ok(out_dtype) || !ok(compute)) return PE_ERR_INVALID_ARG;
  if (compute == PE_FP32) {
    if (in_dtype != PE_FP32 || out_dtype != PE_FP32) {
      g_last_error = "pe_polar_ex: fp32 compute takes fp32 input and output";
      return PE_ERR_UNSUPPORTED;
    }
    return checked_call(c, in, out, shapes, count, PE_FP32, PE_FP32, stream, [&] {
      return polar_impl(c, in, out, nullptr, shapes, count, iters, PE_FP32, stream, 0.0, 0.0);
    });
  }
  const int io = (in_dtype == PE_FP32 ? 1 : 0) | (out_dtype == PE_FP32 ? 2 : 0);
  return checked_call(c, in, out, shapes, count, in_dtype, out_dtype, stream, [&] {
    return polar_impl(c, in, out, nullptr, shapes, count, iters, PE_BF16, stream, 0.0, 0.0, nullptr, nullptr, io);
  });
}

extern "C" pe_status pe_polar_split(pe_ctx c, const void* in, void* out, int64_t rows, int64_t cols, int iters,
                                      pe_allreduce_fn allreduce, void* user, void* stream) {
  if (!c || !in || !out || iters < 1) return PE_ERR_INVALID_ARG;
  if (!allreduce) {                      // the context's own communicator (pe_attach_comm)
    if (!pe_ctx_dist(c)) {
      g_last_error = "pe_polar_split: no allreduce callback and no communicator (pe_attach_comm)";
      return PE_ERR_INVALID_ARG;
    }
    allreduce = pe_comm_allreduce;
    user = c;
  }
  const int64_t shp[2] = {rows, cols};
  const void* ins[1] = {in};
  void* outs[1] = {out};
  SplitCtx sh{allreduce, user};
  return polar_impl(c, ins, outs, nullptr, shp, 1, iters, PE_BF16, stream, 0.0, 0.0, nullptr, &sh);
}

extern "C" pe_status pe_split_slot_bytes(int64_t rows, int64_t cols, int64_t* bytes) {
  if (rows < 1 || cols < 1 || !bytes) return PE_ERR_INVALID_ARG;
  const size_t g = rup((size_t)rows * rup((size_t)rows, 8) * sizeof(float), 256);
  *bytes = (int64_t)(256 + 2 * g);
  return PE_OK;
}

extern "C" pe_status pe_polar_split_peers(pe_ctx c, const void* in, void* out, int64_t rows, int64_t cols, int iters,
                                          void* const* slots, int rank, int world, pe_barrier_fn barrier, void* user,
                                          void* stream) {
  if (!c || !in || !out || iters < 1 || !slots || !barrier || world < 1 || rank < 0 || rank >= world)
    return PE_ERR_INVALID_ARG;
  for (int r = 0; r < world; ++r)
    if (!slots[r] || (reinterpret_cast<uintptr_t>(slots[r]) & 255)) {
      g_last_error = "pe_polar_split_peers: every slot must be a 256-byte aligned device pointer";
      return PE_ERR_INVALID_ARG;
    }
  const int64_t shp[2] = {rows, cols};
  const void* ins[1] = {in};
  void* outs[1] = {out};
  SplitCtx sh{nullptr, user};
  sh.slots = slots;
  sh.rank = rank;
  sh.world = world;
  sh.barrier = barrier;
  return polar_impl(c, ins, outs, nullptr, shp, 1, iters, PE_BF16, stream, 0.0, 0.0, nullptr, &sh);
}

extern "C" pe_status pe_muon_step(pe_ctx c, void* const* W, void* const* M, const void* const* G,
                                  const int64_t* shapes, int count, double beta, double lr, int iters,
                                  void* stream) {
  if (!c || count < 0 || (count > 0 && (!W || !M || !G))) return PE_ERR_INVALID_ARG;
  if (!std::isfinite(beta) || !std::isfinite(lr)) return PE_ERR_INVALID_ARG;
  for (int i = 0; i < count; ++i)
    for (int j = 0; j < count; ++j)
      if (W[i] == M[j] || W[i] == G[j] || M[i] == G[j]) {
        g_last_error = "pe_muon_step: W, M and G buffers must be distinct";
        return PE_ERR_INVALID_ARG;
      }
  return polar_impl(c, M, W, count > 0 ? G : nullptr, shapes, count, iters, PE_BF16, stream, beta, lr);
}

// End-to-end entry on host buffers.  The batch is cut into G groups of about
// equal bytes and software-pipelined over three streams: H2D copies of group
// g+1 and D2H copies of group g-1 overlap the compute of group g (PCIe is full
// duplex, so both directions also overlap each other).
extern "C" pe_status pe_polar_host(pe_ctx c, const void* const* in, void* const* out, const int64_t* shapes,
                                   int count, int iters, pe_dtype dtype, void* stream_) {
  if (!c || iters < 1 || (dtype != PE_BF16 && dtype != PE_FP32)) return PE_ERR_INVALID_ARG;
  if (count == 0) { c->last_launches = 0; return PE_OK; }
  if (!in || !out) return PE_ERR_INVALID_ARG;
  pe_status s = validate_shapes(shapes, count);
  if (s != PE_OK) return s;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream_);
  PE_CUDA(cudaSetDevice(c->device));
  const size_t es = (dtype == PE_BF16) ? 2 : 4;
  std::vector<size_t> off(count), nb(count);
  size_t total = 0;
  for (int i = 0; i < count; ++i) {
    if (!in[i] || !out[i]) return PE_ERR_INVALID_ARG;
    nb[i] = (size_t)shapes[2 * i] * shapes[2 * i + 1] * es;
    off[i] = total;
    total += rup(nb[i], 256);
  }
  if (total > c->staging_bytes) {
    if (c->staging) { PE_CUDA(cudaDeviceSynchronize()); cudaFree(c->staging); c->staging = nullptr; }
    if (cudaMalloc(&c->staging, total) != cudaSuccess) { cudaGetLastError(); c->staging_bytes = 0; return PE_ERR_WORKSPACE; }
    c->staging_bytes = total;
  }
  if (!c->s_h2d) {
    PE_CUDA(cudaStreamCreateWithFlags(&c->s_h2d, cudaStreamNonBlocking));
    PE_CUDA(cudaStreamCreateWithFlags(&c->s_d2h, cudaStreamNonBlocking));
  }
  // groups: contiguous index ranges of ~equal bytes: up to 8 of >= 16 MB,
  // more (up to 48, >= 256 MB each) for large sets, where the first group's
  // H2D and the last group's D2H are the exposed fill and drain (GPT-2 S on
  // B200 / PCIe 5: G=1 8.1 ms, G=4 7.2 ms, G=8 6.4 ms; Llama-3-8B set, 14 GB
  // each way: G=8 417 ms, G=16 391, G=32 382, G=48 379, profiles/r2_e2e.txt)
  const size_t g_small = std::min<size_t>(8, total / (16u << 20)), g_large = std::min<size_t>(48, total >> 28);
  int G = (int)std::max<size_t>(1, std::min<size_t>((size_t)count, std::max(g_small, g_large)));
  if (const char* gv = getenv("PE_HOST_GROUPS")) G = std::max(1, std::min(count, atoi(gv)));   // experiments
  const bool skip_compute = getenv("PE_HOST_NOCOMPUTE") != nullptr;                          // experiments
  std::vector<int> gbeg(G + 1, count);
  gbeg[0] = 0;
  {
    size_t acc = 0;
    int g = 1;
    for (int i = 0; i < count && g < G; ++i) {
      acc += nb[i];
      if (acc * G >= total * (size_t)g) gbeg[g++] = i + 1;
    }
  }
  while ((int)c->host_ev.size() < 3 * G + 1) {
    cudaEvent_t e;
    PE_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->host_ev.push_back(e);
  }
  cudaEvent_t ev_start = c->host_ev[3 * G];
  PE_CUDA(cudaEventRecord(ev_start, st));           // after earlier work on the caller's stream
  PE_CUDA(cudaStreamWaitEvent(c->s_h2d, ev_start, 0));
  PE_CUDA(cudaStreamWaitEvent(c->s_d2h, ev_start, 0));
  std::vector<void*> dptr(count);
  uint8_t* base = reinterpret_cast<uint8_t*>(c->staging);
  for (int i = 0; i < count; ++i) dptr[i] = base + off[i];
  int launches = 0;
  cudaEvent_t last_ed = nullptr;
  for (int g = 0; g < G; ++g) {
    const int b = gbeg[g], e = gbeg[g + 1];
    if (b >= e) continue;
    cudaEvent_t eh = c->host_ev[3 * g], ec = c->host_ev[3 * g + 1], ed = c->host_ev[3 * g + 2];
    for (int i = b; i < e; ++i)
      PE_CUDA(cudaMemcpyAsync(dptr[i], in[i], nb[i], cudaMemcpyHostToDevice, c->s_h2d));
    PE_CUDA(cudaEventRecord(eh, c->s_h2d));
    PE_CUDA(cudaStreamWaitEvent(st, eh, 0));
    if (!skip_compute) {
      s = polar_impl(c, dptr.data() + b, dptr.data() + b, nullptr, shapes + 2 * b, e - b, iters, dtype, stream_,
                     0.0, 0.0, c->s_h2d);
      if (s != PE_OK) return s;
      launches += c->last_launches;
    }
    PE_CUDA(cudaEventRecord(ec, st));
    PE_CUDA(cudaStreamWaitEvent(c->s_d2h, ec, 0));
    for (int i = b; i < e; ++i)
      PE_CUDA(cudaMemcpyAsync(out[i], dptr[i], nb[i], cudaMemcpyDeviceToHost, c->s_d2h));
    PE_CUDA(cudaEventRecord(ed, c->s_d2h));
    last_ed = ed;
  }
  if (last_ed) PE_CUDA(cudaStreamWaitEvent(st, last_ed, 0));
  PE_CUDA(cudaStreamSynchronize(st));
  c->last_launches = launches;
  return PE_OK;
}

// ---------------------------------------------------------------- host utils
extern "C" pe_status pe_flops(const int64_t* shapes, int count, int iters, int degree, double* flops) {
  if (!flops || count < 0 || iters < 0 || (count > 0 && !shapes)) return PE_ERR_INVALID_ARG;
  if (degree != 3 && degree != 5) return PE_ERR_UNSUPPORTED;
  double f = 0.0;
  for (int i = 0; i < count; ++i) {
    const double r = (double)shapes[2 * i], cc = (double)shapes[2 * i + 1];
    const double m = std::min(r, cc), n = std::max(r, cc);
    double per = m * (m + 1) * n + 2.0 * m * m * n;
    if (degree == 5) per += m * m * (m + 1);
    f += iters * per;
  }
  *flops = f;
  return PE_OK;
}
