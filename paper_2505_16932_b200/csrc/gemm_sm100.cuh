// Grouped persistent tcgen05 GEMM (CTA-pair, cta_group::2) for the three
// products of one Polar Express iteration (Listing 2), bf16 in /
// fp32 accumulate:
//
//   kModeGram   A  = X X^T           both operands K-major rows of X; only
//                                    256x256 tiles with I <= J are computed;
//                                    off-diagonal tiles are also stored
//                                    transposed at (J, I).
//   kModePoly   B  = b A + c (A A^T) A symmetric so A A = A A^T (SYRK on A);
//                                    the epilogue reads the same bf16 A
//                                    (reading R8); mirrored like the Gram.
//   kModeUpdate X' = a X + B X       A-operand B (K-major), B-operand X
//                                    (MN-major: X row-major is N-contiguous).
//
// A cluster of two CTAs on one TPC computes one 256x256 output tile with
// tcgen05.mma.cta_group::2 (M=256, N=256, K=16): CTA r holds rows
// [128r, 128r+128) of the left operand and rows/columns [128r, 128r+128) of
// the right operand in its shared memory, and accumulator rows
// [128r, 128r+128) x 256 columns in its TMEM.  Per CTA:
//   warp 0      TMA producer (64x64 bf16 boxes, 128B swizzle, 6-stage ring;
//               bytes of both CTAs are counted on the leader's barrier)
//   warp 1      leader: single-thread MMA issuer; both: TMEM alloc (512 cols
//               = two 256-column fp32 accumulators -> epilogue of tile i
//               overlaps the main loop of tile i+1)
//   warps 2..9  epilogue: lane quadrant (warp % 4) x column half
//               ((warp-2) / 4): tcgen05.ld -> fp32 epilogue -> bf16 stores
// Grouped scheduling: one launch covers every tile of every matrix of the
// batch; cluster c walks tiles c, c + #clusters, ... of a host-built list
// (longest K first; update tiles column-major for L2 reuse of B).
#pragma once
#include <cuda_bf16.h>

#include "pe_types.h"
#include "ptx.cuh"

namespace pe {

struct GemmArgs {
  const Tile* tiles;
  int ntiles;
  const MatDev* mats;
  const CUtensorMap* tmaps;    // main loop, 4 per matrix: X[0], X[1], A, B (64x64 boxes, 128B swizzle)
  const CUtensorMap* emaps;    // epilogue, 4 per matrix: X[0], X[1], A, B (16-col x 32-row boxes)
  const CUtensorMap* omaps;    // per call: caller output (16x32 boxes), valid where outs[mat] != nullptr
  void* const* outs;           // per matrix final destination (wide, bf16) or nullptr
  int mode;
  int xin;                     // which X buffer holds the current iterate
  int final_iter;              // update writes outs[mat] when non-null
  float a, b, c;
  int dbg;                     // timing experiments only: 1 = no epilogue work, 2 = no operand loads
  long long* stats;            // optional per-CTA wait-cycle counters (8 per CTA) or nullptr
};

__device__ __forceinline__ void load8_bf16(const __nv_bfloat16* p, float* f) {
  uint4 u = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}

__device__ __forceinline__ uint4 pack8_bf16(const float* f) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return u;
}

// Mirrored store of a symmetric-output chunk: element (r, c0+j) -> (c0+j, r).
// Lanes hold consecutive r, so each store instruction writes 64 contiguous bytes.
__device__ __forceinline__ void mirror_chunk16(__nv_bfloat16* dst, int m, int ld, int r, int c0, const float* w) {
  if (r >= m) return;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int c = c0 + j;
    if (c < m) dst[(size_t)c * ld + r] = __float2bfloat16_rn(w[j]);
  }
}

// kSt: smem pipeline stages; kSl: epilogue smem slots per warp.  kSl == 3:
// operand chunks are prefetched one chunk ahead (long-K phases, deep ring);
// kSl == kEpiChunks: a whole tile's operand chunks are prefetched while the
// MMA of that tile runs (short-K phases, where one chunk of lookahead cannot
// hide the TMA latency).
template <int kSt, int kSl>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kGemmThreads, 1) pe_gemm_sm100(const GemmArgs args) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kSt * kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kSt * kStageBytes);
  uint64_t* empty = full + kSt;
  uint64_t* tfull = empty + kSt;
  uint64_t* tempty = tfull + 2;
  uint64_t* xbars = tempty + 2;                              // kEpiWarps x kSl
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xbars + kEpiWarps * kSl);
  uint8_t* epi_smem = smem + kSt * kStageBytes + kBarrierBytes;   // kEpiWarps x kSl x 1 KB

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int mode = args.mode;
  const uint32_t rank = cluster_rank();
  const bool leader = (rank == 0);
  const int cid = blockIdx.x >> 1;
  const int ncl = gridDim.x >> 1;
  long long st_wait_tempty = 0, st_wait_full = 0, st_wait_tfull = 0;
  const long long st_begin = clock64();

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kSt; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 2 * kEpiWarps);
    }
    for (int s = 0; s < kEpiWarps * kSl; ++s) mbar_init(&xbars[s], 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_pair(tmem_slot, kTmemCols);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    // Loads the (tile, k-block) sequence of this cluster into the smem ring and
    // runs an L2 prefetch of the same boxes kPrefetch k-blocks ahead, so the
    // ring's TMA loads hit L2 (the ring alone covers ~kSt x 512 MMA cycles).
    if (elect_one()) {
      const uint32_t full_leader0 = mapa_shared(smem_u32(&full[0]), 0);
      struct Op { const CUtensorMap* A; const CUtensorMap* B; int nk, row_a, col_b; bool diag; };
      auto op_of = [&](int t) -> Op {
        const Tile tl = args.tiles[t];
        const MatDev& md = args.mats[tl.mat];
        const CUtensorMap* maps = args.tmaps + 4 * tl.mat;
        Op o;
        int K;
        if (mode == kModeGram) { o.A = o.B = maps + args.xin; K = md.n; }
        else if (mode == kModePoly) { o.A = o.B = maps + 2; K = md.m; }
        else { o.A = maps + 3; o.B = maps + args.xin; K = md.m; }
        o.nk = (K + kBK - 1) / kBK;
        // diagonal tile of a symmetric phase: both operands are the same row
        // panel, so it is loaded once and the MMA reads it as A and as B
        o.diag = (mode != kModeUpdate) && (tl.tm == tl.tn);
        o.row_a = tl.tm * kBM + (int)rank * (kBM / 2);
        o.col_b = tl.tn * kBN + (int)rank * (kBN / 2);
        return o;
      };
      // prefetch cursor
      int pt = cid, pkb = 0;
      Op po = (pt < args.ntiles) ? op_of(pt) : Op{nullptr, nullptr, 0, 0, 0, false};
      auto prefetch_one = [&]() {
        if (kPrefetch == 0 || pt >= args.ntiles) return;
        tma_prefetch_2d(po.A, pkb * kBK, po.row_a);
        tma_prefetch_2d(po.A, pkb * kBK, po.row_a + 64);
        if (mode != kModeUpdate) {
          tma_prefetch_2d(po.B, pkb * kBK, po.col_b);
          tma_prefetch_2d(po.B, pkb * kBK, po.col_b + 64);
        } else {
          tma_prefetch_2d(po.B, po.col_b, pkb * kBK);
          tma_prefetch_2d(po.B, po.col_b + 64, pkb * kBK);
        }
        if (++pkb == po.nk) {
          pkb = 0;
          pt += ncl;
          if (pt < args.ntiles) po = op_of(pt);
        }
      };
      for (int i = 0; i < kPrefetch; ++i) prefetch_one();
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cid; t < args.ntiles; t += ncl) {
        const Op o = op_of(t);
        for (int kb = 0; kb < o.nk; ++kb) {
          prefetch_one();
          mbar_wait(&empty[stage], phase ^ 1);
          if (leader) mbar_arrive_expect_tx(&full[stage], o.diag ? 2 * kABytes : 2 * kStageBytes);
          const uint32_t bar = full_leader0 + stage * sizeof(uint64_t);
          uint8_t* a_dst = sA + stage * kABytes;
          uint8_t* b_dst = sB + stage * kBBytes;
          tma_load_2d_pair(a_dst, o.A, bar, kb * kBK, o.row_a);
          tma_load_2d_pair(a_dst + kBoxBytes, o.A, bar, kb * kBK, o.row_a + 64);
          if (o.diag) {
            // B operand = A operand (same smem)
          } else if (mode != kModeUpdate) {
            tma_load_2d_pair(b_dst, o.B, bar, kb * kBK, o.col_b);
            tma_load_2d_pair(b_dst + kBoxBytes, o.B, bar, kb * kBK, o.col_b + 64);
          } else {
            tma_load_2d_pair(b_dst, o.B, bar, o.col_b, kb * kBK);
            tma_load_2d_pair(b_dst + kBoxBytes, o.B, bar, o.col_b + 64, kb * kBK);
          }
          if (++stage == kSt) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader CTA)
    if (leader) {
      const uint32_t idesc = idesc_bf16(kBM, kBN, 0, mode == kModeUpdate ? 1 : 0);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = cid; t < args.ntiles; t += ncl) {
        const Tile tl = args.tiles[t];
        const MatDev& md = args.mats[tl.mat];
        const int K = (mode == kModeGram) ? md.n : md.m;
        const int nk = (K + kBK - 1) / kBK;
        const bool diag = (mode != kModeUpdate) && (tl.tm == tl.tn);
        long long t0 = clock64();
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        st_wait_tempty += clock64() - t0;
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kBN;
        for (int kb = 0; kb < nk; ++kb) {
          long long t1 = clock64();
          mbar_wait(&full[stage], phase);
          st_wait_full += clock64() - t1;
          tc_fence_after();
          if (elect_one()) {
            const uint32_t a_addr = smem_u32(sA + stage * kABytes);
            const uint32_t b_addr = diag ? a_addr : smem_u32(sB + stage * kBBytes);
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) {
              const uint64_t adesc = smem_desc_sw128(a_addr + k * 32, 16, 1024);
              const uint64_t bdesc = (mode != kModeUpdate)
                                         ? smem_desc_sw128(b_addr + k * 32, 16, 1024)
                                         : smem_desc_sw128(b_addr + k * 2048, kBoxBytes, 1024);
              umma_bf16_pair(d_tmem, adesc, bdesc, idesc, (kb | k) != 0);
            }
            umma_commit_pair(&empty[stage], 0x3);
          }
          __syncwarp();
          if (++stage == kSt) { stage = 0; phase ^= 1; }
        }
        if (elect_one()) umma_commit_pair(&tfull[acc], 0x3);
        __syncwarp();
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    // Warp ew owns TMEM lane quadrant q (its 32 output rows) and column half
    // `half` (128 columns) of the CTA's 128 x 256 accumulator, processed as
    // 16-column chunks through a 3-slot smem ring: the operand chunk (X for
    // update, A for poly) arrives by TMA, the bf16 result is written back in
    // place and leaves by TMA store; mirrored (transposed) stores of the
    // symmetric phases go straight to global (64 contiguous bytes per store).
    const int ew = warp - 2;
    const int q = warp & 3;
    const int half = ew >> 2;
    uint8_t* slots = epi_smem + ew * kSl * kEpiSlotBytes;
    uint64_t* xbar = xbars + ew * kSl;
    const bool need_load = (mode != kModeGram) && !(args.dbg & 3);
    const bool do_work = !(args.dbg & 1);
    const int emap_in = (mode == kModeUpdate) ? args.xin : 2;
    const uint32_t tempty_leader0 = mapa_shared(smem_u32(&tempty[0]), 0);
    const int row_off = (int)rank * (kBM / 2) + q * 32;

    // iterator over this warp's valid chunks (for operand prefetch)
    auto valid = [&](int tt, int kk) -> bool {
      const Tile tl2 = args.tiles[tt];
      const MatDev& m2 = args.mats[tl2.mat];
      const int nc = (mode == kModeUpdate) ? m2.n : m2.m;
      return tl2.tn * kBN + half * (kBN / 2) + kk * kEpiCols < nc;
    };
    auto advance = [&](int& tt, int& kk) {
      while (tt < args.ntiles) {
        if (kk < kEpiChunks && valid(tt, kk)) return;
        tt += ncl;
        kk = 0;
      }
    };
    auto issue_load = [&](int tt, int kk, int slot) {
      const Tile tl2 = args.tiles[tt];
      mbar_arrive_expect_tx(&xbar[slot], kEpiSlotBytes);
      tma_load_2d(slots + slot * kEpiSlotBytes, args.emaps + 4 * tl2.mat + emap_in, &xbar[slot],
                  tl2.tn * kBN + half * (kBN / 2) + kk * kEpiCols, tl2.tm * kBM + row_off);
    };
    if constexpr (kSl >= kEpiChunks) {
      // ---- tile-prefetch epilogue: slot k <-> chunk k of the current tile
      uint32_t phase_bits = 0;
      auto issue_tile = [&](int tt) {
        if (!need_load || tt >= args.ntiles) return;
        for (int kk = 0; kk < kEpiChunks; ++kk) {
          if (!valid(tt, kk)) break;
          issue_load(tt, kk, kk);
        }
      };
      if (lane == 0) issue_tile(cid);
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = cid; t < args.ntiles; t += ncl) {
        const Tile tl = args.tiles[t];
        const MatDev md = args.mats[tl.mat];
        long long t2 = clock64();
        mbar_wait(&tfull[acc], acc_phase);
        st_wait_tfull += clock64() - t2;
        tc_fence_after();
        const int r0 = tl.tm * kBM + row_off;
        const int r = r0 + lane;
        const uint32_t t_row = tmem_base + acc * kBN + ((uint32_t)(q * 32) << 16) + half * (kBN / 2);
        const int ncols = (mode == kModeUpdate) ? md.n : md.m;
        const bool mirror = (mode != kModeUpdate) && (tl.tn != tl.tm);
        const CUtensorMap* dmap;
        if (mode == kModeGram) dmap = args.emaps + 4 * tl.mat + 2;
        else if (mode == kModePoly) dmap = args.emaps + 4 * tl.mat + 3;
        else if (args.final_iter && args.outs != nullptr && args.outs[tl.mat] != nullptr) dmap = args.omaps + tl.mat;
        else dmap = args.emaps + 4 * tl.mat + (args.xin ^ 1);
        __nv_bfloat16* mdst = reinterpret_cast<__nv_bfloat16*>(mode == kModeGram ? md.A : md.B);
        float v[32];
#pragma unroll 1
        for (int k2 = 0; k2 < kEpiChunks; k2 += 2) {
          if (tl.tn * kBN + half * (kBN / 2) + k2 * kEpiCols >= ncols) break;   // warp-uniform
          tmem_ld32(t_row + k2 * kEpiCols, v);
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            const int k = k2 + h2;
            const int c0 = tl.tn * kBN + half * (kBN / 2) + k * kEpiCols;
            if (c0 < ncols && do_work) {
              if (need_load) {
                mbar_wait(&xbar[k], (phase_bits >> k) & 1u);
                phase_bits ^= 1u << k;
              }
              float w[16];
#pragma unroll
              for (int j = 0; j < 16; ++j) w[j] = v[h2 * 16 + j];
              uint4* sp = reinterpret_cast<uint4*>(slots + k * kEpiSlotBytes + lane * (kEpiCols * 2));
              if (need_load) {
                float o[16];
                load8_bf16(reinterpret_cast<const __nv_bfloat16*>(sp), o);
                load8_bf16(reinterpret_cast<const __nv_bfloat16*>(sp + 1), o + 8);
                if (mode == kModePoly) {
#pragma unroll
                  for (int j = 0; j < 16; ++j) w[j] = __fadd_rn(__fmul_rn(args.b, o[j]), __fmul_rn(args.c, w[j]));
                } else {
#pragma unroll
                  for (int j = 0; j < 16; ++j) w[j] = __fadd_rn(__fmul_rn(args.a, o[j]), w[j]);
                }
              }
              sp[0] = pack8_bf16(w);
              sp[1] = pack8_bf16(w + 8);
              if (mirror) mirror_chunk16(mdst, md.m, md.ldm, r, c0, w);
              fence_async_smem();
              __syncwarp();
              if (lane == 0) {
                tma_store_2d(dmap, slots + k * kEpiSlotBytes, c0, r0);
                bulk_commit();
              }
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive_remote(tempty_leader0 + acc * sizeof(uint64_t));
          bulk_wait_read<0>();          // this tile's stores have left smem: slots are free
          issue_tile(t + ncl);
        }
        __syncwarp();
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    } else {
    int pt = cid, pk = 0;          // next chunk to prefetch
    advance(pt, pk);
    if (need_load && lane == 0 && pt < args.ntiles) issue_load(pt, pk, 0);
    ++pk;
    advance(pt, pk);

    int g = 0;                     // chunks processed by this warp
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = cid; t < args.ntiles; t += ncl) {
      const Tile tl = args.tiles[t];
      const MatDev md = args.mats[tl.mat];
      long long t2 = clock64();
      mbar_wait(&tfull[acc], acc_phase);
      st_wait_tfull += clock64() - t2;
      tc_fence_after();
      const int r0 = tl.tm * kBM + row_off;
      const int r = r0 + lane;
      const uint32_t t_row = tmem_base + acc * kBN + ((uint32_t)(q * 32) << 16) + half * (kBN / 2);
      const int ncols = (mode == kModeUpdate) ? md.n : md.m;
      const bool mirror = (mode != kModeUpdate) && (tl.tn != tl.tm);
      const CUtensorMap* dmap;
      if (mode == kModeGram) dmap = args.emaps + 4 * tl.mat + 2;
      else if (mode == kModePoly) dmap = args.emaps + 4 * tl.mat + 3;
      else if (args.final_iter && args.outs != nullptr && args.outs[tl.mat] != nullptr) dmap = args.omaps + tl.mat;
      else dmap = args.emaps + 4 * tl.mat + (args.xin ^ 1);
      __nv_bfloat16* mdst = reinterpret_cast<__nv_bfloat16*>(mode == kModeGram ? md.A : md.B);
      float v[32];
#pragma unroll 1
      for (int k2 = 0; k2 < kEpiChunks; k2 += 2) {
        if (tl.tn * kBN + half * (kBN / 2) + k2 * kEpiCols >= ncols) break;   // warp-uniform
        tmem_ld32(t_row + k2 * kEpiCols, v);
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int k = k2 + h2;
          const int c0 = tl.tn * kBN + half * (kBN / 2) + k * kEpiCols;
          if (c0 < ncols && do_work) {
            const int slot = g % kSl;
            if (need_load) {
              if (lane == 0) {
                bulk_wait_read<1>();                  // slot of chunk g+1 (last used by g-2) is free
                if (pt < args.ntiles) issue_load(pt, pk, (g + 1) % kSl);
              }
              ++pk;
              advance(pt, pk);
              mbar_wait(&xbar[slot], (uint32_t)((g / kSl) & 1));
            } else {
              if (lane == 0) bulk_wait_read<kSl - 1>();   // slot g%3 (last used by g-3) is free
              __syncwarp();
            }
            float w[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) w[j] = v[h2 * 16 + j];
            uint4* sp = reinterpret_cast<uint4*>(slots + slot * kEpiSlotBytes + lane * (kEpiCols * 2));
            if (need_load) {
              float o[16];
              load8_bf16(reinterpret_cast<const __nv_bfloat16*>(sp), o);
              load8_bf16(reinterpret_cast<const __nv_bfloat16*>(sp + 1), o + 8);
              if (mode == kModePoly) {
#pragma unroll
                for (int j = 0; j < 16; ++j) w[j] = __fadd_rn(__fmul_rn(args.b, o[j]), __fmul_rn(args.c, w[j]));
              } else {
#pragma unroll
                for (int j = 0; j < 16; ++j) w[j] = __fadd_rn(__fmul_rn(args.a, o[j]), w[j]);
              }
            }
            sp[0] = pack8_bf16(w);
            sp[1] = pack8_bf16(w + 8);
            if (mirror) mirror_chunk16(mdst, md.m, md.ldm, r, c0, w);
            fence_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(dmap, slots + slot * kEpiSlotBytes, c0, r0);
              bulk_commit();
            }
            ++g;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(tempty_leader0 + acc * sizeof(uint64_t));
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
    }
    if (lane == 0) bulk_wait<0>();
  }

  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == 1) tmem_dealloc_pair(tmem_base, kTmemCols);
  if (args.stats != nullptr && lane == 0 && (warp == 1 || warp == 2)) {
    long long* st = args.stats + blockIdx.x * 8;
    if (warp == 1) { st[0] = clock64() - st_begin; st[1] = st_wait_tempty; st[2] = st_wait_full; }
    else { st[3] = st_wait_tfull; }
  }
}

template <int kSt, int kSl> constexpr size_t gemm_smem_bytes() {
  return 1024 + (size_t)kSt * kStageBytes + kBarrierBytes + (size_t)kEpiWarps * kSl * kEpiSlotBytes;
}

}  // namespace pe
