// Grouped persistent tcgen05 GEMM for the three products of one Polar
// Express iteration (Listing 2), bf16 in / fp32 accumulate:
//
//   kModeGram   A  = X X^T           both operands K-major rows of X; only
//                                    tiles touching the upper triangle are
//                                    computed, each element c >= r is stored
//                                    at (r,c) and mirrored to (c,r).
//   kModePoly   B  = b A + c (A A^T) A symmetric so A A = A A^T (SYRK on A);
//                                    the epilogue reads the same bf16 A
//                                    (reading R8); mirrored like the Gram.
//   kModeUpdate X' = a X + B X       A-operand B (K-major), B-operand X
//                                    (MN-major: X row-major is N-contiguous).
//
// One launch covers every tile of every matrix of the batch (the "grouped
// persistent scheduler"): CTA b walks tiles b, b+grid, ... of a host-built
// list sorted longest-K first.  Warp roles (192 threads):
//   warp 0      TMA producer: 64x64 bf16 boxes, 128B swizzle, 4-stage ring
//   warp 1      tcgen05.mma issuer (one thread), TMEM owner
//   warps 2..5  epilogue: tcgen05.ld -> fp32 epilogue -> bf16 global stores
// TMEM holds two 128x256 fp32 accumulators so the epilogue of tile i
// overlaps the main loop of tile i+1.
#pragma once
#include <cuda_bf16.h>

#include "pe_types.h"
#include "ptx.cuh"

namespace pe {

struct GemmArgs {
  const Tile* tiles;
  int ntiles;
  const MatDev* mats;
  const CUtensorMap* tmaps;    // 4 per matrix: X[0], X[1], A, B
  void* const* outs;           // per matrix final destination (wide, bf16) or nullptr
  int mode;
  int xin;                     // which X buffer holds the current iterate
  int final_iter;              // update writes outs[mat] when non-null
  float a, b, c;
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

__global__ void __launch_bounds__(kGemmThreads, 1) pe_gemm_sm100(const GemmArgs args) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment for the 128B-swizzle atoms
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages * kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int mode = args.mode;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 128);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < args.ntiles; t += gridDim.x) {
        const Tile tl = args.tiles[t];
        const MatDev& md = args.mats[tl.mat];
        const CUtensorMap* maps = args.tmaps + 4 * tl.mat;
        const CUtensorMap* mapA;
        const CUtensorMap* mapB;
        int K;
        if (mode == kModeGram) {
          mapA = mapB = maps + args.xin;
          K = md.n;
        } else if (mode == kModePoly) {
          mapA = mapB = maps + 2;
          K = md.m;
        } else {
          mapA = maps + 3;
          mapB = maps + args.xin;
          K = md.m;
        }
        const int nk = (K + kBK - 1) / kBK;
        const int row_a = tl.tm * kBM;
        const int col_b = tl.tn * kBN;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], kStageBytes);
          uint8_t* a_dst = sA + stage * kABytes;
          uint8_t* b_dst = sB + stage * kBBytes;
          tma_load_2d(a_dst, mapA, &full[stage], kb * kBK, row_a);
          tma_load_2d(a_dst + kBoxBytes, mapA, &full[stage], kb * kBK, row_a + 64);
          if (mode != kModeUpdate) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
              tma_load_2d(b_dst + q * kBoxBytes, mapB, &full[stage], kb * kBK, col_b + 64 * q);
          } else {
#pragma unroll
            for (int q = 0; q < 4; ++q)
              tma_load_2d(b_dst + q * kBoxBytes, mapB, &full[stage], col_b + 64 * q, kb * kBK);
          }
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t idesc = idesc_bf16(kBM, kBN, 0, mode == kModeUpdate ? 1 : 0);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < args.ntiles; t += gridDim.x) {
      const Tile tl = args.tiles[t];
      const MatDev& md = args.mats[tl.mat];
      const int K = (mode == kModeGram) ? md.n : md.m;
      const int nk = (K + kBK - 1) / kBK;
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * kBN;
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t a_addr = smem_u32(sA + stage * kABytes);
          const uint32_t b_addr = smem_u32(sB + stage * kBBytes);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            const uint64_t adesc = smem_desc_sw128(a_addr + k * 32, 16, 1024);
            const uint64_t bdesc = (mode != kModeUpdate)
                                       ? smem_desc_sw128(b_addr + k * 32, 16, 1024)
                                       : smem_desc_sw128(b_addr + k * 2048, kBoxBytes, 1024);
            umma_bf16(d_tmem, adesc, bdesc, idesc, (kb | k) != 0);
          }
          umma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
      if (elect_one()) umma_commit(&tfull[acc]);
      __syncwarp();
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int ew = warp & 3;            // TMEM lane quadrant accessible by this warp
    const int row_in_tile = ew * 32 + lane;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < args.ntiles; t += gridDim.x) {
      const Tile tl = args.tiles[t];
      const MatDev md = args.mats[tl.mat];
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int r = tl.tm * kBM + row_in_tile;
      const uint32_t t_row = tmem_base + acc * kBN + ((uint32_t)(ew * 32) << 16);
      if (mode != kModeUpdate) {
        // symmetric output (m x m)
        const int m = md.m, ld = md.ldm;
        __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(mode == kModeGram ? md.A : md.B);
        const __nv_bfloat16* Ain = reinterpret_cast<const __nv_bfloat16*>(md.A);
        for (int ch = 0; ch < kBN / 32; ++ch) {
          const int c0 = tl.tn * kBN + ch * 32;
          if (c0 >= m) break;                       // warp-uniform
          float v[32];
          tmem_ld32(t_row + ch * 32, v);
          if (r < m && c0 + 31 >= r) {
            if (mode == kModePoly) {
              float av[32];
              if (c0 + 32 <= m) {
#pragma unroll
                for (int q = 0; q < 4; ++q) load8_bf16(Ain + (size_t)r * ld + c0 + 8 * q, av + 8 * q);
              } else {
                for (int j = 0; j < 32; ++j)
                  av[j] = (c0 + j < m) ? __bfloat162float(Ain[(size_t)r * ld + c0 + j]) : 0.f;
              }
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = __fadd_rn(__fmul_rn(args.b, av[j]), __fmul_rn(args.c, v[j]));
            }
            if (c0 >= r && c0 + 32 <= m) {
#pragma unroll
              for (int q = 0; q < 4; ++q)
                *reinterpret_cast<uint4*>(dst + (size_t)r * ld + c0 + 8 * q) = pack8_bf16(v + 8 * q);
            } else {
              for (int j = 0; j < 32; ++j) {
                const int c = c0 + j;
                if (c >= r && c < m) dst[(size_t)r * ld + c] = __float2bfloat16_rn(v[j]);
              }
            }
          }
          // mirrored store (c, r) for c > r; lanes = consecutive r -> contiguous
          if (r < m) {
#pragma unroll 4
            for (int j = 0; j < 32; ++j) {
              const int c = c0 + j;
              if (c > r && c < m) dst[(size_t)c * ld + r] = __float2bfloat16_rn(v[j]);
            }
          }
        }
      } else {
        const int m = md.m, n = md.n;
        const __nv_bfloat16* X = reinterpret_cast<const __nv_bfloat16*>(md.X[args.xin]);
        __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(md.X[args.xin ^ 1]);
        int ldd = md.ldx;
        if (args.final_iter && args.outs != nullptr && args.outs[tl.mat] != nullptr) {
          dst = reinterpret_cast<__nv_bfloat16*>(args.outs[tl.mat]);
          ldd = md.n;
        }
        for (int ch = 0; ch < kBN / 32; ++ch) {
          const int c0 = tl.tn * kBN + ch * 32;
          if (c0 >= n) break;
          float v[32];
          tmem_ld32(t_row + ch * 32, v);
          if (r < m) {
            float xv[32];
            const bool full_chunk = (c0 + 32 <= n);
            if (full_chunk) {
#pragma unroll
              for (int q = 0; q < 4; ++q) load8_bf16(X + (size_t)r * md.ldx + c0 + 8 * q, xv + 8 * q);
            } else {
              for (int j = 0; j < 32; ++j)
                xv[j] = (c0 + j < n) ? __bfloat162float(X[(size_t)r * md.ldx + c0 + j]) : 0.f;
            }
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __fadd_rn(__fmul_rn(args.a, xv[j]), v[j]);
            if (full_chunk && (ldd % 8) == 0) {
#pragma unroll
              for (int q = 0; q < 4; ++q)
                *reinterpret_cast<uint4*>(dst + (size_t)r * ldd + c0 + 8 * q) = pack8_bf16(v + 8 * q);
            } else {
              for (int j = 0; j < 32; ++j)
                if (c0 + j < n) dst[(size_t)r * ldd + c0 + j] = __float2bfloat16_rn(v[j]);
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem_base, kTmemCols);
}

constexpr size_t gemm_smem_bytes() {
  return 1024 + (size_t)kStages * kStageBytes + (2 * kStages + 4) * sizeof(uint64_t) + 16;
}

}  // namespace pe
