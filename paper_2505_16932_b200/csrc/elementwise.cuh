// HBM-bound passes of the hot path:
//   pe_norm_kernel  -- per-matrix sum of squares (fp64, deterministic
//                      two-level reduction) -> s = ||M||_F * 1.01 + 1e-7
//                      (Listing 2; reading R1/R2), inv = fp32(1/s).
//   pe_copy_kernel  -- X_0 = bf16(fp32(x) * inv) in the wide orientation
//                      (transpose trick P:493), and the final transpose-back
//                      of tall results.  64x64 tiles through smem so
//                      both the read and the write are row-contiguous.
#pragma once
#include <cuda_bf16.h>

#include "pe_types.h"

namespace pe {

constexpr int kNormChunk = 32768;   // elements per norm block
constexpr int kNormThreads = 256;

struct NormArgs {
  const void* const* srcs;     // per matrix, caller layout (rows x cols contiguous)
  const int64_t* elems;        // per matrix element count
  const int* chunk_mat;        // per block: matrix index
  const int* chunk_idx;        // per block: chunk index within the matrix
  const int* nchunks;          // per matrix: number of chunks
  double* partials;            // per block
  unsigned int* counters;      // per matrix, zero at rest (self-resetting)
  float* inv;                  // per matrix: fp32(1 / s)
  int src_f32;                 // 1: fp32 input, 0: bf16
};

__global__ void __launch_bounds__(kNormThreads) pe_norm_kernel(const NormArgs a) {
  const int blk = blockIdx.x;
  const int mat = a.chunk_mat[blk];
  const int ci = a.chunk_idx[blk];
  const int64_t total = a.elems[mat];
  const int64_t begin = (int64_t)ci * kNormChunk;
  const int64_t end = min(begin + (int64_t)kNormChunk, total);
  double acc = 0.0;
  if (a.src_f32) {
    const float* p = reinterpret_cast<const float*>(a.srcs[mat]);
    for (int64_t i = begin + (int64_t)threadIdx.x * 4; i < end; i += (int64_t)kNormThreads * 4) {
      if (i + 4 <= end && ((reinterpret_cast<uintptr_t>(p + i) & 15) == 0)) {
        float4 v = *reinterpret_cast<const float4*>(p + i);
        acc += (double)v.x * v.x + (double)v.y * v.y + (double)v.z * v.z + (double)v.w * v.w;
      } else {
        for (int64_t j = i; j < min(i + 4, end); ++j) acc += (double)p[j] * p[j];
      }
    }
  } else {
    const __nv_bfloat16* p = reinterpret_cast<const __nv_bfloat16*>(a.srcs[mat]);
    for (int64_t i = begin + (int64_t)threadIdx.x * 8; i < end; i += (int64_t)kNormThreads * 8) {
      if (i + 8 <= end && ((reinterpret_cast<uintptr_t>(p + i) & 15) == 0)) {
        uint4 u = *reinterpret_cast<const uint4*>(p + i);
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float2 f = __bfloat1622float2(h[q]);
          acc += (double)(f.x * f.x) + (double)(f.y * f.y);   // bf16^2 is exact in fp32
        }
      } else {
        for (int64_t j = i; j < min(i + 8, end); ++j) {
          float f = __bfloat162float(p[j]);
          acc += (double)(f * f);
        }
      }
    }
  }
  // block reduction in a fixed order (deterministic)
  __shared__ double red[kNormThreads / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffff, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kNormThreads / 32; ++w) s += red[w];
    a.partials[blk] = s;
    __threadfence();
    const unsigned prev = atomicAdd(&a.counters[mat], 1u);
    last = (prev + 1 == (unsigned)a.nchunks[mat]);
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    // partials of this matrix are contiguous blocks [blk - ci, blk - ci + nchunks)
    const int first = blk - ci;
    double s = 0.0;
    for (int k = 0; k < a.nchunks[mat]; ++k) s += *(volatile double*)&a.partials[first + k];
    const double denom = sqrt(s) * 1.01 + 1e-7;
    a.inv[mat] = (float)(1.0 / denom);
    a.counters[mat] = 0u;                          // ready for the next call / graph replay
  }
}

struct CopyArgs {
  const CopyTile* tiles;
  int ntiles;
  const void* const* srcs;     // per matrix source
  void* const* dsts;           // per matrix destination
  const int* src_rows;         // per matrix
  const int* src_cols;
  const int* src_ld;
  const int* dst_ld;
  const int* transpose;        // per matrix: dst = src^T
  const float* scale;          // per matrix multiplier or nullptr
  int src_f32, dst_f32;
};

template <typename T> __device__ __forceinline__ float to_f(T v);
template <> __device__ __forceinline__ float to_f<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T> __device__ __forceinline__ T from_f(float v);
template <> __device__ __forceinline__ float from_f<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

template <typename TS, typename TD>
__device__ __forceinline__ void copy_tile(const CopyArgs& a, const CopyTile ct, float (*tile)[65]) {
  const int mat = ct.mat;
  const TS* src = reinterpret_cast<const TS*>(a.srcs[mat]);
  TD* dst = reinterpret_cast<TD*>(a.dsts[mat]);
  const int R = a.src_rows[mat], C = a.src_cols[mat];
  const int sld = a.src_ld[mat], dld = a.dst_ld[mat];
  const bool tr = a.transpose[mat] != 0;
  const float sc = a.scale ? a.scale[mat] : 1.0f;
  const int r0 = ct.tr * 64, c0 = ct.tc * 64;
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;   // 64 x 4
  for (int i = ty; i < 64; i += 4) {
    const int r = r0 + i, c = c0 + tx;
    float v = 0.f;
    if (r < R && c < C) v = to_f<TS>(src[(size_t)r * sld + c]);
    tile[i][tx] = a.scale ? __fmul_rn(v, sc) : v;
  }
  __syncthreads();
  if (!tr) {
    for (int i = ty; i < 64; i += 4) {
      const int r = r0 + i, c = c0 + tx;
      if (r < R && c < C) dst[(size_t)r * dld + c] = from_f<TD>(tile[i][tx]);
    }
  } else {
    // dst is C x R: dst[c][r] = src[r][c]
    for (int i = ty; i < 64; i += 4) {
      const int c = c0 + i, r = r0 + tx;
      if (r < R && c < C) dst[(size_t)c * dld + r] = from_f<TD>(tile[tx][i]);
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256) pe_copy_kernel(const CopyArgs a) {
  __shared__ float tile[64][65];
  for (int t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
    const CopyTile ct = a.tiles[t];
    if (a.src_f32) {
      if (a.dst_f32) copy_tile<float, float>(a, ct, tile);
      else copy_tile<float, __nv_bfloat16>(a, ct, tile);
    } else {
      if (a.dst_f32) copy_tile<__nv_bfloat16, float>(a, ct, tile);
      else copy_tile<__nv_bfloat16, __nv_bfloat16>(a, ct, tile);
    }
  }
}

}  // namespace pe
