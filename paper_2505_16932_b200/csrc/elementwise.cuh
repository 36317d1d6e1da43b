// HBM-bound passes of the hot path:
//   pe_norm_kernel       per-matrix sum of squares (fp64, deterministic
//                        two-level reduction) -> s = ||M||_F * 1.01 + 1e-7
//                        (Listing 2; readings R1/R2), inv = fp32(1/s).
//   pe_rows_kernel       row-contiguous copy with optional scale: X_0 = M/s for
//                        wide inputs, and the final copy for outputs whose
//                        rows are not 16-byte multiples.  16-byte vectors.
//   pe_transpose_kernel  64x64 tiles through smem: X_0 = (M/s)^T for tall
//                        inputs (transpose trick) and the transpose
//                        back of tall results.  16-byte vectors on
//                        both the read and the write side.
//   pe_planes_kernel     fp32 path: X_0 = M/s split into three bf16 planes
//                        (gemm_sm100.cuh, kP = 3), and the final fp32 result
//                        p0 + p1 + p2; optionally transposed (tall inputs).
#pragma once
#include <cuda_bf16.h>

#include "pe_types.h"
#include "ptx.cuh"

namespace pe {

#ifndef PE_NORM_CHUNK
#define PE_NORM_CHUNK 98304
#endif
#ifndef PE_NORM_PERSIST
#define PE_NORM_PERSIST 0
#endif
constexpr int kNormChunk = PE_NORM_CHUNK;   // elements per norm block
constexpr int kNormThreads = 256;
#ifndef PE_NORM_UNROLL
#define PE_NORM_UNROLL 8
#endif
constexpr int kNormUnroll = PE_NORM_UNROLL;

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
  int* zero;                   // fused GEMM schedule: completion counters to clear, or nullptr
  int nzero;
  // Muon step (pe_muon_step, bf16 only): srcs are the momentum buffers M,
  // updated in place to M = bf16(beta M + (1 - beta) G) before the norm of
  // the new M is taken
  const void* const* grads;    // G per matrix, or nullptr (plain pe_polar)
  float beta, omb;             // fp32(beta), fp32(1 - beta)
  double* sums;                // sharded calls: write the local sum of squares here instead of inv
  int nblk;                    // chunks in total (the grid is persistent: block b takes chunks b, b + grid, ...)
  double* ssq;                 // spectrum-aware init: per matrix sum of squares, or nullptr
};

// |x| of a bf16 (bit pattern in the low 16 bits of h) as an fp64 value built
// with integer ops: exponent e + (1023 - 127), the 7 mantissa bits on top of
// the fp64 mantissa.  The F2F.F64.F32 conversion it replaces runs at a
// quarter of the issue rate and made the norm pass issue-bound (71 % of HBM)
// when the power cap pulled the SM clock to ~1.1 GHz.  Exact for normal bf16
// values; zero and subnormals become ~2^-127 (their squares, <= 2^-252, vanish
// in any sum of a non-negligible matrix, and a matrix of only such values has
// s = 1e-7 either way); Inf / NaN become 2^128 (the iteration still
// propagates them: X_0 = M inv).
__device__ __forceinline__ double bf16_abs_f64(uint32_t h) {
  return __hiloint2double((int)(((h & 0x7FFFu) << 13) + 0x38000000u), 0);
}

__device__ __forceinline__ double sumsq8_bf16(uint4 u) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
  double acc = 0.0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const double a = bf16_abs_f64(w[q]), b = bf16_abs_f64(w[q] >> 16);
    acc += a * a + b * b;   // exact squares in fp64 (an fp32 square overflows past |x| ~ 1.8e19)
  }
  return acc;
}

// One chunk of one matrix: partial sum of squares, and the matrix's s when
// this is its last chunk to finish.
__device__ __forceinline__ void norm_chunk(const NormArgs& a, const int blk) {
  const int mat = a.chunk_mat[blk];
  const int ci = a.chunk_idx[blk];
  const int64_t total = a.elems[mat];
  const int64_t begin = (int64_t)ci * kNormChunk;
  const int64_t end = min(begin + (int64_t)kNormChunk, total);
  double acc = 0.0;
  if (a.grads != nullptr) {
    // momentum update fused into the norm pass: reads M and G, writes M
    __nv_bfloat16* p = const_cast<__nv_bfloat16*>(reinterpret_cast<const __nv_bfloat16*>(a.srcs[mat]));
    const __nv_bfloat16* gp = reinterpret_cast<const __nv_bfloat16*>(a.grads[mat]);
    const bool al = (((reinterpret_cast<uintptr_t>(p) | reinterpret_cast<uintptr_t>(gp)) & 15) == 0);
    int64_t i = begin + (int64_t)threadIdx.x * 8;
    constexpr int64_t kStride = (int64_t)kNormThreads * 8;
    auto upd = [&](float m, float g) { return __float2bfloat16_rn(__fadd_rn(__fmul_rn(a.beta, m), __fmul_rn(a.omb, g))); };
    if (al) {
      for (; i + 8 <= end; i += kStride) {
        const uint4 mu = *reinterpret_cast<const uint4*>(p + i);
        const uint4 gu = __ldg(reinterpret_cast<const uint4*>(gp + i));
        const __nv_bfloat162* mh = reinterpret_cast<const __nv_bfloat162*>(&mu);
        const __nv_bfloat162* gh = reinterpret_cast<const __nv_bfloat162*>(&gu);
        uint4 ou;
        __nv_bfloat162* oh = reinterpret_cast<__nv_bfloat162*>(&ou);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 mf = __bfloat1622float2(mh[q]), gf = __bfloat1622float2(gh[q]);
          oh[q] = __halves2bfloat162(upd(mf.x, gf.x), upd(mf.y, gf.y));
        }
        *reinterpret_cast<uint4*>(p + i) = ou;
        acc += sumsq8_bf16(ou);
      }
    }
    for (; i < end; i += kStride)
      for (int64_t j = i; j < min(i + 8, end); ++j) {
        const __nv_bfloat16 v = upd(__bfloat162float(p[j]), __bfloat162float(gp[j]));
        p[j] = v;
        const float f = __bfloat162float(v);
        acc += (double)f * f;
      }
  } else if (a.src_f32) {
    const float* p = reinterpret_cast<const float*>(a.srcs[mat]);
    const bool al = ((reinterpret_cast<uintptr_t>(p) & 15) == 0);
    int64_t i = begin + (int64_t)threadIdx.x * 4;
    if (al) {
      for (; i + 4 <= end; i += (int64_t)kNormThreads * 4) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(p + i));
        acc += (double)v.x * v.x + (double)v.y * v.y + (double)v.z * v.z + (double)v.w * v.w;
      }
    }
    for (; i < end; i += (int64_t)kNormThreads * 4)
      for (int64_t j = i; j < min(i + 4, end); ++j) acc += (double)p[j] * p[j];
  } else {
    const __nv_bfloat16* p = reinterpret_cast<const __nv_bfloat16*>(a.srcs[mat]);
    const bool al = ((reinterpret_cast<uintptr_t>(p) & 15) == 0);
    int64_t i = begin + (int64_t)threadIdx.x * 8;
    constexpr int64_t kStride = (int64_t)kNormThreads * 8;
    if (al) {
      // kNormUnroll independent 16-byte loads in flight per thread
      for (; i + (kNormUnroll - 1) * kStride + 8 <= end; i += kNormUnroll * kStride) {
        uint4 u[kNormUnroll];
#pragma unroll
        for (int q = 0; q < kNormUnroll; ++q) u[q] = __ldg(reinterpret_cast<const uint4*>(p + i + q * kStride));
#pragma unroll
        for (int q = 0; q < kNormUnroll; ++q) acc += sumsq8_bf16(u[q]);
      }
      for (; i + 8 <= end; i += kStride) acc += sumsq8_bf16(__ldg(reinterpret_cast<const uint4*>(p + i)));
    }
    for (; i < end; i += kStride)
      for (int64_t j = i; j < min(i + 8, end); ++j) {
        const float f = __bfloat162float(p[j]);
        acc += (double)f * f;
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
    if (a.ssq != nullptr) a.ssq[mat] = s;
    if (a.sums != nullptr) {
      a.sums[mat] = s;                             // all-reduced by the caller, then pe_inv_kernel
    } else {
      const double denom = sqrt(s) * 1.01 + 1e-7;
      a.inv[mat] = (float)(1.0 / denom);
    }
    a.counters[mat] = 0u;                          // ready for the next call / graph replay
  }
  __syncthreads();                                 // red / last are reused by the next chunk
}

// One block per chunk (PE_NORM_PERSIST=1: one wave of blocks walking the
// chunks round-robin -- measured slower, 66 vs 49 us on GPT-2 S, because a
// block's loads stop at every chunk's reduction).  Chunks of 96 Ki elements
// with 8 loads in flight per thread: 42.9 us for the GPT-2 S set (65536 / 4
// loads: 53 us; ncu of that one: SMs active 67 % of the elapsed cycles, a
// 1.46-wave tail); profiles/r1_norm.md.
__global__ void __launch_bounds__(kNormThreads) pe_norm_kernel(const NormArgs a) {
  pdl_trigger();
  pdl_wait();
  for (int i = blockIdx.x * kNormThreads + threadIdx.x; i < a.nzero; i += gridDim.x * kNormThreads) a.zero[i] = 0;
  for (int blk = blockIdx.x; blk < a.nblk; blk += gridDim.x) norm_chunk(a, blk);
}

// Per-matrix parameters of a copy pass (row copy or tile transpose).
struct CopyMat {
  int rows, cols;        // source shape
  int sld, dld;          // leading dims (elements)
  int64_t pstride;       // fp32 path: elements between the three bf16 planes of the workspace side
};

// Work item of the copy passes: a band of rows (row kernel) or a 64x64 tile
// (transpose kernel) of one matrix.
struct CopyItem {
  int mat, a, b, pad;    // rows: a = first row, b = row count; transpose: a = tile row, b = tile col
};

struct CopyArgs {
  const CopyItem* items;
  int nitems;
  const CopyMat* mats;
  const void* const* srcs;     // per matrix source
  void* const* dsts;           // per matrix destination
  const float* scale;          // per matrix multiplier or nullptr
  int pow2;                    // multiply by the power-of-two part of scale only (pow2_part, exact)
  int muon;                    // finalize of pe_muon_step: dst = bf16(dst - lr * src) (Muon W update)
  float lr;
};

template <typename T> struct VecT;
template <> struct VecT<__nv_bfloat16> { static constexpr int N = 8; };
template <> struct VecT<float> { static constexpr int N = 4; };

__device__ __forceinline__ void unpack(const uint4& u, float* f, __nv_bfloat16*) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}
__device__ __forceinline__ void unpack(const uint4& u, float* f, float*) {
  f[0] = __uint_as_float(u.x); f[1] = __uint_as_float(u.y);
  f[2] = __uint_as_float(u.z); f[3] = __uint_as_float(u.w);
}
__device__ __forceinline__ uint4 pack(const float* f, __nv_bfloat16*) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return u;
}
__device__ __forceinline__ uint4 pack(const float* f, float*) {
  return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]), __float_as_uint(f[3]));
}
__device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
__device__ __forceinline__ float to_f(float v) { return v; }
template <typename T> __device__ __forceinline__ T from_f(float v);
template <> __device__ __forceinline__ float from_f<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

// 8 elements of a row <-> fp32 registers (bf16: one 16-byte vector, fp32: two)
__device__ __forceinline__ void load8(const __nv_bfloat16* p, float* f) {
  unpack(*reinterpret_cast<const uint4*>(p), f, (__nv_bfloat16*)nullptr);
}
__device__ __forceinline__ void load8(const float* p, float* f) {
  unpack(*reinterpret_cast<const uint4*>(p), f, (float*)nullptr);
  unpack(*reinterpret_cast<const uint4*>(p + 4), f + 4, (float*)nullptr);
}
__device__ __forceinline__ void store8(__nv_bfloat16* p, const float* f) {
  *reinterpret_cast<uint4*>(p) = pack(f, (__nv_bfloat16*)nullptr);
}
__device__ __forceinline__ void store8(float* p, const float* f) {
  *reinterpret_cast<uint4*>(p) = pack(f, (float*)nullptr);
  *reinterpret_cast<uint4*>(p + 4) = pack(f + 4, (float*)nullptr);
}

// dst[r][c] = scale * src[r][c] for the rows of each item (S, D: element
// types of source and destination; bf16 <-> fp32 conversions for pe_polar_ex).
template <typename S, typename D = S>
__global__ void __launch_bounds__(256) pe_rows_kernel(const CopyArgs a) {
  pdl_trigger();
  pdl_wait();
  constexpr int V = 8;
  for (int it = blockIdx.x; it < a.nitems; it += gridDim.x) {
    const CopyItem ci = a.items[it];
    const CopyMat cm = a.mats[ci.mat];
    const S* src = reinterpret_cast<const S*>(a.srcs[ci.mat]);
    D* dst = reinterpret_cast<D*>(a.dsts[ci.mat]);
    const float sc = a.scale ? (a.pow2 ? pow2_part(a.scale[ci.mat]) : a.scale[ci.mat]) : 1.0f;
    const bool vec = (cm.cols % V == 0) && (cm.sld % V == 0) && (cm.dld % V == 0) &&
                     ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
    if (vec) {
      const int vpr = cm.cols / V;                    // vectors per row
      const int64_t nv = (int64_t)vpr * ci.b;
      for (int64_t e = threadIdx.x; e < nv; e += blockDim.x) {
        const int rr = ci.a + (int)(e / vpr);
        const int cc = (int)(e % vpr) * V;
        float f[V];
        load8(src + (size_t)rr * cm.sld + cc, f);
        if (a.scale) {
#pragma unroll
          for (int j = 0; j < V; ++j) f[j] = __fmul_rn(f[j], sc);
        }
        if (a.muon) {
          float w[V];
          load8(dst + (size_t)rr * cm.dld + cc, w);
#pragma unroll
          for (int j = 0; j < V; ++j) f[j] = __fsub_rn(w[j], __fmul_rn(a.lr, f[j]));
        }
        store8(dst + (size_t)rr * cm.dld + cc, f);
      }
    } else {
      const int64_t ne = (int64_t)cm.cols * ci.b;
      for (int64_t e = threadIdx.x; e < ne; e += blockDim.x) {
        const int rr = ci.a + (int)(e / cm.cols);
        const int cc = (int)(e % cm.cols);
        float f = to_f(src[(size_t)rr * cm.sld + cc]);
        if (a.scale) f = __fmul_rn(f, sc);
        if (a.muon) f = __fsub_rn(to_f(dst[(size_t)rr * cm.dld + cc]), __fmul_rn(a.lr, f));
        dst[(size_t)rr * cm.dld + cc] = from_f<D>(f);
      }
    }
  }
}

// dst (cols x rows) = (scale * src)^T, 64x64 tiles, 256 threads.
template <typename S, typename D = S>
__global__ void __launch_bounds__(256) pe_transpose_kernel(const CopyArgs a) {
  pdl_trigger();
  pdl_wait();
  constexpr int V = VecT<S>::N;                 // source elements per 16-byte vector
  constexpr int VPR = 64 / V;                   // source vectors per 64-element tile row
  constexpr int W = VecT<D>::N;                 // destination elements per 16-byte vector
  constexpr int WPR = 64 / W;
  __shared__ float tile[64][65];
  for (int it = blockIdx.x; it < a.nitems; it += gridDim.x) {
    const CopyItem ci = a.items[it];
    const CopyMat cm = a.mats[ci.mat];
    const S* src = reinterpret_cast<const S*>(a.srcs[ci.mat]);
    D* dst = reinterpret_cast<D*>(a.dsts[ci.mat]);
    const float sc = a.scale ? (a.pow2 ? pow2_part(a.scale[ci.mat]) : a.scale[ci.mat]) : 1.0f;
    const int r0 = ci.a * 64, c0 = ci.b * 64;
    const bool vin = (cm.sld % V == 0) && ((reinterpret_cast<uintptr_t>(src) & 15) == 0);
    const bool vout = (cm.dld % W == 0) && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0);
    // load 64 x 64 (rows r0.., cols c0..)
    for (int e = threadIdx.x; e < 64 * VPR; e += 256) {
      const int i = e / VPR, jv = (e % VPR) * V;
      const int r = r0 + i, c = c0 + jv;
      float f[V];
      if (vin && r < cm.rows && c + V <= cm.cols) {
        unpack(*reinterpret_cast<const uint4*>(src + (size_t)r * cm.sld + c), f, (S*)nullptr);
      } else {
#pragma unroll
        for (int j = 0; j < V; ++j) f[j] = (r < cm.rows && c + j < cm.cols) ? to_f(src[(size_t)r * cm.sld + c + j]) : 0.f;
      }
#pragma unroll
      for (int j = 0; j < V; ++j) tile[i][jv + j] = a.scale ? __fmul_rn(f[j], sc) : f[j];
    }
    __syncthreads();
    // store transposed: dst row = c0 + i (source column), dst cols = r0.. (source rows)
    for (int e = threadIdx.x; e < 64 * WPR; e += 256) {
      const int i = e / WPR, jv = (e % WPR) * W;
      const int dr = c0 + i, dc = r0 + jv;
      if (dr >= cm.cols) continue;
      float f[W];
#pragma unroll
      for (int j = 0; j < W; ++j) f[j] = tile[jv + j][i];
      if (vout && dc + W <= cm.rows) {
        if (a.muon) {
          float w[W];
          unpack(*reinterpret_cast<const uint4*>(dst + (size_t)dr * cm.dld + dc), w, (D*)nullptr);
#pragma unroll
          for (int j = 0; j < W; ++j) f[j] = __fsub_rn(w[j], __fmul_rn(a.lr, f[j]));
        }
        *reinterpret_cast<uint4*>(dst + (size_t)dr * cm.dld + dc) = pack(f, (D*)nullptr);
      } else {
#pragma unroll
        for (int j = 0; j < W; ++j)
          if (dc + j < cm.rows) {
            float v = f[j];
            if (a.muon) v = __fsub_rn(to_f(dst[(size_t)dr * cm.dld + dc + j]), __fmul_rn(a.lr, v));
            dst[(size_t)dr * cm.dld + dc + j] = from_f<D>(v);
          }
      }
    }
    __syncthreads();
  }
}

// fp32 path, one 64x64 tile of the source per item.
//   kSplit: src fp32 caller matrix (rows x cols, ld sld), dst three bf16
//           planes (ld dld, plane stride pstride): dst = split3(scale * src)
//   else:   src three bf16 planes (ld sld, plane stride pstride), dst fp32:
//           dst = p0 + p1 + p2
// kTr: dst is the transpose (cols x rows) of src.
template <bool kSplit, bool kTr>
__global__ void __launch_bounds__(256) pe_planes_kernel(const CopyArgs a) {
  pdl_trigger();
  pdl_wait();
  __shared__ float tile[64][65];
  for (int it = blockIdx.x; it < a.nitems; it += gridDim.x) {
    const CopyItem ci = a.items[it];
    const CopyMat cm = a.mats[ci.mat];
    const float sc = a.scale ? (a.pow2 ? pow2_part(a.scale[ci.mat]) : a.scale[ci.mat]) : 1.0f;
    const int r0 = ci.a * 64, c0 = ci.b * 64;
    auto put = [&](int dr, int dc, float f) {
      if (kSplit) {
        __nv_bfloat16* d = reinterpret_cast<__nv_bfloat16*>(a.dsts[ci.mat]) + (size_t)dr * cm.dld + dc;
        const __nv_bfloat16 h0 = __float2bfloat16_rn(f);
        const float r1 = __fsub_rn(f, __bfloat162float(h0));
        const __nv_bfloat16 h1 = __float2bfloat16_rn(r1);
        d[0] = h0;
        d[cm.pstride] = h1;
        d[2 * cm.pstride] = __float2bfloat16_rn(__fsub_rn(r1, __bfloat162float(h1)));
      } else {
        reinterpret_cast<float*>(a.dsts[ci.mat])[(size_t)dr * cm.dld + dc] = f;
      }
    };
    for (int e = threadIdx.x; e < 64 * 64; e += 256) {
      const int i = e >> 6, j = e & 63;
      const int r = r0 + i, c = c0 + j;
      float f = 0.f;
      if (r < cm.rows && c < cm.cols) {
        const size_t o = (size_t)r * cm.sld + c;
        if (kSplit) {
          f = reinterpret_cast<const float*>(a.srcs[ci.mat])[o];
          if (a.scale) f = __fmul_rn(f, sc);
        } else {
          const __nv_bfloat16* p = reinterpret_cast<const __nv_bfloat16*>(a.srcs[ci.mat]) + o;
          f = __fadd_rn(__fadd_rn(__bfloat162float(p[0]), __bfloat162float(p[cm.pstride])),
                        __bfloat162float(p[2 * cm.pstride]));
        }
        if (!kTr) put(r, c, f);
      }
      if (kTr) tile[i][j] = f;
    }
    if (kTr) {
      __syncthreads();
      for (int e = threadIdx.x; e < 64 * 64; e += 256) {
        const int i = e >> 6, j = e & 63;
        const int dr = c0 + i, dc = r0 + j;          // dst row = source column
        if (dr < cm.cols && dc < cm.rows) put(dr, dc, tile[j][i]);
      }
      __syncthreads();
    }
  }
}

// Sharded calls (pe_polar_split): inv from the all-reduced sum of squares
// (P:494), and the all-reduced fp32 Gram rounded once to the bf16 A the poly
// reads -- scaled by fp32(inv inv) in the first iteration, as the folded
// Gram epilogue does (reading R8).
__global__ void pe_inv_kernel(const double* sums, float* inv) {
  pdl_trigger();
  pdl_wait();
  if (threadIdx.x == 0) inv[0] = (float)(1.0 / (sqrt(sums[0]) * 1.01 + 1e-7));
}
__global__ void __launch_bounds__(256) pe_round_gram_kernel(const float* a32, __nv_bfloat16* a, int64_t n,
                                                            const float* inv, int first) {
  pdl_trigger();
  pdl_wait();
  const float sc = first ? __fmul_rn(inv[0], inv[0]) : 1.0f;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = __float2bfloat16_rn(first ? __fmul_rn(a32[i], sc) : a32[i]);
}

// pe_polar_split_peers: the cross-rank sums over peer-visible slots (slot r =
// rank r's partial results, written by its own kernels; on several GPUs a
// P2P-mapped or NVLS buffer, read here with plain loads), in rank order so
// every rank forms bit-identical sums.  Slot layout: double ||M_r||^2 at byte
// 0, partial Gram of parity p at byte 256 + p * gbytes.
struct PeerSlots {
  const uint8_t* const* slots;   // [world] device pointers
  int world;
  int64_t gbytes;                // bytes of one partial Gram (m * ldm fp32, 256-byte padded)
};
__global__ void pe_inv_peers_kernel(const PeerSlots ps, float* inv) {
  pdl_trigger();
  pdl_wait();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int r = 0; r < ps.world; ++r) s += *reinterpret_cast<const volatile double*>(ps.slots[r]);
    inv[0] = (float)(1.0 / (sqrt(s) * 1.01 + 1e-7));
  }
}
__global__ void __launch_bounds__(256) pe_round_peers_kernel(const PeerSlots ps, int parity, __nv_bfloat16* a,
                                                             int64_t n, const float* inv, int first) {
  pdl_trigger();
  pdl_wait();
  const float sc = first ? __fmul_rn(inv[0], inv[0]) : 1.0f;
  const int64_t off = 256 + parity * ps.gbytes;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float v = 0.f;
    for (int r = 0; r < ps.world; ++r) v = __fadd_rn(v, __ldcg(reinterpret_cast<const float*>(ps.slots[r] + off) + i));
    a[i] = __float2bfloat16_rn(first ? __fmul_rn(v, sc) : v);
  }
}

// Per-call upload of a pe_polar call (pointers, caller tensor maps,
// coefficients) from its mapped pinned host buffer, read over PCIe by the
// SMs: it never waits in the copy engines behind unrelated bulk transfers.
__global__ void __launch_bounds__(256) pe_upload_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                        int n) {
  pdl_trigger();
  // Like every kernel of the library, wait for the previous grid before
  // touching memory: the wait is what chains consecutive calls (a later
  // call's kernels never overlap an earlier call's, whose buffers -- this
  // upload slot four calls back, the plan's workspace -- they reuse).
  pdl_wait();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[i] = src[i];
}

// ---------------------------------------------------------------- debug scan
// Count the non-finite elements (NaN / Inf: all exponent bits set) of one
// buffer of n elements (bf16 or fp32) into *count (pe_count_nonfinite,
// PE_DEBUG_CHECK_FINITE; off the hot path).
template <typename T>
__global__ void __launch_bounds__(256) pe_nonfinite_kernel(const T* __restrict__ x, int64_t n,
                                                           unsigned long long* count) {
  pdl_trigger();
  pdl_wait();
  unsigned long long k = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (sizeof(T) == 2) {
      const uint16_t u = reinterpret_cast<const uint16_t*>(x)[i];
      k += (u & 0x7F80u) == 0x7F80u;
    } else {
      const uint32_t u = reinterpret_cast<const uint32_t*>(x)[i];
      k += (u & 0x7F800000u) == 0x7F800000u;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) k += __shfl_xor_sync(0xffffffffu, k, o);
  if ((threadIdx.x & 31) == 0 && k) atomicAdd(count, k);
}

// ---------------------------------------------------------------- App. H
// Fast rectangular iteration (Alg. 4): with Q_0 = I the first
// iteration of an application is R_1 = Y and Q_1 = h_1(Y) = a_1 I + H_1,
// H_1 = b_1 Y + c_1 Y^2 (the poly GEMM).  This pass writes Q_1 in full
// storage (the later products read it as a plain m x m operand) from H_1's
// upper-block-triangle storage: Q_1 = bf16(fp32(H_1) + a_1) on the diagonal,
// H_1 elsewhere (blocks below the diagonal read transposed).  One 64 x 64
// tile per block, through shared memory (coalesced both ways).
struct ExpandArgs {
  const CopyItem* items;       // (mat, tile row, tile col) of 64 x 64 tiles
  int nitems;
  const MatDev* mats;          // source mats[i].B (H_1), destination mats[i].E[0] (Q_1)
  float a;
};
__global__ void __launch_bounds__(256) pe_expand_kernel(const ExpandArgs e) {
  pdl_trigger();
  pdl_wait();
  // [64][64 + 8] bf16: row pitch 144 bytes keeps 16-byte row segments aligned
  // and spreads the column gathers of the transposed tiles over the banks
  __shared__ __align__(16) __nv_bfloat16 t[64][72];
  const int tid = threadIdx.x;
  for (int it = blockIdx.x; it < e.nitems; it += gridDim.x) {
    const CopyItem ci = e.items[it];
    const MatDev md = e.mats[ci.mat];
    const int r0 = ci.a * 64, c0 = ci.b * 64;
    const bool upper = (r0 / kBM) <= (c0 / kBM);
    const int sr0 = upper ? r0 : c0, sc0 = upper ? c0 : r0;
    const __nv_bfloat16* H = reinterpret_cast<const __nv_bfloat16*>(md.B);
    __nv_bfloat16* Q = reinterpret_cast<__nv_bfloat16*>(md.E[0]);
    const bool vec = (md.ldm % 8 == 0) && (sr0 + 64 <= md.m) && (sc0 + 64 <= md.m) && (r0 + 64 <= md.m) &&
                     (c0 + 64 <= md.m);
    __syncthreads();                                   // previous tile's reads of t are done
    if (vec) {
      // 512 16-byte units (row i, columns 8u .. 8u+7), two per thread
      for (int k = tid; k < 512; k += 256) {
        const int i = k >> 3, u = k & 7;
        *reinterpret_cast<uint4*>(&t[i][8 * u]) =
            *reinterpret_cast<const uint4*>(H + (int64_t)(sr0 + i) * md.ldm + sc0 + 8 * u);
      }
    } else {
      for (int k = tid; k < 64 * 64; k += 256) {
        const int i = k >> 6, j = k & 63, gr = sr0 + i, gc = sc0 + j;
        t[i][j] = (gr < md.m && gc < md.m) ? H[(int64_t)gr * md.ldm + gc] : __float2bfloat16_rn(0.f);
      }
    }
    __syncthreads();
    if (vec) {
      for (int k = tid; k < 512; k += 256) {
        const int i = k >> 3, u = k & 7, gr = r0 + i;
        __align__(16) __nv_bfloat16 v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          v[q] = upper ? t[i][8 * u + q] : t[8 * u + q][i];
          if (gr == c0 + 8 * u + q) v[q] = __float2bfloat16_rn(__fadd_rn(__bfloat162float(v[q]), e.a));
        }
        *reinterpret_cast<uint4*>(Q + (int64_t)gr * md.ldm + c0 + 8 * u) = *reinterpret_cast<const uint4*>(v);
      }
    } else {
      for (int k = tid; k < 64 * 64; k += 256) {
        const int i = k >> 6, j = k & 63, gr = r0 + i, gc = c0 + j;
        if (gr >= md.m || gc >= md.m) continue;
        __nv_bfloat16 v = upper ? t[i][j] : t[j][i];
        if (gr == gc) v = __float2bfloat16_rn(__fadd_rn(__bfloat162float(v), e.a));
        Q[(int64_t)gr * md.ldm + gc] = v;
      }
    }
  }
}

// ---------------------------------------------------------------- App. G
// Spectrum-aware first step (k = 1; reading R17): the power
// method on A_0 = X_0 X_0^T (the iteration-1 Gram, bf16, upper 256-block
// triangle stored) gives the Rayleigh quotient lambda <= sigma_1(X_0)^2, hence
// z = sqrt(lambda) / F with F = ||X_0||_F; if 1/sqrt(2) <= z <= 1 - 1e-6 the
// first step applies p(x) = [a (x/F) + b (x/F)^3] / (1 + |b| 2^-7), (a, b)
// from eq. (init_poly), as B = (b'/F^3) A_0 and
// X_1 = (a'/F) X_0 + B X_0 through the poly and update GEMMs; otherwise
// (a, b) = (1, 0).
constexpr int kSymvRows = 32;        // rows of A per work item (one per lane)
constexpr int kSymvThreads = 256;

struct SymvArgs {
  const MatDev* mats;
  const int* item_mat;       // per item: matrix
  const int* item_r0;        // per item: first row
  int nitems;
  const int* item0;          // per matrix: first item
  const int* nitem;          // per matrix: items
  const int64_t* voff;       // per matrix: offset of its vector (floats)
  const float* vin;          // previous w, or the start vector v0 in the first iteration
  const double* nrm2_in;     // ||previous w||^2 per matrix (normalises vin); nullptr: vin is v0
  float* wout;               // A v
  double* part;              // per item: v.w, w.w, v.v over its rows
  unsigned* counters;        // per matrix, zero at rest (self-resetting)
  double* lam;               // per matrix: v.w / v.v
  double* nrm2_out;          // per matrix: w.w
  float* const* a32;         // per matrix: the Gram in fp32 (upper blocks, leading dim ldm), read instead of
                             // the bf16 A (the Rayleigh quotient of bf16(A) can exceed sigma_1^2, R17)
};

// w = A v for every matrix (one launch per power iteration).  A(r, c) with
// c's 256-block left of r's is read from the stored transposed block as
// A[c][r0 .. r0+31] (4 lanes x 16 bytes per column, 8 columns per warp
// instruction), the rest row-wise as A[r][c .. c+7] (16 bytes per lane).
__device__ __forceinline__ void symv_v8(const float* vin, float vs, int c, int m, float* v) {
  if (c + 8 <= m) {                                  // vin + c is 32-byte aligned (voff % 32 == 0, c % 8 == 0)
    const float4 p = *reinterpret_cast<const float4*>(vin + c);
    const float4 q = *reinterpret_cast<const float4*>(vin + c + 4);
    v[0] = p.x * vs; v[1] = p.y * vs; v[2] = p.z * vs; v[3] = p.w * vs;
    v[4] = q.x * vs; v[5] = q.y * vs; v[6] = q.z * vs; v[7] = q.w * vs;
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = (c + k < m) ? vin[c + k] * vs : 0.f;
  }
}

template <typename TA> __device__ __forceinline__ float symv_ld(const TA* p);
template <> __device__ __forceinline__ float symv_ld<__nv_bfloat16>(const __nv_bfloat16* p) { return __bfloat162float(*p); }
template <> __device__ __forceinline__ float symv_ld<float>(const float* p) { return *p; }
// 8 consecutive elements (16 or 32 bytes, aligned) as floats
__device__ __forceinline__ void symv_ld8(const __nv_bfloat16* p, float* f) {
  const uint4 u = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float2 t = __bfloat1622float2(h[q]);
    f[2 * q] = t.x;
    f[2 * q + 1] = t.y;
  }
}
__device__ __forceinline__ void symv_ld8(const float* p, float* f) {
  const float4 x = *reinterpret_cast<const float4*>(p), y = *reinterpret_cast<const float4*>(p + 4);
  f[0] = x.x; f[1] = x.y; f[2] = x.z; f[3] = x.w; f[4] = y.x; f[5] = y.y; f[6] = y.z; f[7] = y.w;
}

template <typename TA>
__global__ void __launch_bounds__(kSymvThreads) pe_symv_kernel(const SymvArgs a) {
  pdl_trigger();
  pdl_wait();
  constexpr int kW = kSymvThreads / 32;
  __shared__ float lpart[kW][kSymvRows];
  __shared__ float upart[kSymvRows];
  __shared__ bool last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int it = blockIdx.x; it < a.nitems; it += gridDim.x) {
    const int mat = a.item_mat[it], r0 = a.item_r0[it];
    const MatDev md = a.mats[mat];
    const int m = md.m, ld = md.ldm;
    const TA* A = a.a32 ? reinterpret_cast<const TA*>(a.a32[mat]) : reinterpret_cast<const TA*>(md.A);
    const float* vin = a.vin + a.voff[mat];          // iteration 0: the start vector v0 (unnormalised)
    const float vs = a.nrm2_in ? (float)(1.0 / sqrt(a.nrm2_in[mat])) : 1.0f;
    auto v_at = [&](int c) { return vin[c] * vs; };
    const int cl = (r0 / 256) * 256;                 // columns [0, cl): transposed stored blocks
    // part L: lane = (column offset lane / 4, row segment lane % 4 of 8 rows)
    {
      const int seg = lane & 3, rs = r0 + seg * 8;
      float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      const bool full = rs + 8 <= m;
#pragma unroll 4
      for (int c = warp * 8 + (lane >> 2); c < cl; c += kW * 8) {
        const float vc = v_at(c);
        const TA* p = A + (size_t)c * ld + rs;
        if (full) {
          float f[8];
          symv_ld8(p, f);
#pragma unroll
          for (int q = 0; q < 8; ++q) acc[q] += f[q] * vc;
        } else {
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (rs + k < m) acc[k] += symv_ld<TA>(p + k) * vc;
        }
      }
      // lanes with the same segment hold the same rows: reduce over lane / 4
#pragma unroll
      for (int k = 0; k < 8; ++k) {
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], o);
      }
      if (lane < 4) {
#pragma unroll
        for (int k = 0; k < 8; ++k) lpart[warp][lane * 8 + k] = acc[k];
      }
    }
    // part U: warp w takes rows r0 + 4w .. r0 + 4w + 3, 16 bytes of a row per lane
#pragma unroll
    for (int q = 0; q < kSymvRows / kW; ++q) {
      const int rr = r0 + warp * (kSymvRows / kW) + q;
      float acc = 0.f;
      if (rr < m) {
        const TA* row = A + (size_t)rr * ld;
#pragma unroll 4
        for (int c = cl + 8 * lane; c < m; c += 256) {
          float v[8];
          symv_v8(vin, vs, c, m, v);
          if (c + 8 <= m) {
            float f[8];
            symv_ld8(row + c, f);
#pragma unroll
            for (int k = 0; k < 8; ++k) acc += f[k] * v[k];
          } else {
            for (int k = 0; k < 8 && c + k < m; ++k) acc += symv_ld<TA>(row + c + k) * v[k];
          }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) upart[rr - r0] = acc;
    }
    __syncthreads();
    double vw = 0.0, ww = 0.0, vv = 0.0;
    if (warp == 0) {
      const int r = r0 + lane;
      float w = upart[lane];
      for (int k = 0; k < kW; ++k) w += lpart[k][lane];
      if (r < m) {
        a.wout[a.voff[mat] + r] = w;
        const float vr = v_at(r);
        vw = (double)vr * w;
        ww = (double)w * w;
        vv = (double)vr * vr;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        vw += __shfl_xor_sync(0xffffffffu, vw, o);
        ww += __shfl_xor_sync(0xffffffffu, ww, o);
        vv += __shfl_xor_sync(0xffffffffu, vv, o);
      }
      if (lane == 0) {
        a.part[3 * it] = vw;
        a.part[3 * it + 1] = ww;
        a.part[3 * it + 2] = vv;
        __threadfence();
        const unsigned prev = atomicAdd(&a.counters[mat], 1u);
        last = (prev + 1 == (unsigned)a.nitem[mat]);
      }
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
      __threadfence();
      double svw = 0.0, sww = 0.0, svv = 0.0;        // items of the matrix in order (deterministic)
      for (int k = a.item0[mat]; k < a.item0[mat] + a.nitem[mat]; ++k) {
        svw += *(volatile double*)&a.part[3 * k];
        sww += *(volatile double*)&a.part[3 * k + 1];
        svv += *(volatile double*)&a.part[3 * k + 2];
      }
      a.lam[mat] = svv > 0.0 ? svw / svv : 0.0;
      a.nrm2_out[mat] = sww;
      a.counters[mat] = 0u;
    }
    __syncthreads();
  }
}

// Per matrix: z = sqrt(lambda / F^2), F^2 = ssq * inv^2 (= ||X_0||_F^2), and
// the first step's (a/F, b/F^3) from eq. (init_poly), or (1, 0).
// trace(A_0) of the raw fp32 Gram per matrix (one block each, fixed-order
// reduction): ||X_0||_F^2 of the rounded X_0 = bf16(M inv) of fp32 inputs, the
// scale the Rayleigh quotient of that Gram is on (App. G, reading R17)
__global__ void __launch_bounds__(256) pe_trace_kernel(float* const* a32, const MatDev* mats, double* tr, int count) {
  pdl_trigger();
  pdl_wait();
  __shared__ double red[256];
  const int i = blockIdx.x;
  if (i >= count) return;
  const MatDev md = mats[i];
  double s = 0.0;
  for (int j = threadIdx.x; j < md.m; j += blockDim.x) s += (double)a32[i][(size_t)j * md.ldm + j];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) tr[i] = red[0];
}

__global__ void pe_init_coef_kernel(const double* lam, const double* ssq, const float* inv, float* mcoef,
                                    int count, double margin, const int* mflags, const double* tr) {
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  // lam is the Rayleigh quotient of the fp32 Gram the iteration-1 GEMM
  // accumulated: of M M^T for folded bf16 input (flags 8 | 1), of 4^e M M^T
  // for copied bf16 input (flag 8), of X_0 X_0^T = (M/s)(M/s)^T for fp32
  // input; z = sigma_1 / ||.||_F on the same scale
  double f2 = ssq[i] * (double)inv[i] * (double)inv[i];
  // bf16 copies hold M * 2^e (pow2_part): their Gram is 4^e M M^T
  const double p2 = (double)pow2_part(inv[i]);
  double den2 = (mflags[i] & 8) ? ((mflags[i] & 1) ? ssq[i] : ssq[i] * p2 * p2) : f2;
  if (!(mflags[i] & 8) && tr != nullptr) {
    // fp32 input: X_0 = bf16(M inv) is rounded, so its norm is not ||M|| inv;
    // z and F from the same Gram keep z <= sigma_1 / F (the lower bound the
    // step's tail bound sqrt(1 - z^2) relies on)
    f2 = tr[i];
    den2 = tr[i];
  }
  const double z = (den2 > 0.0 && lam[i] > 0.0) ? sqrt(lam[i] / den2) : 0.0;
  float ca = 1.f, cb = 0.f;
  if (z >= 0.70710678118654752 && z <= 1.0 - 1e-6) {
    const double t = sqrt(1.0 - z * z);
    const double den = z * t * (2.0 * z * z - 1.0);
    const double F = sqrt(f2);
    const double a = (z * z * (z + t) - t) / den, b = (t - z) / den;
    // optional margin (pe_set_spectrum_init_ex; default 0 = eq. (init_poly)
    // exactly): divide by 1 + |b| * margin.  With z from the fp32 Gram the
    // paper's step stays finite on every input tried (R17); an earlier z from
    // the bf16 Gram overestimated sigma_1, lifted the tail past 1 and needed
    // a 2^-7 margin to avoid NaN
    const double sc = 1.0 / (1.0 + fabs(b) * margin);
    ca = (float)(a * sc / F);
    cb = (float)(b * sc / (F * F * F));
  }
  mcoef[2 * i] = ca;
  mcoef[2 * i + 1] = cb;
}

}  // namespace pe
