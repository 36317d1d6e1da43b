// Grouped persistent tcgen05 GEMM (CTA pair, cta_group::2) for the three
// products of one Polar Express iteration (Listing 2), bf16 in /
// fp32 accumulate:
//
//   kModeGram   A  = X X^T           both operands rows of X; only the
//                                    256x256 tiles with I <= J are computed
//                                    and stored (upper block triangle).
//   kModePoly   B  = b A + c (A A^T) A symmetric so A A = A A^T (SYRK on A);
//                                    the epilogue reads the same bf16 A
//                                    (reading R8); upper block triangle.
//   kModeUpdate X' = a X + B X       left operand B (K-major), right operand
//                                    X (MN-major: row-major X is N-contiguous).
// The blocks of A and B below the diagonal are never written: a consumer
// that needs block (I, P) with P < I loads the stored block (P, I) and feeds
// it to the MMA as an MN-major operand (the transpose is free in the UMMA
// descriptor), so the symmetric phases write half the bytes.
//
// Normalisation and orientation are folded into the first and last
// iteration (no X_0 buffer, no transpose-back pass) for caller matrices whose
// rows are 16-byte multiples: the first Gram reads the caller's M directly
// (K-major if wide, MN-major -- i.e. M^T -- if tall) and scales its fp32
// accumulator by inv^2, inv = fp32(1/s), s = ||M||_F * 1.01 + 1e-7;
// the first update reads M as its right operand and epilogue operand and
// scales (a M + B M) by inv; the last update writes the caller's buffer,
// transposed through shared memory when the caller's matrix is tall.
//
// A cluster of two CTAs on one TPC computes one 256x256 output tile with
// tcgen05.mma.cta_group::2 (M=256, N=256, K=16): CTA r holds rows
// [128r, 128r+128) of the left operand and rows/columns [128r, 128r+128) of
// the right operand in its shared memory, and accumulator rows
// [128r, 128r+128) x 256 columns in its TMEM.  Per CTA:
//   warp 0      TMA producer (64x64 bf16 boxes, 128B swizzle, kSt-stage
//               ring; bytes of both CTAs are counted on the leader's barrier)
//   warp 1      leader: single-thread MMA issuer; both: TMEM alloc (512 cols
//               = two 256-column fp32 accumulators -> the epilogue of tile i
//               overlaps the main loop of tile i+1)
//   warps 2..9  epilogue: lane quadrant (warp % 4) x column half
//               ((warp-2) / 4), 32-row x 64-column chunks staged in a 4 KB
//               smem slot (128B swizzle): operand chunks arrive by TMA, bf16
//               results leave by TMA store.
// Grouped scheduling: one launch covers every tile of every matrix of the
// batch; cluster c walks tiles c, c + #clusters, ... of a host-built list.
//
// fp32 (kP = 3): every workspace buffer holds three stacked bf16 planes
// v = p0 + p1 + p2 (p0 = bf16(v), p1 = bf16(v - p0), p2 = bf16(v - p0 - p1);
// 24 significand bits, i.e. an fp32 value), and each product is the K-
// concatenation of the six plane products with i + j <= 2:
//   P Q^T ~ sum_{i+j<=2} P_i Q_j^T  =  [P2 P1 P0 P1 P0 P0] [Q0 Q1 Q2 Q0 Q1 Q0]^T
// (dropped terms are O(2^-24) relative).  The main loop is the bf16 one over
// 6x the k-blocks (plane p of a buffer = rows [p m, (p+1) m) of its stacked
// tensor map); the epilogue sums the operand planes, applies the fp32
// arithmetic and splits the result into planes again.  No folding, no
// diagonal single-panel loads.  The tensor core adds every K=16 step into the
// fp32 accumulator with truncation, so the accumulation order is arranged to
// keep each truncating chain short (small plane products first, the big
// p0 q0 chain in passes of <= 16 K blocks split over both TMEM buffers, an
// fp32 running sum across passes; see p3_passes).
#pragma once
#include <cuda_bf16.h>

#include "pe_types.h"
#include "ptx.cuh"

namespace pe {

// Timeline instrumentation (PE_DEBUG_GEMM bit 128, profiles/phase_timeline.py):
// compiled in only with -DPE_GEMM_TIMELINE=1 (PE_NVCC_FLAGS at build time)
#ifndef PE_GEMM_TIMELINE
#define PE_GEMM_TIMELINE 0
#endif
constexpr bool kGemmTimeline = PE_GEMM_TIMELINE != 0;

// per-call matrix flags
constexpr int kFlagFolded = 1;   // iteration 1 reads the caller's M (no X_0 buffer)
constexpr int kFlagTall = 2;     // caller matrix is rows > cols (iterate on M^T)
constexpr int kFlagDirect = 4;   // last update writes the caller's output buffer
constexpr int kFlagScaled = 8;   // iteration 1 reads the unscaled bf16 M (the caller's, or an exact
                                 // oriented copy) and applies 1/s in its epilogues (reading R8)

struct GemmArgs {
  const Tile* tiles;
  int ntiles;
  const MatDev* mats;
  const CUtensorMap* tmaps;    // main loop, 6 per matrix: X[0], X[1] (64x64 boxes), A, B (64 x 128-row
                               // boxes), A, B (64x64 boxes, for transposed reads); 128B swizzle
  const CUtensorMap* emaps;    // epilogue, 4 kP per matrix: X[0], X[1], A, B (64-col x 32-row boxes) x planes
  const CUtensorMap* imaps;    // per call, 2 per matrix: caller input main loop / epilogue chunk
  const CUtensorMap* omaps;    // per call, 1 per matrix: caller output epilogue chunk
  const int* mflags;           // per call, per matrix: kFlag*
  const float* inv;            // per matrix fp32(1/s)
  float* scratch;              // kP = 3: 128 x 256 fp32 per CTA (running sum of the K passes)
  float* const* out32;         // sharded calls: the Gram writes its raw fp32 accumulator here (m x m,
                               // leading dim ldm, blocks on/above the diagonal), not bf16 A; else nullptr
  int out32_both = 0;          // App. G step: the raw fp32 accumulator to out32 AND the usual bf16 A
  int muon;                    // pe_muon_step: the last update's direct output is the weight W,
  float lr;                    // updated to bf16(W - lr * bf16(X'))
  // one phase per launch (nphase == 0): the phase of every tile
  int mode;
  int xin;                     // which X buffer holds the current iterate
  int first_iter, final_iter;
  float a, b, c;
  // fused schedule (nphase = 3T > 0): one launch runs every phase of every
  // matrix; Tile::pad is the phase p (iteration p / 3, mode p % 3), tiles are
  // listed in a dependency-respecting order and a tile of phase p > 0 waits
  // until done[mat * nphase + p - 1] reaches need[mat * 3 + (p - 1) % 3]
  // (every epilogue warp of every tile of that phase has published)
  int nphase;
  const float* coef;           // per iteration fp32 (a, b, c)
  int* done;                   // per (matrix, phase) completion counters, zero at launch
  const int* need;             // per (matrix, mode): 2 * kEpiWarps * tiles
  const float* mcoef;          // spectrum-aware first step (App. G): per matrix (a, b), c = 0; else nullptr
  int lin;                     // odd cubic step (degree-3 table, App. G step): no poly phase; the update
                               // reads A as its left operand and computes X' = a X + b (A X)
  // Fast rectangular iteration (App. H, Alg. 4; plans built for it carry
  // kMapsRect main-loop and kEmapsRect epilogue maps per matrix, see below)
  int tstride, estride;        // main-loop / epilogue (per plane) maps per matrix: 6 / 4, or 11 / 8
  float shift;                 // Gram: added to the diagonal after the scale (Alg. 4's 10^-3 I)
  int psrc;                    // poly source: 0 = A (Y), 1 = R
  int gen;                     // update phase as a generic product of Alg. 4 (the fields below), else 0
  int g_l, g_lmn, g_lsym;      // left operand map (and its transposed-block map when symmetric-stored)
  int g_rx, g_r;               // right operand: the iterate X (caller M when folded), else map g_r (MN-major)
  int g_ein, g_eout;           // epilogue operand map (-1: none, result = acc) / result map (-1: the X logic)
  int g_wide;                  // result columns: 1 = n (X-shaped), 0 = m (square)
  int dbg;                     // timing experiments only: 1 = no epilogue work, 2 = no operand loads,
                               // 8 = all loads hit the same boxes, 16 = no TMEM loads, 32 = no result
                               // stores, 256 = every result store to the same box, 2048 = right
                               // operand not loaded (results are wrong with any of these)
  long long* stats;            // optional per-CTA wait-cycle counters (8 per CTA) or nullptr
};

// Everything the three roles need to know about one tile.
struct TileCfg {
  int mode, xin;               // phase of the tile (see GemmArgs)
  bool first, last;            // first / last iteration
  float a, b, c;               // the iteration's coefficients
  const int* dep;              // fused: counter to wait for before reading operands, or nullptr
  int dep_need;
  int* pub;                    // fused: counter to publish this tile's results to, or nullptr
  const CUtensorMap* A;        // main-loop maps of the left / right operand
  const CUtensorMap* B;
  int nk, row_a, col_b;        // k-blocks; this CTA's first row of A and of B
  bool a_mn, b_mn;             // operand stored MN-major (else K-major)
  bool a_wide, b_wide;         // operand is a symmetric m x m buffer (A or B) of which only the
                               // 256x256 blocks on or above the diagonal are stored; K-major
                               // 128-row boxes, and blocks below the diagonal are read as the
                               // transpose of the stored block (MN-major, 64x64 boxes, maps *mn)
  const CUtensorMap* Amn;
  const CUtensorMap* Bmn;
  int pan_a, pan_b;            // 256-row panel index of the left / right operand rows
  bool diag;                   // symmetric phase, I == J: one panel serves both operands
  const CUtensorMap* ein;      // epilogue operand chunk map (update: X, poly: A)
  bool ein_tr;                 // operand chunk is M^T of a tall caller matrix
  const CUtensorMap* eout;     // result chunk map
  bool eout_tr;                // result chunk is stored transposed (tall caller output)
  bool scaled;                 // first iteration of a bf16-input matrix: 1/s in the epilogue
  bool pre;                    // ... whose X_0 is the copy M * 2^e: the epilogue applies 1/s * 2^-e
  bool muon;                   // result chunk is a Muon weight update of the chunk already at eout
  bool lin;                    // update of a cubic step: left operand A, epilogue a X + b acc
  bool rr;                     // poly of Alg. 4's R: the true product R R, not R R^T -- R = Q T is not
                               // symmetric inside its diagonal blocks, so the right operand's diagonal
                               // K block is read transposed (MN-major) and diagonal tiles share nothing
  bool has_ein;                // the epilogue reads an operand chunk (poly: A/R, update: X/Q)
  int ncols;                   // result columns (n for X-shaped results, m for square ones)
  float shift;                 // Gram: diagonal shift
  int prow;                    // kP = 3: rows per plane of the stacked buffers (= m)
};

// kEdge: the launch is a first or last iteration (folded input / direct
// output possible); the middle iterations compile all of that away.
// kP: planes per buffer (1 = bf16, 3 = fp32 as three bf16 planes); the
// epilogue maps are kP per buffer (one per plane), buffer b plane p at em[kP*b + p].
template <bool kEdge, int kP = 1>
__device__ __forceinline__ TileCfg tile_cfg(const GemmArgs& g, const Tile& tl, uint32_t rank) {
  const MatDev& md = g.mats[tl.mat];
  const CUtensorMap* maps = g.tmaps + g.tstride * tl.mat;
  const CUtensorMap* em = g.emaps + g.estride * kP * tl.mat;
  TileCfg c;
  c.dep = nullptr;
  c.pub = nullptr;
  c.dep_need = 0;
  if (g.nphase > 0) {
    const int p = tl.pad, t = p / 3;
    c.mode = p - 3 * t;
    c.xin = t & 1;
    c.first = (t == 0);
    c.last = (3 * t + 3 == g.nphase);
    c.a = g.coef[3 * t];
    c.b = g.coef[3 * t + 1];
    c.c = g.coef[3 * t + 2];
    c.pub = g.done + tl.mat * g.nphase + p;
    if (p > 0) {
      c.dep = c.pub - 1;
      c.dep_need = g.need[tl.mat * 3 + (p - 1) % 3];
    }
  } else {
    c.mode = g.mode;
    c.xin = g.xin;
    c.first = g.first_iter != 0;
    c.last = g.final_iter != 0;
    c.a = g.a;
    c.b = g.b;
    c.c = g.c;
    if (g.mcoef != nullptr) {              // App. G first step: p(x) = a x + b x^3 per matrix
      c.a = g.mcoef[2 * tl.mat];
      c.b = g.mcoef[2 * tl.mat + 1];
      c.c = 0.f;
    }
  }
  const int fl = kEdge ? g.mflags[tl.mat] : 0;
  const bool fold = kEdge && c.first && (fl & kFlagFolded);
  const bool tall = kEdge && (fl & kFlagTall) != 0;
  const bool scl = kEdge && c.first && (fl & kFlagScaled);
  c.scaled = scl;
  c.pre = scl && !(fl & kFlagFolded);
  c.muon = false;
  c.lin = false;
  c.rr = false;
  c.shift = 0.f;
  c.a_wide = c.b_wide = false;
  c.Amn = c.Bmn = nullptr;
  c.pan_a = tl.tm;
  c.pan_b = tl.tn;
  c.ein = nullptr;
  c.ein_tr = false;
  c.eout_tr = false;
  if (c.mode == kModeGram) {
    c.A = c.B = fold ? g.imaps + 2 * tl.mat : maps + c.xin;
    c.a_mn = c.b_mn = fold && tall;
    c.nk = (md.n + kBK - 1) / kBK;
    c.eout = em + 2 * kP;
    c.shift = g.nphase == 0 ? g.shift : 0.f;
  } else if (c.mode == kModePoly) {
    const bool r = g.nphase == 0 && g.psrc != 0;      // Alg. 4: h(R) from R (maps 9 / 10, emap 7)
    c.rr = r;
    c.A = c.B = maps + (r ? 9 : 2);
    c.Amn = c.Bmn = maps + (r ? 10 : 4);
    c.a_mn = c.b_mn = false;
    c.a_wide = c.b_wide = true;
    c.nk = (md.m + kBK - 1) / kBK;
    c.ein = em + (r ? 7 : 2) * kP;
    c.eout = em + 3 * kP;
  } else {
    const bool gen = g.nphase == 0 && g.gen != 0;
    const bool rx = !gen || g.g_rx != 0;             // right operand is the iterate
    c.scaled = scl && rx;
    c.lin = g.nphase == 0 && g.lin != 0;
    if (gen) {
      c.A = maps + g.g_l;
      c.Amn = g.g_lsym ? maps + g.g_lmn : nullptr;
      c.a_wide = g.g_lsym != 0;      // symmetric-stored (Y, H) or full (Q: K-major 64 x 64 boxes)
    } else {
      c.A = maps + (c.lin ? 2 : 3);   // cubic: B = b A is never formed, the update reads A
      c.Amn = maps + (c.lin ? 4 : 5);
      c.a_wide = true;
    }
    c.a_mn = false;
    c.nk = (md.m + kBK - 1) / kBK;
    if (!rx) {
      c.B = maps + g.g_r;
      c.b_mn = true;
    } else if (fold) {
      c.B = g.imaps + 2 * tl.mat;
      c.b_mn = !tall;                 // wide: M is N-contiguous; tall: M^T rows are M's rows (K-contiguous)
      c.ein = g.imaps + 2 * tl.mat + 1;
      c.ein_tr = tall;
    } else {
      c.B = maps + c.xin;
      c.b_mn = true;
      c.ein = em + kP * c.xin;
    }
    if (gen) {
      c.ein = g.g_ein >= 0 ? em + kP * g.g_ein : nullptr;
      if (c.ein == nullptr) c.ein_tr = false;
    }
    if (gen && g.g_eout >= 0) {
      c.eout = em + kP * g.g_eout;
    } else if (kEdge && c.last && (fl & kFlagDirect)) {
      c.eout = g.omaps + tl.mat;
      c.eout_tr = tall;
      c.muon = g.muon != 0;
    } else {
      c.eout = em + kP * (c.xin ^ 1);
    }
  }
  c.has_ein = c.mode != kModeGram && c.ein != nullptr;
  c.ncols = (c.mode == kModeUpdate && !(g.nphase == 0 && g.gen != 0 && !g.g_wide)) ? md.n : md.m;
  c.diag = (kP == 1) && (c.mode != kModeUpdate) && (tl.tm == tl.tn) && !c.rr;
  c.prow = (kP == 1) ? 0 : md.m;
  c.row_a = tl.tm * kBM + (int)rank * (kBM / 2);
  c.col_b = tl.tn * kBN + (int)rank * (kBN / 2);
  return c;
}

__device__ __forceinline__ void bf16x8_to_f32(const uint4& u, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 t = __bfloat1622float2(h[i]);
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

// Epilogue arithmetic of one half (32 columns) of a 32-row x 64-column chunk
// (thread = row `lane`): w (fp32 accumulator in) -> w (result).  The operand
// is read from `slot` and the bf16 result written back to `slot`.  Slot
// layouts: row-major [32][64] with the TMA 128B swizzle (16-byte unit j of
// row r at r*128 + ((j ^ (r & 7)) * 16)), or -- for the transposed chunks of
// a tall caller matrix -- [64][32] plain (element (c, r) at c*32 + r).
// Rounding points: reading R8.
__device__ __forceinline__ uint32_t sw128_off(int r, int j) { return r * 128 + ((j ^ (r & 7)) << 4); }

template <bool kEdge>
__device__ __forceinline__ void epilogue_math(const GemmArgs& g, const TileCfg& cfg, float inv, uint8_t* slot,
                                             int lane, int half32, float* w, const uint32_t* pre, int dj) {
  // dj: column (within these 32) of this row's diagonal element, if any (Gram shift)
  // pre != nullptr: the operand half was read into packed bf16 pairs before
  // any result of this chunk was written (mixed layouts, see caller)
  const bool tr_in = kEdge && cfg.ein_tr;
  const bool tr_out = kEdge && cfg.eout_tr;
#pragma unroll
  for (int qq = 0; qq < 2; ++qq) {           // 16 columns at a time (register pressure)
    float* wq = w + 16 * qq;
    if (cfg.mode == kModeUpdate && !cfg.has_ein) {
      // generic product of Alg. 4 with no epilogue operand: the result is acc
      if (kEdge && cfg.scaled) {
#pragma unroll
        for (int j = 0; j < 16; ++j) wq[j] = __fmul_rn(wq[j], inv);
      }
    } else if (cfg.mode != kModeGram) {
      float o[16];
      if (kEdge && pre != nullptr) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pre[qq * 8 + j]));
          o[2 * j] = f.x;
          o[2 * j + 1] = f.y;
        }
      } else if (!tr_in) {
#pragma unroll
        for (int v = 0; v < 2; ++v)
          bf16x8_to_f32(*reinterpret_cast<const uint4*>(slot + sw128_off(lane, half32 * 4 + qq * 2 + v)), o + 8 * v);
      } else {
        const __nv_bfloat16* sp = reinterpret_cast<const __nv_bfloat16*>(slot) + lane;
#pragma unroll
        for (int j = 0; j < 16; ++j) o[j] = __bfloat162float(sp[(half32 * 32 + qq * 16 + j) * 32]);
      }
      if (cfg.mode == kModePoly) {
#pragma unroll
        for (int j = 0; j < 16; ++j) wq[j] = __fadd_rn(__fmul_rn(cfg.b, o[j]), __fmul_rn(cfg.c, wq[j]));
      } else {
        if (cfg.lin) {
#pragma unroll
          for (int j = 0; j < 16; ++j) wq[j] = __fadd_rn(__fmul_rn(cfg.a, o[j]), __fmul_rn(cfg.b, wq[j]));
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) wq[j] = __fadd_rn(__fmul_rn(cfg.a, o[j]), wq[j]);
        }
        if (kEdge && cfg.scaled) {
#pragma unroll
          for (int j = 0; j < 16; ++j) wq[j] = __fmul_rn(wq[j], inv);
        }
      }
    } else {
      if (kEdge && cfg.scaled) {
        const float inv2 = __fmul_rn(inv, inv);
#pragma unroll
        for (int j = 0; j < 16; ++j) wq[j] = __fmul_rn(wq[j], inv2);
      }
      if (cfg.shift != 0.f) {            // Alg. 4: Y = X X^T + shift I
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (16 * qq + j == dj) wq[j] = __fadd_rn(wq[j], cfg.shift);
      }
    }
    if (kEdge && cfg.muon) {
      // Muon: the slot holds the weight chunk; W <- bf16(W - lr * bf16(X'))
      if (!tr_out) {
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          uint4* up = reinterpret_cast<uint4*>(slot + sw128_off(lane, half32 * 4 + qq * 2 + v));
          float wo[8];
          bf16x8_to_f32(*up, wo);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            wo[j] = __fsub_rn(wo[j], __fmul_rn(g.lr, __bfloat162float(__float2bfloat16_rn(wq[8 * v + j]))));
          *up = pack8_bf16(wo);
        }
      } else {
        __nv_bfloat16* sp = reinterpret_cast<__nv_bfloat16*>(slot) + lane;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          __nv_bfloat16* e = sp + (half32 * 32 + qq * 16 + j) * 32;
          *e = __float2bfloat16_rn(
              __fsub_rn(__bfloat162float(*e), __fmul_rn(g.lr, __bfloat162float(__float2bfloat16_rn(wq[j])))));
        }
      }
    } else if (!tr_out) {
#pragma unroll
      for (int v = 0; v < 2; ++v)
        *reinterpret_cast<uint4*>(slot + sw128_off(lane, half32 * 4 + qq * 2 + v)) = pack8_bf16(wq + 8 * v);
    } else {
      __nv_bfloat16* sp = reinterpret_cast<__nv_bfloat16*>(slot) + lane;
#pragma unroll
      for (int j = 0; j < 16; ++j) sp[(half32 * 32 + qq * 16 + j) * 32] = __float2bfloat16_rn(wq[j]);
    }
  }
}

// Operand half (32 values of row `lane`) of a chunk, packed as bf16 pairs.
template <bool kTr>
__device__ __forceinline__ void read_operand_half(const uint8_t* slot, int lane, int half32, uint32_t* pre) {
  if (!kTr) {
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const uint4 u = *reinterpret_cast<const uint4*>(slot + sw128_off(lane, half32 * 4 + v));
      pre[4 * v] = u.x; pre[4 * v + 1] = u.y; pre[4 * v + 2] = u.z; pre[4 * v + 3] = u.w;
    }
  } else {
    const uint16_t* sp = reinterpret_cast<const uint16_t*>(slot) + lane;
#pragma unroll
    for (int j = 0; j < 16; ++j)
      pre[j] = (uint32_t)sp[(half32 * 32 + 2 * j) * 32] | ((uint32_t)sp[(half32 * 32 + 2 * j + 1) * 32] << 16);
  }
}

// ---------------------------------------------------------------- fp32 (kP = 3)
// The big (0,0) plane chain of a tile is cut into passes of at most 16 K
// blocks; within a pass it is split over the two TMEM buffers, and the
// epilogue carries the fp32 running sum of the passes in a per-CTA global
// scratch tile.  Every truncating accumulator chain is <= 8 K blocks (32
// MMA steps) long whatever K is.
__host__ __device__ constexpr int p3_passes(int nk) { return nk > 16 ? (nk + 15) / 16 : 1; }
// Split v into three bf16 planes: v - p0 and (v - p0) - p1 are exact in fp32
// (Sterbenz), so p0 + p1 + p2 carries v's 24 significand bits.
__device__ __forceinline__ void split3(float v, float& p0, float& p1, float& p2) {
  p0 = __bfloat162float(__float2bfloat16_rn(v));
  const float r1 = __fsub_rn(v, p0);
  p1 = __bfloat162float(__float2bfloat16_rn(r1));
  p2 = __fsub_rn(r1, p1);
}

// Epilogue arithmetic of one half (32 columns) of a 32-row x 64-column chunk
// whose three planes sit in slots[0..2] (128B-swizzled 4 KB each): the operand
// (poly: A, update: X) is p0 + p1 + p2, the fp32 result is split back into
// the three slots in place.
__device__ __forceinline__ void epilogue_math_p3(const TileCfg& cfg, uint8_t* slots, int lane, int half32, float* w) {
#pragma unroll
  for (int qq = 0; qq < 2; ++qq) {
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      float* wv = w + 16 * qq + 8 * v;
      const uint32_t off = sw128_off(lane, half32 * 4 + qq * 2 + v);
      if (cfg.mode != kModeGram) {
        float o0[8], o1[8], o2[8];
        bf16x8_to_f32(*reinterpret_cast<const uint4*>(slots + off), o0);
        bf16x8_to_f32(*reinterpret_cast<const uint4*>(slots + kEpiSlotBytes + off), o1);
        bf16x8_to_f32(*reinterpret_cast<const uint4*>(slots + 2 * kEpiSlotBytes + off), o2);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float o = __fadd_rn(__fadd_rn(o0[j], o1[j]), o2[j]);
          wv[j] = (cfg.mode == kModePoly) ? __fadd_rn(__fmul_rn(cfg.b, o), __fmul_rn(cfg.c, wv[j]))
                  : cfg.lin ? __fadd_rn(__fmul_rn(cfg.a, o), __fmul_rn(cfg.b, wv[j]))
                            : __fadd_rn(__fmul_rn(cfg.a, o), wv[j]);
        }
      }
      float p0[8], p1[8], p2[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) split3(wv[j], p0[j], p1[j], p2[j]);
      *reinterpret_cast<uint4*>(slots + off) = pack8_bf16(p0);
      *reinterpret_cast<uint4*>(slots + kEpiSlotBytes + off) = pack8_bf16(p1);
      *reinterpret_cast<uint4*>(slots + 2 * kEpiSlotBytes + off) = pack8_bf16(p2);
    }
  }
}

// Epilogue role of the fp32 instantiation: chunk by chunk (three 4 KB plane
// slots per warp): operand planes in by TMA, fp32 arithmetic, result planes
// out by TMA.  The main loop is 6x longer than the bf16 one, so the
// per-chunk load latency stays hidden behind the next tile's MMAs.
__device__ __forceinline__ void epilogue_role_p3(const GemmArgs& args, uint8_t* slots, uint64_t* xbar,
                                                uint64_t* tfull, uint32_t tempty_leader0, uint32_t tmem_base,
                                                int warp, int lane, uint32_t rank, int cid, int ncl) {
  const int ew = warp - 2;
  const int q = warp & 3;
  const int half = ew >> 2;
  const int row_off = (int)rank * (kBM / 2) + q * 32;
  // per-CTA fp32 running sum of the passes, [64 column quads][128 rows][4]:
  // a warp's 32 rows of one column quad are 512 contiguous bytes
  float4* scr = reinterpret_cast<float4*>(args.scratch) + (size_t)blockIdx.x * (kBM / 2) * (kBN / 4);
  const int srow = q * 32 + lane;
  uint32_t acc_phase = 0, xphase = 0;
  for (int t = cid; t < args.ntiles; t += ncl) {
    const Tile tl = args.tiles[t];
    const MatDev md = args.mats[tl.mat];
    const TileCfg cfg = tile_cfg<false, 3>(args, tl, rank);
    const int mode = cfg.mode;
    const bool need_load = (mode != kModeGram);
    if (lane == 0 && need_load && cfg.dep != nullptr) acquire_counter(cfg.dep, cfg.dep_need);
    const int r0 = tl.tm * kBM + row_off;
    const uint32_t t_row = tmem_base + ((uint32_t)(q * 32) << 16) + half * (kBN / 2);
    const int ncols = cfg.ncols;
    const int npass = p3_passes(cfg.nk);
    for (int ps = 0; ps < npass; ++ps) {
      // accumulator of the pass = buffer 0 (+ buffer 1 when the pass's big
      // chain has >= 2 K blocks), plus the running sum of earlier passes
      const int k_lo = ps * cfg.nk / npass, k_hi = (ps + 1) * cfg.nk / npass;
      const bool b1 = (k_hi - k_lo) >= 2;
      const bool last = (ps == npass - 1);
      mbar_wait(&tfull[0], acc_phase);
      tc_fence_after();
#pragma unroll 1
      for (int k = 0; k < kEpiChunks; ++k) {
        const int c0 = tl.tn * kBN + half * (kBN / 2) + k * kEpiCols;
        if (c0 >= ncols) break;                                   // warp-uniform
        if (last) {
          if (lane == 0) {
            bulk_wait_read<0>();                                  // previous chunk's stores left the slots
            if (need_load) {
              mbar_arrive_expect_tx(xbar, 3 * kEpiSlotBytes);
#pragma unroll
              for (int p = 0; p < 3; ++p) tma_load_2d(slots + p * kEpiSlotBytes, cfg.ein + p, xbar, c0, r0);
            }
          }
          __syncwarp();
          if (need_load) {
            mbar_wait(xbar, xphase);
            xphase ^= 1;
          }
        }
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
          if (c0 + 32 * h >= ncols) break;
          float w[32];
          tmem_ld32(t_row + k * kEpiCols + 32 * h, w);
          if (b1) {
            float w2[32];
            tmem_ld32(t_row + kBN + k * kEpiCols + 32 * h, w2);
#pragma unroll
            for (int j = 0; j < 32; ++j) w[j] = __fadd_rn(w[j], w2[j]);
          }
          float4* sp = scr + (size_t)((half * (kBN / 2) + k * kEpiCols + 32 * h) >> 2) * (kBM / 2) + srow;
          if (ps > 0) {
#pragma unroll
            for (int v = 0; v < 8; ++v) {
              const float4 o = sp[v * (kBM / 2)];
              w[4 * v] = __fadd_rn(w[4 * v], o.x);
              w[4 * v + 1] = __fadd_rn(w[4 * v + 1], o.y);
              w[4 * v + 2] = __fadd_rn(w[4 * v + 2], o.z);
              w[4 * v + 3] = __fadd_rn(w[4 * v + 3], o.w);
            }
          }
          if (!last) {
#pragma unroll
            for (int v = 0; v < 8; ++v) sp[v * (kBM / 2)] = make_float4(w[4 * v], w[4 * v + 1], w[4 * v + 2], w[4 * v + 3]);
          } else {
            epilogue_math_p3(cfg, slots, lane, h, w);
          }
        }
        if (last) {
          fence_async_smem();
          __syncwarp();
          if (lane == 0) {
#pragma unroll
            for (int p = 0; p < 3; ++p) tma_store_2d(cfg.eout + p, slots + p * kEpiSlotBytes, c0, r0);
            bulk_commit();
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(tempty_leader0);
      acc_phase ^= 1;
    }
    if (lane == 0 && cfg.pub != nullptr) publish_stores(cfg.pub);
  }
  if (lane == 0) bulk_wait<0>();
}

// kSt: smem pipeline stages; kSl: 4 KB epilogue slots per warp (2 = one per
// chunk, whole-tile operand prefetch; 1 = a single staging slot: the Gram has
// no epilogue operand, poly/update load chunk 1's operand once chunk 0's
// result has left the slot -- the freed 32 KB buy a sixth ring stage; 3 = the
// three plane slots of the fp32 instantiation); kEdge: first/last-iteration
// specialisation; kP: planes per buffer (1 = bf16, 3 = fp32, see top).
template <int kSt, int kSl, bool kEdge, int kP = 1>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kGemmThreads, 1) pe_gemm_sm100(const GemmArgs args) {
  static_assert(kP == 1 || (kP == 3 && kSl == 3 && !kEdge), "fp32 planes: three slots, no folding");
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
  uint8_t* epi_smem = smem + kSt * kStageBytes + kBarrierBytes;   // kEpiWarps x kSl x 4 KB

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = (rank == 0);
  const int cid = blockIdx.x >> 1;
  const int ncl = gridDim.x >> 1;
  long long st_wait_tempty = 0, st_wait_full = 0, st_wait_tfull = 0, st_lat = 0, st_nstage = 0;
  __shared__ long long st_issue[8];     // debug: producer issue time per stage (leader CTA)
  const long long st_begin = clock64();
  // PE_DEBUG_GEMM bit 128: per-CTA %globaltimer timeline of the launch in the
  // stats slots (0 entry, 1 after the PDL wait, 2 first operand stage landed,
  // 3 last MMA committed, 4 last result store issued, 5 stores complete, 6 exit,
  // 7 the last tile's accumulator ready in the epilogue)
  const bool tl_on = kGemmTimeline && (args.dbg & 128) && args.stats != nullptr;
  long long* tl_st = tl_on ? args.stats + blockIdx.x * 8 : nullptr;
  // (bit 128, CTAs 0..63 of a phase-per-launch call: clock64 of the last tile's epilogue steps
  // of warp 2 at stats + 6144 + 512 mode + 8 blockIdx: 0 accumulator ready, 1 first TMEM load,
  // 2 first half computed, 3 chunk 0 computed, 4 its store issued, 5 chunk 1's slot free,
  // 6 chunk 1 computed, 7 the tile's stores have left smem)
  long long* tl_ep = (tl_on && blockIdx.x < 64 && args.nphase == 0)
                         ? args.stats + (6144 - 2048 * args.mode) + 512 * args.mode + blockIdx.x * 8 : nullptr;
  if (tl_on && threadIdx.x == 0) tl_st[0] = (long long)gtimer();

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
  // Everything above overlaps the previous kernel's tail (programmatic
  // dependent launch); nothing below may touch its outputs before this.
  pdl_trigger();
  pdl_wait();
  if (tl_on && threadIdx.x == 0) tl_st[1] = (long long)gtimer();

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (elect_one()) {
      const uint32_t full_leader0 = mapa_shared(smem_u32(&full[0]), 0);
      const uint64_t pol_keep = l2_policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      TileCfg nxt;
      if (cid < args.ntiles) nxt = tile_cfg<kEdge, kP>(args, args.tiles[cid], rank);
      for (int t = cid; t < args.ntiles; t += ncl) {
        const TileCfg o = nxt;
        if (t + ncl < args.ntiles) nxt = tile_cfg<kEdge, kP>(args, args.tiles[t + ncl], rank);   // off the critical path
        if (o.dep != nullptr) acquire_counter(o.dep, o.dep_need);    // fused: operands are complete
        // kP = 3: six plane-pair segments (i, j), small terms first:
        // (2,0) (1,1) (0,2) (1,0) (0,1) (0,0).  The tensor core adds each
        // K=16 step into the fp32 accumulator with truncation; with the big
        // (0,0) chain last, the small terms are never truncated against the
        // big accumulator (256x1024: relF 2.0e-5 big-first, 2.4e-6 now).
        // (kP = 3: the small segments run in pass 0 over all of K, the big
        // (0,0) segment pass by pass, see p3_passes)
        const int npass = (kP == 3) ? p3_passes(o.nk) : 1;
        for (int ps = 0; ps < npass; ++ps)
        for (int sg = (kP == 3 && ps > 0) ? 5 : 0; sg < (kP == 3 ? 6 : 1); ++sg) {
        const int pa = (kP == 3) ? ((0x001012 >> (4 * sg)) & 0xF) * o.prow : 0;
        const int pb = (kP == 3) ? ((0x010210 >> (4 * sg)) & 0xF) * o.prow : 0;
        const bool bigseg = (kP == 1) || sg == 5;
        const int kb_lo = bigseg ? ps * o.nk / npass : 0;
        const int kb_hi = bigseg ? (ps + 1) * o.nk / npass : o.nk;
        for (int kb = kb_lo; kb < kb_hi; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          const bool skip_b = o.diag || (args.dbg & 2048);    // dbg 2048: B operand not loaded (timing only)
          if (leader) mbar_arrive_expect_tx(&full[stage], skip_b ? 2 * kABytes : 2 * kStageBytes);
          if (args.stats != nullptr && leader) st_issue[stage] = clock64();
          const uint32_t bar = full_leader0 + stage * sizeof(uint64_t);
          uint8_t* a_dst = sA + stage * kABytes;
          uint8_t* b_dst = sB + stage * kBBytes;
          const int k0 = (args.dbg & 8) ? 0 : kb * kBK;   // dbg 8: every load hits the same (L2-resident) boxes
          // the update's left operand (B = b A + c A^2) is re-read by every
          // column panel of X: keep it in L2 (evict_last); X streams through
          const bool keep_a = kP == 1 && o.mode == kModeUpdate && !(args.dbg & 16384);
          if (o.a_wide && (kb >> 2) < o.pan_a) {                    // block below the diagonal
            if (keep_a) {
              tma_load_2d_pair_hint(a_dst, o.Amn, bar, o.row_a, k0 + pa, pol_keep);
              tma_load_2d_pair_hint(a_dst + kBoxBytes, o.Amn, bar, o.row_a + 64, k0 + pa, pol_keep);
            } else {
              tma_load_2d_pair(a_dst, o.Amn, bar, o.row_a, k0 + pa);
              tma_load_2d_pair(a_dst + kBoxBytes, o.Amn, bar, o.row_a + 64, k0 + pa);
            }
          } else if (o.a_wide) {
            if (keep_a) tma_load_2d_pair_hint(a_dst, o.A, bar, k0, o.row_a + pa, pol_keep);
            else tma_load_2d_pair(a_dst, o.A, bar, k0, o.row_a + pa);      // one 64 x 128 box
          } else if (!o.a_mn) {
            tma_load_2d_pair(a_dst, o.A, bar, k0, o.row_a + pa);
            tma_load_2d_pair(a_dst + kBoxBytes, o.A, bar, k0, o.row_a + pa + 64);
          } else {
            tma_load_2d_pair(a_dst, o.A, bar, o.row_a, k0);
            tma_load_2d_pair(a_dst + kBoxBytes, o.A, bar, o.row_a + 64, k0);
          }
          if (!skip_b) {          // diagonal tiles: the right operand is the left one
            if (o.b_wide && ((kb >> 2) < o.pan_b || (o.rr && (kb >> 2) == o.pan_b))) {
              tma_load_2d_pair(b_dst, o.Bmn, bar, o.col_b, k0 + pb);
              tma_load_2d_pair(b_dst + kBoxBytes, o.Bmn, bar, o.col_b + 64, k0 + pb);
            } else if (o.b_wide) {
              tma_load_2d_pair(b_dst, o.B, bar, k0, o.col_b + pb);
            } else if (!o.b_mn) {
              tma_load_2d_pair(b_dst, o.B, bar, k0, o.col_b + pb);
              tma_load_2d_pair(b_dst + kBoxBytes, o.B, bar, k0, o.col_b + pb + 64);
            } else {
              tma_load_2d_pair(b_dst, o.B, bar, o.col_b, k0 + pb);
              tma_load_2d_pair(b_dst + kBoxBytes, o.B, bar, o.col_b + 64, k0 + pb);
            }
          }
          if (++stage == kSt) { stage = 0; phase ^= 1; }
        }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader CTA)
    if (leader) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      TileCfg nxt;
      if (cid < args.ntiles) nxt = tile_cfg<kEdge, kP>(args, args.tiles[cid], rank);
      for (int t = cid; t < args.ntiles; t += ncl) {
        const TileCfg o = nxt;
        if (t + ncl < args.ntiles) nxt = tile_cfg<kEdge, kP>(args, args.tiles[t + ncl], rank);
        const int npass = (kP == 3) ? p3_passes(o.nk) : 1;
        for (int ps = 0; ps < npass; ++ps) {
        long long t0 = clock64();
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        st_wait_tempty += clock64() - t0;
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kBN;
        // kP = 3: pass ps = [small segments over all K (pass 0 only)] + the
        // big chain over K blocks [k_lo, k_hi): its first half continues in
        // buffer 0, the second half starts buffer 1 (one tile in flight).
        const int k_lo = ps * o.nk / npass, k_hi = (ps + 1) * o.nk / npass;
        const int n_small = (kP == 3 && ps == 0) ? 5 * o.nk : 0;
        const int n_first = (kP == 3) ? n_small + (k_hi - k_lo + 1) / 2 : o.nk;
        const int nst = n_small + (k_hi - k_lo);
        int kin = (n_small > 0) ? 0 : k_lo;   // K block index within the current segment
        for (int kb = 0; kb < nst; ++kb) {
          if (kb == n_small) kin = k_lo;
          // per k-block operand layout: blocks of a symmetric buffer below
          // the diagonal arrive transposed (MN-major)
          const bool amn = o.a_mn || (o.a_wide && (kin >> 2) < o.pan_a);
          const bool bmn = o.b_mn || (o.b_wide && ((kin >> 2) < o.pan_b || (o.rr && (kin >> 2) == o.pan_b)));
          const uint32_t idesc = idesc_bf16(kBM, kBN, amn, bmn);
          if (++kin == o.nk && kb < n_small) kin = 0;
          long long t1 = clock64();
          mbar_wait(&full[stage], phase);
          const long long t1e = clock64();
          if (tl_on && t == cid && kb == 0 && lane == 0) tl_st[2] = (long long)gtimer();
          st_wait_full += t1e - t1;
          if (args.stats != nullptr) { st_lat += t1e - *(volatile long long*)&st_issue[stage]; ++st_nstage; }
          tc_fence_after();
          if (elect_one()) {
            const uint32_t a_addr = smem_u32(sA + stage * kABytes);
            const uint32_t b_addr = o.diag ? a_addr : smem_u32(sB + stage * kBBytes);
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) {
              // K-major: advance 32 bytes inside the 128B swizzle row;
              // MN-major: advance 16 K-rows (2 KB); LBO = 8 KB between the
              // two 64-element MN atoms of a 128-wide operand.
              const uint64_t adesc = amn ? smem_desc_sw128(a_addr + k * 2048, kBoxBytes, 1024)
                                         : smem_desc_sw128(a_addr + k * 32, 16, 1024);
              const uint64_t bdesc = bmn ? smem_desc_sw128(b_addr + k * 2048, kBoxBytes, 1024)
                                         : smem_desc_sw128(b_addr + k * 32, 16, 1024);
              if (kP == 3 && kb >= n_first)
                umma_bf16_pair(tmem_base + kBN, adesc, bdesc, idesc, (kb != n_first) || k != 0);
              else
                umma_bf16_pair(d_tmem, adesc, bdesc, idesc, (kb | k) != 0);
            }
            umma_commit_pair(&empty[stage], 0x3);
          }
          __syncwarp();
          if (++stage == kSt) { stage = 0; phase ^= 1; }
        }
        if (elect_one()) umma_commit_pair(&tfull[acc], 0x3);
        __syncwarp();
        if (tl_on && lane == 0) tl_st[3] = (long long)gtimer();
        if (kP == 3) {
          acc_phase ^= 1;          // both buffers belong to one pass
        } else {
          acc ^= 1;
          if (acc == 0) acc_phase ^= 1;
        }
        }
      }
    }
  } else if (kP == 3) {
    epilogue_role_p3(args, epi_smem + (warp - 2) * kSl * kEpiSlotBytes, xbars + (warp - 2) * kSl, tfull,
                     mapa_shared(smem_u32(&tempty[0]), 0), tmem_base, warp, lane, rank, cid, ncl);
  } else {
    // ------------------------------------------------------------ epilogue
    // Warp ew owns TMEM lane quadrant q (its 32 output rows) and column half
    // `half` (128 columns) of the CTA's 128 x 256 accumulator: two 32 x 64
    // chunks, each staged in a 4 KB smem slot (128B-swizzled, so the
    // row-per-thread accesses are conflict-free).  The whole tile's operand
    // chunks (A for poly, X for update) are loaded by TMA while the tile's MMA
    // runs; results leave by TMA store.
    const int ew = warp - 2;
    const int q = warp & 3;
    const int half = ew >> 2;
    uint8_t* slots = epi_smem + ew * kSl * kEpiSlotBytes;
    uint64_t* xbar = xbars + ew * kSl;
    auto needs_load = [&](const TileCfg& c2) { return c2.has_ein && !(args.dbg & 3); };
    const bool do_work = !(args.dbg & 1);
    const uint32_t tempty_leader0 = mapa_shared(smem_u32(&tempty[0]), 0);
    const int row_off = (int)rank * (kBM / 2) + q * 32;

    auto col0 = [&](const Tile& tl2, int kk) { return tl2.tn * kBN + half * (kBN / 2) + kk * kEpiCols; };
    auto ncols_of = [&](const Tile&, const TileCfg& c2) { return c2.ncols; };
    auto issue_tile = [&](const Tile& tl2, const TileCfg& c2, int nc) {
      if (c2.dep != nullptr) acquire_counter(c2.dep, c2.dep_need);   // fused: the operand is complete
      const int r0 = tl2.tm * kBM + row_off;
      for (int kk = 0; kk < (kSl == 1 ? 1 : kEpiChunks) && col0(tl2, kk) < nc; ++kk) {
        const int c0 = col0(tl2, kk);
        mbar_arrive_expect_tx(&xbar[kk], kEpiSlotBytes);
        if (!(kEdge && c2.ein_tr)) tma_load_2d(slots + kk * kEpiSlotBytes, c2.ein, &xbar[kk], c0, r0);
        else tma_load_2d(slots + kk * kEpiSlotBytes, c2.ein, &xbar[kk], r0, c0);
      }
    };

    int acc = 0;
    uint32_t acc_phase = 0;
    uint32_t phase_bits = 0;
    Tile ntl{};
    TileCfg ncfg{};
    int nnc = 0;
    if (cid < args.ntiles) {
      ntl = args.tiles[cid];
      ncfg = tile_cfg<kEdge>(args, ntl, rank);
      nnc = ncols_of(ntl, ncfg);
      if (lane == 0 && needs_load(ncfg)) issue_tile(ntl, ncfg, nnc);
    }
    for (int t = cid; t < args.ntiles; t += ncl) {
      const Tile tl = ntl;
      const MatDev md = args.mats[tl.mat];
      const TileCfg cfg = ncfg;
      const bool has_next = t + ncl < args.ntiles;
      if (has_next) {                        // next tile's description, loaded early
        ntl = args.tiles[t + ncl];
        ncfg = tile_cfg<kEdge>(args, ntl, rank);
        nnc = ncols_of(ntl, ncfg);
      }
      const bool need_load = needs_load(cfg);
      const float inv = !cfg.scaled ? 1.0f : cfg.pre ? pow2_residual(args.inv[tl.mat]) : args.inv[tl.mat];
      long long t2 = clock64();
      mbar_wait(&tfull[acc], acc_phase);
      st_wait_tfull += clock64() - t2;
      if (tl_on && ew == 0 && lane == 0) tl_st[7] = (long long)gtimer();
      if (tl_ep != nullptr && ew == 0 && lane == 0) tl_ep[0] = clock64();
      tc_fence_after();
      const int r0 = tl.tm * kBM + row_off;
      const int r = r0 + lane;
      const uint32_t t_row = tmem_base + acc * kBN + ((uint32_t)(q * 32) << 16) + half * (kBN / 2);
      const int ncols = cfg.ncols;
#pragma unroll 1
      for (int k = 0; k < kEpiChunks; ++k) {
        const int c0 = col0(tl, k);
        if (c0 >= ncols || !do_work) break;                  // warp-uniform
        const int xb = (kSl == 1) ? 0 : k;                   // operand barrier / phase bit of this chunk
        uint8_t* slot = slots + (kSl == 1 ? 0 : k) * kEpiSlotBytes;
        const bool tl_rec = tl_ep != nullptr && ew == 0 && lane == 0;
        if (kSl == 1 && need_load && k > 0) {
          // one slot: this chunk's operand is loaded once the previous chunk's
          // result has left the slot
          if (lane == 0) {
            bulk_wait_read<0>();
            mbar_arrive_expect_tx(&xbar[0], kEpiSlotBytes);
            if (!(kEdge && cfg.ein_tr)) tma_load_2d(slot, cfg.ein, &xbar[0], c0, r0);
            else tma_load_2d(slot, cfg.ein, &xbar[0], r0, c0);
          }
          __syncwarp();
        }
        if (need_load) {
          mbar_wait(&xbar[xb], (phase_bits >> xb) & 1u);
          phase_bits ^= 1u << xb;
        }
        if (cfg.mode == kModeGram && args.out32 != nullptr) {
          // sharded call: the partial Gram leaves in fp32 (16-byte stores of
          // this thread's row); the all-reduce and the rounding come later
          float* dst = args.out32[tl.mat] + (size_t)r * md.ldm;
#pragma unroll 1
          for (int h = 0; h < 2; ++h) {
            if (c0 + 32 * h >= ncols) break;
            float w[32];
            tmem_ld32(t_row + k * kEpiCols + 32 * h, w);
            if (r < md.m) {
#pragma unroll
              for (int v = 0; v < 8; ++v) {
                const int col = c0 + 32 * h + 4 * v;
                if (col + 3 < md.m) {
                  *reinterpret_cast<float4*>(dst + col) = make_float4(w[4 * v], w[4 * v + 1], w[4 * v + 2], w[4 * v + 3]);
                } else {
#pragma unroll
                  for (int e = 0; e < 4; ++e)
                    if (col + e < md.m) dst[col + e] = w[4 * v + e];
                }
              }
            }
          }
          if (!args.out32_both) continue;      // App. G: the bf16 A of the same accumulator too
        }
        if (kSl == 1 && k > 0 && !need_load) {
          // single staging slot (Gram: no epilogue operand): the previous
          // chunk's store must have left smem before this chunk is written
          if (lane == 0) bulk_wait_read<0>();
          __syncwarp();
        }
        if (tl_rec && k == 1) tl_ep[5] = clock64();
        if (kEdge && need_load && (cfg.ein_tr != cfg.eout_tr || cfg.muon)) {
          // operand and result layouts differ (tall caller matrix, first or
          // last iteration), or the result updates another chunk (Muon): read
          // the whole operand chunk before the slot is overwritten
          uint32_t pre[2][16];
          if (cfg.ein_tr) { read_operand_half<true>(slot, lane, 0, pre[0]); read_operand_half<true>(slot, lane, 1, pre[1]); }
          else { read_operand_half<false>(slot, lane, 0, pre[0]); read_operand_half<false>(slot, lane, 1, pre[1]); }
          __syncwarp();
          if (cfg.muon) {
            // bring the weight chunk into the slot (same map and box as the store)
            if (lane == 0) {
              fence_async_smem();
              mbar_arrive_expect_tx(&xbar[xb], kEpiSlotBytes);
              if (!cfg.eout_tr) tma_load_2d(slot, cfg.eout, &xbar[xb], c0, r0);
              else tma_load_2d(slot, cfg.eout, &xbar[xb], r0, c0);
            }
            __syncwarp();
            mbar_wait(&xbar[xb], (phase_bits >> xb) & 1u);
            phase_bits ^= 1u << xb;
          }
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (c0 + 32 * h < ncols) {
              float w[32];
              tmem_ld32(t_row + k * kEpiCols + 32 * h, w);
              epilogue_math<kEdge>(args, cfg, inv, slot, lane, h, w, pre[h], r - (c0 + 32 * h));
            }
          }
        } else {
#pragma unroll 1
          for (int h = 0; h < 2; ++h) {
            if (c0 + 32 * h >= ncols) break;
            float w[32];
            if (args.dbg & 16) {
#pragma unroll
              for (int j = 0; j < 32; ++j) w[j] = 0.f;
            } else {
              tmem_ld32(t_row + k * kEpiCols + 32 * h, w);
            }
            if (tl_rec && k == 0 && h == 0) tl_ep[1] = clock64();
            epilogue_math<kEdge>(args, cfg, inv, slot, lane, h, w, nullptr, r - (c0 + 32 * h));
            if (tl_rec && k == 0 && h == 0) tl_ep[2] = clock64();
          }
        }
        if (tl_rec) tl_ep[k == 0 ? 3 : 6] = clock64();
        {                                       // each chunk leaves as soon as it is done
                                                // (measured: 2-4 % faster than one burst per tile)
          fence_async_smem();
          __syncwarp();
          if (lane == 0 && !(args.dbg & 32)) {
            if (cfg.mode == kModeUpdate && !(args.dbg & 16384)) {
              // X' is not read again in this launch: first out of L2
              const uint64_t pol = l2_policy_evict_first();
              if (!(kEdge && cfg.eout_tr)) tma_store_2d_hint(cfg.eout, slot, c0, r0, pol);
              else tma_store_2d_hint(cfg.eout, slot, r0, c0, pol);
            } else if (!(kEdge && cfg.eout_tr)) {
              tma_store_2d(cfg.eout, slot, c0, r0);
            } else {
              tma_store_2d(cfg.eout, slot, r0, c0);
            }
            bulk_commit();
          }
        }
        if (tl_rec && k == 0) tl_ep[4] = clock64();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive_remote(tempty_leader0 + acc * sizeof(uint64_t));
        if (cfg.pub != nullptr) publish_stores(cfg.pub);   // fused: stores complete, counted
        else bulk_wait_read<0>();     // this tile's stores have left smem: slots are free
        if (tl_ep != nullptr && ew == 0) tl_ep[7] = clock64();
        if (has_next && needs_load(ncfg)) issue_tile(ntl, ncfg, nnc);
      }
      __syncwarp();
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
    if (tl_on && ew == 0 && lane == 0) tl_st[4] = (long long)gtimer();
    if (lane == 0) bulk_wait<0>();
    if (tl_on && ew == 0 && lane == 0) tl_st[5] = (long long)gtimer();
  }

  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == 1) tmem_dealloc_pair(tmem_base, kTmemCols);
  if (tl_on) {
    if (threadIdx.x == 0) tl_st[6] = (long long)gtimer();
  } else if (args.stats != nullptr && lane == 0 && (warp == 1 || warp == 2)) {
    long long* st = args.stats + blockIdx.x * 8;
    if (warp == 1) {
      st[0] = clock64() - st_begin; st[1] = st_wait_tempty; st[2] = st_wait_full;
      st[4] = st_lat; st[5] = st_nstage;
    }
    else { st[3] = st_wait_tfull; }
  }
}

template <int kSt, int kSl> constexpr size_t gemm_smem_bytes() {
  return 1024 + (size_t)kSt * kStageBytes + kBarrierBytes + (size_t)kEpiWarps * kSl * kEpiSlotBytes;
}

}  // namespace pe
