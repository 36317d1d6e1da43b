// Device-side data layout shared by the host planner (pe_api.cu) and the
// kernels.  All matrices are held in the "wide" orientation m <= n.
#pragma once
#include <cstdint>

namespace pe {

// bf16 tensor-core path: one 256x256 output tile per CTA pair (cta_group::2)
constexpr int kBM = 256;        // UMMA M of the pair (128 rows per CTA = TMEM lanes)
constexpr int kBN = 256;        // UMMA N (each CTA stages 128 of the right operand)
constexpr int kBK = 64;         // K per pipeline stage (one 128-byte swizzle row of bf16)
constexpr int kBoxBytes = 64 * 64 * 2;                 // one TMA box (64 x 64 bf16)
constexpr int kABytes = (kBM / 2) * kBK * 2;           // 16 KB per CTA
constexpr int kBBytes = (kBN / 2) * kBK * 2;           // 16 KB per CTA
constexpr int kStageBytes = kABytes + kBBytes;         // 32 KB per CTA
constexpr int kEpiWarps = 8;                           // 4 lane quadrants x 2 column halves
constexpr int kGemmThreads = 64 + 32 * kEpiWarps;      // TMA warp, MMA warp, epilogue warps
constexpr int kTmemCols = 512;                         // 2 x 256-column fp32 accumulators
constexpr int kEpiCols = 64;                           // epilogue chunk: 32 rows x 64 columns (128B rows)
constexpr int kEpiChunks = (kBN / 2) / kEpiCols;       // chunks (= smem slots) per warp per tile
constexpr int kEpiSlotBytes = 32 * kEpiCols * 2;       // 4 KB
constexpr int kBarrierBytes = 1024;                    // mbarriers + TMEM slot (rounded up)

constexpr int kModeGram = 0;    // A   = X X^T
constexpr int kModePoly = 1;    // B   = b A + c A A^T    (A symmetric)
constexpr int kModeUpdate = 2;  // X'  = a X + B X

// Per-matrix descriptor (device-resident, built by the planner).
struct MatDev {
  int m, n;          // oriented dims, m <= n
  int ldx, ldm;      // leading dims (elements) of the m x n and m x m buffers
  void* X[2];        // ping-pong iterates (m x n)
  void* A;           // Gram (m x m, symmetric)
  void* B;           // b A + c A^2 (m x m, symmetric)
  int rows, cols;    // caller's shape
  int tall;          // rows > cols: caller matrix is X^T
  int pad;
  void* E[4];        // fast rectangular iteration (App. H, Alg. 4) plans: Q_0, Q_1 (ping-pong Q,
                     // full m x m), T = Y Q (full), R = Q^T Y Q (symmetric); else nullptr
};

// One output tile of a GEMM phase (units: kBM rows, kBN columns).
struct Tile {
  int mat, tm, tn, pad;
};


}  // namespace pe
