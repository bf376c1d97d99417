// Shared-memory tile layout and tcgen05 GEMM issue helpers (sm_100a).
//
// Tile layout ("SW128 tile"): a bf16 matrix stored as [rows][cols] with cols
// split into 64-element (128-B) column blocks; block b lives at
// b * rows * 128 B, row r of a block at r * 128 B, and its 16-B chunk c at
// chunk position (c ^ (r & 7)).  This is exactly what a TMA load with
// CU_TENSOR_MAP_SWIZZLE_128B and a 64-column box writes into a 1024-B
// aligned buffer, and what UMMA's SWIZZLE_128B descriptors read.  The same
// stored tile is a K-major operand (rows = M or N, cols = K) or an MN-major
// operand (rows = K, cols = M or N) -- no transposed copies are needed.
#pragma once
#include "ptx.cuh"

namespace dash {

// Byte offset of the 16-B chunk holding columns [8*chunk, 8*chunk+8) of row r.
__device__ __forceinline__ uint32_t sw128_chunk_offset(int rows, int r, int chunk) {
  const int blk = chunk >> 3, c = chunk & 7;
  return static_cast<uint32_t>(blk * rows * 128 + r * 128 + ((c ^ (r & 7)) << 4));
}

// Issue D(tmem)[M x N] (+)= A[M x K] * B[K x N] as K/16 tcgen05.mma ops.
//   A_MN = false: A stored K-major as an SW128 tile [a_rows = M][K].
//   A_MN = true : A stored MN-major as an SW128 tile [a_rows = K][M].
//   B_MN = false: B stored K-major as [b_rows = N][K]   (i.e. B^T row-major).
//   B_MN = true : B stored MN-major as [b_rows = K][N].
// Must be called by a single thread.
template <int M, int N, int K, bool A_MN, bool B_MN>
__device__ __forceinline__ void umma_gemm(uint32_t d_tmem, uint32_t a_base, int a_rows,
                                          uint32_t b_base, int b_rows, bool accumulate) {
  constexpr uint32_t idesc = ptx::idesc_bf16(M, N, A_MN ? 1 : 0, B_MN ? 1 : 0);
  static_assert(M == 128, "this kernel family uses M = 128 (one TMEM lane per row)");
  static_assert(N % 16 == 0 && N >= 16 && N <= 256, "invalid UMMA N");
  static_assert(K % 16 == 0, "invalid UMMA K");
#pragma unroll
  for (int kk = 0; kk < K / 16; ++kk) {
    uint64_t a, b;
    if (A_MN) {
      a = ptx::sdesc_sw128(a_base + kk * 2048, a_rows * 128, 1024);
    } else {
      a = ptx::sdesc_sw128(a_base + (kk >> 2) * (a_rows * 128) + (kk & 3) * 32, 16, 1024);
    }
    if (B_MN) {
      b = ptx::sdesc_sw128(b_base + kk * 2048, b_rows * 128, 1024);
    } else {
      b = ptx::sdesc_sw128(b_base + (kk >> 2) * (b_rows * 128) + (kk & 3) * 32, 16, 1024);
    }
    ptx::mma_bf16(d_tmem, a, b, idesc, (accumulate || kk > 0) ? 1u : 0u);
  }
}

}  // namespace dash
