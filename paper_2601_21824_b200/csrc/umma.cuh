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

// Shared-memory descriptor of an SW128 tile (no k offset).  K-major operands
// use LBO = 16 B (ignored) and SBO = 1024 B (8-row groups); MN-major operands
// use LBO = the 64-column block stride (rows * 128 B) and SBO = 1024 B.
template <bool MN>
__device__ __forceinline__ uint64_t tile_desc(uint32_t saddr, int rows) {
  return MN ? ptx::sdesc_sw128(saddr, rows * 128, 1024) : ptx::sdesc_sw128(saddr, 16, 1024);
}
// Descriptor increment (in the 16-B address units of the start-address field)
// for K step kk of an operand whose base descriptor is tile_desc<MN>(...).
template <bool MN>
__host__ __device__ constexpr uint32_t kstep(int kk, int rows) {
  return MN ? static_cast<uint32_t>(kk * 2048 / 16)
            : static_cast<uint32_t>(((kk >> 2) * rows * 128 + (kk & 3) * 32) / 16);
}

// Issue D(tmem)[M x N] (+)= A[M x K] * B[K x N] as K/16 tcgen05.mma ops.
//   A_MN = false: A stored K-major as an SW128 tile [A_ROWS = M][K].
//   A_MN = true : A stored MN-major as an SW128 tile [A_ROWS = K][M].
//   B_MN = false: B stored K-major as [B_ROWS = N][K]   (i.e. B^T row-major).
//   B_MN = true : B stored MN-major as [B_ROWS = K][N].
// a_desc / b_desc are the tiles' base descriptors (tile_desc); each K step adds
// a compile-time constant, so an MMA costs one add per operand to issue.
// Must be called by a whole converged warp (one elected lane issues).
template <int M, int N, int K, bool A_MN, bool B_MN, int A_ROWS, int B_ROWS>
__device__ __forceinline__ void umma_gemm_d(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                            bool accumulate) {
  constexpr uint32_t idesc = ptx::idesc_bf16(M, N, A_MN ? 1 : 0, B_MN ? 1 : 0);
  static_assert(M == 128, "this kernel family uses M = 128 (one TMEM lane per row)");
  static_assert(N % 16 == 0 && N >= 16 && N <= 256, "invalid UMMA N");
  static_assert(K % 16 == 0, "invalid UMMA K");
#pragma unroll
  for (int kk = 0; kk < K / 16; ++kk) {
    ptx::mma_bf16_e(d_tmem, a_desc + kstep<A_MN>(kk, A_ROWS), b_desc + kstep<B_MN>(kk, B_ROWS),
                    idesc, (accumulate || kk > 0) ? 1u : 0u);
  }
}

// Convenience form taking shared addresses (probe / non-hot paths).
template <int M, int N, int K, bool A_MN, bool B_MN>
__device__ __forceinline__ void umma_gemm(uint32_t d_tmem, uint32_t a_base, int a_rows,
                                          uint32_t b_base, int b_rows, bool accumulate) {
  constexpr uint32_t idesc = ptx::idesc_bf16(M, N, A_MN ? 1 : 0, B_MN ? 1 : 0);
  const uint64_t ad = tile_desc<A_MN>(a_base, a_rows), bd = tile_desc<B_MN>(b_base, b_rows);
#pragma unroll
  for (int kk = 0; kk < K / 16; ++kk) {
    ptx::mma_bf16_e(d_tmem, ad + kstep<A_MN>(kk, a_rows), bd + kstep<B_MN>(kk, b_rows), idesc,
                    (accumulate || kk > 0) ? 1u : 0u);
  }
}

// D(tmem)[128 x N] (+)= A(tmem)[128 x K] * B[K x N]: A in TMEM at column
// a_tmem (row m in lane m, K packed two bf16 per column, so each K = 16 step
// advances 8 columns); B from an SW128 tile given by its base descriptor.
template <int N, int K, bool B_MN, int B_ROWS>
__device__ __forceinline__ void umma_gemm_ts_d(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                               bool accumulate) {
  constexpr uint32_t idesc = ptx::idesc_bf16(128, N, 0, B_MN ? 1 : 0);
  static_assert(N % 16 == 0 && N >= 16 && N <= 256, "invalid UMMA N");
#pragma unroll
  for (int kk = 0; kk < K / 16; ++kk) {
    ptx::mma_bf16_ts_e(d_tmem, a_tmem + kk * 8, b_desc + kstep<B_MN>(kk, B_ROWS), idesc,
                       (accumulate || kk > 0) ? 1u : 0u);
  }
}
template <int N, int K, bool B_MN>
__device__ __forceinline__ void umma_gemm_ts(uint32_t d_tmem, uint32_t a_tmem, uint32_t b_base,
                                             int b_rows, bool accumulate) {
  constexpr uint32_t idesc = ptx::idesc_bf16(128, N, 0, B_MN ? 1 : 0);
  const uint64_t bd = tile_desc<B_MN>(b_base, b_rows);
#pragma unroll
  for (int kk = 0; kk < K / 16; ++kk) {
    ptx::mma_bf16_ts_e(d_tmem, a_tmem + kk * 8, bd + kstep<B_MN>(kk, b_rows), idesc,
                       (accumulate || kk > 0) ? 1u : 0u);
  }
}

}  // namespace dash
