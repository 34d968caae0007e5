// FP64 tile engine for sm_100a: shared-memory staged operands, warp-level DMMA
// (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4).  tcgen05 has no f64 kind on sm_100a,
// so FP64 contractions run on DMMA; this header is the one contraction core used
// by the Cauchy sampling, the dense fallback update and the HSS multiply.
//
// CTA tile BM x BN with BM = WM*MF*8 and BN = WN*NF*8; each warp owns an
// (MF*8) x (NF*8) sub-tile held in registers.  K advances in BK = 16 chunks.
// Shared strides are = 4 (mod 16) doubles so fragment loads are bank-conflict free.
#pragma once
#include "common.cuh"

namespace hsseig {

template <int MF_, int NF_, int WM_, int WN_, int STAGES_ = 3>
struct Tile {
  static constexpr int MF = MF_, NF = NF_, WM = WM_, WN = WN_, STAGES = STAGES_;
  static constexpr int BM = WM * MF * 8;
  static constexpr int BN = WN * NF * 8;
  static constexpr int BK = 16;
  static constexpr int THREADS = WM * WN * 32;
  static constexpr int SA = BK + 4;                       // A: [BM][SA]
  static constexpr int SB = ((BN + 15) / 16) * 16 + 4;    // B: [BK][SB]
  static constexpr int A_ELEMS = BM * SA;
  static constexpr int B_ELEMS = BK * SB;
  static constexpr int STAGE_ELEMS = A_ELEMS + B_ELEMS;
  static constexpr size_t SMEM_BYTES = sizeof(double) * STAGE_ELEMS * STAGES;
};

template <class T>
struct Acc {
  double c[T::MF][T::NF][2];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int i = 0; i < T::MF; ++i)
#pragma unroll
      for (int j = 0; j < T::NF; ++j) c[i][j][0] = c[i][j][1] = 0.0;
  }
};

// One BK chunk of MMAs from staged tiles sA [BM][SA], sB [BK][SB].
template <class T>
__device__ __forceinline__ void mma_chunk(const double* __restrict__ sA,
                                          const double* __restrict__ sB, Acc<T>& acc, int wm,
                                          int wn, int lane) {
  const int gr = lane >> 2, gc = lane & 3;
#pragma unroll
  for (int kk = 0; kk < T::BK; kk += 4) {
    double a[T::MF], b[T::NF];
#pragma unroll
    for (int i = 0; i < T::MF; ++i) a[i] = sA[(wm * T::MF * 8 + i * 8 + gr) * T::SA + kk + gc];
#pragma unroll
    for (int j = 0; j < T::NF; ++j) b[j] = sB[(kk + gc) * T::SB + wn * T::NF * 8 + j * 8 + gr];
#pragma unroll
    for (int i = 0; i < T::MF; ++i)
#pragma unroll
      for (int j = 0; j < T::NF; ++j) dmma_8x8x4(acc.c[i][j][0], acc.c[i][j][1], a[i], b[j]);
  }
}

// Partial chunk: only the first kv (multiple of 4, <= BK) k-columns are live, and only the
// first jmax n-fragments of this warp carry output columns (both warp-uniform).
template <class T>
__device__ __forceinline__ void mma_chunk_part(const double* __restrict__ sA,
                                               const double* __restrict__ sB, Acc<T>& acc, int wm,
                                               int wn, int lane, int kv, int jmax) {
  const int gr = lane >> 2, gc = lane & 3;
#pragma unroll
  for (int kk = 0; kk < T::BK; kk += 4) {
    if (kk >= kv) break;
    double a[T::MF], b[T::NF];
#pragma unroll
    for (int i = 0; i < T::MF; ++i) a[i] = sA[(wm * T::MF * 8 + i * 8 + gr) * T::SA + kk + gc];
#pragma unroll
    for (int j = 0; j < T::NF; ++j) b[j] = sB[(kk + gc) * T::SB + wn * T::NF * 8 + j * 8 + gr];
#pragma unroll
    for (int j = 0; j < T::NF; ++j) {
      if (j >= jmax) break;
#pragma unroll
      for (int i = 0; i < T::MF; ++i) dmma_8x8x4(acc.c[i][j][0], acc.c[i][j][1], a[i], b[j]);
    }
  }
}

// 16-byte async copies (pairs of doubles); the tail pair of a row copies 8 bytes and
// zero-fills the rest.  Requires 16-byte aligned rows (checked by the caller).
template <class T>
__device__ __forceinline__ void load_a_async16(double* sA, const double* __restrict__ A,
                                               int64_t lda, int64_t M, int64_t m0, int K, int k0,
                                               int tid) {
  constexpr int PR = T::BK / 2;
  constexpr int N = T::BM * PR;
#pragma unroll
  for (int e = tid; e < N; e += T::THREADS) {
    const int r = e / PR, c = (e % PR) * 2;
    const int64_t gr = m0 + r;
    const int gc = k0 + c;
    const int nvalid = (gr < M) ? max(0, min(2, K - gc)) : 0;
    const double* src = nvalid ? (A + gr * lda + gc) : A;
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(sA + r * T::SA + c));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(src),
                 "r"(nvalid * 8));
  }
}

template <class T>
__device__ __forceinline__ void load_b_async16(double* sB, const double* __restrict__ B,
                                               int64_t ldb, int K, int k0, int N, int tid) {
  constexpr int PR = (T::BN + 1) / 2;
  constexpr int NE = T::BK * PR;
#pragma unroll 2
  for (int e = tid; e < NE; e += T::THREADS) {
    const int r = e / PR, c = (e % PR) * 2;
    const int gk = k0 + r;
    const int nvalid = (gk < K) ? max(0, min(2, N - c)) : 0;
    const double* src = nvalid ? (B + (int64_t)gk * ldb + c) : B;
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(sB + r * T::SB + c));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(src),
                 "r"(nvalid * 8));
  }
}

// Async copy of an A chunk: rows [m0, m0+BM) x cols [k0, k0+BK) of row-major A (ld),
// zero-filled outside [0,M) x [0,K).
template <class T>
__device__ __forceinline__ void load_a_async(double* sA, const double* __restrict__ A, int64_t lda,
                                             int64_t M, int64_t m0, int K, int k0, int tid) {
  constexpr int N = T::BM * T::BK;
#pragma unroll 4
  for (int e = tid; e < N; e += T::THREADS) {
    int r = e / T::BK, c = e % T::BK;
    int64_t gr = m0 + r;
    int gc = k0 + c;
    bool ok = (gr < M) && (gc < K);
    const double* src = ok ? (A + gr * lda + gc) : A;
    cp_async8(sA + r * T::SA + c, src, ok);
  }
}

// Async copy of a B chunk: element (kk, n) at B[kk*sr + n*sc]; zero outside [0,K) x [0,N).
template <class T>
__device__ __forceinline__ void load_b_async(double* sB, const double* __restrict__ B, int64_t sr,
                                             int64_t sc, int K, int k0, int N, int n0, int tid) {
  constexpr int NE = T::BK * T::BN;
#pragma unroll 4
  for (int e = tid; e < NE; e += T::THREADS) {
    int r, c;
    if (sc == 1) { r = e / T::BN; c = e % T::BN; }      // coalesce along n
    else { c = e / T::BK; r = e % T::BK; }              // coalesce along k (transposed source)
    int gk = k0 + r, gn = n0 + c;
    bool ok = (gk < K) && (gn < N);
    const double* src = ok ? (B + (int64_t)gk * sr + (int64_t)gn * sc) : B;
    cp_async8(sB + r * T::SB + c, src, ok);
  }
}

// Store the accumulator tile to row-major C (ldc), masked to [0,M) x [0,N).
template <class T>
__device__ __forceinline__ void store_acc(const Acc<T>& acc, double* __restrict__ C, int64_t ldc,
                                          int64_t M, int64_t m0, int N, int n0, int wm, int wn,
                                          int lane) {
  const int gr = lane >> 2, gc = lane & 3;
#pragma unroll
  for (int i = 0; i < T::MF; ++i) {
    int64_t row = m0 + wm * T::MF * 8 + i * 8 + gr;
    if (row >= M) continue;
    double* crow = C + row * ldc;
#pragma unroll
    for (int j = 0; j < T::NF; ++j) {
      int col = n0 + wn * T::NF * 8 + j * 8 + 2 * gc;
      if (col < N) crow[col] = acc.c[i][j][0];
      if (col + 1 < N) crow[col + 1] = acc.c[i][j][1];
    }
  }
}

}  // namespace hsseig
