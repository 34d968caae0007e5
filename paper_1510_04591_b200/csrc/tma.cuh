// TMA + mbarrier helpers and the warp-specialised FP64 DMMA tile geometry (sm_100a).
#pragma once
#include <cudaTypedefs.h>

#include <cstring>

#include "dmma_gemm.cuh"

namespace hsseig {

constexpr int kMaps = 8;  // tensor-map roles of one launch (see hss_mult.cu / cauchy.cu)

struct alignas(128) MapSet {
  CUtensorMap m[kMaps];
};

template <int MF_, int NF_, int WM_, int WN_, int STAGES_>
struct TTile {
  static constexpr int MF = MF_, NF = NF_, WM = WM_, WN = WN_, STAGES = STAGES_;
  static constexpr int BM = WM * MF * 8;
  static constexpr int BN = WN * NF * 8;
  static constexpr int BK = 16;
  static constexpr int SA = BK + 4;             // A box width (doubles) = smem row stride
  static constexpr int SB = ((BN + 15) / 16) * 16 + 4;
  static constexpr int CONSUMERS = WM * WN;
  static constexpr int THREADS = (CONSUMERS + 1) * 32;
  static constexpr int A_BYTES = BM * SA * 8;
  static constexpr int B_BYTES = BK * SB * 8;
  static constexpr int STAGE_BYTES = ((A_BYTES + B_BYTES + 127) / 128) * 128;
  static constexpr size_t SMEM_BYTES = (size_t)STAGE_BYTES * STAGES + 2 * STAGES * 8 + 128;
  // two CTAs per SM when the ring is small enough (more warps to hide DMMA latency)
  static constexpr int MINB = SMEM_BYTES <= 112 * 1024 ? 2 : 1;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
// Consumer release of one ring stage.  The stage's next TMA fill (async proxy) must not
// overtake this warp's fragment reads (generic proxy): ptxas does not make the mbarrier
// arrive wait for outstanding LDS, so the reads are fenced into the async proxy first.
__device__ __forceinline__ void stage_release(uint64_t* b, int lane) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane == 0) mbar_arrive(b);
}
// Tensor maps live in device memory and are rewritten (H2D copy) between launches at the
// same address; the TMA unit may serve a stale cached descriptor unless the issuing thread
// acquires the generic-proxy writes into the tensormap proxy first.
__device__ __forceinline__ void tmap_acquire(const CUtensorMap* map) {
  asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(
                   reinterpret_cast<uint64_t>(map))
               : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// One BK chunk; kv (warp-uniform, a multiple of 4) is the chunk's valid depth.  Operands
// are zero-padded past K (factor slots, TMA out-of-bounds fill), so rounding K up to a
// multiple of 4 is exact; output columns beyond N are computed but never stored.
template <class T>
__device__ __forceinline__ void tmma_chunk(const double* __restrict__ sA, const double* __restrict__ sB,
                                           double (&c)[T::MF][T::NF][2], int wm, int wn, int lane,
                                           int kv = T::BK) {
  const int gr = lane >> 2, gc = lane & 3;
  const double* a0 = sA + (wm * T::MF * 8 + gr) * T::SA + gc;
  const double* b0 = sB + gc * T::SB + wn * T::NF * 8 + gr;
#pragma unroll
  for (int kk = 0; kk < T::BK; kk += 4) {
    if (kk >= kv) break;
    double a[T::MF], b[T::NF];
#pragma unroll
    for (int i = 0; i < T::MF; ++i) a[i] = a0[i * 8 * T::SA + kk];
#pragma unroll
    for (int j = 0; j < T::NF; ++j) b[j] = b0[kk * T::SB + j * 8];
#pragma unroll
    for (int j = 0; j < T::NF; ++j)
#pragma unroll
      for (int i = 0; i < T::MF; ++i) dmma_8x8x4(c[i][j][0], c[i][j][1], a[i], b[j]);
  }
}

// Same chunk with only this warp's first JM n-fragments live (compile-time, straight-line
// code): a tile sized for the widest job of a launch does no DMMA work on the padding of
// narrower jobs (HSS levels mix ranks; the tile covers the largest one).
// FULL: all BK k-columns live (no per-k-step exits, so the compiler can hoist the
// fragment loads of later k-steps over the DMMAs of earlier ones).
template <class T, int JM, bool FULL, int JA>
__device__ __forceinline__ void tmma_chunk_j(const double* __restrict__ sA, const double* __restrict__ sB,
                                             double (&c)[T::MF][JA][2], int wm, int wn, int lane,
                                             int kv) {
  const int gr = lane >> 2, gc = lane & 3;
  const double* a0 = sA + (wm * T::MF * 8 + gr) * T::SA + gc;
  const double* b0 = sB + gc * T::SB + wn * T::NF * 8 + gr;
#pragma unroll
  for (int kk = 0; kk < T::BK; kk += 4) {
    if (!FULL && kk >= kv) break;
    double a[T::MF], b[JM > 0 ? JM : 1];
#pragma unroll
    for (int i = 0; i < T::MF; ++i) a[i] = a0[i * 8 * T::SA + kk];
#pragma unroll
    for (int j = 0; j < JM; ++j) b[j] = b0[kk * T::SB + j * 8];
#pragma unroll
    for (int j = 0; j < JM; ++j)
#pragma unroll
      for (int i = 0; i < T::MF; ++i) dmma_8x8x4(c[i][j][0], c[i][j][1], a[i], b[j]);
  }
}

// One job of a batched two-segment GEMM C = A1 B1 + A2 B2 (tma_gemm_kernel, hss_mult.cu).
struct TJob {
  int32_t am[2], acol[2];            // A map role and column offset per segment (rows = tile)
  int32_t bm[2], brow[2], bcol[2];   // B map role, row and column offset per segment
  int32_t K[2], N, SW;               // segment depths, output width, store width (zero fill)
  double* C;
  int64_t ldc;
};

// Tensor maps reach device memory through a kernel parameter (stream-ordered, no host
// blocking on a pageable copy that would queue behind bulk host<->device traffic).
static __global__ void put_maps_kernel(const __grid_constant__ MapSet maps, MapSet* dst) {
  const uint4* src = reinterpret_cast<const uint4*>(&maps);
  uint4* d = reinterpret_cast<uint4*>(dst);
  for (int i = threadIdx.x; i < (int)(sizeof(MapSet) / 16); i += blockDim.x) d[i] = src[i];
}

// ---------------------------------------------------------------------------- host side
static inline bool upload_maps(const MapSet& maps, MapSet* dst, cudaStream_t s) {
  put_maps_kernel<<<1, 64, 0, s>>>(maps, dst);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError() == cudaSuccess;
}
// Raw operand descriptions (rows, cols, ld) for the map roles of one launch.
struct Operand {
  const double* base;
  uint64_t rows, cols, ld;
};
// Job-table GEMM on the TMA/DMMA engine (hss_mult.cu): shape 0 rank-width tiles for N = n,
// 1 wide tiles, 2 tall-N tiles (BM 96, BN 128).  Maps go to dmaps (device), jobs are device.
int tma_jobs_gemm(int shape, int n, const Operand (&ops)[kMaps], MapSet* dmaps, const TJob* jobs,
                  int njobs, int64_t M, cudaStream_t s);
// Plain C = A B (row-major, 16-byte aligned A / B rows) on the engine; jobs: (N+127)/128
// device TJobs, dmaps: one device MapSet (hss_mult.cu).
int tma_plain_gemm(const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                   int64_t ldc, int64_t M, int64_t N, int64_t K, TJob* jobs, MapSet* dmaps,
                   cudaStream_t s);

static inline PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult qr;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// Row-major (rows x cols, leading dimension ld) float64 matrix, box of box_rows x box_cols.
static inline bool make_map(CUtensorMap* m, const double* base, uint64_t rows, uint64_t cols, uint64_t ld,
                     uint32_t box_cols, uint32_t box_rows) {
  memset(m, 0, sizeof(*m));
  if (!base) return true;   // role unused by this launch
  auto fn = encode_fn();
  if (!fn || rows == 0 || cols == 0) return false;
  cuuint64_t gdim[2] = {cols, rows};
  cuuint64_t gstride[1] = {ld * 8};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), gdim, gstride, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace hsseig
