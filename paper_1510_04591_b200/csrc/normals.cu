// The reference's Gaussian sample block on the device, bit-for-bit.
//
// rand_hss_construct draws Omega = default_rng(seed).standard_normal((k, w))
// (pkg/src/hsseig/hss.py:236-237): NumPy's PCG64 (XSL-RR 128/64) bit stream fed
// through its 256-layer ziggurat for the normal distribution (NumPy
// random/src/distributions: random_standard_normal; third-party, not vendored).
// The generator is sequential and the ziggurat rejects a variable number of
// draws, so the device version works in three passes over the raw stream:
//   1. raw     : every thread jumps the LCG to its segment (O(log n) advance) and
//                writes its 64-bit outputs;
//   2. walk    : every segment parses the rejection chain from the first E entry
//                offsets it can be entered at and records exit position and count;
//   3. resolve : every segment fixes its true entry offset (chains from nearby
//                offsets merge within a few draws, so the look-back is short);
//                a two-level scan turns the per-segment counts into output indices;
//   4. emit    : every segment re-walks from its true entry and writes its normals
//                at their global index.
// The ziggurat tables are NumPy's own (ki/wi/fi), loaded once by the host from the
// installed NumPy and checked against NumPy output before use.
#include <cmath>
#include <cstring>

#include "common.cuh"

namespace hsseig {

typedef unsigned __int128 u128;

constexpr int kSeg = 32;       // raw draws per segment (short: one thread per segment, latency-bound walk)
constexpr int kEntries = 16;   // entry offsets tried per segment
constexpr double kZigR = 3.6541528853610088;
constexpr double kZigInvR = 0.27366123732975828;

__device__ uint64_t g_ki[256];
__device__ double g_wi[256];
__device__ double g_fi[256];
static bool g_tables_loaded = false;

__device__ __forceinline__ u128 mk128(uint64_t hi, uint64_t lo) { return ((u128)hi << 64) | lo; }

__device__ __forceinline__ uint64_t xsl_rr(u128 s) {
  const uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
  const unsigned rot = (unsigned)(s >> 122);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

// state after `delta` LCG steps (PCG's O(log delta) jump)
__device__ u128 lcg_advance(u128 state, u128 delta, u128 mult, u128 plus) {
  u128 acc_mult = 1, acc_plus = 0;
  while (delta > 0) {
    if (delta & 1) {
      acc_mult *= mult;
      acc_plus = acc_plus * mult + plus;
    }
    plus = (mult + 1) * plus;
    mult *= mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

__global__ void raw_kernel(uint64_t sh, uint64_t sl, uint64_t ih, uint64_t il, int64_t L,
                           uint64_t* __restrict__ U) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t p0 = t * kSeg;
  if (p0 >= L) return;
  const u128 mult = mk128(2549297995355413924ull, 4865540595714422341ull);
  const u128 inc = mk128(ih, il);
  u128 s = lcg_advance(mk128(sh, sl), (u128)p0, mult, inc);
  const int64_t pe = p0 + kSeg < L ? p0 + kSeg : L;
  for (int64_t p = p0; p < pe; ++p) {
    s = s * mult + inc;
    U[p] = xsl_rr(s);
  }
}

__device__ __forceinline__ double unit(uint64_t r) { return (double)(r >> 11) * (1.0 / 9007199254740992.0); }

// Parse one normal starting at draw p; returns the next start, writes the value.
// Draws beyond L count as failure (returns L).
// *tail_u receives the raw draw behind the tail-branch log1p (0 otherwise): NumPy evaluates
// that value with the C library's log1p, whose last bit the device log1p does not always
// reproduce, so the host re-evaluates those few values (about 1 in 4000 normals).
__device__ __forceinline__ int64_t one_normal(const uint64_t* __restrict__ U, int64_t p, int64_t L,
                                              double* val, uint64_t* tail_u = nullptr,
                                              int* tail_sign = nullptr) {
  for (;;) {
    if (p >= L) return L;
    uint64_t r = U[p];
    const int idx = (int)(r & 0xff);
    r >>= 8;
    const int sign = (int)(r & 1);
    const uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
    double x = (double)rabs * g_wi[idx];
    if (sign) x = -x;
    if (rabs < g_ki[idx]) { *val = x; return p + 1; }
    if (idx == 0) {
      int64_t q = p + 1;
      for (;;) {
        if (q + 1 >= L) return L;
        const double xx = -kZigInvR * log1p(-unit(U[q]));
        const double yy = -log1p(-unit(U[q + 1]));
        q += 2;
        if (yy + yy > xx * xx) {
          *val = ((rabs >> 8) & 1) ? -(kZigR + xx) : kZigR + xx;
          if (tail_u) {
            *tail_u = U[q - 2];
            *tail_sign = (int)((rabs >> 8) & 1);
          }
          return q;
        }
      }
    }
    if (p + 1 >= L) return L;
    if ((g_fi[idx - 1] - g_fi[idx]) * unit(U[p + 1]) + g_fi[idx] < exp(-0.5 * x * x)) {
      *val = x;
      return p + 2;
    }
    p += 2;  // wedge rejection: the same normal restarts on the next draws
  }
}

// exit position and start count of the chain entering segment t at offset e.  The chain
// from offset 0 is walked in full and its starts kept in a 256-bit map; the chains from
// the other offsets stop as soon as they land on one of those starts (they coincide
// from there on), so each extra entry costs only a few parses.
__global__ void walk_kernel(const uint64_t* __restrict__ U, int64_t L, int nseg,
                            int64_t* __restrict__ exitpos, int32_t* __restrict__ count) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nseg) return;
  const int64_t a = (int64_t)t * kSeg, b = a + kSeg;
  uint32_t bits[kSeg / 32];
#pragma unroll
  for (int q = 0; q < kSeg / 32; ++q) bits[q] = 0u;
  int64_t p = a;
  int c0 = 0;
  double v;
  while (p < b) {
    const int r = (int)(p - a);
    bits[r >> 5] |= 1u << (r & 31);
    p = one_normal(U, p, L, &v);
    ++c0;
  }
  const int64_t x0 = p;
  exitpos[(int64_t)t * kEntries] = x0;
  count[(int64_t)t * kEntries] = c0;
  for (int e = 1; e < kEntries; ++e) {
    p = a + e;
    int c = 0;
    bool merged = false;
    while (p < b) {
      const int r = (int)(p - a);
      if ((bits[r >> 5] >> (r & 31)) & 1u) {
        // chain-0 starts at positions >= r
        int rest = __popc(bits[r >> 5] >> (r & 31));
        for (int q = (r >> 5) + 1; q < kSeg / 32; ++q) rest += __popc(bits[q]);
        c += rest;
        merged = true;
        break;
      }
      p = one_normal(U, p, L, &v);
      ++c;
    }
    exitpos[(int64_t)t * kEntries + e] = merged ? x0 : p;
    count[(int64_t)t * kEntries + e] = c;
  }
}

// true entry offset of every segment (look back to the nearest segment whose exit does
// not depend on its entry, then compose forward), the segment's normal count, and a
// block-local exclusive scan of the counts; bsum[block] = the block's total
constexpr int kResolveThreads = 256;

__global__ void __launch_bounds__(kResolveThreads) resolve_kernel(
    const int64_t* __restrict__ exitpos, const int32_t* __restrict__ count, int nseg,
    int32_t* __restrict__ entry, int64_t* __restrict__ base, int64_t* __restrict__ bsum,
    int32_t* __restrict__ fail) {
  __shared__ int64_t sc[kResolveThreads];
  const int t = blockIdx.x * kResolveThreads + threadIdx.x;
  int64_t c = 0;
  if (t < nseg) {
    int q0 = t - 1;
    while (q0 >= 0) {
      const int64_t* x = exitpos + (int64_t)q0 * kEntries;
      bool merged = true;
      for (int q = 1; q < kEntries; ++q) merged &= (x[q] == x[0]);
      if (merged) break;
      --q0;
    }
    int eq, q;
    if (q0 >= 0) {
      eq = (int)(exitpos[(int64_t)q0 * kEntries] - (int64_t)(q0 + 1) * kSeg);
      q = q0 + 1;
    } else {
      eq = 0;
      q = 0;
    }
    for (; q < t; ++q) {
      if (eq < 0 || eq >= kEntries) { *fail = 1; eq = 0; }
      eq = (int)(exitpos[(int64_t)q * kEntries + eq] - (int64_t)(q + 1) * kSeg);
    }
    if (eq < 0 || eq >= kEntries) { *fail = 1; eq = 0; }
    entry[t] = eq;
    c = count[(int64_t)t * kEntries + eq];
  }
  // block-local exclusive scan (Hillis-Steele over 256 entries)
  sc[threadIdx.x] = c;
  __syncthreads();
  for (int off = 1; off < kResolveThreads; off <<= 1) {
    const int64_t v = threadIdx.x >= off ? sc[threadIdx.x - off] : 0;
    __syncthreads();
    sc[threadIdx.x] += v;
    __syncthreads();
  }
  if (t < nseg) base[t] = sc[threadIdx.x] - c;
  if (threadIdx.x == kResolveThreads - 1) bsum[blockIdx.x] = sc[threadIdx.x];
}

// one block: exclusive scan of the per-block totals (in place); checks the stream length
__global__ void scan_blocks_kernel(int64_t* __restrict__ bsum, int nblk, int64_t n,
                                   int32_t* __restrict__ fail) {
  __shared__ int64_t part[1024];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int per = (nblk + nt - 1) / nt;
  const int s0 = min(nblk, tid * per), s1 = min(nblk, s0 + per);
  int64_t s = 0;
  for (int b = s0; b < s1; ++b) s += bsum[b];
  part[tid] = s;
  __syncthreads();
  if (tid == 0) {
    int64_t acc = 0;
    for (int q = 0; q < nt; ++q) {
      const int64_t v = part[q];
      part[q] = acc;
      acc += v;
    }
    if (acc < n) *fail = 2;   // raw stream too short (never at the sizes the margin covers)
  }
  __syncthreads();
  int64_t acc = part[tid];
  for (int b = s0; b < s1; ++b) {
    const int64_t v = bsum[b];
    bsum[b] = acc;
    acc += v;
  }
}

__global__ void emit_kernel(const uint64_t* __restrict__ U, int64_t L, int nseg,
                            const int32_t* __restrict__ entry, const int64_t* __restrict__ base,
                            const int64_t* __restrict__ bsum, int64_t n, int64_t w, int64_t ldo, double* __restrict__ out,
                            int64_t* __restrict__ tails, int64_t tail_cap,
                            int32_t* __restrict__ fail) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nseg) return;
  const int64_t a = (int64_t)t * kSeg, b = a + kSeg;
  int64_t p = a + entry[t], i = base[t] + bsum[t / kResolveThreads];
  while (p < b && i < n) {
    double v;
    uint64_t tu = 0;
    int tsg = 0;
    bool tail = false;
    {
      uint64_t tmp = ~0ull;
      p = one_normal(U, p, L, &v, &tmp, &tsg);
      if (tmp != ~0ull) { tail = true; tu = tmp; }
    }
    const int64_t o = (i / w) * ldo + (i % w);   // row-major (n / w) x w, leading dimension ldo
    out[o] = v;
    if (tail && tails) {
      const unsigned long long slot = atomicAdd(reinterpret_cast<unsigned long long*>(tails), 1ull);
      if ((int64_t)slot < tail_cap) {
        tails[1 + 3 * slot] = o;
        tails[2 + 3 * slot] = (int64_t)tu;
        tails[3 + 3 * slot] = tsg;
      } else {
        *fail = 3;
      }
    }
    ++i;
  }
}

}  // namespace hsseig

using namespace hsseig;

static int64_t raw_len(int64_t n) { return ((n + n / 16 + 4096 + kSeg - 1) / kSeg) * kSeg; }

extern "C" int hsseig_set_normal_tables(const uint64_t* ki, const double* wi, const double* fi) {
  if (!ki || !wi || !fi) HSS_ARG_FAIL();
  if (cudaMemcpyToSymbol(g_ki, ki, sizeof(uint64_t) * 256) != cudaSuccess ||
      cudaMemcpyToSymbol(g_wi, wi, sizeof(double) * 256) != cudaSuccess ||
      cudaMemcpyToSymbol(g_fi, fi, sizeof(double) * 256) != cudaSuccess)
    return HSSEIG_ERR_CUDA;
  g_tables_loaded = true;
  return HSSEIG_OK;
}

extern "C" int64_t hsseig_normals_work_bytes(int64_t n) {
  const int64_t L = raw_len(n);
  const int64_t nseg = L / kSeg;
  const int64_t nblk = (nseg + kResolveThreads - 1) / kResolveThreads;
  return 8 * L + nseg * kEntries * (8 + 4) + nseg * 4 + (nseg + 1) * 8 + nblk * 8 + 1024;
}

extern "C" int hsseig_pcg64_normals(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                                    uint64_t inc_lo, int64_t n, int64_t w, int64_t ldo, double* out,
                                    void* work, int32_t* fail_dev, int64_t* tails,
                                    int64_t tail_cap, void* stream) {
  if (!g_tables_loaded) HSS_ARG_FAIL();
  if (n < 0 || w < 1 || ldo < w || !out || !work || !fail_dev) HSS_ARG_FAIL();
  if (n == 0) return HSSEIG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t L = raw_len(n);
  const int nseg = (int)(L / kSeg);
  char* wk = static_cast<char*>(work);
  uint64_t* U = reinterpret_cast<uint64_t*>(wk);
  int64_t* exitpos = reinterpret_cast<int64_t*>(wk + 8 * L);
  int32_t* count = reinterpret_cast<int32_t*>(exitpos + (int64_t)nseg * kEntries);
  int32_t* entry = count + (int64_t)nseg * kEntries;
  int64_t* base = reinterpret_cast<int64_t*>(
      (reinterpret_cast<uintptr_t>(entry + nseg) + 7) & ~(uintptr_t)7);
  raw_kernel<<<(nseg + 63) / 64, 64, 0, s>>>(state_hi, state_lo, inc_hi, inc_lo, L, U);
  HSS_CHECK_LAUNCH();
  walk_kernel<<<(nseg + 63) / 64, 64, 0, s>>>(U, L, nseg, exitpos, count);
  HSS_CHECK_LAUNCH();
  const int nblk = (nseg + kResolveThreads - 1) / kResolveThreads;
  int64_t* bsum = base + nseg + 1;
  resolve_kernel<<<nblk, kResolveThreads, 0, s>>>(exitpos, count, nseg, entry, base, bsum, fail_dev);
  HSS_CHECK_LAUNCH();
  scan_blocks_kernel<<<1, 1024, 0, s>>>(bsum, nblk, n, fail_dev);
  HSS_CHECK_LAUNCH();
  if (tails && cudaMemsetAsync(tails, 0, sizeof(int64_t), s) != cudaSuccess) return HSSEIG_ERR_CUDA;
  emit_kernel<<<(nseg + 63) / 64, 64, 0, s>>>(U, L, nseg, entry, base, bsum, n, w, ldo, out, tails,
                                                 tail_cap, fail_dev);
  HSS_CHECK_LAUNCH();
  return HSSEIG_OK;
}

// Ziggurat-tail re-evaluation with the host C library's log1p (NumPy's random_standard_normal
// evaluates the tail as -log1p(-u) / r with libm), then a scatter kernel on the stream that
// reads the (offset, value) pairs from pinned host memory: no Python loop, no blocking upload.
__global__ void tail_scatter_kernel(const int64_t* __restrict__ pairs, int64_t cnt,
                                    double* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < cnt) out[pairs[2 * t]] = __longlong_as_double(pairs[2 * t + 1]);
}

extern "C" int64_t hsseig_normals_fixup(const int64_t* h_tails, int64_t tail_cap, double zig_r,
                                        double zig_inv_r, int64_t* h_pairs, int64_t* d_pairs,
                                        double* out, void* stream) {
  // returns the number of values fixed, or -status
  if (!h_tails || !h_pairs || !d_pairs || !out || tail_cap < 0 || h_tails[0] < 0 ||
      h_tails[0] > tail_cap) {
    set_arg_error(__FILE__, __LINE__);
    return -HSSEIG_ERR_ARG;
  }
  const int64_t cnt = h_tails[0];
  for (int64_t t = 0; t < cnt; ++t) {
    const int64_t* rec = h_tails + 1 + 3 * t;
    const uint64_t u = static_cast<uint64_t>(rec[1]) >> 11;
    const double xx = -zig_inv_r * log1p(-(static_cast<double>(u) * (1.0 / 9007199254740992.0)));
    const double v = rec[2] ? -(zig_r + xx) : zig_r + xx;
    int64_t bits;
    memcpy(&bits, &v, sizeof(bits));
    h_pairs[2 * t] = rec[0];
    h_pairs[2 * t + 1] = bits;
  }
  if (cnt == 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  // the scatter reads the pinned pairs in place (mapped host memory): no copy-engine transfer,
  // which would queue behind a bulk host->device stream (MergePipeline's streamed Q_old)
  const int64_t* src = nullptr;
  void* mapped = nullptr;
  if (cudaHostGetDevicePointer(&mapped, h_pairs, 0) == cudaSuccess && mapped) {
    src = static_cast<const int64_t*>(mapped);
  } else {
    cudaGetLastError();
    if (cudaMemcpyAsync(d_pairs, h_pairs, sizeof(int64_t) * 2 * cnt, cudaMemcpyHostToDevice, s) !=
        cudaSuccess)
      return -HSSEIG_ERR_CUDA;
    src = d_pairs;
  }
  tail_scatter_kernel<<<(unsigned)((cnt + 255) / 256), 256, 0, s>>>(src, cnt, out);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (cudaPeekAtLastError() != cudaSuccess) return -HSSEIG_ERR_CUDA;
  return cnt;
}

