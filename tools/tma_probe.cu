// Minimal TMA + mbarrier probe: load boxes of a row-major FP64 matrix and verify.
#include <cstdio>
#include <vector>
#include "../paper_1510_04591_b200/csrc/tma.cuh"
using namespace hsseig;

__global__ void probe(const MapSet* maps, int c0, int c1, int bc, int br, double* out, int variant) {
  extern __shared__ __align__(128) unsigned char smraw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smraw) + 127) & ~(uintptr_t)127);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 65536);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    if (variant == 1) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(bar, bc * br * 8);
    tma_load_2d(sm, &maps->m[0], c0, c1, bar);
  }
  mbar_wait(bar, 0);
  const double* s = reinterpret_cast<const double*>(sm);
  for (int e = threadIdx.x; e < bc * br; e += blockDim.x) out[e] = s[e];
}

int main(int argc, char** argv) {
  const int rows = 40, cols = 256, ld = 256;
  std::vector<double> h(rows * ld);
  for (int i = 0; i < rows * ld; ++i) h[i] = i;
  double *d, *o;
  cudaMalloc(&d, sizeof(double) * rows * ld);
  cudaMalloc(&o, sizeof(double) * 65536);
  cudaMemcpy(d, h.data(), sizeof(double) * rows * ld, cudaMemcpyHostToDevice);
  MapSet* dm;
  cudaMalloc(&dm, sizeof(MapSet));
  struct Case { int bc, br, c0, c1, variant; };
  Case all[] = {{20, 16, 0, 0, 1}, {20, 64, 0, 0, 1}, {20, 16, 3, 0, 1}, {20, 16, 2, 0, 1},
                 {20, 16, 4, 0, 1}, {20, 32, 2, 5, 1}, {100, 16, 6, 30, 1}, {20, 16, 250, 10, 1}};
  int which = argc > 1 ? atoi(argv[1]) : 0;
  Case cases[1] = {all[which]};
  for (auto& cs : cases) {
    MapSet ms;
    memset(&ms, 0, sizeof(ms));
    bool ok = make_map(&ms.m[0], d, rows, cols, ld, cs.bc, cs.br);
    cudaMemcpy(dm, &ms, sizeof(ms), cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
    probe<<<1, 128, 70000>>>(dm, cs.c0, cs.c1, cs.bc, cs.br, o, cs.variant);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<double> r(cs.bc * cs.br);
    int bad = 0;
    if (e == cudaSuccess) {
      cudaMemcpy(r.data(), o, sizeof(double) * r.size(), cudaMemcpyDeviceToHost);
      for (int a = 0; a < cs.br; ++a) for (int b = 0; b < cs.bc; ++b) {
        int gr = cs.c1 + a, gc = cs.c0 + b;
        double want = (gr < rows && gc < cols) ? h[gr * ld + gc] : 0.0;
        if (r[a * cs.bc + b] != want) ++bad;
      }
    }
    printf("box %dx%d at (%d,%d) variant %d: encode=%d err=%s bad=%d\n", cs.bc, cs.br, cs.c0, cs.c1, cs.variant, ok, cudaGetErrorString(e), bad);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
