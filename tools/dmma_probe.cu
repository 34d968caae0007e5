// DMMA throughput vs independent accumulator chains per warp and warps per SM.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void chains(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[CH][2];
#pragma unroll
  for (int t = 0; t < CH; ++t) { c[t][0] = 0; c[t][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < CH; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < CH; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int CH>
void run(int warps_per_sm, double* out) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int threads = 32 * warps_per_sm;   // one block per SM
  int iters = 4096 * 8 / CH;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  chains<CH><<<sms, threads>>>(out, 16);
  cudaEventRecord(e0);
  chains<CH><<<sms, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double fl = 2.0 * 256 * CH * (double)iters * sms * warps_per_sm;
  printf("chains %2d warps/SM %2d: %6.2f TF/s\n", CH, warps_per_sm, fl / ms / 1e9);
}
int main() {
  double* out;
  cudaMalloc(&out, sizeof(double) * 148 * 1024);
  for (int w : {4, 8, 12, 16, 32}) {
    run<4>(w, out); run<8>(w, out); run<12>(w, out); run<16>(w, out); run<24>(w, out);
  }
  return 0;
}
