// FP64 peak probe: FFMA64 (DFMA) chains and DMMA m8n8k4 chains, timed with CUDA events.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
  for (int t = 0; t < 8; ++t) { c[t][0] = 0; c[t][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0; for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void dmma16_kernel(double* out, int iters) {
  double a[8], b[4], c[4][4];
  for (int t = 0; t < 8; ++t) a[t] = threadIdx.x * 1e-3 + t;
  for (int t = 0; t < 4; ++t) b[t] = 1.0 - threadIdx.x * 1e-4 * t;
  for (int t = 0; t < 4; ++t) for (int u = 0; u < 4; ++u) c[t][u] = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0; for (int t = 0; t < 4; ++t) for (int u = 0; u < 4; ++u) s += c[t][u];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void ddiv_kernel(double* out, int iters, double a) {
  double x0 = threadIdx.x + 1.5, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, s = 0;
  for (int i = 0; i < iters; ++i) {
    s += a / x0 + a / x1 + a / x2 + a / x3;
    x0 += 1.0; x1 += 1.0; x2 += 1.0; x3 += 1.0;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, sizeof(double) * 148 * 64 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    int blocks = sms * 8, threads = 256, iters = 4096;
    cudaEventRecord(e0); dfma_kernel<<<blocks, threads>>>(out, iters, 0.999, 1e-3); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * blocks * threads * (double)iters * 64;
    printf("DFMA: %.2f TF/s\n", fl / ms / 1e9);
    iters = 2048;
    cudaEventRecord(e0); dmma_kernel<<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 256 * 8 * (double)iters * blocks * (threads / 32);
    printf("DMMA m8n8k4: %.2f TF/s\n", fl / ms / 1e9);
    iters = 512;
    cudaEventRecord(e0); dmma16_kernel<<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 16 * 8 * 16 * 4 * (double)iters * blocks * (threads / 32);
    printf("DMMA m16n8k16: %.2f TF/s\n", fl / ms / 1e9);
    iters = 2048;
    cudaEventRecord(e0); ddiv_kernel<<<blocks, threads>>>(out, iters, 3.0); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("DDIV: %.2f Gdiv/s\n", 4.0 * blocks * threads * (double)iters / ms / 1e6);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
