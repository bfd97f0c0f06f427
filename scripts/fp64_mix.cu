// fp64_mix.cu -- do DFMA (FP64 pipe) and DMMA (mma.sync m8n8k4 f64) issue concurrently on sm_100?
// mode 0: even warps DFMA only; 1: odd warps DMMA only; 2: both (even DFMA, odd DMMA).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fp64_mix scripts/fp64_mix.cu
#include <cuda_runtime.h>
#include <cstdio>

__global__ void mix_kernel(double* out, int it_f, int it_m, int mode) {
  const int warp = threadIdx.x >> 5;
  double s = 0;
  if ((warp & 1) == 0 && mode != 1) {
    double x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = threadIdx.x * 1e-9 + u;
    for (int i = 0; i < it_f; ++i) {
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = fma(x[u], 0.9999999, 1e-7);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) s += x[u];
  } else if ((warp & 1) == 1 && mode != 0) {
    double a = 1.0 + threadIdx.x * 1e-12, b = 0.999999;
    double c[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
    for (int i = 0; i < it_m; ++i) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[u][0]), "+d"(c[u][1]) : "d"(a), "d"(b));
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) s += c[u][0] + c[u][1];
  }
  if (s == 12345.678) out[0] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 4, threads = 512;
  const int it_f = 1 << 15, it_m = 1 << 14;
  for (int mode = 0; mode < 3; ++mode) {
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) {
      cudaEventRecord(e0);
      mix_kernel<<<blocks, threads>>>(out, it_f, it_m, mode);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r && ms < best) best = ms;
    }
    const double wh = (double)blocks * threads / 2;  // threads doing each kind
    const double ff = mode != 1 ? 2.0 * 8 * it_f * wh : 0, fm = mode != 0 ? 2.0 * 256 * 4 * (double)it_m * wh / 32 : 0;
    printf("mode %d: %.3f ms  dfma %.2f TF  dmma %.2f TF  total %.2f TF\n", mode, best, ff / best / 1e9,
           fm / best / 1e9, (ff + fm) / best / 1e9);
  }
  return 0;
}
