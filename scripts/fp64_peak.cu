// fp64_peak.cu -- measured fp64 peaks of the B200 ("Measure fp64 on the box").
//
//   dfma : a DFMA loop, 8 independent chains per thread, 148 * 8 CTAs x 256 threads
//   dmma : mma.sync m8n8k4 f64 (the DMMA tensor path), 4 independent accumulators per warp
//   dgemm: cuBLAS DGEMM 8192^3 (what cuBLAS reaches on a large square problem)
//
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/fp64_peak scripts/fp64_peak.cu -lcublas
// Prints one JSON line (TFLOP/s, best of 5, CUDA events).
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) x[u] = threadIdx.x * 1e-9 + u;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = fma(x[u], a, b);
  }
  double s = 0;
#pragma unroll
  for (int u = 0; u < 8; ++u) s += x[u];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-12, b = 0.999999;
  double c[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[u][0]), "+d"(c[u][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int u = 0; u < 4; ++u) s += c[u][0] + c[u][1];
  if (s == 12345.678) out[0] = s;
}

template <typename F>
float best_ms(F&& f, int reps = 5) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  f();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  const int iters = 1 << 16;
  const int blocks = sms * 8, threads = 256;
  const float t_fma = best_ms([&] { dfma_kernel<<<blocks, threads>>>(out, iters, 0.9999999, 1e-7); });
  const double fl_fma = 2.0 * 8 * iters * (double)blocks * threads;
  const float t_mma = best_ms([&] { dmma_kernel<<<blocks, threads>>>(out, iters); });
  const double fl_mma = 2.0 * 8 * 8 * 4 * 4 * (double)iters * blocks * (threads / 32);
  const int N = 8192;
  double *A, *B, *C;
  cudaMalloc(&A, sizeof(double) * N * N);
  cudaMalloc(&B, sizeof(double) * N * N);
  cudaMalloc(&C, sizeof(double) * N * N);
  cudaMemset(A, 0, sizeof(double) * N * N);
  cudaMemset(B, 0, sizeof(double) * N * N);
  cublasHandle_t h;
  cublasCreate(&h);
  const double one = 1.0, zero = 0.0;
  const float t_gemm = best_ms([&] {
    cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, N, N, N, &one, A, N, B, N, &zero, C, N);
  }, 3);
  const double fl_gemm = 2.0 * N * (double)N * N;
  const cudaError_t e = cudaDeviceSynchronize();
  printf("{\"dfma_tflops\": %.2f, \"dmma_tflops\": %.2f, \"cublas_dgemm_8192_tflops\": %.2f, \"sms\": %d, "
         "\"status\": \"%s\"}\n",
         fl_fma / t_fma / 1e9, fl_mma / t_mma / 1e9, fl_gemm / t_gemm / 1e9, sms, cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
