// Probe: batched symmetric eigensolvers at the recycle update's size (t ~ 220, 8 samples).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 scripts/probe_syev.cu -lcusolver -o gpurun_out/probe_syev
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>

#define CK(x) do { auto e = (x); if (e != 0) { printf("%s:%d err %d\n", __FILE__, __LINE__, (int)e); exit(1); } } while (0)

int main(int argc, char** argv) {
  int n = argc > 1 ? atoi(argv[1]) : 220, B = argc > 2 ? atoi(argv[2]) : 8;
  std::vector<double> h((size_t)n * n * B);
  srand(1);
  for (int b = 0; b < B; ++b) {
    std::vector<double> G((size_t)n * n);
    for (auto& x : G) x = rand() / (double)RAND_MAX - 0.5;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        double s = 0;
        for (int k = 0; k < n; ++k) s += G[i * n + k] * G[j * n + k];
        h[(size_t)b * n * n + i * n + j] = s / n;
      }
  }
  double *dA, *dA0, *dW;
  int* info;
  CK(cudaMalloc(&dA, h.size() * 8));
  CK(cudaMalloc(&dA0, h.size() * 8));
  CK(cudaMalloc(&dW, (size_t)n * B * 8));
  CK(cudaMalloc(&info, B * sizeof(int) * 2));
  CK(cudaMemcpy(dA0, h.data(), h.size() * 8, cudaMemcpyHostToDevice));
  cusolverDnHandle_t hd;
  CK(cusolverDnCreate(&hd));
  cusolverDnParams_t prm;
  CK(cusolverDnCreateParams(&prm));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;

  // batched
  size_t wd = 0, wh = 0;
  CK(cusolverDnXsyevBatched_bufferSize(hd, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, dA, n,
                                        CUDA_R_64F, dW, CUDA_R_64F, &wd, &wh, B));
  void* dwork;
  CK(cudaMalloc(&dwork, wd + 8));
  std::vector<char> hwork(wh + 8);
  for (int rep = 0; rep < 4; ++rep) {
    CK(cudaMemcpy(dA, dA0, h.size() * 8, cudaMemcpyDeviceToDevice));
    cudaEventRecord(e0);
    CK(cusolverDnXsyevBatched(hd, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, dA, n,
                              CUDA_R_64F, dW, CUDA_R_64F, dwork, wd, hwork.data(), wh, info, B));
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("XsyevBatched n=%d B=%d: %.3f ms (work %zu B dev, %zu B host)\n", n, B, ms, wd, wh);
  }
  std::vector<double> w1((size_t)n * B);
  CK(cudaMemcpy(w1.data(), dW, w1.size() * 8, cudaMemcpyDeviceToHost));

  // per-matrix syevd
  int lw;
  CK(cusolverDnDsyevd_bufferSize(hd, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dW, &lw));
  double* w2;
  CK(cudaMalloc(&w2, (size_t)lw * 8));
  for (int rep = 0; rep < 3; ++rep) {
    CK(cudaMemcpy(dA, dA0, h.size() * 8, cudaMemcpyDeviceToDevice));
    cudaEventRecord(e0);
    for (int b = 0; b < B; ++b)
      CK(cusolverDnDsyevd(hd, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA + (size_t)b * n * n, n,
                          dW + (size_t)b * n, w2, lw, info));
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("syevd loop n=%d B=%d: %.3f ms\n", n, B, ms);
  }
  std::vector<double> w3((size_t)n * B);
  CK(cudaMemcpy(w3.data(), dW, w3.size() * 8, cudaMemcpyDeviceToHost));
  double md = 0;
  for (size_t i = 0; i < w1.size(); ++i) md = fmax(md, fabs(w1[i] - w3[i]));
  printf("max |eig batched - eig syevd| = %.3e\n", md);

  // syevj batched (Jacobi) for reference, only if n <= 32 supported
  syevjInfo_t sj;
  CK(cusolverDnCreateSyevjInfo(&sj));
  int lwj = 0;
  auto st = cusolverDnDsyevjBatched_bufferSize(hd, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dW,
                                               &lwj, sj, B);
  printf("syevjBatched bufferSize status %d\n", (int)st);
  return 0;
}
