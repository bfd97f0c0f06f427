// Probe: latency of cuSOLVER symmetric eigensolvers for t x t (t ~ 220) fp64 and
// whether 8 of them overlap on 8 streams.  nvcc -O2 -arch=sm_100a probe_cusolver.cu -lcusolver -o probe
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <chrono>
#include <cstdio>
#include <vector>

#define CK(x)                                                             \
  do {                                                                    \
    auto e = (x);                                                         \
    if ((int)e != 0) {                                                    \
      printf("error %d at %s:%d\n", (int)e, __FILE__, __LINE__);          \
      return 1;                                                           \
    }                                                                     \
  } while (0)

int main() {
  const int t = 220, NB = 8;
  std::vector<double> h(t * t);
  for (int i = 0; i < t; ++i)
    for (int j = 0; j <= i; ++j) {
      double v = (i == j) ? t + (i % 7) : 1.0 / (1 + i + j) + 0.01 * ((i * 31 + j * 17) % 13);
      h[i * t + j] = h[j * t + i] = v;
    }
  std::vector<cudaStream_t> st(NB);
  std::vector<cusolverDnHandle_t> hs(NB);
  std::vector<double*> A(NB), Ab(NB), W(NB), work(NB);
  std::vector<int*> info(NB);
  int lwork = 0;
  for (int b = 0; b < NB; ++b) {
    CK(cudaStreamCreateWithFlags(&st[b], cudaStreamNonBlocking));
    CK(cusolverDnCreate(&hs[b]));
    CK(cusolverDnSetStream(hs[b], st[b]));
    CK(cudaMalloc(&A[b], t * t * 8));
    CK(cudaMalloc(&Ab[b], t * t * 8));
    CK(cudaMalloc(&W[b], t * 8));
    CK(cudaMalloc(&info[b], 4));
    CK(cudaMemcpy(Ab[b], h.data(), t * t * 8, cudaMemcpyHostToDevice));
  }
  CK(cusolverDnDsyevd_bufferSize(hs[0], CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, t, A[0], t, W[0], &lwork));
  for (int b = 0; b < NB; ++b) CK(cudaMalloc(&work[b], (size_t)lwork * 8 * 4));
  auto now = [] { return std::chrono::high_resolution_clock::now(); };
  auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
  for (int rep = 0; rep < 3; ++rep) {
    // single
    CK(cudaMemcpyAsync(A[0], Ab[0], t * t * 8, cudaMemcpyDeviceToDevice, st[0]));
    CK(cudaDeviceSynchronize());
    auto t0 = now();
    CK(cusolverDnDsyevd(hs[0], CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, t, A[0], t, W[0], work[0], lwork,
                        info[0]));
    CK(cudaDeviceSynchronize());
    auto t1 = now();
    // 8 streams
    for (int b = 0; b < NB; ++b) CK(cudaMemcpyAsync(A[b], Ab[b], t * t * 8, cudaMemcpyDeviceToDevice, st[b]));
    CK(cudaDeviceSynchronize());
    auto t2 = now();
    for (int b = 0; b < NB; ++b)
      CK(cusolverDnDsyevd(hs[b], CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, t, A[b], t, W[b], work[b], lwork,
                          info[b]));
    auto t2b = now();
    CK(cudaDeviceSynchronize());
    auto t3 = now();
    printf("syevd t=%d: single %.3f ms | 8 streams %.3f ms (host enqueue %.3f ms)\n", t, ms(t0, t1), ms(t2, t3),
           ms(t2, t2b));
  }
  // syevj
  syevjInfo_t params;
  CK(cusolverDnCreateSyevjInfo(&params));
  CK(cusolverDnXsyevjSetTolerance(params, 1e-14));
  CK(cusolverDnXsyevjSetMaxSweeps(params, 20));
  int lj = 0;
  CK(cusolverDnDsyevj_bufferSize(hs[0], CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, t, A[0], t, W[0], &lj,
                                 params));
  double* wj;
  CK(cudaMalloc(&wj, (size_t)lj * 8 * NB));
  for (int rep = 0; rep < 2; ++rep) {
    CK(cudaMemcpy(A[0], Ab[0], t * t * 8, cudaMemcpyDeviceToDevice));
    CK(cudaDeviceSynchronize());
    auto t0 = now();
    CK(cusolverDnDsyevj(hs[0], CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, t, A[0], t, W[0], wj, lj, info[0],
                        params));
    CK(cudaDeviceSynchronize());
    auto t1 = now();
    printf("syevj t=%d: single %.3f ms\n", t, ms(t0, t1));
  }
  // syevdx: 20 largest
  int lx = 0, meig = 0;
  CK(cusolverDnDsyevdx_bufferSize(hs[0], CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, t,
                                  A[0], t, 0.0, 0.0, t - 19, t, &meig, W[0], &lx));
  double* wx;
  CK(cudaMalloc(&wx, (size_t)lx * 8));
  for (int rep = 0; rep < 2; ++rep) {
    CK(cudaMemcpy(A[0], Ab[0], t * t * 8, cudaMemcpyDeviceToDevice));
    CK(cudaDeviceSynchronize());
    auto t0 = now();
    CK(cusolverDnDsyevdx(hs[0], CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, t, A[0], t,
                         0.0, 0.0, t - 19, t, &meig, W[0], wx, lx, info[0]));
    CK(cudaDeviceSynchronize());
    auto t1 = now();
    printf("syevdx (20 largest) t=%d: %.3f ms\n", t, ms(t0, t1));
  }
  // geqrf 428 x 220
  int lq = 0;
  double *Q, *tau;
  CK(cudaMalloc(&Q, 428 * t * 8));
  CK(cudaMalloc(&tau, t * 8));
  CK(cusolverDnDgeqrf_bufferSize(hs[0], 428, t, Q, 428, &lq));
  double* wq;
  CK(cudaMalloc(&wq, (size_t)lq * 8));
  for (int rep = 0; rep < 2; ++rep) {
    CK(cudaDeviceSynchronize());
    auto t0 = now();
    CK(cusolverDnDgeqrf(hs[0], 428, t, Q, 428, tau, wq, lq, info[0]));
    CK(cudaDeviceSynchronize());
    auto t1 = now();
    printf("geqrf 428x%d: %.3f ms\n", t, ms(t0, t1));
  }
  return 0;
}
