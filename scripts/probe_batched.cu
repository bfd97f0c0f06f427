// Probe: batched building blocks of the recycle update at C2 sizes (n = 16384, T = 220, B = 8).
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { auto e = (x); if (e != 0) { printf("%s:%d err %d\n", __FILE__, __LINE__, (int)e); exit(1); } } while (0)

__global__ void fill(double* a, size_t n, unsigned seed) {
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    unsigned h = (unsigned)(i * 2654435761u) ^ seed;
    h ^= h >> 13; h *= 0x5bd1e995; h ^= h >> 15;
    a[i] = (h & 0xffffff) / 16777216.0 - 0.5;
  }
}
__global__ void add_diag(double* G, int T, double v) {
  G[(size_t)blockIdx.x * T * T + threadIdx.x * (T + 1)] += v;
}

int main(int argc, char** argv) {
  int n = argc > 1 ? atoi(argv[1]) : 16384, T = argc > 2 ? atoi(argv[2]) : 220, B = argc > 3 ? atoi(argv[3]) : 8;
  double *A, *G, *Q;
  CK(cudaMalloc(&A, (size_t)n * T * B * 8));
  CK(cudaMalloc(&Q, (size_t)n * T * B * 8));
  CK(cudaMalloc(&G, (size_t)T * T * B * 8));
  fill<<<1024, 256>>>(A, (size_t)n * T * B, 7);
  cublasHandle_t hb;
  CK(cublasCreate(&hb));
  cusolverDnHandle_t hs;
  CK(cusolverDnCreate(&hs));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  const double one = 1.0, zero = 0.0;
  auto timeit = [&](const char* name, auto fn, int reps = 5) {
    fn();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) fn();
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-48s %8.1f us\n", name, ms * 1000 / reps);
  };
  // Gram G = A^T A (A column-major n x T per sample)
  timeit("gram dgemmStridedBatched TxT (n=16384)", [&] {
    CK(cublasDgemmStridedBatched(hb, CUBLAS_OP_T, CUBLAS_OP_N, T, T, n, &one, A, n, (long long)n * T, A, n,
                                 (long long)n * T, &zero, G, T, (long long)T * T, B));
  });
  double* Gp;
  CK(cudaMalloc(&Gp, (size_t)T * T * B * 16 * 8));
  for (int S : {2, 4, 8, 16}) {
    char nm[96];
    snprintf(nm, sizeof nm, "gram split-K S=%d (per-sample strided batch)", S);
    const int c = n / S;
    timeit(nm, [&] {
      for (int b = 0; b < B; ++b)
        CK(cublasDgemmStridedBatched(hb, CUBLAS_OP_T, CUBLAS_OP_N, T, T, c, &one, A + (size_t)b * n * T, n, c,
                                     A + (size_t)b * n * T, n, c, &zero, Gp + (size_t)b * S * T * T, T,
                                     (long long)T * T, S));
    });
    std::vector<const double*> pa(B * S), pb(B * S);
    std::vector<double*> pc(B * S);
    for (int b = 0; b < B; ++b)
      for (int s = 0; s < S; ++s) {
        pa[b * S + s] = A + (size_t)b * n * T + (size_t)s * c;
        pc[b * S + s] = Gp + ((size_t)b * S + s) * T * T;
      }
    const double** dpa;
    double** dpc;
    CK(cudaMalloc(&dpa, B * S * 8));
    CK(cudaMalloc(&dpc, B * S * 8));
    CK(cudaMemcpy(dpa, pa.data(), B * S * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dpc, pc.data(), B * S * 8, cudaMemcpyHostToDevice));
    snprintf(nm, sizeof nm, "gram split-K S=%d (pointer-array batch %d)", S, B * S);
    timeit(nm, [&] {
      CK(cublasDgemmBatched(hb, CUBLAS_OP_T, CUBLAS_OP_N, T, T, c, &one, dpa, n, dpa, n, &zero, dpc, T, B * S));
    });
  }
  timeit("gram dsyrk loop (8 calls)", [&] {
    for (int b = 0; b < B; ++b)
      CK(cublasDsyrk(hb, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, T, n, &one, A + (size_t)b * n * T, n, &zero,
                     G + (size_t)b * T * T, T));
  });
  add_diag<<<B, T>>>(G, T, (double)n);
  std::vector<double*> hp(B), hq(B), ha(B);
  for (int b = 0; b < B; ++b) { hp[b] = G + (size_t)b * T * T; hq[b] = Q + (size_t)b * n * T; ha[b] = A + (size_t)b * n * T; }
  double **dp, **dq, **da;
  CK(cudaMalloc(&dp, B * 8)); CK(cudaMalloc(&dq, B * 8)); CK(cudaMalloc(&da, B * 8));
  CK(cudaMemcpy(dp, hp.data(), B * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dq, hq.data(), B * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(da, ha.data(), B * 8, cudaMemcpyHostToDevice));
  int* info;
  CK(cudaMalloc(&info, B * 4));
  double* G0;
  CK(cudaMalloc(&G0, (size_t)T * T * B * 8));
  CK(cudaMemcpy(G0, G, (size_t)T * T * B * 8, cudaMemcpyDeviceToDevice));
  timeit("potrfBatched T=220 B=8", [&] {
    CK(cudaMemcpyAsync(G, G0, (size_t)T * T * B * 8, cudaMemcpyDeviceToDevice));
    CK(cusolverDnDpotrfBatched(hs, CUBLAS_FILL_MODE_LOWER, T, dp, T, info, B));
  });
  int lw;
  CK(cusolverDnDpotrf_bufferSize(hs, CUBLAS_FILL_MODE_LOWER, T, G, T, &lw));
  double* wk;
  CK(cudaMalloc(&wk, (size_t)lw * 8 + 8));
  timeit("potrf loop (8 calls)", [&] {
    CK(cudaMemcpyAsync(G, G0, (size_t)T * T * B * 8, cudaMemcpyDeviceToDevice));
    for (int b = 0; b < B; ++b)
      CK(cusolverDnDpotrf(hs, CUBLAS_FILL_MODE_LOWER, T, G + (size_t)b * T * T, T, wk, lw, info));
  });
  CK(cudaMemcpy(Q, A, (size_t)n * T * B * 8, cudaMemcpyDeviceToDevice));
  timeit("trsmBatched right Lower^T (n x T)", [&] {
    CK(cublasDtrsmBatched(hb, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, n, T, &one,
                          dp, T, dq, n, B));
  });
  timeit("dgemmStridedBatched A * M (n x T x T)", [&] {
    CK(cublasDgemmStridedBatched(hb, CUBLAS_OP_N, CUBLAS_OP_T, n, T, T, &one, A, n, (long long)n * T, G, T,
                                 (long long)T * T, &zero, Q, n, (long long)n * T, B));
  });
  timeit("dgemmStridedBatched A * X (n x T x 20)", [&] {
    CK(cublasDgemmStridedBatched(hb, CUBLAS_OP_N, CUBLAS_OP_N, n, 20, T, &one, A, n, (long long)n * T, G, T,
                                 (long long)T * T, &zero, Q, n, (long long)n * T, B));
  });
  timeit("dgemmStridedBatched small TxT x T", [&] {
    CK(cublasDgemmStridedBatched(hb, CUBLAS_OP_N, CUBLAS_OP_T, T, T, T, &one, G, T, (long long)T * T, G, T,
                                 (long long)T * T, &zero, Q, T, (long long)T * T, B));
  });
  return 0;
}
