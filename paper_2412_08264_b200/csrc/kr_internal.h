// kr_internal.h -- host-side error plumbing shared by the C ABI translation units.
#pragma once

#include <cuda.h>
#include <cusolverDn.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <string>

#include "../../include/krecycle_b200.h"

namespace kr {

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int check_launch(const char* what);
int validate_op(const kr_op& op);
int ensure_smem(const void* kernel, size_t bytes);
int device_sms();
int cusolver_handle(cusolverDnHandle_t* out, cudaStream_t st);
// 4-D fp64 tensor map (cols, rows, ncols, batch) with leading / batch strides ld, bs (elements)
// and box (box_w, box_h, 1, 1) for the TMA-staged stencil regions; false when the layout is not
// expressible (odd widths or strides, misaligned base) or the driver entry point is missing
bool make_region_tmap(CUtensorMap* map, const double* base, int cols, int rows, int64_t ncols, int64_t batch,
                      int64_t ld, int64_t bs, int box_w, int box_h);

// fp64 tensor-core (DMMA) products of the recycle update (kr_gemm.cu).
// gram: G_b[i][j] = x_i . y_j over n (row-major G; sym: lower triangle computed and mirrored).
// dims (nullable, device): per-sample live rows -- rows past them are zero pad rows and are
// skipped (their products come out as exact zeros); dims_mask bit 0: bounds X's rows, bit 1: Y's.
int64_t gram_dmma_workspace(int batch, int rx, int ry, int64_t n, bool sym);
int gram_dmma(const double* X, int64_t ldx, int64_t bsx, const double* Y, int64_t ldy, int64_t bsy, int batch, int rx,
              int ry, int64_t n, bool sym, double* G, int64_t ldg, int64_t bsg, double* work, int64_t work_len,
              cudaStream_t st, const int32_t* dims = nullptr, int dims_mask = 0);
// rows_mul: Y_b (R2 x L) = alpha F_b (R2 x R1) X_b (R1 x L) + beta Y_b; lower: F is lower triangular;
// dims_mask bit 0: dims bounds the live output rows (the others become beta Y), bit 1: the k extent
int rows_mul_dmma(const double* F, int64_t ldf, int64_t sF, const double* X, int64_t ldX, int64_t sX, double* Y,
                  int64_t ldY, int64_t sY, int R2, int R1, int64_t L, int batch, double alpha, double beta, bool lower,
                  cudaStream_t st, const int32_t* dims = nullptr, int dims_mask = 0);

}  // namespace kr

#define KR_CHECK_ARG(cond, msg)                      \
  do {                                               \
    if (!(cond)) return ::kr::fail(KR_EINVAL, msg);  \
  } while (0)

#define KR_TRY(expr)              \
  do {                            \
    int _kr_rc = (expr);          \
    if (_kr_rc != KR_OK) return _kr_rc; \
  } while (0)
