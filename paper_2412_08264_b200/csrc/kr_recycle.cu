// kr_recycle.cu -- the whole-batch recycle update, orchestrated natively.
//
// Same algorithm as paper_2412_08264_b200/batched.py::recycle_update (which stays
// as the readable reference and the tests' comparison point), issued from C++:
// no Python per-op overhead and no GIL, so the sample groups' host threads run
// truly in parallel, and a host round trip only where a decision needs data
// (shifted Cholesky QR, the pivoted rank drop, the Hessian-condition bracket).
//
// Layout: a block of R vectors of length L per sample is "rows" [B][R][L]; in
// cuBLAS terms an L x R column-major matrix with ld L.  Samples carry t_b <= T
// live rows, the rest zero; every Gram gets an identity pad block (kr_chol_inv),
// so the leading t_b block of each factor is the per-sample factor.
//
// Steps (reference lines in recycling.py):
//   1. A = [V_prev, U_prev] rows                                (:187-199)
//   2. W = orth(A): CholQR2; shifted CholeskyQR3 where CholQR2 declines; where
//      cond(A) may exceed 1e9, pivoted QR of the small R factor (kr_qrcp) with the
//      reference's |R_kk| > 1e-10 |R_00| keep rule (Householder R where even
//      shifted CholeskyQR3 is out of range)                    (:187-199)
//   3. HW = H W, Ht = sym(W^T H W)                               (:226-236, :333-336)
//   4. Ritz: s selected eigenpairs of Ht                         (:226-236)
//      RGen: condition bracket of Ht (exact extremes only inside it) (:290-296);
//            [Jt; Ht] = Q R (CholQR2), Q1^T Q1 = Z diag(alpha^2) Z^T for the s
//            selected pairs, alpha / beta column norms, V_H, X = R^-1 Z  (:275-359)
//   5. U~ = W X (or W V_H), H U~ = (H W) X, C R = H U~, U = U~ R^-1  (:362-383)
//   6. Z = W V_H diag(mu) for the NSC rule                      (stopping.py:69-72)

#include <cusolverDn.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <functional>
#include <map>
#include <tuple>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "kr_common.cuh"
#include "kr_internal.h"

extern "C" {
int64_t kr_gram_workspace(int32_t batch, int32_t rows, int64_t n);
int kr_gram(const double* A, const double* B, int64_t ld, int64_t bs, int32_t batch, int32_t rows, int64_t n,
            double* G, int64_t ldg, int64_t bsg, double* work, int64_t work_len, kr_stream_t stream);
int64_t kr_chol_inv_workspace(int32_t batch, int32_t tmax);
int kr_chol_inv(const double* G, int64_t ldg, int64_t bsg, const int32_t* dims, int32_t batch, int32_t tmax,
                int32_t flags, const double* shift, double* F, int64_t ldf, int64_t bsf, double* stats,
                int32_t* info, uint8_t* skipped, double* work, int64_t work_len, kr_stream_t stream);
int64_t kr_syev_select_workspace(int32_t batch, int32_t tmax);
int kr_syev_select(const double* A, int64_t lda, int64_t bsa, const int32_t* dims, int32_t batch, int32_t tmax,
                   int32_t size_code, int32_t s, double* lam, int64_t bsl, double* Z, int64_t ldz, int64_t bsz,
                   int32_t* nsel, double* work, int64_t work_len, kr_stream_t stream);
int kr_qrcp_small_cluster(double* M, const int32_t* dims, int32_t batch, int32_t tmax, double rtol, double* Q,
                          int32_t* rank, int32_t* perm, double* work, int64_t work_len, kr_stream_t stream);
}

namespace kr {
int hvp_cols(const kr_op* op, const double* V, int64_t ldv, int64_t bsv, int32_t ncols, const int32_t* dims,
             double* HV, int64_t ldo, int64_t bso, cudaStream_t stream);
namespace {

constexpr double CHOLQR_TOL = 1e-7;   // recycling.CHOLQR_TOL
constexpr double RANK_TOL = 1e-10;    // recycling.RANK_TOL (recycling.py:194)
constexpr double PIVOT_COND = 1e9;    // below: pivoted QR keeps every column
constexpr double SHIFT_COND_MAX = 1e14;
constexpr double COND_LIMIT = 1e12;   // recycling.py:291
constexpr int RC_TMAX = KR_TMAX;

// ---------------------------------------------------------------- small kernels

// A[b][j] = V_b[j] (j < k_b), U_b[j - k_b] (j < k_b + s_b), 0 otherwise
__global__ void gather_rows_kernel(const double* V, int64_t ld_v, int64_t bs_v, const int32_t* kd, const double* U,
                                   int64_t ld_u, int64_t bs_u, const int32_t* sd, double* A, int T, int64_t n) {
  const int j = blockIdx.x, b = blockIdx.y;
  const int k = kd[b], s = sd[b];
  const double* src = j < k ? V + b * bs_v + (int64_t)j * ld_v
                            : (j < k + s ? U + b * bs_u + (int64_t)(j - k) * ld_u : nullptr);
  double* dst = A + ((int64_t)b * T + j) * n;
  for (int64_t p = threadIdx.x; p < n; p += blockDim.x) dst[p] = src ? src[p] : 0.0;
}

// out[b] = sum of squares of rows x cols block b (rows of length `cols`, row stride ld);
// a CTA per block, 8 independent loads in flight per thread (fixed order: deterministic)
constexpr int FROB_NT = 512;
__global__ void __launch_bounds__(FROB_NT) frob2_kernel(const double* X, int rows, int64_t cols, int64_t ld, int64_t bs,
                                                        double* out) {
  const int b = blockIdx.x;
  const double* Xb = X + b * bs;
  const int total = rows * (int)cols;
  double s[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  for (int e0 = threadIdx.x; e0 < total; e0 += 8 * FROB_NT) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * FROB_NT;
      if (e < total) {
        const int r = e / (int)cols, c = e - r * (int)cols;
        const double v = Xb[(int64_t)r * ld + c];
        s[u] = fma(v, v, s[u]);
      }
    }
  }
  __shared__ double red[8 * 33 + 8];
  double v1[1] = {((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]))};
  block_sum<1>(v1, red);
  if (threadIdx.x == 0) out[b] = red[0];
}

// out[b] = trace of the T x T block b (= ||A_b||_F^2 for a Gram G_b = A_b A_b^T)
__global__ void trace_kernel(const double* G, int T, double* out) {
  const int b = blockIdx.x;
  double s = 0.0;
  for (int i = threadIdx.x; i < T; i += blockDim.x) s += G[(int64_t)b * T * T + (int64_t)i * (T + 1)];
  __shared__ double red[8 * 33 + 8];
  double v1[1] = {s};
  block_sum<1>(v1, red);
  if (threadIdx.x == 0) out[b] = red[0];
}

// Hs = (Ht + Ht^T)/2 (separate output: other blocks read the transposed entries);
// S rows [b][j] = [Jt[b][j][0..p) , Hs[b][j][0..T)]
__global__ void sym_and_s_kernel(const double* Ht, const double* Jt, int p, int T, double* Hs, double* S) {
  const int b = blockIdx.y, j = blockIdx.x;
  const double* H = Ht + (int64_t)b * T * T;
  double* sr = S ? S + ((int64_t)b * T + j) * (p + T) : nullptr;
  for (int i = threadIdx.x; i < T; i += blockDim.x) {
    const double v = 0.5 * (H[(int64_t)j * T + i] + H[(int64_t)i * T + j]);
    Hs[((int64_t)b * T + j) * T + i] = v;
    if (sr) sr[p + i] = v;
  }
  if (sr)
    for (int i = threadIdx.x; i < p; i += blockDim.x) sr[i] = Jt[((int64_t)b * T + j) * p + i];
}

// GSVD epilogue: Y rows [b][q][0..p+T): alpha = ||Y[:p]|| (clamped to [0,1]), beta = ||Y[p:]||,
// mu = alpha/beta, VH = Y[p:]/beta, VHmu = mu VH; bad[b] |= beta == 0 for a selected q
__global__ void gsvd_epilogue_kernel(const double* Y, int p, int T, int s, const int32_t* nsel, double* mu,
                                     double* VH, double* VHmu, int32_t* bad) {
  const int q = blockIdx.x, b = blockIdx.y;
  const double* y = Y + ((int64_t)b * s + q) * (p + T);
  __shared__ double red[8 * 33 + 8];
  double a2[2] = {0.0, 0.0};
  for (int i = threadIdx.x; i < p + T; i += blockDim.x) {
    const double v = y[i];
    if (i < p) a2[0] += v * v; else a2[1] += v * v;
  }
  block_sum<2>(a2, red);
  const double alpha = fmin(fmax(sqrt(red[0]), 0.0), 1.0), beta = sqrt(red[1]);
  const bool live = q < nsel[b];
  const double bs = beta > 0.0 ? beta : 1.0, m = alpha / bs;
  if (threadIdx.x == 0) {
    mu[(int64_t)b * s + q] = live ? m : 0.0;
    if (live && !(beta > 0.0)) bad[b] = 1;
  }
  for (int i = threadIdx.x; i < T; i += blockDim.x) {
    const double v = live ? y[p + i] / bs : 0.0;
    VH[((int64_t)b * s + q) * T + i] = v;
    VHmu[((int64_t)b * s + q) * T + i] = m * v;
  }
}

// rows of X (B, R, L) scaled to unit norm (side M candidates)
__global__ void normalize_rows_kernel(double* X, int R, int64_t L) {
  const int r = blockIdx.x, b = blockIdx.y;
  double* x = X + ((int64_t)b * R + r) * L;
  __shared__ double red[8 * 33 + 8];
  double v[1] = {0.0};
  for (int64_t i = threadIdx.x; i < L; i += blockDim.x) v[0] += x[i] * x[i];
  block_sum<1>(v, red);
  const double nr = sqrt(red[0]), sc = nr > 0.0 ? 1.0 / nr : 1.0;
  for (int64_t i = threadIdx.x; i < L; i += blockDim.x) x[i] *= sc;
}

// Unit rows with the eigensolver's sign convention (largest-|component| positive)
__global__ void normalize_sign_rows_kernel(double* X, int R, int64_t L) {
  const int r = blockIdx.x, b = blockIdx.y;
  double* x = X + ((int64_t)b * R + r) * L;
  __shared__ double red[8 * 33 + 8];
  __shared__ double smax[256];
  __shared__ int64_t simax[256];
  double v[1] = {0.0};
  double best = -1.0;
  int64_t bi = 0;
  for (int64_t i = threadIdx.x; i < L; i += blockDim.x) {
    v[0] += x[i] * x[i];
    if (fabs(x[i]) > best) {
      best = fabs(x[i]);
      bi = i;
    }
  }
  smax[threadIdx.x] = best;
  simax[threadIdx.x] = bi;
  block_sum<1>(v, red);
  if (threadIdx.x == 0) {  // first index of the largest magnitude
    for (int t = 1; t < (int)blockDim.x; ++t)
      if (smax[t] > smax[0] || (smax[t] == smax[0] && simax[t] < simax[0])) {
        smax[0] = smax[t];
        simax[0] = simax[t];
      }
  }
  __syncthreads();
  const double nr = sqrt(red[0]);
  const double sc = (nr > 0.0 ? 1.0 / nr : 1.0) * (x[simax[0]] < 0.0 ? -1.0 : 1.0);
  __syncthreads();
  for (int64_t i = threadIdx.x; i < L; i += blockDim.x) x[i] *= sc;
}

// Q1t[b][c][i] = QS[b][i][c] for c < p: the first p entries of the rows of QS, transposed
__global__ void transpose_head_kernel(const double* QS, int P, int T, int p, double* Q1t) {
  __shared__ double tile[32][33];
  const int b = blockIdx.z;
  const double* src = QS + (int64_t)b * T * P;
  double* dst = Q1t + (int64_t)b * p * T;
  const int i0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int i = i0 + r, cc = c0 + threadIdx.x;
    tile[r][threadIdx.x] = (i < T && cc < p) ? src[(int64_t)i * P + cc] : 0.0;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int cc = c0 + r, i = i0 + threadIdx.x;
    if (cc < p && i < T) dst[(int64_t)cc * T + i] = tile[threadIdx.x][r];
  }
}

// M (column-major, ld T) <- upper triangle of the t x t R held column-major in A (ld n)
__global__ void copy_r_kernel(const double* A, int64_t n, int t, double* M, int T) {
  const int j = blockIdx.x;
  for (int i = threadIdx.x; i < T; i += blockDim.x) M[(int64_t)j * T + i] = (i <= j && j < t) ? A[(int64_t)j * n + i] : 0.0;
}

// ---------------------------------------------------------------- host helpers

// Thrown by Ctx::take when the caller's workspace is exhausted: the piece is never
// handed out, so nothing is queued on memory past the buffer; kr_recycle_update
// catches it at the C boundary and returns KR_ENOMEM.
struct WorkspaceOverrun {
  int64_t used, cap, want;
};

struct Ctx {
  cudaStream_t st;
  double* cur;
  double* end;
  double* base = cur;
  double* take(int64_t cnt) {
    const int64_t c = (cnt + 31) & ~int64_t(31);  // 256-byte aligned pieces
    if (cnt < 0 || cur + c > end) throw WorkspaceOverrun{cur - base, end - base, cnt};
    double* r = cur;
    cur += c;
    return r;
  }
};

// Y rows (B, R2, L) = F rows (B, R2, R1) @ X rows (B, R1, L)  [+ beta Y]; lower: F is a
// lower-triangular factor (the Cholesky-QR passes) -- half the products are skipped
// kdims (device, nullable): per-sample live rows of X -- the k loop stops there (the rows past
// them are zero pad rows)
int rows_mul(Ctx& c, const double* F, int64_t sF, const double* X, int64_t ldX, int64_t sX, double* Y, int64_t ldY,
             int64_t sY, int R2, int R1, int64_t L, int B, double alpha = 1.0, double beta = 0.0, bool lower = false,
             const int32_t* kdims = nullptr) {
  return rows_mul_dmma(F, R1, sF, X, ldX, sX, Y, ldY, sY, R2, R1, L, B, alpha, beta, lower, c.st, kdims,
                       kdims ? 2 : 0);
}
// F = L^-1 D^-1 of a Cholesky-QR pass (identity pad block); dims: per-sample live rows of the
// square product (pad rows of X are zero, so the pad rows of Y come out zero either way)
int rows_mul_lower(Ctx& c, const double* F, int64_t sF, const double* X, int64_t ldX, int64_t sX, double* Y,
                   int64_t ldY, int64_t sY, int R2, int R1, int64_t L, int B, const int32_t* dims = nullptr) {
  return rows_mul_dmma(F, R1, sF, X, ldX, sX, Y, ldY, sY, R2, R1, L, B, 1.0, 0.0, true, c.st, dims, dims ? 3 : 0);
}

// G (B, Rx, Ry) = X rows (Rx, L) Y rows (Ry, L)^T, rows of stride ld; sym: the result is
// symmetric (a Gram, or W^T H W up to roundoff) -- lower tile blocks computed and mirrored
int gram_xy(Ctx& c, const double* X, const double* Y, int64_t ld, int64_t bs, int B, int Rx, int Ry, int64_t L,
            bool sym, double* G, int64_t ldg, int64_t bsg, const int32_t* dims = nullptr) {
  const int64_t wl = gram_dmma_workspace(B, Rx, Ry, L, sym);
  double* ws = c.take(wl);
  return gram_dmma(X, ld, bs, Y, ld, bs, B, Rx, Ry, L, sym, G, ldg, bsg, ws, wl, c.st, dims, dims ? 3 : 0);
}

// G (B, R, R) = X rows (R, L) X^T for short rows (L small)
int small_gram(Ctx& c, const double* X, int64_t ldX, int64_t sX, double* G, int R, int64_t L, int B) {
  return gram_xy(c, X, X, ldX, sX, B, R, R, L, true, G, R, (int64_t)R * R);
}

// G[i][j] = a_i . b_j (row-major); symmetric in exact arithmetic at every call site
// dims (device, nullable): per-sample live rows (zero pad rows past them)
int gram(Ctx& c, const double* A, const double* Bm, int B, int R, int64_t n, double* G,
         const int32_t* dims = nullptr) {
  return gram_xy(c, A, Bm, n, (int64_t)R * n, B, R, R, n, true, G, R, (int64_t)R * R, dims);
}

template <typename T>
int d2h(Ctx& c, std::vector<T>& host, const T* dev, size_t cnt) {
  host.resize(cnt);
  if (cnt == 0) return KR_OK;
  cudaError_t e = cudaMemcpyAsync(host.data(), dev, cnt * sizeof(T), cudaMemcpyDeviceToHost, c.st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c.st);
  return e == cudaSuccess ? KR_OK : fail(KR_ECUDA, std::string("kr_recycle d2h: ") + cudaGetErrorString(e));
}

// Several small device -> host reads with ONE stream synchronisation: the copies go
// into a per-thread pinned staging buffer (a pageable destination would make every
// cudaMemcpyAsync synchronous on its own), then out into the host vectors.
struct Fetch {
  struct Item {
    const void* dev;
    size_t bytes, off;
    std::function<void(const char*)> out;
  };
  std::vector<Item> items;
  size_t total = 0;
  template <typename T>
  Fetch& add(std::vector<T>& host, const T* dev, size_t cnt) {
    const size_t bytes = cnt * sizeof(T), off = (total + 15) & ~(size_t)15;
    total = off + bytes;
    items.push_back({dev, bytes, off, [&host, cnt](const char* src) {
                       host.resize(cnt);
                       if (cnt) memcpy(host.data(), src, cnt * sizeof(T));
                     }});
    return *this;
  }
  int run(Ctx& c) {
    static thread_local char* buf = nullptr;
    static thread_local size_t cap = 0;
    if (total > cap) {
      if (buf) cudaFreeHost(buf);
      cap = std::max<size_t>(total, 65536);
      if (cudaMallocHost(&buf, cap) != cudaSuccess) {
        buf = nullptr;
        cap = 0;
        return fail(KR_ECUDA, "kr_recycle: pinned staging buffer");
      }
    }
    for (const Item& it : items)
      if (it.bytes && cudaMemcpyAsync(buf + it.off, it.dev, it.bytes, cudaMemcpyDeviceToHost, c.st) != cudaSuccess)
        return fail(KR_ECUDA, "kr_recycle fetch");
    const cudaError_t e = cudaStreamSynchronize(c.st);
    if (e != cudaSuccess) return fail(KR_ECUDA, std::string("kr_recycle fetch: ") + cudaGetErrorString(e));
    for (const Item& it : items) it.out(buf + it.off);
    return KR_OK;
  }
};

// Small host -> device uploads through a per-thread pinned ring (no stream sync: each
// upload has its own slot for the duration of one kr_recycle_update call).  An event
// recorded after every upload lets the next call wait for the last one before it
// resets the ring (a call that returned early on an error may leave copies in flight).
struct UpRing {
  char* buf = nullptr;
  size_t cap = 0, off = 0;
  cudaEvent_t done = nullptr;
  bool pending = false;
  int reset() {
    if (pending && done && cudaEventSynchronize(done) != cudaSuccess)
      return fail(KR_ECUDA, "kr_recycle: upload ring wait");
    pending = false;
    off = 0;
    return KR_OK;
  }
};
UpRing& up_ring() {
  static thread_local UpRing r;
  return r;
}

template <typename T>
int h2d(Ctx& c, T* dev, const T* host, size_t cnt) {
  if (cnt == 0) return KR_OK;
  UpRing& r = up_ring();
  const size_t bytes = cnt * sizeof(T), off = (r.off + 15) & ~(size_t)15;
  if (r.buf == nullptr || off + bytes > r.cap) {  // first use / overflow: synchronous fallback
    cudaError_t e = cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, c.st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c.st);
    if (r.buf == nullptr && cudaMallocHost(&r.buf, 1 << 16) == cudaSuccess) r.cap = 1 << 16;
    return e == cudaSuccess ? KR_OK : fail(KR_ECUDA, std::string("kr_recycle h2d: ") + cudaGetErrorString(e));
  }
  memcpy(r.buf + off, host, bytes);
  r.off = off + bytes;
  if (!r.done && cudaEventCreateWithFlags(&r.done, cudaEventDisableTiming) != cudaSuccess)
    return fail(KR_ECUDA, "kr_recycle h2d event");
  cudaError_t e = cudaMemcpyAsync(dev, r.buf + off, bytes, cudaMemcpyHostToDevice, c.st);
  if (e == cudaSuccess) e = cudaEventRecord(r.done, c.st);
  r.pending = true;
  return e == cudaSuccess ? KR_OK : fail(KR_ECUDA, std::string("kr_recycle h2d: ") + cudaGetErrorString(e));
}

// A per-host-thread side stream for independent work inside one orchestrator call:
// fork (side waits for main), enqueue, join (record on side), wait (main waits).
struct SideStream {
  cudaStream_t st = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int init() {
    if (st) return KR_OK;
    int least = 0, greatest = 0;
    cudaDeviceGetStreamPriorityRange(&least, &greatest);
    if (cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, greatest) != cudaSuccess ||
        cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming) != cudaSuccess)
      return fail(KR_ECUDA, "kr_recycle side stream");
    return KR_OK;
  }
  int fork(cudaStream_t main) {
    KR_TRY(init());
    if (cudaEventRecord(ev_fork, main) != cudaSuccess || cudaStreamWaitEvent(st, ev_fork, 0) != cudaSuccess)
      return fail(KR_ECUDA, "kr_recycle fork");
    return KR_OK;
  }
  int join(cudaStream_t) {
    return cudaEventRecord(ev_join, st) == cudaSuccess ? KR_OK : fail(KR_ECUDA, "kr_recycle join");
  }
  int wait(cudaStream_t main) {
    return cudaStreamWaitEvent(main, ev_join, 0) == cudaSuccess ? KR_OK : fail(KR_ECUDA, "kr_recycle wait");
  }
};

SideStream& side_stream() {
  static thread_local SideStream ss;  // one per host thread (device fixed per thread here)
  return ss;
}

// Lowest-priority side stream for the update's big throughput kernel (H W, thousands of
// blocks): with the groups' own streams at high priority, the other sample group's
// latency-bound kernels are dispatched between its blocks instead of queueing behind
// the whole launch (measured: ~1.2 ms waits of the slower group).
struct LowStream {
  cudaStream_t st = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int run_hvp(const kr_op* op, const double* V, int64_t ldv, int64_t bsv, int32_t ncols, const int32_t* dims,
              double* HV, int64_t ldo, int64_t bso, cudaStream_t main) {
    if (!st) {
      int least = 0, greatest = 0;
      cudaDeviceGetStreamPriorityRange(&least, &greatest);
      if (cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, least) != cudaSuccess ||
          cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming) != cudaSuccess)
        return fail(KR_ECUDA, "kr_recycle low-priority stream");
    }
    if (cudaEventRecord(ev_fork, main) != cudaSuccess || cudaStreamWaitEvent(st, ev_fork, 0) != cudaSuccess)
      return fail(KR_ECUDA, "kr_recycle fork");
    KR_TRY(hvp_cols(op, V, ldv, bsv, ncols, dims, HV, ldo, bso, st));
    if (cudaEventRecord(ev_join, st) != cudaSuccess || cudaStreamWaitEvent(main, ev_join, 0) != cudaSuccess)
      return fail(KR_ECUDA, "kr_recycle join");
    return KR_OK;
  }
};

LowStream& low_stream() {
  static thread_local LowStream ls;
  return ls;
}

// The update's latency-bound one-CTA-per-matrix kernels (Cholesky, eigen-select, pivoted
// QR) on a highest-priority side stream: fork, launch, join.  With the group streams at
// default priority, a sample group's critical-path kernel is dispatched ahead of the
// other group's pending GEMM / stencil blocks.
struct HiStream {
  cudaStream_t st = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  template <typename F>
  int run(cudaStream_t main, F&& launch) {
    // off by default: with four sample groups the fork/join events cost more than the priority
    // gains (A/B: 21.0 vs 21.8 ms/step); KR_HI_LATENCY=1 enables it (it helped with two groups)
    static const bool on = getenv("KR_HI_LATENCY") != nullptr && getenv("KR_HI_LATENCY")[0] == '1';
    if (!on) return launch(main);
    if (!st) {
      int least = 0, greatest = 0;
      cudaDeviceGetStreamPriorityRange(&least, &greatest);
      if (cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, greatest) != cudaSuccess ||
          cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming) != cudaSuccess)
        return fail(KR_ECUDA, "kr_recycle high-priority stream");
    }
    if (cudaEventRecord(ev_fork, main) != cudaSuccess || cudaStreamWaitEvent(st, ev_fork, 0) != cudaSuccess)
      return fail(KR_ECUDA, "kr_recycle fork");
    KR_TRY(launch(st));
    if (cudaEventRecord(ev_join, st) != cudaSuccess || cudaStreamWaitEvent(main, ev_join, 0) != cudaSuccess)
      return fail(KR_ECUDA, "kr_recycle join");
    return KR_OK;
  }
};

HiStream& hi_stream() {
  static thread_local HiStream hs;
  return hs;
}

struct Factor {  // one Cholesky-QR factor of a batch: F (B,T,T), info, stats
  double* F;
  int32_t* info;
  double* stats;
};

int chol(Ctx& c, const double* G, const int32_t* dims, int B, int T, bool scale, const double* shift, Factor& f,
         bool partial = false) {
  const int64_t wl = kr_chol_inv_workspace(B, T);
  double* ws = wl > 0 ? c.take(wl) : nullptr;  // packed factors of t > 228 (L2-resident)
  return hi_stream().run(c.st, [&](cudaStream_t st) {
    return kr_chol_inv(G, T, (int64_t)T * T, dims, B, T, (scale ? 1 : 0) | 2 | (partial ? 8 : 0), shift, f.F, T,
                       (int64_t)T * T, f.stats, f.info, nullptr, ws, wl, st);
  });
}

// CholQR2 of rows A (B, T, L) with dims; Q out (B,T,L) (may alias nothing), F = R^{-T} (B,T,T).
// Returns per-sample device flags through `ok_dev` (1 = fine) for the non-robust use.
struct QrOut {
  double* Q;
  double* F;
  Factor f1, f2;
};

int cholqr2(Ctx& c, const double* A, int B, int T, int64_t L, const int32_t* dims, double* tmpQ, QrOut& o) {
  double* G = c.take((int64_t)B * T * T);
  KR_TRY(L >= 4096 ? gram(c, A, A, B, T, L, G) : small_gram(c, A, L, (int64_t)T * L, G, T, L, B));
  KR_TRY(chol(c, G, dims, B, T, true, nullptr, o.f1));
  KR_TRY(rows_mul_lower(c, o.f1.F, (int64_t)T * T, A, L, (int64_t)T * L, tmpQ, L, (int64_t)T * L, T, T, L, B));
  KR_TRY(L >= 4096 ? gram(c, tmpQ, tmpQ, B, T, L, G) : small_gram(c, tmpQ, L, (int64_t)T * L, G, T, L, B));
  KR_TRY(chol(c, G, dims, B, T, false, nullptr, o.f2));
  KR_TRY(rows_mul_lower(c, o.f2.F, (int64_t)T * T, tmpQ, L, (int64_t)T * L, o.Q, L, (int64_t)T * L, T, T, L, B));
  return rows_mul_lower(c, o.f2.F, (int64_t)T * T, o.f1.F, T, (int64_t)T * T, o.F, T, (int64_t)T * T, T, T, T, B);
}

Factor new_factor(Ctx& c, int B, int T) {
  Factor f;
  f.F = c.take((int64_t)B * T * T);
  f.info = reinterpret_cast<int32_t*>(c.take((B + 1) / 2));
  f.stats = c.take(4 * (int64_t)B);
  return f;
}

bool cholqr_ok(const std::vector<int32_t>& info, const std::vector<double>& st, int b) {
  return info[b] < 0 && st[4 * b + 0] > CHOLQR_TOL * st[4 * b + 1] && st[4 * b + 2] > 0.0;
}

// cuSOLVER work size of the Householder branch (geqrf + orgqr of an n x T block)
int64_t house_lwork(int64_t n, int T) {
  // the cuSOLVER size queries are slow host calls and every workspace query makes them:
  // cached per host thread and shape
  // (keyed by device too: the cuSOLVER handles are per device); a failed query is
  // never cached and falls back to a generous bound
  static thread_local std::map<std::tuple<int, int64_t, int>, int64_t> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(dev, n, T);
  const auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  const int64_t fallback = std::max<int64_t>(1 << 20, 64 * (int64_t)T * T);
  cusolverDnHandle_t sh;
  if (cusolver_handle(&sh, nullptr) != KR_OK) return fallback;
  int lw1 = 0, lw2 = 0;
  if (cusolverDnDgeqrf_bufferSize(sh, (int)n, T, nullptr, (int)n, &lw1) != CUSOLVER_STATUS_SUCCESS ||
      cusolverDnDorgqr_bufferSize(sh, (int)n, T, T, nullptr, (int)n, nullptr, &lw2) != CUSOLVER_STATUS_SUCCESS)
    return fallback;
  const int64_t lw = std::max(lw1, lw2);
  cache[key] = lw;
  return lw;
}

// Orthonormal rows Wb (t x n) spanning the candidate rows Ab when the Cholesky-QR passes
// broke down at row k1 (exactly dependent candidates -- late Lanczos bases lose
// orthogonality): rows [0, k1) by shifted CholeskyQR3 (that block factored), rows
// [k1, t) by a Householder QR of the remainder after two block Gram-Schmidt passes
// against them, its completion directions projected twice more and re-orthonormalised
// (CholQR2).  A Householder QR of n x (t - k1) instead of n x t (~0.5 ms instead of ~4.5 ms
// at n = 16384, t = 220).  ok = false: a pass broke down (brk = its row) -- the caller
// retries with a smaller k1 or takes the full Householder QR.
int block_house(Ctx& c, const double* Ab, int t, int k1, int64_t n, double* Wb, double* Rem, double* hwk, int64_t hwl,
                double* tau, bool& ok, int& brk, bool prefix_ready) {
  ok = false;
  brk = -1;
  const int m = t - k1;
  const double one = 1.0, zero = 0.0, mone = -1.0;
  int32_t* dk = reinterpret_cast<int32_t*>(c.take(2));
  int32_t* dm = reinterpret_cast<int32_t*>(c.take(2));
  double* dsh = c.take(1);
  const double sh = 11.0 * ((double)n * k1 + (double)k1 * (k1 + 1)) * 2.220446049250313e-16 * k1;
  KR_TRY(h2d(c, dk, &k1, 1));
  KR_TRY(h2d(c, dm, &m, 1));
  KR_TRY(h2d(c, dsh, &sh, 1));
  double* G = c.take((int64_t)t * t);
  double* Cp = c.take((int64_t)t * t);
  Factor f1 = new_factor(c, 1, k1), f2 = new_factor(c, 1, k1), f3 = new_factor(c, 1, k1);
  Factor g1 = new_factor(c, 1, m), g2 = new_factor(c, 1, m);
  // leading block: shifted CholeskyQR3 into Wb[0, k1), Rem as scratch -- unless the
  // caller's partial Cholesky-QR passes already left those rows orthonormalised
  if (!prefix_ready) {
  KR_TRY(gram(c, Ab, Ab, 1, k1, n, G));
  KR_TRY(chol(c, G, dk, 1, k1, true, dsh, f1));
  KR_TRY(rows_mul(c, f1.F, 0, Ab, n, 0, Rem, n, 0, k1, k1, n, 1));
  KR_TRY(gram(c, Rem, Rem, 1, k1, n, G));
  KR_TRY(chol(c, G, dk, 1, k1, false, nullptr, f2));
  KR_TRY(rows_mul(c, f2.F, 0, Rem, n, 0, Wb, n, 0, k1, k1, n, 1));
  KR_TRY(gram(c, Wb, Wb, 1, k1, n, G));
  KR_TRY(chol(c, G, dk, 1, k1, false, nullptr, f3));
  KR_TRY(rows_mul(c, f3.F, 0, Wb, n, 0, Rem, n, 0, k1, k1, n, 1));
  KR_TRY(cudaMemcpyAsync(Wb, Rem, sizeof(double) * k1 * n, cudaMemcpyDeviceToDevice, c.st) == cudaSuccess
             ? KR_OK : fail(KR_ECUDA, "block_house copy"));
  std::vector<int32_t> a1, a2, a3;
  KR_TRY(Fetch().add(a1, f1.info, 1).add(a2, f2.info, 1).add(a3, f3.info, 1).run(c));
  for (int v : {a1[0], a2[0], a3[0]})
    if (v >= 0 && (brk < 0 || v < brk)) brk = v;
  if (getenv("KR_RECYCLE_DEBUG") && brk >= 0)
    fprintf(stderr, "  block_house t=%d k1=%d leading block breakdown rows %d %d %d\n", t, k1, a1[0], a2[0], a3[0]);
  if (brk >= 0) return KR_OK;
  }
  // remainder rows, projected twice: Rem -= W1 (W1^T Rem)   (column-major n x m / n x k1 views)
  KR_TRY(cudaMemcpyAsync(Rem, Ab + (int64_t)k1 * n, sizeof(double) * m * n, cudaMemcpyDeviceToDevice, c.st) ==
                 cudaSuccess ? KR_OK : fail(KR_ECUDA, "block_house copy"));
  const int64_t pwl = gram_dmma_workspace(1, m, k1, n, false);
  double* pws = c.take(pwl);
  auto project = [&]() -> int {
    for (int pass = 0; pass < 2; ++pass) {
      // Cp (m x k1, row-major) = Rem rows . W1 rows;  Rem -= Cp W1
      KR_TRY(gram_dmma(Rem, n, 0, Wb, n, 0, 1, m, k1, n, false, Cp, k1, 0, pws, pwl, c.st));
      KR_TRY(rows_mul(c, Cp, 0, Wb, n, 0, Rem, n, 0, m, k1, n, 1, -1.0, 1.0));
    }
    return KR_OK;
  };
  KR_TRY(project());
  // Householder QR of the narrow remainder -> orthonormal Q2 (n x m) in Rem
  cusolverDnHandle_t shd;
  KR_TRY(cusolver_handle(&shd, c.st));
  int lw1 = 0, lw2 = 0;
  cusolverDnDgeqrf_bufferSize(shd, (int)n, m, Rem, (int)n, &lw1);
  cusolverDnDorgqr_bufferSize(shd, (int)n, m, m, Rem, (int)n, tau, &lw2);
  const int lw = std::max(lw1, lw2);
  if (hwk == nullptr || lw + 1 > hwl) return fail(KR_ENOMEM, "kr_recycle: block Householder work buffer");
  int32_t* dinfo = reinterpret_cast<int32_t*>(hwk + lw);
  if (cusolverDnDgeqrf(shd, (int)n, m, Rem, (int)n, tau, hwk, lw, dinfo) != CUSOLVER_STATUS_SUCCESS ||
      cusolverDnDorgqr(shd, (int)n, m, m, Rem, (int)n, tau, hwk, lw, dinfo) != CUSOLVER_STATUS_SUCCESS)
    return fail(KR_ECUDA, "kr_recycle: block Householder QR");
  // completion directions of a rank-deficient remainder are not orthogonal to W1: project, CholQR2
  KR_TRY(project());
  double* W2 = Wb + (int64_t)k1 * n;
  KR_TRY(gram(c, Rem, Rem, 1, m, n, G));
  KR_TRY(chol(c, G, dm, 1, m, false, nullptr, g1));
  KR_TRY(rows_mul_lower(c, g1.F, 0, Rem, n, 0, W2, n, 0, m, m, n, 1));
  KR_TRY(gram(c, W2, W2, 1, m, n, G));
  KR_TRY(chol(c, G, dm, 1, m, false, nullptr, g2));
  KR_TRY(rows_mul_lower(c, g2.F, 0, W2, n, 0, Rem, n, 0, m, m, n, 1));
  KR_TRY(cudaMemcpyAsync(W2, Rem, sizeof(double) * m * n, cudaMemcpyDeviceToDevice, c.st) == cudaSuccess
             ? KR_OK : fail(KR_ECUDA, "block_house copy"));
  std::vector<int32_t> b1, b2;
  KR_TRY(Fetch().add(b1, g1.info, 1).add(b2, g2.info, 1).run(c));
  ok = b1[0] < 0 && b2[0] < 0;
  if (getenv("KR_RECYCLE_DEBUG"))
    fprintf(stderr, "  block_house t=%d k1=%d prefix=%d completion breakdown rows %d %d\n", t, k1, (int)prefix_ready,
            b1[0], b2[0]);
  return KR_OK;
}

int64_t workspace_doubles(const kr_op& op, const kr_recycle_args& a) {
  // generous per-term budget: every Ctx::take of kr_recycle_update is covered with
  // margin (each take also rounds up to 32 doubles); overruns are reported
  const int64_t B = a.batch, T = a.T, n = op_n(op), s = a.s;
  const int64_t p = op.reg_kind == KR_REG_TV ? 1 : (int64_t)op.num_filters * (1 + op.ksize * op.ksize);
  const int64_t P = p + T;
  int64_t w = 0;
  w += 2 * B * T * n;                                   // A, tmpQ
  w += 30 * (B * T * T + 4 * B + 64);                   // T x T factors, Grams, Ht, Hs, Mq, M, Q_R (+ harmonic pencil)
  w += 5 * B * T * P;                                   // Jt, S, QS, CholQR tmp
  w += 8 * B * s * T + 2 * B * s * P;                   // Z, X, coeffs, VH mu, Y, extremes
  w += 4 * B * s * n + 8 * (B * s * s + 4 * B + 64);    // cand, HU, CholQR tmp; prepare factors
  w += 8 * kr_gram_workspace((int32_t)B, (int32_t)T, n);
  w += kr_jadj_workspace(&op, (int32_t)T) + 3 * kr_syev_select_workspace((int32_t)B, (int32_t)T);
  w += house_lwork(n, (int)T) + 64;                     // Householder branch (cuSOLVER work)
  w += T * n + 16 * (T * T + 64);                       // block-Householder branch: remainder rows, factors
  w += 8 * T * T + 4 * T + 65536;                       // pivoted path (tau), slack
  w += 12 * (kr_chol_inv_workspace((int32_t)B, (int32_t)T) + 64);  // packed factors of t > 228 (per Cholesky)
  w += 24 * (kr_chol_inv_workspace(1, (int32_t)T) + 64);          // block-Householder branch's factors
  return w;
}

}  // namespace
}  // namespace kr

using namespace kr;


extern "C" int kr_thread_warmup(void) {
  cusolverDnHandle_t sh;
  KR_TRY(cusolver_handle(&sh, nullptr));
  // one tiny Householder QR on this thread's handle (first-call setup off the hot path)
  const int m = 64, q = 8;
  int lw1 = 0, lw2 = 0;
  cusolverDnDgeqrf_bufferSize(sh, m, q, nullptr, m, &lw1);
  cusolverDnDorgqr_bufferSize(sh, m, q, q, nullptr, m, nullptr, &lw2);
  const int lw = std::max(lw1, lw2);
  double* buf = nullptr;
  if (cudaMalloc(&buf, sizeof(double) * ((size_t)m * q + q + lw + 1)) != cudaSuccess)
    return fail(KR_ENOMEM, "kr_thread_warmup");
  cudaMemset(buf, 0, sizeof(double) * m * q);
  double* A = buf;
  double* tau = A + m * q;
  double* wk = tau + q;
  int32_t* info = reinterpret_cast<int32_t*>(wk + lw);
  const double one = 1.0;
  for (int i = 0; i < q; ++i) cudaMemcpy(A + (size_t)i * m + i, &one, sizeof(double), cudaMemcpyHostToDevice);
  cusolverDnDgeqrf(sh, m, q, A, m, tau, wk, lw, info);
  cusolverDnDorgqr(sh, m, q, q, A, m, tau, wk, lw, info);
  const cudaError_t e = cudaDeviceSynchronize();
  cudaFree(buf);
  return e == cudaSuccess ? KR_OK : fail(KR_ECUDA, "kr_thread_warmup");
}

extern "C" int64_t kr_recycle_workspace(const kr_op* op, const kr_recycle_args* a) {
  if (!op || !a || validate_op(*op) != KR_OK) return -1;
  return workspace_doubles(*op, *a);
}

static int recycle_update_impl(const kr_op* op, const kr_recycle_args* a, double* work, int64_t work_len,
                               kr_stream_t stream);

extern "C" int kr_recycle_update(const kr_op* op, const kr_recycle_args* a, double* work, int64_t work_len,
                                 kr_stream_t stream) {
  try {
    return recycle_update_impl(op, a, work, work_len, stream);
  } catch (const WorkspaceOverrun& e) {
    char msg[200];
    snprintf(msg, sizeof msg, "kr_recycle_update: workspace exhausted (%lld of %lld doubles used, %lld more asked)",
             (long long)e.used, (long long)e.cap, (long long)e.want);
    return fail(KR_ENOMEM, msg);
  }
}

static int recycle_update_impl(const kr_op* op, const kr_recycle_args* a, double* work, int64_t work_len,
                               kr_stream_t stream) {
  KR_CHECK_ARG(op && a, "null argument");
  KR_TRY(validate_op(*op));
  const int B = a->batch, T = a->T, s = a->s;
  const int64_t n = op_n(*op);
  KR_CHECK_ARG(op->batch == B, "operator batch must equal args.batch");
  KR_CHECK_ARG(T >= 1 && T <= RC_TMAX && s >= 1 && s <= T, "need 1 <= s <= T <= KR_TMAX");
  KR_CHECK_ARG(a->vec_type == 0 || a->vec_type == 2 || (a->vec_type == 1 && a->size_code == 1),
               "vec_type: Ritz, harmonic Ritz, or RGen with size L");
  KR_CHECK_ARG(a->vec_type == 0 || op->reg_kind != KR_REG_NONE, "RGen needs a mixed Jacobian");
  KR_CHECK_ARG(work && work_len >= workspace_doubles(*op, *a), "kr_recycle workspace too small");
  const int p = op->reg_kind == KR_REG_TV ? 1 : op->num_filters * (1 + op->ksize * op->ksize);
  const int P = p + T;
  // inner placement (recycling.py:409-415): project with the previous system's operator
  const kr_op* pop = a->op_proj ? a->op_proj : op;
  const bool inner = a->op_proj != nullptr;
  if (inner) {
    KR_TRY(validate_op(*pop));
    KR_CHECK_ARG(pop->batch == B && pop->rows == op->rows && pop->cols == op->cols && pop->reg_kind == op->reg_kind &&
                     pop->num_filters == op->num_filters && pop->ksize == op->ksize,
                 "op_proj must describe the same batch and model family as op");
  }
  Ctx c{(cudaStream_t)stream, work, work + work_len};
  KR_TRY(up_ring().reset());
  static const bool debug = getenv("KR_RECYCLE_DEBUG") != nullptr;
  const auto t_start = std::chrono::steady_clock::now();
  int n_ill = 0, n_house = 0, n_exact = 0, n_block = 0;
  double house_ms = 0.0;
  bool was_shifted = false;
  std::vector<int32_t> t(B), status(B, 0);
  for (int b = 0; b < B; ++b) t[b] = a->kdims[b] + a->sdims[b];

  // ---- 1. candidates A = [V_prev, U_prev] rows
  int32_t* dd = reinterpret_cast<int32_t*>(c.take(B * 4 + 8));  // device ints: kd, sd, td, nsel, misc
  int32_t* d_kd = dd;
  int32_t* d_sd = dd + B;
  int32_t* d_td = dd + 2 * B;
  int32_t* d_ns = dd + 3 * B;
  int32_t* d_bad = dd + 4 * B;
  {
    std::vector<int32_t> hk(5 * B, 0);
    for (int b = 0; b < B; ++b) {
      hk[b] = a->kdims[b];
      hk[B + b] = a->sdims[b];
      hk[2 * B + b] = t[b];
    }
    KR_TRY(h2d(c, dd, hk.data(), hk.size()));
  }
  double* A = c.take((int64_t)B * T * n);
  double* tmpQ = c.take((int64_t)B * T * n);
  gather_rows_kernel<<<dim3(T, B), 256, 0, c.st>>>(a->V, a->ld_v, a->bs_v, d_kd, a->Uprev, a->ld_u, a->bs_u, d_sd, A,
                                                   T, n);
  KR_TRY(check_launch("gather_rows"));

  // ---- 2. W = orth(A) with the reference's rank drop
  double* W = a->W;
  Factor f1 = new_factor(c, B, T), f2 = new_factor(c, B, T), f3 = new_factor(c, B, T);
  double* G = c.take((int64_t)B * T * T);
  double* F = c.take((int64_t)B * T * T);
  double* Ft = c.take((int64_t)B * T * T);
  KR_TRY(gram(c, A, A, B, T, n, G, d_td));
  double* nrm = c.take(2 * B);  // ||A||_F^2 = tr(A A^T) (the Gram is reused below), ||R^-1||_F^2
  trace_kernel<<<B, 256, 0, c.st>>>(G, T, nrm);
  // (partial factors: a sample whose passes break down keeps its orthonormalised leading
  // rows -- the block-Householder branch below starts from them)
  KR_TRY(chol(c, G, d_td, B, T, true, nullptr, f1, true));
  std::vector<int32_t> info1;
  std::vector<double> st1;
  KR_TRY(Fetch().add(info1, f1.info, B).add(st1, f1.stats, 4 * B).run(c));
  std::vector<char> ok1(B);
  bool shifted = false;
  for (int b = 0; b < B; ++b) {
    ok1[b] = t[b] == 0 || cholqr_ok(info1, st1, b);
    shifted |= !ok1[b];
  }
  if (shifted) {  // shifted CholeskyQR3 for the declined samples (sigma = 11 (n t + t(t+1)) u t)
    std::vector<double> sh(B, 0.0);
    for (int b = 0; b < B; ++b)
      if (!ok1[b]) {
        const double tb = t[b];
        sh[b] = 11.0 * (n * tb + tb * (tb + 1)) * 2.220446049250313e-16 * tb;
      }
    double* d_sh = c.take(B);
    KR_TRY(h2d(c, d_sh, sh.data(), B));
    KR_TRY(chol(c, G, d_td, B, T, true, d_sh, f1, true));
  }
  std::vector<int32_t> is1;
  if (shifted) KR_TRY(d2h(c, is1, f1.info, B));
  // first pass into tmpQ or W so that the last pass lands in W (no B x T x n copy back)
  const int npass = shifted ? 2 : 1;
  double* first = (npass % 2 == 1) ? tmpQ : W;
  KR_TRY(rows_mul_lower(c, f1.F, (int64_t)T * T, A, n, (int64_t)T * n, first, n, (int64_t)T * n, T, T, n, B, d_td));
  // second pass (and third when shifted)
  Factor* fp[2] = {&f2, &f3};
  double* cur = first;
  double* nxt = first == W ? tmpQ : W;
  KR_TRY(cudaMemcpyAsync(F, f1.F, sizeof(double) * B * T * T, cudaMemcpyDeviceToDevice, c.st) == cudaSuccess
             ? KR_OK : fail(KR_ECUDA, "kr_recycle copy"));
  for (int pass = 0; pass < npass; ++pass) {
    KR_TRY(gram(c, cur, cur, B, T, n, G, d_td));
    KR_TRY(chol(c, G, d_td, B, T, false, nullptr, *fp[pass], true));
    KR_TRY(rows_mul_lower(c, fp[pass]->F, (int64_t)T * T, cur, n, (int64_t)T * n, nxt, n, (int64_t)T * n, T, T, n, B, d_td));
    KR_TRY(rows_mul_lower(c, fp[pass]->F, (int64_t)T * T, F, T, (int64_t)T * T, Ft, T, (int64_t)T * T, T, T, T, B));
    std::swap(F, Ft);
    std::swap(cur, nxt);
  }
  if (cur != W) KR_TRY(cudaMemcpyAsync(W, cur, sizeof(double) * B * T * n, cudaMemcpyDeviceToDevice, c.st) == cudaSuccess
                           ? KR_OK : fail(KR_ECUDA, "kr_recycle copy W"));
  // condition bound ||A||_F ||R^-1||_F and the later passes' breakdowns
  frob2_kernel<<<B, FROB_NT, 0, c.st>>>(F, T, T, T, (int64_t)T * T, nrm + B);
  std::vector<double> nr;
  std::vector<int32_t> i2, i3;
  {
    Fetch fe;
    fe.add(nr, nrm, 2 * B).add(i2, f2.info, B);
    if (shifted) fe.add(i3, f3.info, B);
    KR_TRY(fe.run(c));
  }
  std::vector<int> ill, hh;  // samples for the pivoted path; of those, the ones needing Householder
  for (int b = 0; b < B; ++b) {
    if (t[b] == 0) continue;
    const double cb = sqrt(nr[b]) * sqrt(nr[B + b]);
    // CholQR2 (ok1) or shifted CholeskyQR3 that factored and stayed within its range
    const bool okb = shifted ? (is1[b] < 0 && i2[b] < 0 && i3[b] < 0 && (ok1[b] || cb <= SHIFT_COND_MAX))
                             : (ok1[b] && i2[b] < 0);
    if (!okb || cb > PIVOT_COND) {
      ill.push_back(b);
      if (!okb) hh.push_back(b);
    }
    if (debug && (!okb || cb > PIVOT_COND))
      fprintf(stderr, "  sample %d t=%d cb=%.3e ok1=%d shifted=%d is1=%d i2=%d i3=%d -> %s\n", b, t[b], cb, (int)ok1[b],
              (int)shifted, shifted ? is1[b] : -9, i2[b], shifted ? i3[b] : -9, okb ? "pivoted" : "householder");
  }
  n_ill = (int)ill.size();
  n_house = (int)hh.size();
  std::vector<int> brow(B, -1);  // first breakdown row of the Cholesky-QR passes (-1: none)
  for (int b : hh) {
    int r = -1;
    for (int v : {shifted ? is1[b] : -1, i2[b], shifted ? i3[b] : -1})
      if (v >= 0 && (r < 0 || v < r)) r = v;
    // no breakdown of the shifted passes but a condition bound beyond their range: split at
    // the unshifted first pass's breakdown row (the leading rows of the successful shifted
    // passes are the shifted CholeskyQR3 of the leading, well-conditioned block)
    if (r < 0 && info1[b] >= 0) r = info1[b];
    brow[b] = r;
  }
  was_shifted = shifted;
  if (!ill.empty()) {
    const int nb = (int)ill.size();
    double* M = c.take((int64_t)nb * T * T);
    double* Qr = c.take((int64_t)nb * T * T);
    int32_t* d_misc = reinterpret_cast<int32_t*>(c.take(2 * nb + 2));
    int32_t* d_rank = d_misc + nb;
    std::vector<int32_t> tdim(nb);
    for (int i = 0; i < nb; ++i) tdim[i] = t[ill[i]];
    KR_TRY(h2d(c, d_misc, tdim.data(), nb));
    double* tau = c.take(T);
    double* hwk = nullptr;
    int64_t hwl = 0;
    double* house_rem = nullptr;  // remainder rows of the block Householder branch
    if (!hh.empty()) {
      hwl = house_lwork(n, T) + 1;
      hwk = c.take(hwl);
      house_rem = c.take((int64_t)T * n);
    }
    // R factors: from the Cholesky-QR basis (R^T = A W^T) or a Householder QR
    for (int i = 0; i < nb; ++i) {
      const int b = ill[i];
      const double one = 1.0, zero = 0.0;
      bool house = std::find(hh.begin(), hh.end(), b) != hh.end();
      // Cholesky-QR broke down at a row: block Householder, where the full one is expensive
      // (n t >= 2^21: ~1 ms and up; small problems keep the full Householder QR)
      if (house && brow[b] >= t[b] / 2 && n * (int64_t)t[b] >= ((int64_t)1 << 21)) {
        if (debug) cudaStreamSynchronize(c.st);
        const auto th0 = std::chrono::steady_clock::now();
        double* Wb = W + (int64_t)b * T * n;
        // rows [0, brow) of W are the partial passes' orthonormalised leading rows; rows
        // [t, T) stay zero; [brow, t) are written by block_house
        if (T > t[b])
          KR_TRY(cudaMemsetAsync(Wb + (int64_t)t[b] * n, 0, sizeof(double) * (T - t[b]) * n, c.st) == cudaSuccess
                     ? KR_OK : fail(KR_ECUDA, "memset"));
        int k1 = brow[b];
        for (int attempt = 0; attempt < 4 && house; ++attempt) {
          bool ok = false;
          int brk = -1;
          KR_TRY(block_house(c, A + (int64_t)b * T * n, t[b], k1, n, Wb, house_rem, hwk, hwl, tau, ok, brk,
                             attempt == 0));
          if (ok) {
            house = false;
            ++n_block;
          } else if (attempt == 0) {
            continue;  // recompute the leading block (shifted CholeskyQR3) instead of reusing it
          } else if (brk >= t[b] / 2 && brk < k1) {
            k1 = brk;
          } else {
            break;
          }
        }
        if (debug) {
          cudaStreamSynchronize(c.st);
          house_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - th0).count();
        }
      }
      if (!house) {  // M column-major R: M[j][i] = a_j . w_i  (col-major M (T x T) = W_col^T A_col)
        KR_TRY(gram_xy(c, A + (int64_t)b * T * n, W + (int64_t)b * T * n, n, 0, 1, T, T, n, false,
                       M + (int64_t)i * T * T, T, 0));
      } else {  // Householder: geqrf/orgqr on A_b (n x t column-major == its rows), W_b = Q rows
        // rare path (rank-deficient candidates): the LAPACK work buffer is sized by cuSOLVER,
        // so it is allocated stream-ordered here instead of from the caller's workspace
        if (debug) cudaStreamSynchronize(c.st);
        const auto th0 = std::chrono::steady_clock::now();
        cusolverDnHandle_t sh;
        KR_TRY(cusolver_handle(&sh, c.st));
        double* Ab = A + (int64_t)b * T * n;
        const int tb = t[b];
        int lw1 = 0, lw2 = 0;
        cusolverDnDgeqrf_bufferSize(sh, (int)n, tb, Ab, (int)n, &lw1);
        cusolverDnDorgqr_bufferSize(sh, (int)n, tb, tb, Ab, (int)n, tau, &lw2);
        const int lw = std::max(lw1, lw2);
        if (hwk == nullptr || lw + 1 > hwl) return fail(KR_ENOMEM, "kr_recycle: Householder work buffer");
        double* wk = hwk;
        int32_t* dinfo = reinterpret_cast<int32_t*>(wk + lw);
        const bool qok = cusolverDnDgeqrf(sh, (int)n, tb, Ab, (int)n, tau, wk, lw, dinfo) == CUSOLVER_STATUS_SUCCESS;
        copy_r_kernel<<<T, 256, 0, c.st>>>(Ab, n, tb, M + (int64_t)i * T * T, T);
        const bool gok = qok && cusolverDnDorgqr(sh, (int)n, tb, tb, Ab, (int)n, tau, wk, lw, dinfo) ==
                                    CUSOLVER_STATUS_SUCCESS;
        cudaMemsetAsync(W + (int64_t)b * T * n, 0, sizeof(double) * T * n, c.st);
        cudaMemcpyAsync(W + (int64_t)b * T * n, Ab, sizeof(double) * tb * n, cudaMemcpyDeviceToDevice, c.st);
        if (debug) {
          cudaStreamSynchronize(c.st);
          house_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - th0).count();
        }
        if (!gok) return fail(KR_ECUDA, "kr_recycle: Householder QR");
      }
    }
    double* qw = c.take(nb * T + 1);
    KR_TRY(hi_stream().run(c.st, [&](cudaStream_t st) {
      return kr_qrcp_small_cluster(M, d_misc, nb, T, RANK_TOL, Qr, d_rank, nullptr, qw, nb * T + 1, st);
    }));
    // W_b <- Q_R[:, :r]^T W_b  (rows beyond the rank are zero)
    for (int i = 0; i < nb; ++i) {
      const int b = ill[i];
      KR_TRY(rows_mul(c, Qr + (int64_t)i * T * T, 0, W + (int64_t)b * T * n, n, 0, tmpQ, n, 0, T, T, n, 1));
      KR_TRY(cudaMemcpyAsync(W + (int64_t)b * T * n, tmpQ, sizeof(double) * T * n, cudaMemcpyDeviceToDevice, c.st)
                     == cudaSuccess ? KR_OK : fail(KR_ECUDA, "kr_recycle copy"));
    }
    std::vector<int32_t> rk;
    KR_TRY(d2h(c, rk, d_rank, nb));
    for (int i = 0; i < nb; ++i) t[ill[i]] = rk[i];
    std::vector<int32_t> ht(t.begin(), t.end());
    KR_TRY(h2d(c, d_td, ht.data(), B));
  }

  // ---- 3. H W and the projected Hessian
  double* HW = a->HW;
  static const bool lowpri = getenv("KR_HVP_LOWPRI") == nullptr || getenv("KR_HVP_LOWPRI")[0] != '0';
  if (lowpri)
    KR_TRY(low_stream().run_hvp(pop, W, n, (int64_t)T * n, T, d_td, HW, n, (int64_t)T * n, c.st));
  else
    KR_TRY(hvp_cols(pop, W, n, (int64_t)T * n, T, d_td, HW, n, (int64_t)T * n, c.st));
  double* Ht = c.take((int64_t)B * T * T);
  KR_TRY(gram(c, W, HW, B, T, n, Ht, d_td));
  double* coeffs = c.take((int64_t)B * s * T);
  double* Xc = nullptr;
  double* VHmu = nullptr;
  std::vector<int32_t> bad(B, 0);
  if (a->vec_type == 0 || a->vec_type == 2) {
    // Ritz (ritz_select, recycling.py:226-236): eigenpairs of sym(W^T H W).
    // Harmonic Ritz (harmonic_ritz_select, :239-272): the pencil A rho = theta B rho with
    // A = sym((HW)^T HW), B = sym((HW)^T W) = sym(W^T H W), reduced by B's Cholesky factor
    // (F = L^-1 D^-1, F B F^T = I): M = F A F^T, rho = F^T z, selection by |theta| (theta > 0
    // for SPD H), candidates W rho / ||W rho|| (= rho / ||rho||, W orthonormal).  A
    // near-singular B (the reference's null-direction branch) is declined to the
    // per-sample path.
    double* Hs = c.take((int64_t)B * T * T);
    sym_and_s_kernel<<<dim3(T, B), 256, 0, c.st>>>(Ht, nullptr, 0, T, Hs, nullptr);
    Ht = Hs;
    double* Msel = Ht;
    Factor fb;
    if (a->vec_type == 2) {
      double* Ag = c.take((int64_t)B * T * T);
      KR_TRY(gram(c, HW, HW, B, T, n, Ag));
      double* As = c.take((int64_t)B * T * T);
      sym_and_s_kernel<<<dim3(T, B), 256, 0, c.st>>>(Ag, nullptr, 0, T, As, nullptr);
      fb = new_factor(c, B, T);
      KR_TRY(chol(c, Ht, d_td, B, T, true, nullptr, fb));
      double* FA = c.take((int64_t)B * T * T);
      double* Mh = c.take((int64_t)B * T * T);
      KR_TRY(rows_mul(c, fb.F, (int64_t)T * T, As, T, (int64_t)T * T, FA, T, (int64_t)T * T, T, T, T, B));
      // Mh = (F A) F^T = F A F^T (symmetric): Mh[i][j] = (FA)_i . F_j
      KR_TRY(gram_xy(c, FA, fb.F, T, (int64_t)T * T, B, T, T, T, false, Mh, T, (int64_t)T * T));
      Msel = Mh;
    }
    const int64_t el = kr_syev_select_workspace(B, T);
    double* zc = a->vec_type == 2 ? c.take((int64_t)B * s * T) : coeffs;
    KR_TRY(hi_stream().run(c.st, [&](cudaStream_t st) { return kr_syev_select(Msel, T, (int64_t)T * T, d_td, B, T, a->size_code, s, nullptr, 0, zc, T,
                          (int64_t)s * T, d_ns, c.take(el), el, st); }));
    if (a->vec_type == 2) {
      KR_TRY(rows_mul(c, zc, (int64_t)s * T, fb.F, T, (int64_t)T * T, coeffs, T, (int64_t)s * T, s, T, T, B));
      normalize_rows_kernel<<<dim3(s, B), 256, 0, c.st>>>(coeffs, s, T);
      std::vector<int32_t> bi;
      std::vector<double> bst;
      KR_TRY(Fetch().add(bi, fb.info, B).add(bst, fb.stats, 4 * B).run(c));
      for (int b = 0; b < B; ++b) {
        const double r = bst[4 * b + 1] > 0.0 ? bst[4 * b] / bst[4 * b + 1] : 0.0;
        if (t[b] > 0 && !(bi[b] < 0 && r * r > 10.0 * RANK_TOL)) {
          status[b] = 1;  // (near-)singular pencil: the reference restricts to B's non-null directions
          if (debug) fprintf(stderr, "  sample %d declined: harmonic pencil B (info %d, pivot ratio %.3e)\n", b, bi[b], r);
        }
      }
    }
  } else {
    // J W
    double* Jt = c.take((int64_t)B * T * p);
    const int64_t jl = kr_jadj_workspace(pop, T);
    KR_TRY(kr_jadj(pop, W, n, (int64_t)T * n, T, Jt, p, (int64_t)T * p, c.take(jl), jl, c.st));
    double* S = c.take((int64_t)B * T * P);
    double* Hs = c.take((int64_t)B * T * T);
    sym_and_s_kernel<<<dim3(T, B), 256, 0, c.st>>>(Ht, Jt, p, T, Hs, S);
    Ht = Hs;
    // condition bracket of Ht: (max L_jj / min L_jj)^2 <= cond <= ||Ht||_F ||L^-1||_F^2
    // (on a side stream: independent of the GSVD's CholQR2 below, whose one-CTA-per-matrix
    // Cholesky kernels it would otherwise wait behind)
    Factor fh = new_factor(c, B, T);
    double* hn = c.take(2 * B);
    SideStream& ss = side_stream();
    KR_TRY(ss.fork(c.st));
    const int64_t hwl_c = kr_chol_inv_workspace(B, T);
    double* hws_c = hwl_c > 0 ? c.take(hwl_c) : nullptr;
    KR_TRY(kr_chol_inv(Ht, T, (int64_t)T * T, d_td, B, T, 2, nullptr, fh.F, T, (int64_t)T * T, fh.stats, fh.info,
                       nullptr, hws_c, hwl_c, ss.st));
    frob2_kernel<<<B, FROB_NT, 0, ss.st>>>(Ht, T, T, T, (int64_t)T * T, hn);
    frob2_kernel<<<B, FROB_NT, 0, ss.st>>>(fh.F, T, T, T, (int64_t)T * T, hn + B);
    KR_TRY(ss.join(c.st));  // joined before the host reads hn / fh (below, after the eigen launch)
    bool joined = false;
    // GSVD: [Jt; Ht] = Q R (CholQR2 of the rows of S)
    QrOut qs;
    qs.Q = c.take((int64_t)B * T * P);
    qs.F = c.take((int64_t)B * T * T);
    qs.f1 = new_factor(c, B, T);
    qs.f2 = new_factor(c, B, T);
    KR_TRY(cholqr2(c, S, B, T, P, d_td, c.take((int64_t)B * T * P), qs));
    // Right singular vectors of Q1 (= first p entries of every row of QS) for the s largest
    // alpha: eigenvectors of Q1^T Q1 (t x t).  When every sample has more candidates than
    // parameters (t_b > p: Q1^T Q1 has rank <= p) and the t x t problem is beyond the
    // shared-memory eigensolver while p x p is not, the same vectors come from the p x p dual
    // Q1 Q1^T y = alpha^2 y as z = Q1^T y / alpha (well conditioned for the LARGEST alpha, the
    // only ones size L selects): C3 at steady state t = 330, p = 208 -- 13 ms of one-CTA-per-
    // matrix eigensolver on the update's critical chain become ~1.5 ms.
    int tmin = T;
    for (int b = 0; b < B; ++b) tmin = t[b] < tmin ? t[b] : tmin;
    const char* de = getenv("KR_GSVD_DUAL");  // (read per call: the tests run both forms)
    const bool dual_off = de && de[0] == '0';
    const bool dual = !dual_off && T > 228 && p <= 228 && p >= s && tmin > p;
    const int64_t el = kr_syev_select_workspace(B, dual ? p : T);
    double* Zs = c.take((int64_t)B * s * T);
    if (!dual) {
      double* Mq = c.take((int64_t)B * T * T);
      KR_TRY(small_gram(c, qs.Q, P, (int64_t)T * P, Mq, T, p, B));
      KR_TRY(hi_stream().run(c.st, [&](cudaStream_t st) { return kr_syev_select(Mq, T, (int64_t)T * T, d_td, B, T, 1, s, nullptr, 0, Zs, T, (int64_t)s * T, d_ns,
                            c.take(el), el, st); }));
    } else {
      double* Q1t = c.take((int64_t)B * p * T);
      transpose_head_kernel<<<dim3((T + 31) / 32, (p + 31) / 32, B), dim3(32, 8), 0, c.st>>>(qs.Q, P, T, p, Q1t);
      KR_TRY(check_launch("transpose_head"));
      double* Md = c.take((int64_t)B * p * p);  // Q1 Q1^T
      KR_TRY(rows_mul(c, Q1t, (int64_t)p * T, qs.Q, P, (int64_t)T * P, Md, p, (int64_t)p * p, p, T, p, B));
      int32_t* d_pd = reinterpret_cast<int32_t*>(c.take((B + 1) / 2 + 1));
      {
        std::vector<int32_t> hp(B, p);
        KR_TRY(h2d(c, d_pd, hp.data(), B));
      }
      double* Yd = c.take((int64_t)B * s * p);
      KR_TRY(hi_stream().run(c.st, [&](cudaStream_t st) { return kr_syev_select(Md, p, (int64_t)p * p, d_pd, B, p, 1, s, nullptr, 0, Yd, p, (int64_t)s * p, d_ns,
                            c.take(el), el, st); }));
      KR_TRY(rows_mul(c, Yd, (int64_t)s * p, Q1t, T, (int64_t)p * T, Zs, T, (int64_t)s * T, s, p, T, B));
      normalize_sign_rows_kernel<<<dim3(s, B), 256, 0, c.st>>>(Zs, s, T);
      KR_TRY(check_launch("normalize_sign_rows"));
    }
    // the bracket decision (host), overlapping the eigen kernel
    if (!joined) {
      KR_TRY(ss.wait(c.st));
      joined = true;
    }
    std::vector<double> hnv, hst;
    std::vector<int32_t> hinf;
    KR_TRY(Fetch().add(hnv, hn, 2 * B).add(hst, fh.stats, 4 * B).add(hinf, fh.info, B).run(c));
    std::vector<int> exact;
    for (int b = 0; b < B; ++b) {
      if (t[b] == 0) continue;
      const double ub = sqrt(hnv[b]) * hnv[B + b];
      const bool scr = hinf[b] < 0 && hst[4 * b] > 0.0 && ub < COND_LIMIT;
      if (!scr) exact.push_back(b);
    }
    n_exact = (int)exact.size();
    if (!exact.empty()) {  // exact extreme eigenvalues where the bracket straddles the limit
      double* ext = c.take(2 * (int64_t)B);
      double* zz = c.take(2 * (int64_t)B * T);
      const int64_t elT = kr_syev_select_workspace(B, T);
      KR_TRY(hi_stream().run(c.st, [&](cudaStream_t st) { return kr_syev_select(Ht, T, (int64_t)T * T, d_td, B, T, 2, 2, ext, 2, zz, T, 2 * (int64_t)T, nullptr,
                            c.take(elT), elT, st); }));
      std::vector<double> ex;
      KR_TRY(d2h(c, ex, ext, 2 * B));
      for (int b : exact) {
        const double lo = ex[2 * b], hi = ex[2 * b + 1], smax = std::max(fabs(lo), fabs(hi));
        if (!(lo > 0.0 && lo >= smax / COND_LIMIT)) status[b] = 1;  // singular: the per-sample path raises
        if (debug && status[b]) fprintf(stderr, "  sample %d declined: W^T H W singular (lo %.3e hi %.3e)\n", b, lo, hi);
      }
    }
    // alpha, beta, mu, V_H from Y = Z Q^T rows; X = R^-1 z
    double* Y = c.take((int64_t)B * s * P);
    KR_TRY(rows_mul(c, Zs, (int64_t)s * T, qs.Q, P, (int64_t)T * P, Y, P, (int64_t)s * P, s, T, P, B));
    double* VHv = a->VH;
    VHmu = c.take((int64_t)B * s * T);
    KR_TRY(cudaMemsetAsync(d_bad, 0, sizeof(int32_t) * B, c.st) == cudaSuccess ? KR_OK : fail(KR_ECUDA, "memset"));
    gsvd_epilogue_kernel<<<dim3(s, B), 256, 0, c.st>>>(Y, p, T, s, d_ns, a->mu, VHv, VHmu, d_bad);
    Xc = c.take((int64_t)B * s * T);
    KR_TRY(rows_mul(c, Zs, (int64_t)s * T, qs.F, T, (int64_t)T * T, Xc, T, (int64_t)s * T, s, T, T, B));
    double* cf = a->side == 1 ? VHv : Xc;
    KR_TRY(cudaMemcpyAsync(coeffs, cf, sizeof(double) * B * s * T, cudaMemcpyDeviceToDevice, c.st) == cudaSuccess
               ? KR_OK : fail(KR_ECUDA, "copy"));
    // QR breakdowns of [Jt; Ht]
    std::vector<int32_t> qi1, qi2;
    std::vector<double> qs1;
    KR_TRY(Fetch().add(qi1, qs.f1.info, B).add(qs1, qs.f1.stats, 4 * B).add(qi2, qs.f2.info, B).run(c));
    for (int b = 0; b < B; ++b)
      if (t[b] > 0 && !(cholqr_ok(qi1, qs1, b) && qi2[b] < 0)) {
        status[b] = 1;
        if (debug)
          fprintf(stderr, "  sample %d declined: GSVD CholQR2 (info %d/%d, pivots %.3e..%.3e)\n", b, qi1[b], qi2[b],
                  qs1[4 * b], qs1[4 * b + 1]);
      }
  }

  // ---- 5. U~ = W coeffs, H U~, C R = H U~, U = U~ R^-1
  double* cand = c.take((int64_t)B * s * n);
  double* HU = c.take((int64_t)B * s * n);
  if (a->vec_type == 1 && a->side == 2) {  // side M: normalised mean of both candidate sets
    KR_TRY(rows_mul(c, a->VH, (int64_t)s * T, W, n, (int64_t)T * n, cand, n, (int64_t)s * n, s, T, n, B, 0.5, 0.0));
    KR_TRY(rows_mul(c, Xc, (int64_t)s * T, W, n, (int64_t)T * n, cand, n, (int64_t)s * n, s, T, n, B, 0.5, 1.0));
    normalize_rows_kernel<<<dim3(s, B), 256, 0, c.st>>>(cand, s, n);
    KR_TRY(kr_hvp(op, cand, n, (int64_t)s * n, s, HU, n, (int64_t)s * n, c.st));
  } else {
    KR_TRY(rows_mul(c, coeffs, (int64_t)s * T, W, n, (int64_t)T * n, cand, n, (int64_t)s * n, s, T, n, B, 1.0, 0.0, false, d_td));
    if (a->reuse_products && !inner)  // (inner: H W is the previous H's, H U~ needs the upcoming one)
      KR_TRY(rows_mul(c, coeffs, (int64_t)s * T, HW, n, (int64_t)T * n, HU, n, (int64_t)s * n, s, T, n, B, 1.0, 0.0, false, d_td));
    else
      KR_TRY(kr_hvp(op, cand, n, (int64_t)s * n, s, HU, n, (int64_t)s * n, c.st));
  }
  QrOut qu;
  qu.Q = a->C;
  qu.F = c.take((int64_t)B * s * s);
  qu.f1 = new_factor(c, B, s);
  qu.f2 = new_factor(c, B, s);
  KR_TRY(cholqr2(c, HU, B, s, n, d_ns, c.take((int64_t)B * s * n), qu));
  KR_TRY(rows_mul(c, qu.F, (int64_t)s * s, cand, n, (int64_t)s * n, a->U, n, (int64_t)s * n, s, s, n, B));
  if (a->vec_type == 1)
    KR_TRY(rows_mul(c, VHmu, (int64_t)s * T, W, n, (int64_t)T * n, a->Z, n, (int64_t)s * n, s, T, n, B, 1.0, 0.0, false, d_td));

  // ---- 6. per-sample outcome
  std::vector<int32_t> ns, ui1, ui2, bd;
  std::vector<double> us1;
  {
    Fetch fe;
    fe.add(ns, d_ns, B).add(ui1, qu.f1.info, B).add(us1, qu.f1.stats, 4 * B).add(ui2, qu.f2.info, B);
    if (a->vec_type == 1) fe.add(bd, d_bad, B);
    KR_TRY(fe.run(c));
  }
  for (int b = 0; b < B; ++b) {
    a->tdims[b] = t[b];
    a->nsel[b] = ns[b];
    if (t[b] == 0 || ns[b] == 0) {
      a->status[b] = 2;
      continue;
    }
    if (!(cholqr_ok(ui1, us1, b) && ui2[b] < 0)) status[b] = 1;
    if (a->vec_type == 1 && bd[b]) status[b] = 1;
    if (debug && status[b])
      fprintf(stderr, "  sample %d declined: prepare CholQR2 (info %d/%d, pivots %.3e..%.3e) beta0 %d\n", b, ui1[b],
              ui2[b], us1[4 * b], us1[4 * b + 1], a->vec_type == 1 ? bd[b] : 0);
    a->status[b] = status[b];
  }
  if (debug)
    fprintf(stderr, "kr_recycle_update: B=%d T=%d shifted=%d ill=%d householder=%d (block %d) exact=%d host %.2f ms (householder %.2f)\n",
            B, T, (int)was_shifted, n_ill, n_house, n_block, n_exact,
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count(), house_ms);
  return check_launch("kr_recycle_update");
}
