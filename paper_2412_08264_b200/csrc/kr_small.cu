// kr_small.cu -- batched Cholesky + triangular inverse of the small Gram matrices
// of the recycle update (the Cholesky-QR passes of recycling._cholqr2 and the
// batched path, and the _hessian_condition screen, recycling.py:290-296).
//
// One CTA per matrix, the t x t lower triangle packed in shared memory
// (t <= CHOL_TMAX), or for larger t (<= CHOL_TMAX_G, the candidate widths of
// C3-C5) in a caller-provided global workspace that stays L2-resident -- the same
// code and arithmetic order either way, so both give bitwise the same factor: scale by D = sqrt(diag G) (optional), add a diagonal shift
// (optional, shifted CholeskyQR), factor G = L L^T (blocked right-looking),
// report the first failing row and the extreme pivots, and overwrite L by
// L^{-1} (blocked forward substitution, one thread per column).  Output F = L^{-1} D^{-1}, a full
// row-major T x T matrix: lower triangle F, zero upper triangle, identity in the
// pad block (rows/columns >= t_b), ready to be the left GEMM operand F @ A.

#include "kr_common.cuh"
#include "kr_internal.h"

namespace kr {
namespace {

constexpr int CNT = 512;
constexpr int CHOL_TMAX = 228;
constexpr int CHOL_TMAX_G = KR_TMAX;
constexpr int NB = 16;
constexpr int NCH_G = (CHOL_TMAX_G + CNT / 2 - 1) / (CNT / 2);  // column chunks of the inverse at t <= 640

struct CholParams {
  const double* G;
  int64_t ldg, bsg;
  const int32_t* dims;
  int T, flags;
  const double* shift;
  double* F;
  int64_t ldf, bsf;
  double* stats;  // per sample: [min L_jj, max L_jj, min D, 0]
  int32_t* info;  // per sample: -1 = factored, else the first failing row
  uint8_t* skipped;  // per sample and row (skip mode): 1 = dependent row removed
  double* gwork;     // nullable: per sample T(T+1)/2 doubles holding the packed factor (t > CHOL_TMAX)
};

__device__ __forceinline__ int64_t pk(int i, int j) { return (int64_t)i * (i + 1) / 2 + j; }

// 1/sqrt(d) for d > 0 without the sqrt/div slow-path calls (which force spills in
// fully unrolled register code): hardware approximation + three Newton steps.
__device__ __forceinline__ double rsqrt_nr(double d) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
#pragma unroll
  for (int it = 0; it < 3; ++it) {
    const double h = 0.5 * d * y;
    y = fma(y, fma(-h, y, 0.5), y);
  }
  return y;
}

template <int NCH>  // column chunks of CNT/2 in the inverse (1 for t <= 256)
__global__ void __launch_bounds__(CNT, 1) chol_inv_kernel(CholParams P) {
  extern __shared__ double sm[];
  const int tid = threadIdx.x;
  const int b = blockIdx.x;
  const int t = P.dims[b];
  const int T = P.T;
  double* D = sm;                 // T
  double* col = D + T;            // T (cached column)
  double* rdiag = col + T;        // NB reciprocal pivots of the current block
  double* Lbb = rdiag + NB;       // NB x (NB + 1) copy of a diagonal block
  // packed lower t(t+1)/2: shared memory, or the sample's slice of the global workspace
  double* A = P.gwork ? P.gwork + (int64_t)blockIdx.x * ((int64_t)P.T * (P.T + 1) / 2) : Lbb + NB * (NB + 1);
  __shared__ int s_fail;
  __shared__ unsigned char skp[CHOL_TMAX_G];
#ifdef KR_CHOL_TIMING
  long long csec[7] = {0, 0, 0, 0, 0, 0, 0}, clast = clock64();
#endif
  const double* Gb = P.G + (int64_t)b * P.bsg;
  const bool scale = P.flags & 1, inv = P.flags & 2, skipmode = P.flags & 4;
  for (int i = tid; i < t; i += CNT) {
    const double g = Gb[(int64_t)i * P.ldg + i];
    D[i] = (scale && g > 0.0) ? sqrt(g) : 1.0;
  }
  if (tid == 0) s_fail = -1;
  for (int i = tid; i < CHOL_TMAX_G; i += CNT) skp[i] = 0;
  __syncthreads();
  const double sh = P.shift ? P.shift[b] : 0.0;
  // lower triangle (as potrf 'L'), rows coalesced, independent loads in flight
  for (int i = tid >> 5; i < t; i += CNT / 32) {
    const double* gi = Gb + (int64_t)i * P.ldg;
    const double di = D[i];
#pragma unroll 4
    for (int j = tid & 31; j <= i; j += 32) A[pk(i, j)] = __ldg(gi + j) / (di * D[j]) + (i == j ? sh : 0.0);
  }
  __syncthreads();
  for (int i = tid; i < t; i += CNT) col[i] = A[pk(i, i)];  // diagonal before factoring
  __syncthreads();
  // a pivot below PIV_RTOL * (its original diagonal) is a breakdown: the row is
  // numerically dependent on the previous ones (exact dependence rounds either way)
  const double piv_rtol = 4.0 * t * 1.1102230246251565e-16;
  // ---- blocked Cholesky (right-looking, NB = 32) ----
#ifdef KR_CHOL_TIMING
    __syncthreads();
    if (tid == 0) { const long long c_ = clock64(); csec[0] += c_ - clast; clast = c_; }
#endif
  const int lane = tid & 31, warp = tid >> 5;
  // diagonal block kb in registers (warp 0): lane = row, column j broadcast by shuffles
  auto diag = [&](int kb) {
    const int nb = min(NB, t - kb);
      double a[NB];
#pragma unroll
      for (int k = 0; k < NB; ++k) a[k] = (lane < nb && k <= lane) ? A[pk(kb + lane, kb + k)] : 0.0;
      int bad = -1;
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        if (j < nb && bad < 0) {
          const double d = __shfl_sync(0xffffffffu, a[j], j);
          if (!(d > piv_rtol * col[kb + j])) {
            if (skipmode) {  // remove the dependent row: zero column below, unit pivot
              if (lane > j) a[j] = 0.0;
              if (lane == j) a[j] = 1.0;
              if (lane == 0) skp[kb + j] = 1;
            } else {
              bad = kb + j;
            }
          } else {
            const double rl = rsqrt_nr(d), ljj = d * rl;
            const double lij = lane == j ? ljj : a[j] * rl;
            if (lane >= j) a[j] = lij;
#pragma unroll
            for (int k = j + 1; k < NB; ++k) {
              const double lkj = __shfl_sync(0xffffffffu, lij, k);
              if (lane >= k) a[k] -= lij * lkj;
            }
          }
        }
      }
      if (lane < nb) {
#pragma unroll
        for (int k = 0; k < NB; ++k)
          if (k <= lane) A[pk(kb + lane, kb + k)] = a[k];
        rdiag[lane] = 1.0 / a[lane];  // (outside the unrolled code)
      }
      if (lane == 0 && bad >= 0) s_fail = bad;
      };
  // trailing update A_ij -= L_i,panel . L_j,panel for rows i >= rs, columns
  // j in [jlo, min(i + 1, jhi)), by warps w = 0 .. nw-1: lanes over j, four rows i0 + nw u
  // at once so each lane's L_j,panel load feeds four entries (every entry accumulates
  // c = 0 .. nb-1 in order)
  auto trailing = [&](int kb, int nb, int rs, int jlo, int jhi, int w, int nw) {
    constexpr int RU = 4;
    for (int i0 = rs + w; i0 < t; i0 += RU * nw) {
      const double* Li[RU];
      int im = i0;
#pragma unroll
      for (int u = 0; u < RU; ++u) {
        const int i = min(i0 + nw * u, t - 1);
        Li[u] = A + pk(i, kb);
        if (i0 + nw * u < t) im = i0 + nw * u;
      }
      const int jm = min(im, jhi - 1);
      for (int j = jlo + lane; j <= jm; j += 32) {
        const double* Lj = A + pk(j, kb);
        double acc[RU] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int c = 0; c < NB; ++c) {
          if (c < nb) {
            const double lj = Lj[c];
#pragma unroll
            for (int u = 0; u < RU; ++u) acc[u] += Li[u][c] * lj;
          }
        }
#pragma unroll
        for (int u = 0; u < RU; ++u) {
          const int i = i0 + nw * u;
          if (i < t && j <= i) A[pk(i, j)] -= acc[u];
        }
      }
    }
  };
  // right-looking blocked Cholesky with one block of look-ahead: after the panel of block
  // kb, the trailing update of the next block column comes first (all warps), then warp 0
  // factors the next diagonal block while warps 1.. finish the rest of the trailing
  // update (the same operations on every entry, reordered across independent entries)
  if (t > 0 && warp == 0) diag(0);
  __syncthreads();
  for (int kb = 0; kb < t; kb += NB) {
    const int nb = min(NB, t - kb);
#ifdef KR_CHOL_TIMING
    __syncthreads();
    if (tid == 0) { const long long c_ = clock64(); csec[1] += c_ - clast; clast = c_; }
#endif
    if (s_fail >= 0) break;
    // panel: rows below solve x L_kk^T = a (forward substitution over the block columns)
    for (int r = kb + nb + tid; r < t; r += CNT) {
      double x[NB];
#pragma unroll
      for (int c = 0; c < NB; ++c) {
        if (c < nb) {
          double v = A[pk(r, kb + c)];
          for (int m = 0; m < c; ++m) v -= x[m] * A[pk(kb + c, kb + m)];
          x[c] = skp[kb + c] ? 0.0 : v * rdiag[c];
          A[pk(r, kb + c)] = x[c];
        }
      }
    }
    __syncthreads();
#ifdef KR_CHOL_TIMING
    __syncthreads();
    if (tid == 0) { const long long c_ = clock64(); csec[2] += c_ - clast; clast = c_; }
#endif
    const int kn = kb + nb;
    if (kn < t) {
      const int nbn = min(NB, t - kn);
      trailing(kb, nb, kn, kn, kn + nbn, warp, CNT / 32);  // next block column
      __syncthreads();
      if (warp == 0)
        diag(kn);
      else
        trailing(kb, nb, kn + nbn, kn + nbn, t, warp - 1, CNT / 32 - 1);  // the rest
      __syncthreads();
    }
#ifdef KR_CHOL_TIMING
    __syncthreads();
    if (tid == 0) { const long long c_ = clock64(); csec[3] += c_ - clast; clast = c_; }
#endif
  }
  __syncthreads();
  const int fail = s_fail;
  if (P.stats) {  // extreme pivots and the smallest row norm, warp 0
    if (warp == 0) {
      double lo = 1e308, hi = 0.0, dm = 1e308;
      for (int j = lane; j < t; j += 32) {
        if (fail < 0 && !skp[j]) {
          lo = fmin(lo, A[pk(j, j)]);
          hi = fmax(hi, A[pk(j, j)]);
        }
        dm = fmin(dm, scale ? sqrt(fmax(Gb[(int64_t)j * P.ldg + j], 0.0)) : 1.0);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        dm = fmin(dm, __shfl_xor_sync(0xffffffffu, dm, o));
      }
      if (lane == 0) {
        P.stats[4 * b + 0] = t ? lo : 1.0;
        P.stats[4 * b + 1] = t ? hi : 1.0;
        P.stats[4 * b + 2] = t ? dm : 1.0;
        P.stats[4 * b + 3] = 0.0;
      }
    }
  }
  if (tid == 0) P.info[b] = fail;
  if (P.skipped)
    for (int i = tid; i < T; i += CNT) P.skipped[(int64_t)b * T + i] = i < t ? skp[i] : 0;
  if (!inv) return;
  double* Fb = P.F + (int64_t)b * P.bsf;
  const bool partial = P.flags & 8;
  if (fail >= 0 && !partial) {  // no factor: identity (callers discard the sample)
    for (int64_t e = tid; e < (int64_t)T * T; e += CNT) {
      const int i = (int)(e / T), j = (int)(e % T);
      Fb[(int64_t)i * P.ldf + j] = i == j ? 1.0 : 0.0;
    }
    return;
  }
  // partial mode: the leading `fail` rows factored (Cholesky is prefix-consistent), so
  // F keeps their inverse and zero rows from the breakdown row on
  const int tf = fail >= 0 ? fail : t;
  // ---- X = L^{-1} by blocked forward substitution ----
  // Block row I (rows ib..ib+nb): V = E_I - L_I,<I X_<I, then X_I = L_II^{-1} V.  A thread
  // owns one column c and one half h of the block rows: 8 accumulators in registers, one
  // contiguous X load per k feeding 8 FMAs with broadcast L operands; the substitution
  // runs on those registers (h = 0 rows first, then h = 1 with them), X_I overwrites L_I.
  for (int ib = 0; ib < tf; ib += NB) {
    const int nb = min(NB, tf - ib);
    const int w = ib + nb;  // columns 0 .. w-1 are nonzero in block row I
    for (int e = tid; e < nb * nb; e += CNT) {
      const int r = e / nb, m = e % nb;
      Lbb[r * (NB + 1) + m] = m <= r ? A[pk(ib + r, ib + m)] : 0.0;
      if (m == r) rdiag[r] = 1.0 / A[pk(ib + r, ib + r)];
    }
    // columns in chunks of CNT/2 (t > 256 needs up to NCH of them): the accumulators of every
    // chunk are formed before any X_I write (they read L_I,<I, which X_I overwrites)
    const int h = tid / (CNT / 2), c0 = tid - h * (CNT / 2);
    const int r0 = 8 * h;
    double acc[NCH][8];
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
#pragma unroll
      for (int u = 0; u < 8; ++u) acc[ch][u] = 0.0;
      const int c = c0 + ch * (CNT / 2);
      // the warp's lanes hold consecutive columns; they all start k at the warp's first
      // column, so the L operands are warp-uniform (broadcast smem loads), and a lane adds
      // fma(l, 0, acc) == acc for its rows k < c (bitwise the per-column loop from k = c)
      const int cw = (c & ~31) < w ? (c & ~31) : w;  // warp's first column (clamped)
      if (cw < w && r0 < nb) {
        const bool act = c < w;
        const double* lp[8];  // rows ib + r0 + u of L (clamped into the matrix)
#pragma unroll
        for (int u = 0; u < 8; ++u) lp[u] = A + pk(min(ib + r0 + u, tf - 1), 0);
        int k = cw;
        for (; k + 3 < ib; k += 4) {
          double xv[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) xv[j] = (act && k + j >= c) ? A[pk(k + j, c)] : 0.0;  // X_(k+j),c
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const double* l = lp[u] + k;
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[ch][u] = fma(l[j], xv[j], acc[ch][u]);
          }
        }
        for (; k < ib; ++k) {
          const double xk = (act && k >= c) ? A[pk(k, c)] : 0.0;
#pragma unroll
          for (int u = 0; u < 8; ++u) acc[ch][u] = fma(lp[u][k], xk, acc[ch][u]);
        }
      }
    }
    __syncthreads();  // every read of L_I,<I done before X_I overwrites it
    double x[NB];
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
      const int c = c0 + ch * (CNT / 2);
      if (h == 0 && c < w) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          if (r < nb) {
            double s = (c == ib + r ? 1.0 : 0.0) - acc[ch][r];
#pragma unroll
            for (int m = 0; m < r; ++m) s -= Lbb[r * (NB + 1) + m] * x[m];
            x[r] = (c <= ib + r) ? s * rdiag[r] : 0.0;
            if (c <= ib + r) A[pk(ib + r, c)] = x[r];
          }
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
      const int c = c0 + ch * (CNT / 2);
      if (h == 1 && c < w && nb > 8) {
#pragma unroll
        for (int m = 0; m < 8; ++m) x[m] = (c <= ib + m) ? A[pk(ib + m, c)] : 0.0;
#pragma unroll
        for (int r = 8; r < NB; ++r) {
          if (r < nb) {
            double s = (c == ib + r ? 1.0 : 0.0) - acc[ch][r - 8];
#pragma unroll
            for (int m = 0; m < r; ++m) s -= Lbb[r * (NB + 1) + m] * x[m];
            x[r] = (c <= ib + r) ? s * rdiag[r] : 0.0;
            if (c <= ib + r) A[pk(ib + r, c)] = x[r];
          }
        }
      }
    }
    __syncthreads();
  }
#ifdef KR_CHOL_TIMING
  __syncthreads();
  if (tid == 0) { const long long c_ = clock64(); csec[4] += c_ - clast; clast = c_; }
#endif
  // ---- F = L^{-1} D^{-1}, full row-major T x T ----
  for (int i = warp; i < T; i += CNT / 32) {
    double* fi = Fb + (int64_t)i * P.ldf;
    for (int j = lane; j < T; j += 32) {
      double v;
      if (i < t && j < t)
        v = (i < tf && j <= i && !skp[i]) ? A[pk(i, j)] / D[j] : 0.0;
      else
        v = i == j ? 1.0 : 0.0;
      fi[j] = v;
    }
  }
#ifdef KR_CHOL_TIMING
  __syncthreads();
  if (tid == 0) { const long long c_ = clock64(); csec[5] += c_ - clast; clast = c_; }
#endif
#ifdef KR_CHOL_TIMING
  if (tid == 0 && b == 0)
    printf("chol t=%d cycles: load %lld diag %lld panel %lld trailing %lld inverse %lld output %lld\n", t, csec[0], csec[1],
           csec[2], csec[3], csec[4], csec[5]);
#endif
}

}  // namespace
}  // namespace kr

using namespace kr;

extern "C" int64_t kr_chol_inv_workspace(int32_t batch, int32_t tmax) {
  if (batch < 0 || tmax < 0) return -1;
  return tmax <= CHOL_TMAX ? 0 : (int64_t)batch * ((int64_t)tmax * (tmax + 1) / 2);
}

extern "C" int kr_chol_inv(const double* G, int64_t ldg, int64_t bsg, const int32_t* dims, int32_t batch,
                           int32_t tmax, int32_t flags, const double* shift, double* F, int64_t ldf, int64_t bsf,
                           double* stats, int32_t* info, uint8_t* skipped, double* work, int64_t work_len,
                           kr_stream_t stream) {
  KR_CHECK_ARG(batch >= 0 && tmax >= 0, "negative size");
  KR_CHECK_ARG(tmax <= CHOL_TMAX_G, "kr_chol_inv: t exceeds 640");
  KR_CHECK_ARG(work_len >= kr_chol_inv_workspace(batch, tmax) && (tmax <= CHOL_TMAX || work),
               "kr_chol_inv: workspace too small (kr_chol_inv_workspace)");
  KR_CHECK_ARG(!(flags & 16) || (work && work_len >= (int64_t)batch * ((int64_t)tmax * (tmax + 1) / 2)),
               "kr_chol_inv: flag 16 needs a batch * t(t+1)/2 workspace");
  KR_CHECK_ARG(ldg >= tmax, "leading dimension smaller than t");
  KR_CHECK_ARG(!(flags & 2) || (F && ldf >= tmax), "inverse requested without an output");
  if (batch == 0) return KR_OK;
  KR_CHECK_ARG(G && dims && info, "null pointer");
  const bool glob = tmax > CHOL_TMAX || (flags & 16);  // bit 4: the workspace variant at any size (tests)
  CholParams P{G, ldg, bsg, dims, tmax, flags, shift, F, ldf, bsf, stats, info, skipped, glob ? work : nullptr};
  const size_t smem =
      (size_t)(2 * tmax + NB + NB * (NB + 1) + (glob ? 0 : (int64_t)tmax * (tmax + 1) / 2)) * sizeof(double);
  if (tmax <= CNT / 2) {
    KR_TRY(ensure_smem((const void*)chol_inv_kernel<1>, smem));
    chol_inv_kernel<1><<<batch, CNT, smem, (cudaStream_t)stream>>>(P);
  } else {
    KR_TRY(ensure_smem((const void*)chol_inv_kernel<NCH_G>, smem));
    chol_inv_kernel<NCH_G><<<batch, CNT, smem, (cudaStream_t)stream>>>(P);
  }
  return check_launch("chol_inv_kernel");
}

// ---------------------------------------------------------------------------
// Batched Gram G_b = A_b B_b^T of row blocks (A_b: rows x n, row stride ld), the
// (B, T, n) x (B, T, n) -> (B, T, T) products of the recycle update (candidate
// Grams, W^T H W).  cuBLAS picks small tiles for T x T outputs with K = n, so
// the pixel dimension is split into S chunks (pointer-array batched DGEMM over
// sample x chunk, pointers built on the device) and the partials are summed in
// fixed chunk order (deterministic).

extern "C" int64_t kr_gram_workspace(int32_t batch, int32_t rows, int64_t n) {
  // kr_gram plans a true Gram (A == B) on the lower tile blocks and a general product on all
  // tiles; their split counts differ, so the workspace covers both
  const int64_t a = kr::gram_dmma_workspace(batch, rows, rows, n, false);
  const int64_t b = kr::gram_dmma_workspace(batch, rows, rows, n, true);
  return a > b ? a : b;
}

extern "C" int kr_gram(const double* A, const double* Bm, int64_t ld, int64_t bs, int32_t batch, int32_t rows,
                       int64_t n, double* G, int64_t ldg, int64_t bsg, double* work, int64_t work_len,
                       kr_stream_t stream) {
  KR_CHECK_ARG(batch >= 0 && rows >= 0 && n >= 0, "negative size");
  KR_CHECK_ARG(ld >= n && ldg >= rows, "leading dimension too small");
  if (batch == 0 || rows == 0) return KR_OK;
  KR_CHECK_ARG(A && Bm && G && work, "null pointer");
  KR_CHECK_ARG(work_len >= kr_gram_workspace(batch, rows, n), "workspace too small");
  // a true Gram (A == B) computes the lower tile blocks and mirrors them
  return kr::gram_dmma(A, ld, bs, Bm, ld, bs, batch, rows, rows, n, A == Bm, G, ldg, bsg, work, work_len,
                       (cudaStream_t)stream);
}

// ---------------------------------------------------------------------------
// Sample-ordered sum of per-sample hypergradient rows (a thread per entry j, the rows
// accumulated left to right: bitwise the reference's sequential accumulation).

namespace kr {
namespace {
__global__ void ordered_sum_kernel(const double* __restrict__ rows, int count, int p, int64_t ld,
                                   double* __restrict__ out) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < p; j += gridDim.x * blockDim.x) {
    double acc = rows[j];
    for (int k = 1; k < count; ++k) acc += rows[(int64_t)k * ld + j];
    out[j] = acc;
  }
}
}  // namespace
}  // namespace kr

extern "C" int kr_ordered_sum(const double* rows, int32_t count, int32_t p, int64_t ld, double* out,
                              kr_stream_t stream) {
  KR_CHECK_ARG(count >= 1 && p >= 0 && ld >= p, "bad ordered-sum shape");
  if (p == 0) return KR_OK;
  KR_CHECK_ARG(rows && out, "null pointer");
  ordered_sum_kernel<<<(p + 255) / 256, 256, 0, (cudaStream_t)stream>>>(rows, count, p, ld, out);
  return check_launch("kr_ordered_sum");
}
