// kr_qrcp.cu -- QR with column pivoting of small t x t matrices, one CTA each.
//
// The reference builds the candidate basis with scipy's pivoted economic QR of
// [V_prev, U_prev] and keeps the pivots with |R_ii| > 1e-10 |R_00|
// (recycling.py:187-199).  For a tall block A = Q_A R (any backward-stable QR),
// pivoted QR of A is Q_A times pivoted QR of the small R, so the device path
// runs this kernel on R: Householder QR with column pivoting (LAPACK geqp3's
// greedy rule: the largest remaining column norm, exactly recomputed each step,
// ties to the lowest index), stopped at the first |R_kk| <= rtol |R_00|.  It
// returns the rank r and Q_R's first r columns, so the kept basis is
// Q_A Q_R[:, :r] (a GEMM), with the reference's drop decisions.
//
// The matrix (column-major, T x T per sample) is worked on in place in global
// memory (L2-resident).  Each reflector is applied with the trailing columns held
// in registers, QC columns per warp in flight, and the same pass returns their
// exact trailing norms for the next pivot choice.

#include <cfloat>

#include "kr_common.cuh"
#include "kr_internal.h"

namespace kr {
namespace {

constexpr int QNT = 256;
constexpr int QW = QNT / 32;

struct QrcpParams {
  double* M;  // in/out work: column j of sample b at M + b*T*T + j*T
  const int32_t* dims;
  int T;
  double rtol;
  double* Q;      // out: Q_R columns, column j of sample b at Q + b*T*T + j*T (first rank columns, rest 0)
  int32_t* rank;  // out
  int32_t* perm;  // out: pivot order (T per sample), nullable
  double* tau;    // work: T per sample
};

constexpr int QR = 8;   // rows per lane (t <= 256)
constexpr int QC = 4;   // columns per warp per round (independent loads in flight)

// Apply H = I - tau v v^T (v = vs[k..t), vs[k] = 1) to columns [j0, t) of M from
// row k, QC columns per warp at a time held in registers; optionally return the
// exact norms^2 of rows (k, t) of the updated columns in cn[].
__device__ void apply_reflector(double* M, int T, int t, int k, int j0, int jend, double tau, const double* vs,
                                double* cn, const int* col = nullptr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int jb = j0 + warp * QC; jb < jend; jb += QW * QC) {
    double c[QC][QR];
#pragma unroll
    for (int u = 0; u < QC; ++u) {
      const int jj = jb + u < jend ? (col ? col[jb + u] : jb + u) : 0;
      const double* cj = M + (int64_t)jj * T;
#pragma unroll
      for (int r = 0; r < QR; ++r) {
        const int i = k + lane + 32 * r;
        c[u][r] = (jb + u < jend && i < t) ? cj[i] : 0.0;
      }
    }
    double d[QC];
#pragma unroll
    for (int u = 0; u < QC; ++u) {
      double s = 0.0;
#pragma unroll
      for (int r = 0; r < QR; ++r) {
        const int i = k + lane + 32 * r;
        if (i < t) s += vs[i] * c[u][r];
      }
      d[u] = s;
    }
#pragma unroll
    for (int u = 0; u < QC; ++u) d[u] = tau * warp_sum(d[u]);
#pragma unroll
    for (int u = 0; u < QC; ++u) {
      double nn = 0.0;
      const int jj = jb + u < jend ? (col ? col[jb + u] : jb + u) : 0;
      double* cj = M + (int64_t)jj * T;
#pragma unroll
      for (int r = 0; r < QR; ++r) {
        const int i = k + lane + 32 * r;
        if (i < t) {
          c[u][r] -= d[u] * vs[i];
          if (jb + u < jend) cj[i] = c[u][r];
          if (i > k) nn += c[u][r] * c[u][r];
        }
      }
      if (cn) {
        nn = warp_sum(nn);
        if (lane == 0 && jb + u < jend) cn[jb + u] = nn;
      }
    }
  }
}

__global__ void __launch_bounds__(QNT, 1) qrcp_kernel(QrcpParams P) {
  __shared__ double cn[256];   // norms^2 of the trailing parts of the columns (exact)
  __shared__ double vs[256];   // current Householder vector
  __shared__ int pv[256];
  __shared__ double s_beta, s_tau, s_r00;
  __shared__ int s_piv, s_rank;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = blockIdx.x, t = P.dims[b], T = P.T;
  double* M = P.M + (int64_t)b * T * T;
  double* tau = P.tau + (int64_t)b * T;
  for (int j = tid; j < t; j += QNT) pv[j] = j;
  for (int j = warp; j < t; j += QW) {  // initial column norms
    const double* cj = M + (int64_t)j * T;
    double s = 0.0;
    for (int i = lane; i < t; i += 32) s += cj[i] * cj[i];
    s = warp_sum(s);
    if (lane == 0) cn[j] = s;
  }
  if (tid == 0) s_rank = t;
  __syncthreads();
  for (int k = 0; k < t; ++k) {
    // pivot: the largest remaining norm, lowest index on ties (warp 0)
    if (warp == 0) {
      double best = -1.0;
      int bi = k;
      for (int j = k + lane; j < t; j += 32)
        if (cn[j] > best) {
          best = cn[j];
          bi = j;
        }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) {
          best = ob;
          bi = oi;
        }
      }
      if (lane == 0) s_piv = bi;
    }
    __syncthreads();
    // pivot swap through the index: column j of the pivoted matrix is physical column pv[j]
    if (tid == 0) {
      const int p = s_piv;
      const int a = pv[k];
      pv[k] = pv[p];
      pv[p] = a;
      const double c = cn[k];
      cn[k] = cn[p];
      cn[p] = c;
    }
    __syncthreads();
    // Householder of column k (larfg), v staged in shared memory
    double* ck = M + (int64_t)pv[k] * T;
    if (warp == 0) {
      double x[QR];
      double s = 0.0;
#pragma unroll
      for (int r = 0; r < QR; ++r) {
        const int i = k + 1 + lane + 32 * r;
        x[r] = i < t ? ck[i] : 0.0;
        s += x[r] * x[r];
      }
      s = warp_sum(s);
      const double alpha = ck[k];
      double beta = alpha, tk = 0.0;
      if (s > 0.0) {
        beta = -copysign(sqrt(alpha * alpha + s), alpha);
        tk = (beta - alpha) / beta;
      }
      const double scal = tk != 0.0 ? 1.0 / (alpha - beta) : 0.0;
#pragma unroll
      for (int r = 0; r < QR; ++r) {
        const int i = k + 1 + lane + 32 * r;
        if (i < t) {
          const double v = x[r] * scal;
          vs[i] = v;
          ck[i] = v;
        }
      }
      if (lane == 0) {
        vs[k] = 1.0;
        s_beta = beta;
        s_tau = tk;
        if (k == 0) s_r00 = fabs(beta);
        ck[k] = beta;
        tau[k] = tk;
      }
    }
    __syncthreads();
    const double beta = s_beta, tk = s_tau;
    if (fabs(beta) <= P.rtol * s_r00 || (k == 0 && s_r00 == 0.0)) {  // recycling.py:194 keep rule
      if (tid == 0) s_rank = k;
      break;
    }
    if (tk != 0.0) {
      apply_reflector(M, T, t, k, k + 1, t, tk, vs, cn, pv);
    } else {
      for (int j = k + 1 + warp; j < t; j += QW) {  // norms still drop row k
        const double* cj = M + (int64_t)pv[j] * T;
        double s = 0.0;
        for (int i = k + 1 + lane; i < t; i += 32) s += cj[i] * cj[i];
        s = warp_sum(s);
        if (lane == 0) cn[j] = s;
      }
    }
    __syncthreads();
  }
  __syncthreads();
  const int r = s_rank;
  if (tid == 0) P.rank[b] = r;
  if (P.perm)
    for (int j = tid; j < T; j += QNT) P.perm[(int64_t)b * T + j] = j < t ? pv[j] : -1;
  // Q_R[:, :r] = H_0 ... H_{r-1} [I_r; 0]  (orgqr, backward accumulation)
  double* Qb = P.Q + (int64_t)b * T * T;
  for (int j = warp; j < T; j += QW)
    for (int i = lane; i < T; i += 32) Qb[(int64_t)j * T + i] = (j < r && i == j) ? 1.0 : 0.0;
  __syncthreads();
  for (int kk = r - 1; kk >= 0; --kk) {
    const double tk = tau[kk];
    if (tk != 0.0) {
      const double* vk = M + (int64_t)pv[kk] * T;
      for (int i = kk + 1 + tid; i < t; i += QNT) vs[i] = vk[i];
      if (tid == 0) vs[kk] = 1.0;
      __syncthreads();
      apply_reflector(Qb, T, t, kk, kk, r, tk, vs, nullptr);
    }
    __syncthreads();
  }
}

}  // namespace
}  // namespace kr

using namespace kr;

extern "C" int kr_qrcp_small(double* M, const int32_t* dims, int32_t batch, int32_t tmax, double rtol, double* Q,
                             int32_t* rank, int32_t* perm, double* work, int64_t work_len, kr_stream_t stream) {
  KR_CHECK_ARG(batch >= 0 && tmax >= 0 && tmax <= 256, "kr_qrcp_small: t must be in [0, 256]");
  KR_CHECK_ARG(work_len >= (int64_t)batch * tmax, "workspace too small");
  if (batch == 0) return KR_OK;
  KR_CHECK_ARG(M && dims && Q && rank && work, "null pointer");
  QrcpParams P{M, dims, tmax, rtol, Q, rank, perm, work};
  qrcp_kernel<<<batch, QNT, 0, (cudaStream_t)stream>>>(P);
  return check_launch("qrcp_kernel");
}
