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
// memory (L2-resident); a warp per column for the Householder application.

#include <cfloat>

#include "kr_common.cuh"
#include "kr_internal.h"

namespace kr {
namespace {

constexpr int QNT = 512;
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

__global__ void __launch_bounds__(QNT, 1) qrcp_kernel(QrcpParams P) {
  __shared__ double cn[256];   // column norms^2 (t <= 256)
  __shared__ int pv[256];
  __shared__ double red_v[QW];
  __shared__ int red_i[QW];
  __shared__ double s_beta, s_tau, s_r00;
  __shared__ int s_piv, s_rank;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = blockIdx.x, t = P.dims[b], T = P.T;
  double* M = P.M + (int64_t)b * T * T;
  double* tau = P.tau + (int64_t)b * T;
  for (int j = tid; j < t; j += QNT) pv[j] = j;
  if (tid == 0) s_rank = t;
  __syncthreads();
  int k = 0;
  for (; k < t; ++k) {
    // exact norms of the trailing parts of the remaining columns (warp per column)
    for (int j = k + warp; j < t; j += QW) {
      const double* cj = M + (int64_t)j * T;
      double s = 0.0;
      for (int i = k + lane; i < t; i += 32) s += cj[i] * cj[i];
      s = warp_sum(s);
      if (lane == 0) cn[j] = s;
    }
    __syncthreads();
    // pivot: the largest norm, lowest index on ties (warp 0)
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
    const int p = s_piv;
    if (p != k) {  // swap columns k and p
      double* ck = M + (int64_t)k * T;
      double* cp = M + (int64_t)p * T;
      for (int i = tid; i < t; i += QNT) {
        const double a = ck[i];
        ck[i] = cp[i];
        cp[i] = a;
      }
      if (tid == 0) {
        const int a = pv[k];
        pv[k] = pv[p];
        pv[p] = a;
      }
    }
    __syncthreads();
    // Householder of column k below the diagonal (larfg)
    double* ck = M + (int64_t)k * T;
    if (warp == 0) {
      double s = 0.0;
      for (int i = k + 1 + lane; i < t; i += 32) s += ck[i] * ck[i];
      s = warp_sum(s);
      if (lane == 0) {
        const double alpha = ck[k];
        double beta = alpha, tk = 0.0;
        if (s > 0.0) {
          beta = -copysign(sqrt(alpha * alpha + s), alpha);
          tk = (beta - alpha) / beta;
        }
        s_beta = beta;
        s_tau = tk;
        if (k == 0) s_r00 = fabs(beta);
      }
    }
    __syncthreads();
    const double beta = s_beta, tk = s_tau;
    if (fabs(beta) <= P.rtol * s_r00 || (k == 0 && s_r00 == 0.0)) {  // recycling.py:194 keep rule
      if (tid == 0) s_rank = k;
      break;
    }
    if (tk != 0.0) {
      const double scal = 1.0 / (ck[k] - beta);
      for (int i = k + 1 + tid; i < t; i += QNT) ck[i] *= scal;
    }
    __syncthreads();
    if (tid == 0) {
      ck[k] = beta;
      tau[k] = tk;
    }
    // apply H_k = I - tau v v^T (v = [1; ck[k+1:]]) to the trailing columns
    if (tk != 0.0)
      for (int j = k + 1 + warp; j < t; j += QW) {
        double* cj = M + (int64_t)j * T;
        double d = (lane == 0) ? cj[k] : 0.0;
        for (int i = k + 1 + lane; i < t; i += 32) d += ck[i] * cj[i];
        d = tk * warp_sum(d);
        if (lane == 0) cj[k] -= d;
        for (int i = k + 1 + lane; i < t; i += 32) cj[i] -= d * ck[i];
      }
    __syncthreads();
  }
  __syncthreads();
  const int r = s_rank;
  if (tid == 0) P.rank[b] = r;
  if (P.perm)
    for (int j = tid; j < T; j += QNT) P.perm[(int64_t)b * T + j] = j < t ? pv[j] : -1;
  // Q_R[:, :r] = H_0 ... H_{r-1} [I_r; 0]  (orgqr, backward accumulation), column per warp
  double* Qb = P.Q + (int64_t)b * T * T;
  for (int j = warp; j < T; j += QW)
    for (int i = lane; i < T; i += 32) Qb[(int64_t)j * T + i] = (j < r && i == j) ? 1.0 : 0.0;
  __syncthreads();
  for (int kk = r - 1; kk >= 0; --kk) {
    const double tk = tau[kk];
    const double* vk = M + (int64_t)kk * T;  // v = [1; vk[kk+1:]]
    if (tk != 0.0)
      for (int j = kk + warp; j < r; j += QW) {
        double* qj = Qb + (int64_t)j * T;
        double d = (lane == 0) ? qj[kk] : 0.0;
        for (int i = kk + 1 + lane; i < t; i += 32) d += vk[i] * qj[i];
        d = tk * warp_sum(d);
        if (lane == 0) qj[kk] -= d;
        for (int i = kk + 1 + lane; i < t; i += 32) qj[i] -= d * vk[i];
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
