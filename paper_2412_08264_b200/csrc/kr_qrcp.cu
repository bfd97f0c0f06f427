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

// ---------------------------------------------------------------------------
// Cluster version: QNC CTAs per matrix, column g owned by CTA g % QNC (slot
// g / QNC) and resident in that CTA's shared memory for the whole factorization.
// Per pivot step: each CTA's best remaining column -> exchanged over DSMEM ->
// the same pivot everywhere (largest norm, lowest current position on ties);
// the owner forms the Householder vector; every CTA reads it over DSMEM and
// updates its own resident columns (exact trailing norms from the same pass).
// Two cluster barriers per step and no global-memory traffic.  Q_R is then
// accumulated with its columns distributed the same way (reflectors from L2).

#include <cooperative_groups.h>
#include <cuda_pipeline.h>

namespace kr {
namespace {

namespace cgc = cooperative_groups;
constexpr int QCN = 256;                  // threads per CTA
constexpr int QCW = QCN / 32;

// Variants by the largest t: cluster size QNC (8 portable, 16 non-portable), rows per
// lane QRR (registers of a column chunk), columns per warp per round QCC.  Resident
// columns per CTA: ceil(t / QNC) (<= 40 x 640 doubles = 200 KB at t = 640).
//   t <= 256: <8, 8, 4>   t <= 448: <8, 14, 2>   t <= 640: <16, 20, 2>
struct QcCand {
  double v;  // best remaining norm^2 of a CTA
  int g;     // its global column (-1: none)
  int pos;   // its current position
};

// Exchange through DSMEM is push-based: a producer stores into every CTA's copy
// before the cluster barrier (release / acquire), so reads after it are local.
template <int QNC, int QRR, int QCC, int TMX>
__global__ void __launch_bounds__(QCN, 1) qrcp_cluster_kernel(QrcpParams P) {
  constexpr int QR = QRR;
  constexpr int QC = QCC;
  constexpr int QCOLS = (TMX + QNC - 1) / QNC;
  extern __shared__ double csm[];
  cgc::cluster_group cluster = cgc::this_cluster();
  const int cr = (int)cluster.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = blockIdx.x / QNC, t = P.dims[b], T = P.T;
  const int qcols = (T + QNC - 1) / QNC;    // resident column slots (runtime T)
  double* cols = csm;                       // [qcols][T] resident columns
  double* vl = cols + (int64_t)qcols * T;   // [T] Householder vector of the current step (pushed by its owner)
  __shared__ double cn[QCOLS];              // trailing norms^2 of the resident columns
  __shared__ int done[QCOLS];               // already pivoted
  __shared__ int pos[TMX];                  // current position of every global column (replicated)
  __shared__ int at[TMX];                   // global column at every position (replicated)
  __shared__ QcCand cand[QNC];              // every CTA's candidate of the step (pushed)
  __shared__ double bt[2];                  // beta, tau of the step (pushed by the owner)
  double* M = P.M + (int64_t)b * T * T;
  const int nloc = (t - cr + QNC - 1) / QNC;  // columns g = cr + QNC * l, l < nloc
  for (int l = warp; l < nloc; l += QCW) {
    const int g = cr + QNC * l;
    const double* src = M + (int64_t)g * T;
    double s = 0.0;
    for (int i = lane; i < t; i += 32) {
      const double x = src[i];
      cols[(int64_t)l * T + i] = x;
      s += x * x;
    }
    s = warp_sum(s);
    if (lane == 0) {
      cn[l] = s;
      done[l] = 0;
    }
  }
  for (int g = tid; g < t; g += QCN) {
    pos[g] = g;
    at[g] = g;
  }
  __syncthreads();
  cluster.sync();
  double r00 = 0.0;
  int rank = t;
#ifdef KR_QRCP_TIMING
  long long qsec[6] = {0, 0, 0, 0, 0, 0}, qlast = clock64();
#endif
  for (int k = 0; k < t; ++k) {
    // 1. this CTA's candidate (warp 0), pushed to every CTA
    if (warp == 0) {
      double best = -1.0;
      int bg = -1, bp = 1 << 30;
      for (int l = lane; l < nloc; l += 32) {
        if (done[l]) continue;
        const int g = cr + QNC * l, p = pos[g];
        if (cn[l] > best || (cn[l] == best && p < bp)) {
          best = cn[l];
          bg = g;
          bp = p;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int og = __shfl_xor_sync(0xffffffffu, bg, o);
        const int op = __shfl_xor_sync(0xffffffffu, bp, o);
        if (ob > best || (ob == best && op < bp)) {
          best = ob;
          bg = og;
          bp = op;
        }
      }
      if (lane < QNC) {
        QcCand* dst = cluster.map_shared_rank(&cand[cr], lane);
        dst->v = best;
        dst->g = bg;
        dst->pos = bp;
      }
    }
#ifdef KR_QRCP_TIMING
    __syncthreads();
    if (tid == 0) { const long long c_ = clock64(); qsec[0] += c_ - qlast; qlast = c_; }
#endif
    __syncwarp();
    cluster.sync();
#ifdef KR_QRCP_TIMING
    __syncthreads();
    if (tid == 0) { const long long c_ = clock64(); qsec[1] += c_ - qlast; qlast = c_; }
#endif
    // 2. the cluster's pivot, decided identically in every CTA from the local copies
    double best = -1.0;
    int pg = -1, pp = 1 << 30;
#pragma unroll
    for (int r = 0; r < QNC; ++r) {
      const double v = cand[r].v;
      const int g = cand[r].g, p = cand[r].pos;
      if (g >= 0 && (v > best || (v == best && p < pp))) {
        best = v;
        pg = g;
        pp = p;
      }
    }
    // position bookkeeping (LAPACK's swap of positions k and pp); pos / at are read by
    // warp 0 only until the final write-back (behind barriers)
    if (tid == 0) {
      const int gk = at[k];
      at[pp] = gk;
      pos[gk] = pp;
      at[k] = pg;
      pos[pg] = k;
    }
#ifdef KR_QRCP_TIMING
    __syncthreads();
    if (tid == 0) { const long long c_ = clock64(); qsec[2] += c_ - qlast; qlast = c_; }
#endif
    const int owner = pg % QNC, lslot = pg / QNC;
    // 3. the owner forms the Householder vector of its column pg (rows k..t) and
    //    pushes it, beta and tau to every CTA (one warp per destination)
    if (cr == owner) {
      if (warp == 0) {
        double* cp = cols + (int64_t)lslot * T;
        double x[QR];
        double s = 0.0;
#pragma unroll
        for (int r = 0; r < QR; ++r) {
          const int i = k + 1 + lane + 32 * r;
          x[r] = i < t ? cp[i] : 0.0;
          s += x[r] * x[r];
        }
        s = warp_sum(s);
        const double alpha = cp[k];
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
            cp[i] = v;
            vl[i] = v;
          }
        }
        if (lane == 0) {
          vl[k] = 1.0;
          bt[0] = beta;
          bt[1] = tk;
          cp[k] = beta;
          done[lslot] = 1;
          P.tau[(int64_t)b * T + k] = tk;
        }
      }
      __syncthreads();  // owner CTA only (cr is uniform per CTA)
      for (int q = warp; q < QNC; q += QCW) {
        if (q == cr) continue;
        double* dv = cluster.map_shared_rank(vl, q);
        for (int i = k + lane; i < t; i += 32) dv[i] = vl[i];
        if (lane < 2) cluster.map_shared_rank(bt, q)[lane] = bt[lane];
      }
    }
#ifdef KR_QRCP_TIMING
    __syncthreads();
    if (tid == 0) { const long long c_ = clock64(); qsec[3] += c_ - qlast; qlast = c_; }
#endif
    __syncwarp();
    cluster.sync();
    // 4. beta / tau / v are local now
    const double beta = bt[0], tk = bt[1];
    if (k == 0) r00 = fabs(beta);
    if (fabs(beta) <= P.rtol * r00 || (k == 0 && r00 == 0.0)) {  // recycling.py:194 keep rule
      rank = k;
      break;
    }
#ifdef KR_QRCP_TIMING
    __syncthreads();
    if (tid == 0) { const long long c_ = clock64(); qsec[4] += c_ - qlast; qlast = c_; }
#endif
    // 5. apply H_k to the resident unpivoted columns; exact trailing norms.  A warp
    // takes QC columns at a time so their reductions are in flight together.
    const int rch = (t - k + 31) / 32;  // row chunks below k (warp-uniform)
    const bool app = tk != 0.0;
    for (int l0 = warp; l0 < nloc; l0 += QC * QCW) {
      double c[QC][QR];
      double d[QC], nn[QC];
      bool act[QC];
      const double* cb[QC];
#pragma unroll
      for (int u = 0; u < QC; ++u) {
        const int l = l0 + u * QCW;
        act[u] = l < nloc && !done[l < nloc ? l : 0];
        cb[u] = cols + (int64_t)(act[u] ? l : 0) * T;
        d[u] = 0.0;
        nn[u] = 0.0;
      }
      // loads are unconditional at clamped rows (masked by selects): no per-element branches
#pragma unroll
      for (int r = 0; r < QR; ++r) {
        if (r >= rch) break;
        const int i = k + lane + 32 * r;
        const int ic = i < t ? i : t - 1;
        const double vi = vl[ic];
#pragma unroll
        for (int u = 0; u < QC; ++u) {
          const double x = cb[u][ic];
          c[u][r] = i < t ? x : 0.0;
          d[u] = fma(vi, c[u][r], d[u]);
        }
      }
      if (app) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
          for (int u = 0; u < QC; ++u) d[u] += __shfl_xor_sync(0xffffffffu, d[u], o);
        }
      }
#pragma unroll
      for (int r = 0; r < QR; ++r) {
        if (r >= rch) break;
        const int i = k + lane + 32 * r;
        const int ic = i < t ? i : t - 1;
        const double vi = vl[ic];
#pragma unroll
        for (int u = 0; u < QC; ++u) {
          const double y = app ? fma(-tk * d[u], vi, c[u][r]) : c[u][r];
          nn[u] = fma((i > k && i < t) ? y : 0.0, y, nn[u]);
          if (app && act[u] && i < t) const_cast<double*>(cb[u])[i] = y;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
        for (int u = 0; u < QC; ++u) nn[u] += __shfl_xor_sync(0xffffffffu, nn[u], o);
      }
      if (lane == 0) {
#pragma unroll
        for (int u = 0; u < QC; ++u)
          if (act[u]) cn[l0 + u * QCW] = nn[u];
      }
    }
#ifdef KR_QRCP_TIMING
    __syncthreads();
    if (tid == 0) { const long long c_ = clock64(); qsec[5] += c_ - qlast; qlast = c_; }
#endif
  }
#ifdef KR_QRCP_TIMING
  if (tid == 0 && b == 0)
    printf("qrcp cta %d: cand %lld sync1 %lld pivot %lld house+sync2 %lld vcopy %lld apply %lld\n", cr, qsec[0], qsec[1],
           qsec[2], qsec[3], qsec[4], qsec[5]);
#endif
  // write back the resident columns (R_piv above the diagonal, reflectors below)
  for (int l = warp; l < nloc; l += QCW) {
    const int g = cr + QNC * l;
    double* dst = M + (int64_t)g * T;
    for (int i = lane; i < t; i += 32) dst[i] = cols[(int64_t)l * T + i];
  }
  if (cr == 0) {
    if (tid == 0) P.rank[b] = rank;
    if (P.perm)
      for (int j = tid; j < T; j += QCN) P.perm[(int64_t)b * T + j] = j < t ? at[j] : -1;
  }
  __syncthreads();
  cluster.sync();  // every CTA's columns and tau are in global memory (cluster-scope release/acquire)
  // Q_R[:, :r]: logical column j held by CTA j % QNC in the columns area
  const int r = rank;
  double* Qb = P.Q + (int64_t)b * T * T;
  const int qloc = (r - cr + QNC - 1) / QNC;  // Q columns j = cr + QNC * l, l < qloc
  for (int l = warp; l < qcols; l += QCW)
    for (int i = lane; i < T; i += 32) cols[(int64_t)l * T + i] = (l < qloc && i == cr + QNC * l) ? 1.0 : 0.0;
  __syncthreads();
  // reflectors r-1 .. 0 applied backwards; the next one streams into the other
  // buffer (cp.async) while the current one is applied, tau staged in shared memory
  double* taus = vl + 2 * T;  // reflector buffers: vl + (k & 1) T
  for (int i = tid; i < r; i += QCN) taus[i] = P.tau[(int64_t)b * T + i];
  auto fetch = [&](int k2) {
    const double* src = M + (int64_t)at[k2] * T;
    double* dst = vl + (k2 & 1) * T;
    for (int i = k2 + 1 + tid; i < t; i += QCN) __pipeline_memcpy_async(dst + i, src + i, sizeof(double));
    __pipeline_commit();
  };
  if (r > 0) fetch(r - 1);
  for (int kk = r - 1; kk >= 0; --kk) {
    if (kk >= 1) {
      fetch(kk - 1);
      __pipeline_wait_prior(1);
    } else {
      __pipeline_wait_prior(0);
    }
    double* vc = vl + (kk & 1) * T;
    if (tid == 0) vc[kk] = 1.0;
    __syncthreads();
    const double tk = taus[kk];
    if (tk != 0.0) {
      const int rch = (t - kk + 31) / 32;
      for (int l0 = warp; l0 < qloc; l0 += QC * QCW) {
        double c[QC][QR], d[QC];
        bool act[QC];
        double* cb[QC];
#pragma unroll
        for (int u = 0; u < QC; ++u) {
          const int l = l0 + u * QCW;
          act[u] = l < qloc && cr + QNC * l >= kk;
          cb[u] = cols + (int64_t)(act[u] ? l : 0) * T;
          d[u] = 0.0;
        }
#pragma unroll
        for (int rr = 0; rr < QR; ++rr) {
          if (rr >= rch) break;
          const int i = kk + lane + 32 * rr;
          const int ic = i < t ? i : t - 1;
          const double vi = i < t ? vc[ic] : 0.0;
#pragma unroll
          for (int u = 0; u < QC; ++u) {
            c[u][rr] = cb[u][ic];
            d[u] = fma(vi, c[u][rr], d[u]);
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
          for (int u = 0; u < QC; ++u) d[u] += __shfl_xor_sync(0xffffffffu, d[u], o);
        }
#pragma unroll
        for (int rr = 0; rr < QR; ++rr) {
          if (rr >= rch) break;
          const int i = kk + lane + 32 * rr;
          const int ic = i < t ? i : t - 1;
          const double vi = vc[ic];
#pragma unroll
          for (int u = 0; u < QC; ++u)
            if (act[u] && i < t) cb[u][i] = fma(-tk * d[u], vi, c[u][rr]);
        }
      }
    }
    __syncthreads();
  }
  for (int j = cr; j < T; j += QNC) {
    const int l = (j - cr) / QNC;
    double* dst = Qb + (int64_t)j * T;
    for (int i = tid; i < T; i += QCN) dst[i] = (j < r) ? cols[(int64_t)l * T + i] : 0.0;
  }
}

}  // namespace
}  // namespace kr

namespace kr {
namespace {
template <int QNC, int QRR, int QCC, int TMX>
int launch_qrcp_cluster(const QrcpParams& P, int batch, cudaStream_t st) {
  const auto kern = qrcp_cluster_kernel<QNC, QRR, QCC, TMX>;
  const int T = P.T;
  const size_t smem = ((size_t)((T + QNC - 1) / QNC) * T + 3 * (size_t)T) * sizeof(double);
  KR_TRY(ensure_smem((const void*)kern, smem));
  if (QNC > 8) {
    static bool np = false;  // per instantiation
    if (!np) {
      if (cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
        return fail(KR_ECUDA, "qrcp: non-portable cluster size");
      np = true;
    }
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(batch * QNC);
  cfg.blockDim = dim3(QCN);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = QNC;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, P);
  return check_launch("qrcp_cluster_kernel");
}
}  // namespace
}  // namespace kr

extern "C" int kr_qrcp_small_cluster(double* M, const int32_t* dims, int32_t batch, int32_t tmax, double rtol,
                                     double* Q, int32_t* rank, int32_t* perm, double* work, int64_t work_len,
                                     kr_stream_t stream) {
  using namespace kr;
  KR_CHECK_ARG(batch >= 0 && tmax >= 0 && tmax <= KR_TMAX, "kr_qrcp_small_cluster: t must be in [0, KR_TMAX]");
  KR_CHECK_ARG(work_len >= (int64_t)batch * tmax, "workspace too small");
  if (batch == 0) return KR_OK;
  KR_CHECK_ARG(M && dims && Q && rank && work, "null pointer");
  QrcpParams P{M, dims, tmax, rtol, Q, rank, perm, work};
  cudaStream_t st = (cudaStream_t)stream;
  if (tmax <= 256) return launch_qrcp_cluster<8, 8, 4, 256>(P, batch, st);
  if (tmax <= 448) return launch_qrcp_cluster<8, 14, 2, 448>(P, batch, st);
  return launch_qrcp_cluster<16, 20, 2, KR_TMAX>(P, batch, st);
}
