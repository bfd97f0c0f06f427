// kr_eig.cu -- selected eigenpairs of a batch of small symmetric matrices.
//
// The recycle update needs, per sample, s of the t eigenpairs of a t x t
// symmetric matrix (t = k_prev + s_prev ~ 220 at C2): the Ritz pairs of
// W^T H W (recycling.py:226-236) or the right singular vectors of Q1 in the
// GSVD (recycling.py:275-313, taken from Q1^T Q1).  Library eigensolvers
// compute all t vectors through many latency-bound launches per matrix
// (cuSOLVER syevd ~2 ms at t = 220; the batched syev ~0.85 ms per matrix).
// Here one CTA owns one matrix for the whole computation:
//
//   1. Householder tridiagonalization (LAPACK sytd2, lower) on the packed
//      lower triangle held in shared memory (t <= EIG_TPACK), or -- for the wider
//      candidate blocks of C3-C5 (t <= KR_TMAX) -- on the full symmetric matrix in
//      a global workspace (L2-resident; rows read coalesced, both triangles
//      updated with a symmetric rounding order so the matrix stays bitwise
//      symmetric, reflector k stored in row k);
//   2. the selected eigenvalues by Sturm-count multisection: the 32 lanes of a
//      warp evaluate 32 points of the bracket per round (x33 per round), with
//      the division-free three-term recurrence (rescaled by powers of two);
//   3. their eigenvectors by inverse iteration on the tridiagonal matrix
//      (LAPACK stein's scheme: LU with partial pivoting, scaled start, growth
//      test, modified Gram-Schmidt inside clusters of close eigenvalues);
//   4. back-transformation through the stored reflectors.
//
// Selection follows recycling.py:202-213 (_select_indices) with the clamp of
// _clamp_dim: s_b = min(s, t_b); S -> the s_b smallest, L -> the s_b largest,
// M -> s_b/2 smallest then the rest largest; output in ascending order.
// Eigenvector signs: largest-magnitude component of the final vector positive.

#include <cfloat>

#include "kr_common.cuh"
#include "kr_internal.h"

namespace kr {
namespace {

constexpr int ENT = 512;
constexpr int EW = ENT / 32;
constexpr int EIG_TPACK = 228;
constexpr int EIG_TGLOB = KR_TMAX;
constexpr int EIG_MAXSEL = 128;
constexpr int EIG_RED = 64;
constexpr int MAXITS = 5;
constexpr int EXTRA = 2;

struct EigParams {
  const double* A;
  int64_t lda, bsa;
  const int32_t* dims;
  int T, size_code, s, nw;  // nw: vectors per inverse-iteration wave
  double* lam;
  int64_t bsl;
  double* Z;
  int64_t ldz, bsz;
  int32_t* nsel;
  double* work;  // per sample: packed reflectors T(T+1)/2 (shared-memory variant) or the full T x T matrix
};

__device__ __forceinline__ int64_t pk(int i, int j) { return (int64_t)i * (i + 1) / 2 + j; }  // i >= j

__device__ __forceinline__ double sym_at(const double* Ap, int i, int j) { return i >= j ? Ap[pk(i, j)] : Ap[pk(j, i)]; }

// 32-bit packed index (t <= EIG_TPACK keeps it far below 2^31): the hot loops' address math
__device__ __forceinline__ int pk32(int i, int j) { return ((i * (i + 1)) >> 1) + j; }  // i >= j

__device__ __forceinline__ double sym_at32(const double* Ap, int i, int j) {
  const int hi = i >= j ? i : j, lo = i >= j ? j : i;  // branch-free: one load per lane
  return Ap[pk32(hi, lo)];
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block sum over ENT threads, broadcast; red holds EW + 1 doubles.
__device__ double bsum(double v, double* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double r = l < EW ? red[l] : 0.0;
    r = warp_sum(r);
    if (l == 0) red[EW] = r;
  }
  __syncthreads();
  return red[EW];
}

// Number of eigenvalues of the tridiagonal (d, e) smaller than x: sign changes
// of the characteristic-polynomial sequence, i.e. negative pivots of
// T - x I = L D L^T (the ratio recurrence q_i = p_i / p_{i-1}, zero pivots
// replaced by -pivmin as in LAPACK).  The polynomial form needs no division;
// its rounding is a relative perturbation of d_i - x and e_i^2 per step, the
// same backward error as the ratio form.  Rescaled by powers of two (exact).
__device__ int sturm_count(const double* __restrict__ d, const double* __restrict__ e2, int t, double x,
                           double pivmin) {
  double pm1 = 1.0;
  double p = d[0] - x;
  if (p == 0.0) p = -pivmin;
  int cnt = p < 0.0;
  auto step = [&](double di, double ei) {
    double pn = fma(di - x, p, -ei * pm1);
    if (pn == 0.0) pn = -pivmin * p;
    cnt += (pn < 0.0) != (p < 0.0);
    pm1 = p;
    p = pn;
    const double ap = fabs(p);
    if (ap > 0x1p+400 || ap < 0x1p-400) {
      int ex;
      frexp(p, &ex);
      p = ldexp(p, -ex);
      pm1 = ldexp(pm1, -ex);
    }
  };
  int i = 1;
  for (; i + 3 < t; i += 4) {  // operands of four steps loaded ahead of the recurrence
    const double d0 = d[i], d1 = d[i + 1], d2 = d[i + 2], d3 = d[i + 3];
    const double f0 = e2[i - 1], f1 = e2[i], f2 = e2[i + 1], f3 = e2[i + 2];
    step(d0, f0);
    step(d1, f1);
    step(d2, f2);
    step(d3, f3);
  }
  for (; i < t; ++i) step(d[i], e2[i - 1]);
  return cnt;
}

// Tridiagonal LU with partial pivoting of T - lambda I (LAPACK lagtf).
// a: diagonal (in: d - lambda, out: U diagonal, stored as reciprocals in ra),
// b: first super-diagonal, c: multipliers, dd: second super-diagonal, piv.
struct TriLU {
  double *a, *b, *c, *dd, *ra;
  unsigned char* piv;
};

__device__ void lagtf(const double* __restrict__ d, const double* __restrict__ e, int t, double lambda, TriLU f,
                      double tol) {
  for (int i = 0; i < t; ++i) f.a[i] = d[i] - lambda;
  for (int i = 0; i + 1 < t; ++i) {
    f.b[i] = e[i];
    f.c[i] = e[i];
  }
  f.piv[0] = 0;
  double scale1 = fabs(f.a[0]) + (t > 1 ? fabs(f.b[0]) : 0.0);
  for (int k = 0; k + 1 < t; ++k) {
    double& ak = f.a[k];
    double& ak1 = f.a[k + 1];
    const double scale2 = fabs(f.c[k]) + fabs(ak1) + (k + 2 < t ? fabs(f.b[k + 1]) : 0.0);
    const double piv1 = ak == 0.0 ? 0.0 : fabs(ak) / scale1;
    if (f.c[k] == 0.0) {
      f.piv[k] = 0;
      scale1 = scale2;
      if (k + 2 < t) f.dd[k] = 0.0;
    } else {
      const double piv2 = fabs(f.c[k]) / scale2;
      if (piv2 <= piv1) {
        f.piv[k] = 0;
        scale1 = scale2;
        f.c[k] = f.c[k] / ak;
        ak1 -= f.c[k] * f.b[k];
        if (k + 2 < t) f.dd[k] = 0.0;
      } else {
        f.piv[k] = 1;
        const double mult = ak / f.c[k];
        ak = f.c[k];
        const double temp = ak1;
        ak1 = f.b[k] - mult * temp;
        if (k + 2 < t) {
          f.dd[k] = f.b[k + 1];
          f.b[k + 1] = -mult * f.dd[k];
        }
        f.b[k] = temp;
        f.c[k] = mult;
      }
    }
  }
  // reciprocal pivots, tiny ones perturbed to +-tol (LAPACK lagts job -1)
  for (int k = 0; k < t; ++k) {
    double ak = f.a[k];
    if (fabs(ak) < tol) ak = copysign(tol, ak == 0.0 ? 1.0 : ak);
    f.ra[k] = 1.0 / ak;
  }
}

// Solve (T - lambda I) y = x in place with the factors (LAPACK lagts, job -1).
__device__ void lagts(const TriLU& f, int t, double* __restrict__ y) {
  // the running element stays in a register (same operations as the in-memory form)
  double prev = y[0];
#pragma unroll 4
  for (int k = 1; k < t; ++k) {
    double yk = y[k];
    const double ck = f.c[k - 1];
    if (!f.piv[k - 1]) {
      yk -= ck * prev;
      y[k - 1] = prev;
      prev = yk;
    } else {
      const double temp = prev;
      y[k - 1] = yk;
      prev = temp - ck * yk;
    }
  }
  y[t - 1] = prev;
  double y1 = 0.0, y2 = 0.0;  // y[k + 1], y[k + 2]
#pragma unroll 4
  for (int k = t - 1; k >= 0; --k) {
    double temp = y[k];
    if (k + 1 < t) temp -= f.b[k] * y1;
    if (k + 2 < t) temp -= f.dd[k] * y2;
    const double yk = temp * f.ra[k];
    y[k] = yk;
    y2 = y1;
    y1 = yk;
  }
}

__device__ __forceinline__ double start_value(int q, int i) {
  // deterministic uniform(-1, 1) start vector (LAPACK larnv's role)
  unsigned h = (unsigned)(q * 7919 + 17) * 2654435761u ^ (unsigned)(i + 1) * 2246822519u;
  h ^= h >> 15;
  h *= 0x2c1b3c6du;
  h ^= h >> 12;
  h *= 0x297a2d39u;
  h ^= h >> 15;
  return (double)(h >> 8) * (2.0 / 16777216.0) - 1.0;
}

template <int RPL, bool GLOB>
__global__ void __launch_bounds__(ENT, 1) eig_select_kernel(EigParams P) {
  extern __shared__ double sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = blockIdx.x;
  const int t = P.dims[b];
  const int T = P.T;
  const int s = P.s < t ? P.s : t;
  const int lo = P.size_code == 0 ? s : (P.size_code == 1 ? 0 : s / 2);
  double* Zb = P.Z + (int64_t)b * P.bsz;
  for (int q = 0; q < P.s; ++q)
    for (int i = tid; i < T; i += ENT) Zb[(int64_t)q * P.ldz + i] = 0.0;
  if (tid == 0 && P.nsel) P.nsel[b] = s;
  if (s == 0) return;

  double* d = sm;
  double* e = d + T;
  double* tau = e + T;
  double* e2 = tau + T;
  double* sel = e2 + T;
  double* red = sel + EIG_MAXSEL;
  double* R = red + EIG_RED;
  __shared__ int s_int[4];

#ifdef KR_EIG_TIMING
  long long ec[12] = {0}, elast = clock64();
#define KR_EMARK(i)                                                   \
  do {                                                                \
    __syncthreads();                                                  \
    if (tid == 0) { const long long c_ = clock64(); ec[i] += c_ - elast; elast = c_; } \
  } while (0)
#else
#define KR_EMARK(i) ((void)0)
#endif
  // ---------------- 1. tridiagonalization ----------------
  double* vv = R;
  double* yv = R + T;
  double* Ap = R + 2 * T;
  const double* Ab = P.A + (int64_t)b * P.bsa;
  double* Af = P.work + (int64_t)b * T * T;  // GLOB: full matrix, row i at Af + i T
  if constexpr (GLOB) {
    double* ww = R + 2 * T;
    for (int i = warp; i < t; i += EW) {
      const double* ai = Ab + (int64_t)i * P.lda;
      for (int j = lane; j < t; j += 32)
        Af[(int64_t)i * T + j] = i == j ? __ldg(ai + j) : 0.5 * (__ldg(ai + j) + __ldg(Ab + (int64_t)j * P.lda + i));
    }
    __syncthreads();
    for (int k = 0; k + 1 < t; ++k) {
      const int m = t - k - 1;
      double* rk = Af + (int64_t)k * T;  // row k == column k (symmetric)
      double part = 0.0;
      for (int i = k + 2 + tid; i < t; i += ENT) {
        const double x = rk[i];
        part += x * x;
      }
      const double xn2 = bsum(part, red);
      const double alpha = rk[k + 1];
      double tk = 0.0, beta = alpha;
      if (xn2 > 0.0) {
        beta = -copysign(sqrt(alpha * alpha + xn2), alpha);
        tk = (beta - alpha) / beta;
        const double scal = 1.0 / (alpha - beta);
        for (int i = tid; i < m; i += ENT) {
          double v = 1.0;
          if (i > 0) {
            v = rk[k + 1 + i] * scal;
            rk[k + 1 + i] = v;
          }
          vv[i] = v;
        }
      }
      if (tid == 0) {
        e[k] = beta;
        tau[k] = tk;
        d[k] = rk[k];
      }
      if (tk == 0.0) continue;  // block-uniform (xn2 is broadcast)
      __syncthreads();
      // y = tau A22 v: a warp per row, two rows in flight, coalesced row reads
      for (int r = warp; r < m; r += 2 * EW) {
        const int r2 = r + EW;
        const bool two = r2 < m;
        const double* a1 = Af + (int64_t)(k + 1 + r) * T + k + 1;
        const double* a2 = Af + (int64_t)(k + 1 + (two ? r2 : r)) * T + k + 1;
        double acc = 0.0, acc2 = 0.0;
        for (int c = lane; c < m; c += 32) {
          const double vc = vv[c];
          acc += a1[c] * vc;
          acc2 += a2[c] * vc;
        }
        acc = warp_sum(acc);
        acc2 = warp_sum(acc2);
        if (lane == 0) {
          yv[r] = tk * acc;
          if (two) yv[r2] = tk * acc2;
        }
      }
      __syncthreads();
      double pv = 0.0;
      for (int r = tid; r < m; r += ENT) pv += yv[r] * vv[r];
      const double kappa = -0.5 * tk * bsum(pv, red);
      for (int r = tid; r < m; r += ENT) ww[r] = fma(kappa, vv[r], yv[r]);
      __syncthreads();
      // A22 -= v w^T + w v^T on both triangles; (r, c) and (c, r) round identically
      for (int r = warp; r < m; r += EW) {
        const double vi = vv[r], wi = ww[r];
        double* row = Af + (int64_t)(k + 1 + r) * T + k + 1;
        for (int c = lane; c < m; c += 32)
          row[c] -= __dadd_rn(__dmul_rn(vi, ww[c]), __dmul_rn(wi, vv[c]));
      }
      __syncthreads();
    }
    if (tid == 0) {
      d[t - 1] = Af[(int64_t)(t - 1) * T + t - 1];
      e[t - 1] = 0.0;
      tau[t - 1] = 0.0;
    }
    __syncthreads();
  } else {
  // (A + A^T) / 2 with coalesced reads: storage rows into the lower triangle, then
  // storage rows again onto the transposed positions
  for (int i = warp; i < t; i += EW) {
    const double* ai = Ab + (int64_t)i * P.lda;
#pragma unroll 4
    for (int j = lane; j <= i; j += 32) Ap[pk(i, j)] = __ldg(ai + j);
  }
  __syncthreads();
  for (int j = warp; j < t; j += EW) {
    const double* aj = Ab + (int64_t)j * P.lda;
#pragma unroll 4
    for (int i = j + 1 + lane; i < t; i += 32) Ap[pk(i, j)] = 0.5 * (Ap[pk(i, j)] + __ldg(aj + i));
  }
  __syncthreads();
  for (int k = 0; k + 1 < t; ++k) {
    const int m = t - k - 1;
    double part = 0.0;
    for (int i = k + 2 + tid; i < t; i += ENT) {
      const double x = Ap[pk(i, k)];
      part += x * x;
    }
    const double xn2 = bsum(part, red);
    KR_EMARK(5);
    const double alpha = Ap[pk(k + 1, k)];
    double tk = 0.0, beta = alpha;
    if (xn2 > 0.0) {
      beta = -copysign(sqrt(alpha * alpha + xn2), alpha);
      tk = (beta - alpha) / beta;
      const double scal = 1.0 / (alpha - beta);
      for (int i = tid; i < m; i += ENT) {
        double v = 1.0;
        if (i > 0) {
          v = Ap[pk(k + 1 + i, k)] * scal;
          Ap[pk(k + 1 + i, k)] = v;
        }
        vv[i] = v;
      }
    }
    if (tid == 0) {
      e[k] = beta;
      tau[k] = tk;
      d[k] = Ap[pk(k, k)];
    }
    if (tk == 0.0) continue;  // block-uniform (xn2 is broadcast)
    __syncthreads();
    KR_EMARK(6);
    // y = tau * A22 v, one warp per row (lower row part + column part via symmetry)
    // two rows per warp at a time (independent chains; each row's lane order and
    // shuffle tree as before)
    for (int r = warp; r < m; r += 2 * EW) {
      const int r2 = r + EW;
      const bool two = r2 < m;
      const int i = k + 1 + r, i2 = k + 1 + (two ? r2 : r);
      double acc = 0.0, acc2 = 0.0;
      for (int c = lane; c < m; c += 32) {
        const double vc = vv[c];
        acc += sym_at32(Ap, i, k + 1 + c) * vc;
        acc2 += sym_at32(Ap, i2, k + 1 + c) * vc;
      }
      acc = warp_sum(acc);
      acc2 = warp_sum(acc2);
      if (lane == 0) {
        yv[r] = tk * acc;
        if (two) yv[r2] = tk * acc2;
      }
    }
    __syncthreads();
    KR_EMARK(7);
    double pv = 0.0;
    for (int r = tid; r < m; r += ENT) pv += yv[r] * vv[r];
    const double kappa = -0.5 * tk * bsum(pv, red);
    KR_EMARK(8);
    // A22 -= v w^T + w v^T with w = y + kappa v (lower part)
    // two rows per warp at a time (every element's update is independent and unchanged)
    for (int r = warp; r < m; r += 2 * EW) {
      const int r2 = r + EW;
      const bool two = r2 < m;
      const double vi = vv[r], wi = yv[r] + kappa * vi;
      const double vi2 = two ? vv[r2] : 0.0, wi2 = two ? yv[r2] + kappa * vi2 : 0.0;
      double* row = Ap + pk32(k + 1 + r, k + 1);
      double* row2 = Ap + pk32(k + 1 + (two ? r2 : r), k + 1);
      const int cmax = two ? r2 : r;
      for (int c = lane; c <= cmax; c += 32) {
        const double vj = vv[c], wj = yv[c] + kappa * vj;
        if (c <= r) row[c] -= vi * wj + wi * vj;
        if (two) row2[c] -= vi2 * wj + wi2 * vj;
      }
    }
    __syncthreads();
    KR_EMARK(9);
  }
  if (tid == 0) {
    d[t - 1] = Ap[pk(t - 1, t - 1)];
    e[t - 1] = 0.0;
    tau[t - 1] = 0.0;
  }
  double* Hb = P.work + (int64_t)b * ((int64_t)T * (T + 1) / 2);
  for (int64_t i = tid; i < pk(t, 0); i += ENT) Hb[i] = Ap[i];
  __syncthreads();
  }  // !GLOB

  KR_EMARK(0);
  // ---------------- 2. selected eigenvalues ----------------
  if (warp == 0) {
    double gl = 1e308, gu = -1e308, tn = 0.0, em = 0.0;
    for (int i = lane; i < t; i += 32) {
      const double off = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < t ? fabs(e[i]) : 0.0);
      gl = fmin(gl, d[i] - off);
      gu = fmax(gu, d[i] + off);
      tn = fmax(tn, fabs(d[i]) + off);
      if (i + 1 < t) {
        e2[i] = e[i] * e[i];
        em = fmax(em, e2[i]);
      }
    }
    gl = -warp_max(-gl);
    gu = warp_max(gu);
    tn = warp_max(tn);
    em = warp_max(em);
    if (lane == 0) {
      const double widen = 2.0 * DBL_EPSILON * fmax(tn, DBL_MIN) * t + DBL_MIN;
      red[0] = gl - widen;
      red[1] = gu + widen;
      red[2] = tn;
      red[3] = DBL_MIN * fmax(1.0, em);
    }
  }
  __syncthreads();
  const double gl = red[0], gu = red[1], tnorm = red[2], pivmin = red[3];
  const double atol = DBL_EPSILON * fmax(tnorm, DBL_MIN);
  for (int q = warp; q < s; q += EW) {
    const int idx = q < lo ? q : t - (s - q);
    double a = gl, bb = gu;
    for (int round = 0; round < 64; ++round) {
      if (bb - a <= atol + 2.0 * DBL_EPSILON * fmax(fabs(a), fabs(bb))) break;
      const double x = a + (bb - a) * ((double)(lane + 1) / 33.0);
      const int c = sturm_count(d, e2, t, x, pivmin);
      const unsigned mask = __ballot_sync(0xffffffffu, c > idx);
      const int ls = mask ? __ffs(mask) - 1 : 32;
      const double xa = __shfl_sync(0xffffffffu, x, ls == 0 ? 0 : ls - 1);
      const double xb = __shfl_sync(0xffffffffu, x, ls == 32 ? 31 : ls);
      if (ls > 0) a = xa;
      if (ls < 32) bb = xb;
    }
    if (lane == 0) sel[q] = 0.5 * (a + bb);
  }
  __syncthreads();

  KR_EMARK(1);
  // ---------------- 3. inverse iteration ----------------
  // clusters of close selected eigenvalues (gap <= 1e-3 ||T||, LAPACK stein's ORTOL);
  // within a cluster the shifts are separated by >= 10 eps |lambda| (PERTOL)
  __shared__ short cl_first[EIG_MAXSEL];
  if (tid == 0) {
    const double ortol = 1e-3 * tnorm;
    int first = 0;
    for (int q = 0; q < s; ++q) {
      if (q > 0 && sel[q] - sel[q - 1] > ortol) first = q;
      if (q > first) {
        const double pertol = 10.0 * DBL_EPSILON * fmax(fabs(sel[q]), atol);
        if (sel[q] - sel[q - 1] < pertol) sel[q] = sel[q - 1] + pertol;
      }
      cl_first[q] = (short)first;
    }
  }
  __syncthreads();
  const int nw = P.nw;
  const double dtpcrt = sqrt(0.1 / t);
  // per active vector: x, a, b, c, dd, ra (6t doubles) + piv (t bytes)
  const int64_t per_vec = 6 * (int64_t)T + (T + 7) / 8;
  // Vectors are processed in waves of nw warps (one vector per warp).  Within a
  // wave all vectors iterate together (block inverse iteration): solve, then
  // modified Gram-Schmidt against the finished members of the cluster (earlier
  // waves) and, in order, against this wave's earlier members -- the role of
  // stein's MGS step.  The wave iterates until every vector passed the growth
  // test, then EXTRA more sweeps (stein's EXTRA), at most MAXITS + EXTRA.
  for (int w0 = 0; w0 < s; w0 += nw) {
    const int q = w0 + warp;
    const bool act = warp < nw && q < s;
    double* xs = R + (int64_t)warp * per_vec;
    TriLU f{xs + T, xs + 2 * T, xs + 3 * T, xs + 4 * T, xs + 5 * T, reinterpret_cast<unsigned char*>(xs + 6 * T)};
    if (act) {
      if (lane == 0) lagtf(d, e, t, sel[q], f, fmax(atol, DBL_MIN));
      for (int i = lane; i < t; i += 32) xs[i] = start_value(q, i);
      __syncwarp();
    }
    if (tid == 0) s_int[0] = 0;
    __syncthreads();
    int conv_at = -1;
    for (int it = 0; it < MAXITS + EXTRA; ++it) {
      if (act) {
        double asum = 0.0;
        for (int i = lane; i < t; i += 32) asum += fabs(xs[i]);
        asum = warp_sum(asum);
        const double scl = t * tnorm * fmax(DBL_EPSILON, fabs(1.0 / f.ra[t - 1])) / fmax(asum, DBL_MIN);
        for (int i = lane; i < t; i += 32) xs[i] *= scl;
        __syncwarp();
        if (lane == 0) lagts(f, t, xs);
        __syncwarp();
        for (int p = cl_first[q]; p < w0; ++p) {
          const double* zp = Zb + (int64_t)p * P.ldz;
          double dot = 0.0;
          for (int i = lane; i < t; i += 32) dot += zp[i] * xs[i];
          dot = warp_sum(dot);
          for (int i = lane; i < t; i += 32) xs[i] -= dot * zp[i];
          __syncwarp();
        }
      }
      __syncthreads();
      if (act) {
        const int f0 = cl_first[q] > w0 ? cl_first[q] : w0;  // first in-wave member of q's cluster
        if (q == f0) {
          for (int q2 = q + 1; q2 < s && q2 < w0 + nw && cl_first[q2] == cl_first[q]; ++q2) {
            double* x2 = R + (int64_t)(q2 - w0) * per_vec;
            for (int p = f0; p < q2; ++p) {
              const double* xp = R + (int64_t)(p - w0) * per_vec;
              double dot = 0.0, nn = 0.0;
              for (int i = lane; i < t; i += 32) {
                dot += xp[i] * x2[i];
                nn += xp[i] * xp[i];
              }
              dot = warp_sum(dot);
              nn = warp_sum(nn);
              const double cf = nn > 0.0 ? dot / nn : 0.0;
              for (int i = lane; i < t; i += 32) x2[i] -= cf * xp[i];
              __syncwarp();
            }
          }
        }
      }
      __syncthreads();
      if (act) {
        double nrm = 0.0;
        for (int i = lane; i < t; i += 32) nrm = fmax(nrm, fabs(xs[i]));
        nrm = warp_max(nrm);
        if (lane == 0 && nrm < dtpcrt) atomicOr(&s_int[0], 1);
      }
      __syncthreads();
      const bool all = s_int[0] == 0;
      __syncthreads();
      if (tid == 0) s_int[0] = 0;
      if (all && conv_at < 0) conv_at = it;
      if (conv_at >= 0 && it - conv_at >= EXTRA) break;
    }
    if (act) {
      double nn = 0.0;
      for (int i = lane; i < t; i += 32) nn += xs[i] * xs[i];
      nn = warp_sum(nn);
      const double scl = 1.0 / sqrt(nn);
      for (int i = lane; i < t; i += 32) Zb[(int64_t)q * P.ldz + i] = xs[i] * scl;
    }
    __syncthreads();
  }

  KR_EMARK(2);
  // ---------------- 4. back-transformation ----------------
  if constexpr (!GLOB) {
    const double* Hb = P.work + (int64_t)b * ((int64_t)T * (T + 1) / 2);
    for (int64_t i = tid; i < pk(t, 0); i += ENT) Ap[i] = Hb[i];
    __syncthreads();
  }
  for (int q = warp; q < s; q += EW) {
    double* zq = Zb + (int64_t)q * P.ldz;
    double z[RPL];
#pragma unroll
    for (int c = 0; c < RPL; ++c) {
      const int i = lane + 32 * c;
      z[c] = i < t ? zq[i] : 0.0;
    }
    for (int k = t - 2; k >= 0; --k) {
      const double tk = tau[k];
      if (tk == 0.0) continue;
      double dot = 0.0, hv[RPL];
#pragma unroll
      for (int c = 0; c < RPL; ++c) {
        const int i = lane + 32 * c;
        hv[c] = (i > k + 1 && i < t) ? (GLOB ? Af[(int64_t)k * T + i] : Ap[pk32(i, k)]) : 1.0;
      }
#pragma unroll
      for (int c = 0; c < RPL; ++c) {
        const int i = lane + 32 * c;
        if (i > k && i < t) dot += hv[c] * z[c];
      }
      dot = tk * warp_sum(dot);
#pragma unroll
      for (int c = 0; c < RPL; ++c) {
        const int i = lane + 32 * c;
        if (i > k && i < t) z[c] -= dot * hv[c];
      }
    }
    // sign: largest-magnitude component positive (first one on ties)
    double amax = -1.0;
    int imax = 0;
    double zmax = 0.0;
#pragma unroll
    for (int c = 0; c < RPL; ++c) {
      const int i = lane + 32 * c;
      if (i < t && fabs(z[c]) > amax) {
        amax = fabs(z[c]);
        imax = i;
        zmax = z[c];
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double oa = __shfl_xor_sync(0xffffffffu, amax, o);
      const int oi = __shfl_xor_sync(0xffffffffu, imax, o);
      const double oz = __shfl_xor_sync(0xffffffffu, zmax, o);
      if (oa > amax || (oa == amax && oi < imax)) {
        amax = oa;
        imax = oi;
        zmax = oz;
      }
    }
    const double sg = zmax < 0.0 ? -1.0 : 1.0;
#pragma unroll
    for (int c = 0; c < RPL; ++c) {
      const int i = lane + 32 * c;
      if (i < t) zq[i] = sg * z[c];
    }
    if (lane == 0 && P.lam) P.lam[(int64_t)b * P.bsl + q] = sel[q];
  }
#ifdef KR_EIG_TIMING
  KR_EMARK(3);
  if (tid == 0 && b == 0)
    printf("eig t=%d s=%d nw=%d cycles: tridiag %lld (norm %lld v %lld matvec %lld pv %lld rank2 %lld) sturm %lld "
           "inverse %lld back %lld\n", t, s, P.nw, ec[0] + ec[5] + ec[6] + ec[7] + ec[8] + ec[9], ec[5], ec[6], ec[7],
           ec[8], ec[9], ec[1], ec[2], ec[3]);
#endif
}

int64_t eig_smem_doubles(int T, int* nw_out) {
  const int64_t base = 4 * (int64_t)T + EIG_MAXSEL + EIG_RED;
  const int64_t r1 = T > EIG_TPACK ? 3 * (int64_t)T : 2 * (int64_t)T + (int64_t)T * (T + 1) / 2;
  const int64_t per_vec = 6 * (int64_t)T + (T + 7) / 8;
  // static smem (cl_first: EIG_MAXSEL shorts, s_int) kept out of the 227 KB opt-in
  const int64_t cap = (227 * 1024 - (int64_t)sizeof(short) * EIG_MAXSEL - 64) / 8 - base;
  int nw = (int)((cap > r1 ? cap : r1) / per_vec);
  if (nw > EW) nw = EW;
  if (nw < 1) nw = 1;
  int64_t r3 = nw * per_vec;
  if (nw_out) *nw_out = nw;
  return base + (r1 > r3 ? r1 : r3);
}

}  // namespace
}  // namespace kr

using namespace kr;

extern "C" int64_t kr_syev_select_workspace(int32_t batch, int32_t tmax) {
  if (batch < 0 || tmax < 0) return -1;
  return (int64_t)batch * (tmax > EIG_TPACK ? (int64_t)tmax * tmax : (int64_t)tmax * (tmax + 1) / 2);
}

extern "C" int kr_syev_select(const double* A, int64_t lda, int64_t bsa, const int32_t* dims, int32_t batch,
                              int32_t tmax, int32_t size_code, int32_t s, double* lam, int64_t bsl, double* Z,
                              int64_t ldz, int64_t bsz, int32_t* nsel, double* work, int64_t work_len,
                              kr_stream_t stream) {
  KR_CHECK_ARG(batch >= 0 && tmax >= 0 && s >= 0, "negative size");
  KR_CHECK_ARG(tmax <= EIG_TGLOB, "kr_syev_select: t exceeds KR_TMAX (640)");
  KR_CHECK_ARG(s <= EIG_MAXSEL, "kr_syev_select: more than 128 selected pairs");
  KR_CHECK_ARG(size_code >= 0 && size_code <= 2, "size code must be 0 (S), 1 (L) or 2 (M)");
  KR_CHECK_ARG(lda >= tmax && ldz >= tmax, "leading dimension smaller than t");
  KR_CHECK_ARG(work_len >= kr_syev_select_workspace(batch, tmax), "workspace too small");
  if (batch == 0 || s == 0 || tmax == 0) return KR_OK;
  KR_CHECK_ARG(A && dims && Z && work, "null pointer");
  EigParams P{A, lda, bsa, dims, tmax, size_code, s, 0, lam, bsl, Z, ldz, bsz, nsel, work};
  const size_t smem = (size_t)eig_smem_doubles(tmax, &P.nw) * sizeof(double);
  if (tmax <= EIG_TPACK) {
    KR_TRY(ensure_smem((const void*)eig_select_kernel<(EIG_TPACK + 31) / 32, false>, smem));
    eig_select_kernel<(EIG_TPACK + 31) / 32, false><<<batch, ENT, smem, (cudaStream_t)stream>>>(P);
  } else {
    KR_TRY(ensure_smem((const void*)eig_select_kernel<(EIG_TGLOB + 31) / 32, true>, smem));
    eig_select_kernel<(EIG_TGLOB + 31) / 32, true><<<batch, ENT, smem, (cudaStream_t)stream>>>(P);
  }
  return check_launch("eig_select_kernel");
}
