/* cpu_stencil.c -- TEST INFRASTRUCTURE ONLY (the oracle's C restatement).
 *
 * Plain C (+ OpenMP over image rows) restatement of the deblurring operators of
 * oracle/cpu_imaging.py, for fixture generation at the BASELINE configs' sizes
 * (256^2 .. 512^2), where scipy's direct convolve2d takes seconds per Hessian
 * product.  Same conventions as cpu_imaging (and the reference's operators.py):
 *
 *   conv_same(x, k)[i][j] = sum_{a,b} k[a][b] x[i - a + c][j - b + c]   (operators.py:309-326:
 *                            scipy convolve2d mode="same", boundary="fill"; zero outside)
 *   corr_same(x, k)[i][j] = sum_{a,b} k[a][b] x[i + a - c][j + b - c]
 *   H v  = scale * A^T A v + ridge * v + sum_j w_j corr(curv_j . conv(v, k_j), k_j)
 *          (cpu_imaging.hessian; operators.py:363-383 generalised), A = the blur
 *          outer(taps, taps), applied as two 1-D passes (it is exactly separable)
 *   J w  per filter j: [-w_j <slope_j, conv(w, k_j)>,
 *                       -w_j (shift(slope_j, w) + shift(curv_j . conv(w, k_j), xhat))]
 *          (cpu_imaging.jacobian; operators.py:386-444 _shift_dot / apply_adjoint)
 *   shift(v, x)[a][b] = sum_p v[p] x[p - (a - c), p - (b - c)]
 *
 * Only the summation order differs from cpu_imaging (checked against it at small
 * sizes in tests/test_oracle.py::test_c_stencil_matches_numpy_oracle).  Never
 * linked into the product.
 */
#include <stdlib.h>
#include <string.h>

static void conv1d_rows(const double* x, double* y, int R, int Cc, const double* t, int b, int flip) {
  const int c = b / 2;
#pragma omp parallel for schedule(static)
  for (int i = 0; i < R; ++i) {
    for (int j = 0; j < Cc; ++j) {
      double s = 0.0;
      for (int a = 0; a < b; ++a) {
        const int jj = flip ? j - a + c : j + a - c;
        if (jj >= 0 && jj < Cc) s += t[a] * x[(long)i * Cc + jj];
      }
      y[(long)i * Cc + j] = s;
    }
  }
}

static void conv1d_cols(const double* x, double* y, int R, int Cc, const double* t, int b, int flip) {
  const int c = b / 2;
#pragma omp parallel for schedule(static)
  for (int i = 0; i < R; ++i) {
    for (int j = 0; j < Cc; ++j) y[(long)i * Cc + j] = 0.0;
    for (int a = 0; a < b; ++a) {
      const int ii = flip ? i - a + c : i + a - c;
      if (ii < 0 || ii >= R) continue;
      const double ta = t[a];
      for (int j = 0; j < Cc; ++j) y[(long)i * Cc + j] += ta * x[(long)ii * Cc + j];
    }
  }
}

/* y = conv_same(x, k) (flip = 1) or corr_same(x, k) (flip = 0), q x q kernel k */
static void conv2d(const double* x, double* y, int R, int Cc, const double* k, int q, int flip) {
  const int c = q / 2;
#pragma omp parallel for schedule(static)
  for (int i = 0; i < R; ++i) {
    for (int j = 0; j < Cc; ++j) y[(long)i * Cc + j] = 0.0;
    for (int a = 0; a < q; ++a) {
      const int ii = flip ? i - a + c : i + a - c;
      if (ii < 0 || ii >= R) continue;
      const double* xr = x + (long)ii * Cc;
      double* yr = y + (long)i * Cc;
      for (int bb = 0; bb < q; ++bb) {
        const double kab = k[a * q + bb];
        const int d = flip ? c - bb : bb - c; /* column offset: x[j + d] */
        const int j0 = d < 0 ? -d : 0, j1 = d > 0 ? Cc - d : Cc;
        for (int j = j0; j < j1; ++j) yr[j] += kab * xr[j + d];
      }
    }
  }
}

/* A^T A v for the separable blur: corr(conv(v, g g^T), g g^T) */
static void blur_ata(const double* v, double* out, double* t1, double* t2, int R, int Cc, const double* taps, int b) {
  conv1d_rows(v, t1, R, Cc, taps, b, 1);
  conv1d_cols(t1, t2, R, Cc, taps, b, 1);
  conv1d_cols(t2, t1, R, Cc, taps, b, 0);
  conv1d_rows(t1, out, R, Cc, taps, b, 0);
}

/* out = H v.  kernels: J x q x q, w: J filter weights, curv: J x n (phi'' at xhat). */
void oc_hvp(const double* v, double* out, int R, int Cc, const double* taps, int b, double scale, double ridge,
            int J, int q, const double* kernels, const double* w, const double* curv) {
  const long n = (long)R * Cc;
  double* t1 = (double*)malloc(sizeof(double) * n);
  double* t2 = (double*)malloc(sizeof(double) * n);
  double* t3 = (double*)malloc(sizeof(double) * n);
  blur_ata(v, out, t1, t2, R, Cc, taps, b);
  for (long p = 0; p < n; ++p) out[p] = scale * out[p] + ridge * v[p];
  for (int j = 0; j < J; ++j) {
    const double* k = kernels + (long)j * q * q;
    conv2d(v, t1, R, Cc, k, q, 1);
    const double* cj = curv + (long)j * n;
    for (long p = 0; p < n; ++p) t1[p] *= cj[p];
    conv2d(t1, t3, R, Cc, k, q, 0);
    for (long p = 0; p < n; ++p) out[p] += w[j] * t3[p];
  }
  free(t1);
  free(t2);
  free(t3);
}

/* out[a][b] = sum_p v[p] x[p - (a - c), p - (b - c)] */
static void shift_dot(const double* v, const double* x, int R, int Cc, int q, double* out) {
  const int c = q / 2;
#pragma omp parallel for collapse(2) schedule(static)
  for (int a = 0; a < q; ++a) {
    for (int bb = 0; bb < q; ++bb) {
      const int da = a - c, db = bb - c;
      const int r0 = da > 0 ? da : 0, r1 = da < 0 ? R + da : R;
      const int c0 = db > 0 ? db : 0, c1 = db < 0 ? Cc + db : Cc;
      double s = 0.0;
      for (int i = r0; i < r1; ++i) {
        const double* vr = v + (long)i * Cc;
        const double* xr = x + (long)(i - da) * Cc - db;
        for (int j = c0; j < c1; ++j) s += vr[j] * xr[j];
      }
      out[a * q + bb] = s;
    }
  }
}

/* out (J (1 + q^2)) = J w.  slope / curv: J x n (phi', phi'' at xhat). */
void oc_jadj(const double* wv, double* out, int R, int Cc, const double* xhat, int J, int q, const double* kernels,
             const double* w, const double* slope, const double* curv) {
  const long n = (long)R * Cc;
  const int q2 = q * q;
  double* cw = (double*)malloc(sizeof(double) * n);
  double* m = (double*)malloc(sizeof(double) * n);
  double* g1 = (double*)malloc(sizeof(double) * q2);
  double* g2 = (double*)malloc(sizeof(double) * q2);
  for (int j = 0; j < J; ++j) {
    const double* k = kernels + (long)j * q2;
    const double* sj = slope + (long)j * n;
    const double* cj = curv + (long)j * n;
    conv2d(wv, cw, R, Cc, k, q, 1);
    double head = 0.0;
    for (long p = 0; p < n; ++p) {
      head += sj[p] * cw[p];
      m[p] = cj[p] * cw[p];
    }
    shift_dot(sj, wv, R, Cc, q, g1);
    shift_dot(m, xhat, R, Cc, q, g2);
    double* o = out + (long)j * (1 + q2);
    o[0] = -w[j] * head;
    for (int i = 0; i < q2; ++i) o[1 + i] = -w[j] * (g1[i] + g2[i]);
  }
  free(cw);
  free(m);
  free(g1);
  free(g2);
}

/* y = conv_same(x, k) -- exported for the prepare step (phi', phi'' at xhat) */
void oc_conv_same(const double* x, double* y, int R, int Cc, const double* k, int q) { conv2d(x, y, R, Cc, k, q, 1); }
