// kr_ops.cu -- operator kernels behind the C ABI:
//   kr_op_prepare  curvature / slope tables at xhat  (operators.py:427 caching)
//   kr_hvp         H V for t columns x B samples     (operators.py:253-261)
//   kr_jadj        J W for t columns x B samples     (operators.py:290-298, 386-444)
//   kr_lower_eval  lower cost + gradient             (operators.py:329-353)
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "kr_common.cuh"
#include "kr_internal.h"

namespace kr {

// ---------------------------------------------------------------------------
// curvature tables

__global__ void prepare_filters_kernel(kr_op op) {
  const int64_t n = op_n(op);
  const int q = op.ksize, rq = q / 2, J = op.num_filters;
  const int b = blockIdx.y;
  const double* x = op.xhat + (int64_t)b * n;
  const double e2 = op.eps * op.eps;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    int y = (int)(p / op.cols), xx = (int)(p % op.cols);
    for (int j = 0; j < J; ++j) {
      const double* kj = op.kernels + j * q * q;
      double u = 0.0;
      for (int a = 0; a < q; ++a) {
        int yy = y - a + rq;
        if (yy < 0 || yy >= op.rows) continue;
        for (int bb = 0; bb < q; ++bb) {
          int xc = xx - bb + rq;
          if (xc < 0 || xc >= op.cols) continue;
          u += kj[a * q + bb] * x[(int64_t)yy * op.cols + xc];
        }
      }
      int64_t o = ((int64_t)b * J + j) * n + p;
      if (op.potential == KR_POT_QUADRATIC) {
        op.slope[o] = 2.0 * u;  // phi'(t) = 2t
        if (op.curv) op.curv[o] = 2.0;
      } else {
        double s = sqrt(u * u + e2);
        op.slope[o] = u / s;           // phi'
        op.curv[o] = e2 / (s * s * s);  // phi'' = eps^2 / (t^2+eps^2)^{3/2}
      }
    }
  }
}

__global__ void prepare_tv_kernel(kr_op op) {
  const int64_t n = op_n(op);
  const int b = blockIdx.y;
  const double* x = op.xhat + (int64_t)b * n;
  const double e2 = op.eps * op.eps;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    int y = (int)(p / op.cols), xx = (int)(p % op.cols);
    double gh = (xx < op.cols - 1) ? x[p + 1] - x[p] : 0.0;
    double gv = (y < op.rows - 1) ? x[p + op.cols] - x[p] : 0.0;
    double s = sqrt(gh * gh + gv * gv + e2);
    double* M = op.curv + (int64_t)b * 3 * n;
    double* S = op.slope + (int64_t)b * 2 * n;
    M[p] = (1.0 - gh * gh / (s * s)) / s;
    M[n + p] = -(gh * gv) / (s * s * s);
    M[2 * n + p] = (1.0 - gv * gv / (s * s)) / s;
    S[p] = gh / s;
    S[n + p] = gv / s;
  }
}

// ---------------------------------------------------------------------------
// H V

template <int Q>
__global__ void __launch_bounds__(NT) hvp_kernel(kr_op op, const double* __restrict__ V, int64_t ldv,
                                                 int64_t bsv, double* __restrict__ HV, int64_t ldo,
                                                 int64_t bso, const int32_t* __restrict__ dims,
                                                 const __grid_constant__ CUtensorMap tmap, int use_tma) {
  extern __shared__ __align__(128) double smem[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t mphase;
  const int tile = blockIdx.x, col = blockIdx.y, b = blockIdx.z;
  if (dims && col >= dims[b]) {  // zero pad column of a batch padded to its widest sample: H 0 = 0
    double* out = HV + b * bso + col * ldo;
    for (int l = threadIdx.x; l < TPX; l += blockDim.x) {
      const int64_t p = tile_pixel(op, tile, l);
      if (p >= 0) out[p] = 0.0;
    }
    return;
  }
  const Geom g = make_geom(op);
  Smem sm = carve(g, smem);
  if (use_tma) tma_mbar_init(&mbar, &mphase);
  load_weights(op, g, sm);
  const double* in = V + b * bsv + col * ldv;
  const TmaSrc t{&tmap, col, b, 1.0, &mbar, &mphase};
  tile_hvp_t<Q>(op, g, sm, b, TileIn{in, 1.0, nullptr, 0.0}, tile, use_tma ? &t : nullptr);
  double* out = HV + b * bso + col * ldo;
  if (op.data_kind == KR_DATA_DENSE) {
    for (int l = threadIdx.x; l < TPX; l += blockDim.x) {
      int64_t p = tile_pixel(op, tile, l);
      if (p >= 0) out[p] = sm.res[l];
    }
  } else {  // the tile's origin once, not per element
    const int tyc = tiles_x(op);
    const int y0 = (tile / tyc) * TH, x0 = (tile % tyc) * TW;
    for (int l = threadIdx.x; l < TPX; l += blockDim.x) {
      const int y = y0 + l / TW, x = x0 + l % TW;
      if (y < op.rows && x < op.cols) out[(int64_t)y * op.cols + x] = sm.res[l];
    }
  }
}

// ---------------------------------------------------------------------------
// J W: per (tile, column, sample) partial sums, then a fixed-order reduce.

__global__ void __launch_bounds__(NT) jadj_filters_kernel(kr_op op, const double* __restrict__ W, int64_t ldw,
                                                          int64_t bsw, double* __restrict__ part) {
  extern __shared__ double smem[];
  const int q = op.ksize, rq = q / 2, q2 = q * q, J = op.num_filters;
  const int RW = TW + 4 * rq, RH = TH + 4 * rq;  // w region with 2rq halo (C_j w on tile+rq, shifts)
  double* Sw = smem;              // RH x RW
  double* Sx = Sw + RH * RW;      // xhat on tile + rq halo: (TH+2rq) x (TW+2rq)
  double* Sk = Sx + (TH + 2 * rq) * (TW + 2 * rq);
  double* red = Sk + J * q2;      // reduction scratch (KR_MAX_KSIZE^2+1)*33
  const int tile = blockIdx.x, col = blockIdx.y, b = blockIdx.z;
  const int ntiles = gridDim.x, ncols = gridDim.y;
  const int tyc = tiles_x(op);
  const int y0 = (tile / tyc) * TH, x0 = (tile % tyc) * TW;
  const int64_t n = op_n(op);
  const double* w = W + b * bsw + col * ldw;
  const double* xh = op.xhat + (int64_t)b * n;
  for (int i = threadIdx.x; i < RH * RW; i += blockDim.x) {
    int yy = i / RW, xx = i - yy * RW;
    int y = y0 - 2 * rq + yy, x = x0 - 2 * rq + xx;
    Sw[i] = (y >= 0 && y < op.rows && x >= 0 && x < op.cols) ? w[(int64_t)y * op.cols + x] : 0.0;
  }
  const int XW = TW + 2 * rq, XH = TH + 2 * rq;
  for (int i = threadIdx.x; i < XH * XW; i += blockDim.x) {
    int yy = i / XW, xx = i - yy * XW;
    int y = y0 - rq + yy, x = x0 - rq + xx;
    Sx[i] = (y >= 0 && y < op.rows && x >= 0 && x < op.cols) ? xh[(int64_t)y * op.cols + x] : 0.0;
  }
  for (int i = threadIdx.x; i < J * q2; i += blockDim.x) Sk[i] = op.kernels[i];
  block_barrier();
  const int P = J * (1 + q2);
  double* outp = part + (((int64_t)b * ncols + col) * ntiles + tile) * P;
  for (int j = 0; j < J; ++j) {
    const double* kj = Sk + j * q2;
    const double* sl = op.slope + ((int64_t)b * J + j) * n;
    const double* cv = (op.potential == KR_POT_QUADRATIC) ? nullptr : op.curv + ((int64_t)b * J + j) * n;
    double acc[1 + KR_MAX_KSIZE * KR_MAX_KSIZE];
    for (int i = 0; i <= q2; ++i) acc[i] = 0.0;
    for (int l = threadIdx.x; l < TPX; l += blockDim.x) {
      int ty = l / TW, tx = l - ty * TW;
      int y = y0 + ty, x = x0 + tx;
      if (y >= op.rows || x >= op.cols) continue;
      int64_t p = (int64_t)y * op.cols + x;
      // C_j w at p (true convolution)
      const double* c = Sw + (ty + 2 * rq) * RW + tx + 2 * rq;
      double cw = 0.0;
      for (int a = 0; a < q; ++a)
        for (int bb = 0; bb < q; ++bb) cw += kj[a * q + bb] * c[-(a - rq) * RW - (bb - rq)];
      double s1 = sl[p];
      double yv = (cv ? cv[p] : 2.0) * cw;
      acc[0] += s1 * cw;
      // shift(phi', w)[a,b] + shift(kappa C w, xhat)[a,b]: x[p - (a-rq, b-rq)]
      const double* cx = Sx + (ty + rq) * XW + tx + rq;
      for (int a = 0; a < q; ++a)
        for (int bb = 0; bb < q; ++bb) {
          int off_w = -(a - rq) * RW - (bb - rq);
          int off_x = -(a - rq) * XW - (bb - rq);
          acc[1 + a * q + bb] += s1 * c[off_w] + yv * cx[off_x];
        }
    }
    // block reduce 1 + q2 values (runtime q): process in chunks of 8
    for (int base = 0; base <= q2; base += 8) {
      double v8[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v8[i] = (base + i <= q2) ? acc[base + i] : 0.0;
      block_sum<8>(v8, red);
      if (threadIdx.x < 8 && base + threadIdx.x <= q2) outp[j * (1 + q2) + base + threadIdx.x] = red[threadIdx.x];
      block_barrier();
    }
  }
}

__global__ void __launch_bounds__(NT) jadj_tv_kernel(kr_op op, const double* __restrict__ W, int64_t ldw,
                                                     int64_t bsw, double* __restrict__ part) {
  __shared__ double red[8 * 33 + 8];
  const int tile = blockIdx.x, col = blockIdx.y, b = blockIdx.z;
  const int ntiles = gridDim.x, ncols = gridDim.y;
  const int tyc = tiles_x(op);
  const int y0 = (tile / tyc) * TH, x0 = (tile % tyc) * TW;
  const int64_t n = op_n(op);
  const double* w = W + b * bsw + col * ldw;
  const double* S = op.slope + (int64_t)b * 2 * n;
  double acc[1] = {0.0};
  for (int l = threadIdx.x; l < TPX; l += blockDim.x) {
    int y = y0 + l / TW, x = x0 + l % TW;
    if (y >= op.rows || x >= op.cols) continue;
    int64_t p = (int64_t)y * op.cols + x;
    double dh = (x < op.cols - 1) ? w[p + 1] - w[p] : 0.0;
    double dv = (y < op.rows - 1) ? w[p + op.cols] - w[p] : 0.0;
    acc[0] += S[p] * dh + S[n + p] * dv;
  }
  block_sum<1>(acc, red);
  if (threadIdx.x == 0) part[((int64_t)b * ncols + col) * ntiles + tile] = red[0];
}

// out[b][col][i] = -w_j * sum_tiles part (fixed order); i runs over P = J(1+q^2) (TV: 1)
__global__ void jadj_reduce_kernel(kr_op op, const double* __restrict__ part, int ntiles, int P,
                                   double* __restrict__ out, int64_t ldo, int64_t bso) {
  const int col = blockIdx.y, b = blockIdx.z, ncols = gridDim.y;
  const int blk = (op.reg_kind == KR_REG_TV) ? 1 : 1 + op.ksize * op.ksize;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P; i += gridDim.x * blockDim.x) {
    const double* src = part + ((int64_t)b * ncols + col) * ntiles * P + i;
    double acc = 0.0;
    for (int t = 0; t < ntiles; ++t) acc += src[(int64_t)t * P];
    double wj = op.fweights[i / blk];
    out[b * bso + col * ldo + i] = -wj * acc;
  }
}

// ---------------------------------------------------------------------------
// lower-level cost + gradient (one tile per block, partial cost per tile)

__global__ void __launch_bounds__(NT) lower_eval_kernel(kr_op op, const double* __restrict__ X,
                                                        const double* __restrict__ Y, double* __restrict__ grad,
                                                        double* __restrict__ part) {
  extern __shared__ double smem[];
  const Geom g = make_geom(op);
  Smem sm = carve(g, smem);
  __shared__ double red[4 * 33 + 4];
  load_weights(op, g, sm);
  const int tile = blockIdx.x, b = blockIdx.z, ntiles = gridDim.x;
  const int tyc = tiles_x(op);
  const int y0 = (tile / tyc) * TH, x0 = (tile % tyc) * TW;
  const int rows = op.rows, cols = op.cols, H = g.H;
  const int64_t n = op_n(op);
  const double* x = X + (int64_t)b * n;
  const double* yv = Y + (int64_t)b * n;
  load_region(op, g, TileIn{x, 1.0, nullptr, 0.0}, y0, x0, sm.S0);
  block_barrier();
  double c_data = 0.0, c_ridge = 0.0, c_reg = 0.0;
  const double* mask = (op.data_kind == KR_DATA_MASK) ? op.mask + (int64_t)b * op.mask_bstride : nullptr;
  for (int l = threadIdx.x; l < TPX; l += blockDim.x) {
    int ty = l / TW, tx = l - ty * TW;
    int y = y0 + ty, xx = x0 + tx;
    double acc = 0.0;
    if (y < rows && xx < cols) {
      double v = sm.S0[(ty + H) * g.RW + tx + H];
      int64_t p = (int64_t)y * cols + xx;
      if (mask && mask[p] != 0.0) {
        double r = v - yv[p];
        c_data += r * r;
        acc = op.data_scale == 1.0 ? r : op.data_scale * r;
      }
      acc += op.ridge * v;
      c_ridge += v * v;
    }
    sm.res[l] = acc;
  }
  block_barrier();
  if (op.data_kind == KR_DATA_BLUR) {
    // residual A x - y on rows [y0-rb, y0+TH+rb) ... computed like tile_blur_normal but subtracting y
    const int rb = g.rb, bs = op.blur_size;
    const double* tp = sm.taps;
    const int w1 = TW + 2 * rb, h1 = TH + 4 * rb;
    double* S1 = sm.SA;
    for (int i = threadIdx.x; i < h1 * w1; i += blockDim.x) {
      int r1 = i / w1, c1 = i - r1 * w1;
      const double* src = sm.S0 + (r1 + H - 2 * rb) * g.RW + c1 + H;
      double acc = 0.0;
      for (int u = 0; u < bs; ++u) acc += tp[u] * src[-u];
      S1[i] = acc;
    }
    block_barrier();
    const int w2 = w1, h2 = TH + 2 * rb;
    double* S2 = sm.SB;
    for (int i = threadIdx.x; i < h2 * w2; i += blockDim.x) {
      int r2 = i / w2, c2 = i - r2 * w2;
      int y = y0 - rb + r2, xx = x0 - rb + c2;
      double acc = 0.0;
      if (y >= 0 && y < rows && xx >= 0 && xx < cols) {
        const double* src = S1 + (r2 + 2 * rb) * w1 + c2;
        for (int u = 0; u < bs; ++u) acc += tp[u] * src[-u * w1];
        acc -= yv[(int64_t)y * cols + xx];
        // data cost counted on the tile's own pixels only
        if (r2 >= rb && r2 < rb + TH && c2 >= rb && c2 < rb + TW) c_data += acc * acc;
      }
      S2[i] = acc;
    }
    block_barrier();
    double* S3 = sm.SA;
    for (int i = threadIdx.x; i < h2 * TW; i += blockDim.x) {
      int r3 = i / TW, c3 = i - r3 * TW;
      const double* src = S2 + r3 * w2 + c3;
      double acc = 0.0;
      for (int u = 0; u < bs; ++u) acc += tp[u] * src[u];
      S3[i] = acc;
    }
    block_barrier();
    for (int l = threadIdx.x; l < TPX; l += blockDim.x) {
      int ty = l / TW, tx = l - ty * TW;
      const double* src = S3 + ty * TW + tx;
      double acc = 0.0;
      for (int u = 0; u < bs; ++u) acc += tp[u] * src[u * TW];
      sm.res[l] += op.data_scale * acc;
    }
    block_barrier();
  }
  if (op.reg_kind == KR_REG_FILTERS) {
    const int q = op.ksize, rq = g.rq;
    const int w4 = TW + 2 * rq, h4 = TH + 2 * rq;
    double* S4 = sm.SA;
    const bool quad = (op.potential == KR_POT_QUADRATIC);
    const double e2 = op.eps * op.eps;
    for (int j = 0; j < op.num_filters; ++j) {
      const double* kj = sm.kw + j * q * q;
      const double wj = sm.fw[j];
      double cj = 0.0;
      for (int i = threadIdx.x; i < h4 * w4; i += blockDim.x) {
        int r4 = i / w4, c4 = i - r4 * w4;
        int y = y0 - rq + r4, xx = x0 - rq + c4;
        double e = 0.0;
        if (y >= 0 && y < rows && xx >= 0 && xx < cols) {
          const double* src = sm.S0 + (r4 + H) * g.RW + c4 + H;
          double u = 0.0;
          for (int a = 0; a < q; ++a)
            for (int bb = 0; bb < q; ++bb) u += kj[a * q + bb] * src[-a * g.RW - bb];
          bool own = (r4 >= rq && r4 < rq + TH && c4 >= rq && c4 < rq + TW);
          if (quad) {
            e = 2.0 * u;
            if (own) cj += u * u;
          } else {
            double s = sqrt(u * u + e2);
            e = u / s;
            if (own) cj += s;
          }
        }
        S4[i] = e;
      }
      c_reg += wj * cj;
      block_barrier();
      for (int l = threadIdx.x; l < TPX; l += blockDim.x) {
        int ty = l / TW, tx = l - ty * TW;
        const double* src = S4 + ty * w4 + tx;
        double acc = 0.0;
        for (int a = 0; a < q; ++a)
          for (int bb = 0; bb < q; ++bb) acc += kj[a * q + bb] * src[a * w4 + bb];
        sm.res[l] += wj * acc;
      }
      block_barrier();
    }
  } else if (op.reg_kind == KR_REG_TV) {
    const int w5 = TW + 1, h5 = TH + 1;
    double* PH = sm.SA;
    double* PV = sm.SA + h5 * w5;
    const double e2 = op.eps * op.eps;
    for (int i = threadIdx.x; i < h5 * w5; i += blockDim.x) {
      int r5 = i / w5, c5 = i - r5 * w5;
      int y = y0 - 1 + r5, xx = x0 - 1 + c5;
      double ph = 0.0, pv = 0.0;
      if (y >= 0 && y < rows && xx >= 0 && xx < cols) {
        const double* c = sm.S0 + (y - y0 + H) * g.RW + (xx - x0 + H);
        double dh = (xx < cols - 1) ? c[1] - c[0] : 0.0;
        double dv = (y < rows - 1) ? c[g.RW] - c[0] : 0.0;
        double s = sqrt(dh * dh + dv * dv + e2);
        ph = dh / s;
        pv = dv / s;
        if (r5 >= 1 && c5 >= 1) c_reg += s;
      }
      PH[i] = ph;
      PV[i] = pv;
    }
    c_reg *= sm.fw[0];
    block_barrier();
    const double wa = sm.fw[0];
    for (int l = threadIdx.x; l < TPX; l += blockDim.x) {
      int ty = l / TW, tx = l - ty * TW;
      int i = (ty + 1) * w5 + tx + 1;
      sm.res[l] += wa * ((-PH[i] + PH[i - 1]) + (-PV[i] + PV[i - w5]));
    }
    block_barrier();
  }
  double* gout = grad + (int64_t)b * n;
  for (int l = threadIdx.x; l < TPX; l += blockDim.x) {
    int64_t p = tile_pixel(op, tile, l);
    if (p >= 0) gout[p] = sm.res[l];
  }
  double v3[3] = {c_data, c_ridge, c_reg};
  block_sum<3>(v3, red);
  if (threadIdx.x < 3) part[((int64_t)b * ntiles + tile) * 3 + threadIdx.x] = red[threadIdx.x];
}

// Lower-level cost and gradient for the configs' model family (blur 9/15/21 + learned
// filters q = 3/5/7, smooth-|.| or quadratic potential) through the HVP's templated tile
// machinery: the separable register-blocked blur with the residual A x - y formed in its
// second pass, and the one-filter-per-warp stage with phi' in place of the curvature
// (operators.py:329-353 generalised; same partial layout as lower_eval_kernel).
template <int Q, int BS>
__global__ void __launch_bounds__(NT) lower_eval_fast_kernel(kr_op op, const double* __restrict__ X,
                                                             const double* __restrict__ Y, double* __restrict__ grad,
                                                             double* __restrict__ part) {
  extern __shared__ __align__(128) double smem[];
  const Geom g = make_geom(op);
  Smem sm = carve(g, smem);
  __shared__ double red[4 * 33 + 4];
  load_weights(op, g, sm);
  const int tile = blockIdx.x, b = blockIdx.z, ntiles = gridDim.x;
  const int tyc = tiles_x(op);
  const int y0 = (tile / tyc) * TH, x0 = (tile % tyc) * TW;
  const int rows = op.rows, cols = op.cols, H = g.H;
  const int64_t n = op_n(op);
  load_region(op, g, TileIn{X + (int64_t)b * n, 1.0, nullptr, 0.0}, y0, x0, sm.S0);
  block_barrier();
  double c_data = 0.0, c_ridge = 0.0, c_reg = 0.0;
  for (int l = threadIdx.x; l < TPX; l += blockDim.x) {
    const int ty = l / TW, tx = l - ty * TW;
    const double v = sm.S0[(ty + H) * g.RW + tx + H];
    double acc = 0.0;
    if (y0 + ty < rows && x0 + tx < cols) {
      acc = op.ridge * v;
      c_ridge += v * v;
    }
    sm.res[l] = acc;
  }
  block_barrier();
  blur_normal_bs<BS, true>(op, g, sm, y0, x0, Y + (int64_t)b * n, &c_data);
  tile_filters_q<Q, true>(op, g, sm, b, y0, x0, &c_reg);
  double* gout = grad + (int64_t)b * n;
  for (int l = threadIdx.x; l < TPX; l += blockDim.x) {
    const int64_t p = tile_pixel(op, tile, l);
    if (p >= 0) gout[p] = sm.res[l];
  }
  double v3[3] = {c_data, c_ridge, c_reg};
  block_sum<3>(v3, red);
  if (threadIdx.x < 3) part[((int64_t)b * ntiles + tile) * 3 + threadIdx.x] = red[threadIdx.x];
}

__global__ void lower_reduce_kernel(kr_op op, const double* __restrict__ part, int ntiles, double* cost) {
  const int b = blockIdx.x;
  if (threadIdx.x != 0) return;
  double d = 0.0, r = 0.0, g = 0.0;
  for (int t = 0; t < ntiles; ++t) {
    const double* s = part + ((int64_t)b * ntiles + t) * 3;
    d += s[0];
    r += s[1];
    g += s[2];
  }
  cost[b] = 0.5 * op.data_scale * d + 0.5 * op.ridge * r + g;
}

}  // namespace kr

// ===========================================================================
// C ABI

using namespace kr;

extern "C" int kr_op_prepare(const kr_op* op, kr_stream_t stream) {
  KR_CHECK_ARG(op != nullptr, "null operator");
  KR_TRY(validate_op(*op));
  if (op->reg_kind == KR_REG_NONE || op->data_kind == KR_DATA_DENSE) return KR_OK;
  KR_CHECK_ARG(op->xhat != nullptr && op->slope != nullptr, "prepare needs xhat and slope buffers");
  const int64_t n = op_n(*op);
  dim3 grid((unsigned)((n + 255) / 256 > 1024 ? 1024 : (n + 255) / 256), op->batch);
  if (op->reg_kind == KR_REG_FILTERS) {
    KR_CHECK_ARG(op->potential == KR_POT_QUADRATIC || op->curv != nullptr, "prepare needs a curv buffer");
    prepare_filters_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(*op);
  } else {
    KR_CHECK_ARG(op->curv != nullptr, "prepare needs a curv buffer");
    prepare_tv_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(*op);
  }
  return check_launch("kr_op_prepare");
}

namespace kr {
int hvp_cols(const kr_op* op, const double* V, int64_t ldv, int64_t bsv, int32_t ncols, const int32_t* dims,
             double* HV, int64_t ldo, int64_t bso, cudaStream_t stream);
}

extern "C" int kr_hvp(const kr_op* op, const double* V, int64_t ldv, int64_t bsv, int32_t ncols, double* HV,
                      int64_t ldo, int64_t bso, kr_stream_t stream) {
  return kr::hvp_cols(op, V, ldv, bsv, ncols, nullptr, HV, ldo, bso, (cudaStream_t)stream);
}

// H V with an optional DEVICE per-sample column count dims[b]: columns >= dims[b] are the zero
// padding of a batch padded to its widest sample and are written as zeros without a stencil.
int kr::hvp_cols(const kr_op* op, const double* V, int64_t ldv, int64_t bsv, int32_t ncols, const int32_t* dims,
                 double* HV, int64_t ldo, int64_t bso, cudaStream_t stream) {
  KR_CHECK_ARG(op != nullptr, "null operator");
  KR_TRY(validate_op(*op));
  if (ncols <= 0 || op->batch <= 0) return KR_OK;
  KR_CHECK_ARG(V != nullptr && HV != nullptr, "null vector");
  KR_CHECK_ARG(ldv >= op_n(*op) && ldo >= op_n(*op), "leading dimension smaller than n");
  Geom g = make_geom(*op);
  size_t smem = (size_t)g.total * sizeof(double);
  const void* fn = KR_PICK_Q(hvp_kernel, q_variant(*op));
  KR_TRY(ensure_smem(fn, smem));
  dim3 grid(num_tiles(*op), ncols, op->batch);
  kr_op opv = *op;
  alignas(64) CUtensorMap tmap;
  int use_tma = (op->data_kind != KR_DATA_DENSE && g.RH * (TW + 2 * g.H) <= g.sa &&
                 make_region_tmap(&tmap, V, op->cols, op->rows, ncols, op->batch, ldv, bsv, TW + 2 * g.H, g.RH))
                    ? 1 : 0;
  if (!use_tma) memset(&tmap, 0, sizeof tmap);
  void* args[] = {&opv, (void*)&V, &ldv, &bsv, &HV, &ldo, &bso, (void*)&dims, &tmap, &use_tma};
  cudaError_t e = cudaLaunchKernel(fn, grid, dim3(NT), args, smem, (cudaStream_t)stream);
  if (e != cudaSuccess) return fail(KR_ECUDA, std::string("kr_hvp launch: ") + cudaGetErrorString(e));
  return check_launch("kr_hvp");
}

// ---------------------------------------------------------------------------
// J W for many columns through the materialised mixed Jacobian (the q^2 lag sums of
// _shift_dot, operators.py:386-408, become rows of a p x n matrix):

namespace kr {

// The mixed Jacobian materialised: J w is linear in w, so J W for many columns is
// one GEMM with the p x n matrix Mt = J (operators.py:411-444 restated per pixel):
//   Mt[j(1+q^2)]     = -w_j C_j^T phi'_j                                  (theta0 head)
//   Mt[j(1+q^2)+1+d] = -w_j [ phi'_j(. + delta_d) + C_j^T(phi''_j . xhat(. - delta_d)) ]
// (the two _shift_dot terms, with <C_j w, phi'' . S_d xhat> = <w, C_j^T(phi'' . S_d xhat)>).
// One block per (tile, filter, sample): phi'_j, phi''_j on the tile + R halo and xhat on
// the tile + 2R halo in smem; C_j^T is the correlation sum_{a,b} k[a][b] u(y-R+a, x-R+b).
template <int Q>
__global__ void __launch_bounds__(NT) jmat_kernel(kr_op op, double* __restrict__ Mt, int64_t bsm) {
  constexpr int R = Q / 2, Q2 = Q * Q;
  constexpr int EW = TW + 2 * R, EH = TH + 2 * R, XW = TW + 4 * R, XH = TH + 4 * R;
  __shared__ double ps[EH * EW];  // phi'_j
  __shared__ double pc[EH * EW];  // phi''_j (2 for the quadratic potential), zero outside
  __shared__ double xs[XH * XW];  // xhat
  const int tile = blockIdx.x, j = blockIdx.y, b = blockIdx.z, J = op.num_filters;
  const int tyc = tiles_x(op);
  const int y0 = (tile / tyc) * TH, x0 = (tile % tyc) * TW;
  const int rows = op.rows, cols = op.cols;
  const int64_t n = op_n(op);
  const bool quad = op.potential == KR_POT_QUADRATIC;
  const double* sl = op.slope + ((int64_t)b * J + j) * n;
  const double* cv = quad ? nullptr : op.curv + ((int64_t)b * J + j) * n;
  const double* xh = op.xhat + (int64_t)b * n;
  for (int i = threadIdx.x; i < EH * EW; i += NT) {
    const int y = y0 - R + i / EW, x = x0 - R + i % EW;
    const bool in = y >= 0 && y < rows && x >= 0 && x < cols;
    const int64_t pp = (int64_t)y * cols + x;
    ps[i] = in ? sl[pp] : 0.0;
    pc[i] = in ? (quad ? 2.0 : cv[pp]) : 0.0;
  }
  for (int i = threadIdx.x; i < XH * XW; i += NT) {
    const int y = y0 - 2 * R + i / XW, x = x0 - 2 * R + i % XW;
    xs[i] = (y >= 0 && y < rows && x >= 0 && x < cols) ? xh[(int64_t)y * cols + x] : 0.0;
  }
  double k[Q2];
#pragma unroll
  for (int i = 0; i < Q2; ++i) k[i] = op.kernels[j * Q2 + i];
  const double nw = -op.fweights[j];
  block_barrier();
  double* base = Mt + (int64_t)b * bsm + (int64_t)j * (1 + Q2) * n;
  for (int l = threadIdx.x; l < TPX; l += NT) {
    const int ty = l / TW, tx = l - ty * TW;
    const int y = y0 + ty, x = x0 + tx;
    if (y >= rows || x >= cols) continue;
    const int64_t p = (int64_t)y * cols + x;
    double h = 0.0;
#pragma unroll
    for (int a = 0; a < Q; ++a)
#pragma unroll
      for (int bb = 0; bb < Q; ++bb) h = fma(k[a * Q + bb], ps[(ty + a) * EW + tx + bb], h);
    base[p] = nw * h;
    for (int d = 0; d < Q2; ++d) {
      const int da = d / Q - R, db = d % Q - R;
      double v = 0.0;
      const double* xr = xs + (ty + R - da) * XW + tx + R - db;
#pragma unroll
      for (int a = 0; a < Q; ++a)
#pragma unroll
        for (int bb = 0; bb < Q; ++bb) v = fma(k[a * Q + bb], pc[(ty + a) * EW + tx + bb] * xr[a * XW + bb], v);
      v += ps[(ty + R + da) * EW + tx + R + db];
      base[(int64_t)(1 + d) * n + p] = nw * v;
    }
  }
}

static bool jw_jmat_path(const kr_op& op, int ncols) { return q_variant(op) > 0 && ncols >= 4; }

// samples per jmat pass: the materialised J of a pass stays under 64 M doubles (512 MB)
static int jmat_chunk(const kr_op& op) {
  const int64_t per = (int64_t)op.num_filters * (1 + op.ksize * op.ksize) * op_n(op);
  int64_t c = ((int64_t)64 << 20) / (per > 0 ? per : 1);
  if (c < 1) c = 1;
  return (int)(c < op.batch ? c : op.batch);
}

}  // namespace kr

extern "C" int64_t kr_jadj_workspace(const kr_op* op, int32_t ncols) {
  if (!op || validate_op(*op) != KR_OK) return -1;
  if (jw_jmat_path(*op, ncols)) {
    const int P = op->num_filters * (1 + op->ksize * op->ksize);
    return (int64_t)jmat_chunk(*op) * P * op_n(*op) + gram_dmma_workspace(jmat_chunk(*op), ncols, P, op_n(*op), false);
  }
  int64_t P = (op->reg_kind == KR_REG_TV) ? 1 : (int64_t)op->num_filters * (1 + op->ksize * op->ksize);
  return (int64_t)op->batch * ncols * num_tiles(*op) * P;
}

// J W through the materialised Jacobian: one jmat launch for all samples, then one
// strided-batched DGEMM  JW_b (cols x p) = W_b Mt_b^T.
static int jadj_jmat(const kr_op& op, const double* W, int64_t ldw, int64_t bsw, int32_t ncols, double* JW,
                     int64_t ldo, int64_t bso, double* work, cudaStream_t st) {
  const int64_t n = op_n(op);
  const int q = op.ksize, P = op.num_filters * (1 + q * q);
  KR_CHECK_ARG(ldo >= P, "output leading dimension smaller than p");
  const int64_t bsm = (int64_t)P * n;
  const void* fn = q == 3 ? (const void*)jmat_kernel<3> : q == 5 ? (const void*)jmat_kernel<5>
                                                               : (const void*)jmat_kernel<7>;
  const int chunk = jmat_chunk(op);
  double* gws = work + (int64_t)chunk * bsm;  // tile partials of the product
  const int64_t gwl = gram_dmma_workspace(chunk, ncols, P, n, false);
  for (int b0 = 0; b0 < op.batch; b0 += chunk) {
    const int nb = (op.batch - b0) < chunk ? (op.batch - b0) : chunk;
    kr_op opv = op;  // samples b0 .. b0+nb-1 as a batch of nb
    opv.batch = nb;
    opv.slope = op.slope + (int64_t)b0 * op.num_filters * n;
    if (op.curv) opv.curv = op.curv + (int64_t)b0 * op.num_filters * n;
    opv.xhat = op.xhat + (int64_t)b0 * n;
    double* Mt = work;
    int64_t bsmv = bsm;
    void* args[] = {&opv, &Mt, &bsmv};
    cudaError_t e = cudaLaunchKernel(fn, dim3(num_tiles(op), op.num_filters, nb), dim3(NT), args, 0, st);
    if (e != cudaSuccess) return fail(KR_ECUDA, std::string("jmat launch: ") + cudaGetErrorString(e));
    KR_TRY(check_launch("jmat"));
    // out (cols x P, row-major, ld ldo): out[c][j] = w_c . Mt_j over the pixels (DMMA, kr_gemm.cu)
    KR_TRY(gram_dmma(W + (int64_t)b0 * bsw, ldw, bsw, Mt, n, bsm, nb, ncols, P, n, false, JW + (int64_t)b0 * bso, ldo,
                     bso, gws, gwl, st));
  }
  return KR_OK;
}

extern "C" int kr_jadj(const kr_op* op, const double* W, int64_t ldw, int64_t bsw, int32_t ncols, double* JW,
                       int64_t ldo, int64_t bso, double* work, int64_t work_len, kr_stream_t stream) {
  KR_CHECK_ARG(op != nullptr, "null operator");
  KR_TRY(validate_op(*op));
  KR_CHECK_ARG(op->reg_kind != KR_REG_NONE && op->data_kind != KR_DATA_DENSE, "operator has no mixed Jacobian");
  if (ncols <= 0 || op->batch <= 0) return KR_OK;
  KR_CHECK_ARG(op->slope != nullptr, "jadj needs the prepared slope table (call kr_op_prepare)");
  KR_CHECK_ARG(work_len >= kr_jadj_workspace(op, ncols), "jadj workspace too small");
  const int ntiles = num_tiles(*op);
  dim3 grid(ntiles, ncols, op->batch);
  cudaStream_t st = (cudaStream_t)stream;
  if (jw_jmat_path(*op, ncols)) return jadj_jmat(*op, W, ldw, bsw, ncols, JW, ldo, bso, work, st);
  int P;
  if (op->reg_kind == KR_REG_FILTERS) {
    const int q = op->ksize, rq = q / 2;
    P = op->num_filters * (1 + q * q);
    KR_CHECK_ARG(ldo >= P, "output leading dimension smaller than p");
    size_t smem = sizeof(double) * ((size_t)(TH + 4 * rq) * (TW + 4 * rq) + (TH + 2 * rq) * (TW + 2 * rq) +
                                    op->num_filters * q * q + 8 * 33 + 8);
    KR_TRY(ensure_smem((const void*)jadj_filters_kernel, smem));
    jadj_filters_kernel<<<grid, NT, smem, st>>>(*op, W, ldw, bsw, work);
  } else {
    P = 1;
    KR_CHECK_ARG(ldo >= 1, "output leading dimension smaller than p");
    jadj_tv_kernel<<<grid, NT, 0, st>>>(*op, W, ldw, bsw, work);
  }
  KR_TRY(check_launch("kr_jadj"));
  dim3 rgrid((P + 127) / 128, ncols, op->batch);
  jadj_reduce_kernel<<<rgrid, 128, 0, st>>>(*op, work, ntiles, P, JW, ldo, bso);
  return check_launch("kr_jadj reduce");
}

extern "C" int64_t kr_lower_workspace(const kr_op* op) {
  if (!op || validate_op(*op) != KR_OK) return -1;
  return (int64_t)op->batch * num_tiles(*op) * 3;
}

extern "C" int kr_lower_eval(const kr_op* op, const double* X, const double* Y, double* cost, double* grad,
                             double* work, int64_t work_len, kr_stream_t stream) {
  KR_CHECK_ARG(op != nullptr, "null operator");
  KR_TRY(validate_op(*op));
  KR_CHECK_ARG(op->data_kind != KR_DATA_DENSE, "dense operators have no lower-level cost");
  KR_CHECK_ARG(X && Y && cost && grad, "null pointer");
  KR_CHECK_ARG(work_len >= kr_lower_workspace(op), "lower workspace too small");
  Geom g = make_geom(*op);
  size_t smem = (size_t)g.total * sizeof(double);
  const int ntiles = num_tiles(*op);
  cudaStream_t st = (cudaStream_t)stream;
  const void* fast = nullptr;
  static const bool generic_only = getenv("KR_LOWER_GENERIC") != nullptr;
  if (!generic_only && op->data_kind == KR_DATA_BLUR && op->reg_kind == KR_REG_FILTERS) {
#define KR_LFAST(QQ, BB) \
    if (op->ksize == QQ && op->blur_size == BB) fast = (const void*)lower_eval_fast_kernel<QQ, BB>;
    KR_LFAST(3, 9) KR_LFAST(3, 15) KR_LFAST(3, 21) KR_LFAST(5, 9) KR_LFAST(5, 15) KR_LFAST(5, 21)
    KR_LFAST(7, 9) KR_LFAST(7, 15) KR_LFAST(7, 21)
#undef KR_LFAST
  }
  if (fast) {
    KR_TRY(ensure_smem(fast, smem));
    kr_op opv = *op;
    void* args[] = {&opv, (void*)&X, (void*)&Y, &grad, &work};
    const cudaError_t e = cudaLaunchKernel(fast, dim3(ntiles, 1, op->batch), dim3(NT), args, smem, st);
    if (e != cudaSuccess) return fail(KR_ECUDA, std::string("kr_lower_eval launch: ") + cudaGetErrorString(e));
  } else {
    KR_TRY(ensure_smem((const void*)lower_eval_kernel, smem));
    lower_eval_kernel<<<dim3(ntiles, 1, op->batch), NT, smem, st>>>(*op, X, Y, grad, work);
  }
  KR_TRY(check_launch("kr_lower_eval"));
  lower_reduce_kernel<<<op->batch, 32, 0, st>>>(*op, work, ntiles, cost);
  return check_launch("kr_lower_eval reduce");
}
