// kr_gemm.cu -- the tall-skinny fp64 products of the recycle update on the fp64 tensor
// cores (mma.sync m8n8k4 f64 = DMMA; tcgen05 has no fp64 kind), hand-written for the
// shapes and the structure the update has:
//
//   gram:      G_b[i][j] = x_i . y_j over n pixels (rows contiguous), t x t from t x n --
//              the Grams of the Cholesky-QR passes and W^T H W (recycling.py:194, 250, 333),
//              J W against the materialised mixed Jacobian.  Symmetric products compute
//              only the tile blocks on and below the diagonal and mirror them (half the
//              flops of a general GEMM); split-K over the pixels with partials summed in
//              fixed order (deterministic).
//   rows_mul:  Y_b = alpha F_b X_b + beta Y_b, (R2 x R1)(R1 x L) with L = n pixels -- the
//              W <- R^-T A passes of the Cholesky-QR (F lower triangular: the k loop of a
//              tile row stops at its diagonal block, half the flops again), the pivoted
//              basis change, U~ = W X, H U~ = (H W) X, Z = W V_H diag(mu).
//
// Both stage their operand tiles with a 3-deep cp.async pipeline into padded shared
// memory (row stride = 4 mod 16 doubles: every fragment load is conflict-free), 8 warps
// per CTA, accumulators in registers.  DMMA issues one instruction per 256 FMAs, so the
// fp64 pipe -- the bound of these products (t/16 >= 20 flop/B at C3) -- is fed by one
// shared load per MMA or less.

#include "kr_common.cuh"
#include "kr_internal.h"

namespace kr {
namespace {

constexpr int GT = 256;      // threads per CTA
constexpr int STAGES = 3;

__device__ __forceinline__ void cp16(void* s, const void* g, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(s)), "l"(g), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp8(void* s, const void* g, int bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(s)), "l"(g), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Two consecutive doubles of a row from global to shared, zero-filled past `valid` doubles.
// V16: one 16-byte copy (both addresses 16-byte aligned).  Dead pairs (valid <= 0: pad rows,
// the tail of the k range) are plain shared stores: a zero-size cp.async still sends its
// request, and thousands of them on one dummy address serialise in L2 (measured: an edge
// tile with 10 live rows took as long as a full one).
template <bool V16>
__device__ __forceinline__ void cp_pair(double* s, const double* g, int64_t valid) {
  if (valid <= 0) {
    if (V16) {
      *reinterpret_cast<double2*>(s) = make_double2(0.0, 0.0);
    } else {
      s[0] = 0.0;
      s[1] = 0.0;
    }
  } else if (V16) {
    cp16(s, g, valid >= 2 ? 16 : 8);
  } else {
    cp8(s, g, 8);
    if (valid >= 2) cp8(s + 1, g + 1, 8);
    else s[1] = 0.0;
  }
}

// ------------------------------------------------------------------ gram

constexpr int GM = 64, GN = 64, GK = 32, GLD = GK + 4;  // tile and padded row stride (36 = 4 mod 16)
constexpr int G_STAGE = (GM + GN) * GLD;                // doubles per stage
constexpr size_t G_SMEM = sizeof(double) * STAGES * G_STAGE;

struct GramParams {
  const double* X;
  const double* Y;
  int64_t ldx, bsx, ldy, bsy;
  int rx, ry;
  int64_t n;
  int S;          // splits of the pixel dimension
  int64_t chunk;  // pixels per split (multiple of GK)
  int sym;        // 1: lower tile blocks only (rx == ry), mirrored by the sum kernel
  int tn;         // tile columns (general case)
  int ntile;      // tiles per (sample, split)
  double* part;   // [batch][S][ntile][GM * GN]
  const int32_t* dims;  // nullable: per-sample live rows (the rows beyond are zero pad rows)
  int dim_x, dim_y;     // dims bounds the rows of X / of Y
};

__device__ __forceinline__ void tile_of(const GramParams& P, int q, int& ti, int& tj) {
  if (P.sym) {
    ti = 0;
    while ((ti + 1) * (ti + 2) / 2 <= q) ++ti;
    tj = q - ti * (ti + 1) / 2;
  } else {
    ti = q / P.tn;
    tj = q - ti * P.tn;
  }
}

template <bool V16>
__global__ void __launch_bounds__(GT, 2) gram_dmma_kernel(const GramParams P) {
  extern __shared__ __align__(16) double gsm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;  // 2 x 4 warps: warp tile 32 x 16
  int ti, tj;
  tile_of(P, blockIdx.x, ti, tj);
  const int sp = blockIdx.y, b = blockIdx.z;
  const double* Xb = P.X + (int64_t)b * P.bsx;
  const double* Yb = P.Y + (int64_t)b * P.bsy;
  const bool same = P.X == P.Y && ti == tj;  // diagonal tile of a true Gram: one operand tile
  // live extents: 8-row MMA blocks past them (tile padding, a sample's zero pad rows) are
  // skipped.  A warp's blocks are dealt cyclically (row blocks wm + 2 mi, column blocks
  // wn + 4 ni), so the live blocks of an edge tile spread evenly over the warps and over the
  // SM's four schedulers (a warp is pinned to one)
  int rx = P.rx, ry = P.ry;
  if (P.dims) {
    const int d = P.dims[b];
    if (P.dim_x && d < rx) rx = d;
    if (P.dim_y && d < ry) ry = d;
  }
  int mcnt = 0, ncnt = 0;  // live row / column blocks of this warp (prefixes: the blocks ascend)
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) mcnt += (ti * GM + (wm + 2 * mi) * 8 < rx) ? 1 : 0;
#pragma unroll
  for (int ni = 0; ni < 2; ++ni) ncnt += (tj * GN + (wn + 4 * ni) * 8 < ry) ? 1 : 0;
  const bool full = mcnt == 4 && ncnt == 2;
  if (ti * GM >= rx || tj * GN >= ry) {  // nothing live in this tile
    double* out = P.part + (((int64_t)b * P.S + blockIdx.y) * P.ntile + blockIdx.x) * (GM * GN);
    for (int e = tid; e < GM * GN; e += GT) out[e] = 0.0;
    return;
  }
  const int64_t k_begin = (int64_t)sp * P.chunk;
  const int64_t k_end = k_begin + P.chunk < P.n ? k_begin + P.chunk : P.n;
  const int nk = k_end > k_begin ? (int)((k_end - k_begin + GK - 1) / GK) : 0;

  auto load = [&](int stage, int kt) {
    double* xs = gsm + stage * G_STAGE;
    double* ys = xs + GM * GLD;
    const int64_t k0 = k_begin + (int64_t)kt * GK;
#pragma unroll
    for (int i = 0; i < (GM * GK / 2) / GT; ++i) {
      const int c = tid + i * GT, row = c / (GK / 2), cc = (c % (GK / 2)) * 2;
      const int64_t pcol = k0 + cc;
      const int gx = ti * GM + row;
      cp_pair<V16>(xs + row * GLD + cc, Xb + (int64_t)gx * P.ldx + pcol, gx < rx ? k_end - pcol : 0);
      if (!same) {
        const int gy = tj * GN + row;
        cp_pair<V16>(ys + row * GLD + cc, Yb + (int64_t)gy * P.ldy + pcol, gy < ry ? k_end - pcol : 0);
      }
    }
  };

  double acc[4][2][2];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;

  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load(s, s);
    cp_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_wait<STAGES - 2>();
    __syncthreads();
    if (kt + STAGES - 1 < nk) load((kt + STAGES - 1) % STAGES, kt + STAGES - 1);
    cp_commit();
    const double* xs = gsm + (kt % STAGES) * G_STAGE;
    const double* ys = same ? xs : xs + GM * GLD;
    const double* xa = xs + (wm * 8 + (lane >> 2)) * GLD + (lane & 3);
    const double* yb = ys + (wn * 8 + (lane >> 2)) * GLD + (lane & 3);
    if (full) {
#pragma unroll
      for (int ks = 0; ks < GK / 4; ++ks) {
        double a[4], bb[2];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) a[mi] = xa[mi * 16 * GLD + ks * 4];
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) bb[ni] = yb[ni * 32 * GLD + ks * 4];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int ni = 0; ni < 2; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], a[mi], bb[ni]);
      }
    } else if (mcnt > 0 && ncnt > 0) {
#pragma unroll
      for (int ks = 0; ks < GK / 4; ++ks) {
        double a[4], bb[2];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) a[mi] = mi < mcnt ? xa[mi * 16 * GLD + ks * 4] : 0.0;
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) bb[ni] = ni < ncnt ? yb[ni * 32 * GLD + ks * 4] : 0.0;
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int ni = 0; ni < 2; ++ni)
            if (mi < mcnt && ni < ncnt) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], a[mi], bb[ni]);
      }
    }
  }
  cp_wait<0>();
  double* out = P.part + (((int64_t)b * P.S + sp) * P.ntile + blockIdx.x) * (GM * GN);
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) {
      const int r = (wm + 2 * mi) * 8 + (lane >> 2), cidx = (wn + 4 * ni) * 8 + 2 * (lane & 3);
      *reinterpret_cast<double2*>(out + r * GN + cidx) = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
    }
}

// G = sum over the splits (fixed order) of the tile partials; symmetric products mirror
// the off-diagonal tiles
__global__ void gram_tile_sum_kernel(const GramParams P, double* G, int64_t ldg, int64_t bsg) {
  const int q = blockIdx.x, b = blockIdx.y;
  int ti, tj;
  tile_of(P, q, ti, tj);
  const double* part = P.part + ((int64_t)b * P.S * P.ntile + q) * (GM * GN);
  double* Gb = G + (int64_t)b * bsg;
  for (int e = threadIdx.x; e < GM * GN; e += blockDim.x) {
    double acc = 0.0;
    for (int s = 0; s < P.S; ++s) acc += part[(int64_t)s * P.ntile * (GM * GN) + e];
    const int gi = ti * GM + e / GN, gj = tj * GN + e % GN;
    if (gi < P.rx && gj < P.ry && !(P.sym && gj > gi)) {  // (the strict upper triangle is the mirror)
      Gb[(int64_t)gi * ldg + gj] = acc;
      if (P.sym && gi != gj) Gb[(int64_t)gj * ldg + gi] = acc;
    }
  }
}

int gram_splits(int batch, int ntile, int64_t n) {
  // The CTAs run in whole waves of 2 per SM, each CTA for n / S pixels: pick the split count
  // that minimises waves x k-tiles per CTA (at t = 330, 16 samples: S = 7 fills 7.95 waves where
  // S = 4 leaves the fifth wave half empty); at least 8 k-tiles per split, at most 32 splits
  int sms = device_sms();
  if (sms < 1) sms = 148;
  const int64_t slots = 2 * (int64_t)sms, base = (int64_t)batch * ntile;
  const int64_t kt = (n + GK - 1) / GK;
  int best = 1;
  int64_t best_cost = -1;
  bool best_wide = false;
  for (int S = 1; S <= 32; ++S) {
    const int64_t per = (kt + S - 1) / S;
    if (S > 1 && per < 8) break;
    const int64_t waves = (base * S + slots - 1) / slots;
    const int64_t cost = waves * (per + 6);  // + pipeline fill / epilogue of a CTA
    // at least ~4 waves when the pixels allow it: with one or two long waves the CTAs of the
    // last wave cannot be balanced (measured: 576 CTAs of 2048 k-tiles slower than 2304 of 512)
    const bool wide = base * S >= 4 * slots;
    if (best_cost < 0 || (wide && !best_wide) || (wide == best_wide && cost < best_cost)) {
      best_cost = cost;
      best = S;
      best_wide = wide;
    }
  }
  return best;
}

void gram_plan(GramParams& P, int batch, int rx, int ry, int64_t n, bool sym) {
  const int tm = (rx + GM - 1) / GM, tn = (ry + GN - 1) / GN;
  P.rx = rx;
  P.ry = ry;
  P.n = n;
  P.sym = sym ? 1 : 0;
  P.tn = tn;
  P.ntile = sym ? tm * (tm + 1) / 2 : tm * tn;
  P.S = gram_splits(batch, P.ntile, n);
  const int64_t per = (n + P.S - 1) / P.S;
  P.chunk = (per + GK - 1) / GK * GK;
}

// ------------------------------------------------------------------ rows_mul

constexpr int MN = 128, MK = 16, MLDF = MK + 4, MLDX = MN + 4;  // 20 and 132 = 4 mod 16

template <int BM>
struct MulGeo {
  static constexpr int WM = BM / 32;        // warps along the rows
  static constexpr int WN = 8 / WM;         // warps along the pixels
  static constexpr int WCOLS = MN / WN;     // pixels per warp (32 or 16)
  static constexpr int NI = WCOLS / 8;
  static constexpr int STAGE = BM * MLDF + MK * MLDX;
  static constexpr size_t SMEM = sizeof(double) * STAGES * STAGE;
};

struct MulParams {
  const double* F;
  int64_t ldf, sF;
  const double* X;
  int64_t ldX, sX;
  double* Y;
  int64_t ldY, sY;
  int R2, R1;
  int64_t L;
  double alpha, beta;
  int lower;    // F lower triangular (zero above the diagonal): the k loop stops at the diagonal block
  int tiles_i;  // row tiles
  int st2;      // 16-byte stores allowed
  const int32_t* dims;  // nullable: per-sample live extent
  int dim_r, dim_k;     // dims bounds the output rows (the rest come out as beta Y) / the k extent
};

template <int BM, bool V16>
__global__ void __launch_bounds__(GT, 2) rows_mul_dmma_kernel(const MulParams P) {
  using Gm = MulGeo<BM>;
  extern __shared__ __align__(16) double gsm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / Gm::WN, wn = warp % Gm::WN;
  // row tiles fastest (they share the X tile through L2), the heavy (lowest) ones first
  const int it = P.tiles_i - 1 - (int)(blockIdx.x % P.tiles_i);
  const int64_t p0 = (int64_t)(blockIdx.x / P.tiles_i) * MN;
  const int i0 = it * BM, b = blockIdx.z;
  const double* Fb = P.F + (int64_t)b * P.sF;
  const double* Xb = P.X + (int64_t)b * P.sX;
  double* Yb = P.Y + (int64_t)b * P.sY;
  int R2 = P.R2, R1 = P.R1;
  if (P.dims) {
    const int d = P.dims[b];
    if (P.dim_r && d < R2) R2 = d;
    if (P.dim_k && d < R1) R1 = d;
  }
  int kend = (P.lower && i0 + BM < R1) ? i0 + BM : R1;
  if (i0 >= R2) kend = 0;  // no live row: the tile is beta Y
  const int nk = (kend + MK - 1) / MK;
  // per 8-row MMA block of this warp (dealt cyclically over the warp rows: block wm + WM mi,
  // so live rows and the triangular k extents balance): the k extent (0 past the live rows; a
  // triangular F stops at the block's last row)
  int kmi[4], kw = 0, kall = 1 << 30;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
    const int rb = i0 + (wm + Gm::WM * mi) * 8;
    kmi[mi] = rb >= R2 ? 0 : (P.lower && rb + 8 < kend) ? rb + 8 : kend;
    kw = kmi[mi] > kw ? kmi[mi] : kw;
    kall = kmi[mi] < kall ? kmi[mi] : kall;
  }

  auto load = [&](int stage, int kt) {
    double* fs = gsm + stage * Gm::STAGE;
    double* xs = fs + BM * MLDF;
    const int k0 = kt * MK;
#pragma unroll
    for (int i = 0; i < (BM * MK) / GT; ++i) {
      const int e = tid + i * GT, row = e / MK, col = e % MK;
      const int gi = i0 + row, gj = k0 + col;
      const bool ok = gi < R2 && gj < kend;
      if (ok) cp8(fs + row * MLDF + col, Fb + (int64_t)gi * P.ldf + gj, 8);
      else fs[row * MLDF + col] = 0.0;
    }
#pragma unroll
    for (int i = 0; i < (MK * MN / 2) / GT; ++i) {
      const int c = tid + i * GT, row = c / (MN / 2), cc = (c % (MN / 2)) * 2;
      const int gj = k0 + row;
      const int64_t pc = p0 + cc;
      cp_pair<V16>(xs + row * MLDX + cc, Xb + (int64_t)gj * P.ldX + pc, gj < kend ? P.L - pc : 0);
    }
  };

  double acc[4][Gm::NI][2];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < Gm::NI; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;

  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load(s, s);
    cp_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_wait<STAGES - 2>();
    __syncthreads();
    if (kt + STAGES - 1 < nk) load((kt + STAGES - 1) % STAGES, kt + STAGES - 1);
    cp_commit();
    const double* fs = gsm + (kt % STAGES) * Gm::STAGE;
    const double* xs = fs + BM * MLDF;
    const double* fa = fs + (wm * 8 + (lane >> 2)) * MLDF + (lane & 3);
    const double* xb = xs + (lane & 3) * MLDX + wn * Gm::WCOLS + (lane >> 2);
#pragma unroll
    for (int ks = 0; ks < MK / 4; ++ks) {
      const int kg = kt * MK + ks * 4;
      if (kg >= kw) break;
      double a[4], bb[Gm::NI];
#pragma unroll
      for (int ni = 0; ni < Gm::NI; ++ni) bb[ni] = xb[ks * 4 * MLDX + ni * 8];
      if (kg + 4 <= kall) {  // every block live at this k-step: branch-free
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) a[mi] = fa[mi * Gm::WM * 8 * MLDF + ks * 4];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int ni = 0; ni < Gm::NI; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], a[mi], bb[ni]);
      } else {
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) a[mi] = kg < kmi[mi] ? fa[mi * Gm::WM * 8 * MLDF + ks * 4] : 0.0;
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
          if (kg < kmi[mi]) {
#pragma unroll
            for (int ni = 0; ni < Gm::NI; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], a[mi], bb[ni]);
          }
      }
    }
  }
  cp_wait<0>();
  const double alpha = P.alpha, beta = P.beta;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
    const int gi = i0 + (wm + Gm::WM * mi) * 8 + (lane >> 2);
    if (gi >= P.R2) continue;
#pragma unroll
    for (int ni = 0; ni < Gm::NI; ++ni) {
      const int64_t pc = p0 + wn * Gm::WCOLS + ni * 8 + 2 * (lane & 3);
      if (pc >= P.L) continue;
      double* y = Yb + (int64_t)gi * P.ldY + pc;
      double v0 = alpha * acc[mi][ni][0], v1 = alpha * acc[mi][ni][1];
      if (P.st2 && pc + 1 < P.L) {
        if (beta != 0.0) {
          const double2 o = *reinterpret_cast<const double2*>(y);
          v0 += beta * o.x;
          v1 += beta * o.y;
        }
        *reinterpret_cast<double2*>(y) = make_double2(v0, v1);
      } else {
        y[0] = beta != 0.0 ? v0 + beta * y[0] : v0;
        if (pc + 1 < P.L) y[1] = beta != 0.0 ? v1 + beta * y[1] : v1;
      }
    }
  }
}

bool al16(const void* p) { return ((uintptr_t)p & 15) == 0; }

template <int BM>
int launch_mul(const MulParams& P, int batch, bool v16, cudaStream_t st) {
  using Gm = MulGeo<BM>;
  const int64_t tiles_p = (P.L + MN - 1) / MN;
  const dim3 grid((unsigned)(tiles_p * P.tiles_i), 1, batch);
  const void* fn = v16 ? (const void*)rows_mul_dmma_kernel<BM, true> : (const void*)rows_mul_dmma_kernel<BM, false>;
  KR_TRY(ensure_smem(fn, Gm::SMEM));
  MulParams Pv = P;
  void* args[] = {&Pv};
  cudaError_t e = cudaLaunchKernel(fn, grid, dim3(GT), args, Gm::SMEM, st);
  if (e != cudaSuccess) return fail(KR_ECUDA, std::string("rows_mul launch: ") + cudaGetErrorString(e));
  return check_launch("rows_mul (dmma)");
}

}  // namespace

int64_t gram_dmma_workspace(int batch, int rx, int ry, int64_t n, bool sym) {
  if (batch <= 0 || rx <= 0 || ry <= 0 || n <= 0) return 1;
  GramParams P{};
  gram_plan(P, batch, rx, ry, n, sym);
  return (int64_t)batch * P.S * P.ntile * (GM * GN);
}

int gram_dmma(const double* X, int64_t ldx, int64_t bsx, const double* Y, int64_t ldy, int64_t bsy, int batch, int rx,
              int ry, int64_t n, bool sym, double* G, int64_t ldg, int64_t bsg, double* work, int64_t work_len,
              cudaStream_t st, const int32_t* dims, int dims_mask) {
  if (batch == 0 || rx == 0 || ry == 0) return KR_OK;
  KR_CHECK_ARG(!sym || rx == ry, "symmetric Gram needs equal row counts");
  GramParams P{};
  gram_plan(P, batch, rx, ry, n, sym);
  KR_CHECK_ARG(work && work_len >= (int64_t)batch * P.S * P.ntile * (GM * GN), "gram workspace too small");
  P.X = X;
  P.Y = Y;
  P.ldx = ldx;
  P.bsx = bsx;
  P.ldy = ldy;
  P.bsy = bsy;
  P.part = work;
  P.dims = dims;
  P.dim_x = dims_mask & 1;
  P.dim_y = (dims_mask >> 1) & 1;
  const bool v16 = al16(X) && al16(Y) && ldx % 2 == 0 && bsx % 2 == 0 && ldy % 2 == 0 && bsy % 2 == 0;
  const void* fn = v16 ? (const void*)gram_dmma_kernel<true> : (const void*)gram_dmma_kernel<false>;
  KR_TRY(ensure_smem(fn, G_SMEM));
  void* args[] = {&P};
  cudaError_t e = cudaLaunchKernel(fn, dim3(P.ntile, P.S, batch), dim3(GT), args, G_SMEM, st);
  if (e != cudaSuccess) return fail(KR_ECUDA, std::string("gram launch: ") + cudaGetErrorString(e));
  gram_tile_sum_kernel<<<dim3(P.ntile, batch), 256, 0, st>>>(P, G, ldg, bsg);
  return check_launch("gram (dmma)");
}

int rows_mul_dmma(const double* F, int64_t ldf, int64_t sF, const double* X, int64_t ldX, int64_t sX, double* Y,
                  int64_t ldY, int64_t sY, int R2, int R1, int64_t L, int batch, double alpha, double beta, bool lower,
                  cudaStream_t st, const int32_t* dims, int dims_mask) {
  if (batch == 0 || R2 == 0 || L == 0) return KR_OK;
  MulParams P{};
  P.F = F;
  P.ldf = ldf;
  P.sF = sF;
  P.X = X;
  P.ldX = ldX;
  P.sX = sX;
  P.Y = Y;
  P.ldY = ldY;
  P.sY = sY;
  P.R2 = R2;
  P.R1 = R1;
  P.L = L;
  P.alpha = alpha;
  P.beta = beta;
  P.lower = lower ? 1 : 0;
  P.dims = dims;
  P.dim_r = dims_mask & 1;
  P.dim_k = (dims_mask >> 1) & 1;
  const bool v16 = al16(X) && ldX % 2 == 0 && sX % 2 == 0;
  P.st2 = (al16(Y) && ldY % 2 == 0 && sY % 2 == 0) ? 1 : 0;
  if (R2 <= 32) {
    P.tiles_i = 1;
    return launch_mul<32>(P, batch, v16, st);
  }
  P.tiles_i = (R2 + 63) / 64;
  return launch_mul<64>(P, batch, v16, st);
}

}  // namespace kr

extern "C" int kr_rows_mul(const double* F, int64_t ldf, int64_t bsf, const double* X, int64_t ldx, int64_t bsx, double* Y,
                           int64_t ldy, int64_t bsy, int32_t r2, int32_t r1, int64_t L, int32_t batch, double alpha,
                           double beta, int32_t lower, kr_stream_t stream) {
  KR_CHECK_ARG(batch >= 0 && r2 >= 0 && r1 >= 0 && L >= 0, "negative size");
  if (batch == 0 || r2 == 0 || L == 0) return KR_OK;
  KR_CHECK_ARG(F && X && Y, "null pointer");
  KR_CHECK_ARG(ldf >= r1 && ldx >= L && ldy >= L, "leading dimension too small");
  return kr::rows_mul_dmma(F, ldf, bsf, X, ldx, bsx, Y, ldy, bsy, r2, r1, L, batch, alpha, beta, lower != 0,
                           (cudaStream_t)stream, nullptr, 0);
}
