// kr_common.cuh -- shared device code: operator descriptor access, tile
// geometry, deterministic block reductions, and the shared-memory tile
// stencils (Hessian-vector product and lower-level gradient).
//
// Reference semantics: operators.py:19-22 (true convolution, zero boundary),
// operators.py:363-383 (H v), operators.py:329-353 (cost / gradient); the
// blur / TV / phi_eps generalisation is documented in DESIGN.md.
#pragma once

#include <cuda.h>  // CUtensorMap (type only; the encoder is resolved through the runtime)
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/krecycle_b200.h"

namespace kr {

#ifdef KR_RMINRES_TIMING
__device__ unsigned long long g_stencil_ns[8];
__device__ __forceinline__ unsigned long long kr_gtime0() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define KR_SMARK(i, last)                                                     \
  do {                                                                        \
    if (threadIdx.x == 0 && blockIdx.x == 0) {                                \
      const unsigned long long t_ = kr_gtime0();                              \
      g_stencil_ns[i] += t_ - last;                                           \
      last = t_;                                                              \
    }                                                                         \
  } while (0)
#else
#define KR_SMARK(i, last) ((void)0)
#endif

// Block barrier preceded by a full-warp reconvergence: thread-0-only sections
// (scalar recurrences, partial reductions) leave warp 0 diverged, and the
// .aligned bar.sync behind __syncthreads() must be reached by converged warps.
__device__ __forceinline__ void block_barrier() {
  __syncwarp();
  __syncthreads();
}

constexpr int TH = 16;        // tile rows
constexpr int TW = 32;        // tile cols
constexpr int TPX = TH * TW;  // pixels per tile
constexpr int NT = 256;       // threads per block for tile kernels
constexpr int PPT = TPX / NT; // tile pixels per thread
constexpr int MAX_SLOTS = 400;  // >= 2 MAX_S + 1 + MAX_NSC (C^T hv, C^T v, v.hv, Z^T hv)

struct Geom {
  int rb;    // blur radius (0 if no blur)
  int rq;    // filter radius (0 if no filters)
  int H;     // halo of the input region
  int RW;    // region width  = TW + 2H
  int RH;    // region height = TH + 2H
  int s0;    // doubles in S0 (input region)
  int sa;    // doubles in SA (scratch A)
  int sb;    // doubles in SB (scratch B)
  int kw;    // doubles of kernel weights (J q^2)
  int total; // total doubles of dynamic smem used by the stencil
};

__host__ __device__ inline int imax(int a, int b) { return a > b ? a : b; }

constexpr int NWARP = NT / 32;  // warps per tile block (the filter stage runs one filter per warp)

// stride of one filter plane of the filter stage (tile_filters_q): = 2 (mod 8) doubles
__host__ __device__ inline int filt_plane_stride(int rq) {
  const int epix = (TW + 2 * rq) * (TH + 2 * rq);
  return ((epix + 7) & ~7) + 2;
}

__host__ __device__ inline Geom make_geom(const kr_op& op) {
  Geom g;
  g.rb = (op.data_kind == KR_DATA_BLUR) ? op.blur_size / 2 : 0;
  g.rq = (op.reg_kind == KR_REG_FILTERS) ? op.ksize / 2 : 0;
  g.H = imax(imax(2 * g.rb, 2 * g.rq), 1);
  // odd row stride (in doubles): the row-run passes map lanes to rows, and an odd
  // stride puts the 32 rows of a warp on distinct bank pairs
  g.RW = TW + 2 * g.H + 1;
  g.RH = TH + 2 * g.H;
  g.s0 = (g.RH * g.RW + 15) & ~15;  // SA starts 128-byte aligned: it is the TMA staging buffer
  const int w1p = TW + 2 * g.rb + 1;  // padded (odd) strides of the blur scratch
  int s1 = (op.data_kind == KR_DATA_BLUR) ? (TH + 4 * g.rb) * w1p : 0;
  int s3 = (op.data_kind == KR_DATA_BLUR) ? (TH + 2 * g.rb) * (TW + 1) : 0;
  int s4 = (op.reg_kind == KR_REG_FILTERS) ? NWARP * filt_plane_stride(g.rq) : 0;
  int s5 = (op.reg_kind == KR_REG_TV) ? 2 * (TH + 1) * (TW + 1) : 0;
  g.sa = imax(imax(s1, s3), imax(s4, s5));
  g.sb = (op.data_kind == KR_DATA_BLUR) ? (TH + 2 * g.rb) * w1p : 0;
  g.kw = (op.reg_kind == KR_REG_FILTERS) ? op.num_filters * op.ksize * op.ksize : 0;
  g.total = g.s0 + g.sa + g.sb + TPX + g.kw + KR_MAX_FILTERS + KR_MAX_BLUR + 1;
  return g;
}

__host__ __device__ inline int64_t op_n(const kr_op& op) { return (int64_t)op.rows * op.cols; }

// Compile-time filter-size variant of the stencil kernels (0 = generic runtime path).
inline int q_variant(const kr_op& op) {
  if (op.reg_kind == KR_REG_FILTERS && op.data_kind != KR_DATA_DENSE &&
      (op.ksize == 3 || op.ksize == 5 || op.ksize == 7))
    return op.ksize;
  return 0;
}

#define KR_PICK_Q(kernel, q) \
  ((q) == 3 ? (const void*)kernel<3> : (q) == 5 ? (const void*)kernel<5> : (q) == 7 ? (const void*)kernel<7> \
                                                                              : (const void*)kernel<0>)

__host__ __device__ inline int tiles_y(const kr_op& op) { return (op.rows + TH - 1) / TH; }
__host__ __device__ inline int tiles_x(const kr_op& op) { return (op.cols + TW - 1) / TW; }
__host__ __device__ inline int num_tiles(const kr_op& op) {
  if (op.data_kind == KR_DATA_DENSE) return (int)((op_n(op) + TPX - 1) / TPX);
  return tiles_y(op) * tiles_x(op);
}

// ---------------------------------------------------------------------------
// deterministic reductions

__device__ inline double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Warp sum of NV values at once by recursive halving ("transpose" reduction):
// at each level a lane keeps half of its values and adds its partner's other half,
// so NV=32 costs 16+8+4+2+1 = 31 shuffles instead of 32*5.  Afterwards value i
// (i < NV) is complete in lane  lane_of(i)  (returned through `owner`).
template <int W, int OFF, int P>
__device__ inline void msum_level(double (&a)[P], int lane) {
  if constexpr (OFF >= 1) {
    if constexpr (W >= 2) {
      constexpr int H = W / 2;
      const bool upper = (lane & OFF) != 0;
#pragma unroll
      for (int i = 0; i < H; ++i) {
        const double keep = upper ? a[i + H] : a[i];
        const double send = upper ? a[i] : a[i + H];
        a[i] = keep + __shfl_xor_sync(0xffffffffu, send, OFF);
      }
    } else {
      a[0] += __shfl_xor_sync(0xffffffffu, a[0], OFF);
    }
    msum_level<(W >= 2 ? W / 2 : 1), OFF / 2, P>(a, lane);
  }
}

template <int NV>
struct MultiSum {
  static constexpr int P = NV <= 1 ? 1 : NV <= 2 ? 2 : NV <= 4 ? 4 : NV <= 8 ? 8 : NV <= 16 ? 16 : 32;
  // value index this lane ends up holding (fully reduced over the warp)
  __device__ static inline int owner(int lane) {
    int idx = 0, w = P;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      if (w > 1) {
        if (lane & off) idx += w / 2;
        w /= 2;
      }
    }
    return idx;
  }
  __device__ static inline double reduce(const double (&v)[NV], int lane) {
    double a[P];
#pragma unroll
    for (int i = 0; i < P; ++i) a[i] = i < NV ? v[i] : 0.0;
    msum_level<P, 16, P>(a, lane);
    return a[0];
  }
};

// Sum NV per-thread values over the block; red is smem of >= NV*33 doubles.
// Result in red[0..NV) after the call (visible to all threads).
template <int NV>
__device__ inline void block_sum(double (&v)[NV], double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if constexpr (NV >= 4) {
    using M = MultiSum<NV>;
    const double s = M::reduce(v, lane);  // lane holds the warp sum of value owner(lane)
    const int idx = M::owner(lane);
    block_barrier();
    if (idx < NV && (lane & ((32 / M::P) - 1)) == 0) red[idx * 32 + warp] = s;
  } else {
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = warp_sum(v[i]);
    block_barrier();
    if (lane == 0) {
#pragma unroll
      for (int i = 0; i < NV; ++i) red[i * 32 + warp] = v[i];
    }
  }
  block_barrier();
  if (threadIdx.x < NV) {
    double acc = 0.0;
    for (int w = 0; w < nw; ++w) acc += red[threadIdx.x * 32 + w];
    red[NV * 32 + threadIdx.x] = acc;
  }
  block_barrier();
  if (threadIdx.x < NV) red[threadIdx.x] = red[NV * 32 + threadIdx.x];
  block_barrier();
}

// ---------------------------------------------------------------------------
// tile stencil: H v on one TH x TW tile of sample b.
//
//   out = data_scale A^T A v + ridge v + sum_j w_j C_j^T (kappa_j . C_j v)   (filters)
//   out = data_scale A^T A v + ridge v + w D^T M D v                         (TV)
//
// `in` describes the sample's input vector (TileIn: the solvers feed the
// unnormalised Lanczos vector and beta, so H sees exactly v = u/beta).  The result is left
// in `res` (smem, TPX doubles, row-major tile).  All threads must call.

struct Smem {
  double* S0;
  double* SA;
  double* SB;
  double* res;
  double* kw;  // kernels
  double* fw;  // filter weights
  double* taps;  // blur taps
};

__device__ inline Smem carve(const Geom& g, double* base) {
  Smem s;
  s.S0 = base;
  s.SA = s.S0 + g.s0;
  s.SB = s.SA + g.sa;
  s.res = s.SB + g.sb;
  s.kw = s.res + TPX;
  s.fw = s.kw + g.kw;
  s.taps = s.fw + KR_MAX_FILTERS;
  return s;
}

// Load the filter bank into smem (call once per block).
__device__ inline void load_weights(const kr_op& op, const Geom& g, Smem& sm) {
  for (int i = threadIdx.x; i < g.kw; i += blockDim.x) sm.kw[i] = op.kernels[i];
  int nf = (op.reg_kind == KR_REG_TV) ? 1 : (op.reg_kind == KR_REG_FILTERS ? op.num_filters : 0);
  for (int i = threadIdx.x; i < nf; i += blockDim.x) sm.fw[i] = op.fweights[i];
  for (int i = threadIdx.x; i < op.blur_size && op.data_kind == KR_DATA_BLUR; i += blockDim.x)
    sm.taps[i] = op.blur_taps[i];
  block_barrier();
}

// Input of a tile stencil: v = a / div, or v = a + coef * b when b != nullptr
// (CG's direction p = r + (rr_new/rr) p_old, formed on the fly), minus
// sum_i U_i mu_i when U != nullptr (recycled CG's deflated direction).
struct TileIn {
  const double* a;
  double div;
  const double* b;
  double coef;
  const double* U = nullptr;
  int64_t ldu = 0;
  int s = 0;
  const double* mu = nullptr;
  __device__ inline double at(int64_t p) const {
    double v = b ? a[p] + coef * b[p] : a[p] / div;
    if (U)
      for (int i = 0; i < s; ++i) v -= U[(int64_t)i * ldu + p] * mu[i];
    return v;
  }
};

// TMA-staged region load (sm_100a cp.async.bulk.tensor): the (RH x (TW + 2H)) box of the
// input vector around the tile is fetched in ONE bulk tensor copy into the scratch SA (the
// tensor map's out-of-bounds fill is zero -- exactly the zero boundary), then copied into
// S0's padded (odd-stride) layout, divided by `div` when it is not 1.  The 4-D tensor is
// (cols, rows, columns, samples) with the caller's leading / batch strides.
struct TmaSrc {
  const CUtensorMap* map;  // nullptr: scalar loads
  int col, b;              // tensor coordinates 2 and 3 of the vector
  double div;
  uint64_t* mbar;          // shared-memory mbarrier (initialised with count 1)
  uint32_t* phase;         // its current phase parity (shared)
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ inline void tma_mbar_init(uint64_t* mbar, uint32_t* phase) {
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mbar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    *phase = 0;
  }
  __syncthreads();
}

__device__ inline void tma_load_region(const TmaSrc& t, const Geom& g, int y0, int x0, double* stage, double* S0) {
  const int BW = TW + 2 * g.H;
  if (threadIdx.x == 0) {
    const uint32_t bytes = (uint32_t)(g.RH * BW * sizeof(double));
    // generic-proxy accesses of the staging buffer (the previous tile's passes) before the
    // async-proxy writes of the bulk copy
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(t.mbar)), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
        "[%6];" ::"r"(smem_u32(stage)),
        "l"(t.map), "r"(x0 - g.H), "r"(y0 - g.H), "r"(t.col), "r"(t.b), "r"(smem_u32(t.mbar))
        : "memory");
  }
  const uint32_t ph = *t.phase;
  asm volatile(
      "{\n\t.reg .pred P1;\n\tKR_TMA_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra KR_TMA_WAIT;\n\t}" ::"r"(smem_u32(t.mbar)),
      "r"(ph)
      : "memory");
  const double div = t.div;
  {
    // (row, column) of the thread's elements carried incrementally: one division per thread
    const int nt = (int)blockDim.x, dq = nt / BW, dm = nt - dq * BW;
    int yy = (int)threadIdx.x / BW, xx = (int)threadIdx.x - yy * BW;
    int o = yy * g.RW + xx;
    const int dro = dq * g.RW + dm, wrap = g.RW - BW;
    for (int i = threadIdx.x; i < g.RH * BW; i += nt) {
      const double v = stage[i];
      S0[o] = div == 1.0 ? v : v / div;
      xx += dm;
      o += dro;
      if (xx >= BW) {
        xx -= BW;
        o += wrap;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) *t.phase = ph ^ 1u;
}

__device__ inline void load_region(const kr_op& op, const Geom& g, const TileIn& in, int y0, int x0,
                                   double* S0) {
  const int rows = op.rows, cols = op.cols;
  for (int i = threadIdx.x; i < g.s0; i += blockDim.x) {
    int yy = i / g.RW, xx = i - yy * g.RW;
    int y = y0 - g.H + yy, x = x0 - g.H + xx;
    double v = 0.0;
    if (y >= 0 && y < rows && x >= 0 && x < cols) v = in.at((int64_t)y * cols + x);
    S0[i] = v;
  }
}

// Dense operator: res[l] = sum_j M[p][j] v[j] for the tile's flat rows.
__device__ inline void tile_hvp_dense(const kr_op& op, int b, const TileIn& in, int tile, double* res) {
  const int64_t n = op_n(op);
  const double* M = op.dense + (int64_t)b * op.dense_bstride;
  for (int l = threadIdx.x; l < TPX; l += blockDim.x) {
    int64_t p = (int64_t)tile * TPX + l;
    double acc = 0.0;
    if (p < n) {
      const double* row = M + p * n;
      for (int64_t j = 0; j < n; ++j) acc += row[j] * in.at(j);
    }
    res[l] = acc;
  }
  block_barrier();
}

// Run length (outputs per thread along a pass) for a pass with `lanes` independent
// lines of `len` outputs and a BS-tap kernel: minimises rounds x (FMAs + loads) per thread.
__host__ __device__ constexpr int pick_run(int lanes, int len, int BS) {
  int best = 1;
  long long best_cost = -1;
  for (int r = 1; r <= 8; ++r) {
    const long long items = (long long)lanes * ((len + r - 1) / r);
    const long long rounds = (items + NT - 1) / NT;
    const long long cost = rounds * (r * BS + r + BS - 1);
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      best = r;
    }
  }
  // a longer run within 3 % of the cheapest: more independent accumulators per thread (the
  // passes are FMA-latency bound with two) and fewer loads per FMA
  for (int r = 8; r > best; --r) {
    const long long items = (long long)lanes * ((len + r - 1) / r);
    const long long rounds = (items + NT - 1) / NT;
    const long long cost = rounds * (r * BS + r + BS - 1);
#ifndef KR_PICK_SLACK
#define KR_PICK_SLACK 3
#endif
    if (cost * 100 <= best_cost * (100 + KR_PICK_SLACK)) return r;
  }
  return best;
}

// Blur data term res += data_scale * A^T A v for a compile-time blur size BS: four
// separable passes, taps in registers, each thread a run of outputs along the pass
// (a sliding window: RUN + BS - 1 loads for RUN * BS FMAs).  Row passes map lanes to
// rows (odd smem strides keep them conflict-free), column passes map lanes to columns.
// Every output accumulates its taps in the order u = 0 .. BS-1 (the generic path's order).
// GRAD = true (the lower-level gradient, operators.py:329-353 generalised): pass 2's
// A x gets y subtracted inside the image (residual A x - y) and the data cost
// sum (A x - y)^2 of the tile's own pixels is accumulated into *dcost.
// init = true: pass 4 writes res instead of accumulating into it (no pointwise term before it).
template <int BS, bool GRAD = false>
__device__ inline void blur_normal_bs(const kr_op& op, const Geom& g, Smem& sm, int y0, int x0,
                                      const double* ydata = nullptr, double* dcost = nullptr, bool init = false) {
  constexpr int RB = BS / 2;
  constexpr int H1 = TH + 4 * RB, W1 = TW + 2 * RB, W1P = W1 + 1, H2 = TH + 2 * RB, W3P = TW + 1;
  constexpr int RX1 = pick_run(H1, W1, BS), RY2 = pick_run(W1, H2, BS), RX3 = pick_run(H2, TW, BS),
                RY4 = pick_run(TW, TH, BS);
  const int H = g.H, RW = g.RW, rows = op.rows, cols = op.cols;
  const int tid = threadIdx.x;
  double tp[BS];
#pragma unroll
  for (int u = 0; u < BS; ++u) tp[u] = sm.taps[u];
  // pass 1: S1[r][c] = sum_u tp[u] S0[r + H - 2RB][c + H - u]   (rows r < H1, cols c < W1)
  double* S1 = sm.SA;
  {
    constexpr int NC = (W1 + RX1 - 1) / RX1;
    for (int item = tid; item < H1 * NC; item += NT) {
      const int r = item % H1, c0 = (item / H1) * RX1;
      const double* src = sm.S0 + (r + H - 2 * RB) * RW + c0 + H - (BS - 1);  // window column m
      double acc[RX1];
#pragma unroll
      for (int i = 0; i < RX1; ++i) acc[i] = 0.0;
#pragma unroll
      for (int m = BS + RX1 - 2; m >= 0; --m) {  // u = i + BS - 1 - m ascending
        const double v = src[m];
#pragma unroll
        for (int i = 0; i < RX1; ++i) {
          const int u = i + BS - 1 - m;
          if (u >= 0 && u < BS) acc[i] = fma(tp[u], v, acc[i]);
        }
      }
#pragma unroll
      for (int i = 0; i < RX1; ++i)
        if (c0 + i < W1) S1[r * W1P + c0 + i] = acc[i];
    }
  }
  block_barrier();
  // pass 2: S2[r][c] = sum_u tp[u] S1[r + 2RB - u][c], zero outside the image (rows r < H2)
  double* S2 = sm.SB;
  {
    constexpr int NR = (H2 + RY2 - 1) / RY2;
    for (int item = tid; item < W1 * NR; item += NT) {
      const int c = item % W1, r0 = (item / W1) * RY2;
      const double* src = S1 + r0 * W1P + c;  // window row m = S1 row r0 + m
      double acc[RY2];
#pragma unroll
      for (int i = 0; i < RY2; ++i) acc[i] = 0.0;
#pragma unroll
      for (int m = BS + RY2 - 2; m >= 0; --m) {  // output i reads S1 row r0 + i + 2RB - u
        const double v = (r0 + m < H1) ? src[m * W1P] : 0.0;
#pragma unroll
        for (int i = 0; i < RY2; ++i) {
          const int u = i + 2 * RB - m;
          if (u >= 0 && u < BS) acc[i] = fma(tp[u], v, acc[i]);
        }
      }
      const int x = x0 - RB + c;
#pragma unroll
      for (int i = 0; i < RY2; ++i) {
        const int r = r0 + i, y = y0 - RB + r;
        if (r < H2) {
          const bool in = y >= 0 && y < rows && x >= 0 && x < cols;
          double v = in ? acc[i] : 0.0;
          if constexpr (GRAD) {
            if (in) {
              v -= ydata[(int64_t)y * cols + x];
              if (r >= RB && r < RB + TH && c >= RB && c < RB + TW) *dcost += v * v;
            }
          }
          S2[r * W1P + c] = v;
        }
      }
    }
  }
  block_barrier();
  // pass 3: S3[r][c] = sum_u tp[u] S2[r][c + u]   (rows r < H2, cols c < TW)
  double* S3 = sm.SA;
  {
    constexpr int NC = (TW + RX3 - 1) / RX3;
    for (int item = tid; item < H2 * NC; item += NT) {
      const int r = item % H2, c0 = (item / H2) * RX3;
      const double* src = S2 + r * W1P + c0;
      double acc[RX3];
#pragma unroll
      for (int i = 0; i < RX3; ++i) acc[i] = 0.0;
#pragma unroll
      for (int m = 0; m < BS + RX3 - 1; ++m) {  // u = m - i ascending
        const double v = (c0 + m < W1) ? src[m] : 0.0;
#pragma unroll
        for (int i = 0; i < RX3; ++i) {
          const int u = m - i;
          if (u >= 0 && u < BS) acc[i] = fma(tp[u], v, acc[i]);
        }
      }
#pragma unroll
      for (int i = 0; i < RX3; ++i)
        if (c0 + i < TW) S3[r * W3P + c0 + i] = acc[i];
    }
  }
  block_barrier();
  // pass 4: res[r][c] += data_scale * sum_u tp[u] S3[r + u][c]
  {
    const double ds = op.data_scale;
    constexpr int NR = (TH + RY4 - 1) / RY4;
    for (int item = tid; item < TW * NR; item += NT) {
      const int c = item % TW, r0 = (item / TW) * RY4;
      const double* src = S3 + r0 * W3P + c;
      double acc[RY4];
#pragma unroll
      for (int i = 0; i < RY4; ++i) acc[i] = 0.0;
#pragma unroll
      for (int m = 0; m < BS + RY4 - 1; ++m) {
        const double v = (r0 + m < H2) ? src[m * W3P] : 0.0;
#pragma unroll
        for (int i = 0; i < RY4; ++i) {
          const int u = m - i;
          if (u >= 0 && u < BS) acc[i] = fma(tp[u], v, acc[i]);
        }
      }
#pragma unroll
      for (int i = 0; i < RY4; ++i)
        if (r0 + i < TH) {
          double* o = sm.res + (r0 + i) * TW + c;
          *o = init ? ds * acc[i] : *o + ds * acc[i];
        }
    }
  }
  block_barrier();
}

__device__ inline void tile_blur_normal_generic(const kr_op& op, const Geom& g, Smem& sm, int y0, int x0,
                                                bool accumulate);

// Blur data term on the loaded region: res (+)= data_scale * A^T A v.
__device__ inline void tile_blur_normal(const kr_op& op, const Geom& g, Smem& sm, int y0, int x0,
                                        bool accumulate) {
  switch (op.blur_size) {
    case 9: blur_normal_bs<9>(op, g, sm, y0, x0, nullptr, nullptr, !accumulate); return;
    case 15: blur_normal_bs<15>(op, g, sm, y0, x0, nullptr, nullptr, !accumulate); return;
    case 21: blur_normal_bs<21>(op, g, sm, y0, x0, nullptr, nullptr, !accumulate); return;
    default: break;
  }
  tile_blur_normal_generic(op, g, sm, y0, x0, accumulate);
}

__device__ inline void tile_blur_normal_generic(const kr_op& op, const Geom& g, Smem& sm, int y0, int x0,
                                                bool accumulate) {
  const int rb = g.rb, bs = op.blur_size, H = g.H;
  const int rows = op.rows, cols = op.cols;
  const double* __restrict__ tp = sm.taps;
  // S1: horizontal conv, rows [y0-2rb, y0+TH+2rb), cols [x0-rb, x0+TW+rb)
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
  // S2 = A v (vertical conv), rows [y0-rb, y0+TH+rb), cols [x0-rb, x0+TW+rb); zero outside image
  const int w2 = w1, h2 = TH + 2 * rb;
  double* S2 = sm.SB;
  for (int i = threadIdx.x; i < h2 * w2; i += blockDim.x) {
    int r2 = i / w2, c2 = i - r2 * w2;
    int y = y0 - rb + r2, x = x0 - rb + c2;
    double acc = 0.0;
    if (y >= 0 && y < rows && x >= 0 && x < cols) {
      const double* src = S1 + (r2 + 2 * rb) * w1 + c2;
      for (int u = 0; u < bs; ++u) acc += tp[u] * src[-u * w1];
    }
    S2[i] = acc;
  }
  block_barrier();
  // S3: horizontal correlation, rows [y0-rb, y0+TH+rb), cols [x0, x0+TW)
  double* S3 = sm.SA;
  for (int i = threadIdx.x; i < h2 * TW; i += blockDim.x) {
    int r3 = i / TW, c3 = i - r3 * TW;
    const double* src = S2 + r3 * w2 + c3;
    double acc = 0.0;
    for (int u = 0; u < bs; ++u) acc += tp[u] * src[u];
    S3[i] = acc;
  }
  block_barrier();
  const double ds = op.data_scale;
  for (int l = threadIdx.x; l < TPX; l += blockDim.x) {
    int ty = l / TW, tx = l - ty * TW;
    const double* src = S3 + ty * TW + tx;
    double acc = 0.0;
    for (int u = 0; u < bs; ++u) acc += tp[u] * src[u * TW];
    if (accumulate) sm.res[l] += ds * acc;
    else sm.res[l] = ds * acc;
  }
  block_barrier();
}

// Learned-filter part of H v for a compile-time filter size Q, filters in groups of 8:
//   stage 1 (fp64 tensor cores, mma.sync m8n8k4 f64 = DMMA): for the group's 8 filters at
//            once, E[p][j] = kappa_j(p) . sum_tap A[p][tap] K[tap][j] on the (TH+2R) x (TW+2R)
//            extended tile -- A the im2col of the loaded region (one LDS per lane per MMA),
//            K the group's taps in registers (Q^2 - 1 taps in k-steps of 4; the last tap
//            is added by two DFMAs per lane on the accumulator fragment -- 4 pipe cycles
//            instead of the 16 of a zero-padded MMA), 8 region pixels per MMA row block; the warps share the region's 8-pixel
//            blocks; E lands in 8 smem planes (plane stride = 2 mod 8 doubles: the epilogue's
//            stores are conflict-free);
//   stage 2 (DFMA, one filter per warp): acc += (w_j k_j) corr E_j on the tile, a lane an
//            8-row x 2-column output block (taps in registers, each region row loaded once
//            per lane as Q+1 doubles in double2 loads: conflict-free quarter warps); Q = 7
//            runs its tap rows in two halves so the taps fit in registers;
// then the per-warp sums are added in warp order (fixed, deterministic) to sm.res.
// DMMA and DFMA share the fp64 pipe on sm_100 (scripts/fp64_mix.cu: 37 TF either way or
// mixed); the MMA form issues one instruction per 256 FMAs instead of 8 and one shared
// load per MMA, which is what bounded the scalar form (profiles/r2_ncu_hvp_c3*.txt).
// GRAD = true: the lower-level gradient's regulariser term sum_j w_j C_j^T phi'(C_j x)
// (stage 1 applies phi' instead of the curvature) and the cost sum_j w_j sum_p phi(C_j x)
// over the tile's own pixels into *rcost.
template <int Q>
struct FiltGeo {
  static constexpr int R = Q / 2, EW = TW + 2 * R, EH = TH + 2 * R, EPIX = EW * EH;
  static constexpr int ESP = ((EPIX + 7) & ~7) + 2;  // plane stride, = 2 (mod 8)
  static constexpr int NK = (Q * Q) / 4;             // full k-steps of 4 taps; Q^2 = 1 (mod 4) for odd Q: the
                                                     // last tap is two DFMAs per lane instead of a zero-padded MMA
  static constexpr int NMT = (EPIX + 7) / 8;         // 8-pixel row blocks of the region
};

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// stage 2 over tap rows [A0, A1): acc[i][e] += sum_{a,bb} kk[a][bb] E[(8br + i + a) EW + 2bc + e + bb]
template <int Q, int A0, int A1>
__device__ inline void filt_stage2(const double* __restrict__ E, const double* __restrict__ kj, double wj, int br,
                                   int bc, double (&acc)[8][2]) {
  using F = FiltGeo<Q>;
  constexpr int EW = F::EW, NA = A1 - A0, NW = Q + 1;
  double kk[NA][Q];
#pragma unroll
  for (int a = 0; a < NA; ++a)
#pragma unroll
    for (int bb = 0; bb < Q; ++bb) kk[a][bb] = wj * kj[(A0 + a) * Q + bb];
#pragma unroll
  for (int sr = A0; sr < 7 + A1; ++sr) {  // region row 8br + sr feeds output rows i = sr - a
    const double2* rp = reinterpret_cast<const double2*>(E + (8 * br + sr) * EW + 2 * bc);
    double w[NW];
#pragma unroll
    for (int u = 0; u < NW / 2; ++u) {
      const double2 v = rp[u];
      w[2 * u] = v.x;
      w[2 * u + 1] = v.y;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int a = sr - i;
      if (a >= A0 && a < A1) {
#pragma unroll
        for (int bb = 0; bb < Q; ++bb) {
          acc[i][0] = fma(kk[a - A0][bb], w[bb], acc[i][0]);
          acc[i][1] = fma(kk[a - A0][bb], w[bb + 1], acc[i][1]);
        }
      }
    }
  }
}

template <int Q, bool GRAD = false>
__device__ inline void tile_filters_q(const kr_op& op, const Geom& g, Smem& sm, int b, int y0, int x0,
                                      double* rcost = nullptr) {
  using F = FiltGeo<Q>;
  constexpr int R = F::R, EW = F::EW, EH_ = F::EH, EPIX = F::EPIX, ESP = F::ESP, NK = F::NK, NMT = F::NMT, QQ = Q * Q;
  static_assert(QQ % 4 == 1, "odd filter size: Q^2 - 1 taps in k-steps of 4 plus one");
  static_assert(TH == 16 && TW == 32 && NWARP == 8, "stage-2 lane blocks assume a 16 x 32 tile and 8 warps");
  const int rows = op.rows, cols = op.cols, H = g.H, RW = g.RW, J = op.num_filters;
  const int64_t n = op_n(op);
  const bool quad = op.potential == KR_POT_QUADRATIC;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int kc = lane & 3, mr = lane >> 2;  // MMA fragment column (tap / filter pair) and row (pixel)
  int aoff[NK > 0 ? NK : 1];                             // im2col offsets of this lane's taps in the region
#pragma unroll
  for (int ks = 0; ks < NK; ++ks) {
    const int tap = 4 * ks + kc;
    aoff[ks] = -((tap / Q) * RW + tap % Q);
  }
  const int alast = -((Q - 1) * RW + (Q - 1));  // the last tap (Q^2 - 1)
  const int bc = lane & 15, br = lane >> 4;  // stage-2 block: rows 8br .. 8br+7, cols 2bc, 2bc+1
  double acc[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
  for (int g0 = 0; g0 < J; g0 += 8) {
    double bw[NK > 0 ? NK : 1];  // B fragment: filter g0 + mr, taps 4 ks + kc
    {
      const int j = g0 + mr;
#pragma unroll
      for (int ks = 0; ks < NK; ++ks) {
        const int tap = 4 * ks + kc;
        bw[ks] = j < J ? sm.kw[j * QQ + tap] : 0.0;
      }
    }
    const int j0 = g0 + 2 * kc;  // this lane's accumulator filters j0, j0 + 1
    const double wl0 = j0 < J ? sm.kw[j0 * QQ + QQ - 1] : 0.0, wl1 = j0 + 1 < J ? sm.kw[(j0 + 1) * QQ + QQ - 1] : 0.0;
    const double* c0p = (quad || GRAD || j0 >= J) ? nullptr : op.curv + ((int64_t)b * J + j0) * n;
    const double* c1p = (quad || GRAD || j0 + 1 >= J) ? nullptr : op.curv + ((int64_t)b * J + j0 + 1) * n;
    double* S4 = sm.SA;
    // this lane's region pixel pe = 8 mt + mr advances by 8 NWARP = 64 pixels per iteration:
    // its row / column in the extended tile, its offset in the loaded region, its global
    // pixel index and its plane slot are carried incrementally (no division, no 64-bit
    // products in the loop)
    constexpr int STEP = 8 * NWARP, DR = STEP / EW, DC = STEP - DR * EW;
    int pe = 8 * warp + mr;
    int re = pe / EW, ce = pe - re * EW;
    int soff = (re + H) * RW + ce + H;                            // offset of the pixel in S0
    int64_t gp = (int64_t)(y0 - R + re) * cols + (x0 - R + ce);   // global pixel index
    double* e0p = S4 + (2 * kc) * ESP + pe;
    for (int mt = warp; mt < NMT; mt += NWARP) {
      const bool live = pe < EPIX;
      const int y = y0 - R + re, x = x0 - R + ce;
      const bool in = live && (unsigned)y < (unsigned)rows && (unsigned)x < (unsigned)cols;
      double cv0 = 0.0, cv1 = 0.0;
      if constexpr (!GRAD) {
        if (in) {
          cv0 = quad ? 2.0 : (c0p ? __ldg(c0p + gp) : 0.0);
          cv1 = quad ? 2.0 : (c1p ? __ldg(c1p + gp) : 0.0);
        }
      }
      // (a padded slot past the region reads the region's last pixel, like the clamp it replaces)
      const double* src = sm.S0 + (live ? soff : (EH_ - 1 + H) * RW + (EW - 1) + H);
      double d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int ks = 0; ks < NK; ++ks) dmma_8x8x4(d0, d1, src[aoff[ks]], bw[ks]);
      {
        const double al = src[alast];
        d0 = fma(al, wl0, d0);
        d1 = fma(al, wl1, d1);
      }
      if (live) {
        double e0, e1;
        if constexpr (GRAD) {
          // phi' and phi of u = (c_j * x) (the potential, operators.py:5-7 / DESIGN section 2);
          // zero outside the image like the curvature path
          e0 = e1 = 0.0;
          if (in) {
            const bool own = re >= R && re < R + TH && ce >= R && ce < R + TW;
            const double u[2] = {d0, d1};
            double e[2];
#pragma unroll
            for (int k = 0; k < 2; ++k) {
              const int j = j0 + k;
              if (quad) {
                e[k] = 2.0 * u[k];
                if (own && j < J) *rcost += sm.fw[j] * (u[k] * u[k]);
              } else {
                const double sq = sqrt(u[k] * u[k] + op.eps * op.eps);
                e[k] = u[k] / sq;
                if (own && j < J) *rcost += sm.fw[j] * sq;
              }
            }
            e0 = e[0];
            e1 = e[1];
          }
        } else {
          e0 = cv0 * d0;
          e1 = cv1 * d1;
        }
        e0p[0] = e0;
        e0p[ESP] = e1;
      }
      pe += STEP;
      e0p += STEP;
      ce += DC;
      re += DR;
      soff += DR * RW + DC;
      gp += (int64_t)DR * cols + DC;
      if (ce >= EW) {
        ce -= EW;
        re += 1;
        soff += RW - EW;
        gp += cols - EW;
      }
    }
    block_barrier();
    const int j = g0 + warp;
    if (j < J) {
      const double* E = S4 + warp * ESP;
      const double* kj = sm.kw + j * QQ;
      const double wj = sm.fw[j];
      if constexpr (Q <= 5) {
        filt_stage2<Q, 0, Q>(E, kj, wj, br, bc, acc);
      } else {
        filt_stage2<Q, 0, Q / 2 + 1>(E, kj, wj, br, bc, acc);
        filt_stage2<Q, Q / 2 + 1, Q>(E, kj, wj, br, bc, acc);
      }
    }
    block_barrier();  // the planes are free again (next group / the per-warp sums)
  }
  double* P = sm.SA;
#pragma unroll
  for (int i = 0; i < 8; ++i)
    *reinterpret_cast<double2*>(P + warp * TPX + (8 * br + i) * TW + 2 * bc) = make_double2(acc[i][0], acc[i][1]);
  block_barrier();
  for (int l = threadIdx.x; l < TPX; l += NT) {
    double a = 0.0;
#pragma unroll
    for (int w = 0; w < NWARP; ++w) a += P[w * TPX + l];
    sm.res[l] += a;
  }
  block_barrier();
}

template <int Q>
__device__ inline void tile_hvp_t(const kr_op& op, const Geom& g, Smem& sm, int b, const TileIn& in, int tile,
                                  const TmaSrc* tma = nullptr);

__device__ inline void tile_hvp(const kr_op& op, const Geom& g, Smem& sm, int b, const TileIn& in, int tile) {
  tile_hvp_t<0>(op, g, sm, b, in, tile);
}

template <int Q>
__device__ inline void tile_hvp_t(const kr_op& op, const Geom& g, Smem& sm, int b, const TileIn& in, int tile,
                                  const TmaSrc* tma) {
  if (op.data_kind == KR_DATA_DENSE) {
    tile_hvp_dense(op, b, in, tile, sm.res);
    return;
  }
  const int tyc = tiles_x(op);
  const int y0 = (tile / tyc) * TH, x0 = (tile % tyc) * TW;
  const int rows = op.rows, cols = op.cols, H = g.H;
  const int64_t n = op_n(op);
#ifdef KR_RMINRES_TIMING
  unsigned long long slast = kr_gtime0();
#endif
  if (tma && tma->map) {
    tma_load_region(*tma, g, y0, x0, sm.SA, sm.S0);
  } else {
    load_region(op, g, in, y0, x0, sm.S0);
    block_barrier();
  }
  KR_SMARK(0, slast);

  // pointwise part: mask data term + ridge (a blur data term without ridge has none: the
  // blur's last pass then writes res instead of accumulating -- 0 + x = x, bitwise the same)
  const bool pointwise = !(op.data_kind == KR_DATA_BLUR && op.ridge == 0.0);
  if (pointwise) {
    const double* mask = (op.data_kind == KR_DATA_MASK) ? op.mask + (int64_t)b * op.mask_bstride : nullptr;
    for (int l = threadIdx.x; l < TPX; l += blockDim.x) {
      int ty = l / TW, tx = l - ty * TW;
      int y = y0 + ty, x = x0 + tx;
      double v = sm.S0[(ty + H) * g.RW + tx + H];
      double acc = 0.0;
      if (y < rows && x < cols) {
        if (mask) acc = (op.data_scale == 1.0 ? mask[(int64_t)y * cols + x] : op.data_scale * mask[(int64_t)y * cols + x]) * v;
        acc += op.ridge * v;
      }
      sm.res[l] = acc;
    }
    block_barrier();
  }
  KR_SMARK(1, slast);
  if (op.data_kind == KR_DATA_BLUR) tile_blur_normal(op, g, sm, y0, x0, pointwise);
  KR_SMARK(2, slast);

  if (Q > 0 && op.reg_kind == KR_REG_FILTERS) {
    tile_filters_q<(Q > 0 ? Q : 1)>(op, g, sm, b, y0, x0);
    KR_SMARK(3, slast);
  } else if (op.reg_kind == KR_REG_FILTERS) {
    const int q = op.ksize, rq = g.rq;
    const int w4 = TW + 2 * rq, h4 = TH + 2 * rq;
    double* S4 = sm.SA;
    const bool quad = (op.potential == KR_POT_QUADRATIC);
    for (int j = 0; j < op.num_filters; ++j) {
      const double* kj = sm.kw + j * q * q;
      const double* cj = quad ? nullptr : op.curv + ((int64_t)b * op.num_filters + j) * n;
      for (int i = threadIdx.x; i < h4 * w4; i += blockDim.x) {
        int r4 = i / w4, c4 = i - r4 * w4;
        int y = y0 - rq + r4, x = x0 - rq + c4;
        double e = 0.0;
        if (y >= 0 && y < rows && x >= 0 && x < cols) {
          const double* src = sm.S0 + (r4 + H) * g.RW + c4 + H;
          double acc = 0.0;
          for (int a = 0; a < q; ++a)
            for (int bb = 0; bb < q; ++bb) acc += kj[a * q + bb] * src[-a * g.RW - bb];
          e = quad ? 2.0 * acc : cj[(int64_t)y * cols + x] * acc;
        }
        S4[i] = e;
      }
      block_barrier();
      const double wj = sm.fw[j];
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
    // p = M D v on rows [y0-1, y0+TH), cols [x0-1, x0+TW); masked where D's row is zero
    const int w5 = TW + 1, h5 = TH + 1;
    double* PH = sm.SA;
    double* PV = sm.SA + h5 * w5;
    const double* M = op.curv + (int64_t)b * 3 * n;
    for (int i = threadIdx.x; i < h5 * w5; i += blockDim.x) {
      int r5 = i / w5, c5 = i - r5 * w5;
      int y = y0 - 1 + r5, x = x0 - 1 + c5;
      double ph = 0.0, pv = 0.0;
      if (y >= 0 && y < rows && x >= 0 && x < cols) {
        const double* c = sm.S0 + (y - y0 + H) * g.RW + (x - x0 + H);
        double dh = (x < cols - 1) ? c[1] - c[0] : 0.0;
        double dv = (y < rows - 1) ? c[g.RW] - c[0] : 0.0;
        int64_t p = (int64_t)y * cols + x;
        double m11 = M[p], m12 = M[n + p], m22 = M[2 * n + p];
        if (x < cols - 1) ph = m11 * dh + m12 * dv;
        if (y < rows - 1) pv = m12 * dh + m22 * dv;
      }
      PH[i] = ph;
      PV[i] = pv;
    }
    block_barrier();
    const double wa = sm.fw[0];
    for (int l = threadIdx.x; l < TPX; l += blockDim.x) {
      int ty = l / TW, tx = l - ty * TW;
      int i = (ty + 1) * w5 + tx + 1;
      // D_h^T p_h = -p_h[x] + p_h[x-1];  D_v^T p_v = -p_v[y] + p_v[y-1]
      double dth = -PH[i] + PH[i - 1];
      double dtv = -PV[i] + PV[i - w5];
      sm.res[l] += wa * (dth + dtv);
    }
    block_barrier();
  }
}

// Global pixel index of tile-local pixel l, or -1 if outside the image.
__device__ inline int64_t tile_pixel(const kr_op& op, int tile, int l) {
  if (op.data_kind == KR_DATA_DENSE) {
    int64_t p = (int64_t)tile * TPX + l;
    return p < op_n(op) ? p : -1;
  }
  const int tyc = tiles_x(op);
  int y = (tile / tyc) * TH + l / TW, x = (tile % tyc) * TW + l % TW;
  if (y >= op.rows || x >= op.cols) return -1;
  return (int64_t)y * op.cols + x;
}

}  // namespace kr
