// kr_rminres.cu -- batched recycled MINRES as ONE persistent cooperative kernel.
//
// Algorithm: /root/reference/pkg/src/krecycle/krylov.py:205-383 (Alg. 3 with the
// corrected sign w += c_k zeta_{k-1}(vt - bt)), stop rules stopping.py:69-118,
// residual recurrence krylov.py:154-181.  B200 structure:
//
//  * one launch runs every iteration of every sample; blocks are partitioned
//    by sample (Gs blocks per sample), grid-wide barriers separate the three
//    reduction phases of an iteration:
//      P1  finish iteration k-1 (Givens, vt / w / residual updates, stop test),
//          v_k = u_{k-1}/beta_k, tile stencil hv_k = H v_k, partial C^T hv_k
//      P2  NSC decision, u = hv_k - C chv_k, partial alpha = v_k . u
//      P3  u -= alpha v_k; u -= beta v_{k-1}, partial ||u||^2
//  * the recycle-space terms b = U chv and H b~ = C chv are carried in s-space
//    (b~_k = U btc_k, btc_k = (chv_k - gamma btc_{k-2} - delta btc_{k-1})/eps~);
//    the solution is w = w_v - U Omega and the residual r = r_v + C Omega with
//    Omega = sum_k step_k btc_k, so U is read once per solve instead of once
//    per iteration (exact in exact arithmetic);
//  * NSC reads Z = W V_H,sel diag(mu_sel) (one n x s block) instead of W (n x t):
//    Z^T r = Z^T r_v + (Z^T C) Omega;
//  * every reduction is a fixed-order two-level sum (warp tree, block, then the
//    sample's blocks in rank order), so results are bitwise reproducible.

#include <string>

#include "kr_common.cuh"
#include "kr_internal.h"
#include "kr_solver.cuh"


namespace kr {

struct SolverWork {
  double* tmp;     // unnormalised next Lanczos vector u (global: read with halo)
  double* u;       // hv - C chv
  double* hv[2];   // H v_k (double-buffered by k parity)
  double* vt[2];   // v~ recurrence
  double* hvt[2];  // H v~ recurrence
  double* rv;      // residual without the C Omega term
  double* wv;      // solution without the -U Omega term
  double* vr[2];   // Lanczos vectors when the basis is not tracked
  double* part;    // [B][NSLOT][Gs] block partials
  int* done;       // finished-sample counter
};

struct Params {
  kr_op op;
  kr_solve_args a;
  SolverWork w;
  int Gs;       // blocks per sample
  int b0;       // first sample of this launch
  int nb;       // samples in this launch
  int nslot;
  int64_t n;
  __device__ inline Partials parts() const { return Partials{w.part, nslot, Gs}; }
};

struct Scalars {
  double beta, beta_prev, alpha, alpha_prev;
  double c1, s1, c2, s2, zeta;
  double gamma, delta, eps_r, step;
  double tol_bd, delta_stop;
  int active, finished, counted, pending, pend_k, pend_broke, do_update, do_hvp, iters, reason;
};

__device__ inline double* vec(double* base, int64_t n, int b) { return base + (int64_t)b * n; }

// Lanczos vector v_k (k >= 1)
__device__ inline double* lanczos(const Params& P, int b, int k, int site = 0) {
#ifdef KR_GUARD
  assert(site != 1 || k >= 1);
  assert(site != 1 || k <= P.a.max_iter);
  assert(site != 2 || k <= P.a.max_iter);
  assert(site != 3 || k <= P.a.max_iter);
  assert(site != 4 || k >= 1);
  assert(b >= 0 && b < P.op.batch);
#endif
  if (P.a.basis) return P.a.basis + (int64_t)b * P.a.bs_basis + (int64_t)(k - 1) * P.a.ld_basis;
  return vec(P.w.vr[k & 1], P.n, b);
}

// All cross-block traffic is within a sample (its Gs blocks share partials), so the
// "grid" barrier is a per-sample barrier: one counter per sample, Gs arrivals.
#ifdef KR_RMINRES_TIMING
__device__ __forceinline__ unsigned long long kr_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define KR_TMARK(i)                                   \
  do {                                                \
    if (threadIdx.x == 0) {                           \
      const unsigned long long t_ = kr_gtime();       \
      tsec[i] += t_ - tlast;                          \
      tlast = t_;                                     \
    }                                                 \
  } while (0)
#else
#define KR_TMARK(i) ((void)0)
#endif

#define KR_GRID_SYNC() grid_barrier(reinterpret_cast<unsigned int*>(P.w.done) + 1 + bl, P.Gs, grid_target)

template <int Q>
__global__ void __launch_bounds__(NT, 2) rminres_kernel(Params P) {
  unsigned int grid_target = 0;
#ifdef KR_RMINRES_TIMING
  unsigned long long tsec[12] = {0}, tlast = kr_gtime();
  int tk = 0;
#endif
  extern __shared__ double smem[];
  const kr_op& op = P.op;
  const kr_solve_args& A = P.a;
  const Geom g = make_geom(op);
  Smem sm = carve(g, smem);
  double* tail = smem + g.total;
  double* slot_acc = tail;               // MAX_SLOTS
  double* chv = slot_acc + MAX_SLOTS;    // MAX_S (also the initial projection t)
  double* btc1 = chv + 2 * MAX_S;  // chv holds C^T hv [0,s) and C^T v [s,2s)
  double* btc2 = btc1 + MAX_S;
  double* omega = btc2 + MAX_S;
  // NSC in s-space: zrv = Z^T r_v, zhA / zhB = Z^T hvt_{k-1} / Z^T hvt_{k-2} (the
  // residual recurrence krylov.py:169-181 applied to Z^T r), zhv = Z^T hv_k
  double* nscv = omega + MAX_S;          // MAX_NSC (squared terms of the NSC value)
  double* zrv = nscv + MAX_NSC;          // MAX_NSC
  double* zhA = zrv + MAX_NSC;           // MAX_NSC
  double* zhB = zhA + MAX_NSC;           // MAX_NSC
  double* zhv = zhB + MAX_NSC;           // MAX_NSC
  double* red = zhv + MAX_NSC;           // RED_DOUBLES
#ifdef KR_VOLATILE_SC
  __shared__ volatile Scalars sc;
#else
  __shared__ Scalars sc;
#endif
  __shared__ double red1[4];  // single-slot reductions

  const int bl = blockIdx.x / P.Gs;      // local sample index
  const int j = blockIdx.x % P.Gs;       // rank within the sample
  const int b = P.b0 + bl;               // global sample index
  const int64_t n = P.n;
  const int s = A.s, ns = (A.stop_kind == 1) ? A.nsc_s : 0;
  // slots: [C^T hv (s) | C^T v (s) | v.hv | Z^T hv (ns)] contiguous (one reduction in P2),
  // then Z^T r0 (setup) and ||u||^2
  const int SL_CHV = 0, SL_ALPHA = 2 * s, SL_ZHV = 2 * s + 1, SL_NSC = 2 * s + 1 + ns, SL_BETA2 = 2 * s + 1 + 2 * ns;
  const int64_t lo = n * j / P.Gs, hi = n * (j + 1) / P.Gs;
  const int ntiles = num_tiles(op);
  const bool leader = (j == 0);
  const bool track = A.track_residual != 0;
  const Partials PP = P.parts();
  KR_ASSERT(b < op.batch && bl < P.nb && s <= MAX_S && 2 * s + 1 + ns <= MAX_SLOTS && ns <= MAX_NSC && hi <= n);

  const double* U = A.U ? A.U + (int64_t)b * A.bs_uc : nullptr;
  const double* C = A.C ? A.C + (int64_t)b * A.bs_uc : nullptr;
  const double* Z = (ns > 0) ? A.Z + (int64_t)b * A.bs_z : nullptr;
  const double* ZtC = (ns > 0 && s > 0) ? A.ZtC + (int64_t)b * ns * s : nullptr;
  const double* gb = A.g + (int64_t)b * n;
  const double* w0 = A.w0 ? A.w0 + (int64_t)b * n : nullptr;
  double* tmp = vec(P.w.tmp, n, b);
  double* ub = vec(P.w.u, n, b);
  double* rv = vec(P.w.rv, n, b);
  double* wv = vec(P.w.wv, n, b);
  double* res_norms = A.res_norms + (int64_t)b * (A.max_iter + 1);
  double* stop_vals = A.stop_vals + (int64_t)b * (A.max_iter + 1);

  load_weights(op, g, sm);
  for (int i = threadIdx.x; i < MAX_SLOTS; i += blockDim.x) slot_acc[i] = 0.0;
  for (int i = threadIdx.x; i < MAX_S; i += blockDim.x) {
    chv[i] = 0.0;
    btc1[i] = 0.0;
    btc2[i] = 0.0;
    omega[i] = 0.0;
  }
  for (int i = threadIdx.x; i < MAX_NSC; i += blockDim.x) {
    zrv[i] = 0.0;
    zhA[i] = 0.0;
    zhB[i] = 0.0;
    zhv[i] = 0.0;
  }
  if (threadIdx.x == 0) {
    sc.active = 1;
    sc.finished = 0;
    sc.counted = 0;
    sc.pending = 0;
    sc.iters = 0;
    sc.reason = R_MAXIT;
    sc.c1 = 1.0;
    sc.s1 = 0.0;
    sc.c2 = 0.0;
    sc.s2 = 0.0;
    sc.beta_prev = 0.0;
    sc.alpha_prev = 0.0;
    sc.delta_stop = A.delta;
  }
  block_barrier();

  // ---------------- setup S1: r0 = g - H w0, partial C^T r0 ----------------
  if (w0) {
    for (int tile = j; tile < ntiles; tile += P.Gs) {
      tile_hvp_t<Q>(op, g, sm, b, TileIn{w0, 1.0, nullptr, 0.0}, tile);
      for (int l = threadIdx.x; l < TPX; l += blockDim.x) {
        int64_t p = tile_pixel(op, tile, l);
        double r = 0.0;
        if (p >= 0) {
          r = gb[p] - sm.res[l];
          tmp[p] = r;
        }
        sm.res[l] = r;
      }
      block_barrier();
    }
  } else {
    for (int64_t p = lo + threadIdx.x; p < hi; p += blockDim.x) tmp[p] = gb[p];  // g - H 0 == g exactly
  }
  // zero the recurrence state
  for (int64_t p = lo + threadIdx.x; p < hi; p += blockDim.x) {
    vec(P.w.vt[0], n, b)[p] = 0.0;
    vec(P.w.vt[1], n, b)[p] = 0.0;
    if (track) {
      vec(P.w.hvt[0], n, b)[p] = 0.0;
      vec(P.w.hvt[1], n, b)[p] = 0.0;
    }
  }
  KR_GRID_SYNC();  // tmp complete (written by tiles when w0 given)
  if (s > 0) {
    slot_dots(C, A.ld_uc, s, lo, hi, [&](int64_t p) { return tmp[p]; }, slot_acc, red);
    write_partials(PP, bl, j, SL_CHV, s, slot_acc);
  }
  KR_GRID_SYNC();
  // ---------------- setup S2: projection onto the recycle space ----------------
  if (s > 0) {
    reduce_slots(PP, bl, SL_CHV, s, chv);  // t = C^T r0
    block_barrier();
  }
  {
    double bsq[1] = {0.0};
    for (int64_t p = lo + threadIdx.x; p < hi; p += blockDim.x) {
      double r = tmp[p];
      double w = w0 ? w0[p] : 0.0;
      if (s > 0) {
        double ut = 0.0, ct = 0.0;
        for (int i = 0; i < s; ++i) {
          ut += U[(int64_t)i * A.ld_uc + p] * chv[i];
          ct += C[(int64_t)i * A.ld_uc + p] * chv[i];
        }
        w = w + ut;  // w = w + U t
        r = r - ct;  // r = r - C t
        tmp[p] = r;
      }
      wv[p] = w;
      if (track) rv[p] = r;
      bsq[0] += r * r;
    }
    block_sum<1>(bsq, red);
    if (threadIdx.x == 0) P.w.part[((int64_t)bl * P.nslot + SL_BETA2) * P.Gs + j] = red[0];
    if (ns > 0) {
      for (int i = threadIdx.x; i < ns; i += blockDim.x) slot_acc[i] = 0.0;
      block_barrier();
      slot_dots(Z, A.ld_z, ns, lo, hi, [&](int64_t p) { return tmp[p]; }, slot_acc, red);
      write_partials(PP, bl, j, SL_NSC, ns, slot_acc);
    }
  }
  // g-scale for the breakdown tolerance (krylov.py:236-237): ||g||
  {
    double gsq[1] = {0.0};
    for (int64_t p = lo + threadIdx.x; p < hi; p += blockDim.x) gsq[0] += gb[p] * gb[p];
    block_sum<1>(gsq, red);
    if (threadIdx.x == 0) P.w.part[((int64_t)bl * P.nslot + SL_ALPHA) * P.Gs + j] = red[0];
  }
  KR_GRID_SYNC();
  reduce_slots(PP, bl, SL_ALPHA, 1, red1);
  if (ns > 0) reduce_slots(PP, bl, SL_NSC, ns, zrv);  // Z^T r0_v
  block_barrier();
  if (threadIdx.x == 0) {
    double gg = red1[0];
    double gn = sqrt(gg);
    sc.tol_bd = BREAKDOWN_RTOL * (gn > 1e-300 ? gn : 1e-300);
  }
  block_barrier();

  // ---------------- main loop ----------------
  KR_TMARK(0);
  for (int k = 1; k <= A.max_iter + 1; ++k) {
    // this sample is finished and reported: its blocks leave (sc is block-shared and
    // identical across the sample's blocks, so all of them leave at the same k)
    if (sc.counted) break;
#ifdef KR_GUARD
    {
      __shared__ int guard_k[NT];
      guard_k[threadIdx.x] = k;
      block_barrier();
      assert(guard_k[0] == k);                                  // warp 0 at the same iteration
      assert(guard_k[(threadIdx.x + 32) % blockDim.x] == k);    // neighbouring warp too
      block_barrier();
    }
#endif
    // ===== P1 =====
#ifdef KR_RMINRES_TIMING
    tk = k;
#endif
    if (sc.active) {
      reduce_slots(PP, bl, SL_BETA2, 1, red1);
      block_barrier();
    }
    KR_TMARK(1);
    if (threadIdx.x == 0) {
      sc.do_update = 0;
      sc.do_hvp = 0;
      if (sc.active) {
        double bb = red1[0];
        double beta_k = sqrt(bb);
        bool broke = beta_k <= sc.tol_bd;
        if (k == 1) {
          sc.beta = beta_k;
          sc.zeta = beta_k;
          if (leader) res_norms[0] = beta_k;
          if (A.stop_kind == 0) {
            if (leader) stop_vals[0] = beta_k;
            if (beta_k < sc.delta_stop) {
              sc.active = 0; sc.finished = 1; sc.iters = 0; sc.reason = R_TOL;
            } else if (broke) {
              sc.active = 0; sc.finished = 1; sc.iters = 0; sc.reason = R_BREAK;
            }
          } else {
            sc.pending = 1; sc.pend_k = 0; sc.pend_broke = broke;
          }
        } else {
          // finish iteration k-1 (krylov.py:298-338)
          const double bp = sc.beta;  // beta_{k-1}
          const double al = sc.alpha;
          double gamma = sc.s2 * bp;
          double delta = sc.c1 * sc.c2 * bp + sc.s1 * al;
          double eps = -sc.s1 * sc.c2 * bp + sc.c1 * al;
          double eps_r = hypot(eps, beta_k);
          if (eps_r == 0.0) {
            sc.active = 0; sc.finished = 1; sc.iters = k - 2; sc.reason = R_BREAK;
          } else {
            double s_new = beta_k / eps_r, c_new = eps / eps_r;
            double zeta_prev = sc.zeta;
            sc.zeta = -s_new * zeta_prev;
            sc.gamma = gamma; sc.delta = delta; sc.eps_r = eps_r;
            sc.step = c_new * zeta_prev;
            sc.do_update = 1;
            sc.c2 = sc.c1; sc.s2 = sc.s1; sc.c1 = c_new; sc.s1 = s_new;
            sc.beta_prev = bp;
            sc.beta = beta_k;
            double rn = fabs(sc.zeta);
            if (leader) res_norms[k - 1] = rn;
            if (A.stop_kind == 0) {
              if (leader) stop_vals[k - 1] = rn;
              if (rn < sc.delta_stop) {
                sc.active = 0; sc.finished = 1; sc.iters = k - 1; sc.reason = R_TOL;
              } else if (broke) {
                sc.active = 0; sc.finished = 1; sc.iters = k - 1; sc.reason = R_BREAK;
              } else if (k - 1 == A.max_iter) {
                sc.active = 0; sc.finished = 1; sc.iters = k - 1; sc.reason = R_MAXIT;
              }
            } else {
              sc.pending = 1; sc.pend_k = k - 1; sc.pend_broke = broke;
            }
          }
        }
        if (sc.active && !(sc.pending && sc.pend_broke) && k <= A.max_iter) sc.do_hvp = 1;
      }
    }
    block_barrier();
    if (sc.do_update) {
      // s-space recurrences (thread per recycle column)
      for (int i = threadIdx.x; i < s; i += blockDim.x) {
        double bt = (chv[i] - sc.gamma * btc2[i] - sc.delta * btc1[i]) / sc.eps_r;
        omega[i] += sc.step * bt;
        btc2[i] = btc1[i];
        btc1[i] = bt;
      }
      // Z^T of the tracked-residual recurrence: hvt_{k-1} = (hv_{k-1} - delta hvt_{k-2}
      // - gamma hvt_{k-3}) / eps~, r_v -= step hvt_{k-1}
      for (int i = threadIdx.x; i < ns; i += blockDim.x) {
        const double zn = (zhv[i] - sc.delta * zhA[i] - sc.gamma * zhB[i]) / sc.eps_r;
        zrv[i] -= sc.step * zn;
        zhB[i] = zhA[i];
        zhA[i] = zn;
      }
      // pointwise updates of iteration k-1
      const int km = k - 1;
      const double* v = lanczos(P, b, km, 1);
      double* vtn = vec(P.w.vt[km & 1], n, b);        // holds vt_{k-3} -> becomes vt_{k-1}
      const double* vto = vec(P.w.vt[(km + 1) & 1], n, b);  // vt_{k-2}
      const double* hvk = vec(P.w.hv[km & 1], n, b);
      double* hvtn = vec(P.w.hvt[km & 1], n, b);
      const double* hvto = vec(P.w.hvt[(km + 1) & 1], n, b);
      const double ga = sc.gamma, de = sc.delta, er = sc.eps_r, st = sc.step;
      // two pixels per thread per round, every load issued before the first store
      for (int64_t p0 = lo + threadIdx.x; p0 < hi; p0 += 2 * NT) {
        const int64_t p1 = p0 + NT;
        const bool h1 = p1 < hi;
        const int64_t q1 = h1 ? p1 : p0;
        const double v0 = v[p0], v1 = v[q1], a0 = vtn[p0], a1 = vtn[q1], o0 = vto[p0], o1 = vto[q1];
        const double w0 = wv[p0], w1 = wv[q1];
        double x0 = 0.0, x1 = 0.0, ho0 = 0.0, ho1 = 0.0, hn0 = 0.0, hn1 = 0.0, r0 = 0.0, r1 = 0.0;
        if (track) {
          x0 = hvk[p0]; x1 = hvk[q1]; ho0 = hvto[p0]; ho1 = hvto[q1]; hn0 = hvtn[p0]; hn1 = hvtn[q1];
          r0 = rv[p0]; r1 = rv[q1];
        }
        const double vt0 = (v0 - ga * a0 - de * o0) / er, vt1 = (v1 - ga * a1 - de * o1) / er;
        vtn[p0] = vt0;
        wv[p0] = w0 + st * vt0;
        if (h1) {
          vtn[p1] = vt1;
          wv[p1] = w1 + st * vt1;
        }
        if (track) {
          const double ht0 = (x0 - de * ho0 - ga * hn0) / er, ht1 = (x1 - de * ho1 - ga * hn1) / er;
          hvtn[p0] = ht0;
          rv[p0] = r0 - st * ht0;
          if (h1) {
            hvtn[p1] = ht1;
            rv[p1] = r1 - st * ht1;
          }
        }
      }
    }
    block_barrier();
    KR_TMARK(2);
    if (sc.pending) {
      // NSC of iteration pend_k (stopping.py:69-72): (Z^T r)_i = zrv_i + (Z^T C Omega)_i,
      // decided here, before the next H v (no pass over Z, no extra grid barrier)
      for (int i = threadIdx.x; i < ns; i += blockDim.x) {
        double z = zrv[i];
        if (ZtC) {
          double c0 = 0.0, c1 = 0.0;
          int l = 0;
          for (; l + 1 < s; l += 2) {
            c0 += ZtC[(int64_t)i * s + l] * omega[l];
            c1 += ZtC[(int64_t)i * s + l + 1] * omega[l + 1];
          }
          if (l < s) c0 += ZtC[(int64_t)i * s + l] * omega[l];
          z += c0 + c1;
        }
        nscv[i] = z * z;
      }
      block_barrier();
      if (threadIdx.x == 0) {
        double ss = 0.0;
        for (int i = 0; i < ns; ++i) ss += nscv[i];
        double val = sqrt(ss);
        const int kk = sc.pend_k;
        if (leader) stop_vals[kk] = val;
        sc.pending = 0;
        if (val < sc.delta_stop) {
          sc.active = 0; sc.finished = 1; sc.iters = kk; sc.reason = R_TOL;
        } else if (sc.pend_broke) {
          sc.active = 0; sc.finished = 1; sc.iters = kk; sc.reason = R_BREAK;
        } else if (kk == A.max_iter) {
          sc.active = 0; sc.finished = 1; sc.iters = kk; sc.reason = R_MAXIT;
        }
        sc.do_hvp = sc.do_hvp && sc.active;
      }
      block_barrier();
    }
    KR_TMARK(3);
    if (sc.finished && !sc.counted) {
      // finalize: w = w_v - U Omega, r = r_v + C Omega (krylov.py:184-202 outputs)
      double* wout = A.w + (int64_t)b * n;
      double* rout = (track && A.r) ? A.r + (int64_t)b * n : nullptr;
      for (int64_t p = lo + threadIdx.x; p < hi; p += blockDim.x) {
        double uo = 0.0, co = 0.0;
        for (int i = 0; i < s; ++i) {
          uo += U[(int64_t)i * A.ld_uc + p] * omega[i];
          co += C[(int64_t)i * A.ld_uc + p] * omega[i];
        }
        wout[p] = wv[p] - uo;
        if (rout) rout[p] = rv[p] + co;
      }
    }
    if (sc.do_hvp) {
      const double beta_k = sc.beta;
      double* vk = lanczos(P, b, k, 2);  // written from the stencil's region (v = u / beta)
      for (int i = threadIdx.x; i < 2 * s + 1 + ns; i += blockDim.x) slot_acc[i] = 0.0;
      block_barrier();
      double* hvk = vec(P.w.hv[k & 1], n, b);
      const int sm8 = s > ns ? s : ns;
      const int npass = sm8 > 0 ? (sm8 + 7) / 8 : 1;
      const bool deferred = npass <= DEF_PASSES;
      if (deferred) {  // warp sums accumulate in red over passes and tiles
        for (int i = threadIdx.x; i < npass * 25 * DEF_STRIDE; i += blockDim.x) red[i] = 0.0;
        block_barrier();
      }
      for (int tile = j; tile < ntiles; tile += P.Gs) {
        KR_TMARK(4);
        tile_hvp_t<Q>(op, g, sm, b, TileIn{tmp, beta_k, nullptr, 0.0}, tile);
        KR_TMARK(5);
        for (int l = threadIdx.x; l < TPX; l += blockDim.x) {
          int64_t p = tile_pixel(op, tile, l);
          if (p >= 0) {
            hvk[p] = sm.res[l];
            if (op.data_kind == KR_DATA_DENSE) {
              vk[p] = tmp[p] / beta_k;
            } else {
              const int ty = l / TW, tx = l - ty * TW;
              vk[p] = sm.S0[(ty + g.H) * g.RW + tx + g.H];
            }
          }
        }
        // partials over this tile: C^T hv, C^T v, Z^T hv (NSC) and v . hv
        // (alpha = v.hv - (C^T v).(C^T hv)), 8 columns per pass; with <= DEF_PASSES passes
        // the warp sums stay in registers (accumulated over the block's tiles) and are
        // combined once after the tile loop
        for (int base = 0; base < sm8 || base == 0; base += 8) {
          double v25[25];
#pragma unroll
          for (int i = 0; i < 25; ++i) v25[i] = 0.0;
          static_assert(TPX == 2 * NT, "two tile pixels per thread");
          {
            // both of the thread's pixels: all 2 x 16 column loads in flight at once
            int64_t pp[2];
            double hh[2], vv[2], cc[2][8], zz[2][8];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int l = threadIdx.x + u * NT;
              pp[u] = tile_pixel(op, tile, l);
              const int64_t q = pp[u] >= 0 ? pp[u] : 0;
              hh[u] = sm.res[l];
              if (op.data_kind == KR_DATA_DENSE) {
                vv[u] = pp[u] >= 0 ? tmp[q] / beta_k : 0.0;
              } else {
                const int ty = l / TW, tx = l - ty * TW;
                vv[u] = sm.S0[(ty + g.H) * g.RW + tx + g.H];
              }
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                cc[u][i] = (pp[u] >= 0 && base + i < s) ? C[(int64_t)(base + i) * A.ld_uc + q] : 0.0;
                zz[u][i] = (pp[u] >= 0 && base + i < ns) ? Z[(int64_t)(base + i) * A.ld_z + q] : 0.0;
              }
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              if (pp[u] < 0) continue;
              const double h = hh[u], v = vv[u];
              if (base == 0) v25[24] += v * h;
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                if (base + i < s) {
                  v25[i] += cc[u][i] * h;
                  v25[8 + i] += cc[u][i] * v;
                }
                if (base + i < ns) v25[16 + i] += zz[u][i] * h;
              }
            }
          }
          if (deferred) {
            def_add<25>(MultiSum<25>::reduce(v25, threadIdx.x & 31), base / 8, red);
            continue;
          }
          block_sum<25>(v25, red);
          if (threadIdx.x < 8 && base + threadIdx.x < s) {
            slot_acc[base + threadIdx.x] += red[threadIdx.x];
            slot_acc[s + base + threadIdx.x] += red[8 + threadIdx.x];
          }
          if (threadIdx.x < 8 && base + threadIdx.x < ns) slot_acc[2 * s + 1 + base + threadIdx.x] += red[16 + threadIdx.x];
          if (threadIdx.x == 0 && base == 0) slot_acc[2 * s] += red[24];
          block_barrier();
        }
        block_barrier();
      }
      if (deferred) {
        // value (pass q, i): i < 8 -> C^T hv column 8q+i, 8..15 -> C^T v column 8q+i-8,
        // 16..23 -> Z^T hv column 8q+i-16, 24 (q = 0) -> v.hv
        for (int c = threadIdx.x; c < s; c += blockDim.x) {
          slot_acc[c] = def_sum(red, (c / 8) * 25 + c % 8);
          slot_acc[s + c] = def_sum(red, (c / 8) * 25 + 8 + c % 8);
        }
        for (int c = threadIdx.x; c < ns; c += blockDim.x) slot_acc[2 * s + 1 + c] = def_sum(red, (c / 8) * 25 + 16 + c % 8);
        if (threadIdx.x == 0) slot_acc[2 * s] = def_sum(red, 24);
        block_barrier();
      }
      write_partials(PP, bl, j, SL_CHV, 2 * s + 1 + ns, slot_acc);  // C^T hv, C^T v, v.hv, Z^T hv
    }
    KR_TMARK(6);
    KR_GRID_SYNC();
    KR_TMARK(7);
    // ===== P2 ===== (the NSC decision moved to P1: s-space recurrence)
    KR_TMARK(8);
    if (sc.do_hvp) {
      // chv = C^T hv, cv = C^T v, alpha = v.hv - cv.chv  (== v.(hv - C chv), krylov.py:269-283)
      // one reduction of the contiguous slots into slot_acc (free until the next dots phase)
      reduce_slots(PP, bl, SL_CHV, 2 * s + 1 + ns, slot_acc);
      block_barrier();
      for (int i = threadIdx.x; i < 2 * s; i += blockDim.x) chv[i] = slot_acc[i];  // chv[0..s), cv at chv[s..2s)
      for (int i = threadIdx.x; i < ns; i += blockDim.x) zhv[i] = slot_acc[2 * s + 1 + i];  // Z^T hv_k for the next P1
      if (threadIdx.x == 0) red1[0] = slot_acc[2 * s];
      block_barrier();
      if (threadIdx.x == 0) {
        double a = red1[0];
        double corr = 0.0;
        for (int i = 0; i < s; ++i) corr += chv[s + i] * chv[i];
        sc.alpha = a - corr;
      }
      block_barrier();
      const double al = sc.alpha, be = sc.beta;
      const double* vk = lanczos(P, b, k, 3);
      const double* vkm = (k > 1) ? lanczos(P, b, k - 1, 4) : nullptr;
      const double* hvk = vec(P.w.hv[k & 1], n, b);
      double bsq[1] = {0.0};
      // two pixels per thread per round; C read 8 columns at a time with all loads in flight
      for (int64_t p0 = lo + threadIdx.x; p0 < hi; p0 += 2 * NT) {
        const int64_t p1 = p0 + NT;
        const bool h1 = p1 < hi;
        const int64_t q1 = h1 ? p1 : p0;
        double x0 = hvk[p0], x1 = hvk[q1];
        const double vk0 = vk[p0], vk1 = vk[q1];
        const double vm0 = vkm ? vkm[p0] : 0.0, vm1 = vkm ? vkm[q1] : 0.0;
        if (s > 0) {
          double cc0 = 0.0, cc1 = 0.0;
          for (int i0 = 0; i0 < s; i0 += 8) {
            double c0[8], c1[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              c0[i] = (i0 + i < s) ? C[(int64_t)(i0 + i) * A.ld_uc + p0] : 0.0;
              c1[i] = (i0 + i < s) ? C[(int64_t)(i0 + i) * A.ld_uc + q1] : 0.0;
            }
#pragma unroll
            for (int i = 0; i < 8; ++i)
              if (i0 + i < s) {
                cc0 += c0[i] * chv[i0 + i];
                cc1 += c1[i] * chv[i0 + i];
              }
          }
          x0 = x0 - cc0;  // vnext = hv - C chv
          x1 = x1 - cc1;
        }
        x0 = x0 - al * vk0;  // vnext -= alpha v
        x1 = x1 - al * vk1;
        x0 = x0 - be * vm0;  // vnext -= beta v_prev
        x1 = x1 - be * vm1;
        tmp[p0] = x0;
        bsq[0] += x0 * x0;
        if (h1) {
          tmp[p1] = x1;
          bsq[0] += x1 * x1;
        }
      }
      block_sum<1>(bsq, red);
      if (threadIdx.x == 0) P.w.part[((int64_t)bl * P.nslot + SL_BETA2) * P.Gs + j] = red[0];
    }
    {
      // evaluate before thread 0 flips `counted` (keeps the barrier below uniform)
      const bool count_now = sc.finished && !sc.counted;
      block_barrier();
      if (count_now && threadIdx.x == 0) {
        sc.counted = 1;
        if (leader) {
          A.iters[b] = sc.iters;
          A.reasons[b] = sc.reason;
          atomicAdd(P.w.done, 1);
        }
      }
      block_barrier();
    }
    KR_TMARK(9);
    KR_GRID_SYNC();
    KR_TMARK(10);
  }
#ifdef KR_RMINRES_TIMING
  if (threadIdx.x == 0 && bl == 0 && (j == 0 || j == P.Gs / 2))
    printf("rminres timing b=%d j=%d/%d k=%d ns: setup %llu | p1-scalar %llu upd %llu nsc %llu vk+fin %llu stencil %llu "
           "dots %llu | gsync1 %llu | p2-nsc %llu p2-u %llu | gsync2 %llu\n",
           b, j, P.Gs, tk, tsec[0], tsec[1], tsec[2], tsec[3], tsec[4], tsec[5], tsec[6], tsec[7], tsec[8], tsec[9],
           tsec[10]);
  if (threadIdx.x == 0 && blockIdx.x == 0)
    printf("stencil block0 ns: region %llu pointwise %llu blur %llu filters %llu\n", g_stencil_ns[0], g_stencil_ns[1],
           g_stencil_ns[2], g_stencil_ns[3]);
#endif
}

}  // namespace kr

using namespace kr;

namespace {

struct Layout {
  int Gs, chunk, nslot;
  int64_t vec_doubles;   // per-sample vector storage
  int64_t part_doubles;  // partials
  int64_t total;         // doubles (plus ints packed at the end)
  size_t smem;
};

int plan(const kr_op& op, const kr_solve_args& a, Layout& L) {
  const int64_t n = op_n(op);
  Geom g = make_geom(op);
  L.smem = sizeof(double) * ((size_t)g.total + MAX_SLOTS + 5 * MAX_S + 5 * MAX_NSC + RED_DOUBLES);
  int sms = device_sms();
  int per_sm = 0;
  if (sms > 0) {
    if (L.smem > 48 * 1024)
      ensure_smem(KR_PICK_Q(rminres_kernel, q_variant(op)), L.smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, KR_PICK_Q(rminres_kernel, q_variant(op)), NT, L.smem);
  }
  if (per_sm < 1) per_sm = 1;
  if (sms < 1) sms = 148;
  int max_blocks = per_sm * sms;
  int B = op.batch;
  L.chunk = B < max_blocks ? B : max_blocks;
  if (L.chunk < 1) L.chunk = 1;
  int want = (int)((n + 511) / 512);
  int nt = num_tiles(op);
  if (want < nt) want = nt;
  int Gs = max_blocks / L.chunk;
  if (Gs > want) Gs = want;
  if (Gs < 1) Gs = 1;
  L.Gs = Gs;
  int ns = a.stop_kind == 1 ? a.nsc_s : 0;
  L.nslot = 2 * a.s + 2 * ns + 2;
  L.vec_doubles = (int64_t)B * n * (a.basis ? 11 : 13);
  L.part_doubles = (int64_t)L.chunk * L.nslot * Gs;
  L.total = L.vec_doubles + L.part_doubles + 2 + (L.chunk + 1) / 2;  // + one barrier counter per sample
  return KR_OK;
}

int check_args(const kr_op& op, const kr_solve_args& a, bool dyn) {
  KR_CHECK_ARG(a.max_iter >= 1, "max_iter must be >= 1");
  KR_CHECK_ARG(a.s >= 0 && a.s <= MAX_S, "recycle dimension must be in [0, 128]");
  KR_CHECK_ARG(a.s == 0 || (a.U && a.C && a.ld_uc >= op_n(op)), "recycle space U/C missing or bad ld");
  KR_CHECK_ARG(a.stop_kind >= 0 && a.stop_kind <= 2, "stop_kind must be 0 (residual), 1 (NSC) or 2 (true hg)");
  KR_CHECK_ARG(a.stop_kind != 2 || (dyn && a.nsc_r0 && a.Z && a.nsc_s >= 1 && a.nsc_s <= MAX_NSC &&
                                    (a.s == 0 || a.ZtC)),
               "the true-hypergradient stop needs a kept basis, J's rows (p <= 128), J U and J w* - J w0");
  KR_CHECK_ARG(a.delta > 0.0, "tolerance must be positive");
  if (a.stop_kind == 1 || a.stop_kind == 2) {
    KR_CHECK_ARG(a.nsc_s >= 1 && a.nsc_s <= MAX_NSC, "NSC needs 1..128 columns");
    KR_CHECK_ARG(a.Z && a.ld_z >= op_n(op), "NSC needs Z");
    KR_CHECK_ARG(a.s == 0 || a.ZtC, "NSC with recycling needs Z^T C");
    // the per-sample kernel evaluates NSC through the tracked residual; the shared-block
    // kernel keeps Z^T r in s-space and forms the vector only when it is asked for
    KR_CHECK_ARG(dyn || a.track_residual, "NSC needs the tracked residual");
  }
  KR_CHECK_ARG(a.g && a.w && a.res_norms && a.stop_vals && a.iters && a.reasons, "missing output buffer");
  KR_CHECK_ARG(!a.basis || a.ld_basis >= op_n(op), "basis leading dimension smaller than n");
  KR_CHECK_ARG(!a.track_residual || a.r, "track_residual needs an r buffer");
  KR_CHECK_ARG(op.reg_kind != KR_REG_FILTERS || op.potential == KR_POT_QUADRATIC || op.curv,
               "operator not prepared (curv)");
  KR_CHECK_ARG(op.reg_kind != KR_REG_TV || op.curv, "operator not prepared (curv)");
  return KR_OK;
}

}  // namespace

namespace kr {
bool rminres_dyn_applies(const kr_op& op, const kr_solve_args& a);
int64_t rminres_dyn_workspace(const kr_op& op, const kr_solve_args& a);
int rminres_dyn(const kr_op& op, const kr_solve_args& a, double* work, int64_t work_len, cudaStream_t st);
}  // namespace kr

extern "C" int64_t kr_rminres_workspace(const kr_op* op, const kr_solve_args* a) {
  if (!op || !a || validate_op(*op) != KR_OK) return -1;
  if (rminres_dyn_applies(*op, *a)) return rminres_dyn_workspace(*op, *a);
  Layout L;
  plan(*op, *a, L);
  return L.total;
}

extern "C" int kr_rminres(const kr_op* op, const kr_solve_args* a, double* work, int64_t work_len,
                          kr_stream_t stream) {
  KR_CHECK_ARG(op && a, "null argument");
  KR_TRY(validate_op(*op));
  if (op->batch == 0) return KR_OK;
  const bool dyn = rminres_dyn_applies(*op, *a);
  KR_TRY(check_args(*op, *a, dyn));
  // with the Lanczos basis kept (every recycled sequence solve): blocks shared by all
  // running samples (kr_rminres_dyn.cu)
  if (dyn) return rminres_dyn(*op, *a, work, work_len, (cudaStream_t)stream);
  Layout L;
  plan(*op, *a, L);
  KR_CHECK_ARG(work && work_len >= L.total, "rminres workspace too small");
  const int64_t n = op_n(*op);
  const int B = op->batch;
  Params P;
  P.op = *op;
  P.a = *a;
  P.n = n;
  P.Gs = L.Gs;
  P.nslot = L.nslot;
  double* cur = work;
  auto take = [&](int64_t cnt) {
    double* r = cur;
    cur += cnt;
    return r;
  };
  P.w.tmp = take(B * n);
  P.w.u = take(B * n);
  P.w.hv[0] = take(B * n);
  P.w.hv[1] = take(B * n);
  P.w.vt[0] = take(B * n);
  P.w.vt[1] = take(B * n);
  P.w.hvt[0] = take(B * n);
  P.w.hvt[1] = take(B * n);
  P.w.rv = take(B * n);
  P.w.wv = take(B * n);
  if (!a->basis) {
    P.w.vr[0] = take(B * n);
    P.w.vr[1] = take(B * n);
  } else {
    P.w.vr[0] = P.w.vr[1] = nullptr;
  }
  take((a->basis ? 11 : 13) * (int64_t)B * n - (cur - work));  // keep layout == plan
  P.w.part = take(L.part_doubles);
  P.w.done = reinterpret_cast<int*>(take(2 + (L.chunk + 1) / 2));
  cudaStream_t st = (cudaStream_t)stream;
  const void* kfn = KR_PICK_Q(rminres_kernel, q_variant(*op));
  KR_TRY(ensure_smem(kfn, L.smem));
  for (int b0 = 0; b0 < B; b0 += L.chunk) {
    P.b0 = b0;
    P.nb = (B - b0) < L.chunk ? (B - b0) : L.chunk;
    cudaMemsetAsync(P.w.done, 0, (4 + 2 * ((L.chunk + 1) / 2)) * sizeof(int), st);
    dim3 grid(P.nb * P.Gs), block(NT);
    void* args[] = {&P};
    cudaError_t e = cudaLaunchCooperativeKernel(kfn, grid, block, args, L.smem, st);
    if (e != cudaSuccess) return fail(KR_ECUDA, std::string("rminres cooperative launch: ") + cudaGetErrorString(e));
  }
  return check_launch("kr_rminres");
}

