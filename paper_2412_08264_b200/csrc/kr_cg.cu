// kr_cg.cu -- batched conjugate gradients as one persistent cooperative kernel.
//
// Algorithm: /root/reference/pkg/src/krecycle/krylov.py:408-483 (plain CG,
// NonSPDError on p^T H p <= 0, basis columns r_k/||r_k||), with the stop rule
// evaluated on the explicit residual (stopping.py:93-118).  Two per-sample
// barriers per iteration: the direction p_k = r_{k-1} + (rr_{k-1}/rr_{k-2}) p_{k-1}
// is formed on the fly inside the stencil load, so it needs no barrier of its own.
//
// Recycled CG (s > 0, Minv = (U^T C)^{-1}): deflated CG (Saad, Yeung, Erhel &
// Guyomarc'h, SIAM J. Sci. Comput. 21 (2000), Alg. 2.2; oracle cpu_krylov.rcg):
// the start is projected, x += U Minv U^T r, r -= C Minv U^T r (one extra barrier),
// and p_k = r + beta p_{k-1} - U mu with mu = Minv C^T r, the C^T r partials riding
// with r.r and the U mu term folded into the same on-the-fly stencil load.

#include <string>

#include "kr_common.cuh"
#include "kr_internal.h"
#include "kr_solver.cuh"


namespace kr {

struct CgParams {
  kr_op op;
  kr_solve_args a;
  double* r;      // [B][n] residual
  double* p[2];   // [B][n] directions by parity
  double* hp;     // [B][n]
  double* wv;     // [B][n] solution
  double* part;
  int* done;
  int Gs, b0, nb, nslot;
  int64_t n;
};

template <int Q>
__global__ void __launch_bounds__(NT, 2) cg_kernel(CgParams P) {
  unsigned int grid_target = 0;
  extern __shared__ double smem[];
  const kr_op& op = P.op;
  const kr_solve_args& A = P.a;
  const Geom g = make_geom(op);
  Smem sm = carve(g, smem);
  double* slot_acc = smem + g.total;
  double* nscv = slot_acc + MAX_SLOTS;
  double* ctr = nscv + MAX_NSC;   // C^T r (or U^T r at the start), MAX_S
  double* mu = ctr + MAX_S;       // Minv C^T r, MAX_S
  double* red = mu + MAX_S;
  __shared__ double s_rr, s_rr_old, s_res, s_php, s_coef;
  __shared__ int s_active, s_finished, s_counted, s_iters, s_reason, s_hvp;
  __shared__ double red1[4];  // single-slot reductions

  const Partials PP{P.part, P.nslot, P.Gs};
  const int bl = blockIdx.x / P.Gs, j = blockIdx.x % P.Gs, b = P.b0 + bl;
  const int64_t n = P.n;
  const int ns = (A.stop_kind == 1) ? A.nsc_s : 0;
  const int s = A.Minv ? A.s : 0;  // deflation columns (recycled CG)
  const int SL_NSC = 0, SL_RR = ns, SL_PHP = ns + 1, SL_CR = ns + 2;  // SL_CR .. SL_CR + s: C^T r
  const double* U = s ? A.U + (int64_t)b * A.bs_uc : nullptr;
  const double* C = s ? A.C + (int64_t)b * A.bs_uc : nullptr;
  const double* Mi = s ? A.Minv + (int64_t)b * s * s : nullptr;
  const int64_t lo = n * j / P.Gs, hi = n * (j + 1) / P.Gs;
  const int ntiles = num_tiles(op);
  const bool leader = (j == 0);
  const double* gb = A.g + (int64_t)b * n;
  const double* w0 = A.w0 ? A.w0 + (int64_t)b * n : nullptr;
  const double* Z = ns ? A.Z + (int64_t)b * A.bs_z : nullptr;
  double* r = P.r + (int64_t)b * n;
  double* hp = P.hp + (int64_t)b * n;
  double* w = P.wv + (int64_t)b * n;
  double* res_norms = A.res_norms + (int64_t)b * (A.max_iter + 1);
  double* stop_vals = A.stop_vals + (int64_t)b * (A.max_iter + 1);

  load_weights(op, g, sm);
  if (threadIdx.x == 0) {
    s_active = 1;
    s_finished = 0;
    s_counted = 0;
    s_iters = 0;
    s_reason = R_MAXIT;
    s_rr_old = 1.0;
  }
  block_barrier();
  // r = g - H w0
  if (w0) {
    for (int tile = j; tile < ntiles; tile += P.Gs) {
      tile_hvp_t<Q>(op, g, sm, b, TileIn{w0, 1.0, nullptr, 0.0}, tile);
      for (int l = threadIdx.x; l < TPX; l += blockDim.x) {
        int64_t p = tile_pixel(op, tile, l);
        if (p >= 0) r[p] = gb[p] - sm.res[l];
      }
      block_barrier();
    }
  } else {
    for (int64_t p = lo + threadIdx.x; p < hi; p += blockDim.x) r[p] = gb[p];
  }
  for (int64_t p = lo + threadIdx.x; p < hi; p += blockDim.x) w[p] = w0 ? w0[p] : 0.0;
  grid_barrier(reinterpret_cast<unsigned int*>(P.done) + 1 + bl, P.Gs, grid_target);  // per-sample
  if (s) {
    // deflated start: y = Minv U^T r, w += U y, r -= C y  (U^T r = 0 afterwards)
    for (int i = threadIdx.x; i < s; i += blockDim.x) slot_acc[i] = 0.0;
    block_barrier();
    slot_dots(U, A.ld_uc, s, lo, hi, [&](int64_t p) { return r[p]; }, slot_acc, red);
    write_partials(PP, bl, j, SL_CR, s, slot_acc);
    grid_barrier(reinterpret_cast<unsigned int*>(P.done) + 1 + bl, P.Gs, grid_target);  // per-sample
    reduce_slots(PP, bl, SL_CR, s, ctr);
    block_barrier();
    for (int i = threadIdx.x; i < s; i += blockDim.x) {
      double y = 0.0;
      for (int l = 0; l < s; ++l) y += Mi[(int64_t)i * s + l] * ctr[l];
      mu[i] = y;
    }
    block_barrier();
    for (int64_t p = lo + threadIdx.x; p < hi; p += blockDim.x) {
      double du = 0.0, dc = 0.0;
      for (int i = 0; i < s; ++i) {
        du += U[(int64_t)i * A.ld_uc + p] * mu[i];
        dc += C[(int64_t)i * A.ld_uc + p] * mu[i];
      }
      w[p] += du;
      r[p] -= dc;
    }
    // all of the sample's SL_CR partials were read before anyone rewrites them below
    grid_barrier(reinterpret_cast<unsigned int*>(P.done) + 1 + bl, P.Gs, grid_target);  // per-sample
  }
  {
    double v[1] = {0.0};
    for (int64_t p = lo + threadIdx.x; p < hi; p += blockDim.x) v[0] += r[p] * r[p];
    block_sum<1>(v, red);
    write_partial1(PP, bl, j, SL_RR, red[0]);
    if (ns) {
      for (int i = threadIdx.x; i < ns; i += blockDim.x) slot_acc[i] = 0.0;
      block_barrier();
      slot_dots(Z, A.ld_z, ns, lo, hi, [&](int64_t p) { return r[p]; }, slot_acc, red);
      write_partials(PP, bl, j, SL_NSC, ns, slot_acc);
    }
    if (s) {
      for (int i = threadIdx.x; i < s; i += blockDim.x) slot_acc[i] = 0.0;
      block_barrier();
      slot_dots(C, A.ld_uc, s, lo, hi, [&](int64_t p) { return r[p]; }, slot_acc, red);
      write_partials(PP, bl, j, SL_CR, s, slot_acc);
    }
  }
  grid_barrier(reinterpret_cast<unsigned int*>(P.done) + 1 + bl, P.Gs, grid_target);  // per-sample

  for (int k = 1; k <= A.max_iter + 1; ++k) {
    if (s_counted) break;  // this sample is reported: its blocks leave together
    // ===== P1: stop test on r_{k-1}, then hp = H p_k =====
    if (ns && s_active) {
      reduce_slots(PP, bl, SL_NSC, ns, nscv);
      block_barrier();
    }
    if (s_active) {
      reduce_slots(PP, bl, SL_RR, 1, red1);
      block_barrier();
    }
    if (s && s_active) {  // mu = Minv C^T r_{k-1}
      reduce_slots(PP, bl, SL_CR, s, ctr);
      block_barrier();
      for (int i = threadIdx.x; i < s; i += blockDim.x) {
        double y = 0.0;
        for (int l = 0; l < s; ++l) y += Mi[(int64_t)i * s + l] * ctr[l];
        mu[i] = y;
      }
    }
    if (threadIdx.x == 0) {
      s_hvp = 0;
      if (s_active) {
        double rr = red1[0];
        double res = sqrt(rr);
        double val = res;
        if (ns) {
          double ss = 0.0;
          for (int i = 0; i < ns; ++i) ss += nscv[i] * nscv[i];
          val = sqrt(ss);
        }
        if (leader) {
          res_norms[k - 1] = res;
          stop_vals[k - 1] = val;
        }
        if (val < A.delta) {
          s_active = 0; s_finished = 1; s_iters = k - 1; s_reason = R_TOL;
        } else if (k - 1 == A.max_iter) {
          s_active = 0; s_finished = 1; s_iters = k - 1; s_reason = R_MAXIT;
        } else {
          s_coef = (k == 1) ? 0.0 : rr / s_rr_old;
          s_rr_old = rr;
          s_res = res;
          s_hvp = 1;
        }
      }
    }
    block_barrier();
    if (s_hvp) {
      double* pk = P.p[k & 1] + (int64_t)b * n;
      const double* po = (k == 1) ? nullptr : P.p[(k + 1) & 1] + (int64_t)b * n;
      const double coef = s_coef, res = s_res;
      double* basis = A.basis ? A.basis + (int64_t)b * A.bs_basis + (int64_t)(k - 1) * A.ld_basis : nullptr;
      for (int64_t p = lo + threadIdx.x; p < hi; p += blockDim.x) {
        double d = po ? r[p] + coef * po[p] : r[p];
        for (int i = 0; i < s; ++i) d -= U[(int64_t)i * A.ld_uc + p] * mu[i];
        pk[p] = d;
        if (basis) basis[p] = (res > 0.0) ? r[p] / res : 0.0;
      }
      double php[1] = {0.0};
      for (int tile = j; tile < ntiles; tile += P.Gs) {
        TileIn tin{r, 1.0, po ? po : r, po ? coef : 0.0};
        if (s) {
          tin.U = U;
          tin.ldu = A.ld_uc;
          tin.s = s;
          tin.mu = mu;
        }
        tile_hvp_t<Q>(op, g, sm, b, tin, tile);
        const int tyc = tiles_x(op);
        for (int l = threadIdx.x; l < TPX; l += blockDim.x) {
          int64_t p = tile_pixel(op, tile, l);
          if (p < 0) continue;
          hp[p] = sm.res[l];
          double pv;
          if (op.data_kind == KR_DATA_DENSE) {
            pv = pk[p];
          } else {
            int ty = l / TW, tx = l - ty * TW;
            pv = sm.S0[(ty + g.H) * g.RW + tx + g.H];
          }
          php[0] += pv * sm.res[l];
          (void)tyc;
        }
        block_barrier();
      }
      block_sum<1>(php, red);
      write_partial1(PP, bl, j, SL_PHP, red[0]);
    }
    grid_barrier(reinterpret_cast<unsigned int*>(P.done) + 1 + bl, P.Gs, grid_target);  // per-sample
    // ===== P2: step =====
    if (s_hvp) {
      reduce_slots(PP, bl, SL_PHP, 1, red1 + 1);
      block_barrier();
      if (threadIdx.x == 0) {
        double php = red1[1];
        s_php = php;
        if (php <= 0.0) {
          s_active = 0; s_finished = 1; s_iters = k; s_reason = R_NONSPD;
        }
      }
      block_barrier();
      if (s_active) {
        const double a = s_rr_old / s_php;
        const double* pk = P.p[k & 1] + (int64_t)b * n;
        double v[1] = {0.0};
        for (int64_t p = lo + threadIdx.x; p < hi; p += blockDim.x) {
          w[p] = w[p] + a * pk[p];
          double rn = r[p] - a * hp[p];
          r[p] = rn;
          v[0] += rn * rn;
        }
        block_sum<1>(v, red);
        write_partial1(PP, bl, j, SL_RR, red[0]);
        if (ns) {
          for (int i = threadIdx.x; i < ns; i += blockDim.x) slot_acc[i] = 0.0;
          block_barrier();
          slot_dots(Z, A.ld_z, ns, lo, hi, [&](int64_t p) { return r[p]; }, slot_acc, red);
          write_partials(PP, bl, j, SL_NSC, ns, slot_acc);
        }
        if (s) {
          for (int i = threadIdx.x; i < s; i += blockDim.x) slot_acc[i] = 0.0;
          block_barrier();
          slot_dots(C, A.ld_uc, s, lo, hi, [&](int64_t p) { return r[p]; }, slot_acc, red);
          write_partials(PP, bl, j, SL_CR, s, slot_acc);
        }
      }
    }
    if (s_finished && !s_counted) {
      double* wout = A.w + (int64_t)b * n;
      double* rout = A.r ? A.r + (int64_t)b * n : nullptr;
      for (int64_t p = lo + threadIdx.x; p < hi; p += blockDim.x) {
        wout[p] = w[p];
        if (rout) rout[p] = r[p];
      }
      block_barrier();
      if (threadIdx.x == 0) {
        s_counted = 1;
        if (leader) {
          A.iters[b] = s_iters;
          A.reasons[b] = s_reason;
          atomicAdd(P.done, 1);
        }
      }
      block_barrier();
    }
    grid_barrier(reinterpret_cast<unsigned int*>(P.done) + 1 + bl, P.Gs, grid_target);  // per-sample
  }
}

}  // namespace kr

using namespace kr;

namespace {

struct CgLayout {
  int Gs, chunk, nslot;
  int64_t total;
  size_t smem;
};

void cg_plan(const kr_op& op, const kr_solve_args& a, CgLayout& L) {
  const int64_t n = op_n(op);
  Geom g = make_geom(op);
  L.smem = sizeof(double) * ((size_t)g.total + MAX_SLOTS + MAX_NSC + 2 * MAX_S + RED_DOUBLES);
  int sms = device_sms(), per_sm = 0;
  if (sms > 0) {
    if (L.smem > 48 * 1024)
      ensure_smem(KR_PICK_Q(cg_kernel, q_variant(op)), L.smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, KR_PICK_Q(cg_kernel, q_variant(op)), NT, L.smem);
  }
  if (per_sm < 1) per_sm = 1;
  if (sms < 1) sms = 148;
  const int max_blocks = per_sm * sms, B = op.batch;
  L.chunk = B < max_blocks ? (B > 0 ? B : 1) : max_blocks;
  int want = (int)((n + 511) / 512);
  if (want < num_tiles(op)) want = num_tiles(op);
  int Gs = max_blocks / L.chunk;
  L.Gs = Gs < 1 ? 1 : (Gs > want ? want : Gs);
  L.nslot = (a.stop_kind == 1 ? a.nsc_s : 0) + 2 + (a.Minv ? a.s : 0);
  L.total = 5 * (int64_t)B * n + (int64_t)L.chunk * L.nslot * L.Gs + 2 + (L.chunk + 1) / 2;
}

}  // namespace

extern "C" int64_t kr_cg_workspace(const kr_op* op, const kr_solve_args* a) {
  if (!op || !a || validate_op(*op) != KR_OK) return -1;
  CgLayout L;
  cg_plan(*op, *a, L);
  return L.total;
}

extern "C" int kr_cg(const kr_op* op, const kr_solve_args* a, double* work, int64_t work_len, kr_stream_t stream) {
  KR_CHECK_ARG(op && a, "null argument");
  KR_TRY(validate_op(*op));
  if (op->batch == 0) return KR_OK;
  KR_CHECK_ARG(a->max_iter >= 1, "max_iter must be >= 1");
  KR_CHECK_ARG(a->stop_kind == 0 || a->stop_kind == 1, "stop_kind must be 0 or 1");
  KR_CHECK_ARG(a->delta > 0.0, "tolerance must be positive");
  KR_CHECK_ARG(a->stop_kind == 0 || (a->Z && a->nsc_s >= 1 && a->nsc_s <= MAX_NSC), "NSC needs Z");
  KR_CHECK_ARG(!a->Minv || (a->s >= 1 && a->s <= MAX_S && a->U && a->C && a->ld_uc >= op_n(*op)),
               "recycled CG needs U, C (s <= 128) with Minv");
  KR_CHECK_ARG(a->g && a->w && a->res_norms && a->stop_vals && a->iters && a->reasons, "missing output buffer");
  CgLayout L;
  cg_plan(*op, *a, L);
  KR_CHECK_ARG(work && work_len >= L.total, "cg workspace too small");
  const int64_t n = op_n(*op);
  const int B = op->batch;
  CgParams P;
  P.op = *op;
  P.a = *a;
  P.n = n;
  P.Gs = L.Gs;
  P.nslot = L.nslot;
  P.r = work;
  P.p[0] = P.r + (int64_t)B * n;
  P.p[1] = P.p[0] + (int64_t)B * n;
  P.hp = P.p[1] + (int64_t)B * n;
  P.wv = P.hp + (int64_t)B * n;
  P.part = P.wv + (int64_t)B * n;
  P.done = reinterpret_cast<int*>(P.part + (int64_t)L.chunk * L.nslot * L.Gs);
  cudaStream_t st = (cudaStream_t)stream;
  const void* kfn = KR_PICK_Q(cg_kernel, q_variant(*op));
  KR_TRY(ensure_smem(kfn, L.smem));
  for (int b0 = 0; b0 < B; b0 += L.chunk) {
    P.b0 = b0;
    P.nb = (B - b0) < L.chunk ? (B - b0) : L.chunk;
    cudaMemsetAsync(P.done, 0, (4 + 2 * ((L.chunk + 1) / 2)) * sizeof(int), st);
    void* args[] = {&P};
    cudaError_t e = cudaLaunchCooperativeKernel(kfn, dim3(P.nb * P.Gs), dim3(NT), args, L.smem, st);
    if (e != cudaSuccess) return fail(KR_ECUDA, std::string("cg cooperative launch: ") + cudaGetErrorString(e));
  }
  return check_launch("kr_cg");
}
