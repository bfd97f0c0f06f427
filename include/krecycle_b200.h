/*
 * krecycle_b200.h -- C ABI of the B200-native recycled hypergradient solve.
 *
 * The reference (arXiv 2412.08264, package `krecycle`) is pure Python and has
 * no FFI; its "operator API" is a duck-typed protocol.  Each entry point below
 * replaces one reference interface (cited as file:line under
 * /root/reference/pkg/src/krecycle/) with plain pointers and sizes:
 *
 *   kr_op_prepare      <- the closures built by foe_hessian / mixed_jacobian
 *                         (operators.py:363-383, 411-444): per-pixel curvature
 *                         phi''(C_j xhat) and slope phi'(C_j xhat) cached once
 *                         per (theta, xhat), like `kx_list` (operators.py:427)
 *   kr_hvp             <- SymmetricOperator.__call__ / apply_matrix
 *                         (operators.py:253-261): H v for t columns, B samples
 *   kr_jadj            <- MixedJacobianOperator.apply_adjoint / _matrix
 *                         (operators.py:290-298): J w for t columns, B samples
 *   kr_lower_eval      <- foe_cost / foe_gradient (operators.py:329-353)
 *   kr_rminres         <- rminres / minres (krylov.py:386-405) with
 *                         _rminres_core (krylov.py:205-383), the residual
 *                         recurrence (krylov.py:154-181) and the stop rules
 *                         ResidualNormRule / NscRule (stopping.py:93-118)
 *   kr_cg              <- cg (krylov.py:408-483)
 *   kr_syev_select     <- the t x t eigen-selection inside ritz_select / gsvd_pair /
 *                         rgen_select (recycling.py:202-213, 226-236, 275-359)
 *   kr_qrcp_small      <- the pivoted QR's column choice and rank drop
 *                         (recycling.py:187-199, 362-383) on the small R factor
 *   kr_chol_inv        <- the t x t factorizations of the QRs in build_candidate_basis,
 *                         gsvd_pair, prepare_recycle and the condition check
 *                         (recycling.py:187-199, 290-313, 362-383)
 *
 * All array pointers are DEVICE pointers (fp64 unless stated), all calls are
 * asynchronous on the given CUDA stream, and every function returns 0 on
 * success or a negative KR_E* code; kr_last_error() gives the message.  The
 * error codes map onto the reference's exceptions: KR_EINVAL -> ValueError,
 * KR_ENONSPD -> NonSPDError, KR_ECUDA -> RuntimeError.
 *
 * Layout: image vectors are row-major (rows x cols), samples contiguous
 * ([batch][n]); a block of t column vectors per sample is [batch][t][ld]
 * (column j of sample b at ptr + b*bs + j*ld), i.e. the numpy n x t matrix of
 * the reference stored column-major.
 */
#ifndef KRECYCLE_B200_H
#define KRECYCLE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* kr_stream_t; /* == cudaStream_t */

#define KR_ABI_VERSION 6

/* Largest candidate width t = k_prev + s_prev of the small dense kernels and the recycle
 * update: BASELINE C5 with s = 80 and 500 iterations (t <= 580), with margin. */
#define KR_TMAX 640

#define KR_OK 0
#define KR_EINVAL (-1)
#define KR_ECUDA (-2)
#define KR_ENONSPD (-3)
#define KR_ENOMEM (-4)

#define KR_MAX_BLUR 31
#define KR_MAX_KSIZE 9
#define KR_MAX_FILTERS 64

/* data term: cost = data_scale/2 ||A x - y||^2 + ridge/2 ||x||^2 */
#define KR_DATA_NONE 0
#define KR_DATA_MASK 1  /* A = row subsampling; A^T A = diag(mask) (operators.py:187-235) */
#define KR_DATA_BLUR 2  /* A = separable Gaussian, true convolution, zero boundary */
#define KR_DATA_DENSE 3 /* H = explicit symmetric matrix (dense_operator, operators.py:269-274) */

#define KR_REG_NONE 0
#define KR_REG_FILTERS 1 /* sum_j w_j sum_p phi((c_j * x)_p) */
#define KR_REG_TV 2      /* w sum_p sqrt(Dh^2 + Dv^2 + eps^2), Neumann forward differences */

#define KR_POT_QUADRATIC 0  /* phi(t) = t^2 (reference FoE, operators.py:5-7) */
#define KR_POT_SMOOTH_ABS 1 /* phi(t) = sqrt(t^2 + eps^2) */

/* One Hessian / Jacobian family for a batch of samples sharing theta. */
typedef struct kr_op {
  int32_t rows, cols, batch;
  int32_t data_kind;
  double data_scale;
  double ridge;
  const double* mask;     /* KR_DATA_MASK: [batch][n] 0/1 (mask_bstride 0 = shared) */
  int64_t mask_bstride;
  const double* dense;    /* KR_DATA_DENSE: [batch][n][n] row-major */
  int64_t dense_bstride;
  int32_t blur_size;      /* odd, <= KR_MAX_BLUR */
  double blur_taps[KR_MAX_BLUR]; /* 1-D normalised taps; blur = outer(taps, taps) */
  int32_t reg_kind;
  int32_t potential;
  double eps;
  int32_t num_filters, ksize;
  const double* kernels;  /* [J][q][q] row-major (the theta layout of operators.py:150-172) */
  const double* fweights; /* [J] exp(a_j) after the +/-30 clamp (operators.py:174-184); TV: [1] */
  double* curv;           /* [batch][J][n] phi''(C_j xhat); TV: [batch][3][n] (m11, m12, m22) */
  double* slope;          /* [batch][J][n] phi'(C_j xhat);  TV: [batch][2][n] (Dh xhat/s, Dv xhat/s) */
  const double* xhat;     /* [batch][n] */
} kr_op;

/* Arguments of one batched recycled-MINRES solve (krylov.py:205-383). */
typedef struct kr_solve_args {
  int32_t max_iter;
  int32_t s;               /* recycle columns (zero-padded columns are allowed) */
  const double* g;         /* [batch][n] right-hand sides */
  const double* w0;        /* [batch][n] initial guesses or NULL (zero) */
  const double* U;         /* [batch][s][ld_uc] */
  const double* C;         /* [batch][s][ld_uc], C^T C = I */
  int64_t ld_uc, bs_uc;
  int32_t stop_kind;       /* 0 = residual norm (stopping.py:93-99), 1 = NSC (stopping.py:102-118),
                              2 = true hypergradient error (stopping.py:121-185; see nsc_r0) */
  double delta;            /* strict: stop when value < delta (stopping.py:89-90) */
  int32_t nsc_s;           /* NSC columns */
  const double* Z;         /* [batch][nsc_s][ld_z]: Z = W V_H,sel diag(mu_sel) (nsc_value, stopping.py:69-72) */
  int64_t ld_z, bs_z;
  const double* ZtC;       /* [batch][nsc_s][s]: Z^T C (row-major nsc_s x s) */
  int32_t track_residual;  /* maintain r by the recurrence (krylov.py:154-181) */
  double* w;               /* out [batch][n] solution */
  double* r;               /* out [batch][n] tracked residual (if track_residual) */
  double* basis;           /* out [batch][max_iter][ld_basis] Lanczos vectors, or NULL */
  int64_t ld_basis, bs_basis;
  double* res_norms;       /* out [batch][max_iter+1] */
  double* stop_vals;       /* out [batch][max_iter+1] */
  int32_t* iters;          /* out [batch] */
  int32_t* reasons;        /* out [batch]: 0 tolerance, 1 max_iter, 2 breakdown, 3 non-SPD */
  const double* Minv;      /* [batch][s][s] (U^T C)^{-1}, row-major: kr_cg deflation (recycled CG); NULL = plain CG */
  const double* nsc_r0;    /* stop_kind 2 (true hypergradient error, stopping.py:121-185): [batch][nsc_s]
                              J w* - J w0 with w* = H^-1 g; Z then holds the rows of J (nsc_s = p <= 128),
                              ZtC = J U, and the value ||J H^-1 r_k|| follows the residual recurrence
                              with Z^T hv_k replaced by J v_k (= J H^-1 H v_k).  Needs a kept basis. */
} kr_solve_args;

int kr_abi_version(void);
const char* kr_last_error(void);
int kr_device_info(int32_t* num_sms, int32_t* cc_major, int32_t* cc_minor);
/* sizeof(kr_op), sizeof(kr_solve_args): lets an FFI binding verify its struct mirror. */
int kr_struct_sizes(int64_t* op_size, int64_t* args_size);

int kr_op_prepare(const kr_op* op, kr_stream_t stream);

int kr_hvp(const kr_op* op, const double* V, int64_t ldv, int64_t bsv, int32_t ncols,
           double* HV, int64_t ldo, int64_t bso, kr_stream_t stream);

int64_t kr_jadj_workspace(const kr_op* op, int32_t ncols);
int kr_jadj(const kr_op* op, const double* W, int64_t ldw, int64_t bsw, int32_t ncols,
            double* JW, int64_t ldo, int64_t bso, double* work, int64_t work_len,
            kr_stream_t stream);

/* Lower-level cost and gradient at X ([batch][n]) for data y ([batch][n] blur / [batch][n] masked-and-scattered):
   cost[b] = data_scale/2 ||A x_b - y_b||^2 + ridge/2 ||x_b||^2 + R(x_b);  grad = d cost / d x. */
int64_t kr_lower_workspace(const kr_op* op);
int kr_lower_eval(const kr_op* op, const double* X, const double* Y, double* cost, double* grad,
                  double* work, int64_t work_len, kr_stream_t stream);

int64_t kr_rminres_workspace(const kr_op* op, const kr_solve_args* args);
int kr_rminres(const kr_op* op, const kr_solve_args* args, double* work, int64_t work_len,
               kr_stream_t stream);

/* CG (krylov.py:408-483); NonSPD curvature is reported through reasons[b] = 3.  With
 * s > 0 and Minv set: recycled (deflated) CG with deflation space U (Saad, Yeung,
 * Erhel & Guyomarc'h 2000; the "recycled CG" of the north star), residuals kept
 * orthogonal to U, directions p = r + beta p - U Minv C^T r. */
int64_t kr_cg_workspace(const kr_op* op, const kr_solve_args* args);
int kr_cg(const kr_op* op, const kr_solve_args* args, double* work, int64_t work_len,
          kr_stream_t stream);

/* Selected eigenpairs of a batch of symmetric t_b x t_b matrices (t_b <= tmax <= 228),
 * the eigen-selection step of ritz_select (recycling.py:226-236, _select_indices
 * :202-213, _clamp_dim) and of gsvd_pair's right singular vectors
 * (recycling.py:275-313, through Q1^T Q1).  Matrix b: element (i, j) at
 * A + b*bsa + j*lda + i (symmetrised as (A + A^T)/2), t_b = dims[b] (DEVICE int32).
 * size_code 0/1/2 = S/L/M: s_b = min(s, t_b) pairs, the s_b smallest (S), the s_b
 * largest (L), or s_b/2 smallest then the rest largest (M), ascending.  Outputs:
 * lam[b*bsl + q], eigenvector q of sample b at Z + b*bsz + q*ldz (rows >= t_b and
 * columns >= s_b zeroed, largest-|component| positive), nsel[b] = s_b (optional). */
int64_t kr_syev_select_workspace(int32_t batch, int32_t tmax);
int kr_syev_select(const double* A, int64_t lda, int64_t bsa, const int32_t* dims, int32_t batch,
                   int32_t tmax, int32_t size_code, int32_t s, double* lam, int64_t bsl, double* Z,
                   int64_t ldz, int64_t bsz, int32_t* nsel, double* work, int64_t work_len,
                   kr_stream_t stream);

/* Batched Cholesky + triangular inverse of the t_b x t_b Gram blocks of the
 * Cholesky-QR passes (recycling._cholqr2 batched; the reference's pivoted QR at
 * recycling.py:187-199, 362-383 and the QR of [Jt; Ht] at :305) and of the
 * W^T H W condition screen (recycling.py:290-296).  G b: element (i, j) at
 * G + b*bsg + i*ldg + j (symmetrised), t_b = dims[b] <= tmax <= KR_TMAX (DEVICE int32).
 * tmax <= 228 works in shared memory (work may be null); larger tmax needs
 * kr_chol_inv_workspace(batch, tmax) doubles of DEVICE work (the packed factors).
 * flags bit 0: scale by D = sqrt(diag G); bit 1: write F; bit 2: skip mode -- a row
 * whose pivot falls below 4 t eps times its diagonal is removed (zero column of L,
 * zero row of F, skipped[b*tmax + i] = 1) instead of stopping; bit 3: partial -- on a
 * breakdown at row i, F keeps the inverse of the leading i x i factor and zero rows
 * i..t_b-1 (otherwise F is the identity).  shift (nullable,
 * DEVICE, per sample) is added to the scaled diagonal.  G_s = L L^T; F = L^{-1} D^{-1}
 * row-major (F + b*bsf + i*ldf + j), zero upper triangle, identity pad block.
 * info[b] = -1 or the first row whose pivot is not positive; stats[4b..4b+3] =
 * (min L_jj, max L_jj, min D, 0) (nullable). */
int64_t kr_chol_inv_workspace(int32_t batch, int32_t tmax);
int kr_chol_inv(const double* G, int64_t ldg, int64_t bsg, const int32_t* dims, int32_t batch,
                int32_t tmax, int32_t flags, const double* shift, double* F, int64_t ldf, int64_t bsf,
                double* stats, int32_t* info, uint8_t* skipped, double* work, int64_t work_len,
                kr_stream_t stream);

/* QR with column pivoting of small matrices (t_b <= tmax <= 256), one CTA each:
 * the pivoted QR of build_candidate_basis / prepare_recycle (recycling.py:187-199,
 * 362-383, scipy qr(pivoting=True)) applied to the R factor of the tall block.
 * M (in/out, DEVICE): column j of sample b at M + b*tmax*tmax + j*tmax; on return
 * column perm[j] (the physical column of pivot j) holds column j of R_piv.  Stops at the first |R_kk| <= rtol |R_00|:
 * rank[b] = k.  Q (out): column j (< rank) of Q_R at Q + b*tmax*tmax + j*tmax, the
 * other columns zero.  perm[b*tmax + j] = original index of pivot j (nullable).
 * work: batch*tmax doubles. */
int kr_qrcp_small(double* M, const int32_t* dims, int32_t batch, int32_t tmax, double rtol, double* Q,
                  int32_t* rank, int32_t* perm, double* work, int64_t work_len, kr_stream_t stream);
/* Same contract, one 4-CTA thread-block cluster per matrix: the columns stay in the
 * CTAs' shared memory and the pivot / reflector exchange goes over DSMEM. */
int kr_qrcp_small_cluster(double* M, const int32_t* dims, int32_t batch, int32_t tmax, double rtol, double* Q,
                          int32_t* rank, int32_t* perm, double* work, int64_t work_len, kr_stream_t stream);

/* Batched Gram of row blocks: G_b[i][j] = a_i . b_j (row-major G, ldg, bsg) for
 * A_b, B_b given as `rows` rows of length n (row stride ld, batch stride bs) -- the
 * (B, t, n) Grams of the recycle update's QRs and W^T H W (recycling.py:194, 250,
 * 333).  Hand-written fp64 tensor-core kernel (mma.m8n8k4 f64, kr_gemm.cu): split-K over
 * the pixel dimension, tile partials summed in fixed order; a true Gram (A == B) computes
 * the lower tile blocks only and mirrors them.  work: kr_gram_workspace doubles. */
int64_t kr_gram_workspace(int32_t batch, int32_t rows, int64_t n);
int kr_gram(const double* A, const double* B, int64_t ld, int64_t bs, int32_t batch, int32_t rows, int64_t n,
            double* G, int64_t ldg, int64_t bsg, double* work, int64_t work_len, kr_stream_t stream);

/* Batched row-block product Y_b = alpha F_b X_b + beta Y_b with F_b (r2 x r1, row-major,
 * ldf, bsf) and X_b / Y_b rows of length L (ldx / ldy, bsx / bsy): the W <- R^-T A passes of
 * the Cholesky-QRs (recycling.py:194, 369), the basis recombinations U~ = W X, H U~ = (H W) X
 * (recycling.py:362-383) and Z = W V_H diag(mu).  lower != 0: F is lower triangular (the k
 * loop of a tile row stops at its diagonal block).  Same fp64 tensor-core kernel family. */
int kr_rows_mul(const double* F, int64_t ldf, int64_t bsf, const double* X, int64_t ldx, int64_t bsx, double* Y,
                int64_t ldy, int64_t bsy, int32_t r2, int32_t r1, int64_t L, int32_t batch, double alpha, double beta,
                int32_t lower, kr_stream_t stream);

/* Whole-batch recycle update (recycling.py:386-465 next_recycle for every sample of
 * the batch at once; outer or inner placement; RGen with size L -- rgen_select :316-359 +
 * gsvd_pair :275-313 -- Ritz -- ritz_select :226-236 -- or harmonic Ritz --
 * harmonic_ritz_select :239-272; prepare_recycle :362-383), orchestrated natively: candidate basis with the reference's pivoted-QR
 * rank drop, H W / J W, the projected pencil, the selected eigenpairs, the new
 * (U, C) and the NSC block Z = W V_H diag(mu).  `op` is the operator of the
 * upcoming system with op->batch == batch.  Host arrays are marked HOST, the rest
 * are DEVICE pointers.  status[b] = 0 done, 1 declined (the caller runs the
 * per-sample reference path for sample b: W^T H W numerically singular, or a
 * breakdown in the GSVD / prepare QR), 2 empty recycle space. */
typedef struct kr_recycle_args {
  int32_t batch, T, s;           /* samples; padded candidate count (<= 228); recycle dim */
  int32_t vec_type;              /* 0 = Ritz, 1 = RGen, 2 = harmonic Ritz */
  int32_t size_code, side;       /* size S/L/M = 0/1/2 (RGen: L only); side R/L/M = 0/1/2 */
  int32_t reuse_products;        /* H U~ = (H W) X_sel instead of s more H v */
  const double* V;               /* previous Lanczos bases: sample b, column j at V + b*bs_v + j*ld_v */
  int64_t ld_v, bs_v;
  const int32_t* kdims;          /* HOST [batch] basis columns */
  const double* Uprev;           /* previous U: sample b, column j at Uprev + b*bs_u + j*ld_u */
  int64_t ld_u, bs_u;
  const int32_t* sdims;          /* HOST [batch] previous recycle dims */
  double* W;                     /* out [batch][T][n] candidate basis rows (orthonormal) */
  double* HW;                    /* out [batch][T][n] H W */
  double* U;                     /* out [batch][s][n] */
  double* C;                     /* out [batch][s][n], C^T C = I */
  double* mu;                    /* out [batch][s] selected mu (RGen) */
  double* VH;                    /* out [batch][s][T] V_H columns as rows (RGen) */
  double* Z;                     /* out [batch][s][n] Z = W V_H diag(mu) rows (RGen) */
  int32_t* tdims;                /* HOST out [batch] candidates kept */
  int32_t* nsel;                 /* HOST out [batch] recycle dims */
  int32_t* status;               /* HOST out [batch] */
  const kr_op* op_proj;          /* HOST, nullable: inner placement (recycling.py:409-415) -- H W and J W
                                    use this operator (the previous system's H and J) while H U~ and
                                    C = H U R^-1 use `op` (the upcoming H); reuse_products is then
                                    ignored (H U~ is s fresh products with the upcoming H) */
} kr_recycle_args;

/* out[j] = (((rows[0][j] + rows[1][j]) + rows[2][j]) + ...), j < p: the sample-ordered sum of
 * per-sample hypergradients (rows: count x p, row stride ld), left to right as the
 * reference accumulates them (bilevel.py:439-446 over samples) -- one launch instead of
 * count - 1 vector adds.  Used after the cross-rank all-gather. */
int kr_ordered_sum(const double* rows, int32_t count, int32_t p, int64_t ld, double* out, kr_stream_t stream);

/* Creates this host thread's cuBLAS / cuSOLVER handles on the current device (both are
 * per thread and expensive on first use); optional, for callers that pin update work
 * to long-lived threads.  Host-side setup only, no reference counterpart. */
int kr_thread_warmup(void);

int64_t kr_recycle_workspace(const kr_op* op, const kr_recycle_args* args);
int kr_recycle_update(const kr_op* op, const kr_recycle_args* args, double* work, int64_t work_len,
                      kr_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* KRECYCLE_B200_H */
