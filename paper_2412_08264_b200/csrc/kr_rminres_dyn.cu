// kr_rminres_dyn.cu -- batched recycled MINRES as ONE persistent cooperative kernel whose
// blocks are shared by all still-running samples (the solve path when the Lanczos basis
// is kept, i.e. every recycled sequence solve).
//
// Algorithm: /root/reference/pkg/src/krecycle/krylov.py:205-383 (Alg. 3 with the
// corrected sign w += c_k zeta_{k-1}(vt - bt)), stop rules stopping.py:69-118, the
// residual recurrence krylov.py:154-181.  Differences from kr_rminres.cu's per-sample
// kernel:
//
//  * Work units are (sample, tile) pairs of the samples still iterating, dealt out to
//    ALL resident blocks every phase: when samples stop (NSC / tolerance / max_iter at
//    different k), their SMs move to the others instead of idling until the slowest
//    sample is done.  Two grid-wide barriers per iteration (A: stencil H v_k + the tile's
//    dot products; B: u = H v_k - C chv - alpha v_k - beta v_{k-1} and ||u||^2).
//  * Per-tile partial sums; the LAST block to finish a sample's tiles in a phase
//    (per-sample arrival counter) reduces them in fixed tile order and runs the sample's
//    scalar recurrences (Givens, stop tests, s-space recycle / NSC recurrences) once,
//    writing the sample's state for the next phase -- results are independent of how
//    units were dealt out (bitwise reproducible, batch-composition independent).
//  * No per-iteration solution / residual vectors: the iterate is w = w0 + U (t0 - Omega)
//    + V y with y = R^{-1} step from the recorded (gamma, delta, eps~, step) (R the upper
//    tri-banded matrix of the vt recurrence vt_k = (v_k - gamma vt_{k-2} - delta vt_{k-1})
//    / eps~, krylov.py:322-326), formed once at the end from the stored basis V; the
//    tracked residual (krylov.py:154-181, only when requested) likewise as
//    r = r0 - C (t0 - Omega) - HV y from the kept H v_k.  Exact in exact arithmetic.
//    This removes ~12 n-vector accesses per iteration (the vt / w / hvt / r updates).
//  * The stop decision of iteration k is taken right after it (end of phase B), so a
//    finished sample's blocks never run another stencil.

#include <cstring>
#include <string>

#include "kr_common.cuh"
#include "kr_internal.h"
#include "kr_solver.cuh"

namespace kr {
namespace dyn {

#ifdef KR_DYN_TIMING
// block 0's time by section of the unit loop (ns): 0 draw / wait for work, 1 stencil, 2 dots,
// 3 arrive + last-block reduction (A), 4 phase B unit, 5 finalisation, 6 publish; 7 = A units
__device__ unsigned long long g_dyn_ns[8];
#define KR_DMARK(i, last)                                         \
  do {                                                            \
    if (threadIdx.x == 0 && blockIdx.x == 0) {                    \
      unsigned long long t_;                                      \
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_));       \
      g_dyn_ns[i] += t_ - last;                                   \
      last = t_;                                                  \
    }                                                             \
  } while (0)
#else
#define KR_DMARK(i, last) ((void)0)
#endif

// M_RUN: next step is phase A (stencil + dots) of iteration k; M_RUNB: phase B of k;
// M_FIN: finalisation (w, r); M_WAIT: skips one super-phase (pipelining offset)
enum Mode : unsigned { M_DONE = 0, M_RUN = 1, M_FIN = 2, M_RUNB = 3, M_WAIT = 4, M_INIT = 0xff };

struct St {
  double beta;       // beta_k: v_k = tmp / beta_k
  double alpha;      // alpha_k (phase A)
  double c1, s1, c2, s2, zeta;
  double tol_bd;
  int k;             // current Lanczos index
  int iters, reason, pad;
};

// per-sample s-vectors (MAX_S == MAX_NSC doubles each)
enum { V_CHV = 0, V_CV, V_BTC1, V_BTC2, V_OMEGA, V_T0, V_ZRV, V_ZHA, V_ZHB, V_ZHV, V_TMO, NVEC };
static_assert(MAX_S == MAX_NSC, "vector slots share one stride");
constexpr int MAX_B = 512;

struct DParams {
  kr_op op;
  kr_solve_args a;
  int64_t n;
  int ntiles, nslot, G, B;
  double* tmp;                 // [B][n] u (unnormalised next Lanczos vector); setup: r0'
  double* hv;                  // [B][n], or [B][max_iter][n] when the residual is tracked
  double* r0;                  // [B][n] g - H w0 (w0 and tracked residual only)
  double* part;                // [B][nslot][ntiles]
  St* st;                      // [B]
  double* vecs;                // [B][NVEC][MAX_S]
  double* hist;                // [B][max_iter + 1][4]: gamma, delta, eps~, step of iteration k
  double* y;                   // [B][max_iter]
  unsigned long long* mode;    // [B]: (phase stamp << 32) | (mode before that phase << 8) | mode
  int* cnt;                    // [B] arrivals in the current phase
  unsigned int* bar;           // grid barrier counter
  unsigned int* grab;          // [2] unit tickets of the current / next super-phase
  int track;                   // residual vector requested (hv keeps every column)
  int vec2;                    // even image width and 16-byte aligned columns: pixel pairs as double2
  int pipe;                    // odd samples run one phase behind the even ones (A and B units overlap)
  int use_tma;                 // the stencil's halo region comes in one bulk tensor copy (tmap over tmp)
  int window;                  // samples iterating at a time (the first `window` unfinished ones)
  int dataflow;                // barrier-free schedule: per-sample phase tickets instead of grid barriers
  int group_b;                 // tiles per draw of a phase-B unit (dataflow schedule)
  int prio;                    // dataflow schedule: draw from the lowest unfinished sample first
  unsigned long long* tick;    // [B] kind << 56 | phase sequence << 32 | tiles dispensed in the current phase
  int* sched;                  // [2] head (first sample that may be unfinished), samples done
  CUtensorMap tmap;            // (cols, rows, 1, B) view of tmp
};

__device__ __forceinline__ double2 ld2cg(const double* p) { return __ldcg(reinterpret_cast<const double2*>(p)); }
__device__ __forceinline__ double2 ld2g(const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); }
__device__ __forceinline__ void st2(double* p, double2 v) { *reinterpret_cast<double2*>(p) = v; }

// The thread's pixel pair of a tile (vec2 mode): row threadIdx.x / 16, columns 2 (threadIdx.x % 16) + {0, 1}.
struct Pair {
  int l;       // tile-local index of the first pixel
  int64_t q;   // global pixel index of the first pixel (0 when outside)
  bool ok;
};
__device__ inline Pair tile_pair(const kr_op& op, int tile) {
  const int tyc = tiles_x(op);
  const int ty = threadIdx.x >> 4, tx = (threadIdx.x & 15) * 2;
  const int y = (tile / tyc) * TH + ty, x = (tile % tyc) * TW + tx;
  Pair r;
  r.l = ty * TW + tx;
  r.ok = y < op.rows && x < op.cols;  // cols even: x + 1 < cols as well
  r.q = r.ok ? (int64_t)y * op.cols + x : 0;
  return r;
}
static_assert(TPX == 2 * NT && TW == 32, "vec2 mode: one pixel pair per thread per tile");

__device__ inline double* vecp(const DParams& P, int b, int which) {
  return P.vecs + ((int64_t)b * NVEC + which) * MAX_S;
}
__device__ inline double* partp(const DParams& P, int b, int slot) {
  return P.part + ((int64_t)b * P.nslot + slot) * P.ntiles;
}
__device__ inline double* hvcol(const DParams& P, int b, int k) {  // H v_k
  return P.track ? P.hv + ((int64_t)b * P.a.max_iter + (k - 1)) * P.n : P.hv + (int64_t)b * P.n;
}
__device__ inline double* vcol(const DParams& P, int b, int k) {  // v_k, basis column k-1
  return P.a.basis + (int64_t)b * P.a.bs_basis + (int64_t)(k - 1) * P.a.ld_basis;
}

// mode of sample b as of the START of phase ph (a change made during ph is stamped ph)
__device__ inline unsigned mode_at(const DParams& P, int b, unsigned ph) {
  const unsigned long long m = *reinterpret_cast<volatile unsigned long long*>(P.mode + b);
  return (unsigned)(m >> 32) == ph ? (unsigned)((m >> 8) & 0xff) : (unsigned)(m & 0xff);
}
__device__ inline void mode_set(const DParams& P, int b, unsigned ph, unsigned prev, unsigned cur) {
  *reinterpret_cast<volatile unsigned long long*>(P.mode + b) =
      ((unsigned long long)ph << 32) | ((unsigned long long)prev << 8) | cur;
}

// Ordered list of the samples whose mode (at the start of phase ph) is in `want` (bit
// mask of modes); identical in every block.
__device__ inline int build_list(const DParams& P, unsigned ph, unsigned want, int* list, int* wsum) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int total = 0;
  for (int b0 = 0; b0 < P.B; b0 += NT) {
    const int b = b0 + threadIdx.x;
    const bool f = b < P.B && ((want >> mode_at(P, b, ph)) & 1u);
    const unsigned m = __ballot_sync(0xffffffffu, f);
    if (lane == 0) wsum[warp] = __popc(m);
    block_barrier();
    int off = total;
    for (int w = 0; w < warp; ++w) off += wsum[w];
    if (f) list[off + __popc(m & ((1u << lane) - 1u))] = b;
    for (int w = 0; w < NWARP; ++w) total += wsum[w];
    block_barrier();
  }
  return total;
}

// Unit done: true in exactly one block per (sample, phase) -- the last to arrive.
__device__ inline bool arrive(const DParams& P, int b, int* flag) {
  __threadfence();
  block_barrier();
  if (threadIdx.x == 0) {
    const int prev = atomicAdd(P.cnt + b, 1);
    *flag = (prev == P.ntiles - 1);
    if (*flag) {
      atomicExch(P.cnt + b, 0);
      __threadfence();
    }
  }
  block_barrier();
  return *flag != 0;
}

// out[i] = sum over tiles (fixed order: lane-strided, fixed shuffle tree) of slot slot0+i
__device__ inline void reduce_tiles(const DParams& P, int b, int slot0, int S, double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int INF = 4;
  for (int i0 = warp; i0 < S; i0 += INF * NWARP) {
    double acc[INF];
#pragma unroll
    for (int u = 0; u < INF; ++u) {
      const int i = i0 + u * NWARP;
      double s = 0.0;
      if (i < S) {
        const double* src = partp(P, b, slot0 + i);
        for (int t = lane; t < P.ntiles; t += 32) s += __ldcg(src + t);
      }
      acc[u] = s;
    }
#pragma unroll
    for (int u = 0; u < INF; ++u) {
      const double v = warp_sum(acc[u]);
      const int i = i0 + u * NWARP;
      if (lane == 0 && i < S) out[i] = v;
    }
  }
  block_barrier();
}

// Per-tile dot products of up to 8 matrix columns per pass with a tile vector x:
// part[slot0 + i][tile] = sum_{p in tile} A_i[p] x(p), i < S.
template <typename XF>
__device__ inline void tile_mdots(const DParams& P, int b, int tile, const double* A, int64_t lda, int S, int slot0,
                                  XF xf, double* red) {
  for (int base = 0; base < S; base += 8) {
    double v8[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v8[i] = 0.0;
    for (int l = threadIdx.x; l < TPX; l += NT) {
      const int64_t p = tile_pixel(P.op, tile, l);
      if (p < 0) continue;
      const double x = xf(l, p);
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (base + i < S) v8[i] += A[(int64_t)(base + i) * lda + p] * x;
    }
    block_sum<8>(v8, red);
    if (threadIdx.x < 8 && base + threadIdx.x < S) partp(P, b, slot0 + base + threadIdx.x)[tile] = red[threadIdx.x];
    block_barrier();
  }
}

// y = R^{-1} step over iterations 1..K (backward tri-banded substitution, carries for
// the two trailing indices); staged through `scratch` (>= 4 * CH doubles) in chunks.
__device__ inline void solve_y(const DParams& P, int b, int K, double* scratch, int CH) {
  const double* H = P.hist + (int64_t)b * (P.a.max_iter + 1) * 4;
  double* Y = P.y + (int64_t)b * P.a.max_iter;
  __shared__ double car[2];
  if (threadIdx.x == 0) car[0] = car[1] = 0.0;
  for (int hi = K; hi >= 1; hi -= CH) {
    const int lo = hi - CH + 1 > 1 ? hi - CH + 1 : 1;  // indices lo..hi
    const int m = hi - lo + 1;
    block_barrier();
    for (int i = threadIdx.x; i < 4 * m; i += NT) scratch[i] = __ldcg(H + 4 * lo + i);
    block_barrier();
    if (threadIdx.x == 0) {
      double a1 = car[0], a2 = car[1];
      for (int j = hi; j >= lo; --j) {
        const double* h = scratch + 4 * (j - lo);  // gamma, delta, eps~, step
        const double yj = (h[3] + a1) / h[2];
        const double n1 = a2 - h[1] * yj;
        a2 = -h[0] * yj;
        a1 = n1;
        scratch[4 * m + (j - lo)] = yj;
      }
      car[0] = a1;
      car[1] = a2;
    }
    block_barrier();
    for (int i = threadIdx.x; i < m; i += NT) Y[lo - 1 + i] = scratch[4 * m + i];
  }
  block_barrier();
}

#define DYN_GRID_SYNC() grid_barrier(P.bar, (unsigned)P.G, grid_target)

// Barrier-free schedule: every sample carries a ticket word
//   [63:56] kind of its current phase (M_RUN / M_RUNB / M_FIN / M_DONE)
//   [55:32] phase sequence number     [31:0] tiles dispensed in this phase.
// A block draws tiles of the current phase of one of the first `window` unfinished samples
// (a group of `group_b` tiles for the short streaming phase B, one tile otherwise); the block
// that completes a phase (last arrival) does the sample's reduction and scalar step and then
// publishes the next phase's word.  No block ever waits for another except by looking for
// work, so samples drift apart and one sample's serial tail (reduction, scalar recurrences)
// overlaps the others' tiles.  Warp 0 collectively: the 32 lanes look at the 32 samples from
// the head in one round trip, one lane draws.  Returns false when every sample is done.
__device__ __forceinline__ unsigned long long tick_word(unsigned kind, unsigned seq, unsigned lo) {
  return ((unsigned long long)kind << 56) | ((unsigned long long)(seq & 0xffffffu) << 32) | lo;
}
constexpr unsigned TICK_DONE_LO = 0x7fffffffu;
__device__ __noinline__ bool grab_unit(const DParams& P, int* b_out, int* tile_out, int* cnt_out, unsigned* md_out,
                                       unsigned* seq_out) {
  const int lane = threadIdx.x & 31;
  unsigned spin = 0;
  for (;;) {
    const int done = *reinterpret_cast<volatile int*>(P.sched + 1);
    const int head = *reinterpret_cast<volatile int*>(P.sched);
    if (done >= P.B) return false;
    const int bb = head + lane;
    const unsigned long long w = bb < P.B ? *reinterpret_cast<volatile unsigned long long*>(P.tick + bb)
                                          : tick_word(M_DONE, 0, TICK_DONE_LO);
    const unsigned kind = (unsigned)(w >> 56), lo = (unsigned)w;
    const bool fin = kind == M_DONE;
    const unsigned fm = __ballot_sync(0xffffffffu, fin);
    const int lead = fm == 0xffffffffu ? 32 : __ffs(~fm) - 1;  // leading finished samples: the head moves on
    if (lane == 0 && lead > 0) atomicMax(P.sched, head + lead < P.B ? head + lead : P.B);
    const int rank = __popc(~fm & ((1u << lane) - 1u));        // unfinished samples before this one
    const bool avail = !fin && rank < P.window && lo < (unsigned)P.ntiles;
    const unsigned am = __ballot_sync(0xffffffffu, avail);
    if (am == 0) {
      if (!(fm == 0xffffffffu && head + 32 < P.B)) __nanosleep(64);
      ++spin;
      continue;
    }
    // prio: lowest unfinished sample first (depth-first: the few leading samples get every
    // block they can use and stay L2-resident, the rest of the window takes the overflow);
    // otherwise a block-dependent start spreads the blocks over the window
    const int start = P.prio ? 0 : (int)((blockIdx.x + spin) & 31u);
    const unsigned rot = start ? ((am >> start) | (am << (32 - start))) : am;
    const int pick = (__ffs(rot) - 1 + start) & 31;
    unsigned long long old = 0;
    int G = 1;
    if (lane == pick) {
      G = kind == M_RUNB ? P.group_b : 1;
      old = atomicAdd(P.tick + bb, (unsigned long long)G);
    }
    old = __shfl_sync(0xffffffffu, old, pick);
    G = __shfl_sync(0xffffffffu, G, pick);
    const unsigned okind = (unsigned)(old >> 56), olo = (unsigned)old;
    if (okind != M_DONE && olo < (unsigned)P.ntiles) {
      __threadfence();
      *b_out = head + pick;
      *tile_out = (int)olo;
      *cnt_out = (int)olo + G <= P.ntiles ? G : P.ntiles - (int)olo;
      *md_out = okind;
      *seq_out = (unsigned)(old >> 32) & 0xffffffu;
      return true;
    }
    ++spin;
  }
}

template <int Q>
__global__ void __launch_bounds__(NT, 2) rminres_dyn_kernel(const __grid_constant__ DParams P) {
  unsigned int grid_target = 0;
  extern __shared__ __align__(128) double smem[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t mphase;
  const kr_op& op = P.op;
  const kr_solve_args& A = P.a;
  const Geom g = make_geom(op);
  Smem sm = carve(g, smem);
  double* slot = smem + g.total;      // MAX_SLOTS (reductions of the last block)
  double* sv = slot + MAX_SLOTS;      // MAX_S (per-unit s-vector: chv / tmo)
  double* red = sv + MAX_S;           // RED_DOUBLES
  __shared__ int list[MAX_B];
  __shared__ int wsum[NWARP];
  __shared__ int s_flag;
  __shared__ int s_unit;
  __shared__ int s_b, s_tile, s_cnt;   // dataflow schedule: the drawn unit
  __shared__ unsigned s_md, s_seq, s_pub;
  __shared__ double sc[8];
  const int64_t n = P.n;
  const int s = A.s, ns = A.stop_kind >= 1 ? A.nsc_s : 0;
  const int nt = P.ntiles, G = P.G;
  const int SL_CHV = 0, SL_CV = s, SL_VHV = 2 * s, SL_ZHV = 2 * s + 1;
  const int CH = (g.s0 + g.sa) / 5;  // solve_y / finalize staging chunk (entries)
  if (P.use_tma) tma_mbar_init(&mbar, &mphase);
  load_weights(op, g, sm);
  unsigned ph = 0;

  // ---------------- S0: r0 = g - H w0; partials C^T r0 (slots 0..s), ||g||^2 (slot s) ----------------
  for (int u = blockIdx.x; u < P.B * nt; u += G) {
    const int b = u / nt, tile = u - b * nt;
    const double* gb = A.g + (int64_t)b * n;
    const double* C = s ? A.C + (int64_t)b * A.bs_uc : nullptr;
    const double* r0src = gb;
    if (A.w0) {
      tile_hvp_t<Q>(op, g, sm, b, TileIn{A.w0 + (int64_t)b * n, 1.0, nullptr, 0.0}, tile);
      double* tb = P.tmp + (int64_t)b * n;
      for (int l = threadIdx.x; l < TPX; l += NT) {
        const int64_t p = tile_pixel(op, tile, l);
        if (p < 0) continue;
        const double r = gb[p] - sm.res[l];
        tb[p] = r;
        if (P.track) P.r0[(int64_t)b * n + p] = r;
      }
      block_barrier();
      r0src = tb;
    }
    if (s) tile_mdots(P, b, tile, C, A.ld_uc, s, 0, [&](int, int64_t p) { return r0src[p]; }, red);
    {
      double v[1] = {0.0};
      for (int l = threadIdx.x; l < TPX; l += NT) {
        const int64_t p = tile_pixel(op, tile, l);
        if (p >= 0) v[0] += gb[p] * gb[p];
      }
      block_sum<1>(v, red);
      if (threadIdx.x == 0) partp(P, b, s)[tile] = red[0];
    }
    if (arrive(P, b, &s_flag)) {
      reduce_tiles(P, b, 0, s + 1, slot);
      double* t0 = vecp(P, b, V_T0);
      for (int i = threadIdx.x; i < s; i += NT) t0[i] = slot[i];
      if (threadIdx.x == 0) {
        const double gn = sqrt(slot[s]);
        P.st[b].tol_bd = BREAKDOWN_RTOL * (gn > 1e-300 ? gn : 1e-300);
      }
    }
    block_barrier();
  }
  DYN_GRID_SYNC();
  ++ph;

  // ---------------- S1: r0' = r0 - C t0; partials ||r0'||^2 (slot 0), Z^T r0' (1..ns) ----------------
  for (int u = blockIdx.x; u < P.B * nt; u += G) {
    const int b = u / nt, tile = u - b * nt;
    const double* gb = A.g + (int64_t)b * n;
    const double* C = s ? A.C + (int64_t)b * A.bs_uc : nullptr;
    double* tb = P.tmp + (int64_t)b * n;
    const double* r0src = A.w0 ? tb : gb;
    for (int i = threadIdx.x; i < s; i += NT) sv[i] = __ldcg(vecp(P, b, V_T0) + i);
    block_barrier();
    double v[1] = {0.0};
    for (int l = threadIdx.x; l < TPX; l += NT) {
      const int64_t p = tile_pixel(op, tile, l);
      if (p < 0) continue;
      double r = r0src[p];
      if (s) {
        double ct = 0.0;
        for (int i = 0; i < s; ++i) ct += C[(int64_t)i * A.ld_uc + p] * sv[i];
        r = r - ct;
      }
      tb[p] = r;
      v[0] += r * r;
    }
    block_sum<1>(v, red);
    if (threadIdx.x == 0) partp(P, b, 0)[tile] = red[0];
    block_barrier();
    if (ns && A.stop_kind == 1) {
      const double* Z = A.Z + (int64_t)b * A.bs_z;
      tile_mdots(P, b, tile, Z, A.ld_z, ns, 1, [&](int, int64_t p) { return tb[p]; }, red);
    }
    if (arrive(P, b, &s_flag)) {
      reduce_tiles(P, b, 0, A.stop_kind == 1 ? 1 + ns : 1, slot);
      double* zrv = vecp(P, b, V_ZRV);
      if (A.stop_kind == 2) {
        // G r0' = J H^-1 (g - H w0 - C t0) = (J w* - J w0) - (J U) t0
        const double* t0 = vecp(P, b, V_T0);
        const double* ZtC = s ? A.ZtC + (int64_t)b * ns * s : nullptr;
        for (int i = threadIdx.x; i < ns; i += NT) {
          double z = A.nsc_r0[(int64_t)b * ns + i];
          for (int l = 0; l < s; ++l) z -= ZtC[(int64_t)i * s + l] * t0[l];
          zrv[i] = z;
          slot[1 + i] = z;
        }
        block_barrier();
      } else {
        for (int i = threadIdx.x; i < ns; i += NT) zrv[i] = slot[1 + i];
      }
      if (threadIdx.x == 0) {
        St& S = P.st[b];
        const double beta = sqrt(slot[0]);
        const bool broke = beta <= S.tol_bd;
        S.beta = beta;
        S.zeta = beta;
        S.c1 = 1.0; S.s1 = 0.0; S.c2 = 0.0; S.s2 = 0.0;
        S.alpha = 0.0;
        double val = beta;
        if (ns) {  // nsc_value of r0' (Omega = 0)
          double ss = 0.0;
          for (int i = 0; i < ns; ++i) ss += slot[1 + i] * slot[1 + i];
          val = sqrt(ss);
        }
        A.res_norms[(int64_t)b * (A.max_iter + 1)] = beta;
        A.stop_vals[(int64_t)b * (A.max_iter + 1)] = val;
        unsigned m = M_RUN;
        if (val < A.delta) { S.iters = 0; S.reason = R_TOL; m = M_FIN; }
        else if (broke) { S.iters = 0; S.reason = R_BREAK; m = M_FIN; }
        if (m == M_RUN && P.pipe && (b & 1)) m = M_WAIT;
        S.k = 1;
        mode_set(P, b, ph, M_INIT, m);
        if (P.dataflow) P.tick[b] = tick_word(m, 1, 0);
      }
      block_barrier();
      // t0 - Omega (Omega = 0) for a sample that finishes here
      const double* t0 = vecp(P, b, V_T0);
      double* tmo = vecp(P, b, V_TMO);
      for (int i = threadIdx.x; i < s; i += NT) tmo[i] = t0[i];
    }
    block_barrier();
  }
  DYN_GRID_SYNC();
  ++ph;

  // ---------------- iterations ----------------
  const int npass = (s > ns ? s : ns) > 0 ? ((s > ns ? s : ns) + 7) / 8 : 1;
  const bool deferred = npass <= DEF_PASSES;
  // true hypergradient error: the "Z" rows are J's and the per-iteration dots are J v_k
  // (= J H^-1 H v_k, the G hv_k of the residual recurrence applied to G = J H^-1)
  const bool zhv_on_v = A.stop_kind == 2;
  for (;;) {
    // One super-phase: every sample with work takes its next step -- phase A (M_RUN: stencil
    // + dots of v_k), phase B (M_RUNB: u, ||u||^2, finish iteration k) or the finalisation
    // (M_FIN: w and r from the stored basis).  Without pipelining all samples are in step
    // (A, B, A, ...); with it the odd samples run one phase behind, so every super-phase
    // mixes compute-heavy A units with streaming B units on the same SMs.
    // Sample window: only the first `window` unfinished samples iterate; a finished sample's
    // place goes to the next one.  Their recycle blocks C and Z (read every iteration) then
    // stay L2-resident from one iteration to the next instead of streaming from HBM for the
    // whole batch; per-sample arithmetic does not depend on the window (bitwise the same).
    int na = 0;
    if (!P.dataflow) {
      na = build_list(P, ph, (1u << M_RUN) | (1u << M_FIN) | (1u << M_RUNB), list, wsum);
      if (na > P.window) na = P.window;
      if (na == 0) break;  // identical in every block (M_WAIT only ever coexists with M_RUN samples)
      if (blockIdx.x == 0)
        for (int b = threadIdx.x; b < P.B; b += NT)
          if (mode_at(P, b, ph) == M_WAIT) mode_set(P, b, ph, M_WAIT, M_RUN);
    }
    // units are taken from a ticket counter (the next ticket requested while the current
    // unit runs): blocks that drew heavy units take fewer -- the super-phase ends when the
    // work does, not when the unluckiest block's fixed share does.  Unit u is tile u / na
    // of list sample u % na (samples interleaved: A and B units mix on every SM, and
    // neighbouring tiles of a sample run concurrently for the halo's L2 reuse).
    unsigned int* tickets = P.grab + (ph & 1);
    if (!P.dataflow) {
      if (blockIdx.x == 0 && threadIdx.x == 0) atomicExch(P.grab + ((ph + 1) & 1), 0u);
      if (threadIdx.x == 0) s_unit = (int)atomicAdd(tickets, 1u);
      block_barrier();
    }
#ifdef KR_DYN_TIMING
    unsigned long long dlast = 0;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(dlast));
#endif
    for (;;) {
      unsigned int next_ticket = 0;
      int b, tile0, tcount = 1;
      unsigned md;
      if (P.dataflow) {
        if (threadIdx.x < 32) {
          int gb = -1, gt = 0, gc = 1;
          unsigned gm = 0, gs = 0;
          if (!grab_unit(P, &gb, &gt, &gc, &gm, &gs)) gb = -1;
          if (threadIdx.x == 0) {
            s_b = gb;
            s_tile = gt;
            s_cnt = gc;
            s_md = gm;
            s_seq = gs;
            s_pub = 0xffu;
          }
        }
        block_barrier();
        if (s_b < 0) break;
        b = s_b;
        tile0 = s_tile;
        tcount = s_cnt;
        md = s_md;
      } else {
        const int u = s_unit;
        if (u >= na * nt) break;
        if (threadIdx.x == 0) next_ticket = atomicAdd(tickets, 1u);
        b = list[u % na];
        tile0 = u / na;
        md = mode_at(P, b, ph);
      }
      KR_DMARK(0, dlast);
      for (int tile = tile0; tile < tile0 + tcount; ++tile) {
      if (md == M_RUN) {
        const double beta = __ldcg(&P.st[b].beta);
        const int k = *reinterpret_cast<volatile int*>(&P.st[b].k);
        const double* tb = P.tmp + (int64_t)b * n;
        const double* C = s ? A.C + (int64_t)b * A.bs_uc : nullptr;
        const double* Z = ns ? A.Z + (int64_t)b * A.bs_z : nullptr;
        double* hvk = hvcol(P, b, k);
        double* vk = vcol(P, b, k);
        const TmaSrc tsrc{&P.tmap, 0, b, beta, &mbar, &mphase};
        tile_hvp_t<Q>(op, g, sm, b, TileIn{tb, beta, nullptr, 0.0}, tile, P.use_tma ? &tsrc : nullptr);
        KR_DMARK(1, dlast);
        if (P.use_tma && !P.dataflow && threadIdx.x == 0 && next_ticket < (unsigned)(na * nt)) {
          // the next unit's halo region into L2 while this unit's dots run (its bulk copy then
          // hits L2; a finalisation unit's region is only a wasted prefetch)
          const int nb = list[next_ticket % na], ntl = next_ticket / na, tyc = tiles_x(op);
          asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global [%0, {%1, %2, %3, %4}];" ::"l"(&P.tmap),
                       "r"((ntl % tyc) * TW - g.H), "r"((ntl / tyc) * TH - g.H), "r"(0), "r"(nb)
                       : "memory");
        }
        if (deferred) {
          for (int i = threadIdx.x; i < npass * 25 * DEF_STRIDE; i += NT) red[i] = 0.0;
          block_barrier();
        }
        if (P.vec2) {
          // one pixel pair per thread: H v_k and v_k written as double2, C / Z read as double2,
          // 8 + 8 column pairs in flight per pass
          const Pair pr = tile_pair(op, tile);
          const int c0 = (pr.l / TW + g.H) * g.RW + (pr.l % TW) + g.H;
          double2 h2 = make_double2(sm.res[pr.l], sm.res[pr.l + 1]);
          double2 v2 = make_double2(sm.S0[c0], sm.S0[c0 + 1]);
          if (pr.ok) {
            st2(hvk + pr.q, h2);
            st2(vk + pr.q, v2);
          } else {
            h2 = v2 = make_double2(0.0, 0.0);
          }
          for (int base = 0; base < 8 * npass; base += 8) {
            double2 cc[8], zz[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              cc[i] = (pr.ok && base + i < s) ? ld2g(C + (int64_t)(base + i) * A.ld_uc + pr.q) : make_double2(0.0, 0.0);
              zz[i] = (pr.ok && base + i < ns) ? ld2g(Z + (int64_t)(base + i) * A.ld_z + pr.q) : make_double2(0.0, 0.0);
            }
            double v25[25];
            v25[24] = base == 0 ? v2.x * h2.x + v2.y * h2.y : 0.0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              v25[i] = cc[i].x * h2.x + cc[i].y * h2.y;
              v25[8 + i] = cc[i].x * v2.x + cc[i].y * v2.y;
              v25[16 + i] = zhv_on_v ? zz[i].x * v2.x + zz[i].y * v2.y : zz[i].x * h2.x + zz[i].y * h2.y;
            }
            if (deferred) {
              def_add<25>(MultiSum<25>::reduce(v25, threadIdx.x & 31), base / 8, red);
              continue;
            }
            block_sum<25>(v25, red);
            if (threadIdx.x < 8 && base + threadIdx.x < s) {
              partp(P, b, SL_CHV + base + threadIdx.x)[tile] = red[threadIdx.x];
              partp(P, b, SL_CV + base + threadIdx.x)[tile] = red[8 + threadIdx.x];
            }
            if (threadIdx.x < 8 && base + threadIdx.x < ns) partp(P, b, SL_ZHV + base + threadIdx.x)[tile] = red[16 + threadIdx.x];
            if (threadIdx.x == 0 && base == 0) partp(P, b, SL_VHV)[tile] = red[24];
            block_barrier();
          }
        } else {
        for (int l = threadIdx.x; l < TPX; l += NT) {
          const int64_t p = tile_pixel(op, tile, l);
          if (p < 0) continue;
          hvk[p] = sm.res[l];
          if (op.data_kind == KR_DATA_DENSE) {
            vk[p] = tb[p] / beta;
          } else {
            const int ty = l / TW, tx = l - ty * TW;
            vk[p] = sm.S0[(ty + g.H) * g.RW + tx + g.H];
          }
        }
        // tile partials: C^T hv, C^T v, v.hv, Z^T hv -- 8 columns per pass, 2 pixels per thread
        for (int base = 0; base < 8 * npass; base += 8) {
          double v25[25];
#pragma unroll
          for (int i = 0; i < 25; ++i) v25[i] = 0.0;
          int64_t pp[2];
          double hh[2], vv[2], cc[2][8], zz[2][8];
#pragma unroll
          for (int uu = 0; uu < 2; ++uu) {
            const int l = threadIdx.x + uu * NT;
            pp[uu] = tile_pixel(op, tile, l);
            const int64_t q = pp[uu] >= 0 ? pp[uu] : 0;
            hh[uu] = sm.res[l];
            if (op.data_kind == KR_DATA_DENSE) {
              vv[uu] = pp[uu] >= 0 ? tb[q] / beta : 0.0;
            } else {
              const int ty = l / TW, tx = l - ty * TW;
              vv[uu] = sm.S0[(ty + g.H) * g.RW + tx + g.H];
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              cc[uu][i] = (pp[uu] >= 0 && base + i < s) ? C[(int64_t)(base + i) * A.ld_uc + q] : 0.0;
              zz[uu][i] = (pp[uu] >= 0 && base + i < ns) ? Z[(int64_t)(base + i) * A.ld_z + q] : 0.0;
            }
          }
#pragma unroll
          for (int uu = 0; uu < 2; ++uu) {
            if (pp[uu] < 0) continue;
            const double h = hh[uu], v = vv[uu];
            if (base == 0) v25[24] += v * h;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              v25[i] += cc[uu][i] * h;
              v25[8 + i] += cc[uu][i] * v;
              v25[16 + i] += zz[uu][i] * (zhv_on_v ? v : h);
            }
          }
          if (deferred) {
            def_add<25>(MultiSum<25>::reduce(v25, threadIdx.x & 31), base / 8, red);
            continue;
          }
          block_sum<25>(v25, red);
          if (threadIdx.x < 8 && base + threadIdx.x < s) {
            partp(P, b, SL_CHV + base + threadIdx.x)[tile] = red[threadIdx.x];
            partp(P, b, SL_CV + base + threadIdx.x)[tile] = red[8 + threadIdx.x];
          }
          if (threadIdx.x < 8 && base + threadIdx.x < ns) partp(P, b, SL_ZHV + base + threadIdx.x)[tile] = red[16 + threadIdx.x];
          if (threadIdx.x == 0 && base == 0) partp(P, b, SL_VHV)[tile] = red[24];
          block_barrier();
        }
        }
        if (deferred) {
          block_barrier();
          for (int c = threadIdx.x; c < s; c += NT) {
            partp(P, b, SL_CHV + c)[tile] = def_sum(red, (c / 8) * 25 + c % 8);
            partp(P, b, SL_CV + c)[tile] = def_sum(red, (c / 8) * 25 + 8 + c % 8);
          }
          for (int c = threadIdx.x; c < ns; c += NT) partp(P, b, SL_ZHV + c)[tile] = def_sum(red, (c / 8) * 25 + 16 + c % 8);
          if (threadIdx.x == 0) partp(P, b, SL_VHV)[tile] = def_sum(red, 24);
        }
        KR_DMARK(2, dlast);
        if (arrive(P, b, &s_flag)) {
          reduce_tiles(P, b, 0, 2 * s + 1 + ns, slot);
          double* chv = vecp(P, b, V_CHV);
          double* cv = vecp(P, b, V_CV);
          double* zhv = vecp(P, b, V_ZHV);
          for (int i = threadIdx.x; i < s; i += NT) {
            chv[i] = slot[SL_CHV + i];
            cv[i] = slot[SL_CV + i];
          }
          for (int i = threadIdx.x; i < ns; i += NT) zhv[i] = slot[SL_ZHV + i];
          if (threadIdx.x == 0) {  // alpha = v.hv - (C^T v).(C^T hv)  (== v.(hv - C chv), krylov.py:269-283)
            double corr = 0.0;
            for (int i = 0; i < s; ++i) corr += slot[SL_CV + i] * slot[SL_CHV + i];
            P.st[b].alpha = slot[SL_VHV] - corr;
            mode_set(P, b, ph, M_RUN, M_RUNB);
            s_pub = M_RUNB;
          }
        }
        block_barrier();
        KR_DMARK(3, dlast);
#ifdef KR_DYN_TIMING
        if (threadIdx.x == 0 && blockIdx.x == 0) g_dyn_ns[7] += 1;
#endif
      } else if (md == M_RUNB) {
        // ===== phase B: u = hv_k - C chv - alpha v_k - beta_k v_{k-1}, ||u||^2; then finish iteration k =====
      St* S = P.st + b;
      const int k = *reinterpret_cast<volatile int*>(&S->k);
      const double al = __ldcg(&S->alpha), be = __ldcg(&S->beta);
      const double* C = s ? A.C + (int64_t)b * A.bs_uc : nullptr;
      for (int i = threadIdx.x; i < s; i += NT) sv[i] = __ldcg(vecp(P, b, V_CHV) + i);
      block_barrier();
      const double* vk = vcol(P, b, k);
      const double* vkm = k > 1 ? vcol(P, b, k - 1) : nullptr;
      const double* hvk = hvcol(P, b, k);
      double* tb = P.tmp + (int64_t)b * n;
      double bsq[1] = {0.0};
      if (P.vec2) {
        // one pixel pair per thread, every load of the pass issued before the first use
        const Pair pr = tile_pair(op, tile);
        if (pr.ok) {
          const double2 h2 = ld2cg(hvk + pr.q), v2 = ld2cg(vk + pr.q);
          const double2 m2 = vkm ? ld2cg(vkm + pr.q) : make_double2(0.0, 0.0);
          double ccx = 0.0, ccy = 0.0;
          for (int i0 = 0; i0 < s; i0 += 16) {
            double2 c16[16];
#pragma unroll
            for (int i = 0; i < 16; ++i)
              c16[i] = (i0 + i < s) ? ld2g(C + (int64_t)(i0 + i) * A.ld_uc + pr.q) : make_double2(0.0, 0.0);
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (i0 + i < s) {
                ccx += c16[i].x * sv[i0 + i];
                ccy += c16[i].y * sv[i0 + i];
              }
          }
          double2 x;
          x.x = ((h2.x - ccx) - al * v2.x) - be * m2.x;  // vnext = hv - C chv - alpha v - beta v_prev
          x.y = ((h2.y - ccy) - al * v2.y) - be * m2.y;
          st2(tb + pr.q, x);
          bsq[0] = x.x * x.x + x.y * x.y;
        }
      } else
      for (int l = threadIdx.x; l < TPX; l += NT) {
        const int64_t p = tile_pixel(op, tile, l);
        if (p < 0) continue;
        double x = hvk[p];
        if (s) {
          double cc = 0.0;
          for (int i0 = 0; i0 < s; i0 += 8) {
            double c8[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) c8[i] = (i0 + i < s) ? C[(int64_t)(i0 + i) * A.ld_uc + p] : 0.0;
#pragma unroll
            for (int i = 0; i < 8; ++i)
              if (i0 + i < s) cc += c8[i] * sv[i0 + i];
          }
          x = x - cc;  // vnext = hv - C chv
        }
        x = x - al * vk[p];                     // vnext -= alpha v
        x = x - be * (vkm ? vkm[p] : 0.0);      // vnext -= beta v_prev
        tb[p] = x;
        bsq[0] += x * x;
      }
      block_sum<1>(bsq, red);
      if (threadIdx.x == 0) partp(P, b, 0)[tile] = red[0];
      if (arrive(P, b, &s_flag)) {
        reduce_tiles(P, b, 0, 1, slot);
        // finish iteration k (krylov.py:298-381) -- scalars on thread 0
        if (threadIdx.x == 0) {
          const double bnew = sqrt(slot[0]);
          const bool broke = bnew <= S->tol_bd;
          const double bp = S->beta, a0 = S->alpha;
          const double gamma = S->s2 * bp;
          const double delta = S->c1 * S->c2 * bp + S->s1 * a0;
          const double eps = -S->s1 * S->c2 * bp + S->c1 * a0;
          const double eps_r = hypot(eps, bnew);
          sc[5] = broke ? 1.0 : 0.0;
          if (eps_r == 0.0) {
            sc[4] = -1.0;  // breakdown before the update: k - 1 iterations
          } else {
            const double s_new = bnew / eps_r, c_new = eps / eps_r;
            const double zeta_prev = S->zeta;
            S->zeta = -s_new * zeta_prev;
            const double step = c_new * zeta_prev;
            double* h = P.hist + ((int64_t)b * (A.max_iter + 1) + k) * 4;
            h[0] = gamma; h[1] = delta; h[2] = eps_r; h[3] = step;
            S->c2 = S->c1; S->s2 = S->s1; S->c1 = c_new; S->s1 = s_new;
            S->beta = bnew;
            sc[0] = gamma; sc[1] = delta; sc[2] = eps_r; sc[3] = step; sc[4] = 1.0;
            A.res_norms[(int64_t)b * (A.max_iter + 1) + k] = fabs(S->zeta);
          }
        }
        block_barrier();
        const bool upd = sc[4] > 0.0;
        if (upd) {
          const double ga = sc[0], de = sc[1], er = sc[2], st = sc[3];
          double* chv = vecp(P, b, V_CHV);
          double* b1 = vecp(P, b, V_BTC1);
          double* b2 = vecp(P, b, V_BTC2);
          double* om = vecp(P, b, V_OMEGA);
          for (int i = threadIdx.x; i < s; i += NT) {  // b~ recurrence in s-space
            const double bt = (chv[i] - ga * b2[i] - de * b1[i]) / er;
            om[i] += st * bt;
            b2[i] = b1[i];
            b1[i] = bt;
          }
          double* zrv = vecp(P, b, V_ZRV);
          double* zA = vecp(P, b, V_ZHA);
          double* zB = vecp(P, b, V_ZHB);
          const double* zhv = vecp(P, b, V_ZHV);
          for (int i = threadIdx.x; i < ns; i += NT) {  // Z^T of the tracked-residual recurrence
            const double zn = (zhv[i] - de * zA[i] - ga * zB[i]) / er;
            zrv[i] -= st * zn;
            zB[i] = zA[i];
            zA[i] = zn;
          }
          block_barrier();
          if (ns) {  // nsc_value (stopping.py:69-72): || Z^T r_v + (Z^T C) Omega ||
            const double* ZtC = s ? A.ZtC + (int64_t)b * ns * s : nullptr;
            for (int i = threadIdx.x; i < ns; i += NT) {
              double z = zrv[i];
              if (ZtC) {
                double c0 = 0.0, c1 = 0.0;
                int l = 0;
                for (; l + 1 < s; l += 2) {
                  c0 += ZtC[(int64_t)i * s + l] * om[l];
                  c1 += ZtC[(int64_t)i * s + l + 1] * om[l + 1];
                }
                if (l < s) c0 += ZtC[(int64_t)i * s + l] * om[l];
                z += c0 + c1;
              }
              slot[i] = z * z;
            }
            block_barrier();
          }
        }
        if (threadIdx.x == 0) {
          unsigned m = M_RUN;
          if (!upd) {
            S->iters = k - 1;
            S->reason = R_BREAK;
            m = M_FIN;
          } else {
            double val = fabs(S->zeta);
            if (ns) {
              double ss = 0.0;
              for (int i = 0; i < ns; ++i) ss += slot[i];
              val = sqrt(ss);
            }
            A.stop_vals[(int64_t)b * (A.max_iter + 1) + k] = val;
            if (val < A.delta) { S->iters = k; S->reason = R_TOL; m = M_FIN; }
            else if (sc[5] > 0.0) { S->iters = k; S->reason = R_BREAK; m = M_FIN; }
            else if (k == A.max_iter) { S->iters = k; S->reason = R_MAXIT; m = M_FIN; }
            else S->k = k + 1;
          }
          sc[6] = (double)m;
          mode_set(P, b, ph, M_RUNB, m);
          s_pub = m;
        }
        block_barrier();
        if (sc[6] == (double)M_FIN) {
          // y = R^{-1} step and t0 - Omega for the finalisation in the next phase
          solve_y(P, b, *reinterpret_cast<volatile int*>(&S->iters), sm.S0, CH);
          const double* t0 = vecp(P, b, V_T0);
          const double* om = vecp(P, b, V_OMEGA);
          double* tmo = vecp(P, b, V_TMO);
          for (int i = threadIdx.x; i < s; i += NT) tmo[i] = t0[i] - om[i];
        }
      }
      block_barrier();
      } else {  // M_FIN: w = w0 + U (t0 - Omega) + V y;  r = r0 - C (t0 - Omega) - HV y
        const int K = *reinterpret_cast<volatile int*>(&P.st[b].iters);
        const double* U = s ? A.U + (int64_t)b * A.bs_uc : nullptr;
        const double* C = s ? A.C + (int64_t)b * A.bs_uc : nullptr;
        const double* Yb = P.y + (int64_t)b * A.max_iter;
        for (int i = threadIdx.x; i < s; i += NT) sv[i] = __ldcg(vecp(P, b, V_TMO) + i);
        block_barrier();
        double wacc[PPT], racc[PPT];
        int64_t pp[PPT];
#pragma unroll
        for (int uu = 0; uu < PPT; ++uu) {
          pp[uu] = tile_pixel(op, tile, threadIdx.x + uu * NT);
          const int64_t q = pp[uu] >= 0 ? pp[uu] : 0;
          double w = A.w0 ? A.w0[(int64_t)b * n + q] : 0.0;
          double r = 0.0;
          if (P.track) r = A.w0 ? P.r0[(int64_t)b * n + q] : A.g[(int64_t)b * n + q];
          double uo = 0.0, co = 0.0;
          for (int i = 0; i < s; ++i) {
            uo += U[(int64_t)i * A.ld_uc + q] * sv[i];
            if (P.track) co += C[(int64_t)i * A.ld_uc + q] * sv[i];
          }
          wacc[uu] = w + uo;
          racc[uu] = r - co;
        }
        double* ys = sm.S0;  // y staged in chunks (the stencil scratch is free here)
        for (int j0 = 0; j0 < K; j0 += CH) {
          const int m = (K - j0) < CH ? (K - j0) : CH;
          block_barrier();
          for (int i = threadIdx.x; i < m; i += NT) ys[i] = __ldcg(Yb + j0 + i);
          block_barrier();
#pragma unroll
          for (int uu = 0; uu < PPT; ++uu) {
            const int64_t q = pp[uu] >= 0 ? pp[uu] : 0;
            const double* V = A.basis + (int64_t)b * A.bs_basis + (int64_t)j0 * A.ld_basis + q;
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
            int j = 0;
            for (; j + 3 < m; j += 4) {
              a0 += V[(int64_t)j * A.ld_basis] * ys[j];
              a1 += V[(int64_t)(j + 1) * A.ld_basis] * ys[j + 1];
              a2 += V[(int64_t)(j + 2) * A.ld_basis] * ys[j + 2];
              a3 += V[(int64_t)(j + 3) * A.ld_basis] * ys[j + 3];
            }
            for (; j < m; ++j) a0 += V[(int64_t)j * A.ld_basis] * ys[j];
            wacc[uu] += (a0 + a1) + (a2 + a3);
            if (P.track) {
              const double* HVc = P.hv + ((int64_t)b * A.max_iter + j0) * n + q;
              double h0 = 0.0, h1 = 0.0;
              int jj = 0;
              for (; jj + 1 < m; jj += 2) {
                h0 += HVc[(int64_t)jj * n] * ys[jj];
                h1 += HVc[(int64_t)(jj + 1) * n] * ys[jj + 1];
              }
              if (jj < m) h0 += HVc[(int64_t)jj * n] * ys[jj];
              racc[uu] -= h0 + h1;
            }
          }
        }
#pragma unroll
        for (int uu = 0; uu < PPT; ++uu) {
          if (pp[uu] < 0) continue;
          A.w[(int64_t)b * n + pp[uu]] = wacc[uu];
          if (P.track && A.r) A.r[(int64_t)b * n + pp[uu]] = racc[uu];
        }
        if (arrive(P, b, &s_flag)) {
          if (threadIdx.x == 0) {
            A.iters[b] = P.st[b].iters;
            A.reasons[b] = P.st[b].reason;
            mode_set(P, b, ph, M_FIN, M_DONE);
            s_pub = M_DONE;
          }
        }
        block_barrier();
      }
      block_barrier();
      if (md == M_RUNB) KR_DMARK(4, dlast);
      else if (md != M_RUN) KR_DMARK(5, dlast);
      }  // tiles of the drawn unit
      if (P.dataflow) {
        // the block that completed the sample's phase publishes the next one (after all of
        // its own post-processing above: the barrier orders the block's writes, the fence
        // makes them visible before the word)
        if (threadIdx.x == 0 && s_pub != 0xffu) {
          __threadfence();
          if (s_pub == M_DONE) {
            atomicExch(P.tick + b, tick_word(M_DONE, 0, TICK_DONE_LO));
            __threadfence();
            atomicAdd(P.sched + 1, 1);
          } else {
            atomicExch(P.tick + b, tick_word(s_pub, s_seq + 1, 0));
          }
        }
      } else {
        if (threadIdx.x == 0) s_unit = (int)next_ticket;
      }
      block_barrier();
      KR_DMARK(6, dlast);
    }
    if (P.dataflow) break;
    DYN_GRID_SYNC();
    ++ph;
  }
}

}  // namespace dyn
}  // namespace kr

using namespace kr;
using namespace kr::dyn;

namespace {

struct DynLayout {
  int G, nslot, ntiles;
  int64_t total;
  size_t smem;
  bool track;
};

void dyn_plan(const kr_op& op, const kr_solve_args& a, DynLayout& L) {
  const int64_t n = op_n(op);
  const Geom g = make_geom(op);
  const int B = op.batch;
  L.smem = sizeof(double) * ((size_t)g.total + MAX_SLOTS + MAX_S + RED_DOUBLES);
  L.ntiles = num_tiles(op);
  const int ns = a.stop_kind >= 1 ? a.nsc_s : 0;
  L.nslot = imax(imax(2 * a.s + 1 + ns, a.s + 1), 1 + ns);
  L.track = a.track_residual && a.r;
  int sms = device_sms(), per_sm = 0;
  const void* kfn = KR_PICK_Q(rminres_dyn_kernel, q_variant(op));
  if (sms > 0) {
    if (L.smem > 48 * 1024) ensure_smem(kfn, L.smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, NT, L.smem);
  }
  if (per_sm < 1) per_sm = 1;
  if (sms < 1) sms = 148;
  L.G = per_sm * sms;
  const int64_t hv = L.track ? (int64_t)B * a.max_iter * n : (int64_t)B * n;
  L.total = (int64_t)B * n + hv + ((a.w0 && L.track) ? (int64_t)B * n : 0) + (int64_t)B * L.nslot * L.ntiles +
            (int64_t)B * (sizeof(St) / 8) + (int64_t)B * NVEC * MAX_S + (int64_t)B * (a.max_iter + 1) * 4 +
            (int64_t)B * a.max_iter + B /*mode*/ + (B + 2) /*cnt, bar (as doubles)*/ + B /*tick*/ + 2 /*sched*/ + 8;
}

}  // namespace

namespace kr {

bool rminres_dyn_applies(const kr_op& op, const kr_solve_args& a) {
  static const bool off = getenv("KR_RMINRES_DYN") && getenv("KR_RMINRES_DYN")[0] == '0';
  return !off && a.basis != nullptr && op.batch >= 1 && op.batch <= MAX_B;
}

int64_t rminres_dyn_workspace(const kr_op& op, const kr_solve_args& a) {
  DynLayout L;
  dyn_plan(op, a, L);
  return L.total;
}

int rminres_dyn(const kr_op& op, const kr_solve_args& a, double* work, int64_t work_len, cudaStream_t st) {
  DynLayout L;
  dyn_plan(op, a, L);
  KR_CHECK_ARG(work && work_len >= L.total, "rminres workspace too small");
  const int64_t n = op_n(op);
  const int B = op.batch;
  DParams P;
  P.op = op;
  P.a = a;
  P.n = n;
  P.ntiles = L.ntiles;
  P.nslot = L.nslot;
  P.G = L.G;
  P.B = B;
  P.track = L.track ? 1 : 0;
  double* cur = work;
  auto take = [&](int64_t cnt) {
    double* r = cur;
    cur += cnt;
    return r;
  };
  P.tmp = take((int64_t)B * n);
  P.hv = take(L.track ? (int64_t)B * a.max_iter * n : (int64_t)B * n);
  P.r0 = (a.w0 && L.track) ? take((int64_t)B * n) : nullptr;
  P.part = take((int64_t)B * L.nslot * L.ntiles);
  P.st = reinterpret_cast<St*>(take((int64_t)B * (sizeof(St) / 8)));
  P.vecs = take((int64_t)B * NVEC * MAX_S);
  P.hist = take((int64_t)B * (a.max_iter + 1) * 4);
  P.y = take((int64_t)B * a.max_iter);
  P.mode = reinterpret_cast<unsigned long long*>(take(B));
  P.cnt = reinterpret_cast<int*>(take(B + 2));
  P.bar = reinterpret_cast<unsigned int*>(P.cnt + B + 1);
  P.grab = reinterpret_cast<unsigned int*>(P.cnt + B + 2);
  P.tick = reinterpret_cast<unsigned long long*>(take(B));
  P.sched = reinterpret_cast<int*>(take(2));
  // pipelining pays when every super-phase still has several units per block
  const char* pe = getenv("KR_DYN_PIPE");
  P.pipe = pe ? (pe[0] == '1') : 0;  // measured: no gain once units are ticketed (C3: 1326 vs 1315 ms)
  auto al16 = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
  const int ns = a.stop_kind >= 1 ? a.nsc_s : 0;
  P.vec2 = op.data_kind != KR_DATA_DENSE && op.cols % 2 == 0 && al16(P.tmp) && al16(P.hv) && al16(a.basis) &&
           a.ld_basis % 2 == 0 && a.bs_basis % 2 == 0 &&
           (a.s == 0 || (al16(a.C) && a.ld_uc % 2 == 0 && a.bs_uc % 2 == 0)) &&
           (ns == 0 || (al16(a.Z) && a.ld_z % 2 == 0 && a.bs_z % 2 == 0)) && getenv("KR_DYN_SCALAR") == nullptr;
  {
    const Geom g = make_geom(op);
    P.use_tma = (op.data_kind != KR_DATA_DENSE && g.RH * (TW + 2 * g.H) <= g.sa &&
                 make_region_tmap(&P.tmap, P.tmp, op.cols, op.rows, 1, B, n, n, TW + 2 * g.H, g.RH))
                    ? 1 : 0;
    if (!P.use_tma) memset(&P.tmap, 0, sizeof P.tmap);
  }
  {
    const char* we = getenv("KR_DYN_WINDOW");
    int w = we ? atoi(we) : 0;
    P.window = w > 0 ? w : MAX_B;
    const char* de = getenv("KR_DYN_DATAFLOW");
    P.dataflow = (de && de[0] == '1') ? 1 : 0;
    if (P.dataflow) P.pipe = 0;
    const char* ge = getenv("KR_DYN_GROUPB");
    P.group_b = ge && atoi(ge) > 0 ? atoi(ge) : 4;
    const char* pr = getenv("KR_DYN_PRIO");
    P.prio = (pr && pr[0] == '1') ? 1 : 0;
  }
  const void* kfn = KR_PICK_Q(rminres_dyn_kernel, q_variant(op));
  KR_TRY(ensure_smem(kfn, L.smem));
  cudaMemsetAsync(P.vecs, 0, sizeof(double) * (size_t)B * NVEC * MAX_S, st);
  cudaMemsetAsync(P.mode, 0xff, sizeof(unsigned long long) * (size_t)B, st);
  cudaMemsetAsync(P.cnt, 0, sizeof(double) * (size_t)(B + 2), st);
  cudaMemsetAsync(P.tick, 0, sizeof(double) * (size_t)(B + 2), st);
  void* args[] = {&P};
  cudaError_t e = cudaLaunchCooperativeKernel(kfn, dim3(P.G), dim3(NT), args, L.smem, st);
  if (e != cudaSuccess) return fail(KR_ECUDA, std::string("rminres cooperative launch: ") + cudaGetErrorString(e));
#ifdef KR_DYN_TIMING
  {
    cudaStreamSynchronize(st);
    unsigned long long h[8] = {};
    cudaMemcpyFromSymbol(h, kr::dyn::g_dyn_ns, sizeof h);
    unsigned long long z[8] = {};
    cudaMemcpyToSymbol(kr::dyn::g_dyn_ns, z, sizeof z);
    fprintf(stderr, "dyn block0 us: draw %.0f stencil %.0f dots %.0f arriveA %.0f phaseB %.0f fin %.0f publish %.0f; A units %llu\n",
            h[0] / 1e3, h[1] / 1e3, h[2] / 1e3, h[3] / 1e3, h[4] / 1e3, h[5] / 1e3, h[6] / 1e3, h[7]);
  }
#endif
  return check_launch("kr_rminres (dyn)");
}

}  // namespace kr
