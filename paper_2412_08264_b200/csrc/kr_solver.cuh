// kr_solver.cuh -- helpers shared by the persistent Krylov kernels: block
// partial sums per sample and their fixed-order (deterministic) reduction.
#pragma once

#include <cassert>

#include "kr_common.cuh"

#ifdef KR_GUARD
#define KR_ASSERT(c) assert(c)
#else
#define KR_ASSERT(c) ((void)0)
#endif

namespace kr {

constexpr int MAX_S = 128;                // recycle columns
constexpr int MAX_NSC = 128;              // NSC columns
constexpr double BREAKDOWN_RTOL = 1e-13;  // krylov.py:50

enum Reason { R_TOL = 0, R_MAXIT = 1, R_BREAK = 2, R_NONSPD = 3 };

// Block partials of one launch: part[sample][slot][rank].
struct Partials {
  double* part;
  int nslot;
  int Gs;
  __device__ inline double* at(int bl, int slot) const {
    KR_ASSERT(bl >= 0 && slot >= 0 && slot < nslot);
    return part + ((int64_t)bl * nslot + slot) * Gs;
  }
};

// Deferred cross-warp reductions.  A pass reduces NV per-thread values inside each
// warp (MultiSum, no block barrier) and keeps the lane-owned warp sum in a register;
// after all passes the warp sums go to smem (stride DEF_STRIDE per value) and ONE
// barrier later each value is summed over the warps in warp order -- the same
// order as block_sum, without a block barrier per pass.
constexpr int DEF_PASSES = 4;   // passes kept in registers
constexpr int DEF_STRIDE = 9;   // >= warps per block (8) + 1, odd: conflict-free
constexpr int RED_DOUBLES = 912;  // reduction scratch: max(25 * 33 + 25, 25 * DEF_PASSES * DEF_STRIDE)

template <int NV>
__device__ inline void def_add(double r, int pass, double* red) {  // r: this lane's MultiSum<NV> result
  using M = MultiSum<NV>;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int idx = M::owner(lane);
  if (idx < NV && (lane & ((32 / M::P) - 1)) == 0) red[(pass * NV + idx) * DEF_STRIDE + warp] += r;
}

__device__ inline double def_sum(const double* red, int v) {
  const int nw = blockDim.x >> 5;
  double acc = 0.0;
  for (int w = 0; w < nw; ++w) acc += red[v * DEF_STRIDE + w];
  return acc;
}

// acc_out[i] += sum_{p in [lo,hi)} A_i[p] * x(p), i < S; A_i = A + i*lda (16 columns per pass).
// red needs 16 * DEF_PASSES * DEF_STRIDE doubles for the deferred path (S <= 64).
template <typename XF>
__device__ inline void slot_dots(const double* __restrict__ A, int64_t lda, int S, int64_t lo, int64_t hi,
                                 XF xf, double* acc_out, double* red) {
  const int npass = (S + 15) / 16;
  if (npass <= DEF_PASSES) {
    block_barrier();  // red may still be read by an earlier reduction
    for (int i = threadIdx.x; i < npass * 16 * DEF_STRIDE; i += blockDim.x) red[i] = 0.0;
    block_barrier();
    for (int pass = 0; pass < npass; ++pass) {
      const int base = pass * 16;
      double v16[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) v16[i] = 0.0;
      for (int64_t p = lo + threadIdx.x; p < hi; p += blockDim.x) {
        double x = xf(p);
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (base + i < S) v16[i] += A[(int64_t)(base + i) * lda + p] * x;
      }
      def_add<16>(MultiSum<16>::reduce(v16, threadIdx.x & 31), pass, red);
    }
    block_barrier();
    for (int i = threadIdx.x; i < S; i += blockDim.x) acc_out[i] += def_sum(red, i);
    block_barrier();
    return;
  }
  for (int base = 0; base < S; base += 16) {
    double v16[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v16[i] = 0.0;
    for (int64_t p = lo + threadIdx.x; p < hi; p += blockDim.x) {
      double x = xf(p);
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (base + i < S) v16[i] += A[(int64_t)(base + i) * lda + p] * x;
    }
    block_sum<16>(v16, red);
    if (threadIdx.x < 16 && base + threadIdx.x < S) acc_out[base + threadIdx.x] += red[threadIdx.x];
    block_barrier();
  }
}

__device__ inline void write_partials(const Partials& P, int bl, int j, int slot0, int S, const double* acc) {
  KR_ASSERT(j >= 0 && j < P.Gs && S >= 0 && slot0 + S <= P.nslot && S <= MAX_SLOTS);
  for (int i = threadIdx.x; i < S; i += blockDim.x) P.at(bl, slot0 + i)[j] = acc[i];
}

__device__ inline void write_partial1(const Partials& P, int bl, int j, int slot, double v) {
  if (threadIdx.x == 0) P.at(bl, slot)[j] = v;
}

// out[i] = sum over the sample's Gs blocks.  A warp per slot: lanes read the
// Gs partials coalesced (8 slots in flight per warp), then a fixed shuffle tree
// -- deterministic (the same order every run and for every block).  Callers
// synchronise the block before reading out[].
__device__ inline void reduce_slots(const Partials& P, int bl, int slot0, int S, double* out) {
  constexpr int INF = 8;  // slots in flight per warp
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i0 = warp; i0 < S; i0 += INF * nw) {
    double acc[INF];
#pragma unroll
    for (int u = 0; u < INF; ++u) {
      const int i = i0 + u * nw;
      double a = 0.0;
      if (i < S) {
        const double* src = P.at(bl, slot0 + i);
        for (int jj = lane; jj < P.Gs; jj += 32) a += src[jj];
      }
      acc[u] = a;
    }
#pragma unroll
    for (int u = 0; u < INF; ++u) {
      const double v = warp_sum(acc[u]);
      const int i = i0 + u * nw;
      if (lane == 0 && i < S) out[i] = v;
    }
  }
}

// Grid-wide barrier for a cooperative launch.  Thread 0 of every block arrives
// with a release add on a monotone counter and polls it with acquire loads
// (ld.acquire.gpu also invalidates the SM's L1, so the block's later plain loads
// see the other blocks' writes).  The __syncwarp inside block_barrier() keeps
// lanes 1..31 of warp 0 from entering the aligned bar.sync while lane 0 is still
// polling -- cooperative_groups' grid.sync() does not, and on sm_100 that let
// warp 0 fall one block barrier behind its siblings.
__device__ __forceinline__ void grid_barrier(unsigned int* counter, unsigned int nblocks, unsigned int& target) {
  block_barrier();
  if (threadIdx.x == 0) {
    target += nblocks;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(counter) : "memory");
    unsigned int v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
    } while ((int)(v - target) < 0);
  }
  block_barrier();
}

// Blocks per sample and samples per launch for a cooperative launch.
struct LaunchPlan {
  int Gs;
  int chunk;
};

}  // namespace kr
