// The n = 8 Ax_helm element-pair body shared by the stand-alone K1 kernel
// (ax.cu: ax_helm8s_kernel) and the fused Ax+dssum kernel (axdss.cu).
//
// One-pencil mapping with a bank-swizzled shared layout.  In the generic
// ax_helm_kernel the t-direction reads us_[i][j][q] (and f3s) come from 4 rows
// j at a 64-byte stride, so rows j and j+2 hit the same banks (2-way conflict,
// 16 of the ~70 wavefronts of a warp-layer).  Here column c of row r is stored at
// c ^ (((r >> 1) & 1) * 4): the 4 rows of a warp land on distinct banks, and the
// (q, q+1) pairs stay adjacent, so the t-direction operand pair is one
// conflict-free LDS.128.  Per warp-layer wavefronts 70 -> 46.  Arithmetic and
// accumulation order are those of ax_helm_kernel (kernels/_numba.py:86-131,
// same results bit for bit).
#pragma once
#include "common.cuh"

namespace sf {

template <int N>
struct DMat {
  double v[N * N];
};

#ifndef SF_AX_UNROLL
#define SF_AX_UNROLL 2
#endif
constexpr int kAxUnroll = SF_AX_UNROLL;
#ifndef SF_AX8S_MINB
#define SF_AX8S_MINB 4
#endif

// 128 threads: elements 2*pair and 2*pair+1 (64 threads each).
// PRE: the operator is applied to pre .* u (the Jacobi-preconditioned Krylov
// vector, `precond(v)` then `apply_a`, krylov.py:106-107) without materialising
// it: each u value is scaled as it is loaded (one IEEE multiply, the same bits
// as `inv_diag * v`), including the masked rows that pass u through.
// MASS: false compiles the mass term out (callers pass it only when lam_mass == 0,
// where the reference skips the term, _numba.py:128); true keeps the runtime test.
template <bool EX, bool MASK, bool PRE = false, bool MASS = true>
__device__ __forceinline__ void ax8s_pair(const DMat<8>& D, const double* __restrict__ g,
                                          const double* __restrict__ b, const double* __restrict__ u,
                                          double* __restrict__ w, long long E, double lv, double lm,
                                          const uint32_t* __restrict__ inmask,
                                          const uint32_t* __restrict__ outsel, long long pair,
                                          unsigned long long* signal = nullptr,
                                          const double* __restrict__ pre = nullptr) {
  constexpr int N = 8, NN = 64, NNN = 512, EPB = 2, WPE = 16;
  __shared__ __align__(16) double us_[EPB][NNN];
  __shared__ __align__(16) double f1s[EPB][NNN];
  __shared__ __align__(16) double f2s[EPB][NNN];
  __shared__ __align__(16) double f3s[EPB][NNN];
  const int le = threadIdx.x >> 6;
  const int t = threadIdx.x & 63;
  const int j = t >> 3, k = t & 7;
  const int sj = ((j >> 1) & 1) << 2;
  const int st = j * N + (k ^ sj);  // swizzled smem slot of (j, k) within a layer
  const long long e = pair * EPB + le;
  const bool active = e < E;
  const long long base = e * NNN + t;
  const long long gstride = E * (long long)NNN;
  double* su = us_[le];
  double* s1 = f1s[le];
  double* s2 = f2s[le];
  double* s3 = f3s[le];
#define SW(row) ((((row) >> 1) & 1) << 2)

  // this thread's mask bits, one per layer (bit i <-> point (i, j, k)), gathered
  // up front so the output loop has no dependent loads
  // (the warp's 8 words per mask come in with one load per lane and are
  // broadcast by shuffles: 2 loads per thread instead of 16)
  uint32_t inb = 0xffu, outb = 0xffu;
  if constexpr (MASK) {
    inb = 0u;
    outb = 0u;
    uint32_t win = 0u, wout = 0u;
    if (active) {
      const long long wi = e * WPE + 2 * (threadIdx.x & 7) + (t >> 5);
      win = __ldg(inmask + wi);
      wout = __ldg(outsel + wi);
    }
#pragma unroll
    for (int i = 0; i < N; ++i) {
      inb |= ((__shfl_sync(0xffffffffu, win, i) >> (t & 31)) & 1u) << i;
      outb |= ((__shfl_sync(0xffffffffu, wout, i) >> (t & 31)) & 1u) << i;
    }
  }
  double um[N];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double uv = active ? __ldg(u + base + i * NN) : 0.0;
    if constexpr (PRE) uv = active ? __dmul_rn(__ldg(pre + base + i * NN), uv) : 0.0;
    if constexpr (MASK) {
      if (!((inb >> i) & 1u)) uv = 0.0;
    }
    um[i] = uv;
    su[i * NN + st] = uv;
  }
  double dj[N], dk[N];
#pragma unroll
  for (int q = 0; q < N; ++q) {
    dj[q] = D.v[j * N + q];
    dk[q] = D.v[k * N + q];
  }
  const double* gp = g + (active ? base : 0);
  // (a per-thread cp.async ring holding 3 layers of G in shared memory was
  // measured slower: 238 vs 220 us at 32^3 -- the extra LDGSTS/LDS traffic costs
  // more than the deeper prefetch gains)
  double gn[6];
#pragma unroll
  for (int m = 0; m < 6; ++m) gn[m] = active ? __ldg(gp + m * gstride) : 0.0;
  __syncthreads();
  // fused kernel: publish the previous Ax job of this block (its stores have
  // long completed while this job's loads were in flight, so the fence is cheap)
  if (signal != nullptr && threadIdx.x == 0) {
    __threadfence();
    atomicAdd(signal, 1ull);
  }

#pragma unroll (kAxUnroll)
  for (int i = 0; i < N; ++i) {
    double gc[6];
#pragma unroll
    for (int m = 0; m < 6; ++m) gc[m] = gn[m];
    if (i + 1 < N) {
#pragma unroll
      for (int m = 0; m < 6; ++m) gn[m] = active ? __ldg(gp + (i + 1) * NN + m * gstride) : 0.0;
    }
    double ar = 0.0, as = 0.0, at = 0.0;
    // (splitting these three chains further into even/odd halves measured
    // slower: 230 vs 216 us at 32^3)
#pragma unroll
    for (int q = 0; q < N; ++q) {
      ar = mac<EX>(ar, D.v[i * N + q], um[q]);
      as = mac<EX>(as, dj[q], su[i * NN + q * N + (k ^ SW(q))]);
    }
#pragma unroll
    for (int q = 0; q < N; q += 2) {
      const double2 tv = *reinterpret_cast<const double2*>(su + i * NN + j * N + (q ^ sj));
      at = mac<EX>(at, dk[q], tv.x);
      at = mac<EX>(at, dk[q + 1], tv.y);
    }
    s1[i * NN + st] = add<EX>(add<EX>(mul<EX>(gc[0], ar), mul<EX>(gc[1], as)), mul<EX>(gc[2], at));
    s2[i * NN + st] = add<EX>(add<EX>(mul<EX>(gc[1], ar), mul<EX>(gc[3], as)), mul<EX>(gc[4], at));
    s3[i * NN + st] = add<EX>(add<EX>(mul<EX>(gc[2], ar), mul<EX>(gc[4], as)), mul<EX>(gc[5], at));
  }
#pragma unroll
  for (int q = 0; q < N; ++q) {
    dj[q] = D.v[q * N + j];
    dk[q] = D.v[q * N + k];
  }
  // mass term: B is streamed one layer ahead (issued before the barrier) so its
  // load latency hides behind the contraction instead of stalling each output
  // layer (ncu/profile: the Helmholtz operator ran 1.5x the Poisson one)
  const bool mass = MASS && lm != 0.0;
  double bnext = 0.0;
  if constexpr (MASS) bnext = (mass && active) ? __ldg(b + base) : 0.0;
  __syncthreads();
  if (!active) return;

#pragma unroll (kAxUnroll)
  for (int i = 0; i < N; ++i) {
    double bi = 0.0;
    if constexpr (MASS) {
      bi = bnext;
      if (mass && i + 1 < N) bnext = __ldg(b + base + (i + 1) * NN);
    }
    double acc = 0.0;
    if constexpr (EX) {
      // the reference's single interleaved accumulator (_numba.py:119-126)
#pragma unroll
      for (int q = 0; q < N; q += 2) {
        const double2 t3 = *reinterpret_cast<const double2*>(s3 + i * NN + j * N + (q ^ sj));
        acc = mac<EX>(acc, D.v[q * N + i], s1[q * NN + st]);
        acc = mac<EX>(acc, dj[q], s2[i * NN + q * N + (k ^ SW(q))]);
        acc = mac<EX>(acc, dk[q], t3.x);
        acc = mac<EX>(acc, D.v[(q + 1) * N + i], s1[(q + 1) * NN + st]);
        acc = mac<EX>(acc, dj[q + 1], s2[i * NN + (q + 1) * N + (k ^ SW(q + 1))]);
        acc = mac<EX>(acc, dk[q + 1], t3.y);
      }
    } else {
      // production: three independent DFMA chains (r, s, t) instead of one
      // 24-long chain -- ncu showed 'wait' (fixed-latency dependency) as the
      // second stall reason; the sum differs from the reference's order only
      // by rounding (<= 1e-15 relative)
      double ar = 0.0, as = 0.0, at = 0.0;
#pragma unroll
      for (int q = 0; q < N; q += 2) {
        const double2 t3 = *reinterpret_cast<const double2*>(s3 + i * NN + j * N + (q ^ sj));
        ar = fma(D.v[q * N + i], s1[q * NN + st], ar);
        as = fma(dj[q], s2[i * NN + q * N + (k ^ SW(q))], as);
        at = fma(dk[q], t3.x, at);
        ar = fma(D.v[(q + 1) * N + i], s1[(q + 1) * NN + st], ar);
        as = fma(dj[q + 1], s2[i * NN + (q + 1) * N + (k ^ SW(q + 1))], as);
        at = fma(dk[q + 1], t3.y, at);
      }
      acc = (ar + as) + at;
    }
    double wv = mul<EX>(lv, acc);
    if (mass) wv = add<EX>(wv, mul<EX>(mul<EX>(lm, bi), su[i * NN + st]));
    if constexpr (MASK) {
      if (!((outb >> i) & 1u)) {
        wv = __ldg(u + base + i * NN);
        if constexpr (PRE) wv = __dmul_rn(__ldg(pre + base + i * NN), wv);
      }
    }
    w[base + i * NN] = wv;
  }
#undef SW
}

}  // namespace sf
