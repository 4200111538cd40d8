// Element-local tensor-product kernels: Ax_helm (K1), local_grad3 (grad_ref) and
// the one-axis contractions apply_{r,s,t}.
//
// Reference semantics (file:line under /root/reference/pkg/src/semflow):
//   ax_helmholtz_local  kernels/_numba.py:86-131
//   grad_ref            kernels/_numba.py:63-83
//   apply_r/s/t         kernels/_numba.py:15-60
//   make_global_op body operators.py:51-54 (masked variant, fused here)
//
// Layout: scalar field (E, n, n, n) float64, C order, axes (element, r, s, t) --
// t is fastest.  geom is (6, E, n, n, n) packed rr, rs, rt, ss, st, tt.
//
// Thread mapping ("r-pencils").  One element is handled by n*n threads; thread
// t = j*n + k owns the pencil u[0..n-1][j][k] along r.  For a fixed layer i the
// n*n threads of an element touch n*n consecutive doubles, so every global load
// and store of u, geom, b and w is a fully coalesced 8-byte-per-lane access
// (256 B per warp instruction) and each byte of HBM is read exactly once.
//   * the r-derivative is register-local (D[i][q] is warp-uniform and comes from
//     the kernel-parameter constant bank as a DFMA operand),
//   * the s- and t-derivatives read the element's u volume from shared memory;
//     for a warp the addresses depend only on k (s-derivative) or only on j
//     (t-derivative), so every LDS is a conflict-free broadcast,
//   * the transposed contraction keeps f1 (r-component of G grad u) in registers
//     and f2, f3 in shared memory, preserving the reference's single interleaved
//     accumulator over q (`_numba.py:119-126`).
#include "ax8s.cuh"

namespace sf {

template <int N>
struct AxCfg {
  static constexpr int NN = N * N;
  static constexpr int NNN = N * N * N;
  static constexpr int EPB = (128 / NN) > 0 ? (128 / NN) : 1;  // elements per block
  static constexpr int THREADS = EPB * NN;
  static constexpr int WPE = (NNN + 31) / 32;  // mask words per element
};

// bit for local point p of element e in a packed per-element bitmask
__device__ __forceinline__ bool mask_bit(const uint32_t* __restrict__ m, long long e, int wpe,
                                         int p) {
  return (__ldg(m + e * wpe + (p >> 5)) >> (p & 31)) & 1u;
}

// K1.  w = lam_visc * D^T G D um + lam_mass * B um, um = inmask ? u : 0.
// With MASK, the written value is w where outsel is set and u elsewhere
// (outsel = mask | shared: shared points are finalised by the dssum kernel).
//
// Register budget: the layer loops are not fully unrolled (SF_AX_UNROLL) so the
// live state per thread is the u pencil, one layer of G (plus the prefetched next
// layer) and the thread's two rows of D -- ~80-100 registers, 5-6 blocks (20-24
// warps) per SM, enough loads in flight to cover HBM latency.  f1, f2, f3 live in
// shared memory (4 element volumes, 16 KB per element at n = 8).
#ifndef SF_AX_MINB
#define SF_AX_MINB 5
#endif
template <int N, bool EX, bool MASK>
__global__ void __launch_bounds__(AxCfg<N>::THREADS, (N == 8 ? SF_AX_MINB : 1))
ax_helm_kernel(DMat<N> D, const double* __restrict__ g, const double* __restrict__ b,
               const double* __restrict__ u, double* __restrict__ w, long long E, double lv,
               double lm, const uint32_t* __restrict__ inmask,
               const uint32_t* __restrict__ outsel) {
  using C = AxCfg<N>;
  constexpr int NN = C::NN, NNN = C::NNN;
  __shared__ double us_[C::EPB][NNN];
  __shared__ double f1s[C::EPB][NNN];
  __shared__ double f2s[C::EPB][NNN];
  __shared__ double f3s[C::EPB][NNN];

  const int le = threadIdx.x / NN;
  const int t = threadIdx.x - le * NN;
  const int j = t / N, k = t - (t / N) * N;
  const long long e = (long long)blockIdx.x * C::EPB + le;
  const bool active = e < E;
  const long long base = e * NNN + t;
  const long long gstride = E * (long long)NNN;

  double um[N];   // masked pencil the operator acts on
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double uv = active ? __ldg(u + base + i * NN) : 0.0;
    if constexpr (MASK) {
      if (!(active && mask_bit(inmask, e, C::WPE, i * NN + t))) uv = 0.0;
    }
    um[i] = uv;
    us_[le][i * NN + t] = uv;
  }
  double dj[N], dk[N];
#pragma unroll
  for (int q = 0; q < N; ++q) {
    dj[q] = D.v[j * N + q];
    dk[q] = D.v[k * N + q];
  }
  // G of layer 0 in flight while the block synchronises
  const double* gp = g + (active ? base : 0);
  double gn[6];
#pragma unroll
  for (int m = 0; m < 6; ++m) gn[m] = active ? __ldg(gp + m * gstride) : 0.0;
  __syncthreads();

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
#pragma unroll
    for (int q = 0; q < N; ++q) {
      ar = mac<EX>(ar, D.v[i * N + q], um[q]);
      as = mac<EX>(as, dj[q], us_[le][i * NN + q * N + k]);
      at = mac<EX>(at, dk[q], us_[le][i * NN + j * N + q]);
    }
    // (g0*gr + g1*gs) + g2*gt, as written in _numba.py:116-118
    f1s[le][i * NN + t] = add<EX>(add<EX>(mul<EX>(gc[0], ar), mul<EX>(gc[1], as)), mul<EX>(gc[2], at));
    f2s[le][i * NN + t] = add<EX>(add<EX>(mul<EX>(gc[1], ar), mul<EX>(gc[3], as)), mul<EX>(gc[4], at));
    f3s[le][i * NN + t] = add<EX>(add<EX>(mul<EX>(gc[2], ar), mul<EX>(gc[4], as)), mul<EX>(gc[5], at));
  }
#pragma unroll
  for (int q = 0; q < N; ++q) {  // columns of D for the transposed contraction
    dj[q] = D.v[q * N + j];
    dk[q] = D.v[q * N + k];
  }
  __syncthreads();
  if (!active) return;

  const bool mass = lm != 0.0;
#pragma unroll (kAxUnroll)
  for (int i = 0; i < N; ++i) {
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < N; ++q) {
      acc = mac<EX>(acc, D.v[q * N + i], f1s[le][q * NN + t]);
      acc = mac<EX>(acc, dj[q], f2s[le][i * NN + q * N + k]);
      acc = mac<EX>(acc, dk[q], f3s[le][i * NN + j * N + q]);
    }
    double wv = mul<EX>(lv, acc);
    if (mass) wv = add<EX>(wv, mul<EX>(mul<EX>(lm, __ldg(b + base + i * NN)), us_[le][i * NN + t]));
    if constexpr (MASK) {
      // unselected points (masked, unshared) return the operator input
      if (!mask_bit(outsel, e, C::WPE, i * NN + t)) wv = __ldg(u + base + i * NN);
    }
    w[base + i * NN] = wv;
  }
}

// K1 for n = 8: the one-pencil kernel with a bank-swizzled shared layout
// (body in ax8s.cuh, shared with the fused Ax+dssum kernel).
template <bool EX, bool MASK, bool PRE = false, bool MASS = true>
__global__ void __launch_bounds__(128, SF_AX8S_MINB)
ax_helm8s_kernel(DMat<8> D, const double* __restrict__ g, const double* __restrict__ b,
                 const double* __restrict__ u, double* __restrict__ w, long long E, double lv,
                 double lm, const uint32_t* __restrict__ inmask, const uint32_t* __restrict__ outsel,
                 const double* __restrict__ pre = nullptr, long long pair0 = 0) {
  ax8s_pair<EX, MASK, PRE, MASS>(D, g, b, u, w, E, lv, lm, inmask, outsel, (long long)blockIdx.x + pair0,
                                 nullptr, pre);
}

// Poisson-type operators (lam_mass == 0) run the variant without the mass term:
// the B prefetch register would otherwise cost the common case ~8 %.
template <bool EX, bool MASK, bool PRE>
static void launch8s(dim3 grid, cudaStream_t st, const DMat<8>& D, const double* g, const double* b,
                     const double* u, double* w, long long E, double lv, double lm, const uint32_t* inmask,
                     const uint32_t* outsel, const double* pre, long long pair0 = 0) {
  if (lm != 0.0)
    ax_helm8s_kernel<EX, MASK, PRE, true><<<grid, 128, 0, st>>>(D, g, b, u, w, E, lv, lm, inmask, outsel, pre,
                                                                pair0);
  else
    ax_helm8s_kernel<EX, MASK, PRE, false><<<grid, 128, 0, st>>>(D, g, b, u, w, E, lv, lm, inmask, outsel, pre,
                                                                 pair0);
}

// n = 8 production kernel: bulk-copy-fed persistent Ax (ax8t.cu); 0 selects the
// register-prefetch kernel below (ax8s.cuh) -- sf_set_ax_kernel, for A/B runs.
int ax_helm8t(const DMat<8>& D, const double* g, const double* b, const double* u, double* w, long long E,
              long long e0, long long e1, double lv, double lm, const uint32_t* inmask, const uint32_t* outsel,
              const double* pre, int exact, cudaStream_t st);
int g_ax_kernel = 1;

// Elements [e0, e1) of an E-element field (e0 even; strides use E): the boundary /
// interior split that lets the multi-GPU operator post its halo exchange before
// the interior elements are computed.
int ax_helm8_range(const double* d_host, const double* g, const double* b, const double* u, const double* pre,
                   double* w, long long E, long long e0, long long e1, double lv, double lm,
                   const uint32_t* inmask, const uint32_t* outsel, int exact, cudaStream_t st) {
  if (e0 < 0 || e1 > E || e0 > e1 || (e0 & 1) || ((e1 & 1) && e1 != E)) {
    set_error("ax_range: bad element range [%lld, %lld) of %lld (ends must be even or E)", e0, e1, E);
    return SF_ERR_ARG;
  }
  if ((inmask == nullptr) != (outsel == nullptr)) {
    set_error("ax_range: inmask and outsel must both be given or both be null");
    return SF_ERR_ARG;
  }
  if (e1 == e0) return SF_OK;
  DMat<8> D;
  for (int x = 0; x < 64; ++x) D.v[x] = d_host[x];
  if (g_ax_kernel == 1) {
    const int r = ax_helm8t(D, g, b, u, w, E, e0, e1, lv, lm, inmask, outsel, pre, exact, st);
    if (r != SF_ERR_UNSUPPORTED) return r;
  }
  const long long p0 = e0 / 2, p1 = (e1 + 1) / 2;
  dim3 grid((unsigned)(p1 - p0));
  const bool masked = inmask != nullptr;
#define R(EXV, MV, PV) launch8s<EXV, MV, PV>(grid, st, D, g, b, u, w, E, lv, lm, inmask, outsel, pre, p0)
  if (exact) {
    if (pre) { if (masked) R(true, true, true); else R(true, false, true); }
    else { if (masked) R(true, true, false); else R(true, false, false); }
  } else {
    if (pre) { if (masked) R(false, true, true); else R(false, false, true); }
    else { if (masked) R(false, true, false); else R(false, false, false); }
  }
#undef R
  return check_launch("ax_range");
}

// K1 for n = 8, two pencils per thread (experimental, -DSF_AX_PENCIL2; measured
// 305 us vs 246 us for the one-pencil kernel at 32^3, kept for further tuning).  One warp owns one element; lane (j, kk)
// owns the r-pencils (j, 2kk) and (j, 2kk+1).  Global accesses are 16-byte
// vectors (a warp moves one contiguous 512 B element layer per instruction).  In
// shared memory the s-derivative pair and the t-derivative row are fetched once
// for both pencils (LDS.128), roughly halving the shared-memory wavefronts per
// point against the one-pencil kernel, which is what bounds it (ncu: l1tex 72 %,
// short-scoreboard stalls).  The layer loops are not unrolled so the live state
// stays ~100 registers.  Each element is private to its warp: __syncwarp only.
// Per-point arithmetic and accumulation order are identical to ax_helm_kernel.
#ifndef SF_AX8_MINB
#define SF_AX8_MINB 7
#endif
#ifndef SF_AX8_EPB
#define SF_AX8_EPB 2
#endif
constexpr int AX8_EPB = SF_AX8_EPB;  // elements (warps) per block

template <bool EX, bool MASK>
__global__ void __launch_bounds__(32 * AX8_EPB, SF_AX8_MINB)
ax_helm_n8_kernel(DMat<8> D, const double* __restrict__ g, const double* __restrict__ b,
                  const double* __restrict__ u, double* __restrict__ w, long long E, double lv,
                  double lm, const uint32_t* __restrict__ inmask,
                  const uint32_t* __restrict__ outsel) {
  constexpr int N = 8, NN = 64, NNN = 512;
  constexpr int PJ = 10, LAY = N * PJ, VOL = N * LAY;  // padded smem rows: conflict-free LDS.128
  // us_: element u, layer i overwritten by f3 once every lane is past layer i
  __shared__ __align__(16) double us_[AX8_EPB][VOL];
  __shared__ __align__(16) double f1s[AX8_EPB][VOL];
  __shared__ __align__(16) double f2s[AX8_EPB][VOL];
  __shared__ __align__(16) double Dr[N * PJ];   // D row-major, padded rows
  __shared__ __align__(16) double Dc[N * PJ];   // D^T row-major, padded rows
  for (int x = threadIdx.x; x < NN; x += blockDim.x) {
    Dr[(x >> 3) * PJ + (x & 7)] = D.v[x];
    Dc[(x >> 3) * PJ + (x & 7)] = D.v[(x & 7) * N + (x >> 3)];
  }
  __syncthreads();
  const int le = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int j = lane >> 2, k0 = (lane & 3) * 2;
  const long long e = (long long)blockIdx.x * AX8_EPB + le;
  if (e >= E) return;  // whole warp exits together; no block barrier below
  const int jk = j * N + k0;        // global layer offset
  const int sjk = j * PJ + k0;      // shared layer offset
  const long long base = e * NNN + jk;
  const long long gstride = E * (long long)NNN;
  const int wsel = j >> 2, bsh = (j & 3) * 8 + k0;  // mask word offset / bit within a layer
  double* su = us_[le];
  double* s1 = f1s[le];
  double* s2 = f2s[le];

  double um0[N], um1[N];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double2 v = __ldg(reinterpret_cast<const double2*>(u + base + i * NN));
    if constexpr (MASK) {
      const uint32_t wd = __ldg(inmask + e * 16 + 2 * i + wsel) >> bsh;
      if (!(wd & 1u)) v.x = 0.0;
      if (!(wd & 2u)) v.y = 0.0;
    }
    um0[i] = v.x;
    um1[i] = v.y;
    *reinterpret_cast<double2*>(su + i * LAY + sjk) = v;
  }
  double dj[N];
#pragma unroll
  for (int q = 0; q < N; ++q) dj[q] = Dr[j * PJ + q];
  const double* gp = g + base;
  double2 gn[6];
#pragma unroll
  for (int m = 0; m < 6; ++m) gn[m] = __ldg(reinterpret_cast<const double2*>(gp + m * gstride));
  __syncwarp();

#pragma unroll 1
  for (int i = 0; i < N; ++i) {
    double2 gv[6];
#pragma unroll
    for (int m = 0; m < 6; ++m) gv[m] = gn[m];
    if (i + 1 < N) {
#pragma unroll
      for (int m = 0; m < 6; ++m)
        gn[m] = __ldg(reinterpret_cast<const double2*>(gp + (i + 1) * NN + m * gstride));
    }
    double ar0 = 0.0, ar1 = 0.0, as0 = 0.0, as1 = 0.0, at0 = 0.0, at1 = 0.0;
#pragma unroll
    for (int q = 0; q < N; ++q) {
      const double dq = Dr[i * PJ + q];
      ar0 = mac<EX>(ar0, dq, um0[q]);
      ar1 = mac<EX>(ar1, dq, um1[q]);
      const double2 sv = *reinterpret_cast<const double2*>(su + i * LAY + q * PJ + k0);
      as0 = mac<EX>(as0, dj[q], sv.x);
      as1 = mac<EX>(as1, dj[q], sv.y);
    }
#pragma unroll
    for (int q = 0; q < N; q += 2) {
      const double2 tv = *reinterpret_cast<const double2*>(su + i * LAY + j * PJ + q);
      const double2 da = *reinterpret_cast<const double2*>(Dr + k0 * PJ + q);
      const double2 db = *reinterpret_cast<const double2*>(Dr + (k0 + 1) * PJ + q);
      at0 = mac<EX>(at0, da.x, tv.x);
      at1 = mac<EX>(at1, db.x, tv.x);
      at0 = mac<EX>(at0, da.y, tv.y);
      at1 = mac<EX>(at1, db.y, tv.y);
    }
    double2 v1, v2, v3;
    v1.x = add<EX>(add<EX>(mul<EX>(gv[0].x, ar0), mul<EX>(gv[1].x, as0)), mul<EX>(gv[2].x, at0));
    v1.y = add<EX>(add<EX>(mul<EX>(gv[0].y, ar1), mul<EX>(gv[1].y, as1)), mul<EX>(gv[2].y, at1));
    v2.x = add<EX>(add<EX>(mul<EX>(gv[1].x, ar0), mul<EX>(gv[3].x, as0)), mul<EX>(gv[4].x, at0));
    v2.y = add<EX>(add<EX>(mul<EX>(gv[1].y, ar1), mul<EX>(gv[3].y, as1)), mul<EX>(gv[4].y, at1));
    v3.x = add<EX>(add<EX>(mul<EX>(gv[2].x, ar0), mul<EX>(gv[4].x, as0)), mul<EX>(gv[5].x, at0));
    v3.y = add<EX>(add<EX>(mul<EX>(gv[2].y, ar1), mul<EX>(gv[4].y, as1)), mul<EX>(gv[5].y, at1));
    *reinterpret_cast<double2*>(s1 + i * LAY + sjk) = v1;
    *reinterpret_cast<double2*>(s2 + i * LAY + sjk) = v2;
    __syncwarp();  // every lane has read u layer i
    *reinterpret_cast<double2*>(su + i * LAY + sjk) = v3;
  }
#pragma unroll
  for (int q = 0; q < N; ++q) dj[q] = Dc[j * PJ + q];  // column j of D
  __syncwarp();

  const bool mass = lm != 0.0;
#pragma unroll 1
  for (int i = 0; i < N; ++i) {
    double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
    for (int q = 0; q < N; q += 2) {
      const double2 t3 = *reinterpret_cast<const double2*>(su + i * LAY + j * PJ + q);
      const double2 ca = *reinterpret_cast<const double2*>(Dc + k0 * PJ + q);        // D[q..q+1][k0]
      const double2 cb = *reinterpret_cast<const double2*>(Dc + (k0 + 1) * PJ + q);  // D[q..q+1][k0+1]
      const double2 ci = *reinterpret_cast<const double2*>(Dc + i * PJ + q);         // D[q..q+1][i]
      const double2 ra = *reinterpret_cast<const double2*>(s1 + q * LAY + sjk);
      const double2 rb = *reinterpret_cast<const double2*>(s1 + (q + 1) * LAY + sjk);
      const double2 sa = *reinterpret_cast<const double2*>(s2 + i * LAY + q * PJ + k0);
      const double2 sb = *reinterpret_cast<const double2*>(s2 + i * LAY + (q + 1) * PJ + k0);
      acc0 = mac<EX>(acc0, ci.x, ra.x);
      acc1 = mac<EX>(acc1, ci.x, ra.y);
      acc0 = mac<EX>(acc0, dj[q], sa.x);
      acc1 = mac<EX>(acc1, dj[q], sa.y);
      acc0 = mac<EX>(acc0, ca.x, t3.x);
      acc1 = mac<EX>(acc1, cb.x, t3.x);
      acc0 = mac<EX>(acc0, ci.y, rb.x);
      acc1 = mac<EX>(acc1, ci.y, rb.y);
      acc0 = mac<EX>(acc0, dj[q + 1], sb.x);
      acc1 = mac<EX>(acc1, dj[q + 1], sb.y);
      acc0 = mac<EX>(acc0, ca.y, t3.y);
      acc1 = mac<EX>(acc1, cb.y, t3.y);
    }
    double2 wv;
    wv.x = mul<EX>(lv, acc0);
    wv.y = mul<EX>(lv, acc1);
    if (mass) {
      const double2 bv = __ldg(reinterpret_cast<const double2*>(b + base + i * NN));
      const double2 uv = *reinterpret_cast<const double2*>(u + base + i * NN);
      double u0 = uv.x, u1 = uv.y;
      if constexpr (MASK) {
        const uint32_t wd = __ldg(inmask + e * 16 + 2 * i + wsel) >> bsh;
        if (!(wd & 1u)) u0 = 0.0;
        if (!(wd & 2u)) u1 = 0.0;
      }
      wv.x = add<EX>(wv.x, mul<EX>(mul<EX>(lm, bv.x), u0));
      wv.y = add<EX>(wv.y, mul<EX>(mul<EX>(lm, bv.y), u1));
    }
    if constexpr (MASK) {
      const uint32_t sel = __ldg(outsel + e * 16 + 2 * i + wsel) >> bsh;
      if ((sel & 3u) != 3u) {
        const double2 uv = __ldg(reinterpret_cast<const double2*>(u + base + i * NN));
        if (!(sel & 1u)) wv.x = uv.x;
        if (!(sel & 2u)) wv.y = uv.y;
      }
    }
    *reinterpret_cast<double2*>(w + base + i * NN) = wv;
  }
}

// grad_ref: three reference derivatives with separate sequential accumulators
// (`_numba.py:63-83`).
template <int N, bool EX>
__global__ void __launch_bounds__(AxCfg<N>::THREADS)
grad_ref_kernel(DMat<N> D, const double* __restrict__ u, double* __restrict__ ur,
                double* __restrict__ us, double* __restrict__ ut, long long E) {
  using C = AxCfg<N>;
  constexpr int NN = C::NN, NNN = C::NNN;
  __shared__ double us_[C::EPB][NNN];
  const int le = threadIdx.x / NN;
  const int t = threadIdx.x - le * NN;
  const int j = t / N, k = t - (t / N) * N;
  const long long e = (long long)blockIdx.x * C::EPB + le;
  const bool active = e < E;
  const long long base = e * NNN + t;
  double up[N];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    up[i] = active ? __ldg(u + base + i * NN) : 0.0;
    us_[le][i * NN + t] = up[i];
  }
  double dj[N], dk[N];
#pragma unroll
  for (int q = 0; q < N; ++q) {
    dj[q] = D.v[j * N + q];
    dk[q] = D.v[k * N + q];
  }
  __syncthreads();
  if (!active) return;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double ar = 0.0, as = 0.0, at = 0.0;
#pragma unroll
    for (int q = 0; q < N; ++q) {
      ar = mac<EX>(ar, D.v[i * N + q], up[q]);
      as = mac<EX>(as, dj[q], us_[le][i * NN + q * N + k]);
      at = mac<EX>(at, dk[q], us_[le][i * NN + j * N + q]);
    }
    ur[base + i * NN] = ar;
    us[base + i * NN] = as;
    ut[base + i * NN] = at;
  }
}

// apply_{r,s,t}: out = A (m x n) contracted along one axis, rectangular allowed.
// One block per element; the element and A sit in shared memory; each output
// point is one sequential dot over the contracted index (`_numba.py:15-60`).
// Elements may be non-cubic (d0, d1, d2): the dealiasing chain contracts one
// axis at a time from n to m points (operators.py:141-147).
template <int AXIS, bool EX>
__global__ void apply_axis_kernel(const double* __restrict__ a, int m, int d0, int d1, int d2,
                                  const double* __restrict__ u, double* __restrict__ out,
                                  long long E) {
  extern __shared__ double sm[];
  const int n = AXIS == 0 ? d0 : (AXIS == 1 ? d1 : d2);
  const int o0 = AXIS == 0 ? m : d0, o1 = AXIS == 1 ? m : d1, o2 = AXIS == 2 ? m : d2;
  double* as = sm;          // m*n
  double* ue = sm + m * n;  // d0*d1*d2
  const long long e = blockIdx.x;
  const int nin = d0 * d1 * d2;
  for (int x = threadIdx.x; x < m * n; x += blockDim.x) as[x] = a[x];
  for (int x = threadIdx.x; x < nin; x += blockDim.x) ue[x] = u[e * nin + x];
  __syncthreads();
  const int nout = o0 * o1 * o2;
  for (int x = threadIdx.x; x < nout; x += blockDim.x) {
    const int i0 = x / (o1 * o2), i1 = (x / o2) % o1, i2 = x % o2;
    double acc = 0.0;
    for (int q = 0; q < n; ++q) {
      double uv;
      int p;
      if (AXIS == 0) { p = i0; uv = ue[(q * d1 + i1) * d2 + i2]; }
      else if (AXIS == 1) { p = i1; uv = ue[(i0 * d1 + q) * d2 + i2]; }
      else { p = i2; uv = ue[(i0 * d1 + i1) * d2 + q]; }
      acc = mac<EX>(acc, as[p * n + q], uv);
    }
    out[e * nout + x] = acc;
  }
}

// ----------------------------------------------------------------------------
// host-side dispatch over the polynomial order

template <int N>
static DMat<N> load_dmat(const double* d_host) {
  DMat<N> D;
  for (int x = 0; x < N * N; ++x) D.v[x] = d_host[x];
  return D;
}

template <int N>
static int launch_ax(const double* d_host, const double* g, const double* b, const double* u,
                     double* w, long long E, double lv, double lm, const uint32_t* inmask,
                     const uint32_t* outsel, int exact, cudaStream_t st, const double* pre) {
  using C = AxCfg<N>;
  if (E <= 0) return SF_OK;
  DMat<N> D = load_dmat<N>(d_host);
  dim3 grid((unsigned)((E + C::EPB - 1) / C::EPB));
  const bool masked = inmask != nullptr;
  if constexpr (N == 8) {
    if (g_ax_kernel == 1) {
      const int r = ax_helm8t(D, g, b, u, w, E, 0, E, lv, lm, inmask, outsel, pre, exact, st);
      if (r != SF_ERR_UNSUPPORTED) return r;
    }
  }
  if (pre != nullptr) {
    // fused Jacobi scaling: n = 8 swizzled kernel only
    if constexpr (N == 8) {
      dim3 g8((unsigned)((E + 1) / 2));
      if (exact) {
        if (masked) launch8s<true, true, true>(g8, st, D, g, b, u, w, E, lv, lm, inmask, outsel, pre);
        else launch8s<true, false, true>(g8, st, D, g, b, u, w, E, lv, lm, nullptr, nullptr, pre);
      } else {
        if (masked) launch8s<false, true, true>(g8, st, D, g, b, u, w, E, lv, lm, inmask, outsel, pre);
        else launch8s<false, false, true>(g8, st, D, g, b, u, w, E, lv, lm, nullptr, nullptr, pre);
      }
      return check_launch("ax_helm8s_pre");
    } else {
      set_error("ax_helm: the fused pre-scaling is implemented for n = 8 only (got n = %d)", N);
      return SF_ERR_UNSUPPORTED;
    }
  }
  if constexpr (N == 8) {
#ifdef SF_AX_PENCIL2
    dim3 g8((unsigned)((E + AX8_EPB - 1) / AX8_EPB));
    if (exact) {
      if (masked) ax_helm_n8_kernel<true, true><<<g8, 32 * AX8_EPB, 0, st>>>(D, g, b, u, w, E, lv, lm, inmask, outsel);
      else ax_helm_n8_kernel<true, false><<<g8, 32 * AX8_EPB, 0, st>>>(D, g, b, u, w, E, lv, lm, nullptr, nullptr);
    } else {
      if (masked) ax_helm_n8_kernel<false, true><<<g8, 32 * AX8_EPB, 0, st>>>(D, g, b, u, w, E, lv, lm, inmask, outsel);
      else ax_helm_n8_kernel<false, false><<<g8, 32 * AX8_EPB, 0, st>>>(D, g, b, u, w, E, lv, lm, nullptr, nullptr);
    }
    return check_launch("ax_helm_n8");
#elif !defined(SF_AX8_UNSWIZZLED)
    dim3 g8((unsigned)((E + 1) / 2));
    if (exact) {
      if (masked) launch8s<true, true, false>(g8, st, D, g, b, u, w, E, lv, lm, inmask, outsel, nullptr);
      else launch8s<true, false, false>(g8, st, D, g, b, u, w, E, lv, lm, nullptr, nullptr, nullptr);
    } else {
      if (masked) launch8s<false, true, false>(g8, st, D, g, b, u, w, E, lv, lm, inmask, outsel, nullptr);
      else launch8s<false, false, false>(g8, st, D, g, b, u, w, E, lv, lm, nullptr, nullptr, nullptr);
    }
    return check_launch("ax_helm8s");
#endif
  }
  if (exact) {
    if (masked) ax_helm_kernel<N, true, true><<<grid, C::THREADS, 0, st>>>(D, g, b, u, w, E, lv, lm, inmask, outsel);
    else ax_helm_kernel<N, true, false><<<grid, C::THREADS, 0, st>>>(D, g, b, u, w, E, lv, lm, nullptr, nullptr);
  } else {
    if (masked) ax_helm_kernel<N, false, true><<<grid, C::THREADS, 0, st>>>(D, g, b, u, w, E, lv, lm, inmask, outsel);
    else ax_helm_kernel<N, false, false><<<grid, C::THREADS, 0, st>>>(D, g, b, u, w, E, lv, lm, nullptr, nullptr);
  }
  return check_launch("ax_helm");
}

template <int N>
static int launch_grad(const double* d_host, const double* u, double* ur, double* us, double* ut,
                       long long E, int exact, cudaStream_t st) {
  using C = AxCfg<N>;
  if (E <= 0) return SF_OK;
  DMat<N> D = load_dmat<N>(d_host);
  dim3 grid((unsigned)((E + C::EPB - 1) / C::EPB));
  if (exact) grad_ref_kernel<N, true><<<grid, C::THREADS, 0, st>>>(D, u, ur, us, ut, E);
  else grad_ref_kernel<N, false><<<grid, C::THREADS, 0, st>>>(D, u, ur, us, ut, E);
  return check_launch("grad_ref");
}

#define SF_DISPATCH_N(n, CALL)                          \
  switch (n) {                                          \
    case 2: return CALL(2); case 3: return CALL(3);     \
    case 4: return CALL(4); case 5: return CALL(5);     \
    case 6: return CALL(6); case 7: return CALL(7);     \
    case 8: return CALL(8); case 9: return CALL(9);     \
    case 10: return CALL(10);                           \
    default: set_error("polynomial size n=%d unsupported (2..10)", n); return SF_ERR_UNSUPPORTED; \
  }

int ax_helm(const double* d_host, int n, const double* g, const double* b, const double* u,
            double* w, long long E, double lv, double lm, const uint32_t* inmask,
            const uint32_t* outsel, int exact, cudaStream_t st, const double* pre) {
  if ((inmask == nullptr) != (outsel == nullptr)) {
    set_error("ax_helm: inmask and outsel must both be given or both be null");
    return SF_ERR_ARG;
  }
#define CALL(NV) launch_ax<NV>(d_host, g, b, u, w, E, lv, lm, inmask, outsel, exact, st, pre)
  SF_DISPATCH_N(n, CALL)
#undef CALL
}

int grad_ref(const double* d_host, int n, const double* u, double* ur, double* us, double* ut,
             long long E, int exact, cudaStream_t st) {
#define CALL(NV) launch_grad<NV>(d_host, u, ur, us, ut, E, exact, st)
  SF_DISPATCH_N(n, CALL)
#undef CALL
}

int apply_axis3(int axis, const double* a, int m, int d0, int d1, int d2, const double* u, double* out,
                long long E, int exact, cudaStream_t st) {
  if (E <= 0) return SF_OK;
  const int n = axis == 0 ? d0 : (axis == 1 ? d1 : d2);
  if (axis < 0 || axis > 2 || m <= 0 || d0 <= 0 || d1 <= 0 || d2 <= 0) {
    set_error("apply_axis: bad axis/shape (%d; %d x [%d %d %d])", axis, m, d0, d1, d2);
    return SF_ERR_ARG;
  }
  size_t smem = sizeof(double) * ((size_t)m * n + (size_t)d0 * d1 * d2);
  if (smem > 200 * 1024) {
    set_error("apply_axis: element too large for shared memory");
    return SF_ERR_UNSUPPORTED;
  }
  if (smem > 48 * 1024) {
    cudaFuncSetAttribute(apply_axis_kernel<0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(apply_axis_kernel<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(apply_axis_kernel<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(apply_axis_kernel<0, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(apply_axis_kernel<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(apply_axis_kernel<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  dim3 grid((unsigned)E);
  int threads = 128;
#define SF_AXIS_LAUNCH(AX, EXV) \
  apply_axis_kernel<AX, EXV><<<grid, threads, smem, st>>>(a, m, d0, d1, d2, u, out, E)
  if (exact) {
    if (axis == 0) SF_AXIS_LAUNCH(0, true);
    else if (axis == 1) SF_AXIS_LAUNCH(1, true);
    else SF_AXIS_LAUNCH(2, true);
  } else {
    if (axis == 0) SF_AXIS_LAUNCH(0, false);
    else if (axis == 1) SF_AXIS_LAUNCH(1, false);
    else SF_AXIS_LAUNCH(2, false);
  }
#undef SF_AXIS_LAUNCH
  return check_launch("apply_axis");
}

int apply_axis(int axis, const double* a, int m, int n, const double* u, double* out, long long E,
               int exact, cudaStream_t st) {
  return apply_axis3(axis, a, m, n, n, n, u, out, E, exact, st);
}

}  // namespace sf
