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
#if !defined(SF_AX8_UNSWIZZLED)
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
