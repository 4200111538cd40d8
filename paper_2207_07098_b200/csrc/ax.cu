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
#include "common.cuh"

namespace sf {

template <int N>
struct DMat {
  double v[N * N];
};

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
template <int N, bool EX, bool MASK>
__global__ void __launch_bounds__(AxCfg<N>::THREADS)
ax_helm_kernel(DMat<N> D, const double* __restrict__ g, const double* __restrict__ b,
               const double* __restrict__ u, double* __restrict__ w, long long E, double lv,
               double lm, const uint32_t* __restrict__ inmask,
               const uint32_t* __restrict__ outsel) {
  using C = AxCfg<N>;
  constexpr int NN = C::NN, NNN = C::NNN;
  __shared__ double us_[C::EPB][NNN];
  __shared__ double f2s[C::EPB][NNN];
  __shared__ double f3s[C::EPB][NNN];

  const int le = threadIdx.x / NN;
  const int t = threadIdx.x - le * NN;
  const int j = t / N, k = t - (t / N) * N;
  const long long e = (long long)blockIdx.x * C::EPB + le;
  const bool active = e < E;
  const long long base = e * NNN + t;
  const long long gstride = E * (long long)NNN;

  double up[N];   // original pencil (kept for the masked output select)
  double um[N];   // masked pencil the operator acts on
#pragma unroll
  for (int i = 0; i < N; ++i) {
    up[i] = active ? __ldg(u + base + i * NN) : 0.0;
    bool in = true;
    if constexpr (MASK) in = active && mask_bit(inmask, e, C::WPE, i * NN + t);
    um[i] = in ? up[i] : 0.0;
    us_[le][i * NN + t] = um[i];
  }
  double dj[N], dk[N];
#pragma unroll
  for (int q = 0; q < N; ++q) {
    dj[q] = D.v[j * N + q];
    dk[q] = D.v[k * N + q];
  }
  __syncthreads();

  double f1[N];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double ar = 0.0, as = 0.0, at = 0.0;
#pragma unroll
    for (int q = 0; q < N; ++q) {
      ar = mac<EX>(ar, D.v[i * N + q], um[q]);
      as = mac<EX>(as, dj[q], us_[le][i * NN + q * N + k]);
      at = mac<EX>(at, dk[q], us_[le][i * NN + j * N + q]);
    }
    double g0 = 0, g1 = 0, g2 = 0, g3 = 0, g4 = 0, g5 = 0;
    if (active) {
      const double* gp = g + base + i * NN;
      g0 = __ldg(gp);
      g1 = __ldg(gp + gstride);
      g2 = __ldg(gp + 2 * gstride);
      g3 = __ldg(gp + 3 * gstride);
      g4 = __ldg(gp + 4 * gstride);
      g5 = __ldg(gp + 5 * gstride);
    }
    // (g0*gr + g1*gs) + g2*gt, as written in _numba.py:116-118
    f1[i] = add<EX>(add<EX>(mul<EX>(g0, ar), mul<EX>(g1, as)), mul<EX>(g2, at));
    f2s[le][i * NN + t] = add<EX>(add<EX>(mul<EX>(g1, ar), mul<EX>(g3, as)), mul<EX>(g4, at));
    f3s[le][i * NN + t] = add<EX>(add<EX>(mul<EX>(g2, ar), mul<EX>(g4, as)), mul<EX>(g5, at));
  }
#pragma unroll
  for (int q = 0; q < N; ++q) {  // columns of D for the transposed contraction
    dj[q] = D.v[q * N + j];
    dk[q] = D.v[q * N + k];
  }
  __syncthreads();
  if (!active) return;

  const bool mass = lm != 0.0;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < N; ++q) {
      acc = mac<EX>(acc, D.v[q * N + i], f1[q]);
      acc = mac<EX>(acc, dj[q], f2s[le][i * NN + q * N + k]);
      acc = mac<EX>(acc, dk[q], f3s[le][i * NN + j * N + q]);
    }
    double wv = mul<EX>(lv, acc);
    if (mass) wv = add<EX>(wv, mul<EX>(mul<EX>(lm, __ldg(b + base + i * NN)), um[i]));
    if constexpr (MASK) {
      if (!mask_bit(outsel, e, C::WPE, i * NN + t)) wv = up[i];
    }
    w[base + i * NN] = wv;
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
template <int AXIS, bool EX>
__global__ void apply_axis_kernel(const double* __restrict__ a, int m, int n,
                                  const double* __restrict__ u, double* __restrict__ out,
                                  long long E) {
  extern __shared__ double sm[];
  double* as = sm;          // m*n
  double* ue = sm + m * n;  // n^3
  const long long e = blockIdx.x;
  const int nnn = n * n * n;
  for (int x = threadIdx.x; x < m * n; x += blockDim.x) as[x] = a[x];
  for (int x = threadIdx.x; x < nnn; x += blockDim.x) ue[x] = u[e * nnn + x];
  __syncthreads();
  const int nout = m * n * n;
  for (int x = threadIdx.x; x < nout; x += blockDim.x) {
    int i0, i1, i2;  // output index (d0, d1, d2) with the contracted axis of extent m
    if (AXIS == 0) { i0 = x / (n * n); i1 = (x / n) % n; i2 = x % n; }
    else if (AXIS == 1) { i0 = x / (m * n); i1 = (x / n) % m; i2 = x % n; }
    else { i0 = x / (n * m); i1 = (x / m) % n; i2 = x % m; }
    double acc = 0.0;
    for (int q = 0; q < n; ++q) {
      double uv;
      int p;
      if (AXIS == 0) { p = i0; uv = ue[(q * n + i1) * n + i2]; }
      else if (AXIS == 1) { p = i1; uv = ue[(i0 * n + q) * n + i2]; }
      else { p = i2; uv = ue[(i0 * n + i1) * n + q]; }
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
                     const uint32_t* outsel, int exact, cudaStream_t st) {
  using C = AxCfg<N>;
  if (E <= 0) return SF_OK;
  DMat<N> D = load_dmat<N>(d_host);
  dim3 grid((unsigned)((E + C::EPB - 1) / C::EPB));
  const bool masked = inmask != nullptr;
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
            const uint32_t* outsel, int exact, cudaStream_t st) {
  if ((inmask == nullptr) != (outsel == nullptr)) {
    set_error("ax_helm: inmask and outsel must both be given or both be null");
    return SF_ERR_ARG;
  }
#define CALL(NV) launch_ax<NV>(d_host, g, b, u, w, E, lv, lm, inmask, outsel, exact, st)
  SF_DISPATCH_N(n, CALL)
#undef CALL
}

int grad_ref(const double* d_host, int n, const double* u, double* ur, double* us, double* ut,
             long long E, int exact, cudaStream_t st) {
#define CALL(NV) launch_grad<NV>(d_host, u, ur, us, ut, E, exact, st)
  SF_DISPATCH_N(n, CALL)
#undef CALL
}

int apply_axis(int axis, const double* a, int m, int n, const double* u, double* out, long long E,
               int exact, cudaStream_t st) {
  if (E <= 0) return SF_OK;
  if (axis < 0 || axis > 2 || m <= 0 || n <= 0) {
    set_error("apply_axis: bad axis/shape (%d, %d, %d)", axis, m, n);
    return SF_ERR_ARG;
  }
  size_t smem = sizeof(double) * ((size_t)m * n + (size_t)n * n * n);
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
  if (exact) {
    if (axis == 0) apply_axis_kernel<0, true><<<grid, threads, smem, st>>>(a, m, n, u, out, E);
    else if (axis == 1) apply_axis_kernel<1, true><<<grid, threads, smem, st>>>(a, m, n, u, out, E);
    else apply_axis_kernel<2, true><<<grid, threads, smem, st>>>(a, m, n, u, out, E);
  } else {
    if (axis == 0) apply_axis_kernel<0, false><<<grid, threads, smem, st>>>(a, m, n, u, out, E);
    else if (axis == 1) apply_axis_kernel<1, false><<<grid, threads, smem, st>>>(a, m, n, u, out, E);
    else apply_axis_kernel<2, false><<<grid, threads, smem, st>>>(a, m, n, u, out, E);
  }
  return check_launch("apply_axis");
}

}  // namespace sf
