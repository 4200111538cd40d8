// Strong-form derivative operators (K3), weak divergence / cdtp (K4), the
// CFL reduction and the BDF/EXT history combination (K8).
//
// Reference semantics:
//   grad              operators.py:59-66   out[l] = rx[0,l]*ur + rx[1,l]*us + rx[2,l]*ut
//   div               operators.py:69-76   out = 0; out += (...) for l = 0, 1, 2
//   curl              operators.py:79-88
//   advect/advect_vec operators.py:108-126 (c0*g0 + c1*g1) + c2*g2 (collocation)
//   weak_grad_dot     operators.py:91-105  apply_r(D^T,f0) + apply_s(D^T,f1) + apply_t(D^T,f2)
//   cfl               operators.py:161-182
//   BDF/EXT sums      timestep.py:227-232
//
// All of these are element-local.  One block of n^3 threads handles one element
// (one thread per point); the element's input fields are staged in shared memory
// so the reference derivatives are shared-memory contractions.  rx is the
// (3, 3, E, n, n, n) array rx[s, l] = dr_s/dx_l.
#include "reduce.cuh"

namespace sf {

template <int N>
struct DM2 {
  double v[N * N];
};

template <int N, bool EX>
__device__ __forceinline__ void ref_derivs(const DM2<N>& D, const double* __restrict__ ue, int i,
                                           int j, int k, double& ar, double& as, double& at) {
  constexpr int NN = N * N;
  ar = 0.0; as = 0.0; at = 0.0;
#pragma unroll
  for (int q = 0; q < N; ++q) {
    ar = mac<EX>(ar, D.v[i * N + q], ue[q * NN + j * N + k]);
    as = mac<EX>(as, D.v[j * N + q], ue[i * NN + q * N + k]);
    at = mac<EX>(at, D.v[k * N + q], ue[i * NN + j * N + q]);
  }
}

// physical derivative d/dx_l from reference derivatives (operators.py:64-65);
// r[s][l] = rx[s, l] at this point, loaded before the shared-memory barrier so
// the nine metric loads overlap the element staging instead of stalling here
template <bool EX>
__device__ __forceinline__ double chain(const double (&r)[3][3], int l, double ar, double as, double at) {
  return add<EX>(add<EX>(mul<EX>(r[0][l], ar), mul<EX>(r[1][l], as)), mul<EX>(r[2][l], at));
}

enum DerivOp { OP_GRAD = 0, OP_DIV = 1, OP_CURL = 2, OP_ADVECT = 3 };

// in: NF fields of P points each (in[f] contiguous planes at stride P)
// OP_GRAD   in u          -> out[0..2]
// OP_DIV    in v0,v1,v2   -> out[0]
// OP_CURL   in v0,v1,v2   -> out[0..2]
// OP_ADVECT in v0,v1,v2 (advected), c in `c` -> out[0..2], times `sign`
template <int N, bool EX, int OP>
__global__ void __launch_bounds__(N * N * N)
deriv_kernel(DM2<N> D, const double* __restrict__ in, const double* __restrict__ c,
             const double* __restrict__ rx, double* __restrict__ out, long long E, double sign) {
  constexpr int NN = N * N, NNN = N * N * N;
  constexpr int NF = (OP == OP_GRAD) ? 1 : 3;
  __shared__ double ue[NF][NNN];
  const long long e = blockIdx.x;
  const long long PT = E * NNN;
  const int x = threadIdx.x;
  const long long p = e * NNN + x;
#pragma unroll
  for (int f = 0; f < NF; ++f) ue[f][x] = __ldg(in + f * PT + p);
  double r[3][3];
#pragma unroll
  for (int sl = 0; sl < 9; ++sl) r[sl / 3][sl % 3] = __ldg(rx + sl * PT + p);
  double c0 = 0.0, c1 = 0.0, c2 = 0.0;
  if constexpr (OP == OP_ADVECT) {
    c0 = __ldg(c + p);
    c1 = __ldg(c + PT + p);
    c2 = __ldg(c + 2 * PT + p);
  }
  __syncthreads();
  const int i = x / NN, j = (x / N) % N, k = x % N;
  if constexpr (OP == OP_GRAD) {
    double ar, as, at;
    ref_derivs<N, EX>(D, ue[0], i, j, k, ar, as, at);
#pragma unroll
    for (int l = 0; l < 3; ++l) out[l * PT + p] = chain<EX>(r, l, ar, as, at);
  } else if constexpr (OP == OP_DIV) {
    double acc = 0.0;
#pragma unroll
    for (int l = 0; l < 3; ++l) {
      double ar, as, at;
      ref_derivs<N, EX>(D, ue[l], i, j, k, ar, as, at);
      acc = add<EX>(acc, chain<EX>(r, l, ar, as, at));
    }
    out[p] = acc;
  } else if constexpr (OP == OP_CURL) {
    // g_f[m] = d v_f / d x_m ; only the six off-diagonal entries are needed
    double g[3][3];
#pragma unroll
    for (int f = 0; f < 3; ++f) {
      double ar, as, at;
      ref_derivs<N, EX>(D, ue[f], i, j, k, ar, as, at);
#pragma unroll
      for (int m = 0; m < 3; ++m) g[f][m] = (m == f) ? 0.0 : chain<EX>(r, m, ar, as, at);
    }
    out[0 * PT + p] = sub<EX>(g[2][1], g[1][2]);
    out[1 * PT + p] = sub<EX>(g[0][2], g[2][0]);
    out[2 * PT + p] = sub<EX>(g[1][0], g[0][1]);
  } else {  // OP_ADVECT
#pragma unroll
    for (int f = 0; f < 3; ++f) {
      double ar, as, at;
      ref_derivs<N, EX>(D, ue[f], i, j, k, ar, as, at);
      const double g0 = chain<EX>(r, 0, ar, as, at);
      const double g1 = chain<EX>(r, 1, ar, as, at);
      const double g2 = chain<EX>(r, 2, ar, as, at);
      const double a = add<EX>(add<EX>(mul<EX>(c0, g0), mul<EX>(c1, g1)), mul<EX>(c2, g2));
      out[f * PT + p] = sign * a;  // sign is +-1: exact
    }
  }
}

// weak_grad_dot: f_s = bm * (rx[s,0] w0 + rx[s,1] w1 + rx[s,2] w2);
// r = (apply_r(D^T, f0) + apply_s(D^T, f1)) + apply_t(D^T, f2)
template <int N, bool EX>
__global__ void __launch_bounds__(N * N * N)
cdtp_kernel(DM2<N> D, const double* __restrict__ w, const double* __restrict__ rx,
            const double* __restrict__ bm, double* __restrict__ out, long long E) {
  constexpr int NN = N * N, NNN = N * N * N;
  __shared__ double f[3][NNN];
  const long long e = blockIdx.x;
  const long long PT = E * NNN;
  const int x = threadIdx.x;
  const long long p = e * NNN + x;
  const double w0 = __ldg(w + p), w1 = __ldg(w + PT + p), w2 = __ldg(w + 2 * PT + p);
  const double b = __ldg(bm + p);
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    const double r0 = __ldg(rx + (s * 3 + 0) * PT + p);
    const double r1 = __ldg(rx + (s * 3 + 1) * PT + p);
    const double r2 = __ldg(rx + (s * 3 + 2) * PT + p);
    f[s][x] = mul<EX>(b, add<EX>(add<EX>(mul<EX>(r0, w0), mul<EX>(r1, w1)), mul<EX>(r2, w2)));
  }
  __syncthreads();
  const int i = x / NN, j = (x / N) % N, k = x % N;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll
  for (int q = 0; q < N; ++q) {
    a0 = mac<EX>(a0, D.v[q * N + i], f[0][q * NN + j * N + k]);
    a1 = mac<EX>(a1, D.v[q * N + j], f[1][i * NN + q * N + k]);
    a2 = mac<EX>(a2, D.v[q * N + k], f[2][i * NN + j * N + q]);
  }
  out[p] = add<EX>(add<EX>(a0, a1), a2);
}

// CFL: max_p sum_s |rx[s,0] v0 + rx[s,1] v1 + rx[s,2] v2| / dxi_s ; max is exact,
// so the atomicMax on the (non-negative) bit pattern is deterministic.
template <int N, bool EX>
__global__ void __launch_bounds__(N * N * N)
cfl_kernel(const double* __restrict__ v, const double* __restrict__ rx, DM2<N> dxi_pack,
           long long E, unsigned long long* __restrict__ out_bits) {
  constexpr int NN = N * N, NNN = N * N * N;
  const long long e = blockIdx.x;
  const long long PT = E * NNN;
  const int x = threadIdx.x;
  const long long p = e * NNN + x;
  const int idx[3] = {x / NN, (x / N) % N, x % N};
  const double v0 = __ldg(v + p), v1 = __ldg(v + PT + p), v2 = __ldg(v + 2 * PT + p);
  double total = 0.0;
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    const double r0 = __ldg(rx + (s * 3 + 0) * PT + p);
    const double r1 = __ldg(rx + (s * 3 + 1) * PT + p);
    const double r2 = __ldg(rx + (s * 3 + 2) * PT + p);
    const double uh = add<EX>(add<EX>(mul<EX>(r0, v0), mul<EX>(r1, v1)), mul<EX>(r2, v2));
    total = add<EX>(total, fabs(uh) / dxi_pack.v[idx[s]]);
  }
  // block max then one atomic per block
  __shared__ double red[NNN];
  red[x] = total;
  __syncthreads();
  for (int s = 1; s < NNN; s <<= 1) {
    if ((x % (2 * s)) == 0 && x + s < NNN) red[x] = fmax(red[x], red[x + s]);
    __syncthreads();
  }
  if (x == 0) atomicMax(out_bits, (unsigned long long)__double_as_longlong(red[0]));
}

// vhat_dt = sum_q (alpha_q/dt) v_q + beta_q nl_q ; omega = sum_q beta_q curl_q
// (timestep.py:227-232; accumulation starts from zeros and runs over q in order,
// the two updates of vhat_dt per q are separate roundings as in numpy)
struct BdfExtOp {
  static constexpr int K = 0;
  double* vhat;
  double* omega;
  const double* vel[3];
  const double* nl[3];
  const double* crl[3];
  double a_dt[3];
  double beta[3];
  int order;
  struct In { double v[3], n[3], c[3]; };
  __device__ void prologue() {}
  __device__ __forceinline__ In load(long long p, const double*) const {
    In in;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const bool on = q < order;
      in.v[q] = on ? __ldg(vel[q] + p) : 0.0;
      in.n[q] = on ? __ldg(nl[q] + p) : 0.0;
      in.c[q] = on ? __ldg(crl[q] + p) : 0.0;
    }
    return in;
  }
  __device__ __forceinline__ void finish(long long p, const In& in, double (&)[1]) const {
    double vh = 0.0, om = 0.0;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      if (q < order) {
        vh = __dadd_rn(vh, __dmul_rn(a_dt[q], in.v[q]));
        vh = __dadd_rn(vh, __dmul_rn(beta[q], in.n[q]));
        om = __dadd_rn(om, __dmul_rn(beta[q], in.c[q]));
      }
    }
    vhat[p] = vh;
    omega[p] = om;
  }
};

// ---------------------------------------------------------------- dispatch
template <int N>
static DM2<N> dm2(const double* h) {
  DM2<N> D;
  for (int x = 0; x < N * N; ++x) D.v[x] = h[x];
  return D;
}

template <int N>
static int launch_deriv(int op, const double* d_host, const double* in, const double* c,
                        const double* rx, double* out, long long E, double sign, int exact,
                        cudaStream_t st) {
  if (E <= 0) return SF_OK;
  DM2<N> D = dm2<N>(d_host);
  dim3 grid((unsigned)E), block(N * N * N);
#define L(EXV, OPV) deriv_kernel<N, EXV, OPV><<<grid, block, 0, st>>>(D, in, c, rx, out, E, sign)
  if (exact) {
    switch (op) {
      case OP_GRAD: L(true, OP_GRAD); break;
      case OP_DIV: L(true, OP_DIV); break;
      case OP_CURL: L(true, OP_CURL); break;
      case OP_ADVECT: L(true, OP_ADVECT); break;
      default: set_error("deriv: bad op %d", op); return SF_ERR_ARG;
    }
  } else {
    switch (op) {
      case OP_GRAD: L(false, OP_GRAD); break;
      case OP_DIV: L(false, OP_DIV); break;
      case OP_CURL: L(false, OP_CURL); break;
      case OP_ADVECT: L(false, OP_ADVECT); break;
      default: set_error("deriv: bad op %d", op); return SF_ERR_ARG;
    }
  }
#undef L
  return check_launch("deriv");
}

template <int N>
static int launch_cdtp(const double* d_host, const double* w, const double* rx, const double* bm,
                       double* out, long long E, int exact, cudaStream_t st) {
  if (E <= 0) return SF_OK;
  DM2<N> D = dm2<N>(d_host);
  if (exact) cdtp_kernel<N, true><<<(unsigned)E, N * N * N, 0, st>>>(D, w, rx, bm, out, E);
  else cdtp_kernel<N, false><<<(unsigned)E, N * N * N, 0, st>>>(D, w, rx, bm, out, E);
  return check_launch("cdtp");
}

template <int N>
static int launch_cfl(const double* v, const double* rx, const double* dxi, long long E,
                      unsigned long long* out_bits, int exact, cudaStream_t st) {
  if (E <= 0) return SF_OK;
  DM2<N> X;
  for (int x = 0; x < N * N; ++x) X.v[x] = x < N ? dxi[x] : 0.0;
  if (exact) cfl_kernel<N, true><<<(unsigned)E, N * N * N, 0, st>>>(v, rx, X, E, out_bits);
  else cfl_kernel<N, false><<<(unsigned)E, N * N * N, 0, st>>>(v, rx, X, E, out_bits);
  return check_launch("cfl");
}

#define SF_DISPATCH_N2(n, CALL)                          \
  switch (n) {                                           \
    case 2: return CALL(2); case 3: return CALL(3);      \
    case 4: return CALL(4); case 5: return CALL(5);      \
    case 6: return CALL(6); case 7: return CALL(7);      \
    case 8: return CALL(8); case 9: return CALL(9);      \
    case 10: return CALL(10);                            \
    default: set_error("polynomial size n=%d unsupported (2..10)", n); return SF_ERR_UNSUPPORTED; \
  }

int deriv(int op, const double* d_host, int n, const double* in, const double* c, const double* rx,
          double* out, long long E, double sign, int exact, cudaStream_t st) {
#define CALL(NV) launch_deriv<NV>(op, d_host, in, c, rx, out, E, sign, exact, st)
  SF_DISPATCH_N2(n, CALL)
#undef CALL
}

int cdtp(const double* d_host, int n, const double* w, const double* rx, const double* bm,
         double* out, long long E, int exact, cudaStream_t st) {
#define CALL(NV) launch_cdtp<NV>(d_host, w, rx, bm, out, E, exact, st)
  SF_DISPATCH_N2(n, CALL)
#undef CALL
}

int cfl_max(const double* v, const double* rx, const double* dxi_host, int n, long long E,
            unsigned long long* out_bits, int exact, cudaStream_t st) {
#define CALL(NV) launch_cfl<NV>(v, rx, dxi_host, E, out_bits, exact, st)
  SF_DISPATCH_N2(n, CALL)
#undef CALL
}

int bdf_ext(double* vhat, double* omega, const double* const* vel, const double* const* nl,
            const double* const* crl, const double* a_dt, const double* beta, int order,
            long long P3, cudaStream_t st) {
  if (order < 1 || order > 3) { set_error("bdf_ext: order %d", order); return SF_ERR_ARG; }
  BdfExtOp op{};
  op.vhat = vhat;
  op.omega = omega;
  for (int q = 0; q < 3; ++q) {
    op.vel[q] = q < order ? vel[q] : nullptr;
    op.nl[q] = q < order ? nl[q] : nullptr;
    op.crl[q] = q < order ? crl[q] : nullptr;
    op.a_dt[q] = q < order ? a_dt[q] : 0.0;
    op.beta[q] = q < order ? beta[q] : 0.0;
  }
  op.order = order;
  RedWork none{nullptr, nullptr};
  return launch_map_reduce(op, P3, none, nullptr, st, "bdf_ext");
}

}  // namespace sf
