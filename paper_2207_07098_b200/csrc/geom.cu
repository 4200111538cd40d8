// Function-space setup on the device: GLL coordinates and geometric factors.
//
// Reference semantics (space.py):
//   _trilinear_coords  :182-192  coords[l,e,i,j,k] = sum_c corners[e,c,l] * wc[c,i,j,k]
//                                (numpy einsum without optimize accumulates c = 0..7
//                                 sequentially from 0.0 -- reproduced bit-for-bit)
//   build_space        :214-245  xr via apply_{r,s,t}(D, coords[l]); c12, c20, c01 by
//                                np.cross; jac = sum_l a0[l] c12[l]; rx = [c12,c20,c01]/jac;
//                                bm = (w_i w_j) w_k * jac; geom[m] = bm * sum_l rx[s,l] rx[t,l]
// Every operation here is issued without contraction (EX arithmetic) so the
// device-built geometry is bit-identical to a numba-lane build_space: the GLL
// coordinates decide the gather-scatter numbering (which must be bit-exact) and
// exact metrics make the whole operator chain comparable bit-for-bit.
#include "common.cuh"

namespace sf {

// corners: (E, 8, 3) ; wc: (8, NNN) ; coords: (3, E, NNN)
__global__ void trilinear_coords_kernel(const double* __restrict__ corners,
                                        const double* __restrict__ wc, int nnn, long long E,
                                        double* __restrict__ coords) {
  const long long total = E * nnn;
  for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < total;
       x += (long long)gridDim.x * blockDim.x) {
    const long long e = x / nnn;
    const int p = (int)(x - e * nnn);
#pragma unroll
    for (int l = 0; l < 3; ++l) {
      double acc = 0.0;
#pragma unroll
      for (int c = 0; c < 8; ++c)
        acc = __dadd_rn(acc, __dmul_rn(corners[(e * 8 + c) * 3 + l], wc[c * nnn + p]));
      coords[l * total + x] = acc;
    }
  }
}

template <int N>
struct GM {
  double d[N * N];
  double w3[N * N * N];
};

// one block (n^3 threads) per element
template <int N>
__global__ void __launch_bounds__(N * N * N)
metrics_kernel(GM<N> G, const double* __restrict__ coords, long long E, double* __restrict__ rx,
               double* __restrict__ jac, double* __restrict__ bm, double* __restrict__ geom) {
  constexpr int NN = N * N, NNN = N * N * N;
  __shared__ double xs[3][NNN];
  const long long e = blockIdx.x;
  const long long PT = E * NNN;
  const int x = threadIdx.x;
  const long long p = e * NNN + x;
#pragma unroll
  for (int l = 0; l < 3; ++l) xs[l][x] = coords[l * PT + p];
  __syncthreads();
  const int i = x / NN, j = (x / N) % N, k = x % N;
  double a[3][3];  // a[s][l] = dx_l / dr_s  (= xr[l, s])
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    double ar = 0.0, as = 0.0, at = 0.0;
#pragma unroll
    for (int q = 0; q < N; ++q) {
      ar = __dadd_rn(ar, __dmul_rn(G.d[i * N + q], xs[l][q * NN + j * N + k]));
      as = __dadd_rn(as, __dmul_rn(G.d[j * N + q], xs[l][i * NN + q * N + k]));
      at = __dadd_rn(at, __dmul_rn(G.d[k * N + q], xs[l][i * NN + j * N + q]));
    }
    a[0][l] = ar;
    a[1][l] = as;
    a[2][l] = at;
  }
  // np.cross(u, v): (u1 v2 - u2 v1, u2 v0 - u0 v2, u0 v1 - u1 v0)
  auto cross = [](const double* u, const double* v, double* c) {
    c[0] = __dsub_rn(__dmul_rn(u[1], v[2]), __dmul_rn(u[2], v[1]));
    c[1] = __dsub_rn(__dmul_rn(u[2], v[0]), __dmul_rn(u[0], v[2]));
    c[2] = __dsub_rn(__dmul_rn(u[0], v[1]), __dmul_rn(u[1], v[0]));
  };
  double c[3][3];  // c[s] = reciprocal vector s (rows of the inverse Jacobian * J)
  cross(a[1], a[2], c[0]);
  cross(a[2], a[0], c[1]);
  cross(a[0], a[1], c[2]);
  double J = 0.0;
#pragma unroll
  for (int l = 0; l < 3; ++l) J = __dadd_rn(J, __dmul_rn(a[0][l], c[0][l]));
  jac[p] = J;
  double r[3][3];
#pragma unroll
  for (int s = 0; s < 3; ++s)
#pragma unroll
    for (int l = 0; l < 3; ++l) {
      r[s][l] = __ddiv_rn(c[s][l], J);
      rx[(s * 3 + l) * PT + p] = r[s][l];
    }
  const double b = __dmul_rn(G.w3[x], J);
  bm[p] = b;
  const int ps[6] = {0, 0, 0, 1, 1, 2}, pt[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
  for (int m = 0; m < 6; ++m) {
    double acc = 0.0;
#pragma unroll
    for (int l = 0; l < 3; ++l) acc = __dadd_rn(acc, __dmul_rn(r[ps[m]][l], r[pt[m]][l]));
    geom[m * PT + p] = __dmul_rn(b, acc);
  }
}

int trilinear_coords(const double* corners, const double* wc, int n, long long E, double* coords,
                     cudaStream_t st) {
  if (E <= 0) return SF_OK;
  const int nnn = n * n * n;
  long long total = E * nnn;
  long long blocks = (total + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  trilinear_coords_kernel<<<(unsigned)blocks, 256, 0, st>>>(corners, wc, nnn, E, coords);
  return check_launch("trilinear_coords");
}

template <int N>
static int launch_metrics(const double* d_host, const double* w_host, const double* coords,
                          long long E, double* rx, double* jac, double* bm, double* geom,
                          cudaStream_t st) {
  if (E <= 0) return SF_OK;
  GM<N> G;
  for (int x = 0; x < N * N; ++x) G.d[x] = d_host[x];
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < N; ++j)
      for (int k = 0; k < N; ++k) {
        volatile double wij = w_host[i] * w_host[j];  // (w_i w_j) w_k, numpy broadcast order
        G.w3[(i * N + j) * N + k] = wij * w_host[k];
      }
  metrics_kernel<N><<<(unsigned)E, N * N * N, 0, st>>>(G, coords, E, rx, jac, bm, geom);
  return check_launch("metrics");
}

int metrics(const double* d_host, const double* w_host, int n, const double* coords, long long E,
            double* rx, double* jac, double* bm, double* geom, cudaStream_t st) {
  switch (n) {
#define C(NV) case NV: return launch_metrics<NV>(d_host, w_host, coords, E, rx, jac, bm, geom, st);
    C(2) C(3) C(4) C(5) C(6) C(7) C(8) C(9) C(10)
#undef C
    default: set_error("metrics: n=%d unsupported (2..10)", n); return SF_ERR_UNSUPPORTED;
  }
}

}  // namespace sf
