// Over-integrated convective term in one launch (reference operators.py:129-158,
// Dealias.advect via advect_vec, :119-126):
//
//   out_f = sign * project_back(wjac_f * sum_l to_fine(c_l) * to_fine(grad_l v_f)) / bm
//
// to_fine = apply_t(J, apply_s(J, apply_r(J, .))) with J the n -> m = ceil(3n/2)
// Gauss-Legendre interpolation matrix, project_back the same with J^T.  The
// unfused chain moves seven m^3 fields per component through HBM (m^3 / n^3 =
// 3.4x a GLL field each); here one CTA takes one element: c interpolated once into
// shared memory, then per component the GLL gradient (chain rule with rx), three
// interpolations, the fine-grid product, the weighting and the projection, all in
// shared memory.  HBM sees c, v, rx, wjac_f, bm once and out once.
//
// Every contraction is one thread's sequential sum over the contracted index in
// ascending order, starting from 0.0 -- the numba lane's loop (kernels/_numba.py
// apply_r/s/t) -- and the products / sums between stages are those of the
// reference expression, so EX=true is bit-identical to the reference chain.
#include "common.cuh"

namespace sf {

template <int N, int M>
struct DealiasMats {
  double D[N * N];   // GLL derivative
  double J[M * N];   // GLL -> GL interpolation, row p = J[p * N + i]
  double Jt[N * M];  // its transpose (projection), row a = Jt[a * M + p]
};

// In a contraction the output index p of the matrix row varies fastest across
// the threads of a warp for the t axis (and every few threads for s): the
// matrix is read column-major there, mat_cm[i * R + p], so a warp's lanes hit
// consecutive addresses instead of one row stride apart (6-way bank conflicts
// at R = 12, N = 8).

// smem layout (doubles): cf 3 m^3 | fine m^3 | tf m^3 | t1 max(m n n, n m m) |
// t2 max(m m n, n n m) | u n^3 | g 3 n^3
template <int N, int M>
__host__ __device__ constexpr int dealias_smem_doubles() {
  constexpr int MN = (M * N * N > N * M * M) ? M * N * N : N * M * M;
  constexpr int MM = (M * M * N > N * N * M) ? M * M * N : N * N * M;
  return 5 * M * M * M + MN + MM + 4 * N * N * N;
}

// out (A, B, C) with A = rows of mat applied on axis `axis` of in (I0, I1, I2):
// three specialisations written out so every loop bound is a constant
template <int R, int I0, int I1, int I2, bool EX>
__device__ __forceinline__ void contract_r(const double* __restrict__ mat, const double* __restrict__ in,
                                           double* __restrict__ out) {
  // out[p, j, k] = sum_i mat[p, i] in[i, j, k]
  for (int x = threadIdx.x; x < R * I1 * I2; x += blockDim.x) {
    const int p = x / (I1 * I2), jk = x - p * (I1 * I2);
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < I0; ++i) s = mac<EX>(s, mat[p * I0 + i], in[i * I1 * I2 + jk]);
    out[x] = s;
  }
}
template <int R, int I0, int I1, int I2, bool EX>
__device__ __forceinline__ void contract_s(const double* __restrict__ mat_cm, const double* __restrict__ in,
                                           double* __restrict__ out) {
  // out[i, p, k] = sum_j mat[p, j] in[i, j, k]   (mat column-major: mat_cm[j * R + p])
  for (int x = threadIdx.x; x < I0 * R * I2; x += blockDim.x) {
    const int i = x / (R * I2), rem = x - i * (R * I2), p = rem / I2, k = rem - p * I2;
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < I1; ++j) s = mac<EX>(s, mat_cm[j * R + p], in[(i * I1 + j) * I2 + k]);
    out[x] = s;
  }
}
template <int R, int I0, int I1, int I2, bool EX>
__device__ __forceinline__ void contract_t(const double* __restrict__ mat_cm, const double* __restrict__ in,
                                           double* __restrict__ out) {
  // out[i, j, p] = sum_k mat[p, k] in[i, j, k]   (mat column-major: mat_cm[k * R + p])
  for (int x = threadIdx.x; x < I0 * I1 * R; x += blockDim.x) {
    const int ij = x / R, p = x - ij * R;
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < I2; ++k) s = mac<EX>(s, mat_cm[k * R + p], in[ij * I2 + k]);
    out[x] = s;
  }
}

template <int N, int M, bool EX>
__device__ __forceinline__ void to_fine(const double* J, const double* Jcm, const double* in, double* t1,
                                        double* t2, double* out) {
  contract_r<M, N, N, N, EX>(J, in, t1);
  __syncthreads();
  contract_s<M, M, N, N, EX>(Jcm, t1, t2);
  __syncthreads();
  contract_t<M, M, M, N, EX>(Jcm, t2, out);
  __syncthreads();
}

template <int N, int M, bool EX>
__global__ void __launch_bounds__(512) dealias_advect_kernel(DealiasMats<N, M> mats, const double* __restrict__ c,
                                                             const double* __restrict__ v,
                                                             const double* __restrict__ rx,
                                                             const double* __restrict__ wjf,
                                                             const double* __restrict__ bm, long long E, double sign,
                                                             double* __restrict__ out) {
  constexpr int NNN = N * N * N, MMM = M * M * M;
  constexpr int MN = (M * N * N > N * M * M) ? M * N * N : N * M * M;
  constexpr int MM = (M * M * N > N * N * M) ? M * M * N : N * N * M;
  extern __shared__ double sm[];
  double* cf = sm;                 // 3 MMM
  double* fine = cf + 3 * MMM;     // MMM
  double* tf = fine + MMM;         // MMM
  double* t1 = tf + MMM;           // MN
  double* t2 = t1 + MN;            // MM
  double* u = t2 + MM;             // NNN
  double* g = u + NNN;             // 3 NNN
  __shared__ DealiasMats<N, M> mt;
  for (int x = threadIdx.x; x < N * N; x += blockDim.x) mt.D[x] = mats.D[x];
  for (int x = threadIdx.x; x < M * N; x += blockDim.x) {
    mt.J[x] = mats.J[x];
    mt.Jt[x] = mats.Jt[x];
  }
  const long long e = blockIdx.x;
  const long long PT = E * NNN;
  const long long base = e * NNN;
  // the advecting field on the fine grid, once per element
  for (int l = 0; l < 3; ++l) {
    for (int x = threadIdx.x; x < NNN; x += blockDim.x) u[x] = __ldg(c + l * PT + base + x);
    __syncthreads();
    to_fine<N, M, EX>(mt.J, mt.Jt, u, t1, t2, cf + l * MMM);
  }
  for (int f = 0; f < 3; ++f) {
    for (int x = threadIdx.x; x < NNN; x += blockDim.x) u[x] = __ldg(v + f * PT + base + x);
    __syncthreads();
    // GLL gradient: g_l = rx[0,l] ur + rx[1,l] us + rx[2,l] ut (operators.py:59-66)
    for (int x = threadIdx.x; x < NNN; x += blockDim.x) {
      const int i = x / (N * N), j = (x / N) % N, k = x % N;
      double ar = 0.0, as = 0.0, at = 0.0;
#pragma unroll
      for (int q = 0; q < N; ++q) {
        ar = mac<EX>(ar, mt.D[i * N + q], u[(q * N + j) * N + k]);
        as = mac<EX>(as, mt.D[j * N + q], u[(i * N + q) * N + k]);
        at = mac<EX>(at, mt.D[k * N + q], u[(i * N + j) * N + q]);
      }
#pragma unroll
      for (int l = 0; l < 3; ++l) {
        const double r0 = __ldg(rx + (0 * 3 + l) * PT + base + x);
        const double r1 = __ldg(rx + (1 * 3 + l) * PT + base + x);
        const double r2 = __ldg(rx + (2 * 3 + l) * PT + base + x);
        g[l * NNN + x] = add<EX>(add<EX>(mul<EX>(r0, ar), mul<EX>(r1, as)), mul<EX>(r2, at));
      }
    }
    __syncthreads();
    // fine = cf0 * gf0; fine += cf1 * gf1; fine += cf2 * gf2 (operators.py:150-152)
    for (int l = 0; l < 3; ++l) {
      to_fine<N, M, EX>(mt.J, mt.Jt, g + l * NNN, t1, t2, tf);
      for (int x = threadIdx.x; x < MMM; x += blockDim.x) {
        const double pr = mul<EX>(cf[l * MMM + x], tf[x]);
        fine[x] = (l == 0) ? pr : add<EX>(fine[x], pr);
      }
      __syncthreads();
    }
    // weak = project_back(wjac_f * fine) / bm (operators.py:153-154)
    for (int x = threadIdx.x; x < MMM; x += blockDim.x) fine[x] = mul<EX>(__ldg(wjf + e * MMM + x), fine[x]);
    __syncthreads();
    contract_r<N, M, M, M, EX>(mt.Jt, fine, t1);
    __syncthreads();
    contract_s<N, N, M, M, EX>(mt.J, t1, t2);      // Jt column-major is J row-major
    __syncthreads();
    for (int x = threadIdx.x; x < NNN; x += blockDim.x) {
      const int ij = x / N, p = x - ij * N;
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < M; ++k) s = mac<EX>(s, mt.J[k * N + p], t2[ij * M + k]);
      out[f * PT + base + x] = sign * (s / __ldg(bm + base + x));   // sign is +-1: exact
    }
    __syncthreads();
  }
}

template <int N, int M>
static int launch_dealias(const double* D, const double* J, const double* c, const double* v, const double* rx,
                          const double* wjf, const double* bm, long long E, double sign, double* out, int exact,
                          cudaStream_t st) {
  DealiasMats<N, M> m;
  for (int i = 0; i < N * N; ++i) m.D[i] = D[i];
  for (int p = 0; p < M; ++p)
    for (int i = 0; i < N; ++i) {
      m.J[p * N + i] = J[p * N + i];
      m.Jt[i * M + p] = J[p * N + i];
    }
  const size_t smem = (size_t)dealias_smem_doubles<N, M>() * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(dealias_advect_kernel<N, M, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(dealias_advect_kernel<N, M, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  if (E <= 0) return SF_OK;
  if (exact)
    dealias_advect_kernel<N, M, true><<<(unsigned)E, 512, smem, st>>>(m, c, v, rx, wjf, bm, E, sign, out);
  else
    dealias_advect_kernel<N, M, false><<<(unsigned)E, 512, smem, st>>>(m, c, v, rx, wjf, bm, E, sign, out);
  return check_launch("dealias_advect");
}

}  // namespace sf

extern "C" {

// out (3, E, n^3) = sign * Dealias.advect_vec(c, v) (operators.py:119-158) for
// (n, m) = (8, 12), (6, 9), (4, 6); D (n x n) and J (m x n) are HOST arrays,
// wjac_f (E, m^3) = fine quadrature weights x Jacobian on the fine grid.
int sf_dealias_advect_f64(const double* d_host, const double* j_host, int n, int m, const double* c,
                          const double* v, const double* rx, const double* wjac_f, const double* bm, long long E,
                          double sign, double* out, int exact, void* stream) {
  using namespace sf;
  if (!d_host || !j_host || !c || !v || !rx || !wjac_f || !bm || !out || E < 0) {
    set_error("sf_dealias_advect_f64: bad arguments");
    return SF_ERR_ARG;
  }
  cudaStream_t st = as_stream(stream);
  if (n == 8 && m == 12) return launch_dealias<8, 12>(d_host, j_host, c, v, rx, wjac_f, bm, E, sign, out, exact, st);
  if (n == 6 && m == 9) return launch_dealias<6, 9>(d_host, j_host, c, v, rx, wjac_f, bm, E, sign, out, exact, st);
  if (n == 4 && m == 6) return launch_dealias<4, 6>(d_host, j_host, c, v, rx, wjac_f, bm, E, sign, out, exact, st);
  set_error("sf_dealias_advect_f64: (n, m) = (%d, %d) not instantiated", n, m);
  return SF_ERR_UNSUPPORTED;
}

}  // extern "C"
