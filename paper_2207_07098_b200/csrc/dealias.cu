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
// Every contraction output is one thread's sequential sum over the contracted
// index in ascending order, starting from 0.0 -- the numba lane's loop
// (kernels/_numba.py apply_r/s/t) -- and the products / sums between stages are
// those of the reference expression, so EX=true is bit-identical to the chain.
//
// Register blocking: a thread loads one input line (the n or m values along the
// contracted axis) into registers and produces every output of that line; the
// matrices sit in the kernel's parameter (constant) bank and are indexed with
// compile-time constants, so each FMA reads one register and one constant -- no
// shared-memory traffic for the matrices and one shared load per 8-12 FMAs
// (the one-output-per-thread form was shared-memory bound at ~12 % of the FP64
// pipe).  Inputs of the t-axis contractions are stored with an odd line stride
// (n+1, m+1) so the lanes of a warp read distinct banks.
#include "common.cuh"

namespace sf {

template <int N, int M>
struct DealiasMats {
  double D[N * N];   // GLL derivative
  double J[M * N];   // GLL -> GL interpolation, J[p * N + i]
};

// Every shared buffer keeps its contiguous lines at an odd pitch (n+1 or m+1
// doubles) so the lanes of a warp, which walk lines, hit distinct banks.
// smem layout (doubles): cf 3 m m (m+1) | fine | tf | t1 max(m n (n+1), n m (m+1)) |
// t2 max(m m (n+1), n n (m+1)) | u n^3 | g 3 n^3
template <int N, int M>
__host__ __device__ constexpr int dealias_smem_doubles() {
  constexpr int FP = M * M * (M + 1);
  constexpr int T1 = (M * N * (N + 1) > N * M * (M + 1)) ? M * N * (N + 1) : N * M * (M + 1);
  constexpr int T2 = (M * M * (N + 1) > N * N * (M + 1)) ? M * M * (N + 1) : N * N * (M + 1);
  return 5 * FP + T1 + T2 + 4 * N * N * N;
}

// One register-blocked contraction line: a[0..I) (the values along the
// contracted axis) -> outputs o in [O0, O0 + OC) of rows of the row-major matrix
// mat (R x I) or, with TR, of its transpose (mat I x R read as mat[i * R + o]);
// every matrix index is a compile-time constant (parameter bank).
template <int I, int O0, int OC, int R, bool TR, bool EX>
__device__ __forceinline__ void line(const double* mat, const double (&a)[I], double* out, int ostride) {
#pragma unroll
  for (int o = O0; o < O0 + OC; ++o) {
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < I; ++i) s = mac<EX>(s, TR ? mat[i * R + o] : mat[o * I + i], a[i]);
    out[o * ostride] = s;
  }
}

// A contraction phase: LINES input lines x 2 output halves.  The half is the slow
// index of the thread id (warp-uniform except at one boundary warp), so both
// halves run with compile-time matrix indices.
template <int I, int R, bool TR, bool EX, int LINES, class Load, class Out>
__device__ __forceinline__ void phase(const double* mat, Load load, Out outp) {
  constexpr int H = R / 2;
  for (int x = threadIdx.x; x < 2 * LINES; x += blockDim.x) {
    const int half = x / LINES, ln = x - half * LINES;
    double a[I];
#pragma unroll
    for (int i = 0; i < I; ++i) a[i] = load(ln, i);
    int stride;
    double* o = outp(ln, stride);
    if (half == 0)
      line<I, 0, H, R, TR, EX>(mat, a, o, stride);
    else
      line<I, H, R - H, R, TR, EX>(mat, a, o, stride);
  }
}

// GLL (N^3) -> GL (M^3): apply_t(J, apply_s(J, apply_r(J, in))); out lines pitch M+1
template <int N, int M, bool EX>
__device__ __forceinline__ void to_fine(const DealiasMats<N, M>& m, const double* __restrict__ in,
                                        double* __restrict__ t1, double* __restrict__ t2,
                                        double* __restrict__ out) {
  // r: t1[p][j][k] = sum_i J[p][i] in[i][j][k]; line (j, k); t1 lines pitch N+1
  phase<N, M, false, EX, N * N>(
      m.J, [&](int ln, int i) { return in[i * N * N + ln]; },
      [&](int ln, int& st) {
        st = N * (N + 1);
        const int j = ln / N, k = ln - j * N;
        return t1 + j * (N + 1) + k;
      });
  __syncthreads();
  // s: t2[p][q][k] = sum_j J[q][j] t1[p][j][k]; line (p, k); t2 lines pitch N+1
  phase<N, M, false, EX, M * N>(
      m.J, [&](int ln, int j) { const int p = ln / N, k = ln - p * N; return t1[(p * N + j) * (N + 1) + k]; },
      [&](int ln, int& st) {
        st = N + 1;
        const int p = ln / N, k = ln - p * N;
        return t2 + p * M * (N + 1) + k;
      });
  __syncthreads();
  // t: out[p][q][r] = sum_k J[r][k] t2[p][q][k]; line (p, q)
  phase<N, M, false, EX, M * M>(
      m.J, [&](int ln, int k) { return t2[ln * (N + 1) + k]; },
      [&](int ln, int& st) {
        st = 1;
        return out + ln * (M + 1);
      });
  __syncthreads();
}

template <int N, int M, bool EX>
__global__ void __launch_bounds__(256, 2) dealias_advect_kernel(const __grid_constant__ DealiasMats<N, M> mats,
                                                             const double* __restrict__ c,
                                                             const double* __restrict__ v,
                                                             const double* __restrict__ rx,
                                                             const double* __restrict__ wjf,
                                                             const double* __restrict__ bm, long long E,
                                                             double sign, double* __restrict__ out) {
  constexpr int NNN = N * N * N, MMM = M * M * M;
  constexpr int FP = M * M * (M + 1);   // a fine field, lines at pitch M+1
  constexpr int T1 = (M * N * (N + 1) > N * M * (M + 1)) ? M * N * (N + 1) : N * M * (M + 1);
  constexpr int T2 = (M * M * (N + 1) > N * N * (M + 1)) ? M * M * (N + 1) : N * N * (M + 1);
  extern __shared__ double sm[];
  double* cf = sm;                 // 3 FP
  double* fine = cf + 3 * FP;      // FP
  double* tf = fine + FP;          // FP
  double* t1 = tf + FP;            // T1
  double* t2 = t1 + T1;            // T2
  double* u = t2 + T2;             // NNN
  double* g = u + NNN;             // 3 NNN
  const DealiasMats<N, M>& m = mats;
  const long long e = blockIdx.x;
  const long long PT = E * NNN;
  const long long base = e * NNN;
  // the advecting field on the fine grid, once per element
  for (int l = 0; l < 3; ++l) {
    for (int x = threadIdx.x; x < NNN; x += blockDim.x) u[x] = __ldg(c + l * PT + base + x);
    __syncthreads();
    to_fine<N, M, EX>(m, u, t1, t2, cf + l * FP);
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
        ar = mac<EX>(ar, m.D[i * N + q], u[(q * N + j) * N + k]);
        as = mac<EX>(as, m.D[j * N + q], u[(i * N + q) * N + k]);
        at = mac<EX>(at, m.D[k * N + q], u[(i * N + j) * N + q]);
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
      to_fine<N, M, EX>(m, g + l * NNN, t1, t2, tf);
      for (int x = threadIdx.x; x < MMM; x += blockDim.x) {
        const int y = (x / M) * (M + 1) + x % M;
        const double pr = mul<EX>(cf[l * FP + y], tf[y]);
        fine[y] = (l == 0) ? pr : add<EX>(fine[y], pr);
      }
      __syncthreads();
    }
    // weak = project_back(wjac_f * fine) / bm (operators.py:153-154); J^T[a][p] = J[p][a]
    for (int x = threadIdx.x; x < MMM; x += blockDim.x) {
      const int y = (x / M) * (M + 1) + x % M;
      fine[y] = mul<EX>(__ldg(wjf + e * MMM + x), fine[y]);
    }
    __syncthreads();
    // r: t1[a][q][r] = sum_p J[p][a] fine[p][q][r]; line (q, r); t1 lines pitch M+1
    phase<M, N, true, EX, M * M>(
        m.J, [&](int ln, int p) { const int q = ln / M, r = ln - q * M; return fine[(p * M + q) * (M + 1) + r]; },
        [&](int ln, int& st) {
          st = M * (M + 1);
          const int q = ln / M, r = ln - q * M;
          return t1 + q * (M + 1) + r;
        });
    __syncthreads();
    // s: t2[a][b][r] = sum_q J[q][b] t1[a][q][r]; line (a, r); t2 lines pitch M+1
    phase<M, N, true, EX, N * M>(
        m.J, [&](int ln, int q) { const int a0 = ln / M, r = ln - a0 * M; return t1[(a0 * M + q) * (M + 1) + r]; },
        [&](int ln, int& st) {
          st = M + 1;
          const int a0 = ln / M, r = ln - a0 * M;
          return t2 + a0 * N * (M + 1) + r;
        });
    __syncthreads();
    // t: w[a][b][c] = sum_r J[r][c] t2[a][b][r] into u (n^3), then / bm, * sign
    phase<M, N, true, EX, N * N>(
        m.J, [&](int ln, int r) { return t2[ln * (M + 1) + r]; },
        [&](int ln, int& st) {
          st = 1;
          return u + ln * N;
        });
    __syncthreads();
    for (int x = threadIdx.x; x < NNN; x += blockDim.x)
      out[f * PT + base + x] = sign * (u[x] / __ldg(bm + base + x));   // sign is +-1: exact
    __syncthreads();
  }
}

template <int N, int M>
static int launch_dealias(const double* D, const double* J, const double* c, const double* v, const double* rx,
                          const double* wjf, const double* bm, long long E, double sign, double* out, int exact,
                          cudaStream_t st) {
  DealiasMats<N, M> m;
  for (int i = 0; i < N * N; ++i) m.D[i] = D[i];
  for (int i = 0; i < M * N; ++i) m.J[i] = J[i];
  const size_t smem = (size_t)dealias_smem_doubles<N, M>() * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(dealias_advect_kernel<N, M, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(dealias_advect_kernel<N, M, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  if (E <= 0) return SF_OK;
  if (exact)
    dealias_advect_kernel<N, M, true><<<(unsigned)E, 256, smem, st>>>(m, c, v, rx, wjf, bm, E, sign, out);
  else
    dealias_advect_kernel<N, M, false><<<(unsigned)E, 256, smem, st>>>(m, c, v, rx, wjf, bm, E, sign, out);
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
