// Multiplicity-weighted inner products (glsc3, K5) and the fused Krylov vector
// updates (K6 CG, K7 GMRES MGS / projection), all on the deterministic
// map-reduce skeleton of reduce.cuh.
//
// Reference semantics:
//   GatherScatter.dot     space.py:72-76   sum((a * invmult) * b)
//   FunctionSpace.integral space.py:159-161 sum(bm * u)          (unweighted)
//   pcg                   krylov.py:36-75
//   gmres (MGS + update)  krylov.py:78-160
//   ProjectionSpace       krylov.py:163-236
//
// Scalars produced by one kernel and consumed by the next (alpha, beta, h_ij,
// projection coefficients) stay in device memory: kernels read them through
// pointers, so the host never has to round-trip them.  Every division that the
// reference performs on host floats (alpha = rz / pap, ...) is performed by each
// thread with the same IEEE operation, so all threads see the same value.
#include "reduce.cuh"

namespace sf {

// weight 1/mult for point p, or 1 when no multiplicity is given (plain dot)
__device__ __forceinline__ double wgt(const uint8_t* __restrict__ mult, long long p,
                                      const double* im_tab) {
  return mult ? im_tab[__ldg(mult + p)] : 1.0;
}

// ---------------------------------------------------------------- dots
// out[k] = sum_p (a_k[p] * w[p]) * b_k[p] for up to 4 (a, b) pairs
template <int KK>
struct DotOp {
  static constexpr int K = KK;
  const double* a[4];
  const double* b[4];
  const uint8_t* mult;
  __device__ void prologue() {}
  __device__ __forceinline__ void point(long long p, const double* im_tab, double (&acc)[K]) const {
    const double w = wgt(mult, p, im_tab);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double aw = mult ? __ldg(a[k] + p) * w : __ldg(a[k] + p);
      acc[k] = fma(aw, __ldg(b[k] + p), acc[k]);
    }
  }
};

int dot_multi(int K, const double* const* a, const double* const* b, const uint8_t* mult,
              long long P, RedWork wk, double* out, cudaStream_t st) {
  switch (K) {
#define CASE(KV)                                                              \
  case KV: {                                                                  \
    DotOp<KV> op;                                                             \
    for (int k = 0; k < KV; ++k) { op.a[k] = a[k]; op.b[k] = b[k]; }         \
    op.mult = mult;                                                           \
    return launch_map_reduce(op, P, wk, out, st, "dot");                      \
  }
    CASE(1) CASE(2) CASE(3) CASE(4)
#undef CASE
    default: set_error("dot_multi: K=%d out of range 1..4", K); return SF_ERR_ARG;
  }
}

// ---------------------------------------------------------------- PCG
// z = M r with M = diag(invdiag) (BlockJacobi, precond.py:58-59) or identity.
__device__ __forceinline__ double prec(const double* __restrict__ invdiag, double r, long long p) {
  return invdiag ? __ldg(invdiag + p) * r : r;
}

// p = M r ; out[0] = <r, p>_w                      (krylov.py:48-50)
struct CgInitOp {
  static constexpr int K = 1;
  const double* r;
  const double* invdiag;
  double* pv;
  const uint8_t* mult;
  __device__ void prologue() {}
  __device__ __forceinline__ void point(long long p, const double* im_tab, double (&acc)[K]) const {
    const double rv = r[p];
    const double z = prec(invdiag, rv, p);
    pv[p] = z;
    acc[0] = fma(rv * wgt(mult, p, im_tab), z, acc[0]);
  }
};

// alpha = rz / pap ; x += alpha p ; r -= alpha ap ; out = (<r,r>_w, <r, M r>_w)
// (krylov.py:63-71; the preconditioned inner product is computed even on the
// converged iteration, where the reference skips it -- it is then unused)
struct CgUpdateOp {
  static constexpr int K = 2;
  double* x;
  double* r;
  const double* pv;
  const double* ap;
  const double* invdiag;
  const uint8_t* mult;
  const double* rz;
  const double* pap;
  double alpha;
  __device__ void prologue() { alpha = *rz / *pap; }
  __device__ __forceinline__ void point(long long p, const double* im_tab, double (&acc)[K]) const {
    x[p] = fma(alpha, pv[p], x[p]);
    const double rv = fma(-alpha, ap[p], r[p]);
    r[p] = rv;
    const double rw = rv * wgt(mult, p, im_tab);
    acc[0] = fma(rw, rv, acc[0]);
    acc[1] = fma(rw, prec(invdiag, rv, p), acc[1]);
  }
};

// beta = rz_new / rz ; p = M r + beta p            (krylov.py:72-74)
struct CgDirOp {
  static constexpr int K = 0;
  double* pv;
  const double* r;
  const double* invdiag;
  const double* rz_new;
  const double* rz;
  double beta;
  __device__ void prologue() { beta = *rz_new / *rz; }
  __device__ __forceinline__ void point(long long p, const double*, double (&)[1]) const {
    pv[p] = fma(beta, pv[p], prec(invdiag, r[p], p));
  }
};

int cg_init(const double* r, const double* invdiag, double* pv, const uint8_t* mult, long long P,
            RedWork wk, double* out, cudaStream_t st) {
  CgInitOp op{r, invdiag, pv, mult};
  return launch_map_reduce(op, P, wk, out, st, "cg_init");
}

int cg_update(double* x, double* r, const double* pv, const double* ap, const double* invdiag,
              const uint8_t* mult, const double* rz, const double* pap, long long P, RedWork wk,
              double* out, cudaStream_t st) {
  CgUpdateOp op{x, r, pv, ap, invdiag, mult, rz, pap, 0.0};
  return launch_map_reduce(op, P, wk, out, st, "cg_update");
}

int cg_direction(double* pv, const double* r, const double* invdiag, const double* rz_new,
                 const double* rz, long long P, cudaStream_t st) {
  CgDirOp op{pv, r, invdiag, rz_new, rz, 0.0};
  RedWork none{nullptr, nullptr};
  return launch_map_reduce(op, P, none, nullptr, st, "cg_direction");
}

// ---------------------------------------------------------------- GMRES / projection
// One modified-Gram-Schmidt sweep step (krylov.py:112-115 / 119-122):
//   if vprev: w -= (*hprev) * vprev          (the update of the previous i)
//   out[0] = <w, vnext>_w   if vnext         (the next h_{i j})
//   out[1] = <w, w>_w       if want_norm     (norm_before / norm_after)
// A second pair (w2, v2prev) lets the projection basis update ad and d together
// (krylov.py:230-231): w2 -= (*hprev) * v2prev.
struct MgsOp {
  static constexpr int K = 2;
  double* w;
  const double* vprev;
  const double* hprev;
  const double* vnext;
  double* w2;
  const double* v2prev;
  const uint8_t* mult;
  int want_norm;
  double h;
  __device__ void prologue() { h = vprev ? *hprev : 0.0; }
  __device__ __forceinline__ void point(long long p, const double* im_tab, double (&acc)[K]) const {
    double wv = w[p];
    if (vprev) {
      wv = fma(-h, vprev[p], wv);
      w[p] = wv;
    }
    if (w2) w2[p] = fma(-h, v2prev[p], w2[p]);
    const double ww = wv * wgt(mult, p, im_tab);
    if (vnext) acc[0] = fma(ww, __ldg(vnext + p), acc[0]);
    if (want_norm) acc[1] = fma(ww, wv, acc[1]);
  }
};

int mgs_step(double* w, const double* vprev, const double* hprev, const double* vnext, double* w2,
             const double* v2prev, const uint8_t* mult, int want_norm, long long P, RedWork wk,
             double* out, cudaStream_t st) {
  MgsOp op{w, vprev, hprev, vnext, w2, v2prev, mult, want_norm, 0.0};
  return launch_map_reduce(op, P, wk, out, st, "mgs_step");
}

// x = x0 + sum_i coef[i] * M v_i, accumulated in i order (krylov.py:153-154 for
// GMRES with zs[i] = M v_i recomputed bit-identically; krylov.py:207-209 for the
// projection guess with M = I and x0 = 0).  x0 may alias x; x0 == nullptr -> 0.
struct LinCombOp {
  static constexpr int K = 0;
  double* x;
  const double* x0;
  const double* const* v;  // device array of nv pointers
  const double* coef;      // device array of nv scalars
  const double* invdiag;
  int nv;
  __device__ void prologue() {}
  __device__ __forceinline__ void point(long long p, const double*, double (&)[1]) const {
    double acc = x0 ? x0[p] : 0.0;
    for (int i = 0; i < nv; ++i) acc = fma(coef[i], prec(invdiag, __ldg(v[i] + p), p), acc);
    x[p] = acc;
  }
};

int lincomb(double* x, const double* x0, const double* const* v, const double* coef,
            const double* invdiag, int nv, long long P, cudaStream_t st) {
  LinCombOp op{x, x0, v, coef, invdiag, nv};
  RedWork none{nullptr, nullptr};
  return launch_map_reduce(op, P, none, nullptr, st, "lincomb");
}

// r = b - ax ; out[0] = <r, r>_w                   (krylov.py:155-157)
struct ResidualOp {
  static constexpr int K = 1;
  double* r;
  const double* b;
  const double* ax;
  const uint8_t* mult;
  __device__ void prologue() {}
  __device__ __forceinline__ void point(long long p, const double* im_tab, double (&acc)[K]) const {
    const double rv = b[p] - ax[p];
    r[p] = rv;
    acc[0] = fma(rv * wgt(mult, p, im_tab), rv, acc[0]);
  }
};

int residual(double* r, const double* b, const double* ax, const uint8_t* mult, long long P,
             RedWork wk, double* out, cudaStream_t st) {
  ResidualOp op{r, b, ax, mult};
  return launch_map_reduce(op, P, wk, out, st, "residual");
}

// y = x / (*s)  (IEEE division, krylov.py:98,149 `r / beta`, `w / norm_after`)
// optionally also y2 = x2 / (*s) (projection basis append, krylov.py:235-236)
struct ScaleDivOp {
  static constexpr int K = 0;
  double* y;
  const double* x;
  double* y2;
  const double* x2;
  const double* s;
  double sv;
  __device__ void prologue() { sv = *s; }
  __device__ __forceinline__ void point(long long p, const double*, double (&)[1]) const {
    y[p] = x[p] / sv;
    if (y2) y2[p] = x2[p] / sv;
  }
};

int scale_div(double* y, const double* x, double* y2, const double* x2, const double* s,
              long long P, cudaStream_t st) {
  ScaleDivOp op{y, x, y2, x2, s, 0.0};
  RedWork none{nullptr, nullptr};
  return launch_map_reduce(op, P, none, nullptr, st, "scale_div");
}

}  // namespace sf
