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
//
// Each Op splits its per-point work into load() (all global reads) and finish()
// (arithmetic, stores, partial sums) so map_reduce_kernel can keep several
// points' loads in flight per thread.
#include "reduce.cuh"

namespace sf {
int peer_allreduce(const PeerCtx& c, const double* in, int k, double* out, cudaStream_t st);
}

namespace sf {

// weight 1/mult for point p, or 1 when no multiplicity is given (plain dot)
__device__ __forceinline__ double wgt(const uint8_t* __restrict__ mult, long long p,
                                      const double* im_tab) {
  return mult ? im_tab[__ldg(mult + p)] : 1.0;
}

// z = M r with M = diag(invdiag) (BlockJacobi, precond.py:58-59) or identity.
__device__ __forceinline__ double ldprec(const double* __restrict__ invdiag, long long p) {
  return invdiag ? __ldg(invdiag + p) : 1.0;
}

// ---------------------------------------------------------------- dots
// out[k] = sum_p (a_k[p] * w[p]) * b_k[p] for up to 4 (a, b) pairs
template <int KK>
struct DotOp {
  static constexpr int K = KK;
  const double* a[4];
  const double* b[4];
  const uint8_t* mult;
  struct In { double a[KK], b[KK], w; };
  __device__ void prologue() {}
  __device__ __forceinline__ In load(long long p, const double* im_tab) const {
    In in;
    in.w = wgt(mult, p, im_tab);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      in.a[k] = __ldg(a[k] + p);
      in.b[k] = __ldg(b[k] + p);
    }
    return in;
  }
  __device__ __forceinline__ void finish(long long, const In& in, double (&acc)[K]) const {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const double aw = mult ? in.a[k] * in.w : in.a[k];
      acc[k] = fma(aw, in.b[k], acc[k]);
    }
  }
};

int dot1_vec(const double* a, const double* b, const uint8_t* mult, long long P, RedWork wk,
             double* out, cudaStream_t st, const PeerCtx* peer);  // vectorised weighted dot (below)

int dot_multi(int K, const double* const* a, const double* const* b, const uint8_t* mult,
              long long P, RedWork wk, double* out, cudaStream_t st) {
  if (K == 1 && mult) {
    const int r = dot1_vec(a[0], b[0], mult, P, wk, out, st, nullptr);
    if (r >= 0) return r;  // -1: not vectorisable (alignment / odd P), use the generic path
  }
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
// p = M r ; out[0] = <r, p>_w                      (krylov.py:48-50)
struct CgInitOp {
  static constexpr int K = 1;
  const double* r;
  const double* invdiag;
  double* pv;
  const uint8_t* mult;
  struct In { double r, d, w; };
  __device__ void prologue() {}
  __device__ __forceinline__ In load(long long p, const double* im_tab) const {
    return In{r[p], ldprec(invdiag, p), wgt(mult, p, im_tab)};
  }
  __device__ __forceinline__ void finish(long long p, const In& in, double (&acc)[K]) const {
    const double z = invdiag ? in.d * in.r : in.r;
    pv[p] = z;
    acc[0] = fma(in.r * in.w, z, acc[0]);
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
  struct In { double x, r, p, ap, d, w; };
  __device__ void prologue() { alpha = *rz / *pap; }
  __device__ __forceinline__ In load(long long p, const double* im_tab) const {
    return In{x[p], r[p], pv[p], ap[p], ldprec(invdiag, p), wgt(mult, p, im_tab)};
  }
  __device__ __forceinline__ void finish(long long p, const In& in, double (&acc)[K]) const {
    x[p] = fma(alpha, in.p, in.x);
    const double rv = fma(-alpha, in.ap, in.r);
    r[p] = rv;
    const double rw = rv * in.w;
    acc[0] = fma(rw, rv, acc[0]);
    acc[1] = fma(rw, invdiag ? in.d * rv : rv, acc[1]);
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
  struct In { double p, r, d; };
  __device__ void prologue() { beta = *rz_new / *rz; }
  __device__ __forceinline__ In load(long long p, const double*) const {
    return In{pv[p], r[p], ldprec(invdiag, p)};
  }
  __device__ __forceinline__ void finish(long long p, const In& in, double (&)[1]) const {
    pv[p] = fma(beta, in.p, invdiag ? in.d * in.r : in.r);
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
template <bool PREV, bool NEXT, bool NORM, bool W2>
struct MgsOp {
  static constexpr int K = 2;
  double* w;
  const double* vprev;
  const double* hprev;
  const double* vnext;
  double* w2;
  const double* v2prev;
  const uint8_t* mult;
  double h;
  struct In { double w, vp, vn, w2, v2p, m; };
  __device__ void prologue() { h = PREV ? *hprev : 0.0; }
  __device__ __forceinline__ In load(long long p, const double* im_tab) const {
    In in{};
    in.w = w[p];
    if constexpr (PREV) in.vp = __ldg(vprev + p);
    if constexpr (NEXT) in.vn = __ldg(vnext + p);
    if constexpr (W2) {
      in.w2 = w2[p];
      in.v2p = __ldg(v2prev + p);
    }
    if constexpr (NEXT || NORM) in.m = wgt(mult, p, im_tab);
    return in;
  }
  __device__ __forceinline__ void finish(long long p, const In& in, double (&acc)[K]) const {
    double wv = in.w;
    if constexpr (PREV) {
      wv = fma(-h, in.vp, wv);
      w[p] = wv;
    }
    if constexpr (W2) w2[p] = fma(-h, in.v2p, in.w2);
    if constexpr (NEXT || NORM) {
      const double ww = wv * in.m;
      if constexpr (NEXT) acc[0] = fma(ww, in.vn, acc[0]);
      if constexpr (NORM) acc[1] = fma(ww, wv, acc[1]);
    }
  }
};

// Vectorised MGS pass: 16-byte loads of point pairs (each warp instruction moves
// a contiguous 512 B run), SF_MGS_U pairs per lane in flight.  Same per-point
// arithmetic as MgsOp; used when P is even and every array is 16-byte aligned.
// Measured at 64^3 (tools/vec_bench.py): 2 blocks/SM minimum (no register cap
// below 128) runs the prev+next pass in 637 us vs 647 us at 4; U only changes the
// per-thread point order (hence the dot's rounding), so it stays at 2; streaming
// cache hints (ld/st.global.cs) cost 7 %.
#ifndef SF_MGS_MINB
#define SF_MGS_MINB 2
#endif
#ifndef SF_MGS_U
#define SF_MGS_U 2
#endif
template <bool PREV, bool NEXT, bool NORM, bool W2, int KOUT = 2>
__global__ void __launch_bounds__(RED_THREADS, SF_MGS_MINB)
mgs2_kernel(double* __restrict__ w, const double* __restrict__ vprev, const double* __restrict__ hprev,
            const double* __restrict__ vnext, double* __restrict__ w2, const double* __restrict__ v2prev,
            const uint8_t* __restrict__ mult, long long P2, RedWork wk, double* __restrict__ out,
            PeerCtx peer, const double* __restrict__ gate) {
  // gated pass (GMRES second MGS sweep decided on the device): every block of
  // every rank reads the same global flag, so all skip together -- no partials,
  // no counter update, no peer traffic
  if (gate != nullptr && *gate == 0.0) return;
  constexpr int U = SF_MGS_U;
  __shared__ double im_tab[256];
  init_im_tab(im_tab);
  __syncthreads();
  const double h = PREV ? *hprev : 0.0;
  double acc[2] = {0.0, 0.0};
  const int lane = threadIdx.x & 31;
  const long long gwarp = ((long long)blockIdx.x * RED_THREADS + threadIdx.x) >> 5;
  const long long span = 32LL * U;
  const long long wstride = (long long)gridDim.x * (RED_THREADS / 32) * span;
  double2* w_2 = reinterpret_cast<double2*>(w);
  double2* w2_2 = reinterpret_cast<double2*>(w2);
  for (long long base = gwarp * span + lane; base < P2; base += wstride) {
    double2 wv[U], vp[U], vn[U], x2[U], v2[U];
    double m0[U], m1[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const long long i = base + 32 * q;
      if (i < P2) {
        wv[q] = w_2[i];
        if constexpr (PREV) vp[q] = __ldg(reinterpret_cast<const double2*>(vprev) + i);
        if constexpr (NEXT) vn[q] = __ldg(reinterpret_cast<const double2*>(vnext) + i);
        if constexpr (W2) {
          x2[q] = w2_2[i];
          v2[q] = __ldg(reinterpret_cast<const double2*>(v2prev) + i);
        }
        if constexpr (NEXT || NORM) {
          const uchar2 mm = __ldg(reinterpret_cast<const uchar2*>(mult) + i);
          m0[q] = im_tab[mm.x];
          m1[q] = im_tab[mm.y];
        }
      }
    }
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const long long i = base + 32 * q;
      if (i < P2) {
        double a = wv[q].x, b = wv[q].y;
        if constexpr (PREV) {
          a = fma(-h, vp[q].x, a);
          b = fma(-h, vp[q].y, b);
          w_2[i] = make_double2(a, b);
        }
        if constexpr (W2) w2_2[i] = make_double2(fma(-h, v2[q].x, x2[q].x), fma(-h, v2[q].y, x2[q].y));
        if constexpr (NEXT || NORM) {
          const double wa = a * m0[q], wb = b * m1[q];
          if constexpr (NEXT) {
            acc[0] = fma(wa, vn[q].x, acc[0]);
            acc[0] = fma(wb, vn[q].y, acc[0]);
          }
          if constexpr (NORM) {
            acc[1] = fma(wa, a, acc[1]);
            acc[1] = fma(wb, b, acc[1]);
          }
        }
      }
    }
  }
  if constexpr (KOUT == 2) {
    finish_reduce<2>(acc, wk, out, &peer);
  } else {
    double a1[1] = {acc[0]};
    finish_reduce<1>(a1, wk, out, &peer);
  }
}

// <a, b>_{1/mult} through the vectorised pass (w = a read-only, v_next = b):
// the same (a * 1/mult) * b per point as DotOp<1>
int dot1_vec(const double* a, const double* b, const uint8_t* mult, long long P, RedWork wk,
             double* out, cudaStream_t st, const PeerCtx* peer) {
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (P % 2 != 0 || !al(a) || !al(b) || (reinterpret_cast<uintptr_t>(mult) & 1) != 0) return -1;
  const long long P2 = P / 2;
  unsigned blocks = RED_BLOCKS;
  long long need = (P2 + RED_THREADS - 1) / RED_THREADS;
  if (need < (long long)blocks) blocks = (unsigned)(need > 0 ? need : 1);
  mgs2_kernel<false, true, false, false, 1><<<blocks, RED_THREADS, 0, st>>>(
      const_cast<double*>(a), nullptr, nullptr, b, nullptr, nullptr, mult, P2, wk, out,
      peer ? *peer : PeerCtx{}, nullptr);
  return check_launch("dot");
}

template <bool PREV, bool NEXT, bool NORM, bool W2>
static int mgs_launch(double* w, const double* vprev, const double* hprev, const double* vnext,
                      double* w2, const double* v2prev, const uint8_t* mult, long long P,
                      RedWork wk, double* out, cudaStream_t st, const PeerCtx* peer,
                      const double* gate) {
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  const bool vec = (P % 2 == 0) && mult && al(w) && (!PREV || al(vprev)) && (!NEXT || al(vnext)) &&
                   (!W2 || (al(w2) && al(v2prev))) && ((reinterpret_cast<uintptr_t>(mult) & 1) == 0);
  if (vec) {
    const long long P2 = P / 2;
    unsigned blocks = RED_BLOCKS;
    long long need = (P2 + RED_THREADS - 1) / RED_THREADS;
    if (need < (long long)blocks) blocks = (unsigned)(need > 0 ? need : 1);
    mgs2_kernel<PREV, NEXT, NORM, W2><<<blocks, RED_THREADS, 0, st>>>(w, vprev, hprev, vnext, w2, v2prev,
                                                                      mult, P2, wk, out,
                                                                      peer ? *peer : PeerCtx{}, gate);
    return check_launch("mgs_step");
  }
  if (gate != nullptr) {
    set_error("mgs_step: a gated pass needs 16-byte aligned arrays and an even point count");
    return SF_ERR_UNSUPPORTED;
  }
  MgsOp<PREV, NEXT, NORM, W2> op{w, vprev, hprev, vnext, w2, v2prev, mult, 0.0};
  const int r = launch_map_reduce(op, P, wk, out, st, "mgs_step");
  if (r != SF_OK || peer == nullptr || peer->world <= 1) return r;
  return peer_allreduce(*peer, out, 2, out, st);  // unfused fallback: separate peer kernel
}

int mgs_step(double* w, const double* vprev, const double* hprev, const double* vnext, double* w2,
             const double* v2prev, const uint8_t* mult, int want_norm, long long P, RedWork wk,
             double* out, cudaStream_t st, const PeerCtx* peer, const double* gate) {
  if (w2 && !vprev) w2 = nullptr;  // w2 is only ever updated together with w
  const int code = (vprev ? 8 : 0) | (vnext ? 4 : 0) | (want_norm ? 2 : 0) | (w2 ? 1 : 0);
  switch (code) {
#define C(CODE, A, B, N, W) \
  case CODE: return mgs_launch<A, B, N, W>(w, vprev, hprev, vnext, w2, v2prev, mult, P, wk, out, st, peer, gate);
    C(0, false, false, false, false) C(2, false, false, true, false)
    C(4, false, true, false, false) C(6, false, true, true, false)
    C(8, true, false, false, false) C(9, true, false, false, true)
    C(10, true, false, true, false) C(11, true, false, true, true)
    C(12, true, true, false, false) C(13, true, true, false, true)
    C(14, true, true, true, false) C(15, true, true, true, true)
#undef C
    default: set_error("mgs_step: bad argument combination"); return SF_ERR_ARG;
  }
}

// GMRES Arnoldi step bookkeeping on the device (krylov.py:110-123, 149), so the
// host never has to stop the stream inside an iteration.  blk is the iteration's
// scalar block: first-sweep pairs at [2i, 2i+1] (h_i, <w,w>), the second sweep
// at o2 + 2i, and [o3] = reorthogonalise flag, [o3+1] = final norm.
//   phase 0: flag = sqrt(na2) < 0.7071 * sqrt(nb2); norm = sqrt(na2)
//   phase 1: if flag, norm = sqrt(na2 of the second sweep)
//   phase 2: phase 0, and the second sweep's first coefficient <w, v_0> is taken
//            from [2(j+1)], where the first sweep's last pass left it (that pass
//            also dotted the updated w with v_0: the same per-point products and
//            reduction tree as a separate pass, one read of w fewer)
// (IEEE sqrt and the same comparison the host evaluates: identical decision.)
__global__ void gmres_gate_kernel(double* blk, int j, int o2, int o3, int phase) {
  if (threadIdx.x != 0) return;
  if (phase == 0 || phase == 2) {
    const double nb = sqrt(blk[1]);
    const double na = sqrt(blk[2 * (j + 1) + 1]);
    blk[o3] = (na < 0.7071 * nb) ? 1.0 : 0.0;
    blk[o3 + 1] = na;
    if (phase == 2) blk[o2] = blk[2 * (j + 1)];
  } else if (blk[o3] != 0.0) {
    blk[o3 + 1] = sqrt(blk[o2 + 2 * (j + 1) + 1]);
  }
}

int gmres_gate(double* blk, int j, int o2, int o3, int phase, cudaStream_t st) {
  gmres_gate_kernel<<<1, 32, 0, st>>>(blk, j, o2, o3, phase);
  return check_launch("gmres_gate");
}

// x = x0 + sum_i coef[i] * M v_i, accumulated in i order (krylov.py:153-154 for
// GMRES with zs[i] = M v_i recomputed bit-identically; krylov.py:207-209 for the
// projection guess with M = I and x0 = 0).  x0 may alias x; x0 == nullptr -> 0.
// Each thread carries 4 independent points through the i loop so 4 loads of
// every basis vector are in flight at once.
__global__ void __launch_bounds__(RED_THREADS)
lincomb_kernel(double* x, const double* x0, const double* const* __restrict__ v,
               const double* __restrict__ coef, const double* __restrict__ invdiag, int nv,
               long long P) {
  const int lane = threadIdx.x & 31;
  const long long gwarp = ((long long)blockIdx.x * RED_THREADS + threadIdx.x) >> 5;
  const long long wstride = (long long)gridDim.x * (RED_THREADS / 32) * 128;
  const long long stride = 32;
  for (long long p0 = gwarp * 128 + lane; p0 < P; p0 += wstride) {
    double acc[4], d[4];
    bool ok[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const long long p = p0 + q * stride;
      ok[q] = p < P;
      acc[q] = (ok[q] && x0) ? x0[p] : 0.0;
      d[q] = (ok[q] && invdiag) ? __ldg(invdiag + p) : 1.0;
    }
    for (int i = 0; i < nv; ++i) {
      const double c = __ldg(coef + i);
      const double* vi = v[i];
      double vv[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) vv[q] = ok[q] ? __ldg(vi + p0 + q * stride) : 0.0;
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = fma(c, invdiag ? d[q] * vv[q] : vv[q], acc[q]);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (ok[q]) x[p0 + q * stride] = acc[q];
  }
}

int lincomb(double* x, const double* x0, const double* const* v, const double* coef,
            const double* invdiag, int nv, long long P, cudaStream_t st) {
  if (P <= 0) return SF_OK;
  long long need = (P + 4LL * RED_THREADS - 1) / (4LL * RED_THREADS);
  unsigned blocks = (unsigned)(need < RED_BLOCKS ? (need > 0 ? need : 1) : RED_BLOCKS);
  lincomb_kernel<<<blocks, RED_THREADS, 0, st>>>(x, x0, v, coef, invdiag, nv, P);
  return check_launch("lincomb");
}

// r = b - ax ; out[0] = <r, r>_w                   (krylov.py:155-157)
struct ResidualOp {
  static constexpr int K = 1;
  double* r;
  const double* b;
  const double* ax;
  const uint8_t* mult;
  struct In { double b, ax, w; };
  __device__ void prologue() {}
  __device__ __forceinline__ In load(long long p, const double* im_tab) const {
    return In{b[p], ax[p], wgt(mult, p, im_tab)};
  }
  __device__ __forceinline__ void finish(long long p, const In& in, double (&acc)[K]) const {
    const double rv = in.b - in.ax;
    r[p] = rv;
    acc[0] = fma(rv * in.w, rv, acc[0]);
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
  struct In { double x, x2; };
  __device__ void prologue() { sv = *s; }
  __device__ __forceinline__ In load(long long p, const double*) const {
    return In{x[p], y2 ? x2[p] : 0.0};
  }
  __device__ __forceinline__ void finish(long long p, const In& in, double (&)[1]) const {
    y[p] = in.x / sv;
    if (y2) y2[p] = in.x2 / sv;
  }
};

// Vectorised y = x / s (and y2 = x2 / s): 16-byte pair loads/stores, a warp
// moves contiguous 512 B runs, SD_U pairs per lane in flight; the same IEEE
// division per point as ScaleDivOp.  GMRES normalises in place (y == x), so the
// vector pointers carry no __restrict__ (each thread loads its pairs before it
// stores them, which is all in-place use needs).
constexpr int SD_U = 2;
__global__ void __launch_bounds__(RED_THREADS)
scale_div2_kernel(double2* y, const double2* x, double2* y2, const double2* x2,
                  const double* __restrict__ s, long long P2) {
  const double sv = *s;
  const int lane = threadIdx.x & 31;
  const long long gwarp = ((long long)blockIdx.x * RED_THREADS + threadIdx.x) >> 5;
  const long long span = 32LL * SD_U;
  const long long wstride = (long long)gridDim.x * (RED_THREADS / 32) * span;
  for (long long base = gwarp * span + lane; base < P2; base += wstride) {
    double2 a[SD_U], b[SD_U];
#pragma unroll
    for (int q = 0; q < SD_U; ++q) {
      const long long i = base + 32 * q;
      if (i < P2) {
        a[q] = x[i];
        if (y2) b[q] = x2[i];
      }
    }
#pragma unroll
    for (int q = 0; q < SD_U; ++q) {
      const long long i = base + 32 * q;
      if (i < P2) {
        y[i] = make_double2(a[q].x / sv, a[q].y / sv);
        if (y2) y2[i] = make_double2(b[q].x / sv, b[q].y / sv);
      }
    }
  }
}

int scale_div(double* y, const double* x, double* y2, const double* x2, const double* s,
              long long P, cudaStream_t st) {
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (P % 2 == 0 && al(y) && al(x) && (!y2 || (al(y2) && al(x2)))) {
    const long long P2 = P / 2;
    unsigned blocks = RED_BLOCKS;
    const long long need = (P2 + RED_THREADS * SD_U - 1) / (RED_THREADS * SD_U);
    if (need < (long long)blocks) blocks = (unsigned)(need > 0 ? need : 1);
    scale_div2_kernel<<<blocks, RED_THREADS, 0, st>>>(
        reinterpret_cast<double2*>(y), reinterpret_cast<const double2*>(x), reinterpret_cast<double2*>(y2),
        reinterpret_cast<const double2*>(x2), s, P2);
    return check_launch("scale_div");
  }
  ScaleDivOp op{y, x, y2, x2, s, 0.0};
  RedWork none{nullptr, nullptr};
  return launch_map_reduce(op, P, none, nullptr, st, "scale_div");
}

}  // namespace sf
