// Ax_helm for n = 8 fed by bulk asynchronous copies (K1, the production kernel).
//
// Reference: ax_helmholtz_local, kernels/_numba.py:86-131; the masked global
// operator body, operators.py:51-54; the Jacobi-preconditioned application
// `z = precond(v); w = apply_a(z)`, krylov.py:106-107.  Per-point arithmetic and
// accumulation order are those of ax8s.cuh (bit-identical in both modes).
//
// Why.  The register-prefetch kernel (ax8s.cuh) keeps one layer of G per thread
// in flight: ~30 KB of loads per SM, about half of what HBM latency x bandwidth
// needs, so it stalls on long-scoreboard at ~54 % of DRAM peak (ncu, 32^3).  Here
// every element's operands are six 4 KB runs of G, one of u (+ pre, B, the two
// 64-byte mask rows), contiguous in HBM; one producer lane moves them into a
// ring of shared-memory stages with `cp.async.bulk` (UBLKCP) completing on an
// mbarrier, so the bytes in flight are bounded by shared memory (~100+ KB per
// SM), not by registers.
//
// Layout.  One persistent CTA per SM: 8 compute warps + 1 producer warp.  A warp
// computes a whole element; lane (j, kp), j = lane >> 2, kp = lane & 3, owns the
// two r-pencils (j, 2kp) and (j, 2kp+1), so every shared-memory access of its own
// points is one LDS.128 and the t-derivative's row is shared by both pencils.
//   forward  (per layer i): r-derivative from the register pencil, s/t from the
//            stage (broadcast / rotated LDS.128, conflict-free), G from the stage;
//            f1 stays in registers, f2/f3 go to the warp's 8 KB scratch
//            (pair-swizzled rows).  The stage is released after the forward pass.
//   output   (per layer i): r-contraction from the f1 registers, s/t from scratch,
//            mass term and the masked pass-through from registers, one STG.128 per
//            lane (a warp writes 512 contiguous bytes per layer).
// PRE/MASK: the warp rewrites its own points of the staged u as
// (inmask ? pre * u : 0) before the derivatives read it.
#include <cuda/std/cstdint>

#include "ax8s.cuh"

namespace sf {

namespace ax8t {

constexpr int N = 8, NN = 64, NNN = 512;
constexpr int CW = 7;                          // compute warps (8 warps in all: up to 255 registers)
constexpr int THREADS = (CW + 1) * 32;         // + producer warp
constexpr int FIELD = NNN * 8;                 // bytes of one element field (4 KB)
constexpr int SCRATCH = 2 * FIELD;             // f2, f3 of one element per warp
constexpr int SMEM_MAX = 232448;               // sm_100 dynamic shared memory per block
constexpr int HEAD = 2048;                     // mbarriers + the two D tables

__host__ __device__ constexpr int stage_bytes(bool pre, bool mass, bool mask) {
  return 7 * FIELD + (pre ? FIELD : 0) + (mass ? FIELD : 0) + (mask ? 128 : 0);
}
__host__ __device__ constexpr int n_stages(bool pre, bool mass, bool mask) {
  return (SMEM_MAX - HEAD - CW * SCRATCH) / stage_bytes(pre, mass, mask) > 6
             ? 6
             : (SMEM_MAX - HEAD - CW * SCRATCH) / stage_bytes(pre, mass, mask);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy completing `bytes` on the stage's mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// scratch rows: pair p of row r stored at pair p ^ ((r >> 1) & 3) -- the 8 rows
// read together by the t-contraction land on 8 distinct 16-byte bank groups
__device__ __forceinline__ int swz(int r, int p) { return r * N + 2 * (p ^ ((r >> 1) & 3)); }

// sum_q D[q][i] f1[q][j][k] + D[q][j] f2[i][q][k] + D[q][k] f3[i][j][q] for
// k = 2 kp + c: the reference's single interleaved chain (EX, _numba.py:119-126)
// or three DFMA chains (production)
template <bool EX>
__device__ __forceinline__ double out_point(const DMat<8>& D, const double (&f1)[N], const double (&djT)[N],
                                            const double (&dkT)[N], const double* f2s, const double* f3s, int i,
                                            int j, int kp, int c) {
  if constexpr (EX) {
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < N; q += 2) {
      const double2 t3 = *reinterpret_cast<const double2*>(f3s + i * NN + swz(j, q >> 1));
      const double s2a = f2s[i * NN + swz(q, kp) + c];
      const double s2b = f2s[i * NN + swz(q + 1, kp) + c];
      acc = mac<EX>(acc, D.v[q * N + i], f1[q]);
      acc = mac<EX>(acc, djT[q], s2a);
      acc = mac<EX>(acc, dkT[q], t3.x);
      acc = mac<EX>(acc, D.v[(q + 1) * N + i], f1[q + 1]);
      acc = mac<EX>(acc, djT[q + 1], s2b);
      acc = mac<EX>(acc, dkT[q + 1], t3.y);
    }
    return acc;
  } else {
    double ar = 0.0, as = 0.0, at = 0.0;
#pragma unroll
    for (int q = 0; q < N; q += 2) {
      const double2 t3 = *reinterpret_cast<const double2*>(f3s + i * NN + swz(j, q >> 1));
      const double s2a = f2s[i * NN + swz(q, kp) + c];
      const double s2b = f2s[i * NN + swz(q + 1, kp) + c];
      ar = fma(D.v[q * N + i], f1[q], ar);
      as = fma(djT[q], s2a, as);
      at = fma(dkT[q], t3.x, at);
      ar = fma(D.v[(q + 1) * N + i], f1[q + 1], ar);
      as = fma(djT[q + 1], s2b, as);
      at = fma(dkT[q + 1], t3.y, at);
    }
    return (ar + as) + at;
  }
}

template <bool EX, bool MASK, bool PRE, bool MASS>
__global__ void __launch_bounds__(THREADS, 1)
ax8t_kernel(DMat<8> D, const double* __restrict__ g, const double* __restrict__ b,
            const double* __restrict__ u, double* __restrict__ w, long long E, long long e0, long long e1,
            double lv, double lm, const uint32_t* __restrict__ inmask, const uint32_t* __restrict__ outsel,
            const double* __restrict__ pre) {
  constexpr int S = n_stages(PRE, MASS, MASK);
  constexpr int SB = stage_bytes(PRE, MASS, MASK);
  constexpr int OFF_PRE = 7 * FIELD;
  constexpr int OFF_B = OFF_PRE + (PRE ? FIELD : 0);
  constexpr int OFF_M = OFF_B + (MASS ? FIELD : 0);
  extern __shared__ __align__(1024) unsigned char smem[];
  // Barriers.  empty[s]: stage s released (waited only by the producer, in order).
  // full[w]: the data of compute warp w's next element has landed -- one barrier
  // per CONSUMER, not per stage: successive uses of a stage go to different warps,
  // and a parity wait by a warp two phases ahead of a stage's barrier would pass
  // spuriously.  A warp waits on its own barrier in order (CW >= S keeps a
  // barrier's previous use consumed before the producer re-arms it).
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + CW;
  double* Dr = reinterpret_cast<double*>(smem + 1024);   // D row-major
  double* Dc = Dr + NN;                                  // D transposed
  unsigned char* stages = smem + HEAD;
  double* scratch_all = reinterpret_cast<double*>(stages + S * SB);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long n_el = e1 - e0;
  // this CTA's elements: e0 + blockIdx.x + n * gridDim.x, n = 0 .. cnt-1
  const long long cnt = n_el > blockIdx.x ? (n_el - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  static_assert(CW >= S, "a full barrier is re-armed only after its previous element was consumed");
  if (threadIdx.x == 0) {
    for (int x = 0; x < CW; ++x) mbar_init(full + x, 1);
    for (int x = 0; x < S; ++x) mbar_init(empty + x, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int x = threadIdx.x; x < NN; x += blockDim.x) {
    Dr[x] = D.v[x];
    Dc[x] = D.v[(x & 7) * N + (x >> 3)];
  }
  __syncthreads();

  const long long gstride = E * (long long)NNN;
  if (warp == CW) {
    // ------------------------------------------------------------ producer
    if (lane != 0) return;
    const uint64_t pol = policy_evict_first();   // every operand byte is read once
    for (long long n = 0; n < cnt; ++n) {
      const int s = (int)(n % S);
      const unsigned ph = (unsigned)((n / S) & 1);
      if (n >= S) mbar_wait(empty + s, ph ^ 1u);
      const long long e = e0 + blockIdx.x + n * gridDim.x;
      unsigned char* st = stages + s * SB;
      uint64_t* fb = full + (int)(n % CW);
      mbar_expect_tx(fb, SB);
      bulk_g2s(st, u + e * NNN, FIELD, fb, pol);
#pragma unroll
      for (int m = 0; m < 6; ++m) bulk_g2s(st + (1 + m) * FIELD, g + m * gstride + e * NNN, FIELD, fb, pol);
      if constexpr (PRE) bulk_g2s(st + OFF_PRE, pre + e * NNN, FIELD, fb, pol);
      if constexpr (MASS) bulk_g2s(st + OFF_B, b + e * NNN, FIELD, fb, pol);
      if constexpr (MASK) {
        bulk_g2s(st + OFF_M, inmask + e * 16, 64, fb, pol);
        bulk_g2s(st + OFF_M + 64, outsel + e * 16, 64, fb, pol);
      }
    }
    return;
  }

  // -------------------------------------------------------------- compute warps
  const int j = lane >> 2, kp = lane & 3;
  const int k0 = 2 * kp;
  double* f2s = scratch_all + warp * (SCRATCH / 8);
  double* f3s = f2s + NNN;
  // Thread-dependent rows/columns of D come from the shared tables, reloaded at
  // the start of each pass (24 values each; keeping all 48 resident spills):
  //   forward  s: D[j][q]          t: D[k][q] (production: pair-rotated, see below)
  //   output   s: D[q][j]          t: D[q][k]        (r uses the uniform D[q][i])
  const int jr = (j >> 1) & 3;

  for (long long n = warp; n < cnt; n += CW) {
    const int s = (int)(n % S);
    const long long e = e0 + blockIdx.x + n * gridDim.x;
    unsigned char* st = stages + s * SB;
    double* su = reinterpret_cast<double*>(st);
    const double* sg = reinterpret_cast<const double*>(st + FIELD);
    mbar_wait(full + warp, (unsigned)((n / CW) & 1));

    // own pencils (j, k0) and (j, k0+1): um = the vector the operator acts on,
    // (inmask ? pre .* u : 0)
    double um0[N], um1[N];
    uint32_t inb = 0xffffu, outb = 0xffffu;   // bit 2i+c <-> point (i, j, k0+c)
    if constexpr (MASK) {
      const uint32_t* sm = reinterpret_cast<const uint32_t*>(st + OFF_M);
      inb = 0u;
      outb = 0u;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const int wd = 2 * i + (j >> 2), sh = (j & 3) * 8 + k0;
        inb |= ((sm[wd] >> sh) & 3u) << (2 * i);
        outb |= ((sm[16 + wd] >> sh) & 3u) << (2 * i);
      }
    }
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double2 v = *reinterpret_cast<const double2*>(su + i * NN + j * N + k0);
      if constexpr (PRE) {
        const double2 p = *reinterpret_cast<const double2*>(
            reinterpret_cast<const double*>(st + OFF_PRE) + i * NN + j * N + k0);
        v.x = __dmul_rn(p.x, v.x);
        v.y = __dmul_rn(p.y, v.y);
      }
      um0[i] = ((inb >> (2 * i)) & 1u) ? v.x : 0.0;
      um1[i] = ((inb >> (2 * i + 1)) & 1u) ? v.y : 0.0;
    }
    if constexpr (PRE || MASK) {
      // the derivatives read neighbours' points from the stage: store the
      // transformed values back (own points only), then make them warp-visible
#pragma unroll
      for (int i = 0; i < N; ++i)
        *reinterpret_cast<double2*>(su + i * NN + j * N + k0) = make_double2(um0[i], um1[i]);
      __syncwarp();
    }
    // mass term (lm * B) * um, formed while the stage holds B
    double mb0[N], mb1[N];
    if constexpr (MASS) {
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const double2 bv = *reinterpret_cast<const double2*>(
            reinterpret_cast<const double*>(st + OFF_B) + i * NN + j * N + k0);
        mb0[i] = mul<EX>(mul<EX>(lm, bv.x), um0[i]);
        mb1[i] = mul<EX>(mul<EX>(lm, bv.y), um1[i]);
      }
    }

    // ---------------------------------------------------------------- forward
    double dj[N], dt0[N], dt1[N];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      // production reads the t-row pairs in the order (m + jr) & 3 (conflict-free
      // LDS.128 for the 8 rows of a warp); entry 2m+x then holds q = 2 pm + x
      const int pm = EX ? m : ((m + jr) & 3);
      const double2 a = *reinterpret_cast<const double2*>(Dr + j * N + 2 * m);
      const double2 b0 = *reinterpret_cast<const double2*>(Dr + k0 * N + 2 * pm);
      const double2 b1 = *reinterpret_cast<const double2*>(Dr + (k0 + 1) * N + 2 * pm);
      dj[2 * m] = a.x;
      dj[2 * m + 1] = a.y;
      dt0[2 * m] = b0.x;
      dt0[2 * m + 1] = b0.y;
      dt1[2 * m] = b1.x;
      dt1[2 * m + 1] = b1.y;
    }
    double f1a[N], f1b[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double ar0 = 0.0, as0 = 0.0, at0 = 0.0, ar1 = 0.0, as1 = 0.0, at1 = 0.0;
      const double* sl = su + i * NN;
#pragma unroll
      for (int q = 0; q < N; ++q) {
        const double2 sv = *reinterpret_cast<const double2*>(sl + q * N + k0);
        ar0 = mac<EX>(ar0, D.v[i * N + q], um0[q]);
        as0 = mac<EX>(as0, dj[q], sv.x);
        ar1 = mac<EX>(ar1, D.v[i * N + q], um1[q]);
        as1 = mac<EX>(as1, dj[q], sv.y);
      }
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        // exact mode: pairs in reference order q = 0..7 (2-way bank conflicts)
        const int pm = EX ? m : ((m + jr) & 3);
        const double2 tv = *reinterpret_cast<const double2*>(sl + j * N + 2 * pm);
        at0 = mac<EX>(at0, dt0[2 * m], tv.x);
        at1 = mac<EX>(at1, dt1[2 * m], tv.x);
        at0 = mac<EX>(at0, dt0[2 * m + 1], tv.y);
        at1 = mac<EX>(at1, dt1[2 * m + 1], tv.y);
      }
      double2 gm[6];
#pragma unroll
      for (int m = 0; m < 6; ++m) gm[m] = *reinterpret_cast<const double2*>(sg + m * NNN + i * NN + j * N + k0);
      f1a[i] = add<EX>(add<EX>(mul<EX>(gm[0].x, ar0), mul<EX>(gm[1].x, as0)), mul<EX>(gm[2].x, at0));
      f1b[i] = add<EX>(add<EX>(mul<EX>(gm[0].y, ar1), mul<EX>(gm[1].y, as1)), mul<EX>(gm[2].y, at1));
      const double f2a = add<EX>(add<EX>(mul<EX>(gm[1].x, ar0), mul<EX>(gm[3].x, as0)), mul<EX>(gm[4].x, at0));
      const double f2b = add<EX>(add<EX>(mul<EX>(gm[1].y, ar1), mul<EX>(gm[3].y, as1)), mul<EX>(gm[4].y, at1));
      const double f3a = add<EX>(add<EX>(mul<EX>(gm[2].x, ar0), mul<EX>(gm[4].x, as0)), mul<EX>(gm[5].x, at0));
      const double f3b = add<EX>(add<EX>(mul<EX>(gm[2].y, ar1), mul<EX>(gm[4].y, as1)), mul<EX>(gm[5].y, at1));
      *reinterpret_cast<double2*>(f2s + i * NN + swz(j, kp)) = make_double2(f2a, f2b);
      *reinterpret_cast<double2*>(f3s + i * NN + swz(j, kp)) = make_double2(f3a, f3b);
      // keep the next layer's shared loads below this point: hoisting all eight
      // layers' loads (the full unroll) would spill
      asm volatile("" ::: "memory");
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + s);   // stage consumed: the producer may refill it

    // ----------------------------------------------------------------- output
    double djT[N], dkT0[N], dkT1[N];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const double2 a = *reinterpret_cast<const double2*>(Dc + j * N + 2 * m);
      const double2 b0 = *reinterpret_cast<const double2*>(Dc + k0 * N + 2 * m);
      const double2 b1 = *reinterpret_cast<const double2*>(Dc + (k0 + 1) * N + 2 * m);
      djT[2 * m] = a.x;
      djT[2 * m + 1] = a.y;
      dkT0[2 * m] = b0.x;
      dkT0[2 * m + 1] = b0.y;
      dkT1[2 * m] = b1.x;
      dkT1[2 * m + 1] = b1.y;
    }
    double* wp = w + e * NNN + j * N + k0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double res[2];
      res[0] = out_point<EX>(D, f1a, djT, dkT0, f2s, f3s, i, j, kp, 0);
      res[1] = out_point<EX>(D, f1b, djT, dkT1, f2s, f3s, i, j, kp, 1);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        double wv = mul<EX>(lv, res[c]);
        if constexpr (MASS) {
          if (lm != 0.0) wv = add<EX>(wv, c ? mb1[i] : mb0[i]);
        }
        if constexpr (MASK) {
          if (!((outb >> (2 * i + c)) & 1u)) {
            // Dirichlet row (not shared): the operator input passes through
            const long long pidx = e * NNN + i * NN + j * N + k0 + c;
            wv = __ldg(u + pidx);
            if constexpr (PRE) wv = __dmul_rn(__ldg(pre + pidx), wv);
          }
        }
        res[c] = wv;
      }
      *reinterpret_cast<double2*>(wp + i * NN) = make_double2(res[0], res[1]);
      asm volatile("" ::: "memory");
    }
    __syncwarp();   // every lane is done with the scratch before the next element
  }
}

}  // namespace ax8t

static int g_sms = 0;

template <bool EX, bool MASK, bool PRE, bool MASS>
static int launch_one(const DMat<8>& D, const double* g, const double* b, const double* u, double* w,
                      long long E, long long e0, long long e1, double lv, double lm, const uint32_t* inmask,
                      const uint32_t* outsel, const double* pre, cudaStream_t st) {
  using namespace ax8t;
  constexpr int S = n_stages(PRE, MASS, MASK);
  constexpr int smem = HEAD + S * stage_bytes(PRE, MASS, MASK) + CW * SCRATCH;
  static_assert(smem <= SMEM_MAX, "ax8t shared memory");
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(ax8t_kernel<EX, MASK, PRE, MASS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    configured = true;
  }
  if (g_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const long long n_el = e1 - e0;
  const unsigned grid = (unsigned)(n_el < g_sms ? n_el : g_sms);
  ax8t_kernel<EX, MASK, PRE, MASS><<<grid, THREADS, smem, st>>>(D, g, b, u, w, E, e0, e1, lv, lm, inmask, outsel,
                                                                pre);
  return check_launch("ax8t");
}

// Elements [e0, e1) of an E-element field, n = 8.  Returns SF_ERR_UNSUPPORTED when
// an operand is not 16-byte aligned (the caller then uses the register kernel).
int ax_helm8t(const DMat<8>& D, const double* g, const double* b, const double* u, double* w, long long E,
              long long e0, long long e1, double lv, double lm, const uint32_t* inmask, const uint32_t* outsel,
              const double* pre, int exact, cudaStream_t st) {
  auto al = [](const void* p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (!al(g) || !al(b) || !al(u) || !al(w) || !al(pre) || !al(inmask) || !al(outsel)) return SF_ERR_UNSUPPORTED;
  if (e1 <= e0) return SF_OK;
  const bool masked = inmask != nullptr, mass = lm != 0.0;
#define L(EXV, MV, PV, BV) return launch_one<EXV, MV, PV, BV>(D, g, b, u, w, E, e0, e1, lv, lm, inmask, outsel, pre, st)
#define LB(EXV, MV, PV) \
  if (mass) L(EXV, MV, PV, true); else L(EXV, MV, PV, false)
#define LP(EXV, MV) \
  if (pre) { LB(EXV, MV, true); } else { LB(EXV, MV, false); }
  if (exact) {
    if (masked) { LP(true, true); } else { LP(true, false); }
  } else {
    if (masked) { LP(false, true); } else { LP(false, false); }
  }
#undef LP
#undef LB
#undef L
}

}  // namespace sf
