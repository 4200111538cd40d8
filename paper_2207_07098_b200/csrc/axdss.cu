// Fused global operator, n = 8: Ax_helm (K1) and the shared-node dssum (K2) in
// ONE launch (operators.py:51-54: mask*gs.add(ax(mask*u)) + (1-mask)*u).
//
// Why.  K2 is latency-bound (scattered 8-byte accesses to the face copies, ncu:
// long-scoreboard stalls, ~40 % of DRAM peak) while K1 streams u and G.  Run back
// to back, the dssum's latency is exposed in full; interleaved with Ax work on
// the same SMs it could hide behind the Ax blocks' streaming.
//
// How.  The Ax element pairs are cut into chunks of about one wave.  The dssum
// items (shared gids) are assigned to the chunk holding their highest element
// and packed per (chunk, multiplicity class) into dssum blocks.  A schedule
// orders the work  A0 .. A_L D0 A_{L+1} D1 ...  (D_c after A_{c+L}, L = lag).
// An Ax block bumps its chunk's counter once its elements are written (fence +
// atomic, release); a dssum block spins (acquire) until the chunks [lo_c, c]
// its items read are complete.  No grid-wide barrier.
//
// Measured (32^3, B200): the interleaved dssum costs ~40 us instead of 88 us,
// but the dssum blocks run at the Ax kernel's occupancy (4 x 128 threads per
// SM, too few loads in flight for scattered gathers) and every Ax block pays a
// release fence: 310 us plain / 340 us masked against 308 / 333 us for the two
// kernels.  A persistent, ticket-scheduled variant was slower still (ticket
// latency per job).  The path is therefore OPT-IN (SEMFLOW_B200_FUSED=1); it is
// kept, tested bit-exact, as the base for a halo-overlapped multi-GPU operator.
//
// Results are bit-identical to K1 followed by K2: each element's arithmetic is
// ax8s_pair, each gid is summed by one thread in the reference order
// (kernels/_numba.py:134-153, sequential, starting from 0.0).
#include "ax8s.cuh"

namespace sf {

// Device view of the plan built by GatherScatter.fused_plan (space.py).
struct FusedPlan {
  const int* sched;   // [n_blocks] slot -> >= 0: Ax element pair, < 0: -1 - dssum block
  const int4* dtab;   // [n_dblk] {chunk, class 2/4/8/0(generic), first item, count}
  const int* need;    // [n_chunks] Ax blocks per chunk
  const int* lo;      // [n_chunks] lowest Ax chunk read by dssum chunk c
  const int2* p2;     // pairs
  const int4* p4;     // quads
  const int4* p8;     // octets (two int4 each)
  const int* goff;    // generic CSR offsets [n_gen + 1]
  const int* gperm;   // generic CSR entries
  int n_blocks;
  int chunk_pairs;    // Ax element pairs per chunk
  int n_chunks;
};

constexpr int DSS_THREADS = 128;
#ifndef SF_DSS_BATCH
#define SF_DSS_BATCH 4
#endif
constexpr int DSS_BATCH = SF_DSS_BATCH;  // pair gids in flight per thread

__device__ __forceinline__ unsigned long long ld_acquire_gpu(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ double ldv(const double* v, int p) { return __ldcg(v + (p & 0x7fffffff)); }

template <int MODE>
__device__ __forceinline__ void put(double* __restrict__ v, const double* __restrict__ u, int p, double s) {
  if (MODE == 2 && p < 0) {
    p &= 0x7fffffff;
    v[p] = __ldg(u + p);
  } else {
    v[p] = s;
  }
}

template <int MODE>
__device__ __forceinline__ void dss_items(const FusedPlan& pl, int4 d, double* __restrict__ v,
                                          const double* __restrict__ u) {
  const int first = d.z, end = d.z + d.w;
  if (d.y == 2) {
    for (int i0 = first + threadIdx.x; i0 < end; i0 += DSS_THREADS * DSS_BATCH) {
      int2 q[DSS_BATCH];
      double a[DSS_BATCH], b[DSS_BATCH];
#pragma unroll
      for (int k = 0; k < DSS_BATCH; ++k) {
        const int i = i0 + k * DSS_THREADS;
        q[k] = i < end ? __ldg(pl.p2 + i) : make_int2(0, 0);
      }
#pragma unroll
      for (int k = 0; k < DSS_BATCH; ++k) {
        if (i0 + k * DSS_THREADS < end) {
          a[k] = ldv(v, q[k].x);
          b[k] = ldv(v, q[k].y);
        }
      }
#pragma unroll
      for (int k = 0; k < DSS_BATCH; ++k) {
        if (i0 + k * DSS_THREADS < end) {
          const double s = __dadd_rn(__dadd_rn(0.0, a[k]), b[k]);
          put<MODE>(v, u, q[k].x, s);
          put<MODE>(v, u, q[k].y, s);
        }
      }
    }
  } else if (d.y == 4) {
    for (int i0 = first + threadIdx.x; i0 < end; i0 += DSS_THREADS * 2) {
      int4 q[2];
      double a[2][4];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int i = i0 + k * DSS_THREADS;
        q[k] = i < end ? __ldg(pl.p4 + i) : make_int4(0, 0, 0, 0);
      }
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        if (i0 + k * DSS_THREADS < end) {
          a[k][0] = ldv(v, q[k].x);
          a[k][1] = ldv(v, q[k].y);
          a[k][2] = ldv(v, q[k].z);
          a[k][3] = ldv(v, q[k].w);
        }
      }
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        if (i0 + k * DSS_THREADS < end) {
          double s = 0.0;
#pragma unroll
          for (int o = 0; o < 4; ++o) s = __dadd_rn(s, a[k][o]);
          put<MODE>(v, u, q[k].x, s);
          put<MODE>(v, u, q[k].y, s);
          put<MODE>(v, u, q[k].z, s);
          put<MODE>(v, u, q[k].w, s);
        }
      }
    }
  } else if (d.y == 8) {
    for (int i = first + threadIdx.x; i < end; i += DSS_THREADS) {
      const int4 qa = __ldg(pl.p8 + 2 * i), qb = __ldg(pl.p8 + 2 * i + 1);
      const int idx[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
      double a[8];
#pragma unroll
      for (int o = 0; o < 8; ++o) a[o] = ldv(v, idx[o]);
      double s = 0.0;
#pragma unroll
      for (int o = 0; o < 8; ++o) s = __dadd_rn(s, a[o]);
#pragma unroll
      for (int o = 0; o < 8; ++o) put<MODE>(v, u, idx[o], s);
    }
  } else {
    for (int i = first + threadIdx.x; i < end; i += DSS_THREADS) {
      const int o0 = __ldg(pl.goff + i), o1 = __ldg(pl.goff + i + 1);
      double s = 0.0;
      for (int o = o0; o < o1; ++o) s = __dadd_rn(s, ldv(v, __ldg(pl.gperm + o)));
      for (int o = o0; o < o1; ++o) put<MODE>(v, u, __ldg(pl.gperm + o), s);
    }
  }
}

// One block per schedule slot, slot = blockIdx.x.  Blocks are dispatched in
// index order (the property single-pass scans rely on), so a dssum block only
// waits on Ax blocks that are already resident or retired.  Counters are 64-bit
// and never reset: launch number `epoch` of a plan finds chunk c complete when
// its counter reaches (epoch + 1) * need[c].
template <bool EX, int MODE>
__global__ void __launch_bounds__(128, SF_AX8S_MINB)
ax_dssum8_kernel(DMat<8> D, const double* __restrict__ g, const double* __restrict__ b,
                    const double* __restrict__ u, double* __restrict__ w, long long E, double lv,
                    double lm, const uint32_t* __restrict__ inmask, const uint32_t* __restrict__ outsel,
                    FusedPlan pl, unsigned long long* __restrict__ sync, unsigned long long epoch) {
  const int job = __ldg(pl.sched + blockIdx.x);
  if (job >= 0) {
    ax8s_pair<EX, MODE == 2>(D, g, b, u, w, E, lv, lm, inmask, outsel, (long long)job);
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(sync + 1 + job / pl.chunk_pairs, 1ull);
    }
  } else {
    if (threadIdx.x == 0) {
      const int4 d = __ldg(pl.dtab + (-1 - job));
      for (int c = __ldg(pl.lo + d.x); c <= d.x; ++c) {
        const unsigned long long need = (epoch + 1ull) * (unsigned long long)__ldg(pl.need + c);
        while (ld_acquire_gpu(sync + 1 + c) < need) __nanosleep(64);
      }
    }
    __syncthreads();
#ifndef SF_FUSED_NO_DSS
    dss_items<MODE>(pl, __ldg(pl.dtab + (-1 - job)), w, u);
#endif
  }
}

// meta (host, int64): {n_jobs, chunk_pairs, n_chunks, off_sched, off_dtab,
//                       off_need, off_lo, off_p2, off_p4, off_p8, off_goff, off_gperm}
// offsets in int32 words from `plan`; sync: n_chunks + 1 zero-initialised uint64.
int ax_dssum8(const double* d_host, const double* g, const double* b, const double* u, double* w,
              long long E, double lv, double lm, const uint32_t* inmask, const uint32_t* outsel,
              int mode, const int* plan, const long long* meta, unsigned long long* sync,
              unsigned long long epoch, int exact, cudaStream_t st) {
  if (E <= 0) return SF_OK;
  if ((inmask == nullptr) != (outsel == nullptr) || (mode == 2) != (inmask != nullptr) ||
      (mode != 0 && mode != 2)) {
    set_error("ax_dssum: mode %d inconsistent with the masks (0 = plain, 2 = masked)", mode);
    return SF_ERR_ARG;
  }
  if (plan == nullptr || meta == nullptr || sync == nullptr || meta[0] <= 0 || meta[1] <= 0) {
    set_error("ax_dssum: missing or empty plan");
    return SF_ERR_ARG;
  }
  DMat<8> D;
  for (int x = 0; x < 64; ++x) D.v[x] = d_host[x];
  FusedPlan pl;
  pl.sched = plan + meta[3];
  pl.dtab = reinterpret_cast<const int4*>(plan + meta[4]);
  pl.need = plan + meta[5];
  pl.lo = plan + meta[6];
  pl.p2 = reinterpret_cast<const int2*>(plan + meta[7]);
  pl.p4 = reinterpret_cast<const int4*>(plan + meta[8]);
  pl.p8 = reinterpret_cast<const int4*>(plan + meta[9]);
  pl.goff = plan + meta[10];
  pl.gperm = plan + meta[11];
  pl.n_blocks = (int)meta[0];
  pl.chunk_pairs = (int)meta[1];
  pl.n_chunks = (int)meta[2];
#define SF_FUSED_LAUNCH(EXV, MV, IM, OS)                                                   \
  ax_dssum8_kernel<EXV, MV><<<pl.n_blocks, 128, 0, st>>>(D, g, b, u, w, E, lv, lm, IM, OS, pl, \
                                                         sync, epoch)
  if (exact) {
    if (mode == 2) SF_FUSED_LAUNCH(true, 2, inmask, outsel);
    else SF_FUSED_LAUNCH(true, 0, nullptr, nullptr);
  } else {
    if (mode == 2) SF_FUSED_LAUNCH(false, 2, inmask, outsel);
    else SF_FUSED_LAUNCH(false, 0, nullptr, nullptr);
  }
#undef SF_FUSED_LAUNCH
  return check_launch("ax_dssum8");
}

}  // namespace sf
