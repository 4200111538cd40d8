// Hybrid overlapping Schwarz preconditioner, application (reference
// precond.py:94-250, HybridSchwarz.__call__ at :239-250).  Stream-ordered
// launches, no host synchronisation, CUDA-graph capturable:
//
//   gather    rg[g] = r[first copy of g]; rw[g] = wsqrt[g] * rg[g]      (:241-242)
//   restrict  rc = P^T rg: per element corner sums, then per vertex     (:246-247)
//   coarse    fixed-iteration Jacobi-CG on the vertex problem (:205-230), one
//             persistent launch with software grid barriers
//   local     sol_e = A_e^{-1} rw[sub_e] for every subdomain (:243-244): the
//             explicit inverses of the DISTINCT subdomain matrices; the operand
//             Rw = rw[sub] is gathered here (rows grouped by class) and each
//             class's products are one FP64 GEMM (cuBLAS, issued by the host)
//   finalize  z[g] = (sum over subdomains holding g, ascending) sol * wsqrt[g]
//             + sum_v (ascending) P[g, v] xc[v]; z = rg on constrained g  (:244-249)
//   scatter   out[p] = z[gid[p]]                                          (:250)
//
// The prolongation P (trilinear weights of a point to the corners of its
// element, precond.py:184-201) is not stored: P[g, v] = tw[p_g, c] with p_g the
// local index of g's first copy and c the corner of that element at vertex v.
// All sums run in the reference's order (ascending subdomain / gid / vertex) and
// in fixed trees for the coarse dots: deterministic, atomics only in the barrier.
#include <cstring>

#include "common.cuh"
#include "../../include/semflow_b200.h"

namespace sf {

__global__ void sch_gather_kernel(const double* __restrict__ r, const long long* __restrict__ first,
                                  const double* __restrict__ wsqrt, long long G, double* __restrict__ rg,
                                  double* __restrict__ rw) {
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < G;
       g += (long long)gridDim.x * blockDim.x) {
    SF_CHECK(first[g] >= 0);
    const double v = r[first[g]];
    rg[g] = v;
    rw[g] = __dmul_rn(wsqrt[g], v);
  }
}

// Restriction rc = P^T rg in two deterministic stages.
//   element: se[e][c] = sum over the points p of e that carry their gid's owned
//            first copy (rflag) of tw[p, c] * rg[node(p)] -- each gid counted once;
//            a warp per element, lane-strided points, a fixed xor tree
//   vertex:  rc[v] = sum over the (e, c) at vertex v, ascending e, of se[e][c]
// (the reference sums per vertex over gids ascending, precond.py:246; the coarse
// solve is approximate, one rounding order is as good as another, this one reads
// every point once and coalesced instead of ~(2n-1)^3 scattered gids per vertex)
__global__ void sch_restrict_elem_kernel(const double* __restrict__ rg, const long long* __restrict__ node,
                                         const uint8_t* __restrict__ rflag, const double* __restrict__ tw,
                                         int nnn, long long E, double* __restrict__ se) {
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long e = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; e < E; e += warps) {
    double acc[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c] = 0.0;
    for (int p = lane; p < nnn; p += 32) {
      const long long q = e * nnn + p;
      if (rflag[q]) {
        const double v = rg[node[q]];
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[c] = __dadd_rn(acc[c], __dmul_rn(tw[p * 8 + c], v));
      }
    }
#pragma unroll
    for (int c = 0; c < 8; ++c)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[c] = __dadd_rn(acc[c], __shfl_xor_sync(0xffffffffu, acc[c], o));
    if (lane < 8) {
      double mine = acc[0];
#pragma unroll
      for (int c = 1; c < 8; ++c)
        if (lane == c) mine = acc[c];
      se[e * 8 + lane] = mine;
    }
  }
}

__global__ void sch_restrict_vert_kernel(const double* __restrict__ se, const long long* __restrict__ vptr,
                                         const long long* __restrict__ vent, long long nv,
                                         const uint8_t* __restrict__ vfixed, double* __restrict__ rc) {
  for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < nv;
       v += (long long)gridDim.x * blockDim.x) {
    double acc = 0.0;
    if (!vfixed[v])
      for (long long k = vptr[v]; k < vptr[v + 1]; ++k) acc = __dadd_rn(acc, se[vent[k]]);
    rc[v] = acc;
  }
}

// ----------------------------------------------------------------- coarse CG

struct CoarseArgs {
  long long nv;
  int width;                        // ELL row width of the coarse matrix
  const int* col;                   // (nv, width), padded with the row's own index, value 0
  const double* val;
  const double* inv_diag;
  const double* rc;
  double* x;                        // output
  double* r;
  double* z;
  double* p;
  double* ap;
  double* part;                     // 2 * gridDim partial sums (ping-pong)
  unsigned* bar;                    // [0] arrivals, [1] exits
  int iters;
};

__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    while (true) {
      unsigned v;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
      if (v >= target) break;
      __nanosleep(32);
    }
  }
  __syncthreads();
}

// fixed-order block sum of one value per thread; result valid in thread 0
__device__ __forceinline__ double block_sum(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s = __dadd_rn(s, sh[i]);
  __syncthreads();
  return s;
}

// every block combines the partials of all blocks in block order: the same
// scalar on every block, a pure function of the data and gridDim
__device__ __forceinline__ double grid_dot(double mine, double* part, int slot, unsigned* bar,
                                           unsigned& nbar, double* sh) {
  const double b = block_sum(mine, sh);
  if (threadIdx.x == 0) part[slot * gridDim.x + blockIdx.x] = b;
  nbar += gridDim.x;
  grid_barrier(bar, nbar);
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (unsigned i = 0; i < gridDim.x; ++i) s = __dadd_rn(s, ((volatile double*)part)[slot * gridDim.x + i]);
    sh[32] = s;
  }
  __syncthreads();
  const double s = sh[32];
  __syncthreads();
  return s;
}

__global__ void __launch_bounds__(256) sch_coarse_cg_kernel(CoarseArgs a) {
  __shared__ double sh[33];
  unsigned nbar = 0;
  int slot = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long t0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  // x = 0; r = rc; z = D r; p = z; rz = <r, z>
  double loc = 0.0;
  for (long long v = t0; v < a.nv; v += stride) {
    const double rv = a.rc[v];
    const double zv = __dmul_rn(a.inv_diag[v], rv);
    a.x[v] = 0.0;
    a.r[v] = rv;
    a.z[v] = zv;
    a.p[v] = zv;
    loc = __dadd_rn(loc, __dmul_rn(rv, zv));
  }
  double rz = grid_dot(loc, a.part, slot, a.bar, nbar, sh);
  slot ^= 1;
  if (rz > 0.0) {
    for (int it = 0; it < a.iters; ++it) {
      // ap = A p; <p, ap>
      loc = 0.0;
      for (long long v = t0; v < a.nv; v += stride) {
        double s = 0.0;
        const int* c = a.col + v * a.width;
        const double* w = a.val + v * a.width;
        for (int k = 0; k < a.width; ++k) s = __dadd_rn(s, __dmul_rn(w[k], __ldcg(a.p + c[k])));
        a.ap[v] = s;
        loc = __dadd_rn(loc, __dmul_rn(a.p[v], s));
      }
      const double pap = grid_dot(loc, a.part, slot, a.bar, nbar, sh);
      slot ^= 1;
      if (!(pap > 0.0)) break;
      const double alpha = rz / pap;
      loc = 0.0;
      for (long long v = t0; v < a.nv; v += stride) {
        a.x[v] = __dadd_rn(a.x[v], __dmul_rn(alpha, a.p[v]));
        const double rv = __dsub_rn(a.r[v], __dmul_rn(alpha, a.ap[v]));
        a.r[v] = rv;
        const double zv = __dmul_rn(a.inv_diag[v], rv);
        a.z[v] = zv;
        loc = __dadd_rn(loc, __dmul_rn(rv, zv));
      }
      const double rz_new = grid_dot(loc, a.part, slot, a.bar, nbar, sh);
      slot ^= 1;
      if (!(rz_new > 0.0)) break;
      const double beta = rz_new / rz;
      for (long long v = t0; v < a.nv; v += stride) a.p[v] = __dadd_rn(a.z[v], __dmul_rn(beta, a.p[v]));
      rz = rz_new;
      nbar += gridDim.x;
      grid_barrier(a.bar, nbar);        // p complete before the next product
    }
  }
  // the last block out resets the barrier words for the next launch
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(a.bar + 1, 1u) == gridDim.x - 1) {
      a.bar[0] = 0u;
      a.bar[1] = 0u;
      __threadfence();
    }
  }
}

// ----------------------------------------------------------------- local solves

// Rw[p][j] = rw[sub[p][j]]: the weighted residual of every subdomain slot, rows in
// class order (the operand of the per-class solve GEMM sol_c = Rw_c inv_c^T)
__global__ void sch_gather_rw_kernel(const double* __restrict__ rw, const int* __restrict__ sub, long long n,
                                     long long L, double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    SF_CHECK(sub[i] >= 0 && sub[i] <= L);     // rw[L] is the zero padding slot
    out[i] = rw[sub[i]];
  }
}

// z[g] = con ? rg : (sum_k sol[pos[k]]) * wsqrt + sum over the corners of g's
// first element in ascending vertex id of tw[p*8+c] * xc[vertex]
__global__ void sch_finalize_kernel(const double* __restrict__ sol, const double* __restrict__ sol_recv,
                                    long long n_sol, const long long* __restrict__ off,
                                    const int* __restrict__ pos, const double* __restrict__ wsqrt,
                                    const long long* __restrict__ first, int nnn,
                                    const int* __restrict__ cvert, const uint8_t* __restrict__ ccorn,
                                    const double* __restrict__ tw, const double* __restrict__ xc,
                                    const uint8_t* __restrict__ con, const double* __restrict__ rg,
                                    long long G, double* __restrict__ z) {
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < G;
       g += (long long)gridDim.x * blockDim.x) {
    if (con[g]) { z[g] = rg[g]; continue; }
    double acc = 0.0;
    for (long long k = off[g]; k < off[g + 1]; ++k) {
      const long long q = pos[k];            // own subdomains' slots, then the peers' (N > 1)
      SF_CHECK(q >= 0 && (q < n_sol || sol_recv != nullptr));
      acc = __dadd_rn(acc, q < n_sol ? sol[q] : sol_recv[q - n_sol]);
    }
    const long long fp = first[g];
    const long long e = fp / nnn;
    const int p = (int)(fp - e * nnn);
    double pc = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int c = ccorn[e * 8 + k];
      pc = __dadd_rn(pc, __dmul_rn(tw[p * 8 + c], xc[cvert[e * 8 + k]]));
    }
    z[g] = __dadd_rn(__dmul_rn(acc, wsqrt[g]), pc);
  }
}

__global__ void sch_scatter_kernel(const double* __restrict__ z, const long long* __restrict__ gid,
                                   long long P, long long G, double* __restrict__ out) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < P;
       p += (long long)gridDim.x * blockDim.x) {
    SF_CHECK(gid[p] >= 0 && gid[p] < G);
    out[p] = z[gid[p]];
  }
}

// out[v] = sum over ranks in rank order of the partial restrictions: own partial
// at position `rank`, the peers' (ascending rank, self skipped) in recv
__global__ void sch_rank_sum_kernel(const double* __restrict__ own, const double* __restrict__ recv, int rank,
                                    int world, long long nv, double* __restrict__ out) {
  for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < nv;
       v += (long long)gridDim.x * blockDim.x) {
    double acc = 0.0;
    int k = 0;
    for (int q = 0; q < world; ++q) {
      if (q == rank) acc = __dadd_rn(acc, own[v]);
      else acc = __dadd_rn(acc, recv[(long long)(k++) * nv + v]);
    }
    out[v] = acc;
  }
}

// copy the current bank of a double-banked NVLink inbox (csrc/halo.cu) to out
__global__ void halo_unbank_kernel(const double* __restrict__ bank0, const unsigned long long* __restrict__ seq,
                                   long long stride, long long n, double* __restrict__ out) {
  const double* src = bank0 + (long long)(*seq & 1ull) * stride;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = src[i];
}

static unsigned grid_for(long long n) {
  long long b = (n + 255) / 256;
  if (b < 1) b = 1;
  if (b > 148 * 16) b = 148 * 16;
  return (unsigned)b;
}

}  // namespace sf

extern "C" {

int sf_schwarz_coarse_blocks(void) {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

static int bad(const SfSchwarz* s, const char* what) {
  if (!s || s->S <= 0 || s->G < 0) {
    sf::set_error("%s: bad arguments", what);
    return 1;
  }
  return 0;
}

// stage 1: rg / rw of this rank's nodes (gids with a local copy)
int sf_schwarz_gather_f64(const SfSchwarz* s, const double* r, void* stream) {
  using namespace sf;
  if (bad(s, "sf_schwarz_gather_f64") || !r) return SF_ERR_ARG;
  sch_gather_kernel<<<grid_for(s->G), 256, 0, as_stream(stream)>>>(r, s->first, s->wsqrt, s->G, s->rg, s->rw);
  return check_launch("schwarz gather");
}

// stage 2: restriction of the owned nodes -> rc_part
int sf_schwarz_restrict_f64(const SfSchwarz* s, void* stream) {
  using namespace sf;
  if (bad(s, "sf_schwarz_restrict_f64")) return SF_ERR_ARG;
  const long long E = s->P / s->nnn;
  sch_restrict_elem_kernel<<<grid_for(E * 32), 256, 0, as_stream(stream)>>>(s->rg, s->gid, s->rflag, s->tw, s->nnn,
                                                                          E, s->se);
  if (int e = check_launch("schwarz restrict (elements)")) return e;
  sch_restrict_vert_kernel<<<grid_for(s->nv), 256, 0, as_stream(stream)>>>(s->se, s->pt_ptr, s->pt_ent, s->nv,
                                                                          s->vfixed, s->rc_part);
  return check_launch("schwarz restrict (vertices)");
}

// N > 1: rc = rank-order sum of every rank's rc_part (own + received partials)
int sf_schwarz_rank_sum_f64(const SfSchwarz* s, const double* recv, int rank, int world, void* stream) {
  using namespace sf;
  if (bad(s, "sf_schwarz_rank_sum_f64")) return SF_ERR_ARG;
  sch_rank_sum_kernel<<<grid_for(s->nv), 256, 0, as_stream(stream)>>>(s->rc_part, recv, rank, world, s->nv, s->rc);
  return check_launch("schwarz rank sum");
}

// stage 3: coarse Jacobi-CG (one persistent launch) rc -> xc
int sf_schwarz_coarse_f64(const SfSchwarz* s, void* stream) {
  using namespace sf;
  if (bad(s, "sf_schwarz_coarse_f64")) return SF_ERR_ARG;
  CoarseArgs a;
  a.nv = s->nv; a.width = s->ac_width; a.col = s->ac_col; a.val = s->ac_val; a.inv_diag = s->ac_inv_diag;
  a.rc = s->rc; a.x = s->xc; a.r = s->cr; a.z = s->cz; a.p = s->cp; a.ap = s->cap; a.part = s->cpart;
  a.bar = s->cbar; a.iters = s->coarse_iters;
  sch_coarse_cg_kernel<<<s->coarse_blocks, 256, 0, as_stream(stream)>>>(a);
  return check_launch("schwarz coarse");
}

// stage 4a: the solve operand Rw = rw[sub] (rows in class order); the per-class
// products sol_c = Rw_c inv_c^T are FP64 GEMMs issued by the host (cuBLAS)
int sf_schwarz_gather_rw_f64(const SfSchwarz* s, void* stream) {
  using namespace sf;
  if (bad(s, "sf_schwarz_gather_rw_f64")) return SF_ERR_ARG;
  const long long n = s->n_sol;
  sch_gather_rw_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(s->rw, s->sub, n, s->L, s->rwg);
  return check_launch("schwarz gather rw");
}

// stage 5: ordered overlap sums (own + received solutions) + prolongation -> z
int sf_schwarz_finalize_f64(const SfSchwarz* s, void* stream) {
  using namespace sf;
  if (bad(s, "sf_schwarz_finalize_f64")) return SF_ERR_ARG;
  sch_finalize_kernel<<<grid_for(s->G), 256, 0, as_stream(stream)>>>(
      s->sol, s->sol_recv, s->n_sol, s->acc_off, s->acc_pos, s->wsqrt, s->first, s->nnn, s->cvert, s->ccorn, s->tw,
      s->xc, s->constrained, s->rg, s->G, s->z);
  return check_launch("schwarz finalize");
}

// stage 6: out[p] = z[node of p]
int sf_schwarz_scatter_f64(const SfSchwarz* s, double* out, void* stream) {
  using namespace sf;
  if (bad(s, "sf_schwarz_scatter_f64") || !out) return SF_ERR_ARG;
  sch_scatter_kernel<<<grid_for(s->P), 256, 0, as_stream(stream)>>>(s->z, s->gid, s->P, s->G, out);
  return check_launch("schwarz scatter");
}

// copy the current bank of an NVLink halo inbox to out (n doubles)
int sf_halo_unbank_f64(const double* bank0, const unsigned long long* seq, long long stride, long long n,
                       double* out, void* stream) {
  using namespace sf;
  if (n <= 0) return SF_OK;
  if (!bank0 || !seq || !out) {
    set_error("sf_halo_unbank_f64: bad arguments");
    return SF_ERR_ARG;
  }
  halo_unbank_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(bank0, seq, stride, n, out);
  return check_launch("halo unbank");
}

}  // extern "C"
