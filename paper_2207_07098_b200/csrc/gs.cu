// Gather-scatter (direct stiffness summation, "dssum" / QQ^T) kernels (K2).
//
// Reference semantics:
//   gs_gather   kernels/_numba.py:134-143  sums[g] = 0.0 + v[perm[o0]] + v[perm[o0+1]] ...
//               (sequential, ascending local index within the gid segment)
//   gs_scatter  kernels/_numba.py:146-153  out[perm[o]] = sums[g]
//   GatherScatter.add / avg   space.py:38-60 (avg multiplies by 1.0/count)
//   make_global_op            operators.py:51-54 (masked finalisation)
//
// The production dssum works on the *shared* part of the map only: gids with
// multiplicity > 1 (S_g of them, S_l local copies).  Unshared points are
// identity under QQ^T and are never touched.  One thread owns one shared gid and
// sums its copies sequentially in the reference order, so the result is
// bit-identical to the numba lane and independent of launch geometry; there are
// no atomics.  perm entries are int32 local indices; in the masked-operator map a
// negative entry (bit 31 set) marks a Dirichlet-masked copy, which receives the
// operator input u instead of the sum (`mask*gs.add(w) + (1-mask)*u`).
#include "common.cuh"

namespace sf {

__global__ void gs_gather_kernel(const double* __restrict__ vals, const long long* __restrict__ perm,
                                 const long long* __restrict__ off, long long n_gid,
                                 double* __restrict__ sums) {
  long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_gid) return;
  double acc = 0.0;
  for (long long o = off[g]; o < off[g + 1]; ++o) acc = __dadd_rn(acc, vals[perm[o]]);
  sums[g] = acc;
}

__global__ void gs_scatter_kernel(const double* __restrict__ sums, const long long* __restrict__ perm,
                                  const long long* __restrict__ off, long long n_gid,
                                  double* __restrict__ out) {
  long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_gid) return;
  const double v = sums[g];
  for (long long o = off[g]; o < off[g + 1]; ++o) out[perm[o]] = v;
}

// MODE 0: add (QQ^T).  MODE 1: avg (sum * (1.0/count)).  MODE 2: masked-operator
// finalisation (negative perm entry -> write u[idx]).
// Entries >= n_local refer to copies owned by another rank: their raw values
// were received into `recv` (entry - n_local), they are summed in place in the
// global order and never written (their owner finalises them).
template <int MODE>
__global__ void dssum_shared_kernel(double* __restrict__ v, const int* __restrict__ off,
                                    const int* __restrict__ perm, int n_shared,
                                    const double* __restrict__ u, const double* __restrict__ recv,
                                    int n_local) {
  int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_shared) return;
  const int o0 = __ldg(off + g), o1 = __ldg(off + g + 1);
  double acc = 0.0;
  for (int o = o0; o < o1; ++o) {
    const int p = __ldg(perm + o) & 0x7fffffff;
    acc = __dadd_rn(acc, p < n_local ? v[p] : __ldg(recv + (p - n_local)));
  }
  if (MODE == 1) acc = __dmul_rn(acc, __drcp_rn((double)(o1 - o0)));
  for (int o = o0; o < o1; ++o) {
    int p = __ldg(perm + o);
    if (MODE == 2 && p < 0) {
      p &= 0x7fffffff;
      v[p] = u[p];
    } else if (p < n_local) {
      v[p] = acc;
    }
  }
}

// Multiplicity-class dssum.  The shared gids are stored class by class: n2 pairs,
// n4 quads and n8 octets (fixed stride, no offsets: box-mesh faces, edges and
// vertices), then n_gen gids of any other count through CSR offsets (unstructured
// meshes, multi-rank interfaces).  A pair costs one int2 index load, two value
// loads and two stores -- the offsets load is gone from the dependent chain that
// bounds the CSR kernel (ncu: 30 cycles of long-scoreboard stall per instruction,
// 39 % of DRAM peak).  Per-gid order and arithmetic are unchanged.
// The pairs segment is padded to a multiple of 4 ints so the quads and octets
// that follow are 16-byte aligned for their int4 loads.
__host__ __device__ __forceinline__ long long pairs_span(int n2) { return (2LL * n2 + 3) & ~3LL; }

// masked finalisation value: the operator input u, or pre .* u when the operator
// was applied to the Jacobi-scaled vector on the fly (sf_ax_pre_f64)
__device__ __forceinline__ double dss_input(const double* __restrict__ u, const double* __restrict__ pre,
                                           int p) {
  const double x = u[p];
  return pre != nullptr ? __dmul_rn(__ldg(pre + p), x) : x;
}

template <int MODE>
__device__ __forceinline__ void dss_finish(double* __restrict__ v, const double* __restrict__ u,
                                           const int* idx, int c, double acc, int n_local,
                                           const double* __restrict__ pre = nullptr) {
  if (MODE == 1) acc = __dmul_rn(acc, __drcp_rn((double)c));
  for (int o = 0; o < c; ++o) {
    int p = idx[o];
    if (MODE == 2 && p < 0) {
      p &= 0x7fffffff;
      SF_CHECK(p < n_local);
      v[p] = dss_input(u, pre, p);
    } else if (p < n_local) {
      v[p] = acc;
    }
  }
}

__device__ __forceinline__ double dss_load(const double* __restrict__ v, const double* __restrict__ recv,
                                           int p, int n_local) {
  p &= 0x7fffffff;
  SF_CHECK(p < n_local || recv != nullptr);   // a remote copy needs the halo inbox
  return p < n_local ? v[p] : __ldg(recv + (p - n_local));
}

template <int MODE>
__global__ void __launch_bounds__(256)
dssum_cls_kernel(double* __restrict__ v, const int* __restrict__ perm, int n2, int n4, int n8,
                 const int* __restrict__ gen_off, int n_gen, const double* __restrict__ u,
                 const double* __restrict__ recv, int n_local) {
  int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g < n2) {
    const int2 q = __ldg(reinterpret_cast<const int2*>(perm) + g);
    const int idx[2] = {q.x, q.y};
    double acc = 0.0;
    acc = __dadd_rn(acc, dss_load(v, recv, q.x, n_local));
    acc = __dadd_rn(acc, dss_load(v, recv, q.y, n_local));
    dss_finish<MODE>(v, u, idx, 2, acc, n_local);
    return;
  }
  g -= n2;
  const int* p4 = perm + pairs_span(n2);
  if (g < n4) {
    const int4 q = __ldg(reinterpret_cast<const int4*>(p4) + g);
    const int idx[4] = {q.x, q.y, q.z, q.w};
    double acc = 0.0;
#pragma unroll
    for (int o = 0; o < 4; ++o) acc = __dadd_rn(acc, dss_load(v, recv, idx[o], n_local));
    dss_finish<MODE>(v, u, idx, 4, acc, n_local);
    return;
  }
  g -= n4;
  const int* p8 = p4 + 4LL * n4;
  if (g < n8) {
    const int4 qa = __ldg(reinterpret_cast<const int4*>(p8) + 2 * g);
    const int4 qb = __ldg(reinterpret_cast<const int4*>(p8) + 2 * g + 1);
    const int idx[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
    double acc = 0.0;
#pragma unroll
    for (int o = 0; o < 8; ++o) acc = __dadd_rn(acc, dss_load(v, recv, idx[o], n_local));
    dss_finish<MODE>(v, u, idx, 8, acc, n_local);
    return;
  }
  g -= n8;
  if (g < n_gen) {
    const int* pg = p8 + 8LL * n8;
    const int o0 = __ldg(gen_off + g), o1 = __ldg(gen_off + g + 1);
    double acc = 0.0;
    for (int o = o0; o < o1; ++o) acc = __dadd_rn(acc, dss_load(v, recv, __ldg(pg + o), n_local));
    if (MODE == 1) acc = __dmul_rn(acc, __drcp_rn((double)(o1 - o0)));
    for (int o = o0; o < o1; ++o) {
      int p = __ldg(pg + o);
      if (MODE == 2 && p < 0) {
        p &= 0x7fffffff;
        v[p] = u[p];
      } else if (p < n_local) {
        v[p] = acc;
      }
    }
  }
}

// Element-blocked dssum.  Same classes and per-gid arithmetic as dssum_cls_kernel,
// but block b owns every gid whose lowest local copy lies in elements
// [b*EB, (b+1)*EB), all classes (pairs, then quads, octets, generic).  ncu on the
// class-by-class kernel: DRAM traffic 3.74 GB per launch at 64^3 against 1.67 GB
// of algorithmic bytes -- a copy on a t-face uses 8 B of its 32 B sector, and the
// sectors shared by face, edge and vertex copies were fetched once per class pass
// (edges and vertices run long after the faces of the same element).  Keeping an
// element range's classes together in one block lets those sectors hit in L2.
// bstart: 4 x (nb + 1) item offsets (per class, relative to the class start).
#ifndef SF_DSS_PB
#define SF_DSS_PB 2
#endif
constexpr int DSS_PB = SF_DSS_PB;

template <int MODE>
__global__ void __launch_bounds__(256)
dssum_blk_kernel(double* __restrict__ v, const int* __restrict__ perm, int n2, int n4, int n8,
                 const int* __restrict__ gen_off, const int* __restrict__ bstart, int nb,
                 const double* __restrict__ u, const double* __restrict__ pre,
                 const double* __restrict__ recv, int n_local,
                 const unsigned long long* __restrict__ recv_seq, long long recv_bank) {
  const int b = blockIdx.x;
  // NVLink halo inbox: the bank of the current exchange is chosen by the call
  // number in device memory (halo.cu), so the launch arguments never change
  if (recv_seq != nullptr) recv += (long long)(*recv_seq & 1ull) * recv_bank;
  const int2* p2 = reinterpret_cast<const int2*>(perm);
  const int4* p4 = reinterpret_cast<const int4*>(perm + pairs_span(n2));
  const int4* p8 = reinterpret_cast<const int4*>(perm + pairs_span(n2) + 4LL * n4);
  const int* pg = perm + pairs_span(n2) + 4LL * n4 + 8LL * n8;
  {
    const int s = __ldg(bstart + b), e = __ldg(bstart + b + 1);
    // DSS_PB pairs per thread in flight: all index loads, then all value loads,
    // then the sums and stores (the kernel is latency-bound: ncu long-scoreboard)
    for (int g = s + threadIdx.x; g < e; g += DSS_PB * blockDim.x) {
      int2 q[DSS_PB];
      double a0[DSS_PB], a1[DSS_PB];
#pragma unroll
      for (int k = 0; k < DSS_PB; ++k) {
        const int gk = g + k * blockDim.x;
        q[k] = gk < e ? __ldg(p2 + gk) : make_int2(0, 0);
      }
#pragma unroll
      for (int k = 0; k < DSS_PB; ++k) {
        if (g + k * blockDim.x < e) {
          a0[k] = dss_load(v, recv, q[k].x, n_local);
          a1[k] = dss_load(v, recv, q[k].y, n_local);
        }
      }
#pragma unroll
      for (int k = 0; k < DSS_PB; ++k) {
        if (g + k * blockDim.x < e) {
          const int ik[2] = {q[k].x, q[k].y};
          dss_finish<MODE>(v, u, ik, 2, __dadd_rn(__dadd_rn(0.0, a0[k]), a1[k]), n_local, pre);
        }
      }
    }
  }
  {
    const int s = __ldg(bstart + (nb + 1) + b), e = __ldg(bstart + (nb + 1) + b + 1);
    for (int g = s + threadIdx.x; g < e; g += blockDim.x) {
      const int4 q = __ldg(p4 + g);
      const int idx[4] = {q.x, q.y, q.z, q.w};
      double a[4];
#pragma unroll
      for (int o = 0; o < 4; ++o) a[o] = dss_load(v, recv, idx[o], n_local);
      double acc = 0.0;
#pragma unroll
      for (int o = 0; o < 4; ++o) acc = __dadd_rn(acc, a[o]);
      dss_finish<MODE>(v, u, idx, 4, acc, n_local, pre);
    }
  }
  {
    const int s = __ldg(bstart + 2 * (nb + 1) + b), e = __ldg(bstart + 2 * (nb + 1) + b + 1);
    for (int g = s + threadIdx.x; g < e; g += blockDim.x) {
      const int4 qa = __ldg(p8 + 2 * g), qb = __ldg(p8 + 2 * g + 1);
      const int idx[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
      double a[8];
#pragma unroll
      for (int o = 0; o < 8; ++o) a[o] = dss_load(v, recv, idx[o], n_local);
      double acc = 0.0;
#pragma unroll
      for (int o = 0; o < 8; ++o) acc = __dadd_rn(acc, a[o]);
      dss_finish<MODE>(v, u, idx, 8, acc, n_local, pre);
    }
  }
  {
    const int s = __ldg(bstart + 3 * (nb + 1) + b), e = __ldg(bstart + 3 * (nb + 1) + b + 1);
    for (int g = s + threadIdx.x; g < e; g += blockDim.x) {
      const int o0 = __ldg(gen_off + g), o1 = __ldg(gen_off + g + 1);
      double acc = 0.0;
      for (int o = o0; o < o1; ++o) acc = __dadd_rn(acc, dss_load(v, recv, __ldg(pg + o), n_local));
      if (MODE == 1) acc = __dmul_rn(acc, __drcp_rn((double)(o1 - o0)));
      for (int o = o0; o < o1; ++o) {
        int p = __ldg(pg + o);
        if (MODE == 2 && p < 0) {
          p &= 0x7fffffff;
          v[p] = dss_input(u, pre, p);
        } else if (p < n_local) {
          v[p] = acc;
        }
      }
    }
  }
}

__global__ void gather_kernel(double* __restrict__ out, const double* __restrict__ v,
                              const int* __restrict__ idx, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = v[idx[i]];
}

// out[j] = buf[0*k + j] + buf[1*k + j] + ... in rank order (deterministic allreduce)
__global__ void rank_sum_kernel(const double* __restrict__ buf, int world, int k,
                                double* __restrict__ out) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= k) return;
  double acc = 0.0;
  for (int r = 0; r < world; ++r) acc = __dadd_rn(acc, buf[r * k + j]);
  out[j] = acc;
}

int gs_gather(const double* vals, const long long* perm, const long long* off, long long n_gid,
              double* sums, cudaStream_t st) {
  if (n_gid <= 0) return SF_OK;
  int th = 256;
  gs_gather_kernel<<<(unsigned)((n_gid + th - 1) / th), th, 0, st>>>(vals, perm, off, n_gid, sums);
  return check_launch("gs_gather");
}

int gs_scatter(const double* sums, const long long* perm, const long long* off, long long n_gid,
               double* out, cudaStream_t st) {
  if (n_gid <= 0) return SF_OK;
  int th = 256;
  gs_scatter_kernel<<<(unsigned)((n_gid + th - 1) / th), th, 0, st>>>(sums, perm, off, n_gid, out);
  return check_launch("gs_scatter");
}

int dssum_shared(double* v, const int* off, const int* perm, int n_shared, int mode,
                 const double* u, const double* recv, int n_local, cudaStream_t st) {
  if (n_shared <= 0) return SF_OK;
  if (recv == nullptr) n_local = 0x7fffffff;
  int th = 256;
  unsigned grid = (unsigned)((n_shared + th - 1) / th);
  switch (mode) {
    case 0: dssum_shared_kernel<0><<<grid, th, 0, st>>>(v, off, perm, n_shared, nullptr, recv, n_local); break;
    case 1: dssum_shared_kernel<1><<<grid, th, 0, st>>>(v, off, perm, n_shared, nullptr, recv, n_local); break;
    case 2:
      if (u == nullptr) { set_error("dssum_shared: masked mode needs u"); return SF_ERR_ARG; }
      dssum_shared_kernel<2><<<grid, th, 0, st>>>(v, off, perm, n_shared, u, recv, n_local);
      break;
    default: set_error("dssum_shared: bad mode %d", mode); return SF_ERR_ARG;
  }
  return check_launch("dssum_shared");
}

int dssum_cls(double* v, const int* perm, int n2, int n4, int n8, const int* gen_off, int n_gen,
              int mode, const double* u, const double* recv, int n_local, cudaStream_t st) {
  const long long total = (long long)n2 + n4 + n8 + n_gen;
  if (total <= 0) return SF_OK;
  if (recv == nullptr) n_local = 0x7fffffff;
  int th = 256;
  unsigned grid = (unsigned)((total + th - 1) / th);
  switch (mode) {
    case 0: dssum_cls_kernel<0><<<grid, th, 0, st>>>(v, perm, n2, n4, n8, gen_off, n_gen, nullptr, recv, n_local); break;
    case 1: dssum_cls_kernel<1><<<grid, th, 0, st>>>(v, perm, n2, n4, n8, gen_off, n_gen, nullptr, recv, n_local); break;
    case 2:
      if (u == nullptr) { set_error("dssum_cls: masked mode needs u"); return SF_ERR_ARG; }
      dssum_cls_kernel<2><<<grid, th, 0, st>>>(v, perm, n2, n4, n8, gen_off, n_gen, u, recv, n_local);
      break;
    default: set_error("dssum_cls: bad mode %d", mode); return SF_ERR_ARG;
  }
  return check_launch("dssum_cls");
}

int dssum_blk(double* v, const int* perm, int n2, int n4, int n8, const int* gen_off, const int* bstart,
              int nb, int mode, const double* u, const double* pre, const double* recv, int n_local,
              const unsigned long long* recv_seq, long long recv_bank, cudaStream_t st) {
  if (nb <= 0) return SF_OK;
  if (recv == nullptr) {
    n_local = 0x7fffffff;
    recv_seq = nullptr;
  }
  switch (mode) {
    case 0: dssum_blk_kernel<0><<<nb, 256, 0, st>>>(v, perm, n2, n4, n8, gen_off, bstart, nb, nullptr, nullptr, recv, n_local, recv_seq, recv_bank); break;
    case 1: dssum_blk_kernel<1><<<nb, 256, 0, st>>>(v, perm, n2, n4, n8, gen_off, bstart, nb, nullptr, nullptr, recv, n_local, recv_seq, recv_bank); break;
    case 2:
      if (u == nullptr) { set_error("dssum_blk: masked mode needs u"); return SF_ERR_ARG; }
      dssum_blk_kernel<2><<<nb, 256, 0, st>>>(v, perm, n2, n4, n8, gen_off, bstart, nb, u, pre, recv, n_local, recv_seq, recv_bank);
      break;
    default: set_error("dssum_blk: bad mode %d", mode); return SF_ERR_ARG;
  }
  return check_launch("dssum_blk");
}

int gather(double* out, const double* v, const int* idx, long long n, cudaStream_t st) {
  if (n <= 0) return SF_OK;
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  gather_kernel<<<(unsigned)blocks, 256, 0, st>>>(out, v, idx, n);
  return check_launch("gather");
}

int rank_sum(const double* buf, int world, int k, double* out, cudaStream_t st) {
  if (k <= 0) return SF_OK;
  rank_sum_kernel<<<(k + 127) / 128, 128, 0, st>>>(buf, world, k, out);
  return check_launch("rank_sum");
}

}  // namespace sf
