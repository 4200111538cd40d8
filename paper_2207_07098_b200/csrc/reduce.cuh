// Deterministic fused map-reduce skeleton used by every glsc3-style kernel.
//
// A kernel instantiates `map_reduce<Op>`: each of the RED_BLOCKS x RED_THREADS
// threads walks a fixed grid-stride slice of the P points calling Op::point(p,
// acc) (which may also write vectors -- the fused CG / GMRES updates), then K
// sums are folded by a fixed warp-shuffle tree, a fixed cross-warp order, and
// finally by the last block to arrive, which combines the per-block partials in
// block order and writes out[0..K-1].  The summation order is a pure function of
// P, so results are reproducible run to run (the reference contract,
// kernels/__init__.py:19-22) -- but they are not the OpenBLAS `np.dot` order
// (space.py:76), which no parallel reduction can reproduce.
#pragma once
#include <type_traits>

#include "common.cuh"
#include "peer.cuh"

namespace sf {

struct RedWork {
  double* partials;    // [K_MAX * RED_BLOCKS]
  unsigned* counter;   // one zero-initialised counter, reset by the last block
};
constexpr int K_MAX = 4;

// 1/m lookup for the multiplicity weights: im_tab[m] = 1.0 / m (IEEE division,
// bit-identical to `invmult = 1.0 / mult`, space.py:313).
__device__ __forceinline__ void init_im_tab(double* tab) {
  for (int m = threadIdx.x; m < 256; m += blockDim.x) tab[m] = m ? 1.0 / (double)m : 0.0;
}

template <int K>
__device__ __forceinline__ void finish_reduce(double (&acc)[K], RedWork wk, double* __restrict__ out,
                                              const PeerCtx* peer = nullptr) {
  __shared__ double red[RED_THREADS / 32][K];
  __shared__ double fin[K];
  __shared__ bool am_last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double v = acc[k];
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) v += __shfl_down_sync(0xffffffffu, v, s);
    if (lane == 0) red[warp][k] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double v = 0.0;
      for (int w = 0; w < RED_THREADS / 32; ++w) v += red[w][k];
      wk.partials[k * RED_BLOCKS + blockIdx.x] = v;
    }
    __threadfence();
    unsigned prev = atomicAdd(wk.counter, 1u);
    am_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  const int nb = gridDim.x;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double v = 0.0;
    for (int b = threadIdx.x; b < nb; b += RED_THREADS)
      v += ((volatile double*)wk.partials)[k * RED_BLOCKS + b];
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) v += __shfl_down_sync(0xffffffffu, v, s);
    if (lane == 0) red[warp][k] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double v = 0.0;
      for (int w = 0; w < RED_THREADS / 32; ++w) v += red[w][k];
      fin[k] = v;
    }
    *wk.counter = 0u;
  }
  __syncthreads();
  if (warp != 0) return;
  if (peer != nullptr && peer->world > 1) {
    // fused cross-GPU reduction over NVLink peer memory (peer.cuh): the rank's
    // partials leave the kernel already summed over all ranks
    peer_allreduce_warp(*peer, lane < K ? fin[lane] : 0.0, K, out);
  } else if (lane < K) {
    out[lane] = fin[lane];
  }
}

// Each thread handles UNR independent grid-stride points per trip: all loads of
// the UNR points are issued before any result is stored (Op::load / Op::finish),
// so a thread keeps UNR x (bytes per point) in flight -- the single-point loop
// could not hoist a load of point p+stride above the store to point p (possible
// aliasing) and stalled at ~5 TB/s.
constexpr int RED_UNR = 4;

// per-Op unroll depth: Op::UNR when declared (read-only ops carry few registers
// per point and want more bytes in flight), RED_UNR otherwise
template <class Op, class = void>
struct UnrOf { static constexpr int value = RED_UNR; };
template <class Op>
struct UnrOf<Op, std::void_t<decltype(Op::UNR)>> { static constexpr int value = Op::UNR; };

template <class Op>
__global__ void __launch_bounds__(RED_THREADS) map_reduce_kernel(Op op, long long P, RedWork wk,
                                                                 double* __restrict__ out) {
  constexpr int K = Op::K;
  constexpr int U = UnrOf<Op>::value;
  __shared__ double im_tab[256];
  init_im_tab(im_tab);
  __syncthreads();
  Op o = op;
  o.prologue();
  double acc[K > 0 ? K : 1];
#pragma unroll
  for (int k = 0; k < (K > 0 ? K : 1); ++k) acc[k] = 0.0;
  // a warp walks contiguous spans of 32*RED_UNR points (each load instruction is a
  // fully coalesced 256 B run and the warp's RED_UNR runs are adjacent: good DRAM
  // locality); warps stride over the array
  const int lane = threadIdx.x & 31;
  const long long gwarp = ((long long)blockIdx.x * RED_THREADS + threadIdx.x) >> 5;
  const long long span = 32LL * U;
  const long long wstride = (long long)gridDim.x * (RED_THREADS / 32) * span;
  for (long long base = gwarp * span + lane; base < P; base += wstride) {
    typename Op::In in[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const long long p = base + 32 * q;
      if (p < P) in[q] = o.load(p, im_tab);
    }
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const long long p = base + 32 * q;
      if (p < P) o.finish(p, in[q], acc);
    }
  }
  if constexpr (K > 0) finish_reduce<K>(acc, wk, out);
}

template <class Op>
inline int launch_map_reduce(const Op& op, long long P, RedWork wk, double* out, cudaStream_t st,
                             const char* name) {
  unsigned blocks = RED_BLOCKS;
  long long need = (P + RED_THREADS - 1) / RED_THREADS;
  if (need < (long long)blocks) blocks = (unsigned)(need > 0 ? need : 1);
  map_reduce_kernel<Op><<<blocks, RED_THREADS, 0, st>>>(op, P, wk, out);
  return check_launch(name);
}

}  // namespace sf
