// Peer-memory (NVLink) reduction context and the device routine shared by
// peer.cu (standalone kernel) and the fused Krylov kernels (vec.cu).
#pragma once
#include <cstring>

#include "common.cuh"

#define PEER_MAX_RANKS 8
#define PEER_KMAX 4
#define PEER_TIMEOUT_NS 5000000000ull  // 5 s: a rank that never arrives is an error, not a hang

namespace sf {

struct PeerCtx {
  double* box[PEER_MAX_RANKS];  // every rank's mailbox (own + IPC-mapped peers)
  int world;
  int rank;
  // Device word counting the reductions this rank has EXECUTED (stream-ordered:
  // every kernel that uses the context runs on the rank's compute stream).  A
  // call publishes and waits for *seq + 1 and stores it back when done, so a
  // gated pass that returns early consumes no number and the bank parity stays
  // in step with the calls that really exchange -- on every rank alike, because
  // every rank gates on the same all-reduced scalars.  Kernel arguments never
  // change from call to call, so CUDA graphs can capture these kernels.
  unsigned long long* seq;
  unsigned* error;              // set to 1 on poll timeout; later calls return at once
  // slot layout: [bank][rank][PEER_KMAX values, flag word, padding] = 64 B per slot
  static constexpr int SLOT = 8;
  __host__ __device__ static constexpr int slot_off(int bank, int r) {
    return (bank * PEER_MAX_RANKS + r) * SLOT;
  }
  static int box_doubles(int) { return 2 * PEER_MAX_RANKS * SLOT; }
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Executed by ONE full warp.  Lane j (< k) holds this rank's partial j in
// `mine_j`; out[0..k) receives the rank-order sum on every rank (written by lane
// 0).  Returns false (and sets *c.error, out = NaN) on timeout.  Once the error
// flag is set every later call returns NaN at once: a dead peer makes the solver
// see NaN scalars within one call instead of waiting 5 s per reduction.
__device__ __forceinline__ bool peer_allreduce_warp(const PeerCtx& c, double mine_j, int k,
                                                    double* out) {
  const int lane = threadIdx.x & 31;
  if (*(volatile const unsigned*)c.error != 0u) {
    if (lane < k) out[lane] = __longlong_as_double(0x7ff8000000000000ll);
    return false;
  }
  const unsigned long long seq = *(volatile const unsigned long long*)c.seq + 1ull;
  const int bank = (int)(seq & 1ull);
  double v[PEER_KMAX];
#pragma unroll
  for (int j = 0; j < PEER_KMAX; ++j) v[j] = __shfl_sync(0xffffffffu, mine_j, j);
  // 1. publish into every rank's mailbox (lane r -> rank r; NVLink stores for peers)
  if (lane < c.world) {
    double* dst = c.box[lane] + PeerCtx::slot_off(bank, c.rank);
#pragma unroll
    for (int j = 0; j < PEER_KMAX; ++j)
      if (j < k) dst[j] = v[j];
    // the values were written by this lane: its st.release.sys orders them before
    // the flag for every acquirer (no separate fence.sys, ~1-2 us per reduction)
    st_release_sys(reinterpret_cast<unsigned long long*>(dst + PEER_KMAX), seq);
  }
  // 2. lane r waits (acquire) for rank r's slot in my mailbox and reads it
  const double* mine = c.box[c.rank];
  bool ok = true;
  double sv[PEER_KMAX];
#pragma unroll
  for (int j = 0; j < PEER_KMAX; ++j) sv[j] = 0.0;
  if (lane < c.world) {
    const double* slot = mine + PeerCtx::slot_off(bank, lane);
    const unsigned long long* flag = reinterpret_cast<const unsigned long long*>(slot + PEER_KMAX);
    const unsigned long long t0 = global_ns();
    while (ld_acquire_sys(flag) != seq) {
      if (global_ns() - t0 > PEER_TIMEOUT_NS) { ok = false; break; }
    }
#pragma unroll
    for (int j = 0; j < PEER_KMAX; ++j)
      if (j < k) sv[j] = ((volatile const double*)slot)[j];
  }
  ok = __all_sync(0xffffffffu, ok);
  if (!ok) {
    if (lane < k) out[lane] = __longlong_as_double(0x7ff8000000000000ll);
    if (lane == 0) atomicExch(c.error, 1u);
    return false;
  }
  if (lane == 0) *c.seq = seq;   // every lane has read its slot: the call is done
  // 3. rank-order sum (identical on every rank)
  double acc[PEER_KMAX];
#pragma unroll
  for (int j = 0; j < PEER_KMAX; ++j) acc[j] = 0.0;
  for (int r = 0; r < c.world; ++r) {
#pragma unroll
    for (int j = 0; j < PEER_KMAX; ++j) acc[j] = __dadd_rn(acc[j], __shfl_sync(0xffffffffu, sv[j], r));
  }
  if (lane == 0)
    for (int j = 0; j < k; ++j) out[j] = acc[j];
  return true;
}

}  // namespace sf
