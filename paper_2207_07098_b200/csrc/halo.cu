// NVLink halo exchange for the multi-GPU dssum (collective C1).
//
// The NCCL path (gather kernel + ncclSend/ncclRecv + a stream wait) costs a
// fixed ~60 us of host and launch overhead per exchange, and the NCCL kernel
// then spins until the peer arrives (measured 320 us per exchange inside a
// 2-GPU TGV step).  Here the exchange is two small kernels on the compute
// stream and no host involvement:
//   halo_put   gathers this rank's interface copies straight into every peer's
//              IPC-mapped inbox (NVLink stores), then -- last block, after a
//              system-scope fence from every block -- publishes the call's
//              sequence number in each peer's flag word (release);
//   halo_wait  one warp polls this rank's own flag words (acquire) until every
//              peer's data for the sequence number has landed.
// The dssum kernel then reads the inbox as its receive buffer.  Inboxes are
// double-banked by sequence parity: a rank cannot start writing bank b for call
// s+2 before its peer finished reading bank b for call s, because its own
// halo_wait for s+1 waits on data the peer only sends after that read (stream
// order on the peer).  The summation order of the dssum is unchanged, so the
// result is bitwise the same as with NCCL.
//
// The call number lives in DEVICE memory (a word in the rank's own inbox header,
// advanced by the put's last block), not in a kernel argument: halo_wait and the
// dssum read it to pick the flag value and the bank.  Kernel arguments are then
// identical from call to call, so an operator application that contains an
// exchange can be captured once in a CUDA graph and replayed.
//
// Inbox layout (doubles): [flags: PEER_MAX_RANKS uint64][call number at
// HALO_SEQ][pad to 32][bank 0: n_recv][bank 1: n_recv]; rank r's data goes at its
// recv offset in each bank.
#include "peer.cuh"

namespace sf {

constexpr int HALO_HEADER = 32;  // doubles before bank 0
constexpr int HALO_SEQ = 16;     // header word holding the rank's call number

struct HaloPeers {
  int n;                                        // peers
  int rank[PEER_MAX_RANKS];                     // their ranks
  long long start[PEER_MAX_RANKS + 1];          // segments of the send list
  double* dst[PEER_MAX_RANKS];                  // peer inbox bank 0 + this rank's recv offset
  long long stride[PEER_MAX_RANKS];             // peer's bank stride (doubles)
  unsigned long long* flag[PEER_MAX_RANKS];     // peer's flag word for this rank
};

__global__ void halo_put_kernel(const double* __restrict__ v, const int* __restrict__ send_idx,
                                HaloPeers hp, unsigned long long* __restrict__ seqp,
                                unsigned* __restrict__ counter, const unsigned* __restrict__ error) {
  // after a peer failure every exchange is a no-op (the host raises at its next check)
  if (*(volatile const unsigned*)error != 0u) return;
  // every block reads the call number before the last block advances it
  const unsigned long long seq = *(volatile const unsigned long long*)seqp + 1ull;
  const int bank = (int)(seq & 1ull);
  const long long total = hp.start[hp.n];
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    int q = 0;
    while (q + 1 < hp.n && i >= hp.start[q + 1]) ++q;
    hp.dst[q][bank * hp.stride[q] + (i - hp.start[q])] = __ldg(v + __ldg(send_idx + i));
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    if (atomicAdd(counter, 1u) == gridDim.x - 1u) {
      *counter = 0u;  // rearm for the next call on this stream
      *seqp = seq;
      __threadfence_system();
      for (int q = 0; q < hp.n; ++q) st_release_sys(hp.flag[q], seq);
    }
  }
}

__global__ void halo_wait_kernel(const unsigned long long* __restrict__ flags, HaloPeers hp,
                                 unsigned* __restrict__ error) {
  const int lane = threadIdx.x;
  if (*(volatile const unsigned*)error != 0u) return;
  const unsigned long long seq = *(volatile const unsigned long long*)(flags + HALO_SEQ);
  bool ok = true;
  if (lane < hp.n) {
    const unsigned long long* f = flags + hp.rank[lane];
    const unsigned long long t0 = global_ns();
    while (ld_acquire_sys(f) < seq) {
      if (global_ns() - t0 > PEER_TIMEOUT_NS) { ok = false; break; }
    }
  }
  if (!__all_sync(0xffffffffu, ok) && lane == 0) atomicExch(error, 1u);
}

}  // namespace sf

extern "C" {

int sf_halo_inbox_doubles(long long n_recv) { return (int)(sf::HALO_HEADER + 2 * n_recv); }

int sf_halo_header_doubles(void) { return sf::HALO_HEADER; }

// Push this rank's interface copies to every peer and publish the next call
// number (own_inbox[HALO_SEQ] + 1, advanced in device memory).
//   send_idx: concatenated local indices, peer q's segment = [seg[q], seg[q+1])
//   peer_rank / peer_dst / peer_stride / peer_flag: per peer (n_peers <= 8)
int sf_halo_put_f64(const double* v, const int* send_idx, int n_peers, const int* peer_rank,
                    const long long* seg, double* const* peer_dst, const long long* peer_stride,
                    unsigned long long* const* peer_flag, unsigned long long* own_inbox, unsigned* counter,
                    const unsigned* error, void* stream) {
  using namespace sf;
  if (n_peers <= 0) return SF_OK;
  if (n_peers > PEER_MAX_RANKS || !v || !send_idx || !counter || !own_inbox || !error) {
    set_error("sf_halo_put_f64: bad arguments (n_peers=%d)", n_peers);
    return SF_ERR_ARG;
  }
  HaloPeers hp;
  std::memset(&hp, 0, sizeof(hp));
  hp.n = n_peers;
  for (int q = 0; q < n_peers; ++q) {
    hp.rank[q] = peer_rank[q];
    hp.start[q] = seg[q];
    hp.dst[q] = peer_dst[q];
    hp.stride[q] = peer_stride[q];
    hp.flag[q] = peer_flag[q];
  }
  hp.start[n_peers] = seg[n_peers];
  const long long total = seg[n_peers];
  long long blocks = (total + 255) / 256;
  if (blocks < 1) blocks = 1;
  if (blocks > 148 * 4) blocks = 148 * 4;
  halo_put_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(v, send_idx, hp, own_inbox + HALO_SEQ,
                                                                  counter, error);
  return check_launch("halo_put");
}

// Wait (on the stream) until every peer published the current call number
// (own_flags[HALO_SEQ], advanced by this rank's put) into this rank's flags.
int sf_halo_wait(const unsigned long long* own_flags, int n_peers, const int* peer_rank,
                 unsigned* error, void* stream) {
  using namespace sf;
  if (n_peers <= 0) return SF_OK;
  if (n_peers > PEER_MAX_RANKS || !own_flags || !error) {
    set_error("sf_halo_wait: bad arguments (n_peers=%d)", n_peers);
    return SF_ERR_ARG;
  }
  HaloPeers hp;
  std::memset(&hp, 0, sizeof(hp));
  hp.n = n_peers;
  for (int q = 0; q < n_peers; ++q) hp.rank[q] = peer_rank[q];
  halo_wait_kernel<<<1, 32, 0, as_stream(stream)>>>(own_flags, hp, error);
  return check_launch("halo_wait");
}

}  // extern "C"
