// Cross-GPU reduction of glsc3 partials over NVLink peer memory (C2 in SURVEY
// §2.3), replacing the NCCL all-gather on the Krylov critical path.
//
// Every rank owns a mailbox in its HBM, exported to the other ranks of the node
// with CUDA IPC.  A reduction of k partials (k <= PEER_KMAX):
//   1. each rank stores its k values into slot[rank] of EVERY rank's mailbox
//      (plain st.global on peer-mapped pointers -> NVLink writes), then a
//      system-scope fence and a release store of the call's sequence number;
//   2. it polls its own mailbox until all `world` slots carry that number and
//      sums the slots in rank order -- every rank computes the identical value,
//      deterministic for a given GPU count (same order as the NCCL path).
// Mailboxes are double-banked by sequence parity: a rank can run at most one call
// ahead of any peer (it cannot finish call n+1 without the peer's n+1 data), so it
// never overwrites a bank a peer is still reading.  Polling is bounded
// (PEER_TIMEOUT_NS of %globaltimer); on timeout the kernel records an error flag
// instead of hanging the GPU.
//
// The same device routine runs inside the MGS / glsc3 kernel's last block
// (mgs2_kernel), fusing the collective into the compute kernel.
#include "common.cuh"
#include "peer.cuh"

namespace sf {

__global__ void peer_allreduce_kernel(PeerCtx c, const double* __restrict__ in, int k,
                                      double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const double mine = lane < k ? in[lane] : 0.0;
  __syncwarp();  // every lane has read `in` before lane 0 may overwrite it (in == out)
  peer_allreduce_warp(c, mine, k, out);
}

int peer_allreduce(const PeerCtx& c, const double* in, int k, double* out, cudaStream_t st) {
  if (k < 1 || k > PEER_KMAX) {
    set_error("peer_allreduce: k=%d out of range 1..%d", k, PEER_KMAX);
    return SF_ERR_ARG;
  }
  peer_allreduce_kernel<<<1, 32, 0, st>>>(c, in, k, out);
  return check_launch("peer_allreduce");
}

}  // namespace sf

extern "C" {

int sf_ipc_handle_bytes(void) { return (int)sizeof(cudaIpcMemHandle_t); }

// mailbox memory comes straight from cudaMalloc (an IPC handle names a whole
// allocation, so the exported pointer must be an allocation base)
int sf_dev_alloc_zero(long long bytes, void** out) {
  cudaError_t e = cudaMalloc(out, (size_t)bytes);
  if (e == cudaSuccess) e = cudaMemset(*out, 0, (size_t)bytes);
  if (e != cudaSuccess) {
    sf::set_error("cudaMalloc/cudaMemset: %s", cudaGetErrorString(e));
    return sf::SF_ERR_CUDA;
  }
  return sf::SF_OK;
}

int sf_dev_free(void* p) {
  cudaError_t e = cudaFree(p);
  if (e != cudaSuccess) {
    sf::set_error("cudaFree: %s", cudaGetErrorString(e));
    return sf::SF_ERR_CUDA;
  }
  return sf::SF_OK;
}

int sf_peer_mailbox_doubles(int world) { return sf::PeerCtx::box_doubles(world); }

int sf_ipc_get_handle(void* dev_ptr, unsigned char* handle_out) {
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, dev_ptr);
  if (e != cudaSuccess) {
    sf::set_error("cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
    return sf::SF_ERR_CUDA;
  }
  memcpy(handle_out, &h, sizeof(h));
  return sf::SF_OK;
}

int sf_ipc_open_handle(const unsigned char* handle, void** dev_ptr_out) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) {
    sf::set_error("cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
    return sf::SF_ERR_CUDA;
  }
  return sf::SF_OK;
}

int sf_ipc_close_handle(void* dev_ptr) {
  cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
  if (e != cudaSuccess) {
    sf::set_error("cudaIpcCloseMemHandle: %s", cudaGetErrorString(e));
    return sf::SF_ERR_CUDA;
  }
  return sf::SF_OK;
}

int sf_peer_allreduce_f64(double* const* boxes, int world, int rank, unsigned long long* seq,
                          unsigned* error, const double* in, int k, double* out, void* stream) {
  if (world < 1 || world > PEER_MAX_RANKS || rank < 0 || rank >= world) {
    sf::set_error("sf_peer_allreduce_f64: bad world/rank %d/%d", world, rank);
    return sf::SF_ERR_ARG;
  }
  sf::PeerCtx c{};
  for (int r = 0; r < world; ++r) c.box[r] = boxes[r];
  c.world = world;
  c.rank = rank;
  c.seq = seq;
  c.error = error;
  return sf::peer_allreduce(c, in, k, out, sf::as_stream(stream));
}

}  // extern "C"
