// C ABI of libsemflow_b200.so -- the drop-in boundary (see include/semflow_b200.h
// for the reference interface each entry point replaces).  Plain pointers, sizes
// and a cudaStream_t passed as void*; every function returns an int status
// (0 = ok) and leaves a message for sf_last_error() on failure.
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "common.cuh"
#include "reduce.cuh"
#include "peer.cuh"

#include "../../include/semflow_b200.h"

namespace sf {

static thread_local char g_err[512] = {0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return SF_ERR_CUDA;
  }
  return SF_OK;
}

// implemented in ax.cu, gs.cu, vec.cu, ops.cu, geom.cu
int ax_helm(const double*, int, const double*, const double*, const double*, double*, long long,
            double, double, const uint32_t*, const uint32_t*, int, cudaStream_t, const double*);
int grad_ref(const double*, int, const double*, double*, double*, double*, long long, int,
             cudaStream_t);
int apply_axis(int, const double*, int, int, const double*, double*, long long, int, cudaStream_t);
int apply_axis3(int, const double*, int, int, int, int, const double*, double*, long long, int,
                cudaStream_t);
int gs_gather(const double*, const long long*, const long long*, long long, double*, cudaStream_t);
int gs_scatter(const double*, const long long*, const long long*, long long, double*, cudaStream_t);
int dssum_shared(double*, const int*, const int*, int, int, const double*, const double*, int,
                 cudaStream_t);
int gather(double*, const double*, const int*, long long, cudaStream_t);
int dssum_cls(double*, const int*, int, int, int, const int*, int, int, const double*, const double*,
              int, cudaStream_t);
int rank_sum(const double*, int, int, double*, cudaStream_t);
int ax_helm8_range(const double*, const double*, const double*, const double*, const double*, double*, long long,
                   long long, long long, double, double, const uint32_t*, const uint32_t*, int, cudaStream_t);
int dssum_blk(double*, const int*, int, int, int, const int*, const int*, int, int, const double*,
              const double*, const double*, int, const unsigned long long*, long long, cudaStream_t);
int dot_multi(int, const double* const*, const double* const*, const uint8_t*, long long, RedWork,
              double*, cudaStream_t);
int cg_init(const double*, const double*, double*, const uint8_t*, long long, RedWork, double*,
            cudaStream_t);
int cg_update(double*, double*, const double*, const double*, const double*, const uint8_t*,
              const double*, const double*, long long, RedWork, double*, cudaStream_t);
int cg_direction(double*, const double*, const double*, const double*, const double*, long long,
                 cudaStream_t);
int mgs_step(double*, const double*, const double*, const double*, double*, const double*,
             const uint8_t*, int, long long, RedWork, double*, cudaStream_t, const PeerCtx*,
             const double*);
int gmres_gate(double*, int, int, int, int, cudaStream_t);
int dot1_vec(const double*, const double*, const uint8_t*, long long, RedWork, double*, cudaStream_t,
             const PeerCtx*);
int peer_allreduce(const PeerCtx&, const double*, int, double*, cudaStream_t);
int lincomb(double*, const double*, const double* const*, const double*, const double*, int,
            long long, cudaStream_t);
int residual(double*, const double*, const double*, const uint8_t*, long long, RedWork, double*,
             cudaStream_t);
int scale_div(double*, const double*, double*, const double*, const double*, long long,
              cudaStream_t);
int deriv(int, const double*, int, const double*, const double*, const double*, double*, long long,
          double, int, cudaStream_t);
int cdtp(const double*, int, const double*, const double*, const double*, double*, long long, int,
         cudaStream_t);
int cfl_max(const double*, const double*, const double*, int, long long, unsigned long long*, int,
            cudaStream_t);
int bdf_ext(double*, double*, const double* const*, const double* const*, const double* const*,
            const double*, const double*, int, long long, cudaStream_t);
int trilinear_coords(const double*, const double*, int, long long, double*, cudaStream_t);
int metrics(const double*, const double*, int, const double*, long long, double*, double*, double*,
            double*, cudaStream_t);
extern int g_ax_kernel;

}  // namespace sf

using namespace sf;

extern "C" {

const char* sf_version(void) { return "semflow_b200 0.1.0 (sm_100a, fp64)"; }
const char* sf_last_error(void) { return g_err; }

int sf_red_workspace_doubles(void) { return K_MAX * RED_BLOCKS; }

// n = 8 Ax kernel: 1 = bulk-copy-fed persistent kernel (default), 0 = register-
// prefetch kernel.  Process-wide; for A/B measurements (tools/ax_variants.py).
int sf_set_ax_kernel(int which) {
  if (which != 0 && which != 1) {
    set_error("sf_set_ax_kernel: expected 0 or 1, got %d", which);
    return SF_ERR_ARG;
  }
  g_ax_kernel = which;
  return SF_OK;
}

int sf_apply_axis_f64(int axis, const double* a, int m, int n, const double* u, double* out,
                      long long E, int exact, void* stream) {
  return apply_axis(axis, a, m, n, u, out, E, exact, as_stream(stream));
}

int sf_apply_axis3_f64(int axis, const double* a, int m, int d0, int d1, int d2, const double* u,
                       double* out, long long E, int exact, void* stream) {
  return apply_axis3(axis, a, m, d0, d1, d2, u, out, E, exact, as_stream(stream));
}

int sf_grad_ref_f64(const double* d_host, int n, const double* u, double* ur, double* us,
                    double* ut, long long E, int exact, void* stream) {
  return grad_ref(d_host, n, u, ur, us, ut, E, exact, as_stream(stream));
}

int sf_ax_helm_f64(const double* d_host, int n, const double* g, const double* b, const double* u,
                   double* w, long long E, double lam_visc, double lam_mass, int exact,
                   void* stream) {
  return ax_helm(d_host, n, g, b, u, w, E, lam_visc, lam_mass, nullptr, nullptr, exact,
                 as_stream(stream), nullptr);
}

int sf_gs_gather_f64(const double* vals, const long long* perm, const long long* offsets,
                     long long n_gid, double* sums, void* stream) {
  return gs_gather(vals, perm, offsets, n_gid, sums, as_stream(stream));
}

int sf_gs_scatter_f64(const double* sums, const long long* perm, const long long* offsets,
                      long long n_gid, double* out, void* stream) {
  return gs_scatter(sums, perm, offsets, n_gid, out, as_stream(stream));
}

int sf_ax_masked_f64(const double* d_host, int n, const double* g, const double* b,
                     const double* u, double* w, long long E, double lam_visc, double lam_mass,
                     const uint32_t* inmask, const uint32_t* outsel, int exact, void* stream) {
  if (!inmask || !outsel) {
    set_error("sf_ax_masked_f64: inmask and outsel are required");
    return SF_ERR_ARG;
  }
  return ax_helm(d_host, n, g, b, u, w, E, lam_visc, lam_mass, inmask, outsel, exact,
                 as_stream(stream), nullptr);
}

int sf_ax_pre_f64(const double* d_host, int n, const double* g, const double* b, const double* u,
                  const double* pre, double* w, long long E, double lam_visc, double lam_mass,
                  const uint32_t* inmask, const uint32_t* outsel, int exact, void* stream) {
  if (!pre || (inmask == nullptr) != (outsel == nullptr)) {
    set_error("sf_ax_pre_f64: pre is required; inmask/outsel both or neither");
    return SF_ERR_ARG;
  }
  return ax_helm(d_host, n, g, b, u, w, E, lam_visc, lam_mass, inmask, outsel, exact,
                 as_stream(stream), pre);
}

int sf_ax_range_f64(const double* d_host, int n, const double* g, const double* b, const double* u,
                    const double* pre, double* w, long long E, long long e0, long long e1, double lam_visc,
                    double lam_mass, const uint32_t* inmask, const uint32_t* outsel, int exact, void* stream) {
  if (n != 8) {
    set_error("sf_ax_range_f64: element ranges are implemented for n = 8 (got %d)", n);
    return SF_ERR_UNSUPPORTED;
  }
  return ax_helm8_range(d_host, g, b, u, pre, w, E, e0, e1, lam_visc, lam_mass, inmask, outsel, exact,
                        as_stream(stream));
}

int sf_dssum_f64(double* v, const int* offsets, const int* perm, int n_shared, int mode,
                 const double* u, const double* recv, int n_local, void* stream) {
  return dssum_shared(v, offsets, perm, n_shared, mode, u, recv, n_local, as_stream(stream));
}

int sf_dssum_cls_f64(double* v, const int* perm, int n2, int n4, int n8, const int* gen_offsets,
                     int n_gen, int mode, const double* u, const double* recv, int n_local,
                     void* stream) {
  return dssum_cls(v, perm, n2, n4, n8, gen_offsets, n_gen, mode, u, recv, n_local, as_stream(stream));
}

int sf_dssum_blk_f64(double* v, const int* perm, int n2, int n4, int n8, const int* gen_offsets,
                     const int* block_start, int n_blocks, int mode, const double* u, const double* pre,
                     const double* recv, int n_local, const unsigned long long* recv_seq,
                     long long recv_bank, void* stream) {
  return dssum_blk(v, perm, n2, n4, n8, gen_offsets, block_start, n_blocks, mode, u, pre, recv, n_local,
                   recv_seq, recv_bank, as_stream(stream));
}

int sf_gather_f64(double* out, const double* v, const int* idx, long long n, void* stream) {
  return gather(out, v, idx, n, as_stream(stream));
}

int sf_rank_sum_f64(const double* buf, int world, int k, double* out, void* stream) {
  return rank_sum(buf, world, k, out, as_stream(stream));
}

int sf_glsc3_f64(int K, const double* const* a, const double* const* b, const uint8_t* mult,
                 long long P, double* partials, unsigned* counter, double* out, void* stream) {
  return dot_multi(K, a, b, mult, P, RedWork{partials, counter}, out, as_stream(stream));
}

int sf_cg_init_f64(const double* r, const double* invdiag, double* p, const uint8_t* mult,
                   long long P, double* partials, unsigned* counter, double* out, void* stream) {
  return cg_init(r, invdiag, p, mult, P, RedWork{partials, counter}, out, as_stream(stream));
}

int sf_cg_update_f64(double* x, double* r, const double* p, const double* ap,
                     const double* invdiag, const uint8_t* mult, const double* rz,
                     const double* pap, long long P, double* partials, unsigned* counter,
                     double* out, void* stream) {
  return cg_update(x, r, p, ap, invdiag, mult, rz, pap, P, RedWork{partials, counter}, out,
                   as_stream(stream));
}

int sf_cg_direction_f64(double* p, const double* r, const double* invdiag, const double* rz_new,
                        const double* rz, long long P, void* stream) {
  return cg_direction(p, r, invdiag, rz_new, rz, P, as_stream(stream));
}

int sf_mgs_step_f64(double* w, const double* vprev, const double* hprev, const double* vnext,
                    double* w2, const double* v2prev, const uint8_t* mult, int want_norm,
                    long long P, double* partials, unsigned* counter, double* out,
                    const double* gate, void* stream) {
  return mgs_step(w, vprev, hprev, vnext, w2, v2prev, mult, want_norm, P,
                  RedWork{partials, counter}, out, as_stream(stream), nullptr, gate);
}

int sf_gmres_gate_f64(double* blk, int j, int o2, int o3, int phase, void* stream) {
  return gmres_gate(blk, j, o2, o3, phase, as_stream(stream));
}

static int make_peer(PeerCtx& c, double* const* boxes, int world, int rank, unsigned long long* seq,
                     unsigned* error) {
  if (world < 1 || world > PEER_MAX_RANKS || rank < 0 || rank >= world) {
    set_error("peer context: bad world/rank %d/%d", world, rank);
    return SF_ERR_ARG;
  }
  c = PeerCtx{};
  for (int r = 0; r < world; ++r) c.box[r] = boxes[r];
  c.world = world;
  c.rank = rank;
  c.seq = seq;
  c.error = error;
  return SF_OK;
}

int sf_mgs_step_peer_f64(double* w, const double* vprev, const double* hprev, const double* vnext,
                         double* w2, const double* v2prev, const uint8_t* mult, int want_norm,
                         long long P, double* partials, unsigned* counter, double* out,
                         double* const* boxes, int world, int rank, unsigned long long* seq,
                         unsigned* error, const double* gate, void* stream) {
  PeerCtx c;
  int st = make_peer(c, boxes, world, rank, seq, error);
  if (st != SF_OK) return st;
  return mgs_step(w, vprev, hprev, vnext, w2, v2prev, mult, want_norm, P,
                  RedWork{partials, counter}, out, as_stream(stream), &c, gate);
}

int sf_glsc3_peer_f64(const double* a, const double* b, const uint8_t* mult, long long P,
                      double* partials, unsigned* counter, double* out, double* const* boxes,
                      int world, int rank, unsigned long long* seq, unsigned* error, void* stream) {
  PeerCtx c;
  int st = make_peer(c, boxes, world, rank, seq, error);
  if (st != SF_OK) return st;
  const int r = mult ? dot1_vec(a, b, mult, P, RedWork{partials, counter}, out, as_stream(stream), &c)
                     : -1;
  if (r >= 0) return r;
  const double* pa[1] = {a};
  const double* pb[1] = {b};
  st = dot_multi(1, pa, pb, mult, P, RedWork{partials, counter}, out, as_stream(stream));
  if (st != SF_OK) return st;
  return peer_allreduce(c, out, 1, out, as_stream(stream));
}

int sf_lincomb_f64(double* x, const double* x0, const double* const* v, const double* coef,
                   const double* invdiag, int nv, long long P, void* stream) {
  return lincomb(x, x0, v, coef, invdiag, nv, P, as_stream(stream));
}

int sf_residual_f64(double* r, const double* b, const double* ax, const uint8_t* mult, long long P,
                    double* partials, unsigned* counter, double* out, void* stream) {
  return residual(r, b, ax, mult, P, RedWork{partials, counter}, out, as_stream(stream));
}

int sf_scale_div_f64(double* y, const double* x, double* y2, const double* x2, const double* s,
                     long long P, void* stream) {
  return scale_div(y, x, y2, x2, s, P, as_stream(stream));
}

int sf_deriv_f64(int op, const double* d_host, int n, const double* in, const double* c,
                 const double* rx, double* out, long long E, double sign, int exact,
                 void* stream) {
  return deriv(op, d_host, n, in, c, rx, out, E, sign, exact, as_stream(stream));
}

int sf_cdtp_f64(const double* d_host, int n, const double* w, const double* rx, const double* bm,
                double* out, long long E, int exact, void* stream) {
  return cdtp(d_host, n, w, rx, bm, out, E, exact, as_stream(stream));
}

int sf_cfl_f64(const double* v, const double* rx, const double* dxi_host, int n, long long E,
               unsigned long long* out_bits, int exact, void* stream) {
  return cfl_max(v, rx, dxi_host, n, E, out_bits, exact, as_stream(stream));
}

int sf_bdf_ext_f64(double* vhat, double* omega, const double* const* vel, const double* const* nl,
                   const double* const* crl, const double* a_dt, const double* beta, int order,
                   long long P3, void* stream) {
  return bdf_ext(vhat, omega, vel, nl, crl, a_dt, beta, order, P3, as_stream(stream));
}

int sf_trilinear_coords_f64(const double* corners, const double* wc, int n, long long E,
                            double* coords, void* stream) {
  return trilinear_coords(corners, wc, n, E, coords, as_stream(stream));
}

int sf_metrics_f64(const double* d_host, const double* w_host, int n, const double* coords,
                   long long E, double* rx, double* jac, double* bm, double* geom, void* stream) {
  return metrics(d_host, w_host, n, coords, E, rx, jac, bm, geom, as_stream(stream));
}

}  // extern "C"
