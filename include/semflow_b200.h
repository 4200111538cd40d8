/*
 * semflow_b200.h -- C ABI of libsemflow_b200.so, the B200 (sm_100a) drop-in for
 * the matrix-free spectral-element hot path of the `semflow` reference
 * (arXiv 2207.07098 restated in Python, /root/reference/pkg/src/semflow).
 *
 * Conventions
 *   - All arrays are DEVICE pointers unless the parameter name ends in `_host`.
 *   - Fields are float64, C order: scalar (E, n, n, n) with axes (element, r, s, t),
 *     vector (3, E, n, n, n); geometric factors g (6, E, n, n, n) packed
 *     rr, rs, rt, ss, st, tt; rx (3, 3, E, n, n, n) with rx[s][l] = dr_s/dx_l.
 *     (space.py:1-6, 102-122)
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Every entry point returns 0 on success and a nonzero SF_ERR_* code on
 *     failure; sf_last_error() returns the (thread-local) message.
 *   - `exact` != 0 selects non-contracted arithmetic (no FMA) in the same loop
 *     order as the reference numba lane, giving bit-identical results for the
 *     element kernels; exact == 0 is the production (DFMA) path.
 *   - Reductions use a caller-owned workspace: `partials` holds
 *     sf_red_workspace_doubles() doubles and `counter` one zero-initialised
 *     unsigned (it is reset by the kernel).  Reductions are deterministic: the
 *     summation order depends only on the problem size.
 *   - n (points per direction, order + 1) must be in 2..10.
 *
 * The python binding that loads this library is
 * paper_2207_07098_b200/_lib.py; INTEGRATION.md shows how the reference's own
 * kernel lane (semflow/kernels/__init__.py) binds it.
 */
#ifndef SEMFLOW_B200_H
#define SEMFLOW_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SF_OK 0
#define SF_ERR_ARG 1
#define SF_ERR_CUDA 2
#define SF_ERR_UNSUPPORTED 3

const char* sf_version(void);
const char* sf_last_error(void);
/* doubles needed for the `partials` reduction workspace */
int sf_red_workspace_doubles(void);

/* ---------------------------------------------------------------------------
 * Kernel lane -- the reference's plugin API, semflow/kernels/__init__.py:47-53
 * ------------------------------------------------------------------------- */

/* apply_r / apply_s / apply_t (axis 0 / 1 / 2): out = a (m x n) contracted along
 * one reference axis of u (E, n, n, n); out has that axis of extent m.
 * Replaces kernels/_numba.py:15-60 (apply_r :15, apply_s :31, apply_t :47). */
int sf_apply_axis_f64(int axis, const double* a, int m, int n, const double* u, double* out,
                      long long E, int exact, void* stream);
/* The same contraction on non-cubic elements u (E, d0, d1, d2): axis `axis`
 * (extent d_axis) is replaced by m -- the reference kernels accept any element
 * shape, which the dealiasing chain needs (operators.py:141-147). */
int sf_apply_axis3_f64(int axis, const double* a, int m, int d0, int d1, int d2, const double* u,
                       double* out, long long E, int exact, void* stream);

/* grad_ref: (ur, us, ut) = reference derivatives of u.  d_host is the n x n GLL
 * differentiation matrix in host memory.  Replaces kernels/_numba.py:63-83. */
int sf_grad_ref_f64(const double* d_host, int n, const double* u, double* ur, double* us,
                    double* ut, long long E, int exact, void* stream);

/* ax_helmholtz_local: w = lam_visc * D^T G D u + lam_mass * B u per element
 * (lam_mass == 0 skips the mass term).  Replaces kernels/_numba.py:86-131. */
int sf_ax_helm_f64(const double* d_host, int n, const double* g, const double* b, const double* u,
                   double* w, long long E, double lam_visc, double lam_mass, int exact,
                   void* stream);

/* gs_gather: sums[g] = sum of vals[perm[o]] for o in [offsets[g], offsets[g+1]),
 * sequential in perm order.  Replaces kernels/_numba.py:134-143. */
int sf_gs_gather_f64(const double* vals, const long long* perm, const long long* offsets,
                     long long n_gid, double* sums, void* stream);

/* gs_scatter: out[perm[o]] = sums[g] (in place).  Replaces kernels/_numba.py:146-153. */
int sf_gs_scatter_f64(const double* sums, const long long* perm, const long long* offsets,
                      long long n_gid, double* out, void* stream);

/* ---------------------------------------------------------------------------
 * Device operator API -- the performance boundary (device-resident fields)
 * ------------------------------------------------------------------------- */

/* Masked element operator, first half of make_global_op's closure
 * (operators.py:51-54): um = inmask ? u : 0; w = lam_visc D^T G D um + lam_mass B um;
 * the value stored is w where `outsel` is set and u where it is clear.
 * inmask/outsel are packed per-element bitmasks: ceil(n^3/32) uint32 words per
 * element, bit p of element e = local point p.  Callers set outsel = mask OR
 * shared, then finish with sf_dssum_f64(mode=2). */
int sf_ax_masked_f64(const double* d_host, int n, const double* g, const double* b,
                     const double* u, double* w, long long E, double lam_visc, double lam_mass,
                     const uint32_t* inmask, const uint32_t* outsel, int exact, void* stream);

/* Selects the n = 8 Ax_helm kernel behind sf_ax_helm_f64 / sf_ax_masked_f64 /
 * sf_ax_pre_f64 / sf_ax_range_f64: 1 (default) = persistent kernel fed by bulk
 * asynchronous copies into a shared-memory ring, 0 = register-prefetch kernel.
 * Both are bit-identical; process-wide switch for A/B measurements. */
int sf_set_ax_kernel(int which);

/* The element operator (plain / masked / pre-scaled) on elements [e0, e1) of an
 * E-element field (n = 8; e0 even, e1 even or E; geometry strides use E): the
 * multi-GPU operator computes the halo elements first, posts the NVLink halo
 * exchange, then the interior.  pre, inmask/outsel optional. */
int sf_ax_range_f64(const double* d_host, int n, const double* g, const double* b, const double* u,
                    const double* pre, double* w, long long E, long long e0, long long e1, double lam_visc,
                    double lam_mass, const uint32_t* inmask, const uint32_t* outsel, int exact, void* stream);

/* In-place dssum (QQ^T) over the shared part of the gather-scatter map:
 * offsets (n_shared+1) / perm (int32 local indices) of the gids with
 * multiplicity > 1, grouped by gid with ascending local index (space.py:303-305).
 * mode 0: add (GatherScatter.add, space.py:38-49)
 * mode 1: avg (GatherScatter.avg, space.py:51-60: sum * (1.0/count))
 * mode 2: masked operator finalisation (operators.py:53-54): copies whose perm
 *         entry is negative (bit 31 set) receive u[idx] instead of the sum.
 * Each shared gid is summed by one thread in reference order: bit-identical to
 * gs_gather + gs_scatter, atomics-free.
 * Multi-GPU: perm entries >= n_local name copies owned by other ranks, whose raw
 * values are read from recv[entry - n_local] and never written (recv == NULL:
 * single rank, n_local ignored).  Summation stays in global copy order, so the
 * result is bitwise independent of the rank count. */
int sf_dssum_f64(double* v, const int* offsets, const int* perm, int n_shared, int mode,
                 const double* u, const double* recv, int n_local, void* stream);

/* The same dssum with the shared gids stored by multiplicity class (the layout
 * space.GatherScatter uses): perm holds n2 index pairs (the segment padded to a
 * multiple of 4 ints, so perm must be 16-byte aligned), then n4 quadruples, then
 * n8 octets (fixed stride, no offsets), then the CSR part of n_gen gids of any
 * other multiplicity (gen_offsets, n_gen+1 entries relative to that part).  Same
 * modes, flags, halo convention and per-gid order as sf_dssum_f64. */
int sf_dssum_cls_f64(double* v, const int* perm, int n2, int n4, int n8, const int* gen_offsets,
                     int n_gen, int mode, const double* u, const double* recv, int n_local,
                     void* stream);

/* The class-layout dssum scheduled by element range (the production kernel):
 * thread block b owns the gids whose lowest local copy lies in its element range,
 * all classes, so the 32-byte sectors shared by face, edge and vertex copies of
 * those elements are fetched from HBM once.  block_start: 4 x (n_blocks + 1)
 * item offsets, one row per class (pairs, quads, octets, generic), each relative
 * to its class.  Same modes, flags, halo convention and per-gid order as
 * sf_dssum_f64 (bit-identical results).  pre (optional, mode 2): masked copies
 * receive pre[p] * u[p] -- the input of an operator applied by sf_ax_pre_f64.
 * recv_seq (optional, device): the receive buffer is double-banked (NVLink halo
 * inbox, sf_halo_put_f64) and the copies are read from
 * recv + (*recv_seq & 1) * recv_bank -- the bank of the current exchange. */
int sf_dssum_blk_f64(double* v, const int* perm, int n2, int n4, int n8, const int* gen_offsets,
                     const int* block_start, int n_blocks, int mode, const double* u, const double* pre,
                     const double* recv, int n_local, const unsigned long long* recv_seq,
                     long long recv_bank, void* stream);

/* Ax_helm of the Jacobi-scaled vector pre .* u without materialising it
 * (`z = precond(v); w = apply_a(z)`, krylov.py:106-107 with BlockJacobi,
 * precond.py:58-59): each u value is multiplied by pre as it is loaded, the same
 * IEEE product `inv_diag * v` rounds to.  inmask/outsel optional (both or
 * neither, as in sf_ax_masked_f64).  n = 8 only (SF_ERR_UNSUPPORTED otherwise). */
int sf_ax_pre_f64(const double* d_host, int n, const double* g, const double* b, const double* u,
                  const double* pre, double* w, long long E, double lam_visc, double lam_mass,
                  const uint32_t* inmask, const uint32_t* outsel, int exact, void* stream);

/* out[i] = v[idx[i]] -- packs a rank's interface values for the halo exchange. */
int sf_gather_f64(double* out, const double* v, const int* idx, long long n, void* stream);

/* out[j] = buf[0*k+j] + buf[1*k+j] + ... (rank order): finishes an all-gather
 * based, deterministic allreduce of k glsc3 partials over `world` ranks. */
int sf_rank_sum_f64(const double* buf, int world, int k, double* out, void* stream);

/* glsc3: out[k] = sum_p (a_k[p] / mult[p]) * b_k[p] for K = 1..4 pairs
 * (GatherScatter.dot, space.py:72-76).  a, b are HOST arrays of K device
 * pointers; mult is the uint8 multiplicity per local point (NULL = unweighted,
 * FunctionSpace.integral, space.py:159-161).  out is a device array. */
int sf_glsc3_f64(int K, const double* const* a, const double* const* b, const uint8_t* mult,
                 long long P, double* partials, unsigned* counter, double* out, void* stream);

/* PCG building blocks (krylov.py:36-75 with BlockJacobi, precond.py:43-59);
 * invdiag == NULL means no preconditioner.  Scalars are device pointers.
 *   cg_init:      p = M r;                           out[0] = <r, p>
 *   cg_update:    alpha = *rz / *pap; x += alpha p; r -= alpha ap;
 *                 out[0] = <r, r>, out[1] = <r, M r>
 *   cg_direction: p = M r + (*rz_new / *rz) p                                   */
int sf_cg_init_f64(const double* r, const double* invdiag, double* p, const uint8_t* mult,
                   long long P, double* partials, unsigned* counter, double* out, void* stream);
int sf_cg_update_f64(double* x, double* r, const double* p, const double* ap,
                     const double* invdiag, const uint8_t* mult, const double* rz,
                     const double* pap, long long P, double* partials, unsigned* counter,
                     double* out, void* stream);
int sf_cg_direction_f64(double* p, const double* r, const double* invdiag, const double* rz_new,
                        const double* rz, long long P, void* stream);

/* One modified Gram-Schmidt step (gmres krylov.py:109-123; ProjectionSpace.absorb
 * krylov.py:229-231): if vprev, w -= (*hprev) vprev and, if w2, w2 -= (*hprev) v2prev;
 * out[0] = <w, vnext> (if vnext), out[1] = <w, w> (if want_norm).
 * gate (device scalar, may be NULL): when *gate == 0 the pass is skipped entirely
 * (the conditional second Gram-Schmidt sweep decided on the device; needs
 * 16-byte aligned arrays and an even P). */
int sf_mgs_step_f64(double* w, const double* vprev, const double* hprev, const double* vnext,
                    double* w2, const double* v2prev, const uint8_t* mult, int want_norm,
                    long long P, double* partials, unsigned* counter, double* out,
                    const double* gate, void* stream);

/* GMRES Arnoldi bookkeeping on the device (krylov.py:110-123): blk holds the
 * iteration's scalars (first sweep pairs at 2i, second sweep at o2 + 2i);
 * phase 0 writes blk[o3] = (norm_after < 0.7071 norm_before) and blk[o3+1] =
 * norm_after, phase 1 replaces blk[o3+1] by the second sweep's norm if blk[o3];
 * phase 2 is phase 0 plus blk[o2] = blk[2(j+1)] (the first sweep's last pass
 * also computed <w, v_0>, the second sweep's first coefficient). */
int sf_gmres_gate_f64(double* blk, int j, int o2, int o3, int phase, void* stream);

/* x = x0 + sum_i coef[i] * M v[i] accumulated in i order; v is a DEVICE array
 * of nv pointers, coef a device array (gmres update krylov.py:150-154 with
 * zs[i] = M vs[i]; ProjectionSpace.prepare krylov.py:206-209 with M = I). */
int sf_lincomb_f64(double* x, const double* x0, const double* const* v, const double* coef,
                   const double* invdiag, int nv, long long P, void* stream);

/* r = b - ax; out[0] = <r, r>  (krylov.py:155-157) */
int sf_residual_f64(double* r, const double* b, const double* ax, const uint8_t* mult, long long P,
                    double* partials, unsigned* counter, double* out, void* stream);

/* y = x / *s (and y2 = x2 / *s if y2) -- krylov.py:98, 149, 235-236 */
int sf_scale_div_f64(double* y, const double* x, double* y2, const double* x2, const double* s,
                     long long P, void* stream);

/* Strong-form operators (operators.py): op 0 grad (:59-66, in u -> out 3 comps),
 * 1 div (:69-76, in v -> out), 2 curl (:79-88, in v -> out v), 3 advect_vec
 * (:108-126, collocation; in v, c -> out = sign * (c . grad) v). */
int sf_deriv_f64(int op, const double* d_host, int n, const double* in, const double* c,
                 const double* rx, double* out, long long E, double sign, int exact,
                 void* stream);

/* weak_grad_dot / cdtp (operators.py:91-105): out = sum_s D_s^T (bm rx_s . w) */
int sf_cdtp_f64(const double* d_host, int n, const double* w, const double* rx, const double* bm,
                double* out, long long E, int exact, void* stream);

/* cfl (operators.py:161-182) without the dt factor: *out_bits = max(*out_bits,
 * bits of max_p sum_s |rx_s . v| / dxi_s).  Initialise *out_bits to 0. */
int sf_cfl_f64(const double* v, const double* rx, const double* dxi_host, int n, long long E,
               unsigned long long* out_bits, int exact, void* stream);

/* BDF/EXT history sums (timestep.py:227-232) over P3 = 3*E*n^3 values:
 * vhat = sum_q a_dt[q] vel[q] + beta[q] nl[q]; omega = sum_q beta[q] crl[q].
 * vel/nl/crl are HOST arrays of `order` device pointers. */
int sf_bdf_ext_f64(double* vhat, double* omega, const double* const* vel, const double* const* nl,
                   const double* const* crl, const double* a_dt, const double* beta, int order,
                   long long P3, void* stream);

/* ---------------------------------------------------------------------------
 * Multi-GPU: NVLink peer-memory reduction (replaces the NCCL all-gather of
 * glsc3 partials on the Krylov critical path)
 * ------------------------------------------------------------------------- */

/* size of a cudaIpcMemHandle_t in bytes */
int sf_ipc_handle_bytes(void);
/* doubles in one rank's mailbox (double-banked slots of up to 4 partials) */
int sf_peer_mailbox_doubles(int world);
/* zero-initialised cudaMalloc allocation (IPC handles name whole allocations) */
int sf_dev_alloc_zero(long long bytes, void** out);
int sf_dev_free(void* p);
int sf_ipc_get_handle(void* dev_ptr, unsigned char* handle_out);
int sf_ipc_open_handle(const unsigned char* handle, void** dev_ptr_out);
int sf_ipc_close_handle(void* dev_ptr);
/* out[0..k) = sum over ranks (rank order) of every rank's in[0..k), k <= 4.
 * boxes: HOST array of `world` mailbox pointers (own + IPC-opened peers);
 * seq: DEVICE uint64 counting the reductions this rank has executed (zero
 * before the first; each call exchanges *seq + 1 and advances it, so a gated
 * pass that skips consumes no number and graph-captured calls stay in step);
 * error: device flag set to 1 if a peer did not arrive within 5 s -- then out is
 * NaN, and every later call returns NaN at once.  in and out may alias. */
int sf_peer_allreduce_f64(double* const* boxes, int world, int rank, unsigned long long* seq,
                          unsigned* error, const double* in, int k, double* out, void* stream);

/* Fused compute + collective: sf_mgs_step_f64 / the weighted glsc3 whose last
 * thread block publishes the rank's partials to every peer over NVLink and
 * returns the rank-order global sums in `out` (no separate collective).  The
 * peer arguments are those of sf_peer_allreduce_f64. */
int sf_mgs_step_peer_f64(double* w, const double* vprev, const double* hprev, const double* vnext,
                         double* w2, const double* v2prev, const uint8_t* mult, int want_norm,
                         long long P, double* partials, unsigned* counter, double* out,
                         double* const* boxes, int world, int rank, unsigned long long* seq,
                         unsigned* error, const double* gate, void* stream);
int sf_glsc3_peer_f64(const double* a, const double* b, const uint8_t* mult, long long P,
                      double* partials, unsigned* counter, double* out, double* const* boxes,
                      int world, int rank, unsigned long long* seq, unsigned* error, void* stream);

/* NVLink halo exchange of the multi-GPU dssum (replaces the NCCL send/recv of
 * the interface copies; SURVEY 8e collective C1).  Each rank owns an IPC-exported
 * inbox of sf_halo_inbox_doubles(n_recv) doubles: 32 header doubles (uint64 flag
 * per sender rank), then two banks of n_recv values (bank = seq & 1) laid out as
 * the dssum's receive buffer.  Header word 16 is the rank's exchange counter
 * (device memory, zero at allocation): the call number seq = counter + 1.
 *   sf_halo_put_f64: v[send_idx[i]] for peer q's segment [seg[q], seg[q+1]) is
 *     stored at peer_dst[q][bank * peer_stride[q] + i - seg[q]] (NVLink stores);
 *     after a system-scope fence the last block advances own_inbox's counter and
 *     writes seq to peer_flag[q] (release).  counter: a zeroed device uint32,
 *     re-armed by the kernel.  No-op once *error is set.
 *   sf_halo_wait: one warp waits (acquire) until own_flags[peer_rank[q]] >= seq
 *     for every peer; sets *error after 5 s instead of hanging.
 * Both are stream-ordered and take the same arguments on every call (CUDA-graph
 * capturable); the dssum that follows reads the bank through recv_seq. */
int sf_halo_inbox_doubles(long long n_recv);
int sf_halo_header_doubles(void);
int sf_halo_put_f64(const double* v, const int* send_idx, int n_peers, const int* peer_rank,
                    const long long* seg, double* const* peer_dst, const long long* peer_stride,
                    unsigned long long* const* peer_flag, unsigned long long* own_inbox,
                    unsigned* counter, const unsigned* error, void* stream);
int sf_halo_wait(const unsigned long long* own_flags, int n_peers, const int* peer_rank,
                 unsigned* error, void* stream);

/* ---------------------------------------------------------------------------
 * Function-space setup (space.py:182-245), bit-identical to build_space
 * ------------------------------------------------------------------------- */

/* coords (3, E, n^3) = sum_c corners[e, c, l] * wc[c, p] (space.py:182-192);
 * corners (E, 8, 3), wc (8, n^3) trilinear corner weights, device arrays. */
int sf_trilinear_coords_f64(const double* corners, const double* wc, int n, long long E,
                            double* coords, void* stream);

/* rx (9 planes), jac, bm, geom (6 planes) from coords (space.py:214-245). */
int sf_metrics_f64(const double* d_host, const double* w_host, int n, const double* coords,
                   long long E, double* rx, double* jac, double* bm, double* geom, void* stream);

/* Over-integrated convection in one launch (Dealias.advect via advect_vec,
 * operators.py:119-158): out (3, E, n^3) = sign * project_back(wjac_f *
 * sum_l to_fine(c_l) to_fine(grad_l v_f)) / bm, every fine-grid field in shared
 * memory.  d_host (n x n) GLL derivative and j_host (m x n) GLL -> GL
 * interpolation are HOST arrays; (n, m) in {(8, 12), (6, 9), (4, 6)}; wjac_f
 * (E, m^3); exact = 1: the reference's contraction order without FMA. */
int sf_dealias_advect_f64(const double* d_host, const double* j_host, int n, int m, const double* c,
                          const double* v, const double* rx, const double* wjac_f, const double* bm, long long E,
                          double sign, double* out, int exact, void* stream);

/* ---------------------------------------------------------------------------
 * Hybrid overlapping Schwarz preconditioner (precond.py:94-250)
 * ------------------------------------------------------------------------- */

/* Device state of one HybridSchwarz (built by precond.HybridSchwarz; every
 * pointer is device memory).  G global ids, P local points, nv mesh vertices,
 * S = padded subdomain size, nnn = n^3. */
typedef struct SfSchwarz {
  long long G, P, nv;
  int nnn, S;
  const long long* first;       /* (G) local index of each gid's first copy */
  const long long* gid;         /* (P) */
  const double* wsqrt;          /* (G) 1 / sqrt(overlap count) */
  double* rg;                   /* (G) work: gathered residual */
  double* rw;                   /* (G + 1) work: wsqrt * rg, rw[G] = 0 (padding slot) */
  const long long* pt_ptr;      /* (nv + 1) restriction rows: vertex -> (element, corner) */
  const long long* pt_ent;      /*   entries element * 8 + corner, ascending element */
  const double* tw;             /* (nnn, 8) trilinear corner weights */
  const uint8_t* vfixed;        /* (nv) constrained vertices */
  double* rc_part;              /* (nv) work: this rank's restriction (owned gids) */
  double* rc;                   /* (nv) work: restricted residual (= rc_part on one rank) */
  int ac_width;                 /* coarse matrix, ELL (nv, ac_width), ascending columns */
  const int* ac_col;
  const double* ac_val;
  const double* ac_inv_diag;
  double *xc, *cr, *cz, *cp, *cap;   /* (nv) coarse CG vectors; xc = coarse solution */
  double* cpart;                /* (2 * coarse_blocks) partial sums */
  unsigned* cbar;               /* (2) grid-barrier words, zero between launches */
  int coarse_iters, coarse_blocks;
  const int* sub;               /* (E, S) nodes of each subdomain slot, rows grouped by class;
                                   padding slots name rw's zero slot */
  double* rwg;                  /* (E, S) work: rw[sub], the solve GEMM operand */
  double* sol;                  /* (E, S) work: local solutions (class-ordered rows) */
  const double* sol_recv;       /* N > 1: the peers' solutions on this rank's gids */
  long long n_sol;              /* E * S: acc_pos >= n_sol index sol_recv */
  const long long* acc_off;     /* (G + 1) overlap accumulation: gid -> sol slots, */
  const int* acc_pos;           /*   ascending global subdomain */
  const int* cvert;             /* (E, 8) element corners, ascending vertex id */
  const uint8_t* ccorn;         /* (E, 8) their corner numbers */
  const uint8_t* constrained;   /* (G) Dirichlet gids */
  double* z;                    /* (G) work: assembled correction */
  const uint8_t* rflag;         /* (P) point carries its gid's owned first copy */
  double* se;                   /* (E, 8) work: per element corner restriction sums */
  long long L;                  /* nodes incl. the peers' layer nodes; rw has L + 1 */
} SfSchwarz;

/* out = M^-1 r for the hybrid Schwarz preconditioner (HybridSchwarz.__call__,
 * precond.py:239-250), in stream-ordered stages (no host sync, deterministic):
 *   gather      rg, rw of this rank's nodes (G counts them; all gids on one rank)
 *   restrict    this rank's coarse restriction (owned gids) -> rc_part
 *   rank_sum    N > 1: rc = rank-order sum of the all-gathered partials
 *   coarse      fixed-iteration Jacobi-CG on the vertex problem (one launch)
 *   gather_rw   rwg = rw[sub], then per class sol_c = rwg_c inv_c^T (FP64 GEMM
 *               issued by the caller)
 *   finalize    ordered overlap sums (own + received solutions) + prolongation
 *   scatter     out[p] = z[node of p]
 * N > 1: the layer residuals, restriction partials and subdomain solutions
 * travel over NVLink between the stages (halo put/wait + sf_halo_unbank_f64). */
int sf_schwarz_gather_f64(const SfSchwarz* s, const double* r, void* stream);
int sf_schwarz_restrict_f64(const SfSchwarz* s, void* stream);
int sf_schwarz_rank_sum_f64(const SfSchwarz* s, const double* recv, int rank, int world, void* stream);
int sf_schwarz_coarse_f64(const SfSchwarz* s, void* stream);
int sf_schwarz_gather_rw_f64(const SfSchwarz* s, void* stream);
int sf_schwarz_finalize_f64(const SfSchwarz* s, void* stream);
int sf_schwarz_scatter_f64(const SfSchwarz* s, double* out, void* stream);
/* out[0..n) = the current bank of a double-banked halo inbox (bank 0 at bank0,
 * bank stride `stride`, call counter *seq; csrc/halo.cu) */
int sf_halo_unbank_f64(const double* bank0, const unsigned long long* seq, long long stride, long long n,
                       double* out, void* stream);
/* blocks of the coarse CG launch (= SM count) */
int sf_schwarz_coarse_blocks(void);

#ifdef __cplusplus
}
#endif

#endif /* SEMFLOW_B200_H */
