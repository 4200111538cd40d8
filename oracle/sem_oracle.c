/*
 * sem_oracle.c -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * CPU restatement of the reference's element kernels (the numba lane,
 * /root/reference/pkg/src/semflow/kernels/_numba.py) in plain C.  Loop nests and
 * accumulation order follow the reference line by line and the file is compiled
 * with -ffp-contract=off, so every output is bit-identical to the numba lane
 * (pinned against tests/golden/kernels.npz by tests/test_oracle.py).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may load
 * this library (oracle/liboracle.so, built by oracle/Makefile).
 *
 * Layout: fields (E, n, n, n) C order; g (6, E, n, n, n).
 */
#include <pthread.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <unistd.h>

/* ---- minimal static-schedule parallel-for over [0, N) on pthreads ---------
 * (no OpenMP runtime in this image); each index is processed by exactly one
 * thread with the serial loop body, so results do not depend on the count. */
typedef void (*range_fn)(long long lo, long long hi, void* ctx);
struct job { range_fn fn; void* ctx; long long lo, hi; };
static void* run_job(void* p) { struct job* j = (struct job*)p; j->fn(j->lo, j->hi, j->ctx); return NULL; }

int or_num_threads(void) {
  const char* s = getenv("ORACLE_THREADS");
  int t = s ? atoi(s) : (int)sysconf(_SC_NPROCESSORS_ONLN);
  return t < 1 ? 1 : (t > 256 ? 256 : t);
}

static void parallel_for(long long N, range_fn fn, void* ctx) {
  int T = or_num_threads();
  if (N < 2 * T || T == 1) { fn(0, N, ctx); return; }
  pthread_t th[256];
  struct job jobs[256];
  for (int t = 0; t < T; ++t) {
    jobs[t].fn = fn; jobs[t].ctx = ctx;
    jobs[t].lo = N * t / T; jobs[t].hi = N * (t + 1) / T;
    pthread_create(&th[t], NULL, run_job, &jobs[t]);
  }
  for (int t = 0; t < T; ++t) pthread_join(th[t], NULL);
}

#define IDX(e, i, j, k) ((((size_t)(e) * n + (i)) * n + (j)) * n + (k))

/* _numba.py:15-60 -- one-axis contraction with an m x n matrix a */
struct apply_ctx { int axis; const double* a; int m, n; const double* u; double* out; };
static void apply_range(long long lo, long long hi, void* cp) {
  struct apply_ctx* c = (struct apply_ctx*)cp;
  const int n = c->n, m = c->m, axis = c->axis;
  const double *a = c->a, *u = c->u;
  for (long long e = lo; e < hi; ++e)
    for (int x = 0; x < n; ++x)
      for (int y = 0; y < n; ++y)
        for (int p = 0; p < m; ++p) {
          double acc = 0.0;
          size_t o;
          if (axis == 0) {
            for (int q = 0; q < n; ++q) acc += a[p * n + q] * u[IDX(e, q, x, y)];
            o = (((size_t)e * m + p) * n + x) * n + y;
          } else if (axis == 1) {
            for (int q = 0; q < n; ++q) acc += a[p * n + q] * u[IDX(e, x, q, y)];
            o = (((size_t)e * n + x) * m + p) * n + y;
          } else {
            for (int q = 0; q < n; ++q) acc += a[p * n + q] * u[IDX(e, x, y, q)];
            o = (((size_t)e * n + x) * n + y) * m + p;
          }
          c->out[o] = acc;
        }
}
void or_apply_axis(int axis, const double* a, int m, int n, const double* u, double* out,
                   long long E) {
  struct apply_ctx c = {axis, a, m, n, u, out};
  parallel_for(E, apply_range, &c);
}

/* _numba.py:63-83 -- three reference derivatives, separate sequential sums */
struct grad_ctx { const double* d; int n; const double* u; double *ur, *us, *ut; };
static void grad_range(long long lo, long long hi, void* cp) {
  struct grad_ctx* c = (struct grad_ctx*)cp;
  const int n = c->n;
  const double *d = c->d, *u = c->u;
  for (long long e = lo; e < hi; ++e)
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j)
        for (int k = 0; k < n; ++k) {
          double ar = 0.0, as = 0.0, at = 0.0;
          for (int q = 0; q < n; ++q) {
            ar += d[i * n + q] * u[IDX(e, q, j, k)];
            as += d[j * n + q] * u[IDX(e, i, q, k)];
            at += d[k * n + q] * u[IDX(e, i, j, q)];
          }
          c->ur[IDX(e, i, j, k)] = ar;
          c->us[IDX(e, i, j, k)] = as;
          c->ut[IDX(e, i, j, k)] = at;
        }
}
void or_grad_ref(const double* d, int n, const double* u, double* ur, double* us, double* ut,
                 long long E) {
  struct grad_ctx c = {d, n, u, ur, us, ut};
  parallel_for(E, grad_range, &c);
}

/* _numba.py:86-131 -- local weak Helmholtz action, interleaved transposed sum */
struct ax_ctx { const double *d, *g, *b, *u; int n; double* w; long long E; double lv, lm; };
static void ax_range(long long lo, long long hi, void* cp) {
  struct ax_ctx* c = (struct ax_ctx*)cp;
  const int n = c->n;
  const size_t NNN = (size_t)n * n * n;
  const size_t PT = (size_t)c->E * NNN;
  const double *d = c->d, *g = c->g, *u = c->u;
  double ur[1000], us[1000], ut[1000], f1[1000], f2[1000], f3[1000];
  for (long long e = lo; e < hi; ++e) {
    const double* ue = u + (size_t)e * NNN;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j)
        for (int k = 0; k < n; ++k) {
          double ar = 0.0, as = 0.0, at = 0.0;
          for (int q = 0; q < n; ++q) {
            ar += d[i * n + q] * ue[(q * n + j) * n + k];
            as += d[j * n + q] * ue[(i * n + q) * n + k];
            at += d[k * n + q] * ue[(i * n + j) * n + q];
          }
          int p = (i * n + j) * n + k;
          ur[p] = ar;
          us[p] = as;
          ut[p] = at;
        }
    for (size_t p = 0; p < NNN; ++p) {
      size_t gp = (size_t)e * NNN + p;
      double g0 = g[gp], g1 = g[PT + gp], g2 = g[2 * PT + gp];
      double g3 = g[3 * PT + gp], g4 = g[4 * PT + gp], g5 = g[5 * PT + gp];
      f1[p] = g0 * ur[p] + g1 * us[p] + g2 * ut[p];
      f2[p] = g1 * ur[p] + g3 * us[p] + g4 * ut[p];
      f3[p] = g2 * ur[p] + g4 * us[p] + g5 * ut[p];
    }
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j)
        for (int k = 0; k < n; ++k) {
          double acc = 0.0;
          for (int q = 0; q < n; ++q) {
            acc += d[q * n + i] * f1[(q * n + j) * n + k];
            acc += d[q * n + j] * f2[(i * n + q) * n + k];
            acc += d[q * n + k] * f3[(i * n + j) * n + q];
          }
          double wv = c->lv * acc;
          size_t gp = (size_t)e * NNN + (size_t)(i * n + j) * n + k;
          if (c->lm != 0.0) wv += c->lm * c->b[gp] * u[gp];
          c->w[gp] = wv;
        }
  }
}
void or_ax_helm(const double* d, int n, const double* g, const double* b, const double* u,
                double* w, long long E, double lv, double lm) {
  if (n > 10) return;
  struct ax_ctx c = {d, g, b, u, n, w, E, lv, lm};
  parallel_for(E, ax_range, &c);
}

/* _numba.py:134-153 -- sequential per-gid sum in perm order / broadcast */
struct gs_ctx { const double* vals; const long long *perm, *off; double* out; int scatter; };
static void gs_range(long long lo, long long hi, void* cp) {
  struct gs_ctx* c = (struct gs_ctx*)cp;
  for (long long g = lo; g < hi; ++g) {
    if (c->scatter) {
      for (long long o = c->off[g]; o < c->off[g + 1]; ++o) c->out[c->perm[o]] = c->vals[g];
    } else {
      double acc = 0.0;
      for (long long o = c->off[g]; o < c->off[g + 1]; ++o) acc += c->vals[c->perm[o]];
      c->out[g] = acc;
    }
  }
}
void or_gs_gather(const double* vals, const long long* perm, const long long* off, long long n_gid,
                  double* sums) {
  struct gs_ctx c = {vals, perm, off, sums, 0};
  parallel_for(n_gid, gs_range, &c);
}
void or_gs_scatter(const double* sums, const long long* perm, const long long* off,
                   long long n_gid, double* out) {
  struct gs_ctx c = {sums, perm, off, out, 1};
  parallel_for(n_gid, gs_range, &c);
}

/* space.py:182-192 -- trilinear GLL coordinates, c accumulated 0..7 from 0.0 */
struct co_ctx { const double *corners, *wc; int nnn; long long E; double* coords; };
static void co_range(long long lo, long long hi, void* cp) {
  struct co_ctx* c = (struct co_ctx*)cp;
  const size_t PT = (size_t)c->E * c->nnn;
  for (long long e = lo; e < hi; ++e)
    for (int p = 0; p < c->nnn; ++p)
      for (int l = 0; l < 3; ++l) {
        double acc = 0.0;
        for (int k = 0; k < 8; ++k) acc += c->corners[((size_t)e * 8 + k) * 3 + l] * c->wc[k * c->nnn + p];
        c->coords[l * PT + (size_t)e * c->nnn + p] = acc;
      }
}
void or_trilinear_coords(const double* corners, const double* wc, int nnn, long long E,
                         double* coords) {
  struct co_ctx c = {corners, wc, nnn, E, coords};
  parallel_for(E, co_range, &c);
}
