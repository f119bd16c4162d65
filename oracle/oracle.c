/* oracle.c — plain CPU oracle for the RK4 + 2SHOC NLSE step.  TEST INFRASTRUCTURE ONLY
 * (see oracle.h for the scope rule and the paper passages each function follows).
 * Compile: gcc -O2 -ffp-contract=off -fno-fast-math -fopenmp                           */
#include "oracle.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---- point iteration helpers ---------------------------------------------------- */
typedef struct { int64_t n[3], st[3], total; } geom;

static geom mk_geom(const orc_problem *P) {
  geom g;
  g.n[0] = P->n[0]; g.n[1] = P->dims > 1 ? P->n[1] : 1; g.n[2] = P->dims > 2 ? P->n[2] : 1;
  g.st[0] = 1; g.st[1] = g.n[0]; g.st[2] = g.n[0] * g.n[1]; g.total = g.n[0] * g.n[1] * g.n[2];
  return g;
}

static int valid(const orc_problem *P) {
  if (!P || P->dims < 1 || P->dims > 3 || !(P->a > 0.0)) return 0;
  if (P->bc == ORC_BC_MSD && P->dims != 1) return 0; /* MSD: 1D only (reading R28) */
  for (int d = 0; d < P->dims; ++d)
    if (P->n[d] < 5 || !(P->h[d] > 0.0)) return 0;
  return 1;
}

/* Parallelism only splits the set of independent output points into contiguous ranges;
 * every point's arithmetic is the same whatever the thread count.                      */
#define PAR_MIN 4096
#define FEP_LOOP(g, nth_, tid_, ...)                                                      \
  {                                                                                      \
    const int64_t p0_ = (g).total * (tid_) / (nth_), p1_ = (g).total * ((tid_) + 1) / (nth_); \
    int64_t ix[3] = {p0_ % (g).n[0], (p0_ / (g).n[0]) % (g).n[1], p0_ / ((g).n[0] * (g).n[1])}; \
    for (int64_t p = p0_; p < p1_; ++p) {                                                \
      __VA_ARGS__                                                                        \
      if (++ix[0] == (g).n[0]) { ix[0] = 0; if (++ix[1] == (g).n[1]) { ix[1] = 0; ++ix[2]; } } \
    }                                                                                    \
  }
#define FOR_EACH_POINT(g, ...)                                                            \
  if ((g).total > PAR_MIN) {                                                             \
    _Pragma("omp parallel") {                                                            \
      int64_t nth_ = 1, tid_ = 0;                                                        \
      FEP_THREADS(nth_, tid_);                                                           \
      FEP_LOOP(g, nth_, tid_, __VA_ARGS__)                                               \
    }                                                                                    \
  } else FEP_LOOP(g, 1, 0, __VA_ARGS__)
#ifdef _OPENMP
#define FEP_THREADS(nth, tid) do { nth = omp_get_num_threads(); tid = omp_get_thread_num(); } while (0)
#else
#define FEP_THREADS(nth, tid) do { nth = 1; tid = 0; } while (0)
#endif

/* is the point with indices ix a boundary point (any index 0 or n-1 on an existing axis)? */
static inline int is_boundary(const geom *g, int dims, const int64_t ix[3]) {
  for (int d = 0; d < dims; ++d)
    if (ix[d] == 0 || ix[d] == g->n[d] - 1) return 1;
  return 0;
}

/* Steps 1-5 of the oracle; D[d] and N are caller scratch. */
static void lap_core(const orc_problem *P, const double *psi, double *L, double *D[3], double *N) {
  const geom g = mk_geom(P);
  const int dims = P->dims;

  /* 1. N_p = s |psi_p|^2 - V_p                                      (`nbnb1`)  */
  FOR_EACH_POINT(g, {
    double re = psi[2 * p], im = psi[2 * p + 1];
    double v = P->V ? P->V[p] : 0.0;
    N[p] = P->s * (re * re + im * im) - v;
  })

  /* 2. D_d = (psi[p+e_d] - 2 psi[p] + psi[p-e_d]) / h_d^2 where 1 <= index_d <= n_d-2
   *    (`2shoc1d` P:131, `2d2shocMs1` P:173-176, `3d2shocMs1` P:266-271).  Elsewhere 0. */
  for (int d = 0; d < dims; ++d) {
    const int64_t st = g.st[d], nd = g.n[d];
    const double ih2 = 1.0 / (P->h[d] * P->h[d]);
    double *Dd = D[d];
    FOR_EACH_POINT(g, {
      int64_t i = ix[d];
      if (i >= 1 && i <= nd - 2) {
        for (int c = 0; c < 2; ++c)
          Dd[2 * p + c] = (psi[2 * (p + st) + c] - 2.0 * psi[2 * p + c] + psi[2 * (p - st) + c]) * ih2;
      } else {
        Dd[2 * p] = 0.0;
        Dd[2 * p + 1] = 0.0;
      }
    })
  }

  /* 3.-4. lambda_b at boundary points (Dirichlet `dbc_lap` P:402; Laplacian-zero P:431),
   *    then the face fill D_d(b) = lambda_b - sum_{e != d} D_e(b) at d-face points
   *    (reading R8: "...or on the separate spatial derivatives", P:429
   *    "rearranging the boundary condition").  D values used on the right-hand side are
   *    the step-2 (tangential, interior-along-e) values: a d-face point is interior along
   *    every e != d, so no face fill ever overwrites a value another face fill reads.   */
  for (int d = 0; d < dims; ++d) {
    const int64_t nd = g.n[d];
    FOR_EACH_POINT(g, {
      int64_t i = ix[d];
      int face = (i == 0 || i == nd - 1); /* ... and all other indices interior */
      for (int e = 0; e < dims; ++e) {
        if (e == d) continue;
        if (ix[e] == 0 || ix[e] == g.n[e] - 1) face = 0;
      }
      if (face) {
        double lr = 0.0, li = 0.0;
        if (P->bc == ORC_BC_DIRICHLET) {
          lr = -(N[p] * psi[2 * p]) / P->a;
          li = -(N[p] * psi[2 * p + 1]) / P->a;
        } else if (P->bc == ORC_BC_MSD) {
          /* `msdbc_lap`: Lap_b = [Im(i Lap_{b-1} / Psi_{b-1}) + (N_{b-1} - N_b)/a] Psi_b,
           * Im(i z) = Re(z), with Lap_{b-1} the step-1 value D_{b-1} (reading R28).        */
          const int64_t q = (i == 0) ? p + 1 : p - 1;
          const double pr = psi[2 * q], pi = psi[2 * q + 1];
          const double re_ratio = (D[d][2 * q] * pr + D[d][2 * q + 1] * pi) / (pr * pr + pi * pi);
          const double fac = re_ratio + (N[q] - N[p]) / P->a;
          lr = fac * psi[2 * p];
          li = fac * psi[2 * p + 1];
        }
        for (int e = 0; e < dims; ++e) {
          if (e == d) continue;
          lr = lr - D[e][2 * p];
          li = li - D[e][2 * p + 1];
        }
        D[d][2 * p] = lr;
        D[d][2 * p + 1] = li;
      }
    })
  }

  /* 5. L_p = sum_d 7/6 D_d[p] - (D_d[p+e_d] + D_d[p-e_d]) / 12 at interior p
   *    (`2shoc1d2` P:132, `2d2shocMs2` P:177, `3d2shocMs2` P:272-275); CD: sum_d D_d[p];
   *    boundary points: L_b = lambda_b.                                         */
  FOR_EACH_POINT(g, {
    if (is_boundary(&g, dims, ix)) {
      if (P->bc == ORC_BC_DIRICHLET) {
        L[2 * p] = -(N[p] * psi[2 * p]) / P->a;
        L[2 * p + 1] = -(N[p] * psi[2 * p + 1]) / P->a;
      } else if (P->bc == ORC_BC_MSD) { /* 1D: the face value filled above */
        L[2 * p] = D[0][2 * p];
        L[2 * p + 1] = D[0][2 * p + 1];
      } else {
        L[2 * p] = 0.0;
        L[2 * p + 1] = 0.0;
      }
    } else {
      for (int c = 0; c < 2; ++c) {
        double acc = 0.0;
        for (int d = 0; d < dims; ++d) {
          const int64_t st = g.st[d];
          double term;
          if (P->scheme == ORC_SCHEME_CD)
            term = D[d][2 * p + c];
          else
            term = (7.0 / 6.0) * D[d][2 * p + c] - (D[d][2 * (p + st) + c] + D[d][2 * (p - st) + c]) / 12.0;
          acc = acc + term;
        }
        L[2 * p + c] = acc;
      }
    }
  })
}

typedef struct { double *D[3]; double *N; double *L; } scratch;

static int scratch_alloc(const orc_problem *P, scratch *w) {
  geom g = mk_geom(P);
  memset(w, 0, sizeof(*w));
  w->N = (double *)malloc(sizeof(double) * (size_t)g.total);
  w->L = (double *)malloc(sizeof(double) * 2 * (size_t)g.total);
  int ok = w->N && w->L;
  for (int d = 0; d < P->dims; ++d) {
    w->D[d] = (double *)malloc(sizeof(double) * 2 * (size_t)g.total);
    ok = ok && w->D[d];
  }
  return ok ? 0 : -1;
}
static void scratch_free(scratch *w) {
  for (int d = 0; d < 3; ++d) free(w->D[d]);
  free(w->N);
  free(w->L);
}

int orc_laplacian(const orc_problem *P, const double *psi, double *L) {
  if (!valid(P) || !psi || !L) return -1;
  scratch w;
  if (scratch_alloc(P, &w)) { scratch_free(&w); return -1; }
  lap_core(P, psi, L, w.D, w.N);
  scratch_free(&w);
  return 0;
}

/* 6. F = i (a L + N psi) at interior points; Dirichlet boundary F_b = 0
 *    exactly (`dbc_ut`, reading R10); Laplacian-zero F_b = i N_b psi_b (R9). */
static void rhs_core(const orc_problem *P, const double *psi, double *F, scratch *w) {
  const geom g = mk_geom(P);
  lap_core(P, psi, w->L, w->D, w->N);
  const double *L = w->L, *N = w->N;
  FOR_EACH_POINT(g, {
    double re = psi[2 * p], im = psi[2 * p + 1];
    if (is_boundary(&g, P->dims, ix)) {
      if (P->bc == ORC_BC_DIRICHLET) {
        F[2 * p] = 0.0;
        F[2 * p + 1] = 0.0;
      } else { /* i * (N psi) */
        F[2 * p] = -(N[p] * im);
        F[2 * p + 1] = N[p] * re;
      }
    } else {
      /* i * (x + i y) = -y + i x with x + i y = a L + N psi */
      double xr = P->a * L[2 * p] + N[p] * re;
      double xi = P->a * L[2 * p + 1] + N[p] * im;
      F[2 * p] = -xi;
      F[2 * p + 1] = xr;
    }
  })
  if (P->bc == ORC_BC_MSD) {
    /* `msdbc_ut`: Psi_t,b = i Im(Psi_t,b-1 / Psi_b-1) Psi_b, after the interior. */
    const int64_t n = g.n[0];
    const int64_t bs[2] = {0, n - 1}, qs[2] = {1, n - 2};
    for (int k = 0; k < 2; ++k) {
      const int64_t b = bs[k], q = qs[k];
      const double pr = psi[2 * q], pi = psi[2 * q + 1];
      const double m = (F[2 * q + 1] * pr - F[2 * q] * pi) / (pr * pr + pi * pi);
      F[2 * b] = -(m * psi[2 * b + 1]);
      F[2 * b + 1] = m * psi[2 * b];
    }
  }
}

int orc_rhs(const orc_problem *P, const double *psi, double *F) {
  if (!valid(P) || !psi || !F) return -1;
  scratch w;
  if (scratch_alloc(P, &w)) { scratch_free(&w); return -1; }
  rhs_core(P, psi, F, &w);
  scratch_free(&w);
  return 0;
}

/* 7. Classic RK4 as the paper writes it (`RK4`):
 *   1) Ktot = F(Psi)              6) Ktmp = F(Psitmp)
 *   2) Psitmp = Psi + k/2 Ktot    7) Ktot = Ktot + 2 Ktmp
 *   3) Ktmp = F(Psitmp)           8) Psitmp = Psi + k Ktmp
 *   4) Ktot = Ktot + 2 Ktmp       9) Ktmp = F(Psitmp)
 *   5) Psitmp = Psi + k/2 Ktmp   10) Psi = Psi + k/6 (Ktot + Ktmp)                    */
int orc_rk4(const orc_problem *P, double *psi, double dt, int64_t nsteps) {
  if (!valid(P) || !psi || !(dt > 0.0) || nsteps < 0) return -1;
  const geom g = mk_geom(P);
  const int64_t M = 2 * g.total;
  scratch w;
  double *Ktot = (double *)malloc(sizeof(double) * (size_t)M);
  double *Ktmp = (double *)malloc(sizeof(double) * (size_t)M);
  double *Ptmp = (double *)malloc(sizeof(double) * (size_t)M);
  if (!Ktot || !Ktmp || !Ptmp || scratch_alloc(P, &w)) {
    free(Ktot); free(Ktmp); free(Ptmp); scratch_free(&w);
    return -1;
  }
  const double k = dt;
  for (int64_t n = 0; n < nsteps; ++n) {
    rhs_core(P, psi, Ktot, &w);                                          /* 1 */
#pragma omp parallel for schedule(static) if (M > PAR_MIN)
    for (int64_t q = 0; q < M; ++q) Ptmp[q] = psi[q] + (k / 2.0) * Ktot[q]; /* 2 */
    rhs_core(P, Ptmp, Ktmp, &w);                                          /* 3 */
#pragma omp parallel for schedule(static) if (M > PAR_MIN)
    for (int64_t q = 0; q < M; ++q) {
      Ktot[q] = Ktot[q] + 2.0 * Ktmp[q];                                  /* 4 */
      Ptmp[q] = psi[q] + (k / 2.0) * Ktmp[q];                             /* 5 */
    }
    rhs_core(P, Ptmp, Ktmp, &w);                                          /* 6 */
#pragma omp parallel for schedule(static) if (M > PAR_MIN)
    for (int64_t q = 0; q < M; ++q) {
      Ktot[q] = Ktot[q] + 2.0 * Ktmp[q];                                  /* 7 */
      Ptmp[q] = psi[q] + k * Ktmp[q];                                     /* 8 */
    }
    rhs_core(P, Ptmp, Ktmp, &w);                                          /* 9 */
#pragma omp parallel for schedule(static) if (M > PAR_MIN)
    for (int64_t q = 0; q < M; ++q) psi[q] = psi[q] + (k / 6.0) * (Ktot[q] + Ktmp[q]); /* 10 */
  }
  free(Ktot); free(Ktmp); free(Ptmp);
  scratch_free(&w);
  return 0;
}

int orc_N_minmax(const orc_problem *P, const double *psi, double *nmin, double *nmax) {
  if (!valid(P) || !psi || !nmin || !nmax) return -1;
  const geom g = mk_geom(P);
  double lo = INFINITY, hi = -INFINITY;
  for (int64_t p = 0; p < g.total; ++p) { /* serial, fixed order */
    double re = psi[2 * p], im = psi[2 * p + 1];
    double v = P->V ? P->V[p] : 0.0;
    double N = P->s * (re * re + im * im) - v;
    if (N < lo) lo = N;
    if (N > hi) hi = N;
  }
  *nmin = lo;
  *nmax = hi;
  return 0;
}

/* Table 2 (`t:sumresults`), values x 1/12, typed from the paper. */
static const int G1[] = {64, 63, 46, 12, -3, -4};
static const int G2[] = {128, 127, 126, 110, 109, 92, 24, 9, 8, -6, -7, -8};
static const int G3[] = {192, 191, 190, 189, 174, 173, 172, 156, 155, 138,
                         36, 21, 20, 6, 5, 4, -9, -10, -11, -12};

int orc_table2_G(int d, int *out12) {
  const int *G = d == 1 ? G1 : (d == 2 ? G2 : G3);
  int n = d == 1 ? 6 : (d == 2 ? 12 : 20);
  if (d < 1 || d > 3) return 0;
  for (int i = 0; i < n; ++i) out12[i] = G[i];
  return n;
}

double orc_kmax_from_N(int dims, const double h[3], double a, double nmin, double nmax) {
  if (dims < 1 || dims > 3 || !(a > 0.0)) return -1.0;
  int iso = 1;
  for (int d = 1; d < dims; ++d)
    if (h[d] != h[0]) iso = 0;
  if (iso) {
    /* `kdfull`: k < sqrt(8) / max{||B||, max_{i,g} |L_i - g|} * h^2 / a,
     * L_i = (h^2/a) N_i, B = 0.  |L - g| is convex in L, so over L in [Lmin, Lmax]
     * its maximum is attained at an endpoint: scan the two endpoints against every g. */
    int G[20];
    int nG = orc_table2_G(dims, G);
    double hh = h[0] * h[0];
    double Lmin = (hh / a) * nmin, Lmax = (hh / a) * nmax;
    double M = 0.0; /* ||B||_inf = 0 */
    for (int q = 0; q < nG; ++q) {
      double g = (double)G[q] / 12.0;
      double e1 = fabs(Lmin - g), e2 = fabs(Lmax - g);
      if (e1 > M) M = e1;
      if (e2 > M) M = e2;
    }
    return sqrt(8.0) / M * hh / a;
  }
  /* Reading R17 (anisotropic extension, not in the paper): Gershgorin on the sum of
   * per-axis operators, -a Lap in [-(4/12) a H, (64/12) a H], H = sum_d 1/h_d^2, so the
   * linearised spectrum i(a Lap + N) has |mu| <= max((64/12) a H - Nmin, Nmax + (4/12) a H). */
  double H = 0.0;
  for (int d = 0; d < dims; ++d) H = H + 1.0 / (h[d] * h[d]);
  double m1 = (64.0 / 12.0) * a * H - nmin;
  double m2 = nmax + (4.0 / 12.0) * a * H;
  double M = fabs(m1) > fabs(m2) ? fabs(m1) : fabs(m2);
  return sqrt(8.0) / M;
}

double orc_kmax(const orc_problem *P, const double *psi) {
  double lo, hi;
  if (orc_N_minmax(P, psi, &lo, &hi)) return -1.0;
  return orc_kmax_from_N(P->dims, P->h, P->a, lo, hi);
}

/* Test-infrastructure knob (no arithmetic): OpenMP threads for the oracle's point loops.
 * n > 0 sets the count; returns the count now in effect. */
int orc_set_threads(int n) {
  if (n > 0) omp_set_num_threads(n);
  return omp_get_max_threads();
}
