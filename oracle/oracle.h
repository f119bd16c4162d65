/* oracle.h — plain, slow, obviously-correct CPU oracle for the RK4 + 2SHOC NLSE step.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or call this library.  It shares no
 * code, headers, tables or constants with the CUDA library (paper_1109_1027_b200/).
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, cited as P:line):
 *   NLSE  i Psi_t + a Lap(Psi) - V Psi + s|Psi|^2 Psi = 0                (`NLSE`)
 *   F(Psi) = i [ a Lap(Psi) + (s|Psi|^2 - V) Psi ]
 *   Lap by the two-step compact scheme in its per-axis ("multi-storage") form:
 *     step 1  D_d = delta_d^2 Psi                 (`2shoc1d`, `2d2shocMs1`, `3d2shocMs1`)
 *     step 2  Lap = sum_d 7/6 D_d - (D_d(+e_d) + D_d(-e_d))/12
 *                                                 (`2shoc1d2`, `2d2shocMs2`, `3d2shocMs2`)
 *   boundary rule for the intermediate D (readings R8,R9):
 *     lambda_b = -(s|Psi_b|^2 - V_b) Psi_b / a     (Dirichlet, `dbc_lap`)
 *     lambda_b = 0                                 (Laplacian-zero)
 *     D_d(b) = lambda_b - sum_{e != d} D_e(b)      at d-face points b
 *     Lap_b  = lambda_b
 *   Psi_t boundary:  F_b = 0 (Dirichlet, `dbc_ut`);  F_b = i N_b Psi_b
 *     (Laplacian-zero, reading R9)
 *   MSD (1D only): lambda_b = [Re(D_{b-1}/Psi_{b-1}) + (N_{b-1}-N_b)/a] Psi_b
 *     (`msdbc_lap`, reading R28); F_b = i Im(F_{b-1}/Psi_{b-1}) Psi_b (`msdbc_ut`)
 *   RK4 exactly as the paper's 10-step listing with K_tot, K_tmp, Psi_tmp (`RK4`,
 *     P:366-382).
 *   CD scheme (RK4+CD): Lap = sum_d D_d, same boundary values.
 *
 * Arithmetic: IEEE double, explicit (re, im) pairs, no FMA contraction
 * (-ffp-contract=off), fixed loop order; OpenMP splits independent output points only.
 * Layout: row-major [z][y][x], x fastest, complex interleaved (re, im).
 */
#ifndef NLSE_ORACLE_H
#define NLSE_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_BC_DIRICHLET = 0, ORC_BC_LAPZERO = 1, ORC_BC_MSD = 2 };
enum { ORC_SCHEME_2SHOC = 0, ORC_SCHEME_CD = 1 };

typedef struct {
  int dims;          /* 1, 2, 3 */
  int64_t n[3];      /* counts x, y, z (unused axes = 1) */
  double h[3];       /* spacing per axis */
  double a, s;       /* NLSE parameters */
  const double *V;   /* potential per point (double), or NULL for V = 0 */
  int bc;            /* ORC_BC_* */
  int scheme;        /* ORC_SCHEME_* */
} orc_problem;

/* Lap(psi) -> L (interior: 2SHOC / CD; boundary points: lambda_b).  0 or -1. */
int orc_laplacian(const orc_problem *P, const double *psi, double *L);
/* F(psi) -> F, boundary rows per the BC. */
int orc_rhs(const orc_problem *P, const double *psi, double *F);
/* nsteps classic RK4 steps of size dt, in place (the paper's listing). */
int orc_rk4(const orc_problem *P, double *psi, double dt, int64_t nsteps);
/* min / max over all points of N = s|psi|^2 - V. */
int orc_N_minmax(const orc_problem *P, const double *psi, double *nmin, double *nmax);
/* Stability bound `kdfull` with B = 0 (Table 1 Dirichlet; Laplacian-zero by
 * reading R14) and the G set of Table 2, from the extreme values of N
 * (N = s|psi|^2 - V) over the whole grid.  Isotropic h: the paper's formula
 *   k = sqrt(8) h^2 / (a max_{i, g in G(d)} |L_i - g|),  L_i = (h^2/a) N_i.
 * Anisotropic h: reading R17.  Returns kmax (> 0) or a negative value. */
double orc_kmax_from_N(int dims, const double h[3], double a, double nmin, double nmax);
double orc_kmax(const orc_problem *P, const double *psi);
/* The G set of Table 2 for d (1..3), in units of 1/12; returns its size. */
int orc_table2_G(int d, int *out12);
/* Test-infrastructure knob: OpenMP threads of the point loops (n > 0 sets); returns the count
 * in effect. */
int orc_set_threads(int n);

#ifdef __cplusplus
}
#endif
#endif
