/* icgen.h — seeded synthetic inputs (initial states Psi0 and potentials V) for the
 * 2SHOC/RK4 NLSE workloads.  This module is INPUT GENERATION ONLY: it contains
 * none of the method's arithmetic (no differences, no Laplacian, no RK4), so it
 * may be shared by the CPU oracle (oracle/) and by the harness that feeds the
 * CUDA library (tests/, bench.py).  The CUDA library itself never links it.
 *
 * Grid convention ("x_i = x_min + h i"): coordinate of index i
 * along axis d is xmin[d] + i*h[d].  Layout of every output box is row-major
 * [z][y][x] with x fastest and complex values interleaved (re, im) — the same
 * memory as torch.complex64 / complex128.
 *
 * Random numbers: counter-based SplitMix64 keyed by (seed, stream) and indexed
 * by the GLOBAL linear index (k*Ny + j)*Nx + i, so any box / z-slab of a grid is
 * generated identically to the same region of the whole grid.
 */
#ifndef ICGEN_H
#define ICGEN_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum icg_kind {
  ICG_NOISE = 0,        /* p0*((2u1-1) + i(2u2-1)) + p1 + i*p2                          */
  ICG_BRIGHT_SECH = 1,  /* p0*sech(p1*x) * exp(i*p2)          (C1: sqrt2 sech x)         */
  ICG_DARK_TANH = 2,    /* tanh(x)*(1 + p0*(2u0-1))           (C2)                       */
  ICG_TF_VORTEX2D = 3,  /* sqrt(max(0,p0 - V)) * prod_j (x-xj + i(y-yj))/|.|  (C3)
                           V = p1*x^2 + p1*y^2; p2 = #vortices; xj = p3 + p4*u3(2j),
                           yj = p3 + p4*u3(2j+1)                                        */
  ICG_TF_RING3D = 4,    /* sqrt(max(0,p0 - V)) * ((rho-p2) + i z)/|.| + p3*noise  (C4)
                           V = p1*(x^2+y^2+z^2)                                          */
  ICG_GAUSS_NOISE = 5,  /* exp(-r^2/p0) + p1*noise                              (C5)   */
  ICG_GAUSS_EXACT = 6,  /* exp(-r^2/(2 p0)) * exp(-i p1 t), t = p2  (PAPER 2dexpsol /
                           3dexpsol; p1 = dims)                  */
  ICG_SMOOTH_NOISE = 7, /* smooth analytic field + p0*noise at all points (tests):
                           (1+0.3 sin(x+0.5y-0.7z)) exp(i(0.8x - 0.6y + 0.4z))
                           * exp(-p1 r^2)                                              */
  ICG_DARK_MOVING = 8   /* co-moving dark soliton (`1dmds`) at time p4:
                           sqrt(Om/s) tanh(sqrt(|Om|/(2a)) (x - c t))
                           * exp(i[(c/(2a)) x + (Om - c^2/(4a)) t]);  p0=c, p1=Om, p2=a, p3=s */
};

typedef struct {
  int kind;
  int dims;            /* 1, 2, 3                                                        */
  int64_t n[3];        /* GLOBAL counts (x, y, z); unused axes = 1                       */
  double xmin[3];      /* coordinate of index 0 per axis                                 */
  double h[3];         /* spacing per axis                                               */
  uint64_t seed;
  double p[8];         /* kind-specific parameters (see enum)                            */
} icg_spec;

/* One U[0,1) draw: (splitmix64(idx ^ key) >> 11) * 2^-53,
 * key = (seed * 0x100000001B3) ^ (stream << 56).                                       */
double icg_uniform(uint64_t seed, uint32_t stream, uint64_t idx);

/* Fill the box [lo, lo+cnt) (per axis, x,y,z) of the global grid.  out has
 * cnt[0]*cnt[1]*cnt[2] complex elements.  Returns 0, or -1 on bad arguments.        */
int icg_fill_c128(const icg_spec *spec, const int64_t lo[3], const int64_t cnt[3], double *out);
int icg_fill_c64(const icg_spec *spec, const int64_t lo[3], const int64_t cnt[3], float *out);

/* Separable harmonic potential V = ((w0 (x-c0)^2) + w1 (y-c1)^2) + w2 (z-c2)^2 (terms
 * of absent axes omitted), materialised in double over the box.                      */
int icg_harmonic(int dims, const double xmin[3], const double h[3], const double w[3],
                 const double c[3], const int64_t lo[3], const int64_t cnt[3], double *V);

#ifdef __cplusplus
}
#endif
#endif
