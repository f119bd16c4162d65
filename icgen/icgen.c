/* icgen.c — seeded synthetic inputs for the 2SHOC/RK4 NLSE workloads.
 * Input generation only (see icgen.h); shared by oracle-side and CUDA-side harnesses.
 * Workload recipes: SURVEY.md §8(d) "Concrete inputs", BASELINE.json configs[0..4],
 * and the paper's accuracy experiments.                        */
#include "icgen.h"
#include <math.h>
#include <stddef.h>

static inline uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

double icg_uniform(uint64_t seed, uint32_t stream, uint64_t idx) {
  uint64_t key = (seed * 0x100000001B3ULL) ^ ((uint64_t)stream << 56);
  return (double)(splitmix64(idx ^ key) >> 11) * (1.0 / 9007199254740992.0);
}

/* value of the field at global index (i,j,k) -> (re, im) */
static void eval_point(const icg_spec *s, int64_t i, int64_t j, int64_t k, double *re, double *im) {
  const double x = s->xmin[0] + (double)i * s->h[0];
  const double y = s->dims > 1 ? s->xmin[1] + (double)j * s->h[1] : 0.0;
  const double z = s->dims > 2 ? s->xmin[2] + (double)k * s->h[2] : 0.0;
  const uint64_t gidx = ((uint64_t)k * (uint64_t)s->n[1] + (uint64_t)j) * (uint64_t)s->n[0] + (uint64_t)i;
  const double *p = s->p;
  double r = 0.0, m = 0.0;
  switch (s->kind) {
  case ICG_NOISE:
    r = p[0] * (2.0 * icg_uniform(s->seed, 1, gidx) - 1.0) + p[1];
    m = p[0] * (2.0 * icg_uniform(s->seed, 2, gidx) - 1.0) + p[2];
    break;
  case ICG_BRIGHT_SECH: {
    double amp = p[0] / cosh(p[1] * x);
    r = amp * cos(p[2]);
    m = amp * sin(p[2]);
  } break;
  case ICG_DARK_TANH: {
    double eps = p[0] * (2.0 * icg_uniform(s->seed, 0, gidx) - 1.0);
    r = tanh(x) * (1.0 + eps);
    m = 0.0;
  } break;
  case ICG_TF_VORTEX2D: {
    double V = p[1] * x * x + p[1] * y * y;
    double amp = sqrt(fmax(0.0, p[0] - V));
    double pr = 1.0, pi = 0.0;
    int nv = (int)p[2];
    for (int v = 0; v < nv; ++v) {
      double xj = p[3] + p[4] * icg_uniform(s->seed, 3, (uint64_t)(2 * v));
      double yj = p[3] + p[4] * icg_uniform(s->seed, 3, (uint64_t)(2 * v + 1));
      double dr = x - xj, di = y - yj, mod = hypot(dr, di);
      double fr = 0.0, fi = 0.0;
      if (mod > 0.0) { fr = dr / mod; fi = di / mod; }
      double tr = pr * fr - pi * fi, ti = pr * fi + pi * fr;
      pr = tr; pi = ti;
    }
    r = amp * pr;
    m = amp * pi;
  } break;
  case ICG_TF_RING3D: {
    double V = p[1] * (x * x + y * y + z * z);
    double amp = sqrt(fmax(0.0, p[0] - V));
    double rho = sqrt(x * x + y * y);
    double dr = rho - p[2], di = z, mod = hypot(dr, di);
    double fr = 0.0, fi = 0.0;
    if (mod > 0.0) { fr = dr / mod; fi = di / mod; }
    r = amp * fr + p[3] * (2.0 * icg_uniform(s->seed, 1, gidx) - 1.0);
    m = amp * fi + p[3] * (2.0 * icg_uniform(s->seed, 2, gidx) - 1.0);
  } break;
  case ICG_GAUSS_NOISE: {
    double r2 = x * x + y * y + z * z;
    r = exp(-r2 / p[0]) + p[1] * (2.0 * icg_uniform(s->seed, 1, gidx) - 1.0);
    m = p[1] * (2.0 * icg_uniform(s->seed, 2, gidx) - 1.0);
  } break;
  case ICG_GAUSS_EXACT: {
    double r2 = x * x + y * y + z * z;
    double amp = exp(-r2 / (2.0 * p[0]));
    double ph = -p[1] * p[2];
    r = amp * cos(ph);
    m = amp * sin(ph);
  } break;
  case ICG_SMOOTH_NOISE: {
    double r2 = x * x + y * y + z * z;
    double amp = (1.0 + 0.3 * sin(x + 0.5 * y - 0.7 * z)) * exp(-p[1] * r2);
    double ph = 0.8 * x - 0.6 * y + 0.4 * z;
    r = amp * cos(ph) + p[0] * (2.0 * icg_uniform(s->seed, 1, gidx) - 1.0);
    m = amp * sin(ph) + p[0] * (2.0 * icg_uniform(s->seed, 2, gidx) - 1.0);
  } break;
  case ICG_DARK_MOVING: {
    const double c = p[0], Om = p[1], a = p[2], sn = p[3], t = p[4];
    const double amp = sqrt(Om / sn) * tanh(sqrt(fabs(Om) / (2.0 * a)) * (x - c * t));
    const double ph = (c / (2.0 * a)) * x + (Om - c * c / (4.0 * a)) * t;
    r = amp * cos(ph);
    m = amp * sin(ph);
  } break;
  default:
    r = NAN; m = NAN;
  }
  *re = r;
  *im = m;
}

static int check_box(const icg_spec *s, const int64_t lo[3], const int64_t cnt[3]) {
  if (!s || !lo || !cnt || s->dims < 1 || s->dims > 3) return -1;
  for (int d = 0; d < 3; ++d) {
    if (cnt[d] < 0 || lo[d] < 0 || lo[d] + cnt[d] > s->n[d]) return -1;
    if (d >= s->dims && (s->n[d] != 1)) return -1;
  }
  return 0;
}

int icg_fill_c128(const icg_spec *s, const int64_t lo[3], const int64_t cnt[3], double *out) {
  if (check_box(s, lo, cnt) || !out) return -1;
  const int64_t rows = cnt[1] * cnt[2];
#pragma omp parallel for schedule(static)
  for (int64_t row = 0; row < rows; ++row) {
    const int64_t kk = row / cnt[1], jj = row % cnt[1];
    double *o = out + 2 * row * cnt[0];
    for (int64_t ii = 0; ii < cnt[0]; ++ii)
      eval_point(s, lo[0] + ii, lo[1] + jj, lo[2] + kk, &o[2 * ii], &o[2 * ii + 1]);
  }
  return 0;
}

int icg_fill_c64(const icg_spec *s, const int64_t lo[3], const int64_t cnt[3], float *out) {
  if (check_box(s, lo, cnt) || !out) return -1;
  const int64_t rows = cnt[1] * cnt[2];
#pragma omp parallel for schedule(static)
  for (int64_t row = 0; row < rows; ++row) {
    const int64_t kk = row / cnt[1], jj = row % cnt[1];
    float *o = out + 2 * row * cnt[0];
    for (int64_t ii = 0; ii < cnt[0]; ++ii) {
      double re, im;
      eval_point(s, lo[0] + ii, lo[1] + jj, lo[2] + kk, &re, &im);
      o[2 * ii] = (float)re;
      o[2 * ii + 1] = (float)im;
    }
  }
  return 0;
}

int icg_harmonic(int dims, const double xmin[3], const double h[3], const double w[3],
                 const double c[3], const int64_t lo[3], const int64_t cnt[3], double *V) {
  if (dims < 1 || dims > 3 || !V) return -1;
  const int64_t rows = cnt[1] * cnt[2];
#pragma omp parallel for schedule(static)
  for (int64_t row = 0; row < rows; ++row) {
    const int64_t kk = row / cnt[1], jj = row % cnt[1];
    double vy = 0.0, vz = 0.0;
    if (dims > 1) { double y = xmin[1] + (double)(lo[1] + jj) * h[1] - c[1]; vy = w[1] * (y * y); }
    if (dims > 2) { double z = xmin[2] + (double)(lo[2] + kk) * h[2] - c[2]; vz = w[2] * (z * z); }
    double *o = V + row * cnt[0];
    for (int64_t ii = 0; ii < cnt[0]; ++ii) {
      double x = xmin[0] + (double)(lo[0] + ii) * h[0] - c[0];
      double v = w[0] * (x * x);
      if (dims > 1) v = v + vy;
      if (dims > 2) v = v + vz;
      o[ii] = v;
    }
  }
  return 0;
}
