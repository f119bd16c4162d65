// stage_line.cuh — fused RK4-stage kernel for 1D grids, and the reductions.
//
// 1D has no tile to stage: each thread evaluates one point from five coalesced
// neighbouring loads (L1 serves the overlap), with the face rule of DESIGN.md R8 reduced to
// 1D (D(b) = lambda_b, `dbc_lap` P:402) realised as a ghost value computed in registers:
//   ghost(-1) = h^2 lambda_0 + 2 Psi_0 - Psi_1,   ghost(N) = h^2 lambda_{N-1} + 2 Psi_{N-1} - Psi_{N-2}.
#pragma once
#include "stage_stream.cuh"

namespace nlse {

template <typename R, int MODE>
__global__ void __launch_bounds__(256) stage_line_kernel(const cplx<R> *__restrict__ Tin, const cplx<R> *__restrict__ psi,
                                                         const cplx<R> *__restrict__ acc, const StageParams<R> P) {
  using CT = cplx<R>;
  const int n = P.nx;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const CT c = Tin[i];
    const bool bnd = i == 0 || i == n - 1;
    const R V = potential(P, int(i), 0, 0);
    const R N = fma(P.s, norm2(c), -V);
    CT L, F;
    if (!bnd) {
      const CT m1 = Tin[i - 1], p1 = Tin[i + 1];
      CT m2, p2;
      if (i >= 2) m2 = Tin[i - 2];
      else m2 = axpy(R(2) * m1 - c, P.hx2, lambda_b(P, m1, potential(P, 0, 0, 0)));
      if (i <= n - 3) p2 = Tin[i + 2];
      else p2 = axpy(R(2) * p1 - c, P.hx2, lambda_b(P, p1, potential(P, n - 1, 0, 0)));
      L = P.cx * (R(16) * (m1 + p1) - (m2 + p2) - R(30) * c);
      F = mk<R>(-fma(P.a, L.im, N * c.im), fma(P.a, L.re, N * c.re));
    } else {
      L = lambda_b(P, c, V);
      F = P.bc == 0 ? mk<R>(R(0), R(0)) : mk<R>(-(N * c.im), N * c.re);
    }
    if (MODE == M_LAP) {
      P.out_T[i] = L;
    } else if (MODE == M_S1) {
      P.out_acc[i] = axpy(c, P.ca, F);
      P.out_T[i] = axpy(c, P.cb, F);
    } else if (MODE == M_S2 || MODE == M_S3) {
      P.out_acc[i] = axpy(acc[i], P.ca, F);
      P.out_T[i] = axpy(psi[i], P.cb, F);
    } else {
      P.out_T[i] = axpy(acc[i], P.cb, F);
    }
  }
}

// ---------------------------------------------------------------------------------------
// min / max of N = s|Psi|^2 - V over the local grid (for `kdfull`), and a finiteness scan.
// One partial (min, max, nonfinite-count) triple per block; the host folds them.
template <typename R>
__global__ void __launch_bounds__(256) reduce_N_kernel(const cplx<R> *__restrict__ psi, const StageParams<R> P,
                                                       double *__restrict__ part) {
  double lo = INFINITY, hi = -INFINITY, bad = 0;
  const int64_t total = int64_t(P.nx) * P.ny * P.nz;
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < total; q += int64_t(gridDim.x) * blockDim.x) {
    const int gx = int(q % P.nx);
    const int64_t r = q / P.nx;
    const int gy = int(r % P.ny), lz = int(r / P.ny);
    const cplx<R> c = psi[(int64_t(lz) * P.ny + gy) * P.pitch + gx];
    if (!isfinite(c.re) || !isfinite(c.im)) bad += 1;
    const double N = double(fma(P.s, norm2(c), -potential(P, gx, gy, lz)));
    lo = fmin(lo, N);
    hi = fmax(hi, N);
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    bad += __shfl_xor_sync(0xffffffffu, bad, o);
  }
  __shared__ double s[3][8];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { s[0][w] = lo; s[1][w] = hi; s[2][w] = bad; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < int(blockDim.x >> 5); ++i) {
      lo = fmin(lo, s[0][i]);
      hi = fmax(hi, s[1][i]);
      bad += s[2][i];
    }
    part[3 * blockIdx.x] = lo;
    part[3 * blockIdx.x + 1] = hi;
    part[3 * blockIdx.x + 2] = bad;
  }
}

// Pitched <-> dense copies are done with cudaMemcpy2DAsync by the host; no kernel needed.

}  // namespace nlse
