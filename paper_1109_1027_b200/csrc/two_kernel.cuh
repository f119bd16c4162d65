// two_kernel.cuh — the paper's own single-storage 2SHOC realisation ("TWO_KERNEL" variant),
// kept beside the fused kernel as the paper-faithful comparison point.
//
// Kernel A (step 1, `2d2shocs1` P:205-214, `3d2shocs` P:286-308):
//     D = sum_d delta_d^2 Psi at interior points, D_b = lambda_b at boundary points
//     (`dbc_lap` P:399-404; Laplacian-zero P:431), stored to HBM (one extra field).
// Kernel B (step 2 + RHS + RK4 stage combine):
//   isotropic h, the paper's printed stencils (`2d2shocs2` P:218-232, `3d2shocs2`
//   P:312-354; 1D `2shoc1d2` P:132):
//     L = -1/12 (sum_{2d neighbours} D - (16 - 2d) D) + 1/(6h^2) (sum_{edge-midpoints} Psi - 4 p Psi),
//     p = d(d-1)/2 coordinate planes;
//   anisotropic h (reading R17): the same operator written per axis,
//     L = D - sum_d (D(+e_d) + D(-e_d) - 2D)/12
//           + sum_{d<e} (h_d^2 + h_e^2)/12 * delta_d^2 delta_e^2 Psi.
// Shard seams: D is also evaluated on the two planes adjacent to the slab (from the 2-plane
// Psi halo), so one halo exchange per stage serves both steps.
#pragma once
#include "stage_stream.cuh"

namespace nlse {

template <typename R> struct TwoParams {
  int iso;
  R w2;             // isotropic: 1/(6 h^2)
  R cde[3];         // anisotropic pair weights (h_d^2 + h_e^2)/(12 h_d^2 h_e^2) for (x,y),(x,z),(y,z)
};

template <typename R> static void two_params(int dims, const double h[3], TwoParams<R> &Q) {
  Q.iso = 1;
  for (int d = 1; d < dims; ++d)
    if (h[d] != h[0]) Q.iso = 0;
  Q.w2 = R(1.0 / (6.0 * h[0] * h[0]));
  // kernel axes: x = axis 0, y = axis 1 (3D), z = streamed axis (dims-1)
  const double hx = h[0], hy = dims == 3 ? h[1] : 1.0, hz = dims >= 2 ? h[dims - 1] : 1.0;
  auto c = [](double a, double b) { return (a * a + b * b) / (12.0 * a * a * b * b); };
  Q.cde[0] = R(c(hx, hy));
  Q.cde[1] = R(c(hx, hz));
  Q.cde[2] = R(c(hy, hz));
}

template <typename R> struct PlaneView {  // stencil-input planes incl. the 2-plane halos
  const cplx<R> *in, *lo, *hi;
  int nz;
  int64_t plane;
  __device__ __forceinline__ const cplx<R> *operator()(int p) const {
    if (p >= 0 && p < nz) return in + int64_t(p) * plane;
    if (p < 0) return lo + int64_t(p + 2) * plane;
    return hi + int64_t(p - nz) * plane;
  }
};

// Every two-kernel launch walks ZC consecutive planes per block (blockIdx.z = plane chunk):
// one point per thread and plane, x / y neighbours through L1, the plane k+1 loads of one
// iteration re-read from L1 as plane k's centre in the next.  (One block per plane meant
// 1.8 M blocks of 256 points for C4, and block scheduling, not HBM, bounded the kernels.)
constexpr int TWO_ZC = 16;

// Kernel A: D on local planes [-1, nz] (index shifted by +1 in the D buffer).
template <int DIMS, typename R>
__global__ void __launch_bounds__(256) two_d_kernel(PlaneView<R> T, cplx<R> *__restrict__ D, const StageParams<R> P) {
  // 3D blocks cover 32 x 8 points of a plane, 1D/2D blocks 256 points of a row
  const int gx = DIMS == 3 ? blockIdx.x * 32 + (threadIdx.x & 31) : blockIdx.x * 256 + threadIdx.x;
  const int gy = DIMS == 3 ? blockIdx.y * 8 + (threadIdx.x >> 5) : 0;
  if (gx >= P.nx || gy >= P.ny) return;
  const int z_begin = DIMS >= 2 ? int(blockIdx.z) * TWO_ZC - 1 : 0;
  const int z_end = DIMS >= 2 ? min(z_begin + TWO_ZC, P.nz + 1) : 1;
  const int o = gy * int(P.pitch) + gx;  // in-plane offset (a plane has < 2^31 elements)
  const int pitch = int(P.pitch);
  const bool xy_bnd = gx == 0 || gx == P.nx - 1 || (DIMS == 3 && (gy == 0 || gy == P.ny - 1));
  cplx<R> *Dp = D + (DIMS >= 2 ? int64_t(z_begin + 1) * P.plane : 0) + o;
  // z register queue: the centre column at planes lz-1, lz, lz+1 (plane lz+1 is the only new
  // centre load per plane; planes beyond a global face read a valid buffer and go unused)
  cplx<R> cm = DIMS >= 2 ? T(z_begin - 1)[o] : mk<R>(R(0), R(0)), c0 = T(DIMS >= 2 ? z_begin : 0)[o];
  for (int lz = z_begin; lz < z_end; ++lz, Dp += (DIMS >= 2 ? P.plane : 0)) {
    const cplx<R> cp = DIMS >= 2 ? T(lz + 1)[o] : c0;
    const int gz = P.z0 + lz;
    const cplx<R> *pl = T(DIMS >= 2 ? lz : 0) + o;
    const cplx<R> c = c0;
    if (!(DIMS >= 2 && (gz < 0 || gz >= P.NZ))) {  // beyond a global face: never read
      cplx<R> d;
      if (xy_bnd || (DIMS >= 2 && (gz == 0 || gz == P.NZ - 1))) {
        d = lambda_b(P, c, potential(P, gx, gy, lz));
      } else {
        d = d2(pl[-1], c, pl[1], P.ihx2);
        if (DIMS == 3) d = d + d2(pl[-pitch], c, pl[pitch], P.ihy2);
        if (DIMS >= 2) d = d + d2(cm, c, cp, P.ihz2);
      }
      *Dp = d;
    }
    cm = c0;
    c0 = cp;
  }
}

// Output of kernel B at local index g: L (MODE 5) or the Psi-space RK4 stage combine.
template <typename R, int MODE>
__device__ __forceinline__ void two_store(const StageParams<R> &P, int64_t g, cplx<R> c, cplx<R> L, cplx<R> F,
                                          const cplx<R> *__restrict__ psi, const cplx<R> *__restrict__ acc) {
  if (MODE == M_LAP) {
    P.out_T[g] = L;
  } else if (MODE == M_S1) {
    P.out_acc[g] = axpy(c, P.ca, F);
    P.out_T[g] = axpy(c, P.cb, F);
  } else if (MODE == M_S2 || MODE == M_S3) {
    P.out_acc[g] = axpy(acc[g], P.ca, F);
    P.out_T[g] = axpy(psi[g], P.cb, F);
  } else {
    P.out_T[g] = axpy(acc[g], P.cb, F);
  }
}

// Kernel B: step 2 + F + stage combine (MODE 1-4) or L (MODE 5) on local planes [0, nz).
template <int DIMS, typename R, int MODE>
__global__ void __launch_bounds__(256, 4) two_step2_kernel(PlaneView<R> T, const cplx<R> *__restrict__ D,
                                                         const cplx<R> *__restrict__ psi,
                                                         const cplx<R> *__restrict__ acc, const StageParams<R> P,
                                                         const TwoParams<R> Q) {
  // 3D blocks cover 32 x 8 points of a plane, 1D/2D blocks 256 points of a row
  const int gx = DIMS == 3 ? blockIdx.x * 32 + (threadIdx.x & 31) : blockIdx.x * 256 + threadIdx.x;
  const int gy = DIMS == 3 ? blockIdx.y * 8 + (threadIdx.x >> 5) : 0;
  if (gx >= P.nx || gy >= P.ny) return;
  const int o = gy * int(P.pitch) + gx;  // in-plane offset (a plane has < 2^31 elements)
  const int pitch = int(P.pitch);
  const bool xy_bnd = gx == 0 || gx == P.nx - 1 || (DIMS == 3 && (gy == 0 || gy == P.ny - 1));
  const int z_begin = DIMS >= 2 ? int(blockIdx.z) * TWO_ZC : 0;
  const int z_end = DIMS >= 2 ? min(z_begin + TWO_ZC, P.nz) : 1;
  const int64_t dz = DIMS >= 2 ? P.plane : 0;
  const cplx<R> *Dc = D + (DIMS >= 2 ? int64_t(z_begin + 1) * P.plane : 0) + o;
  int64_t g = int64_t(z_begin) * P.plane + o;
  const cplx<R> zero = mk<R>(R(0), R(0));
  // z register queues (planes k-1, k, k+1): the Psi centre, the Psi "cross" neighbours
  // (x-1, x+1, y-1, y+1) and the D centre; per plane only plane k+1's centre and cross, plane
  // k's diagonals and D's in-plane neighbours are loaded (14 loads per point instead of 21 in
  // 3D: the L1 pipe is what bounds this kernel).  Boundary threads skip the neighbour loads.
  struct Cross { cplx<R> xm, xp, ym, yp; };
  auto cross_at = [&](const cplx<R> *q) -> Cross {
    if (xy_bnd) return {zero, zero, zero, zero};
    return {q[-1], q[1], DIMS == 3 ? q[-pitch] : zero, DIMS == 3 ? q[pitch] : zero};
  };
  const cplx<R> *q0 = T(z_begin) + o;
  cplx<R> cm = DIMS >= 2 ? T(z_begin - 1)[o] : zero, c0 = q0[0];
  Cross xm_ = DIMS >= 2 ? cross_at(T(z_begin - 1) + o) : Cross{zero, zero, zero, zero}, x0_ = cross_at(q0);
  cplx<R> dm = DIMS >= 2 ? Dc[-dz] : zero, d0 = Dc[0];
  for (int lz = z_begin; lz < z_end; ++lz, Dc += dz, g += dz) {
    const int gz = P.z0 + lz;
    const cplx<R> *pl = T(lz) + o;
    const cplx<R> *zp = DIMS >= 2 ? T(lz + 1) + o : pl;
    const cplx<R> cp = DIMS >= 2 ? zp[0] : zero;
    const Cross xp_ = DIMS >= 2 ? cross_at(zp) : Cross{zero, zero, zero, zero};
    const cplx<R> dp = DIMS >= 2 ? Dc[dz] : zero;
    const cplx<R> c = c0;
    const R V = potential(P, gx, gy, lz);
    const R N = fma(P.s, norm2(c), -V);
    cplx<R> L, F;
    if (!(xy_bnd || (DIMS >= 2 && (gz == 0 || gz == P.NZ - 1)))) {
      cplx<R> sx = Dc[-1] + Dc[1];
      cplx<R> sy = DIMS == 3 ? Dc[-pitch] + Dc[pitch] : zero;
      cplx<R> sz = DIMS >= 2 ? dm + dp : zero;
      if (Q.iso) {
        // -1/12 (sum of 2d D-neighbours - (16 - 2d) D) + 1/(6h^2) (edge-midpoints - 4 p Psi)
        L = R(-1.0 / 12.0) * ((sx + sy + sz) - R(16 - 2 * DIMS) * d0);
        if (DIMS >= 2) {
          // edge midpoints minus 4 Psi per coordinate plane, the centre subtracted per plane
          // (each group of four sums to 4 Psi exactly for a constant field, so L = 0 exactly)
          cplx<R> e = axpy((xm_.xm + xm_.xp) + (xp_.xm + xp_.xp), R(-4), c);
          if (DIMS == 3) {
            e = e + axpy((pl[-pitch - 1] + pl[-pitch + 1]) + (pl[pitch - 1] + pl[pitch + 1]), R(-4), c);
            e = e + axpy((xm_.ym + xm_.yp) + (xp_.ym + xp_.yp), R(-4), c);
          }
          L = L + Q.w2 * e;
        }
      } else {
        L = d0 - R(1.0 / 12.0) * ((sx + sy + sz) - R(2 * DIMS) * d0);
        // sum_{d<e} (h_d^2+h_e^2)/12 delta_d^2 delta_e^2 Psi, each cross difference written as
        // [corners - 2 (face neighbours of both axes) + 4 Psi] / (h_d^2 h_e^2)
        auto cross = [&](cplx<R> corners, cplx<R> fd, cplx<R> fe, R w) {
          return w * ((corners - R(2) * (fd + fe)) + R(4) * c);
        };
        const cplx<R> fx = x0_.xm + x0_.xp;
        if (DIMS >= 2) {
          const cplx<R> fz = cm + cp;
          L = L + cross((xm_.xm + xm_.xp) + (xp_.xm + xp_.xp), fx, fz, Q.cde[1]);
          if (DIMS == 3) {
            const cplx<R> fy = x0_.ym + x0_.yp;
            L = L + cross((pl[-pitch - 1] + pl[-pitch + 1]) + (pl[pitch - 1] + pl[pitch + 1]), fx, fy, Q.cde[0]);
            L = L + cross((xm_.ym + xm_.yp) + (xp_.ym + xp_.yp), fy, fz, Q.cde[2]);
          }
        }
      }
      F = mk<R>(-fma(P.a, L.im, N * c.im), fma(P.a, L.re, N * c.re));
    } else {
      L = lambda_b(P, c, V);
      F = P.bc == 0 ? zero : mk<R>(-(N * c.im), N * c.re);
    }
    two_store<R, MODE>(P, g, c, L, F, psi, acc);
    cm = c0;
    c0 = cp;
    xm_ = x0_;
    x0_ = xp_;
    dm = d0;
    d0 = dp;
  }
}

template <int DIMS, typename R>
static cudaError_t launch_two_impl(int stage, const cplx<R> *in, const cplx<R> *lo, const cplx<R> *hi,
                                   const cplx<R> *psi, const cplx<R> *acc, cplx<R> *D, const StageParams<R> &P,
                                   const TwoParams<R> &Q, cudaStream_t st) {
  PlaneView<R> T{in, lo ? lo : in, hi ? hi : in, P.nz, P.plane};
  dim3 blk(256);
  const int bx = DIMS == 3 ? (P.nx + 31) / 32 : (P.nx + 255) / 256;
  dim3 ga(bx, DIMS == 3 ? (P.ny + 7) / 8 : 1, DIMS >= 2 ? (P.nz + 2 + TWO_ZC - 1) / TWO_ZC : 1);
  two_d_kernel<DIMS, R><<<ga, blk, 0, st>>>(T, D, P);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  dim3 gb(bx, DIMS == 3 ? (P.ny + 7) / 8 : 1, DIMS >= 2 ? (P.nz + TWO_ZC - 1) / TWO_ZC : 1);
  switch (stage) {
    case 1: two_step2_kernel<DIMS, R, M_S1><<<gb, blk, 0, st>>>(T, D, psi, acc, P, Q); break;
    case 2: two_step2_kernel<DIMS, R, M_S2><<<gb, blk, 0, st>>>(T, D, psi, acc, P, Q); break;
    case 3: two_step2_kernel<DIMS, R, M_S3><<<gb, blk, 0, st>>>(T, D, psi, acc, P, Q); break;
    case 4: two_step2_kernel<DIMS, R, M_S4><<<gb, blk, 0, st>>>(T, D, psi, acc, P, Q); break;
    default: two_step2_kernel<DIMS, R, M_LAP><<<gb, blk, 0, st>>>(T, D, psi, acc, P, Q); break;
  }
  return cudaGetLastError();
}


// ---------------------------------------------------------------------------------------
// Multi-storage variant ("TWO_KERNEL_MS", variant 3): the paper's per-axis form
// (`2d2shocMs1/2` P:185-200, `3d2shocMs1/2` P:262-280; "2X/3X storage" of Tables 4-5).
// Kernel A stores D_d = delta_d^2 Psi for every axis d (dims fields); at a d-face point b
// that is interior along the other axes it stores the face rule (reading R8)
//     D_d(b) = lambda_b - sum_{e != d} delta_e^2 Psi_b,
// and lambda_b at edge/corner points (never read).  Kernel B:
//     L = sum_d 7/6 D_d - (D_d(+e_d) + D_d(-e_d)) / 12,   L_b = lambda_b.
// D_d for axis d (kernel axes x, y, z) lives at D + d * Dfield.
template <int DIMS, typename R>
__global__ void __launch_bounds__(256) two_dms_kernel(PlaneView<R> T, cplx<R> *__restrict__ D, int64_t Dfield,
                                                      const StageParams<R> P) {
  const int gx = DIMS == 3 ? blockIdx.x * 32 + (threadIdx.x & 31) : blockIdx.x * 256 + threadIdx.x;
  const int gy = DIMS == 3 ? blockIdx.y * 8 + (threadIdx.x >> 5) : 0;
  if (gx >= P.nx || gy >= P.ny) return;
  const int64_t o = int64_t(gy) * P.pitch + gx;
  const int z_begin = DIMS >= 2 ? int(blockIdx.z) * TWO_ZC - 1 : 0;
  const int z_end = DIMS >= 2 ? min(z_begin + TWO_ZC, P.nz + 1) : 1;
  for (int lz = z_begin; lz < z_end; ++lz) {
  const int gz = P.z0 + lz;
  if (DIMS >= 2 && (gz < 0 || gz >= P.NZ)) continue;
  const cplx<R> *pl = T(DIMS >= 2 ? lz : 0);
  const cplx<R> c = pl[o];
  // kernel axes present: x always, y in 3D, z (streamed) in 2D/3D
  const bool fx = gx == 0 || gx == P.nx - 1;
  const bool fy = DIMS == 3 && (gy == 0 || gy == P.ny - 1);
  const bool fz = DIMS >= 2 && (gz == 0 || gz == P.NZ - 1);
  const int nf = int(fx) + int(fy) + int(fz);
  cplx<R> dx = mk<R>(R(0), R(0)), dy = dx, dz = dx;
  if (!fx) dx = d2(pl[o - 1], c, pl[o + 1], P.ihx2);
  if (DIMS == 3 && !fy) dy = d2(pl[o - P.pitch], c, pl[o + P.pitch], P.ihy2);
  if (DIMS >= 2 && !fz) dz = d2(T(lz - 1)[o], c, T(lz + 1)[o], P.ihz2);
  cplx<R> lam = mk<R>(R(0), R(0));
  if (nf) lam = lambda_b(P, c, potential(P, gx, gy, lz));
  // face rule on a single face; lambda_b on edges/corners (never read)
  if (fx) dx = nf == 1 ? (lam - dy) - dz : lam;
  if (fy) dy = nf == 1 ? (lam - dx) - dz : lam;
  if (fz) dz = nf == 1 ? (lam - dx) - dy : lam;
  const int64_t g = (int64_t(DIMS >= 2 ? lz + 1 : 0)) * P.plane + o;
  D[g] = dx;
  if (DIMS == 3) D[Dfield + g] = dy;
  if (DIMS >= 2) D[(DIMS - 1) * Dfield + g] = dz;
  }
}

template <int DIMS, typename R, int MODE>
__global__ void __launch_bounds__(256) two_step2ms_kernel(PlaneView<R> T, const cplx<R> *__restrict__ D,
                                                          int64_t Dfield, const cplx<R> *__restrict__ psi,
                                                          const cplx<R> *__restrict__ acc, const StageParams<R> P) {
  const int gx = DIMS == 3 ? blockIdx.x * 32 + (threadIdx.x & 31) : blockIdx.x * 256 + threadIdx.x;
  const int gy = DIMS == 3 ? blockIdx.y * 8 + (threadIdx.x >> 5) : 0;
  if (gx >= P.nx || gy >= P.ny) return;
  const int64_t o = int64_t(gy) * P.pitch + gx;
  const int z_end = DIMS >= 2 ? min(int(blockIdx.z + 1) * TWO_ZC, P.nz) : 1;
  for (int lz = DIMS >= 2 ? int(blockIdx.z) * TWO_ZC : 0; lz < z_end; ++lz) {
  const int gz = P.z0 + lz;
  const cplx<R> c = T(lz)[o];
  const bool bnd = gx == 0 || gx == P.nx - 1 || (DIMS == 3 && (gy == 0 || gy == P.ny - 1)) ||
                   (DIMS >= 2 && (gz == 0 || gz == P.NZ - 1));
  const R V = potential(P, gx, gy, lz);
  const R N = fma(P.s, norm2(c), -V);
  cplx<R> L, F;
  if (!bnd) {
    const int64_t dzs = DIMS >= 2 ? P.plane : 0;
    const cplx<R> *Dx = D + (DIMS >= 2 ? int64_t(lz + 1) * P.plane : 0) + o;
    const R w0 = R(7.0 / 6.0), w1 = R(1.0 / 12.0);
    L = w0 * Dx[0] - w1 * (Dx[-1] + Dx[1]);
    if (DIMS == 3) {
      const cplx<R> *Dy = Dx + Dfield;
      L = L + (w0 * Dy[0] - w1 * (Dy[-P.pitch] + Dy[P.pitch]));
    }
    if (DIMS >= 2) {
      const cplx<R> *Dz = Dx + (DIMS - 1) * Dfield;
      L = L + (w0 * Dz[0] - w1 * (Dz[-dzs] + Dz[dzs]));
    }
    F = mk<R>(-fma(P.a, L.im, N * c.im), fma(P.a, L.re, N * c.re));
  } else {
    L = lambda_b(P, c, V);
    F = P.bc == 0 ? mk<R>(R(0), R(0)) : mk<R>(-(N * c.im), N * c.re);
  }
  two_store<R, MODE>(P, int64_t(lz) * P.plane + o, c, L, F, psi, acc);
  }
}

template <int DIMS, typename R>
static cudaError_t launch_two_ms_impl(int stage, const cplx<R> *in, const cplx<R> *lo, const cplx<R> *hi,
                                      const cplx<R> *psi, const cplx<R> *acc, cplx<R> *D, int64_t Dfield,
                                      const StageParams<R> &P, cudaStream_t st) {
  PlaneView<R> T{in, lo ? lo : in, hi ? hi : in, P.nz, P.plane};
  dim3 blk(256);
  const int bx = DIMS == 3 ? (P.nx + 31) / 32 : (P.nx + 255) / 256;
  dim3 ga(bx, DIMS == 3 ? (P.ny + 7) / 8 : 1, DIMS >= 2 ? (P.nz + 2 + TWO_ZC - 1) / TWO_ZC : 1);
  two_dms_kernel<DIMS, R><<<ga, blk, 0, st>>>(T, D, Dfield, P);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  dim3 gb(bx, DIMS == 3 ? (P.ny + 7) / 8 : 1, DIMS >= 2 ? (P.nz + TWO_ZC - 1) / TWO_ZC : 1);
  switch (stage) {
    case 1: two_step2ms_kernel<DIMS, R, M_S1><<<gb, blk, 0, st>>>(T, D, Dfield, psi, acc, P); break;
    case 2: two_step2ms_kernel<DIMS, R, M_S2><<<gb, blk, 0, st>>>(T, D, Dfield, psi, acc, P); break;
    case 3: two_step2ms_kernel<DIMS, R, M_S3><<<gb, blk, 0, st>>>(T, D, Dfield, psi, acc, P); break;
    case 4: two_step2ms_kernel<DIMS, R, M_S4><<<gb, blk, 0, st>>>(T, D, Dfield, psi, acc, P); break;
    default: two_step2ms_kernel<DIMS, R, M_LAP><<<gb, blk, 0, st>>>(T, D, Dfield, psi, acc, P); break;
  }
  return cudaGetLastError();
}

}  // namespace nlse
