// stage_line.cuh — fused RK4-stage kernel for 1D grids, and the reductions.
//
// 1D has no tile to stage: each thread evaluates one point from five coalesced
// neighbouring loads (L1 serves the overlap), with the face rule of DESIGN.md R8 reduced to
// 1D (D(b) = lambda_b, `dbc_lap` P:402) realised as a ghost value computed in registers:
//   ghost(-1) = h^2 lambda_0 + 2 Psi_0 - Psi_1,   ghost(N) = h^2 lambda_{N-1} + 2 Psi_{N-1} - Psi_{N-2}.
#pragma once
#include "stage_stream.cuh"

namespace nlse {

// MSD boundary (`msdbc_lap`; reading R28): at boundary b with inward
// neighbour q, lambda_b = [Re(D_q / Psi_q) + (N_q - N_b)/a] Psi_b, D_q = delta^2 Psi at q.
template <typename R>
__device__ __forceinline__ cplx<R> msd_lambda(const cplx<R> *__restrict__ Tin, int b, int q, const StageParams<R> &P) {
  using CT = cplx<R>;
  const CT cb = Tin[b], cq = Tin[q], cf = Tin[2 * q - b];
  const CT D = P.ihx2 * ((cb + cf) - R(2) * cq);
  const R nq = norm2(cq);
  const R re = fma(D.re, cq.re, D.im * cq.im) / nq;
  const R Nq = fma(P.s, nq, -potential(P, q, 0, 0)), Nb = fma(P.s, norm2(cb), -potential(P, b, 0, 0));
  return (re + (Nq - Nb) * P.inv_a) * cb;
}

// MSD = false compiles the MSD branches out (handles with another BC).
template <typename R, bool MSD = true>
__device__ __forceinline__ cplx<R> line_lambda(const cplx<R> *__restrict__ Tin, int b, int n, const StageParams<R> &P) {
  if (MSD && P.bc == 2) return msd_lambda(Tin, b, b == 0 ? 1 : n - 2, P);
  return lambda_b(P, Tin[b], potential(P, b, 0, 0));
}

// Interior point i of the 1D stage: the 5-point wide form with ghost values at the ends
// (ghost = h^2 lambda_b + 2 Psi_b - Psi_{b+n}); returns t with F = i t.
template <typename R, bool MSD = true>
__device__ __forceinline__ cplx<R> line_interior(const cplx<R> *__restrict__ Tin, int64_t i, int n,
                                                const StageParams<R> &P, cplx<R> &c, cplx<R> &L) {
  using CT = cplx<R>;
  c = Tin[i];
  const CT m1 = Tin[i - 1], p1 = Tin[i + 1];
  CT m2, p2;
  if (i >= 2) m2 = Tin[i - 2];
  else m2 = axpy(R(2) * m1 - c, P.hx2, line_lambda<R, MSD>(Tin, 0, n, P));
  if (i <= n - 3) p2 = Tin[i + 2];
  else p2 = axpy(R(2) * p1 - c, P.hx2, line_lambda<R, MSD>(Tin, n - 1, n, P));
  L = lap5(R(2) * c, P.c1x, P.cx, m1, p1, m2, p2);  // 2SHOC wide form, or CD (cx = 0)
  const R N = fma(P.s, norm2(c), -potential(P, int(i), 0, 0));
  return axpy(N * c, P.a, L);  // a L + N c
}

// One point of the 1D stage: returns t with F = i t (and L for the Laplacian output).
template <typename R, bool MSD = true>
__device__ __forceinline__ cplx<R> line_point(const cplx<R> *__restrict__ Tin, int64_t i, int n, const StageParams<R> &P,
                                             cplx<R> &c, cplx<R> &L) {
  using CT = cplx<R>;
  if (i != 0 && i != n - 1) return line_interior<R, MSD>(Tin, i, n, P, c, L);
  c = Tin[i];
  L = line_lambda<R, MSD>(Tin, int(i), n, P);
  if (MSD && P.bc == 2) {
    // `msdbc_ut`: Psi_t,b = i Im(Psi_t,q / Psi_q) Psi_b, i.e. t_b = Re(t_q / Psi_q) Psi_b
    const int q = i == 0 ? 1 : n - 2;
    CT cq, Lq;
    const CT tq = line_interior<R, MSD>(Tin, q, n, P, cq, Lq);
    return (fma(tq.re, cq.re, tq.im * cq.im) / norm2(cq)) * c;
  }
  const R N = fma(P.s, norm2(c), -potential(P, int(i), 0, 0));
  return P.bc == 0 ? mk<R>(R(0), R(0)) : N * c;
}

template <typename R, int MODE>
__global__ void __launch_bounds__(256) stage_line_kernel(const cplx<R> *__restrict__ Tin, const cplx<R> *__restrict__ psi,
                                                         const cplx<R> *__restrict__ acc, const cplx<R> *__restrict__ t3,
                                                         const StageParams<R> P) {
  using CT = cplx<R>;
  const int n = P.nx;
  for (int64_t i0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i0 < n; i0 += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = P.rev ? n - 1 - i0 : i0;  // reversed: start on what the last stage wrote last
    CT c, L;
    const CT t = line_point(Tin, i, n, P, c, L);
    if (MODE == M_LAP) {
      P.out_T[i] = L;
    } else if (MODE == M_S1) {
      P.out_acc[i] = iaxpy(c, P.ca, t);
      P.out_T[i] = iaxpy(c, P.cb, t);
    } else if (MODE == M_S1R) {
      P.out_T[i] = iaxpy(c, P.cb, t);
    } else if (MODE == M_S2R) {
      const CT ps = psi[i];
      P.out_acc[i] = iaxpy(axpy(ps, R(1.0 / 3.0), c - ps), P.ca, t);
      P.out_T[i] = iaxpy(ps, P.cb, t);
    } else if (MODE == M_S3R) {
      P.out_T[i] = iaxpy(psi[i], P.cb, t);
    } else if (MODE == M_S4R) {
      P.out_T[i] = iaxpy(axpy(acc[i], R(1.0 / 3.0), c - psi[i]), P.cb, t);
    } else if (MODE == M_S4X) {  // write-light stage 4: acc holds T_A, t3 holds T_B
      const CT ps = psi[i];
      const CT dsum = axpy(acc[i] - ps, R(2), t3[i] - ps) + (c - ps);
      P.out_T[i] = iaxpy(axpy(ps, R(1.0 / 3.0), dsum), P.cb, t);
    } else if (MODE == M_S2Y) {  // carried sum (variant 7): Q = 3 acc - Psi
      const CT ps = psi[i];
      P.out_acc[i] = iaxpy(axpy(c - ps, R(2), ps), P.ca, t);
      P.out_T[i] = iaxpy(ps, P.cb, t);
    } else if (MODE == M_S4Y) {  // Psi' = (Q + T_C + k/2 K4) / 3; a Dirichlet end keeps T_C = Psi_b
      P.out_T[i] = ((i == 0 || i == n - 1) && P.bc == 0) ? c : carry3(acc[i], c, P.cb, t);
    } else if (MODE == M_S2 || MODE == M_S3) {
      P.out_acc[i] = iaxpy(acc[i], P.ca, t);
      P.out_T[i] = iaxpy(psi[i], P.cb, t);
    } else {
      P.out_T[i] = iaxpy(acc[i], P.cb, t);
    }
  }
}

// 1D stage over tiles of 256 * PT points staged in shared memory (coalesced loads, one read
// per point plus a 4-point halo per tile, conflict-free strided reads); the two points at each
// grid end (ghost / MSD rules) go through line_point on global memory.  Same arithmetic as
// stage_line_kernel.
template <typename R, int MODE, int PT>
__global__ void __launch_bounds__(256) line_tile_kernel(const cplx<R> *__restrict__ Tin, const cplx<R> *__restrict__ psi,
                                                        const cplx<R> *__restrict__ acc, const cplx<R> *__restrict__ t3,
                                                        const StageParams<R> P) {
  using CT = cplx<R>;
  constexpr int TILE = 256 * PT;
  __shared__ __align__(16) CT sT[TILE + 8];  // sT[k] = Tin[t0 - 4 + k]
  const int n = P.nx;
  const int64_t t0 = int64_t(P.rev ? gridDim.x - 1 - blockIdx.x : blockIdx.x) * TILE;
  for (int k = threadIdx.x; k < TILE + 8; k += 256) {
    const int64_t g = t0 - 4 + k;
    sT[k] = (g >= 0 && g < n) ? Tin[g] : mk<R>(R(0), R(0));
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < PT; ++q) {
    const int64_t i = t0 + q * 256 + threadIdx.x;
    if (i >= n) break;
    CT c, L, t;
    if (i < 2 || i >= n - 2) {
      t = line_point(Tin, i, n, P, c, L);
    } else {
      const CT *pp = sT + (i - t0 + 4);
      c = pp[0];
      L = lap5(R(2) * c, P.c1x, P.cx, pp[-1], pp[1], pp[-2], pp[2]);
      const R N = fma(P.s, norm2(c), -potential(P, int(i), 0, 0));
      t = axpy(N * c, P.a, L);
    }
    if (MODE == M_LAP) {
      P.out_T[i] = L;
    } else if (MODE == M_S1) {
      P.out_acc[i] = iaxpy(c, P.ca, t);
      P.out_T[i] = iaxpy(c, P.cb, t);
    } else if (MODE == M_S1R) {
      P.out_T[i] = iaxpy(c, P.cb, t);
    } else if (MODE == M_S2R) {
      const CT ps = psi[i];
      P.out_acc[i] = iaxpy(axpy(ps, R(1.0 / 3.0), c - ps), P.ca, t);
      P.out_T[i] = iaxpy(ps, P.cb, t);
    } else if (MODE == M_S3R) {
      P.out_T[i] = iaxpy(psi[i], P.cb, t);
    } else if (MODE == M_S4R) {
      P.out_T[i] = iaxpy(axpy(acc[i], R(1.0 / 3.0), c - psi[i]), P.cb, t);
    } else if (MODE == M_S4X) {  // write-light stage 4: acc holds T_A, t3 holds T_B
      const CT ps = psi[i];
      const CT dsum = axpy(acc[i] - ps, R(2), t3[i] - ps) + (c - ps);
      P.out_T[i] = iaxpy(axpy(ps, R(1.0 / 3.0), dsum), P.cb, t);
    } else if (MODE == M_S2Y) {  // carried sum (variant 7): Q = 3 acc - Psi
      const CT ps = psi[i];
      P.out_acc[i] = iaxpy(axpy(c - ps, R(2), ps), P.ca, t);
      P.out_T[i] = iaxpy(ps, P.cb, t);
    } else if (MODE == M_S4Y) {  // Psi' = (Q + T_C + k/2 K4) / 3; a Dirichlet end keeps T_C = Psi_b
      P.out_T[i] = ((i == 0 || i == n - 1) && P.bc == 0) ? c : carry3(acc[i], c, P.cb, t);
    } else if (MODE == M_S2 || MODE == M_S3) {
      P.out_acc[i] = iaxpy(acc[i], P.ca, t);
      P.out_T[i] = iaxpy(psi[i], P.cb, t);
    } else {
      P.out_T[i] = iaxpy(acc[i], P.cb, t);
    }
  }
}

// Persistent 1D stage: each CTA walks segments of SEG points; one thread prefetches the next
// NS-1 segments (stencil input with a 4-point halo, and the pointwise streams) into a ring of
// shared-memory slots with one contiguous cp.async.bulk per stream, so the whole CTA computes
// from shared memory while the following segments stream in.  Segments touching either end of
// the grid are loaded with plain loads (out-of-range halo entries are never read: the two
// points at each end go through line_point on global memory).  Same arithmetic as
// line_tile_kernel.
// complex64: 512-point segments, 4 ring stages, >= 3 CTAs per SM (C2 c64 0.0994 -> 0.0724
// ms/step against 1024-point segments with one CTA per SM: more loads in flight per SM).
// (complex128 with 512-point segments, 4 stages, 2 CTAs per SM: the same 0.131 ms/step.)
template <typename R> struct LineStream {
  static constexpr int SEG = sizeof(R) == 4 ? 512 : 1024, NS = sizeof(R) == 4 ? 4 : 3, NT = 256;
  static constexpr int MINB = sizeof(R) == 4 ? 3 : 1;  // CTAs per SM (launch bound)
};
template <typename R, int MODE> __host__ __device__ constexpr int line_npa() {
  return MODE == M_S4X ? 3 : ((MODE == M_S4R || MODE == M_S2 || MODE == M_S3 || MODE == M_S4) ? 2 :
                              ((MODE == M_S2R || MODE == M_S3R || MODE == M_S2Y || MODE == M_S4Y) ? 1 : 0));
}
template <typename R, int MODE> __host__ __device__ constexpr size_t line_stream_smem() {
  using LS = LineStream<R>;
  return size_t(LS::NS) * ((LS::SEG + 8) + size_t(line_npa<R, MODE>()) * LS::SEG) * sizeof(cplx<R>) + 8 * LS::NS;
}

template <typename R, int MODE>
__global__ void __launch_bounds__(256, LineStream<R>::MINB) line_stream_kernel(const cplx<R> *__restrict__ Tin, const cplx<R> *__restrict__ psi,
                                                             const cplx<R> *__restrict__ acc, const cplx<R> *__restrict__ t3,
                                                             const StageParams<R> P) {
  using CT = cplx<R>;
  using LS = LineStream<R>;
  constexpr int SEG = LS::SEG, NS = LS::NS, NPA = line_npa<R, MODE>();
  constexpr int SLOT = (SEG + 8) + NPA * SEG;  // complex per ring stage: T (+halo), then the P streams
  extern __shared__ __align__(1024) unsigned char lsm[];
  CT *ring = reinterpret_cast<CT *>(lsm);
  uint64_t *full = reinterpret_cast<uint64_t *>(lsm + size_t(NS) * SLOT * sizeof(CT));
  const int n = P.nx;
  const int nseg = (n + SEG - 1) / SEG;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) mbar_init(&full[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const CT *pstream[3] = {MODE == M_S4Y ? acc : psi, acc, t3};  // M_S4Y streams the carried sum alone
  auto seg_of = [&](int j) { const int sg = blockIdx.x + j * gridDim.x; return P.rev ? nseg - 1 - sg : sg; };
  auto interior = [&](int sg) { return int64_t(sg) * SEG - 4 >= 0 && int64_t(sg + 1) * SEG + 4 <= n; };
  auto issue = [&](int j) {  // thread 0: prefetch segment j into ring stage j % NS
    const int sg = seg_of(j);
    uint64_t *bar = &full[j % NS];
    if (!interior(sg)) {
      mbar_arrive(bar);  // loaded by the whole CTA after the wait
      return;
    }
    CT *slot = ring + size_t(j % NS) * SLOT;
    const uint32_t tb = uint32_t((SEG + 8) * sizeof(CT)), pb = uint32_t(SEG * sizeof(CT));
    mbar_arrive_expect_tx(bar, tb + NPA * pb);
    const uint64_t pol = policy_evict_normal();
    bulk_load_hint(slot, Tin + int64_t(sg) * SEG - 4, tb, bar, pol);
#pragma unroll
    for (int q = 0; q < NPA; ++q) bulk_load_hint(slot + (SEG + 8) + q * SEG, pstream[q] + int64_t(sg) * SEG, pb, bar, pol);
  };
  const int njobs = blockIdx.x < nseg ? (nseg - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  if (threadIdx.x == 0)
    for (int j = 0; j < NS - 1 && j < njobs; ++j) issue(j);
  for (int j = 0; j < njobs; ++j) {
    if (threadIdx.x == 0 && j + NS - 1 < njobs) issue(j + NS - 1);
    const int sg = seg_of(j);
    CT *slot = ring + size_t(j % NS) * SLOT;
    mbar_wait(&full[j % NS], (j / NS) & 1);
    const int64_t t0 = int64_t(sg) * SEG;
    if (!interior(sg)) {  // grid-end segment: plain loads, halo entries outside the grid zeroed
      for (int k = threadIdx.x; k < SEG + 8; k += LS::NT) {
        const int64_t g = t0 - 4 + k;
        slot[k] = (g >= 0 && g < n) ? Tin[g] : mk<R>(R(0), R(0));
      }
      for (int q = 0; q < NPA; ++q)
        for (int k = threadIdx.x; k < SEG; k += LS::NT) {
          const int64_t g = t0 + k;
          slot[(SEG + 8) + q * SEG + k] = g < n ? pstream[q][g] : mk<R>(R(0), R(0));
        }
      __syncthreads();
    }
    const CT *sT = slot, *sP = slot + (SEG + 8);
#pragma unroll
    for (int q = 0; q < SEG / LS::NT; ++q) {
      const int kk = q * LS::NT + threadIdx.x;
      const int64_t i = t0 + kk;
      if (i >= n) break;
      CT c, L, t;
      if (i < 2 || i >= n - 2) {
        t = line_point(Tin, i, n, P, c, L);
      } else {
        const CT *pp = sT + kk + 4;
        c = pp[0];
        L = lap5(R(2) * c, P.c1x, P.cx, pp[-1], pp[1], pp[-2], pp[2]);
        const R N = fma(P.s, norm2(c), -potential(P, int(i), 0, 0));
        t = axpy(N * c, P.a, L);
      }
      const CT ps = NPA > 0 ? sP[kk] : c, a1 = NPA > 1 ? sP[SEG + kk] : c, a2 = NPA > 2 ? sP[2 * SEG + kk] : c;
      if (MODE == M_LAP) {
        P.out_T[i] = L;
      } else if (MODE == M_S1R) {
        P.out_T[i] = iaxpy(c, P.cb, t);
      } else if (MODE == M_S2R) {
        P.out_acc[i] = iaxpy(axpy(ps, R(1.0 / 3.0), c - ps), P.ca, t);
        P.out_T[i] = iaxpy(ps, P.cb, t);
      } else if (MODE == M_S3R) {
        P.out_T[i] = iaxpy(ps, P.cb, t);
      } else if (MODE == M_S4R) {
        P.out_T[i] = iaxpy(axpy(a1, R(1.0 / 3.0), c - ps), P.cb, t);
      } else if (MODE == M_S4X) {
        const CT dsum = axpy(a1 - ps, R(2), a2 - ps) + (c - ps);
        P.out_T[i] = iaxpy(axpy(ps, R(1.0 / 3.0), dsum), P.cb, t);
      } else if (MODE == M_S2Y) {
        P.out_acc[i] = iaxpy(axpy(c - ps, R(2), ps), P.ca, t);
        P.out_T[i] = iaxpy(ps, P.cb, t);
      } else if (MODE == M_S4Y) {  // the one pointwise stream is the carried sum Q
        P.out_T[i] = ((i == 0 || i == n - 1) && P.bc == 0) ? c : carry3(ps, c, P.cb, t);
      } else if (MODE == M_S1) {
        P.out_acc[i] = iaxpy(c, P.ca, t);
        P.out_T[i] = iaxpy(c, P.cb, t);
      } else if (MODE == M_S2 || MODE == M_S3) {
        P.out_acc[i] = iaxpy(a1, P.ca, t);
        P.out_T[i] = iaxpy(ps, P.cb, t);
      } else {  // M_S4
        P.out_T[i] = iaxpy(a1, P.cb, t);
      }
    }
    __syncthreads();  // every thread is done with this ring stage before it is refilled
  }
}

// Resident small-grid 1D solver: the whole grid (Psi, T_A, T_B, acc) lives in one CTA's
// shared memory and the CTA runs all nsteps x 4 stages of an nlse2shoc_rk4 call, separated
// by barriers.  Same per-point arithmetic as stage_line_kernel; one launch per call instead
// of 4 per step (C1: 2000 steps on 1024 points is otherwise launch-latency bound).
template <typename R, bool MSD>
__global__ void __launch_bounds__(1024, 1) resident_line_kernel(cplx<R> *__restrict__ psi_g, int64_t nsteps, R dt,
                                                                const StageParams<R> P) {
  using CT = cplx<R>;
  extern __shared__ __align__(16) unsigned char rsm[];
  const int n = P.nx;
  CT *psi = reinterpret_cast<CT *>(rsm), *TA = psi + n, *TB = TA + n, *acc = TB + n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) psi[i] = psi_g[i];
  __syncthreads();
  const R c6 = dt / R(6), c3 = dt / R(3), c2 = dt / R(2);
  for (int64_t step = 0; step < nsteps; ++step) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {  // stage 1
      CT c, L;
      const CT t = line_point<R, MSD>(psi, i, n, P, c, L);
      acc[i] = iaxpy(c, c6, t);
      TA[i] = iaxpy(c, c2, t);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {  // stage 2
      CT c, L;
      const CT t = line_point<R, MSD>(TA, i, n, P, c, L);
      acc[i] = iaxpy(acc[i], c3, t);
      TB[i] = iaxpy(psi[i], c2, t);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {  // stage 3
      CT c, L;
      const CT t = line_point<R, MSD>(TB, i, n, P, c, L);
      acc[i] = iaxpy(acc[i], c3, t);
      TA[i] = iaxpy(psi[i], dt, t);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {  // stage 4
      CT c, L;
      const CT t = line_point<R, MSD>(TA, i, n, P, c, L);
      psi[i] = iaxpy(acc[i], c6, t);
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) psi_g[i] = psi[i];
}

// ---------------------------------------------------------------------------------------
// min / max of N = s|Psi|^2 - V over the local grid (for `kdfull`), and a finiteness scan.
// One partial (min, max, nonfinite-count) triple per block; the host folds them.
template <typename R>
__global__ void __launch_bounds__(256) reduce_N_kernel(const cplx<R> *__restrict__ psi, const StageParams<R> P,
                                                       double *__restrict__ part) {
  // Each warp scans one contiguous range of the (caller-layout, pitch == nx) field, lanes
  // interleaved for coalescing; the (x, y, z) index of its lane advances by 32 per iteration
  // with carries instead of a division per element.
  R lo = R(INFINITY), hi = R(-INFINITY);
  double bad = 0;
  const int64_t total = int64_t(P.nx) * P.ny * P.nz;
  const int64_t nwarps = int64_t(gridDim.x) * (blockDim.x >> 5);
  const int64_t wid = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t chunk = ((total + nwarps - 1) / nwarps + 31) & ~int64_t(31);
  const int64_t q0 = wid * chunk + (threadIdx.x & 31), q1 = min(total, (wid + 1) * chunk);
  if (q0 < q1) {
    int gx = int(q0 % P.nx);
    int64_t r = q0 / P.nx;
    int gy = int(r % P.ny), lz = int(r / P.ny);
    for (int64_t q = q0; q < q1; q += 32) {
      const cplx<R> c = psi[q];
      if (!isfinite(c.re) || !isfinite(c.im)) bad += 1;
      const R N = fma(P.s, norm2(c), -potential(P, gx, gy, lz));
      lo = fmin(lo, N);
      hi = fmax(hi, N);
      gx += 32;
      while (gx >= P.nx) {
        gx -= P.nx;
        if (++gy == P.ny) {
          gy = 0;
          ++lz;
        }
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    bad += __shfl_xor_sync(0xffffffffu, bad, o);
  }
  __shared__ R s[2][8];
  __shared__ double sb[8];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { s[0][w] = lo; s[1][w] = hi; sb[w] = bad; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < int(blockDim.x >> 5); ++i) {
      lo = fmin(lo, s[0][i]);
      hi = fmax(hi, s[1][i]);
      bad += sb[i];
    }
    const int b = blockIdx.x;
    part[3 * b] = double(lo);
    part[3 * b + 1] = double(hi);
    part[3 * b + 2] = bad;
  }
}

// Pitched <-> dense copies are done with cudaMemcpy2DAsync by the host; no kernel needed.

}  // namespace nlse
