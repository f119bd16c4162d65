// stage_pair.cuh — temporal blocking: two RK4 stages per pass over HBM.
//
// The four stage launches of one step (stage_stream.cuh) move 12-13 field transfers per
// point-step.  Here one launch runs a PAIR of stages over a (column, z-chunk) tile:
//
//   pair A (stages 1+2):  reads Psi (halo 4)                -> writes acc, T_B
//   pair B (stages 3+4):  reads T_B (halo 4), Psi (halo 2), acc -> writes Psi^{n+1}
//
// 7 field transfers per point-step plus the wider halos.  Inside a pair, phase A evaluates
// the first stage on the tile grown by the 2-cell stencil radius (the "extended" region) for
// plane j and keeps the result T_mid in a 5-plane shared-memory ring; phase B evaluates the
// second stage on the tile for plane k = j - 2 from that ring, exactly like the single-stage
// kernel evaluates it from T planes in HBM.  Every formula is the one of stage_stream.cuh:
// the 5-point-per-axis wide form of the 2SHOC Laplacian, the ghost-value form of
// the boundary rule (R8/R9) applied to each phase's own input, the Psi_t boundary
// rule, and the reconstructed-accumulator stage combines:
//   phase A of pair A:  T_A  = Psi + k/2 F(Psi)
//   phase B of pair A:  acc  = Psi + (T_A - Psi)/3 + k/3 F(T_A),   T_B = Psi + k/2 F(T_A)
//   phase A of pair B:  T_A' = Psi + k F(T_B)
//   phase B of pair B:  Psi' = acc + (T_A' - Psi)/3 + k/6 F(T_A')
// Psi' cannot overwrite Psi in place (neighbouring tiles still read Psi's halo), so the
// driver ping-pongs Psi between the caller's buffer and the T_A workspace.
// Single-slab (unsharded) handles only.
#pragma once
#include "stage_stream.cuh"

namespace nlse {

enum PairKind { PAIR_A = 0, PAIR_B = 1 };

// W_IN: input slot row (x0-4 ...), W_EX: mid / Psi-ext slot row (x0-2 ...); rings: RI input
// planes (5 pinned + prefetch), 5 mid planes, RPS Psi-ext planes and RA acc tiles (pair B).
template <int DIMS, typename R> struct PCfg;
// 3D complex64 tiles: 60 x 16, 15 consumer warps x 1 row (16 warps, 128 registers).  Sweep
// (C4 768^3 ms per step, one B200): 64 x 16 / 8 warps x 2 rows (168 registers) 18.5;
// 60 x 16 / 15 x 1 13.5 (kept); 48 x 20 / 15 x 1 14.7.  The per-stage kernels take 8.8:
// DESIGN.md §6 says why the pairs lose.
template <> struct PCfg<3, float> {
  static constexpr int TX = 60, TY = 16, PPX = 2, RPW = 1, NCW = 15;
  static constexpr int W_IN = 68, NBOX_IN = 1, W_EX = 64, NBOX_EX = 1, NBOXP = 1;
  static constexpr int RI_A = 9, RI_B = 7, RPS = 4, RA = 2;
};
template <> struct PCfg<3, double> {
  static constexpr int TX = 32, TY = 16, PPX = 1, RPW = 2, NCW = 8;
  static constexpr int W_IN = 40, NBOX_IN = 1, W_EX = 36, NBOX_EX = 1, NBOXP = 1;
  static constexpr int RI_A = 8, RI_B = 6, RPS = 4, RA = 2;
};
template <> struct PCfg<2, float> {
  static constexpr int TX = 1024, TY = 1, PPX = 4, RPW = 1, NCW = 8;
  static constexpr int W_IN = 1040, NBOX_IN = 5, W_EX = 1040, NBOX_EX = 5, NBOXP = 4;
  static constexpr int RI_A = 16, RI_B = 10, RPS = 6, RA = 4;
};
template <> struct PCfg<2, double> {
  static constexpr int TX = 512, TY = 1, PPX = 2, RPW = 1, NCW = 8;
  static constexpr int W_IN = 520, NBOX_IN = 5, W_EX = 520, NBOX_EX = 5, NBOXP = 4;
  static constexpr int RI_A = 16, RI_B = 10, RPS = 6, RA = 4;
};

template <int DIMS, typename R> struct PLayout {
  using C = PCfg<DIMS, R>;
  static constexpr int HI = DIMS == 3 ? 4 : 0, HE = DIMS == 3 ? 2 : 0;  // y-halo rows of input / ext slots
  static constexpr int IROWS = C::TY + 2 * HI, EROWS = C::TY + 2 * HE;
  static constexpr int ISLOT = C::W_IN * IROWS, ESLOT = C::W_EX * EROWS, PTILE = C::TX * C::TY;
  static constexpr int EPC = sizeof(cplx<R>) / 8;
  static constexpr int BW_IN = C::W_IN * EPC / C::NBOX_IN, BW_EX = C::W_EX * EPC / C::NBOX_EX;
  static constexpr int BWP = C::TX * EPC / C::NBOXP;
  static constexpr uint32_t ISLOT_B = ISLOT * sizeof(cplx<R>), ESLOT_B = ESLOT * sizeof(cplx<R>);
  static constexpr uint32_t PTILE_B = PTILE * sizeof(cplx<R>);
  static constexpr int NTHREADS = (C::NCW + 1) * 32;
  static constexpr int RM = 5;
  static constexpr int EXW = C::TX + 4, EXH = DIMS == 3 ? C::TY + 4 : 1;  // extended region
  static constexpr int NTASK_A = (EXW / C::PPX) * EXH;
  static_assert(C::W_IN >= C::TX + 8 && C::W_EX >= C::TX + 4, "slot widths");
  static_assert(EXW % C::PPX == 0, "extended row split");
  static_assert(BW_IN <= 256 && BW_EX <= 256 && BWP <= 256, "TMA box inner extent");
  static_assert(C::W_IN * EPC % C::NBOX_IN == 0 && C::W_EX * EPC % C::NBOX_EX == 0 && C::TX * EPC % C::NBOXP == 0, "box split");
  static_assert(ISLOT_B % 128 == 0 && ESLOT_B % 128 == 0 && PTILE_B % 128 == 0, "128-byte aligned slots");
  static_assert((BW_IN * 8) % 128 == 0 || C::NBOX_IN == 1, "input sub-boxes 128-byte aligned");
  static_assert((BW_EX * 8) % 128 == 0 || C::NBOX_EX == 1, "ext sub-boxes 128-byte aligned");
  static_assert((BWP * 8) % 128 == 0 || C::NBOXP == 1, "acc sub-boxes 128-byte aligned");
  static_assert((C::TX / C::PPX) * (C::TY / C::RPW) == C::NCW * 32, "thread map");
  static_assert((C::W_IN * sizeof(cplx<R>)) % 16 == 0 && (C::W_EX * sizeof(cplx<R>)) % 16 == 0, "16-byte rows");
  template <int PAIR> __host__ __device__ static constexpr int ri() { return PAIR == PAIR_A ? C::RI_A : C::RI_B; }
  template <int PAIR> __host__ __device__ static constexpr int rps() { return PAIR == PAIR_A ? 0 : C::RPS; }
  template <int PAIR> __host__ __device__ static constexpr int ra() { return PAIR == PAIR_A ? 0 : C::RA; }
  template <int PAIR> __host__ __device__ static constexpr size_t smem_bytes() {
    return size_t(ri<PAIR>()) * ISLOT_B + size_t(RM + rps<PAIR>()) * ESLOT_B + size_t(ra<PAIR>()) * PTILE_B +
           size_t(2 * (ri<PAIR>() + rps<PAIR>() + ra<PAIR>())) * 8;
  }
};

template <typename R, int N>
__device__ __forceinline__ void sts_run(cplx<R> *p, const cplx<R> *v) {
  using VV = V16<R>;
  static_assert(N % VV::CPV == 0, "run");
#pragma unroll
  for (int i = 0; i < N / VV::CPV; ++i) reinterpret_cast<typename VV::T *>(p)[i] = VV::join(v + i * VV::CPV);
}

template <int DIMS, typename R, int PAIR>
__global__ void __launch_bounds__(PLayout<DIMS, R>::NTHREADS, 1)
    pair_stream_kernel(const __grid_constant__ CUtensorMap tm_in, const __grid_constant__ CUtensorMap tm_ps,
                       const __grid_constant__ CUtensorMap tm_acc, const StageParams<R> P) {
  using C = PCfg<DIMS, R>;
  using LY = PLayout<DIMS, R>;
  using CT = cplx<R>;
  constexpr int TX = C::TX, TY = C::TY, WI = C::W_IN, WE = C::W_EX, HI = LY::HI, HE = LY::HE;
  constexpr int RI = LY::template ri<PAIR>(), RPS = LY::template rps<PAIR>(), RA = LY::template ra<PAIR>();
  constexpr int RM = LY::RM, PPX = C::PPX, RPW = C::RPW, NT = C::NCW * 32;
  constexpr int RPSM = RPS > 0 ? RPS : 1, RAM = RA > 0 ? RA : 1;
  constexpr bool B = PAIR == PAIR_B;
  constexpr int kAU = 8;  // unroll of phase A's task loop

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  CT *iring = reinterpret_cast<CT *>(smem_raw);
  CT *mring = reinterpret_cast<CT *>(smem_raw + size_t(RI) * LY::ISLOT_B);
  CT *sring = reinterpret_cast<CT *>(smem_raw + size_t(RI) * LY::ISLOT_B + size_t(RM) * LY::ESLOT_B);
  CT *aring = reinterpret_cast<CT *>(smem_raw + size_t(RI) * LY::ISLOT_B + size_t(RM + RPS) * LY::ESLOT_B);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + size_t(RI) * LY::ISLOT_B + size_t(RM + RPS) * LY::ESLOT_B +
                                                size_t(RA) * LY::PTILE_B);
  uint64_t *fullI = bars, *emptyI = bars + RI, *fullS = bars + 2 * RI, *emptyS = fullS + RPS, *fullA = emptyS + RPS,
           *emptyA = fullA + RA;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < RI; ++i) {
      mbar_init(&fullI[i], 1);
      mbar_init(&emptyI[i], C::NCW);
    }
    for (int i = 0; i < RPS; ++i) {
      mbar_init(&fullS[i], 1);
      mbar_init(&emptyS[i], C::NCW);
    }
    for (int i = 0; i < RA; ++i) {
      mbar_init(&fullA[i], 1);
      mbar_init(&emptyA[i], C::NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  const int G = gridDim.x;
  const int chunk_len = (P.nz + P.nchunk - 1) / P.nchunk;
  const int ncol = P.ncx * P.ncy;

  if (warp == C::NCW) {
    // ------------------------------------------------------------------ producer warp
    if (lane == 0) {
      prefetch_tmap(&tm_in);
      if (B) {
        prefetch_tmap(&tm_ps);
        prefetch_tmap(&tm_acc);
      }
      const uint64_t pol_keep = policy_evict_last(), pol_stream = policy_evict_first();
      uint32_t icnt = 0, scnt = 0, acnt = 0;
      for (int t = blockIdx.x; t < P.ntiles; t += G) {
        const int chunk = t / ncol, col = t % ncol;
        const int x0 = (col % P.ncx) * TX, y0 = (col / P.ncx) * TY;
        const int kb = chunk * chunk_len, ke = min(P.nz, kb + chunk_len);
        auto produceI = [&](int p) {
          const uint32_t slot = icnt % RI, par = (icnt / RI) & 1;
          mbar_wait_backoff(&emptyI[slot], par ^ 1);
          if (p >= 0 && p < P.nz) {
            mbar_arrive_expect_tx(&fullI[slot], LY::ISLOT_B);
            char *dst = reinterpret_cast<char *>(iring + size_t(slot) * LY::ISLOT);
#pragma unroll
            for (int b = 0; b < C::NBOX_IN; ++b) {
              const int c0 = (x0 - 4) * LY::EPC + b * LY::BW_IN;
              if (DIMS == 3) tma_load_3d_hint(dst + b * LY::BW_IN * 8, &tm_in, &fullI[slot], c0, y0 - 4, p, pol_keep);
              else tma_load_2d_hint(dst + b * LY::BW_IN * 8, &tm_in, &fullI[slot], c0, p, pol_keep);
            }
          } else {
            mbar_arrive(&fullI[slot]);
          }
          ++icnt;
        };
        auto produceS = [&](int p) {
          const uint32_t slot = scnt % RPSM, par = (scnt / RPSM) & 1;
          mbar_wait_backoff(&emptyS[slot], par ^ 1);
          if (p >= 0 && p < P.nz) {
            mbar_arrive_expect_tx(&fullS[slot], LY::ESLOT_B);
            char *dst = reinterpret_cast<char *>(sring + size_t(slot) * LY::ESLOT);
#pragma unroll
            for (int b = 0; b < C::NBOX_EX; ++b) {
              const int c0 = (x0 - 2) * LY::EPC + b * LY::BW_EX;
              if (DIMS == 3) tma_load_3d_hint(dst + b * LY::BW_EX * 8, &tm_ps, &fullS[slot], c0, y0 - 2, p, pol_keep);
              else tma_load_2d_hint(dst + b * LY::BW_EX * 8, &tm_ps, &fullS[slot], c0, p, pol_keep);
            }
          } else {
            mbar_arrive(&fullS[slot]);
          }
          ++scnt;
        };
        auto produceA = [&](int p) {
          const uint32_t slot = acnt % RAM, par = (acnt / RAM) & 1;
          mbar_wait_backoff(&emptyA[slot], par ^ 1);
          mbar_arrive_expect_tx(&fullA[slot], LY::PTILE_B);
          char *dst = reinterpret_cast<char *>(aring + size_t(slot) * LY::PTILE);
#pragma unroll
          for (int b = 0; b < C::NBOXP; ++b) {
            const int c0 = x0 * LY::EPC + b * LY::BWP;
            if (DIMS == 3) tma_load_3d_hint(dst + b * LY::BWP * 8, &tm_acc, &fullA[slot], c0, y0, p, pol_stream);
            else tma_load_2d_hint(dst + b * LY::BWP * 8, &tm_acc, &fullA[slot], c0, p, pol_stream);
          }
          ++acnt;
        };
        for (int p = kb - 4; p < kb; ++p) produceI(p);
        for (int j = kb - 2; j < ke + 2; ++j) {
          produceI(j + 2);
          if (B) {
            produceS(j);
            if (j - 2 >= kb) produceA(j - 2);
          }
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------------- consumer warps
  const int ct = threadIdx.x;
  constexpr int CPT = TX / PPX;
  const int cg = ct % CPT, rg = ct / CPT;
  const int lx0 = cg * PPX, ly0 = rg * RPW;  // phase-B points of this thread (tile-relative)
  const CT zero = mk<R>(R(0), R(0));
  const R cx = P.cx, cy = P.cy, cz = P.cz, pa_ = P.a, ps_ = P.s;
  const R c16x = P.c1x, c16y = P.c1y, c16z = P.c1z, cA = P.cA, ca = P.ca, cb = P.cb;
  const int nx = P.nx, ny = P.ny, nz = P.nz, NZ = P.NZ, z0 = P.z0;
  uint32_t icnt = 0, scnt = 0, acnt = 0, mcnt = 0;

  for (int t = blockIdx.x; t < P.ntiles; t += G) {
    const int chunk = t / ncol, col = t % ncol;
    const int x0 = (col % P.ncx) * TX, y0 = (col / P.ncx) * TY;
    const int kb = chunk * chunk_len, ke = min(nz, kb + chunk_len);
    const uint32_t ib = icnt, sb = scnt, ab = acnt, mb = mcnt;  // counters of planes kb-4, kb-2, kb, kb-2
    // Ring positions advance by one slot per plane iteration (no divisions in the plane loop):
    // jc = current plane j; bI = input slot of plane jc-2; sJ = Psi slot of plane jc; mJ = mid
    // slot of plane jc; (s4, par4) = input slot and phase of plane jc+2; sPar = phase of sJ.
    int jc = kb - 2;
    int bI = int(ib % RI), sJ = int(sb % RPSM), mJ = int(mb % RM);
    int s4 = int((ib + 4) % RI);
    uint32_t par4 = ((ib + 4) / RI) & 1u, sPar = (sb / RPSM) & 1u;
    auto islot = [&](int p) -> CT * {  // p in [jc-2, jc+2]
      int q = bI + (p - jc + 2);
      q = q >= RI ? q - RI : q;
      return iring + size_t(q) * LY::ISLOT;
    };
    auto sslot = [&](int p) -> CT * {  // p in [jc-2, jc]
      int q = sJ + (p - jc);
      q = q < 0 ? q + RPSM : q;
      return sring + size_t(q) * LY::ESLOT;
    };
    auto aslot = [&](int p) -> CT * { return aring + size_t((ab + uint32_t(p - kb)) % RAM) * LY::PTILE; };
    auto mslot = [&](int p) -> CT * {  // p in [jc-4, jc]
      int q = mJ + (p - jc);
      q = q < 0 ? q + RM : q;
      return mring + size_t(q) * LY::ESLOT;
    };
    auto iwait0 = [&](int p) {  // tile start only
      const uint32_t c = ib + uint32_t(p - kb + 4);
      mbar_wait(&fullI[c % RI], (c / RI) & 1);
    };
    auto irelease = [&](int p) {  // p in [jc-2, jc+1]
      int q = bI + (p - jc + 2);
      q = q >= RI ? q - RI : q;
      if (lane == 0) mbar_arrive(&emptyI[q]);
    };
    auto srelease = [&](int p) {  // p in [jc-2, jc]
      int q = sJ + (p - jc);
      q = q < 0 ? q + RPSM : q;
      if (lane == 0) mbar_arrive(&emptyS[q]);
    };
    // input slot position of tile-relative (lx, ly); ext/mid slot position
    auto ati = [&](CT *s, int lx, int ly) -> CT & { return s[(ly + HI) * WI + lx + 4]; };
    auto atm = [&](CT *s, int lx, int ly) -> CT & { return s[(ly + HE) * WE + lx + 2]; };

    // faces the extended region (phase A) / the tile (phase B) touch
    const bool xlo = x0 == 0;
    const bool xhiA = x0 - 2 <= nx - 2 && nx - 2 < x0 + TX + 2, xhiB = x0 <= nx - 2 && nx - 2 < x0 + TX;
    const bool ylo = DIMS == 3 && y0 == 0;
    const bool yhiA = DIMS == 3 && y0 - 2 <= ny - 2 && ny - 2 < y0 + TY + 2;
    const bool yhiB = DIMS == 3 && y0 <= ny - 2 && ny - 2 < y0 + TY;

    R vxr[PPX], vyr[RPW];
#pragma unroll
    for (int q = 0; q < PPX; ++q) vxr[q] = (P.vkind == 1 && x0 + lx0 + q < nx) ? P.vx[x0 + lx0 + q] : R(0);
#pragma unroll
    for (int r = 0; r < RPW; ++r) vyr[r] = (P.vkind == 1 && P.vy && y0 + ly0 + r < ny) ? P.vy[y0 + ly0 + r] : R(0);

    // phase-A tasks of this thread (tile-constant): input-slot run offset, ext offset and the
    // x/y part of a separable harmonic V
    constexpr int NTA = (LY::NTASK_A + NT - 1) / NT;
    int a_in[NTA], a_ex[NTA];
    R a_v[NTA][PPX];
#pragma unroll
    for (int i = 0; i < NTA; ++i) {
      const int task = min(ct + i * NT, LY::NTASK_A - 1);
      const int ex = (task % (LY::EXW / PPX)) * PPX, ey = task / (LY::EXW / PPX);
      a_in[i] = (ey + HI - HE) * WI + ex;
      a_ex[i] = ey * WE + ex;
      const int gy = y0 - HE + ey;
#pragma unroll
      for (int q = 0; q < PPX; ++q) {
        const int gx = x0 - 2 + ex + q;
        R v = R(0);
        if (P.vkind == 1 && gx >= 0 && gx < nx && gy >= 0 && gy < ny) {
          v = P.vx[gx];
          if (DIMS == 3 && P.vy) v = v + P.vy[gy];
        }
        a_v[i][q] = v;
      }
    }
    // lean planes: no boundary point, no ghost, no array potential in the region a phase covers
    // (every point in [2, n-3]: the ghosts at -1 and n are read by the points 1 and n-2)
    const bool leanA = P.vkind != 2 && x0 - 2 >= 2 && x0 + TX + 2 <= nx - 2 &&
                       (DIMS == 2 || (y0 - 2 >= 2 && y0 + TY + 2 <= ny - 2));
    const bool leanB = P.vkind != 2 && x0 >= 2 && x0 + TX <= nx - 2 && (DIMS == 2 || (y0 >= 2 && y0 + TY <= ny - 2));

    CT qm2[RPW][PPX], qm1[RPW][PPX], qp1[RPW][PPX];
    cplx<R> *outT = P.out_T + int64_t(kb) * P.plane + int64_t(y0 + ly0) * P.pitch + (x0 + lx0);
    cplx<R> *outA = B ? nullptr : P.out_acc + (outT - P.out_T);

    for (int p = kb - 4; p < kb; ++p) iwait0(p);
    for (int j = kb - 2; j < ke + 2; ++j) {
      mbar_wait(&fullI[s4], par4);  // input plane j+2
      if (B) mbar_wait(&fullS[sJ], sPar);  // Psi plane j
      const int gzj = z0 + j;
      const bool jin = j >= 0 && j < nz;
      if (j == kb + 2) {
        // seed phase B's streamed-axis queue (mid planes kb-2, kb-1, kb+1, complete since the
        // last barrier) before phase A below overwrites the slot of plane kb-3
#pragma unroll
        for (int r = 0; r < RPW; ++r) {
          lds_run<R, PPX>(&atm(mslot(kb - 2), lx0, ly0 + r), qm2[r]);
          lds_run<R, PPX>(&atm(mslot(kb - 1), lx0, ly0 + r), qm1[r]);
          lds_run<R, PPX>(&atm(mslot(kb + 1), lx0, ly0 + r), qp1[r]);
        }
      }
      // ================================================================ phase A, plane j
      if (jin && gzj >= 1 && gzj <= NZ - 2) {
        const bool zgl = P.lo_face && gzj == 1, zgh = P.hi_face && gzj == NZ - 2;
        if (xlo || xhiA || ylo || yhiA || zgl || zgh) {
          CT *s0 = islot(j), *sm = islot(j - 1), *sp = islot(j + 1);
          // x faces, rows of the extended region
          for (int task = ct; task < 2 * LY::EXH; task += NT) {
            const bool hi = task >= LY::EXH;
            if (hi ? !xhiA : !xlo) continue;
            const int ly = (task % LY::EXH) - HE, gy = y0 + ly;
            if (DIMS == 3 && (gy < 1 || gy > ny - 2)) continue;
            const int bx = hi ? nx - 1 : 0, lb = bx - x0, n = hi ? -1 : 1;
            const CT cbv = ati(s0, lb, ly), cin = ati(s0, lb + n, ly);
            CT D = lambda_b(P, cbv, potential(P, bx, gy, j));
            D = D - d2(ati(sm, lb, ly), cbv, ati(sp, lb, ly), P.ihz2);
            if (DIMS == 3) D = D - d2(ati(s0, lb, ly - 1), cbv, ati(s0, lb, ly + 1), P.ihy2);
            ati(s0, lb - n, ly) = axpy(R(2) * cbv - cin, P.hx2, D);
          }
          if (DIMS == 3) {
            for (int task = ct; task < 2 * LY::EXW; task += NT) {
              const bool hi = task >= LY::EXW;
              if (hi ? !yhiA : !ylo) continue;
              const int lx = (task % LY::EXW) - 2, gx = x0 + lx;
              if (gx < 1 || gx > nx - 2) continue;
              const int by = hi ? ny - 1 : 0, lb = by - y0, n = hi ? -1 : 1;
              const CT cbv = ati(s0, lx, lb), cin = ati(s0, lx, lb + n);
              CT D = lambda_b(P, cbv, potential(P, gx, by, j));
              D = D - d2(ati(sm, lx, lb), cbv, ati(sp, lx, lb), P.ihz2);
              D = D - d2(ati(s0, lx - 1, lb), cbv, ati(s0, lx + 1, lb), P.ihx2);
              ati(s0, lx, lb - n) = axpy(R(2) * cbv - cin, P.hy2, D);
            }
          }
          // streamed-axis faces: ghost plane -1 (j = 1) / NZ (j = NZ-2) into its ring slot
          if (zgl || zgh) {
            CT *sbp = zgl ? sm : sp, *sg = zgl ? islot(j - 2) : islot(j + 2);
            const int pb = zgl ? j - 1 : j + 1;
            for (int task = ct; task < LY::EXW * LY::EXH; task += NT) {
              const int lx = (task % LY::EXW) - 2, ly = (task / LY::EXW) - HE;
              const int gx = x0 + lx, gy = y0 + ly;
              if (gx < 1 || gx > nx - 2 || (DIMS == 3 && (gy < 1 || gy > ny - 2))) continue;
              const CT cbv = ati(sbp, lx, ly), cin = ati(s0, lx, ly);
              CT D = lambda_b(P, cbv, potential(P, gx, gy, pb));
              D = D - d2(ati(sbp, lx - 1, ly), cbv, ati(sbp, lx + 1, ly), P.ihx2);
              if (DIMS == 3) D = D - d2(ati(sbp, lx, ly - 1), cbv, ati(sbp, lx, ly + 1), P.ihy2);
              ati(sg, lx, ly) = axpy(R(2) * cbv - cin, P.hz2, D);
            }
          }
          fence_proxy_async_smem();  // generic writes to TMA slots precede their refills
          named_bar_sync(1, NT);
        }
      }
      if (jin && leanA && gzj >= 2 && gzj <= NZ - 3) {
        const CT *s0 = islot(j), *sm1 = islot(j - 1), *sm2 = islot(j - 2), *sp1 = islot(j + 1), *sp2 = islot(j + 2);
        const CT *ps = B ? sslot(j) : nullptr;
        CT *md = mslot(j);
        const R vzj = (P.vkind == 1 && P.vz) ? P.vz[z0 + j] : R(0);
#pragma unroll (kAU)
        for (int i = 0; i < NTA; ++i) {
          if (NTA * NT != LY::NTASK_A && ct + i * NT >= LY::NTASK_A) break;  // warp-uniform when possible
          const int o = a_in[i];
          CT run[PPX + 4];
          lds_run<R, PPX + 4>(s0 + o, run);
          CT zm2[PPX], zm1[PPX], zp1[PPX], zp2[PPX];
          lds_run<R, PPX>(sm2 + o + 2, zm2);
          lds_run<R, PPX>(sm1 + o + 2, zm1);
          lds_run<R, PPX>(sp1 + o + 2, zp1);
          lds_run<R, PPX>(sp2 + o + 2, zp2);
          CT ym2[PPX], ym1[PPX], yp1[PPX], yp2[PPX];
          if (DIMS == 3) {
            lds_run<R, PPX>(s0 + o + 2 - 2 * WI, ym2);
            lds_run<R, PPX>(s0 + o + 2 - WI, ym1);
            lds_run<R, PPX>(s0 + o + 2 + WI, yp1);
            lds_run<R, PPX>(s0 + o + 2 + 2 * WI, yp2);
          }
          CT psv[PPX];
          if (B) lds_run<R, PPX>(ps + a_ex[i], psv);
          CT out[PPX];
#pragma unroll
          for (int q = 0; q < PPX; ++q) {
            const CT c = run[q + 2];
            // sum_d (16 (g-1 + g+1 - 2 g0) - (g-2 + g+2 - 2 g0)) / (12 h_d^2)
            CT L = lap_wide<DIMS>(c, c16x, cx, c16y, cy, c16z, cz, run[q + 1], run[q + 3], run[q], run[q + 4],
                                 ym1[q], yp1[q], ym2[q], yp2[q], zm1[q], zp1[q], zm2[q], zp2[q]);
            const R N = fma(ps_, norm2(c), -(a_v[i][q] + vzj));
            const CT tF = axpy(N * c, pa_, L);
            out[q] = B ? iaxpy(psv[q], cA, tF) : iaxpy(c, cA, tF);
          }
          sts_run<R, PPX>(md + a_ex[i], out);
        }
      } else if (jin) {
        const CT *s0 = islot(j), *sm1 = islot(j - 1), *sm2 = islot(j - 2), *sp1 = islot(j + 1), *sp2 = islot(j + 2);
        const CT *ps = B ? sslot(j) : nullptr;
        CT *md = mslot(j);
        const R vzj = (P.vkind == 1 && P.vz) ? P.vz[z0 + j] : R(0);
        const bool zintj = gzj >= 1 && gzj <= NZ - 2;
        for (int task = ct; task < LY::NTASK_A; task += NT) {
          const int ex = (task % (LY::EXW / PPX)) * PPX, ey = task / (LY::EXW / PPX);
          const int lx = ex - 2, ly = ey - HE, gy = y0 + ly;
          if (DIMS == 3 && (gy < 0 || gy >= ny)) continue;
          const int o = (ey + HI - HE) * WI + ex;  // run start (x = gx - 2) in an input slot
          CT run[PPX + 4];
          lds_run<R, PPX + 4>(s0 + o, run);
          CT zm2[PPX], zm1[PPX], zp1[PPX], zp2[PPX];
          lds_run<R, PPX>(sm2 + o + 2, zm2);
          lds_run<R, PPX>(sm1 + o + 2, zm1);
          lds_run<R, PPX>(sp1 + o + 2, zp1);
          lds_run<R, PPX>(sp2 + o + 2, zp2);
          CT ym2[PPX], ym1[PPX], yp1[PPX], yp2[PPX];
          if (DIMS == 3) {
            lds_run<R, PPX>(s0 + o + 2 - 2 * WI, ym2);
            lds_run<R, PPX>(s0 + o + 2 - WI, ym1);
            lds_run<R, PPX>(s0 + o + 2 + WI, yp1);
            lds_run<R, PPX>(s0 + o + 2 + 2 * WI, yp2);
          }
          CT psv[PPX];
          if (B) lds_run<R, PPX>(ps + ey * WE + ex, psv);
          CT out[PPX];
#pragma unroll
          for (int q = 0; q < PPX; ++q) {
            const int gx = x0 + lx + q;
            const CT c = run[q + 2];
            // sum_d (16 (g-1 + g+1 - 2 g0) - (g-2 + g+2 - 2 g0)) / (12 h_d^2)
            CT L = lap_wide<DIMS>(c, c16x, cx, c16y, cy, c16z, cz, run[q + 1], run[q + 3], run[q], run[q + 4],
                                 ym1[q], yp1[q], ym2[q], yp2[q], zm1[q], zp1[q], zm2[q], zp2[q]);
            const bool valid = gx >= 0 && gx < nx;
            R V = R(0);
            if (valid) {
              if (P.vkind == 2) V = potential(P, gx, gy, j);
              else if (P.vkind == 1) V = (P.vx[gx] + (DIMS == 3 && P.vy ? P.vy[gy] : R(0))) + vzj;
            }
            const R N = fma(ps_, norm2(c), -V);
            const bool bnd = gx == 0 || gx == nx - 1 || (DIMS == 3 && (gy == 0 || gy == ny - 1)) || !zintj;
            const CT tF = bnd ? (P.bc == 0 ? zero : N * c) : axpy(N * c, pa_, L);
            out[q] = valid ? (B ? iaxpy(psv[q], cA, tF) : iaxpy(c, cA, tF)) : zero;
          }
          sts_run<R, PPX>(md + ey * WE + ex, out);
        }
      }
      named_bar_sync(1, NT);  // mid plane j complete

      // ================================================================ phase B, plane k
      const int k = j - 2;
      if (k >= kb) {
        const int gz = z0 + k;
        const bool zint = gz >= 1 && gz <= NZ - 2;
        if (zint && (xlo || xhiB || ylo || yhiB)) {
          CT *s0 = mslot(k), *sm = mslot(k - 1), *sp = mslot(k + 1);
          for (int task = ct; task < 2 * TY; task += NT) {
            const bool hi = task >= TY;
            if (hi ? !xhiB : !xlo) continue;
            const int ly = task % TY, gy = y0 + ly;
            if (DIMS == 3 && (gy < 1 || gy > ny - 2)) continue;
            if (gy >= ny) continue;
            const int bx = hi ? nx - 1 : 0, lb = bx - x0, n = hi ? -1 : 1;
            const CT cbv = atm(s0, lb, ly), cin = atm(s0, lb + n, ly);
            CT D = lambda_b(P, cbv, potential(P, bx, gy, k));
            D = D - d2(atm(sm, lb, ly), cbv, atm(sp, lb, ly), P.ihz2);
            if (DIMS == 3) D = D - d2(atm(s0, lb, ly - 1), cbv, atm(s0, lb, ly + 1), P.ihy2);
            atm(s0, lb - n, ly) = axpy(R(2) * cbv - cin, P.hx2, D);
          }
          if (DIMS == 3) {
            for (int task = ct; task < 2 * TX; task += NT) {
              const bool hi = task >= TX;
              if (hi ? !yhiB : !ylo) continue;
              const int lx = task % TX, gx = x0 + lx;
              if (gx < 1 || gx > nx - 2) continue;
              const int by = hi ? ny - 1 : 0, lb = by - y0, n = hi ? -1 : 1;
              const CT cbv = atm(s0, lx, lb), cin = atm(s0, lx, lb + n);
              CT D = lambda_b(P, cbv, potential(P, gx, by, k));
              D = D - d2(atm(sm, lx, lb), cbv, atm(sp, lx, lb), P.ihz2);
              D = D - d2(atm(s0, lx - 1, lb), cbv, atm(s0, lx + 1, lb), P.ihx2);
              atm(s0, lx, lb - n) = axpy(R(2) * cbv - cin, P.hy2, D);
            }
          }
          named_bar_sync(1, NT);
        }
        const bool zg_lo = P.lo_face && gz == 1, zg_hi = P.hi_face && gz == NZ - 2;
        const CT *pa = nullptr;
        if (B) {
          const uint32_t c = ab + uint32_t(k - kb);
          mbar_wait(&fullA[c % RAM], (c / RAM) & 1);
          pa = aslot(k);
        }
        const R vzk = (P.vkind == 1 && P.vz) ? P.vz[z0 + k] : R(0);
        const CT *m0 = &atm(mslot(k), lx0, ly0) - 2, *mp2 = &atm(mslot(k + 2), lx0, ly0);
        auto bloop = [&](auto lean_c) {
          constexpr bool LEAN = decltype(lean_c)::value;
#pragma unroll
        for (int r = 0; r < RPW; ++r) {
          const int gy = y0 + ly0 + r;
          CT run[PPX + 4];
          lds_run<R, PPX + 4>(m0 + r * WE, run);
          CT zp2[PPX];
          lds_run<R, PPX>(mp2 + r * WE, zp2);
          if (!LEAN && (zg_lo || zg_hi)) {
            const CT *sbp = &atm(mslot(zg_lo ? k - 1 : k + 1), lx0, ly0 + r);
#pragma unroll
            for (int q = 0; q < PPX; ++q) {
              const int gx = x0 + lx0 + q;
              if (gx < 1 || gx > nx - 2 || (DIMS == 3 && (gy < 1 || gy > ny - 2))) continue;
              const CT cbv = zg_lo ? qm1[r][q] : qp1[r][q];
              const CT *pb = sbp + q;
              CT D = lambda_b(P, cbv, potential(P, gx, gy, zg_lo ? k - 1 : k + 1));
              D = D - d2(pb[-1], cbv, pb[1], P.ihx2);
              if (DIMS == 3) D = D - d2(pb[-WE], cbv, pb[WE], P.ihy2);
              const CT g = axpy(R(2) * cbv - run[q + 2], P.hz2, D);
              if (zg_lo) qm2[r][q] = g;
              else zp2[q] = g;
            }
          }
          CT ym2[PPX], ym1[PPX], yp1[PPX], yp2[PPX];
          if (DIMS == 3) {
            lds_run<R, PPX>(m0 + r * WE + 2 - 2 * WE, ym2);
            lds_run<R, PPX>(m0 + r * WE + 2 - WE, ym1);
            lds_run<R, PPX>(m0 + r * WE + 2 + WE, yp1);
            lds_run<R, PPX>(m0 + r * WE + 2 + 2 * WE, yp2);
          }
          CT psv[PPX], acv[PPX];
          if (B) {
            lds_run<R, PPX>(&atm(sslot(k), lx0, ly0 + r), psv);
            lds_run<R, PPX>(pa + (ly0 + r) * TX + lx0, acv);
          } else {
            lds_run<R, PPX>(&ati(islot(k), lx0, ly0 + r), psv);
          }
          CT oT[PPX], oA[PPX];
          bool valid[PPX];
#pragma unroll
          for (int q = 0; q < PPX; ++q) {
            const int gx = x0 + lx0 + q;
            const CT c = run[q + 2];
            // sum_d (16 (g-1 + g+1 - 2 g0) - (g-2 + g+2 - 2 g0)) / (12 h_d^2)
            CT L = lap_wide<DIMS>(c, c16x, cx, c16y, cy, c16z, cz, run[q + 1], run[q + 3], run[q], run[q + 4],
                                 ym1[q], yp1[q], ym2[q], yp2[q], qm1[r][q], qp1[r][q], qm2[r][q], zp2[q]);
            valid[q] = LEAN || (gx < nx && gy < ny);
            R V;
            if (!LEAN && P.vkind == 2) V = valid[q] ? potential(P, gx, gy, k) : R(0);
            else V = (vxr[q] + vyr[r]) + vzk;
            const R N = fma(ps_, norm2(c), -V);
            const bool bnd = !LEAN && (gx == 0 || gx == nx - 1 || (DIMS == 3 && (gy == 0 || gy == ny - 1)) || !zint);
            const CT tF = bnd ? (P.bc == 0 ? zero : N * c) : axpy(N * c, pa_, L);
            if (B) {
              oT[q] = iaxpy(axpy(acv[q], R(1.0 / 3.0), c - psv[q]), cb, tF);
            } else {
              oA[q] = iaxpy(axpy(psv[q], R(1.0 / 3.0), c - psv[q]), ca, tF);
              oT[q] = iaxpy(psv[q], cb, tF);
            }
          }
          using VV = V16<R>;
          bool all = true;
#pragma unroll
          for (int q = 0; q < PPX; ++q) all = all && valid[q];
          cplx<R> *oTr = outT + int64_t(r) * P.pitch;
          cplx<R> *oAr = B ? nullptr : outA + int64_t(r) * P.pitch;
          if (all) {
#pragma unroll
            for (int v = 0; v < PPX / VV::CPV; ++v) {
              st_stream(reinterpret_cast<typename VV::T *>(oTr) + v, VV::join(oT + v * VV::CPV));
              if (!B) st_stream(reinterpret_cast<typename VV::T *>(oAr) + v, VV::join(oA + v * VV::CPV));
            }
          } else {
#pragma unroll
            for (int q = 0; q < PPX; ++q) {
              if (!valid[q]) continue;
              oTr[q] = oT[q];
              if (!B) oAr[q] = oA[q];
            }
          }
#pragma unroll
          for (int q = 0; q < PPX; ++q) {
            qm2[r][q] = qm1[r][q];
            qm1[r][q] = run[q + 2];
            qp1[r][q] = zp2[q];
          }
        }
        };
        if (leanB && gz >= 2 && gz <= NZ - 3) bloop(std::true_type{});
        else bloop(std::false_type{});
        outT += P.plane;
        if (!B) outA += P.plane;
        if (B) {
          __syncwarp();
          const uint32_t c = ab + uint32_t(k - kb);
          if (lane == 0) mbar_arrive(&emptyA[c % RAM]);
        }
      }
      // plane j-2 of the input (and of Psi-ext) is no longer read
      __syncwarp();
      irelease(j - 2);
      if (B && j - 2 >= kb - 2) srelease(j - 2);
      // advance the ring positions to plane j+1
      ++jc;
      bI = bI + 1 == RI ? 0 : bI + 1;
      mJ = mJ + 1 == RM ? 0 : mJ + 1;
      if (++s4 == RI) {
        s4 = 0;
        par4 ^= 1u;
      }
      if (++sJ == RPSM) {
        sJ = 0;
        sPar ^= 1u;
      }
    }
    __syncwarp();
    for (int p = ke; p < ke + 4; ++p) irelease(p);
    if (B)
      for (int p = ke; p < ke + 2; ++p) srelease(p);
    icnt += uint32_t(ke - kb + 8);
    scnt += B ? uint32_t(ke - kb + 4) : 0u;
    acnt += B ? uint32_t(ke - kb) : 0u;
    mcnt += uint32_t(ke - kb + 4);
    // the next tile's first phase A overwrites mid slots this tile's last phase B read
    named_bar_sync(1, NT);
  }
}

}  // namespace nlse
