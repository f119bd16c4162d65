// nlse2shoc.cu — host runtime of libnlse2shoc.so: the C-ABI declared in include/nlse2shoc.h
// (handle, validation, workspace, TMA descriptors, launch plan, NCCL z-slab halo exchange)
// plus the kernel instantiations.  Product code: shares nothing with oracle/ or icgen/.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "nlse2shoc.h"
#include "stage_line.cuh"
#include "stage_stream.cuh"
#include "two_kernel.cuh"
#include "stage_pair.cuh"

#ifdef NLSE_WITH_NCCL
#include <nccl.h>
#endif

using namespace nlse;

// ------------------------------------------------------------------------------- errors
static thread_local std::string g_last_error;

static nlse2shoc_status fail(nlse2shoc_status st, const std::string &msg) {
  g_last_error = msg;
  return st;
}
#define CUDA_TRY(expr)                                                                        \
  do {                                                                                        \
    cudaError_t e_ = (expr);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      return fail(e_ == cudaErrorMemoryAllocation ? NLSE2SHOC_ENOMEM : NLSE2SHOC_ECUDA,       \
                  std::string(#expr) + ": " + cudaGetErrorString(e_));                        \
  } while (0)
#define TRY(expr)                                \
  do {                                           \
    nlse2shoc_status s_ = (expr);                \
    if (s_ != NLSE2SHOC_OK) return s_;           \
  } while (0)
#ifdef NLSE_WITH_NCCL
#define NCCL_TRY(expr)                                                                               \
  do {                                                                                               \
    ncclResult_t r_ = (expr);                                                                        \
    if (r_ != ncclSuccess) return fail(NLSE2SHOC_ENCCL, std::string(#expr) + ": " + ncclGetErrorString(r_)); \
  } while (0)
#endif

// --------------------------------------------------------------------------- TMA encode
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void *p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// ------------------------------------------------------------------------------ handle
struct Field {  // one pitched field of the local slab (+ its two halo buffers when sharded)
  void *ptr = nullptr;
  void *halo_lo = nullptr, *halo_hi = nullptr;
  CUtensorMap tm{}, tm_lo{}, tm_hi{};  // stencil-input boxes (tile + halo) over the slab / halos
  CUtensorMap tm_pt{};                 // pointwise tile boxes (Psi^n, acc reads)
  CUtensorMap tm_in4{}, tm_ex{}, tm_ppt{};  // stage-pair kernel: halo-4 input, halo-2 Psi, acc tile
};

// z-chunk layout of a stage launch (StageParams nchunk / ns / ls / mlen).
struct ZLayout {
  int nchunk = 1, ns = 0, ls = 0, mlen = 1;
};

struct nlse2shoc_s {
  int dims = 0;
  int64_t N[3] = {1, 1, 1};  // global counts
  double h[3] = {1, 1, 1};
  double a = 1, s = 0;
  nlse2shoc_potential V{};
  int bc = 0, dtype = 0, device = 0, variant = 0, scheme = 0;
  int D_fields = 0;  // D fields allocated for the two-kernel variants
  int rng_b = 0, rng_e = 0;  // plane range of the next stage launch (0, 0: the whole slab)
  int reserve_sms = 0;       // SMs left free for a concurrent NCCL exchange (interior launches)
  cudaStream_t comm_st = nullptr;  // edge-first halo exchange: side stream + events
  cudaStream_t cap_st = nullptr;   // private stream for CUDA-graph capture
  cudaEvent_t ev_edge = nullptr, ev_recv = nullptr;
  nlse2shoc_alloc_fn alloc = nullptr;  // device allocator captured at create (null: cudaMalloc)
  nlse2shoc_free_fn dfree = nullptr;
  void *alloc_ctx = nullptr;
  size_t S = 8;  // bytes per complex
  // slab (streamed axis = dims-1)
  int rank = 0, nranks = 1;
  int64_t z0 = 0, nz = 1;   // local slab along the streamed axis
  int64_t nx = 1, ny = 1;   // kernel view: x, y (3D only; 1 otherwise)
  int64_t NZ = 1;           // global streamed count
  int64_t pitch = 0, plane = 0, local_elems = 0;
  bool sharded = false;
  // workspace
  Field psiw, TA, TB, acc, D;
  void *vtab = nullptr;  // vx | vy | vz tables (precision R)
  size_t vx_off = 0, vy_off = 0, vz_off = 0;
  double *red = nullptr;  // reduction partials (device)
  int red_blocks = 0;
  size_t bytes = 0;
  int num_sms = 148;
  int64_t launches = 0;
  // execution-path options (nlse2shoc_set_option): results are the same up to the rounding
  // differences stated in include/nlse2shoc.h
  int opt_graph = 1, opt_overlap = 1, opt_resident = 1, opt_reverse = 1, opt_lean = 3, opt_zchunks = 0;
  int opt_sched = -1;         // -1: automatic (dynamic)
  int opt_tail = 1;           // option TAIL_CHUNKS
  int opt_check_every = 0;    // option CHECK_EVERY (steps between non-finite scans; 0: none)
  std::map<uint64_t, ZLayout> zmemo;  // z-chunk layouts chosen so far (zlayout_dynamic)
  unsigned *sched = nullptr;  // dynamic tile schedule counters {next tile, finished CTAs}
  // one instantiated RK4-step graph, reused by later calls with the same psi, dt and settings
  // (gen counts set_variant / set_scheme / set_option calls)
  cudaGraphExec_t gexec = nullptr;
  const void *g_psi = nullptr;
  double g_dt = 0.0;
  int g_kind = 0;
  uint64_t gen = 0, g_gen = 0;
  int64_t g_launches = 0;
  // z-slab halos: one cudaMalloc arena (exportable by CUDA IPC) holding, per field role
  // (0 Psi, 1 T_A, 2 T_B, 3 acc), the 2 low and 2 high halo planes, then two arrival counters
  // of the fused exchange: cnt[0] raised by the lower neighbour, cnt[1] by the upper one
  char *arena = nullptr;
  size_t halo_bytes = 0, arena_bytes = 0;
  unsigned long long *cnt = nullptr;
  // fused exchange: the neighbours' halo buffers per role and counters
  void *peer_lo[4] = {}, *peer_hi[4] = {};
  unsigned long long *peer_sig_lo = nullptr, *peer_sig_hi = nullptr;
  void *ipc_lo = nullptr, *ipc_hi = nullptr;  // neighbours' arenas opened by CUDA IPC
  bool peers = false;                          // peer pointers connected
  bool fusing = false;                         // the running rk4 call mirrors edge planes
  int opt_fused = 1;                           // option FUSED_EXCHANGE
  unsigned long long fused_epoch = 0;          // mirrored stage launches so far
  // loopback (single-GPU emulation of z-slab sharding, SURVEY §4 T3'): virtual slabs that
  // exchange halos by device copies instead of NCCL; empty for ordinary handles
  std::vector<nlse2shoc_s *> slabs;
  bool loop_member = false;
  void *Lw = nullptr;  // pitched staging for the Laplacian output (odd-N_x complex64 only)
  bool ws_external = false;  // T_A, T_B, acc live in the caller's workspace (nlse2shoc_set_workspace)
#ifdef NLSE_WITH_NCCL
  ncclComm_t comm = nullptr;
#endif
};

// Device allocator: cudaMalloc, or the caller's (e.g. torch's caching allocator) when set
// through nlse2shoc_set_allocator before create.
static nlse2shoc_alloc_fn g_alloc = nullptr;
static nlse2shoc_free_fn g_free = nullptr;
static void *g_alloc_ctx = nullptr;

template <typename T> static cudaError_t dev_malloc(nlse2shoc_t H, T **p, size_t n) {
  if (H->alloc) {
    int dev = 0;
    cudaGetDevice(&dev);
    void *q = H->alloc(n, dev, H->alloc_ctx);
    *p = reinterpret_cast<T *>(q);
    return q ? cudaSuccess : cudaErrorMemoryAllocation;
  }
  return cudaMalloc(reinterpret_cast<void **>(p), n);
}

static cudaError_t dev_free(nlse2shoc_t H, void *p) {
  if (!p) return cudaSuccess;
  if (H->dfree) {
    int dev = 0;
    cudaGetDevice(&dev);
    H->dfree(p, dev, H->alloc_ctx);
    return cudaSuccess;
  }
  return cudaFree(p);
}

static const char *kErr[] = {"ok", "invalid argument", "out of device memory", "CUDA error", "NCCL error",
                             "non-finite value", "unsupported"};

// ------------------------------------------------------------------------ small helpers
static bool finite_pos(double v) { return std::isfinite(v) && v > 0.0; }

static nlse2shoc_status encode_map(CUtensorMap *tm, void *base, int dims_tensor, uint64_t inner_elems8,
                                   uint64_t rows, uint64_t planes, uint64_t pitch_bytes, uint64_t plane_bytes,
                                   uint32_t box0, uint32_t box1,
                                   CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B) {
  auto enc = get_encode();
  if (!enc) return fail(NLSE2SHOC_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t gdim[3] = {inner_elems8, rows, planes};
  cuuint64_t gstr[2] = {pitch_bytes, plane_bytes};
  cuuint32_t box[3] = {box0, box1, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, dims_tensor, base, gdim, gstr, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(NLSE2SHOC_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
  return NLSE2SHOC_OK;
}

// L2 promotion of the stencil-input (halo) boxes: 64 B, so a halo column's 16-byte row piece
// brings in its whole 64-byte DRAM burst, which the x-neighbour tile's halo read hits in L2
// (C4: 9.75 -> 9.48 ms/step; none and 256 B measured worse).  Pointwise (Psi^n / acc) boxes:
// 256 B.
static CUtensorMapL2promotion tma_promo() { return CU_TENSOR_MAP_L2_PROMOTION_L2_64B; }
static CUtensorMapL2promotion tma_promo_p() { return CU_TENSOR_MAP_L2_PROMOTION_L2_256B; }

template <int DIMS, typename R> struct Maps {
  using LY = Layout<DIMS, R>;
  using C = Cfg<DIMS, R>;
  // stencil-input map (tile + halo box) over a field with `planes` planes
  static nlse2shoc_status stencil(nlse2shoc_t H, CUtensorMap *tm, void *base, int64_t planes) {
    const uint64_t S = sizeof(cplx<R>);
    if (DIMS == 3)
      return encode_map(tm, base, 3, uint64_t(H->nx) * LY::EPC, uint64_t(H->ny), uint64_t(planes), H->pitch * S,
                        H->plane * S, LY::BW, LY::SROWS, tma_promo());
    return encode_map(tm, base, 2, uint64_t(H->nx) * LY::EPC, uint64_t(planes), 1, H->pitch * S, H->pitch * S * planes,
                      LY::BW, 1, tma_promo());
  }
  // pointwise (Psi^n / acc) map: tile box without halo
  static nlse2shoc_status point(nlse2shoc_t H, CUtensorMap *tm, void *base) {
    const uint64_t S = sizeof(cplx<R>);
    if (DIMS == 3)
      return encode_map(tm, base, 3, uint64_t(H->nx) * LY::EPC, uint64_t(H->ny), uint64_t(H->nz), H->pitch * S,
                        H->plane * S, LY::BWP, C::TY, tma_promo_p());
    return encode_map(tm, base, 2, uint64_t(H->nx) * LY::EPC, uint64_t(H->nz), 1, H->pitch * S, H->plane * S * H->nz,
                      LY::BWP, 1, tma_promo_p());
  }
};

// tensor maps of the stage-pair kernel (stage_pair.cuh geometry)
template <int DIMS, typename R> struct PMaps {
  using LY = PLayout<DIMS, R>;
  using C = PCfg<DIMS, R>;
  static nlse2shoc_status enc(nlse2shoc_t H, CUtensorMap *tm, void *base, uint32_t bw, uint32_t rows) {
    const uint64_t S = sizeof(cplx<R>);
    if (DIMS == 3)
      return encode_map(tm, base, 3, uint64_t(H->nx) * LY::EPC, uint64_t(H->ny), uint64_t(H->nz), H->pitch * S,
                        H->plane * S, bw, rows, tma_promo());
    return encode_map(tm, base, 2, uint64_t(H->nx) * LY::EPC, uint64_t(H->nz), 1, H->pitch * S, H->plane * S * H->nz,
                      bw, 1, tma_promo());
  }
  static nlse2shoc_status all(nlse2shoc_t H, Field &f) {
    TRY(enc(H, &f.tm_in4, f.ptr, LY::BW_IN, LY::IROWS));
    TRY(enc(H, &f.tm_ex, f.ptr, LY::BW_EX, LY::EROWS));
    return enc(H, &f.tm_ppt, f.ptr, LY::BWP, C::TY);
  }
};

template <typename R> static void fill_params(nlse2shoc_t H, StageParams<R> &P) {
  std::memset(&P, 0, sizeof(P));
  P.nx = int(H->nx);
  P.ny = int(H->ny);
  P.nz = int(H->nz);
  P.zb = H->rng_e > 0 ? H->rng_b : 0;  // plane range of this launch (edge / interior split)
  P.ze = H->rng_e > 0 ? H->rng_e : int(H->nz);
  P.z0 = int(H->z0);
  P.NZ = int(H->NZ);
  P.lo_face = H->z0 == 0;
  P.hi_face = H->z0 + H->nz == H->NZ;
  P.has_lo_halo = H->dims > 1 && !P.lo_face;
  P.has_hi_halo = H->dims > 1 && !P.hi_face;
  P.pitch = H->pitch;
  P.plane = H->plane;
  // physical spacing of kernel axes: x = axis 0; y = axis 1 (3D); streamed = axis dims-1
  const double hx = H->h[0], hy = H->dims == 3 ? H->h[1] : 1.0, hz = H->dims >= 2 ? H->h[H->dims - 1] : 1.0;
  const double hh[3] = {hx * hx, hy * hy, hz * hz};
  double w1[3], w2[3];
  for (int d = 0; d < 3; ++d) {
    if (H->scheme == NLSE2SHOC_SCHEME_CD) {  // `uttmp`: delta^2 per axis
      w1[d] = 1.0 / hh[d];
      w2[d] = 0.0;
    } else {  // 5-point wide form of the two-step scheme: (16, -1, -30)/(12 h^2)
      w1[d] = 16.0 / (12.0 * hh[d]);
      w2[d] = 1.0 / (12.0 * hh[d]);
    }
  }
  P.cx = R(w2[0]);
  P.cy = R(w2[1]);
  P.cz = R(w2[2]);
  P.c1x = R(w1[0]);
  P.c1y = R(w1[1]);
  P.c1z = R(w1[2]);
  P.ihx2 = R(1.0 / (hx * hx));
  P.ihy2 = R(1.0 / (hy * hy));
  P.ihz2 = R(1.0 / (hz * hz));
  P.hx2 = R(hx * hx);
  P.hy2 = R(hy * hy);
  P.hz2 = R(hz * hz);
  P.a = R(H->a);
  P.s = R(H->s);
  P.inv_a = R(1.0 / H->a);
  P.bc = H->bc;
  P.lean = H->opt_lean;
  P.sched = (H->opt_sched != 0) ? H->sched : nullptr;
  P.vkind = int(H->V.kind);
  if (H->V.kind == NLSE2SHOC_V_HARMONIC) {
    const R *t = reinterpret_cast<const R *>(H->vtab);
    P.vx = t + H->vx_off;
    P.vy = H->dims == 3 ? t + H->vy_off : nullptr;
    P.vz = H->dims >= 2 ? t + H->vz_off : nullptr;
  }
  if (H->V.kind == NLSE2SHOC_V_ARRAY) P.varr = reinterpret_cast<const R *>(H->V.data);
}

// ------------------------------------------------------------------------ launch plans
// Kernel attributes are per device: remember, per kernel instantiation, which devices have
// been configured (a process may drive several GPUs).
static bool attr_needed(std::atomic<uint64_t> &mask) {
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = uint64_t(1) << (dev & 63);
  return (mask.load(std::memory_order_relaxed) & bit) == 0;
}
static void attr_done(std::atomic<uint64_t> &mask) {
  int dev = 0;
  cudaGetDevice(&dev);
  mask.fetch_or(uint64_t(1) << (dev & 63), std::memory_order_relaxed);
}

template <int DIMS, typename R, int MODE> static nlse2shoc_status set_smem_attr() {
  static std::atomic<uint64_t> done{0};
  if (attr_needed(done)) {
    CUDA_TRY(cudaFuncSetAttribute(stage_stream_kernel<DIMS, R, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(Layout<DIMS, R>::template smem_bytes<MODE>())));
    attr_done(done);
  }
  return NLSE2SHOC_OK;
}

// The kernels give chunk c the planes [c L, min((c+1) L, n)) with L = ceil(n / nchunk): a count
// whose last chunks would start at or past n (e.g. n = 33, nchunk = 8: L = 5, chunk 7 starts
// at 35) is replaced by the smallest count with the same L, so every chunk is non-empty.
static int zchunks_normalised(int n, int nchunk) {
  if (n <= 0 || nchunk <= 1) return 1;
  const int L = (n + nchunk - 1) / nchunk;
  return (n + L - 1) / L;
}

// Dynamic tile schedule: choose the middle chunk count nm and the short end chunks (ns of ls
// planes at each end) minimising  ncol * (planes + chunks * p) / G + tail,  where the tail is
// one middle tile (mlen + p) unless the traversal ends on short chunk rows, which absorb it:
// max(ls + p, mlen + p - S / G), S = the short-tile work at the end of the order.  (The
// kernel's fused-exchange order runs chunks 0 and nchunk-1 first, so it ends on ns - 1 short
// rows; forward and reversed traversals end on ns.)  Middle chunks at most maxl planes when
// that is possible.  Memoised per handle (the search is ~40k evaluations).
static ZLayout zlayout_dynamic(nlse2shoc_t H, int nzr, int ncol, int G, double p, int maxl, bool fused_order) {
  const int tail = H->opt_tail;
  const uint64_t key = (uint64_t(nzr) << 40) ^ (uint64_t(ncol) << 20) ^ (uint64_t(G) << 4) ^
                       (uint64_t(p == 2.0) << 3) ^ (uint64_t(maxl == 64) << 2) ^ (uint64_t(fused_order) << 1) ^
                       uint64_t(tail != 0);
  auto it = H->zmemo.find(key);
  if (it != H->zmemo.end()) return it->second;
  static const int NS[] = {0, 1, 2, 3, 4, 6, 8, 12, 16, 24, 32, 48, 64};
  static const int LS[] = {1, 2, 3, 4, 6, 8, 12, 16, 24, 32};
  ZLayout best, best_any;
  double bestc = 1e300, bestc_any = 1e300;
  for (int ns : NS) {
    if (ns > 0 && !tail) break;
    for (int ls : LS) {
      if (ns == 0 && ls > 1) break;
      const int mid = nzr - 2 * ns * (ns ? ls : 0);
      if (mid < 1) break;
      for (int nm = 1; nm <= 256 && 4 * nm <= mid + 3; ++nm) {
        const int mlen = (mid + nm - 1) / nm;
        const int nme = (mid + mlen - 1) / mlen;  // non-empty middle chunks
        if (nme != nm) continue;
        const double work = double(ncol) * (mid + nme * p + 2.0 * ns * (ls + p)) / G;
        const int send = ns == 0 ? 0 : (fused_order && nme + 2 * ns >= 3 ? ns - 1 : ns);
        double tl = mlen + p;
        if (send > 0) tl = std::max(double(ls) + p, mlen + p - double(ncol) * send * (ls + p) / G);
        const double c = work + tl;
        ZLayout z;
        z.nchunk = nme + 2 * ns;
        z.ns = ns;
        z.ls = ns ? ls : 0;
        z.mlen = mlen;
        if (c < bestc_any - 1e-9) { bestc_any = c; best_any = z; }
        if (mlen <= maxl && c < bestc - 1e-9) { bestc = c; best = z; }
      }
    }
  }
  if (bestc > 1e299) best = best_any;
  H->zmemo[key] = best;
  return best;
}

template <int DIMS, typename R, int MODE>
static nlse2shoc_status launch_stream(nlse2shoc_t H, Field &in, const CUtensorMap *tm_psi, const CUtensorMap *tm_acc,
                                      StageParams<R> P, cudaStream_t st, const CUtensorMap *tm_t3 = nullptr) {
  using C = Cfg<DIMS, R>;
  using LY = Layout<DIMS, R>;
  TRY((set_smem_attr<DIMS, R, MODE>()));
  const size_t smem = LY::template smem_bytes<MODE>();
  int occ = 1;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, stage_stream_kernel<DIMS, R, MODE>, LY::NTHREADS, smem));
  occ = std::max(occ, 1);
  const int G0 = std::max(1, H->num_sms - H->reserve_sms) * occ;
  P.ncx = int((H->nx + C::TX - 1) / C::TX);
  P.ncy = DIMS == 3 ? int((H->ny + C::TY - 1) / C::TY) : 1;
  const int ncol = P.ncx * P.ncy;
  // z-chunks: minimise rounds * (chunk length + priming cost).  3D: chunks of at most 64 planes
  // where possible — neighbouring tiles of a round then stay close in z and their halo reads
  // hit L2 (C4: 110-plane chunks 9.35 ms/step, 55-plane chunks 9.24).
  // Dynamic schedule (P.sched): tiles are taken in order by whichever CTA is free, so the cost
  // is the total work plus the tail, with p the priming cost in planes per tile (measured: 2 for
  // complex64, 4 for complex128 tiles; C4 as 8 slabs of 96 planes 9.72 -> 9.46 ms/step with
  // 24-plane chunks, C5W c64 2.13 -> 2.08).  The tail is one tile unless the traversal ends on
  // short chunks (option TAIL_CHUNKS: ns chunks of ls planes at each end of the range, see
  // zlayout_dynamic), which then only have to outlast the last long tile.
  const int nzr = P.ze - P.zb;  // planes this launch computes
  ZLayout zl;
  if (H->opt_zchunks > 0) {
    zl.nchunk = std::max(1, zchunks_normalised(nzr, std::min<int>(H->opt_zchunks, nzr)));
    zl.mlen = (nzr + zl.nchunk - 1) / zl.nchunk;
  } else if (P.sched) {
    const bool fused_order = P.cnt != nullptr;  // the kernel's edge-chunks-first order
    zl = zlayout_dynamic(H, nzr, ncol, G0, sizeof(R) == 4 ? 2.0 : 4.0, DIMS == 3 ? 64 : 1 << 30, fused_order);
  } else {
    int best = 1, best_any = 1;
    double bestc = 1e300, bestc_any = 1e300;
    for (int nc = 1; nc <= 256 && 4 * nc <= nzr + 3; ++nc) {
      const double L = std::ceil(double(nzr) / nc);
      const double c = std::ceil(double(ncol) * nc / G0) * (L + 1.5);
      if (c < bestc_any - 1e-9) { bestc_any = c; best_any = nc; }
      if ((DIMS != 3 || L <= 64.0) && c < bestc - 1e-9) { bestc = c; best = nc; }
    }
    if (bestc > 1e299) best = best_any;
    zl.nchunk = std::max(1, zchunks_normalised(nzr, best));
    zl.mlen = (nzr + zl.nchunk - 1) / zl.nchunk;
  }
  P.nchunk = zl.nchunk;
  P.ns = zl.ns;
  P.ls = zl.ls;
  P.mlen = zl.mlen;
  P.ntiles = ncol * zl.nchunk;
  const int G = std::min(G0, P.ntiles);
  P.in_T = reinterpret_cast<const cplx<R> *>(in.ptr);
  const CUtensorMap *lo = P.has_lo_halo ? &in.tm_lo : &in.tm;
  const CUtensorMap *hi = P.has_hi_halo ? &in.tm_hi : &in.tm;
  stage_stream_kernel<DIMS, R, MODE><<<G, LY::NTHREADS, smem, st>>>(in.tm, *lo, *hi, tm_psi ? *tm_psi : in.tm,
                                                                   tm_acc ? *tm_acc : in.tm, tm_t3 ? *tm_t3 : in.tm, P);
  CUDA_TRY(cudaGetLastError());
  ++H->launches;
  return NLSE2SHOC_OK;
}

// Stage-pair (temporal blocking) launch, variant 4: one persistent grid per pair.
template <int DIMS, typename R, int PAIR>
static nlse2shoc_status launch_pair(nlse2shoc_t H, const CUtensorMap &tin, const CUtensorMap &tps,
                                    const CUtensorMap &tacc, StageParams<R> P, cudaStream_t st) {
  using C = PCfg<DIMS, R>;
  using LY = PLayout<DIMS, R>;
  const size_t smem = LY::template smem_bytes<PAIR>();
  static std::atomic<uint64_t> attr{0};
  if (attr_needed(attr)) {
    CUDA_TRY(cudaFuncSetAttribute(pair_stream_kernel<DIMS, R, PAIR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(smem)));
    attr_done(attr);
  }
  int occ = 1;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pair_stream_kernel<DIMS, R, PAIR>, LY::NTHREADS, smem));
  occ = std::max(occ, 1);
  const int G0 = H->num_sms * occ;
  P.ncx = int((H->nx + C::TX - 1) / C::TX);
  P.ncy = DIMS == 3 ? int((H->ny + C::TY - 1) / C::TY) : 1;
  const int ncol = P.ncx * P.ncy;
  // z-chunks: minimise rounds * (chunk length + priming cost of 4 extra phase-A planes)
  int best = 1;
  double bestc = 1e300;
  for (int nc = 1; nc <= 256 && nc <= H->nz; ++nc) {
    const double rounds = std::ceil(double(ncol) * nc / G0);
    const double c = rounds * (std::ceil(double(H->nz) / nc) + 4.0);
    if (c < bestc - 1e-9) { bestc = c; best = nc; }
  }
  if (H->opt_zchunks > 0) best = std::min<int>(H->opt_zchunks, int(H->nz));
  best = zchunks_normalised(int(H->nz), best);
  P.nchunk = best;
  P.ntiles = ncol * best;
  const int G = std::min(G0, P.ntiles);
  pair_stream_kernel<DIMS, R, PAIR><<<G, LY::NTHREADS, smem, st>>>(tin, tps, tacc, P);
  CUDA_TRY(cudaGetLastError());
  ++H->launches;
  return NLSE2SHOC_OK;
}

// One RK4 step of the stage-pair form: X = Psi^n (read), Y = Psi^{n+1} (written), X != Y.
template <int DIMS, typename R>
static nlse2shoc_status pair_step(nlse2shoc_t H, Field &X, Field &Y, double dt, cudaStream_t st) {
  StageParams<R> P;
  fill_params<R>(H, P);
  P.cA = R(dt / 2.0);
  P.ca = R(dt / 3.0);
  P.cb = R(dt / 2.0);
  P.out_T = reinterpret_cast<cplx<R> *>(H->TB.ptr);
  P.out_acc = reinterpret_cast<cplx<R> *>(H->acc.ptr);
  TRY((launch_pair<DIMS, R, PAIR_A>(H, X.tm_in4, X.tm_in4, X.tm_in4, P, st)));
  P.cA = R(dt);
  P.ca = R(0);
  P.cb = R(dt / 6.0);
  P.out_T = reinterpret_cast<cplx<R> *>(Y.ptr);
  P.out_acc = nullptr;
  return launch_pair<DIMS, R, PAIR_B>(H, H->TB.tm_in4, X.tm_ex, H->acc.tm_ppt, P, st);
}

static nlse2shoc_status rk4_pairs(nlse2shoc_t H, Field &psi, double dt, int64_t nsteps, cudaStream_t st) {
  Field *X = &psi, *Y = &H->TA;
  const bool f32 = H->dtype == NLSE2SHOC_C64;
  for (int64_t n = 0; n < nsteps; ++n) {
    if (H->dims == 3) TRY(f32 ? (pair_step<3, float>(H, *X, *Y, dt, st)) : (pair_step<3, double>(H, *X, *Y, dt, st)));
    else TRY(f32 ? (pair_step<2, float>(H, *X, *Y, dt, st)) : (pair_step<2, double>(H, *X, *Y, dt, st)));
    std::swap(X, Y);
  }
  if (X != &psi)
    CUDA_TRY(cudaMemcpyAsync(psi.ptr, X->ptr, size_t(H->local_elems) * H->S, cudaMemcpyDeviceToDevice, st));
  return NLSE2SHOC_OK;
}

template <typename R, int MODE>
static nlse2shoc_status launch_line(nlse2shoc_t H, const void *in, const void *psi, const void *acc, StageParams<R> P,
                                    cudaStream_t st, const void *t3 = nullptr) {
  const int threads = 256;
  // Grids of >= 16 segments: the persistent bulk-copy ring, as many CTAs per SM as its shared
  // memory allows (r2: C2 c64 0.0994 -> 0.0724 ms/step with 512-point segments and >= 3 CTAs
  // per SM, c128 0.146 -> 0.130 from the occupancy-sized grid).  Smaller grids: complex128 the
  // grid-stride kernel (L1 serves the stencil overlap), complex64 tiles of 256 points.
  if (H->nx >= 16 * LineStream<R>::SEG) {
    static std::atomic<uint64_t> attr{0};
    const size_t smem = line_stream_smem<R, MODE>();
    if (attr_needed(attr)) {
      CUDA_TRY(cudaFuncSetAttribute(line_stream_kernel<R, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      attr_done(attr);
    }
    const int64_t nseg = (H->nx + LineStream<R>::SEG - 1) / LineStream<R>::SEG;
    int occ = 1;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, line_stream_kernel<R, MODE>, LineStream<R>::NT, smem));
    const int grid = int(std::min<int64_t>(nseg, int64_t(H->num_sms) * std::max(occ, 1)));
    line_stream_kernel<R, MODE><<<grid, LineStream<R>::NT, smem, st>>>(
        reinterpret_cast<const cplx<R> *>(in), reinterpret_cast<const cplx<R> *>(psi),
        reinterpret_cast<const cplx<R> *>(acc), reinterpret_cast<const cplx<R> *>(t3), P);
  } else if (sizeof(R) == 8) {
    const int64_t blocks = std::min<int64_t>((H->nx + threads - 1) / threads, int64_t(H->num_sms) * 8);
    stage_line_kernel<R, MODE><<<int(blocks), threads, 0, st>>>(
        reinterpret_cast<const cplx<R> *>(in), reinterpret_cast<const cplx<R> *>(psi),
        reinterpret_cast<const cplx<R> *>(acc), reinterpret_cast<const cplx<R> *>(t3), P);
  } else {
    constexpr int PT = 1;
    const int64_t blocks = (H->nx + threads * PT - 1) / (threads * PT);
    line_tile_kernel<R, MODE, PT><<<int(blocks), threads, 0, st>>>(
        reinterpret_cast<const cplx<R> *>(in), reinterpret_cast<const cplx<R> *>(psi),
        reinterpret_cast<const cplx<R> *>(acc), reinterpret_cast<const cplx<R> *>(t3), P);
  }
  CUDA_TRY(cudaGetLastError());
  ++H->launches;
  return NLSE2SHOC_OK;
}

// ------------------------------------------------------------------------- halo (NCCL)
static nlse2shoc_status halo_exchange(nlse2shoc_t H, Field &f, cudaStream_t st) {
  if (!H->sharded || H->nranks == 1) return NLSE2SHOC_OK;
#ifdef NLSE_WITH_NCCL
  const size_t bytes = size_t(2 * H->plane) * H->S;
  char *base = reinterpret_cast<char *>(f.ptr);
  NCCL_TRY(ncclGroupStart());
  if (H->rank > 0) {
    NCCL_TRY(ncclSend(base, bytes, ncclChar, H->rank - 1, H->comm, st));
    NCCL_TRY(ncclRecv(f.halo_lo, bytes, ncclChar, H->rank - 1, H->comm, st));
  }
  if (H->rank < H->nranks - 1) {
    NCCL_TRY(ncclSend(base + size_t(H->nz - 2) * H->plane * H->S, bytes, ncclChar, H->rank + 1, H->comm, st));
    NCCL_TRY(ncclRecv(f.halo_hi, bytes, ncclChar, H->rank + 1, H->comm, st));
  }
  NCCL_TRY(ncclGroupEnd());
  return NLSE2SHOC_OK;
#else
  (void)f;
  (void)st;
  return fail(NLSE2SHOC_EUNSUPPORTED, "built without NCCL");
#endif
}

// elements of one D field of the two-kernel variants (local planes [-1, nz])
static int64_t D_field_elems(nlse2shoc_t H) { return H->plane * (H->dims >= 2 ? H->nz + 2 : 1); }

template <int DIMS, typename R>
static nlse2shoc_status launch_two(int, int stage, const cplx<R> *in, const cplx<R> *lo, const cplx<R> *hi,
                                   const cplx<R> *psi, const cplx<R> *acc, cplx<R> *D, const StageParams<R> &P,
                                   const TwoParams<R> &Q, cudaStream_t st, int64_t &launches) {
  CUDA_TRY((launch_two_impl<DIMS, R>(stage, in, lo, hi, psi, acc, D, P, Q, st)));
  launches += 2;
  return NLSE2SHOC_OK;
}

// ----------------------------------------------------------------------- stage drivers
// Stage s = 1..4 of an RK4 step reads X_{s-1} as its stencil input (X_0 = Psi^n) and writes
// the next stage input and the accumulator (Psi-space form):
//   1: acc = Psi + k/6 K1,  T_A = Psi + k/2 K1        3: acc += k/3 K3,  T_A = Psi + k K3
//   2: acc += k/3 K2,       T_B = Psi + k/2 K2        4: Psi = acc + k/6 K4
// s = 5 is the Laplacian (Psi -> L).
// Carried-sum combine (DESIGN.md §5, 12 transfers): the default (variant 0) and variant 7.
// Write-light combine (13 transfers): variant 5 (the default until r2's carried sum).
static bool carried(const nlse2shoc_t H) { return H->variant == 0 || H->variant == 7; }
static bool write_light(const nlse2shoc_t H) { return H->variant == 5; }

// role of stage s's stencil input in the halo arena: 0 Psi, 1 T_A, 2 T_B, 3 acc
static int input_role(const nlse2shoc_t H, int s) {
  if (s == 1 || s == 5) return 0;
  if (s == 4 && write_light(H)) return 3;
  return s == 3 ? 2 : 1;
}

// (write-light: stage 3 writes T_C into acc's buffer, which is stage 4's stencil input)
static Field &stage_input(nlse2shoc_t H, Field &psi, int s) {
  if (s == 4 && write_light(H)) return H->acc;
  return (s == 1 || s == 5) ? psi : (s == 3 ? H->TB : H->TA);
}

template <int DIMS, typename R, int MODE>
static nlse2shoc_status launch_mode(nlse2shoc_t H, Field &psi, Field &in, StageParams<R> &P, cudaStream_t st) {
  if (H->variant == 3) {  // two-kernel, multi-storage (per-axis D_d stored)
    CUDA_TRY((launch_two_ms_impl<DIMS, R>(MODE, reinterpret_cast<const cplx<R> *>(in.ptr),
                                          reinterpret_cast<const cplx<R> *>(in.halo_lo),
                                          reinterpret_cast<const cplx<R> *>(in.halo_hi),
                                          reinterpret_cast<const cplx<R> *>(psi.ptr),
                                          reinterpret_cast<const cplx<R> *>(H->acc.ptr),
                                          reinterpret_cast<cplx<R> *>(H->D.ptr), D_field_elems(H), P, st)));
    H->launches += 2;
    return NLSE2SHOC_OK;
  }
  if (H->variant == 1) {  // two-kernel (stored D)
    TwoParams<R> Q;
    two_params<R>(H->dims, H->h, Q);
    return launch_two<DIMS, R>(0, MODE, reinterpret_cast<const cplx<R> *>(in.ptr),
                               reinterpret_cast<const cplx<R> *>(in.halo_lo), reinterpret_cast<const cplx<R> *>(in.halo_hi),
                               reinterpret_cast<const cplx<R> *>(psi.ptr), reinterpret_cast<const cplx<R> *>(H->acc.ptr),
                               reinterpret_cast<cplx<R> *>(H->D.ptr), P, Q, st, H->launches);
  }
  if constexpr (DIMS == 1) return launch_line<R, MODE>(H, in.ptr, psi.ptr, H->acc.ptr, P, st);
  else return launch_stream<DIMS, R, MODE>(H, in, &psi.tm_pt, &H->acc.tm_pt, P, st);
}

template <int DIMS, typename R>
static nlse2shoc_status launch_stage(nlse2shoc_t H, Field &psi, int s, double dt, void *L, cudaStream_t st) {
  StageParams<R> P;
  fill_params<R>(H, P);
  // stages 2 and 4 walk the grid backwards: the planes the previous stage wrote last are still
  // in L2 when this stage starts (option REVERSE_ORDER)
  P.rev = (H->opt_reverse && (s == 2 || s == 4)) ? 1 : 0;
  // base pointers of the pointwise streams (must match the maps passed to launch_stream)
  P.in_P[0] = reinterpret_cast<const cplx<R> *>(psi.ptr);
  P.in_P[1] = reinterpret_cast<const cplx<R> *>(H->acc.ptr);
  P.in_P[2] = nullptr;
  Field &in = stage_input(H, psi, s);
  if (H->fusing && s <= 4) {
    // fused exchange: this stage's output is the next stage's input (stage 4: Psi^{n+1})
    const int r = input_role(H, s == 4 ? 1 : s + 1);
    P.mir_lo = reinterpret_cast<cplx<R> *>(H->peer_lo[r]);
    P.mir_hi = reinterpret_cast<cplx<R> *>(H->peer_hi[r]);
    P.sig_lo = H->peer_sig_lo;
    P.sig_hi = H->peer_sig_hi;
    P.cnt = H->cnt;
    P.wait_lo = H->peer_lo[r] != nullptr;
    P.wait_hi = H->peer_hi[r] != nullptr;
    P.peer_sys = H->ipc_lo != nullptr || H->ipc_hi != nullptr;
    P.rev = 0;  // edge chunks first (the kernel's chunk order), not the reversed traversal
  }
  cplx<R> *pPsi = reinterpret_cast<cplx<R> *>(psi.ptr), *pA = reinterpret_cast<cplx<R> *>(H->TA.ptr),
          *pB = reinterpret_cast<cplx<R> *>(H->TB.ptr), *pAcc = reinterpret_cast<cplx<R> *>(H->acc.ptr);
  // reconstructed-accumulator form (13 transfers per point-step): variant 6
  const bool recon = H->variant == 6;
  if (carried(H)) {
    // carried-sum form (12 transfers per point-step): stage 2 also stores
    // Q = 3 acc - Psi; stage 3 writes T_C over T_A; stage 4 forms (Q + T_C + k/2 K4) / 3
    switch (s) {
      case 1:
        P.cb = R(dt / 2.0); P.out_T = pA;
        if constexpr (DIMS >= 2) return launch_stream<DIMS, R, M_S1R>(H, in, &psi.tm_pt, &H->acc.tm_pt, P, st);
        else return launch_line<R, M_S1R>(H, in.ptr, psi.ptr, H->acc.ptr, P, st);
      case 2:
        P.ca = R(dt); P.cb = R(dt / 2.0); P.out_T = pB; P.out_acc = pAcc;
        if constexpr (DIMS >= 2) return launch_stream<DIMS, R, M_S2Y>(H, in, &psi.tm_pt, &H->acc.tm_pt, P, st);
        else return launch_line<R, M_S2Y>(H, in.ptr, psi.ptr, H->acc.ptr, P, st);
      case 3:
        P.cb = R(dt); P.out_T = pA;  // T_C
        if constexpr (DIMS >= 2) return launch_stream<DIMS, R, M_S3R>(H, in, &psi.tm_pt, &H->acc.tm_pt, P, st);
        else return launch_line<R, M_S3R>(H, in.ptr, psi.ptr, H->acc.ptr, P, st);
      case 4:
        P.cb = R(dt / 2.0); P.out_T = pPsi;  // k/2 K4 joins the numerator of the division by 3
        if constexpr (DIMS >= 2) return launch_stream<DIMS, R, M_S4Y>(H, in, &psi.tm_pt, &H->acc.tm_pt, P, st);
        else return launch_line<R, M_S4Y>(H, in.ptr, psi.ptr, H->acc.ptr, P, st);
      default:
        break;
    }
  }
  if (write_light(H)) {  // write-light form: T_A, T_B, T_C; acc never stored
    switch (s) {
      case 1:
        P.cb = R(dt / 2.0); P.out_T = pA;
        if constexpr (DIMS >= 2) return launch_stream<DIMS, R, M_S1R>(H, in, &psi.tm_pt, &H->acc.tm_pt, P, st);
        else return launch_line<R, M_S1R>(H, in.ptr, psi.ptr, H->acc.ptr, P, st);
      case 2:
        P.cb = R(dt / 2.0); P.out_T = pB;
        if constexpr (DIMS >= 2) return launch_stream<DIMS, R, M_S3R>(H, in, &psi.tm_pt, &H->acc.tm_pt, P, st);
        else return launch_line<R, M_S3R>(H, in.ptr, psi.ptr, H->acc.ptr, P, st);
      case 3:
        P.cb = R(dt); P.out_T = pAcc;  // T_C
        if constexpr (DIMS >= 2) return launch_stream<DIMS, R, M_S3R>(H, in, &psi.tm_pt, &H->acc.tm_pt, P, st);
        else return launch_line<R, M_S3R>(H, in.ptr, psi.ptr, H->acc.ptr, P, st);
      case 4:
        P.cb = R(dt / 6.0); P.out_T = pPsi;
        if constexpr (DIMS >= 2)
        {
          P.in_P[1] = reinterpret_cast<const cplx<R> *>(H->TA.ptr);
          P.in_P[2] = reinterpret_cast<const cplx<R> *>(H->TB.ptr);
          return launch_stream<DIMS, R, M_S4X>(H, in, &psi.tm_pt, &H->TA.tm_pt, P, st, &H->TB.tm_pt);
        }
        else return launch_line<R, M_S4X>(H, in.ptr, psi.ptr, H->TA.ptr, P, st, H->TB.ptr);
      default:
        break;
    }
  }
  switch (s) {
    case 1:
      P.ca = R(dt / 6.0); P.cb = R(dt / 2.0); P.out_T = pA; P.out_acc = pAcc;
      if (recon) {
        if constexpr (DIMS >= 2) return launch_stream<DIMS, R, M_S1R>(H, in, &psi.tm_pt, &H->acc.tm_pt, P, st);
        else return launch_line<R, M_S1R>(H, in.ptr, psi.ptr, H->acc.ptr, P, st);
      }
      return launch_mode<DIMS, R, M_S1>(H, psi, in, P, st);
    case 2:
      P.ca = R(dt / 3.0); P.cb = R(dt / 2.0); P.out_T = pB; P.out_acc = pAcc;
      if (recon) {
        if constexpr (DIMS >= 2) return launch_stream<DIMS, R, M_S2R>(H, in, &psi.tm_pt, &H->acc.tm_pt, P, st);
        else return launch_line<R, M_S2R>(H, in.ptr, psi.ptr, H->acc.ptr, P, st);
      }
      return launch_mode<DIMS, R, M_S2>(H, psi, in, P, st);
    case 3:
      P.ca = R(dt / 3.0); P.cb = R(dt); P.out_T = pA; P.out_acc = pAcc;
      if (recon) {
        if constexpr (DIMS >= 2) return launch_stream<DIMS, R, M_S3R>(H, in, &psi.tm_pt, &H->acc.tm_pt, P, st);
        else return launch_line<R, M_S3R>(H, in.ptr, psi.ptr, H->acc.ptr, P, st);
      }
      return launch_mode<DIMS, R, M_S3>(H, psi, in, P, st);
    case 4:
      P.ca = R(0); P.cb = R(dt / 6.0); P.out_T = pPsi; P.out_acc = nullptr;
      if (recon) {
        if constexpr (DIMS >= 2) return launch_stream<DIMS, R, M_S4R>(H, in, &psi.tm_pt, &H->acc.tm_pt, P, st);
        else return launch_line<R, M_S4R>(H, in.ptr, psi.ptr, H->acc.ptr, P, st);
      }
      return launch_mode<DIMS, R, M_S4>(H, psi, in, P, st);
    default:
      P.out_T = reinterpret_cast<cplx<R> *>(L);
      return launch_mode<DIMS, R, M_LAP>(H, psi, in, P, st);
  }
}

// NVTX ranges (per call, per stage, per halo exchange) for nsys / ncu --nvtx range
// filters; the NVTX v3 calls are no-ops unless a tool is attached.  Inside a CUDA-graph
// capture they mark the enqueue of the captured step, not its replays.
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange &) = delete;
  NvtxRange &operator=(const NvtxRange &) = delete;
};

static nlse2shoc_status stage(nlse2shoc_t H, Field &psi, int s, double dt, void *L, cudaStream_t st) {
  static const char *const names[] = {"", "nlse2shoc stage 1", "nlse2shoc stage 2", "nlse2shoc stage 3",
                                      "nlse2shoc stage 4", "nlse2shoc laplacian stage"};
  NvtxRange nvtx_r(names[s >= 1 && s <= 5 ? s : 0]);
  const bool f32 = H->dtype == NLSE2SHOC_C64;
  switch (H->dims) {
    case 1: return f32 ? launch_stage<1, float>(H, psi, s, dt, L, st) : launch_stage<1, double>(H, psi, s, dt, L, st);
    case 2: return f32 ? launch_stage<2, float>(H, psi, s, dt, L, st) : launch_stage<2, double>(H, psi, s, dt, L, st);
    default: return f32 ? launch_stage<3, float>(H, psi, s, dt, L, st) : launch_stage<3, double>(H, psi, s, dt, L, st);
  }
}

// A "view" is the list of slabs a call works on: one handle (single GPU, or this rank's
// slab under NCCL sharding), or the virtual slabs of a loopback handle.
struct View {
  std::vector<nlse2shoc_t> hs;
  std::vector<Field> psis;
};

// Halo exchange of stage s's stencil input (2 planes per side): NCCL for a real shard,
// device-to-device copies between the virtual slabs of a loopback handle.
static nlse2shoc_status exchange(View &v, int s, cudaStream_t st) {
  NvtxRange nvtx_r("nlse2shoc halo exchange");
  const size_t P = v.hs.size();
  if (P == 1) return halo_exchange(v.hs[0], stage_input(v.hs[0], v.psis[0], s), st);
  for (size_t i = 0; i < P; ++i) {
    nlse2shoc_t H = v.hs[i];
    Field &f = stage_input(H, v.psis[i], s);
    const size_t b2 = size_t(2 * H->plane) * H->S;
    if (i > 0) {
      nlse2shoc_t Hn = v.hs[i - 1];
      Field &g = stage_input(Hn, v.psis[i - 1], s);
      CUDA_TRY(cudaMemcpyAsync(f.halo_lo, reinterpret_cast<char *>(g.ptr) + size_t(Hn->nz - 2) * Hn->plane * Hn->S, b2,
                               cudaMemcpyDeviceToDevice, st));
    }
    if (i + 1 < P) {
      Field &g = stage_input(v.hs[i + 1], v.psis[i + 1], s);
      CUDA_TRY(cudaMemcpyAsync(f.halo_hi, g.ptr, b2, cudaMemcpyDeviceToDevice, st));
    }
  }
  return NLSE2SHOC_OK;
}

// Small 1D grids: one resident CTA runs the whole call (stage_line.cuh).
template <typename R> static nlse2shoc_status rk4_resident_1d(nlse2shoc_t H, Field &psi, double dt, int64_t nsteps,
                                                              cudaStream_t st) {
  StageParams<R> P;
  fill_params<R>(H, P);
  const size_t smem = size_t(4) * size_t(H->nx) * sizeof(cplx<R>);
  static std::atomic<uint64_t> attr{0};
  if (attr_needed(attr)) {
    CUDA_TRY(cudaFuncSetAttribute(resident_line_kernel<R, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CUDA_TRY(cudaFuncSetAttribute(resident_line_kernel<R, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr_done(attr);
  }
  if (H->bc == NLSE2SHOC_BC_MSD)
    resident_line_kernel<R, true><<<1, 1024, smem, st>>>(reinterpret_cast<cplx<R> *>(psi.ptr), nsteps, R(dt), P);
  else
    resident_line_kernel<R, false><<<1, 1024, smem, st>>>(reinterpret_cast<cplx<R> *>(psi.ptr), nsteps, R(dt), P);
  CUDA_TRY(cudaGetLastError());
  ++H->launches;
  return NLSE2SHOC_OK;
}

static bool resident_ok(nlse2shoc_t H) {
  return H->dims == 1 && H->slabs.empty() && !H->sharded && H->variant != 1 && H->variant != 3 &&
         size_t(4) * size_t(H->nx) * H->S <= size_t(200) * 1024 && H->opt_resident;
}

// Edge-first halo exchange: per stage, the 2 edge planes at each slab end
// (the ones that read halos and that the neighbours need) are computed first, their exchange
// runs on a side stream while the interior planes are computed, and the next stage's edges
// wait for it.  Fused 2D/3D variants on slabs of >= 8 planes (option OVERLAP).
static bool overlap_ok(const View &v) {
  bool multi = v.hs.size() > 1;
  for (nlse2shoc_t H : v.hs) {
    if (!H->opt_overlap || H->dims < 2 || (H->variant != 0 && H->variant != 2 && H->variant != 5 && H->variant != 6 && H->variant != 7) || H->nz < 8)
      return false;
    multi = multi || (H->sharded && H->nranks > 1);
  }
  return multi;
}

static nlse2shoc_status stage_range(nlse2shoc_t H, Field &psi, int s, double dt, int zb, int ze, cudaStream_t st) {
  H->rng_b = zb;
  H->rng_e = ze;
  const nlse2shoc_status r = stage(H, psi, s, dt, nullptr, st);
  H->rng_b = H->rng_e = 0;
  return r;
}

// Graph cache: the last instantiated step graph of a handle, valid for the same stencil-input
// base pointer, dt, kind and settings generation.
static bool graph_cached(nlse2shoc_t H, const void *psi, double dt, int kind) {
  return H->gexec && H->g_psi == psi && H->g_dt == dt && H->g_kind == kind && H->g_gen == H->gen;
}
static void graph_drop(nlse2shoc_t H) {
  if (H->gexec) cudaGraphExecDestroy(H->gexec);  // deferred by the driver until pending launches end
  H->gexec = nullptr;
  H->g_kind = 0;
}
static nlse2shoc_status graph_replay(nlse2shoc_t H, int64_t nsteps, cudaStream_t st) {
  cudaError_t el = cudaSuccess;
  for (int64_t n = 0; n < nsteps && el == cudaSuccess; ++n) el = cudaGraphLaunch(H->gexec, st);
  if (el != cudaSuccess) return fail(NLSE2SHOC_ECUDA, std::string("graph launch: ") + cudaGetErrorString(el));
  return NLSE2SHOC_OK;
}
// End the capture on cs, instantiate and remember the graph in H.
static nlse2shoc_status graph_finish(nlse2shoc_t H, cudaStream_t cs, nlse2shoc_status r, const void *psi, double dt,
                                     int kind) {
  cudaGraph_t graph = nullptr;
  const cudaError_t ec = cudaStreamEndCapture(cs, &graph);
  if (r != NLSE2SHOC_OK) {
    if (graph) cudaGraphDestroy(graph);
    return r;
  }
  if (ec != cudaSuccess) return fail(NLSE2SHOC_ECUDA, std::string("graph capture: ") + cudaGetErrorString(ec));
  graph_drop(H);
  const cudaError_t ei = cudaGraphInstantiate(&H->gexec, graph, 0);
  cudaGraphDestroy(graph);
  if (ei != cudaSuccess) {
    H->gexec = nullptr;
    return fail(NLSE2SHOC_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(ei));
  }
  H->g_psi = psi;
  H->g_dt = dt;
  H->g_kind = kind;
  H->g_gen = H->gen;
  return NLSE2SHOC_OK;
}

// One RK4 step of the edge-first schedule, enqueued on st (the side stream joins and rejoins
// st through events, so the whole step can be captured in a CUDA graph).
static nlse2shoc_status overlapped_step(View &v, double dt, cudaStream_t st) {
  nlse2shoc_t H0 = v.hs[0];
  cudaStream_t cs = H0->comm_st;
  for (int s = 1; s <= 4; ++s) {
    for (size_t i = 0; i < v.hs.size(); ++i) {
      const int nz = int(v.hs[i]->nz);
      TRY(stage_range(v.hs[i], v.psis[i], s, dt, 0, 2, st));
      TRY(stage_range(v.hs[i], v.psis[i], s, dt, nz - 2, nz, st));
    }
    // stage s's output is stage s+1's input (s = 4: Psi, the next step's stage 1 input)
    CUDA_TRY(cudaEventRecord(H0->ev_edge, st));
    CUDA_TRY(cudaStreamWaitEvent(cs, H0->ev_edge, 0));
    TRY(exchange(v, s == 4 ? 1 : s + 1, cs));
    CUDA_TRY(cudaEventRecord(H0->ev_recv, cs));
    for (size_t i = 0; i < v.hs.size(); ++i) {
      // a real NCCL exchange runs kernels: leave it a few SMs beside the persistent grid
      nlse2shoc_t H = v.hs[i];
      H->reserve_sms = (H->sharded && H->nranks > 1) ? 8 : 0;
      const nlse2shoc_status r = stage_range(H, v.psis[i], s, dt, 2, int(H->nz) - 2, st);
      H->reserve_sms = 0;
      TRY(r);
    }
    CUDA_TRY(cudaStreamWaitEvent(st, H0->ev_recv, 0));
  }
  return NLSE2SHOC_OK;
}

// Sharded / loopback calls: the edge-first step (3 launches per slab and stage, the exchange
// and its two events) is captured once into a CUDA graph, NCCL group included, and replayed
// nsteps times (option CUDA_GRAPH; calls of one step run eagerly).
static nlse2shoc_status run_rk4_overlapped(View &v, double dt, int64_t nsteps, cudaStream_t st) {
  nlse2shoc_t H0 = v.hs[0];
  if (!H0->comm_st) {
    CUDA_TRY(cudaStreamCreateWithFlags(&H0->comm_st, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&H0->ev_edge, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&H0->ev_recv, cudaEventDisableTiming));
  }
  TRY(exchange(v, 1, st));  // Psi's halos for the first stage
  if (nsteps < 2 || !H0->opt_graph) {
    for (int64_t n = 0; n < nsteps; ++n) TRY(overlapped_step(v, dt, st));
    return NLSE2SHOC_OK;
  }
  if (!graph_cached(H0, v.psis[0].ptr, dt, 2)) {
    if (!H0->cap_st) CUDA_TRY(cudaStreamCreateWithFlags(&H0->cap_st, cudaStreamNonBlocking));
    for (nlse2shoc_t H : v.hs) H->launches = 0;
    CUDA_TRY(cudaStreamBeginCapture(H0->cap_st, cudaStreamCaptureModeRelaxed));
    const nlse2shoc_status r = overlapped_step(v, dt, H0->cap_st);
    TRY(graph_finish(H0, H0->cap_st, r, v.psis[0].ptr, dt, 2));
    int64_t per_step = 0;
    for (nlse2shoc_t H : v.hs) per_step += H->launches;
    H0->g_launches = per_step;
  }
  TRY(graph_replay(H0, nsteps, st));
  for (nlse2shoc_t H : v.hs) H->launches = 0;
  H0->launches = H0->g_launches * nsteps;
  return NLSE2SHOC_OK;
}

// Single-slab calls of >= 4 steps: the four stage launches of one step are captured once
// into a CUDA graph (on a private stream) and the graph is replayed nsteps times on the
// caller's stream, which trims per-launch overhead on small grids (option CUDA_GRAPH).

static nlse2shoc_status run_rk4_graph(View &v, double dt, int64_t nsteps, cudaStream_t st) {
  nlse2shoc_t H = v.hs[0];
  if (!graph_cached(H, v.psis[0].ptr, dt, 1)) {
    if (!H->cap_st) CUDA_TRY(cudaStreamCreateWithFlags(&H->cap_st, cudaStreamNonBlocking));
    H->launches = 0;
    CUDA_TRY(cudaStreamBeginCapture(H->cap_st, cudaStreamCaptureModeRelaxed));
    nlse2shoc_status r = NLSE2SHOC_OK;
    for (int s = 1; s <= 4 && r == NLSE2SHOC_OK; ++s) r = stage(H, v.psis[0], s, dt, nullptr, H->cap_st);
    TRY(graph_finish(H, H->cap_st, r, v.psis[0].ptr, dt, 1));
    H->g_launches = H->launches;
  }
  TRY(graph_replay(H, nsteps, st));
  H->launches = H->g_launches * nsteps;
  return NLSE2SHOC_OK;
}

// Fused exchange: every slab runs each stage as ONE launch whose kernel
// stores its edge planes into the neighbours' halo buffers and raises their arrival counters;
// there is no exchange step and no edge / interior split.  Fused variants, 2D/3D, slabs with
// connected peers (loopback siblings, or ranks joined by nlse2shoc_connect_peers).
static bool fused_ok(const View &v) {
  for (nlse2shoc_t H : v.hs)
    if (!H->peers || !H->opt_fused || H->dims < 2 ||
        (H->variant != 0 && H->variant != 2 && H->variant != 5 && H->variant != 6 && H->variant != 7))
      return false;
  return true;
}

static nlse2shoc_status fused_step(View &v, double dt, cudaStream_t st) {
  for (int s = 1; s <= 4; ++s)
    for (size_t i = 0; i < v.hs.size(); ++i) {
      v.hs[i]->fusing = true;
      const nlse2shoc_status r = stage(v.hs[i], v.psis[i], s, dt, nullptr, st);
      v.hs[i]->fusing = false;
      TRY(r);
    }
  return NLSE2SHOC_OK;
}

static nlse2shoc_status run_rk4_fused(View &v, double dt, int64_t nsteps, cudaStream_t st) {
  nlse2shoc_t H0 = v.hs[0];
  TRY(exchange(v, 1, st));  // the caller's Psi: halos of the first stage (once per call)
  if (nsteps < 2 || !H0->opt_graph) {
    for (int64_t n = 0; n < nsteps; ++n) TRY(fused_step(v, dt, st));
    return NLSE2SHOC_OK;
  }
  if (!graph_cached(H0, v.psis[0].ptr, dt, 3)) {
    if (!H0->cap_st) CUDA_TRY(cudaStreamCreateWithFlags(&H0->cap_st, cudaStreamNonBlocking));
    for (nlse2shoc_t H : v.hs) H->launches = 0;
    CUDA_TRY(cudaStreamBeginCapture(H0->cap_st, cudaStreamCaptureModeRelaxed));
    const nlse2shoc_status r = fused_step(v, dt, H0->cap_st);
    TRY(graph_finish(H0, H0->cap_st, r, v.psis[0].ptr, dt, 3));
    int64_t per_step = 0;
    for (nlse2shoc_t H : v.hs) per_step += H->launches;
    H0->g_launches = per_step;
  }
  TRY(graph_replay(H0, nsteps, st));
  for (nlse2shoc_t H : v.hs) H->launches = 0;
  H0->launches = H0->g_launches * nsteps;
  return NLSE2SHOC_OK;
}

static nlse2shoc_status run_rk4(View &v, double dt, int64_t nsteps, cudaStream_t st) {
  if (v.hs.size() == 1 && v.hs[0]->variant == 4) return rk4_pairs(v.hs[0], v.psis[0], dt, nsteps, st);
  if (v.hs.size() == 1 && resident_ok(v.hs[0])) {
    nlse2shoc_t H = v.hs[0];
    return H->dtype == NLSE2SHOC_C64 ? rk4_resident_1d<float>(H, v.psis[0], dt, nsteps, st)
                                     : rk4_resident_1d<double>(H, v.psis[0], dt, nsteps, st);
  }
  if (fused_ok(v)) return run_rk4_fused(v, dt, nsteps, st);
  if (overlap_ok(v)) return run_rk4_overlapped(v, dt, nsteps, st);
  if (v.hs.size() == 1 && !v.hs[0]->sharded && nsteps >= 4 && v.hs[0]->opt_graph) return run_rk4_graph(v, dt, nsteps, st);
  for (int64_t n = 0; n < nsteps; ++n)
    for (int s = 1; s <= 4; ++s) {
      TRY(exchange(v, s, st));
      for (size_t i = 0; i < v.hs.size(); ++i) TRY(stage(v.hs[i], v.psis[i], s, dt, nullptr, st));
    }
  return NLSE2SHOC_OK;
}

// ------------------------------------------------------------------------------ create
static nlse2shoc_status alloc_field(nlse2shoc_t H, Field &f) {
  const size_t bytes = size_t(H->local_elems) * H->S;
  CUDA_TRY(dev_malloc(H, &f.ptr, bytes));
  H->bytes += bytes;
  return NLSE2SHOC_OK;
}

// Halo arena of a sharded handle (layout in nlse2shoc_s).  cudaMalloc, not the caller's
// allocator: its base is what CUDA IPC exports to the neighbour ranks.
static Field &role_field(nlse2shoc_t H, int r) { return r == 0 ? H->psiw : (r == 1 ? H->TA : (r == 2 ? H->TB : H->acc)); }
static nlse2shoc_status alloc_arena(nlse2shoc_t H) {
  H->halo_bytes = ((size_t(2 * H->plane) * H->S + 255) / 256) * 256;
  H->arena_bytes = 8 * H->halo_bytes + 256;
  CUDA_TRY(cudaMalloc(reinterpret_cast<void **>(&H->arena), H->arena_bytes));
  CUDA_TRY(cudaMemset(H->arena, 0, H->arena_bytes));
  H->bytes += H->arena_bytes;
  for (int r = 0; r < 4; ++r) {
    role_field(H, r).halo_lo = H->arena + size_t(2 * r) * H->halo_bytes;
    role_field(H, r).halo_hi = H->arena + size_t(2 * r + 1) * H->halo_bytes;
  }
  H->cnt = reinterpret_cast<unsigned long long *>(H->arena + 8 * H->halo_bytes);
  return NLSE2SHOC_OK;
}

template <typename R> static nlse2shoc_status encode_field_maps(nlse2shoc_t H, Field &f) {
  if (H->dims >= 2) {
    if (H->dims == 3) TRY((PMaps<3, R>::all(H, f)));
    else TRY((PMaps<2, R>::all(H, f)));
  }
  if (H->dims == 3) {
    TRY((Maps<3, R>::point(H, &f.tm_pt, f.ptr)));
    TRY((Maps<3, R>::stencil(H, &f.tm, f.ptr, H->nz)));
    if (f.halo_lo) TRY((Maps<3, R>::stencil(H, &f.tm_lo, f.halo_lo, 2)));
    if (f.halo_hi) TRY((Maps<3, R>::stencil(H, &f.tm_hi, f.halo_hi, 2)));
  } else if (H->dims == 2) {
    TRY((Maps<2, R>::point(H, &f.tm_pt, f.ptr)));
    TRY((Maps<2, R>::stencil(H, &f.tm, f.ptr, H->nz)));
    if (f.halo_lo) TRY((Maps<2, R>::stencil(H, &f.tm_lo, f.halo_lo, 2)));
    if (f.halo_hi) TRY((Maps<2, R>::stencil(H, &f.tm_hi, f.halo_hi, 2)));
  }
  return NLSE2SHOC_OK;
}

static nlse2shoc_status encode_maps(nlse2shoc_t H, Field &f) {
  return H->dtype == NLSE2SHOC_C64 ? encode_field_maps<float>(H, f) : encode_field_maps<double>(H, f);
}

template <typename R> static void build_tables(nlse2shoc_t H, std::vector<unsigned char> &host) {
  // per-axis harmonic tables w_d (x_d - c_d)^2, x_d = xmin_d + i h_d, evaluated in double
  const int ax_x = 0, ax_y = 1, ax_z = H->dims - 1;
  std::vector<R> t;
  auto add = [&](int ax, int64_t n) {
    size_t off = t.size();
    for (int64_t i = 0; i < n; ++i) {
      const double x = H->V.xmin[ax] + double(i) * H->h[ax] - H->V.c[ax];
      t.push_back(R(H->V.w[ax] * (x * x)));
    }
    while (t.size() % 4) t.push_back(R(0));
    return off;
  };
  H->vx_off = add(ax_x, H->N[0]);
  H->vy_off = H->dims == 3 ? add(ax_y, H->N[1]) : 0;
  H->vz_off = H->dims >= 2 ? add(ax_z, H->N[ax_z]) : 0;
  host.resize(t.size() * sizeof(R));
  std::memcpy(host.data(), t.data(), host.size());
}

static nlse2shoc_status create_impl(nlse2shoc_t *out, int dims, const int64_t N[3], const double h[3], double a,
                                    double s, const nlse2shoc_potential *V, nlse2shoc_bc bc, nlse2shoc_dtype dtype,
                                    int rank, int nranks, const void *id128, int loop = 0) {
  // loop > 0: this is virtual slab `rank` of a loopback handle (sharded layout, no NCCL);
  // loop < 0: the loopback parent of -loop virtual slabs (owns only the staging buffers)
  if (!out) return fail(NLSE2SHOC_EINVAL, "out is NULL");
  *out = nullptr;
  if (dims < 1 || dims > 3) return fail(NLSE2SHOC_EINVAL, "dims must be 1, 2 or 3");
  if (!N || !h) return fail(NLSE2SHOC_EINVAL, "N / h is NULL");
  for (int d = 0; d < 3; ++d) {
    if (d < dims) {
      if (N[d] < 5) return fail(NLSE2SHOC_EINVAL, "N[d] must be >= 5");
      if (N[d] > (int64_t(1) << 31) - 64) return fail(NLSE2SHOC_EINVAL, "N[d] too large");
      if (!finite_pos(h[d])) return fail(NLSE2SHOC_EINVAL, "h[d] must be finite and > 0");
    } else if (N[d] != 1) {
      return fail(NLSE2SHOC_EINVAL, "N[d] must be 1 for unused axes");
    }
  }
  if (!finite_pos(a)) return fail(NLSE2SHOC_EINVAL, "a must be finite and > 0");
  if (!std::isfinite(s)) return fail(NLSE2SHOC_EINVAL, "s must be finite");
  if (bc != NLSE2SHOC_BC_DIRICHLET && bc != NLSE2SHOC_BC_LAPZERO && bc != NLSE2SHOC_BC_MSD)
    return fail(NLSE2SHOC_EINVAL, "bad bc");
  if (bc == NLSE2SHOC_BC_MSD && dims != 1)
    return fail(NLSE2SHOC_EUNSUPPORTED, "the MSD boundary is implemented for 1D grids only");
  if (dtype != NLSE2SHOC_C64 && dtype != NLSE2SHOC_C128) return fail(NLSE2SHOC_EINVAL, "bad dtype");
  nlse2shoc_potential pv{};
  pv.kind = NLSE2SHOC_V_NONE;
  if (V) pv = *V;
  if (pv.kind != NLSE2SHOC_V_NONE && pv.kind != NLSE2SHOC_V_HARMONIC && pv.kind != NLSE2SHOC_V_ARRAY)
    return fail(NLSE2SHOC_EINVAL, "bad potential kind");
  if (pv.kind == NLSE2SHOC_V_ARRAY && !pv.data) return fail(NLSE2SHOC_EINVAL, "V.data is NULL");
  if (pv.kind == NLSE2SHOC_V_HARMONIC)
    for (int d = 0; d < dims; ++d)
      if (!std::isfinite(pv.w[d]) || !std::isfinite(pv.c[d]) || !std::isfinite(pv.xmin[d]))
        return fail(NLSE2SHOC_EINVAL, "non-finite harmonic parameters");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(NLSE2SHOC_EINVAL, "bad rank / nranks");
  if ((nranks > 1 || loop != 0) && dims == 1) return fail(NLSE2SHOC_EINVAL, "1D grids are not sharded (replicas only)");
#ifndef NLSE_WITH_NCCL
  if (nranks > 1 && loop == 0) return fail(NLSE2SHOC_EUNSUPPORTED, "built without NCCL");
#endif

  auto *H = new nlse2shoc_s();
  H->alloc = g_alloc;
  H->dfree = g_free;
  H->alloc_ctx = g_alloc_ctx;
  H->dims = dims;
  for (int d = 0; d < 3; ++d) { H->N[d] = N[d]; H->h[d] = d < dims ? h[d] : 1.0; }
  H->a = a;
  H->s = s;
  H->V = pv;
  H->bc = bc;
  H->dtype = dtype;
  H->S = dtype == NLSE2SHOC_C64 ? 8 : 16;
  H->rank = rank;
  H->nranks = nranks;
  H->sharded = id128 != nullptr || loop > 0;
  H->loop_member = loop > 0;
  cudaGetDevice(&H->device);
  cudaDeviceGetAttribute(&H->num_sms, cudaDevAttrMultiProcessorCount, H->device);
  H->NZ = dims >= 2 ? N[dims - 1] : 1;
  H->nx = N[0];
  H->ny = dims == 3 ? N[1] : 1;
  int64_t z0 = 0, nz = H->NZ;
  if (dims >= 2) nlse2shoc_split(H->NZ, nranks, rank, &z0, &nz);
  if (dims >= 2 && nz < 2) { delete H; return fail(NLSE2SHOC_EINVAL, "each slab needs >= 2 planes"); }
  H->z0 = z0;
  H->nz = dims >= 2 ? nz : 1;
  if (loop > 0 && pv.kind == NLSE2SHOC_V_ARRAY)  // virtual slab: its part of the whole-grid V
    H->V.data = reinterpret_cast<const char *>(pv.data) + size_t(z0) * size_t(N[0]) * size_t(dims == 3 ? N[1] : 1) *
                                                        (dtype == NLSE2SHOC_C64 ? sizeof(float) : sizeof(double));
  if (dims == 1) H->nz = 1;
  const int64_t cpv = 16 / int64_t(H->S);
  H->pitch = dims == 1 ? H->nx : ((H->nx + cpv - 1) / cpv) * cpv;
  H->plane = H->pitch * H->ny;
  H->local_elems = H->plane * H->nz;
  *out = H;  // from here on, destroy() cleans up on failure

  nlse2shoc_status st = NLSE2SHOC_OK;
  auto chk = [&](nlse2shoc_status r) { if (st == NLSE2SHOC_OK) st = r; };
  if (loop < 0) {  // loopback parent: virtual slabs + staging buffers only
    const int P = -loop;
    for (int i = 0; i < P && st == NLSE2SHOC_OK; ++i) {
      nlse2shoc_t S = nullptr;
      chk(create_impl(&S, dims, N, h, a, s, V, bc, dtype, i, P, nullptr, 1));
      if (S) H->slabs.push_back(S);
    }
    // virtual slabs are each other's peers (same device): the fused exchange needs no IPC
    for (size_t i = 0; st == NLSE2SHOC_OK && i < H->slabs.size(); ++i) {
      nlse2shoc_t S = H->slabs[i];
      nlse2shoc_t lo = i > 0 ? H->slabs[i - 1] : nullptr, hi = i + 1 < H->slabs.size() ? H->slabs[i + 1] : nullptr;
      for (int r = 0; r < 4; ++r) {
        S->peer_lo[r] = lo ? role_field(lo, r).halo_hi : nullptr;
        S->peer_hi[r] = hi ? role_field(hi, r).halo_lo : nullptr;
      }
      S->peer_sig_lo = lo ? lo->cnt + 1 : nullptr;  // the lower slab's "from above" counter
      S->peer_sig_hi = hi ? hi->cnt : nullptr;      // the upper slab's "from below" counter
      S->peers = true;
    }
    if (st == NLSE2SHOC_OK && H->pitch != H->nx) {
      chk(alloc_field(H, H->psiw));
      if (st == NLSE2SHOC_OK && dev_malloc(H, &H->Lw, size_t(H->local_elems) * H->S) != cudaSuccess)
        chk(fail(NLSE2SHOC_ENOMEM, "staging allocation failed"));
    }
    if (st != NLSE2SHOC_OK) {
      std::string keep = g_last_error;
      nlse2shoc_destroy(H);
      *out = nullptr;
      g_last_error = keep;
    }
    return st;
  }
  chk(alloc_field(H, H->TA));
  chk(alloc_field(H, H->TB));
  chk(alloc_field(H, H->acc));
  if (st == NLSE2SHOC_OK && H->pitch != H->nx && !H->loop_member) {
    chk(alloc_field(H, H->psiw));
    if (st == NLSE2SHOC_OK && dev_malloc(H, &H->Lw, size_t(H->local_elems) * H->S) != cudaSuccess)
      chk(fail(NLSE2SHOC_ENOMEM, "staging allocation failed"));
  }
  if (st == NLSE2SHOC_OK && H->sharded) chk(alloc_arena(H));  // halos of all four field roles
  if (st == NLSE2SHOC_OK) {
    chk(encode_maps(H, H->TA));
    chk(encode_maps(H, H->TB));
    chk(encode_maps(H, H->acc));
    if (H->psiw.ptr) chk(encode_maps(H, H->psiw));
  }
  if (st == NLSE2SHOC_OK && pv.kind == NLSE2SHOC_V_HARMONIC) {
    std::vector<unsigned char> host;
    if (dtype == NLSE2SHOC_C64) build_tables<float>(H, host);
    else build_tables<double>(H, host);
    if (dev_malloc(H, &H->vtab, host.size()) != cudaSuccess) chk(fail(NLSE2SHOC_ENOMEM, "table allocation failed"));
    else if (cudaMemcpy(H->vtab, host.data(), host.size(), cudaMemcpyHostToDevice) != cudaSuccess)
      chk(fail(NLSE2SHOC_ECUDA, "table upload failed"));
    H->bytes += host.size();
  }
  if (st == NLSE2SHOC_OK) {
    if (dev_malloc(H, &H->sched, 2 * sizeof(unsigned)) != cudaSuccess) chk(fail(NLSE2SHOC_ENOMEM, "counter allocation failed"));
    else if (cudaMemset(H->sched, 0, 2 * sizeof(unsigned)) != cudaSuccess) chk(fail(NLSE2SHOC_ECUDA, "counter reset failed"));
  }
  if (st == NLSE2SHOC_OK) {
    H->red_blocks = H->num_sms * 4;
    if (dev_malloc(H, &H->red, sizeof(double) * 3 * H->red_blocks) != cudaSuccess)
      chk(fail(NLSE2SHOC_ENOMEM, "reduction buffer allocation failed"));
  }
#ifdef NLSE_WITH_NCCL
  if (st == NLSE2SHOC_OK && H->sharded && id128) {
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    ncclResult_t r = ncclCommInitRank(&H->comm, nranks, id, rank);
    if (r != ncclSuccess) chk(fail(NLSE2SHOC_ENCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r)));
  }
#endif
  if (st == NLSE2SHOC_OK) {
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) chk(fail(NLSE2SHOC_ECUDA, cudaGetErrorString(e)));
  }
  if (st != NLSE2SHOC_OK) {
    std::string keep = g_last_error;
    nlse2shoc_destroy(H);
    *out = nullptr;
    g_last_error = keep;
  }
  return st;
}

// --------------------------------------------------------------------------- psi views
// The caller's Psi is used in place (zero-copy) when its rows are whole 16-byte vectors;
// otherwise (complex64 with odd N_x in 2D/3D) it is staged through a pitched copy.
static nlse2shoc_status wrap_psi(nlse2shoc_t S, void *base, Field &w) {
  w = Field();
  w.ptr = base;
  w.halo_lo = S->psiw.halo_lo;
  w.halo_hi = S->psiw.halo_hi;
  if (S->dims >= 2) {
    if (S->dtype == NLSE2SHOC_C64) {
      TRY(encode_field_maps<float>(S, w));
    } else {
      TRY(encode_field_maps<double>(S, w));
    }
  }
  return NLSE2SHOC_OK;
}

// Build the view of a call on psi (caller layout).  *work receives the pitched base the
// kernels use (== psi on the zero-copy path).
static nlse2shoc_status make_view(nlse2shoc_t H, void *psi, View &v, void **work, cudaStream_t st,
                                  bool padded = false) {
  void *base = psi;
  if (H->pitch != H->nx && !padded) {
    base = H->psiw.ptr;
    CUDA_TRY(cudaMemcpy2DAsync(base, H->pitch * H->S, psi, H->nx * H->S, H->nx * H->S, H->ny * H->nz,
                               cudaMemcpyDeviceToDevice, st));
  }
  *work = base;
  v.hs.clear();
  v.psis.clear();
  if (H->slabs.empty()) {
    v.hs.push_back(H);
    v.psis.emplace_back();
    if (base == H->psiw.ptr) v.psis.back() = H->psiw;
    else TRY(wrap_psi(H, base, v.psis.back()));
    return NLSE2SHOC_OK;
  }
  for (nlse2shoc_t S : H->slabs) {
    v.hs.push_back(S);
    v.psis.emplace_back();
    TRY(wrap_psi(S, reinterpret_cast<char *>(base) + size_t(S->z0) * S->plane * S->S, v.psis.back()));
  }
  return NLSE2SHOC_OK;
}

static nlse2shoc_status unstage(nlse2shoc_t H, void *dst, const void *work, cudaStream_t st) {
  if (work == dst) return NLSE2SHOC_OK;
  CUDA_TRY(cudaMemcpy2DAsync(dst, H->nx * H->S, work, H->pitch * H->S, H->nx * H->S, H->ny * H->nz,
                             cudaMemcpyDeviceToDevice, st));
  return NLSE2SHOC_OK;
}

static void reset_launches(nlse2shoc_t H) {
  H->launches = 0;
  for (nlse2shoc_t S : H->slabs) S->launches = 0;
}

// Every call runs on the handle's device and restores the caller's current device.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) == cudaSuccess && prev != dev) cudaSetDevice(dev);
    else prev = -1;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

static nlse2shoc_status check_ptr(const void *p, const char *name) {
  if (!p) return fail(NLSE2SHOC_EINVAL, std::string(name) + " is NULL");
  if (reinterpret_cast<uintptr_t>(p) % 16) return fail(NLSE2SHOC_EINVAL, std::string(name) + " is not 16-byte aligned");
  return NLSE2SHOC_OK;
}

// D fields of the two-kernel variants on local planes [-1, nz] (seam planes are recomputed
// from the Psi halo): one (single storage, variant 1) or dims (multi-storage, variant 3).

static nlse2shoc_status ensure_D(nlse2shoc_t H, int nfields) {
  if (H->D.ptr && H->D_fields >= nfields) return NLSE2SHOC_OK;
  const size_t bytes = size_t(D_field_elems(H)) * H->S;
  if (H->D.ptr) {
    CUDA_TRY(dev_free(H, H->D.ptr));
    H->D.ptr = nullptr;
    H->bytes -= bytes * size_t(H->D_fields);
    H->D_fields = 0;
  }
  CUDA_TRY(dev_malloc(H, &H->D.ptr, bytes * size_t(nfields)));
  H->bytes += bytes * size_t(nfields);
  H->D_fields = nfields;
  return NLSE2SHOC_OK;
}

template <typename R> static nlse2shoc_status reduce_N(nlse2shoc_t H, const void *psi, double out[3], cudaStream_t st) {
  if (!H->slabs.empty()) {  // loopback: fold the virtual slabs
    out[0] = INFINITY;
    out[1] = -INFINITY;
    out[2] = 0;
    for (nlse2shoc_t S : H->slabs) {
      double r[3];
      TRY(reduce_N<R>(S, reinterpret_cast<const char *>(psi) + size_t(S->z0) * S->nx * S->ny * S->S, r, st));
      out[0] = std::min(out[0], r[0]);
      out[1] = std::max(out[1], r[1]);
      out[2] += r[2];
    }
    return NLSE2SHOC_OK;
  }
  StageParams<R> P;
  fill_params<R>(H, P);
  P.pitch = H->nx;  // caller layout
  const int64_t total = H->nx * H->ny * H->nz;
  const int blocks = int(std::min<int64_t>(H->red_blocks, (total + 255) / 256));
  reduce_N_kernel<R><<<blocks, 256, 0, st>>>(reinterpret_cast<const cplx<R> *>(psi), P, H->red);
  CUDA_TRY(cudaGetLastError());
  std::vector<double> part(3 * blocks);
  CUDA_TRY(cudaMemcpyAsync(part.data(), H->red, sizeof(double) * 3 * blocks, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  out[0] = INFINITY;
  out[1] = -INFINITY;
  out[2] = 0;
  for (int b = 0; b < blocks; ++b) {
    out[0] = std::min(out[0], part[3 * b]);
    out[1] = std::max(out[1], part[3 * b + 1]);
    out[2] += part[3 * b + 2];
  }
#ifdef NLSE_WITH_NCCL
  if (H->sharded && H->nranks > 1 && H->comm) {
    double *d = H->red;  // reuse: [-min, max, bad]
    double v[3] = {-out[0], out[1], out[2]};
    CUDA_TRY(cudaMemcpyAsync(d, v, sizeof(v), cudaMemcpyHostToDevice, st));
    NCCL_TRY(ncclAllReduce(d, d, 2, ncclFloat64, ncclMax, H->comm, st));
    NCCL_TRY(ncclAllReduce(d + 2, d + 2, 1, ncclFloat64, ncclSum, H->comm, st));
    CUDA_TRY(cudaMemcpyAsync(v, d, sizeof(v), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    out[0] = -v[0];
    out[1] = v[1];
    out[2] = v[2];
  }
#endif
  return NLSE2SHOC_OK;
}

// ===================================================================================== ABI
extern "C" {

nlse2shoc_status nlse2shoc_split(int64_t n_slow, int nranks, int rank, int64_t *z0, int64_t *nz) {
  if (!z0 || !nz || nranks < 1 || rank < 0 || rank >= nranks || n_slow < 1) return fail(NLSE2SHOC_EINVAL, "bad split");
  const int64_t base = n_slow / nranks, rem = n_slow % nranks;
  *nz = base + (rank < rem ? 1 : 0);
  *z0 = int64_t(rank) * base + std::min<int64_t>(rank, rem);
  return NLSE2SHOC_OK;
}

nlse2shoc_status nlse2shoc_create(nlse2shoc_t *out, int dims, const int64_t N[3], const double h[3], double a, double s,
                                  const nlse2shoc_potential *V, nlse2shoc_bc bc, nlse2shoc_dtype dtype) {
  return create_impl(out, dims, N, h, a, s, V, bc, dtype, 0, 1, nullptr);
}

nlse2shoc_status nlse2shoc_get_unique_id(void *id128) {
  if (!id128) return fail(NLSE2SHOC_EINVAL, "id128 is NULL");
#ifdef NLSE_WITH_NCCL
  ncclUniqueId id;
  NCCL_TRY(ncclGetUniqueId(&id));
  static_assert(sizeof(id) == 128, "nccl unique id size");
  std::memcpy(id128, &id, sizeof(id));
  return NLSE2SHOC_OK;
#else
  return fail(NLSE2SHOC_EUNSUPPORTED, "built without NCCL");
#endif
}

nlse2shoc_status nlse2shoc_create_sharded(nlse2shoc_t *out, int dims, const int64_t N[3], const double h[3], double a,
                                          double s, const nlse2shoc_potential *V, nlse2shoc_bc bc,
                                          nlse2shoc_dtype dtype, const void *id128, int rank, int nranks) {
  if (!id128) return fail(NLSE2SHOC_EINVAL, "id128 is NULL");
  return create_impl(out, dims, N, h, a, s, V, bc, dtype, rank, nranks, id128);
}

nlse2shoc_status nlse2shoc_create_loopback(nlse2shoc_t *out, int dims, const int64_t N[3], const double h[3],
                                           double a, double s, const nlse2shoc_potential *V, nlse2shoc_bc bc,
                                           nlse2shoc_dtype dtype, int nslabs) {
  if (nslabs < 1) return fail(NLSE2SHOC_EINVAL, "nslabs must be >= 1");
  return create_impl(out, dims, N, h, a, s, V, bc, dtype, 0, 1, nullptr, -nslabs);
}

nlse2shoc_status nlse2shoc_local_extent(nlse2shoc_t H, int64_t *z0, int64_t *nz) {
  if (!H || !z0 || !nz) return fail(NLSE2SHOC_EINVAL, "NULL argument");
  *z0 = H->dims >= 2 ? H->z0 : 0;
  *nz = H->dims >= 2 ? H->nz : H->N[0];
  return NLSE2SHOC_OK;
}

size_t nlse2shoc_workspace_bytes(nlse2shoc_t H) {
  if (!H) return 0;
  size_t b = H->bytes;
  for (nlse2shoc_t S : H->slabs) b += S->bytes;
  return b;
}

nlse2shoc_status nlse2shoc_set_variant(nlse2shoc_t H, int variant) {
  if (!H) return fail(NLSE2SHOC_EINVAL, "NULL handle");
  DeviceGuard dg(H->device);
  if (variant < 0 || variant > 7)
    return fail(NLSE2SHOC_EINVAL, "variant must be 0 (fused default), 1 (two-kernel), 2 (fused, 16-transfer "
                                  "accumulator), 3 (two-kernel, multi-storage), 4 (stage pairs), 5 (fused, "
                                  "write-light), 6 (fused, reconstructed accumulator) or 7 (fused, carried sum)");
  if (variant == 4 && (H->dims < 2 || !H->slabs.empty() || H->sharded))
    return fail(NLSE2SHOC_EUNSUPPORTED, "the stage-pair variant needs a single-slab 2D/3D handle");
  if ((variant == 1 || variant == 3) && H->scheme != NLSE2SHOC_SCHEME_2SHOC)
    return fail(NLSE2SHOC_EUNSUPPORTED, "the two-kernel variants are 2SHOC forms");
  for (nlse2shoc_t S : H->slabs) TRY(nlse2shoc_set_variant(S, variant));
  if ((variant == 1 || variant == 3) && H->slabs.empty()) TRY(ensure_D(H, variant == 3 ? H->dims : 1));
  H->variant = variant;
  ++H->gen;
  return NLSE2SHOC_OK;
}

nlse2shoc_status nlse2shoc_set_option(nlse2shoc_t H, int option, int64_t value) {
  if (!H) return fail(NLSE2SHOC_EINVAL, "NULL handle");
  if (value < 0 || value > (int64_t(1) << 30)) return fail(NLSE2SHOC_EINVAL, "option value out of range");
  const int v = int(value);
  switch (option) {
    case NLSE2SHOC_OPT_CUDA_GRAPH: H->opt_graph = v != 0; break;
    case NLSE2SHOC_OPT_OVERLAP: H->opt_overlap = v != 0; break;
    case NLSE2SHOC_OPT_RESIDENT_1D: H->opt_resident = v != 0; break;
    case NLSE2SHOC_OPT_REVERSE_ORDER: H->opt_reverse = v != 0; break;
    case NLSE2SHOC_OPT_LEAN_STEPS: H->opt_lean = v & 3; break;
    case NLSE2SHOC_OPT_ZCHUNKS: H->opt_zchunks = v; break;
    case NLSE2SHOC_OPT_TILE_SCHEDULE: H->opt_sched = v >= 2 ? -1 : v; break;
    case NLSE2SHOC_OPT_FUSED_EXCHANGE: H->opt_fused = v != 0; break;
    case NLSE2SHOC_OPT_TAIL_CHUNKS: H->opt_tail = v != 0; break;
    case NLSE2SHOC_OPT_CHECK_EVERY: H->opt_check_every = v; break;
    default: return fail(NLSE2SHOC_EINVAL, "unknown option");
  }
  ++H->gen;
  for (nlse2shoc_t S : H->slabs) TRY(nlse2shoc_set_option(S, option, value));
  return NLSE2SHOC_OK;
}

nlse2shoc_status nlse2shoc_ipc_handle(nlse2shoc_t H, void *handle64) {
  if (!H || !handle64) return fail(NLSE2SHOC_EINVAL, "NULL argument");
  if (!H->arena || H->slabs.size() || H->loop_member) return fail(NLSE2SHOC_EINVAL, "not a sharded (NCCL) handle");
  DeviceGuard dg(H->device);
  cudaIpcMemHandle_t h;
  static_assert(sizeof(h) == 64, "CUDA IPC handle size");
  CUDA_TRY(cudaIpcGetMemHandle(&h, H->arena));
  std::memcpy(handle64, &h, sizeof(h));
  return NLSE2SHOC_OK;
}

nlse2shoc_status nlse2shoc_connect_peers(nlse2shoc_t H, const void *lower64, const void *upper64) {
  if (!H) return fail(NLSE2SHOC_EINVAL, "NULL handle");
  if (!H->arena || H->slabs.size() || H->loop_member) return fail(NLSE2SHOC_EINVAL, "not a sharded (NCCL) handle");
  if ((lower64 != nullptr) != (H->rank > 0) || (upper64 != nullptr) != (H->rank < H->nranks - 1))
    return fail(NLSE2SHOC_EINVAL, "give exactly the neighbours this rank has (lower iff rank > 0, upper iff rank < nranks-1)");
  if (H->peers) return fail(NLSE2SHOC_EINVAL, "peers already connected");
  DeviceGuard dg(H->device);
  char *base[2] = {nullptr, nullptr};
  const void *hs[2] = {lower64, upper64};
  for (int i = 0; i < 2; ++i) {
    if (!hs[i]) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, hs[i], sizeof(h));
    void *p = nullptr;
    CUDA_TRY(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    base[i] = reinterpret_cast<char *>(p);
    (i ? H->ipc_hi : H->ipc_lo) = p;
  }
  // every rank's arena has the same layout (same plane size): role r's low halo at 2r, high at
  // 2r+1 halo blocks, counters after the 8 blocks
  for (int r = 0; r < 4; ++r) {
    H->peer_lo[r] = base[0] ? base[0] + size_t(2 * r + 1) * H->halo_bytes : nullptr;
    H->peer_hi[r] = base[1] ? base[1] + size_t(2 * r) * H->halo_bytes : nullptr;
  }
  H->peer_sig_lo = base[0] ? reinterpret_cast<unsigned long long *>(base[0] + 8 * H->halo_bytes) + 1 : nullptr;
  H->peer_sig_hi = base[1] ? reinterpret_cast<unsigned long long *>(base[1] + 8 * H->halo_bytes) : nullptr;
  H->peers = true;
  ++H->gen;
  return NLSE2SHOC_OK;
}

nlse2shoc_status nlse2shoc_set_scheme(nlse2shoc_t H, int scheme) {
  if (!H) return fail(NLSE2SHOC_EINVAL, "NULL handle");
  if (scheme != NLSE2SHOC_SCHEME_2SHOC && scheme != NLSE2SHOC_SCHEME_CD)
    return fail(NLSE2SHOC_EINVAL, "scheme must be 0 (2SHOC) or 1 (CD)");
  if (scheme == NLSE2SHOC_SCHEME_CD && (H->variant == 1 || H->variant == 3))
    return fail(NLSE2SHOC_EUNSUPPORTED, "the two-kernel variants are 2SHOC forms");
  for (nlse2shoc_t S : H->slabs) TRY(nlse2shoc_set_scheme(S, scheme));
  H->scheme = scheme;
  ++H->gen;
  return NLSE2SHOC_OK;
}

nlse2shoc_status nlse2shoc_laplacian(nlse2shoc_t H, const void *psi, void *L, void *stream) {
  NvtxRange nvtx_r("nlse2shoc_laplacian");
  if (!H) return fail(NLSE2SHOC_EINVAL, "NULL handle");
  DeviceGuard dg(H->device);
  TRY(check_ptr(psi, "psi"));
  TRY(check_ptr(L, "L"));
  if (psi == L) return fail(NLSE2SHOC_EINVAL, "psi and L must be distinct");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  reset_launches(H);
  View v;
  void *work = nullptr;
  TRY(make_view(H, const_cast<void *>(psi), v, &work, st));
  // output: the caller's L directly, or the pitched staging buffer
  void *dst = H->pitch == H->nx ? L : H->Lw;
  TRY(exchange(v, 5, st));
  for (size_t i = 0; i < v.hs.size(); ++i) {
    nlse2shoc_t S = v.hs[i];
    // loopback slabs write their part of the full L; a real shard owns the whole local L
    void *Li = H->slabs.empty() ? dst : reinterpret_cast<char *>(dst) + size_t(S->z0) * S->plane * S->S;
    TRY(stage(S, v.psis[i], 5, 0.0, Li, st));
  }
  return unstage(H, L, dst, st);
}

static nlse2shoc_status rk4_entry(nlse2shoc_t H, void *psi, double dt, int64_t nsteps, void *stream, bool padded) {
  NvtxRange nvtx_r("nlse2shoc_rk4");
  if (!H) return fail(NLSE2SHOC_EINVAL, "NULL handle");
  DeviceGuard dg(H->device);
  TRY(check_ptr(psi, "psi"));
  if (padded && (reinterpret_cast<uintptr_t>(psi) & 15)) return fail(NLSE2SHOC_EINVAL, "padded psi must be 16-byte aligned");
  if (!finite_pos(dt)) return fail(NLSE2SHOC_EINVAL, "dt must be finite and > 0");
  if (nsteps < 0) return fail(NLSE2SHOC_EINVAL, "nsteps must be >= 0");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  reset_launches(H);
  if (nsteps == 0) return NLSE2SHOC_OK;
  if (H->opt_check_every > 0) {
    // failure detection (option CHECK_EVERY): chunks of n steps, each followed by a scan of Psi
    if (padded && H->pitch != H->nx) return fail(NLSE2SHOC_EUNSUPPORTED, "CHECK_EVERY scans the dense layout");
    int64_t launches = 0;
    for (int64_t done = 0; done < nsteps;) {
      const int64_t n = std::min<int64_t>(H->opt_check_every, nsteps - done);
      View v;
      void *work = nullptr;
      TRY(make_view(H, psi, v, &work, st, padded));
      TRY(run_rk4(v, dt, n, st));
      TRY(unstage(H, psi, work, st));
      launches += nlse2shoc_last_launch_count(H);
      done += n;
      double r[3];
      if (H->dtype == NLSE2SHOC_C64) TRY(reduce_N<float>(H, psi, r, st));
      else TRY(reduce_N<double>(H, psi, r, st));
      if (r[2] > 0)
        return fail(NLSE2SHOC_ENONFINITE, std::to_string(int64_t(r[2])) + " non-finite values after step " +
                                              std::to_string(done) + " of " + std::to_string(nsteps));
      reset_launches(H);
    }
    H->launches = launches;
    return NLSE2SHOC_OK;
  }
  View v;
  void *work = nullptr;
  TRY(make_view(H, psi, v, &work, st, padded));
  TRY(run_rk4(v, dt, nsteps, st));
  return unstage(H, psi, work, st);
}

nlse2shoc_status nlse2shoc_rk4(nlse2shoc_t H, void *psi, double dt, int64_t nsteps, void *stream) {
  return rk4_entry(H, psi, dt, nsteps, stream, false);
}

nlse2shoc_status nlse2shoc_rk4_padded(nlse2shoc_t H, void *psi, double dt, int64_t nsteps, void *stream) {
  return rk4_entry(H, psi, dt, nsteps, stream, true);
}

nlse2shoc_status nlse2shoc_padded_layout(nlse2shoc_t H, int64_t pitch[3], int64_t offset[3]) {
  if (!H || !pitch || !offset) return fail(NLSE2SHOC_EINVAL, "NULL argument");
  pitch[0] = H->pitch;        // elements per x-row
  pitch[1] = H->plane;        // elements per plane (pitch * N_y; 2D: per row)
  pitch[2] = H->local_elems;  // elements of the local field
  offset[0] = offset[1] = offset[2] = 0;  // no ghost layers in memory: ghosts are formed on chip
  return NLSE2SHOC_OK;
}

size_t nlse2shoc_stage_workspace_bytes(nlse2shoc_t H) {
  if (!H) return 0;
  const size_t f = ((size_t(H->local_elems) * H->S + 255) / 256) * 256;
  return 3 * f;
}

nlse2shoc_status nlse2shoc_set_workspace(nlse2shoc_t H, void *dev, size_t bytes) {
  if (!H) return fail(NLSE2SHOC_EINVAL, "NULL handle");
  DeviceGuard dg(H->device);
  if (!H->slabs.empty() || H->loop_member)
    return fail(NLSE2SHOC_EUNSUPPORTED, "set_workspace: loopback handles own their slabs' workspaces");
  if (!dev || (reinterpret_cast<uintptr_t>(dev) & 255)) return fail(NLSE2SHOC_EINVAL, "workspace must be a 256-byte aligned device pointer");
  if (bytes < nlse2shoc_stage_workspace_bytes(H)) return fail(NLSE2SHOC_EINVAL, "workspace smaller than nlse2shoc_stage_workspace_bytes");
  cudaPointerAttributes pa;
  if (cudaPointerGetAttributes(&pa, dev) != cudaSuccess || pa.type != cudaMemoryTypeDevice || pa.device != H->device) {
    cudaGetLastError();
    return fail(NLSE2SHOC_EINVAL, "workspace is not device memory of the handle's device");
  }
  CUDA_TRY(cudaDeviceSynchronize());  // nothing in flight may still use the old fields
  graph_drop(H);
  const size_t f = nlse2shoc_stage_workspace_bytes(H) / 3, own = size_t(H->local_elems) * H->S;
  // release the handle's own fields first, so that an error below never leaves a field the
  // handle would free pointing into the caller's memory
  if (!H->ws_external)
    for (Field *fl : {&H->TA, &H->TB, &H->acc})
      if (fl->ptr) {
        void *p = fl->ptr;
        fl->ptr = nullptr;
        H->bytes -= own;
        CUDA_TRY(dev_free(H, p));
      }
  H->ws_external = true;
  ++H->gen;
  int i = 0;
  for (Field *fl : {&H->TA, &H->TB, &H->acc}) {
    fl->ptr = reinterpret_cast<char *>(dev) + size_t(i++) * f;
    TRY(encode_maps(H, *fl));
  }
  return NLSE2SHOC_OK;
}

nlse2shoc_status nlse2shoc_stability_bound(nlse2shoc_t H, const void *psi, double *kmax, void *stream) {
  NvtxRange nvtx_r("nlse2shoc_stability_bound");
  if (!H || !kmax) return fail(NLSE2SHOC_EINVAL, "NULL argument");
  DeviceGuard dg(H->device);
  TRY(check_ptr(psi, "psi"));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  double r[3];
  if (H->dtype == NLSE2SHOC_C64) TRY(reduce_N<float>(H, psi, r, st));
  else TRY(reduce_N<double>(H, psi, r, st));
  // `kdfull`: k < sqrt(8) / max(||B||, max_{i,g} |L_i - g|) h^2/a with B = 0 and
  // G (Table 2) spanning [-4d/12, 64d/12] (Gershgorin endpoints of -h^2 Lap).  Written for a
  // per-axis sum so that anisotropic h reduces to it (reading R17): with H = sum_d 1/h_d^2 the
  // spectrum of (a Lap + N) lies in [Nmin - (64/12) a H, Nmax + (4/12) a H].
  // CD (reading R29): -h^2 delta^2 has Gershgorin interval [0, 4] per axis.
  double Hs = 0.0;
  for (int d = 0; d < H->dims; ++d) Hs += 1.0 / (H->h[d] * H->h[d]);
  const bool cd = H->scheme == NLSE2SHOC_SCHEME_CD;
  const double m1 = std::fabs((cd ? 4.0 : 64.0 / 12.0) * H->a * Hs - r[0]);
  const double m2 = std::fabs(r[1] + (cd ? 0.0 : 4.0 / 12.0) * H->a * Hs);
  *kmax = std::sqrt(8.0) / std::max(m1, m2);
  if (r[2] > 0) return fail(NLSE2SHOC_ENONFINITE, "psi contains non-finite values");
  return NLSE2SHOC_OK;
}

nlse2shoc_status nlse2shoc_check_finite(nlse2shoc_t H, const void *psi, void *stream) {
  if (!H) return fail(NLSE2SHOC_EINVAL, "NULL handle");
  DeviceGuard dg(H->device);
  TRY(check_ptr(psi, "psi"));
  double r[3];
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (H->dtype == NLSE2SHOC_C64) TRY(reduce_N<float>(H, psi, r, st));
  else TRY(reduce_N<double>(H, psi, r, st));
  if (r[2] > 0) return fail(NLSE2SHOC_ENONFINITE, std::to_string(int64_t(r[2])) + " non-finite values");
  return NLSE2SHOC_OK;
}

int64_t nlse2shoc_exchange_timeouts(nlse2shoc_t H) {
  if (!H) return -1;
  DeviceGuard dg(H->device);
  if (cudaDeviceSynchronize() != cudaSuccess) return -2;
  int64_t n = 0;
  std::vector<nlse2shoc_t> hs = H->slabs;
  if (hs.empty()) hs.push_back(H);
  for (nlse2shoc_t S : hs) {
    if (!S->cnt) continue;
    unsigned long long v = 0;
    if (cudaMemcpy(&v, S->cnt + 4, sizeof(v), cudaMemcpyDeviceToHost) != cudaSuccess) return -2;
    n += int64_t(v);
  }
  return n;
}

int64_t nlse2shoc_last_launch_count(nlse2shoc_t H) {
  if (!H) return -1;
  int64_t n = H->launches;
  for (nlse2shoc_t S : H->slabs) n += S->launches;
  return n;
}

nlse2shoc_status nlse2shoc_set_allocator(nlse2shoc_alloc_fn alloc, nlse2shoc_free_fn free_fn, void *ctx) {
  if ((alloc == nullptr) != (free_fn == nullptr)) return fail(NLSE2SHOC_EINVAL, "alloc and free must both be set or both NULL");
  g_alloc = alloc;
  g_free = free_fn;
  g_alloc_ctx = ctx;
  return NLSE2SHOC_OK;
}

const char *nlse2shoc_strerror(nlse2shoc_status st) {
  const int i = -int(st);
  if (i < 0 || i > 6) return "unknown status";
  return kErr[i];
}

const char *nlse2shoc_last_error(void) { return g_last_error.c_str(); }

int64_t nlse2shoc_checked_violations(void) {
#ifdef NLSE_CHECKED
  unsigned long long v = 0;
  if (cudaDeviceSynchronize() != cudaSuccess || cudaMemcpyFromSymbol(&v, g_nlse_violations, sizeof(v)) != cudaSuccess)
    return -2;
  return int64_t(v);
#else
  return -1;
#endif
}

const char *nlse2shoc_version(void) {
#ifdef NLSE_CHECKED
#define NLSE_VARIANT_TAG " checked"
#else
#define NLSE_VARIANT_TAG ""
#endif
#ifdef NLSE_WITH_NCCL
  return "nlse2shoc 0.2 sm_100a nccl" NLSE_VARIANT_TAG;
#else
  return "nlse2shoc 0.2 sm_100a" NLSE_VARIANT_TAG;
#endif
}

void nlse2shoc_destroy(nlse2shoc_t H) {
  if (!H) return;
  DeviceGuard dg(H->device);
  cudaDeviceSynchronize();
  for (nlse2shoc_t S : H->slabs) nlse2shoc_destroy(S);
  if (H->Lw) dev_free(H, H->Lw);
  for (Field *f : {&H->TA, &H->TB, &H->acc, &H->psiw, &H->D}) {
    if (H->ws_external && (f == &H->TA || f == &H->TB || f == &H->acc)) continue;  // the caller's memory
    if (f->ptr) dev_free(H, f->ptr);
  }
  if (H->ipc_lo) cudaIpcCloseMemHandle(H->ipc_lo);
  if (H->ipc_hi) cudaIpcCloseMemHandle(H->ipc_hi);
  if (H->arena) cudaFree(H->arena);
  if (H->vtab) dev_free(H, H->vtab);
  if (H->red) dev_free(H, H->red);
  if (H->sched) dev_free(H, H->sched);
  graph_drop(H);
  if (H->ev_edge) cudaEventDestroy(H->ev_edge);
  if (H->ev_recv) cudaEventDestroy(H->ev_recv);
  if (H->comm_st) cudaStreamDestroy(H->comm_st);
  if (H->cap_st) cudaStreamDestroy(H->cap_st);
#ifdef NLSE_WITH_NCCL
  if (H->comm) ncclCommDestroy(H->comm);
#endif
  delete H;
}

}  // extern "C"
