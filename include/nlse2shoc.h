/* nlse2shoc.h — C-ABI of the B200 (sm_100a) RK4 + 2SHOC NLSE library (libnlse2shoc.so).
 *
 * The library integrates the nonlinear Schrodinger equation
 *     i Psi_t + a Lap(Psi) - V(r) Psi + s |Psi|^2 Psi = 0          (PAPER.md `NLSE`)
 * with the method of lines: classic fourth-order Runge-Kutta in time (`RK4`)
 * and the two-step high-order compact (2SHOC) Laplacian in space:
 *     step 1   D_d = delta_d^2 Psi                      (`2shoc1d`, `2d2shocMs1`, `3d2shocMs1`)
 *     step 2   Lap = sum_d 7/6 D_d - (D_d(+e_d) + D_d(-e_d))/12
 *                                                      (`2shoc1d2`, `2d2shocMs2`, `3d2shocMs2`)
 * with the paper's boundary rule for the intermediate D (DESIGN.md
 * readings R8/R9) and the Psi_t boundary condition (`dbc_ut`).
 * PAPER.md = /root/reference/PAPER.md (read at build time only; P:n = line n).
 *
 * Conventions shared by every call
 *  - Grid: dims in {1,2,3}; N[3] = point counts along (x, y, z) (unused axes: 1);
 *    coordinate of index i along axis d is xmin[d] + i*h[d]; every index 0 and
 *    N[d]-1 is a boundary point.  N[d] >= 5 on every used axis.
 *  - Field layout: row-major [z][y][x], x fastest, complex interleaved (re, im): the memory
 *    of a contiguous torch.complex64 / complex128 tensor of shape (Nz, Ny, Nx) (dims dropped
 *    from the left for 1D/2D).  Sharded handles: the local z-slab [z0, z0+nz) only.
 *  - Pointers marked "device" are CUDA device pointers on the handle's device, 16-byte
 *    aligned, caller-owned (the library never frees them).
 *  - Every call returns nlse2shoc_status (0 = OK, < 0 = error); nothing aborts.  Detail of
 *    the last error on the calling thread: nlse2shoc_last_error().
 *  - Work is enqueued on the caller's CUDA stream (cudaStream_t passed as void*; NULL = the
 *    legacy default stream) and the call returns after enqueue, except where noted "syncs".
 *    Asynchronous faults surface at the caller's next synchronisation.
 *  - A handle is not thread-safe; distinct handles are independent.
 */
#ifndef NLSE2SHOC_H
#define NLSE2SHOC_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct nlse2shoc_s *nlse2shoc_t;

typedef enum {
  NLSE2SHOC_OK = 0,
  NLSE2SHOC_EINVAL = -1,       /* invalid argument (see each call)                       */
  NLSE2SHOC_ENOMEM = -2,       /* device allocation failed                               */
  NLSE2SHOC_ECUDA = -3,        /* CUDA runtime / driver error                            */
  NLSE2SHOC_ENCCL = -4,        /* NCCL error (sharded handles)                           */
  NLSE2SHOC_ENONFINITE = -5,   /* non-finite value found by nlse2shoc_check_finite       */
  NLSE2SHOC_EUNSUPPORTED = -6  /* option not built (e.g. no NCCL in this build)          */
} nlse2shoc_status;

/* Boundary conditions.
 *  DIRICHLET: Lap_b = lambda_b = -(s|Psi_b|^2 - V_b) Psi_b / a (`dbc_lap`) for step 1,
 *             Psi_t,b = 0 exactly (`dbc_ut`).
 *  LAPZERO:   "Laplacian-zero": lambda_b = 0, Psi_t,b = i (s|Psi_b|^2 - V_b) Psi_b
 *             (reading R9).
 * At a d-face point b (index_d in {0, N_d-1}, all other indices interior) the per-axis
 * intermediate is D_d(b) = lambda_b - sum_{e != d} delta_e^2 Psi_b (reading R8).          */
/*  MSD:       modulus-squared Dirichlet, 1D only (EUNSUPPORTED otherwise):
 *             lambda_b = [Re(D_{b-1}/Psi_{b-1}) + (N_{b-1} - N_b)/a] Psi_b (`msdbc_lap`, reading
 *             R28), Psi_t,b = i Im(Psi_t,b-1 / Psi_b-1) Psi_b (`msdbc_ut`).  The stability bound
 *             omits Table 1's MSD B term.                                                     */
typedef enum { NLSE2SHOC_BC_DIRICHLET = 0, NLSE2SHOC_BC_LAPZERO = 1, NLSE2SHOC_BC_MSD = 2 } nlse2shoc_bc;

typedef enum { NLSE2SHOC_C64 = 0, NLSE2SHOC_C128 = 1 } nlse2shoc_dtype;

typedef enum { NLSE2SHOC_V_NONE = 0, NLSE2SHOC_V_HARMONIC = 1, NLSE2SHOC_V_ARRAY = 2 } nlse2shoc_vkind;

/* Potential V(r) of `NLSE`.
 *  NONE:      V = 0.
 *  HARMONIC:  V = w[0](x-c[0])^2 + w[1](y-c[1])^2 + w[2](z-c[2])^2 (absent axes dropped),
 *             x = xmin[0] + i h[0] etc.; evaluated on the fly from per-axis tables (no HBM
 *             field).
 *  ARRAY:     data = device pointer to N[0]*N[1]*N[2] (sharded: the local slab) real values
 *             of the handle's precision (float for C64, double for C128) in the field layout;
 *             borrowed: the caller keeps it alive and unchanged until destroy.
 * xmin is also used by nothing else (coordinates only enter through V).                   */
typedef struct {
  nlse2shoc_vkind kind;
  double xmin[3];
  double w[3];
  double c[3];
  const void *data;
} nlse2shoc_potential;

/* Create a single-GPU handle on the current CUDA device.  Every later call on the handle runs
 * on that device whatever device is current, and restores the caller's current device.
 *  out   : receives the handle (host pointer).
 *  dims  : 1, 2 or 3.          N : counts (x, y, z), N[d] >= 5 for d < dims, 1 otherwise.
 *  h     : spacing per axis, finite and > 0 (anisotropic allowed; R17).
 *  a     : > 0, finite.  s : finite.  V : NULL means V_NONE.
 *  bc, dtype : see enums.
 * Allocates the workspace (3 fields for the fused RK4: two stage buffers and the RK4
 * accumulator; see nlse2shoc_workspace_bytes).  EINVAL / ENOMEM / ECUDA.              */
nlse2shoc_status nlse2shoc_create(nlse2shoc_t *out, int dims, const int64_t N[3], const double h[3],
                                  double a, double s, const nlse2shoc_potential *V, nlse2shoc_bc bc,
                                  nlse2shoc_dtype dtype);

/* z-slab sharding (3D, and 2D along y) over nranks processes, one GPU each.
 * N is GLOBAL; this rank owns the slowest-axis slab [z0, z0+nz) given by
 * nlse2shoc_local_extent (even split, remainder to the first ranks; nz >= 2).  The
 * caller's Psi / L / V.data are the LOCAL slab.  id128 is the 128-byte NCCL unique id that
 * rank 0 obtained from nlse2shoc_get_unique_id and broadcast (e.g. with torch.distributed).
 * Collective: every rank must call it, and afterwards every rank must make the same
 * sequence of laplacian / rk4 / stability_bound calls with the same dt and nsteps
 * (a mismatch deadlocks inside NCCL; not detected).  EUNSUPPORTED if built without NCCL. */
nlse2shoc_status nlse2shoc_get_unique_id(void *id128);
nlse2shoc_status nlse2shoc_create_sharded(nlse2shoc_t *out, int dims, const int64_t N[3], const double h[3],
                                          double a, double s, const nlse2shoc_potential *V, nlse2shoc_bc bc,
                                          nlse2shoc_dtype dtype, const void *id128, int rank, int nranks);
/* Halo exchange fused into the stage kernels (the
 * compact stencil keeps the exchange to 2 planes per side).  With peers connected, rk4 runs
 * each RK4 stage as one kernel launch per rank that also stores its two edge planes on each
 * side straight into the neighbour's halo buffer (CUDA IPC mapping over NVLink) and raises an
 * arrival counter there with a system-scope atomic; a kernel reading its halo planes first
 * waits on its own counter.  No NCCL call and no separate exchange step remain in the step
 * (one NCCL send/recv of Psi's halos per rk4 call).  Option FUSED_EXCHANGE switches back to
 * the NCCL exchange.  Loopback handles connect their virtual slabs automatically.
 *  ipc_handle:    64-byte CUDA IPC handle of this rank's halo arena (cudaMalloc'd at create).
 *  connect_peers: open the neighbours' handles: lower64 iff rank > 0, upper64 iff
 *                 rank < nranks-1 (EINVAL otherwise, or if already connected).  Each rank
 *                 must connect before its next rk4 call; the binding's Solver.connect_peers()
 *                 gathers the handles with torch.distributed.                              */
nlse2shoc_status nlse2shoc_ipc_handle(nlse2shoc_t, void *handle64);
/* Fused exchange diagnostics: arrival waits that gave up after ~4 s (a neighbour that never
 * arrived: ranks calling differently, or a dead rank) since create, summed over the handle's
 * slabs; the kernel finishes instead of hanging, and the result of that call is invalid.
 * Syncs the device.  -1 for a NULL handle, -2 on a CUDA error.                             */
int64_t nlse2shoc_exchange_timeouts(nlse2shoc_t);
nlse2shoc_status nlse2shoc_connect_peers(nlse2shoc_t, const void *lower64, const void *upper64);

/* Single-GPU emulation of the z-slab sharding (2D/3D): one handle holding nslabs virtual
 * slabs, split exactly like nlse2shoc_split, that exchange their 2-plane halos by
 * device-to-device copies instead of NCCL and run the same kernels as real shards.  The
 * caller's Psi / L are the WHOLE grid.  Results are bitwise identical to a single-slab
 * handle (no reduction in the step; halos are exact copies); used to test the sharded
 * path where only one GPU is available.  EINVAL for dims = 1 or nslabs < 1.            */
nlse2shoc_status nlse2shoc_create_loopback(nlse2shoc_t *out, int dims, const int64_t N[3], const double h[3],
                                           double a, double s, const nlse2shoc_potential *V, nlse2shoc_bc bc,
                                           nlse2shoc_dtype dtype, int nslabs);
/* Slab owned by this handle along the slowest axis (z in 3D, y in 2D, whole grid in 1D). */
nlse2shoc_status nlse2shoc_local_extent(nlse2shoc_t, int64_t *z0, int64_t *nz);
/* Split rule used by create_sharded (pure host function, no handle needed). */
nlse2shoc_status nlse2shoc_split(int64_t n_slow, int nranks, int rank, int64_t *z0, int64_t *nz);

/* Device bytes the handle allocated (workspace + halos + tables). */
size_t nlse2shoc_workspace_bytes(nlse2shoc_t);

/* Caller-owned stage workspace (SURVEY §8(b) "optional: torch-owned").  The three stage
 * fields of the RK4 combine (T_A, T_B, acc) are placed in `dev` (device memory
 * of the handle's device, 256-byte aligned, at least nlse2shoc_stage_workspace_bytes(H) =
 * 3 fields each rounded up to 256 B); the handle frees the ones it allocated at create and
 * never frees `dev`, which the caller keeps alive until destroy or the next set_workspace.
 * Several handles of the same size that never run concurrently may share one workspace.
 * Syncs the device.  EINVAL: NULL / misaligned / too small / not device memory of this
 * device; EUNSUPPORTED for loopback handles (their slabs own their workspaces).          */
size_t nlse2shoc_stage_workspace_bytes(nlse2shoc_t);
nlse2shoc_status nlse2shoc_set_workspace(nlse2shoc_t, void *dev, size_t bytes);

/* The layout the kernels use in place (SURVEY §8(b) "optional zero-copy Psi"): pitch[0] =
 * elements per x-row, pitch[1] = elements per plane (2D: per row), pitch[2] = elements of the
 * local field; offset[] = 0 — there are no ghost layers in memory (ghost values are formed on
 * chip).  pitch[0] equals N_x except for complex64 with odd N_x in 2D/3D, whose
 * rows are padded to a whole 16-byte vector: nlse2shoc_rk4 stages such a dense Psi through a
 * pitched copy (2 field passes per call), and nlse2shoc_rk4_padded takes Psi already in this
 * layout (16-byte aligned; the pad element of each row is ignored and left untouched) and
 * skips the copy.  For every other handle the two calls are the same.                    */
nlse2shoc_status nlse2shoc_padded_layout(nlse2shoc_t, int64_t pitch[3], int64_t offset[3]);
nlse2shoc_status nlse2shoc_rk4_padded(nlse2shoc_t, void *psi_padded, double dt, int64_t nsteps, void *stream);

/* 0 = FUSED (default): one kernel per RK4 stage computes the whole 2SHOC Laplacian (both
 *     steps, D never stored), the RHS and the RK4 stage combine, 12 field transfers per
 *     point-step, in the carried-sum form (= variant 7).
 * 5 = FUSED_WRITE_LIGHT: stages 1-3 store only T_A = Psi + k/2 K1, T_B = Psi + k/2 K2,
 *     T_C = Psi + k K3 (T_C in the accumulator's buffer); stage 4 forms Psi' = Psi +
 *     ((T_A - Psi) + 2 (T_B - Psi) + (T_C - Psi))/3 + k/6 K4 (the accumulator is never
 *     stored: acc = (T_A + 2 T_B)/3 in exact arithmetic).
 * 6 = FUSED_RECON: stage 1 stores only T_A = Psi + k/2 K1, stage 2 forms acc = Psi + (T_A -
 *     Psi)/3 + k/3 K2, stage 3 stores only T_A = Psi + k K3, stage 4 forms Psi' = acc +
 *     (T_A - Psi)/3 + k/6 K4.
 * 7 = FUSED_CARRIED (12 transfers per point-step, the fewest with one pass per stage:
 *     every stage reads its stencil input and writes its output, stages 2-3 read Psi, one
 *     carried field is written once and read once): stage 2 also stores Q = 3 acc - Psi =
 *     [2 Psi + (T_A - Psi)] + k K2, stage 3 writes T_C = Psi + k K3 over T_A, and stage 4
 *     forms Psi' = (Q + T_C + k/2 K4)/3 from T_C and Q alone, with the sum carried exactly and
 *     a correctly rounded division by 3 (one rounding of size ulp(Psi) per step; stationary
 *     fields and Dirichlet boundary values are reproduced to the bit).
 * 1 = TWO_KERNEL: the paper's single-storage scheme (`2d2shocs1/2`, `3d2shocs`):
 *     kernel A stores D = sum_d delta_d^2 Psi (D_b = lambda_b), kernel B applies step 2 +
 *     RHS + combine.  One more field of workspace (allocated on first use).
 * 2 = FUSED_ACC16: as 0 but stage 1 stores acc = Psi + k/6 K1 explicitly (16 transfers per
 *     point-step, the SURVEY §8(a) a6 form).
 * 3 = TWO_KERNEL_MS: the paper's multi-storage scheme (`2d2shocMs1/2` P:185-200,
 *     `3d2shocMs1/2` P:262-280, the "2X/3X storage" rows of Tables 4-5): kernel A stores
 *     D_d = delta_d^2 Psi per axis (face rule of DESIGN.md reading R8 at d-faces), kernel B
 *     applies L = sum_d 7/6 D_d - (D_d(+e_d) + D_d(-e_d))/12.  dims more fields of workspace.
 * 4 = STAGE_PAIRS (temporal blocking): one launch runs stages 1+2 and one
 *     runs stages 3+4 over each tile, the first stage of a pair evaluated on the tile grown by
 *     the stencil radius and kept in shared memory: 7 field transfers per point-step plus the
 *     wider halos.  Results are bit-identical to variant 6.  Psi^{n+1} is written to the T_A
 *     workspace on odd steps and copied back once per call.  2D/3D single-slab handles only
 *     (EUNSUPPORTED otherwise).
 * Variants 1 and 3 are 2SHOC forms: EUNSUPPORTED with the CD scheme.
 * EINVAL for other values.                                                             */
nlse2shoc_status nlse2shoc_set_variant(nlse2shoc_t, int variant);

/* Spatial scheme (default 2SHOC).  CD = the paper's second-order comparison scheme RK4+CD
 * (`uttmp`): Lap = sum_d delta_d^2 Psi, same boundary rules (L_b = lambda_b,
 * F_b per the BC), same kernels with the +-2 weights set to zero.  stability_bound then uses
 * the CD Gershgorin interval (reading R29).  EUNSUPPORTED with variant 1 (the
 * two-kernel variant is the paper's 2SHOC storage scheme); EINVAL for other values.     */
typedef enum { NLSE2SHOC_SCHEME_2SHOC = 0, NLSE2SHOC_SCHEME_CD = 1 } nlse2shoc_scheme;
nlse2shoc_status nlse2shoc_set_scheme(nlse2shoc_t, int scheme);

/* Execution-path options of a handle (applied to every later call; a loopback handle passes
 * them to its virtual slabs).  None changes the arithmetic of a point: every option selects
 * between code paths that evaluate the same expressions, so results are bit-identical
 * unless noted.  Defaults in brackets.
 *  CUDA_GRAPH    [1] single-slab rk4 calls of >= 4 steps capture one step's launches in a
 *                    CUDA graph and replay it (fewer launch overheads).
 *  OVERLAP       [1] sharded / loopback 2D-3D fused variants: edge planes first, halo
 *                    exchange on a side stream beside the interior planes.
 *  RESIDENT_1D   [1] small 1D grids (4 fields <= 200 KB) run the whole call in one CTA.
 *  REVERSE_ORDER [1] stages 2 and 4 walk the tiles backwards (L2 reuse).  Changes the
 *                    order of nothing but the tiles: bit-identical.
 *  LEAN_STEPS    [3] branch-free plane steps of the fused 2D/3D kernel: bit 1 = tiles with
 *                    no boundary point and no ghost, bit 2 = 3D tiles touching an x/y face
 *                    (ghost fill + face rule inline).  0 = the general step everywhere.
 *  ZCHUNKS       [0] fused 2D/3D kernels: number of chunks the streamed axis is split into
 *                    (0 = automatic); values that would leave empty chunks are reduced to the
 *                    smallest count with the same chunk length.
 *  TILE_SCHEDULE [2] fused 2D/3D kernels: 0 = static (CTA b takes tiles b, b + G, ...),
 *                    1 = dynamic (tiles claimed in order from a counter in device memory,
 *                    so neighbouring tiles are streamed at nearly the same time whatever
 *                    each CTA's speed, and their halo re-reads hit L2), 2 = automatic =
 *                    dynamic (C4 8.83 -> 8.07 ms/step; C3 c128 2.49 -> 2.38, c64 1.50 ->
 *                    1.28 with the dynamic chunk model).  Dynamic needs the calls on a
 *                    handle to be ordered on one stream at a time (the counter is the
 *                    handle's).
 *  FUSED_EXCHANGE [1] sharded / loopback handles with peers: halo exchange fused into the
 *                    stage kernels (see nlse2shoc_connect_peers); 0 = the edge-first NCCL /
 *                    copy exchange (OVERLAP).
 *  TAIL_CHUNKS  [1] fused 2D/3D kernels with the dynamic schedule: the z-chunk layout may
 *                    end the streamed range on short chunks at both ends, so that the last
 *                    tiles of a traversal (in either direction) are short and the CTAs
 *                    finish together; 0 = equal chunks.  Bit-identical.
 * Single-slab and sharded rk4 calls keep their instantiated CUDA graph and replay it in
 * later calls with the same psi pointer and dt (any set_* call drops it).
 *  CHECK_EVERY   [0] failure detection (an explicit scheme past its
 *                    stability bound blows up): n > 0 makes rk4 scan Psi for NaN / Inf after
 *                    every n steps (each scan syncs the stream; sharded: collective) and
 *                    return ENONFINITE as soon as one is found, nlse2shoc_last_error() naming
 *                    the number of steps taken; Psi then holds the state at that step.  0 = no
 *                    scan, rk4 stays asynchronous.  The arithmetic is unchanged (n steps at a
 *                    time replay the same step graph).  EUNSUPPORTED in nlse2shoc_rk4_padded
 *                    when the pitch differs from N_x (the scan reads the dense layout).
 * EINVAL for an unknown option or a negative value.                                     */
typedef enum {
  NLSE2SHOC_OPT_CUDA_GRAPH = 0,
  NLSE2SHOC_OPT_OVERLAP = 1,
  NLSE2SHOC_OPT_RESIDENT_1D = 2,
  NLSE2SHOC_OPT_REVERSE_ORDER = 3,
  NLSE2SHOC_OPT_LEAN_STEPS = 4,
  NLSE2SHOC_OPT_ZCHUNKS = 5,
  NLSE2SHOC_OPT_TILE_SCHEDULE = 6,
  NLSE2SHOC_OPT_FUSED_EXCHANGE = 7,
  NLSE2SHOC_OPT_TAIL_CHUNKS = 8,
  NLSE2SHOC_OPT_CHECK_EVERY = 9
} nlse2shoc_option;
nlse2shoc_status nlse2shoc_set_option(nlse2shoc_t, int option, int64_t value);

/* L = Lap(psi) by 2SHOC; boundary points get L_b = lambda_b.  psi, L: device,
 * field layout, distinct.  Sharded: halo exchange included (collective).             */
nlse2shoc_status nlse2shoc_laplacian(nlse2shoc_t, const void *psi, void *L, void *stream);

/* nsteps classic RK4 steps of size dt in place on psi (device, field layout).
 * dt finite > 0, nsteps >= 0.  The result is the same polynomial as the paper's listing
 * evaluated with a Psi-space accumulator.               */
nlse2shoc_status nlse2shoc_rk4(nlse2shoc_t, void *psi, double dt, int64_t nsteps, void *stream);

/* kmax of `kdfull` from psi (device): B = 0 (Table 1 Dirichlet; Laplacian-zero
 * by reading R14), G of Table 2 via its closed form g in [-4d/12, 64d/12] (isotropic h);
 * anisotropic h: reading R17.  Sharded: global over all ranks (collective).  Syncs. */
nlse2shoc_status nlse2shoc_stability_bound(nlse2shoc_t, const void *psi, double *kmax, void *stream);

/* Scan psi (device) for NaN/Inf; returns ENONFINITE if any is found.  Syncs. */
nlse2shoc_status nlse2shoc_check_finite(nlse2shoc_t, const void *psi, void *stream);

/* Number of CUDA kernels the last laplacian / rk4 call enqueued (instrumentation). */
int64_t nlse2shoc_last_launch_count(nlse2shoc_t);

/* Device allocator for every buffer the library owns (workspace fields, halos, tables, D).
 * Process-wide; captured by each handle at create and used until its destroy, so a handle
 * always frees with the allocator it allocated with.  alloc(bytes, device, ctx) returns a
 * device pointer aligned to >= 256 B, or NULL (-> ENOMEM); free(ptr, device, ctx) releases it.
 * Both NULL restores cudaMalloc/cudaFree.  The Python binding installs torch's caching
 * allocator here, so all device memory is PyTorch's (north star: "PyTorch used only for
 * device memory, streams and process groups").  NCCL's internal buffers are NCCL's own.
 * EINVAL if exactly one of alloc / free is NULL.                                          */
typedef void *(*nlse2shoc_alloc_fn)(size_t bytes, int device, void *ctx);
typedef void (*nlse2shoc_free_fn)(void *ptr, int device, void *ctx);
nlse2shoc_status nlse2shoc_set_allocator(nlse2shoc_alloc_fn alloc, nlse2shoc_free_fn free_fn, void *ctx);

const char *nlse2shoc_strerror(nlse2shoc_status);
const char *nlse2shoc_last_error(void);
/* Checked build (libnlse2shoc_checked.so, -DNLSE_CHECKED): number of global stores of the
 * 2D/3D stage kernels that fell outside their buffer (skipped, not performed) since load;
 * syncs the device.  -1 in normal builds (no checks compiled), -2 on a CUDA error.      */
int64_t nlse2shoc_checked_violations(void);

/* Library version string, e.g. "nlse2shoc 0.2 sm_100a nccl" (" checked" appended). */
const char *nlse2shoc_version(void);
void nlse2shoc_destroy(nlse2shoc_t);

#ifdef __cplusplus
}
#endif
#endif
