/*
 * pf.h -- C ABI of libpf, the B200-native PVD phase-field DNS time step.
 *
 * The library advances the coupled (c, phi, rho) phase-field model of physical vapour
 * deposition of arXiv 2312.05410 (section 4.1) with second-order
 * central differences and the explicit midpoint method (section 4.2 "Dataset":
 * "second-order-central-difference stencils for all spatial derivatives and an explicit
 * midpoint method for time integration").  The discrete model, readings R-1..R-20 and the
 * data layout are in DESIGN.md sections 2, 3 and 6.
 *
 * Conventions (all calls):
 *  - Every call returns a pf_status; no C++ exception crosses this ABI.  On failure
 *    pf_last_error(ctx) (or pf_last_error(NULL) for pf_create*) holds a message valid
 *    until the next call on that ctx / thread.
 *  - Host buffers are owned by the caller, row-major, index (m*ny_local + j)*nx + i,
 *    j = 0 the bottom (substrate) row, unpadded, local rows only in slab mode.
 *    NULL means "skip this field".  Pinned host memory is used as is (faster copies).
 *  - The ctx owns all device memory, streams, CUDA graphs and the NCCL communicator
 *    and releases them in pf_free.  Calls on one ctx must be serialised (SPEC S:270
 *    "one writer"); distinct ctxs are independent.
 *  - Torch (or any other caller) only supplies the process group used to broadcast the
 *    NCCL unique id; no compute happens outside this library.
 */
#ifndef PF_H
#define PF_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PF_ABI_VERSION 7u

typedef struct pf_ctx pf_ctx; /* opaque */

typedef enum {
    PF_OK = 0,
    PF_ERR_ARG = 1,          /* invalid argument / parameter                         */
    PF_ERR_UNSTABLE_DT = 2,  /* dt violates the stability bound R-18 */
    PF_ERR_NOMEM = 3,        /* device or host allocation failed                     */
    PF_ERR_CUDA = 4,         /* CUDA runtime error (message names it)                */
    PF_ERR_NCCL = 5,         /* NCCL error (slab mode)                               */
    PF_ERR_BLOWUP = 6,       /* non-finite value detected ("blow-up")     */
    PF_ERR_STATE = 7,        /* call not allowed in the current state                */
    PF_ERR_ABI = 8           /* pf_params.abi_version != PF_ABI_VERSION              */
} pf_status;

typedef enum { PF_F64 = 0, PF_F32 = 1 } pf_precision;

/* Initial-condition recipes (reading R-14 of BASELINE.json configs[0..4]). */
typedef enum {
    PF_IC_FILM = 0,            /* phi = [j < ic_height] + U(+-noise_phi); c = ic_c0 + noise  */
    PF_IC_ROUGH_SUBSTRATE = 1, /* phi = 1/2(1 - tanh((j - H_i)/delta)), H_i = H + amp sin(2 pi i/lambda) */
    PF_IC_COLUMNS = 2,         /* tanh film at ic_height; ic_ncols columns, c = ic_c_lo / ic_c_hi */
    PF_IC_NONE = 3             /* all fields zero; caller uses pf_set_fields             */
} pf_ic;

/* Every physical / numerical parameter of the model (SPEC S:158-161 SolverConfig, the symbols
 * of P:302-343).  Readings: R-2..R-4 free energy, R-6 mobility, R-7 M_phi, R-9 vapour,
 * R-10 velocity, R-13 values, R-15 per-member rates. */
typedef struct {
    uint32_t abi_version;            /* must be PF_ABI_VERSION                               */
    int32_t nx, ny;                  /* GLOBAL grid; x periodic, y no-flux; nx, ny >= 8 */
    int32_t n_members;               /* members held by this ctx (ensemble, grid.z)          */
    int32_t member_offset;           /* global id of local member 0: keys seeds and rates    */
    int32_t precision;               /* pf_precision: storage and arithmetic type            */
    double dx, dt;                   /* grid spacing, time step                              */
    double kappa_c, kappa_phi;       /* gradient-energy coefficients (R-2)                   */
    double W_c, W_phi;               /* well heights (R-2)                                   */
    double M_A_bulk, M_B_bulk, M_A_surf, M_B_surf, sigma_surf; /* P:312-324 (R-6)            */
    double M_phi;                    /* interface mobility (R-7)                             */
    double D_rho, rho_in;            /* vapour diffusivity and top reservoir density (R-9, R-12) */
    double v0, theta_deg;            /* deposition speed and angle: v = v0_m (cos, -sin) (R-10) */
    double rate_lo, rate_hi;         /* v0_m = v0 (lo + (hi-lo) U(seed, 8m+3, 0)) (R-15)     */
    double theta_span;               /* theta_m = theta_deg + theta_span U(seed, 8m+4, 0) degrees
                                        (0: every member at theta_deg; R-21, P:352 sweeps 50..90) */
    double mob_lo, mob_hi;           /* species mobility sweep (R-23, "species mobilities"):
                                        member m scales M_A (bulk, surf) by a = lo + (hi-lo) U(seed,
                                        8m+5, 0) and M_B by b (stream 8m+6); 1, 1 = no sweep     */
    double noise_rho;                /* stochastic inflow (R-27): > 0 replaces the top
                                        reservoir rho_in by a per-step, per-column draw from
                                        N(rho_in, noise_rho^2) truncated to [0, 2 rho_in]; 0 = off */
    int32_t fe_model;                /* composition free energy: 0 = W_c c^2 (1-c)^2 phi (R-2);
                                        1 = regular solution [omega c(1-c) + temp_rs (c ln c +
                                        (1-c) ln(1-c))] phi (R-28, north_star wording)           */
    double omega, temp_rs;           /* regular-solution interaction and temperature (R-28)   */
    int32_t ic;                      /* pf_ic                                                */
    int32_t ic_ncols;                /* PF_IC_COLUMNS: number of columns                    */
    double ic_height, ic_amp, ic_wavelength;
    double ic_c0, ic_c_lo, ic_c_hi;
    double noise_c, noise_phi;       /* noise amplitudes (uniform +-a, or Gaussian std for c) */
    int32_t noise_c_gaussian;        /* 1: c = c0 + noise_c N(0,1) (Box-Muller, R-16)        */
    int32_t check_every;             /* blow-up / diagnostics check period in steps (>= 1)   */
    uint64_t seed;                   /* counter-RNG seed (R-16)                              */
    int32_t device;                  /* CUDA device ordinal                                  */
    int32_t graph_steps;             /* steps per captured CUDA graph (0 = no graphs)        */
    int32_t kernel_path;             /* stage kernel: 0 auto (single-domain grids of <= 2^19 cells in
                                        all: the band small-grid kernel where its bands fit, else
                                        the persistent small-grid kernel; larger grids: the pair
                                        kernel when nx % 4 == 0 and nx >= 16, else the tile
                                        kernel), 1 tile, 3 pair streaming, 5 warp-specialised step
                                        (experimental), 6 band small-grid (state resident in shared
                                        memory, neighbour flags; PF_ERR_ARG where it does not fit),
                                        7 persistent small-grid (grid barriers); 2 and 4 (the
                                        round-1 one-column and fused-step kernels) are retired and
                                        rejected with PF_ERR_ARG                                */
    int32_t overlap_halo;            /* slab modes: 1 = update the 2-row boundary bands first and
                                        overlap the halo exchange with the interior update
                                        (needs >= 8 rows per slab), 0 = exchange after the stage */
    int32_t halo_transport;          /* slab modes, how the 2 boundary rows reach the neighbours
                                        after every stage:
                                        0 = NCCL send/recv (pf_create_slab) or device-to-device
                                            copies (pf_create_loopback);
                                        1 = peer stores: one kernel per slab and stage writes the
                                            rows straight into the neighbours' ghost rows (CUDA-IPC
                                            mappings over NVLink in pf_create_slab, exchanged once
                                            over the NCCL communicator at create; device pointers in
                                            loopback) and increments an arrival counter in the
                                            receiver's memory, which the receiver's stream awaits
                                            with cuStreamWaitValue32.  Results are bitwise those of
                                            transport 0.  Disables CUDA graphs for the ctx.
                                        2 = NCCL send / receive to SELF (pf_create with n_slabs > 1
                                            only; pf_create_slab rejects it): the slabs of a one-GPU
                                            context exchange through a 1-rank communicator, each
                                            transfer a ncclSend matched by a ncclRecv in one group,
                                            issued by the code transport 0 runs across ranks, and
                                            the diagnostics through ncclAllGather -- the one-GPU
                                            stand-in that executes the NCCL path.  Bitwise those of
                                            transport 0; no CUDA graphs.                           */
} pf_params;

/* Fill *out with the preset of BASELINE.json configs[cfg-1] (cfg = 1..5; R-13, R-14).
 * Errors: PF_ERR_ARG for an unknown cfg or out == NULL. */
pf_status pf_default_params(int32_t cfg, pf_params *out);

/* sizeof(pf_params) as compiled into the library (lets bindings verify their struct mirror). */
uint32_t pf_params_size(void);

/* Host-only: the seeded initial fields of GLOBAL member `member` (row a0 of SURVEY 8(a);
 * recipes R-14, RNG R-16) for global rows [y0, y0+rows), written row-major (row, x) as fp64
 * into caller-owned buffers of rows*nx doubles.  This is exactly what pf_create uploads
 * (before rounding to fp32 for PF_F32).  Needs no GPU.  Errors: PF_ERR_ARG. */
pf_status pf_initial_fields(const pf_params *p, int64_t member, int32_t y0, int32_t rows,
                            double *c, double *phi, double *rho);

/* Host-only: velocity (v_x, v_y) = v0_m (cos theta, -sin theta) of GLOBAL member `member`
 * (R-10, R-15) and the stability limit of R-18 for p.  Need no GPU.  Errors: PF_ERR_ARG. */
pf_status pf_member_velocity(const pf_params *p, int64_t member, double *v_x, double *v_y);
/* Host-only: composition mobilities of GLOBAL member `member` (R-6, R-23):
 * out = {M_A^bulk, M_B^bulk, M_A^surf, M_B^surf}.  Errors: PF_ERR_ARG. */
pf_status pf_member_mobility(const pf_params *p, int64_t member, double out[4]);
/* Host-only: the stochastic reservoir row (R-27) of GLOBAL member `member` for global step
 * `step` (the draw both midpoint stages of that step see): out[nx]; rho_in when noise_rho == 0.
 * Errors: PF_ERR_ARG. */
pf_status pf_inflow_row(const pf_params *p, int64_t member, int64_t step, double *out);
pf_status pf_dt_limit(const pf_params *p, double *dt_max);

/* Create a single-GPU context holding p->n_members independent members of the full
 * nx x ny grid, generate their seeded initial conditions on the host (a0, R-14..R-16) and
 * upload them.  Validates p (nx, ny >= 8, dx, dt > 0, ...) and the stability bound R-18.
 * Errors: PF_ERR_ABI, PF_ERR_ARG, PF_ERR_UNSTABLE_DT, PF_ERR_NOMEM, PF_ERR_CUDA.
 * On error *out is NULL and pf_last_error(NULL) explains. */
pf_status pf_create(const pf_params *p, pf_ctx **out);

/* 128-byte NCCL unique id for pf_create_slab (call on rank 0, broadcast the bytes).
 * Errors: PF_ERR_NCCL. */
pf_status pf_nccl_unique_id(uint8_t out[128]);

/* Create rank `rank` of an nranks-way y-slab decomposition of the global grid:
 * rank r owns global rows [r ny/nranks, (r+1) ny/nranks) (ny % nranks == 0, ny/nranks >= 2);
 * the 2-row halo of c, phi, rho is exchanged with ranks r-1 / r+1 after every midpoint stage
 * over NCCL (P:348 stages; BASELINE configs[3] "2-cell halo exchanged per stage").
 * `uid` comes from pf_nccl_unique_id on rank 0.  Errors: as pf_create plus PF_ERR_NCCL. */
pf_status pf_create_slab(const pf_params *p, int32_t rank, int32_t nranks,
                         const uint8_t uid[128], pf_ctx **out);

/* Host-only: the y-slab decomposition of rank `rank` of `nranks` over ny global rows
 * (the plan pf_create_slab / pf_create_loopback use):
 *   out[0] = y0, first owned global row        out[1] = ny_local = ny / nranks
 *   out[2] = rank below (r-1), -1 at the substrate   out[3] = rank above (r+1), -1 at the top
 *   out[4] = first local row sent down (0)     out[5] = first local row sent up (ny_local-2)
 *   out[6] = first ghost row filled from below (-2)  out[7] = first ghost row filled from above
 *            (ny_local).
 * Every message carries 2 full padded rows (ghost columns included) of c, phi and rho of every
 * member.  Errors: PF_ERR_ARG (ny % nranks != 0, ny / nranks < 2, rank out of range). */
pf_status pf_halo_plan(int32_t ny, int32_t nranks, int32_t rank, int32_t out[8]);

/* Single-process multi-slab context ("loopback"): nslabs y-slabs of every member on ONE
 * device, with the halo exchange done by device-to-device copies.  Same arithmetic and
 * exchange schedule as pf_create_slab, used to test the decomposition without NCCL.
 * Host buffers for get/set still cover the FULL grid.  Errors: as pf_create. */
pf_status pf_create_loopback(const pf_params *p, int32_t nslabs, pf_ctx **out);

/* Advance every member by n >= 0 explicit midpoint steps: per step, stage 1
 * u* = u^n + dt/2 R(u^n) and stage 2 u^{n+1} = u^n + dt R(u*), each one fused kernel pass.
 * Every check_every steps and at the end, the non-finite count is checked:
 * PF_ERR_BLOWUP names the field and step window; the state is left as computed and
 * further pf_step calls fail with PF_ERR_STATE until pf_set_fields.  Synchronous.
 * Errors: PF_ERR_ARG (n < 0), PF_ERR_STATE, PF_ERR_BLOWUP, PF_ERR_CUDA, PF_ERR_NCCL. */
pf_status pf_step(pf_ctx *ctx, int64_t n);

/* End-to-end run from host memory (the call bench.py's e2e times): equivalent to
 * pf_set_fields(ctx, -1, c_in, phi_in, rho_in); pf_step(ctx, n); pf_get_fields(ctx, -1, c_out,
 * phi_out, rho_out) -- bitwise the same result -- but pipelined over `chunks` groups of members
 * (members are independent): the upload of chunk k+1 and the download of chunk k-1 overlap the
 * steps of chunk k on separate streams (pinned host buffers make the copies asynchronous).  With
 * chunks >= 3 the first and last chunks hold ~1/8 of the members each (short exposed copies).
 * Buffers: all members stacked, as for member = -1; NULL inputs keep the device state, NULL
 * outputs are skipped.  The blow-up check runs once per chunk at the end of the call (the reported
 * step window is the whole call).  Single-GPU fp64 contexts with chunks >= 2 pipeline; other
 * contexts run the three calls in sequence.  Synchronous.
 * Errors: as pf_set_fields, pf_step, pf_get_fields. */
pf_status pf_run_host(pf_ctx *ctx, int64_t n, const double *c_in, const double *phi_in, const double *rho_in,
                      double *c_out, double *phi_out, double *rho_out, int32_t chunks);

/* Trajectory / dataset driver ("50 time snapshots equally spaced
 * taken over the entire course of the simulation", dataset shape members x (50, 256, 256)):
 * n_snapshots snapshots of the composite composition field, snapshot 0 = the current state and
 * snapshot s after s * steps_between further steps (pf_step, with its blow-up checks).  The
 * composite field is c where phi > 1/2 and 0 in the vapour.  out (caller-owned,
 * fp64): [member][snapshot][ny_local][nx]; times (optional, NULL to skip): t of each snapshot.
 * Each snapshot is copied to the host on a separate stream while the next steps run (pinned
 * host memory makes the copies asynchronous).  Synchronous.
 * Errors: PF_ERR_ARG, PF_ERR_NOMEM, PF_ERR_STATE, and pf_step's errors. */
pf_status pf_trajectory(pf_ctx *ctx, int32_t n_snapshots, int64_t steps_between, double *out, double *times);

/* The same trajectory streamed to a FILE (SURVEY 8(f) NEXT-1 "adds I/O and a trajectory file";
 * P:354-355 dataset of trajectories x (50, 256, 256)): snapshot s of every member is copied to a
 * pinned host buffer while the next steps run and a writer thread appends it to `path`.
 * Layout (little-endian):
 *   header, 96 bytes: char magic[8] = "PFTRAJ01"; uint32 header_bytes (= 96 + 64 members),
 *     uint32 version = 1; int32 nx, ny_global, y0, ny_rows, members, member_offset, n_snapshots,
 *     dtype (0 = float64, 1 = float32); int64 steps_between, step0 (pf_info steps before
 *     snapshot 0); float64 dt, t0, dx, rho_in;
 *   members records of 8 float64: global member id, v_x, v_y, M_A^bulk, M_B^bulk, M_A^surf,
 *     M_B^surf, 0 (R-10, R-15, R-21, R-23);
 *   data: [n_snapshots][members][ny_rows][nx] of dtype, the composite composition c[phi > 1/2]
 *     (identical to pf_trajectory's values; float32 = rounded);
 *   footer: float64 t of every snapshot.
 * Synchronous.  Errors: PF_ERR_ARG (bad arguments, I/O failure: message names the path),
 * PF_ERR_NOMEM, PF_ERR_STATE and pf_step's errors (the file is then incomplete). */
pf_status pf_trajectory_file(pf_ctx *ctx, const char *path, int32_t n_snapshots, int64_t steps_between,
                             int32_t dtype);

/* Copy member `member` (0..n_members-1, or -1 = all members, stacked) to host buffers of
 * ny_local*nx doubles each (times n_members for -1).  fp32 fields are widened to double.
 * Errors: PF_ERR_ARG, PF_ERR_CUDA. */
pf_status pf_get_fields(pf_ctx *ctx, int32_t member, double *c, double *phi, double *rho);

/* Inverse of pf_get_fields: overwrite the member's state from host buffers (fp32 fields are
 * rounded to nearest).  Clears a blow-up state.  Fields passed as NULL are left unchanged.
 * In slab mode the halo rows are refreshed by an exchange before returning (collective:
 * every rank must call it).  Errors: PF_ERR_ARG, PF_ERR_CUDA, PF_ERR_NCCL. */
pf_status pf_set_fields(pf_ctx *ctx, int32_t member, const double *c, const double *phi,
                        const double *rho);

/* Diagnostics of member `member` (north_star "Reductions"), accumulated in fp64 in a fixed
 * order (deterministic for a fixed launch shape and nranks):
 *   out[0] = dx^2 sum c (mass of c), out[1] = dx^2 sum phi, out[2] = dx^2 sum rho,
 *   out[3] = E_h, out[4] = number of cells with a non-finite field.
 * Slab mode: global values (per-rank partials all-gathered and summed in rank order;
 * collective).  Errors: PF_ERR_ARG, PF_ERR_CUDA, PF_ERR_NCCL. */
pf_status pf_diagnostics(pf_ctx *ctx, int32_t member, double out[5]);

/* Steps taken, simulated time, first global row and number of rows held by this ctx.
 * Any pointer may be NULL.  Errors: PF_ERR_ARG. */
pf_status pf_info(pf_ctx *ctx, int64_t *steps, double *t, int32_t *y0, int32_t *ny_local);

/* Grid and ensemble held by this ctx: global nx, ny and the number of members (host buffers of
 * pf_get_fields / pf_trajectory are sized from these).  Any pointer may be NULL.  Errors: PF_ERR_ARG. */
pf_status pf_shape(pf_ctx *ctx, int32_t *nx, int32_t *ny, int32_t *members);

/* Override the step counter and time (used when resuming from saved fields).
 * Errors: PF_ERR_ARG. */
pf_status pf_set_time(pf_ctx *ctx, int64_t steps, double t);

/* Kernel launches issued by this ctx since creation (stage + diagnostics + exchange kernels);
 * used by the benchmark to report its launch count.  Errors: PF_ERR_ARG. */
pf_status pf_launch_count(pf_ctx *ctx, int64_t *launches);

/* Stage-kernel profiling (bench.py's roofline): while enabled (enable != 0), every stage
 * launch of pf_step is bracketed by CUDA events on the ctx's stream and CUDA graphs are not
 * used; enabling resets the record.  pf_profile_read returns out[0] = total ms of stage-1
 * launches, out[1] = their count, out[2] = total ms of stage-2 launches, out[3] = count,
 * out[4] = total ms of diagnostics launches (pairs), out[5] = their count.
 * Errors: PF_ERR_ARG, PF_ERR_CUDA. */
pf_status pf_profile(pf_ctx *ctx, int32_t enable);
pf_status pf_profile_read(pf_ctx *ctx, double out[6]);

/* The cudaStream_t (as void*) every kernel and copy of this ctx is issued on, so a caller can
 * time the ctx's work with CUDA events recorded on the same stream.  Errors: PF_ERR_ARG. */
pf_status pf_stream(pf_ctx *ctx, void **stream);

/* ---- NEXT-2: microstructure statistics of the paper's evaluation
 * (section 2.3 "spatial autocorrelation S2^(A,A)(r, t)", section 4.5 "Rel. L2";
 * SPEC S:456-526; readings R-24..R-26).  Context-free; run on the current CUDA device; inputs and
 * outputs are host buffers of fp64.  Errors are status codes only (PF_ERR_ARG, PF_ERR_NOMEM,
 * PF_ERR_CUDA; no message).
 *   Indicator I = [comp >= threshold] of a composite field (vapour c = 0, R-24).
 *   S2(r) = (1/N) sum_x I(x) I(x + r), periodic, N = nx ny cells, computed as
 *   IFFT(|FFT(I)|^2) / N^2 with cuFFT; maps are centred: s2[b][ny/2 + dy][nx/2 + dx].
 *   Radial profile: mean of the centred map over bins round(|r|), bins 0 .. pf_s2_nbins - 1 (R-25). */
int32_t pf_s2_nbins(int32_t nx, int32_t ny);
/* comp: [batch][ny][nx] composite fields; s2 (or NULL): [batch][ny][nx]; radial (or NULL):
 * [batch][nbins] with nbins == pf_s2_nbins(nx, ny). */
pf_status pf_s2(const double *comp, int32_t nx, int32_t ny, int32_t batch, double threshold, double *s2,
                double *radial, int32_t nbins);
/* out[b] = ||S2(true_b) - S2(pred_b)||_2 / ||S2(true_b)||_2 for batch pairs of fields. */
pf_status pf_s2_rel_l2(const double *comp_true, const double *comp_pred, int32_t nx, int32_t ny, int32_t batch,
                       double threshold, double *out);

/* Last error message of ctx (ctx == NULL: the calling thread's last create error). */
const char *pf_last_error(const pf_ctx *ctx);

/* Debug: the guard zones around every state buffer of a checked build (-DPF_GUARD_BYTES=N, built by
 * __graft_entry__.build() as paper_2312_05410_b200/_variants/libpf_checked.so, with device-side
 * bounds checks that trap).  *guard_bytes = N (0 in the production build, where *corrupted = 0);
 * *corrupted = guard bytes that no longer hold their fill pattern, i.e. evidence of an out-of-bounds
 * global write.  Synchronises the ctx stream.  Errors: PF_ERR_ARG (NULL), PF_ERR_CUDA.  (Stands in
 * for compute-sanitizer memcheck, which the GPU pool does not allow.) */
pf_status pf_debug_guards(pf_ctx *ctx, int64_t *guard_bytes, int64_t *corrupted);

/* Diagnostics of a PF_TRACE build (PF_NVCC_EXTRA=-DPF_TRACE=1 python -m
 * paper_2312_05410_b200.build --out=...; tools/trace_stage1.py); zeros
 * in a normal build.  They read the fp64 stage-1 pair kernel's timeline of its last launch:
 *   pf_debug_trace:       out[5][512][2] int64 -- per warp (compute warps 0-3, producer = 4) and box:
 *                         full-barrier wait start / end (producer: empty wait start / TMA issue), ns of
 *                         the global timer, block 37 only;
 *   pf_debug_block_spans: out[1024][3] int64 -- per block: start (after the dependent-launch wait),
 *                         SM id, end of compute warp 0.
 * out: host memory the caller owns.  Returns a cudaError_t value (0 = success). */
int pf_debug_trace(long long *out);
int pf_debug_block_spans(long long *out);
/* Diagnostic of a PF_TRACE build: the small-grid step kernel's (kernel_path 7) phase timeline of
 * its last launch, out[160 blocks][64 steps][8] int64 global-timer ns: [0] tile start, [1] u^n
 * loaded, [2] stage-1 mu/M, [3] u*, [4] stage-2 mu/M, [5] tile written, [6] grid barrier passed.
 * Zeros in a normal build.  out: host memory the caller owns.  Returns a cudaError_t value. */
int pf_debug_step_trace(long long *out);
/* Diagnostic of a PF_TRACE build: the band kernel's (kernel_path 6) phase timeline of its last
 * launch, out[16 blocks][128 stages][4] int64 clock64 cycles of thread 0 of the first cluster's
 * blocks: [0] after phase A (mu/M), [1] after phase B (update), [2] after the stage's cluster
 * barrier, [3] stage start.  Zeros in a normal build.  Returns a cudaError_t value. */
int pf_debug_band_trace(long long *out);

/* Release everything the ctx owns.  NULL-safe.  Slab mode: collective (NCCL teardown). */
void pf_free(pf_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* PF_H */
