// pf_internal.h -- shared between the host runtime (pf_host.cpp) and the kernels (pf_kernels.cu).
// Not part of the ABI.  See DESIGN.md section 6 for the layout.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

// Device-side bounds checks of the checked build (-DPF_DEVICE_CHECKS, see pf_debug_guards in
// include/pf.h): a failed check prints its location and traps (the launch fails loudly).
#ifdef PF_DEVICE_CHECKS
#include <cstdio>
#define PF_DCHECK(cond)                                                                         \
    do {                                                                                        \
        if (!(cond)) {                                                                          \
            printf("PF_DCHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond, \
                   (int)blockIdx.x, (int)threadIdx.x);                                          \
            __trap();                                                                           \
        }                                                                                       \
    } while (0)
#else
#define PF_DCHECK(cond) \
    do {                \
    } while (0)
#endif

namespace pf {

// Device layout of one state buffer:
//   [member][field = c, phi, rho][row = -2 .. ny_loc+1][x = -gx .. nx+gx-1]
// Row r of a field lives at storage row r + 2 and column x at storage column x + gx, so the
// ghost frame is physically present: gx = 32 bytes / sizeof(real) ghost columns on each side
// hold the periodic copies, two ghost rows below / above hold the y-mirror rows (c, phi), the
// rho reservoir value rho_in (top) or, at a slab-interior face, the neighbouring slab's rows.
// The streaming kernel keeps the frame up to date as it writes; fill_ghosts rebuilds it after
// host writes.  With the frame present, a TMA box needs no wrap or mirror logic.
struct Layout {
    int nx, ny, ny_loc, y0;      // global grid, owned rows, first owned global row
    int members;
    int path;                    // stage kernel: 0 auto (= 3 when eligible), 1 tile, 2 stream, 3 pair
    int gx;                      // ghost columns per side (32 B / element size)
    int pitch;                   // elements per storage row = nx + 2 gx
    int64_t fstride;             // elements per field  = (ny_loc + 4) * pitch
    int64_t mstride;             // elements per member = 3 * fstride
    int r0, r1;                  // row window [r0, r1) a stage launch updates (default [0, ny_loc))
    int g0, g1;                  // rows [g0, g1) inside the window that the launch skips (g0 == g1:
                                 // none; pair kernel only: both 2-row boundary bands of the slab
                                 // overlap schedule in ONE launch)
    int m0;                      // first member of a stage launch (members = its count; default 0)
    __host__ __device__ int64_t at(int r, int x) const { return (int64_t)(r + 2) * pitch + (x + gx); }
    __host__ __device__ int rows() const { return r1 - r0 - (g1 - g0); }   // rows a launch updates
};

// Coefficients of the discrete model, folded on the host once per ctx.
struct Coef {
    double inv_dx2, half_inv_dx2, inv_2dx;
    double kc_dx2, kp_dx2;          // kappa_c/dx^2, kappa_phi/dx^2
    double W_c, W2c, W2p;           // W_c, 2 W_c, 2 W_phi
    double MBb, dMb, MBs, dMs;      // mobilities shared by all members (when mob < 2)
    int mob;                        // 0 shared with M_A = M_B, 1 shared, 2 per member (R-23)
    double inv_sigma;               // 1/sigma_surf
    double Mp_dx2, Dr_dx2;          // M_phi/dx^2, D_rho/dx^2
    double rho_in;
    double dx2;                     // dx^2 (diagnostics)
    double half_kc, half_kp;        // kappa/2 (diagnostics)
    double W_p;                     // W_phi (diagnostics)
    int fe;                         // composition free energy: 0 polynomial (R-2), 1 regular solution (R-28)
    double omega, temp;             // regular-solution Omega, T (R-28)
};

// Streaming-kernel plan of one slab (host-built once per ctx): strip geometry and the 3D TMA
// tensor maps (x, storage row, member*3 + field) of the two state buffers.
struct StreamPlan {
    bool ok = false;
    int kind = 0;                   // 1: stream_kernel (one column per lane), 2: pair_kernel
    int ncw = 0, Wo = 0, strips = 0;
    int box_x = 0;                  // Wo + 2 halo columns (16 B each side)
    CUtensorMap mapU[2], mapUs[2];  // box (box_x, 2 or 4 rows, 3) over U / Us (index: rows == 4)
    // fused-step kernel (kernel_path 4): one pass per midpoint step, u^n in U -> u^{n+1} in Us,
    // then the host swaps U and Us (and these maps)
    bool fused = false;
    bool ws = false;                // kernel_path 5: the warp-specialised step kernel (fmap*, fWo, ...)
    int fncw = 0, fWo = 0, fstrips = 0, fbox = 0;
    CUtensorMap fmapU, fmapUs;      // box (fbox, 1 row, 3) over U / Us
};
// Swap the roles of the two state buffers in a plan (after a fused step).
void swap_plan_buffers(StreamPlan &P);

// Per-member record of the `vel` device array: v_x, v_y, M_B^bulk, M_A^bulk - M_B^bulk, M_B^surf,
// M_A^surf - M_B^surf (storage precision; R-10, R-15, R-21, R-6, R-23).
constexpr int kMembStride = 6;

// Number of values in a per-member diagnostics record (internal).
// [0] sum c, [1] sum phi, [2] sum rho, [3] E_h, [4] cells with any non-finite field,
// [5] non-finite c, [6] non-finite phi, [7] non-finite rho.
constexpr int kDiag = 8;

// Build the streaming plan (tensor maps) for buffers U, Us of layout L; plan.ok = false when
// the grid is not eligible or the tile path is forced (then the tile kernel is used).
cudaError_t make_stream_plan(int precision, const Layout &L, void *U, void *Us, StreamPlan &plan);
// stage: out = base + coef * R(in).  stage 1: in = U, base = U, out = Us; stage 2: in = Us,
// base = U, out = U (each cell reads its own base value before writing it).
// vel: the per-member record array (kMembStride values per member, pf_cell.cuh).
cudaError_t launch_stage(int precision, const Layout &L, const StreamPlan &plan, const Coef &K, int stage,
                         const void *in, const void *base, void *out, const void *vel, double coef,
                         cudaStream_t s);
// Fused step: out (the other buffer) = u^{n+1} of the state in the buffer P.fmapU describes.
cudaError_t launch_fused(int precision, const Layout &L, const StreamPlan &P, const Coef &K, void *out, const void *vel,
                         double dt, cudaStream_t s);
// Small-grid path: nsteps midpoint steps of every member in one cooperative launch (U holds the
// state before and after; owned cells only, the ghost frame is left stale).
// flags: one unsigned per tile (zeroed once; nullptr = a grid barrier per step), epoch: the steps
// counted on them by earlier launches of this ctx.
cudaError_t launch_persistent(int precision, const Layout &L, const Coef &K, void *U, void *Us, const void *vel,
                              double dt, int64_t nsteps, unsigned *flags, uint32_t epoch, cudaStream_t s);
// Small-grid band path (pf_band.cu): every member is one thread-block cluster of <= 16 blocks,
// each block a band of >= 2 full-width rows held in shared memory for a whole launch; halo rows are
// pushed into the neighbours' shared memory (DSMEM) between two cluster barriers per stage.
struct BandPlan {
    bool ok = false;
    int bands_per_member = 0, blocks = 0, hmax = 0;
    size_t smem = 0;            // dynamic shared memory per block
};
bool make_band_plan(int precision, const Layout &L, BandPlan &B);
// nsteps midpoint steps of every member (U holds the state before and after; owned cells only).
cudaError_t launch_band(int precision, const Layout &L, const BandPlan &B, const Coef &K, void *U, const void *vel,
                        double dt, int64_t nsteps, cudaStream_t s);

// Rebuild the ghost frame of a buffer from its owned cells (periodic columns; mirror rows and
// the rho reservoir at global y boundaries).  Slab-interior ghost rows are left to the exchange.
cudaError_t launch_fill_ghosts(int precision, const Layout &L, double rho_in, void *state, cudaStream_t s);
constexpr int kFillLaunches = 2;
// diag: per-member kDiag doubles into out[members * kDiag]; `partials` scratch of
// members * diag_blocks() * kDiag doubles.  The energy's top y-face of the last owned row is
// included only when the next global row exists (uses the ghost row in slab mode).
int diag_blocks(const Layout &L);
cudaError_t launch_diag(int precision, const Layout &L, const Coef &K, const void *state,
                        double *partials, double *out, cudaStream_t s);
// Stochastic inflow (R-27): the step's truncated-Gaussian reservoir rows of rho in U and Us for
// members [L.m0, L.m0 + L.members) (global ids gmember0 + m); no-op unless this is the top slab.
cudaError_t launch_inflow(int precision, const Layout &L, double rho_in, double sigma, uint64_t seed,
                          int64_t gmember0, int64_t step, void *U, void *Us, cudaStream_t s);
// Composite snapshot field (c where phi > 1/2, else 0) of every member of a slab, fp64, into
// dst[m * dst_mstride + (row0 + r) * nx + x].
cudaError_t launch_composite(int precision, const Layout &L, const void *state, double *dst, int64_t dst_mstride,
                             int row0, cudaStream_t s);
// field <-> contiguous fp64 [members][ny_loc][nx].
cudaError_t launch_pack_f64(int precision, const Layout &L, int field, int member0, int nmem,
                            const void *state, double *dst, cudaStream_t s);
cudaError_t launch_unpack_f64(int precision, const Layout &L, int field, int member0, int nmem,
                              const double *src, void *state, cudaStream_t s);
// B11 halo push (pf_halo.cu; halo_transport = 1): the two boundary rows of every (member, field)
// of `src` stored straight into the neighbours' ghost rows, then one system-scope increment of
// the receiver's arrival counter per block and direction (halo_push_blocks(...) per exchange).
struct HaloPush {
    const char *src;      // this slab's state buffer written by the stage
    char *dst[2];         // [0] the slab below's same buffer, [1] the slab above's (nullptr: none)
    unsigned *flag[2];    // [0] the slab below's "from above" counter, [1] the slab above's "from below"
    int64_t rowb;         // bytes per storage row (pitch * element size)
    int64_t fstride_b;    // bytes per field (members are 3 fields apart)
    int rows;             // owned rows per slab (the same on every slab)
    int nchunks;          // members * 3
};
int halo_push_blocks(int members, int64_t rowb);
cudaError_t launch_halo_push(const HaloPush &h, cudaStream_t s);

// Number of kernel launches made by one launch_stage / launch_diag call.
constexpr int kStageLaunches = 1;
constexpr int kDiagLaunches = 2;

}  // namespace pf
