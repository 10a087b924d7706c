// pf_internal.h -- shared between the host runtime (pf_host.cpp) and the kernels (pf_kernels.cu).
// Not part of the ABI.  See DESIGN.md section 6 for the layout.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace pf {

// Device layout of one state buffer:
//   [member][field = c, phi, rho][row = -2 .. ny_loc+1][x = 0 .. nx-1]
// Row r of a field lives at storage row r + 2: two ghost rows below and above the owned rows
// carry the neighbouring slab's rows in slab mode.  x has no ghost columns (periodic wrap is
// done by index in the kernels).
struct Layout {
    int nx, ny, ny_loc, y0;      // global grid, owned rows, first owned global row
    int members;
    int path;                    // stage kernel: 0 auto (streaming when eligible), 1 tile, 2 streaming
    int64_t fstride;             // elements per field  = (ny_loc + 4) * nx
    int64_t mstride;             // elements per member = 3 * fstride
};

// Coefficients of the discrete model, folded on the host once per ctx.
struct Coef {
    double inv_dx2, half_inv_dx2, inv_2dx;
    double kc_dx2, kp_dx2;          // kappa_c/dx^2, kappa_phi/dx^2
    double W_c, W2c, W2p;           // W_c, 2 W_c, 2 W_phi
    double MBb, dMb, MBs, dMs;      // M_B_bulk, M_A_bulk - M_B_bulk, M_B_surf, M_A_surf - M_B_surf
    double inv_sigma;               // 1/sigma_surf
    double Mp_dx2, Dr_dx2;          // M_phi/dx^2, D_rho/dx^2
    double rho_in;
    double dx2;                     // dx^2 (diagnostics)
    double half_kc, half_kp;        // kappa/2 (diagnostics)
    double W_p;                     // W_phi (diagnostics)
};

// Number of values in a per-member diagnostics record (internal).
// [0] sum c, [1] sum phi, [2] sum rho, [3] E_h, [4] cells with any non-finite field,
// [5] non-finite c, [6] non-finite phi, [7] non-finite rho.
constexpr int kDiag = 8;

// Launchers (pf_kernels.cu).  All return the cudaError_t of the launch.
// stage: out = base + coef * R(in)   (base may alias out: each cell reads its own base value
// before writing it; `in` must not alias `out`).
cudaError_t launch_stage(int precision, const Layout &L, const Coef &K, const void *in,
                         const void *base, void *out, const void *vel, double coef,
                         cudaStream_t s);
// diag: per-member kDiag doubles into out[members * kDiag]; `partials` scratch of
// members * diag_blocks() * kDiag doubles.  The energy's top y-face of the last owned row is
// included only when the next global row exists (uses the ghost row in slab mode).
int diag_blocks(const Layout &L);
cudaError_t launch_diag(int precision, const Layout &L, const Coef &K, const void *state,
                        double *partials, double *out, cudaStream_t s);
// field <-> contiguous fp64 [members][ny_loc][nx] (for fp32 storage; fp64 uses memcpy).
cudaError_t launch_pack_f64(int precision, const Layout &L, int field, int member0, int nmem,
                            const void *state, double *dst, cudaStream_t s);
cudaError_t launch_unpack_f64(int precision, const Layout &L, int field, int member0, int nmem,
                              const double *src, void *state, cudaStream_t s);
// Number of kernel launches made by one launch_stage / launch_diag call.
constexpr int kStageLaunches = 1;
constexpr int kDiagLaunches = 2;

}  // namespace pf
