// pf_cell.cuh -- per-cell arithmetic of the discrete model, shared by every stage
// kernel (tile kernel and streaming kernel).  Every operation is an explicit round-to-nearest
// intrinsic (add / mul / fma), so no compiler contraction choice can differ between call sites:
// each cell's value is the same bit pattern on every code path, tiling, x-translation and slab
// decomposition (reading R-19).
#pragma once
#include <cstdint>

namespace pf {

template <typename real>
struct KC {                    // coefficients folded into the compute precision
    real half_inv_dx2, inv_2dx, kc_dx2, kp_dx2, W_c, W2c, W2p;
    real MBb, dMb, MBs, dMs, inv_sigma, Mp_dx2, Dr_dx2, rho_in, coef;
};

__device__ __forceinline__ double add_(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double mul_(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double fma_(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ double exp_(double x) { return exp(x); }
__device__ __forceinline__ float add_(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float sub_(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float mul_(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fma_(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ float exp_(float x) { return expf(x); }

// Row a2 (constitutive pass): mu_c, mu_phi and M_c of one cell from its value and its four
// neighbours (l = i-1, r = i+1, d = j-1, u = j+1).  P:310-331; readings R-1..R-7.
// The neighbour sums are ((l + r) + (d + u)): symmetric in (d, u), so a mirrored ghost row
// (u[-1] = u[0], u[-2] = u[1]) yields bit-identical mu / M to the cell it mirrors, and the
// boundary-face fluxes vanish exactly.
template <typename real>
__device__ __forceinline__ void constitutive(const KC<real> &k, real c, real p, real cl, real cr,
                                             real cd, real cu, real pl, real pr, real pd, real pu,
                                             real &mu_c, real &mu_p, real &M) {
    const real one = real(1), two = real(2), m2 = real(-2), m4 = real(-4);
    const real lc = fma_(m4, c, add_(add_(cl, cr), add_(cd, cu)));   // dx^2 L(c)
    const real lp = fma_(m4, p, add_(add_(pl, pr), add_(pd, pu)));   // dx^2 L(phi)
    const real c1 = mul_(c, sub_(one, c));                            // c(1-c)
    const real t2c = fma_(m2, c, one);                                // 1-2c
    // mu_c = 2 W_c c(1-c)(1-2c) phi - kappa_c L(c)                              (R-2, R-4)
    mu_c = fma_(-k.kc_dx2, lc, mul_(mul_(mul_(k.W2c, c1), t2c), p));
    // mu_phi = W_c c^2(1-c)^2 + 2 W_phi phi(1-phi)(1-2phi) - kappa_phi L(phi)    (R-3)
    const real p1 = mul_(p, sub_(one, p));                            // phi(1-phi)
    const real t2p = fma_(m2, p, one);                                // 1-2phi
    mu_p = fma_(-k.kp_dx2, lp, fma_(k.W_c, mul_(c1, c1), mul_(mul_(k.W2p, p1), t2p)));
    // M_c = M_bulk + e (M_surf_mix - M_bulk)                         (R-5, R-6)
    const real ch = fmin(fmax(c, real(0)), one);                     // clamp(c, 0, 1)
    const real h = mul_(mul_(ch, ch), fma_(m2, ch, real(3)));         // smoothstep h(c)
    const real pp = mul_(mul_(p, p), fma_(m2, p, real(3)));           // 1/4 (2 - phit)(1 + phit)^2
    const real q = mul_(fma_(two, p, -one), k.inv_sigma);             // phit / sigma_surf
    const real e = exp_(-mul_(q, q));
    const real mb = mul_(pp, fma_(h, k.dMb, k.MBb));
    const real ms = fma_(h, k.dMs, k.MBs);
    M = fma_(e, sub_(ms, mb), mb);
}

// Rows a3-a5: right-hand sides and the Euler-form stage update of one cell.
//   R_c   = sum of face fluxes (M_a + M_b)/2 (mu_b - mu_a)/dx^2   (conservative)
//   S     = rho (v_x G_x phi + v_y G_y phi)                        (R-10)
//   R_phi = M_phi L(mu_phi) + S                                    (R-7)
//   R_rho = D_rho L(rho) - v . G(rho) - S                          (R-9)
//   out   = base + coef R                                          (R-11)
// Arguments: centre (0) and neighbours (l, r, d, u) of M, mu_c, mu_phi, rho; phi neighbours.
// A face flux is the same expression seen from both of its cells, so the divergence telescopes.
template <typename real>
__device__ __forceinline__ void cell_update(const KC<real> &k, real vx, real vy,
                                            real M0, real Ml, real Mr, real Md, real Mu,
                                            real m0, real ml, real mr, real md, real mu,
                                            real q0, real ql, real qr, real qd, real qu,
                                            real pl, real pr, real pd, real pu,
                                            real r0, real rl, real rr, real rd, real ru,
                                            real bc, real bp, real br,
                                            real &oc, real &op, real &orr) {
    const real m4 = real(-4);
    const real fe = mul_(add_(M0, Mr), sub_(mr, m0));
    const real fw = mul_(add_(Ml, M0), sub_(m0, ml));
    const real fn = mul_(add_(M0, Mu), sub_(mu, m0));
    const real fs = mul_(add_(Md, M0), sub_(m0, md));
    const real Rc = mul_(add_(sub_(fe, fw), sub_(fn, fs)), k.half_inv_dx2);
    const real lq = fma_(m4, q0, add_(add_(ql, qr), add_(qd, qu)));          // dx^2 L(mu_phi)
    const real S = mul_(r0, mul_(fma_(vx, sub_(pr, pl), mul_(vy, sub_(pu, pd))), k.inv_2dx));
    const real Rp = fma_(k.Mp_dx2, lq, S);
    const real lr = fma_(m4, r0, add_(add_(rl, rr), add_(rd, ru)));          // dx^2 L(rho)
    const real adv = mul_(fma_(vx, sub_(rr, rl), mul_(vy, sub_(ru, rd))), k.inv_2dx);
    const real Rr = sub_(fma_(k.Dr_dx2, lr, -adv), S);
    oc = fma_(k.coef, Rc, bc);
    op = fma_(k.coef, Rp, bp);
    orr = fma_(k.coef, Rr, br);
}

}  // namespace pf
