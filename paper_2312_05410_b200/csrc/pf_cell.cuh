// pf_cell.cuh -- per-cell arithmetic of the discrete model, shared by every stage
// kernel (tile kernel and streaming kernel) so that each cell's value is produced by the same
// expression sequence on every code path (bitwise invariance across paths, tilings and slabs).
#pragma once
#include <cstdint>

namespace pf {

template <typename real>
struct KC {                    // coefficients folded into the compute precision
    real half_inv_dx2, inv_2dx, kc_dx2, kp_dx2, W_c, W2c, W2p;
    real MBb, dMb, MBs, dMs, inv_sigma, Mp_dx2, Dr_dx2, rho_in, coef;
};

template <typename real>
__device__ __forceinline__ real dexp(real x);
template <>
__device__ __forceinline__ double dexp<double>(double x) { return exp(x); }
template <>
__device__ __forceinline__ float dexp<float>(float x) { return expf(x); }

// Row a2 (constitutive pass): mu_c, mu_phi and M_c of one cell from its value and its four
// neighbours (l = i-1, r = i+1, d = j-1, u = j+1).  P:310-331; readings R-1..R-7.
// The neighbour sums are ((l + r) + (d + u)): symmetric in (d, u), so a mirrored ghost row
// (u[-1] = u[0], u[-2] = u[1]) yields bit-identical mu / M to the cell it mirrors, and the
// boundary-face fluxes vanish exactly.
template <typename real>
__device__ __forceinline__ void constitutive(const KC<real> &k, real c, real p, real cl, real cr,
                                             real cd, real cu, real pl, real pr, real pd, real pu,
                                             real &mu_c, real &mu_p, real &M) {
    const real lc = ((cl + cr) + (cd + cu)) - real(4) * c;   // dx^2 L(c)
    const real lp = ((pl + pr) + (pd + pu)) - real(4) * p;   // dx^2 L(phi)
    const real omc = real(1) - c;
    const real c1 = c * omc;                                 // c(1-c)
    // mu_c = 2 W_c c(1-c)(1-2c) phi - kappa_c L(c)                              (R-2, R-4)
    mu_c = k.W2c * c1 * (real(1) - real(2) * c) * p - k.kc_dx2 * lc;
    // mu_phi = W_c c^2(1-c)^2 + 2 W_phi phi(1-phi)(1-2phi) - kappa_phi L(phi)    (R-3)
    mu_p = k.W_c * (c1 * c1) + k.W2p * (p * (real(1) - p)) * (real(1) - real(2) * p) - k.kp_dx2 * lp;
    // M_c = M_bulk + e (M_surf_mix - M_bulk)                         (R-5, R-6)
    real ch = c < real(0) ? real(0) : c;
    ch = ch > real(1) ? real(1) : ch;
    const real h = ch * ch * (real(3) - real(2) * ch);        // smoothstep h(c)
    const real pp = p * p * (real(3) - real(2) * p);          // 1/4 (2 - phit)(1 + phit)^2
    const real q = (real(2) * p - real(1)) * k.inv_sigma;      // phit / sigma_surf
    const real e = dexp<real>(-(q * q));
    const real mb = pp * (k.MBb + h * k.dMb);
    const real ms = k.MBs + h * k.dMs;
    M = mb + e * (ms - mb);
}

// Rows a3-a5: right-hand sides and the Euler-form stage update of one cell.
//   R_c   = sum of face fluxes (M_a + M_b)/2 (mu_b - mu_a)/dx^2   (conservative)
//   S     = rho (v_x G_x phi + v_y G_y phi)                        (R-10)
//   R_phi = M_phi L(mu_phi) + S                                    (R-7)
//   R_rho = D_rho L(rho) - v . G(rho) - S                          (R-9)
//   out   = base + coef R                                          (R-11)
// Arguments: centre (0) and neighbours (l, r, d, u) of M, mu_c, mu_phi, rho; phi neighbours.
template <typename real>
__device__ __forceinline__ void cell_update(const KC<real> &k, real vx, real vy,
                                            real M0, real Ml, real Mr, real Md, real Mu,
                                            real m0, real ml, real mr, real md, real mu,
                                            real q0, real ql, real qr, real qd, real qu,
                                            real pl, real pr, real pd, real pu,
                                            real r0, real rl, real rr, real rd, real ru,
                                            real bc, real bp, real br,
                                            real &oc, real &op, real &orr) {
    const real fe = (M0 + Mr) * (mr - m0);
    const real fw = (Ml + M0) * (m0 - ml);
    const real fn = (M0 + Mu) * (mu - m0);
    const real fs = (Md + M0) * (m0 - md);
    const real Rc = ((fe - fw) + (fn - fs)) * k.half_inv_dx2;
    const real lq = ((ql + qr) + (qd + qu)) - real(4) * q0;          // dx^2 L(mu_phi)
    const real S = r0 * ((vx * (pr - pl) + vy * (pu - pd)) * k.inv_2dx);
    const real Rp = k.Mp_dx2 * lq + S;
    const real lr = ((rl + rr) + (rd + ru)) - real(4) * r0;          // dx^2 L(rho)
    const real adv = (vx * (rr - rl) + vy * (ru - rd)) * k.inv_2dx;
    const real Rr = (k.Dr_dx2 * lr - adv) - S;
    oc = bc + k.coef * Rc;
    op = bp + k.coef * Rp;
    orr = br + k.coef * Rr;
}

}  // namespace pf
